timeout 300 python tools/e2e_breakdown.py 32 2>&1 | tail -12
timeout 300 python tools/e2e_probe.py 32 2>&1 | tail -16
