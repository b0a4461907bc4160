timeout 900 python -m pytest -q tests -m gpu -x -k "topk or summary or reductions" 2>&1 | tail -3
timeout 300 python tools/summary_timing.py 32 2>&1 | tail -5
