timeout 900 python -m pytest -q tests -m gpu -x -k "topk or summary or reductions or report or circuit_io or sample" 2>&1 | tail -3
timeout 300 python tools/summary_timing.py 32 2>&1 | tail -5
timeout 300 python tools/summary_timing.py 28 2>&1 | tail -5
timeout 300 python tools/e2e_breakdown.py 32 2>&1 | tail -3
