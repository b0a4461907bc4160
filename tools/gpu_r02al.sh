timeout 900 python -m pytest -q tests -m gpu -x -k "topk or summary or argmax or report or measure or circuit_io" 2>&1 | tail -3
timeout 300 python tools/e2e_breakdown.py 32 2>&1 | tail -10
