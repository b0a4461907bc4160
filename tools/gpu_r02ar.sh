timeout 600 python -m pytest -q tests -m gpu -x -k "topk or summary or reductions" 2>&1 | tail -2
for n in 12 20; do timeout 100 python tools/summary_timing.py $n 2>&1 | tail -6; done
timeout 300 python bench.py --workload c1 --steps 20 --warmup 3 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('c1', d['ms_per_step'], d['e2e']['ms_per_step'], d['e2e'].get('serial_ms_per_step'))"
