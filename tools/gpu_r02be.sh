timeout 1500 python -m pytest -q tests/test_jit.py tests/test_parity_gpu.py tests/test_baseline_sizes_gpu.py tests/test_edge_gpu.py -m gpu -x -k "not c2_sweep_n28 and not c2_sweep_n24" 2>&1 | tail -2
timeout 600 python bench.py --no-c2 --no-cpu-baseline --steps 3 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('c4', d['ms_per_step'], d['e2e']['ms_per_step'], 'cold', d['e2e']['cold_first_call_ms'])"
timeout 600 python bench.py --workload c3 --steps 5 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('c3', d['ms_per_step'], d['e2e']['ms_per_step'], 'cold', d['e2e']['cold_first_call_ms'])"
