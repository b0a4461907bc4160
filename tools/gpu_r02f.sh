# round-2: tile search in the pass planner (C4 n=32: 14 -> 9 passes), parity + timing
timeout 1500 python -m pytest -q tests/test_jit.py tests/test_edge_gpu.py tests/test_parity_gpu.py tests/test_baseline_sizes_gpu.py tests/test_partition_gpu.py -m gpu -x -k "not c2_sweep_n28 and not c2_sweep_n24" --durations=5 > gpurun_out/r02f_tests.log 2>&1; echo "pytest rc=$?"; tail -8 gpurun_out/r02f_tests.log
for env in "" "QCS_NO_TILE_SEARCH=1"; do
  env $env timeout 300 python bench.py --no-c2 --no-cpu-baseline --steps 3 > gpurun_out/r02f_bench.log 2>&1; echo "[c4 $env] rc=$?"; python -c "
import json;d=json.loads(open('gpurun_out/r02f_bench.log').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['roofline']['passes_per_step'], d['roofline']['rounds_per_step'], d['roofline']['full_sweeps_per_step'], d['e2e']['ms_per_step'], d['clocks'])"
  env $env timeout 300 python bench.py --workload c5 --n-circuit 32 --no-cpu-baseline --steps 3 > gpurun_out/r02f_bench5.log 2>&1; echo "[c5/32 $env] rc=$?"; python -c "
import json;d=json.loads(open('gpurun_out/r02f_bench5.log').read().strip().splitlines()[-1]);print(d['ms_per_step'], d.get('roofline',{}).get('passes_per_step'), d['clocks'])"
done
timeout 300 python bench.py --workload c3 --no-cpu-baseline --steps 5 > gpurun_out/r02f_bench3.log 2>&1; echo "[c3] rc=$?"; tail -c 600 gpurun_out/r02f_bench3.log
