# round-2: the light-cone round scheduler + scale chaining, parity and A/B timing
timeout 1500 python -m pytest -q tests/test_jit.py tests/test_edge_gpu.py tests/test_parity_gpu.py tests/test_baseline_sizes_gpu.py tests/test_shim_gpu.py -m gpu -x -k "not c2_sweep_n28 and not c2_sweep_n24" --durations=8 > gpurun_out/r02d_tests.log 2>&1; echo "pytest rc=$?"; tail -14 gpurun_out/r02d_tests.log
for env in "" "QCS_NO_SCALE_CHAIN=1" "QCS_NO_ROUND_SCHED=1"; do
  env $env timeout 300 python bench.py --no-c2 --no-cpu-baseline --steps 3 > gpurun_out/r02d_bench.log 2>&1; echo "[$env] rc=$?"; python -c "
import json;d=json.loads(open('gpurun_out/r02d_bench.log').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['roofline']['rounds_per_step'], d['e2e']['ms_per_step'], d['clocks'])"
done
