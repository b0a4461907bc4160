# round-2: lazy +-1 signs in the specialised kernels (QCS_JIT_LAZY_SIGNS); parity + A/B
timeout 1500 python -m pytest -q tests/test_jit.py tests/test_edge_gpu.py tests/test_parity_gpu.py tests/test_baseline_sizes_gpu.py tests/test_partition_gpu.py tests/test_shim_gpu.py -m gpu -x -k "not c2_sweep_n28 and not c2_sweep_n24" > gpurun_out/r02o_tests.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/r02o_tests.log
for env in "" "QCS_JIT_LAZY_SIGNS=0"; do
  for w in c4 c5 c3; do
    env $env timeout 300 python bench.py --workload $w --no-c2 --no-cpu-baseline --steps 3 > gpurun_out/r02o_b.log 2>&1; echo "[$w $env] rc=$?"; python -c "
import json;d=json.loads(open('gpurun_out/r02o_b.log').read().strip().splitlines()[-1]);r=d['roofline'];print(round(d['ms_per_step'],2), r['passes_per_step'], round(r['fp64']['frac'],3), round(r['frac'],3), d['e2e']['ms_per_step'], d['clocks']['sm_mhz'])"
  done
done
