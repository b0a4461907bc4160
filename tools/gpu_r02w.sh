# round-2: 16-register (4-bit) rounds in the specialised kernels (QCS_JIT_W4=1); parity + A/B
QCS_JIT_W4=1 timeout 1500 python -m pytest -q tests/test_jit.py tests/test_edge_gpu.py tests/test_parity_gpu.py tests/test_baseline_sizes_gpu.py -m gpu -x -k "not c2_sweep_n28 and not c2_sweep_n24" > gpurun_out/r02w_tests.log 2>&1; echo "pytest W4 rc=$?"; tail -3 gpurun_out/r02w_tests.log
for env in "QCS_JIT_W4=1" "" "QCS_JIT_W4=1 QCS_W4_MINB=3" "QCS_JIT_W4=1" ""; do
  for w in c4 c5; do
    env $env timeout 300 python bench.py --workload $w --no-c2 --no-cpu-baseline --steps 5 > gpurun_out/r02w_b.log 2>&1; echo "[$w $env] rc=$?"; python -c "
import json;d=json.loads(open('gpurun_out/r02w_b.log').read().strip().splitlines()[-1]);r=d['roofline'];print(round(d['ms_per_step'],2), r['rounds_per_step'], round(r['fp64']['frac'],3), d['clocks']['sm_mhz'])"
  done
done
