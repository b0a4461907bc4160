# round-2: normalised round tables (QCS_NO_TABLE_NORM); parity + alternating A/B
timeout 1500 python -m pytest -q tests/test_jit.py tests/test_edge_gpu.py tests/test_parity_gpu.py tests/test_baseline_sizes_gpu.py -m gpu -x -k "not c2_sweep_n28 and not c2_sweep_n24" > gpurun_out/r02v_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02v_tests.log
for rep in 1 2; do
for env in "" "QCS_NO_TABLE_NORM=1"; do
  for w in c4 c5; do
    env $env timeout 300 python bench.py --workload $w --no-c2 --no-cpu-baseline --steps 5 > gpurun_out/r02v_b.log 2>&1; echo "[$w $env] rc=$?"; python -c "
import json;d=json.loads(open('gpurun_out/r02v_b.log').read().strip().splitlines()[-1]);r=d['roofline'];print(round(d['ms_per_step'],2), round(r['fp64']['frac'],3), d['clocks']['sm_mhz'])"
  done
done
done
