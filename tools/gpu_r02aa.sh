# round-2: persistent pipelined pass kernels (QCS_PERSIST) -- parity, then A/B on C4 / C5 / C3
timeout 1500 python -m pytest -q tests/test_jit.py tests/test_edge_gpu.py tests/test_parity_gpu.py tests/test_baseline_sizes_gpu.py -m gpu -x -k "not c2_sweep_n28 and not c2_sweep_n24" > gpurun_out/r02aa_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02aa_tests.log
ab() {  # $1 workload, $2 env
  env $2 timeout 300 python bench.py --workload $1 --no-c2 --no-cpu-baseline --steps 5 > gpurun_out/r02aa_b.log 2>&1; echo -n "[$1 $2] rc=$? "; python -c "
import json;d=json.loads(open('gpurun_out/r02aa_b.log').read().strip().splitlines()[-1]);r=d['roofline'];print(round(d['ms_per_step'],3), r['passes_per_step'], r['rounds_per_step'], round(r['fp64']['frac'],3), d['clocks']['sm_mhz'])" || tail -5 gpurun_out/r02aa_b.log
}
for rep in 1 2; do
  for w in c4 c5 c3; do ab $w "QCS_PERSIST=0"; ab $w "QCS_PERSIST=1";  ab $w "QCS_PERSIST=2"; done
done
ab c4 "QCS_PERSIST=1 QCS_PLAN_ONE_POLICY=1"
ab c3 "QCS_PERSIST=0 QCS_W4_MIN_GATES=0"
