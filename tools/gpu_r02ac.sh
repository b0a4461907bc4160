# split static / group-dependent sign flips (QCS_JIT_SPLIT_SIGNS): parity + A/B; where the W3 persistent kernel fails
timeout 1500 python -m pytest -q tests/test_jit.py tests/test_edge_gpu.py tests/test_parity_gpu.py tests/test_baseline_sizes_gpu.py -m gpu -x -k "not c2_sweep_n28 and not c2_sweep_n24" > gpurun_out/r02ac_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02ac_tests.log
ab() {  # $1 workload, $2 env
  env $2 timeout 300 python bench.py --workload $1 --no-c2 --no-cpu-baseline --steps 5 > gpurun_out/r02ac_b.log 2>&1; echo -n "[$1 $2] rc=$? "; python -c "
import json;d=json.loads(open('gpurun_out/r02ac_b.log').read().strip().splitlines()[-1]);r=d['roofline'];print(round(d['ms_per_step'],3), r['passes_per_step'], r['rounds_per_step'], round(r['fp64']['frac'],3), d['clocks']['sm_mhz'])" 2>/dev/null || tail -2 gpurun_out/r02ac_b.log
}
for rep in 1 2; do
  for w in c4 c5; do ab $w "QCS_JIT_SPLIT_SIGNS=0"; ab $w "QCS_JIT_SPLIT_SIGNS=1"; done
done
ab c4 "QCS_PERSIST=2"
ab c4 "QCS_PERSIST_SLOTS=3 QCS_W4_MINB=1"
for n in 26 28 29 30; do
  env QCS_PERSIST=2 CUDA_LAUNCH_BLOCKING=1 timeout 120 python tools/persist_check.py c3 $n 2>&1 | tail -1 | cut -c1-150
done
