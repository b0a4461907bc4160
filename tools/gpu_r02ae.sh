# persistent kernels with two barriers per slot: cold-process norm checks, the C3 W3 shape, then parity + A/B
for i in 1 2 3; do env QCS_PERSIST=1 timeout 300 python tools/norm_check.py 32 2 2>&1 | tail -1; done
env QCS_PERSIST=2 timeout 300 python tools/norm_check.py 32 2 2>&1 | tail -1
for n in 26 30; do env QCS_PERSIST=2 timeout 120 python tools/persist_check.py c3 $n 2>&1 | tail -2 | cut -c1-200; env QCS_PERSIST=0 timeout 120 python tools/persist_check.py c3 $n 2>&1 | tail -2 | cut -c1-200; done
timeout 1500 python -m pytest -q tests/test_jit.py tests/test_edge_gpu.py tests/test_parity_gpu.py tests/test_baseline_sizes_gpu.py -m gpu -x -k "not c2_sweep_n28 and not c2_sweep_n24" > gpurun_out/r02ae_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02ae_tests.log
ab() {  # $1 workload, $2 env
  env $2 timeout 300 python bench.py --workload $1 --no-c2 --no-cpu-baseline --steps 5 > gpurun_out/r02ae_b.log 2>&1; echo -n "[$1 $2] rc=$? "; python -c "
import json;d=json.loads(open('gpurun_out/r02ae_b.log').read().strip().splitlines()[-1]);r=d['roofline'];print(round(d['ms_per_step'],3), r['passes_per_step'], r['rounds_per_step'], round(r['fp64']['frac'],3), d['clocks']['sm_mhz'])" 2>/dev/null || tail -2 gpurun_out/r02ae_b.log
}
for w in c4 c3 c5; do ab $w "QCS_PERSIST=0"; ab $w "QCS_PERSIST=1"; ab $w "QCS_PERSIST=2"; done
