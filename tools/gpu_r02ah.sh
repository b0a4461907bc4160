# 16-register rounds on passes with relabellings (QCS_W4_PERMS=1): C5 family A/B + parity
ab() {  # $1 workload, $2 env
  env $2 timeout 300 python bench.py --workload $1 --no-c2 --no-cpu-baseline --steps 5 > gpurun_out/r02ah_b.log 2>&1; echo -n "[$1 $2] rc=$? "; python -c "
import json;d=json.loads(open('gpurun_out/r02ah_b.log').read().strip().splitlines()[-1]);r=d['roofline'];print(round(d['ms_per_step'],3), r['passes_per_step'], r['rounds_per_step'], round(r['fp64']['frac'],3), d['clocks']['sm_mhz'])" 2>/dev/null || tail -2 gpurun_out/r02ah_b.log
}
for rep in 1 2; do ab c5 "QCS_W4_PERMS=0"; ab c5 "QCS_W4_PERMS=1"; ab c5 "QCS_W4_PERMS=1 QCS_W4_MINB=3"; done
QCS_W4_PERMS=1 timeout 900 python -m pytest -q tests/test_jit.py tests/test_baseline_sizes_gpu.py -m gpu -x -k "relabel or c5 or random" 2>&1 | tail -3
