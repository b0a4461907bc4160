# generalised persistent form (relabelled passes with direct stores, cp.async tiles): parity + A/B
timeout 900 python -m pytest -q tests/test_jit.py -m gpu -x -k "pipelined" 2>&1 | tail -3
for c in "c5 26" "c5 30"; do for e in 0 2; do env QCS_PERSIST=$e timeout 200 python tools/persist_check.py $c 2>&1 | tail -3 | cut -c1-220; done; done
env QCS_PERSIST=2 timeout 300 python tools/norm_check.py 32 2 c5 2>&1 | tail -1
ab() {  # $1 workload, $2 env
  env $2 timeout 300 python bench.py --workload $1 --no-c2 --no-cpu-baseline --steps 5 > gpurun_out/r02aj_b.log 2>&1; echo -n "[$1 $2] rc=$? "; python -c "
import json;d=json.loads(open('gpurun_out/r02aj_b.log').read().strip().splitlines()[-1]);r=d['roofline'];print(round(d['ms_per_step'],3), r['passes_per_step'], r['rounds_per_step'], round(r['fp64']['frac'],3), round(r['frac'],3), d['clocks']['sm_mhz'])" 2>/dev/null || tail -2 gpurun_out/r02aj_b.log
}
for rep in 1 2; do ab c5 "QCS_PERSIST=1"; ab c5 "QCS_PERSIST=2"; done
ab c4 "QCS_PERSIST=1"; ab c4 "QCS_PERSIST=2"
ab c3 "QCS_PERSIST=1"; ab c3 "QCS_PERSIST=2"
