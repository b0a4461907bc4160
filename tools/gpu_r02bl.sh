# compact launches for passes that skip most tiles (QCS_NO_COMPACT_LAUNCH=1 restores the full grid): parity + A/B
timeout 1500 python -m pytest -q tests/test_baseline_sizes_gpu.py tests/test_parity_gpu.py tests/test_jit.py tests/test_edge_gpu.py -m gpu -x -k "not c2_sweep" 2>&1 | tail -2
ab() {  # $1 workload, $2 env
  env $2 timeout 300 python bench.py --workload $1 --no-c2 --no-cpu-baseline --steps 5 > gpurun_out/r02bl_b.log 2>&1; echo -n "[$1 $2] rc=$? "; python -c "
import json;d=json.loads(open('gpurun_out/r02bl_b.log').read().strip().splitlines()[-1]);r=d['roofline'];print(round(d['ms_per_step'],3), r['passes_per_step'], round(r['fp64']['frac'],3), round(r['frac'],3), d['clocks']['sm_mhz'], round(d['e2e']['ms_per_step'],2), d['e2e']['max_norm_error'])" 2>/dev/null || tail -2 gpurun_out/r02bl_b.log
}
for rep in 1 2; do ab c4 "QCS_NO_COMPACT_LAUNCH=1"; ab c4 ""; done
ab c3 "QCS_NO_COMPACT_LAUNCH=1"; ab c3 ""
