# wider tile-search seed window for plans of many passes (C5 family: 25 -> 23 passes): parity + A/B
timeout 1200 python -m pytest -q tests/test_baseline_sizes_gpu.py tests/test_jit.py tests/test_edge_gpu.py -m gpu -x -k "c5 or relabel or random" 2>&1 | tail -2
ab() {  # $1 workload, $2 env
  env $2 timeout 300 python bench.py --workload $1 --no-c2 --no-cpu-baseline --steps 5 > gpurun_out/r02aw_b.log 2>&1; echo -n "[$1 $2] rc=$? "; python -c "
import json;d=json.loads(open('gpurun_out/r02aw_b.log').read().strip().splitlines()[-1]);r=d['roofline'];print(round(d['ms_per_step'],3), r['passes_per_step'], round(r['fp64']['frac'],3), round(r['frac'],3), d['clocks']['sm_mhz'], round(d['e2e']['ms_per_step'],2))" 2>/dev/null || tail -2 gpurun_out/r02aw_b.log
}
for rep in 1 2; do ab c5 "QCS_TILE_DEEP_SEEDS=0"; ab c5 "QCS_TILE_DEEP_SEEDS=400"; done
ab c4 ""
