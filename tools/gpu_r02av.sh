ab() {  # $1 workload, $2 env
  env $2 timeout 300 python bench.py --workload $1 --no-c2 --no-cpu-baseline --steps 5 > gpurun_out/r02av_b.log 2>&1; echo -n "[$1 $2] rc=$? "; python -c "
import json;d=json.loads(open('gpurun_out/r02av_b.log').read().strip().splitlines()[-1]);r=d['roofline'];print(round(d['ms_per_step'],3), r['passes_per_step'], round(r['fp64']['frac'],3), round(r['frac'],3), d['clocks']['sm_mhz'])" 2>/dev/null || tail -2 gpurun_out/r02av_b.log
}
for rep in 1 2; do for w in c4 c3 c5; do ab $w "QCS_TMA_L2PROMO=256"; ab $w "QCS_TMA_L2PROMO=128"; ab $w "QCS_TMA_L2PROMO=0"; done; done
