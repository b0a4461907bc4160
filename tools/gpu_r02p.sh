# round-2: lazy signs A/B, alternating repetitions (power-cap clock noise)
for rep in 1 2 3; do
for env in "" "QCS_JIT_LAZY_SIGNS=0"; do
    env $env timeout 300 python bench.py --workload c4 --no-c2 --no-cpu-baseline --steps 5 > gpurun_out/r02p_b.log 2>&1; echo "[c4 $env] rc=$?"; python -c "
import json;d=json.loads(open('gpurun_out/r02p_b.log').read().strip().splitlines()[-1]);r=d['roofline'];print(round(d['ms_per_step'],2), round(r['fp64']['frac'],3), d['clocks']['sm_mhz'], round(d['ms_per_step']*d['clocks']['sm_mhz']/1965,2))"
done
done
