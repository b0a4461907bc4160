# round-2: how many iterated TMA boxes pay (QCS_TMA_MAX_ITER)
for it in 1 2 3 4; do
  for w in c4 c5; do
    QCS_TMA_MAX_ITER=$it timeout 300 python bench.py --workload $w --no-c2 --no-cpu-baseline --steps 3 > gpurun_out/r02n_b.log 2>&1; echo "[$w iter<=$it] rc=$?"; python -c "
import json;d=json.loads(open('gpurun_out/r02n_b.log').read().strip().splitlines()[-1]);r=d['roofline'];print(round(d['ms_per_step'],2), r['passes_per_step'], round(r['fp64']['frac'],3), round(r['frac'],3), d['clocks']['sm_mhz'])"
  done
done
