# round-2: C4 kernel launch knobs (resident tiles per SM, group-loop unroll)
for env in "" "QCS_JIT_MINB=2" "QCS_JIT_UNROLL=2" "QCS_JIT_MINB=2 QCS_JIT_UNROLL=2" "QCS_JIT_BANKSWAP=0"; do
    env $env timeout 300 python bench.py --no-c2 --no-cpu-baseline --steps 5 > gpurun_out/r02u_b.log 2>&1; echo "[c4 $env] rc=$?"; python -c "
import json;d=json.loads(open('gpurun_out/r02u_b.log').read().strip().splitlines()[-1]);r=d['roofline'];print(round(d['ms_per_step'],2), round(r['fp64']['frac'],3), d['clocks']['sm_mhz'])"
done
