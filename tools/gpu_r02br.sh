# the earlier switches re-checked under the final plan (two deferred qubits)
ab() {  # $1 workload, $2 env
  env $2 timeout 300 python bench.py --workload $1 --no-c2 --no-cpu-baseline --steps 5 > gpurun_out/r02br_b.log 2>&1; echo -n "[$1 $2] rc=$? "; python -c "
import json;d=json.loads(open('gpurun_out/r02br_b.log').read().strip().splitlines()[-1]);r=d['roofline'];print(round(d['ms_per_step'],3), r['passes_per_step'], r['rounds_per_step'], round(r['fp64']['instr_per_amplitude'],1), round(r['fp64']['frac'],3), d['clocks']['sm_mhz'])" 2>/dev/null || tail -2 gpurun_out/r02br_b.log
}
for e in "" "QCS_NO_SCALE_CHAIN=1" "QCS_JIT_W4=0" "QCS_PERSIST=0" "QCS_PERSIST=2" "QCS_NO_ROUND_SCHED=1" "QCS_NO_TABLE_NORM=1" "QCS_W4_MINB=1" ""; do ab c4 "$e"; done
