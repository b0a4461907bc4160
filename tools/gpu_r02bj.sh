# deferred qubits (QCS_DEFER=k): the operations outside the light cone of the k top qubits run first, on the 2^-k support
ab() {  # $1 workload, $2 env
  env $2 timeout 300 python bench.py --workload $1 --no-c2 --no-cpu-baseline --steps 5 > gpurun_out/r02bj_b.log 2>&1; echo -n "[$1 $2] rc=$? "; python -c "
import json;d=json.loads(open('gpurun_out/r02bj_b.log').read().strip().splitlines()[-1]);r=d['roofline'];print(round(d['ms_per_step'],3), r['passes_per_step'], round(r['fp64']['frac'],3), round(r['frac'],3), d['clocks']['sm_mhz'], round(d['e2e']['ms_per_step'],2), d['e2e']['max_norm_error'])" 2>/dev/null || tail -2 gpurun_out/r02bj_b.log
}
for k in 0 1 2 3 4 5; do ab c4 "QCS_DEFER=$k"; done
for k in 0 2 3; do ab c5 "QCS_DEFER=$k"; done
QCS_DEFER=2 timeout 900 python -m pytest -q tests/test_baseline_sizes_gpu.py tests/test_parity_gpu.py -m gpu -x -k "not c2_sweep" 2>&1 | tail -2
