# round-2: tile gaps ride in the TMA run dims (more passes load/store as TMA boxes); parity + A/B; C3 knob sweep
timeout 1500 python -m pytest -q tests/test_jit.py tests/test_edge_gpu.py tests/test_parity_gpu.py tests/test_baseline_sizes_gpu.py -m gpu -x -k "not c2_sweep_n28 and not c2_sweep_n24" > gpurun_out/r02z_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02z_tests.log
ab() {  # $1 workload, $2 env
  env $2 timeout 300 python bench.py --workload $1 --no-c2 --no-cpu-baseline --steps 5 > gpurun_out/r02z_b.log 2>&1; echo -n "[$1 $2] rc=$? "; python -c "
import json;d=json.loads(open('gpurun_out/r02z_b.log').read().strip().splitlines()[-1]);r=d['roofline'];print(round(d['ms_per_step'],3), r['passes_per_step'], r['rounds_per_step'], round(r['fp64']['frac'],3), d['clocks']['sm_mhz'])"
}
for rep in 1 2; do
  for w in c4 c5 c3; do ab $w ""; ab $w "QCS_TMA_GAP_DIMS=1"; done
done
for e in "QCS_JIT_W4=0" "QCS_NO_ROUND_SCHED=1" "QCS_NO_TILE_SEARCH=1" "QCS_NO_TMA_ITER=1" "QCS_NO_SCALE_CHAIN=1" "QCS_NO_TABLE_NORM=1" ""; do ab c3 "$e"; done
