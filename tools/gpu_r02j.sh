# round-2: dense engine + bench modes + sampling tests; C5 family A/B of the round-2 planner switches
timeout 900 python -m pytest -q tests/test_dense_gpu.py tests/test_bench_modes.py tests/test_sample_gpu.py -m gpu -x -rs > gpurun_out/r02j_tests.log 2>&1; echo "pytest rc=$?"; tail -12 gpurun_out/r02j_tests.log
for env in "" "QCS_NO_TILE_SEARCH=1" "QCS_NO_ROUND_SCHED=1" "QCS_NO_WHT_MERGE=1" "QCS_PIVOT_LARGER=1" "QCS_NO_SCALE_CHAIN=1"; do
  env $env timeout 300 python bench.py --workload c5 --n-circuit 32 --no-cpu-baseline --steps 3 > gpurun_out/r02j_c5.log 2>&1; echo "[c5/32 $env] rc=$?"; python -c "
import json;d=json.loads(open('gpurun_out/r02j_c5.log').read().strip().splitlines()[-1]);r=d['roofline'];print(round(d['ms_per_step'],1), r['passes_per_step'], r['rounds_per_step'], round(r['fp64']['frac'],3), round(r['frac'],3), d['clocks']['sm_mhz'])"
done
timeout 300 python bench.py --workload rh-signs > gpurun_out/r02j_rh.log 2> gpurun_out/r02j_rh_rows.csv; echo "rh-signs rc=$?"; head -c 400 gpurun_out/r02j_rh.log; echo; cat gpurun_out/r02j_rh_rows.csv | head -30
