# round-2 checkpoint 6 (final): full GPU suite, smoke, the default bench line, the reference arm, every workload's line,
# the C4 n=32 launch list, full captures of a heavy and a light persistent C4 pass and of a C5-family pass
timeout 2400 python -m pytest tests -m gpu -q -rs --durations=8 > gpurun_out/r02ax_gputest.log 2>&1; echo "pytest rc=$?"; tail -14 gpurun_out/r02ax_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02ax_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/r02ax_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r02ax_bench.log | head -c 2500; echo
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02ax_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/r02ax_ref.log | head -c 600; echo
for w in c1 c3 c5 rh-signs; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 > gpurun_out/r02ax_$w.log 2>&1; echo "[$w] rc=$?"; tail -1 gpurun_out/r02ax_$w.log | head -c 500; echo
done
timeout 900 python bench.py --workload c2 --steps 3 --warmup 3 > gpurun_out/r02ax_c2.log 2>&1; echo "[c2] rc=$?"
timeout 300 python tools/c4_once.py 32 10 > gpurun_out/r02ax_c4once.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum --clock-control none --csv --log-file gpurun_out/r02ax_c4_launches.csv python tools/c4_once.py 32 10 > gpurun_out/r02ax_ncu.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qcs_pass -s 3 -c 1 -o gpurun_out/r02ax_c4heavy python tools/c4_once.py 28 10 > gpurun_out/r02ax_ncu2.log 2>&1; echo "ncu heavy rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qcs_pass -s 6 -c 1 -o gpurun_out/r02ax_c4light python tools/c4_once.py 28 10 > gpurun_out/r02ax_ncu3.log 2>&1; echo "ncu light rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qcs_pass -s 8 -c 1 -o gpurun_out/r02ax_c5pass python tools/c5_once.py 28 20 > gpurun_out/r02ax_ncu4.log 2>&1; echo "ncu c5 rc=$?"
