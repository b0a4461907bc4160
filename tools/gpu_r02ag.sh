# round-2 checkpoint 4 (persistent pipelined passes, split sign flips, two-policy tile search): full GPU suite, smoke,
# the default bench line, the reference arm, every workload's line, the C4 n=32 launch list
timeout 2400 python -m pytest tests -m gpu -q -rs --durations=10 > gpurun_out/r02ag_gputest.log 2>&1; echo "pytest rc=$?"; tail -16 gpurun_out/r02ag_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02ag_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/r02ag_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r02ag_bench.log | head -c 3000; echo
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02ag_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/r02ag_ref.log | head -c 1500; echo
for w in c1 c3 c5 rh-signs; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 > gpurun_out/r02ag_$w.log 2>&1; echo "[$w] rc=$?"; tail -1 gpurun_out/r02ag_$w.log | head -c 1200; echo
done
timeout 900 python bench.py --workload c2 --steps 3 --warmup 3 > gpurun_out/r02ag_c2.log 2>&1; echo "[c2] rc=$?"; tail -1 gpurun_out/r02ag_c2.log | head -c 1200; echo
timeout 300 python tools/c4_once.py 32 10 > gpurun_out/r02ag_c4once.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum --clock-control none --csv --log-file gpurun_out/r02ag_c4_launches.csv python tools/c4_once.py 32 10 > gpurun_out/r02ag_ncu.log 2>&1; echo "ncu rc=$?"
