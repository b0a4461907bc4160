# round-2 checkpoint 3 (4-bit rounds, normalised tables): full GPU suite, smoke, the default bench line, the reference arm, C4 launch list
timeout 2400 python -m pytest tests -m gpu -q -rs --durations=10 > gpurun_out/r02x_gputest.log 2>&1; echo "pytest rc=$?"; tail -16 gpurun_out/r02x_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02x_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/r02x_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r02x_bench.log | head -c 2500; echo
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02x_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/r02x_ref.log | head -c 1500; echo
timeout 300 python tools/c4_once.py 32 10 > gpurun_out/r02x_c4once.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum --clock-control none --csv --log-file gpurun_out/r02x_c4_launches.csv python tools/c4_once.py 32 10 > gpurun_out/r02x_ncu.log 2>&1; echo "ncu rc=$?"
