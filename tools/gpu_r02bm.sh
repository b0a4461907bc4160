# round-2 checkpoint 8 (final): deferred qubits + compact launches: full GPU suite, smoke, bench, reference arm, workloads, launch list, per-rank compute
timeout 2400 python -m pytest tests -m gpu -q -rs --durations=8 > gpurun_out/r02bm_gputest.log 2>&1; echo "pytest rc=$?"; tail -14 gpurun_out/r02bm_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02bm_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/r02bm_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r02bm_bench.log | head -c 1800; echo
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02bm_ref.log 2>&1; echo "ref rc=$?"
for w in c1 c3 c5; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 > gpurun_out/r02bm_$w.log 2>&1; echo "[$w] rc=$?"; tail -1 gpurun_out/r02bm_$w.log | head -c 300; echo
done
timeout 300 python tools/c4_once.py 32 10 > gpurun_out/r02bm_c4once.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum --clock-control none --csv --log-file gpurun_out/r02bm_c4_launches.csv python tools/c4_once.py 32 10 > gpurun_out/r02bm_ncu.log 2>&1; echo "ncu launches rc=$?"
timeout 600 python tools/shard_rank_compute.py 32 2>&1 | tail -4
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29701 bench.py --gpus 1 --sharded --steps 3 --warmup 2 > gpurun_out/r02bm_sharded.log 2>&1; echo "sharded rc=$?"
