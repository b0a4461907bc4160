timeout 900 python -m pytest -q tests/test_partition_gpu.py -m gpu -x 2>&1 | tail -3
for extra in "" "--peer"; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29701 bench.py --gpus 1 --sharded $extra --steps 3 --warmup 2 > gpurun_out/r02bc_sharded.log 2>&1; echo "sharded $extra rc=$?"; tail -1 gpurun_out/r02bc_sharded.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['e2e']['ms_per_step'], d['gpu_launches'], d['clocks']['sm_mhz'])"
done
cp gpurun_out/r02bc_sharded.log gpurun_out/r02bc_sharded_peer.log
