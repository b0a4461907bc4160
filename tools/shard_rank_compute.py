"""Per-rank COMPUTE of the sharded C4 circuit, measured on one GPU: rank 0's local batches (the
fused passes on its 2^(n-g) shard, local swaps included) at world sizes 2/4/8 with the exchange
replaced by a no-op (the blocks stay where they are: the amplitudes are not the circuit's, the
kernels and their sizes are).  Not a scaling measurement -- there is no second GPU and no
traffic here -- but it shows what a rank spends outside the exchange, and finds slow local work."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2411_15332_b200 import configs  # noqa: E402
from paper_2411_15332_b200.partition import DeviceBackend, ShardedState, circuit_ops  # noqa: E402


class NullTransport:
    def swap_blocks(self, backend, k, pairs, chunk):
        backend.block(k, pairs[0][1], 0, 1)  # (the shard's content is no longer known, as after a real exchange)


n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
c = configs.c4_circuit(n)
ops = circuit_ops(c)
for world in (1, 2, 4, 8):
    g = world.bit_length() - 1
    be = DeviceBackend(n - g, 0)
    sh = ShardedState(n, world, 0, be, NullTransport() if world > 1 else None, initial=c.initial)

    def step():
        sh.reset(c.initial)
        sh.run(ops)
        sh.flush()
    for _ in range(2):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(3):
        step()
    e1.record()
    e1.synchronize()
    host = (time.perf_counter() - t0) / 3
    print(f"world {world}: shard 2^{n - g}, rank-0 compute {e0.elapsed_time(e1) / 3:8.2f} ms per circuit "
          f"(host loop {1e3 * host:7.2f} ms), remaps {sh.swaps // 5}")
    del sh, be
    torch.cuda.empty_cache()
