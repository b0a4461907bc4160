"""World-size-1 NCCL smoke of the real transport code on one GPU: DistTransport.swap_blocks and
.exchange with CUDA tensors, the partner being this rank itself (NCCL matches a grouped send and
receive to self).  What comes back is what was sent, so the shard must be unchanged; what this
exercises is the NCCL point-to-point batch on complex128 views, the chunked double-buffered
staging, the side-stream copies and the event ordering -- the code a multi-GPU run takes, which
the gloo and in-process transports of the other tests never touch."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    port = int(sys.argv[1]) if len(sys.argv) > 1 else 29611
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", world_size=1, rank=0)
    from paper_2411_15332_b200.partition import DeviceBackend, DistTransport
    n_local = 22
    be = DeviceBackend(n_local, 0)
    be.state.randomize(11)
    be.sync()
    before = be.tensor.clone()
    tr = DistTransport()
    k = 2
    pairs = [(0, 1, 0), (0, 3, 2)]          # (peer, my block, the partner's block): peer = self
    tr.swap_blocks(be, k, pairs, chunk=1 << 16)   # 16 chunks per block, two staging slots
    torch.cuda.synchronize()
    assert torch.equal(be.tensor, before), "the shard changed under a self exchange"
    send = be.block(k, 1, 0, 1 << 12)
    recv = be.empty(1 << 12)
    tr.exchange(send, recv, 0)
    torch.cuda.synchronize()
    assert torch.equal(send, recv)
    # the peer-memory path at world size 1: a symmetric-memory shard, the rendezvous, its barrier,
    # and the swap kernel through the mapped "partner" buffer (this rank's own): the two halves of
    # the shard trade places
    try:
        from paper_2411_15332_b200.partition import SymmetricTransport
        sb = DeviceBackend(n_local, 0, symmetric=True)
        sb.state.randomize(12)
        sb.sync()
        ref = sb.tensor.clone()
        st = SymmetricTransport()
        st.attach(sb)
        half = 1 << (n_local - 1)
        st.barrier()
        sb.swap_peer(0, st.peer_buffer(0)[half:], half)
        st.barrier()
        torch.cuda.synchronize()
        assert torch.equal(sb.tensor[:half], ref[half:]) and torch.equal(sb.tensor[half:], ref[:half])
        print("symmetric memory swap ok")
    except (ImportError, RuntimeError, AttributeError) as e:  # no symmetric memory on this box / build
        print("symmetric memory path skipped:", type(e).__name__, str(e)[:200])
    dist.destroy_process_group()
    print("nccl self exchange ok")


main()
