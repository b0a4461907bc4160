"""The partitioner with real B200 kernels: P ranks emulated by P threads on one GPU, each with
its own device shard (DeviceBackend: a torch tensor wrapped by qcs_state_wrap) and an
in-process transport for the remap exchanges.  Compared with the single-GPU
engine (qcsim.simulate) on the same circuits ('a fake partition running
P shards on one GPU, which exercises the exchange logic without NVLink')."""
import numpy as np
import pytest

from partition_helpers import ThreadTransport, circuit_ops, gather, run_ops, run_ranks

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 4, 8])
def test_emulated_ranks_match_single_gpu(world):
    from paper_2411_15332_b200 import configs
    from paper_2411_15332_b200 import qcsim as Q
    from paper_2411_15332_b200.partition import DeviceBackend, ShardedState
    g = world.bit_length() - 1
    for c in (configs.c4_circuit(n=16, layers=2), configs.c5_circuit(n=17, layers=2, global_qubits=g)):
        want = Q.simulate(c, Q.Engine.rh_dax).final.download()
        hub = ThreadTransport()

        def rank_fn(r):
            st = ShardedState(c.n, world, r, DeviceBackend(c.n - g), hub.endpoint(r), initial=c.initial,
                              chunk_elems=1 << 12)
            run_ops(st, circuit_ops(c))
            return st, st.local_numpy()

        outs = run_ranks(world, rank_fn)
        got = gather([o[0] for o in outs], [o[1] for o in outs])
        assert np.abs(got - want).max() < 1e-12
        assert np.linalg.norm(got - want) < 1e-10
        assert all(o[0].swaps > 0 for o in outs)


@pytest.mark.parametrize("mode", ["split", "remap"])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_emulated_peer_gates_match_single_gpu(world, mode):
    """Peer mode on one GPU: the P shards are P buffers on the device, so the partner
    loads/stores of qcs_apply_split (mode split) and qcs_swap_peer (remaps) are plain device
    accesses (NVLink P2P on a multi-GPU box)."""
    from paper_2411_15332_b200 import configs
    from paper_2411_15332_b200 import qcsim as Q
    from paper_2411_15332_b200.partition import DeviceBackend, ShardedState
    g = world.bit_length() - 1
    for c in (configs.c4_circuit(n=16, layers=2), configs.c5_circuit(n=17, layers=2, global_qubits=g),
              Q.build_grover(15, 12345, 3)):
        want = Q.simulate(c, Q.Engine.rh_dax).final.download()
        hub = ThreadTransport(world, peers=True)

        def rank_fn(r):
            st = ShardedState(c.n, world, r, DeviceBackend(c.n - g), hub.endpoint(r), initial=c.initial,
                              chunk_elems=1 << 12, mode=mode)
            assert st.peer
            run_ops(st, circuit_ops(c))
            return st, st.local_numpy()

        outs = run_ranks(world, rank_fn)
        got = gather([o[0] for o in outs], [o[1] for o in outs])
        assert np.abs(got - want).max() < 1e-12
        assert np.linalg.norm(got - want) < 1e-10
        if mode == "split":
            assert all(o[0].splits > 0 for o in outs)
        else:
            assert all(o[0].swaps > 0 and o[0].splits == 0 for o in outs)


@pytest.mark.parametrize("world", [2, 4])
def test_emulated_ranks_specialised_kernels(world):
    """The same sharded circuits with every local pass as a specialised kernel (jit mode 3:
    pivoted gates, relabellings, group scalars), against the single-GPU interpreter."""
    from paper_2411_15332_b200 import configs
    from paper_2411_15332_b200 import qcsim as Q
    from paper_2411_15332_b200.partition import DeviceBackend, ShardedState
    g = world.bit_length() - 1
    old = Q.jit_mode()
    try:
        for c in (configs.c4_circuit(n=16, layers=2), configs.c5_circuit(n=17, layers=2, global_qubits=g)):
            Q.set_jit_mode(0)
            want = Q.simulate(c, Q.Engine.rh_dax).final.download()
            Q.set_jit_mode(3)
            hub = ThreadTransport()

            def rank_fn(r):
                st = ShardedState(c.n, world, r, DeviceBackend(c.n - g), hub.endpoint(r), initial=c.initial,
                                  chunk_elems=1 << 12)
                run_ops(st, circuit_ops(c))
                return st, st.local_numpy()

            outs = run_ranks(world, rank_fn)
            got = gather([o[0] for o in outs], [o[1] for o in outs])
            assert np.abs(got - want).max() < 1e-12
            assert np.linalg.norm(got - want) < 1e-10
    finally:
        Q.set_jit_mode(old)


def test_split_gate_bit_exact():
    """One gate on a global qubit through qcs_apply_split equals the single-GPU gate kernel
    bit for bit (both follow dax_mvm's arithmetic)."""
    from conftest import bits_equal, random_state
    from paper_2411_15332_b200 import qcsim as Q
    from paper_2411_15332_b200.partition import DeviceBackend, ShardedState
    n, world = 14, 4
    x = random_state(n, 11)
    G = Q.gate_catalog_lookup
    for gate, qubits in ((G("Hadamard"), [0]), (G("U", [0.3, 1.7, 2.9]), [1]), (G("CNOT"), [6, 0]),
                         (G("Toffoli"), [9, 4, 1]), (G("Pauli-Y"), [0])):
        s = Q.DeviceState.from_numpy(x)
        s.apply_gate(gate, qubits)
        want = s.download()
        hub = ThreadTransport(world, peers=True)

        def rank_fn(r):
            import torch
            st = ShardedState(n, world, r, DeviceBackend(n - 2), hub.endpoint(r), mode="split")
            local = x.reshape(world, -1)[r]
            st.backend.tensor.copy_(torch.from_numpy(local.copy()))
            st.apply_gate(gate.matrix, qubits, gate.name)
            return st, st.local_numpy()

        outs = run_ranks(world, rank_fn)
        got = gather([o[0] for o in outs], [o[1] for o in outs])
        assert all(o[0].splits == 1 and o[0].swaps == 0 for o in outs), gate.name
        assert bits_equal(got, want), gate.name


def test_nccl_transport_self_exchange():
    """The NCCL transport (DistTransport.swap_blocks / .exchange on CUDA tensors) run for real at
    world size 1, the partner being the rank itself (tools/nccl_self_exchange.py): the chunked,
    double-buffered send/recv path a multi-GPU run takes, which needs no second GPU to execute.
    In a subprocess with a time limit (a process group per test process; an NCCL build that
    cannot send to self would hang rather than fail)."""
    import os
    import socket
    import subprocess
    import sys

    from conftest import ROOT
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    try:
        out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "nccl_self_exchange.py"), str(port)],
                             capture_output=True, text=True, timeout=240, cwd=ROOT)
    except subprocess.TimeoutExpired:
        pytest.skip("NCCL send/recv to self did not complete on this box")
    assert out.returncode == 0 and "nccl self exchange ok" in out.stdout, out.stderr[-2000:]


def test_world1_sharded_equals_simulate_and_defers_the_reset():
    """One rank: the sharded path hands the whole circuit to the fused engine with the reset
    folded in (the shard is known to be |initial>, its memory untouched until the run writes it),
    so the result is bit for bit simulate's; a reader of the shard's tensor in between sees the
    basis state (the deferred reset is written first)."""
    from conftest import bits_equal
    from paper_2411_15332_b200 import configs
    from paper_2411_15332_b200 import qcsim as Q
    from paper_2411_15332_b200.partition import DeviceBackend, ShardedState
    c = configs.c4_circuit(n=18, layers=3)
    want = Q.simulate(c, Q.Engine.rh_dax).final.download()
    be = DeviceBackend(c.n)
    st = ShardedState(c.n, 1, 0, be, None, initial=c.initial)
    assert be.known == c.initial and be.stale
    st.run(circuit_ops(c))
    st.flush()
    assert be.known is None and not be.stale
    assert bits_equal(st.local_numpy(), want)
    st.reset(5)
    assert be.stale
    t = be.tensor  # an outside reader: the reset is materialised, the content no longer assumed
    assert not be.stale and be.known is None
    assert complex(t[5].item()) == 1.0 and float(t.abs().sum().item()) == 1.0


def test_bench_sharded_arm_on_one_gpu():
    """bench.py --sharded under torchrun with one rank: the N > 1 code path (NCCL process group,
    DeviceBackend, ShardedState, exchange accounting, the JSON line) runs on one B200."""
    import json
    import os
    import socket
    import subprocess
    import sys

    from conftest import ROOT
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1", "--master-addr",
           "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"), "--gpus", "1", "--sharded",
           "--n-circuit", "22", "--steps", "2", "--warmup", "1", "--no-clocks"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 1 and d["scaling"] == "strong" and d["gpu_launches"] > 0
    assert any("NCCL" in s for s in d["comm_init"]) and d["exchange"]["remaps_per_step"] == 0
