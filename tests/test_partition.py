"""Multi-rank partitioner (paper_2411_15332_b200/partition.py) on the CPU.

* world 2 and 4 with torch.distributed over gloo (separate processes, 127.0.0.1), the shard
  compute done by the C oracle: the exchange / remap / reduction logic is what is under test;
* P threads in one process with an in-process transport (many layouts quickly).
Reference results: the oracle on the full state ("P-GPU versus 1-GPU
equality on the same circuit")."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT
from partition_helpers import (OracleBackend, ThreadTransport, circuit_ops, gather, oracle_full, run_ops,
                               run_ops_one_by_one, run_ranks)


def circuits():
    from paper_2411_15332_b200 import configs
    from paper_2411_15332_b200 import qcsim as Q
    return {
        "c4": configs.c4_circuit(n=8, layers=2),
        "c5": configs.c5_circuit(n=9, layers=2, global_qubits=2),
        "grover": Q.build_grover(7, 77, 3),
        "c1": configs.c1_circuit(n=6, layers=1),
    }


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("name", ["c4", "c5", "grover", "c1"])
def test_threads_match_full_state(oracle, world, name):
    from paper_2411_15332_b200.partition import ShardedState
    c = circuits()[name]
    want = oracle_full(oracle, c)
    hub = ThreadTransport()
    g = world.bit_length() - 1

    def rank_fn(r):
        st = ShardedState(c.n, world, r, OracleBackend(c.n - g, oracle), hub.endpoint(r), initial=c.initial,
                          chunk_elems=7)
        run_ops(st, circuit_ops(c))
        return st, st.local_numpy()

    outs = run_ranks(world, rank_fn)
    got = gather([o[0] for o in outs], [o[1] for o in outs])
    assert np.abs(got - want).max() < 1e-12
    assert sum(o[0].swaps for o in outs) > 0 or name == "c1" and world == 2


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("name", ["c4", "c5", "grover"])
def test_threads_one_op_at_a_time(oracle, world, name):
    """Immediate mode (apply_gate / apply_diag / apply_rh one by one): no reordering across
    operations, a remap whenever a gate needs a global qubit."""
    from paper_2411_15332_b200.partition import ShardedState
    c = circuits()[name]
    want = oracle_full(oracle, c)
    hub = ThreadTransport()
    g = world.bit_length() - 1

    def rank_fn(r):
        st = ShardedState(c.n, world, r, OracleBackend(c.n - g, oracle), hub.endpoint(r), initial=c.initial,
                          chunk_elems=5)
        run_ops_one_by_one(st, circuit_ops(c))
        return st, st.local_numpy()

    outs = run_ranks(world, rank_fn)
    assert np.abs(gather([o[0] for o in outs], [o[1] for o in outs]) - want).max() < 1e-12


@pytest.mark.parametrize("world,layers", [(2, 2), (4, 2), (8, 3)])
def test_c4_one_batched_remap_per_layer(oracle, world, layers):
    """The scheduler runs every gate it can before exchanging (later layers' gates included),
    then brings the global qubits the waiting gates need down in ONE remap: H^n plus `layers`
    RY layers cost at most layers + 1 remaps, each moving at most (2^g - 1)/2^g of a shard.
    (Qubit-at-a-time swaps would cost g half-shard exchanges per layer.)"""
    from paper_2411_15332_b200 import configs
    from paper_2411_15332_b200.partition import ShardedState
    c = configs.c4_circuit(n=9, layers=layers)
    want = oracle_full(oracle, c)
    hub = ThreadTransport()
    g = world.bit_length() - 1

    def rank_fn(r):
        st = ShardedState(c.n, world, r, OracleBackend(c.n - g, oracle), hub.endpoint(r), chunk_elems=16)
        run_ops(st, circuit_ops(c))
        return st, st.local_numpy()

    outs = run_ranks(world, rank_fn)
    assert np.abs(gather([o[0] for o in outs], [o[1] for o in outs]) - want).max() < 1e-12
    for st, _ in outs:
        s = st.exchange_stats()
        assert 1 <= s["remaps"] <= layers + 1 and s["qubits"] <= g * (layers + 1)
        shard = 16 << (c.n - g)
        assert s["bytes_sent"] <= s["remaps"] * shard * (world - 1) // world


class _ScheduleOnlyBackend:
    """No amplitudes: records the local batches the scheduler hands over."""

    def __init__(self, n_local):
        self.n = n_local
        self.batches = []

    def set_basis(self, index):
        pass

    def run(self, ops):
        self.batches.append(len(ops))

    def sync(self):
        pass


class _CountingTransport:
    def swap_blocks(self, backend, k, pairs, chunk):
        pass


@pytest.mark.parametrize("world", [2, 4, 8])
def test_c4_n32_schedule_one_remap(world):
    """BASELINE configs[3] sharded (host only, no amplitudes): the cone the scheduler runs before
    its first exchange leaves the ring qubits far from the global ones finished, and the remap
    evicts THOSE (latest next use), so the whole 10-layer circuit costs one remap -- (2^g - 1)/2^g
    of a shard on the wire -- and two local batches.  (Evicting the top local qubits, which the
    next layer needs, cost 10 remaps and 5 / 7 / 7.9 shards at 2 / 4 / 8 ranks.)"""
    from paper_2411_15332_b200 import configs
    from paper_2411_15332_b200.partition import ShardedState
    c = configs.c4_circuit(32)
    g = world.bit_length() - 1
    be = _ScheduleOnlyBackend(c.n - g)
    st = ShardedState(c.n, world, 0, be, _CountingTransport(), initial=c.initial)
    st.run(circuit_ops(c))
    st.flush()
    s = st.exchange_stats()
    shard = 16 << (c.n - g)
    assert s["remaps"] == 1 and s["qubits"] == g
    assert s["bytes_sent"] == shard * (world - 1) // world
    assert len(be.batches) == 2 and sum(be.batches) <= 992 + 32 + g  # the gates (H^n as 32) + the local swaps


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("name", ["c4", "c5", "grover"])
def test_threads_peer_remap_match_full_state(oracle, world, name):
    """Remaps over mapped partner shards (the CPU model of qcs_swap_peer: each rank of a pair
    swaps one half of the block pair between two barriers)."""
    from paper_2411_15332_b200.partition import ShardedState
    c = circuits()[name]
    want = oracle_full(oracle, c)
    hub = ThreadTransport(world, peers=True)
    g = world.bit_length() - 1

    def rank_fn(r):
        st = ShardedState(c.n, world, r, OracleBackend(c.n - g, oracle), hub.endpoint(r), initial=c.initial)
        assert st.peer and st.mode == "remap"
        run_ops(st, circuit_ops(c))
        return st, st.local_numpy()

    outs = run_ranks(world, rank_fn)
    assert np.abs(gather([o[0] for o in outs], [o[1] for o in outs]) - want).max() < 1e-12
    assert all(o[0].swaps > 0 and o[0].splits == 0 for o in outs)


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("name", ["c4", "c5", "grover", "c1"])
def test_threads_peer_gates_match_full_state(oracle, world, name):
    """Split mode: gates mixing only a global qubit run over the partner shard (the CPU model of
    qcs_apply_split), everything else through remaps."""
    from paper_2411_15332_b200.partition import ShardedState
    c = circuits()[name]
    want = oracle_full(oracle, c)
    hub = ThreadTransport(world, peers=True)
    g = world.bit_length() - 1

    def rank_fn(r):
        st = ShardedState(c.n, world, r, OracleBackend(c.n - g, oracle), hub.endpoint(r), initial=c.initial,
                          chunk_elems=7, mode="split")
        assert st.peer
        run_ops(st, circuit_ops(c))
        return st, st.local_numpy()

    outs = run_ranks(world, rank_fn)
    got = gather([o[0] for o in outs], [o[1] for o in outs])
    assert np.abs(got - want).max() < 1e-12
    if name in ("c4", "grover"):  # H / RY on global qubits: no exchange at all
        assert all(o[0].swaps == 0 and o[0].splits > 0 for o in outs)


def test_split_blocks_for_controlled_gates(oracle):
    """CNOT / Toffoli with local controls and a global target, CNOT with a global control
    (identity blocks on half the ranks), a global-target Swap (two mixing qubits: swap path)."""
    from paper_2411_15332_b200 import qcsim as Q
    from paper_2411_15332_b200.partition import ShardedState
    n, world = 7, 4
    rng = np.random.default_rng(3)
    G = Q.gate_catalog_lookup
    steps = [Q.hadamard_all(n),
             Q.CircuitStep.of_gates([Q.Placement(G("RY", [0.3]), 4)]),
             Q.CircuitStep.of_gates([Q.Placement(G("CNOT"), qubits=[5, 0])]),
             Q.CircuitStep.of_gates([Q.Placement(G("Toffoli"), qubits=[6, 3, 1])]),
             Q.CircuitStep.of_gates([Q.Placement(G("CNOT"), qubits=[1, 0])]),
             Q.CircuitStep.of_gates([Q.Placement(G("U", [float(x) for x in rng.uniform(0, 6, 3)]), 1)]),
             Q.CircuitStep.of_gates([Q.Placement(G("Swap"), qubits=[0, 5])]),
             Q.CircuitStep.of_gates([Q.Placement(G("RX", [1.1]), 0)])]
    c = Q.Circuit(n, steps)
    want = oracle_full(oracle, c)
    hub = ThreadTransport(world, peers=True)

    def rank_fn(r):
        st = ShardedState(n, world, r, OracleBackend(n - 2, oracle), hub.endpoint(r), chunk_elems=3, mode="split")
        run_ops(st, circuit_ops(c))
        return st, st.local_numpy()

    outs = run_ranks(world, rank_fn)
    assert np.abs(gather([o[0] for o in outs], [o[1] for o in outs]) - want).max() < 1e-12
    assert all(o[0].splits >= 3 and o[0].swaps >= 1 for o in outs)


def test_global_controls_and_diagonals_need_no_exchange(oracle):
    from paper_2411_15332_b200 import qcsim as Q
    from paper_2411_15332_b200.partition import ShardedState
    n, world = 6, 4
    c = Q.Circuit(n, [Q.hadamard_all(n),
                      Q.CircuitStep.of_gates([Q.Placement(Q.gate_catalog_lookup("CZ"), qubits=[0, 4])]),
                      Q.CircuitStep.of_gates([Q.Placement(Q.gate_catalog_lookup("CNOT"), qubits=[1, 5])]),
                      Q.CircuitStep.of_gates([Q.Placement(Q.gate_catalog_lookup("RZ", [0.7]), 0)]),
                      Q.CircuitStep.of_gates([Q.Placement(Q.gate_catalog_lookup("Toffoli"), qubits=[0, 1, 3])]),
                      Q.CircuitStep.of_diag(Q.DiagSign([5, 40], False))])
    want = oracle_full(oracle, c)
    hub = ThreadTransport()
    ops = circuit_ops(c)
    ops[0] = ("rh_local_only",)

    def rank_fn(r):
        st = ShardedState(n, world, r, OracleBackend(n - 2, oracle), hub.endpoint(r))
        # H on all qubits without moving qubits: local WHT + H on the two global qubits would
        # swap, so prepare the uniform state by hand instead
        st.backend.tensor.fill_(1.0 / np.sqrt(2 ** n))
        run_ops(st, ops[1:])
        return st, st.local_numpy()

    outs = run_ranks(world, rank_fn)
    assert all(o[0].swaps == 0 for o in outs)
    assert np.abs(gather([o[0] for o in outs], [o[1] for o in outs]) - want).max() < 1e-12


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, name, result_path):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle_py import Oracle
    from paper_2411_15332_b200.partition import DistTransport, ShardedState
    Oracle.lib()
    c = circuits()[name]
    g = world.bit_length() - 1
    st = ShardedState(c.n, world, rank, OracleBackend(c.n - g, Oracle), DistTransport(), initial=c.initial,
                      chunk_elems=5)
    run_ops(st, circuit_ops(c))
    loc = torch.from_numpy(st.local_numpy())
    amap = torch.from_numpy(st.logical_amplitude_map())
    if rank == 0:
        locs = [torch.zeros_like(loc) for _ in range(world)]
        maps = [torch.zeros_like(amap) for _ in range(world)]
    else:
        locs = maps = None
    dist.gather(torch.view_as_real(loc), [torch.view_as_real(x) for x in locs] if locs else None, dst=0)
    dist.gather(amap, maps, dst=0)
    if rank == 0:
        full = np.zeros(1 << c.n, dtype=np.complex128)
        for lo, mp_ in zip(locs, maps):
            full[mp_.numpy()] = lo.numpy()
        np.save(result_path, full)
    dist.destroy_process_group()


@pytest.mark.parametrize("world,name", [(2, "c5"), (4, "c4"), (2, "grover")])
def test_gloo_ranks_match_full_state(oracle, tmp_path, world, name):
    path = str(tmp_path / "full.npy")
    mp.start_processes(_gloo_worker, args=(world, _free_port(), name, path), nprocs=world, join=True,
                       start_method="spawn")
    want = oracle_full(oracle, circuits()[name])
    assert np.abs(np.load(path) - want).max() < 1e-12


class _SharedPeerTransport:
    """gloo processes whose shards live in shared memory: peer_buffer maps the partner's shard
    (the CPU stand-in for NVLink peer memory), barrier is the gloo barrier."""

    def __init__(self, shards):
        from paper_2411_15332_b200.partition import DistTransport
        self.inner = DistTransport()
        self.shards = shards

    def exchange(self, send, recv, peer):
        self.inner.exchange(send, recv, peer)

    def peer_buffer(self, peer):
        return self.shards[peer]

    def barrier(self):
        dist.barrier()


def _gloo_peer_worker(rank, world, port, name, shards, result_path, mode):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle_py import Oracle
    from paper_2411_15332_b200.partition import ShardedState
    Oracle.lib()
    c = circuits()[name]
    g = world.bit_length() - 1
    backend = OracleBackend(c.n - g, Oracle)
    backend.tensor = shards[rank]  # this rank's shard is the shared one the partners map
    st = ShardedState(c.n, world, rank, backend, _SharedPeerTransport(shards), initial=c.initial, chunk_elems=5,
                      mode=mode)
    assert st.peer
    run_ops(st, circuit_ops(c))
    st.flush()
    dist.barrier()
    amap = torch.from_numpy(st.logical_amplitude_map())
    maps = [torch.zeros_like(amap) for _ in range(world)] if rank == 0 else None
    dist.gather(amap, maps, dst=0)
    if rank == 0:
        full = np.zeros(1 << c.n, dtype=np.complex128)
        for r, mp_ in enumerate(maps):
            full[mp_.numpy()] = shards[r].numpy()
        np.save(result_path, np.array([full, st.splits, st.swaps], dtype=object), allow_pickle=True)
    dist.destroy_process_group()


@pytest.mark.parametrize("world,name,mode", [(2, "c4", "split"), (4, "grover", "split"), (2, "c5", "split"),
                                            (4, "c4", "remap"), (4, "c5", "remap")])
def test_gloo_peer_mode_match_full_state(oracle, tmp_path, world, name, mode):
    """World 2 / 4 processes over gloo with the partner shards mapped (through shared memory
    here, NVLink on the GPU box): split mode runs gates mixing one global qubit on the partner's
    shard; remap mode swaps remap blocks over the mapping (qcs_swap_peer's contract)."""
    c = circuits()[name]
    g = world.bit_length() - 1
    shards = [torch.zeros(1 << (c.n - g), dtype=torch.complex128).share_memory_() for _ in range(world)]
    path = str(tmp_path / "full.npy")
    mp.start_processes(_gloo_peer_worker, args=(world, _free_port(), name, shards, path, mode), nprocs=world,
                       join=True, start_method="spawn")
    full, splits, swaps = np.load(path, allow_pickle=True)
    assert np.abs(full - oracle_full(oracle, c)).max() < 1e-12
    assert (splits > 0) if mode == "split" else (swaps > 0 and splits == 0)
