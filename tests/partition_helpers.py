"""Test-side pieces for the partitioner: a CPU shard backend (the oracle does the local compute:
tests may use it) and an in-process transport that lets P threads stand in for P ranks."""
import threading

import numpy as np
import torch


class OracleBackend:
    """Local shard as a CPU complex128 tensor; local steps through the C oracle."""

    def __init__(self, n_local, oracle):
        self.n = n_local
        self.O = oracle
        self.tensor = torch.zeros(1 << n_local, dtype=torch.complex128)

    def set_basis(self, index):
        self.tensor.zero_()
        if index is not None:
            self.tensor[index] = 1.0

    def _set(self, arr):
        self.tensor.copy_(torch.from_numpy(arr))

    def apply(self, matrix, local_qubits, name="custom"):
        self._set(self.O.apply_step(self.n, [(list(local_qubits), np.asarray(matrix))], self.tensor.numpy()))

    def apply_diag(self, flipped, flip_rest):
        self._set(self.O.apply_diag(self.n, flipped, flip_rest, self.tensor.numpy()))

    def apply_rh(self):
        self._set(self.O.wht(self.n, self.tensor.numpy()))

    def block(self, k, j, start, count):
        b = (1 << (self.n - k)) * j + start
        return self.tensor[b: b + count]

    def swap_peer(self, offset, peer_block, count):
        """qcs_swap_peer's contract on the CPU."""
        mine = self.tensor[offset: offset + count]
        tmp = mine.clone()
        mine.copy_(peer_block[:count])
        peer_block[:count].copy_(tmp)

    def apply_split(self, peer, self_bit, sel_bits, blocks, skip):
        """qcs_apply_split's contract on the CPU: this rank's half of the pairs, both outputs,
        dax_mvm order (acc = 0; += m[r][c] * x_c over the nonzero entries, ascending c)."""
        half = 1 << (self.n - 1)
        mine, other = self.tensor.numpy(), peer.numpy()
        for j in range(half):
            i = (half if self_bit else 0) | j
            v = 0
            for b in sel_bits:
                v = (v << 1) | ((i >> b) & 1)
            if skip >> v & 1:
                continue
            x = (other[i], mine[i]) if self_bit else (mine[i], other[i])
            out = []
            for r in range(2):
                acc = 0j
                for c in range(2):
                    if blocks[v][r][c] != 0:
                        acc = acc + blocks[v][r][c] * x[c]
                out.append(acc)
            mine[i], other[i] = (out[1], out[0]) if self_bit else (out[0], out[1])

    def empty(self, count):
        return torch.empty(count, dtype=torch.complex128)

    def sync(self):
        pass

    def numpy(self):
        return self.tensor.numpy().copy()


class ThreadTransport:
    """P threads in one process exchanging through mailboxes (an emulated fabric).  With
    peers=True the endpoints also map the other shards (peer_buffer) and share a barrier: the
    emulated NVLink of the fused global-qubit gates."""

    def __init__(self, world=None, peers=False):
        self.cv = threading.Condition()
        self.box = {}
        self.peers = peers
        self.backends = {}
        self.bar = threading.Barrier(world) if peers else None

    def endpoint(self, rank):
        return _PeerEndpoint(self, rank) if self.peers else _Endpoint(self, rank)


class _Endpoint:
    def __init__(self, hub, rank):
        self.hub, self.rank = hub, rank

    def exchange(self, send, recv, peer):
        with self.hub.cv:  # per-(source, destination) FIFO: messages are matched in order
            self.hub.box.setdefault((self.rank, peer), []).append(send.clone())
            self.hub.cv.notify_all()
            while not self.hub.box.get((peer, self.rank)):
                self.hub.cv.wait()
            data = self.hub.box[(peer, self.rank)].pop(0)
        recv.copy_(data)


class _PeerEndpoint(_Endpoint):
    def attach(self, backend):
        self.hub.backends[self.rank] = backend
        self.hub.bar.wait()

    def peer_buffer(self, peer):
        return self.hub.backends[peer].tensor

    def barrier(self):
        # GPU emulation: every rank's kernels go to the device's default stream, so a host
        # barrier after issuing orders them
        self.hub.bar.wait()


def run_ranks(world, fn):
    """Run fn(rank) in `world` threads; re-raise the first failure."""
    errs, outs = [None] * world, [None] * world

    def body(r):
        try:
            outs[r] = fn(r)
        except BaseException as e:  # noqa: BLE001
            errs[r] = e

    ths = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    for e in errs:
        if e is not None:
            raise e
    return outs


def gather(states, parts):
    """Assemble the logical state from every rank's (ShardedState, local amplitudes)."""
    n = states[0].n
    full = np.zeros(1 << n, dtype=np.complex128)
    for st, loc in zip(states, parts):
        full[st.logical_amplitude_map()] = loc
    return full


def circuit_ops(circuit):
    from paper_2411_15332_b200.partition import circuit_ops as ops
    return ops(circuit)


def run_ops(state, ops):
    """The whole list through the scheduler (reordering, batched remaps)."""
    state.run(ops)
    state.flush()


def run_ops_one_by_one(state, ops):
    """Immediate mode: one operation at a time (no reordering across operations)."""
    for op in ops:
        if op[0] == "gate":
            state.apply_gate(op[1], op[2], op[3])
        elif op[0] == "diag":
            state.apply_diag(op[1], op[2])
        else:
            state.apply_rh()


def oracle_full(oracle, circuit):
    x = np.zeros(1 << circuit.n, dtype=np.complex128)
    x[circuit.initial] = 1
    for st in circuit.steps:
        if int(st.kind) == 1:
            x = oracle.apply_diag(circuit.n, st.diag.flipped, st.diag.flip_rest, x)
        elif st.is_hadamard_all(circuit.n):
            x = oracle.wht(circuit.n, x)
        else:
            x = oracle.apply_step(circuit.n, [(p.qubit_list(), p.gate.matrix) for p in st.placements], x)
    return x
