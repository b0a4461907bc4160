"""State-vector partitioner over P = 2^g ranks (BASELINE north star item 5).

Rank r holds the 2^(n-g) amplitudes whose top g basis bits equal r, i.e. whose *physical*
qubits 0..g-1 (qubit 0 is the most significant bit, core.hpp:64-66) spell r.  A logical-to-
physical qubit map lets qubits move between the global and the local part lazily:

* a gate whose matrix does not mix values of its global qubits (diagonal gates, controls on
  global qubits, the C4 CZ ring) is reduced to the block selected by the rank's global bits and
  applied locally -- no communication;
* a gate that mixes exactly one qubit, a global one (H, RX, RY, U3, X, Y on a global qubit;
  CNOT / Toffoli with local controls and a global target), runs as one kernel over peer
  memory when the transport maps the partner shard (``peer_buffer``): each rank takes half of
  the amplitude pairs, loads the partner's amplitude over NVLink and stores both outputs
  (qcs_apply_split) -- the exchange and the arithmetic are fused, nothing is staged;
* any other gate touching a global qubit first swaps that qubit with the most significant
  local qubit: the ranks r and r ^ bit exchange one contiguous half of their shards (pairwise
  send/recv, chunked through a bounded staging buffer), the map records the swap, and the gate
  then runs locally;
* H on all qubits (the RH step) is a local Walsh-Hadamard transform over the local qubits plus
  one H per global qubit (each after its swap);
* diagonal sign steps (Grover oracle / Z0) translate their basis indices through the map; each
  rank negates the ones it owns (or all but those).

Communication uses torch.distributed point-to-point operations (NCCL over NVLink on the GPU
box; gloo in the CPU tests) for the swaps, and peer loads/stores (torch symmetric memory,
``SymmetricTransport``) for the fused gates.  Local compute goes through a backend: ``DeviceBackend`` runs the
B200 kernels through the C ABI on a torch-owned device shard (``qcs_state_wrap``); the tests
plug in CPU backends.  Nothing here touches amplitudes on the host in the device path.
"""
from __future__ import annotations

import math
from typing import List, Optional, Sequence

import numpy as np


def _bits(x: int, n: int) -> List[int]:
    return [(x >> (n - 1 - q)) & 1 for q in range(n)]


class DeviceBackend:
    """A local shard of n_local qubits in a torch CUDA tensor, updated by libqcs_b200 kernels."""

    def __init__(self, n_local: int, device: int = 0, symmetric: bool = False):
        import torch

        from . import qcsim as Q
        self.torch = torch
        self.Q = Q
        self.n = n_local
        self.device = device
        if symmetric:  # peer-mappable (torch symmetric memory): SymmetricTransport rendezvous
            import torch.distributed._symmetric_memory as symm_mem
            self.tensor = symm_mem.empty(1 << n_local, dtype=torch.complex128, device=f"cuda:{device}")
            self.tensor.zero_()
        else:
            self.tensor = torch.zeros(1 << n_local, dtype=torch.complex128, device=f"cuda:{device}")
        stream = torch.cuda.current_stream(device).cuda_stream
        import ctypes as C
        h = C.c_void_p()
        Q._check(Q.L.lib().qcs_state_wrap(n_local, device, C.c_void_p(self.tensor.data_ptr()), C.c_void_p(stream),
                                          C.byref(h)))
        self.state = Q.DeviceState(n_local, 0, device, _handle=h)

    def set_basis(self, index: Optional[int]) -> None:
        self.tensor.zero_()
        if index is not None:
            self.tensor[index] = 1.0

    def apply(self, matrix: np.ndarray, local_qubits: Sequence[int], name: str = "custom") -> None:
        self.state.apply_gate(self.Q.custom_gate(matrix, name), list(local_qubits))

    def apply_diag(self, flipped: Sequence[int], flip_rest: bool) -> None:
        self.state.apply_diag(self.Q.DiagSign(list(flipped), flip_rest))

    def apply_rh(self) -> None:
        self.state.apply_rh()

    def run(self, ops) -> None:
        """Apply a batch of local operations with one fused qcs_simulate call."""
        Q = self.Q
        steps = []
        for op in ops:
            if op[0] == "gate":
                steps.append(Q.CircuitStep.of_gates([Q.Placement(Q.custom_gate(op[1], op[3]), qubits=list(op[2]))]))
            elif op[0] == "diag":
                steps.append(Q.CircuitStep.of_diag(Q.DiagSign(list(op[1]), op[2])))
            else:
                steps.append(Q.hadamard_all(self.n))
        if steps:
            Q.run(Q.Circuit(self.n, steps), self.state, Q.Engine.rh_dax)

    def apply_split(self, peer, self_bit: int, sel_bits: Sequence[int], blocks: np.ndarray, skip: int) -> None:
        """A gate on a global qubit, fused with the exchange: `peer` is the partner shard
        (a tensor in this device's address space)."""
        self.state.apply_split(peer.data_ptr(), self_bit, sel_bits, blocks, skip)

    def half(self, upper: bool):
        h = 1 << (self.n - 1)
        return self.tensor[h:] if upper else self.tensor[:h]

    def chunk(self, upper: bool, start: int, count: int):
        base = (1 << (self.n - 1)) if upper else 0
        return self.tensor[base + start: base + start + count]

    def empty(self, count: int):
        return self.torch.empty(count, dtype=self.torch.complex128, device=self.tensor.device)

    def sync(self) -> None:
        self.torch.cuda.synchronize(self.device)

    def numpy(self) -> np.ndarray:
        self.sync()
        return self.tensor.cpu().numpy()


class DistTransport:
    """Pairwise exchange over torch.distributed (NCCL or gloo)."""

    def __init__(self):
        import torch.distributed as dist
        self.dist = dist

    def exchange(self, send, recv, peer: int) -> None:
        import torch
        s = torch.view_as_real(send) if send.is_complex() else send
        r = torch.view_as_real(recv) if recv.is_complex() else recv
        ops = [self.dist.P2POp(self.dist.isend, s, peer), self.dist.P2POp(self.dist.irecv, r, peer)]
        for req in self.dist.batch_isend_irecv(ops):
            req.wait()


class SymmetricTransport(DistTransport):
    """DistTransport plus the partner shards mapped over NVLink (torch symmetric memory): the
    fused global-qubit gates load and store them directly.  The backend must be a
    DeviceBackend(..., symmetric=True); `attach` is collective."""

    def attach(self, backend) -> None:
        import torch.distributed._symmetric_memory as symm_mem
        self.backend = backend
        self.handle = symm_mem.rendezvous(backend.tensor, self.dist.group.WORLD)

    def peer_buffer(self, peer: int):
        import torch
        return self.handle.get_buffer(peer, (self.backend.tensor.numel(),), torch.complex128)

    def barrier(self) -> None:
        self.handle.barrier(channel=0)  # stream-ordered: orders the GPU work on every rank


class ShardedState:
    """An n-qubit state sharded over `world` ranks (a power of two); this object is rank `rank`."""

    def __init__(self, n: int, world: int, rank: int, backend, transport=None, initial: int = 0,
                 chunk_elems: int = 1 << 24, peer: Optional[bool] = None):
        g = int(round(math.log2(world)))
        if 1 << g != world:
            raise ValueError("world size must be a power of two")
        if n - g < 1:
            raise ValueError("each shard needs at least one local qubit")
        self.n, self.g, self.world, self.rank = n, g, world, rank
        self.backend = backend
        self.transport = transport
        self.chunk = chunk_elems
        self.phys = list(range(n))  # phys[logical qubit] = physical qubit
        self.swaps = 0              # global<->local exchanges performed
        self.exchanged_bytes = 0    # bytes sent by this rank
        self.pending = []           # local operations not yet handed to the backend
        self.splits = 0             # gates run over peer memory (no exchange)
        can_peer = (transport is not None and hasattr(transport, "peer_buffer") and hasattr(transport, "barrier")
                    and hasattr(backend, "apply_split"))
        self.peer = can_peer if peer is None else (bool(peer) and can_peer)
        if self.peer and hasattr(transport, "attach"):
            transport.attach(backend)
        self.set_basis(initial)

    # ------------------------------------------------------------ index mapping
    def _to_phys_index(self, logical_index: int) -> int:
        lb = _bits(logical_index, self.n)
        p = 0
        for q in range(self.n):
            if lb[q]:
                p |= 1 << (self.n - 1 - self.phys[q])
        return p

    def _owner(self, phys_index: int):
        nl = self.n - self.g
        return phys_index >> nl, phys_index & ((1 << nl) - 1)

    def _rank_bit(self, phys_qubit: int) -> int:
        """Value of global physical qubit `phys_qubit` (< g) on this rank."""
        return (self.rank >> (self.g - 1 - phys_qubit)) & 1

    # ------------------------------------------------------------ local work, batched
    def _local(self, op) -> None:
        self.pending.append(op)

    def flush(self) -> None:
        """Hand the pending local operations to the backend (one fused launch sequence)."""
        if not self.pending:
            return
        ops, self.pending = self.pending, []
        if hasattr(self.backend, "run"):
            self.backend.run(ops)
            return
        for op in ops:
            if op[0] == "gate":
                self.backend.apply(op[1], op[2], op[3])
            elif op[0] == "diag":
                self.backend.apply_diag(op[1], op[2])
            else:
                self.backend.apply_rh()

    def set_basis(self, logical_index: int) -> None:
        self.pending = []
        owner, local = self._owner(self._to_phys_index(logical_index))
        self.backend.set_basis(local if owner == self.rank else None)

    # ------------------------------------------------------------ exchange
    def _swap_global_local(self, gq: int, lq: int) -> None:
        """Swap physical global qubit gq with physical local qubit lq == g (the top local bit):
        ranks r and r ^ bit exchange their halves whose top local bit differs from their own
        global bit; the amplitude (global = a, local = b) moves to (global = b, local = a)."""
        assert gq < self.g and lq == self.g
        self.flush()
        if self.world > 1:
            a = self._rank_bit(gq)
            peer = self.rank ^ (1 << (self.g - 1 - gq))
            half = 1 << (self.n - self.g - 1)
            upper = a == 0  # I send (and receive into) my half with local bit 1 - a
            tmp = self.backend.empty(min(self.chunk, half))
            for start in range(0, half, self.chunk):
                cnt = min(self.chunk, half - start)
                mine = self.backend.chunk(upper, start, cnt)
                recv = tmp[:cnt]
                self.backend.sync()
                self.transport.exchange(mine, recv, peer)
                mine.copy_(recv)
                self.exchanged_bytes += 16 * cnt
            self.swaps += 1
        # logical qubits at physical gq and lq trade places
        qa = self.phys.index(gq)
        qb = self.phys.index(lq)
        self.phys[qa], self.phys[qb] = lq, gq

    # ------------------------------------------------------------ operations
    def apply_gate(self, matrix: np.ndarray, logical_qubits: Sequence[int], name: str = "custom") -> None:
        """One placement (gate-local order: local index bit k-1-i <-> logical_qubits[i])."""
        m = np.asarray(matrix, dtype=np.complex128)
        k = len(logical_qubits)
        phys = [self.phys[q] for q in logical_qubits]
        glob = [i for i, p in enumerate(phys) if p < self.g]
        if glob:
            # does the gate keep every global qubit's value (block diagonal in them)?
            r_idx, c_idx = np.nonzero(m)
            gmask = sum(1 << (k - 1 - i) for i in glob)
            if np.all((r_idx & gmask) == (c_idx & gmask)):
                want = sum(self._rank_bit(phys[i]) << (k - 1 - i) for i in glob)
                loc = [i for i in range(k) if i not in glob]
                if not loc:  # all qubits global: a scalar phase on this rank's shard
                    d = m[want, want]
                    if d != 1:
                        self._local(("gate", np.array([[d, 0], [0, d]]), [0], name))  # phase on any qubit
                    return
                sel = [want | sum(((j >> (len(loc) - 1 - t)) & 1) << (k - 1 - loc[t]) for t in range(len(loc)))
                       for j in range(1 << len(loc))]
                sub = m[np.ix_(sel, sel)]
                self._local(("gate", sub, [phys[i] - self.g for i in loc], name))
                return
            if self.peer and self._split_gate(m, phys, name):
                return
            # bring each mixing global qubit local (swap with the top local qubit, which must
            # not be one of this gate's own qubits: move it aside first if needed)
            for i in glob:
                if self.phys[logical_qubits[i]] >= self.g:
                    continue
                top = self.g
                if top in [self.phys[q] for q in logical_qubits]:
                    # the top local qubit carries one of our targets: exchange it with a free
                    # local qubit (a local SWAP gate) before bringing the global qubit down
                    used = {self.phys[q] for q in logical_qubits}
                    free = next(p for p in range(self.g + 1, self.n) if p not in used)
                    self._local_swap(top, free)
                self._swap_global_local(self.phys[logical_qubits[i]], top)
            phys = [self.phys[q] for q in logical_qubits]
        self._local(("gate", m, [p - self.g for p in phys], name))

    def _split_gate(self, m: np.ndarray, phys: List[int], name: str) -> bool:
        """The gate mixes exactly one of its qubits and that one is global: run it over peer
        memory (qcs_apply_split).  Its other qubits only select 2x2 blocks -- global ones by
        this rank's bits, local ones (<= 2) per amplitude.  False: not of that form."""
        k = len(phys)
        r_idx, c_idx = np.nonzero(m)
        mixing = [i for i in range(k) if np.any(((r_idx ^ c_idx) >> (k - 1 - i)) & 1)]
        if len(mixing) != 1 or phys[mixing[0]] >= self.g:
            return False
        ig = mixing[0]
        sel = [i for i in range(k) if i != ig and phys[i] >= self.g]
        if len(sel) > 2:
            return False
        fixed = sum(self._rank_bit(phys[i]) << (k - 1 - i) for i in range(k) if i != ig and phys[i] < self.g)
        nl = self.n - self.g
        sel_bits = [nl - 1 - (phys[i] - self.g) for i in sel]
        nb = 1 << len(sel)
        blocks = np.zeros((nb, 2, 2), dtype=np.complex128)
        skip = 0
        for v in range(nb):
            base = fixed | sum(((v >> (len(sel) - 1 - t)) & 1) << (k - 1 - sel[t]) for t in range(len(sel)))
            idx = [base, base | (1 << (k - 1 - ig))]
            blocks[v] = m[np.ix_(idx, idx)]
            if np.array_equal(blocks[v], np.eye(2)):
                skip |= 1 << v
        # every rank takes part in both barriers (they are world-wide); a rank pair whose blocks
        # are all the identity (a global control that is off) launches nothing
        self.flush()
        self.transport.barrier()  # the partner's earlier work on its shard is done
        if skip != (1 << nb) - 1:
            self.backend.apply_split(self.transport.peer_buffer(self.rank ^ (1 << (self.g - 1 - phys[ig]))),
                                     self._rank_bit(phys[ig]), sel_bits, blocks, skip)
            self.splits += 1
        self.transport.barrier()  # ... and ours before either shard is used again
        return True

    def _local_swap(self, pa: int, pb: int) -> None:
        swap = np.eye(4, dtype=np.complex128)[[0, 2, 1, 3]]
        self._local(("gate", swap, [pa - self.g, pb - self.g], "Swap"))
        qa, qb = self.phys.index(pa), self.phys.index(pb)
        self.phys[qa], self.phys[qb] = pb, pa

    def apply_step(self, placements) -> None:
        """placements: [(matrix, logical_qubits, name), ...] with disjoint qubits."""
        for m, qs, name in placements:
            self.apply_gate(m, qs, name)

    def apply_diag(self, flipped: Sequence[int], flip_rest: bool) -> None:
        mine = []
        for x in flipped:
            owner, local = self._owner(self._to_phys_index(int(x)))
            if owner == self.rank:
                mine.append(local)
        if mine or flip_rest:
            self._local(("diag", sorted(set(mine)), flip_rest))

    def apply_rh(self) -> None:
        """H on all n qubits: local WHT over the local qubits, then one H per global qubit."""
        self._local(("rh",))
        if self.g:
            h = np.array([[1, 1], [1, -1]], dtype=np.complex128) / math.sqrt(2.0)
            for q in [q for q in range(self.n) if self.phys[q] < self.g]:
                self.apply_gate(h, [q], "Hadamard")

    # ------------------------------------------------------------ inspection
    def local_numpy(self) -> np.ndarray:
        self.flush()
        return self.backend.numpy()

    def logical_amplitude_map(self):
        """(logical index for each local index of this shard) -- for gathering in tests."""
        nl = self.n - self.g
        inv = [0] * self.n  # inv[physical] = logical
        for q, p in enumerate(self.phys):
            inv[p] = q
        out = np.empty(1 << nl, dtype=np.int64)
        for local in range(1 << nl):
            phys = (self.rank << nl) | local
            pb = _bits(phys, self.n)
            li = 0
            for p in range(self.n):
                if pb[p]:
                    li |= 1 << (self.n - 1 - inv[p])
            out[local] = li
        return out
