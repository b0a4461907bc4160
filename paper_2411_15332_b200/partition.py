"""State-vector partitioner over P = 2^g ranks (BASELINE north star item 5).

Rank r holds the 2^(n-g) amplitudes whose top g basis bits equal r.  Those are the *physical*
qubits 0..g-1 (qubit 0 is the most significant bit, core.hpp:64-66).  A logical-to-physical
qubit map lets qubits move between the global and the local part lazily.

``run(ops)`` schedules a whole operation list:

* Block reduction.  An operation that does not mix the values of its global qubits runs
  locally.  This covers diagonal gates, controls on global qubits and the C4 CZ ring.  Its
  matrix is reduced to the block this rank's global bits select, so it needs no communication.
* Reordering.  Operations whose qubits are disjoint commute, and so do diagonal operations.
  The scheduler runs every operation it can before it exchanges anything: a whole layer of
  local gates, then the gates waiting on global qubits.
* Batched remap.  When only operations that mix global qubits are left, one remap brings ALL
  the global qubits they need down at once.  The top k local physical qubits go up in exchange.
  It is an all-to-all among the 2^k ranks that differ in those global bits: rank r swaps its
  block j (top local bits = j) with block a of the rank whose global bits are j, where a is r's
  own value of those bits.  Per remap each rank moves (2^k - 1)/2^k of its shard.  Doing one
  qubit at a time would move half a shard per qubit, and qubits would shuttle back and forth.
  - DistTransport: grouped send/recv to all 2^k - 1 partners per chunk (NCCL over NVLink on
    the GPU box, gloo in the CPU tests).  It is double-buffered: a copy stream writes chunk c
    into place while chunk c+1 is on the wire.  There is no host synchronisation.
  - SymmetricTransport: the partner shards are mapped over NVLink (torch symmetric memory).
    Each rank of a pair runs the swap kernel on one half of the block pair (qcs_swap_peer):
    nothing is staged, and every amplitude crosses the link once each way.
* mode="split" is the alternative for peer transports.  A gate that mixes exactly one qubit,
  a global one, runs as one kernel over the partner's shard (qcs_apply_split).  Everything else
  still remaps.
* Diagonal sign steps (the Grover oracle, Z0) translate their basis indices through the map.
  Each rank negates the indices it owns (or all but those).

Local compute goes through a backend.  ``DeviceBackend`` runs the B200 kernels through the C ABI
on a torch-owned device shard (``qcs_state_wrap``).  It flushes queued local operations as one
fused ``qcs_simulate`` call.  The tests plug in CPU backends.  Nothing here touches amplitudes
on the host in the device path.
"""
from __future__ import annotations

import math
import os
import time
from typing import List, Optional, Sequence

import numpy as np

_H = np.array([[1, 1], [1, -1]], dtype=np.complex128) / math.sqrt(2.0)


def _bits(x: int, n: int) -> List[int]:
    return [(x >> (n - 1 - q)) & 1 for q in range(n)]


def circuit_ops(circuit):
    """Circuit -> flat op list: ('gate', m, qubits, name) / ('diag', flipped, flip_rest) / ('rh',)."""
    ops = []
    for st in circuit.steps:
        if int(st.kind) == 1:
            ops.append(("diag", list(st.diag.flipped), st.diag.flip_rest))
        elif st.is_hadamard_all(circuit.n):
            ops.append(("rh",))
        else:
            for p in st.placements:
                ops.append(("gate", p.gate.matrix, p.qubit_list(), p.gate.name))
    return ops


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
            self._tensor = symm_mem.empty(1 << n_local, dtype=torch.complex128, device=f"cuda:{device}")
            self._tensor.zero_()
        else:
            self._tensor = torch.zeros(1 << n_local, dtype=torch.complex128, device=f"cuda:{device}")
        stream = torch.cuda.current_stream(device).cuda_stream
        import ctypes as C
        h = C.c_void_p()
        Q._check(Q.L.lib().qcs_state_wrap(n_local, device, C.c_void_p(self._tensor.data_ptr()), C.c_void_p(stream),
                                          C.byref(h)))
        self.state = Q.DeviceState(n_local, 0, device, _handle=h)

    @property
    def tensor(self):
        """The shard as a torch tensor, for readers and writers outside this class: a deferred
        reset is written first, and the shard's content is no longer taken as known."""
        self._materialise()
        self.known = None
        return self._tensor

    def set_basis(self, index: Optional[int]) -> None:
        # what the shard holds, until something else writes it: the next batch starts from it.
        # The memory is written only when someone needs it (_materialise): a batch that starts
        # from a basis state folds the reset into its first pass and never reads the old content.
        self.known = "zero" if index is None else int(index)
        self.stale = True

    def _materialise(self) -> None:
        if getattr(self, "stale", False):
            self.stale = False
            self._tensor.zero_()
            if isinstance(self.known, int):
                self._tensor[self.known] = 1.0

    def run(self, ops) -> None:
        """Apply a batch of local operations with one fused qcs_simulate call.  A run of
        Hadamards covering every local qubit becomes the RH step (butterflies, one scale).
        A shard known to be a basis state runs the batch with the reset folded in (the passes
        skip the tiles outside the support reached so far, as the single-GPU simulate does); a
        shard known to be all zeros stays all zeros under these linear operations: nothing runs."""
        Q = self.Q
        known, self.known = getattr(self, "known", None), None
        if known == "zero":
            self.known = "zero"
            return
        steps = []
        hs = []

        def flush_h():
            if len(hs) == self.n and len({q for q in hs}) == self.n:
                steps.append(Q.hadamard_all(self.n))
            else:
                h = Q.gate_catalog_lookup("Hadamard")
                steps.extend(Q.CircuitStep.of_gates([Q.Placement(h, qubits=[q])]) for q in hs)
            hs.clear()
        for op in ops:
            if op[0] == "gate" and op[3] == "Hadamard" and len(op[2]) == 1 and op[2][0] not in hs:
                hs.append(op[2][0])
                continue
            if hs:
                flush_h()
            if op[0] == "gate":
                steps.append(Q.CircuitStep.of_gates([Q.Placement(Q.custom_gate(op[1], op[3]), qubits=list(op[2]))]))
            elif op[0] == "diag":
                steps.append(Q.CircuitStep.of_diag(Q.DiagSign(list(op[1]), op[2])))
            else:
                steps.append(Q.hadamard_all(self.n))
        if hs:
            flush_h()
        if steps:
            if isinstance(known, int):
                self.stale = False  # the run writes |known> itself
            else:
                self._materialise()
            Q.run(Q.Circuit(self.n, steps), self.state, Q.Engine.rh_dax,
                  reset_index=known if isinstance(known, int) else None)
        else:
            self.known = known

    def apply_split(self, peer, self_bit: int, sel_bits: Sequence[int], blocks: np.ndarray, skip: int) -> None:
        """A gate on a global qubit, fused with the exchange: `peer` is the partner shard
        (a tensor in this device's address space)."""
        self._materialise()
        self.known = None
        self.state.apply_split(peer.data_ptr(), self_bit, sel_bits, blocks, skip)

    def swap_peer(self, offset: int, peer_block, count: int) -> None:
        """Swap this shard's [offset, offset+count) with `peer_block` (qcs_swap_peer)."""
        Q = self.Q
        import ctypes as C
        self._materialise()
        self.known = None
        Q._check(Q.L.lib().qcs_swap_peer(self.state.handle, offset, C.c_void_p(peer_block.data_ptr()), count))

    def block(self, k: int, j: int, start: int, count: int):
        """Elements [start, start+count) of block j of 2^k (by the top k local bits)."""
        b = (1 << (self.n - k)) * j + start
        self._materialise()
        self.known = None  # a view the transports write through
        return self._tensor[b: b + count]

    def empty(self, count: int):
        return self.torch.empty(count, dtype=self.torch.complex128, device=self._tensor.device)

    def sync(self) -> None:
        self._materialise()
        self.torch.cuda.synchronize(self.device)

    def numpy(self) -> np.ndarray:
        self.sync()
        return self._tensor.cpu().numpy()


class DistTransport:
    """Exchanges over torch.distributed point-to-point operations (NCCL or gloo)."""

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

    def swap_blocks(self, backend, k: int, pairs, chunk: int) -> None:
        """pairs: [(peer, my_block, peer_block)]; my block j of 2^k is swapped in place with the
        partner's block (the partner makes the matching call).  One grouped send/recv to every
        partner per chunk; received chunks land in a staging slot and are copied into place on
        a side stream while the next chunk is on the wire (two slots)."""
        import torch
        if not pairs:
            return
        size = 1 << (backend.n - k)
        step = min(chunk, size)
        probe = backend.block(k, pairs[0][1], 0, 1)
        cuda = probe.is_cuda
        slots = [backend.empty(len(pairs) * step) for _ in range(2)]
        side = torch.cuda.Stream(probe.device) if cuda else None
        cur = torch.cuda.current_stream(probe.device) if cuda else None
        done = [None, None]
        for ci, start in enumerate(range(0, size, step)):
            cnt = min(step, size - start)
            slot = ci & 1
            if done[slot] is not None:
                cur.wait_event(done[slot])  # the slot's previous chunk has been copied out
            ops = []
            for b, (peer, mine, _theirs) in enumerate(pairs):
                src = backend.block(k, mine, start, cnt)
                dst = slots[slot][b * step: b * step + cnt]
                ops.append(self.dist.P2POp(self.dist.isend, torch.view_as_real(src), peer))
                ops.append(self.dist.P2POp(self.dist.irecv, torch.view_as_real(dst), peer))
            for req in self.dist.batch_isend_irecv(ops):
                req.wait()  # CUDA: the current stream waits for the transfers (the host does not)
            if cuda:
                ev = torch.cuda.Event()
                ev.record(cur)
                side.wait_event(ev)
                with torch.cuda.stream(side):
                    for b, (peer, mine, _theirs) in enumerate(pairs):
                        backend.block(k, mine, start, cnt).copy_(slots[slot][b * step: b * step + cnt])
                    done[slot] = torch.cuda.Event()
                    done[slot].record(side)
            else:
                for b, (peer, mine, _theirs) in enumerate(pairs):
                    backend.block(k, mine, start, cnt).copy_(slots[slot][b * step: b * step + cnt])
        if cuda:
            for ev in done:
                if ev is not None:
                    cur.wait_event(ev)
            for s_ in slots:
                s_.record_stream(side)


class SymmetricTransport(DistTransport):
    """DistTransport plus the partner shards mapped over NVLink (torch symmetric memory): remaps
    run the peer swap kernel, and mode="split" gates load and store the partner shard directly.
    The backend must be a DeviceBackend(..., symmetric=True); `attach` is collective."""

    def attach(self, backend) -> None:
        import torch.distributed._symmetric_memory as symm_mem
        self.backend = backend
        self.handle = symm_mem.rendezvous(backend.tensor, self.dist.group.WORLD)

    def peer_buffer(self, peer: int):
        import torch
        return self.handle.get_buffer(peer, (self.backend.tensor.numel(),), torch.complex128)

    def barrier(self) -> None:
        self.handle.barrier(channel=0)  # stream-ordered: orders the GPU work on every rank


def swap_blocks_peer(transport, backend, k: int, pairs, rank: int) -> None:
    """The remap over peer memory: for each partner, the lower rank swaps the first half of the
    block pair and the higher rank the second half (qcs_swap_peer), between two barriers."""
    size = 1 << (backend.n - k)
    h = size // 2
    if hasattr(backend, "_materialise"):
        backend._materialise()  # a deferred reset is written before the partners may read the shard
    transport.barrier()  # every partner's earlier work on its shard is done
    for peer, mine, theirs in pairs:
        lo, cnt = (0, h) if rank < peer else (h, size - h)
        pbuf = transport.peer_buffer(peer)
        off = size * theirs + lo
        backend.swap_peer(size * mine + lo, pbuf[off: off + cnt], cnt)
    transport.barrier()  # ... and the swaps before either shard is used again


class ShardedState:
    """An n-qubit state sharded over `world` ranks (a power of two); this object is rank `rank`."""

    def __init__(self, n: int, world: int, rank: int, backend, transport=None, initial: int = 0,
                 chunk_elems: int = 1 << 22, peer: Optional[bool] = None, mode: str = "remap"):
        g = int(round(math.log2(world)))
        if 1 << g != world:
            raise ValueError("world size must be a power of two")
        if n - g < 1:
            raise ValueError("each shard needs at least one local qubit")
        if mode not in ("remap", "split"):
            raise ValueError("mode is 'remap' or 'split'")
        self.n, self.g, self.world, self.rank = n, g, world, rank
        self.backend = backend
        self.transport = transport
        self.chunk = chunk_elems
        self.mode = mode
        self.phys = list(range(n))  # phys[logical qubit] = physical qubit
        self.pending = []           # local operations not yet handed to the backend
        can_peer = (transport is not None and hasattr(transport, "peer_buffer") and hasattr(transport, "barrier"))
        self.peer = can_peer if peer is None else (bool(peer) and can_peer)
        if self.peer and hasattr(transport, "attach"):
            transport.attach(backend)
        self._timing = False
        self.reset_stats()
        self.set_basis(initial)

    # ------------------------------------------------------------ statistics
    def reset_stats(self) -> None:
        self.swaps = 0              # remaps performed (global<->local exchanges)
        self.remapped_qubits = 0    # qubits moved by them
        self.exchanged_bytes = 0    # bytes sent by this rank
        self.splits = 0             # gates run over peer memory (mode="split")
        self._events = []
        self._host_ms = 0.0

    def timing(self, on: bool) -> None:
        """CUDA events around every exchange (on the current stream) for exchange_stats()."""
        self._timing = on

    def exchange_stats(self) -> dict:
        ms = self._host_ms
        for a, b in self._events:
            b.synchronize()
            ms += a.elapsed_time(b)
        return {"remaps": self.swaps, "qubits": self.remapped_qubits, "bytes_sent": self.exchanged_bytes,
                "splits": self.splits, "ms": ms}

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

    def _rank_bit(self, phys_qubit: int, rank: Optional[int] = None) -> int:
        """Value of global physical qubit `phys_qubit` (< g) on rank `rank` (default: this one)."""
        r = self.rank if rank is None else rank
        return (r >> (self.g - 1 - phys_qubit)) & 1

    # ------------------------------------------------------------ local work, batched
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

    def reset(self, logical_index: int = 0) -> None:
        """Back to |logical_index> with the identity qubit map."""
        self.phys = list(range(self.n))
        self.set_basis(logical_index)

    # ------------------------------------------------------------ exchange
    def _timed(self, fn) -> None:
        if self._timing:
            import torch
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            self._events.append((a, b))
        else:
            fn()

    def _remap(self, gq: List[int]) -> None:
        """Swap the global physical qubits gq[i] with the local physical qubits g + i (the top
        len(gq) local bits): one all-to-all among the 2^k ranks differing in those global bits."""
        k = len(gq)
        if k == 0:
            return
        self.flush()
        if self.world > 1:
            a = 0
            for p in gq:
                a = (a << 1) | self._rank_bit(p)
            pairs = []
            for d in range(1, 1 << k):  # XOR order: the pairs of each d are disjoint
                j = a ^ d
                peer = self.rank
                for i, p in enumerate(gq):
                    bit = (j >> (k - 1 - i)) & 1
                    mask = 1 << (self.g - 1 - p)
                    peer = (peer & ~mask) | (bit * mask)
                pairs.append((peer, j, a))
            nl = self.n - self.g

            def move():
                if self.peer:  # the peer swap kernel over mapped partner shards
                    swap_blocks_peer(self.transport, self.backend, k, pairs, self.rank)
                elif hasattr(self.transport, "swap_blocks"):  # grouped send/recv
                    self.transport.swap_blocks(self.backend, k, pairs, self.chunk)
                else:
                    self._swap_pairwise(k, pairs)
            self._timed(move)
            self.exchanged_bytes += 16 * len(pairs) * (1 << (nl - k))
            self.swaps += 1
            self.remapped_qubits += k
        for i, p in enumerate(gq):  # logical qubits at physical p and g + i trade places
            qa, qb = self.phys.index(p), self.phys.index(self.g + i)
            self.phys[qa], self.phys[qb] = self.g + i, p

    def _swap_pairwise(self, k: int, pairs) -> None:
        """Transports with only a blocking pairwise exchange (the in-process test fabric): one
        partner at a time in XOR order, chunked through a bounded staging buffer."""
        size = 1 << (self.n - self.g - k)
        step = min(self.chunk, size)
        tmp = self.backend.empty(step)
        for peer, mine, _theirs in pairs:
            for start in range(0, size, step):
                cnt = min(step, size - start)
                blk = self.backend.block(k, mine, start, cnt)
                recv = tmp[:cnt]
                self.backend.sync()
                self.transport.exchange(blk, recv, peer)
                blk.copy_(recv)

    def _local_swap(self, pa: int, pb: int) -> None:
        # As three CNOTs -- X-like gates the fused planner lowers to address relabellings inside a
        # pass -- rather than one Swap, a two-target gate that takes a shared-memory round and keeps
        # its pass off the 16-register kernels: rank 0's compute for C4 n=32 at 2 / 4 / 8 ranks
        # 128 / 77 / 42 ms with Swap, 121 / 75 / 39 ms with CNOTs (QCS_LOCAL_SWAP=swap: A/B).
        style = os.environ.get("QCS_LOCAL_SWAP", "cnot")
        if style == "cnot":
            cnot = np.eye(4, dtype=np.complex128)[[0, 1, 3, 2]]
            a, b = pa - self.g, pb - self.g
            for qs in ([a, b], [b, a], [a, b]):
                self.pending.append(("gate", cnot, qs, "CNOT"))
        else:
            swap = np.eye(4, dtype=np.complex128)[[0, 2, 1, 3]]
            self.pending.append(("gate", swap, [pa - self.g, pb - self.g], "Swap"))
        qa, qb = self.phys.index(pa), self.phys.index(pb)
        self.phys[qa], self.phys[qb] = pb, pa

    def _bring_local(self, need: List[int], protect: set, upcoming: List[set]) -> None:
        """Remap the logical qubits `need` (global now) to local positions g..g+k-1.  The local
        qubits that become global in exchange are the ones used latest among `upcoming` (the
        remaining operations' qubit sets) and not by the waiting operations (`protect`); each is
        first brought to a top local position by a local Swap."""
        k = min(len(need), self.g, self.n - self.g)
        need = need[:k]
        free = [pp for pp in range(self.g + k, self.n) if self.phys.index(pp) not in protect]
        clash = [i for i in range(k) if self.phys.index(self.g + i) in protect]
        if len(free) < len(clash):
            raise RuntimeError("no free local qubit to make room for a remap")
        inv = {p: q for q, p in enumerate(self.phys)}

        def next_use(pp):
            q = inv[pp]
            for t, qs in enumerate(upcoming):
                if q in qs:
                    return t
            return len(upcoming)
        # The k local qubits that trade places with the incoming ones become global: pick the
        # ones used latest among the remaining operations (never again, if there are such --
        # a layered circuit's cone leaves qubits far from the global ones finished), not whichever
        # sit at the top local positions.  Evicting a qubit the next layer needs costs a remap
        # per layer (C4 at n=32 on 2 ranks: 10 remaps, 5 shards on the wire, 18 passes); evicting
        # finished ones costs one (0.5 shards, 11 passes).  A local Swap (fused into the pending
        # batch) brings each chosen qubit to a top position first.
        cands = [pp for pp in range(self.g, self.n) if inv[pp] not in protect]
        victims = sorted(cands, key=lambda pp: (-next_use(pp), pp))[:k]
        slots = [self.g + i for i in range(k)]
        stay = [pp for pp in slots if pp in victims]          # already in place
        move = [pp for pp in victims if pp not in slots]       # to be swapped up
        for p in slots:
            if p in stay:
                continue
            if not move:
                if inv[p] in protect:
                    raise RuntimeError("no free local qubit to make room for a remap")
                continue
            best = move.pop(0)
            self._local_swap(p, best)
            inv = {pp: q for q, pp in enumerate(self.phys)}
        self._remap([self.phys[q] for q in need])

    # ------------------------------------------------------------ operations
    def _analyse(self, op):
        """-> (qubits, diagonal, mixing qubits) of an operation; a sign step touches all qubits."""
        if op[0] == "diag":
            return None, True, []
        m = np.asarray(op[1])
        qs = list(op[2])
        k = len(qs)
        r_idx, c_idx = np.nonzero(m)
        mixing = [qs[i] for i in range(k) if np.any(((r_idx ^ c_idx) >> (k - 1 - i)) & 1)]
        return qs, not mixing, mixing

    def _emit_local(self, op) -> None:
        """Queue an operation none of whose mixing qubits is global (block reduction)."""
        if op[0] == "diag":
            mine = []
            for x in op[1]:
                owner, local = self._owner(self._to_phys_index(int(x)))
                if owner == self.rank:
                    mine.append(local)
            if mine or op[2]:
                self.pending.append(("diag", sorted(set(mine)), op[2]))
            return
        _, m, logical_qubits, name = op
        m = np.asarray(m, dtype=np.complex128)
        k = len(logical_qubits)
        phys = [self.phys[q] for q in logical_qubits]
        glob = [i for i, p in enumerate(phys) if p < self.g]
        if not glob:
            self.pending.append(("gate", m, [p - self.g for p in phys], name))
            return
        want = sum(self._rank_bit(phys[i]) << (k - 1 - i) for i in glob)
        loc = [i for i in range(k) if i not in glob]
        if not loc:  # all qubits global: a scalar phase on this rank's shard
            d = m[want, want]
            if d != 1:
                self.pending.append(("gate", np.array([[d, 0], [0, d]]), [0], name))
            return
        sel = [want | sum(((j >> (len(loc) - 1 - t)) & 1) << (k - 1 - loc[t]) for t in range(len(loc)))
               for j in range(1 << len(loc))]
        sub = m[np.ix_(sel, sel)]
        self.pending.append(("gate", sub, [phys[i] - self.g for i in loc], name))

    def run(self, ops) -> None:
        """Apply an operation list ('gate', m, qubits, name) / ('diag', flipped, flip_rest) /
        ('rh',), reordering commuting operations so that every exchange is one batched remap."""
        flat = []
        for op in ops:
            if op[0] == "rh":  # H on every qubit, as n commuting one-qubit gates
                flat += [("gate", _H, [q], "Hadamard") for q in range(self.n)]
            else:
                flat.append(op)
        info = [self._analyse(op) for op in flat]
        pending = list(range(len(flat)))
        while pending:
            busy_nd, busy_d = set(), set()
            sign_blocked = nd_blocked = False
            remaining, waiting = [], []
            for i in pending:
                qs, diag, mixing = info[i]
                if qs is None:  # a sign step: commutes with diagonal operations only
                    conflict = nd_blocked
                else:
                    conflict = any(q in busy_nd for q in qs) or (not diag and (sign_blocked or any(q in busy_d for q in qs)))
                if not conflict:
                    glob_mix = [q for q in mixing if self.phys[q] < self.g]
                    if not glob_mix:
                        self._emit_local(flat[i])
                        continue
                    if self.mode == "split" and self.peer and self._split_gate(flat[i]):
                        continue
                    waiting.append(i)
                remaining.append(i)
                if qs is None:
                    sign_blocked = True
                else:
                    (busy_d if diag else busy_nd).update(qs)
                    nd_blocked |= not diag
            pending = remaining
            if not pending:
                break
            if not waiting:
                raise RuntimeError("scheduler stalled")  # cannot happen: the first pending op waits
            upcoming = [set(info[i][0]) if info[i][0] is not None else set(range(self.n)) for i in pending]
            try:  # everything the waiting operations need, in one remap
                self._bring_local(*self._needs(waiting, info), upcoming)
            except RuntimeError:  # too few free local qubits to protect them all: the first one
                self._bring_local(*self._needs(waiting[:1], info), upcoming)

    def _needs(self, waiting, info):
        need, protect = [], set()
        for i in waiting:
            qs, _diag, mixing = info[i]
            protect.update(qs)
            for q in mixing:
                if self.phys[q] < self.g and q not in need:
                    need.append(q)
        return need, protect

    def _split_gate(self, op) -> bool:
        """mode="split": the gate mixes exactly one of its qubits and that one is global: run it
        over peer memory (qcs_apply_split).  Its other qubits only select 2x2 blocks -- global
        ones by this rank's bits, local ones (<= 2) per amplitude.  False: not of that form."""
        _, m, logical_qubits, name = op
        m = np.asarray(m, dtype=np.complex128)
        phys = [self.phys[q] for q in logical_qubits]
        k = len(phys)
        r_idx, c_idx = np.nonzero(m)
        mixing = [i for i in range(k) if np.any(((r_idx ^ c_idx) >> (k - 1 - i)) & 1)]
        if len(mixing) != 1 or phys[mixing[0]] >= self.g or not hasattr(self.backend, "apply_split"):
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
        if hasattr(self.backend, "_materialise"):
            self.backend._materialise()  # a deferred reset is written before the partner reads the shard
        self.transport.barrier()  # the partner's earlier work on its shard is done
        if skip != (1 << nb) - 1:
            self.backend.apply_split(self.transport.peer_buffer(self.rank ^ (1 << (self.g - 1 - phys[ig]))),
                                     self._rank_bit(phys[ig]), sel_bits, blocks, skip)
            self.splits += 1
        self.transport.barrier()  # ... and ours before either shard is used again
        return True

    # immediate forms (one operation at a time)
    def apply_gate(self, matrix: np.ndarray, logical_qubits: Sequence[int], name: str = "custom") -> None:
        """One placement (gate-local order: local index bit k-1-i <-> logical_qubits[i])."""
        self.run([("gate", np.asarray(matrix, dtype=np.complex128), list(logical_qubits), name)])

    def apply_step(self, placements) -> None:
        """placements: [(matrix, logical_qubits, name), ...] with disjoint qubits."""
        self.run([("gate", np.asarray(m, dtype=np.complex128), list(qs), name) for m, qs, name in placements])

    def apply_diag(self, flipped: Sequence[int], flip_rest: bool) -> None:
        self.run([("diag", list(flipped), flip_rest)])

    def apply_rh(self) -> None:
        """H on all n qubits: local Hadamards on the local qubits, one remap for the global ones."""
        self.run([("rh",)])

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
