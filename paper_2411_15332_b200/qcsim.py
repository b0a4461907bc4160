"""Python mirror of the reference's qcsim API, backed by the B200 engine (libqcs_b200.so).

Names, argument meanings and errors follow the reference headers (paths under
/root/reference/proj/include/qcsim): ``gate_catalog_lookup`` (gates.hpp:36), ``Placement`` /
``DiagSign`` / ``CircuitStep`` / ``Circuit`` (circuit.hpp:12-50), ``build_grover`` (:55),
``build_qnn_neuron`` (:63), ``Engine`` / ``StepReport`` / ``SimReport`` / ``SimOptions`` /
``simulate`` / ``memory_report`` (engine.hpp:10-49), ``step_matrix_dax`` / ``step_matrix_das``
(engine.hpp:38-39), ``dax_mvm`` (dax.hpp:37), ``das_mvm`` (das.hpp:39), ``rh_mvm`` (rh.hpp:64)
and the DAX1 / DAS1 dump formats (dax.hpp:42-45, das.hpp:43-47).

Every state update runs on the GPU through the C ABI; nothing here computes amplitudes.
Generalisation over the reference: ``Placement`` accepts an explicit ``qubits`` list (any
distinct qubits, gate-local order) besides the reference's contiguous ``first_qubit``.
"""
from __future__ import annotations

import ctypes as C
import enum
import io
import math
import struct
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _lib as L


# ---------------------------------------------------------------- errors (core.hpp:13-36)
class SimError(RuntimeError):
    pass


class CapacityError(SimError):
    pass


class DimensionError(SimError):
    pass


class EncodingError(SimError):
    pass


class ParseError(SimError):
    pass


class CudaError(SimError):
    """The device failed, or there is no CUDA device (there is no CPU fallback)."""


_ERRORS = {L.QCS_ERR_CAPACITY: CapacityError, L.QCS_ERR_DIMENSION: DimensionError,
           L.QCS_ERR_ENCODING: EncodingError, L.QCS_ERR_PARSE: ParseError, L.QCS_ERR_SIM: SimError,
           L.QCS_ERR_CUDA: CudaError, L.QCS_ERR_NCCL: CudaError, L.QCS_ERR_ARG: ValueError}


def _check(rc: int) -> None:
    if rc != L.QCS_OK:
        msg = L.lib().qcs_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, SimError)(msg)


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _vptr(a: np.ndarray):
    return C.c_void_p(a.ctypes.data)


# ---------------------------------------------------------------- gates (gates.hpp)
@dataclass
class GateInfo:
    name: str
    arity: int
    param_count: int
    zero_ratio: float


@dataclass
class GateSpec:
    name: str
    arity: int
    params: List[float]
    matrix: np.ndarray  # 2^arity x 2^arity complex128, row-major
    declared_zero_ratio: float = 0.0


def gate_catalog() -> List[GateInfo]:
    lib = L.lib()
    out = []
    for i in range(lib.qcs_gate_catalog_size()):
        name, a, p, r = C.c_char_p(), C.c_int(), C.c_int(), C.c_double()
        _check(lib.qcs_gate_catalog_entry(i, C.byref(name), C.byref(a), C.byref(p), C.byref(r)))
        out.append(GateInfo(name.value.decode(), a.value, p.value, r.value))
    return out


def canonical_params(name: str) -> List[float]:
    out = (C.c_double * 4)()
    k = C.c_int()
    _check(L.lib().qcs_canonical_params(name.encode(), out, C.byref(k)))
    return list(out[: k.value])


def gate_known(name: str) -> bool:
    try:
        canonical_params(name)
        return True
    except SimError:
        return False


_RATIOS = None  # catalog name -> declared zero ratio (the catalog is constant)


def gate_catalog_lookup(name: str, params: Sequence[float] = ()) -> GateSpec:
    p = np.ascontiguousarray(np.asarray(params, dtype=np.float64).reshape(-1))
    m = np.zeros(64, np.complex128)
    ar = C.c_int()
    canon = C.c_char_p()
    _check(L.lib().qcs_gate_lookup(name.encode(), _dptr(p) if p.size else None, p.size,
                                   m.ctypes.data_as(C.POINTER(C.c_double)), C.byref(ar), C.byref(canon)))
    d = 1 << ar.value
    global _RATIOS
    if _RATIOS is None:
        _RATIOS = {g.name: g.zero_ratio for g in gate_catalog()}
    ratio = _RATIOS.get(canon.value.decode(), 0.0)
    return GateSpec(canon.value.decode(), ar.value, list(map(float, p)), m[: d * d].reshape(d, d).copy(), ratio)


def custom_gate(matrix, name: str = "custom") -> GateSpec:
    m = np.ascontiguousarray(np.asarray(matrix, dtype=np.complex128))
    k = int(round(math.log2(m.shape[0])))
    if m.shape != (1 << k, 1 << k):
        raise DimensionError("gate matrix must be 2^k x 2^k")
    return GateSpec(name, k, [], m)


# ---------------------------------------------------------------- circuits (circuit.hpp)
@dataclass
class Placement:
    gate: GateSpec
    first_qubit: int = 0
    qubits: Optional[List[int]] = None  # generalisation: explicit qubit list (gate-local order)

    def qubit_list(self) -> List[int]:
        if self.qubits is not None:
            return list(self.qubits)
        return list(range(self.first_qubit, self.first_qubit + self.gate.arity))


@dataclass
class DiagSign:
    flipped: List[int] = field(default_factory=list)
    flip_rest: bool = False

    def negated(self, index: int) -> bool:  # circuit.cpp:9-12
        return (index in set(self.flipped)) != self.flip_rest


class StepKind(enum.IntEnum):
    gates = 0
    diag = 1


@dataclass
class CircuitStep:
    kind: StepKind = StepKind.gates
    placements: List[Placement] = field(default_factory=list)
    diag: DiagSign = field(default_factory=DiagSign)
    stage: int = 0

    @staticmethod
    def of_gates(placements: List[Placement], stage: int = 0) -> "CircuitStep":
        return CircuitStep(StepKind.gates, list(placements), DiagSign(), stage)

    @staticmethod
    def of_diag(d: DiagSign, stage: int = 0) -> "CircuitStep":
        return CircuitStep(StepKind.diag, [], DiagSign(sorted(int(x) for x in d.flipped), bool(d.flip_rest)), stage)

    def is_hadamard_all(self, n: int) -> bool:  # circuit.cpp:31-39
        if self.kind != StepKind.gates or len(self.placements) != n:
            return False
        covered = 0
        for p in self.placements:
            if p.gate.name != "Hadamard" or p.gate.arity != 1:
                return False
            covered |= 1 << p.qubit_list()[0]
        return covered == (1 << n) - 1


@dataclass
class Circuit:
    n: int = 0
    steps: List[CircuitStep] = field(default_factory=list)
    initial: int = 0

    def validate(self) -> None:  # circuit.cpp:41-62
        if self.n < 1:
            raise DimensionError("circuit needs n >= 1 qubits")
        dim = 1 << self.n
        if self.initial >= dim:
            raise DimensionError("initial basis index out of range")
        for st in self.steps:
            if st.kind == StepKind.diag:
                if any(i >= dim for i in st.diag.flipped):
                    raise DimensionError("diagonal step index out of range")
                continue
            covered = 0
            for p in st.placements:
                qs = p.qubit_list()
                if min(qs) < 0 or max(qs) >= self.n:
                    raise DimensionError("gate placement out of range")
                for q in qs:
                    if covered >> q & 1:
                        raise DimensionError("overlapping gate placements in a step")
                    covered |= 1 << q


def hadamard_all(n: int, stage: int = 0) -> CircuitStep:
    h = gate_catalog_lookup("Hadamard")
    return CircuitStep.of_gates([Placement(h, q) for q in range(n)], stage)


def grover_auto_iterations(n: int) -> int:  # circuit.cpp:75-78
    return max(1, int(math.floor(math.pi / 4.0 * math.sqrt(math.exp2(n)))))


def build_grover(n: int, marked: int, iterations: int = 0) -> Circuit:  # circuit.cpp:80-96
    if n < 1:
        raise DimensionError("Grover needs n >= 1")
    if marked >= (1 << n):
        raise DimensionError("marked index out of range")
    iters = iterations if iterations > 0 else grover_auto_iterations(n)
    c = Circuit(n, [hadamard_all(n)])
    for _ in range(iters):
        c.steps.append(CircuitStep.of_diag(DiagSign([marked], False)))  # oracle
        c.steps.append(hadamard_all(n))
        c.steps.append(CircuitStep.of_diag(DiagSign([0], True)))  # Z0
        c.steps.append(hadamard_all(n))
    return c


def qnn_total_qubits(input_qubits: int) -> int:  # circuit.cpp:98-103
    if input_qubits < 1:
        raise DimensionError("neuron needs at least one input qubit")
    enc = 0
    while (1 << enc) < input_qubits:
        enc += 1
    return input_qubits + enc + 1


def build_qnn_neuron(input_qubits: int, encode_angles: Sequence[float], weights: Sequence[int]) -> Circuit:
    """circuit.cpp:105-149: RY encoding, Z sign flips + Toffoli aggregation, controlled copy."""
    if len(encode_angles) != input_qubits or len(weights) != input_qubits:
        raise SimError("angle and weight lists must match the input qubit count")
    if any(w not in (1, -1) for w in weights):
        raise SimError("weights must be +1 or -1")
    n = qnn_total_qubits(input_qubits)
    enc = n - input_qubits - 1
    c = Circuit(n)
    c.steps.append(CircuitStep.of_gates(
        [Placement(gate_catalog_lookup("RY", [encode_angles[q]]), q) for q in range(input_qubits)], 1))
    z = gate_catalog_lookup("Pauli-Z")
    pz = [Placement(z, q) for q in range(input_qubits) if weights[q] == -1]
    if pz:
        c.steps.append(CircuitStep.of_gates(pz, 2))
    ccx = gate_catalog_lookup("CCX")
    for e in range(enc):
        first = input_qubits - 2 + e
        if first >= 0:
            c.steps.append(CircuitStep.of_gates([Placement(ccx, first)], 2))
    c.steps.append(CircuitStep.of_gates([Placement(gate_catalog_lookup("Controlled-X"), n - 2)], 3))
    return c


# ---------------------------------------------------------------- engine (engine.hpp)
class Engine(enum.IntEnum):
    dense = 0
    dax = 1
    das = 2
    rh_dax = 3


_ENGINE_NAMES = {Engine.dense: "dense", Engine.dax: "dax", Engine.das: "das", Engine.rh_dax: "rh-dax"}


def engine_name(e: Engine) -> str:
    return _ENGINE_NAMES[Engine(e)]


def engine_from_name(name: str) -> Engine:
    for e, s in _ENGINE_NAMES.items():
        if s == name:
            return e
    if name == "rh_dax":
        return Engine.rh_dax
    raise ParseError("unknown engine: " + name)


class SignMethod(enum.IntEnum):
    nonopt = 0
    quarter = 1
    block = 2
    logarithm = 3


@dataclass
class SimOptions:
    sign_method: SignMethod = SignMethod.logarithm
    block_size: int = 0
    fuse: bool = True  # B200 extension: fuse operations into shared-memory passes


_STRUCT = {0: "dense", 1: "dax", 2: "das", 3: "rh"}


@dataclass
class StepReport:
    structure: str = ""
    stage: int = 0
    matrix_bytes: int = 0
    dense_bytes: int = 0
    entry_count: int = 0
    sign_count: int = 0
    madd_count: int = 0


class DeviceState:
    """A StateVector (core.hpp:64-76) resident in HBM.  ``amps`` downloads on demand."""

    def __init__(self, n: int, basis_index: int = 0, device: int = 0, _handle=None):
        self.n = n
        self.device = device
        if _handle is not None:
            self._h = _handle
        else:
            h = C.c_void_p()
            _check(L.lib().qcs_state_create(n, device, basis_index, C.byref(h)))
            self._h = h

    @classmethod
    def from_numpy(cls, amps: np.ndarray, device: int = 0) -> "DeviceState":
        a = np.ascontiguousarray(amps, dtype=np.complex128)
        n = int(round(math.log2(a.size)))
        if a.size != 1 << n:
            raise DimensionError("state length must be a power of two")
        s = cls(n, 0, device)
        s.upload(a)
        return s

    @property
    def handle(self):
        return self._h

    def dim(self) -> int:
        return 1 << self.n

    def upload(self, a: np.ndarray, first: int = 0) -> None:
        a = np.ascontiguousarray(a, dtype=np.complex128)
        _check(L.lib().qcs_state_upload(self._h, _vptr(a), first, a.size))
        self.sync()

    def download(self, first: int = 0, count: Optional[int] = None) -> np.ndarray:
        count = self.dim() - first if count is None else count
        out = np.empty(count, np.complex128)
        _check(L.lib().qcs_state_download(self._h, _vptr(out), first, count))
        return out

    @property
    def amps(self) -> np.ndarray:
        return self.download()

    def set_basis(self, index: int) -> None:
        _check(L.lib().qcs_state_set_basis(self._h, index))

    def randomize(self, seed: int) -> None:
        _check(L.lib().qcs_state_random(self._h, seed))

    def copy_from(self, other: "DeviceState") -> None:
        _check(L.lib().qcs_state_copy(self._h, other._h))

    def wait_for(self, other: "DeviceState") -> None:
        """Work enqueued on this state from now on starts after everything enqueued on `other`
        so far (device-side ordering, the host does not block)."""
        _check(L.lib().qcs_state_wait(self._h, other._h))

    def sync(self) -> None:
        _check(L.lib().qcs_state_sync(self._h))

    def norm(self) -> float:
        out = C.c_double()
        _check(L.lib().qcs_norm(self._h, C.byref(out)))
        return out.value

    def probabilities(self) -> np.ndarray:
        out = np.empty(self.dim(), np.float64)
        _check(L.lib().qcs_probabilities(self._h, _vptr(out), L.QCS_MEM_HOST))
        return out

    def argmax(self):
        i, p = C.c_uint64(), C.c_double()
        _check(L.lib().qcs_argmax(self._h, C.byref(i), C.byref(p)))
        return i.value, p.value

    def topk(self, k: int = 16):
        idx = (C.c_uint64 * k)()
        pr = (C.c_double * k)()
        _check(L.lib().qcs_topk(self._h, k, idx, pr))
        return list(idx), list(pr)

    def summary(self, k: int = 16):
        """(norm, [top-k indices], [their probabilities]) from one pass over the state; the argmax
        is the first index.  What render_report needs, without downloading 2^n values."""
        nrm = C.c_double()
        idx = (C.c_uint64 * k)()
        pr = (C.c_double * k)()
        _check(L.lib().qcs_summary(self._h, k, C.byref(nrm), idx, pr))
        return nrm.value, list(idx), list(pr)

    def summary_begin(self, k: int = 16) -> None:
        """The summary pass and its read-back, queued on the state's stream (qcs_summary_begin)."""
        _check(L.lib().qcs_summary_begin(self._h, k))
        self._summary_k = k

    def summary_end(self):
        """Wait for summary_begin's result: (norm, [top-k indices], [probabilities])."""
        k = getattr(self, "_summary_k", 16)
        nrm = C.c_double()
        idx = (C.c_uint64 * k)()
        pr = (C.c_double * k)()
        _check(L.lib().qcs_summary_end(self._h, C.byref(nrm), idx, pr))
        return nrm.value, list(idx), list(pr)

    def sample(self, count: int, seed: int):
        """render_report's seeded samples (circuit_io.cpp:114-128), drawn on the device: returns
        ([indices], acc) with acc the sequential sum of the probabilities.  Index-exact against
        the reference (the device reproduces its rounded sequential CDF)."""
        out = (C.c_uint64 * max(count, 1))()
        tot = C.c_double()
        _check(L.lib().qcs_sample(self._h, seed & 0xFFFFFFFFFFFFFFFF, count, out, C.byref(tot)))
        return list(out)[:count], tot.value

    def rh_mvm(self, value: float, method: "SignMethod" = None, block_size: int = 0):
        """rh_mvm(RhMatrix{n, value}, s, method, &stats, block_size) in place (qcs_rh_mvm,
        rh.hpp:64-66): returns (sign_count, madd_count) as RhMvmStats."""
        m = int(SignMethod.logarithm if method is None else method)
        sc, mc = C.c_uint64(), C.c_uint64()
        _check(L.lib().qcs_rh_mvm(self._h, self.n, float(value), m, int(block_size), C.byref(sc), C.byref(mc)))
        return int(sc.value), int(mc.value)

    def gather(self, indices) -> np.ndarray:
        idx = np.ascontiguousarray(np.asarray(indices, dtype=np.uint64))
        out = np.empty(idx.size, np.complex128)
        _check(L.lib().qcs_gather(self._h, idx.ctypes.data_as(C.POINTER(C.c_uint64)), idx.size, _dptr(out)))
        return out

    def distance(self, other: "DeviceState"):
        """(max_i |a_i - b_i|, ||a - b||_2), reduced on the device (no download).  B200-specific."""
        mx, l2 = C.c_double(), C.c_double()
        _check(L.lib().qcs_state_distance(self._h, other._h, C.byref(mx), C.byref(l2)))
        return mx.value, l2.value

    # one step at a time
    def apply_step(self, placements: Sequence[Placement]) -> None:
        arr, keep = _placements(placements)
        _check(L.lib().qcs_apply_step(self._h, arr, len(placements)))

    def apply_gate(self, gate: GateSpec, qubits: Sequence[int]) -> None:
        self.apply_step([Placement(gate, qubits=list(qubits))])

    def apply_diag(self, d: DiagSign) -> None:
        f = np.ascontiguousarray(np.asarray(d.flipped, dtype=np.uint64))
        _check(L.lib().qcs_apply_diag(self._h, f.ctypes.data_as(C.POINTER(C.c_uint64)) if f.size else None,
                                      f.size, int(d.flip_rest)))

    def apply_split(self, peer_ptr: int, self_bit: int, sel_bits: Sequence[int], blocks: np.ndarray,
                    skip_mask: int = 0) -> None:
        """A gate on a shard-global qubit over the partner shard at device address `peer_ptr`
        (qcs_apply_split; partition.py drives it).  blocks: (2^len(sel_bits), 2, 2) complex."""
        b = np.ascontiguousarray(np.asarray(blocks, dtype=np.complex128).reshape(-1, 2, 2))
        sel = (C.c_int * max(1, len(sel_bits)))(*[int(x) for x in sel_bits])
        _check(L.lib().qcs_apply_split(self._h, C.c_void_p(int(peer_ptr)), int(self_bit), len(sel_bits), sel,
                                       b.ctypes.data_as(C.POINTER(C.c_double)), int(skip_mask)))

    def apply_rh(self) -> None:
        _check(L.lib().qcs_apply_rh(self._h))

    def record(self, slot: int) -> None:
        _check(L.lib().qcs_event_record(self._h, slot))

    def elapsed_ms(self, a: int, b: int) -> float:
        ms = C.c_float()
        _check(L.lib().qcs_event_elapsed_ms(self._h, a, b, C.byref(ms)))
        return ms.value

    def timing(self, enable: bool = True) -> None:
        """Per-launch CUDA-event timing by kernel class (see qcs_timing_enable)."""
        _check(L.lib().qcs_timing_enable(self._h, int(enable)))

    def timing_reset(self) -> None:
        _check(L.lib().qcs_timing_reset(self._h))

    def timing_report(self) -> dict:
        """{kernel_class: (launches, total_ms, algorithmic_bytes)}; synchronises the stream."""
        k = C.c_int()
        _check(L.lib().qcs_timing_count(self._h, C.byref(k)))
        out = {}
        for i in range(k.value):
            name, n, ms, b = C.c_char_p(), C.c_uint64(), C.c_double(), C.c_double()
            _check(L.lib().qcs_timing_entry(self._h, i, C.byref(name), C.byref(n), C.byref(ms), C.byref(b)))
            out[name.value.decode()] = (n.value, ms.value, b.value)
        return out

    def close(self) -> None:
        if getattr(self, "_h", None):
            L.lib().qcs_state_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


StateVector = DeviceState


def _placements(placements: Sequence[Placement]):
    """-> (ctypes array of qcs_placement, keep-alive list).  Qubits and matrices of all the
    placements are packed into one int32 and one complex128 array (two numpy calls, not two per
    placement): marshalling dominates the host cost of small circuits."""
    n = len(placements)
    arr = (L.qcs_placement * max(1, n))()
    if n == 0:
        return arr, []
    qlists = [p.qubit_list() for p in placements]
    mats = [p.gate.matrix for p in placements]
    for p, q, m in zip(placements, qlists, mats):
        if len(q) != p.gate.arity or np.size(m) != 4 ** p.gate.arity:
            raise DimensionError("placement matrix / qubit count does not match the gate arity")
    qs = np.fromiter((x for q in qlists for x in q), dtype=np.int32)
    ms = np.concatenate([np.asarray(m, dtype=np.complex128).ravel() for m in mats])
    names = [p.gate.name.encode() for p in placements]
    qa, ma = qs.ctypes.data, ms.ctypes.data
    qo = mo = 0
    for i, p in enumerate(placements):
        k = p.gate.arity
        e = arr[i]
        e.arity = k
        e.qubits = qa + 4 * qo
        e.matrix = ma + 16 * mo
        e.name = names[i]
        qo += k
        mo += 1 << (2 * k)
    return arr, [qs, ms, names]


def _steps(steps: Sequence[CircuitStep]):
    arr = (L.qcs_step * max(1, len(steps)))()
    keep = []
    gate_steps = [st for st in steps if st.kind != StepKind.diag]
    pa, k = _placements([p for st in gate_steps for p in st.placements])
    keep += [pa, k]
    base = C.addressof(pa)
    size = C.sizeof(L.qcs_placement)
    off = 0
    for i, st in enumerate(steps):
        e = arr[i]
        e.kind = int(st.kind)
        e.stage = st.stage
        if st.kind == StepKind.diag:
            f = np.ascontiguousarray(np.asarray(st.diag.flipped, dtype=np.uint64))
            keep.append(f)
            e.flipped = f.ctypes.data if f.size else None
            e.num_flipped = f.size
            e.flip_rest = int(st.diag.flip_rest)
        else:
            e.placements = base + size * off
            e.num_placements = len(st.placements)
            off += len(st.placements)
    return arr, keep


@dataclass
class SimReport:
    final: DeviceState
    steps: List[StepReport]
    total_sign_count: int = 0
    total_madd_count: int = 0
    _probs: Optional[np.ndarray] = None

    @property
    def probabilities(self) -> np.ndarray:  # core.cpp:36-40, computed on the device
        if self._probs is None:
            self._probs = self.final.probabilities()
        return self._probs


def _reports(raw, count) -> List[StepReport]:
    return [StepReport(_STRUCT[raw[i].structure], raw[i].stage, raw[i].matrix_bytes, raw[i].dense_bytes,
                       raw[i].entry_count, raw[i].sign_count, raw[i].madd_count) for i in range(count)]


def simulate(c: Circuit, engine: Engine = Engine.rh_dax, opts: Optional[SimOptions] = None,
             device: int = 0, state: Optional[DeviceState] = None) -> SimReport:
    """engine.cpp:153-210.  ``state`` (optional) is reused and reset to |initial>."""
    opts = opts or SimOptions()
    c.validate()
    if state is None:
        state = DeviceState(c.n, c.initial, device)
    elif state.n != c.n:
        raise DimensionError("state qubit count mismatch")
    arr, keep = _steps(c.steps)
    # reset: start from |initial> (folded into the first pass when it sweeps the whole state)
    o = L.qcs_sim_options(int(opts.sign_method), int(opts.block_size), int(bool(opts.fuse)), 1, int(c.initial))
    rep = (L.qcs_step_report * max(1, len(c.steps)))()
    _check(L.lib().qcs_simulate(state.handle, arr, len(c.steps), int(engine), C.byref(o), rep))
    steps = _reports(rep, len(c.steps))
    mask = (1 << 64) - 1
    return SimReport(state, steps, sum(s.sign_count for s in steps) & mask, sum(s.madd_count for s in steps) & mask)


def run(c: Circuit, state: DeviceState, engine: Engine = Engine.rh_dax, opts: Optional[SimOptions] = None,
        reset_index: Optional[int] = None) -> List[StepReport]:
    """Apply the circuit's steps to `state` as it is (no reset to |initial>): the in-place form
    of simulate used by the partitioner between exchanges.  reset_index: the state is to start
    from the basis state |reset_index> (qcs_sim_options.reset: folded into the first pass, and
    the passes skip the tiles outside the support reached so far)."""
    opts = opts or SimOptions()
    if state.n != c.n:
        raise DimensionError("state qubit count mismatch")
    arr, keep = _steps(c.steps)
    o = L.qcs_sim_options(int(opts.sign_method), int(opts.block_size), int(bool(opts.fuse)))
    if reset_index is not None:
        o = L.qcs_sim_options(int(opts.sign_method), int(opts.block_size), int(bool(opts.fuse)), 1, int(reset_index))
    rep = (L.qcs_step_report * max(1, len(c.steps)))()
    _check(L.lib().qcs_simulate(state.handle, arr, len(c.steps), int(engine), C.byref(o), rep))
    return _reports(rep, len(c.steps))


def memory_report(c: Circuit, engine: Engine) -> List[StepReport]:  # engine.cpp:212-234
    c.validate()
    arr, keep = _steps(c.steps)
    rep = (L.qcs_step_report * max(1, len(c.steps)))()
    _check(L.lib().qcs_memory_report(c.n, arr, len(c.steps), int(engine), rep))
    return _reports(rep, len(c.steps))


def plan_stats(c: Circuit, engine: Engine = Engine.rh_dax, opts: Optional[SimOptions] = None) -> dict:
    """The fused-pass plan simulate() would launch for `c` (host only, no device): operation,
    pass, round counts.  B200-specific; the reference has no planner."""
    opts = opts or SimOptions()
    arr, keep = _steps(c.steps)
    # from |initial>, as simulate() runs it (support tracking, the reset folded into pass 1)
    o = L.qcs_sim_options(int(opts.sign_method), int(opts.block_size), int(bool(opts.fuse)), 1, int(c.initial))
    info = L.qcs_plan_info()
    _check(L.lib().qcs_plan_stats(c.n, arr, len(c.steps), int(engine), C.byref(o), C.byref(info)))
    return {f: int(getattr(info, f)) for f, _ in L.qcs_plan_info._fields_}


def plan_verify(c: Circuit, engine: Engine = Engine.rh_dax, opts: Optional[SimOptions] = None) -> int:
    """Host-only addressing proof of the plan's specialised kernels (qcs_plan_verify): raises
    SimError if any register round's shared-memory addressing is not a permutation of its tile.
    Returns the number of passes checked.  B200-specific."""
    opts = opts or SimOptions()
    arr, keep = _steps(c.steps)
    o = L.qcs_sim_options(int(opts.sign_method), int(opts.block_size), int(bool(opts.fuse)), 1, int(c.initial))
    k = C.c_int64()
    _check(L.lib().qcs_plan_verify(c.n, arr, len(c.steps), int(engine), C.byref(o), C.byref(k)))
    return int(k.value)


def set_jit_mode(mode: int) -> None:
    """0: every fused pass runs on the interpreter kernel; 1 (default): passes with enough work
    run as kernels specialised to their operation list (compiled once per structure, NVRTC);
    2: all.  Results are bit-identical.  B200-specific."""
    _check(L.lib().qcs_set_jit_mode(int(mode)))


def jit_mode() -> int:
    return int(L.lib().qcs_get_jit_mode())


def set_pipeline_mode(mode: int) -> None:
    """Which specialised pass kernels run in the persistent pipelined form (one CTA per SM, a ring
    of TMA tile slots, two compute groups): 0 none, 1 passes with 16-amplitude register rounds
    (default), 2 every eligible pass.  Bit-identical results.  B200-specific."""
    _check(L.lib().qcs_set_pipeline_mode(int(mode)))


def pipeline_mode() -> int:
    return int(L.lib().qcs_get_pipeline_mode())


def plan_compile(c: Circuit, engine: Engine = Engine.rh_dax, opts: Optional[SimOptions] = None) -> dict:
    """Generate and compile (NVRTC, host only) the specialised kernel of every tile pass of the
    plan of `c`.  B200-specific check/tool: {"kernels": passes compiled, "cubin_bytes": code size}."""
    opts = opts or SimOptions()
    arr, keep = _steps(c.steps)
    o = L.qcs_sim_options(int(opts.sign_method), int(opts.block_size), int(bool(opts.fuse)))
    k, b = C.c_int64(), C.c_int64()
    _check(L.lib().qcs_plan_compile(c.n, arr, len(c.steps), int(engine), C.byref(o), C.byref(k), C.byref(b)))
    return {"kernels": int(k.value), "cubin_bytes": int(b.value)}


# ---------------------------------------------------------------- compressed structures
@dataclass
class DaxMatrix:  # dax.hpp:22-28
    rows: int
    cols: int
    row: np.ndarray    # uint64 entry rows
    col: np.ndarray    # uint64 entry cols
    value: np.ndarray  # complex128

    def __eq__(self, o) -> bool:
        return (self.rows == o.rows and self.cols == o.cols and np.array_equal(self.row, o.row)
                and np.array_equal(self.col, o.col) and np.array_equal(self.value, o.value))


@dataclass
class DasMatrix:  # das.hpp:21-27
    rows: int
    cols: int
    dis: np.ndarray            # uint64
    last_in_row: np.ndarray    # uint8 0/1
    value: np.ndarray          # complex128

    def __eq__(self, o) -> bool:
        return (self.rows == o.rows and self.cols == o.cols and np.array_equal(self.dis, o.dis)
                and np.array_equal(self.last_in_row, o.last_in_row) and np.array_equal(self.value, o.value))


def dax_memory_bytes(m: DaxMatrix) -> int:  # dax.cpp:105
    return 24 * len(m.row)


def das_memory_bytes(m: DasMatrix) -> int:  # das.cpp:152
    return 24 * len(m.dis)


def _encode(step: CircuitStep, n: int, das: bool, device: int):
    if step.kind == StepKind.diag:
        raise SimError("diagonal steps have no placement encoding; use diag_dax")
    arr, keep = _placements(step.placements)
    cnt = C.c_uint64()
    fn = L.lib().qcs_step_das if das else L.lib().qcs_step_dax
    rc = fn(n, arr, len(step.placements), device, None, None, None, 0, L.QCS_MEM_HOST, C.byref(cnt))
    if rc not in (L.QCS_OK, L.QCS_ERR_CAPACITY):
        _check(rc)
    k = cnt.value
    a = np.empty(k, np.uint64)
    b = np.empty(k, np.uint8 if das else np.uint64)
    v = np.empty(k, np.complex128)
    _check(fn(n, arr, len(step.placements), device, _vptr(a), _vptr(b), _vptr(v), k, L.QCS_MEM_HOST, C.byref(cnt)))
    return a, b, v


def step_matrix_dax(step: CircuitStep, n: int, device: int = 0) -> DaxMatrix:
    """engine.cpp:135-142, materialised by the device encoder (byte-identical)."""
    if step.kind == StepKind.diag:
        dim = 1 << n
        idx = np.arange(dim, dtype=np.uint64)
        vals = np.ones(dim, np.complex128)
        neg = np.zeros(dim, bool)
        if step.diag.flipped:
            neg[np.asarray(step.diag.flipped, dtype=np.int64)] = True
        if step.diag.flip_rest:
            neg = ~neg
        vals[neg] = -1.0
        return DaxMatrix(dim, dim, idx, idx.copy(), vals)
    r, c, v = _encode(step, n, False, device)
    return DaxMatrix(1 << n, 1 << n, r, c, v)


def step_matrix_das(step: CircuitStep, n: int, device: int = 0) -> DasMatrix:
    """engine.cpp:144-151, materialised by the device encoder (byte-identical)."""
    if step.kind == StepKind.diag:
        d = step_matrix_dax(step, n)
        return DasMatrix(d.rows, d.cols, d.row.copy(), np.ones(d.rows, np.uint8), d.value)
    dis, last, v = _encode(step, n, True, device)
    return DasMatrix(1 << n, 1 << n, dis, last, v)


def dax_mvm(m: DaxMatrix, s: DeviceState) -> DeviceState:  # dax.cpp:96-103
    if m.rows != m.cols or m.cols != s.dim():
        raise DimensionError("DAX MVM shape mismatch")
    out = DeviceState(s.n, 0, s.device)
    r = np.ascontiguousarray(m.row, np.uint64)
    c = np.ascontiguousarray(m.col, np.uint64)
    v = np.ascontiguousarray(m.value, np.complex128)
    _check(L.lib().qcs_dax_mvm(_vptr(r), _vptr(c), _vptr(v), r.size, L.QCS_MEM_HOST, s.handle, out.handle))
    return out


def das_mvm(m: DasMatrix, s: DeviceState) -> DeviceState:  # das.cpp:131-150
    if m.rows != m.cols or m.cols != s.dim():
        raise DimensionError("DAS MVM shape mismatch")
    out = DeviceState(s.n, 0, s.device)
    d = np.ascontiguousarray(m.dis, np.uint64)
    l = np.ascontiguousarray(m.last_in_row, np.uint8)
    v = np.ascontiguousarray(m.value, np.complex128)
    _check(L.lib().qcs_das_mvm(_vptr(d), _vptr(l), _vptr(v), d.size, L.QCS_MEM_HOST, s.handle, out.handle))
    return out


def rh_mvm(s: DeviceState) -> DeviceState:
    """rh_mvm(rh_build(n), s) (rh.hpp:64-66) as a device Walsh-Hadamard butterfly; out-of-place."""
    out = DeviceState(s.n, 0, s.device)
    out.copy_from(s)
    out.apply_rh()
    return out


def dense_cap() -> int:  # core.hpp:38-44 (the dense engine's element cap)
    return int(L.lib().qcs_dense_cap())


def set_dense_cap(cap: int) -> None:
    _check(L.lib().qcs_set_dense_cap(int(cap)))


class DeviceEncoded:
    """A step's DAX or DAS structure materialised in DEVICE memory by the device encoder
    (qcs_step_dax / qcs_step_das with QCS_MEM_DEVICE), for the device MVMs -- the reference's
    step_matrix_* + *_mvm pipeline (engine.cpp:192-199) without host round trips."""

    def __init__(self, step: CircuitStep, n: int, das: bool, device: int = 0):
        import torch
        self.n, self.das, self.device = n, das, device
        arr, keep = _placements(step.placements)
        fn = L.lib().qcs_step_das if das else L.lib().qcs_step_dax
        cnt = C.c_uint64()
        rc = fn(n, arr, len(step.placements), device, None, None, None, 0, L.QCS_MEM_DEVICE, C.byref(cnt))
        if rc not in (L.QCS_OK, L.QCS_ERR_CAPACITY):
            _check(rc)
        k = int(cnt.value)
        dev = torch.device("cuda", device)
        self.a = torch.empty(max(k, 1), dtype=torch.int64, device=dev)
        self.b = torch.empty(max(k, 1), dtype=torch.uint8 if das else torch.int64, device=dev)
        self.v = torch.empty(max(k, 1), dtype=torch.complex128, device=dev)
        _check(fn(n, arr, len(step.placements), device, C.c_void_p(self.a.data_ptr()), C.c_void_p(self.b.data_ptr()),
                  C.c_void_p(self.v.data_ptr()), k, L.QCS_MEM_DEVICE, C.byref(cnt)))
        self.count = int(cnt.value)
        torch.cuda.synchronize(dev)

    def mvm(self, s: "DeviceState", out: "DeviceState") -> None:
        """out = M s (dax.cpp:96-103 / das.cpp:131-150) on the device entries."""
        ptr = lambda t: C.c_void_p(t.data_ptr())
        if self.das:
            _check(L.lib().qcs_das_mvm(ptr(self.a), ptr(self.b), ptr(self.v), self.count, L.QCS_MEM_DEVICE,
                                       s.handle, out.handle))
        else:
            _check(L.lib().qcs_dax_mvm(ptr(self.a), ptr(self.b), ptr(self.v), self.count, L.QCS_MEM_DEVICE,
                                       s.handle, out.handle))

    def close(self) -> None:
        self.a = self.b = self.v = None


def step_matrix_dax_device(step: CircuitStep, n: int, device: int = 0) -> DeviceEncoded:
    return DeviceEncoded(step, n, False, device)


def step_matrix_das_device(step: CircuitStep, n: int, device: int = 0) -> DeviceEncoded:
    return DeviceEncoded(step, n, True, device)


def rh_build_value(n: int) -> float:  # rh.cpp:18-21
    if n < 1:
        raise DimensionError("RH needs n >= 1")
    return math.exp2(-0.5 * n)


# ---------------------------------------------------------------- dumps (dax.cpp:107-138, das.cpp:154-187)
def dax_dump(m: DaxMatrix) -> bytes:
    buf = io.BytesIO()
    buf.write(b"DAX1" + struct.pack("<QQQ", m.rows, m.cols, len(m.row)))
    rec = np.empty((len(m.row), 4), np.uint64)
    rec[:, 0] = m.row
    rec[:, 1] = m.col
    rec[:, 2:] = np.ascontiguousarray(m.value).view(np.uint64).reshape(-1, 2)
    buf.write(rec.astype("<u8").tobytes())
    return buf.getvalue()


def dax_load(data: bytes) -> DaxMatrix:
    if len(data) < 4 or data[:4] != b"DAX1":
        raise ParseError("bad DAX dump magic")
    if len(data) < 28:
        raise ParseError("truncated DAX dump")
    rows, cols, count = struct.unpack_from("<QQQ", data, 4)
    body = data[28:28 + 32 * count]
    if len(body) != 32 * count:
        raise ParseError("truncated DAX dump")
    rec = np.frombuffer(body, "<u8").reshape(-1, 4)
    return DaxMatrix(rows, cols, rec[:, 0].copy(), rec[:, 1].copy(),
                     np.ascontiguousarray(rec[:, 2:]).view(np.complex128).reshape(-1).copy())


def das_dump(m: DasMatrix) -> bytes:
    flag = np.uint64(1) << np.uint64(63)
    rec = np.empty((len(m.dis), 3), np.uint64)
    rec[:, 0] = np.asarray(m.dis, np.uint64) | np.where(np.asarray(m.last_in_row) != 0, flag, np.uint64(0))
    rec[:, 1:] = np.ascontiguousarray(m.value).view(np.uint64).reshape(-1, 2)
    return b"DAS1" + struct.pack("<QQQ", m.rows, m.cols, len(m.dis)) + rec.astype("<u8").tobytes()


def das_load(data: bytes) -> DasMatrix:
    if len(data) < 4 or data[:4] != b"DAS1":
        raise ParseError("bad DAS dump magic")
    if len(data) < 28:
        raise ParseError("truncated DAS dump")
    rows, cols, count = struct.unpack_from("<QQQ", data, 4)
    body = data[28:28 + 24 * count]
    if len(body) != 24 * count:
        raise ParseError("truncated DAS dump")
    rec = np.frombuffer(body, "<u8").reshape(-1, 3)
    flag = np.uint64(1) << np.uint64(63)
    return DasMatrix(rows, cols, rec[:, 0] & ~flag, ((rec[:, 0] & flag) != 0).astype(np.uint8),
                     np.ascontiguousarray(rec[:, 1:]).view(np.complex128).reshape(-1).copy())
