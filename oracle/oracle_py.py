"""ctypes access to the parity checkers.  TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline / ``--impl reference``
legs import this module.  The product (``paper_2411_15332_b200``) never does.

Two checkers live here:

* ``Oracle``   -- our C restatement ``oracle/liboracle.so`` (built from ``qcs_oracle.c``);
* ``Reference`` -- the UNMODIFIED reference library compiled from /root/reference/proj/src into
  ``oracle/_ref/libqcsim_ref.so`` (``oracle/ref_capi.cpp`` marshals arguments only).  It exists on
  a GPU box only when it was built here and shipped with the snapshot; callers must tolerate
  ``Reference.available() == False``.

Complex arrays are numpy ``complex128`` (byte-identical to ``std::complex<double>``).
Placements are ``(qubits, matrix)`` pairs: ``qubits`` is the list of reference qubit indices in
gate-local order (qubit 0 = most significant basis bit), ``matrix`` a ``2^k x 2^k`` complex array.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libqcsim_ref.so")
IO_SO = os.path.join(HERE, "_ref", "libqcsim_io.so")

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_cp = np.ctypeslib.ndpointer(dtype=np.complex128, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")


def flatten_placements(placements):
    """-> (np, arity[int32], qubits[int32], mats[complex128 flat]) in the C-ABI layout."""
    arity = np.array([len(q) for q, _ in placements], dtype=np.int32)
    qubits = np.array([x for q, _ in placements for x in q], dtype=np.int32)
    mats = [np.ascontiguousarray(m, dtype=np.complex128).reshape(-1) for _, m in placements]
    for (q, m), flat in zip(placements, mats):
        if flat.size != 4 ** len(q):
            raise ValueError("matrix size does not match arity")
    mats = np.concatenate(mats) if mats else np.zeros(0, np.complex128)
    if qubits.size == 0:
        qubits = np.zeros(1, np.int32)
    if arity.size == 0:
        arity = np.zeros(1, np.int32)
    if mats.size == 0:
        mats = np.zeros(1, np.complex128)
    return len(placements), arity, qubits, np.ascontiguousarray(mats)


class OracleError(RuntimeError):
    pass


class Oracle:
    """The C restatement (qcs_oracle.c)."""

    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            if not os.path.exists(ORACLE_SO):
                raise OracleError(f"{ORACLE_SO} missing: run `make -C oracle oracle`")
            L = C.CDLL(ORACLE_SO)
            L.orc_step_row_capacity.restype = C.c_long
            L.orc_step_row_capacity.argtypes = [C.c_int, C.c_int, _ip, _ip, _cp]
            L.orc_apply_step.restype = C.c_int
            L.orc_apply_step.argtypes = [C.c_int, C.c_int, _ip, _ip, _cp, _cp, _cp]
            L.orc_step_dax.restype = C.c_long
            L.orc_step_dax.argtypes = [C.c_int, C.c_int, _ip, _ip, _cp, _u64p, _u64p, _cp, C.c_long]
            L.orc_step_das.restype = C.c_long
            L.orc_step_das.argtypes = [C.c_int, C.c_int, _ip, _ip, _cp, _u64p, _u8p, _cp, C.c_long]
            L.orc_dax_mvm.restype = C.c_int
            L.orc_dax_mvm.argtypes = [C.c_int, _u64p, _u64p, _cp, C.c_long, _cp, _cp]
            L.orc_das_mvm.restype = C.c_int
            L.orc_das_mvm.argtypes = [C.c_int, _u64p, _u8p, _cp, C.c_long, _cp, _cp]
            L.orc_apply_diag.restype = C.c_int
            L.orc_apply_diag.argtypes = [C.c_int, _u64p, C.c_uint64, C.c_int, _cp, _cp]
            L.orc_rh_mvm.restype = C.c_int
            L.orc_rh_mvm.argtypes = [C.c_int, _cp, _cp]
            L.orc_wht.restype = C.c_int
            L.orc_wht.argtypes = [C.c_int, _cp, _cp]
            L.orc_norm.restype = C.c_double
            L.orc_norm.argtypes = [C.c_int, _cp]
            L.orc_probabilities.restype = None
            L.orc_probabilities.argtypes = [C.c_int, _cp, _dp]
            cls._lib = L
        return cls._lib

    @classmethod
    def apply_step(cls, n, placements, state):
        L = cls.lib()
        npl, ar, qb, mt = flatten_placements(placements)
        out = np.empty_like(state)
        rc = L.orc_apply_step(n, npl, ar, qb, mt, np.ascontiguousarray(state), out)
        if rc:
            raise OracleError(f"orc_apply_step rc={rc}")
        return out

    @classmethod
    def step_dax(cls, n, placements):
        L = cls.lib()
        npl, ar, qb, mt = flatten_placements(placements)
        cap = L.orc_step_row_capacity(n, npl, ar, qb, mt) << n
        rows = np.empty(cap, np.uint64)
        cols = np.empty(cap, np.uint64)
        vals = np.empty(cap, np.complex128)
        cnt = L.orc_step_dax(n, npl, ar, qb, mt, rows, cols, vals, cap)
        if cnt < 0:
            raise OracleError(f"orc_step_dax rc={cnt}")
        return rows[:cnt].copy(), cols[:cnt].copy(), vals[:cnt].copy()

    @classmethod
    def step_das(cls, n, placements):
        L = cls.lib()
        npl, ar, qb, mt = flatten_placements(placements)
        cap = L.orc_step_row_capacity(n, npl, ar, qb, mt) << n
        dis = np.empty(cap, np.uint64)
        last = np.empty(cap, np.uint8)
        vals = np.empty(cap, np.complex128)
        cnt = L.orc_step_das(n, npl, ar, qb, mt, dis, last, vals, cap)
        if cnt == -3:
            raise OracleError("DAS cannot represent an all-zero row")
        if cnt < 0:
            raise OracleError(f"orc_step_das rc={cnt}")
        return dis[:cnt].copy(), last[:cnt].copy(), vals[:cnt].copy()

    @classmethod
    def dax_mvm(cls, n, rows, cols, vals, state):
        out = np.empty(1 << n, np.complex128)
        rc = cls.lib().orc_dax_mvm(n, rows, cols, vals, len(rows), np.ascontiguousarray(state), out)
        if rc:
            raise OracleError(f"orc_dax_mvm rc={rc}")
        return out

    @classmethod
    def das_mvm(cls, n, dis, last, vals, state):
        out = np.empty(1 << n, np.complex128)
        rc = cls.lib().orc_das_mvm(n, dis, last, vals, len(dis), np.ascontiguousarray(state), out)
        if rc:
            raise OracleError(f"orc_das_mvm rc={rc}")
        return out

    @classmethod
    def apply_diag(cls, n, flipped, flip_rest, state):
        f = np.ascontiguousarray(np.sort(np.asarray(flipped, dtype=np.uint64)))
        if f.size == 0:
            f = np.zeros(0, np.uint64)
        out = np.empty_like(state)
        rc = cls.lib().orc_apply_diag(n, f if f.size else np.zeros(1, np.uint64), f.size, int(flip_rest),
                                      np.ascontiguousarray(state), out)
        if rc:
            raise OracleError(f"orc_apply_diag rc={rc}")
        return out

    @classmethod
    def rh_mvm(cls, n, state):
        out = np.empty_like(state)
        rc = cls.lib().orc_rh_mvm(n, np.ascontiguousarray(state), out)
        if rc:
            raise OracleError(f"orc_rh_mvm rc={rc}")
        return out

    @classmethod
    def wht(cls, n, state):
        out = np.empty_like(state)
        rc = cls.lib().orc_wht(n, np.ascontiguousarray(state), out)
        if rc:
            raise OracleError(f"orc_wht rc={rc}")
        return out

    @classmethod
    def norm(cls, n, state):
        return cls.lib().orc_norm(n, np.ascontiguousarray(state))

    @classmethod
    def probabilities(cls, n, state):
        p = np.empty(1 << n, np.float64)
        cls.lib().orc_probabilities(n, np.ascontiguousarray(state), p)
        return p


class Reference:
    """The reference library itself (oracle/_ref/libqcsim_ref.so), when it was built."""

    _lib = None
    ENGINES = {"dense": 0, "dax": 1, "das": 2, "rh-dax": 3}
    SIGN_METHODS = {"nonopt": 0, "quarter": 1, "block": 2, "logarithm": 3}

    @staticmethod
    def available():
        return os.path.exists(REF_SO)

    @classmethod
    def lib(cls):
        if cls._lib is None:
            if not cls.available():
                raise OracleError(f"{REF_SO} missing: build with `make -C oracle ref` where /root/reference exists")
            L = C.CDLL(REF_SO)
            L.ref_last_error.restype = C.c_char_p
            L.ref_catalog_size.restype = C.c_int
            L.ref_catalog_entry.argtypes = [C.c_int, C.c_char_p, C.c_int, C.POINTER(C.c_int),
                                            C.POINTER(C.c_int), C.POINTER(C.c_double)]
            L.ref_gate_lookup.argtypes = [C.c_char_p, _dp, C.c_int, _cp, C.POINTER(C.c_int)]
            L.ref_canonical_params.argtypes = [C.c_char_p, _dp, C.POINTER(C.c_int)]
            L.ref_step_dax.restype = C.c_long
            L.ref_step_dax.argtypes = [C.c_int, C.c_int, _ip, _ip, _cp, _u64p, _u64p, _cp, C.c_long]
            L.ref_step_dump.restype = C.c_long
            L.ref_step_dump.argtypes = [C.c_int, C.c_int, _ip, _ip, _cp, C.c_int, C.c_char_p, C.c_long]
            L.ref_step_das.restype = C.c_long
            L.ref_step_das.argtypes = [C.c_int, C.c_int, _ip, _ip, _cp, _u64p, _u8p, _cp, C.c_long]
            L.ref_apply_step.argtypes = [C.c_int, C.c_int, _ip, _ip, _cp, C.c_int, _cp, _cp,
                                         C.POINTER(C.c_double), C.POINTER(C.c_double)]
            L.ref_dax_mvm.argtypes = [C.c_int, _u64p, _u64p, _cp, C.c_long, _cp, _cp]
            L.ref_das_mvm.argtypes = [C.c_int, _u64p, _u8p, _cp, C.c_long, _cp, _cp]
            L.ref_rh_mvm.argtypes = [C.c_int, _cp, _cp, C.c_int, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
            L.ref_simulate.argtypes = [C.c_int, C.c_uint64, C.c_int, _ip, _ip, _ip, _ip, _ip, _cp,
                                       C.POINTER(C.c_char_p), _u64p, _u64p, _ip, C.c_int, C.c_int, _cp,
                                       _u64p, C.POINTER(C.c_double)]
            L.ref_grover.argtypes = [C.c_int, C.c_uint64, C.c_int, C.c_int, _cp, C.POINTER(C.c_int)]
            L.ref_grover_auto_iterations.restype = C.c_uint64
            L.ref_grover_auto_iterations.argtypes = [C.c_int]
            L.ref_qnn.argtypes = [C.c_int, _dp, _ip, C.c_int, _cp, C.POINTER(C.c_int)]
            L.ref_random_unit_state.restype = None
            L.ref_random_unit_state.argtypes = [C.c_int, C.c_uint64, _cp]
            L.ref_quadrant_sign.argtypes = [C.c_uint64, C.c_uint64, C.c_int]
            cls._lib = L
        return cls._lib

    @classmethod
    def _check(cls, rc, what):
        if rc:
            raise OracleError(f"{what}: rc={rc}: {cls.lib().ref_last_error().decode()}")

    @classmethod
    def catalog(cls):
        L = cls.lib()
        out = []
        buf = C.create_string_buffer(64)
        for i in range(L.ref_catalog_size()):
            a, p, r = C.c_int(), C.c_int(), C.c_double()
            L.ref_catalog_entry(i, buf, 64, C.byref(a), C.byref(p), C.byref(r))
            out.append((buf.value.decode(), a.value, p.value, r.value))
        return out

    @classmethod
    def gate(cls, name, params=()):
        L = cls.lib()
        p = np.ascontiguousarray(np.asarray(params, dtype=np.float64).reshape(-1))
        out = np.zeros(64, np.complex128)
        ar = C.c_int()
        cls._check(L.ref_gate_lookup(name.encode(), p if p.size else np.zeros(1), p.size, out, C.byref(ar)),
                   f"gate {name}")
        d = 1 << ar.value
        return out[: d * d].reshape(d, d).copy()

    @classmethod
    def canonical_params(cls, name):
        out = np.zeros(8)
        k = C.c_int()
        cls._check(cls.lib().ref_canonical_params(name.encode(), out, C.byref(k)), name)
        return list(out[: k.value])

    @classmethod
    def step_dax(cls, n, placements):
        L = cls.lib()
        npl, ar, qb, mt = flatten_placements(placements)
        cap = 1
        for q, _ in placements:
            cap *= 1 << len(q)
        cap <<= n
        rows = np.empty(cap, np.uint64)
        cols = np.empty(cap, np.uint64)
        vals = np.empty(cap, np.complex128)
        cnt = L.ref_step_dax(n, npl, ar, qb, mt, rows, cols, vals, cap)
        if cnt < 0:
            raise OracleError(f"ref_step_dax rc={cnt}: {L.ref_last_error().decode()}")
        return rows[:cnt].copy(), cols[:cnt].copy(), vals[:cnt].copy()

    @classmethod
    def step_das(cls, n, placements):
        L = cls.lib()
        npl, ar, qb, mt = flatten_placements(placements)
        cap = 1
        for q, _ in placements:
            cap *= 1 << len(q)
        cap <<= n
        dis = np.empty(cap, np.uint64)
        last = np.empty(cap, np.uint8)
        vals = np.empty(cap, np.complex128)
        cnt = L.ref_step_das(n, npl, ar, qb, mt, dis, last, vals, cap)
        if cnt < 0:
            raise OracleError(f"ref_step_das rc={cnt}: {L.ref_last_error().decode()}")
        return dis[:cnt].copy(), last[:cnt].copy(), vals[:cnt].copy()

    @classmethod
    def step_dump(cls, n, placements, das=False):
        """dax_dump(step_matrix_dax(step)) / das_dump(step_matrix_das(step)) bytes (native steps)."""
        L = cls.lib()
        npl, ar, qb, mt = flatten_placements(placements)
        cap = 28
        ent = 1
        for q, _ in placements:
            ent *= 1 << len(q)
        cap += (24 if das else 32) * (ent << n)
        buf = C.create_string_buffer(cap)
        k = L.ref_step_dump(n, npl, ar, qb, mt, 1 if das else 0, buf, cap)
        if k < 0:
            raise OracleError(f"ref_step_dump rc={k}: {L.ref_last_error().decode()}")
        return buf.raw[:k]

    @classmethod
    def apply_step(cls, n, placements, state, engine="dax"):
        """-> (out_state, t_build_s, t_mvm_s): step_matrix_{dax,das} then {dax,das}_mvm."""
        L = cls.lib()
        npl, ar, qb, mt = flatten_placements(placements)
        out = np.empty_like(state)
        tb, tm = C.c_double(), C.c_double()
        cls._check(L.ref_apply_step(n, npl, ar, qb, mt, 2 if engine == "das" else 1,
                                    np.ascontiguousarray(state), out, C.byref(tb), C.byref(tm)),
                   "ref_apply_step")
        return out, tb.value, tm.value

    @classmethod
    def dax_mvm(cls, n, rows, cols, vals, state):
        out = np.empty(1 << n, np.complex128)
        cls._check(cls.lib().ref_dax_mvm(n, rows, cols, vals, len(rows), np.ascontiguousarray(state), out),
                   "ref_dax_mvm")
        return out

    @classmethod
    def das_mvm(cls, n, dis, last, vals, state):
        out = np.empty(1 << n, np.complex128)
        cls._check(cls.lib().ref_das_mvm(n, dis, last, vals, len(dis), np.ascontiguousarray(state), out),
                   "ref_das_mvm")
        return out

    @classmethod
    def rh_mvm(cls, n, state, method="logarithm"):
        out = np.empty_like(state)
        sc, mc = C.c_uint64(), C.c_uint64()
        cls._check(cls.lib().ref_rh_mvm(n, np.ascontiguousarray(state), out, cls.SIGN_METHODS[method],
                                        C.byref(sc), C.byref(mc)), "ref_rh_mvm")
        return out, sc.value, mc.value

    @classmethod
    def simulate(cls, n, steps, engine="rh-dax", initial=0, sign_method="logarithm"):
        """steps: list of ('gates', [(name, qubits, matrix), ...], stage) or
        ('diag', flipped, flip_rest, stage).  Returns (final_state, reports, seconds)."""
        L = cls.lib()
        kind, stage, nplace, arity, qubits, mats, names, nflip, flipped, frest = ([] for _ in range(10))
        for st in steps:
            if st[0] == "diag":
                kind.append(1)
                stage.append(st[3] if len(st) > 3 else 0)
                nplace.append(0)
                nflip.append(len(st[1]))
                flipped.extend(int(x) for x in st[1])
                frest.append(int(st[2]))
            else:
                kind.append(0)
                stage.append(st[2] if len(st) > 2 else 0)
                nplace.append(len(st[1]))
                nflip.append(0)
                frest.append(0)
                for name, q, m in st[1]:
                    arity.append(len(q))
                    qubits.extend(q)
                    mats.append(np.ascontiguousarray(m, np.complex128).reshape(-1))
                    names.append(name.encode())
        i32 = lambda v: np.ascontiguousarray(np.array(v if v else [0], dtype=np.int32))
        u64 = lambda v: np.ascontiguousarray(np.array(v if v else [0], dtype=np.uint64))
        mats = np.ascontiguousarray(np.concatenate(mats) if mats else np.zeros(1, np.complex128))
        name_arr = (C.c_char_p * max(1, len(names)))(*names)
        out = np.empty(1 << n, np.complex128)
        rep = np.zeros(6 * max(1, len(steps)), np.uint64)
        secs = C.c_double()
        cls._check(L.ref_simulate(n, initial, len(steps), i32(kind), i32(stage), i32(nplace), i32(arity),
                                  i32(qubits), mats, name_arr, u64(nflip), u64(flipped), i32(frest),
                                  cls.ENGINES[engine], cls.SIGN_METHODS[sign_method], out, rep,
                                  C.byref(secs)), "ref_simulate")
        structures = ["dense", "dax", "das", "rh"]
        reports = [dict(structure=structures[int(rep[6 * s + 5])], matrix_bytes=int(rep[6 * s]),
                        dense_bytes=int(rep[6 * s + 1]), entry_count=int(rep[6 * s + 2]),
                        sign_count=int(rep[6 * s + 3]), madd_count=int(rep[6 * s + 4]))
                   for s in range(len(steps))]
        return out, reports, secs.value

    @classmethod
    def grover(cls, n, marked, iterations=0, engine="rh-dax"):
        out = np.empty(1 << n, np.complex128)
        ns = C.c_int()
        cls._check(cls.lib().ref_grover(n, marked, iterations, cls.ENGINES[engine], out, C.byref(ns)),
                   "ref_grover")
        return out

    @classmethod
    def grover_auto_iterations(cls, n):
        return int(cls.lib().ref_grover_auto_iterations(n))

    @classmethod
    def qnn(cls, angles, weights, engine="rh-dax"):
        L = cls.lib()
        k = len(angles)
        nq = C.c_int()
        # qnn_total_qubits: inputs + ceil(log2 inputs) + 1
        enc = 0
        while (1 << enc) < k:
            enc += 1
        out = np.empty(1 << (k + enc + 1), np.complex128)
        cls._check(L.ref_qnn(k, np.ascontiguousarray(angles, dtype=np.float64),
                             np.ascontiguousarray(weights, dtype=np.int32), cls.ENGINES[engine], out,
                             C.byref(nq)), "ref_qnn")
        return out

    @classmethod
    def random_unit_state(cls, n, seed):
        out = np.empty(1 << n, np.complex128)
        cls.lib().ref_random_unit_state(n, seed, out)
        return out

    @classmethod
    def quadrant_sign(cls, r, c, n):
        return cls.lib().ref_quadrant_sign(r, c, n)


class ReferenceIO:
    """The reference's front end (oracle/_ref/libqcsim_io.so: circuit_io.cpp + the engine)."""

    _lib = None

    @staticmethod
    def available():
        return os.path.exists(IO_SO)

    @classmethod
    def lib(cls):
        if cls._lib is None:
            if not cls.available():
                raise OracleError(f"{IO_SO} missing: build with `make -C oracle io` where /root/reference exists")
            L = C.CDLL(IO_SO)
            L.io_last_error.restype = C.c_char_p
            L.io_sample.restype = C.c_long
            L.io_sample.argtypes = [C.c_int, _cp, C.c_int, C.c_ulonglong, _u64p]
            cls._lib = L
        return cls._lib

    @classmethod
    def sample(cls, n, amps, count, seed):
        """render_report's samples (circuit_io.cpp:114-128) for the state `amps`."""
        out = np.zeros(max(count, 1), np.uint64)
        k = cls.lib().io_sample(n, np.ascontiguousarray(amps, np.complex128), count, seed, out)
        if k < 0:
            raise OracleError(f"io_sample rc={k}: {cls.lib().io_last_error().decode()}")
        return [int(x) for x in out[:k]]


# ------------------------------------------------------------ sampling restatement (pure Python)
class MT19937_64:
    """std::mt19937_64 (the reference seeds it with the report seed, circuit_io.cpp:116)."""

    def __init__(self, seed: int):
        self.mt = [0] * 312
        self.mt[0] = seed & 0xFFFFFFFFFFFFFFFF
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & 0xFFFFFFFFFFFFFFFF
        self.i = 312

    def __call__(self) -> int:
        if self.i >= 312:
            mt = self.mt
            for k in range(312):
                y = (mt[k] & 0xFFFFFFFF80000000) | (mt[(k + 1) % 312] & 0x7FFFFFFF)
                v = mt[(k + 156) % 312] ^ (y >> 1)
                if y & 1:
                    v ^= 0xB5026F5AA96619E9
                mt[k] = v
            self.i = 0
        y = self.mt[self.i]
        self.i += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & 0xFFFFFFFFFFFFFFFF


def _uniform(rng, hi):
    """uniform_real_distribution<double>(0, hi) over generate_canonical<double, 53> (libstdc++)."""
    import math
    c = float(rng()) / 18446744073709551616.0
    if c >= 1.0:
        c = math.nextafter(1.0, 0.0)
    return (hi - 0.0) * c + 0.0


def sequential_sample(probs, count, seed):
    """circuit_io.cpp:114-128 restated: sequential rounded CDF, lower_bound per draw."""
    rng = MT19937_64(seed)
    cdf = np.empty(len(probs), np.float64)
    acc = 0.0
    for i, p in enumerate(np.asarray(probs, np.float64).tolist()):
        acc += p
        cdf[i] = acc
    return [int(np.searchsorted(cdf, _uniform(rng, acc), side="left")) for _ in range(count)], acc
