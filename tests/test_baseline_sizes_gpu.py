"""Parity at the BASELINE.json sizes (VERDICT r1 "next round" item 1).

- C3 (configs[2]): 30-qubit Grover, 8 iterations, against the closed form of SURVEY.md section 8c
  (a_marked = sin((2k+1)t), a_other = cos((2k+1)t)/sqrt(2^n - 1), t = asin(2^{-n/2})), which
  follows the reference's Z0 semantics (circuit.cpp:92).
- C2 (configs[1]): the 28-qubit single-gate sweep at targets {0, 13, 27} for all 12 gates,
  bit-exact against the oracle's streaming dax_mvm (oracle/qcs_oracle.c, dax.cpp:96-103).
- C4 (configs[3]) and the C5 family at n=32 (64 GiB states): no CPU oracle fits, so the default
  fused engine is checked against the per-gate kernels (each bit-exact against the oracle at
  n <= 28, test_parity_gpu.py) and against the interpreter kernel (jit mode 0), compared on the
  device (qcs_state_distance) within the north-star tolerance, plus the norm.
"""
import numpy as np
import pytest

from conftest import bits_equal

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

TOL_AMP = 1e-12
TOL_L2 = 1e-10


@pytest.fixture(scope="module")
def Q():
    from paper_2411_15332_b200 import qcsim
    return qcsim


@pytest.fixture(scope="module")
def cfg():
    from paper_2411_15332_b200 import configs
    return configs


def free_bytes():
    import torch
    free, _ = torch.cuda.mem_get_info(0)
    return free


def test_c3_grover_n30_closed_form(Q, cfg):
    n, k = 30, 8
    marked = cfg.c3_marked(n)
    c = cfg.c3_circuit(n, k)
    rep = Q.simulate(c, Q.Engine.rh_dax)
    a_m, a_o = cfg.grover_closed_form(n, k)
    rng = np.random.default_rng(30)
    idx = [marked, 0, (1 << n) - 1, marked ^ 1, marked ^ (1 << (n - 1))]
    idx += [int(v) for v in rng.integers(0, 1 << n, 59)]
    idx = np.array(idx, np.uint64)
    got = rep.final.gather(idx)
    want = np.where(idx == marked, a_m, a_o).astype(np.complex128)
    assert np.abs(got - want).max() <= TOL_AMP
    i, p = rep.final.argmax()
    assert i == marked and abs(p - a_m * a_m) <= 1e-12
    assert abs(rep.final.norm() - 1.0) <= 1e-12
    rep.final.close()


def test_c2_sweep_n28_sampled_targets_bit_exact(Q, cfg, oracle):
    n = 28
    s = Q.DeviceState(n)
    s.randomize(cfg.seed_of(2))
    x = s.download()
    done = set()
    for g in cfg.c2_sweep(n, seed=cfg.seed_of(2)):
        if g.qubits[-1] not in (0, 13, 27):
            continue
        s.upload(x)
        s.apply_gate(g.gate, g.qubits)
        got = s.download()
        want = oracle.apply_step(n, [(g.qubits, g.gate.matrix)], x)
        assert bits_equal(got, want), (g.label, g.qubits, float(np.abs(got - want).max()))
        done.add(g.label)
        del got, want
    assert done == set(cfg.C2_GATES)
    s.close()


def per_gate(Q, c, state):
    """The circuit step by step through the per-gate kernels (one HBM pass per gate, dax_mvm's
    arithmetic) and the RH butterflies; no fusion across gates."""
    state.set_basis(c.initial)
    for st in c.steps:
        if st.is_hadamard_all(c.n):
            state.apply_rh()
        elif int(st.kind) == 1:
            state.apply_diag(st.diag)
        else:
            for p in st.placements:
                state.apply_gate(p.gate, p.qubit_list())


@pytest.mark.parametrize("family", ["c4", "c5"])
def test_n32_fused_vs_per_gate_vs_interpreter(Q, cfg, family):
    n = 32
    if free_bytes() < 2 * (16 << n) + (4 << 30):
        pytest.skip("two 64 GiB states do not fit")
    c = cfg.c4_circuit(n) if family == "c4" else cfg.c5_circuit(n, global_qubits=3)
    a = Q.DeviceState(n)
    b = Q.DeviceState(n)
    try:
        Q.simulate(c, Q.Engine.rh_dax, state=a)  # the default: fused, specialised pass kernels
        assert abs(a.norm() - 1.0) <= 1e-12
        per_gate(Q, c, b)
        mx, l2 = a.distance(b)
        assert mx <= TOL_AMP and l2 <= TOL_L2, (family, "per-gate", mx, l2)
        old = Q.jit_mode()
        try:
            Q.set_jit_mode(0)  # every pass on the interpreter kernel
            Q.simulate(c, Q.Engine.rh_dax, state=b)
        finally:
            Q.set_jit_mode(old)
        mx, l2 = a.distance(b)
        assert mx <= TOL_AMP and l2 <= TOL_L2, (family, "interpreter", mx, l2)
        # a few amplitudes read back through the ordinary path agree as well
        idx = np.array([0, 1, 12345, (1 << n) - 1], np.uint64)
        assert np.abs(a.gather(idx) - b.gather(idx)).max() <= TOL_AMP
    finally:
        a.close()
        b.close()


def test_state_distance_small(Q):
    from conftest import random_state
    x = random_state(10, 1)
    y = x.copy()
    y[17] += 1e-3j
    a, b = Q.DeviceState.from_numpy(x), Q.DeviceState.from_numpy(y)
    mx, l2 = a.distance(b)
    assert abs(mx - 1e-3) < 1e-15 and abs(l2 - 1e-3) < 1e-15
    assert a.distance(a) == (0.0, 0.0)


@pytest.mark.parametrize("initial", [0, (1 << 23) - 1, (0b101 << 21) | 0x1234])
def test_deferred_qubits_from_any_basis_state(Q, cfg, initial):
    """n = 24 (the planner defers the top qubits of a layered nearest-neighbour circuit run from a
    basis state: the operations outside their light cone run first, on the sub-cube the state is
    still confined to).  The fused result must equal the per-gate kernels' -- which run the steps
    in circuit order on the whole state -- within the 1e-12 bar, whatever the basis state's bits
    on the deferred qubits; and with fewer layers than the ring is long the plan does defer
    (fewer FP64 instructions per amplitude than gates would cost on the whole state)."""
    n = 24
    c = cfg.c4_circuit(n, layers=6)
    c.initial = initial
    st = Q.plan_stats(c)
    gates = sum(len(s.placements) for s in c.steps if int(s.kind) == 0 and not s.is_hadamard_all(n))
    assert st["fp64_ops"] / float(1 << n) < 0.9 * (2.0 * 6 * n), (st, gates)  # RY alone would cost 2 per qubit-layer
    a = Q.DeviceState(n)
    b = Q.DeviceState(n)
    try:
        Q.simulate(c, Q.Engine.rh_dax, state=a)
        assert abs(a.norm() - 1.0) <= 1e-12
        per_gate(Q, c, b)
        mx, l2 = a.distance(b)
        assert mx <= TOL_AMP and l2 <= TOL_L2, (initial, mx, l2)
    finally:
        a.close()
        b.close()


@pytest.mark.parametrize("seed", range(4))
def test_deferred_qubits_random_chain_circuits(Q, seed):
    """Random layered circuits on a chain at n = 21..23: any one-qubit catalog gate on every qubit
    per layer (X-like, diagonal, dense, complex), then random diagonal couplings on
    nearest-neighbour pairs (a few of them long-range), from a random basis state.  Few layers
    against the chain's length, so the planner defers the top qubits; fused vs the per-gate
    kernels within 1e-12."""
    rng = np.random.default_rng(4200 + seed)
    n = int(rng.integers(21, 24))
    one = [i for i in Q.gate_catalog() if i.arity == 1]
    diag2 = ["Controlled-Z", "CPhase", "RZZ", "CRZ", "CU1"]
    steps = [Q.hadamard_all(n)] if seed % 2 == 0 else []
    for _ in range(int(rng.integers(3, 6))):
        pl = []
        for q in range(n):
            info = one[int(rng.integers(0, len(one)))]
            pl.append(Q.Placement(Q.gate_catalog_lookup(info.name, list(rng.uniform(0, 2 * np.pi, info.param_count))), q))
        steps.append(Q.CircuitStep.of_gates(pl))
        for start in (0, 1):
            for q in range(start, n - 1, 2):
                name = diag2[int(rng.integers(0, len(diag2)))]
                info = next(i for i in Q.gate_catalog() if i.name == name)
                g = Q.gate_catalog_lookup(name, list(rng.uniform(0, 2 * np.pi, info.param_count)))
                far = int(rng.integers(0, n)) if rng.random() < 0.05 else q + 1
                if far == q:
                    far = q + 1
                steps.append(Q.CircuitStep.of_gates([Q.Placement(g, qubits=[q, far])]))
    c = Q.Circuit(n, steps, int(rng.integers(0, 1 << n)))
    a = Q.DeviceState(n)
    b = Q.DeviceState(n)
    try:
        Q.simulate(c, Q.Engine.rh_dax, state=a)
        per_gate(Q, c, b)
        mx, l2 = a.distance(b)
        assert mx <= TOL_AMP and l2 <= TOL_L2, (seed, n, mx, l2)
    finally:
        a.close()
        b.close()


def test_c4_n33_fills_the_hbm(Q, cfg):
    """A 33-qubit state (128 GiB: updates are in place, one buffer per state) on one 180 GB B200:
    the C4 layers at n = 33 keep the norm to rounding, and a few amplitudes agree with the same
    circuit run with every pass on the interpreter kernel."""
    n = 33
    if free_bytes() < (16 << n) + (6 << 30):
        pytest.skip("a 128 GiB state does not fit")
    c = cfg.c4_circuit(n, layers=3)
    a = Q.DeviceState(n)
    try:
        Q.simulate(c, Q.Engine.rh_dax, state=a)
        assert abs(a.norm() - 1.0) <= 1e-12
        idx = np.array([0, 1, 12345, (1 << n) - 1, (1 << 32) + 77], np.uint64)
        got = a.gather(idx)
        old = Q.jit_mode()
        try:
            Q.set_jit_mode(0)
            Q.simulate(c, Q.Engine.rh_dax, state=a)
        finally:
            Q.set_jit_mode(old)
        assert np.abs(a.gather(idx) - got).max() <= TOL_AMP
    finally:
        a.close()
