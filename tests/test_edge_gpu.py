"""Edge cases through the B200 engine against the oracle: empty and one-qubit circuits,
non-zero initial basis states, degenerate sign steps, and fused random circuits over the whole
catalog on multi-tile states (shared-memory gate rounds, controls inside and outside the
tile, bundles, missed-tile programs).  Bars as in test_parity_gpu.py."""
import numpy as np
import pytest

from conftest import bits_equal, canon_zero

pytestmark = pytest.mark.gpu

TOL_AMP = 1e-12
TOL_L2 = 1e-10


@pytest.fixture(scope="module")
def Q():
    from paper_2411_15332_b200 import qcsim
    return qcsim


def oracle_run(oracle, c):
    x = np.zeros(1 << c.n, np.complex128)
    x[c.initial] = 1
    for st in c.steps:
        if int(st.kind) == 1:
            x = oracle.apply_diag(c.n, sorted(set(st.diag.flipped)), st.diag.flip_rest, x)
        elif st.is_hadamard_all(c.n):
            x = oracle.wht(c.n, x)
        else:
            x = oracle.apply_step(c.n, [(p.qubit_list(), p.gate.matrix) for p in st.placements], x)
    return x


def test_empty_circuit_is_the_basis_state(Q):
    for n, init in ((1, 0), (1, 1), (9, 300), (13, 8191)):
        rep = Q.simulate(Q.Circuit(n, [], init), Q.Engine.rh_dax)
        want = np.zeros(1 << n, np.complex128)
        want[init] = 1
        assert bits_equal(rep.final.download(), want)
        assert rep.steps == [] and rep.total_madd_count == 0


@pytest.mark.parametrize("engine", ["dense", "dax", "das", "rh_dax"])
def test_one_qubit_circuits(Q, oracle, engine):
    G = Q.gate_catalog_lookup
    for init in (0, 1):
        c = Q.Circuit(1, [Q.hadamard_all(1), Q.CircuitStep.of_gates([Q.Placement(G("T"), 0)]),
                          Q.CircuitStep.of_diag(Q.DiagSign([1], False)), Q.hadamard_all(1),
                          Q.CircuitStep.of_gates([Q.Placement(G("RY", [0.4]), 0)])], init)
        want = oracle_run(oracle, c)
        for fuse in (False, True):
            got = Q.simulate(c, getattr(Q.Engine, engine), Q.SimOptions(fuse=fuse)).final.download()
            assert np.abs(got - want).max() <= TOL_AMP, (engine, init, fuse)


def test_degenerate_sign_steps(Q, oracle):
    """Duplicated indices flip once, an empty list without flip_rest is the identity, an empty
    list with flip_rest negates everything: bit-exact one step at a time, within the bar fused
    between other steps."""
    from conftest import random_state
    n = 14
    rng = np.random.default_rng(9)
    signs = [Q.DiagSign([5, 5, 77, 5], False), Q.DiagSign([], False), Q.DiagSign([], True),
             Q.DiagSign([int(i) for i in rng.choice(1 << n, 200, replace=False)], True)]
    x = random_state(n, 21)
    s = Q.DeviceState.from_numpy(x)
    want = x
    for d in signs:
        s.apply_diag(d)
        want = oracle.apply_diag(n, sorted(set(d.flipped)), d.flip_rest, want)
        assert bits_equal(s.download(), want)
    steps = [Q.hadamard_all(n)] + [Q.CircuitStep.of_diag(d) for d in signs[:3]]
    steps += [Q.CircuitStep.of_gates([Q.Placement(Q.gate_catalog_lookup("RX", [0.9]), 3)]),
              Q.CircuitStep.of_diag(signs[3]), Q.hadamard_all(n)]
    c = Q.Circuit(n, steps, 17)
    want = oracle_run(oracle, c)
    for fuse in (True, False):
        got = Q.simulate(c, Q.Engine.rh_dax, Q.SimOptions(fuse=fuse)).final.download()
        assert np.abs(got - want).max() <= TOL_AMP, fuse


@pytest.mark.parametrize("seed", range(4))
def test_random_catalog_circuits_fused(Q, oracle, seed):
    """Random circuits over all 38 catalog gates (any arity, reversed / non-adjacent qubits) on
    n = 13..17: several 12-bit tiles, so every kind of tile operation and round meets tile
    boundaries.  Fused and stepwise against the oracle."""
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(13, 18))
    infos = Q.gate_catalog()
    steps = [Q.hadamard_all(n)]
    for _ in range(40):
        used, pl = set(), []
        for _ in range(int(rng.integers(1, 4))):
            info = infos[int(rng.integers(0, len(infos)))]
            free = [q for q in range(n) if q not in used]
            if len(free) < info.arity:
                break
            qs = [int(q) for q in rng.choice(free, info.arity, replace=False)]
            used.update(qs)
            g = Q.gate_catalog_lookup(info.name, list(rng.uniform(0, 2 * np.pi, info.param_count)))
            pl.append(Q.Placement(g, qubits=qs))
        if pl:
            steps.append(Q.CircuitStep.of_gates(pl))
        if rng.random() < 0.15:
            steps.append(Q.CircuitStep.of_diag(Q.DiagSign([int(rng.integers(0, 1 << n))], bool(rng.random() < 0.5))))
    c = Q.Circuit(n, steps, int(rng.integers(0, 1 << n)))
    want = oracle_run(oracle, c)
    for fuse in (True, False):
        got = Q.simulate(c, Q.Engine.rh_dax, Q.SimOptions(fuse=fuse)).final.download()
        assert np.abs(got - want).max() <= TOL_AMP, fuse
        assert np.linalg.norm(got - want) <= TOL_L2, fuse


def test_abi_argument_errors(Q):
    """The B200-only entry points fail loudly on bad arguments (status codes, no crash)."""
    import ctypes as C
    L = Q.L
    lib = L.lib()
    s = Q.DeviceState(6)
    buf = np.zeros(2 << 6)
    rc = lib.qcs_state_download_async(s.handle, buf.ctypes.data_as(C.c_void_p), 0, 1 << 6)
    assert rc == L.QCS_ERR_ARG  # pageable memory: only pinned buffers may be read back asynchronously
    hp = C.c_void_p()
    Q._check(lib.qcs_host_alloc(16 << 6, C.byref(hp)))
    try:
        Q._check(lib.qcs_state_download_async(s.handle, hp, 0, 1 << 6))
        s.sync()
    finally:
        lib.qcs_host_free(hp)
    blocks = np.eye(2, dtype=np.complex128).reshape(1, 2, 2)
    bp = blocks.ctypes.data_as(C.POINTER(C.c_double))
    assert lib.qcs_apply_split(s.handle, None, 0, 0, None, bp, 0) == L.QCS_ERR_ARG
    import torch
    t = torch.zeros(1 << 6, dtype=torch.complex128, device="cuda")  # a partner shard
    assert lib.qcs_apply_split(s.handle, C.c_void_p(t.data_ptr()), 2, 0, None, bp, 0) == L.QCS_ERR_ARG
    sel = (C.c_int * 1)(9)
    assert lib.qcs_apply_split(s.handle, C.c_void_p(t.data_ptr()), 0, 1, sel, bp, 0) == L.QCS_ERR_DIMENSION
    assert lib.qcs_apply_split(s.handle, C.c_void_p(t.data_ptr()), 0, 3, sel, bp, 0) == L.QCS_ERR_ARG


def test_state_wait_orders_streams(Q, oracle):
    """qcs_state_wait: B's work waits for A's (device-side); both results as computed alone."""
    n = 20
    a, b = Q.DeviceState(n), Q.DeviceState(n)
    a.randomize(7)
    b.randomize(7)
    want = a.download()
    h = Q.gate_catalog_lookup("Hadamard")
    for q in range(n):
        a.apply_gate(h, [q])
    b.wait_for(a)
    b.wait_for(b)  # waiting on itself is a no-op
    for q in range(n):
        b.apply_gate(h, [q])
    b.wait_for(a)
    for q in range(n):
        b.apply_gate(h, [q])
    got_b = b.download()
    assert np.abs(got_b - want).max() <= 1e-12  # H^n H^n = I
    assert np.abs(a.download() - oracle.wht(n, want)).max() <= 1e-12
    a.close()
    b.close()


def test_plan_cache_reuse_and_invalidation(Q, oracle):
    """simulate() on the same state reuses a circuit's plan (and its uploaded tables) when the
    steps repeat exactly; a changed angle, another circuit in between, or a new jit mode plans
    afresh.  Every result against the oracle."""
    n = 14
    G = Q.gate_catalog_lookup

    def circ(theta):
        return Q.Circuit(n, [Q.hadamard_all(n), Q.CircuitStep.of_gates(
            [Q.Placement(G("RY", [theta]), q) for q in range(n)]), Q.CircuitStep.of_gates(
            [Q.Placement(G("Controlled-X"), q) for q in range(0, n - 1, 2)])], 3)

    def want(c):
        return oracle_run(oracle, c)

    st = Q.DeviceState(n)
    a, b = circ(0.3), circ(0.7)
    wa, wb = want(a), want(b)
    old = Q.jit_mode()
    try:
        for c, w in ((a, wa), (a, wa), (b, wb), (a, wa), (b, wb), (b, wb)):
            rep = Q.simulate(c, Q.Engine.rh_dax, state=st)
            assert np.abs(st.download() - w).max() <= TOL_AMP
            assert len(rep.steps) == 3
        Q.set_jit_mode(2 if old != 2 else 0)
        Q.simulate(a, Q.Engine.rh_dax, state=st)
        assert np.abs(st.download() - wa).max() <= TOL_AMP
    finally:
        Q.set_jit_mode(old)
    st.close()


@pytest.mark.parametrize("seed", range(6))
def test_light_cone_planner_random_layers(Q, oracle, seed):
    """The round-2 planner on layered circuits it reorders: random one-qubit catalog gates on
    every qubit per layer, then diagonal couplings (CZ, CPhase, RZZ, CRZ, CU1) on random pairs --
    the light-cone round scheduler, 16-register rounds, scale chaining, table normalisation and
    the tile search all engage.  Against the oracle at n = 14..20, default jit mode and every
    pass specialised (mode 3)."""
    rng = np.random.default_rng(900 + seed)
    n = int(rng.integers(14, 21))
    one = [i for i in Q.gate_catalog() if i.arity == 1]
    diag2 = ["Controlled-Z", "CPhase", "RZZ", "CRZ", "CU1"]
    steps = [Q.hadamard_all(n)]
    for _ in range(int(rng.integers(3, 7))):
        pl = []
        for q in range(n):
            info = one[int(rng.integers(0, len(one)))]
            pl.append(Q.Placement(Q.gate_catalog_lookup(info.name, list(rng.uniform(0, 2 * np.pi, info.param_count))), q))
        steps.append(Q.CircuitStep.of_gates(pl))
        perm = [int(x) for x in rng.permutation(n)]
        for k in range(0, n - 1, 2):
            name = diag2[int(rng.integers(0, len(diag2)))]
            info = next(i for i in Q.gate_catalog() if i.name == name)
            g = Q.gate_catalog_lookup(name, list(rng.uniform(0, 2 * np.pi, info.param_count)))
            steps.append(Q.CircuitStep.of_gates([Q.Placement(g, qubits=[perm[k], perm[k + 1]])]))
    c = Q.Circuit(n, steps, 0)
    want = oracle_run(oracle, c)
    old = Q.jit_mode()
    try:
        for mode in (1, 3):
            Q.set_jit_mode(mode)
            got = Q.simulate(c, Q.Engine.rh_dax).final.download()
            assert np.abs(got - want).max() <= TOL_AMP, (mode, n)
            assert np.linalg.norm(got - want) <= TOL_L2, (mode, n)
    finally:
        Q.set_jit_mode(old)
    st = Q.plan_stats(c)
    assert st["tile_passes"] >= 1 and Q.plan_verify(c) >= 1
