"""GPU parity: the B200 engine (through the C ABI) against the pinned CPU oracle.

Bar (BASELINE.json north_star): bit-exact for compressed-gate index structures and
permutation-only gates; per-amplitude |delta| <= 1e-12 (L2 <= 1e-10) for floating-point gates.
Single-placement steps are bit-exact for every gate (the kernels use dax_mvm's arithmetic).
"""
import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, bits_equal, canon_zero, random_state

pytestmark = pytest.mark.gpu

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


def run_gate(Q, n, gate, qubits, x):
    s = Q.DeviceState.from_numpy(x)
    s.apply_gate(gate, qubits)
    return s.download()


# ------------------------------------------------------------------ single-gate sweep (C2)
@pytest.mark.parametrize("n", [6, 12, 18])
def test_c2_sweep_bit_exact(Q, cfg, oracle, n):
    x = random_state(n, 4242 + n)
    for g in cfg.c2_sweep(n, seed=cfg.seed_of(2)):
        got = run_gate(Q, n, g.gate, g.qubits, x)
        want = oracle.apply_step(n, [(g.qubits, g.gate.matrix)], x)
        assert bits_equal(got, want), (n, g.label, g.qubits, np.abs(got - want).max())


def test_c2_sweep_golden_n12(Q, golden):
    from paper_2411_15332_b200 import configs as cfg
    g = golden("sweep_n12.npz")
    s0 = g["state"]
    for i, sg in enumerate(cfg.c2_sweep(12, seed=cfg.seed_of(2))):
        got = run_gate(Q, 12, sg.gate, sg.qubits, s0)
        assert hashlib.sha256(got.tobytes()).hexdigest() == g["sha"][i], (sg.label, sg.qubits)


def test_c2_sweep_n24_sampled(Q, cfg, oracle):
    n = 24
    x = random_state(n, 24)
    sweep = cfg.c2_sweep(n, seed=cfg.seed_of(2))
    s = Q.DeviceState.from_numpy(x)
    for g in sweep:
        if g.qubits[-1] not in (0, 11, 23):
            continue
        s.upload(x)
        s.apply_gate(g.gate, g.qubits)
        want = oracle.apply_step(n, [(g.qubits, g.gate.matrix)], x)
        assert bits_equal(s.download(), want), (g.label, g.qubits)


def test_every_catalog_gate_every_placement(Q, oracle):
    """All 38 catalog gates at random angles, every ordered qubit tuple of n=5 (covers reversed
    and non-adjacent multi-qubit placements)."""
    import itertools
    n = 5
    x = random_state(n, 5)
    rng = np.random.default_rng(5)
    for info in Q.gate_catalog():
        g = Q.gate_catalog_lookup(info.name, list(rng.uniform(0, 2 * np.pi, info.param_count)))
        for qs in itertools.permutations(range(n), info.arity):
            got = run_gate(Q, n, g, list(qs), x)
            want = oracle.apply_step(n, [(list(qs), g.matrix)], x)
            assert bits_equal(canon_zero(got), canon_zero(want)), (info.name, qs)


def test_multi_placement_steps(Q, oracle):
    rng = np.random.default_rng(17)
    cat = [g for g in Q.gate_catalog()]
    for trial in range(40):
        n = int(rng.integers(3, 12))
        pl, q = [], 0
        exact = True
        while q < n:
            ar = 1 + int(rng.integers(0, min(n - q, 3)))
            fits = [c for c in cat if c.arity == ar]
            info = fits[int(rng.integers(0, len(fits)))]
            g = Q.gate_catalog_lookup(info.name, list(rng.uniform(0, 6.28, info.param_count)))
            pl.append(Q.Placement(g, q))
            vals = g.matrix[g.matrix != 0]
            exact &= bool(np.all(np.isin(vals, [1, -1, 1j, -1j])))
            q += ar + int(rng.integers(0, 2))
        x = random_state(n, trial)
        s = Q.DeviceState.from_numpy(x)
        s.apply_step(pl)
        got = s.download()
        want = oracle.apply_step(n, [(p.qubit_list(), p.gate.matrix) for p in pl], x)
        if exact:
            assert bits_equal(canon_zero(got), canon_zero(want))
        assert np.abs(got - want).max() <= TOL_AMP
        assert np.linalg.norm(got - want) <= TOL_L2


# ------------------------------------------------------------------ diagonal sign steps
def test_diag_steps_bit_exact(Q, oracle):
    n = 10
    x = random_state(n, 3)
    for flipped, rest in [([5], False), ([0], True), ([1, 7, 1023, 7], False), ([], True), ([3, 900], True)]:
        s = Q.DeviceState.from_numpy(x)
        s.apply_diag(Q.DiagSign(flipped, rest))
        assert bits_equal(s.download(), oracle.apply_diag(n, sorted(set(flipped)), rest, x))


# ------------------------------------------------------------------ RH / Walsh-Hadamard
@pytest.mark.parametrize("n", [1, 2, 5, 12, 13, 20, 25])
def test_rh_matches_oracle(Q, oracle, n):
    x = random_state(n, 77 + n)
    s = Q.DeviceState.from_numpy(x)
    s.apply_rh()
    got = s.download()
    want = oracle.wht(n, x) if n > 12 else oracle.rh_mvm(n, x)
    assert np.abs(got - want).max() <= TOL_AMP
    assert np.linalg.norm(got - want) <= TOL_L2
    s.apply_rh()  # involution
    assert np.abs(s.download() - x).max() <= 1e-12


def test_grover_matches_closed_form(Q, cfg):
    for n, k in ((10, 3), (16, 8), (22, 8)):
        marked = cfg.c3_marked(n)
        rep = Q.simulate(Q.build_grover(n, marked, k), Q.Engine.rh_dax)
        a_m, a_o = cfg.grover_closed_form(n, k)
        idx = np.array([0, 1, marked, (marked + 1) % (1 << n), (1 << n) - 1], np.uint64)
        got = rep.final.gather(idx)
        want = np.where(idx == marked, a_m, a_o)
        assert np.abs(got - want).max() <= 1e-12, n
        assert rep.final.argmax()[0] == marked
        assert abs(rep.final.norm() - 1) < 1e-12


def test_grover_golden_reference(Q, golden):
    g = golden("grover.npz")
    for n in range(4, 11):
        rep = Q.simulate(Q.build_grover(n, (1 << n) - 3), Q.Engine.rh_dax)
        assert np.abs(rep.final.download() - g[f"n{n}"]).max() <= 1e-12


@pytest.mark.parametrize("n", [13, 16, 19])
def test_sign_sandwiches_fused_vs_oracle(Q, oracle, n):
    """Sign steps between H^n steps and gates: the fused planner runs the tiles no sign step
    reaches with a simplified (often empty) program.  Lists of 1, 5 and 80 (> 64: searched
    per element) indices, flip_rest both ways, against the oracle step by step."""
    rng = np.random.default_rng(n)
    H = Q.hadamard_all(n)
    ry = Q.gate_catalog_lookup("RY", [0.37])
    signs = [Q.DiagSign([int(i) for i in rng.choice(1 << n, k, replace=False)], rest)
             for k, rest in ((1, False), (1, True), (5, False), (80, True), (0, True), (3, True))]
    steps = [H]
    for d in signs:
        steps += [Q.CircuitStep.of_diag(d), H]
    steps.insert(4, Q.CircuitStep.of_gates([Q.Placement(ry, 2)]))
    c = Q.Circuit(n, steps)
    st = Q.plan_stats(c)
    assert st["alt_passes"] > 0
    x = np.zeros(1 << n, np.complex128)
    x[0] = 1
    for step in steps:
        if step.is_hadamard_all(n):
            x = oracle.wht(n, x)
        elif int(step.kind) == 1:
            x = oracle.apply_diag(n, sorted(set(step.diag.flipped)), step.diag.flip_rest, x)
        else:
            x = oracle.apply_step(n, [(p.qubit_list(), p.gate.matrix) for p in step.placements], x)
    for fuse in (True, False):
        got = Q.simulate(c, Q.Engine.rh_dax, Q.SimOptions(fuse=fuse)).final.download()
        assert np.abs(got - x).max() <= TOL_AMP, fuse
        assert np.linalg.norm(got - x) <= TOL_L2, fuse


# ------------------------------------------------------------------ whole circuits
def test_c1_against_reference_golden(Q, cfg, golden):
    g = golden("c1.npz")
    for eng in (Q.Engine.rh_dax, Q.Engine.dax, Q.Engine.das, Q.Engine.dense):
        rep = Q.simulate(cfg.c1_circuit(), eng)
        got = rep.final.download()
        assert np.abs(got - g["final"]).max() <= TOL_AMP, eng
        assert np.linalg.norm(got - g["final"]) <= TOL_L2
    rep = Q.simulate(cfg.c1_circuit(), Q.Engine.rh_dax)
    assert [s.structure for s in rep.steps] == list(g["structure"])
    assert [s.entry_count for s in rep.steps] == [int(v) for v in g["entry_count"]]
    assert [s.sign_count for s in rep.steps] == [int(v) for v in g["sign_count"]]
    assert [s.madd_count for s in rep.steps] == [int(v) for v in g["madd_count"]]


def test_qnn_neuron_golden(Q, golden):
    g = golden("qnn.npz")
    c = Q.build_qnn_neuron(8, list(g["angles"]), [int(w) for w in g["weights"]])
    for eng in (Q.Engine.rh_dax, Q.Engine.dax):
        got = Q.simulate(c, eng).final.download()
        assert np.abs(got - g["final"]).max() <= 1e-12


def test_reference_engine_tests(Q):
    # test_engine.cpp:134-149 and :193-205
    rep = Q.simulate(Q.build_grover(5, 13), Q.Engine.rh_dax)
    assert rep.steps[0].structure == "rh" and rep.steps[0].matrix_bytes == 16
    assert rep.steps[0].sign_count == 16 * 4
    assert rep.steps[1].structure == "dax" and rep.steps[1].entry_count == 32
    q = Q.simulate(Q.build_grover(5, 13), Q.Engine.rh_dax, Q.SimOptions(sign_method=Q.SignMethod.quarter))
    assert q.steps[0].sign_count == 16 * 16
    assert np.abs(q.final.download() - rep.final.download()).max() < 1e-12
    pi = np.pi
    r = Q.simulate(Q.build_qnn_neuron(2, [pi, pi], [1, 1]), Q.Engine.dense)
    assert abs(r.probabilities[15] - 1) < 1e-10


def test_small_c4_c5_against_oracle(Q, cfg, oracle):
    """The C4 / C5 circuit families at reduced n (their full sizes have no CPU oracle)."""
    for c in (cfg.c4_circuit(n=10, layers=3), cfg.c5_circuit(n=11, layers=3, global_qubits=2)):
        x = np.zeros(1 << c.n, np.complex128)
        x[0] = 1
        for st in c.steps:
            if st.is_hadamard_all(c.n):
                x = oracle.wht(c.n, x)
            else:
                x = oracle.apply_step(c.n, [(p.qubit_list(), p.gate.matrix) for p in st.placements], x)
        got = Q.simulate(c, Q.Engine.rh_dax).final.download()
        assert np.abs(got - x).max() <= TOL_AMP
        assert np.linalg.norm(got - x) <= TOL_L2


def test_errors_mirror_reference(Q):
    with pytest.raises(Q.DimensionError):
        Q.DeviceState(0)
    with pytest.raises(Q.DimensionError):
        Q.DeviceState(3, 8)
    c = Q.Circuit(2, [Q.CircuitStep.of_gates([Q.Placement(Q.gate_catalog_lookup("H"), 0),
                                              Q.Placement(Q.gate_catalog_lookup("X"), 0)])])
    with pytest.raises(Q.DimensionError):
        Q.simulate(c)
    big = Q.Circuit(14, [Q.hadamard_all(14)])
    with pytest.raises(Q.CapacityError):
        Q.simulate(big, Q.Engine.dense)


# ------------------------------------------------------------------ device encoder (DAX / DAS)
def test_encoder_bytes_vs_oracle_and_golden(Q, oracle):
    with open(os.path.join(GOLDEN, "steps.json")) as f:
        recs = json.load(f)

    def sha(*arrs):
        return hashlib.sha256(np.concatenate([np.ascontiguousarray(a).view(np.uint64) for a in arrs]).tobytes()).hexdigest()
    for r in recs:
        pl = [Q.Placement(Q.gate_catalog_lookup(nm, Q.canonical_params(nm)), qs[0])
              for nm, qs in zip(r["names"], r["qubits"])]
        st = Q.CircuitStep.of_gates(pl)
        d = Q.step_matrix_dax(st, r["n"])
        assert sha(d.row, d.col, d.value) == r["dax"]
        s = Q.step_matrix_das(st, r["n"])
        assert sha(s.dis, s.last_in_row.astype(np.uint64), s.value) == r["das"]
        # DAX1 / DAS1 dumps of the device-encoded steps, byte for byte the reference's dax_dump /
        # das_dump of the same steps (dax.cpp:107-118, das.cpp:154-165)
        bx, bs = Q.dax_dump(d), Q.das_dump(s)
        assert len(bx) == r["dax_dump_len"] and hashlib.sha256(bx).hexdigest() == r["dax_dump"]
        assert len(bs) == r["das_dump_len"] and hashlib.sha256(bs).hexdigest() == r["das_dump"]
        assert Q.dax_dump(Q.dax_load(bx)) == bx and Q.das_dump(Q.das_load(bs)) == bs


def test_dumps_vs_live_reference(Q):
    """Bigger steps than the fixtures (n up to 14, 1-3 qubit gates with gaps): the device encoder's
    dumps equal the compiled reference's dax_dump / das_dump bytes (oracle/_ref, when shipped)."""
    from oracle.oracle_py import Reference
    if not Reference.available():
        pytest.skip("oracle/_ref/libqcsim_ref.so not shipped")
    rng = np.random.default_rng(21)
    cat = Q.gate_catalog()
    for t in range(12):
        n = int(rng.integers(9, 15))
        pl, q = [], 0
        while q < n:
            ar = 1 + int(rng.integers(0, min(n - q, 3)))
            fits = [c for c in cat if c.arity == ar]
            info = fits[int(rng.integers(0, len(fits)))]
            pl.append(Q.Placement(Q.gate_catalog_lookup(info.name, Q.canonical_params(info.name)), q))
            q += ar + int(rng.integers(0, 3))
        st = Q.CircuitStep.of_gates(pl)
        ref_pl = [(p.qubit_list(), p.gate.matrix) for p in pl]
        assert Q.dax_dump(Q.step_matrix_dax(st, n)) == Reference.step_dump(n, ref_pl, das=False), t
        assert Q.das_dump(Q.step_matrix_das(st, n)) == Reference.step_dump(n, ref_pl, das=True), t


def test_encoder_general_placements_and_mvm(Q, oracle):
    rng = np.random.default_rng(9)
    cat = Q.gate_catalog()
    for t in range(30):
        n = int(rng.integers(3, 11))
        ar = int(rng.choice([1, 2, 3]))
        info = [c for c in cat if c.arity == ar][int(rng.integers(0, 100)) % len([c for c in cat if c.arity == ar])]
        g = Q.gate_catalog_lookup(info.name, list(rng.uniform(0, 6.28, info.param_count)))
        qs = [int(v) for v in rng.choice(n, ar, replace=False)]
        pl = [Q.Placement(g, qubits=qs)]
        rest = [q for q in range(n) if q not in qs]
        if rest:
            h = Q.gate_catalog_lookup("RY", [0.3])
            pl.append(Q.Placement(h, rest[0]))
        st = Q.CircuitStep.of_gates(pl)
        d = Q.step_matrix_dax(st, n)
        want = oracle.step_dax(n, [(p.qubit_list(), p.gate.matrix) for p in pl])
        assert bits_equal(d.row, want[0]) and bits_equal(d.col, want[1]) and bits_equal(d.value, want[2])
        x = random_state(n, t)
        out = Q.dax_mvm(d, Q.DeviceState.from_numpy(x)).download()
        assert bits_equal(out, oracle.dax_mvm(n, *want, x))
        try:
            dd, ll, vv = oracle.step_das(n, [(p.qubit_list(), p.gate.matrix) for p in pl])
        except Exception:
            continue
        s = Q.step_matrix_das(st, n)
        assert bits_equal(s.dis, dd) and bits_equal(s.last_in_row, ll) and bits_equal(s.value, vv)
        out2 = Q.das_mvm(s, Q.DeviceState.from_numpy(x)).download()
        assert bits_equal(out2, oracle.das_mvm(n, dd, ll, vv, x))


def test_encoder_n20_full_step_and_dump_roundtrip(Q, oracle):
    n = 20
    h = Q.gate_catalog_lookup("H")
    st = Q.CircuitStep.of_gates([Q.Placement(h, 3), Q.Placement(Q.gate_catalog_lookup("CCX"), 10)])
    d = Q.step_matrix_dax(st, n)
    want = oracle.step_dax(n, [(p.qubit_list(), p.gate.matrix) for p in st.placements])
    assert all(bits_equal(a, b) for a, b in zip((d.row, d.col, d.value), want))
    assert Q.dax_load(Q.dax_dump(d)) == d
    s = Q.step_matrix_das(st, n)
    assert Q.das_load(Q.das_dump(s)) == s


def test_das_mvm_malformed(Q):
    x = Q.DeviceState(2)
    m = Q.DasMatrix(4, 4, np.array([5], np.uint64), np.array([1], np.uint8), np.array([1.0 + 0j]))
    with pytest.raises(Q.EncodingError):
        Q.das_mvm(m, x)


# ------------------------------------------------------------------ reductions
def test_reductions(Q, oracle):
    n = 16
    x = random_state(n, 1)
    s = Q.DeviceState.from_numpy(x)
    assert bits_equal(s.probabilities(), oracle.probabilities(n, x))
    assert abs(s.norm() - oracle.norm(n, x)) < 1e-13
    p = oracle.probabilities(n, x)
    i, pi = s.argmax()
    assert i == int(np.argmax(p)) and pi == p[i]
    idx, pr = s.topk(16)
    order = np.argsort(-p, kind="stable")[:16]
    assert list(idx) == [int(v) for v in order]
    s.randomize(5)
    assert abs(s.norm() - 1) < 1e-12


@pytest.mark.parametrize("n", [1, 3, 5, 9, 13, 21])
def test_topk_ties_and_sizes(Q, n):
    """top-k against a stable sort (ties to the lower index, as std::max_element): states with
    many equal probabilities (a uniform superposition with a few raised entries, basis states,
    fewer than k nonzero entries), every k, from 2 amplitudes up to more than one batch per warp."""
    dim = 1 << n
    rng = np.random.default_rng(n)
    cases = [np.full(dim, 1.0 / np.sqrt(dim), np.complex128)]
    x = cases[0].copy()
    for j in rng.choice(dim, min(dim, 5), replace=False):
        x[j] *= 1.5
    cases.append(x)
    b = np.zeros(dim, np.complex128)
    b[dim - 1] = 1.0
    cases.append(b)
    q = rng.integers(0, 4, dim).astype(np.float64) + 1j * rng.integers(0, 4, dim)  # heavy ties
    cases.append(q.astype(np.complex128))
    cases.append(random_state(n, 40 + n))
    for x in cases:
        s = Q.DeviceState.from_numpy(x)
        p = x.real * x.real + x.imag * x.imag
        order = np.argsort(-p, kind="stable")
        for k in (1, 2, 7, 16):
            idx, pr = s.topk(k)
            m = min(k, dim)
            assert [int(v) for v in idx[:m]] == [int(v) for v in order[:m]], (n, k)
            assert list(pr[:m]) == [p[v] for v in order[:m]]
        nrm, idx, pr = s.summary(16)
        assert abs(nrm - np.sqrt(p.sum())) <= 1e-12 * max(1.0, np.sqrt(p.sum()))
        m = min(16, dim)
        assert [int(v) for v in idx[:m]] == [int(v) for v in order[:m]]


@pytest.mark.slow
def test_c2_full_size_properties(Q, cfg):
    """n = 28 (BASELINE C2 size): norm preservation and X/H involutions on the device."""
    n = 28
    s = Q.DeviceState(n)
    s.randomize(cfg.seed_of(2))
    probe = np.array([0, 1, 12345, (1 << n) - 1], np.uint64)
    before = s.gather(probe)
    xg = Q.gate_catalog_lookup("X")
    hg = Q.gate_catalog_lookup("H")
    for q in (0, 13, 27):
        s.apply_gate(xg, [q])
        s.apply_gate(xg, [q])
    assert bits_equal(s.gather(probe), before)
    for q in (0, 27):
        s.apply_gate(hg, [q])
        s.apply_gate(hg, [q])
    assert np.abs(s.gather(probe) - before).max() < 1e-15
    assert abs(s.norm() - 1) < 1e-12


@pytest.mark.parametrize("n", [22, 23])
def test_pass_pairs_around_sign_steps_vs_oracle(Q, oracle, n):
    """Grover-like circuits with several marked indices (one and three per oracle step, flip_rest
    both ways): the planner pairs the H_low passes around each skip pass (plan_stats
    paired_passes) and runs them only on the tiles the sign steps reach; against the oracle."""
    rng = np.random.default_rng(n)
    H = Q.hadamard_all(n)
    steps = [H]
    for it in range(4):
        marked = [int(i) for i in rng.choice(1 << n, 1 + 2 * (it % 2), replace=False)]
        steps += [Q.CircuitStep.of_diag(Q.DiagSign(marked, it == 2)), H,
                  Q.CircuitStep.of_diag(Q.DiagSign([0], True)), H]
    c = Q.Circuit(n, steps)
    assert Q.plan_stats(c)["paired_passes"] > 0
    x = np.zeros(1 << n, np.complex128)
    x[0] = 1
    for st in steps:
        if st.is_hadamard_all(n):
            x = oracle.wht(n, x)
        else:
            x = oracle.apply_diag(n, sorted(set(st.diag.flipped)), st.diag.flip_rest, x)
    got = Q.simulate(c, Q.Engine.rh_dax).final.download()
    assert np.abs(got - x).max() <= TOL_AMP
    assert np.linalg.norm(got - x) <= TOL_L2
