"""Pin the C restatement (oracle/qcs_oracle.c) before trusting it as the parity checker.

1. Known answers copied from the reference's own unit tests:
   test_dax.cpp, test_das.cpp, test_rh.cpp, acceptance.cpp.
2. Golden fixtures produced by the compiled reference (tests/golden/make_golden.py).
3. Live comparison against oracle/_ref when it was built here.
"""
import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, bits_equal, random_state

X = np.array([[0, 1], [1, 0]], np.complex128)
Y = np.array([[0, complex(-0.0, -1.0)], [1j, 0]], np.complex128)
H = np.full((2, 2), 1 / np.sqrt(2), np.complex128)
H[1, 1] = -1 / np.sqrt(2)
I2 = np.eye(2, dtype=np.complex128)
CCX = np.eye(8, dtype=np.complex128)
CCX[6:, 6:] = [[0, 1], [1, 0]]


def sha(*arrs):
    return hashlib.sha256(np.concatenate([np.ascontiguousarray(a).view(np.uint64) for a in arrs]).tobytes()).hexdigest()


# --------------------------------------------------------- known answers (reference unit tests)
def test_dax_yx_worked_example(oracle):
    # test_dax.cpp:11-22 and :69-79: Y (x) X has entries at linear indices 3, 6, 9, 12 with
    # values -i, -i, i, i; the MTP entry[1] is (row 1, col 2, -i).
    r, c, v = oracle.step_dax(2, [([0], Y), ([1], X)])
    assert list(r * 4 + c) == [3, 6, 9, 12]
    assert list(v) == [-1j, -1j, 1j, 1j]
    assert (r[1], c[1]) == (1, 2)
    assert 24 * len(r) == 96  # dax_memory_bytes


def test_dax_x_and_identity_fill(oracle):
    r, c, v = oracle.step_dax(1, [([0], X)])  # test_dax.cpp:24-30
    assert list(zip(r, c, v)) == [(0, 1, 1), (1, 0, 1)]
    r, c, v = oracle.step_dax(2, [])  # I (x) I: test_dax.cpp:81-88
    assert list(r) == [0, 1, 2, 3] and list(c) == [0, 1, 2, 3]
    r, c, v = oracle.step_dax(4, [([0, 1, 2], CCX), ([3], X)])  # CCX (x) X: 16 entries
    assert len(r) == 16


def test_das_worked_examples(oracle):
    # test_das.cpp:12-32
    d, l, v = oracle.step_das(2, [([0], Y), ([1], X)])
    assert list(d) == [3, 2, 1, 0] and list(l) == [1, 1, 1, 1] and list(v) == [-1j, -1j, 1j, 1j]
    d, l, v = oracle.step_das(1, [([0], X)])
    assert list(d) == [1, 0] and list(l) == [1, 1]
    d, l, v = oracle.step_das(1, [([0], H)])
    h = 1 / np.sqrt(2)
    assert list(d) == [0, 0, 0, 0] and list(l) == [0, 1, 0, 1] and list(v) == [h, h, h, -h]
    d, l, v = oracle.step_das(2, [([0], X), ([1], X)])  # X (x) X distances 3, 2, 1, 0
    assert list(d) == [3, 2, 1, 0]
    d, l, v = oracle.step_das(2, [])  # I (x) I distances 0..3
    assert list(d) == [0, 1, 2, 3]


def test_das_rejects_all_zero_row(oracle):
    from oracle.oracle_py import OracleError
    m = np.zeros((2, 2), np.complex128)
    m[0, 0] = 1
    with pytest.raises(OracleError):
        oracle.step_das(1, [([0], m)])


def test_dax_mvm_goldens(oracle):
    # test_dax.cpp:130-150: X [0.6, 0.8] = [0.8, 0.6]; (Y (x) X)|00> = i|11>; identity is exact
    s = np.array([0.6, 0.8], np.complex128)
    assert list(oracle.apply_step(1, [([0], X)], s)) == [0.8, 0.6]
    s2 = np.zeros(4, np.complex128)
    s2[0] = 1
    out = oracle.apply_step(2, [([0], Y), ([1], X)], s2)
    assert out[3] == 1j and not out[:3].any()
    r = random_state(3, 99)
    assert bits_equal(oracle.apply_step(3, [], r), r + 0.0)


def test_das_mvm_ccx(oracle):
    # test_das.cpp:129-150: CCX |110> = |111>
    d, l, v = oracle.step_das(3, [([0, 1, 2], CCX)])
    s = np.zeros(8, np.complex128)
    s[6] = 1
    out = oracle.das_mvm(3, d, l, v, s)
    assert out[7] == 1 and out[6] == 0


def test_dax_zero_products_dropped(oracle):
    # test_dax.cpp:111-121: 1e-200 * 1e-200 underflows to 0 and is not stored
    a = np.array([[1e-200, 1.0], [1.0, 1.0]], np.complex128)
    r, c, v = oracle.step_dax(2, [([0], a), ([1], a)])
    assert (v != 0).all()
    assert len(r) == 16 - 1


def test_rh_quarter_and_wht(oracle):
    # test_rh.cpp:165-179: n=1 and n=3 uniform outputs
    s = np.zeros(8, np.complex128)
    s[0] = 1
    for f in (oracle.rh_mvm, oracle.wht):
        out = f(3, s)
        assert np.allclose(out, 1 / np.sqrt(8), atol=1e-14)
    # involution and dense agreement (acceptance.cpp:218-237)
    for n in (1, 4, 9):
        x = random_state(n, 2000 + n)
        once = oracle.rh_mvm(n, x)
        assert abs(np.linalg.norm(once) - 1) < 1e-9
        assert np.abs(oracle.rh_mvm(n, once) - x).max() < 1e-9
        Hn = np.array([[1.0]])
        for _ in range(n):
            Hn = np.kron(Hn, H.real)
        assert np.abs(Hn @ x - oracle.wht(n, x)).max() < 1e-12


def test_dense_agreement_mvm(oracle):
    # test_dax.cpp:152-168: compressed MVM within 1e-12 of dense for n <= 8
    rng = np.random.default_rng(31)
    for n in range(1, 9):
        mats = [np.linalg.qr(rng.standard_normal((2, 2)) + 1j * rng.standard_normal((2, 2)))[0] for _ in range(n)]
        M = np.array([[1.0 + 0j]])
        for m in mats:
            M = np.kron(M, m)
        x = random_state(n, n)
        out = oracle.apply_step(n, [([q], m) for q, m in enumerate(mats)], x)
        assert np.abs(out - M @ x).max() < 1e-12


# --------------------------------------------------------- golden fixtures from the reference
def test_oracle_matches_reference_sweep_fixtures(oracle, golden):
    import paper_2411_15332_b200.configs as cfg
    for n in (6, 12):
        g = golden(f"sweep_n{n}.npz")
        s = g["state"]
        sweep = cfg.c2_sweep(n, seed=cfg.seed_of(2))
        assert [x.label for x in sweep] == list(g["labels"])
        for i, sg in enumerate(sweep):
            out = oracle.apply_step(n, [(sg.qubits, sg.gate.matrix)], s)
            if "outputs" in g:
                assert bits_equal(out, g["outputs"][i]), (n, sg.label, sg.qubits)
            assert hashlib.sha256(out.tobytes()).hexdigest() == g["sha"][i], (n, sg.label, sg.qubits)


def test_oracle_matches_reference_step_bytes(oracle, golden):
    from paper_2411_15332_b200 import qcsim as Q
    with open(os.path.join(GOLDEN, "steps.json")) as f:
        recs = json.load(f)
    for r in recs:
        pl = [(qs, Q.gate_catalog_lookup(name, Q.canonical_params(name)).matrix)
              for name, qs in zip(r["names"], r["qubits"])]
        rr, cc, vv = oracle.step_dax(r["n"], pl)
        assert len(rr) == r["count"]
        assert sha(rr, cc, vv) == r["dax"]
        d, l, v = oracle.step_das(r["n"], pl)
        assert sha(d, l.astype(np.uint64), v) == r["das"]
        # the host DAX1 / DAS1 writers on the oracle's entries == the reference's dump bytes
        dim = 1 << r["n"]
        bx = Q.dax_dump(Q.DaxMatrix(dim, dim, rr, cc, vv))
        bs = Q.das_dump(Q.DasMatrix(dim, dim, d, l, v))
        assert hashlib.sha256(bx).hexdigest() == r["dax_dump"] and len(bx) == r["dax_dump_len"]
        assert hashlib.sha256(bs).hexdigest() == r["das_dump"] and len(bs) == r["das_dump_len"]


def test_oracle_grover_and_c1(oracle, golden):
    import paper_2411_15332_b200.configs as cfg
    # C1 through the oracle step by step, against the reference's final state (within the
    # reference's own RH tolerance: rh_mvm sums in a different order than the butterfly)
    c = cfg.c1_circuit()
    s = np.zeros(1 << c.n, np.complex128)
    s[0] = 1
    for st in c.steps:
        if st.is_hadamard_all(c.n):
            s = oracle.wht(c.n, s)
        else:
            s = oracle.apply_step(c.n, [(p.qubit_list(), p.gate.matrix) for p in st.placements], s)
    assert np.abs(s - golden("c1.npz")["final"]).max() < 1e-12
    g = golden("grover.npz")
    for n in range(4, 11):
        a_m, a_o = cfg.grover_closed_form(n, int(np.floor(np.pi / 4 * np.sqrt(2 ** n))))
        want = np.full(1 << n, a_o)
        want[(1 << n) - 3] = a_m
        assert np.abs(g[f"n{n}"] - want).max() < 1e-12


# --------------------------------------------------------- live reference comparison
def test_oracle_matches_reference_random_steps(oracle, reference):
    rng = np.random.default_rng(11)
    cat = reference.catalog()
    for t in range(80):
        n = int(rng.integers(2, 9))
        pl, q = [], 0
        while q < n:
            ar = 1 + int(rng.integers(0, min(n - q, 3)))
            fits = [c for c in cat if c[1] == ar]
            name, _, npar, _ = fits[int(rng.integers(0, len(fits)))]
            pl.append((list(range(q, q + ar)), reference.gate(name, list(rng.uniform(0, 6.3, npar)))))
            q += ar + int(rng.integers(0, 2))
        x = reference.random_unit_state(n, t)
        assert all(bits_equal(a, b) for a, b in zip(reference.step_dax(n, pl), oracle.step_dax(n, pl)))
        assert all(bits_equal(a, b) for a, b in zip(reference.step_das(n, pl), oracle.step_das(n, pl)))
        assert bits_equal(reference.apply_step(n, pl, x)[0], oracle.apply_step(n, pl, x))


def test_oracle_matches_projector_decomposition(oracle, reference):
    rng = np.random.default_rng(12)
    cat = reference.catalog()
    for t in range(60):
        n = int(rng.integers(3, 9))
        ar = int(rng.choice([2, 3]))
        fits = [c for c in cat if c[1] == ar]
        name, _, npar, _ = fits[int(rng.integers(0, len(fits)))]
        qs = [int(x) for x in rng.choice(n, ar, replace=False)]
        pl = [(qs, reference.gate(name, list(rng.uniform(0, 6.3, npar))))]
        x = reference.random_unit_state(n, 100 + t)
        assert all(bits_equal(a, b) for a, b in zip(reference.step_dax(n, pl), oracle.step_dax(n, pl)))
        assert bits_equal(reference.apply_step(n, pl, x)[0], oracle.apply_step(n, pl, x))


def test_oracle_rh_matches_reference(oracle, reference):
    for n in range(1, 11):
        x = reference.random_unit_state(n, 808 + n)
        r, sc, mc = reference.rh_mvm(n, x)
        assert bits_equal(r, oracle.rh_mvm(n, x))
        assert mc == (4 * (1 << (n - 1)) ** 2) % (1 << 64)
        assert np.abs(r - oracle.wht(n, x)).max() < 1e-12
