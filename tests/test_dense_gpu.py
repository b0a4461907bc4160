"""The paper's Matrix method on the device: Engine.dense materialises each
step's 2^n x 2^n operator (step_matrix_dense, engine.cpp:126-133: the left fold of dense_tensor
over the per-qubit factors, core.cpp:55-72) and applies dense_mvm (core.cpp:74-87) -- byte for
byte the reference's dense engine, checked against the compiled reference (oracle/_ref) on the
same circuits: random catalog circuits, the C1 family, Grover with its sign steps, the dense-cap
CapacityError."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def Q():
    from paper_2411_15332_b200 import qcsim
    return qcsim


@pytest.fixture(scope="module")
def R():
    from oracle.oracle_py import Reference
    if not Reference.available():
        pytest.skip("oracle/_ref/libqcsim_ref.so not shipped")
    return Reference


def ref_steps(c):
    out = []
    for st in c.steps:
        if int(st.kind) == 1:
            out.append(("diag", list(st.diag.flipped), bool(st.diag.flip_rest), st.stage))
        else:
            out.append(("gates", [(p.gate.name, p.qubit_list(), p.gate.matrix) for p in st.placements], st.stage))
    return out


def random_contiguous_circuit(Q, seed, n, nsteps):
    rng = np.random.default_rng(seed)
    cat = Q.gate_catalog()
    steps = []
    for _ in range(nsteps):
        if rng.random() < 0.15:
            f = sorted({int(v) for v in rng.integers(0, 1 << n, int(rng.integers(0, 4)))})
            steps.append(Q.CircuitStep.of_diag(Q.DiagSign(f, bool(rng.random() < 0.5))))
            continue
        pl, q = [], int(rng.integers(0, 2))
        while q < n:
            ar = 1 + int(rng.integers(0, min(n - q, 3)))
            fits = [c for c in cat if c.arity == ar]
            info = fits[int(rng.integers(0, len(fits)))]
            params = list(rng.uniform(-4, 4, info.param_count)) if info.param_count else []
            pl.append(Q.Placement(Q.gate_catalog_lookup(info.name, params), q))
            q += ar + int(rng.integers(0, 3))
        steps.append(Q.CircuitStep.of_gates(pl))
    return Q.Circuit(n, steps, int(rng.integers(0, 1 << n)))


def check(Q, R, c):
    rep = Q.simulate(c, Q.Engine.dense)
    want, wrep, _ = R.simulate(c.n, ref_steps(c), engine="dense", initial=c.initial)
    got = rep.final.download()
    assert got.view(np.uint64).tobytes() == want.view(np.uint64).tobytes(), float(np.abs(got - want).max())
    assert [s.structure for s in rep.steps] == [w["structure"] for w in wrep]
    assert [s.madd_count for s in rep.steps] == [w["madd_count"] for w in wrep]
    assert [s.matrix_bytes for s in rep.steps] == [w["matrix_bytes"] for w in wrep]


@pytest.mark.parametrize("seed", range(6))
def test_random_circuits_bit_exact(Q, R, seed):
    check(Q, R, random_contiguous_circuit(Q, seed, 3 + seed, 10))


def test_c1_family_and_grover_bit_exact(Q, R):
    from paper_2411_15332_b200 import configs
    check(Q, R, configs.c1_circuit(9, 2))
    check(Q, R, Q.build_grover(8, 37, 3))


def test_dense_cap(Q):
    c = Q.Circuit(14, [Q.hadamard_all(14)])
    with pytest.raises(Q.CapacityError):
        Q.simulate(c, Q.Engine.dense)
    d = Q.Circuit(14, [Q.CircuitStep.of_diag(Q.DiagSign([1], False))])
    with pytest.raises(Q.CapacityError, match="diagonal step exceeds dense cap"):
        Q.simulate(d, Q.Engine.dense)


def test_non_contiguous_steps_within_tolerance(Q):
    """A placement the reference cannot express (reversed CNOT) runs through the fused kernels
    inside a dense-engine circuit; the state still matches the other engines."""
    n = 6
    cnot = Q.gate_catalog_lookup("CNOT")
    h = Q.gate_catalog_lookup("Hadamard")
    c = Q.Circuit(n, [Q.CircuitStep.of_gates([Q.Placement(h, 0), Q.Placement(h, 3)]),
                      Q.CircuitStep.of_gates([Q.Placement(cnot, qubits=[4, 1])]),
                      Q.CircuitStep.of_gates([Q.Placement(Q.gate_catalog_lookup("RY", [0.3]), 2)])])
    a = Q.simulate(c, Q.Engine.dense).final.download()
    b = Q.simulate(c, Q.Engine.dax).final.download()
    assert np.abs(a - b).max() < 1e-12
