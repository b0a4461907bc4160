"""Host logic without a GPU: circuit builders, validation, report accounting, dump formats,
BASELINE workload generators (mirrors of the reference's test_engine / test_io goldens)."""
import numpy as np
import pytest


@pytest.fixture(scope="module")
def Q():
    from paper_2411_15332_b200 import qcsim
    return qcsim


def test_engine_names(Q):
    for e in Q.Engine:
        assert Q.engine_from_name(Q.engine_name(e)) == e
    assert Q.engine_from_name("rh_dax") == Q.Engine.rh_dax
    with pytest.raises(Q.ParseError):
        Q.engine_from_name("sparse")


def test_grover_builder(Q):
    # test_engine.cpp:151-157
    assert Q.grover_auto_iterations(2) == 1
    assert Q.grover_auto_iterations(4) == 3
    assert Q.grover_auto_iterations(10) == 25
    assert len(Q.build_grover(2, 0).steps) == 1 + 4
    assert len(Q.build_grover(10, 7).steps) == 1 + 4 * 25
    with pytest.raises(Q.DimensionError):
        Q.build_grover(0, 0)
    with pytest.raises(Q.DimensionError):
        Q.build_grover(3, 8)
    c = Q.build_grover(5, 13)
    assert c.steps[0].is_hadamard_all(5) and c.steps[1].diag.flipped == [13]
    assert c.steps[3].diag.flip_rest and c.steps[3].diag.flipped == [0]


def test_qnn_builder(Q):
    assert [Q.qnn_total_qubits(k) for k in (1, 2, 4, 8)] == [2, 4, 7, 12]
    with pytest.raises(Q.DimensionError):
        Q.qnn_total_qubits(0)
    with pytest.raises(Q.SimError):
        Q.build_qnn_neuron(2, [0.0], [1, 1])
    with pytest.raises(Q.SimError):
        Q.build_qnn_neuron(2, [0.0, 0.0], [1, 2])
    c = Q.build_qnn_neuron(8, [0.1] * 8, [1, -1, 1, 1, -1, 1, -1, 1])
    assert c.n == 12 and any(s.stage >= 2 for s in c.steps)


def test_validation(Q):
    h, x = Q.gate_catalog_lookup("H"), Q.gate_catalog_lookup("X")
    with pytest.raises(Q.DimensionError):
        Q.Circuit(2, [Q.CircuitStep.of_gates([Q.Placement(h, 0), Q.Placement(x, 0)])]).validate()
    with pytest.raises(Q.DimensionError):
        Q.Circuit(2, [Q.CircuitStep.of_gates([Q.Placement(Q.gate_catalog_lookup("CCX"), 0)])]).validate()
    with pytest.raises(Q.DimensionError):
        Q.Circuit(1, [], 2).validate()
    with pytest.raises(Q.DimensionError):
        Q.Circuit(2, [Q.CircuitStep.of_diag(Q.DiagSign([4]))]).validate()


def test_memory_report_matches_reference_formulas(Q):
    # test_engine.cpp:226-254 and acceptance.cpp:239-265
    for n in (2, 6, 12, 18):
        c = Q.Circuit(n, [Q.CircuitStep.of_gates([Q.Placement(Q.gate_catalog_lookup("X"), q) for q in range(n)])])
        r = Q.memory_report(c, Q.Engine.dax)[0]
        assert r.entry_count == 1 << n
        assert r.dense_bytes / r.matrix_bytes == (2.0 / 3.0) * 2.0 ** n
    c = Q.Circuit(24, [Q.hadamard_all(24)])
    assert Q.memory_report(c, Q.Engine.dax)[0].entry_count == 1 << 48
    rh = Q.memory_report(c, Q.Engine.rh_dax)[0]
    assert rh.structure == "rh" and rh.matrix_bytes == 16
    g = Q.build_grover(5, 13)
    r = Q.memory_report(g, Q.Engine.rh_dax)
    assert r[0].structure == "rh" and r[1].structure == "dax" and r[1].entry_count == 32
    assert r[0].dense_bytes == 1 << 14
    big = Q.memory_report(Q.Circuit(31, [Q.hadamard_all(31)]), Q.Engine.dense)[0]
    assert big.dense_bytes == (1 << 64) - 1  # saturates for 2n + 4 >= 64 (engine.cpp:82-85)


def test_memory_report_vs_reference_simulate(Q, reference):
    from paper_2411_15332_b200 import configs
    c = configs.c1_circuit()
    steps = []
    for st in c.steps:
        steps.append(("gates", [(p.gate.name, p.qubit_list(), p.gate.matrix) for p in st.placements], st.stage))
    for eng in ("dax", "das", "rh-dax"):
        _, ref, _ = reference.simulate(c.n, steps, engine=eng)
        mine = Q.memory_report(c, Q.engine_from_name(eng))
        for a, b in zip(mine, ref):
            assert (a.structure, a.matrix_bytes, a.dense_bytes, a.entry_count) == \
                   (b["structure"], b["matrix_bytes"], b["dense_bytes"], b["entry_count"])


def test_dump_formats(Q):
    # dax dump of Y (x) X: 4 + 3*8 + 4*32 = 156 B (test_dax.cpp:176-190); das: 124 B
    yx = np.kron(Q.gate_catalog_lookup("Y").matrix, Q.gate_catalog_lookup("X").matrix)
    r, c = np.nonzero(yx)
    d = Q.DaxMatrix(4, 4, r.astype(np.uint64), c.astype(np.uint64), yx[r, c])
    b = Q.dax_dump(d)
    assert len(b) == 156 and b[:4] == b"DAX1"
    assert Q.dax_load(b) == d
    s = Q.DasMatrix(4, 4, np.array([3, 2, 1, 0], np.uint64), np.ones(4, np.uint8), yx[r, c])
    b2 = Q.das_dump(s)
    assert len(b2) == 124 and b2[:4] == b"DAS1"
    assert Q.das_load(b2) == s
    with pytest.raises(Q.ParseError):
        Q.dax_load(b"nope")
    with pytest.raises(Q.ParseError):
        Q.das_load(b2[:40])


def test_config_generators():
    from paper_2411_15332_b200 import configs
    assert configs.c1_updates() == 152 << 12
    c1 = configs.c1_circuit()
    assert sum(len(s.placements) if not s.is_hadamard_all(12) else 12 for s in c1.steps) == 152
    sweep = configs.c2_sweep(28)
    assert len(sweep) == 336
    for g in sweep:
        assert len(set(g.qubits)) == len(g.qubits) and all(0 <= q < 28 for q in g.qubits)
    assert [g.qubits[-1] for g in sweep[:28]] == list(range(28))
    assert configs.c3_updates() == 526 << 30
    c4 = configs.c4_circuit()
    assert sum(len(s.placements) for s in c4.steps) == 992
    assert configs.c4_updates() == 992 << 32
    c5 = configs.c5_circuit()
    assert sum(len(s.placements) for s in c5.steps) == 1075
    for st in c5.steps[2::2]:
        assert any(min(p.qubit_list()) < 3 for p in st.placements)
    am, ao = configs.grover_closed_form(30, 8)
    assert abs(am ** 2 + (2 ** 30 - 1) * ao ** 2 - 1) < 1e-12
