"""Front end: parse_circuit_json / render_report / sampling against the
reference's own circuit_io.cpp (fixtures in tests/golden/io.json, tests/golden/make_golden.py io)."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN


@pytest.fixture(scope="module")
def io():
    with open(os.path.join(GOLDEN, "io.json")) as f:
        return json.load(f)


def test_parse_errors_match_reference(io):
    from paper_2411_15332_b200 import circuit_io as IO
    from paper_2411_15332_b200 import qcsim as Q
    cls = {2: Q.DimensionError, 4: Q.ParseError, 5: Q.SimError}
    for e in io["errors"]:
        with pytest.raises(cls[e["code"]]) as ei:
            IO.parse_circuit_json(e["circuit"])
        assert str(ei.value) == e["message"]
        assert type(ei.value) is cls[e["code"]]
    with pytest.raises(Q.ParseError, match="circuit JSON"):
        IO.parse_circuit_json("{not json")
    with pytest.raises(Q.ParseError, match="cannot open circuit file"):
        IO.load_circuit_file("/nonexistent/c.json")


def test_parse_matches_structure(io):
    from paper_2411_15332_b200 import circuit_io as IO
    c = IO.parse_circuit_json(io["reports"][0]["circuit"])
    assert c.n == 5 and c.initial == 3 and len(c.steps) == 6
    assert c.steps[2].diag.flipped == [7] and not c.steps[2].diag.flip_rest
    assert c.steps[4].diag.flip_rest and c.steps[4].diag.flipped == [1, 2, 3]
    assert c.steps[0].placements[1].gate.name == "Controlled-X" and c.steps[0].placements[1].first_qubit == 1


def test_mt19937_64_and_canonical():
    from oracle.oracle_py import MT19937_64
    r = MT19937_64(5489)  # the C++ standard's check value: the 10000th draw of a default engine
    for _ in range(9999):
        r()
    assert r() == 9981545732273789042


def test_json_number_format():
    from paper_2411_15332_b200.circuit_io import _num
    for x, s in [(0.0, "0.0"), (1.0, "1.0"), (0.5, "0.5"), (1e-05, "1e-05"), (0.000123, "0.000123"),
                 (1.2345e-17, "1.2345e-17"), (0.48883412228140133, "0.48883412228140133"), (1e16, "1e+16")]:
        assert _num(x) == s


def test_gate_expression_matches_reference_dense():
    from paper_2411_15332_b200 import circuit_io as IO
    from paper_2411_15332_b200 import qcsim as Q
    yx = IO.parse_gate_expression("Y x X")
    assert yx[0, 3] == -1j and yx[1, 2] == -1j and yx[2, 1] == 1j and yx[3, 0] == 1j
    m = IO.parse_gate_expression("CCX * Pauli-X")
    assert m.shape == (16, 16) and np.count_nonzero(m) == 16
    with pytest.raises(Q.ParseError):
        IO.parse_gate_expression("X y Z")
    with pytest.raises(Q.ParseError):
        IO.parse_gate_expression("X x")


@pytest.mark.gpu
def test_render_report_matches_reference(io):
    from paper_2411_15332_b200 import circuit_io as IO
    from paper_2411_15332_b200 import qcsim as Q
    for r in io["reports"]:
        c = IO.parse_circuit_json(r["circuit"])
        rep = Q.simulate(c, Q.engine_from_name(r["engine"]))
        got = IO.render_report(rep, c.n, IO.ReportOptions(r["format"], r["samples"], r["seed"], r["engine"]))
        if r["name"] == "exact_perm":  # exact values: the final state is bit-identical
            assert got == r["output"], (r["engine"], r["format"])
        elif r["format"] == "json":
            a, b = json.loads(got), json.loads(r["output"])
            assert a.keys() == b.keys() and a["steps"] == b["steps"] and a["argmax"] == b["argmax"]
            assert np.abs(np.array(a["probabilities"]) - np.array(b["probabilities"])).max() < 1e-12
            assert a.get("samples") == b.get("samples")
        else:
            lg, lr = got.splitlines(), r["output"].splitlines()
            assert len(lg) == len(lr)
            assert [x for x in lg if "probab" not in x and "norm" not in x] == \
                   [x for x in lr if "probab" not in x and "norm" not in x]


def test_sampling_restatement_pinned_to_reference():
    """oracle_py.sequential_sample (the Python restatement the device sampler is checked against)
    equals the reference's render_report samples (circuit_io.cpp:114-128), ties included."""
    from oracle.oracle_py import ReferenceIO, sequential_sample
    if not ReferenceIO.available():
        pytest.skip("oracle/_ref/libqcsim_io.so not built")
    rng = np.random.default_rng(3)
    for n in (4, 9, 12):
        x = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
        x /= np.linalg.norm(x)
        p = x.real * x.real + x.imag * x.imag
        assert ReferenceIO.sample(n, x, 300, 17 + n) == sequential_sample(p, 300, 17 + n)[0]
    x = np.full(1 << 10, complex(3 * 2.0 ** -27, 4 * 2.0 ** -27))
    x[0] = complex(0.5, 0.5)
    p = x.real * x.real + x.imag * x.imag
    assert ReferenceIO.sample(10, x, 200, 1) == sequential_sample(p, 200, 1)[0]
