"""Seeded sampling on the device (reference circuit_io.cpp:114-128).

qcs_sample reproduces render_report's samples index for index: std::mt19937_64(seed), draws of
uniform_real_distribution<double>(0, acc), std::lower_bound on the SEQUENTIAL rounded CDF.  The
checkers are the reference's own render_report run on the same state (oracle/_ref/libqcsim_io.so,
``ReferenceIO.sample``) and the Python restatement ``oracle_py.sequential_sample``.  The states
include the cases where a parallel scan would round differently from the sequential chain:
ties to even at every add, many binade changes, leading/trailing zero runs, an all-zero state,
unnormalised sums, partial chunks (n < 12) and chunk-aligned sizes.
"""
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _ref_sample(n, amps, count, seed):
    from oracle.oracle_py import ReferenceIO, sequential_sample
    if ReferenceIO.available():
        return ReferenceIO.sample(n, amps, count, seed)
    p = amps.real * amps.real + amps.imag * amps.imag
    return sequential_sample(p, count, seed)[0]


def _random_state(n, seed):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    return (x / np.linalg.norm(x)).astype(np.complex128)


def _tie_state(n, seed):
    """p_0 = 0.5 exactly, then p = 25 * 2^-54 (amplitude (3, 4) * 2^-27) at random places: with the
    sum in [0.5, 1) every such add is 12.5 ulps, a tie resolved by the parity of the running sum."""
    rng = np.random.default_rng(seed)
    x = np.zeros(1 << n, np.complex128)
    pick = rng.random(1 << n)
    x[pick < 0.6] = complex(3 * 2.0 ** -27, 4 * 2.0 ** -27)
    x[(pick >= 0.6) & (pick < 0.7)] = complex(2.0 ** -27, 0)          # 2^-54: a quarter ulp, dropped
    other = pick >= 0.9
    x[other] = (rng.standard_normal(other.sum()) + 1j * rng.standard_normal(other.sum())) * 2.0 ** -27
    x[0] = complex(0.5, 0.5)
    return x


def _device_sample(x, count, seed):
    from paper_2411_15332_b200 import qcsim as Q
    s = Q.DeviceState.from_numpy(x)
    return s.sample(count, seed)


@pytest.mark.parametrize("n", [5, 11, 12, 13, 16])
def test_random_states_match_reference(n):
    x = _random_state(n, 100 + n)
    for seed in (0, 7, 2024):
        got, acc = _device_sample(x, 400, seed)
        assert got == _ref_sample(n, x, 400, seed), (n, seed)
        p = x.real * x.real + x.imag * x.imag
        from oracle.oracle_py import sequential_sample
        assert acc == sequential_sample(p, 0, seed)[1]  # the final sequential sum, exactly


@pytest.mark.parametrize("n", [12, 15])
def test_tie_to_even_chain(n):
    x = _tie_state(n, n)
    p = x.real * x.real + x.imag * x.imag
    from oracle.oracle_py import sequential_sample
    want, acc_ref = sequential_sample(p, 600, 99)
    got, acc = _device_sample(x, 600, 99)
    assert acc == acc_ref
    assert got == want
    assert got == _ref_sample(n, x, 600, 99)


def test_zero_runs_and_degenerate_states():
    n = 14
    x = _random_state(n, 5)
    x[: 5000] = 0          # leading zeros spanning a whole chunk and part of the next
    x[-7000:] = 0          # trailing zeros: the CDF plateaus at acc
    x *= 3.0               # unnormalised: acc ~ 9 * (kept mass)
    assert _device_sample(x, 300, 3)[0] == _ref_sample(n, x, 300, 3)
    z = np.zeros(1 << n, np.complex128)
    got, acc = _device_sample(z, 10, 1)
    assert acc == 0.0 and got == _ref_sample(n, z, 10, 1) == [0] * 10
    one = np.zeros(1 << n, np.complex128)
    one[12345] = 1.0
    assert _device_sample(one, 20, 4)[0] == [12345] * 20
    assert _device_sample(one, 0, 4)[0] == []


def test_basis_and_uniform_states():
    from paper_2411_15332_b200 import qcsim as Q
    n = 13
    s = Q.DeviceState(n)
    s.apply_rh()                 # uniform: every probability equal, boundaries evenly spaced
    x = s.download()
    got, acc = s.sample(500, 11)
    assert got == _ref_sample(n, x, 500, 11)
    from oracle.oracle_py import sequential_sample
    assert acc == sequential_sample(x.real * x.real + x.imag * x.imag, 0, 11)[1]
    b = Q.DeviceState(n, 4321)   # a basis state: probability 1 at one index, exact
    got, acc = b.sample(50, 2)
    assert acc == 1.0 and got == [4321] * 50


def test_render_report_n24_samples_on_device_fast():
    """An n=24 circuit renders with 256 samples in under a second, index-equal to the reference's
    render_report on the same final state; nothing of size 2^n is downloaded for it."""
    from paper_2411_15332_b200 import circuit_io as IO
    from paper_2411_15332_b200 import configs
    from paper_2411_15332_b200 import qcsim as Q
    n = 24
    rep = Q.simulate(configs.c4_circuit(n, 2), Q.Engine.rh_dax)
    rep.final.sample(1, 0)  # warm (allocations)
    t0 = time.perf_counter()
    out = IO.render_report(rep, n, IO.ReportOptions("json", 256, 77, "rh-dax"))
    dt = time.perf_counter() - t0
    assert dt < 1.0, dt
    import json
    j = json.loads(out)
    assert len(j["samples"]) == 256 and j["seed"] == 77
    x = rep.final.download()
    assert j["samples"] == _ref_sample(n, x, 256, 77)


def test_large_state_samples_consistent_with_probabilities():
    """n=28 (4 GiB): the final sum is the norm to rounding and every sample's amplitude is
    nonzero (the index-exact checks run where the reference can take the state)."""
    from paper_2411_15332_b200 import qcsim as Q
    n = 28
    rep = Q.simulate(Q.build_grover(n, 123456, 3), Q.Engine.rh_dax)
    got, acc = rep.final.sample(200, 5)
    assert abs(acc - 1.0) < 1e-9
    amps = rep.final.gather(sorted(set(got)))
    assert np.all(np.abs(amps) > 0)


def test_summary_begin_end_equals_summary():
    """qcs_summary_begin/_end (the split form a serving loop uses) returns what qcs_summary does,
    and refuses a second pending summary or an end without a begin."""
    from paper_2411_15332_b200 import qcsim as Q
    x = _random_state(14, 9)
    s = Q.DeviceState.from_numpy(x)
    want = s.summary(16)
    s.summary_begin(16)
    with pytest.raises(ValueError):  # QCS_ERR_ARG
        s.summary_begin(16)
    assert s.summary_end() == want
    with pytest.raises(ValueError):
        s.summary_end()
    s.summary_begin(5)
    got = s.summary_end()
    assert got[1] == want[1][:5] and got[2] == want[2][:5] and got[0] == want[0]
