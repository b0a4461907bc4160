"""Fused-pass planner (host only, no GPU): pass counts through qcs_plan_stats.

The planner is B200-specific (the reference applies one step at a time, engine.cpp:153-210);
these tests pin its contract: every operation is scheduled, fusing never needs more HBM
sweeps than stepwise execution, and the BASELINE circuits get the pass counts DESIGN.md
quotes."""
import numpy as np
import pytest

from paper_2411_15332_b200 import configs
from paper_2411_15332_b200 import qcsim as Q

STEPWISE = Q.SimOptions(fuse=False)


def test_c1_is_one_pass():
    st = Q.plan_stats(configs.c1_circuit())
    assert st["passes"] == 1 and st["tile_passes"] == 1
    assert st["max_tile_bits"] == 12


def test_c3_grover_pass_count():
    st = Q.plan_stats(configs.c3_circuit(30))
    assert st["passes"] == 35          # 8 iterations, A.oracle.A and C.Z0.C fused
    assert Q.plan_stats(configs.c3_circuit(30), opts=STEPWISE)["passes"] > st["passes"]


def test_grover_sign_passes_skip_missed_tiles():
    # each oracle / Z0 step sits in a pass mirrored around it (H_b ... sign ... H_b): on the
    # tiles it does not reach the pass is a scalar, carried by another pass, so only the
    # reached tiles are launched
    for n in (22, 30):
        st = Q.plan_stats(configs.c3_circuit(n))
        assert st["skip_passes"] == st["alt_passes"] == 16, n


def test_grover_pass_pairs_around_skip_passes():
    # between two skip passes, the H_low passes come in pairs H_low Q H_low with Q a skip pass:
    # H_low H_low = 2^12 I, so each pair runs only on the 2^9 H_low tiles that Q's one reached
    # tile meets; at n = 30 three passes remain full sweeps (the first H^n)
    st = Q.plan_stats(configs.c3_circuit(30))
    assert st["paired_passes"] == 16
    assert st["passes"] - st["skip_passes"] - st["paired_passes"] == 3
    # no pairs where the middle pass is not a skip pass
    assert Q.plan_stats(configs.c4_circuit(24, 2))["paired_passes"] == 0


def test_rh_is_ceil_passes():
    # H on every qubit: a 12-bit tile takes bits 0..11, later tiles 9 new bits each (0..2 fixed)
    for n, want in [(12, 1), (21, 2), (28, 3), (30, 3), (32, 4)]:
        c = Q.Circuit(n, [Q.hadamard_all(n)])
        assert Q.plan_stats(c)["passes"] == want, n


def test_rh_engine_only_for_rh_dax():
    c = Q.Circuit(14, [Q.hadamard_all(14)])
    rh = Q.plan_stats(c, Q.Engine.rh_dax)
    dax = Q.plan_stats(c, Q.Engine.dax)
    assert rh["ops"] == 15             # the scale plus 14 butterflies
    assert dax["ops"] == 14            # 14 Hadamard placements
    assert rh["passes"] == dax["passes"] == 2


@pytest.mark.parametrize("seed", range(6))
def test_fused_never_needs_more_passes(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(13, 26))
    names = ["Hadamard", "Pauli-X", "T", "RY", "Controlled-X", "Controlled-Z", "Swap"]
    steps = []
    for _ in range(int(rng.integers(5, 30))):
        name = names[int(rng.integers(0, len(names)))]
        g = Q.gate_catalog_lookup(name, [float(rng.uniform(0, 6.28))] if name == "RY" else [])
        qs = [int(q) for q in rng.choice(n, g.arity, replace=False)]
        steps.append(Q.CircuitStep.of_gates([Q.Placement(g, qubits=qs)]))
    c = Q.Circuit(n, steps)
    fused = Q.plan_stats(c)
    step = Q.plan_stats(c, opts=STEPWISE)
    assert fused["passes"] <= step["passes"]
    assert step["ops"] == len(steps)
    assert fused["ops"] <= step["ops"]
    assert fused["passes"] == fused["tile_passes"] + fused["single_passes"]


def test_small_states_run_one_op_per_pass():
    c = Q.Circuit(2, [Q.CircuitStep.of_gates([Q.Placement(Q.gate_catalog_lookup("Hadamard"), 0)]),
                      Q.CircuitStep.of_gates([Q.Placement(Q.gate_catalog_lookup("Pauli-X"), 1)])])
    st = Q.plan_stats(c)
    assert st["tile_passes"] == 0 and st["single_passes"] == st["passes"] == 2


def test_invalid_circuit_rejected_like_simulate():
    with pytest.raises(Q.SimError):
        Q.plan_stats(Q.Circuit(3, [Q.CircuitStep.of_gates([Q.Placement(Q.gate_catalog_lookup("Pauli-X"), 5)])]))
