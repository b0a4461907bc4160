"""Pass kernels specialised at run time (csrc/jit.cpp, NVRTC) against the interpreter kernel
k_tile: the generated source must compile for every kind of tile operation and round (CPU,
NVRTC only), and on the GPU both forms must give bit-identical states up to the sign of exact
zeros (same arithmetic, same order; X-like gates become register swaps instead of 0*x0 + 1*x1)
(mode 2), and with pivoted gates (mode 3, the default for big passes) agree with the oracle,
on circuits that exercise gates (real / complex, bundled, controls inside and outside
the tile), diagonal tables and phases on 1-3 bits, sign flips and sign steps with missed-tile
programs, butterflies, scales and shared-memory gate rounds."""
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import bits_equal, canon_zero


@pytest.fixture(scope="module")
def Q():
    from paper_2411_15332_b200 import qcsim
    return qcsim


@pytest.fixture(scope="module")
def cfg():
    from paper_2411_15332_b200 import configs
    return configs


def random_catalog_circuit(Q, seed, n, nsteps=40):
    """Random steps over the whole gate catalog (any arity, reversed / non-adjacent qubits), with
    sign steps mixed in (as tests/test_edge_gpu.py)."""
    rng = np.random.default_rng(100 + seed)
    infos = Q.gate_catalog()
    steps = [Q.hadamard_all(n)]
    for _ in range(nsteps):
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
    return Q.Circuit(n, steps, int(rng.integers(0, 1 << n)))


def sign_sandwich(Q, n):
    rng = np.random.default_rng(n)
    H = Q.hadamard_all(n)
    signs = [Q.DiagSign([int(i) for i in rng.choice(1 << n, k, replace=False)], rest)
             for k, rest in ((1, False), (1, True), (5, False), (80, True), (0, True))]
    steps = [H]
    for d in signs:
        steps += [Q.CircuitStep.of_diag(d), H]
    steps.insert(4, Q.CircuitStep.of_gates([Q.Placement(Q.gate_catalog_lookup("RY", [0.37]), 2)]))
    return Q.Circuit(n, steps)


def test_generated_sources_compile(Q, cfg):
    """Every tile pass of these plans becomes a kernel that NVRTC compiles for sm_100a."""
    circuits = [random_catalog_circuit(Q, 0, 13, 24), sign_sandwich(Q, 13), cfg.c4_circuit(14, 2),
                cfg.c5_circuit(14, 2, global_qubits=2)]
    for c in circuits:
        st = Q.plan_stats(c)
        r = Q.plan_compile(c)
        assert r["kernels"] == st["tile_passes"] > 0
        assert r["cubin_bytes"] > 0


def test_addressing_proof(Q, cfg):
    """qcs_plan_verify (host only): every register round of every specialised pass kernel of the
    BASELINE families and of random whole-catalog circuits, in every jit mode that changes the
    generated code (relabellings, pivots), addresses each shared-memory slot of its tile exactly
    once -- in bounds and a permutation -- for every thread, group iteration and register; and a
    relabelled last round's direct HBM stores cover the tile exactly once.  (compute-sanitizer is
    closed on the GPU pool; this is the memcheck of the generated kernels' data accesses.)"""
    old = Q.jit_mode()
    try:
        for mode in (1, 3):
            Q.set_jit_mode(mode)
            checked = 0
            for n in (12, 16, 20, 24, 28, 32):
                checked += Q.plan_verify(cfg.c4_circuit(n, 10))
                checked += Q.plan_verify(cfg.c5_circuit(max(n, 16), 20, global_qubits=2))
                checked += Q.plan_verify(cfg.c3_circuit(n) if n >= 16 else cfg.c1_circuit())
            for seed in range(6):
                checked += Q.plan_verify(random_catalog_circuit(Q, seed, 13 + seed, 40))
            checked += Q.plan_verify(sign_sandwich(Q, 15))
            assert checked > 300
    finally:
        Q.set_jit_mode(old)


def test_plans_do_not_depend_on_history(Q, cfg):
    """The same circuit plans the same way whatever was planned before (a read past the
    operation list once made relabelled plans depend on heap contents)."""
    old = Q.jit_mode()
    try:
        Q.set_jit_mode(3)
        c = cfg.c5_circuit(15, 3, global_qubits=2)
        first = Q.plan_stats(c)
        for other in (random_catalog_circuit(Q, 0, 13), sign_sandwich(Q, 15), cfg.c4_circuit(11, 3)):
            Q.plan_stats(other)
            assert Q.plan_stats(c) == first
    finally:
        Q.set_jit_mode(old)


def test_disk_cache_of_compiled_kernels(tmp_path):
    """QCS_JIT_CACHE=<dir>: a second process finds the compiled pass kernels on disk (each entry
    one file holding its full source as the key and a hash of the cubin, published by an atomic
    rename of a mkstemp file) instead of compiling them."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import time; t = time.time(); from paper_2411_15332_b200 import configs, qcsim as Q; "
            "r = Q.plan_compile(configs.c4_circuit(14, 2)); print(r['kernels'], r['cubin_bytes'], time.time() - t)")
    env = dict(os.environ, QCS_JIT_CACHE=str(tmp_path))
    runs = [subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, check=True)
            .stdout.split() for _ in range(2)]
    assert runs[0][:2] == runs[1][:2] and int(runs[0][0]) > 0
    entries = [f for f in os.listdir(tmp_path) if f.endswith(".kc")]
    assert len(entries) == int(runs[0][0])
    assert not [f for f in os.listdir(tmp_path) if not f.endswith(".kc")]  # no temp files left
    assert float(runs[1][2]) < float(runs[0][2])
    # a torn entry (cut short) is recompiled and replaced, never loaded
    victim = os.path.join(tmp_path, entries[0])
    with open(victim, "r+b") as f:
        f.truncate(os.path.getsize(victim) // 2)
    again = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, check=True)
    assert again.stdout.split()[:2] == runs[0][:2]
    assert os.path.getsize(victim) > 0 and len([f for f in os.listdir(tmp_path) if f.endswith(".kc")]) == len(entries)


def test_jit_mode_switch(Q):
    old = Q.jit_mode()
    try:
        for m in (0, 2, 3, 1):
            Q.set_jit_mode(m)
            assert Q.jit_mode() == m
        with pytest.raises(ValueError):
            Q.set_jit_mode(4)
    finally:
        Q.set_jit_mode(old)


def same(a, b):
    """Bit for bit after mapping -0.0 to +0.0."""
    return bits_equal(canon_zero(a), canon_zero(b))


def run_mode(Q, c, mode, fuse=True):
    old = Q.jit_mode()
    Q.set_jit_mode(mode)
    try:
        return Q.simulate(c, Q.Engine.rh_dax, Q.SimOptions(fuse=fuse)).final.download()
    finally:
        Q.set_jit_mode(old)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(3))
def test_specialised_equals_interpreter_random(Q, seed):
    """(Every pass compiles its own kernel here, ~0.5 s each: the stepwise form only once.)"""
    n = 13 + seed
    c = random_catalog_circuit(Q, seed, n)
    for fuse in ((True, False) if seed == 0 else (True,)):
        assert same(run_mode(Q, c, 2, fuse), run_mode(Q, c, 0, fuse)), (seed, fuse)


@pytest.mark.gpu
def test_specialised_equals_interpreter_circuits(Q, cfg):
    circuits = [sign_sandwich(Q, 16), cfg.c4_circuit(16, 3), cfg.c5_circuit(16, 3, global_qubits=2),
                cfg.c3_circuit(18), cfg.c1_circuit()]
    for c in circuits:
        assert same(run_mode(Q, c, 2), run_mode(Q, c, 0)), c.n


TOL_AMP, TOL_L2 = 1e-12, 1e-10


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


@pytest.mark.gpu
def test_pivoted_gates_against_oracle(Q, cfg, oracle):
    """Mode 3: every tile pass specialised, with pivoted gates (row scales folded into the
    rounds' diagonal tables: a different rounding, so the floating-point bar) against the
    oracle."""
    G = Q.gate_catalog_lookup
    # a deferred row scale of a controlled gate is a diagonal on its control bits too: a later
    # gate on the control bit in the same round must keep it from moving (regression)
    ctrl_chain = Q.Circuit(12, [Q.hadamard_all(12)] + [Q.CircuitStep.of_gates([p]) for p in (
        Q.Placement(G("RX", [5.703]), qubits=[0]),
        Q.Placement(G("CU", [2.54, 4.966, 2.455, 3.298]), qubits=[11, 9]),
        Q.Placement(G("CU", [3.229, 1.978, 4.731, 1.819]), qubits=[0, 11]))])
    # (random whole-catalog circuits compile ~2 s per pass: shared-memory gate rounds)
    circuits = [random_catalog_circuit(Q, 0, 13), random_catalog_circuit(Q, 5, 14, 16)]
    circuits += [ctrl_chain, sign_sandwich(Q, 15), cfg.c4_circuit(11, 3), cfg.c5_circuit(15, 3, global_qubits=2),
                 cfg.c3_circuit(14), cfg.c1_circuit()]
    for c in circuits:
        want = oracle_run(oracle, c)
        for fuse in (True,):
            got = run_mode(Q, c, 3, fuse)
            assert np.abs(got - want).max() <= TOL_AMP, (c.n, fuse)
            assert np.linalg.norm(got - want) <= TOL_L2, (c.n, fuse)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(2))
def test_default_mode_relabels_big_passes(Q, cfg, seed):
    """At n = 23 (2048 tiles per pass) the default mode lowers X-like gates (X, CNOT, the X of Y)
    to relabellings and conjugates later diagonals ahead of them: the C5 family and random
    whole-catalog circuits (controls inside and outside the tile, reversed pairs) agree with the
    interpreter, which the oracle checks elsewhere."""
    c = cfg.c5_circuit(23, 4, global_qubits=2) if seed == 0 else random_catalog_circuit(Q, 7, 23, 30)
    got, want = run_mode(Q, c, 1), run_mode(Q, c, 0)
    assert np.abs(got - want).max() <= TOL_AMP
    assert np.linalg.norm(got - want) <= TOL_L2


@pytest.mark.gpu
def test_default_mode_specialises_big_passes(Q, cfg):
    """At n = 22 the C4 passes (1024 tiles x >= 32 rounds) take the specialised kernels with
    pivoted gates in the default mode: within the bar of the (oracle-checked) interpreter."""
    c = cfg.c4_circuit(22, 2)
    got, want = run_mode(Q, c, 1), run_mode(Q, c, 0)
    assert np.abs(got - want).max() <= TOL_AMP
    assert np.linalg.norm(got - want) <= TOL_L2


# ---------------------------------------------------------------- persistent pipelined form
def run_pipeline(Q, c, pmode):
    old = Q.pipeline_mode()
    Q.set_pipeline_mode(pmode)
    try:
        return Q.simulate(c, Q.Engine.rh_dax).final.download()  # a fresh state: a fresh plan cache
    finally:
        Q.set_pipeline_mode(old)


def test_pipelined_sources_compile_and_address(Q, cfg):
    """CPU: with every eligible pass in the persistent pipelined form (mode 2) the generated
    sources still compile for sm_100a and pass the addressing proof; the plans are the same."""
    old = Q.pipeline_mode()
    try:
        for mode in (0, 2):
            Q.set_pipeline_mode(mode)
            for c in (cfg.c4_circuit(24, 3), cfg.c3_circuit(24)):
                st = Q.plan_stats(c)
                assert Q.plan_compile(c)["kernels"] == st["tile_passes"]
                assert Q.plan_verify(c) == st["tile_passes"]
        with pytest.raises(ValueError):
            Q.set_pipeline_mode(3)
    finally:
        Q.set_pipeline_mode(old)
    assert Q.pipeline_mode() == old


@pytest.mark.gpu
@pytest.mark.parametrize("family", ["c4", "c3", "random"])
def test_pipelined_equals_one_tile_per_cta(Q, cfg, family):
    """The persistent pipelined kernels (one CTA per SM, two compute groups over a ring of TMA
    tile slots) run the same arithmetic in the same order as the one-tile-per-CTA kernels: the
    states are bit-identical, for the default (16-register passes) and with every eligible pass
    pipelined (8-register rounds, butterflies: short tiles, where a group that runs ahead of the
    other's loads once read a slot that was not its own)."""
    c = {"c4": lambda: cfg.c4_circuit(24, 4), "c3": lambda: cfg.c3_circuit(24),
         "random": lambda: random_catalog_circuit(Q, 11, 23, 30)}[family]()
    want = run_pipeline(Q, c, 0)
    for pmode in (1, 2):
        for rep in range(2):  # the first run is the cold one (compiles, first touch of the state)
            assert bits_equal(run_pipeline(Q, c, pmode), want), (family, pmode, rep)
