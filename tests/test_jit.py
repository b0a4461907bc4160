"""Pass kernels specialised at run time (csrc/jit.cpp, NVRTC) against the interpreter kernel
k_tile: the generated source must compile for every kind of tile operation and round (CPU,
NVRTC only), and on the GPU both forms must give bit-identical states up to the sign of exact
zeros (same arithmetic, same order; X-like gates become register swaps instead of 0*x0 + 1*x1)
on circuits that exercise gates (real / complex, bundled, controls inside and outside
the tile), diagonal tables and phases on 1-3 bits, sign flips and sign steps with missed-tile
programs, butterflies, scales and shared-memory gate rounds."""
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


def test_jit_mode_switch(Q):
    old = Q.jit_mode()
    try:
        for m in (0, 2, 1):
            Q.set_jit_mode(m)
            assert Q.jit_mode() == m
        with pytest.raises(ValueError):
            Q.set_jit_mode(3)
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
@pytest.mark.parametrize("seed", range(4))
def test_specialised_equals_interpreter_random(Q, seed):
    n = 13 + seed
    c = random_catalog_circuit(Q, seed, n)
    for fuse in (True, False):
        assert same(run_mode(Q, c, 2, fuse), run_mode(Q, c, 0, fuse)), (seed, fuse)


@pytest.mark.gpu
def test_specialised_equals_interpreter_circuits(Q, cfg):
    circuits = [sign_sandwich(Q, 16), cfg.c4_circuit(16, 3), cfg.c5_circuit(16, 3, global_qubits=2),
                cfg.c3_circuit(18), cfg.c1_circuit()]
    for c in circuits:
        assert same(run_mode(Q, c, 2), run_mode(Q, c, 0)), c.n


@pytest.mark.gpu
def test_default_mode_specialises_big_passes(Q, cfg):
    """At n = 22 the C4 passes (1024 tiles x >= 32 rounds) take the specialised kernels in the
    default mode; same bits as the interpreter."""
    c = cfg.c4_circuit(22, 2)
    assert same(run_mode(Q, c, 1), run_mode(Q, c, 0))
