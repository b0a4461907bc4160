"""The BASELINE.json workloads as seeded circuits (synthetic inputs).

Seeds are 20241122 + config number.  Angles are uniform in [0, 2*pi) from numpy's
``default_rng(seed)``; random states are i.i.d. Gaussian re/im, L2-normalised.  The reference
publishes no dataset for this path; these generators stand in with the configs' stated shapes.

amplitude-updates (the metric's unit) = sum over gates of 2^n, where an H on all qubits counts
as n gates and the Grover oracle / Z0 count as one each.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Tuple

import numpy as np

from . import qcsim as Q

SEED = 20241122
TWO_PI = 2.0 * np.pi


def seed_of(config: int) -> int:
    return SEED + config


# ------------------------------------------------------------------ C1: 12-qubit QNN-style
def c1_circuit(n: int = 12, layers: int = 4, seed: int = seed_of(1)) -> Q.Circuit:
    """H on all qubits; then per layer: RY(theta_q) on every qubit (one step), the CNOT chain
    q -> q+1 for q = 0..n-2 (one step each), RZ(phi_q) on every qubit (one step)."""
    rng = np.random.default_rng(seed)
    c = Q.Circuit(n, [Q.hadamard_all(n)])
    cx = Q.gate_catalog_lookup("Controlled-X")
    for _ in range(layers):
        theta = rng.uniform(0.0, TWO_PI, n)
        phi = rng.uniform(0.0, TWO_PI, n)
        c.steps.append(Q.CircuitStep.of_gates([Q.Placement(Q.gate_catalog_lookup("RY", [theta[q]]), q)
                                               for q in range(n)]))
        for q in range(n - 1):
            c.steps.append(Q.CircuitStep.of_gates([Q.Placement(cx, q)]))
        c.steps.append(Q.CircuitStep.of_gates([Q.Placement(Q.gate_catalog_lookup("RZ", [phi[q]]), q)
                                               for q in range(n)]))
    return c


def c1_updates(n: int = 12, layers: int = 4) -> int:
    return (n + layers * (n + (n - 1) + n)) << n  # 152 gates at n = 12


# ------------------------------------------------------------------ C2: single-gate sweep
C2_GATES = ["X", "Y", "Z", "S", "T", "CNOT", "CZ", "SWAP", "Toffoli", "H", "RX", "U3"]


@dataclass
class SweepGate:
    label: str          # C2_GATES label
    gate: Q.GateSpec
    qubits: List[int]   # gate-local order: controls first, target last


def c2_sweep(n: int = 28, seed: int = seed_of(2)) -> List[SweepGate]:
    """Every C2 gate with its target swept over all n qubits; controls / partners drawn from the
    same rng, distinct from the target (and from each other)."""
    rng = np.random.default_rng(seed)
    out = []
    names = {"X": "Pauli-X", "Y": "Pauli-Y", "Z": "Pauli-Z", "S": "S", "T": "T", "CNOT": "Controlled-X",
             "CZ": "Controlled-Z", "SWAP": "Swap", "Toffoli": "CCX", "H": "Hadamard", "RX": "RX", "U3": "U"}
    for label in C2_GATES:
        for t in range(n):
            others = [q for q in range(n) if q != t]
            params: List[float] = []
            if label == "RX":
                params = [float(rng.uniform(0.0, TWO_PI))]
            elif label == "U3":
                params = [float(x) for x in rng.uniform(0.0, TWO_PI, 3)]
            g = Q.gate_catalog_lookup(names[label], params)
            if label in ("CNOT", "CZ", "SWAP"):
                c = int(rng.choice(others))
                qs = [c, t]
            elif label == "Toffoli":
                c1, c2 = (int(x) for x in rng.choice(others, 2, replace=False))
                qs = [c1, c2, t]
            else:
                qs = [t]
            out.append(SweepGate(label, g, qs))
    return out


def c2_updates(n: int = 28) -> int:
    return len(C2_GATES) * n << n


# ------------------------------------------------------------------ C3: Grover
def c3_marked(n: int = 30, seed: int = seed_of(3)) -> int:
    return int(np.random.default_rng(seed).integers(0, 1 << n))


def c3_circuit(n: int = 30, iterations: int = 8, seed: int = seed_of(3)) -> Q.Circuit:
    return Q.build_grover(n, c3_marked(n, seed), iterations)


def c3_updates(n: int = 30, iterations: int = 8) -> int:
    return (n + iterations * (1 + n + 1 + n)) << n  # 526 gate-equivalents at n = 30


def grover_closed_form(n: int, iterations: int) -> Tuple[float, float]:
    """Amplitudes after k Grover iterations with the reference's Z0 (circuit.cpp:92):
    a_marked = sin((2k+1) t), a_other = cos((2k+1) t) / sqrt(2^n - 1), t = asin(2^{-n/2})."""
    t = np.arcsin(2.0 ** (-n / 2.0))
    a = (2 * iterations + 1) * t
    return float(np.sin(a)), float(np.cos(a) / np.sqrt(2.0 ** n - 1.0))


# ------------------------------------------------------------------ C4: 32-qubit QNN
def c4_circuit(n: int = 32, layers: int = 10, seed: int = seed_of(4)) -> Q.Circuit:
    """H all; per layer RY(theta_q) all, RZ(phi_q) all, CZ ring (q, q+1 mod n) as three steps
    (even pairs, odd pairs, the wrap pair (n-1, 0))."""
    rng = np.random.default_rng(seed)
    c = Q.Circuit(n, [Q.hadamard_all(n)])
    cz = Q.gate_catalog_lookup("Controlled-Z")
    for _ in range(layers):
        theta = rng.uniform(0.0, TWO_PI, n)
        phi = rng.uniform(0.0, TWO_PI, n)
        c.steps.append(Q.CircuitStep.of_gates([Q.Placement(Q.gate_catalog_lookup("RY", [theta[q]]), q)
                                               for q in range(n)]))
        c.steps.append(Q.CircuitStep.of_gates([Q.Placement(Q.gate_catalog_lookup("RZ", [phi[q]]), q)
                                               for q in range(n)]))
        c.steps.append(Q.CircuitStep.of_gates([Q.Placement(cz, q) for q in range(0, n - 1, 2)]))
        c.steps.append(Q.CircuitStep.of_gates([Q.Placement(cz, q) for q in range(1, n - 1, 2)]))
        c.steps.append(Q.CircuitStep.of_gates([Q.Placement(cz, qubits=[n - 1, 0])]))
    return c


def c4_updates(n: int = 32, layers: int = 10) -> int:
    return (n + layers * 3 * n) << n  # 992 gates at n = 32


# ------------------------------------------------------------------ C5: 35-qubit random circuit
C5_POOL = ["Pauli-X", "Pauli-Y", "Pauli-Z", "S", "T", "Hadamard", "RX", "RY", "RZ"]


def c5_circuit(n: int = 35, layers: int = 20, global_qubits: int = 3, seed: int = seed_of(5)) -> Q.Circuit:
    """H all; per layer one gate per qubit from C5_POOL (angles U[0, 2pi)), then CNOT on
    floor(n/2) disjoint pairs from a shuffle, resampled until a pair touches the top
    `global_qubits` qubits (the shard-global ones)."""
    rng = np.random.default_rng(seed)
    c = Q.Circuit(n, [Q.hadamard_all(n)])
    cx = Q.gate_catalog_lookup("Controlled-X")
    for _ in range(layers):
        pl = []
        for q in range(n):
            name = C5_POOL[int(rng.integers(0, len(C5_POOL)))]
            params = [float(rng.uniform(0.0, TWO_PI))] if name in ("RX", "RY", "RZ") else []
            pl.append(Q.Placement(Q.gate_catalog_lookup(name, params), q))
        c.steps.append(Q.CircuitStep.of_gates(pl))
        while True:
            perm = [int(x) for x in rng.permutation(n)]
            pairs = [(perm[2 * i], perm[2 * i + 1]) for i in range(n // 2)]
            if any(a < global_qubits or b < global_qubits for a, b in pairs):
                break
        c.steps.append(Q.CircuitStep.of_gates([Q.Placement(cx, qubits=[a, b]) for a, b in pairs]))
    return c


def c5_updates(n: int = 35, layers: int = 20) -> int:
    return (n + layers * (n + n // 2)) << n  # 1075 gates at n = 35
