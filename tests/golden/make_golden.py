"""Regenerate the golden fixtures in tests/golden/ from the UNMODIFIED reference library.

    make -C oracle ref && python tests/golden/make_golden.py

Needs oracle/_ref/libqcsim_ref.so (built from /root/reference/proj/src, so only where the
reference is mounted).  The fixtures are small and committed; the GPU box never reads
/root/reference.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle_py import Reference as R  # noqa: E402
from paper_2411_15332_b200 import configs  # noqa: E402

RNG_SEED = 7


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def steps_for_reference(circuit):
    """Python Circuit -> Reference.simulate step list (names + native placements)."""
    out = []
    for st in circuit.steps:
        if int(st.kind) == 1:
            out.append(("diag", list(st.diag.flipped), st.diag.flip_rest, st.stage))
        else:
            out.append(("gates", [(p.gate.name, p.qubit_list(), p.gate.matrix) for p in st.placements], st.stage))
    return out


def main():
    rng = np.random.default_rng(RNG_SEED)
    # --- gate catalog bytes (gates.cpp:169-222) at canonical and random parameters
    names, arity, params, mats = [], [], [], []
    for name, k, npar, _ in R.catalog():
        sets = [R.canonical_params(name)] + [list(rng.uniform(-7, 7, npar)) for _ in range(3 if npar else 0)]
        for p in sets:
            names.append(name)
            arity.append(k)
            params.append(np.pad(np.asarray(p, float), (0, 4 - len(p))))
            mats.append(np.pad(R.gate(name, p).reshape(-1), (0, 64 - 4 ** k)))
    np.savez_compressed(os.path.join(HERE, "gates.npz"), names=np.array(names), arity=np.array(arity),
                        params=np.array(params), mats=np.array(mats))

    # --- C1 (12-qubit QNN-style) final state, reference rh-dax engine with layer steps
    c1 = configs.c1_circuit()
    final, reports, secs = R.simulate(c1.n, steps_for_reference(c1), engine="rh-dax")
    np.savez_compressed(os.path.join(HERE, "c1.npz"), final=final,
                        structure=np.array([r["structure"] for r in reports]),
                        entry_count=np.array([r["entry_count"] for r in reports], np.uint64),
                        sign_count=np.array([r["sign_count"] for r in reports], np.uint64),
                        madd_count=np.array([r["madd_count"] for r in reports], np.uint64),
                        matrix_bytes=np.array([r["matrix_bytes"] for r in reports], np.uint64))
    print(f"C1 reference simulate: {secs:.2f} s")

    # --- Grover (reference build_grover + simulate, rh-dax), n = 4..10 auto iterations
    gro = {}
    for n in range(4, 11):
        marked = (1 << n) - 3
        gro[f"n{n}"] = R.grover(n, marked, 0, "rh-dax")
    gro["n10_k3"] = R.grover(10, 777, 3, "rh-dax")
    np.savez_compressed(os.path.join(HERE, "grover.npz"), **gro)

    # --- QNN neuron (acceptance.cpp:293-319 angles/weights)
    pi = np.pi
    ang = [pi / 3, 0.9, pi / 5, 2.2, 0.4, 1.7, pi / 7, 2.9]
    w = [1, -1, 1, 1, -1, 1, 1, -1]
    np.savez_compressed(os.path.join(HERE, "qnn.npz"), angles=np.array(ang), weights=np.array(w),
                        final=R.qnn(ang, w, "rh-dax"))

    # --- C2 sweep at n = 6 (full outputs) and n = 12 (sha256 of output bytes), reference
    #     step_matrix_dax (+ projector decomposition for non-adjacent controls) then dax_mvm
    for n, full in ((6, True), (12, False)):
        s = R.random_unit_state(n, 1000 + n)
        outs, hashes, labels, qubits = [], [], [], []
        for g in configs.c2_sweep(n, seed=configs.seed_of(2)):
            o, _, _ = R.apply_step(n, [(g.qubits, g.gate.matrix)], s)
            labels.append(g.label)
            qubits.append(np.pad(g.qubits, (0, 3 - len(g.qubits)), constant_values=-1))
            if full:
                outs.append(o)
            hashes.append(sha(o))
        payload = dict(state=s, labels=np.array(labels), qubits=np.array(qubits), sha=np.array(hashes))
        if full:
            payload["outputs"] = np.array(outs)
        np.savez_compressed(os.path.join(HERE, f"sweep_n{n}.npz"), **payload)

    # --- random native steps: reference DAX / DAS bytes (sha) and MVM outputs (sha), n <= 8
    cat = R.catalog()
    recs = []
    for t in range(60):
        n = int(rng.integers(2, 9))
        pl, q = [], 0
        while q < n:
            ar = 1 + int(rng.integers(0, min(n - q, 3)))
            fits = [c for c in cat if c[1] == ar]
            name, _, npar, _ = fits[int(rng.integers(0, len(fits)))]
            pl.append((name, list(range(q, q + ar)), R.gate(name, R.canonical_params(name))))
            q += ar + int(rng.integers(0, 2))
        plc = [(qs, m) for _, qs, m in pl]
        r_, c_, v_ = R.step_dax(n, plc)
        d_, l_, dv_ = R.step_das(n, plc)
        s = R.random_unit_state(n, 5000 + t)
        o, _, _ = R.apply_step(n, plc, s)
        recs.append(dict(n=n, names=[x[0] for x in pl], qubits=[x[1] for x in pl], seed=5000 + t,
                         dax=sha(np.concatenate([r_, c_, v_.view(np.uint64)])),
                         das=sha(np.concatenate([d_, l_.astype(np.uint64), dv_.view(np.uint64)])),
                         count=len(r_), mvm=sha(o)))
    with open(os.path.join(HERE, "steps.json"), "w") as f:
        json.dump(recs, f, indent=0)
    print("golden fixtures written")


if __name__ == "__main__":
    main()
