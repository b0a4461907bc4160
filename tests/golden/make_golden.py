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
        # the reference's own DAX1 / DAS1 serialisation of the same steps (dax.cpp:107-118,
        # das.cpp:154-165), hashed: the byte-level parity surface of SURVEY.md section 8f row 2
        dump_x = R.step_dump(n, plc, das=False)
        dump_s = R.step_dump(n, plc, das=True)
        recs.append(dict(n=n, names=[x[0] for x in pl], qubits=[x[1] for x in pl], seed=5000 + t,
                         dax=sha(np.concatenate([r_, c_, v_.view(np.uint64)])),
                         das=sha(np.concatenate([d_, l_.astype(np.uint64), dv_.view(np.uint64)])),
                         count=len(r_), mvm=sha(o),
                         dax_dump=hashlib.sha256(dump_x).hexdigest(), dax_dump_len=len(dump_x),
                         das_dump=hashlib.sha256(dump_s).hexdigest(), das_dump_len=len(dump_s)))
    with open(os.path.join(HERE, "steps.json"), "w") as f:
        json.dump(recs, f, indent=0)
    print("golden fixtures written")




def make_io_fixtures():
    """Reference front end (parse_circuit_json -> simulate -> render_report), oracle/_ref/libqcsim_io.so."""
    import subprocess

    def io_run(text, engine, fmt, samples, seed):
        # one process per call: keeps every reference run independent of the others
        out = subprocess.run([sys.executable, __file__, "io-one", text, engine, fmt, str(samples), str(seed)],
                             capture_output=True, text=True)
        code, _, body = out.stdout.partition("\n")
        return int(code), body
    circuits = {
        # exact values only: final states are bit-identical, so reports must be byte-identical
        "exact_perm": {"qubits": 5, "initial": 3, "steps": [
            [{"gate": "X", "targets": [0]}, {"gate": "CNOT", "targets": [1, 2]}],
            [{"gate": "Toffoli", "targets": [2, 3, 4]}], {"oracle": 7}, [{"gate": "SWAP", "targets": [0, 1]}],
            {"diag": {"flipped": [1, 2, 3], "flip_rest": True}}, [{"gate": "S", "targets": [4]}]]},
        "grover6": {"qubits": 6, "steps": [
            [{"gate": "H", "targets": [q]} for q in range(6)], {"oracle": 37},
            [{"gate": "H", "targets": [q]} for q in range(6)], {"z0": True},
            [{"gate": "H", "targets": [q]} for q in range(6)], {"oracle": 37},
            [{"gate": "H", "targets": [q]} for q in range(6)], {"z0": True},
            [{"gate": "H", "targets": [q]} for q in range(6)]]},
        "float_mix": {"qubits": 4, "steps": [
            [{"gate": "RY", "targets": [0], "params": [0.3]}, {"gate": "U", "targets": [1], "params": [1.1, 0.2, 2.5]},
             {"gate": "RXX", "targets": [2, 3], "params": [0.7]}],
            [{"gate": "CH", "targets": [0, 1]}, {"gate": "T", "targets": [3]}],
            [{"gate": "CCX", "targets": [1, 2, 3]}]]},
    }
    recs = []
    for name, circ in circuits.items():
        text = json.dumps(circ)
        for engine in ("rh-dax", "dax"):
            for fmt, samples, seed in (("json", 0, 0), ("json", 7, 99), ("csv", 0, 0), ("human", 5, 42)):
                n, body = io_run(text, engine, fmt, samples, seed)
                assert n >= 0, body
                recs.append(dict(name=name, circuit=text, engine=engine, format=fmt, samples=samples, seed=seed,
                                 output=body))
    errors = []
    for text in ['{"qubits": 2}', '[1, 2]', '{"qubits": 2, "steps": [[{"gate": "H"}]]}',
                 '{"qubits": 2, "steps": [[{"gate": "CNOT", "targets": [1, 0]}]]}',
                 '{"qubits": 2, "steps": [[{"gate": "CNOT", "targets": [0]}]]}',
                 '{"qubits": 2, "steps": [7]}', '{"qubits": 2, "steps": [[{"gate": "Nope", "targets": [0]}]]}',
                 '{"qubits": 2, "steps": [[{"gate": "H", "targets": [2]}]]}', '{"qubits": 2, "steps": [{"oracle": 4}]}',
                 '{"qubits": 2, "steps": [[{"gate": "H", "targets": [0]}, {"gate": "X", "targets": [0]}]]}']:
        n, body = io_run(text, "dax", "json", 0, 0)
        errors.append(dict(circuit=text, code=-n, message=body))
    with open(os.path.join(HERE, "io.json"), "w") as f:
        json.dump(dict(reports=recs, errors=errors), f, indent=0)
    print("io fixtures written")


if __name__ == "__main__":
    # the front-end library and the core reference library define the same symbols: one per process
    if len(sys.argv) > 1 and sys.argv[1] == "io":
        make_io_fixtures()
    elif len(sys.argv) > 1 and sys.argv[1] == "io-one":
        import ctypes as C
        lib = C.CDLL(os.path.join(ROOT, "oracle", "_ref", "libqcsim_io.so"))
        lib.io_run.restype = C.c_long
        lib.io_run.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_int, C.c_ulonglong, C.c_char_p, C.c_long]
        lib.io_last_error.restype = C.c_char_p
        buf = C.create_string_buffer(1 << 22)
        a = sys.argv[2:]
        n = lib.io_run(a[0].encode(), a[1].encode(), a[2].encode(), int(a[3]), int(a[4]), buf, len(buf))
        sys.stdout.write(f"{n}\n" + (buf.value.decode() if n >= 0 else lib.io_last_error().decode()))
    else:
        main()
