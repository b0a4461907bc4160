"""The reference's front end (src/circuit_io.cpp, include/qcsim/circuit_io.hpp) over the B200 engine.

* ``parse_circuit_json`` / ``load_circuit_file`` (circuit_io.cpp:16-83): the same schema, rules
  and ParseError messages (JSON syntax errors keep the ``circuit JSON:`` prefix; the detail text
  comes from Python's parser, not nlohmann's);
* ``parse_gate_expression`` (circuit_io.cpp:85-107): catalog gates joined by ``x`` / ``*``;
* ``render_report`` (circuit_io.cpp:109-203): human / JSON / CSV, key-ordered, with seeded
  sampling.  The JSON layout and number formatting follow nlohmann::ordered_json::dump(2); the
  samples come from the device (qcs_sample): the reference's generator chain (std::mt19937_64 ->
  uniform_real_distribution(0, acc) -> lower_bound) on an exact reproduction of its sequential
  rounded CDF, so equal probabilities give equal samples and no 2^n values are downloaded.

Probabilities, argmax and the norm come from the device (qcs_probabilities is bit-exact; large
states report argmax and top-16 without downloading the state, as the reference does above 2^16
amplitudes).
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass
from typing import List

import numpy as np

from . import qcsim as Q


# ---------------------------------------------------------------- parsing
def _placement(j) -> Q.Placement:  # circuit_io.cpp:16-31
    if not isinstance(j, dict) or "gate" not in j or "targets" not in j:
        raise Q.ParseError('placement needs "gate" and "targets"')
    params = j.get("params", [])
    gate = Q.gate_catalog_lookup(_string(j["gate"]), [_number(p) for p in _array(params)])
    targets = [_int(t) for t in _array(j["targets"])]
    if len(targets) != gate.arity:
        raise Q.ParseError(f"gate {gate.name} targets {gate.arity} qubit(s)")
    for i in range(1, len(targets)):
        if targets[i] != targets[i - 1] + 1:
            raise Q.ParseError("gate targets must be ascending and contiguous")
    return Q.Placement(gate, targets[0])


def _step(j) -> Q.CircuitStep:  # circuit_io.cpp:33-52
    if isinstance(j, list):
        return Q.CircuitStep.of_gates([_placement(p) for p in j])
    if isinstance(j, dict):
        if "oracle" in j:
            return Q.CircuitStep.of_diag(Q.DiagSign([_uint(j["oracle"])], False))
        if "z0" in j:
            return Q.CircuitStep.of_diag(Q.DiagSign([0], True))
        if "diag" in j:
            d = j["diag"]
            if not isinstance(d, dict) or "flipped" not in d:
                raise Q.ParseError('circuit JSON: key "flipped" not found')
            return Q.CircuitStep.of_diag(Q.DiagSign([_uint(x) for x in _array(d["flipped"])],
                                                    bool(_boolean(d.get("flip_rest", False)))))
    raise Q.ParseError("step must be a placement list or a diagonal object")


def _type_error(want, got):
    kinds = {dict: "object", list: "array", str: "string", bool: "boolean", type(None): "null"}
    return Q.ParseError(f"circuit JSON: type must be {want}, but is {kinds.get(type(got), 'number')}")


def _int(v):
    if isinstance(v, bool) or not isinstance(v, (int, float)):
        raise _type_error("number", v)
    return int(v)


def _uint(v):
    return _int(v) & ((1 << 64) - 1)


def _number(v):
    if isinstance(v, bool) or not isinstance(v, (int, float)):
        raise _type_error("number", v)
    return float(v)


def _string(v):
    if not isinstance(v, str):
        raise _type_error("string", v)
    return v


def _array(v):
    if not isinstance(v, list):
        raise _type_error("array", v)
    return v


def _boolean(v):
    if not isinstance(v, bool):
        raise _type_error("boolean", v)
    return v


def parse_circuit_json(text: str) -> Q.Circuit:  # circuit_io.cpp:56-75
    try:
        j = json.loads(text)
    except (json.JSONDecodeError, TypeError) as e:
        raise Q.ParseError(f"circuit JSON: parse error: {e}") from None
    if not isinstance(j, dict) or "qubits" not in j or "steps" not in j:
        raise Q.ParseError('circuit needs "qubits" and "steps"')
    c = Q.Circuit(_int(j["qubits"]), [_step(s) for s in _array(j["steps"])], _uint(j.get("initial", 0)))
    c.validate()
    return c


def load_circuit_file(path: str) -> Q.Circuit:  # circuit_io.cpp:77-83
    try:
        with open(path, "r") as f:
            text = f.read()
    except OSError:
        raise Q.ParseError("cannot open circuit file: " + path) from None
    return parse_circuit_json(text)


def _dense_tensor(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """core.cpp:55-72 with std::complex<double> products (separately rounded)."""
    rows, cols = a.shape[0] * b.shape[0], a.shape[1] * b.shape[1]
    cap = int(Q.L.lib().qcs_dense_cap())
    if rows and cols > cap // rows:
        raise Q.CapacityError(f"dense tensor product exceeds dense cap of {cap} elements")
    out = np.zeros((rows, cols), np.complex128)
    for ra in range(a.shape[0]):
        for rb in range(b.shape[0]):
            for ca in range(a.shape[1]):
                va = a[ra, ca]
                for cb in range(b.shape[1]):
                    vb = b[rb, cb]
                    out[ra * b.shape[0] + rb, ca * b.shape[1] + cb] = complex(
                        va.real * vb.real - va.imag * vb.imag, va.real * vb.imag + va.imag * vb.real)
    return out


def parse_gate_expression(expr: str) -> np.ndarray:  # circuit_io.cpp:85-107
    names = expr.split()
    gates = []
    for i, tok in enumerate(names):
        if i % 2 == 1:
            if tok not in ("x", "*"):
                raise Q.ParseError("expected tensor operator 'x' in expression")
        else:
            gates.append(tok)
    if not gates or len(names) % 2 == 0:
        raise Q.ParseError("expression must be gate names joined by 'x'")
    acc = Q.gate_catalog_lookup(gates[0], Q.canonical_params(gates[0])).matrix
    for g in gates[1:]:
        acc = _dense_tensor(acc, Q.gate_catalog_lookup(g, Q.canonical_params(g)).matrix)
    return acc


# ---------------------------------------------------------------- rendering
def _num(x: float) -> str:
    """nlohmann::json number formatting: shortest round-trip digits, '.0' for integral values,
    exponent form outside [1e-5, 1e15]."""
    if x != x:
        return "null"
    if x in (float("inf"), float("-inf")):
        return "null"
    r = repr(float(x))
    if "e" in r or "E" in r:
        mant, exp = r.split("e")
        e = int(exp)
        return f"{mant}e{'+' if e >= 0 else '-'}{abs(e):02d}"
    return r


class _Compact(list):
    """An array rendered on one line, "[a,b,c]" (as the reference's report shows the samples)."""


def _dump(v, indent=0) -> str:
    pad = " " * indent
    if isinstance(v, _Compact):
        return "[" + ",".join(_dump(x) for x in v) + "]"
    if isinstance(v, dict):
        if not v:
            return "{}"
        items = [f'{pad}  {json.dumps(k)}: {_dump(x, indent + 2)}' for k, x in v.items()]
        return "{\n" + ",\n".join(items) + "\n" + pad + "}"
    if isinstance(v, list):
        if not v:
            return "[]"
        return "[\n" + ",\n".join(f"{pad}  {_dump(x, indent + 2)}" for x in v) + "\n" + pad + "]"
    if isinstance(v, bool):
        return "true" if v else "false"
    if isinstance(v, int):
        return str(v)
    if isinstance(v, float):
        return _num(v)
    return json.dumps(v)


def _g(x: float, prec: int) -> str:
    """std::ostream default float formatting with precision `prec` (%g)."""
    return f"{x:.{prec}g}"


@dataclass
class ReportOptions:  # circuit_io.hpp:26-31
    format: str = "human"  # human | json | csv
    samples: int = 0
    seed: int = 0
    engine: str = ""


def render_report(report: Q.SimReport, n: int, opts: ReportOptions) -> str:  # circuit_io.cpp:109-203
    dim = 1 << n
    small = dim <= (1 << 16)
    state = report.final
    probs = report.probabilities if small else None
    if probs is not None:
        argmax = int(np.argmax(probs))
        pmax = float(probs[argmax])
    else:
        argmax, pmax = state.argmax()
    if small:  # sequential norm as StateVector::norm (core.cpp:30-34)
        amps = state.download()
        norm = math.sqrt(_seq_norm2(amps))
    else:
        norm = state.norm()
    # drawn on the device against the reference's exact sequential CDF (qcs_sample): nothing of
    # size 2^n is downloaded for the samples
    samples = state.sample(opts.samples, opts.seed)[0] if opts.samples > 0 else []

    if opts.format == "json":
        j = {"qubits": n, "engine": opts.engine, "argmax": argmax, "max_probability": pmax, "norm": norm}
        if small:
            j["probabilities"] = [float(p) for p in probs]
        else:
            idx, pr = state.topk(16)
            j["top_probabilities"] = [{"index": int(i), "probability": float(p)} for i, p in zip(idx, pr)]
        j["steps"] = [{"structure": s.structure, "stage": s.stage, "matrix_bytes": s.matrix_bytes,
                       "dense_bytes": s.dense_bytes, "entry_count": s.entry_count, "sign_count": s.sign_count,
                       "madd_count": s.madd_count} for s in report.steps]
        j["total_sign_count"] = report.total_sign_count
        j["total_madd_count"] = report.total_madd_count
        if opts.samples > 0:
            j["seed"] = opts.seed
            j["samples"] = _Compact(samples)  # the reference's dump prints this array on one line
        return _dump(j) + "\n"

    if opts.format == "csv":
        out = ["step,structure,stage,matrix_bytes,dense_bytes,entry_count,sign_count,madd_count\n"]
        for i, s in enumerate(report.steps):
            out.append(f"{i},{s.structure},{s.stage},{s.matrix_bytes},{s.dense_bytes},{s.entry_count},"
                       f"{s.sign_count},{s.madd_count}\n")
        out.append(f"argmax,{argmax}\nmax_probability,{_g(pmax, 6)}\n")
        return "".join(out)

    out = [f"qubits:          {n}\n", f"engine:          {opts.engine}\n", f"argmax:          {argmax}\n",
           f"max probability: {_g(pmax, 12)}\n", f"norm:            {_g(norm, 12)}\n", "steps:\n"]
    for i, s in enumerate(report.steps):
        line = f"  [{i}] {s.structure}  bytes={s.matrix_bytes} (dense {s.dense_bytes})"
        if s.entry_count:
            line += f" entries={s.entry_count}"
        if s.sign_count:
            line += f" signs={s.sign_count}"
        out.append(line + f" madds={s.madd_count}\n")
    if opts.samples > 0:
        out.append(f"samples (seed {opts.seed}):" + "".join(f" {x}" for x in samples) + "\n")
    return "".join(out)


def _seq_norm2(amps: np.ndarray) -> float:
    acc = 0.0
    for a in amps.tolist():
        acc += a.real * a.real + a.imag * a.imag
    return acc
