"""The reference CLI's ``bench`` suites (tools/qcsim_cli.cpp:84-239) on the B200 engine.

``qcsim bench <suite> --sizes ... --engines ...`` prints one row per (size, engine):
suite, n, engine, seconds, memory_bytes, sign_count, multiply_count, status, note.  The suites:

* ``mtp``      (qcsim_cli.cpp:120-142) X on every qubit, the step's structure materialised:
  DAX / DAS by the device encoder (qcs_step_dax / das, device output), dense by the Matrix
  method's device build (timed with its MVM: the device has no separate dense-build entry);
* ``mvm``      (:144-176) the same step through the structure's MVM (device dax_mvm / das_mvm on
  the encoded entries, the dense engine's build + dense_mvm), multiply_count = entries (dense:
  rows * cols);
* ``rh-signs`` (:178-202) rh_mvm with each sign method (qcs_rh_mvm: the device runs the same
  butterflies for every method; the counters are the reference's, checked against the Table-2
  formulas exactly as the reference asserts them -> status "counter-mismatch" otherwise);
* ``grover``   (:204-220) build_grover(n, 2^n / 3) through simulate, argmax asserted;
* ``qnn``      (:222-239) build_qnn_neuron with seeded angles / weights through simulate.

A CapacityError becomes a row with status "capacity-error" (:371-376).  Seconds are host wall
clock around synchronous device work, as the reference times its CPU work.
"""
from __future__ import annotations

import json
import math
import time
from dataclasses import dataclass, field
from typing import List

from . import qcsim as Q


@dataclass
class BenchRow:  # qcsim_cli.cpp:72-82
    suite: str
    n: int
    engine: str
    seconds: float = 0.0
    memory_bytes: int = 0
    sign_count: int = 0
    multiply_count: int = 0
    status: str = "ok"
    note: str = ""
    extra: dict = field(default_factory=dict)


def table2_count(method: int, n: int, b: int) -> int:  # qcsim_cli.cpp:109-118
    half = 1 << (n - 1)
    if method == Q.SignMethod.nonopt:
        return (half * 2) * (half * 2)
    if method == Q.SignMethod.quarter:
        return half * half
    if method == Q.SignMethod.block:
        return half * (half // b + b - 1)
    return half * (n - 1)


def optimal_block_size(n: int) -> int:  # rh.cpp:68-75
    half = 1 << (n - 1)
    best, b = 1, 1
    while b <= half:
        if half // b + b - 1 < half // best + best - 1:
            best = b
        b <<= 1
    return best


def _x_all(n: int) -> Q.CircuitStep:
    x = Q.gate_catalog_lookup("Pauli-X")
    return Q.CircuitStep.of_gates([Q.Placement(x, q) for q in range(n)])


def _sync_time(fn):
    t0 = time.perf_counter()
    out = fn()
    return time.perf_counter() - t0, out


def bench_mtp(n: int, engine: Q.Engine) -> BenchRow:
    row = BenchRow("mtp", n, Q.engine_name(engine))
    step = _x_all(n)
    if engine == Q.Engine.dense:
        dim = 1 << n
        if dim > Q.dense_cap() // dim:
            raise Q.CapacityError(f"dense tensor product exceeds dense cap of {Q.dense_cap()} elements")
        s = Q.DeviceState(n)
        row.seconds, _ = _sync_time(lambda: (Q.simulate(Q.Circuit(n, [step]), engine, state=s), s.sync()))
        row.memory_bytes = dim * dim * 16
        row.note = "device build timed with its dense_mvm"
        s.close()
        return row
    enc = Q.step_matrix_das_device if engine == Q.Engine.das else Q.step_matrix_dax_device
    row.seconds, m = _sync_time(lambda: enc(step, n))
    row.memory_bytes = 24 * m.count
    m.close()
    return row


def bench_mvm(n: int, engine: Q.Engine, seed: int) -> BenchRow:
    row = BenchRow("mvm", n, Q.engine_name(engine))
    step = _x_all(n)
    s = Q.DeviceState(n)
    s.randomize(seed)
    if engine == Q.Engine.dense:
        dim = 1 << n
        if dim > Q.dense_cap() // dim:
            raise Q.CapacityError(f"dense tensor product exceeds dense cap of {Q.dense_cap()} elements")
        Q.run(Q.Circuit(n, [step]), s, engine)  # warm (allocations)
        s.sync()
        row.seconds, _ = _sync_time(lambda: (Q.run(Q.Circuit(n, [step]), s, engine), s.sync()))
        row.memory_bytes = dim * dim * 16
        row.multiply_count = dim * dim
        row.note = "device build + dense_mvm"
    else:
        enc = Q.step_matrix_das_device if engine == Q.Engine.das else Q.step_matrix_dax_device
        m = enc(step, n)
        row.memory_bytes = 24 * m.count
        out = Q.DeviceState(n)
        m.mvm(s, out)  # warm
        out.sync()
        row.seconds, _ = _sync_time(lambda: (m.mvm(s, out), out.sync()))
        row.multiply_count = m.count
        out.close()
        m.close()
    s.close()
    return row


def bench_rh_signs(n: int, seed: int) -> List[BenchRow]:
    rows = []
    s = Q.DeviceState(n)
    s.randomize(seed)
    value = 2.0 ** (-0.5 * n)  # rh_build (rh.cpp:20)
    for method in (Q.SignMethod.nonopt, Q.SignMethod.quarter, Q.SignMethod.block, Q.SignMethod.logarithm):
        row = BenchRow("rh-signs", n, "rh:" + method.name)
        b = optimal_block_size(n) if method == Q.SignMethod.block and n >= 2 else 1
        s.rh_mvm(value, method, b if method == Q.SignMethod.block else 0)  # warm
        s.sync()
        row.seconds, stats = _sync_time(lambda: (s.rh_mvm(value, method, b if method == Q.SignMethod.block else 0),
                                                 s.sync())[0])
        row.memory_bytes = 16
        row.sign_count, row.multiply_count = stats
        expected = table2_count(method, n, b)
        if row.sign_count != expected:
            row.status = "counter-mismatch"
            row.note = f"expected {expected}"
        rows.append(row)
    s.close()
    return rows


def bench_grover(n: int, engine: Q.Engine) -> BenchRow:
    row = BenchRow("grover", n, Q.engine_name(engine))
    marked = (1 << n) // 3
    c = Q.build_grover(n, marked)
    row.seconds, rep = _sync_time(lambda: _sim_sync(c, engine))
    row.memory_bytes = max(s.matrix_bytes for s in rep.steps)
    row.sign_count = rep.total_sign_count
    row.multiply_count = rep.total_madd_count
    argmax = rep.final.argmax()[0]
    row.note = f"argmax={argmax}"
    if argmax != marked:
        row.status = "argmax-mismatch"
    rep.final.close()
    return row


class _MT19937_64:
    """std::mt19937_64, for the qnn suite's seeded angles and weights (qcsim_cli.cpp:223-229)."""

    def __init__(self, seed: int):
        self.mt = [seed & 0xFFFFFFFFFFFFFFFF]
        for i in range(1, 312):
            p = self.mt[-1]
            self.mt.append((6364136223846793005 * (p ^ (p >> 62)) + i) & 0xFFFFFFFFFFFFFFFF)
        self.i = 312

    def __call__(self) -> int:
        if self.i >= 312:
            mt = self.mt
            for k in range(312):
                y = (mt[k] & 0xFFFFFFFF80000000) | (mt[(k + 1) % 312] & 0x7FFFFFFF)
                mt[k] = mt[(k + 156) % 312] ^ (y >> 1) ^ (0xB5026F5AA96619E9 if y & 1 else 0)
            self.i = 0
        y = self.mt[self.i]
        self.i += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        return (y ^ (y >> 43)) & 0xFFFFFFFFFFFFFFFF


def bench_qnn(inputs: int, engine: Q.Engine, seed: int) -> BenchRow:
    rng = _MT19937_64(seed)
    angles, weights = [], []
    for _ in range(inputs):  # qcsim_cli.cpp:223-229: uniform_real_distribution(0, 3), rng() & 1
        c = rng() / 18446744073709551616.0
        angles.append((3.0 - 0.0) * (c if c < 1.0 else math.nextafter(1.0, 0.0)) + 0.0)
        weights.append(1 if (rng() & 1) else -1)
    c = Q.build_qnn_neuron(inputs, angles, weights)
    row = BenchRow("qnn", c.n, Q.engine_name(engine))
    row.seconds, rep = _sync_time(lambda: _sim_sync(c, engine))
    row.memory_bytes = max(s.matrix_bytes for s in rep.steps)
    row.sign_count = rep.total_sign_count
    row.multiply_count = rep.total_madd_count
    row.note = f"inputs={inputs}"
    rep.final.close()
    return row


def _sim_sync(c, engine):
    rep = Q.simulate(c, engine)
    rep.final.sync()
    return rep


def run_suite(suite: str, sizes: List[int], engines: List[Q.Engine], seed: int = 0) -> List[BenchRow]:
    """qcsim_cli.cpp:344-379."""
    rows: List[BenchRow] = []
    for n in sizes:
        if suite == "rh-signs":
            rows += bench_rh_signs(n, seed)
            continue
        for e in engines:
            try:
                if suite == "mtp":
                    rows.append(bench_mtp(n, e))
                elif suite == "mvm":
                    rows.append(bench_mvm(n, e, seed))
                elif suite == "grover":
                    rows.append(bench_grover(n, e))
                elif suite == "qnn":
                    rows.append(bench_qnn(n, e, seed))
                else:
                    raise Q.ParseError("unknown bench suite: " + suite)
            except Q.CapacityError as err:
                rows.append(BenchRow(suite, n, Q.engine_name(e), status="capacity-error", note=str(err)))
    return rows


def render_bench(rows: List[BenchRow], fmt: str = "csv") -> str:  # qcsim_cli.cpp:84-107
    if fmt == "json":
        return json.dumps([{"suite": r.suite, "n": r.n, "engine": r.engine, "seconds": r.seconds,
                            "memory_bytes": r.memory_bytes, "sign_count": r.sign_count,
                            "multiply_count": r.multiply_count, "status": r.status, "note": r.note}
                           for r in rows], indent=2) + "\n"
    out = ["suite,n,engine,seconds,memory_bytes,sign_count,multiply_count,status,note\n"]
    for r in rows:
        out.append(f"{r.suite},{r.n},{r.engine},{r.seconds:.9g},{r.memory_bytes},{r.sign_count},"
                   f"{r.multiply_count},{r.status},{r.note}\n")
    return "".join(out)


def rh_signs(args) -> int:
    """bench.py --workload rh-signs: the rh-signs suite at n = 4..28 (or --n-circuit), rows on
    stderr in the reference's CSV, and one JSON line: H^n applications as n gate-equivalents each
     per second over the timed rh_mvm calls."""
    import sys
    sizes = [args.n_circuit] if args.n_circuit else [4, 8, 12, 16, 20, 24, 28]
    rows = run_suite("rh-signs", sizes, [], seed=0)
    sys.stderr.write(render_bench(rows))
    secs = sum(r.seconds for r in rows)
    updates = sum(r.n * (1 << r.n) for r in rows)
    line = {"metric": "amplitude-updates/sec per circuit and % of HBM roofline at n qubits, 1/2/4/8 B200",
            "value": updates / secs, "unit": "amplitude-updates/s", "n_gpus": 1, "steps": len(rows),
            "warmup": 1, "ms_per_step": 1e3 * secs / len(rows), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "c128", "data": "synthetic",
            "config": {"workload": "rh-signs suite (qcsim_cli.cpp:178-202)", "sizes": sizes},
            "rows": [r.__dict__ for r in rows],
            "counters_ok": all(r.status == "ok" for r in rows)}
    line["rows"] = [{k: v for k, v in d.items() if k != "extra"} for d in line["rows"]]
    print(json.dumps(line), flush=True)
    return 0 if line["counters_ok"] else 1


__all__ = ["BenchRow", "run_suite", "render_bench", "rh_signs", "table2_count", "optimal_block_size"]
