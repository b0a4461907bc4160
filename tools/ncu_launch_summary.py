"""Summarise an ncu launch list of tools/sweep_once.py (one C2 sweep) per gate, per target bit
and per kernel class.

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file launches.csv python tools/sweep_once.py
    python tools/ncu_launch_summary.py launches.csv out.json

ncu's launches are serialised and cold-cache: compare shares and per-launch DRAM bytes, not the
absolute times, with the bench's CUDA-event numbers.
"""
import csv
import json
import os
import sys
from collections import OrderedDict, defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2411_15332_b200 import configs  # noqa: E402

GATE_KERNELS = ("k_diag1", "k_pair", "k_quad", "k_gate")


def load(path):
    rows = OrderedDict()
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        k = int(r["ID"])
        e = rows.setdefault(k, {"name": r["Kernel Name"]})
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        if r["Metric Name"] == "gpu__time_duration.sum":
            e["us"] = v * {"ns": 1e-3, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(unit, 1.0)
        else:
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1)
            e[r["Metric Name"]] = v * scale
    return list(rows.values())


def engine_class(kernel, label):
    """The engine's timing class (gate_kernels.cu launch_k names) of one launch."""
    if "k_quad" in kernel:
        return "gate_quad_monomial"
    if "k_diag1" in kernel:
        return "gate_diag1"
    if "k_pair" in kernel:
        return "gate_pair_dense" if label in ("H", "RX", "U3") else "gate_pair_monomial"
    return "gate_generic"


def main(src, dst, n=28):
    launches = [e for e in load(src) if any(k in e["name"] for k in GATE_KERNELS)]
    sweep = configs.c2_sweep(n, seed=configs.seed_of(2))
    if len(launches) != len(sweep):
        raise SystemExit(f"{len(launches)} gate launches for {len(sweep)} sweep gates")
    per_gate = defaultdict(list)
    per_bit = defaultdict(list)
    per_class = defaultdict(list)
    for g, e in zip(sweep, launches):
        name = g.label
        per_gate[name].append(e)
        per_bit[f"{name}@q{'-'.join(map(str, g.qubits))}"].append(e)
        per_class[engine_class(e["name"], name)].append(e)

    def agg(es):
        us = sum(e["us"] for e in es) / len(es)
        b = sum(e.get("dram__bytes_read.sum", 0) + e.get("dram__bytes_write.sum", 0) for e in es) / len(es)
        return {"launches": len(es), "avg_us": us, "dram_GB_per_launch": b / 1e9, "GBps": b / us / 1e3}

    total = sum(e["us"] for e in launches)
    out = {"source": f"ncu launch list of tools/sweep_once.py at n={n} ({os.path.basename(src)}); "
                     "cold-cache serialised launches: compare shares, not absolutes",
           "total_gate_kernel_ms": total / 1e3,
           "per_gate": {k: {**agg(v), "share": sum(e['us'] for e in v) / total} for k, v in per_gate.items()},
           "per_class": {k: agg(v) for k, v in per_class.items()},
           "per_target": {k: agg(v) for k, v in per_bit.items()}}
    with open(dst, "w") as f:
        json.dump(out, f, indent=1)
    # DRAM bytes per launch by class, read by bench.py for roofline.traffic
    traffic = os.path.join(os.path.dirname(dst), "ncu_traffic.json")
    with open(traffic, "w") as f:
        json.dump({k: v["dram_GB_per_launch"] * 1e9 for k, v in out["per_class"].items()}, f, indent=1)
    for k, v in out["per_gate"].items():
        print(f"{k:10s} {v['avg_us']:9.1f} us  {v['GBps']:7.0f} GB/s  share {v['share']:.3f}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 28)
