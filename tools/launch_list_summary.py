"""Summarise an ncu launch list of the C4 circuit (gpu__time_duration, dram bytes, FP64 SASS
counts per launch) into profiles/r02_ncu_launches_c4_n32.json.

    python tools/launch_list_summary.py gpurun_out/<list>.csv <n> <planner fp64/amp> [what]
"""
import csv
import json
import sys
from collections import defaultdict


def main(path, n, planner, what=""):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    d = defaultdict(dict)
    for r in rows[start + 1:]:
        k = int(r[hdr.index("ID")])
        d[k]["kernel"] = r[hdr.index("Kernel Name")]
        d[k][r[hdr.index("Metric Name")]] = float(r[hdr.index("Metric Value")].replace(",", ""))
    amps = 2 ** n
    launches = []
    for k in sorted(d):
        x = d[k]
        f = sum(x.get(m, 0.0) for m in ("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
                                       "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
                                       "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum"))
        dram = x.get("dram__bytes_read.sum", 0.0) + x.get("dram__bytes_write.sum", 0.0)
        launches.append({"id": k, "kernel": x["kernel"][:40], "ms": x["gpu__time_duration.sum"] / 1e6,
                         "dram_GB": dram / 1e9, "sweeps": dram / (32 * amps), "fp64_per_amp": f / amps})
    tp = [l for l in launches if l["kernel"] == "qcs_pass" or l["kernel"].startswith("void qcs::<unnamed>::k_tile")]
    out = {"what": what, "launches": launches, "tile_pass_total_ms": sum(l["ms"] for l in tp),
           "tile_pass_dram_GB": sum(l["dram_GB"] for l in tp), "tile_pass_sweeps": sum(l["sweeps"] for l in tp),
           "tile_pass_fp64_per_amp": sum(l["fp64_per_amp"] for l in tp), "planner_fp64_per_amp": planner}
    return out


if __name__ == "__main__":
    res = main(sys.argv[1], int(sys.argv[2]), float(sys.argv[3]), sys.argv[4] if len(sys.argv) > 4 else "")
    json.dump(res, sys.stdout, indent=1)
