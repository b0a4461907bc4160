"""Summarise one kernel of an `ncu --set full --import-source on` report as JSON for profiles/.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r01_ncu_xxx.json "what was profiled"

Keeps: duration, IPC, issue-slot use, occupancy, DRAM bytes and throughput, warp-stall mix, the
SASS opcode mix and the hottest source lines (instructions executed / stall samples).
"""
import csv
import io
import json
import subprocess
import sys
from collections import Counter

NCU = "ncu"


def run(args):
    return subprocess.run([NCU, *args], capture_output=True, text=True, check=True).stdout


def raw_metrics(rep):
    rows = list(csv.reader(io.StringIO(run(["-i", rep, "--page", "raw", "--csv"]))))
    head, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(head, units, vals)}


def num(x):
    try:
        return float(x.replace(",", ""))
    except (ValueError, AttributeError):
        return None


def source_view(rep):
    rows = list(csv.reader(io.StringIO(run(["-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]))))
    head = next(r for r in rows if r and r[0] == "Line No")
    ie, ss = head.index("Instructions Executed"), head.index("Warp Stall Sampling (All Samples)")
    lines, ops = [], Counter()
    for r in rows[rows.index(head) + 1:]:
        if not r:
            continue
        if r[0].isdigit():
            n, s = num(r[ie]), num(r[ss])
            if n is not None and s is not None:
                lines.append((int(n), int(s), int(r[0]), r[1].strip()[:120]))
        elif len(r) > ie:
            n = num(r[ie])
            t = r[3].strip().split()
            if n and t:
                ops[(t[1] if t[0].startswith("@") else t[0]).split(".")[0]] += n
    return lines, ops


def main(rep, out, what):
    m = raw_metrics(rep)
    pick = {
        "duration": "gpu__time_duration.sum",
        "dram_bytes_read": "dram__bytes_read.sum",
        "dram_bytes_write": "dram__bytes_write.sum",
        "dram_throughput_pct": "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "ipc_active": "sm__inst_executed.avg.per_cycle_active",
        "issue_slots_busy_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
        "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
        "registers_per_thread": "launch__registers_per_thread",
        "grid_size": "launch__grid_size",
        "block_size": "launch__block_size",
        "shared_mem_per_block": "launch__shared_mem_per_block_dynamic",
        "inst_executed": "smsp__inst_executed.sum",
        "smem_bank_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smem_wavefronts": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    }
    res = {"what": what, "kernel": m.get("Kernel Name", ("", ""))[0]}
    for k, name in pick.items():
        if name in m:
            v, u = m[name]
            res[k] = num(v)
            if u:
                res[k + "_unit"] = u
    stalls = {k.split("stalled_")[1]: num(v) for k, (v, _) in m.items()
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued")}
    tot = sum(v for v in stalls.values() if v) or 1.0
    res["stall_share"] = {k: round(v / tot, 4) for k, v in sorted(stalls.items(), key=lambda kv: -(kv[1] or 0))
                          if v and v / tot >= 0.01}
    lines, ops = source_view(rep)
    ti = sum(x[0] for x in lines) or 1
    ts = sum(x[1] for x in lines) or 1
    to = sum(ops.values()) or 1
    res["opcode_share"] = {k: round(v / to, 4) for k, v in ops.most_common(14)}
    res["top_source_lines"] = [{"line": ln, "inst_share": round(n / ti, 4), "stall_share": round(s / ts, 4),
                                "source": src} for n, s, ln, src in sorted(lines, reverse=True)[:16]]
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps({k: v for k, v in res.items() if not isinstance(v, (list, dict))}, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
