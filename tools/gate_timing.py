"""Per-(gate, target) device time of the single-gate kernel at n qubits (CUDA events per launch)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2411_15332_b200 import configs  # noqa: E402
from paper_2411_15332_b200 import qcsim as Q  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=28)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--targets", default="0,1,2,3,4,8,16,24,25,26,27")
a = ap.parse_args()
s = Q.DeviceState(a.n)
s.randomize(1)
s.timing(True)
want = {int(x) for x in a.targets.split(",")}
rows = []
for g in configs.c2_sweep(a.n):
    bit = a.n - 1 - g.qubits[-1]
    if bit not in want:
        continue
    s.apply_gate(g.gate, g.qubits)
    s.timing_reset()
    for _ in range(a.reps):
        s.apply_gate(g.gate, g.qubits)
    rep = s.timing_report()
    (cls, (cnt, ms, by)), = rep.items()
    rows.append({"gate": g.label, "target_bit": bit, "ctrl_bits": [a.n - 1 - q for q in g.qubits[:-1]], "cls": cls,
                 "us": round(1e3 * ms / cnt, 1), "GBps": round(by / (ms / 1e3) / 1e9, 1)})
for r in rows:
    print(json.dumps(r))
