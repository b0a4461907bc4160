"""One C2 sweep (12 gates x n targets) on a random n-qubit state -- a short command for ncu."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2411_15332_b200 import configs  # noqa: E402
from paper_2411_15332_b200 import qcsim as Q  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=28)
ap.add_argument("--rh", action="store_true", help="also apply H^n (RH) once")
a = ap.parse_args()
s = Q.DeviceState(a.n)
s.randomize(configs.seed_of(2))
for g in configs.c2_sweep(a.n, seed=configs.seed_of(2)):
    s.apply_gate(g.gate, g.qubits)
if a.rh:
    s.apply_rh()
s.sync()
print("norm", s.norm())
