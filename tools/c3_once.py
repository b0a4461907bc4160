"""Grover (C3 shape) through simulate() once -- a short ncu target for the fused tile passes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_15332_b200 import configs  # noqa: E402
from paper_2411_15332_b200 import qcsim as Q  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
it = int(sys.argv[2]) if len(sys.argv) > 2 else 1
rep = Q.simulate(configs.c3_circuit(n, it), Q.Engine.rh_dax)
print("argmax", rep.final.argmax(), "marked", configs.c3_marked(n))
