"""C5-shaped random circuit through simulate() once -- an ncu target."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_15332_b200 import configs  # noqa: E402
from paper_2411_15332_b200 import qcsim as Q  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
layers = int(sys.argv[2]) if len(sys.argv) > 2 else 20
rep = Q.simulate(configs.c5_circuit(n, layers), Q.Engine.rh_dax)
print("norm", rep.final.norm())
