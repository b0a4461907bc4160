"""A circuit with and without the persistent pipelined pass kernels (two processes' worth of
settings are process-wide, so this runs ONE setting; compare the printed checksums)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from paper_2411_15332_b200 import configs  # noqa: E402
from paper_2411_15332_b200 import qcsim as Q  # noqa: E402

which, n = sys.argv[1], int(sys.argv[2])
c = {"c3": lambda: configs.c3_circuit(n), "c4": lambda: configs.c4_circuit(n, 10),
     "c5": lambda: configs.c5_circuit(n, 20, global_qubits=2)}[which]()
rep = Q.simulate(c, Q.Engine.rh_dax)
idx = np.array([0, 1, 5, (1 << n) - 1, (1 << n) // 3, 12345], dtype=np.uint64)
print(which, n, os.environ.get("QCS_PERSIST"), "norm %.15f" % rep.final.norm(), rep.final.gather(idx))
