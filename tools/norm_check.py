"""C4 at n qubits simulated `reps` times on one state (reset each time): prints norm - 1 per run.
A pipelining race or a wrong sign shows as a norm defect far above rounding (1e-13)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_15332_b200 import configs  # noqa: E402
from paper_2411_15332_b200 import qcsim as Q  # noqa: E402

n, reps = int(sys.argv[1]), int(sys.argv[2])
which = sys.argv[3] if len(sys.argv) > 3 else "c4"
c = configs.c4_circuit(n) if which == "c4" else configs.c5_circuit(n, global_qubits=3)
st = Q.DeviceState(n)
out = []
for _ in range(reps):
    Q.simulate(c, Q.Engine.rh_dax, state=st)
    out.append(st.norm() - 1.0)
print(which, n, {k: os.environ.get(k) for k in ("QCS_PERSIST", "QCS_JIT_SPLIT_SIGNS", "QCS_PERSIST_SLOTS")}, ["%.2e" % x for x in out])
