"""Where the host waits in the C4 e2e loop: per request, the time Q.simulate takes to return
(host planning + launches) and the time the read-back then waits, serial and pipelined."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_15332_b200 import configs  # noqa: E402
from paper_2411_15332_b200 import qcsim as Q  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
circuits = [configs.c4_circuit(n, seed=77 + i) for i in range(6)]
a, b = Q.DeviceState(n), Q.DeviceState(n)
for s in (a, b):
    Q.simulate(circuits[0], Q.Engine.rh_dax, state=s)
    s.summary(16)
print("serial")
for c in circuits:
    t0 = time.perf_counter()
    Q.simulate(c, Q.Engine.rh_dax, state=a)
    t1 = time.perf_counter()
    a.summary(16)
    t2 = time.perf_counter()
    print(f"  simulate returns {1e3 * (t1 - t0):7.2f} ms, summary waits {1e3 * (t2 - t1):7.2f} ms")
print("pipelined")
prev = None
pair = [a, b]
for i, c in enumerate(circuits):
    st = pair[i % 2]
    t0 = time.perf_counter()
    if prev is not None:
        prev.summary_begin(16)
        st.wait_for(prev)
    t1 = time.perf_counter()
    Q.simulate(c, Q.Engine.rh_dax, state=st)
    t2 = time.perf_counter()
    if prev is not None:
        prev.summary_end()
    t3 = time.perf_counter()
    print(f"  begin+wait {1e3 * (t1 - t0):6.2f} ms, simulate returns {1e3 * (t2 - t1):7.2f} ms, end waits {1e3 * (t3 - t2):7.2f} ms")
    prev = st
