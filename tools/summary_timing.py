"""Time the read-back reductions on a random state of n qubits: norm, argmax, top-16 + norm (summary)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_15332_b200 import qcsim as Q  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
st = Q.DeviceState(n)
st.randomize(7)
st.sync()
for name, fn in (("norm", st.norm), ("argmax", st.argmax), ("summary(16)", lambda: st.summary(16)), ("topk(16)", lambda: st.topk(16)),
                 ("sample(16)", lambda: st.sample(16, 5)), ("sample(4096)", lambda: st.sample(4096, 5))):
    fn()
    t0 = time.perf_counter()
    for _ in range(3):
        fn()
    dt = (time.perf_counter() - t0) / 3
    print(f"{name:12s} {1e3 * dt:8.2f} ms  {16.0 * (1 << n) / dt / 1e9:8.1f} GB/s")
