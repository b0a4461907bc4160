"""Serial C4 e2e requests (fresh angles, summary read-back) with per-kernel-class device timing on:
where the ~30 ms between the device-timed circuit and the host-timed request go."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_15332_b200 import configs  # noqa: E402
from paper_2411_15332_b200 import qcsim as Q  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
circuits = [configs.c4_circuit(n, seed=177 + i) for i in range(6)]
a = Q.DeviceState(n)
Q.simulate(circuits[0], Q.Engine.rh_dax, state=a)
a.summary(16)
a.sync()
for timing in (False, True):
    a.timing(timing)
    for c in circuits[1:]:
        if timing:
            a.timing_reset()
        t0 = time.perf_counter()
        Q.simulate(c, Q.Engine.rh_dax, state=a)
        t1 = time.perf_counter()
        a.summary(16)
        t2 = time.perf_counter()
        rep = a.timing_report() if timing else {}
        dev = {k: round(v[1], 2) for k, v in rep.items()}
        print(f"timing={timing} simulate returns {1e3 * (t1 - t0):6.2f} ms, summary waits {1e3 * (t2 - t1):7.2f} ms, "
              f"request {1e3 * (t2 - t0):7.2f} ms, device classes {dev}")
a.timing(False)
