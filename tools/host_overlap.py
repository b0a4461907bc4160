"""Host time per simulate() call and whether it overlaps the device: C3/C4 through simulate() K
times back to back (events on the state's stream) with and without per-launch timing."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_15332_b200 import configs  # noqa: E402
from paper_2411_15332_b200 import qcsim as Q  # noqa: E402

for name, c in [("c3", configs.c3_circuit(30)), ("c1", configs.c1_circuit())]:
    st = Q.DeviceState(c.n)
    for _ in range(3):
        Q.simulate(c, Q.Engine.rh_dax, state=st)
    st.sync()
    for timing in (False, True):
        st.timing(timing)
        st.record(0)
        host = []
        for _ in range(5):
            t0 = time.perf_counter()
            Q.simulate(c, Q.Engine.rh_dax, state=st)
            host.append(1e3 * (time.perf_counter() - t0))
        st.record(1)
        st.sync()
        print(name, "timing" if timing else "plain", "device ms/step", round(st.elapsed_ms(0, 1) / 5, 3),
              "host ms/call", [round(h, 2) for h in host])
        st.timing(False)
    st.close()
