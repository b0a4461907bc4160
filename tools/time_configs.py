"""Time the BASELINE circuits C1 / C3 / C4 through qcsim.simulate (device state, CUDA events)."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2411_15332_b200 import configs  # noqa: E402
from paper_2411_15332_b200 import qcsim as Q  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--which", default="c1,c3,c4")
ap.add_argument("--n3", type=int, default=30)
ap.add_argument("--n4", type=int, default=32)
ap.add_argument("--n5", type=int, default=32)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--fuse", type=int, default=1)
a = ap.parse_args()

jobs = {"c1": (lambda: configs.c1_circuit(), configs.c1_updates()),
        "c3": (lambda: configs.c3_circuit(a.n3), configs.c3_updates(a.n3)),
        "c4": (lambda: configs.c4_circuit(a.n4), configs.c4_updates(a.n4)),
        "c5": (lambda: configs.c5_circuit(a.n5), configs.c5_updates(a.n5))}
for key in a.which.split(","):
    build, updates = jobs[key]
    c = build()
    st = Q.DeviceState(c.n)
    opts = Q.SimOptions(fuse=bool(a.fuse))
    Q.simulate(c, Q.Engine.rh_dax, opts, state=st)  # warm-up
    st.sync()
    st.timing(True)
    st.timing_reset()
    times = []
    for _ in range(a.reps):
        st.record(0)
        t0 = time.perf_counter()
        Q.simulate(c, Q.Engine.rh_dax, opts, state=st)
        st.record(1)
        st.sync()
        times.append(st.elapsed_ms(0, 1))
        host = time.perf_counter() - t0
    rep = st.timing_report()
    st.timing(False)
    ms = float(np.median(times))
    out = {"config": key, "n": c.n, "ms": ms, "updates_per_s": updates / (ms / 1e3), "host_s_last": host,
           "kernels": {k: {"launches": v[0] / a.reps, "ms": v[1] / a.reps, "GBps": v[2] / (v[1] / 1e3) / 1e9}
                       for k, v in rep.items()}}
    if key == "c3":
        marked = configs.c3_marked(a.n3)
        am, ao = configs.grover_closed_form(a.n3, 8)
        got = st.gather([marked, 0, 1])
        out["err_vs_closed_form"] = float(max(abs(got[0] - am), abs(got[1] - ao), abs(got[2] - ao)))
    out["norm"] = st.norm()
    print(json.dumps(out), flush=True)
    st.close()
