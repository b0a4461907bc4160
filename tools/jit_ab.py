"""Final-state hash and time of BASELINE circuits through simulate(), for comparing the pass
kernels (QCS_JIT=0: interpreter k_tile; default / force: specialised per-pass kernels).

    QCS_JIT=0 python tools/jit_ab.py c4:24 c5:24 c3:22 c1:12
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_15332_b200 import configs  # noqa: E402
from paper_2411_15332_b200 import qcsim as Q  # noqa: E402

build = {"c1": lambda n: configs.c1_circuit(n), "c3": lambda n: configs.c3_circuit(n),
         "c4": lambda n: configs.c4_circuit(n), "c5": lambda n: configs.c5_circuit(n),
         "c4l2": lambda n: configs.c4_circuit(n, 2)}
reps = int(os.environ.get("REPS", "3"))


def digest(st):
    """sha256 of the whole state up to 2^24 amplitudes, else of 2^20 strided amplitudes."""
    if st.n <= 24:
        return hashlib.sha256(st.download().tobytes()).hexdigest()[:16]
    stride = 1 << (st.n - 20)
    idx = np.arange(0, 1 << st.n, stride, dtype=np.uint64) + np.uint64(12345 % stride)
    return hashlib.sha256(st.gather(idx).tobytes()).hexdigest()[:16]
for arg in sys.argv[1:]:
    key, n = arg.split(":")
    c = build[key](int(n))
    st = Q.DeviceState(c.n)
    t0 = time.perf_counter()
    Q.simulate(c, Q.Engine.rh_dax, state=st)  # warm-up (compiles pass kernels)
    st.sync()
    first = time.perf_counter() - t0
    h = digest(st)
    times = []
    for _ in range(reps):
        st.set_basis(0)
        st.record(0)
        Q.simulate(c, Q.Engine.rh_dax, state=st)
        st.record(1)
        st.sync()
        times.append(st.elapsed_ms(0, 1))
    h2 = digest(st)
    print(json.dumps({"config": arg, "jit": os.environ.get("QCS_JIT", "default"), "sha": h, "repeat_sha_same": h == h2,
                      "first_s": round(first, 2), "ms": round(sorted(times)[len(times) // 2], 3),
                      "norm": st.norm()}), flush=True)
    st.close()
