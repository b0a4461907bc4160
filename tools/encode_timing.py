"""Time the device DAX / DAS encoders (qcs_step_dax / qcs_step_das, output in device memory) and
the explicit-entry MVMs (qcs_dax_mvm / qcs_das_mvm) on one placement at n qubits.

    python tools/encode_timing.py [n]

Host wall-clock around synchronous calls (each call finishes its device work before it
returns), best of 3; bytes are the entries written (24 B accounted, 32 B stored) or read.
"""
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2411_15332_b200 import qcsim as Q  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 26
lib = Q.L.lib()
out = {"n": n}
for name, qubits in (("Hadamard", [3]), ("Controlled-X", [2, 9]), ("Swap", [0, n - 1])):
    g = Q.gate_catalog_lookup(name)
    arr, keep = Q._placements([Q.Placement(g, qubits=qubits)])
    cnt = C.c_uint64()
    Q._check(lib.qcs_step_dax(n, arr, 1, 0, None, None, None, 0, Q.L.QCS_MEM_DEVICE, C.byref(cnt)))
    e = cnt.value
    rows = torch.empty(e, dtype=torch.int64, device="cuda")
    cols = torch.empty(e, dtype=torch.int64, device="cuda")
    vals = torch.empty(2 * e, dtype=torch.float64, device="cuda")
    dis = torch.empty(e, dtype=torch.int64, device="cuda")
    last = torch.empty(e, dtype=torch.uint8, device="cuda")

    def best(f):
        ts = []
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            f()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        return min(ts)

    p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    t_dax = best(lambda: Q._check(lib.qcs_step_dax(n, arr, 1, 0, p(rows), p(cols), p(vals), e, Q.L.QCS_MEM_DEVICE,
                                                   C.byref(cnt))))
    t_das = best(lambda: Q._check(lib.qcs_step_das(n, arr, 1, 0, p(dis), p(last), p(vals), e, Q.L.QCS_MEM_DEVICE,
                                                   C.byref(cnt))))
    s_in = Q.DeviceState(n)
    s_in.randomize(5)
    s_out = Q.DeviceState(n)
    Q._check(lib.qcs_step_dax(n, arr, 1, 0, p(rows), p(cols), p(vals), e, Q.L.QCS_MEM_DEVICE, C.byref(cnt)))
    t_dmvm = best(lambda: Q._check(lib.qcs_dax_mvm(p(rows), p(cols), p(vals), e, Q.L.QCS_MEM_DEVICE, s_in.handle,
                                                   s_out.handle)))
    Q._check(lib.qcs_step_das(n, arr, 1, 0, p(dis), p(last), p(vals), e, Q.L.QCS_MEM_DEVICE, C.byref(cnt)))
    t_smvm = best(lambda: Q._check(lib.qcs_das_mvm(p(dis), p(last), p(vals), e, Q.L.QCS_MEM_DEVICE, s_in.handle,
                                                   s_out.handle)))
    out[name] = {"entries": e, "dax_encode_ms": 1e3 * t_dax, "das_encode_ms": 1e3 * t_das,
                 "dax_encode_GBps_written": 32 * e / t_dax / 1e9, "das_encode_GBps_written": 25 * e / t_das / 1e9,
                 "dax_mvm_ms": 1e3 * t_dmvm, "das_mvm_ms": 1e3 * t_smvm,
                 "dax_mvm_Gentries_per_s": e / t_dmvm / 1e9, "das_mvm_Gentries_per_s": e / t_smvm / 1e9}
    s_in.close()
    s_out.close()
    del rows, cols, vals, dis, last
    torch.cuda.empty_cache()
print(json.dumps(out, indent=1))
