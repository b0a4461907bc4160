"""A small run over every kernel family of libqcs_b200, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck, one tool per gpurun call):

    compute-sanitizer --tool memcheck python tools/sanitize_run.py

n = 14..16 so the tools finish in minutes.  Covers: the single-gate kernels (k_pair / k_diag1 /
k_quad / k_gate), the fused tile passes as interpreter (k_tile: TMA + mbarrier) and as NVRTC-
specialised kernels (qcs_pass, pivots, relabellings, skip / paired passes), diagonal sign steps,
the device DAX/DAS encoders and explicit MVMs, reductions, top-k, sampling, and the split
(peer-memory) kernel on an emulated rank pair.  Prints "sanitize run ok" at the end.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_15332_b200 import configs  # noqa: E402
from paper_2411_15332_b200 import qcsim as Q  # noqa: E402


def main():
    n = 14
    rng = np.random.default_rng(1)
    x = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    x = (x / np.linalg.norm(x)).astype(np.complex128)
    s = Q.DeviceState.from_numpy(x)
    for g in configs.c2_sweep(n, seed=configs.seed_of(2))[::5]:  # gate kernels
        s.apply_gate(g.gate, g.qubits)
    s.apply_diag(Q.DiagSign([3, 77, 1000], False))
    s.apply_diag(Q.DiagSign([0], True))
    s.apply_rh()
    s.norm()
    s.argmax()
    s.topk(16)
    s.probabilities()
    s.sample(64, 3)
    s.gather([0, 5, (1 << n) - 1])
    # fused passes: interpreter and specialised kernels, every family
    for mode in (0, 3):
        Q.set_jit_mode(mode)
        for c in (configs.c4_circuit(16, 3), configs.c5_circuit(16, 3, global_qubits=2), Q.build_grover(16, 1234, 3),
                  configs.c1_circuit()):
            Q.simulate(c, Q.Engine.rh_dax).final.norm()
    Q.set_jit_mode(1)
    # device encoders and explicit-entry MVMs
    st = Q.CircuitStep.of_gates([Q.Placement(Q.gate_catalog_lookup("Hadamard"), 2),
                                 Q.Placement(Q.gate_catalog_lookup("CNOT"), 5)])
    d = Q.step_matrix_dax(st, 12)
    a = Q.step_matrix_das(st, 12)
    v = Q.DeviceState.from_numpy(x[: 1 << 12] / np.linalg.norm(x[: 1 << 12]))
    Q.dax_mvm(d, v)
    Q.das_mvm(a, v)
    # the split kernel over a partner shard (two emulated ranks' shards on one device) and the
    # peer swap kernel, as partition.py drives them
    import ctypes as C
    from paper_2411_15332_b200 import _lib as L
    lo, hi = Q.DeviceState.from_numpy(x[: 1 << 13] * 1.0), Q.DeviceState.from_numpy(x[1 << 13:] * 1.0)
    h = np.array([[1, 1], [1, -1]], np.complex128) / np.sqrt(2.0)
    for st_, self_bit in ((lo, 0), (hi, 1)):
        peer = hi if st_ is lo else lo
        info = [C.c_int(), C.c_int(), C.c_void_p(), C.c_void_p()]
        Q._check(L.lib().qcs_state_info(peer.handle, C.byref(info[0]), C.byref(info[1]), C.byref(info[2]),
                                        C.byref(info[3])))
        st_.apply_split(info[2].value, self_bit, [], h.reshape(1, 2, 2), 0)
        st_.sync() if hasattr(st_, "sync") else None
        Q._check(L.lib().qcs_swap_peer(st_.handle, 0, info[2], 1 << 10))
    print("sanitize run ok")


if __name__ == "__main__":
    main()
