"""Time qcs_apply_rh (H on every qubit as fused butterfly passes) at n qubits, CUDA events."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2411_15332_b200 import qcsim as Q  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
reps = 5
s = Q.DeviceState(n)
s.randomize(7)
s.apply_rh()
s.sync()
s.timing(True)
s.timing_reset()
s.record(0)
for _ in range(reps):
    s.apply_rh()
s.record(1)
s.sync()
ms = s.elapsed_ms(0, 1) / reps
rep = s.timing_report()
k = rep["tile_pass"]
passes = k[0] / reps
print(f"n={n} rh {ms:.3f} ms, {passes:.0f} passes, {ms / passes:.3f} ms/pass, "
      f"{k[2] / (k[1] / 1e3) / 1e9:.0f} GB/s over tile passes, norm {s.norm():.15f}")
