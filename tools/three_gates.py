"""Z(16), CNOT(13 -> 16), X(16) once each on a 28-qubit random state -- a short ncu target."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_15332_b200 import qcsim as Q  # noqa: E402

n = 28
s = Q.DeviceState(n)
s.randomize(1)
q = lambda bit: n - 1 - bit
for name, bits in (("Pauli-Z", [16]), ("Controlled-X", [13, 16]), ("Pauli-X", [16]), ("Pauli-Z", [0])):
    s.apply_gate(Q.gate_catalog_lookup(name), [q(b) for b in bits])
s.sync()
print("ok", s.norm())
