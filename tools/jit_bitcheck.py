"""C4 family at n qubits, L layers: interpreter (jit mode 0) vs specialised pass kernels (modes 1, 2),
compared bit for bit.  usage: python tools/jit_bitcheck.py 30 10"""
import sys, numpy as np
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_15332_b200 import configs, qcsim as Q
n = int(sys.argv[1]); L = int(sys.argv[2])
c = configs.c4_circuit(n, L)
res = {}
for m in (0, 1, 2):
    Q.set_jit_mode(m)
    res[m] = Q.simulate(c, Q.Engine.rh_dax).final.download()
for m in (1, 2):
    d = res[m].view(np.uint64) != res[0].view(np.uint64)
    print(n, L, 'mode', m, 'bits differ:', int(d.sum()), 'maxabs', float(np.abs(res[m]-res[0]).max()))
