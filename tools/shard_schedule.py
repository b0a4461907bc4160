"""Host-only: how the sharded scheduler cuts a circuit at P ranks -- the remaps (exchanged shard
fractions) and, per local batch between them, the passes the fused planner needs (no tensors)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from paper_2411_15332_b200 import configs  # noqa: E402
from paper_2411_15332_b200 import qcsim as Q  # noqa: E402
from paper_2411_15332_b200.partition import ShardedState, circuit_ops  # noqa: E402


class PlanBackend:
    def __init__(self, n_local):
        self.n = n_local
        self.batches = []

    def set_basis(self, index):
        pass

    def run(self, ops):
        self.batches.append(list(ops))

    def sync(self):
        pass


class CountTransport:
    def swap_blocks(self, backend, k, pairs, chunk):
        pass


def batch_circuit(n, ops):
    steps, hs = [], []

    def flush_h():
        if len(hs) == n and len(set(hs)) == n:
            steps.append(Q.hadamard_all(n))
        else:
            h = Q.gate_catalog_lookup("Hadamard")
            steps.extend(Q.CircuitStep.of_gates([Q.Placement(h, qubits=[q])]) for q in hs)
        hs.clear()
    for op in ops:
        if op[0] == "gate" and op[3] == "Hadamard" and len(op[2]) == 1 and op[2][0] not in hs:
            hs.append(op[2][0])
            continue
        if hs:
            flush_h()
        if op[0] == "gate":
            steps.append(Q.CircuitStep.of_gates([Q.Placement(Q.custom_gate(op[1], op[3]), qubits=list(op[2]))]))
        elif op[0] == "diag":
            steps.append(Q.CircuitStep.of_diag(Q.DiagSign(list(op[1]), op[2])))
        else:
            steps.append(Q.hadamard_all(n))
    if hs:
        flush_h()
    return Q.Circuit(n, steps)


def main():
    w = sys.argv[1] if len(sys.argv) > 1 else "c4"
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 32
    for world in (1, 2, 4, 8):
        g = world.bit_length() - 1
        c = {"c4": lambda: configs.c4_circuit(n), "c5": lambda: configs.c5_circuit(n, global_qubits=max(g, 1)),
             "c3": lambda: configs.c3_circuit(n)}[w]()
        be = PlanBackend(n - g)
        sh = ShardedState(n, world, 0, be, CountTransport() if world > 1 else None, initial=c.initial)
        sh.run(circuit_ops(c))
        sh.flush()
        st = sh.exchange_stats()
        shard = 16 << (n - g)
        passes = []
        for ops in be.batches:
            ps = Q.plan_stats(batch_circuit(n - g, ops))
            passes.append((len(ops), ps["passes"], ps["sweep_amps"] / float(1 << (n - g))))
        print(f"{w} n={n} P={world}: remaps {st['remaps']}, shards sent {st['bytes_sent'] / shard:.3f}, "
              f"batches (ops, passes, sweeps): {passes}, total passes {sum(p[1] for p in passes)}")


main()
