#!/usr/bin/env python
"""Benchmark: amplitude-updates/s of the single-gate sweep (BASELINE.json configs[1], "C2").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--n 28]

One step = the whole C2 sweep: X, Y, Z, S, T, CNOT, CZ, SWAP, Toffoli, H, RX(theta),
U3(theta, phi, lambda) with the target swept over all n qubits (controls at seeded distinct
qubits) -- 12 * n single-gate steps applied in place to an n-qubit complex128 random state
resident in HBM.  amplitude-updates per step = 12 * n * 2^n.

Prints ONE JSON line (rank 0).  Timing: CUDA events on the state's stream, warm-up first,
barrier + synchronize on both sides, max over ranks.  The 4 GiB state is 32x the 126 MB L2,
so no L2 flush is needed between iterations.  N > 1 runs N independent replicas (one per GPU,
weak scaling); the sharded multi-GPU path is not this benchmark's workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "amplitude-updates/sec per circuit and % of HBM roofline at n qubits, 1/2/4/8 B200"
UNIT = "amplitude-updates/s"


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


class Dist:
    """torch.distributed plumbing for N > 1 (barrier + max over ranks); inert at N = 1."""

    def __init__(self, world, local_rank, backend="nccl"):
        self.world = world
        self.pg = None
        if world > 1:
            import torch
            import torch.distributed as dist
            torch.cuda.set_device(local_rank)
            dist.init_process_group(backend, device_id=torch.device("cuda", local_rank)
                                    if backend == "nccl" else None)
            self.dist = dist
            self.torch = torch

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def max(self, v: float) -> float:
        if self.world == 1:
            return v
        t = self.torch.tensor([v], dtype=self.torch.float64, device="cuda")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                if out.returncode == 0 and out.stdout.strip():
                    self.samples.append([x.strip() for x in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        smax = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 4 + i and s[4 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": reasons, "samples": len(self.samples)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic(kernel_class: str):
    """DRAM bytes per launch of the dominant kernel class from the committed ncu summary."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f)
        return d.get(kernel_class)
    except Exception:
        return None


# ------------------------------------------------------------------ CPU baselines (rank 0, N = 1)
def cpu_sample_pairs(n_sample: int, count: int):
    from paper_2411_15332_b200 import configs
    sweep = configs.c2_sweep(n_sample, seed=configs.seed_of(2))
    step = max(1, len(sweep) // count)
    return [sweep[i] for i in range(0, len(sweep), step)][:count]


def reference_sample(n_sample: int, pairs, threads: int):
    """Time the reference's own pipeline (step_matrix_dax + dax_mvm, engine.cpp:192-199) on the
    sampled (gate, target) runs; `threads` runs execute concurrently (the library is reentrant,
    ctypes releases the GIL).  Returns (updates/s, seconds, kind)."""
    from oracle.oracle_py import Oracle, Reference
    use_ref = Reference.available()
    rng = np.random.default_rng(0)
    x = (rng.standard_normal(1 << n_sample) + 1j * rng.standard_normal(1 << n_sample))
    x = (x / np.linalg.norm(x)).astype(np.complex128)
    work = list(pairs)
    lock = threading.Lock()

    def worker():
        while True:
            with lock:
                if not work:
                    return
                g = work.pop()
            if use_ref:
                Reference.apply_step(n_sample, [(g.qubits, g.gate.matrix)], x)
            else:
                Oracle.apply_step(n_sample, [(g.qubits, g.gate.matrix)], x)

    t0 = time.perf_counter()
    ths = [threading.Thread(target=worker) for _ in range(max(1, threads))]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    secs = time.perf_counter() - t0
    return len(pairs) * (1 << n_sample) / secs, secs, ("reference" if use_ref else "port")


def host_threads():
    n = os.cpu_count() or 1
    try:
        avail = os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
    except Exception:
        avail = 64 << 30
    return max(1, min(n, int(avail // (3 << 30)), 64))


# ------------------------------------------------------------------ arms
def run_reference_arm(args, rank, world):
    if rank != 0:
        return 0
    n_sample = min(args.n, 24)
    threads = host_threads()
    pairs_per_step = max(threads, 4)
    for _ in range(args.warmup):
        reference_sample(n_sample, cpu_sample_pairs(n_sample, pairs_per_step), threads)
    total_updates = 0
    total_secs = 0.0
    kind = "reference"
    for _ in range(args.steps):
        pairs = cpu_sample_pairs(n_sample, pairs_per_step)
        v, secs, kind = reference_sample(n_sample, pairs, threads)
        total_updates += len(pairs) << n_sample
        total_secs += secs
    value = total_updates / total_secs
    sample = (f"{pairs_per_step} single-gate runs per step from the C2 sweep at n={n_sample} "
              f"(reference step_matrix_dax + dax_mvm per gate, {threads} concurrent host threads)")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total_secs / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
            "config": {"workload": f"C2 single-gate sweep (sampled at n={n_sample})", "n_qubits": args.n,
                       "gates": "X,Y,Z,S,T,CNOT,CZ,SWAP,Toffoli,H,RX,U3", "parallelism": "host threads"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind, "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_b200_arm(args, rank, world, local_rank):
    from paper_2411_15332_b200 import _lib, configs
    from paper_2411_15332_b200 import qcsim as Q
    import ctypes as C

    dist = Dist(world, local_rank)
    n = args.n
    dev = local_rank if world > 1 else 0
    lib = _lib.lib()
    sweep = configs.c2_sweep(n, seed=configs.seed_of(2))
    placements = [Q._placements([Q.Placement(g.gate, qubits=g.qubits)]) for g in sweep]
    updates_per_step = len(sweep) << n
    state = Q.DeviceState(n, 0, dev)
    state.randomize(configs.seed_of(2))
    h = state.handle

    def step():
        for arr, _keep in placements:
            rc = lib.qcs_apply_step(h, arr, 1)
            if rc:
                Q._check(rc)

    for _ in range(args.warmup):
        step()
    state.sync()
    dist.barrier()
    launches0 = lib.qcs_kernel_launches()
    state.timing(True)
    state.timing_reset()
    with ClockSampler(dev) as clocks:
        state.sync()
        dist.barrier()
        state.record(0)
        for _ in range(args.steps):
            step()
        state.record(1)
        state.sync()
        ms = state.elapsed_ms(0, 1)
    dist.barrier()
    launches = lib.qcs_kernel_launches() - launches0
    timing = state.timing_report()
    state.timing(False)
    ms_max = dist.max(ms)
    value = world * updates_per_step * args.steps / (ms_max / 1e3)

    # roofline of the dominant kernel class (largest share of device time)
    dom = max(timing.items(), key=lambda kv: kv[1][1])
    dom_launches, dom_ms, dom_bytes = dom[1]
    peak, peak_kind = measured_peaks()
    achieved = (dom_bytes / dom_launches) / (dom_ms / dom_launches / 1e3) / 1e9
    traffic = ncu_traffic(dom[0])
    total_kernel_ms = sum(v[1] for v in timing.values())
    all_bytes = sum(v[2] for v in timing.values())

    # e2e: the public C ABI with host buffers.  Every step (one request) uploads its input
    # state from pinned memory, runs the sweep and reads the result back into pinned memory.
    # Two requests are in flight on two states (two streams), so one request's PCIe copies
    # overlap the other's sweep -- the way a serving loop uses the API (the reference arm
    # likewise runs concurrent requests on all host threads).  Each sweep waits for the
    # previous request's sweep (qcs_state_wait) before its result's read-back is enqueued, so
    # the sweeps run back to back instead of sharing the GPU and then leaving it idle while
    # both streams copy.  The serial form (one state, copies not overlapped) is reported
    # alongside.
    e2e_steps = max(2, args.steps)
    nbytes = 16 << n
    bufs = []
    for _ in range(3):  # input (read by both uploads), one output per state
        hp = C.c_void_p()
        Q._check(lib.qcs_host_alloc(nbytes, C.byref(hp)))
        bufs.append(hp)
    state2 = Q.DeviceState(n, 0, dev)
    states = [state, state2]
    try:
        hin, hout = bufs[0], bufs[1:]
        Q._check(lib.qcs_state_download(h, hin, 0, 1 << n))

        def run_sweep(st):
            for arr, _keep in placements:
                rc = lib.qcs_apply_step(st, arr, 1)
                if rc:
                    Q._check(rc)

        def request(i, last):
            st, prev = states[i % 2].handle, states[(i - 1) % 2].handle
            Q._check(lib.qcs_state_upload(st, hin, 0, 1 << n))
            if i > 0:
                Q._check(lib.qcs_state_wait(st, prev))  # after request i-1's sweep
            run_sweep(st)
            if i > 0:
                Q._check(lib.qcs_state_download_async(prev, hout[(i - 1) % 2], 0, 1 << n))
            if last:
                Q._check(lib.qcs_state_download_async(st, hout[i % 2], 0, 1 << n))

        def request_serial(i, last):
            st = states[0].handle
            Q._check(lib.qcs_state_upload(st, hin, 0, 1 << n))
            run_sweep(st)
            Q._check(lib.qcs_state_download_async(st, hout[0], 0, 1 << n))

        def timed(fn, count):
            for st in states:
                st.sync()
            dist.barrier()
            t0 = time.perf_counter()
            for i in range(count):
                fn(i, i == count - 1)
            for st in states:
                st.sync()
            return dist.max(1e3 * (time.perf_counter() - t0))

        e2e_ms = timed(request, e2e_steps)
        serial_ms = timed(request_serial, max(1, min(3, args.steps)))
        serial_steps = max(1, min(3, args.steps))
    finally:
        state2.close()
        for hp in bufs:
            lib.qcs_host_free(hp)
    e2e_value = world * updates_per_step * e2e_steps / (e2e_ms / 1e3)
    e2e_serial = world * updates_per_step * serial_steps / (serial_ms / 1e3)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        n_sample = min(n, 22)
        pairs = cpu_sample_pairs(n_sample, 12)
        v, secs, kind = reference_sample(n_sample, pairs, 1)
        cpu = {"value": v, "unit": UNIT, "cores": 1, "kind": kind,
               "sample": f"{len(pairs)} C2 single-gate runs at n={n_sample}, "
                         f"{'reference step_matrix_dax + dax_mvm' if kind == 'reference' else 'oracle port'}, "
                         f"1 thread, {secs:.1f} s"}

    csum = clocks.summary()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "c128 (f64 complex)", "data": "synthetic",
        "config": {"workload": f"C2 single-gate sweep, n={n}", "n_qubits": n,
                   "gates_per_step": len(sweep), "amplitude_updates_per_step": updates_per_step,
                   "state_bytes": 16 << n, "l2": "state 32x larger than L2, no flush needed",
                   "parallelism": "replicas" if world > 1 else "single GPU", "seed": configs.seed_of(2)},
        "roofline": {"bound": "hbm", "kernel": dom[0], "achieved": achieved, "peak": peak,
                     "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                     "frac_nominal_8TBs": achieved / 8000.0, "traffic": traffic,
                     "algorithmic_bytes_per_launch": dom_bytes / dom_launches,
                     "avg_launch_us": 1e3 * dom_ms / dom_launches, "launches": dom_launches,
                     "share_of_kernel_time": dom_ms / total_kernel_ms,
                     "all_kernels_GBps": all_bytes / (total_kernel_ms / 1e3) / 1e9,
                     "all_kernels_frac": all_bytes / (total_kernel_ms / 1e3) / 1e9 / peak},
        "kernel_classes": {k: {"launches": v[0], "ms": round(v[1], 3), "GBps": v[2] / (v[1] / 1e3) / 1e9}
                           for k, v in timing.items()},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes,
                "steps": e2e_steps, "requests_in_flight": 2, "timer": "host wall clock, both streams synced",
                "serial_value": e2e_serial},
        "gpu_launches": int(launches),
        "clocks": csum,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    state.close()
    dist.close()
    return 0


def run_circuit_arm(args, rank, world, local_rank):
    """Whole BASELINE circuits (C1, C3, C4, C5) through the fused engine.  World 1: qcsim.simulate
    on one device state.  World > 1: the state sharded over the ranks by its top log2(world)
    qubits (paper_2411_15332_b200/partition.py), half-shard exchanges over NCCL ("strong" scaling:
    the circuit is fixed)."""
    import torch
    from paper_2411_15332_b200 import configs
    from paper_2411_15332_b200 import qcsim as Q
    w = args.workload
    n = args.n_circuit
    build = {"c1": lambda: configs.c1_circuit(n or 12), "c3": lambda: configs.c3_circuit(n or 30),
             "c4": lambda: configs.c4_circuit(n or 32), "c5": lambda: configs.c5_circuit(n or 35)}[w]
    c = build()
    updates = {"c1": configs.c1_updates(c.n), "c3": configs.c3_updates(c.n), "c4": configs.c4_updates(c.n),
               "c5": configs.c5_updates(c.n)}[w]
    dist = Dist(world, local_rank)
    dev = local_rank if world > 1 else 0
    torch.cuda.set_device(dev)
    if world == 1:
        state = Q.DeviceState(c.n, c.initial, dev)

        def step():
            Q.simulate(c, Q.Engine.rh_dax, state=state)
        sync = state.sync
        plan = Q.plan_stats(c)
    else:
        from paper_2411_15332_b200.partition import DeviceBackend, DistTransport, ShardedState
        g = world.bit_length() - 1
        if args.peer:  # fused global-qubit gates over NVLink peer memory (torch symmetric memory)
            from paper_2411_15332_b200.partition import SymmetricTransport
            backend = DeviceBackend(c.n - g, dev, symmetric=True)
            sh = ShardedState(c.n, world, rank, backend, SymmetricTransport(), initial=c.initial)
        else:  # half-shard swaps over NCCL send/recv
            backend = DeviceBackend(c.n - g, dev)
            sh = ShardedState(c.n, world, rank, backend, DistTransport(), initial=c.initial, peer=False)
        ops = []
        for st in c.steps:
            if int(st.kind) == 1:
                ops.append(("diag", list(st.diag.flipped), st.diag.flip_rest))
            elif st.is_hadamard_all(c.n):
                ops.append(("rh",))
            else:
                ops += [("gate", p.gate.matrix, p.qubit_list(), p.gate.name) for p in st.placements]

        def step():
            sh.phys = list(range(c.n))
            sh.set_basis(c.initial)
            for op in ops:
                if op[0] == "gate":
                    sh.apply_gate(op[1], op[2], op[3])
                elif op[0] == "diag":
                    sh.apply_diag(op[1], op[2])
                else:
                    sh.apply_rh()
            sh.flush()

        def sync():
            torch.cuda.synchronize(dev)
    for _ in range(args.warmup):
        step()
    sync()
    dist.barrier()
    if world == 1:  # events on the state's own stream, per-launch timing of the kernel classes
        state.timing(True)
        state.timing_reset()
        with ClockSampler(dev) as clocks:
            state.record(0)
            for _ in range(args.steps):
                step()
            state.record(1)
            sync()
        ms = state.elapsed_ms(0, 1)
        timing = state.timing_report()
        state.timing(False)
    else:
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(dev) as clocks:
            ev0.record()
            for _ in range(args.steps):
                step()
            sync()
            ev1.record()
            ev1.synchronize()
        ms = dist.max(ev0.elapsed_time(ev1))
    value = updates * args.steps / (ms / 1e3)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "c128 (f64 complex)",
            "data": "synthetic", "config": {"workload": f"{w.upper()} circuit, n={c.n}", "n_qubits": c.n,
                                            "amplitude_updates_per_step": updates,
                                            "parallelism": f"sharded over {world} ranks (top qubits)" if world > 1
                                            else "single GPU, fused passes"},
            "clocks": clocks.summary()}
    if world == 1:
        peak, peak_kind = measured_peaks()
        k_ms = sum(v[1] for v in timing.values())
        k_bytes = sum(v[2] for v in timing.values())
        achieved = k_bytes / (k_ms / 1e3) / 1e9
        # algorithmic bytes: 32 B per amplitude per HBM pass (tile passes and single-op gate kernels)
        line["roofline"] = {"bound": "hbm", "kernel": "all passes", "achieved": achieved, "peak": peak,
                            "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                            "frac_nominal_8TBs": achieved / 8000.0, "traffic": None,
                            "passes_per_step": plan["passes"], "skip_passes_per_step": plan["skip_passes"],
                            "kernel_ms_per_step": k_ms / args.steps,
                            # the launched passes' algorithmic bytes at copy bandwidth (skip passes and
                            # pass pairs move only the tiles they reach)
                            "pass_floor_ms": k_bytes / args.steps / (peak * 1e9) * 1e3,
                            "full_sweeps_per_step": k_bytes / args.steps / (32.0 * (1 << c.n))}
        line["kernel_classes"] = {k: {"launches": v[0] / args.steps, "ms": round(v[1] / args.steps, 3),
                                      "GBps": v[2] / (v[1] / 1e3) / 1e9} for k, v in timing.items()}
        line["gpu_launches"] = int(sum(v[0] for v in timing.values()))
        state.close()
    if world > 1:
        line["exchanges_per_step"] = sh.swaps / (args.steps + args.warmup)
        line["peer_gates_per_step"] = sh.splits / (args.steps + args.warmup)
        line["config"]["global_qubit_gates"] = "peer-memory kernel" if sh.peer else "NCCL half-shard swaps"
    if rank == 0:
        print(json.dumps(line), flush=True)
    dist.close()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n", type=int, default=28)
    ap.add_argument("--workload", default="c2", choices=["c2", "c1", "c3", "c4", "c5"],
                    help="c2 (default): the single-gate sweep; c1/c3/c4/c5: whole BASELINE circuits")
    ap.add_argument("--n-circuit", type=int, default=0, help="qubits for c1/c3/c4/c5 (default: BASELINE size)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--peer", action="store_true",
                    help="c4/c5 under torchrun: gates on global qubits as one kernel over NVLink peer memory "
                         "(qcs_apply_split) instead of NCCL half-shard swaps")
    args = ap.parse_args()
    rank, world, local_rank = dist_env()
    if args.impl == "reference":
        return run_reference_arm(args, rank, world)
    if args.workload != "c2":
        return run_circuit_arm(args, rank, world, local_rank)
    return run_b200_arm(args, rank, world, local_rank)


if __name__ == "__main__":
    sys.exit(main())
