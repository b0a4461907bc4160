"""bench.py's host-side contract, on the CPU: the standalone C4 gate list of the reference arm is
the product's C4 circuit, the reference arm imports nothing from the product package, and the
`--gpus 2` launcher path (torchrun, gloo, remap exchanges, dry run) prints the JSON line."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT


def test_c4_gate_list_matches_configs():
    sys.path.insert(0, ROOT)
    import bench
    from paper_2411_15332_b200 import configs
    for n, layers in ((32, 10), (9, 2)):
        c = configs.c4_circuit(n, layers)
        mine = bench.c4_gate_list(n, layers)
        theirs = [(p.gate.name, list(p.gate.params), p.qubit_list()) for st in c.steps for p in st.placements]
        assert len(mine) == len(theirs) == n + 3 * n * layers
        for a, b in zip(mine, theirs):
            assert a[0] == b[0] and a[2] == b[2] and np.array_equal(a[1], b[1])
    assert bench.workload_config("c4", 32)["amplitude_updates_per_step"] == configs.c4_updates(32)


def test_reference_arm_is_standalone():
    """--impl reference runs the compiled reference (or the oracle port) and never imports the
    product package; its config equals the b200 arm's."""
    code = ("import sys, json; sys.argv = ['bench.py', '--impl', 'reference', '--steps', '1', '--warmup', '0', "
            "'--ref-n', '12']; sys.path.insert(0, %r); import bench; bench.main(); "
            "assert not any(m.startswith('paper_2411_15332_b200') for m in sys.modules), 'product imported'" % ROOT)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    sys.path.insert(0, ROOT)
    import bench
    assert line["impl"] == "reference" and line["config"] == bench.workload_config("c4", 32)
    assert line["cpu_baseline"]["kind"] in ("reference", "port") and line["e2e"]["h2d_bytes_per_step"] == 0


@pytest.mark.timeout(900)
def test_gpus2_launcher_dry_run():
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env.pop("RANK", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run",
                          "--n-circuit", "10", "--steps", "2", "--warmup", "1"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1  # rank 0 only
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["dry_run"] is True
    ex = d["exchange"]
    assert ex["remaps_per_step"] >= 1 and ex["bytes_sent_per_step_per_rank"] > 0
    assert 0 < ex["shards_moved_per_step"] <= 11
    assert any("gloo" in s for s in d["comm_init"])
    for k in ("metric", "value", "unit", "steps", "warmup", "ms_per_step", "config"):
        assert k in d
