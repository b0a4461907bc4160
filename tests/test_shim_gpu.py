"""The reference's own acceptance suite (tests/acceptance.cpp, 11 criteria) with its
src/engine.cpp replaced by shim/engine_b200.cpp -- i.e. qcsim::simulate / step_matrix_dax /
step_matrix_das / memory_report running on the B200 through the C ABI.  Criteria 10 (Grover on
every engine vs the dense Matrix engine, n = 4..12) and 11 (12-qubit neuron) exercise the GPU."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
BIN = os.path.join(ROOT, "oracle", "_ref", "acceptance_b200")


def test_reference_acceptance_suite_on_b200():
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/acceptance_b200 not built (needs the reference sources at build time)")
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "all 11 criteria passed" in out.stdout
