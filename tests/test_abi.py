"""The C-ABI library loads, exports every symbol include/qcs_abi.h declares, and the host-only
entry points behave like the reference (no GPU needed)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import ROOT, bits_equal


def declared_symbols():
    with open(os.path.join(ROOT, "include", "qcs_abi.h")) as f:
        text = f.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(qcs_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2411_15332_b200 import _lib
    lib = _lib.load()
    syms = declared_symbols()
    assert len(syms) > 40
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert set(syms) <= set(_lib.SIGNATURES), set(syms) - set(_lib.SIGNATURES)


def test_library_is_built_for_sm100a():
    import subprocess
    from paper_2411_15332_b200 import _lib
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_device_fails_loudly():
    from paper_2411_15332_b200 import qcsim as Q
    n = C.c_int()
    rc = Q.L.lib().qcs_device_count(C.byref(n))
    if rc == 0 and n.value > 0:
        pytest.skip("a CUDA device is present")
    with pytest.raises(Q.CudaError):
        Q.DeviceState(4)


def test_catalog_matches_reference_golden(golden):
    from paper_2411_15332_b200 import qcsim as Q
    g = golden("gates.npz")
    assert len(Q.gate_catalog()) == 38
    for name, k, p, m in zip(g["names"], g["arity"], g["params"], g["mats"]):
        info = next(x for x in Q.gate_catalog() if x.name == name)
        got = Q.gate_catalog_lookup(str(name), list(p[: info.param_count])).matrix.reshape(-1)
        assert bits_equal(got, m[: 4 ** int(k)]), name


def test_catalog_errors_and_aliases():
    from paper_2411_15332_b200 import qcsim as Q
    with pytest.raises(Q.SimError, match="unknown gate"):
        Q.gate_catalog_lookup("Frobnicator")
    with pytest.raises(Q.SimError, match="takes 1 parameter"):
        Q.gate_catalog_lookup("RX", [])
    with pytest.raises(Q.SimError):
        Q.gate_catalog_lookup("Hadamard", [0.5])
    for alias, name in [("H", "Hadamard"), ("CNOT", "Controlled-X"), ("Toffoli", "CCX"), ("SWAP", "Swap"),
                        ("CZ", "Controlled-Z"), ("Tdg", "T-adjoint"), ("Fredkin", "CSwap")]:
        assert Q.gate_catalog_lookup(alias).name == name
    assert Q.canonical_params("U") == [1.1, 0.7, 0.3]
    # catalog classes (test_core.cpp:9-21) and unitarity
    for info in Q.gate_catalog():
        m = Q.gate_catalog_lookup(info.name, Q.canonical_params(info.name)).matrix
        assert np.allclose(m @ m.conj().T, np.eye(m.shape[0]), atol=1e-12)
        assert float(np.mean(m == 0)) == info.zero_ratio


def test_dense_cap_roundtrip():
    from paper_2411_15332_b200 import _lib
    lib = _lib.lib()
    assert lib.qcs_dense_cap() == 1 << 26
    lib.qcs_set_dense_cap(1 << 10)
    assert lib.qcs_dense_cap() == 1 << 10
    lib.qcs_set_dense_cap(1 << 26)
