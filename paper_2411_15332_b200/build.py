"""Build libqcs_b200.so in-tree with nvcc for sm_100a (no JIT, no torch extension cache).

    python -m paper_2411_15332_b200.build          # or build() from __graft_entry__

Every source compiles with ``-fmad=false``: the kernels reproduce the reference's
separately-rounded complex arithmetic (x86-64 SSE2 without FMA) for bit-exact parity.
"""
from __future__ import annotations

import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libqcs_b200.so")
OBJ = os.path.join(HERE, "_build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++20", "-lineinfo", "-fmad=false", "-Xcompiler", "-fPIC",
          "-I" + os.path.join(ROOT, "include"), "-I" + CSRC, "--expt-relaxed-constexpr"]
# tuning experiments only (e.g. "-DQCS_TILE_NG=1"); part of the build stamp
COMMON += os.environ.get("QCS_EXTRA_NVCC", "").split()

SOURCES = ["gates.cpp", "ops.cpp", "planner.cpp", "engine.cpp", "abi.cpp", "timing.cpp",
           "gate_kernels.cu", "tile_kernels.cu", "state_kernels.cu", "encode_kernels.cu", "peer_kernels.cu", "sample_kernels.cu", "dense_kernels.cu",
           "jit.cpp"]
# embedded into the library for the run-time (NVRTC) pass kernels, jit.cpp
JIT_HEADERS = [("kJitSrcKernels", "kernels.hpp"), ("kJitSrcDevice", "tile_device.cuh")]


def _hash(paths):
    h = hashlib.sha256()
    for p in paths:
        with open(p, "rb") as f:
            h.update(f.read())
    h.update(" ".join(ARCH + COMMON).encode())
    return h.hexdigest()[:16]


def _embed_jit_sources() -> str:
    """_build/jit_src.cpp: the device headers as string constants for NVRTC (jit.cpp)."""
    path = os.path.join(OBJ, "jit_src.cpp")
    parts = ["namespace qcs {"]
    for sym, name in JIT_HEADERS:
        with open(os.path.join(CSRC, name)) as f:
            text = f.read()
        if ")qcsjit\"" in text:
            raise RuntimeError(f"{name} contains the raw-string delimiter")
        parts.append(f'extern const char* const {sym};\nconst char* const {sym} = R"qcsjit({text})qcsjit";')
    parts.append("}  // namespace qcs\n")
    with open(path, "w") as f:
        f.write("\n".join(parts))
    return path


def build(verbose: bool = False, force: bool = False) -> str:
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".hpp", ".cuh"))]
    headers.append(os.path.join(ROOT, "include", "qcs_abi.h"))
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    stamp = os.path.join(OBJ, "stamp")
    digest = _hash(sorted(headers) + srcs)
    if not force and os.path.exists(OUT) and os.path.exists(stamp) and open(stamp).read() == digest:
        return OUT
    os.makedirs(OBJ, exist_ok=True)
    srcs = srcs + [_embed_jit_sources()]
    objs = []
    procs = []
    for s in srcs:
        o = os.path.join(OBJ, os.path.basename(s) + ".o")
        lang = ["-x", "cu"] if s.endswith(".cu") else []
        cmd = [NVCC, *ARCH, *COMMON, *lang, "-c", s, "-o", o]
        if verbose:
            print(" ".join(cmd), flush=True)
        procs.append((s, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(o)
    failed = []
    for s, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            failed.append((s, out.decode(errors="replace")))
        elif verbose and out:
            print(out.decode(errors="replace"))
    if failed:
        msg = "\n".join(f"--- {s}\n{o}" for s, o in failed)
        raise RuntimeError(f"nvcc failed:\n{msg}")
    cudalib = os.path.join(os.path.dirname(os.path.dirname(NVCC)), "lib64")
    link = [NVCC, *ARCH, "-shared", "-o", OUT, *objs, "-Xcompiler", "-fPIC", "-lnvrtc", "-L" + cudalib,
            "-Xlinker", "-rpath=" + cudalib] + os.environ.get("QCS_EXTRA_LINK", "").split()
    if verbose:
        print(" ".join(link), flush=True)
    subprocess.run(link, check=True)
    with open(stamp, "w") as f:
        f.write(digest)
    return OUT


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
