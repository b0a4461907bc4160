"""The TMA tensor-map layout of fused-pass tiles (kernels.hpp tma_layout), checked on the host:
for random tile bit sets over n-bit states, walking every element of the box through the dims'
extents, strides and coordinates must visit exactly the tile's amplitudes at a random tile base,
in ascending local-index order (the order the register rounds address shared memory in), with
every coordinate inside its dim.  Both layouts: gaps riding in the run dims below them (default)
and the round-1 one-dim-per-gap form (QCS_TMA_GAP_DIMS=1)."""
import os
import subprocess
import tempfile

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2411_15332_b200", "csrc")

DRIVER = r"""
#include "kernels.hpp"
#include <cstdio>
int main() {
    unsigned long long S; int n, gap;
    while (std::scanf("%llu %d %d", &S, &n, &gap) == 3) {
        qcs::TmaDim L[16];
        const int r = qcs::tma_layout(S, n, L, gap != 0);
        std::printf("%d", r);
        for (int d = 0; d < r && d < 16; ++d) std::printf(" %d %d %d", L[d].pos, L[d].len, L[d].inlen);
        std::printf("\n");
    }
}
"""


@pytest.fixture(scope="module")
def layout_exe():
    d = tempfile.mkdtemp()
    src, exe = os.path.join(d, "t.cpp"), os.path.join(d, "t")
    open(src, "w").write(DRIVER)
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", CSRC, "-I", "/usr/local/cuda/include", src, "-o", exe],
                   check=True)
    return exe


def layouts(exe, cases):
    inp = "".join(f"{S} {n} {g}\n" for S, n, g in cases)
    out = subprocess.run([exe], input=inp, capture_output=True, text=True, check=True).stdout.split("\n")
    res = []
    for line in out[:len(cases)]:
        v = [int(x) for x in line.split()]
        res.append((v[0], [tuple(v[1 + 3 * i: 4 + 3 * i]) for i in range(min(v[0], 16))]))
    return res


def walk(dims, base):
    """Amplitude index of every box element in box order (dim 0 fastest): the kernel's coordinates
    (tile_device.cuh tma_coord) plus the box offsets, times the dims' strides."""
    coords, strides, boxes = [], [], []
    for d, (pos, ln, inl) in enumerate(dims):
        if d == 0:
            c = (base & ((1 << ln) - 1)) << 1  # doubles
            assert c + 16 <= 2 << ln
            coords.append(c), boxes.append(16), strides.append(None)
        else:
            c = (base >> pos) & ((1 << ln) - 1) if ln > inl else 0
            assert c + (1 << inl) <= 1 << ln, "box leaves its dim"
            assert c < 2 ** 31
            coords.append(c), boxes.append(1 << inl), strides.append(1 << pos)  # amplitudes
    idx = np.zeros(1, dtype=np.int64)
    for d in range(len(dims)):
        if d == 0:
            el = (coords[0] + np.arange(16)) >> 1  # two doubles per amplitude
            # keep one entry per amplitude (the real part's slot)
            el = el[::2]
            idx = el.astype(np.int64)
        else:
            add = (coords[d] + np.arange(boxes[d], dtype=np.int64)) * strides[d]
            idx = (idx[None, :] + add[:, None]).reshape(-1)
    return idx


def deposit_all(S, base):
    bits = [b for b in range(64) if S >> b & 1]
    out = np.zeros(1 << len(bits), dtype=np.int64)
    for i, b in enumerate(bits):
        half = 1 << i
        out[half:2 * half] = out[:half] | (1 << b)
    return out | base


@pytest.mark.parametrize("gap", [0, 1])
def test_tma_layout_addresses_the_tile(layout_exe, gap):
    rng = np.random.default_rng(7 + gap)
    cases = []
    for _ in range(400):
        n = int(rng.integers(3, 37))
        m = int(rng.integers(3, min(n, 12) + 1))
        others = rng.permutation(np.arange(3, n))[: m - 3] if n > 3 else []
        S = 7
        for b in others:
            S |= 1 << int(b)
        cases.append((S, n, gap))
    seen_ranks = set()
    for (S, n, _), (rank, dims) in zip(cases, layouts(layout_exe, cases)):
        seen_ranks.add(rank)
        if rank > 16:  # the one-dim-per-gap form on scattered tiles (never encodable)
            assert gap
            continue
        # every state bit below n is covered exactly once, in order
        cover = 0
        for pos, ln, inl in dims:
            assert pos == cover and 0 <= inl <= ln and (inl <= 8 or pos == 0)
            assert ln <= 31
            cover += ln
        assert cover == n
        base = int(rng.integers(0, 1 << n)) & ~S
        got = walk(dims, base)
        assert np.array_equal(got, deposit_all(S, base)), (S, n, dims)
    assert min(seen_ranks) <= 3 and max(seen_ranks) >= 5


def test_gaps_cost_no_dims(layout_exe):
    """A tile of 4 separate runs above the low bits fits 5 dims only when its gaps ride along."""
    S = 7 | (1 << 7) | (1 << 12) | (1 << 20) | (1 << 27)
    (r0, _), (r1, _) = layouts(layout_exe, [(S, 32, 0), (S, 32, 1)])
    assert r0 == 5 and r1 == 10
    # the widest gaps get dims of their own (31-bit coordinates)
    (r2, dims), = layouts(layout_exe, [(7 | (1 << 35), 36, 0)])
    assert r2 == 4 and dims == [(0, 3, 3), (3, 31, 0), (34, 1, 0), (35, 1, 1)]
