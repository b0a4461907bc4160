// peer_kernels.cu -- gates on a shard-global qubit, computed straight over peer memory (sm_100a).
//
// A state sharded by its top qubits (partition.py) keeps the amplitude pair of a gate on a
// global qubit on two ranks: x0 on the rank whose global bit is 0, x1 on its partner, at the
// same local index.  Instead of exchanging half shards and running the gate locally, each rank
// takes the pairs in one half of the local index space (local top bit == its own global bit),
// loads the partner's amplitude over NVLink (P2P load), computes both outputs and stores the
// partner's back (P2P store): the exchange and the arithmetic are one kernel and overlap per
// pair.  Pairs never overlap between the two ranks, so no atomics; the callers order the two
// kernels with a barrier on each side.
//
// Arithmetic follows dax_mvm (dax.cpp:96-103): acc = 0; acc += m[r][c] * x_c for the nonzero
// entries in ascending column order, separately rounded (-fmad=false), so the result equals
// the single-GPU gate kernels' and the reference's bit for bit.  Blocks that are exactly the
// identity (a local control that is off) are not touched.
#include <cstdint>

#include "common.hpp"
#include "kernels.hpp"

namespace qcs {
namespace {

using u64 = std::uint64_t;

__device__ __forceinline__ double2 madd(double2 acc, double2 v, double2 x) {
    const double pr = __dsub_rn(__dmul_rn(v.x, x.x), __dmul_rn(v.y, x.y));
    const double pi = __dadd_rn(__dmul_rn(v.x, x.y), __dmul_rn(v.y, x.x));
    return make_double2(__dadd_rn(acc.x, pr), __dadd_rn(acc.y, pi));
}

__device__ __forceinline__ double2 row(const SplitParams& p, int v, int r, double2 x0, double2 x1) {
    double2 acc = make_double2(0.0, 0.0);
    if (p.nz[v] >> (2 * r) & 1) acc = madd(acc, p.m[v][2 * r], x0);
    if (p.nz[v] >> (2 * r + 1) & 1) acc = madd(acc, p.m[v][2 * r + 1], x1);
    return acc;
}

__global__ void __launch_bounds__(256) k_split_pair(double2* __restrict__ self, double2* __restrict__ peer,
                                                    const __grid_constant__ SplitParams p) {
    const u64 half = u64(1) << (p.nl - 1);
    const u64 base = p.self_bit ? half : 0;
    const u64 stride = u64(gridDim.x) * blockDim.x;
    for (u64 j = u64(blockIdx.x) * blockDim.x + threadIdx.x; j < half; j += stride) {
        const u64 i = base | j;
        int v = 0;
        for (int s = 0; s < p.nsel; ++s) v = (v << 1) | int((i >> p.sel[s]) & 1);
        if (p.skip >> v & 1) continue;
        const double2 xs = __ldcs(self + i), xp = __ldcs(peer + i);
        const double2 x0 = p.self_bit ? xp : xs, x1 = p.self_bit ? xs : xp;
        const double2 o0 = row(p, v, 0, x0, x1), o1 = row(p, v, 1, x0, x1);
        __stcs(self + i, p.self_bit ? o1 : o0);
        __stcs(peer + i, p.self_bit ? o0 : o1);
    }
}

// Swap [self, self + count) with [peer, peer + count): the data movement of a global<->local
// qubit remap (partition.py).  Each rank of a pair swaps one half of the block pair, so every
// amplitude crosses the link once each way and nothing is staged.  32-byte vectors (two
// amplitudes) when both ends are 32-byte aligned.
__global__ void __launch_bounds__(256) k_swap_peer(double2* __restrict__ self, double2* __restrict__ peer, u64 count) {
    const u64 stride = u64(gridDim.x) * blockDim.x;
    for (u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride) {
        const double2 a = __ldcs(self + i), b = __ldcs(peer + i);
        __stcs(self + i, b);
        __stcs(peer + i, a);
    }
}

}  // namespace

void launch_swap_peer(double2* self, double2* peer, std::uint64_t count, cudaStream_t st) {
    if (!count) return;
    const u64 want = (count + 255) / 256;
    const unsigned grid = unsigned(want < 1 ? 1 : (want > 148 * 16 ? 148 * 16 : want));
    // algorithmic bytes: both blocks read and written once (half of it over the peer link)
    TimedLaunch tl("swap_peer", 64.0 * double(count), st);
    k_swap_peer<<<grid, 256, 0, st>>>(self, peer, count);
    check_launch("k_swap_peer");
}

void launch_split_pair(double2* self, double2* peer, const SplitParams& p, cudaStream_t st) {
    const u64 half = u64(1) << (p.nl - 1);
    const u64 want = (half + 255) / 256;
    const unsigned grid = unsigned(want < 1 ? 1 : (want > 148 * 16 ? 148 * 16 : want));
    // algorithmic bytes: every touched pair read and written, half of it over the peer link
    TimedLaunch tl("split_pair", 64.0 * double(half), st);
    k_split_pair<<<grid, 256, 0, st>>>(self, peer, p);
    check_launch("k_split_pair");
}

}  // namespace qcs
