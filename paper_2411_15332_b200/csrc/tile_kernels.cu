// tile_kernels.cu -- fused shared-memory passes (sm_100a).
//
// A pass owns a set S of m basis-bit positions (the tile bits).  Each CTA loads the 2^m
// amplitudes of one tile -- all indices that agree outside S -- into shared memory, applies
// a list of operations, and writes the tile back: one HBM round trip (32 B per amplitude)
// for the whole list.  S always contains the lowest basis bits so every warp load covers
// contiguous 512-byte runs.
//
// Operations (TileOp): gates whose target bits lie in S (controls may lie outside S: they
// are constant over a tile), diagonal gates and sign steps anywhere (a tile knows its full
// indices), unnormalised Walsh-Hadamard butterflies over bits of S, and a real scale.  The
// Walsh-Hadamard path is the RH structure of the reference (rh.cpp:92-156: scale by
// 2^{-n/2} first, then +-1 sums), computed as radix-8 register butterflies instead of the
// reference's O(4^n) sign loop.  Gate rows use dax_mvm's arithmetic (see gate_kernels.cu).
#include <cstdint>

#include "common.hpp"
#include "kernels.hpp"

namespace qcs {
namespace {

using u64 = std::uint64_t;
constexpr int kTileThreads = 512;
constexpr int kMaxTileBits = 12;  // 64 KiB of amplitudes per CTA -> 3 CTAs per SM
constexpr int kLoBits = 5;

__device__ __forceinline__ double2 madd(double2 acc, double2 v, double2 x) {
    const double pr = __dsub_rn(__dmul_rn(v.x, x.x), __dmul_rn(v.y, x.y));
    const double pi = __dadd_rn(__dmul_rn(v.x, x.y), __dmul_rn(v.y, x.x));
    return make_double2(__dadd_rn(acc.x, pr), __dadd_rn(acc.y, pi));
}

__device__ __forceinline__ double2 neg_exact(double2 x) {
    const double pr = __dsub_rn(__dmul_rn(-1.0, x.x), __dmul_rn(0.0, x.y));
    const double pi = __dadd_rn(__dmul_rn(-1.0, x.y), __dmul_rn(0.0, x.x));
    return make_double2(__dadd_rn(0.0, pr), __dadd_rn(0.0, pi));
}

__device__ __forceinline__ unsigned insert_zero(unsigned t, int b) {
    return ((t >> b) << (b + 1)) | (t & ((1u << b) - 1));
}

__device__ __forceinline__ bool listed(const u64* f, u64 nf, u64 i) {
    u64 lo = 0, hi = nf;
    while (lo < hi) {
        const u64 mid = (lo + hi) >> 1;
        if (__ldg(f + mid) < i) lo = mid + 1; else hi = mid;
    }
    return lo < nf && __ldg(f + lo) == i;
}

struct TileCtx {
    double2* sm;
    const u64* lo_tab;
    const u64* hi_tab;
    int m;
    int lo_bits;
    u64 base;
    __device__ __forceinline__ u64 global(unsigned j) const {
        return base | lo_tab[j & ((1u << lo_bits) - 1)] | hi_tab[j >> lo_bits];
    }
};

__device__ void op_gate(const TileCtx& c, const TileOp& o) {
    if (o.gctrl_mask && (c.base & o.gctrl_mask) != o.gctrl_val) return;
    const int k = o.k, nf = o.nfree, nrows = o.nrows;
    const unsigned ngroups = 1u << (c.m - k);
    unsigned moff[8];
#pragma unroll
    for (int mm = 0; mm < 8; ++mm) {
        unsigned off = 0;
#pragma unroll
        for (int i = 0; i < 3; ++i)
            if (i < nf && (mm >> i & 1)) off |= o.lfree_bit[i];
        moff[mm] = off;
    }
    for (unsigned g = threadIdx.x; g < ngroups; g += blockDim.x) {
        unsigned lb = g;
        for (int i = 0; i < k; ++i) lb = insert_zero(lb, o.lbit[i]);
        lb |= o.lfixed_val;
        double2 x[8];
#pragma unroll
        for (int mm = 0; mm < 8; ++mm)
            if (mm < (1 << nf) && (o.load_mask >> mm & 1)) x[mm] = c.sm[lb | moff[mm]];
        double2 out[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            if (r < nrows) {
                double2 acc = make_double2(0.0, 0.0);
                for (int z = 0; z < o.nnz[r]; ++z) {
                    const int cm = o.col_member[r][z];
                    double2 xv = x[0];
#pragma unroll
                    for (int mm = 1; mm < 8; ++mm)
                        if (cm == mm) xv = x[mm];
                    acc = madd(acc, o.val[r][z], xv);
                }
                out[r] = acc;
            }
        }
#pragma unroll
        for (int r = 0; r < 8; ++r)
            if (r < nrows) c.sm[lb | moff[o.row_member[r]]] = out[r];
    }
}

__device__ void op_diag(const TileCtx& c, const TileOp& o) {
    const unsigned sz = 1u << c.m;
    for (unsigned j = threadIdx.x; j < sz; j += blockDim.x) {
        const u64 gidx = c.global(j);
        int g = 0;
        for (int i = 0; i < o.k; ++i) g = (g << 1) | int((gidx >> o.dpos[i]) & 1);
        if (!o.dskip[g]) c.sm[j] = madd(make_double2(0.0, 0.0), o.val[0][g], c.sm[j]);
    }
}

__device__ void op_sign(const TileCtx& c, const TileOp& o, const u64* flipped, u64 tile_mask) {
    const u64* f = flipped + o.flip_off;
    if (!o.flip_rest) {
        // few listed indices: negate those that fall in this tile
        for (u64 e = threadIdx.x; e < o.flip_cnt; e += blockDim.x) {
            const u64 idx = __ldg(f + e);
            if ((idx & ~tile_mask) != c.base) continue;
            if (e > 0 && __ldg(f + e - 1) == idx) continue;
            // local index: compress the tile bits of idx
            unsigned j = 0;
            for (int b = c.m - 1; b >= 0; --b) {
                // find global position of local bit b via the tables: bit b of j selects
                const u64 gb = b < c.lo_bits ? c.lo_tab[1u << b] : c.hi_tab[1u << (b - c.lo_bits)];
                j = (j << 1) | ((idx & gb) ? 1u : 0u);
            }
            c.sm[j] = neg_exact(c.sm[j]);
        }
        return;
    }
    const unsigned sz = 1u << c.m;
    for (unsigned j = threadIdx.x; j < sz; j += blockDim.x)
        if (!listed(f, o.flip_cnt, c.global(j))) c.sm[j] = neg_exact(c.sm[j]);
}

// Butterflies over up to 3 local bits per round, held in registers.
__device__ void op_wht(const TileCtx& c, unsigned mask) {
    int bits[16], nb = 0;
    for (int b = 0; b < c.m; ++b)
        if (mask >> b & 1) bits[nb++] = b;
    for (int r0 = 0; r0 < nb; r0 += 3) {
        const int R = nb - r0 < 3 ? nb - r0 : 3;
        const int b0 = bits[r0], b1 = R > 1 ? bits[r0 + 1] : 0, b2 = R > 2 ? bits[r0 + 2] : 0;
        const unsigned ngroups = 1u << (c.m - R);
        for (unsigned g = threadIdx.x; g < ngroups; g += blockDim.x) {
            unsigned lb = insert_zero(g, b0);
            if (R > 1) lb = insert_zero(lb, b1);
            if (R > 2) lb = insert_zero(lb, b2);
            const unsigned o1 = 1u << b0, o2 = R > 1 ? 1u << b1 : 0u, o3 = R > 2 ? 1u << b2 : 0u;
            if (R == 1) {
                const double2 x = c.sm[lb], y = c.sm[lb | o1];
                c.sm[lb] = make_double2(x.x + y.x, x.y + y.y);
                c.sm[lb | o1] = make_double2(x.x - y.x, x.y - y.y);
            } else if (R == 2) {
                double2 v[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) v[q] = c.sm[lb | ((q & 1) ? o1 : 0u) | ((q & 2) ? o2 : 0u)];
#pragma unroll
                for (int s = 1; s < 4; s <<= 1)
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        if (!(q & s)) {
                            const double2 x = v[q], y = v[q | s];
                            v[q] = make_double2(x.x + y.x, x.y + y.y);
                            v[q | s] = make_double2(x.x - y.x, x.y - y.y);
                        }
#pragma unroll
                for (int q = 0; q < 4; ++q) c.sm[lb | ((q & 1) ? o1 : 0u) | ((q & 2) ? o2 : 0u)] = v[q];
            } else {
                double2 v[8];
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    v[q] = c.sm[lb | ((q & 1) ? o1 : 0u) | ((q & 2) ? o2 : 0u) | ((q & 4) ? o3 : 0u)];
#pragma unroll
                for (int s = 1; s < 8; s <<= 1)
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        if (!(q & s)) {
                            const double2 x = v[q], y = v[q | s];
                            v[q] = make_double2(x.x + y.x, x.y + y.y);
                            v[q | s] = make_double2(x.x - y.x, x.y - y.y);
                        }
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    c.sm[lb | ((q & 1) ? o1 : 0u) | ((q & 2) ? o2 : 0u) | ((q & 4) ? o3 : 0u)] = v[q];
            }
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kTileThreads) k_tile(double2* __restrict__ a, const __grid_constant__ TilePass p,
                                                       const TileOp* __restrict__ ops,
                                                       const u64* __restrict__ flipped) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int m = p.m;
    const int lo_bits = m < kLoBits ? m : kLoBits;
    double2* sm = reinterpret_cast<double2*>(smem_raw);
    u64* lo_tab = reinterpret_cast<u64*>(sm + (1u << m));
    u64* hi_tab = lo_tab + (1u << lo_bits);
    for (unsigned j = threadIdx.x; j < (1u << lo_bits); j += blockDim.x) {
        u64 v = 0;
        for (int b = 0; b < lo_bits; ++b)
            if (j >> b & 1) v |= u64(1) << p.bits[b];
        lo_tab[j] = v;
    }
    for (unsigned j = threadIdx.x; j < (1u << (m - lo_bits)); j += blockDim.x) {
        u64 v = 0;
        for (int b = lo_bits; b < m; ++b)
            if (j >> (b - lo_bits) & 1) v |= u64(1) << p.bits[b];
        hi_tab[j] = v;
    }
    u64 base = blockIdx.x;
    u64 tile_mask = 0;
    for (int b = 0; b < m; ++b) {  // bits[] ascending: insert zeros from the lowest position up
        const int pos = p.bits[b];
        base = ((base >> pos) << (pos + 1)) | (base & ((u64(1) << pos) - 1));
        tile_mask |= u64(1) << pos;
    }
    __syncthreads();
    TileCtx c{sm, lo_tab, hi_tab, m, lo_bits, base};
    const unsigned sz = 1u << m;
    for (unsigned j = threadIdx.x; j < sz; j += blockDim.x) sm[j] = __ldcs(a + c.global(j));
    __syncthreads();
    for (int i = 0; i < p.op_count; ++i) {
        const TileOp& o = ops[p.op_begin + i];
        switch (o.kind) {
            case TOP_GATE: op_gate(c, o); break;
            case TOP_DIAG: op_diag(c, o); break;
            case TOP_SIGN: op_sign(c, o, flipped, tile_mask); break;
            case TOP_WHT: op_wht(c, o.wht_mask); break;
            case TOP_SCALE:
                for (unsigned j = threadIdx.x; j < sz; j += blockDim.x)
                    sm[j] = make_double2(sm[j].x * o.scale, sm[j].y * o.scale);
                break;
            default: break;
        }
        __syncthreads();
    }
    for (unsigned j = threadIdx.x; j < sz; j += blockDim.x) __stcs(a + c.global(j), sm[j]);
}

}  // namespace

int tile_max_bits() { return kMaxTileBits; }

void launch_tile_pass(double2* amps, int n, const TilePass& p, const TileOp* ops_dev,
                      const std::uint64_t* flipped_dev, cudaStream_t st) {
    if (p.m < 1 || p.m > kMaxTileBits || p.m > n) raise(QCS_ERR_ARG, "tile bits out of range");
    const int lo_bits = p.m < kLoBits ? p.m : kLoBits;
    const std::size_t smem = (std::size_t(1) << p.m) * sizeof(double2) +
                             ((std::size_t(1) << lo_bits) + (std::size_t(1) << (p.m - lo_bits))) * sizeof(u64);
    static bool attr_set[64] = {};  // the attribute is per device
    int dev = 0;
    QCS_CUDA(cudaGetDevice(&dev));
    if (dev < 64 && !attr_set[dev]) {
        const int max_smem = (1 << kMaxTileBits) * 16 + ((1 << kLoBits) + (1 << (kMaxTileBits - kLoBits))) * 8;
        QCS_CUDA(cudaFuncSetAttribute(k_tile, cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem));
        attr_set[dev] = true;
    }
    const u64 tiles = u64(1) << (n - p.m);
    if (tiles > 0x7fffffffull) raise(QCS_ERR_CAPACITY, "too many tiles for one launch");
    TimedLaunch tl("tile_pass", 32.0 * double(u64(1) << n), st);
    k_tile<<<unsigned(tiles), kTileThreads, smem, st>>>(amps, p, ops_dev, flipped_dev);
    check_launch("k_tile");
}

}  // namespace qcs
