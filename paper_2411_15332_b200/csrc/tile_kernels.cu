// tile_kernels.cu -- fused shared-memory passes (sm_100a).
//
// A pass owns a set S of m basis-bit positions, the tile bits (S always holds bits 0..2, so a
// tile is made of 128-byte runs).  Each CTA moves the 2^m amplitudes of one tile -- the indices
// that agree outside S -- from HBM into shared memory, runs the pass's operations, and writes
// the tile back: one HBM round trip, 32 B per amplitude, for the whole operation list.  Where
// the bit layout fits a <= 5-dim tensor map the tile moves as ONE TMA box each way
// (cp.async.bulk.tensor + mbarrier; the 128-byte TMA swizzle is exactly the layout below);
// otherwise every thread issues 16-byte cp.async copies.
//
// Operations execute in rounds: in a round each thread holds 8 amplitudes in registers that
// differ exactly in three tile bits (the round bits) and applies every operation of the round
// to them; rounds are separated by one shared-memory exchange and a barrier.  Shared memory is
// XOR-swizzled (position = j ^ ((j >> 3) & 7)) so 16-byte accesses spread over the banks
// whichever three bits a round owns.  The pass description -- rounds and compact operations --
// travels in the kernel parameter space (<= 32 KB), i.e. the constant bank: every thread
// reads the same operation at the same time, which the constant cache broadcasts.
//
// Register operations: a one-target gate as a dense 2x2 (controls anywhere; tile-bit controls
// per register, controls outside the tile once per CTA), up to three consecutive uncontrolled
// gates bundled into one operation, a diagonal phase on up to three basis bits, +-1 diagonals
// as pending sign flips, a diagonal sign step (Grover oracle / Z0, engine.cpp:62-80),
// unnormalised Walsh-Hadamard butterflies (rh.cpp:92-156: scale by 2^{-n/2}, then +-1 sums)
// and a real scale.  Gates on 2-3 targets run straight on shared memory in rounds of their
// own.  Tiles no sign step reaches run the pass's simplified program, or nothing.
//
// Arithmetic: a fused pass reorders the reference's per-step fold anyway, so it is held to the
// 1e-12 bar and uses fused multiply-adds (half the FP64 instructions).  Passes of a single
// operation never come here: the engine runs them with the bit-exact gate kernels.
#include <algorithm>
#include <cstdint>

#include <cuda.h>

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

__device__ __forceinline__ double2 neg_exact(double2 x) {
    const double pr = __dsub_rn(__dmul_rn(-1.0, x.x), __dmul_rn(0.0, x.y));
    const double pi = __dadd_rn(__dmul_rn(-1.0, x.y), __dmul_rn(0.0, x.x));
    return make_double2(__dadd_rn(0.0, pr), __dadd_rn(0.0, pi));
}

__device__ __forceinline__ unsigned swz(unsigned j) { return j ^ ((j >> 3) & 7u); }

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

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// ---- TMA: the whole tile as one tensor-map box (cp.async.bulk.tensor), 128-byte swizzle
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void tma_load(void* dst, const CUtensorMap* map, const int (&c)[5], int rank,
                                         unsigned long long* bar) {
    const unsigned d = smem_u32(dst), b = smem_u32(bar);
    const auto m = reinterpret_cast<unsigned long long>(map);
    switch (rank) {
        case 2:
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                         " [%0], [%1, {%2, %3}], [%4];" ::"r"(d), "l"(m), "r"(c[0]), "r"(c[1]), "r"(b) : "memory");
            break;
        case 3:
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                         " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(d), "l"(m), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(b)
                         : "memory");
            break;
        case 4:
            asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                         " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(d), "l"(m), "r"(c[0]), "r"(c[1]), "r"(c[2]),
                         "r"(c[3]), "r"(b)
                         : "memory");
            break;
        default:
            asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                         " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(d), "l"(m), "r"(c[0]), "r"(c[1]), "r"(c[2]),
                         "r"(c[3]), "r"(c[4]), "r"(b)
                         : "memory");
            break;
    }
}
__device__ __forceinline__ void tma_store(const CUtensorMap* map, const int (&c)[5], int rank, const void* src) {
    const unsigned s_ = smem_u32(src);
    const auto m = reinterpret_cast<unsigned long long>(map);
    switch (rank) {
        case 2:
            asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(m),
                         "r"(c[0]), "r"(c[1]), "r"(s_)
                         : "memory");
            break;
        case 3:
            asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(m),
                         "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(s_)
                         : "memory");
            break;
        case 4:
            asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(
                             m),
                         "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(s_)
                         : "memory");
            break;
        default:
            asm volatile(
                "cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(m),
                "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(s_)
                : "memory");
            break;
    }
    asm volatile("cp.async.bulk.commit_group;\ncp.async.bulk.wait_group.read 0;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\nfence.mbarrier_init.release.cluster;\n" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait0(unsigned long long* bar) {
    asm volatile(
        "{\n.reg .pred done;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], 0;\n"
        "@!done bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar))
        : "memory");
}

// Fused passes are held to the 1e-12 tolerance (their operation order already differs from the
// reference's per-step fold), so their complex products use fused multiply-adds: half the
// FP64 instructions of the separately rounded form, never less accurate.  Products by exactly
// 0, +-1, +-i stay exact.
__device__ __forceinline__ double2 cmul_f(double2 v, double2 x) {
    return make_double2(fma(v.x, x.x, -v.y * x.y), fma(v.x, x.y, v.y * x.x));
}
__device__ __forceinline__ double2 cmul2_f(double2 a, double2 x0, double2 b, double2 x1) {
    return make_double2(fma(a.x, x0.x, fma(-a.y, x0.y, fma(b.x, x1.x, -b.y * x1.y))),
                        fma(a.x, x0.y, fma(a.y, x0.x, fma(b.x, x1.y, b.y * x1.x))));
}

// One-target gate as a dense 2x2 on the register pairs along bit T; `en` = the registers whose
// tile-local controls hold (0xff without controls).  One straight-line form for every gate keeps
// the register allocation of the round loop free of per-kind copies.
template <int T, bool CTRL>
__device__ __forceinline__ void gate1(double2 (&v)[8], const double2* c, unsigned en) {
    const double2 a0 = c[0], b0 = c[1], a1 = c[2], b1 = c[3];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        if (q & (1 << T)) continue;
        const double2 x0 = v[q], x1 = v[q | (1 << T)];
        const double2 n0 = cmul2_f(a0, x0, b0, x1), n1 = cmul2_f(a1, x0, b1, x1);
        const bool on = !CTRL || ((en >> q) & 1u);
        v[q] = on ? n0 : x0;
        v[q | (1 << T)] = on ? n1 : x1;
    }
}

// Apply and clear the pending +-1 flips (bit q of negacc: negate register q) by xor of the sign
// bits: straight-line, so the round loop keeps one register assignment.
template <int NG>
__device__ __forceinline__ void flip_signs(double2 (&v)[NG][8], unsigned (&negacc)[NG]) {
#pragma unroll
    for (int r = 0; r < NG; ++r) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const long long m = (long long)((negacc[r] >> q) & 1u) << 63;
            v[r][q] = make_double2(__longlong_as_double(__double_as_longlong(v[r][q].x) ^ m),
                                   __longlong_as_double(__double_as_longlong(v[r][q].y) ^ m));
        }
        negacc[r] = 0;
    }
}

template <int B>
__device__ __forceinline__ void butterfly(double2 (&v)[8]) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        if (q & (1 << B)) continue;
        const double2 a = v[q], b = v[q | (1 << B)];
        v[q] = make_double2(a.x + b.x, a.y + b.y);
        v[q | (1 << B)] = make_double2(a.x - b.x, a.y - b.y);
    }
}

// Diagonal phase: entry index g from up to three basis bits; bits held in registers vary with
// q, the others are constant over the thread's group (taken from the group's first element).
// One-bit diagonal on register bit T: entry 0 on the registers with bit T clear, entry 1 on the
// others; an entry that is exactly 1 (skip bit) is not applied.
template <int T>
__device__ __forceinline__ void diag_reg(double2 (&v)[8], double2 c0, double2 c1, unsigned skip) {
    if (!(skip & 1u)) {
#pragma unroll
        for (int q = 0; q < 8; ++q)
            if (!(q >> T & 1)) v[q] = cmul_f(c0, v[q]);
    }
    if (!(skip & 2u)) {
#pragma unroll
        for (int q = 0; q < 8; ++q)
            if (q >> T & 1) v[q] = cmul_f(c1, v[q]);
    }
}

__device__ __forceinline__ void diag_op(double2 (&v)[8], const RegOp& o, const TileOp* big, u64 g0) {
    const int dk = o.dk;
    if (dk == 1) {  // S, T, RZ, phase gates: no per-register entry selection
        const unsigned skip = o.dskip;
        if (o.dreg[0] == 0xff) {  // the bit is constant over the group: one entry for all 8
            const int g = int((g0 >> o.dpos[0]) & 1);
            if (skip >> g & 1) return;
            const double2 d = g ? o.c[1] : o.c[0];
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = cmul_f(d, v[q]);
            return;
        }
        const int rb = o.dreg[0];
        if (rb == 0) diag_reg<0>(v, o.c[0], o.c[1], skip);
        else if (rb == 1) diag_reg<1>(v, o.c[0], o.c[1], skip);
        else diag_reg<2>(v, o.c[0], o.c[1], skip);
        return;
    }
    if (dk <= 2) {  // the host tabulated the register part of g for every q (2 bits each)
        int cg = 0;
        if (o.dreg[0] == 0xff && dk >= 1) cg |= int((g0 >> o.dpos[0]) & 1) << (dk - 1);
        if (dk == 2 && o.dreg[1] == 0xff) cg |= int((g0 >> o.dpos[1]) & 1);
        const unsigned tab = o.dtab, skip = o.dskip;
        const double2 c0 = o.c[0], c1 = o.c[1], c2 = o.c[2], c3 = o.c[3];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int g = cg | int((tab >> (2 * q)) & 3u);
            double2 d = c0;
            if (g == 1) d = c1;
            if (g == 2) d = c2;
            if (g == 3) d = c3;
            const double2 r = cmul_f(d, v[q]);
            if (!(skip >> g & 1)) v[q] = r;
        }
        return;
    }
    int cg = 0;
    int regbit[3] = {-1, -1, -1};
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        if (i >= dk) break;
        const int sh = dk - 1 - i;
        if (o.dreg[i] < 3) regbit[i] = o.dreg[i];
        else cg |= int((g0 >> o.dpos[i]) & 1) << sh;
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        int g = cg;
#pragma unroll
        for (int i = 0; i < 3; ++i)
            if (i < dk && regbit[i] >= 0) g |= ((q >> regbit[i]) & 1) << (dk - 1 - i);
        if (o.dskip >> g & 1) continue;
        double2 d;
        if (dk < 3) {  // select among the four entries in registers (no dynamic indexing)
            d = o.c[0];
            if (g == 1) d = o.c[1];
            if (g == 2) d = o.c[2];
            if (g == 3) d = o.c[3];
        } else {
            d = big[o.ref].val[0][g];
        }
        v[q] = cmul_f(d, v[q]);
    }
}

// Gates on 2 or 3 targets, straight on shared memory (rare: after control peeling the catalog
// leaves only Swap-like and 4x4/8x8 dense gates here).
template <int K>
__device__ __noinline__ void smem_gate(double2* sm, const TileOp& o, int m, unsigned stride) {
    constexpr int NM = 1 << K;
    int asc[K];
#pragma unroll
    for (int i = 0; i < K; ++i) asc[i] = o.tl[K - 1 - i];
    const unsigned ngroups = 1u << (m - K);
    for (unsigned g = threadIdx.x; g < ngroups; g += stride) {
        unsigned lb = g;
#pragma unroll
        for (int i = 0; i < K; ++i) lb = insert_zero(lb, asc[i]);
        if (o.lctrl_mask && (lb & o.lctrl_mask) != o.lctrl_val) continue;
        unsigned pos[NM];
        double2 x[NM];
#pragma unroll
        for (int mm = 0; mm < NM; ++mm) {
            unsigned j = lb;
#pragma unroll
            for (int i = 0; i < K; ++i)
                if (mm >> (K - 1 - i) & 1) j |= 1u << o.tl[i];
            pos[mm] = swz(j);
            x[mm] = sm[pos[mm]];
        }
        double2 out[NM];
#pragma unroll
        for (int r = 0; r < NM; ++r) {
            if (r < o.nrows) {
                double2 acc = make_double2(0.0, 0.0);
#pragma unroll
                for (int z = 0; z < NM; ++z) {
                    if (z < o.nnz[r]) {
                        const int cm = o.col_member[r][z];
                        double2 xv = x[0];
#pragma unroll
                        for (int mm = 1; mm < NM; ++mm)
                            if (cm == mm) xv = x[mm];
                        acc = madd(acc, o.val[r][z], xv);
                    }
                }
                out[r] = acc;
            }
        }
#pragma unroll
        for (int r = 0; r < NM; ++r) {
            if (r < o.nrows) {
                unsigned p = pos[0];
#pragma unroll
                for (int mm = 1; mm < NM; ++mm)
                    if (o.row_member[r] == mm) p = pos[mm];
                sm[p] = out[r];
            }
        }
    }
}

constexpr int kThreads = 256;
// gate/diagonal passes: groups per thread in the register rounds, and the resident-tile
// target that sets their register budget (compile-time tuning knobs)
#ifndef QCS_TILE_NG
#define QCS_TILE_NG 1
#endif
#ifndef QCS_TILE_MINB
#define QCS_TILE_MINB 3
#endif
#ifndef QCS_TILE_TMA  // tiles move as one tensor-map TMA box where the bit layout allows
#define QCS_TILE_TMA 1
#endif
#ifndef QCS_TILE_BITS  // tile size (log2 amplitudes): 12 = 64 KB of shared memory per tile
#define QCS_TILE_BITS 12
#endif
constexpr int kMaxBits = QCS_TILE_BITS;

enum : unsigned { F_GATE = 1, F_DIAG = 2, F_SIGN = 4, F_SMEM = 8 };

// dynamic shared memory: 1 KB alignment slack, the tile, its run offsets (>= 16 bytes), mbarrier
constexpr std::size_t tile_smem(int m) {
    return 1024 + (std::size_t(1) << m) * 16 + std::max<std::size_t>(16, (std::size_t(1) << (m - 3)) * 8) + 16;
}

// F: the operation kinds present in the pass (the host picks the instantiation), so a pass
// without gates or diagonals compiles to the lean butterfly/sign kernel.
template <unsigned F>
// butterfly / sign-only passes are lean enough for 3 resident tiles per SM (the smem limit);
// passes with gates or diagonals: QCS_TILE_MINB resident tiles (3 measured best on B200: C4
// 1.74 -> 1.42 s, C5-shaped 3.52 -> 3.08 s; 80 registers, no spills); passes with shared-memory
// gate rounds (a non-inlined call) keep 2 tiles and 128 registers
__global__ void __launch_bounds__(kThreads, (F & F_SMEM) ? 2 : (F & (F_GATE | F_DIAG)) ? QCS_TILE_MINB : 3)
    k_tile(double2* __restrict__ a, const __grid_constant__ PassParams P, const TileOp* __restrict__ big,
           const u64* __restrict__ flipped, const u64* __restrict__ tables, const __grid_constant__ CUtensorMap tmap) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const int m = P.m;
    const unsigned sz = 1u << m;
    const unsigned ngroups = sz >> 3;  // 8 amplitudes per group
    // 1024-byte aligned tile (the TMA 128-byte swizzle repeats every 1 KB), then the run offsets
    // and the tile's mbarrier
    // (offset from smem_raw, not an integer-cast pointer: keeps the accesses in the shared space)
    const unsigned align_pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
    double2* sm = reinterpret_cast<double2*>(smem_raw + align_pad);
    u64* hi_tab = reinterpret_cast<u64*>(sm + sz);  // basis offset of local bits 3..m-1 (host table)
    auto* bar = reinterpret_cast<unsigned long long*>(hi_tab + (ngroups < 2 ? 2 : ngroups));
    const unsigned t = threadIdx.x, bt = blockDim.x;
    for (unsigned j = 2 * t; j < ngroups; j += 2 * bt) cp_async16(hi_tab + j, tables + P.hi_off + j);
    // basis offset of the tile: its index deposited into the bits outside the tile (host-listed runs)
    u64 base = 0;
    {
        u64 tile = P.list_cnt ? __ldg(tables + P.list_off + blockIdx.x) : u64(blockIdx.x);
        for (int i = 0; i < P.nruns; ++i) {
            base |= (tile & ((u64(1) << P.run_len[i]) - 1)) << P.run_pos[i];
            tile >>= P.run_len[i];
        }
    }
    // sign steps whose listed indices miss this tile act uniformly (negate all or nothing):
    // decide that once per tile (bit s = sign op s has a listed index inside the tile)
    unsigned sign_hit = 0;
    if (F & F_SIGN) {
        u64 tile_mask = 0;
        for (int b = 0; b < m; ++b) tile_mask |= u64(1) << P.bits[b];
        for (int oi = 0; oi < P.nops; ++oi) {
            const RegOp& o = P.ops[oi];
            if ((o.kind & KF_KIND) != TOP_SIGN) continue;
            const TileOp& so = big[o.ref];
            bool hit = so.flip_cnt > 64;  // long lists: search per element
            for (u64 e = 0; e < so.flip_cnt && !hit; ++e) hit = (__ldg(flipped + so.flip_off + e) & ~tile_mask) == base;
            if (hit) sign_hit |= 1u << (o.sidx & 31);
        }
    }
    // tiles no sign step reaches run the pass's simplified program (or nothing at all)
    int rb = 0, re = P.nrounds;
    if ((F & F_SIGN) && P.alt_mode != ALT_NONE && sign_hit == 0) {
        if (P.alt_mode == ALT_SKIP) return;  // the pass is the identity here: no HBM traffic
        rb = P.alt_begin;
        re = rb + P.alt_nrounds;
    }
    // TMA: the tile is one box of the host's tensor map over the state; the coordinates of the
    // bit runs outside the tile come from the tile base (runs inside start at 0)
    int tc[5] = {0, 0, 0, 0, 0};
    if (P.tma_rank) {
        for (int d = 1; d < P.tma_rank; ++d)
            if (P.tma_gap_len[d]) tc[d] = int((base >> P.tma_gap_pos[d]) & ((u64(1) << P.tma_gap_len[d]) - 1));
        if (t == 0) {
            mbar_init(bar);
            mbar_expect_tx(bar, sz * 16u);
            tma_load(sm, &tmap, tc, P.tma_rank, bar);
        }
    }
    cp_async_wait_all();  // the run-offset table
    __syncthreads();
    if (P.tma_rank) {
        mbar_wait0(bar);
    } else {
        // j = t + k * bt: with bt a power of two >= 8, the run offset splits into the thread part
        // hi_tab[t >> 3] and the CTA-uniform part hi_tab[k * bt / 8] (deposit is linear on disjoint bits)
        if (t < sz) {
            const u64 gt = base | (t & 7u) | hi_tab[t >> 3];
            const unsigned rs = bt >> 3;
            for (unsigned j = t, k = 0; j < sz; j += bt, k += rs) cp_async16(sm + swz(j), a + (gt | hi_tab[k]));
        }
        cp_async_wait_all();
        __syncthreads();
    }
    for (int ri = rb; ri < re; ++ri) {
        const RoundDesc& R = P.rounds[ri];
        if ((F & F_SMEM) && (R.flags & RD_SMEM)) {
            for (int oi = R.op_begin; oi < R.op_begin + R.op_count; ++oi) {
                const TileOp& o = big[P.ops[oi].ref];
                if (!(o.gctrl_mask && (base & o.gctrl_mask) != o.gctrl_val)) {
                    if (o.gcase == 2) smem_gate<2>(sm, o, m, bt);
                    else smem_gate<3>(sm, o, m, bt);
                }
                __syncthreads();
            }
            continue;
        }
        const int r0 = R.r[0], r1 = R.r[1], r2 = R.r[2];
        const unsigned ro[3] = {1u << r0, 1u << r1, 1u << r2};
        unsigned off[8], soff[8];  // register q's local offset, and its swizzled form
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            off[q] = ((q & 1) ? ro[0] : 0u) | ((q & 2) ? ro[1] : 0u) | ((q & 4) ? ro[2] : 0u);
            soff[q] = swz(off[q]);  // swz is xor-linear: swz(lb | off) = swz(lb) ^ swz(off)
        }
        // NG groups per thread at once: gate-heavy passes are FP64/issue bound, and two
        // independent register groups per operation halve the per-operation dispatch cost
        constexpr int NG = (F & (F_GATE | F_DIAG)) ? QCS_TILE_NG : 1;
        for (unsigned gb = t; gb < ngroups; gb += NG * bt) {
            unsigned lb[NG];
            bool ok[NG];
            u64 g0[NG];
            unsigned negacc[NG];
            double2 v[NG][8];
#pragma unroll
            for (int r = 0; r < NG; ++r) {
                const unsigned g = gb + unsigned(r) * bt;
                ok[r] = g < ngroups;
                lb[r] = insert_zero(insert_zero(insert_zero(ok[r] ? g : gb, r0), r1), r2);
                const unsigned slb = swz(lb[r]);
#pragma unroll
                for (int q = 0; q < 8; ++q) v[r][q] = sm[slb ^ soff[q]];
                g0[r] = base | (lb[r] & 7u) | hi_tab[lb[r] >> 3];  // basis index of register 0
                negacc[r] = 0;  // pending sign flips of the +-1 diagonals (they commute)
            }
            for (int oi = R.op_begin; oi < R.op_begin + R.op_count; ++oi) {
                const RegOp& o = P.ops[oi];
                const int kb = o.kind;  // low bits: kind; KF_GCTRL: controls outside the tile
                if ((F & F_DIAG) && (kb & KF_FLUSH)) flip_signs<NG>(v, negacc);  // before a butterfly / gate
                if ((kb & KF_GCTRL) && (base & o.gctrl_mask) != o.gctrl_val) continue;
                if ((F & F_DIAG) && (kb & KF_SIGNED) && (kb & KF_BUNDLE)) {
                    const auto* e = reinterpret_cast<const SignEntry*>(P.pool + o.ref);
                    const int ne = o.t;
                    const unsigned cst = o.smask & 0xffu;
#pragma unroll
                    for (int r = 0; r < NG; ++r) {
                        unsigned acc = cst;
                        for (int i = 0; i < ne; ++i) {
                            const unsigned sm_ = e[i].smask, cmk = e[i].cmask, dk = e[i].dk;
                            int cg = 0;
                            if (cmk & 1u) cg |= int((g0[r] >> e[i].p0) & 1) << (dk - 1);
                            if (cmk & 2u) cg |= int((g0[r] >> e[i].p1) & 1);
                            acc ^= (sm_ >> (8 * cg)) & 0xffu;
                        }
                        negacc[r] ^= acc;
                    }
                    continue;
                }
                if ((F & F_DIAG) && (kb & KF_SIGNED)) {
                    // +-1 diagonal: the host tabulated, for each value of the bits that are
                    // constant over the group, which registers flip (one byte per value)
                    const int dk = o.dk, p0 = o.dpos[0], p1 = o.dpos[1];
                    const bool c0 = o.dreg[0] == 0xff, c1 = dk == 2 && o.dreg[1] == 0xff;
                    const unsigned sm_ = o.smask;
#pragma unroll
                    for (int r = 0; r < NG; ++r) {
                        int cg = 0;
                        if (c0) cg |= int((g0[r] >> p0) & 1) << (dk - 1);
                        if (c1) cg |= int((g0[r] >> p1) & 1);
                        negacc[r] ^= (sm_ >> (8 * cg)) & 0xffu;
                    }
                    continue;
                }
                const int kind = kb & KF_KIND;
                if (kind == TOP_WHT) {
                    const int tm = o.t;
#pragma unroll
                    for (int r = 0; r < NG; ++r) {
                        if (tm & 1) butterfly<0>(v[r]);
                        if (tm & 2) butterfly<1>(v[r]);
                        if (tm & 4) butterfly<2>(v[r]);
                    }
                } else if (kind == TOP_SCALE) {
                    const double sc = o.c[0].x;
#pragma unroll
                    for (int r = 0; r < NG; ++r)
#pragma unroll
                        for (int q = 0; q < 8; ++q) v[r][q] = make_double2(v[r][q].x * sc, v[r][q].y * sc);
                } else if ((F & F_GATE) && kind == TOP_GATE && (kb & KF_BUNDLE)) {
                    const int tm = o.t;
                    const double2* pc = P.pool + o.ref;
#pragma unroll
                    for (int r = 0; r < NG; ++r) {
                        if (tm & 1) gate1<0, false>(v[r], pc, 0xffu);
                        if (tm & 2) gate1<1, false>(v[r], pc + 4, 0xffu);
                        if (tm & 4) gate1<2, false>(v[r], pc + 8, 0xffu);
                    }
                } else if ((F & F_GATE) && kind == TOP_GATE) {
                    const int tt = o.t;
                    const unsigned cm = o.lctrl_mask, cv = o.lctrl_val;
#pragma unroll
                    for (int r = 0; r < NG; ++r) {
                        if (cm) {
                            unsigned en = 0;
#pragma unroll
                            for (int q = 0; q < 8; ++q) en |= unsigned(((lb[r] | off[q]) & cm) == cv) << q;
                            if (tt == 0) gate1<0, true>(v[r], o.c, en);
                            else if (tt == 1) gate1<1, true>(v[r], o.c, en);
                            else gate1<2, true>(v[r], o.c, en);
                        } else {
                            if (tt == 0) gate1<0, false>(v[r], o.c, 0xffu);
                            else if (tt == 1) gate1<1, false>(v[r], o.c, 0xffu);
                            else gate1<2, false>(v[r], o.c, 0xffu);
                        }
                    }
                } else if ((F & F_DIAG) && kind == TOP_DIAG) {
#pragma unroll
                    for (int r = 0; r < NG; ++r) diag_op(v[r], o, big, g0[r]);
                } else if ((F & F_SIGN) && kind == TOP_SIGN) {
                    const TileOp& so = big[o.ref];
#pragma unroll
                    for (int r = 0; r < NG; ++r) {
                        if (!(sign_hit >> (o.sidx & 31) & 1)) {
                            if (so.flip_rest) {
#pragma unroll
                                for (int q = 0; q < 8; ++q) v[r][q] = neg_exact(v[r][q]);
                            }
                        } else {
                            const u64* f = flipped + so.flip_off;
#pragma unroll
                            for (int q = 0; q < 8; ++q) {
                                const unsigned j = lb[r] | off[q];
                                const u64 gi = base | (j & 7u) | hi_tab[j >> 3];
                                if (listed(f, so.flip_cnt, gi) != (so.flip_rest != 0)) v[r][q] = neg_exact(v[r][q]);
                            }
                        }
                    }
                }
            }
            if ((F & F_DIAG) && (R.flags & RD_SIGNS)) flip_signs<NG>(v, negacc);
#pragma unroll
            for (int r = 0; r < NG; ++r) {
                if (!ok[r]) continue;
#pragma unroll
                for (int q = 0; q < 8; ++q) sm[swz(lb[r]) ^ soff[q]] = v[r][q];
            }
        }
        __syncthreads();
    }
    if (P.tma_rank) {  // the tile back as one TMA box
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncthreads();
        if (t == 0) tma_store(&tmap, tc, P.tma_rank, sm);
    } else if (t < sz) {
        const u64 gt = base | (t & 7u) | hi_tab[t >> 3];
        const unsigned rs = bt >> 3;
        for (unsigned j = t, k = 0; j < sz; j += bt, k += rs) __stcs(a + (gt | hi_tab[k]), sm[swz(j)]);
    }
}

template <unsigned F>
void launch_f(double2* amps, const PassParams& p, const TileOp* big_dev, const std::uint64_t* flipped_dev, unsigned tiles,
              const std::uint64_t* tables_dev, const CUtensorMap& tmap, int threads, std::size_t smem, cudaStream_t st) {
    static bool attr_set[64] = {};  // per device and instantiation
    int dev = 0;
    QCS_CUDA(cudaGetDevice(&dev));
    if (dev < 64 && !attr_set[dev]) {
        QCS_CUDA(cudaFuncSetAttribute(k_tile<F>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(tile_smem(kMaxBits))));
        QCS_CUDA(cudaFuncSetAttribute(k_tile<F>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        attr_set[dev] = true;
    }
    k_tile<F><<<tiles, threads, smem, st>>>(amps, p, big_dev, flipped_dev, tables_dev, tmap);
}

// The tensor map that moves a pass's tile as one TMA box: the state as <= 5 dims in ascending
// bit order -- the 8 amplitudes of bits 0..2 (16 doubles, 128 bytes, swizzled like swz), then
// each run of tile bits (<= 8 bits per dim: box = the whole run) and each run of other bits
// (box 1, the coordinate selects the tile).  False when the bit layout needs more dims.
bool tile_tensor_map(double2* amps, int n, PassParams& p, CUtensorMap* map) {
    using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static Encode encode = nullptr;
    static bool looked = false;
    if (!looked) {
        looked = true;
        cudaDriverEntryPointQueryResult q{};
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            encode = reinterpret_cast<Encode>(fn);
        else
            cudaGetLastError();
    }
    if (!encode || n > 36 || p.m < 3) return false;
    u64 tile = 0;
    for (int b = 0; b < p.m; ++b) tile |= u64(1) << p.bits[b];
    cuuint64_t gdim[5], gstride[4];
    cuuint32_t box[5], estr[5] = {1, 1, 1, 1, 1};
    int rank = 1;
    gdim[0] = 16;
    box[0] = 16;
    std::uint8_t gpos[5] = {}, glen[5] = {};
    for (int b = 3; b < n;) {
        const bool in = tile >> b & 1;
        int e = b;
        while (e < n && bool(tile >> e & 1) == in) ++e;
        for (int c = b; c < e;) {
            const int len = in ? std::min(8, e - c) : e - c;
            if (rank >= 5 || (!in && len > 31)) return false;
            gdim[rank] = cuuint64_t(1) << len;
            box[rank] = in ? cuuint32_t(1) << len : 1;
            gstride[rank - 1] = cuuint64_t(16) << c;
            gpos[rank] = std::uint8_t(in ? 0 : c);
            glen[rank] = std::uint8_t(in ? 0 : len);
            ++rank;
            c += len;
        }
        b = e;
    }
    if (rank < 2) {  // a 3-bit state: one more (unit) dim keeps the 2d..5d forms
        gdim[1] = 1;
        box[1] = 1;
        gstride[0] = 128;
        rank = 2;
    }
    if (encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, cuuint32_t(rank), amps, gdim, gstride, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    p.tma_rank = rank;
    for (int d = 0; d < 5; ++d) {
        p.tma_gap_pos[d] = gpos[d];
        p.tma_gap_len[d] = glen[d];
    }
    return true;
}

}  // namespace

int tile_max_bits() { return kMaxBits; }

void launch_tile_pass(double2* amps, int n, PassParams& p, const TileOp* big_dev, const std::uint64_t* flipped_dev,
                      const std::uint64_t* tables_dev, cudaStream_t st) {
    if (p.m < 3 || p.m > kMaxBits || p.m > n) raise(QCS_ERR_ARG, "tile bits out of range");
    const std::size_t smem = tile_smem(p.m);
    CUtensorMap tmap{};
    p.tma_rank = 0;
    if (QCS_TILE_TMA) tile_tensor_map(amps, n, p, &tmap);
    const u64 tiles = p.list_cnt ? u64(p.list_cnt) : u64(1) << (n - p.m);
    if (tiles > 0x7fffffffull) raise(QCS_ERR_CAPACITY, "too many tiles for one launch");
    const int threads = std::min(kThreads, std::max(32, 1 << (p.m - 3)));
    unsigned f = 0;
    for (int r = 0; r < p.nrounds; ++r)
        if (p.rounds[r].flags & RD_SMEM) f |= F_SMEM;
    for (int i = 0; i < p.nops; ++i) {
        const int kind = p.ops[i].kind & KF_KIND;
        if (kind == TOP_GATE) f |= F_GATE;
        if (kind == TOP_DIAG) f |= F_DIAG;
        if (kind == TOP_SIGN) f |= F_SIGN;
    }
    TimedLaunch tl("tile_pass", 32.0 * double(tiles) * double(1u << p.m), st);
    switch (f) {
#define QCS_TILE_CASE(x) \
    case x: launch_f<x>(amps, p, big_dev, flipped_dev, unsigned(tiles), tables_dev, tmap, threads, smem, st); break;
        QCS_TILE_CASE(0) QCS_TILE_CASE(1) QCS_TILE_CASE(2) QCS_TILE_CASE(3) QCS_TILE_CASE(4) QCS_TILE_CASE(5)
        QCS_TILE_CASE(6) QCS_TILE_CASE(7) QCS_TILE_CASE(8) QCS_TILE_CASE(9) QCS_TILE_CASE(10) QCS_TILE_CASE(11)
        QCS_TILE_CASE(12) QCS_TILE_CASE(13) QCS_TILE_CASE(14) QCS_TILE_CASE(15)
#undef QCS_TILE_CASE
        default: raise(QCS_ERR_SIM, "internal: no tile kernel for this operation mix");
    }
    check_launch("k_tile");
}

}  // namespace qcs
