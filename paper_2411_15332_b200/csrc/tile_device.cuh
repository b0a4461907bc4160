// tile_device.cuh -- device building blocks of the fused tile passes (sm_100a), shared by the
// interpreter kernel k_tile (tile_kernels.cu, built by nvcc) and the per-pass specialised kernels
// generated at run time (jit.cpp, built by NVRTC).  Compiles under NVRTC: no host headers.
//
// A pass owns a set S of m basis-bit positions, the tile bits (S always holds bits 0..2, so a
// tile is made of 128-byte runs).  Each CTA moves the 2^m amplitudes of one tile -- the indices
// that agree outside S -- from HBM into shared memory (tile_begin), runs the pass's operations in
// register rounds, and writes the tile back (tile_end): one HBM round trip, 32 B per amplitude,
// for the whole operation list.  Where the bit layout fits a <= 5-dim tensor map the tile moves
// as ONE TMA box each way (cp.async.bulk.tensor + mbarrier; the 128-byte TMA swizzle is exactly
// the shared-memory layout); otherwise every thread issues 16-byte cp.async copies.
//
// Shared memory is XOR-swizzled (position = j ^ ((j >> 3) & 7)) so 16-byte accesses spread over
// the banks whichever three bits a round holds in registers.
#pragma once

#include "kernels.hpp"

namespace qcs {
namespace tile {

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
__device__ __forceinline__ void tma_load(void* dst, const TmapParam* map, const int (&c)[5], int rank,
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
__device__ __forceinline__ void tma_store(const TmapParam* map, const int (&c)[5], int rank, const void* src) {
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
}
__device__ __forceinline__ void tma_store_commit_wait() {
    asm volatile("cp.async.bulk.commit_group;\ncp.async.bulk.wait_group.read 0;\n" ::: "memory");
}
// coordinate of dim d of the box at basis index g (tile bits zero): the state bits the dim spans
// (kernels.hpp tma_layout); dim 0 counts doubles, two per amplitude
__device__ __forceinline__ int tma_coord(const PassParams& P, u64 g, int d) {
    if (d >= P.tma_rank || !P.tma_gap_len[d]) return 0;
    return int(((g >> P.tma_gap_pos[d]) & ((u64(1) << P.tma_gap_len[d]) - 1)) << (d == 0 ? 1 : 0));
}
// coordinates of box i of a tile whose top `iter` local bits are iterated: the tile base with i
// deposited into those bits, read out per gap dimension
__device__ __forceinline__ void tma_box_coords(const PassParams& P, u64 base, unsigned i, int (&cc)[5]) {
    u64 g = base;
    for (int k = 0; k < int(P.tma_iter); ++k)
        if (i >> k & 1) g |= u64(1) << P.bits[P.m - int(P.tma_iter) + k];
    for (int d = 0; d < 5; ++d) cc[d] = tma_coord(P, g, d);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count = 1u) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\nfence.mbarrier_init.release.cluster;\n" ::"r"(smem_u32(bar)),
                 "r"(count)
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
template <int T, bool CTRL, int NR>
__device__ __forceinline__ void gate1(double2 (&v)[NR], const double2* c, unsigned en) {
    const double2 a0 = c[0], b0 = c[1], a1 = c[2], b1 = c[3];
#pragma unroll
    for (int q = 0; q < NR; ++q) {
        if (q & (1 << T)) continue;
        const double2 x0 = v[q], x1 = v[q | (1 << T)];
        const double2 n0 = cmul2_f(a0, x0, b0, x1), n1 = cmul2_f(a1, x0, b1, x1);
        const bool on = !CTRL || ((en >> q) & 1u);
        v[q] = on ? n0 : x0;
        v[q | (1 << T)] = on ? n1 : x1;
    }
}

// The same with real coefficients (RY, H, X, CNOT, the real factor of a phase-split gate): half
// the FP64 instructions of the complex form.
template <int T, bool CTRL, int NR>
__device__ __forceinline__ void gate1r(double2 (&v)[NR], const double2* c, unsigned en) {
    const double a0 = c[0].x, b0 = c[1].x, a1 = c[2].x, b1 = c[3].x;
#pragma unroll
    for (int q = 0; q < NR; ++q) {
        if (q & (1 << T)) continue;
        const double2 x0 = v[q], x1 = v[q | (1 << T)];
        const double2 n0 = make_double2(fma(a0, x0.x, b0 * x1.x), fma(a0, x0.y, b0 * x1.y));
        const double2 n1 = make_double2(fma(a1, x0.x, b1 * x1.x), fma(a1, x0.y, b1 * x1.y));
        const bool on = !CTRL || ((en >> q) & 1u);
        v[q] = on ? n0 : x0;
        v[q | (1 << T)] = on ? n1 : x1;
    }
}

// Pivoted form (specialised kernels, KF_PIVOT): row r = x[piv_r] + rho_r * x[other] on the
// register pairs along bit T of the registers in EN; the row scales sit in the round's table.
// NEG bit q: the pair (q, q | 1 << T) holds registers of opposite pending sign (lazy +-1 flips,
// jit.cpp SignTrack): both rows use -rho (a free operand negation in the DFMAs).
template <int T, bool P0, bool P1, bool Z0, bool Z1, bool REAL, unsigned EN, unsigned NEG = 0u, int NR>
__device__ __forceinline__ void gate1p(double2 (&v)[NR], double2 rho0_, double2 rho1_) {
#pragma unroll
    for (int q = 0; q < NR; ++q) {
        if ((q & (1 << T)) || !((EN >> q) & 1u)) continue;
        const bool ng = (NEG >> q) & 1u;
        const double2 rho0 = ng ? make_double2(-rho0_.x, -rho0_.y) : rho0_;
        const double2 rho1 = ng ? make_double2(-rho1_.x, -rho1_.y) : rho1_;
        const double2 x0 = v[q], x1 = v[q | (1 << T)];
        const double2 p0 = P0 ? x1 : x0, o0 = P0 ? x0 : x1, p1 = P1 ? x1 : x0, o1 = P1 ? x0 : x1;
        double2 n0 = p0, n1 = p1;
        if (!Z0) n0 = REAL ? make_double2(fma(rho0.x, o0.x, p0.x), fma(rho0.x, o0.y, p0.y))
                           : make_double2(fma(rho0.x, o0.x, fma(-rho0.y, o0.y, p0.x)), fma(rho0.x, o0.y, fma(rho0.y, o0.x, p0.y)));
        if (!Z1) n1 = REAL ? make_double2(fma(rho1.x, o1.x, p1.x), fma(rho1.x, o1.y, p1.y))
                           : make_double2(fma(rho1.x, o1.x, fma(-rho1.y, o1.y, p1.x)), fma(rho1.x, o1.y, fma(rho1.y, o1.x, p1.y)));
        v[q] = n0;
        v[q | (1 << T)] = n1;
    }
}

// x with its sign flipped when bit 0 of s is set (sign-bit xor: exact, no FP64 instruction)
__device__ __forceinline__ double2 flipd2(double2 x, unsigned s) {
    const long long m = (long long)(s & 1u) << 63;
    return make_double2(__longlong_as_double(__double_as_longlong(x.x) ^ m),
                        __longlong_as_double(__double_as_longlong(x.y) ^ m));
}
__device__ __forceinline__ double flipd(double x, unsigned s) {
    return __longlong_as_double(__double_as_longlong(x) ^ ((long long)(s & 1u) << 63));
}
// negate the registers in mask (bit q: register q)
template <int NR>
__device__ __forceinline__ void flip_mask(double2 (&v)[NR], unsigned mask) {
#pragma unroll
    for (int q = 0; q < NR; ++q) v[q] = flipd2(v[q], mask >> q);
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

template <int B, int NR>
__device__ __forceinline__ void butterfly(double2 (&v)[NR]) {
#pragma unroll
    for (int q = 0; q < NR; ++q) {
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
template <int T, int NR>
__device__ __forceinline__ void diag_reg(double2 (&v)[NR], double2 c0, double2 c1, unsigned skip) {
    if (!(skip & 1u)) {
#pragma unroll
        for (int q = 0; q < NR; ++q)
            if (!(q >> T & 1)) v[q] = cmul_f(c0, v[q]);
    }
    if (!(skip & 2u)) {
#pragma unroll
        for (int q = 0; q < NR; ++q)
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
enum : unsigned { F_GATE = 1, F_DIAG = 2, F_SIGN = 4, F_SMEM = 8 };

// dynamic shared memory: 1 KB alignment slack, the tile, its run offsets (>= 16 bytes), mbarrier
constexpr unsigned long tile_smem(int m) {
    return 1024ul + (1ul << m) * 16 + ((1ul << (m - 3)) * 8 > 16 ? (1ul << (m - 3)) * 8 : 16ul) + 16;
}

// negate the registers in M (a literal) when cond (0 / 1, uniform over the group) is set: one xor
// of the sign word per component
template <unsigned M, int NR>
__device__ __forceinline__ void flip_cond(double2 (&v)[NR], unsigned cond) {
    const int hm = int(cond << 31);
#pragma unroll
    for (int q = 0; q < NR; ++q)
        if ((M >> q) & 1u)
            v[q] = make_double2(__hiloint2double(__double2hiint(v[q].x) ^ hm, __double2loint(v[q].x)),
                                __hiloint2double(__double2hiint(v[q].y) ^ hm, __double2loint(v[q].y)));
}

// One group of 8 register amplitudes: apply and clear pending +-1 flips (bit q: negate register q)
template <int NR>
__device__ __forceinline__ void flip_signs1(double2 (&v)[NR], unsigned& negacc) {
#pragma unroll
    for (int q = 0; q < NR; ++q) {
        const long long m = (long long)((negacc >> q) & 1u) << 63;
        v[q] = make_double2(__longlong_as_double(__double_as_longlong(v[q].x) ^ m),
                            __longlong_as_double(__double_as_longlong(v[q].y) ^ m));
    }
    negacc = 0;
}

struct TileCtx;
__device__ __forceinline__ void tile_end(double2* a, const PassParams& P, const TmapParam& tmap, const TileCtx& c);

struct TileCtx {
    double2* sm;          // the tile (swizzled), 1 KB aligned
    u64* hi_tab;          // basis offset of local bits 3..m-1 (runs of 8), copied from the host table
    unsigned long long* bar;
    u64 base;             // basis index of the tile's first amplitude
    unsigned sign_hit;    // bit s: sign step s has a listed index inside this tile
    int rb, re;           // rounds to run: the main program or the missed-tile alternative
    int tc[5];            // TMA box coordinates
};

// Load the tile: returns false when the pass is the identity on it (ALT_SKIP, no sign step
// reaches it), and then nothing moves.
template <unsigned F>
__device__ __forceinline__ bool tile_begin(double2* a, const PassParams& P, const TileOp* big, const u64* flipped,
                                           const u64* tables, const TmapParam& tmap, unsigned char* smem_raw,
                                           TileCtx& c) {
    const int m = P.m;
    const unsigned sz = 1u << m;
    const unsigned ngroups = sz >> 3;  // 8 amplitudes per group
    // 1024-byte aligned tile (the TMA 128-byte swizzle repeats every 1 KB), then the run offsets
    // and the tile's mbarrier (offsets from smem_raw keep the accesses in the shared space)
    const unsigned align_pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
    c.sm = reinterpret_cast<double2*>(smem_raw + align_pad);
    c.hi_tab = reinterpret_cast<u64*>(c.sm + sz);
    c.bar = reinterpret_cast<unsigned long long*>(c.hi_tab + (ngroups < 2 ? 2 : ngroups));
    const unsigned t = threadIdx.x, bt = blockDim.x;
    // basis offset of the tile: its index deposited into the bits outside the tile (host-listed runs)
    u64 base = 0;
    {
        u64 tl = P.list_cnt ? __ldg(tables + P.list_off + blockIdx.x) : u64(blockIdx.x);
        for (int i = 0; i < P.nruns; ++i) {
            base |= (tl & ((u64(1) << P.run_len[i]) - 1)) << P.run_pos[i];
            tl >>= P.run_len[i];
        }
    }
    base |= P.base_or;
    c.base = base;
    // zero, and the next pass reads it as zero: nothing to do (before any asynchronous copy)
    if (P.smask && (base & P.smask) != P.sval) return false;
    for (unsigned j = 2 * t; j < ngroups; j += 2 * bt) cp_async16(c.hi_tab + j, tables + P.hi_off + j);
    // sign steps whose listed indices miss this tile act uniformly (negate all or nothing):
    // decide that once per tile
    c.sign_hit = 0;
    if (F & F_SIGN) {
        u64 tile_mask = 0;
        for (int b = 0; b < m; ++b) tile_mask |= u64(1) << P.bits[b];
        for (int oi = 0; oi < P.nops; ++oi) {
            const RegOp& o = P.ops[oi];
            if ((o.kind & KF_KIND) != TOP_SIGN) continue;
            const TileOp& so = big[o.ref];
            bool hit = so.flip_cnt > 64;  // long lists: search per element
            for (u64 e = 0; e < so.flip_cnt && !hit; ++e) hit = (__ldg(flipped + so.flip_off + e) & ~tile_mask) == base;
            if (hit) c.sign_hit |= 1u << (o.sidx & 31);
        }
    }
    // tiles no sign step reaches run the pass's simplified program (or nothing at all)
    c.rb = 0;
    c.re = P.nrounds;
    if ((F & F_SIGN) && P.alt_mode != ALT_NONE && c.sign_hit == 0) {
        if (P.alt_mode == ALT_SKIP) {  // the pass is the identity here: no HBM traffic
            cp_async_wait_all();         // (no copy may land after the CTA exits)
            return false;
        }
        c.rb = P.alt_begin;
        c.re = c.rb + P.alt_nrounds;
    }
    for (int d = 0; d < 5; ++d) c.tc[d] = tma_coord(P, base, d);
    if (P.init || (P.zmask && (base & P.zmask) != P.zval)) {
        // the pass starts from |init_index> (zeros and at most one 1), or from a tile the
        // circuit has not reached yet (zeros): nothing to load
        for (unsigned j = t; j < sz; j += bt) c.sm[j] = make_double2(0.0, 0.0);
        cp_async_wait_all();  // the run-offset table
        __syncthreads();
        u64 tile_mask = 0;
        unsigned local = 0;
        for (int b = 0; b < m; ++b) {
            tile_mask |= u64(1) << P.bits[b];
            local |= unsigned((P.init_index >> P.bits[b]) & 1) << b;
        }
        if (!(P.init && (P.init_index & ~tile_mask) == base)) {
            // zeros in, and every operation is linear: zeros out, without the rounds
            tile_end(a, P, tmap, c);
            return false;
        }
        if (t == 0) c.sm[swz(local)] = make_double2(1.0, 0.0);
        __syncthreads();
        return true;
    }
    // TMA: the tile is one box of the host's tensor map over the state; the coordinates of the
    // bit runs outside the tile come from the tile base (runs inside start at 0)
    if (P.tma_rank) {
        if (t == 0) {
            mbar_init(c.bar);
            mbar_expect_tx(c.bar, sz * 16u);
            if (!P.tma_iter) {
                tma_load(c.sm, &tmap, c.tc, P.tma_rank, c.bar);
            } else {  // one box per value of the iterated top local bits, contiguous in shared memory
                const unsigned nb = 1u << P.tma_iter, chunk = sz >> P.tma_iter;
                for (unsigned i = 0; i < nb; ++i) {
                    int cc[5];
                    tma_box_coords(P, base, i, cc);
                    tma_load(c.sm + i * chunk, &tmap, cc, P.tma_rank, c.bar);
                }
            }
        }
    }
    cp_async_wait_all();  // the run-offset table
    __syncthreads();
    if (P.tma_rank) {
        mbar_wait0(c.bar);
    } else {
        // j = t + k * bt: with bt a power of two >= 8, the run offset splits into the thread part
        // hi_tab[t >> 3] and the CTA-uniform part hi_tab[k * bt / 8] (deposit is linear on disjoint bits)
        if (t < sz) {
            const u64 gt = base | (t & 7u) | c.hi_tab[t >> 3];
            const unsigned rs = bt >> 3;
            for (unsigned j = t, k = 0; j < sz; j += bt, k += rs) cp_async16(c.sm + swz(j), a + (gt | c.hi_tab[k]));
        }
        cp_async_wait_all();
        __syncthreads();
    }
    return true;
}

// Write the tile back (after the last round's barrier).
__device__ __forceinline__ void tile_end(double2* a, const PassParams& P, const TmapParam& tmap, const TileCtx& c) {
    const unsigned t = threadIdx.x, bt = blockDim.x, sz = 1u << P.m;
    if (P.tma_rank) {  // the tile back as one TMA box
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncthreads();
        if (t == 0) {
            if (!P.tma_iter) {
                tma_store(&tmap, c.tc, P.tma_rank, c.sm);
            } else {
                const unsigned nb = 1u << P.tma_iter, chunk = sz >> P.tma_iter;
                for (unsigned i = 0; i < nb; ++i) {
                    int cc[5];
                    tma_box_coords(P, c.base, i, cc);
                    tma_store(&tmap, cc, P.tma_rank, c.sm + i * chunk);
                }
            }
            tma_store_commit_wait();
        }
    } else if (t < sz) {
        const u64 gt = c.base | (t & 7u) | c.hi_tab[t >> 3];
        const unsigned rs = bt >> 3;
        for (unsigned j = t, k = 0; j < sz; j += bt, k += rs) __stcs(a + (gt | c.hi_tab[k]), c.sm[swz(j)]);
    }
}


// ---------------------------------------------------------------- persistent pipelined passes
// One CTA per SM walks its share of the pass's tiles (tile = blockIdx.x + k * gridDim.x) through a
// ring of S shared-memory slots.  Two groups of 256 threads compute alternate tiles (group k & 1
// takes the CTA's k-th tile, in slot k % S; named barrier 1 + group), so while both groups work
// the ring's other slots are being written back and refilled by TMA: the HBM round trip of a tile
// hides behind the arithmetic of its neighbours instead of sitting between a CTA's launch and its
// first round.  The thread that issues a tile's store waits until the store has read the slot,
// then loads the CTA's (k + S)-th tile into it.  Each slot has TWO mbarriers, taken in turn by
// its uses (barrier use & 1, parity (use >> 1) & 1): with an odd ring the uses of a slot
// alternate between the groups, and a group that waits for use u + 1 on a single barrier whose
// phase u is still incomplete (the other group's tile has not landed yet) would see the
// "preceding" phase u - 1 as the one it asked for and run on a slot that is not its own.  With
// two barriers the group that waits on one has itself consumed that barrier's previous phase.
struct PersistCtx {
    double2* sm0;              // slot 0 (1 KB aligned); slot s at sm0 + (s << m)
    u64* hi_tab;               // the pass's run-offset table (as in TileCtx)
    unsigned long long* full;  // 2 S mbarriers (slot s, use parity p: full[2 s + p]): the slot's tile has landed
    u64 ntiles;
};

__device__ __forceinline__ u64 tile_base_of(const PassParams& P, u64 tl) {
    u64 base = 0;
    for (int i = 0; i < P.nruns; ++i) {
        base |= (tl & ((u64(1) << P.run_len[i]) - 1)) << P.run_pos[i];
        tl >>= P.run_len[i];
    }
    return base | P.base_or;
}
__device__ __forceinline__ void group_sync(unsigned grp) {
    asm volatile("bar.sync %0, 256;\n" ::"r"(grp + 1u) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n.reg .pred done;\nWAITP_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n"
        "@!done bra WAITP_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(parity)
        : "memory");
}
// one thread: the tile at basis offset `base` into `dst` (completes on `bar`)
__device__ __forceinline__ void tile_load_async(const PassParams& P, const TmapParam& tmap, u64 base, double2* dst,
                                                unsigned long long* bar) {
    const unsigned sz = 1u << P.m;
    mbar_expect_tx(bar, sz * 16u);
    if (!P.tma_iter) {
        int cc[5];
        for (int d = 0; d < 5; ++d) cc[d] = tma_coord(P, base, d);
        tma_load(dst, &tmap, cc, P.tma_rank, bar);
    } else {
        const unsigned nb = 1u << P.tma_iter, chunk = sz >> P.tma_iter;
        for (unsigned i = 0; i < nb; ++i) {
            int cc[5];
            tma_box_coords(P, base, i, cc);
            tma_load(dst + i * chunk, &tmap, cc, P.tma_rank, bar);
        }
    }
}
// one thread: the slot back to its tile; returns once the store has read the slot
__device__ __forceinline__ void tile_store_read(const PassParams& P, const TmapParam& tmap, u64 base, const double2* src) {
    const unsigned sz = 1u << P.m;
    if (!P.tma_iter) {
        int cc[5];
        for (int d = 0; d < 5; ++d) cc[d] = tma_coord(P, base, d);
        tma_store(&tmap, cc, P.tma_rank, src);
    } else {
        const unsigned nb = 1u << P.tma_iter, chunk = sz >> P.tma_iter;
        for (unsigned i = 0; i < nb; ++i) {
            int cc[5];
            tma_box_coords(P, base, i, cc);
            tma_store(&tmap, cc, P.tma_rank, src + i * chunk);
        }
    }
    tma_store_commit_wait();
}

// all 256 threads of a group: the tile at `base` into `dst` as 16-byte cp.async copies (tiles whose
// bit layout needs more than 5 tensor-map dims); each thread's arrival on `bar` (count 256)
// fires when its copies have landed
__device__ __forceinline__ void tile_load_coop(const PassParams& P, const double2* a, u64 base, double2* dst,
                                               const u64* hi_tab, unsigned long long* bar, unsigned t) {
    const unsigned sz = 1u << P.m;
    const u64 gt = base | (t & 7u) | hi_tab[t >> 3];
    for (unsigned j = t, k = 0; j < sz; j += 256u, k += 32u) cp_async16(dst + swz(j), a + (gt | hi_tab[k]));
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

template <unsigned S>
__device__ __forceinline__ void persist_begin(const double2* a, const PassParams& P, const u64* tables,
                                              const TmapParam& tmap, unsigned char* smem_raw, PersistCtx& c) {
    const unsigned sz = 1u << P.m, ngroups = sz >> 3;
    const unsigned align_pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
    c.sm0 = reinterpret_cast<double2*>(smem_raw + align_pad);
    c.hi_tab = reinterpret_cast<u64*>(c.sm0 + S * sz);
    c.full = reinterpret_cast<unsigned long long*>(c.hi_tab + (ngroups < 2 ? 2 : ngroups));
    int out_bits = 0;
    for (int i = 0; i < P.nruns; ++i) out_bits += P.run_len[i];
    c.ntiles = u64(1) << out_bits;
    const unsigned t = threadIdx.x, bt = blockDim.x;
    for (unsigned j = 2 * t; j < ngroups; j += 2 * bt) cp_async16(c.hi_tab + j, tables + P.hi_off + j);
    if (t == 0)
        for (unsigned s = 0; s < 2 * S; ++s) mbar_init(c.full + s, P.tma_rank ? 1u : 256u);
    cp_async_wait_all();
    __syncthreads();
    if (P.tma_rank) {
        if (t == 0)
            for (unsigned s = 0; s < S; ++s) {
                const u64 tile = blockIdx.x + u64(s) * gridDim.x;
                if (tile < c.ntiles) tile_load_async(P, tmap, tile_base_of(P, tile), c.sm0 + s * sz, c.full + 2 * s);
            }
    } else {  // the group that will compute slot s's first tile loads it
        for (unsigned s = t >> 8; s < S; s += 2) {
            const u64 tile = blockIdx.x + u64(s) * gridDim.x;
            if (tile < c.ntiles)
                tile_load_coop(P, a, tile_base_of(P, tile), c.sm0 + s * sz, c.hi_tab, c.full + 2 * s, t & 255u);
        }
    }
}

// after the group's last round on the CTA's k-th tile (in `sm`): write it back and refill the slot
// (bar: the barrier of the slot's NEXT use).  DIRECT: the last round stored its registers
// straight to HBM (relabelled passes), so the slot is free once the group has passed its barrier.
template <unsigned S, bool DIRECT>
__device__ __forceinline__ void persist_end(double2* a, const PassParams& P, const TmapParam& tmap, const PersistCtx& c,
                                            unsigned grp, unsigned t, u64 tile, u64 base, double2* sm,
                                            unsigned long long* bar) {
    const u64 next = tile + u64(S) * gridDim.x;
    if (P.tma_rank) {
        if (!DIRECT) asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        group_sync(grp);
        if (t == 0) {
            if (!DIRECT) tile_store_read(P, tmap, base, sm);
            if (next < c.ntiles) tile_load_async(P, tmap, tile_base_of(P, next), sm, bar);
        }
    } else {
        if (!DIRECT) {  // (the last round ended with the group's barrier)
            const unsigned sz = 1u << P.m;
            const u64 gt = base | (t & 7u) | c.hi_tab[t >> 3];
            for (unsigned j = t, k = 0; j < sz; j += 256u, k += 32u) __stcs(a + (gt | c.hi_tab[k]), sm[swz(j)]);
        }
        group_sync(grp);
        if (next < c.ntiles) tile_load_coop(P, a, tile_base_of(P, next), sm, c.hi_tab, bar, t);
    }
}
// before the CTA exits: every store this thread issued has read its slot (persist_end waits per
// store, so this only documents the invariant), and no cp.async of its own is in flight
__device__ __forceinline__ void persist_finish() {
    asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
    cp_async_wait_all();
}

}  // namespace tile
}  // namespace qcs
