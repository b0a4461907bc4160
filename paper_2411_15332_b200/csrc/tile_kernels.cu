// tile_kernels.cu -- fused shared-memory passes (sm_100a): the interpreter kernel and the launch.
//
// The building blocks (tile load/store, gate forms, diagonals) live in tile_device.cuh; passes
// with enough work run a kernel specialised to their operation list instead (jit.cpp).
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
#include <cmath>
#include <cstdint>

#include <cuda.h>

#include "common.hpp"
#include "kernels.hpp"
#include "tile_device.cuh"

namespace qcs {
namespace {

using namespace tile;

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
static_assert(sizeof(TmapParam) == sizeof(CUtensorMap), "tensor map bytes");

// F: the operation kinds present in the pass (the host picks the instantiation), so a pass
// without gates or diagonals compiles to the lean butterfly/sign kernel.
template <unsigned F>
// butterfly / sign-only passes are lean enough for 3 resident tiles per SM (the smem limit);
// passes with gates or diagonals: QCS_TILE_MINB resident tiles (3 measured best on B200: C4
// 1.74 -> 1.42 s, C5-shaped 3.52 -> 3.08 s; 80 registers, no spills); passes with shared-memory
// gate rounds (a non-inlined call) keep 2 tiles and 128 registers
__global__ void __launch_bounds__(kThreads, (F & F_SMEM) ? 2 : (F & (F_GATE | F_DIAG)) ? QCS_TILE_MINB : 3)
    k_tile(double2* __restrict__ a, const __grid_constant__ PassParams P, const TileOp* __restrict__ big,
           const u64* __restrict__ flipped, const u64* __restrict__ tables, const __grid_constant__ TmapParam tmap) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    TileCtx c;
    if (!tile_begin<F>(a, P, big, flipped, tables, tmap, smem_raw, c)) return;
    double2* const sm = c.sm;
    const u64* const hi_tab = c.hi_tab;
    const u64 base = c.base;
    const unsigned sign_hit = c.sign_hit;
    const int rb = c.rb, re = c.re, m = P.m;
    const unsigned t = threadIdx.x, bt = blockDim.x, ngroups = (1u << m) >> 3;
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
                        if (kb & KF_REAL) {
                            if (tm & 1) gate1r<0, false>(v[r], pc, 0xffu);
                            if (tm & 2) gate1r<1, false>(v[r], pc + 4, 0xffu);
                            if (tm & 4) gate1r<2, false>(v[r], pc + 8, 0xffu);
                        } else {
                            if (tm & 1) gate1<0, false>(v[r], pc, 0xffu);
                            if (tm & 2) gate1<1, false>(v[r], pc + 4, 0xffu);
                            if (tm & 4) gate1<2, false>(v[r], pc + 8, 0xffu);
                        }
                    }
                } else if ((F & F_GATE) && kind == TOP_GATE) {
                    const int tt = o.t;
                    const unsigned cm = o.lctrl_mask, cv = o.lctrl_val;
#pragma unroll
                    for (int r = 0; r < NG; ++r) {
                        unsigned en = 0xffu;
                        if (cm) {
                            en = 0;
#pragma unroll
                            for (int q = 0; q < 8; ++q) en |= unsigned(((lb[r] | off[q]) & cm) == cv) << q;
                        }
                        if (kb & KF_REAL) {
                            if (tt == 0) gate1r<0, true>(v[r], o.c, en);
                            else if (tt == 1) gate1r<1, true>(v[r], o.c, en);
                            else gate1r<2, true>(v[r], o.c, en);
                        } else if (cm) {
                            if (tt == 0) gate1<0, true>(v[r], o.c, en);
                            else if (tt == 1) gate1<1, true>(v[r], o.c, en);
                            else gate1<2, true>(v[r], o.c, en);
                        } else {
                            if (tt == 0) gate1<0, false>(v[r], o.c, 0xffu);
                            else if (tt == 1) gate1<1, false>(v[r], o.c, 0xffu);
                            else gate1<2, false>(v[r], o.c, 0xffu);
                        }
                    }
                } else if ((F & F_DIAG) && kind == TOP_DTAB) {
                    const double2* pc = P.pool + o.ref;
                    const unsigned skip = o.dskip;
#pragma unroll
                    for (int r = 0; r < NG; ++r)
#pragma unroll
                        for (int q = 0; q < 8; ++q)
                            if (!(skip >> q & 1)) v[r][q] = cmul_f(pc[q], v[r][q]);
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
    tile_end(a, P, tmap, c);
}

template <unsigned F>
void launch_f(double2* amps, const PassParams& p, const TileOp* big_dev, const std::uint64_t* flipped_dev, unsigned tiles,
              const std::uint64_t* tables_dev, const TmapParam& tmap, int threads, std::size_t smem, cudaStream_t st) {
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
    const int iter = tile_tma_iter(n, p);
    if (iter < 0) return false;
    u64 tile = 0;
    for (int b = 0; b < p.m - iter; ++b) tile |= u64(1) << p.bits[b];
    TmaDim L[16];
    int rank = tma_layout(tile, n, L, tma_gap_dims());
    if (rank > 5) return false;
    cuuint64_t gdim[5], gstride[4];
    cuuint32_t box[5], estr[5] = {1, 1, 1, 1, 1};
    std::uint8_t gpos[5] = {}, glen[5] = {};
    for (int d = 0; d < rank; ++d) {
        if (d == 0) {  // doubles: 16 per 8 amplitudes, then the gap bits above them
            gdim[0] = cuuint64_t(2) << L[0].len;
            box[0] = 16;
        } else {
            gdim[d] = cuuint64_t(1) << L[d].len;
            box[d] = cuuint32_t(1) << L[d].inlen;
            gstride[d - 1] = cuuint64_t(16) << L[d].pos;
        }
        gpos[d] = std::uint8_t(L[d].pos);
        glen[d] = std::uint8_t(L[d].len > L[d].inlen || d == 0 ? L[d].len : 0);
    }
    if (rank < 2) {  // a 3-bit state: one more (unit) dim keeps the 2d..5d forms
        gdim[1] = 1;
        box[1] = 1;
        gstride[0] = 128;
        rank = 2;
    }
    // L2 promotion 128 B: a 256-byte promotion on a tile whose contiguous runs are 128 bytes fetches
    // the neighbouring tile's 128 bytes as well and counts on that tile's own load hitting them in
    // L2; under the persistent kernels' looser tile order that cost 3-9% extra DRAM traffic on the
    // HBM-bound C4 passes (C4 n=32: 241.0 ms with 256 B, 239.0 ms with 128 B or none; C3 / C5
    // unchanged; tools/gpu_r02av.sh).  QCS_TMA_L2PROMO = 0 / 128 / 256 overrides.
    static const int promo_env = [] { const char* v = std::getenv("QCS_TMA_L2PROMO"); return v ? std::atoi(v) : -1; }();
    const int promo = promo_env >= 0 ? promo_env : 128;
    const CUtensorMapL2promotion l2p = promo == 0     ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                                       : promo == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                                      : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    if (encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, cuuint32_t(rank), amps, gdim, gstride, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, l2p,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    p.tma_rank = rank;
    p.tma_iter = std::uint8_t(iter);
    for (int d = 0; d < 5; ++d) {
        p.tma_gap_pos[d] = gpos[d];
        p.tma_gap_len[d] = glen[d];
    }
    return true;
}

}  // namespace

int tile_max_bits() {
    // QCS_TILE_MAX_BITS (<= the compiled limit): smaller tiles for experiments (planner A/B)
    static const int bits = [] {
        const char* v = std::getenv("QCS_TILE_MAX_BITS");
        const int b = v ? std::atoi(v) : kMaxBits;
        return b >= 6 && b <= kMaxBits ? b : kMaxBits;
    }();
    return bits;
}

int tile_tma_iter(int n, const PassParams& p) {
    if (!QCS_TILE_TMA || n > 36 || p.m < 3) return -1;
    // the boxes cover the lowest m - iter local bits; the top `iter` ones are iterated (one box per
    // value, contiguous in shared memory): the fewest iterated bits that bring the map to <= 5
    // dims, with boxes of at least 64 amplitudes (1 KB)
    auto dims = [&](u64 S) { return tma_layout(S, n, nullptr, tma_gap_dims()); };
    static const bool no_iter = std::getenv("QCS_NO_TMA_ITER") != nullptr;  // A/B switch
    // at most a few big boxes: many small ones (C5's scattered tiles: 32+ boxes of 1-2 KB) were
    // slower than the per-thread cp.async tile (877 vs 819 ms per C5-family circuit at n=32)
    static const int max_iter = [] { const char* v = std::getenv("QCS_TMA_MAX_ITER"); return v ? std::atoi(v) : 2; }();
    int iter = 0;
    u64 tile = 0;
    for (int b = 0; b < p.m; ++b) tile |= u64(1) << p.bits[b];
    while (dims(tile) > 5) {
        if (no_iter || iter >= max_iter || p.m - iter - 1 < 6) return -1;
        tile &= ~(u64(1) << p.bits[p.m - 1 - iter]);
        ++iter;
    }
    return iter;
}

void tile_pass_shape(const PassParams& p, unsigned& f, unsigned& threads) {
    threads = unsigned(std::min(kThreads, std::max(32, 1 << (p.m - 3))));
    f = 0;
    for (int r = 0; r < p.nrounds; ++r)
        if (p.rounds[r].flags & RD_SMEM) f |= F_SMEM;
    for (int i = 0; i < p.nops; ++i) {
        const int kind = p.ops[i].kind & KF_KIND;
        if (kind == TOP_GATE) f |= F_GATE;
        if (kind == TOP_DIAG || kind == TOP_DTAB) f |= F_DIAG;
        if (kind == TOP_SIGN) f |= F_SIGN;
    }
}

namespace {
inline u64 tile_bits(const PassParams& p) {
    u64 t = 0;
    for (int b = 0; b < p.m; ++b) t |= u64(1) << p.bits[b];
    return t;
}
}  // namespace

void launch_tile_pass(double2* amps, int n, PassParams& p, const TileOp* big_dev, const std::uint64_t* flipped_dev,
                      const std::uint64_t* tables_dev, cudaStream_t st, void** jit_slot) {
    if (p.m < 3 || p.m > kMaxBits || p.m > n) raise(QCS_ERR_ARG, "tile bits out of range");
    const std::size_t smem = tile_smem(p.m);
    TmapParam tmap{};
    p.tma_rank = 0;
    p.tma_iter = 0;
    if (QCS_TILE_TMA) tile_tensor_map(amps, n, p, reinterpret_cast<CUtensorMap*>(&tmap));
    const u64 tiles = p.list_cnt ? u64(p.list_cnt) : u64(1) << (n - p.m);
    if (tiles > 0x7fffffffull) raise(QCS_ERR_CAPACITY, "too many tiles for one launch");
    unsigned f = 0, nthreads = 0;
    tile_pass_shape(p, f, nthreads);
    const int threads = int(nthreads);
    // algorithmic bytes: every launched tile is written (16 B per amplitude) and read (16 B) unless
    // it starts from the basis state or lies outside the support reached so far (zmask)
    const double read_frac = p.init ? 0.0 : p.zmask ? std::ldexp(1.0, -__builtin_popcountll(p.zmask)) : 1.0;
    const double active = p.smask ? std::ldexp(1.0, -__builtin_popcountll(p.smask)) : 1.0;  // not skipped
    TimedLaunch tl("tile_pass", 16.0 * active * (1.0 + read_frac) * double(tiles) * double(1u << p.m), st);
    // A pass that skips most of its tiles (smask: the tiles outside the support stay zero and
    // unwritten) launches only the ones it keeps: the runs that turn a block index into a tile
    // base leave the smask bits out, and sval is OR-ed in (base_or).  Launching all 2^(n-m) CTAs
    // to have most return at once cost ~1.4 ms per pass at n=32 (a million empty CTAs).
    static const bool no_compact = std::getenv("QCS_NO_COMPACT_LAUNCH") != nullptr;  // A/B switch
    if (p.smask && !p.list_cnt && !no_compact) {
        static thread_local PassParams q;
        q = p;
        q.nruns = 0;
        int kept = 0;
        for (int b = 0; b < n;) {
            auto out = [&](int x) { return x < n && !(tile_bits(p) >> x & 1) && !(p.smask >> x & 1); };
            if (!out(b)) {
                ++b;
                continue;
            }
            int e = b;
            while (out(e)) ++e;
            q.run_pos[q.nruns] = std::uint8_t(b);
            q.run_len[q.nruns++] = std::uint8_t(e - b);
            kept += e - b;
            b = e;
        }
        q.base_or = p.sval & p.smask;
        const u64 few = u64(1) << kept;
        if (launch_tile_pass_jit(amps, q, f, big_dev, flipped_dev, tables_dev, tmap, unsigned(few), unsigned(threads), smem,
                                 tile_smem(kMaxBits), st, jit_slot)) {
            check_launch("qcs_pass");
            return;
        }
        // (the interpreter kernels below take the full grid and skip in tile_begin)
    } else if (launch_tile_pass_jit(amps, p, f, big_dev, flipped_dev, tables_dev, tmap, unsigned(tiles), unsigned(threads), smem,
                                    tile_smem(kMaxBits), st, jit_slot)) {
        check_launch("qcs_pass");
        return;
    }
    for (int i = 0; i < p.nops; ++i)
        if (((p.ops[i].kind & KF_KIND) == TOP_GATE && (p.ops[i].kind & KF_PIVOT)) || (p.ops[i].kind & KF_KIND) == TOP_PERM)
            raise(QCS_ERR_SIM, "internal: pivoted gates and relabellings need the specialised kernel");
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
