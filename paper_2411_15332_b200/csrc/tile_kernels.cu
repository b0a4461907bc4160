// tile_kernels.cu -- fused shared-memory passes (sm_100a).
//
// A pass owns a set S of m basis-bit positions, the tile bits (S always holds bits 0..2, so
// warp accesses are 128-byte runs).  Each CTA copies the 2^m amplitudes of one tile -- the
// indices that agree outside S -- from HBM into shared memory with cp.async (16 B per
// request, every request of the tile in flight at once), runs the pass's operations, and
// streams the tile back: one HBM round trip, 32 B per amplitude, for the whole operation list.
//
// Operations execute in "rounds": in a round every thread holds 8 amplitudes in registers
// that differ exactly in three tile bits (the round bits) and applies every operation of the
// round to them; rounds are separated by one shared-memory exchange and a barrier.  Shared
// memory is XOR-swizzled (position = j ^ ((j >> 3) & 7)) so the 16-byte accesses of a round
// are bank-conflict free whichever three bits it owns.
//
// Operation kinds: a gate on up to 3 targets among the round bits (controls anywhere: on tile
// bits they are tested per element group, outside the tile once per CTA); a diagonal phase
// on up to 3 basis bits anywhere; a diagonal sign step (Grover oracle / Z0, engine.cpp:62-80);
// unnormalised Walsh-Hadamard butterflies (the RH structure, rh.cpp:92-156: scale by
// 2^{-n/2} first, then +-1 sums); a real scale.  Gate rows use dax_mvm's arithmetic
// (acc = 0; acc += v * x in ascending column order, separately rounded), so a pass holding a
// single gate reproduces the reference bit for bit.
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

// Register index q (3 bits) <-> round bits: local index = lb | (q0 << r0) | (q1 << r1) | (q2 << r2).
struct Round {
    unsigned lb;       // this thread's local base (round bits zero)
    unsigned ro[3];    // 1 << r_i
    __device__ __forceinline__ unsigned local(int q) const {
        return lb | ((q & 1) ? ro[0] : 0u) | ((q & 2) ? ro[1] : 0u) | ((q & 4) ? ro[2] : 0u);
    }
};

// One-target gate in register bit T.  The row tables are decoded once per operation into a
// 2x2 recipe: row r is untouched (identity), one product (monomial), or two products in
// ascending column order -- dax_mvm's accumulation for that row.
struct Gate1 {
    int kind[2];   // 0 untouched, 1 single product, 2 two products
    int col[2];    // column of the single product
    double2 a[2], b[2];
};

__device__ __forceinline__ Gate1 decode1(const TileOp& o) {
    Gate1 g;
    g.kind[0] = g.kind[1] = 0;
    g.col[0] = g.col[1] = 0;
    g.a[0] = g.a[1] = g.b[0] = g.b[1] = make_double2(0.0, 0.0);
#pragma unroll
    for (int r = 0; r < 2; ++r) {  // static indices only: keeps the recipe in registers
        if (r >= o.nrows) break;
        const bool hi = o.row_member[r] != 0;
        const int kind = o.nnz[r], col = o.col_member[r][0];
        const double2 a = o.val[r][0], b = kind > 1 ? o.val[r][1] : make_double2(0.0, 0.0);
        if (hi) {
            g.kind[1] = kind; g.col[1] = col; g.a[1] = a; g.b[1] = b;
        } else {
            g.kind[0] = kind; g.col[0] = col; g.a[0] = a; g.b[0] = b;
        }
    }
    return g;
}

__device__ __forceinline__ double2 row1(const Gate1& g, int r, double2 x0, double2 x1, double2 self) {
    if (g.kind[r] == 0) return self;
    if (g.kind[r] == 1) return madd(make_double2(0.0, 0.0), g.a[r], g.col[r] ? x1 : x0);
    return madd(madd(make_double2(0.0, 0.0), g.a[r], x0), g.b[r], x1);
}

template <int T>
__device__ __forceinline__ void gate_op(double2 (&v)[8], const TileOp& o, const Round& rd) {
    const Gate1 g = decode1(o);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        if (q & (1 << T)) continue;
        if (o.lctrl_mask && (rd.local(q) & o.lctrl_mask) != o.lctrl_val) continue;
        const double2 x0 = v[q], x1 = v[q | (1 << T)];
        v[q] = row1(g, 0, x0, x1, x0);
        v[q | (1 << T)] = row1(g, 1, x0, x1, x1);
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

__device__ __forceinline__ void dispatch_gate(double2 (&v)[8], const TileOp& o, const Round& rd) {
    switch (o.gcase) {  // K and the register bits of the targets, see tile_gate_case()
        case 0: gate_op<0>(v, o, rd); break;
        case 1: gate_op<1>(v, o, rd); break;
        case 2: gate_op<2>(v, o, rd); break;
        default: break;
    }
}

// Gates on 2 or 3 targets run directly on shared memory in their own round (keeps the
// register rounds small): each thread takes groups of 2^K amplitudes.
template <int K>
__device__ __noinline__ void smem_gate(double2* sm, const TileOp& o, int m, unsigned nthreads) {
    constexpr int NM = 1 << K;
    int asc[K];  // target local bits ascending (zero-insertion order)
#pragma unroll
    for (int i = 0; i < K; ++i) asc[i] = o.tl[K - 1 - i];
    const unsigned ngroups = 1u << (m - K);
    for (unsigned g = threadIdx.x; g < ngroups; g += nthreads) {
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
constexpr int kMaxBits = 12;

__global__ void __launch_bounds__(kThreads, 2)
    k_tile(double2* __restrict__ a, const __grid_constant__ TilePass p, const TileRound* __restrict__ rounds,
           const TileOp* __restrict__ ops, const u64* __restrict__ flipped) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int m = p.m;
    const unsigned sz = 1u << m;
    const unsigned nthreads = sz >> 3;  // 8 amplitudes per thread
    double2* sm = reinterpret_cast<double2*>(smem_raw);
    u64* hi_tab = reinterpret_cast<u64*>(sm + sz);  // global offset of local bits 3..m-1
    const unsigned t = threadIdx.x;
    for (unsigned j = t; j < (sz >> 3); j += blockDim.x) {
        u64 v = 0;
        for (int b = 3; b < m; ++b)
            if (j >> (b - 3) & 1) v |= u64(1) << p.bits[b];
        hi_tab[j] = v;
    }
    u64 base = blockIdx.x;
    u64 tile_mask = 0;
    for (int b = 0; b < m; ++b) {
        const int pos = p.bits[b];
        base = ((base >> pos) << (pos + 1)) | (base & ((u64(1) << pos) - 1));
        tile_mask |= u64(1) << pos;
    }
    (void)tile_mask;
    __syncthreads();
    const unsigned bt = blockDim.x;
    // load: consecutive threads take consecutive local indices (bits 0..2 are basis bits 0..2)
    for (unsigned j = t; j < sz; j += bt) cp_async16(sm + swz(j), a + (base | (j & 7u) | hi_tab[j >> 3]));
    cp_async_wait_all();
    __syncthreads();
    for (int ri = 0; ri < p.round_count; ++ri) {
        const TileRound& R = rounds[p.round_begin + ri];
        if (R.smem) {  // gates on 2-3 targets, straight on shared memory
            for (int oi = 0; oi < R.op_count; ++oi) {
                const TileOp& o = ops[R.op_begin + oi];
                if (!(o.gctrl_mask && (base & o.gctrl_mask) != o.gctrl_val)) {
                    if (o.gcase == 2) smem_gate<2>(sm, o, m, bt);
                    else smem_gate<3>(sm, o, m, bt);
                }
                __syncthreads();
            }
            continue;
        }
        for (unsigned g = t; g < nthreads; g += bt) {
            Round rd;
            unsigned lb = g;
            lb = insert_zero(lb, R.rbits[0]);
            lb = insert_zero(lb, R.rbits[1]);
            lb = insert_zero(lb, R.rbits[2]);
            rd.lb = lb;
            rd.ro[0] = 1u << R.rbits[0];
            rd.ro[1] = 1u << R.rbits[1];
            rd.ro[2] = 1u << R.rbits[2];
            double2 v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = sm[swz(rd.local(q))];
            for (int oi = 0; oi < R.op_count; ++oi) {
                const TileOp& o = ops[R.op_begin + oi];
                if (o.gctrl_mask && (base & o.gctrl_mask) != o.gctrl_val) continue;
                switch (o.kind) {
                    case TOP_GATE: dispatch_gate(v, o, rd); break;
                    case TOP_WHT:
                        if (o.wht_mask & 1) butterfly<0>(v);
                        if (o.wht_mask & 2) butterfly<1>(v);
                        if (o.wht_mask & 4) butterfly<2>(v);
                        break;
                    case TOP_SCALE:
#pragma unroll
                        for (int q = 0; q < 8; ++q) v[q] = make_double2(v[q].x * o.scale, v[q].y * o.scale);
                        break;
                    case TOP_DIAG:
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            const unsigned j = rd.local(q);
                            const u64 gi = base | (j & 7u) | hi_tab[j >> 3];
                            int gg = 0;
                            for (int i = 0; i < o.dk; ++i) gg = (gg << 1) | int((gi >> o.dpos[i]) & 1);
                            if (!o.dskip[gg]) v[q] = madd(make_double2(0.0, 0.0), o.val[0][gg], v[q]);
                        }
                        break;
                    case TOP_SIGN: {
                        const u64* f = flipped + o.flip_off;
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            const unsigned j = rd.local(q);
                            const u64 gi = base | (j & 7u) | hi_tab[j >> 3];
                            if (listed(f, o.flip_cnt, gi) != (o.flip_rest != 0)) v[q] = neg_exact(v[q]);
                        }
                        break;
                    }
                    default: break;
                }
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) sm[swz(rd.local(q))] = v[q];
        }
        __syncthreads();
    }
    for (unsigned j = t; j < sz; j += bt) __stcs(a + (base | (j & 7u) | hi_tab[j >> 3]), sm[swz(j)]);
}

}  // namespace

int tile_max_bits() { return kMaxBits; }

void launch_tile_pass(double2* amps, int n, const TilePass& p, const TileRound* rounds_dev, const TileOp* ops_dev,
                      const std::uint64_t* flipped_dev, cudaStream_t st) {
    if (p.m < 3 || p.m > kMaxBits || p.m > n) raise(QCS_ERR_ARG, "tile bits out of range");
    const std::size_t smem = (std::size_t(1) << p.m) * sizeof(double2) + (std::size_t(1) << (p.m - 3)) * sizeof(u64);
    static bool attr_set[64] = {};  // per device
    int dev = 0;
    QCS_CUDA(cudaGetDevice(&dev));
    if (dev < 64 && !attr_set[dev]) {
        const int max_smem = (1 << kMaxBits) * 16 + (1 << (kMaxBits - 3)) * 8;
        QCS_CUDA(cudaFuncSetAttribute(k_tile, cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem));
        QCS_CUDA(cudaFuncSetAttribute(k_tile, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        attr_set[dev] = true;
    }
    const u64 tiles = u64(1) << (n - p.m);
    if (tiles > 0x7fffffffull) raise(QCS_ERR_CAPACITY, "too many tiles for one launch");
    const int threads = std::min(kThreads, std::max(32, 1 << (p.m - 3)));
    TimedLaunch tl("tile_pass", 32.0 * double(u64(1) << n), st);
    k_tile<<<unsigned(tiles), threads, smem, st>>>(amps, p, rounds_dev, ops_dev, flipped_dev);
    check_launch("k_tile");
}

}  // namespace qcs
