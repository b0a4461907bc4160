// gate_kernels.cu -- single-placement gate pass, in place (sm_100a).
//
// Reference: one gates step is step_matrix_dax (engine.cpp:135-142: a 2^n-row DAX built by
// the MTP fold, dax.cpp:58-94) followed by dax_mvm (dax.cpp:96-103).  Here the operator is
// never built: each thread enumerates groups of the touched sub-cube (GateDesc), loads the
// members it needs with 16-byte streaming loads, evaluates the touched rows with dax_mvm's
// arithmetic -- acc = (0,0); acc += v * s[col] in ascending column order, products as
// (ar*br - ai*bi, ar*bi + ai*br), every operation separately rounded (the library is built
// with -fmad=false) -- and stores only those rows.  The result is bit-identical to the
// reference's for single-placement steps.  The pass is HBM-bound: 16 B read + 16 B written
// per touched amplitude, no reuse, so loads/stores carry evict-first hints and each thread
// keeps several independent groups in flight.
//
// Three kernels by group shape, kept lean in registers (occupancy is what hides HBM latency):
//   k_diag1  one member per group: a diagonal entry on a fixed sub-cube (Z, S, T, CZ, CCZ)
//   k_pair   two members: any one-target gate, controls folded into the fixed bits
//            (X, Y, H, RX, RY, U3, RZ, CNOT, CY, CH, Toffoli, ...)
//   k_gate   2-3 free bits: the generic row-table kernel (Swap, iSwap, RXX, DCX, ...)
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "common.hpp"
#include "kernels.hpp"

namespace qcs {
namespace {

using u64 = std::uint64_t;

__device__ __forceinline__ double2 ld_stream(const double2* p) { return __ldcs(p); }
__device__ __forceinline__ void st_stream(double2* p, double2 v) { __stcs(p, v); }

// dax_mvm accumulation step: acc + v * x with each operation rounded separately.
__device__ __forceinline__ double2 madd(double2 acc, double2 v, double2 x) {
    const double pr = __dsub_rn(__dmul_rn(v.x, x.x), __dmul_rn(v.y, x.y));
    const double pi = __dadd_rn(__dmul_rn(v.x, x.y), __dmul_rn(v.y, x.x));
    return make_double2(__dadd_rn(acc.x, pr), __dadd_rn(acc.y, pi));
}

// Insert zero bits at the k ascending positions: group index -> base basis index.
__device__ __forceinline__ u64 insert_zeros(u64 t, int k, const int (&pos)[3]) {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        if (i < k) {
            const int p = pos[i];
            t = ((t >> p) << (p + 1)) | (t & ((u64(1) << p) - 1));
        }
    }
    return t;
}

template <int NF>
__device__ __forceinline__ double2 pick(const double2 (&x)[1 << NF], int m) {
    double2 v = x[0];
#pragma unroll
    for (int j = 1; j < (1 << NF); ++j)
        if (m == j) v = x[j];
    return v;
}

// ---------------------------------------------------------------- one member per group
struct Diag1 {
    int k;
    int pos[3];
    u64 fixed;
    double2 d;
};

template <int ITEMS>
__global__ void __launch_bounds__(256) k_diag1(double2* __restrict__ a, u64 ngroups, const __grid_constant__ Diag1 p) {
    const u64 stride = u64(gridDim.x) * blockDim.x;
    const u64 t0 = u64(blockIdx.x) * blockDim.x + threadIdx.x;
    double2 x[ITEMS];
    u64 idx[ITEMS];
#pragma unroll
    for (int it = 0; it < ITEMS; ++it) {
        idx[it] = insert_zeros(t0 + it * stride, p.k, p.pos) | p.fixed;
        if (t0 + it * stride < ngroups) x[it] = ld_stream(a + idx[it]);
    }
#pragma unroll
    for (int it = 0; it < ITEMS; ++it)
        if (t0 + it * stride < ngroups) st_stream(a + idx[it], madd(make_double2(0.0, 0.0), p.d, x[it]));
}

// ---------------------------------------------------------------- two members per group
struct Pair {
    int k;
    int pos[3];
    u64 fixed;
    u64 off1;        // basis offset of member 1
    int load0, load1;
    int rk[2];       // row kind: 0 untouched, 1 one product (column rc), 2 two products
    int rc[2];
    double2 a[2], b[2];
};

__device__ __forceinline__ double2 pair_row(int rk, int rc, double2 a, double2 b, double2 x0, double2 x1) {
    if (rk == 1) return madd(make_double2(0.0, 0.0), a, rc ? x1 : x0);
    return madd(madd(make_double2(0.0, 0.0), a, x0), b, x1);
}

__device__ __forceinline__ void ld256(const double2* p, double2& a, double2& b) {
    asm volatile("ld.global.cs.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(a.x), "=d"(a.y), "=d"(b.x), "=d"(b.y)
                 : "l"(p));
}
__device__ __forceinline__ void st256(double2* p, double2 a, double2 b) {
    asm volatile("st.global.cs.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(a.x), "d"(a.y), "d"(b.x), "d"(b.y)
                 : "memory");
}

// ADJ: the two members are the halves of one 32-byte sector (the free bit is basis bit 0, both
// loaded and both stored): one 256-bit load and store per group.
template <int ITEMS, bool ADJ>
__global__ void __launch_bounds__(256) k_pair(double2* __restrict__ a, u64 ngroups, const __grid_constant__ Pair p) {
    const u64 stride = u64(gridDim.x) * blockDim.x;
    const u64 t0 = u64(blockIdx.x) * blockDim.x + threadIdx.x;
    double2 x0[ITEMS], x1[ITEMS];
    u64 idx[ITEMS];
#pragma unroll
    for (int it = 0; it < ITEMS; ++it) {
        idx[it] = insert_zeros(t0 + it * stride, p.k, p.pos) | p.fixed;
        if (t0 + it * stride < ngroups) {
            if (ADJ) {
                ld256(a + idx[it], x0[it], x1[it]);
            } else {
                if (p.load0) x0[it] = ld_stream(a + idx[it]);
                if (p.load1) x1[it] = ld_stream(a + (idx[it] | p.off1));
            }
        }
    }
#pragma unroll
    for (int it = 0; it < ITEMS; ++it) {
        if (t0 + it * stride >= ngroups) continue;
        if (ADJ) {
            st256(a + idx[it], pair_row(p.rk[0], p.rc[0], p.a[0], p.b[0], x0[it], x1[it]),
                  pair_row(p.rk[1], p.rc[1], p.a[1], p.b[1], x0[it], x1[it]));
            continue;
        }
        if (p.rk[0]) st_stream(a + idx[it], pair_row(p.rk[0], p.rc[0], p.a[0], p.b[0], x0[it], x1[it]));
        if (p.rk[1]) st_stream(a + (idx[it] | p.off1), pair_row(p.rk[1], p.rc[1], p.a[1], p.b[1], x0[it], x1[it]));
    }
}

// ---------------------------------------------------------------- four members, monomial rows
// Swap, iSwap, DCX, RZZ, CU1-like diagonals on two free bits: each written row is one product.
struct Quad {
    int k;
    int pos[3];
    u64 fixed;
    u64 off[4];
    int load;        // member mask to load
    int nrows;
    int row[4];      // member written by row r
    int col[4];      // member read by row r
    double2 v[4];
};

template <int ITEMS>
__global__ void __launch_bounds__(256) k_quad(double2* __restrict__ a, u64 ngroups, const __grid_constant__ Quad p) {
    const u64 stride = u64(gridDim.x) * blockDim.x;
    const u64 t0 = u64(blockIdx.x) * blockDim.x + threadIdx.x;
    double2 x[ITEMS][4];
    u64 idx[ITEMS];
#pragma unroll
    for (int it = 0; it < ITEMS; ++it) {
        idx[it] = insert_zeros(t0 + it * stride, p.k, p.pos) | p.fixed;
        if (t0 + it * stride < ngroups) {
#pragma unroll
            for (int m = 0; m < 4; ++m)
                if (p.load >> m & 1) x[it][m] = ld_stream(a + (idx[it] | p.off[m]));
        }
    }
#pragma unroll
    for (int it = 0; it < ITEMS; ++it) {
        if (t0 + it * stride >= ngroups) continue;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            if (r >= p.nrows) break;
            const int c = p.col[r];
            const double2 xv = c == 0 ? x[it][0] : c == 1 ? x[it][1] : c == 2 ? x[it][2] : x[it][3];
            st_stream(a + (idx[it] | p.off[p.row[r]]), madd(make_double2(0.0, 0.0), p.v[r], xv));
        }
    }
}

// ---------------------------------------------------------------- generic row tables
// NF: free bits per group; NNZ: max nonzeros per touched row; ITEMS: groups per thread.
template <int NF, int NNZ, int ITEMS>
__global__ void __launch_bounds__(256) k_gate(double2* __restrict__ a, u64 ngroups,
                                              const __grid_constant__ GateDesc d) {
    constexpr int NM = 1 << NF;
    const u64 stride = u64(gridDim.x) * blockDim.x;
    const u64 t0 = u64(blockIdx.x) * blockDim.x + threadIdx.x;
    double2 x[ITEMS][NM];
    u64 base[ITEMS];
#pragma unroll
    for (int it = 0; it < ITEMS; ++it) {
        const u64 g = t0 + it * stride;
        base[it] = insert_zeros(g, d.k, d.pos_asc) | d.fixed_val;
        if (g < ngroups) {
#pragma unroll
            for (int m = 0; m < NM; ++m)
                if (d.load_mask & (1u << m)) x[it][m] = ld_stream(a + (base[it] | d.member_off[m]));
        }
    }
#pragma unroll
    for (int it = 0; it < ITEMS; ++it) {
        if (t0 + it * stride >= ngroups) continue;
        double2 out[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            if (r < d.nrows) {
                double2 acc = make_double2(0.0, 0.0);
#pragma unroll
                for (int z = 0; z < NNZ; ++z)
                    if (z < d.nnz[r]) acc = madd(acc, d.val[r][z], pick<NF>(x[it], d.col_member[r][z]));
                out[r] = acc;
            }
        }
#pragma unroll
        for (int r = 0; r < 8; ++r)
            if (r < d.nrows) st_stream(a + (base[it] | d.member_off[d.row_member[r]]), out[r]);
    }
}

// role of basis bit 0 in a group: -2 fixed gate bit, >= 0 free member bit, -1 not a gate bit
int bit0_role(const GateDesc& d) {
    int b0 = -1;
    for (int i = 0; i < d.k; ++i)
        if (d.pos_asc[i] == 0) b0 = -2;
    for (int i = 0; i < d.nfree; ++i)
        if (d.free_bit[i] == 1) b0 = i;
    return b0;
}

// Algorithmic HBM bytes of one pass: 16 B per member read and per row written, counted per
// 32-byte sector -- a touched amplitude whose basis-bit-0 mate is untouched costs the whole
// sector (SURVEY.md section 8d sector rounding).
double algorithmic_bytes(int n, const GateDesc& d) {
    const double groups = double(u64(1) << (n - d.k));
    const int b0 = bit0_role(d);
    auto cost = [&](unsigned mask) {
        double c = 0;
        for (int m = 0; m < (1 << d.nfree); ++m) {
            if (!(mask >> m & 1)) continue;
            if (b0 == -2) c += 2;
            else if (b0 >= 0) c += (mask >> (m ^ (1 << b0)) & 1) ? 1 : 2;
            else c += 1;
        }
        return c;
    };
    unsigned rows = 0;
    for (int r = 0; r < d.nrows; ++r) rows |= 1u << d.row_member[r];
    return groups * 16.0 * (cost(d.load_mask) + cost(rows));
}

template <class K, class P>
void launch_k(K kernel, double2* a, int n, int k, const GateDesc& d, const P& params, int items, cudaStream_t st,
              const char* cls) {
    const u64 ngroups = u64(1) << (n - k);
    const int threads = 256;
    const u64 per_block = u64(threads) * u64(items);
    const u64 blocks = (ngroups + per_block - 1) / per_block;
    if (blocks > 0x7fffffffull) raise(QCS_ERR_CAPACITY, "state too large for one launch");
    TimedLaunch tl(cls, algorithmic_bytes(n, d), st);
    kernel<<<unsigned(blocks), threads, 0, st>>>(a, ngroups, params);
    check_launch(cls);
}

int max_nnz(const GateDesc& d) {
    int z = 0;
    for (int r = 0; r < d.nrows; ++r) z = d.nnz[r] > z ? d.nnz[r] : z;
    return z;
}

// Tuning hook: QCS_GATE_ITEMS=1|2|4 overrides the groups per thread.
int items_override() {
    static const int v = [] {
        const char* e = std::getenv("QCS_GATE_ITEMS");
        return e ? std::atoi(e) : 0;
    }();
    return v;
}

// Tuning hook: QCS_GATE_ADJ=0 disables the 256-bit adjacent-pair path.
int adj_override() {
    static const int v = [] {
        const char* e = std::getenv("QCS_GATE_ADJ");
        return e ? std::atoi(e) : 1;
    }();
    return v;
}

}  // namespace

void launch_gate(double2* amps, int n, const GateDesc& d, cudaStream_t st) {
    const int b0 = bit0_role(d);
    const int ov = items_override();
    if (d.nfree == 0) {  // measured on B200: bit 0 fixed -> 1 group per thread, else 2
        Diag1 p{};
        p.k = d.k;
        std::memcpy(p.pos, d.pos_asc, sizeof(p.pos));
        p.fixed = d.fixed_val;
        p.d = d.val[0][0];
        const int items = ov ? ov : (b0 == -2 ? 1 : 2);
        if (items == 1) launch_k(k_diag1<1>, amps, n, d.k, d, p, 1, st, "gate_diag1");
        else if (items == 4) launch_k(k_diag1<4>, amps, n, d.k, d, p, 4, st, "gate_diag1");
        else launch_k(k_diag1<2>, amps, n, d.k, d, p, 2, st, "gate_diag1");
        return;
    }
    if (d.nfree == 1) {  // bit 0 in the group -> 4 groups per thread, else 2
        Pair p{};
        p.k = d.k;
        std::memcpy(p.pos, d.pos_asc, sizeof(p.pos));
        p.fixed = d.fixed_val;
        p.off1 = d.member_off[1];
        p.load0 = d.load_mask & 1;
        p.load1 = (d.load_mask >> 1) & 1;
        bool dense = false;
        for (int r = 0; r < d.nrows; ++r) {
            const int m = d.row_member[r];
            p.rk[m] = d.nnz[r];
            p.rc[m] = d.col_member[r][0];
            p.a[m] = d.val[r][0];
            if (d.nnz[r] > 1) {
                p.b[m] = d.val[r][1];
                dense = true;
            }
        }
        const char* cls = dense ? "gate_pair_dense" : "gate_pair_monomial";
        const bool adj = p.off1 == 1 && p.load0 && p.load1 && p.rk[0] && p.rk[1];
        // measured on B200 (tools/gate_timing.py): sector pairs 1 group per thread, bit 0
        // elsewhere in the group 4, otherwise 2
        const int items = ov ? ov : (adj ? 1 : (b0 != -1 ? 4 : 2));
        if (adj && adj_override() != 0) {
            if (items == 1) launch_k(k_pair<1, true>, amps, n, d.k, d, p, 1, st, cls);
            else if (items == 4) launch_k(k_pair<4, true>, amps, n, d.k, d, p, 4, st, cls);
            else launch_k(k_pair<2, true>, amps, n, d.k, d, p, 2, st, cls);
            return;
        }
        if (items == 1) launch_k(k_pair<1, false>, amps, n, d.k, d, p, 1, st, cls);
        else if (items == 4) launch_k(k_pair<4, false>, amps, n, d.k, d, p, 4, st, cls);
        else launch_k(k_pair<2, false>, amps, n, d.k, d, p, 2, st, cls);
        return;
    }
    const int z = max_nnz(d);
    if (d.nfree == 2 && z <= 1 && d.nrows <= 4) {  // Swap, iSwap, DCX, RZZ
        Quad p{};
        p.k = d.k;
        std::memcpy(p.pos, d.pos_asc, sizeof(p.pos));
        p.fixed = d.fixed_val;
        for (int m = 0; m < 4; ++m) p.off[m] = d.member_off[m];
        p.load = int(d.load_mask);
        p.nrows = d.nrows;
        for (int r = 0; r < d.nrows; ++r) {
            p.row[r] = d.row_member[r];
            p.col[r] = d.col_member[r][0];
            p.v[r] = d.val[r][0];
        }
        const int items = ov ? ov : 2;
        if (items == 1) launch_k(k_quad<1>, amps, n, d.k, d, p, 1, st, "gate_quad_monomial");
        else if (items == 4) launch_k(k_quad<4>, amps, n, d.k, d, p, 4, st, "gate_quad_monomial");
        else launch_k(k_quad<2>, amps, n, d.k, d, p, 2, st, "gate_quad_monomial");
        return;
    }
    if (d.nfree == 2) {
        if (z <= 1) launch_k(k_gate<2, 1, 2>, amps, n, d.k, d, d, 2, st, "gate_f2_monomial");  // Swap, iSwap, DCX
        else launch_k(k_gate<2, 4, 1>, amps, n, d.k, d, d, 1, st, "gate_f2_dense");           // RXX, ECR, CU
        return;
    }
    if (z <= 1) launch_k(k_gate<3, 1, 1>, amps, n, d.k, d, d, 1, st, "gate_f3_monomial");
    else launch_k(k_gate<3, 8, 1>, amps, n, d.k, d, d, 1, st, "gate_f3_dense");
}

}  // namespace qcs
