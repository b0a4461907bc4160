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
__device__ __forceinline__ u64 insert_zeros(u64 t, const GateDesc& d) {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        if (i < d.k) {
            const int p = d.pos_asc[i];
            t = ((t >> p) << (p + 1)) | (t & ((u64(1) << p) - 1));
        }
    }
    return t;
}

// acc + v * x, skipping the products by an exact-zero component of v (kind 1: real v, kind 2:
// imaginary v).  Bit-identical to madd: a dropped product is +-0, and adding +-0 to an
// accumulator that started at +0 changes neither its value nor, after the leading 0 + ..., its
// sign (x + +-0 = x for x != 0; +0 + -0 = +0).  Inputs are finite.
__device__ __forceinline__ double2 madd_k(double2 acc, double2 v, int kind, double2 x) {
    if (kind == 1) return make_double2(__dadd_rn(acc.x, __dmul_rn(v.x, x.x)), __dadd_rn(acc.y, __dmul_rn(v.x, x.y)));
    if (kind == 2)
        return make_double2(__dadd_rn(acc.x, -__dmul_rn(v.y, x.y)), __dadd_rn(acc.y, __dmul_rn(v.y, x.x)));
    return madd(acc, v, x);
}

template <int NF>
__device__ __forceinline__ double2 pick(const double2 (&x)[1 << NF], int m) {
    double2 v = x[0];
#pragma unroll
    for (int j = 1; j < (1 << NF); ++j)
        if (m == j) v = x[j];
    return v;
}

// NF: free bits per group; NNZ: max nonzeros per touched row; ITEMS: groups per thread.
template <int NF, int NNZ, int ITEMS>
__global__ void __launch_bounds__(256) k_gate(double2* __restrict__ a, u64 ngroups,
                                              const __grid_constant__ GateDesc d) {
    constexpr int NM = 1 << NF;
    const u64 stride = u64(gridDim.x) * blockDim.x;
    // grid-stride over chunks of ITEMS * stride groups (one chunk when the grid covers all)
    for (u64 t0 = u64(blockIdx.x) * blockDim.x + threadIdx.x; t0 < ngroups; t0 += stride * ITEMS) {
    double2 x[ITEMS][NM];
    u64 base[ITEMS];
#pragma unroll
    for (int it = 0; it < ITEMS; ++it) {
        const u64 g = t0 + it * stride;
        base[it] = insert_zeros(g, d) | d.fixed_val;
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
}

// Persistent grid (QCS_GATE_PERSIST=k: k resident waves) vs one thread per ITEMS groups.
int persist_override() {
    static const int v = [] {
        const char* e = std::getenv("QCS_GATE_PERSIST");
        return e ? std::atoi(e) : 0;
    }();
    return v;
}

// Algorithmic HBM bytes of one pass: 16 B per member read and per row written, counted per
// 32-byte sector -- a touched amplitude whose basis-bit-0 mate is untouched costs the whole
// sector (SURVEY.md section 8d sector rounding).
double algorithmic_bytes(int n, const GateDesc& d) {
    const double groups = double(u64(1) << (n - d.k));
    int bit0 = -1;  // role of basis bit 0 in the group: -2 fixed, >= 0 free member bit, -1 not a gate bit
    for (int i = 0; i < d.k; ++i)
        if (d.pos_asc[i] == 0) bit0 = -2;  // fixed unless it is one of the free bits below
    for (int i = 0; i < d.nfree; ++i)
        if (d.free_bit[i] == 1) bit0 = i;
    auto cost = [&](unsigned mask) {
        double c = 0;
        for (int m = 0; m < (1 << d.nfree); ++m) {
            if (!(mask >> m & 1)) continue;
            if (bit0 == -2) c += 2;
            else if (bit0 >= 0) c += (mask >> (m ^ (1 << bit0)) & 1) ? 1 : 2;
            else c += 1;
        }
        return c;
    };
    unsigned rows = 0;
    for (int r = 0; r < d.nrows; ++r) rows |= 1u << d.row_member[r];
    return groups * 16.0 * (cost(d.load_mask) + cost(rows));
}

template <int NF, int NNZ, int ITEMS>
void launch(double2* a, int n, const GateDesc& d, cudaStream_t st, const char* cls) {
    const u64 ngroups = u64(1) << (n - d.k);
    const int threads = 256;
    const u64 per_block = u64(threads) * ITEMS;
    u64 blocks = (ngroups + per_block - 1) / per_block;
    if (const int waves = persist_override()) {
        int occ = 0;
        QCS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_gate<NF, NNZ, ITEMS>, threads, 0));
        const u64 cap = u64(148) * u64(occ > 0 ? occ : 1) * u64(waves);
        blocks = blocks < cap ? blocks : cap;
    }
    if (blocks > 0x7fffffffull) raise(QCS_ERR_CAPACITY, "state too large for one launch");
    TimedLaunch tl(cls, algorithmic_bytes(n, d), st);
    k_gate<NF, NNZ, ITEMS><<<unsigned(blocks), threads, 0, st>>>(a, ngroups, d);
    check_launch("k_gate");
}

int max_nnz(const GateDesc& d) {
    int z = 0;
    for (int r = 0; r < d.nrows; ++r) z = d.nnz[r] > z ? d.nnz[r] : z;
    return z;
}

}  // namespace

// Tuning hook (QCS_GATE_ITEMS=1|2|4 picks the groups per thread of the f0/f1 kernels).
int items_override() {
    static const int v = [] {
        const char* e = std::getenv("QCS_GATE_ITEMS");
        return e ? std::atoi(e) : 0;
    }();
    return v;
}

void launch_gate(double2* amps, int n, const GateDesc& d, cudaStream_t st) {
    const int z = max_nnz(d);
    const int it = items_override();
    switch (d.nfree) {
        case 0:  // diagonal entry on a fixed sub-cube (Z, S, T, CZ)
            if (it == 1) launch<0, 1, 1>(amps, n, d, st, "gate_f0_diag");
            else if (it == 2) launch<0, 1, 2>(amps, n, d, st, "gate_f0_diag");
            else launch<0, 1, 4>(amps, n, d, st, "gate_f0_diag");
            return;
        case 1:
            if (z <= 1) {  // X, Y, RZ, CNOT, CCX
                if (it == 1) launch<1, 1, 1>(amps, n, d, st, "gate_f1_monomial");
                else if (it == 4) launch<1, 1, 4>(amps, n, d, st, "gate_f1_monomial");
                else launch<1, 1, 2>(amps, n, d, st, "gate_f1_monomial");
            } else {       // H, RX, RY, U3, CH
                if (it == 1) launch<1, 2, 1>(amps, n, d, st, "gate_f1_dense");
                else if (it == 4) launch<1, 2, 4>(amps, n, d, st, "gate_f1_dense");
                else launch<1, 2, 2>(amps, n, d, st, "gate_f1_dense");
            }
            return;
        case 2:
            if (z <= 1) launch<2, 1, 2>(amps, n, d, st, "gate_f2_monomial");  // SWAP, iSwap, RZZ, DCX
            else launch<2, 4, 1>(amps, n, d, st, "gate_f2_dense");             // RXX, ECR, CU
            return;
        default:
            if (z <= 1) launch<3, 1, 1>(amps, n, d, st, "gate_f3_monomial");
            else launch<3, 8, 1>(amps, n, d, st, "gate_f3_dense");
            return;
    }
}

}  // namespace qcs
