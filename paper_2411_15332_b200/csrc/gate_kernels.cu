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
    const u64 t0 = u64(blockIdx.x) * blockDim.x + threadIdx.x;
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
    const u64 blocks = (ngroups + per_block - 1) / per_block;
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

// ---------------------------------------------------------------- sector-granular variant
// Every thread owns whole 32-byte sectors -- amplitude pairs (2u, 2u+1) -- moved with 256-bit
// LDG/STG.  Basis bit 0 is always inside the group: as a free gate bit, as a fixed gate bit
// (the untouched neighbour rides along unchanged), or as a plain bit (the gate rows are applied
// to both halves).  Member index = 2 * pair + bit0.
struct SectorDesc {
    int npos;                 // zero-insertion positions (gate bits and bit 0), ascending
    int pos_asc[4];
    std::uint64_t fixed_val;
    std::uint64_t pair_off[4];
    std::uint32_t load_mask;  // pairs to load
    std::uint32_t store_mask; // pairs to store
    int nrows;
    std::uint8_t row_member[8];
    std::uint8_t nnz[8];
    std::uint8_t col_member[8][4];
    std::uint8_t vkind[8][4];  // 0 complex, 1 real, 2 imaginary coefficient
    double2 val[8][4];
};

// acc + v * x, skipping the products by an exact-zero component of v.  Bit-identical to madd:
// a dropped product is +-0, and adding +-0 to an accumulator that started at +0 changes neither
// its value nor (after the leading 0 + ...) its sign.
__device__ __forceinline__ double2 madd_k(double2 acc, double2 v, int kind, double2 x) {
    if (kind == 1) return make_double2(__dadd_rn(acc.x, __dmul_rn(v.x, x.x)), __dadd_rn(acc.y, __dmul_rn(v.x, x.y)));
    if (kind == 2)
        return make_double2(__dadd_rn(acc.x, -__dmul_rn(v.y, x.y)), __dadd_rn(acc.y, __dmul_rn(v.y, x.x)));
    return madd(acc, v, x);
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

template <int NP>
__device__ __forceinline__ double2 pickm(const double2 (&x)[2 * NP], int m) {
    double2 v = x[0];
#pragma unroll
    for (int j = 1; j < 2 * NP; ++j)
        if (m == j) v = x[j];
    return v;
}

template <int NP, int NR, int NNZ, int ITEMS>
__global__ void __launch_bounds__(256) k_gate_sector(double2* __restrict__ a, u64 ngroups,
                                                     const __grid_constant__ SectorDesc d) {
    const u64 stride = u64(gridDim.x) * blockDim.x;
    const u64 t0 = u64(blockIdx.x) * blockDim.x + threadIdx.x;
    double2 x[ITEMS][2 * NP];
    u64 base[ITEMS];
#pragma unroll
    for (int it = 0; it < ITEMS; ++it) {
        u64 g = t0 + it * stride;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if (i < d.npos) {
                const int p = d.pos_asc[i];
                g = ((g >> p) << (p + 1)) | (g & ((u64(1) << p) - 1));
            }
        }
        base[it] = g | d.fixed_val;
        if (t0 + it * stride < ngroups) {
#pragma unroll
            for (int p = 0; p < NP; ++p)
                if (d.load_mask >> p & 1) ld256(a + (base[it] | d.pair_off[p]), x[it][2 * p], x[it][2 * p + 1]);
        }
    }
#pragma unroll
    for (int it = 0; it < ITEMS; ++it) {
        if (t0 + it * stride >= ngroups) continue;
        double2 out[NR];
#pragma unroll
        for (int r = 0; r < NR; ++r) {
            if (r < d.nrows) {
                double2 acc = make_double2(0.0, 0.0);
#pragma unroll
                for (int z = 0; z < NNZ; ++z)
                    if (z < d.nnz[r]) acc = madd_k(acc, d.val[r][z], d.vkind[r][z], pickm<NP>(x[it], d.col_member[r][z]));
                out[r] = acc;
            }
        }
        double2 y[2 * NP];
#pragma unroll
        for (int m = 0; m < 2 * NP; ++m) y[m] = x[it][m];
#pragma unroll
        for (int r = 0; r < NR; ++r) {
            if (r < d.nrows) {
#pragma unroll
                for (int m = 0; m < 2 * NP; ++m)
                    if (d.row_member[r] == m) y[m] = out[r];
            }
        }
#pragma unroll
        for (int p = 0; p < NP; ++p)
            if (d.store_mask >> p & 1) st256(a + (base[it] | d.pair_off[p]), y[2 * p], y[2 * p + 1]);
    }
}

// GateDesc (member space over the free gate bits) -> SectorDesc; false when it does not fit.
bool to_sector(const GateDesc& d, SectorDesc& s) {
    std::memset(&s, 0, sizeof(s));
    int bit0 = -1;  // -2 fixed gate bit, >= 0 free member bit, -1 not a gate bit
    for (int i = 0; i < d.k; ++i)
        if (d.pos_asc[i] == 0) bit0 = -2;
    for (int i = 0; i < d.nfree; ++i)
        if (d.free_bit[i] == 1) bit0 = i;
    const int other_free = bit0 >= 0 ? d.nfree - 1 : d.nfree;
    const int np = 1 << other_free;
    if (np > 4) return false;
    // positions to zero-insert: the gate bits, plus bit 0 when it is not one of them
    s.npos = 0;
    if (bit0 == -1) s.pos_asc[s.npos++] = 0;
    for (int i = 0; i < d.k; ++i) s.pos_asc[s.npos++] = d.pos_asc[i];
    std::sort(s.pos_asc, s.pos_asc + s.npos);
    s.fixed_val = d.fixed_val & ~std::uint64_t(1);
    // member m (GateDesc) -> (pair, b0)
    auto pair_of = [&](int m) {
        int p = 0, j = 0;
        for (int i = 0; i < d.nfree; ++i) {
            if (i == bit0) continue;
            if (m >> i & 1) p |= 1 << j;
            ++j;
        }
        return p;
    };
    auto b0_of = [&](int m) -> int {
        if (bit0 >= 0) return m >> bit0 & 1;
        if (bit0 == -2) return int(d.fixed_val & 1);
        return 0;
    };
    for (int p = 0; p < np; ++p) {
        std::uint64_t off = 0;
        int j = 0;
        for (int i = 0; i < d.nfree; ++i) {
            if (i == bit0) continue;
            if (p >> j & 1) off |= d.free_bit[i];
            ++j;
        }
        s.pair_off[p] = off;
    }
    const int halves = bit0 == -1 ? 2 : 1;
    s.nrows = 0;
    for (int h = 0; h < halves; ++h)
        for (int r = 0; r < d.nrows; ++r) {
            if (s.nrows >= 8) return false;
            const int rr = s.nrows++;
            auto mem = [&](int m) { return 2 * pair_of(m) + (bit0 == -1 ? h : b0_of(m)); };
            s.row_member[rr] = std::uint8_t(mem(d.row_member[r]));
            s.store_mask |= 1u << pair_of(d.row_member[r]);
            s.nnz[rr] = d.nnz[r];
            if (d.nnz[r] > 4) return false;
            for (int z = 0; z < d.nnz[r]; ++z) {
                s.col_member[rr][z] = std::uint8_t(mem(d.col_member[r][z]));
                const double2 v = d.val[r][z];
                s.val[rr][z] = v;
                s.vkind[rr][z] = v.y == 0.0 ? 1 : (v.x == 0.0 ? 2 : 0);
            }
        }
    for (int m = 0; m < (1 << d.nfree); ++m)
        if (d.load_mask >> m & 1) s.load_mask |= 1u << pair_of(m);
    return true;
}

template <int NP, int NR, int NNZ, int ITEMS>
void launch_sector(double2* a, int n, const GateDesc& g, const SectorDesc& d, cudaStream_t st, const char* cls) {
    const u64 ngroups = u64(1) << (n - d.npos);
    const int threads = 256;
    const u64 per_block = u64(threads) * ITEMS;
    const u64 blocks = (ngroups + per_block - 1) / per_block;
    if (blocks > 0x7fffffffull) raise(QCS_ERR_CAPACITY, "state too large for one launch");
    TimedLaunch tl(cls, algorithmic_bytes(n, g), st);
    k_gate_sector<NP, NR, NNZ, ITEMS><<<unsigned(blocks), threads, 0, st>>>(a, ngroups, d);
    check_launch("k_gate_sector");
}

}  // namespace

void launch_gate(double2* amps, int n, const GateDesc& d, cudaStream_t st) {
    const int z = max_nnz(d);
    SectorDesc s;
    if (n >= 2 && to_sector(d, s)) {
        int np = 0;
        for (int p = 0; p < 4; ++p)
            if ((s.load_mask | s.store_mask) >> p) np = p + 1;
        if (np <= 1) {  // members 2: nnz <= 2
            if (z > 1) launch_sector<1, 4, 2, 4>(amps, n, d, s, st, "sector_p1_dense");
            else launch_sector<1, 4, 1, 4>(amps, n, d, s, st, "sector_p1_monomial");
        } else if (np == 2) {
            if (z <= 1) launch_sector<2, 8, 1, 2>(amps, n, d, s, st, "sector_p2_monomial");
            else if (z <= 2) launch_sector<2, 8, 2, 2>(amps, n, d, s, st, "sector_p2_dense");
            else launch_sector<2, 8, 4, 2>(amps, n, d, s, st, "sector_p2_dense4");
        } else {
            if (z <= 1) launch_sector<4, 8, 1, 1>(amps, n, d, s, st, "sector_p4_monomial");
            else if (z <= 2) launch_sector<4, 8, 2, 1>(amps, n, d, s, st, "sector_p4_dense");
            else launch_sector<4, 8, 4, 1>(amps, n, d, s, st, "sector_p4_dense4");
        }
        return;
    }
    switch (d.nfree) {
        case 0:  // diagonal entry on a fixed sub-cube (Z, S, T, CZ)
            launch<0, 1, 4>(amps, n, d, st, "gate_f0_diag");
            return;
        case 1:
            if (z <= 1) launch<1, 1, 2>(amps, n, d, st, "gate_f1_monomial");  // X, Y, RZ, CNOT, CCX
            else launch<1, 2, 2>(amps, n, d, st, "gate_f1_dense");             // H, RX, RY, U3, CH
            return;
        case 2:
            if (z <= 1) launch<2, 1, 1>(amps, n, d, st, "gate_f2_monomial");  // SWAP, iSwap, RZZ, DCX
            else launch<2, 4, 1>(amps, n, d, st, "gate_f2_dense");             // RXX, ECR, CU
            return;
        default:
            if (z <= 1) launch<3, 1, 1>(amps, n, d, st, "gate_f3_monomial");
            else launch<3, 8, 1>(amps, n, d, st, "gate_f3_dense");
            return;
    }
}

}  // namespace qcs
