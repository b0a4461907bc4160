// dense_kernels.cu -- the paper's "Matrix" method on the device: the dense step operator and its
// MVM, byte for byte the reference's dense engine.
//
//   step_matrix_dense (engine.cpp:126-133): acc = factor_0; acc = dense_tensor(acc, factor_i) --
//     entry (r, c) = ((f0[r0][c0] * f1[r1][c1]) * f2[r2][c2]) ... with 2x2 identities at the
//     uncovered qubits (core.cpp:55-72); a diagonal sign step is the +-1 diagonal (engine.cpp:54-60)
//   dense_mvm (core.cpp:74-87): out[r] = sum_c m[r][c] * s[c], accumulated in column order from 0
//
// Every complex product and sum is separately rounded (the reference's x86-64 build has no FMA;
// this file is compiled with -fmad=false), and the operand order is std::complex's, so the
// matrix bytes -- signed zeros included -- and the MVM results equal the reference's.
#include "common.hpp"
#include "kernels.hpp"

namespace qcs {
namespace {

using u64 = std::uint64_t;

__device__ __forceinline__ double2 cmul_rn(double2 a, double2 b) {  // (a.x + i a.y)(b.x + i b.y)
    return make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                        __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}

// One thread per entry.  Position p of the fold (most significant qubit first) multiplies by
// factor entry (row bits, col bits) of its factor; factors of k qubits take k index bits.
__global__ void k_dense_build(double2* __restrict__ m, int n, DenseFold fold) {
    const u64 dim = u64(1) << n;
    const u64 total = dim * dim;
    for (u64 e = u64(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += u64(gridDim.x) * blockDim.x) {
        const u64 r = e >> n, c = e & (dim - 1);
        double2 acc = make_double2(0.0, 0.0);
        int shift = n;
        for (int f = 0; f < fold.nfactors; ++f) {
            const int k = fold.arity[f];
            shift -= k;
            const unsigned rr = unsigned((r >> shift) & ((1u << k) - 1));
            const unsigned cc = unsigned((c >> shift) & ((1u << k) - 1));
            const double2 v = fold.mat[fold.offset[f] + rr * (1u << k) + cc];
            acc = f == 0 ? v : cmul_rn(acc, v);
        }
        m[e] = acc;
    }
}

// The diagonal sign step as a dense matrix: -1 at the negated indices, +1 elsewhere on the
// diagonal, +0 off it (DenseMatrix's value-initialised zeros).
__global__ void k_dense_diag(double2* __restrict__ m, int n, const u64* __restrict__ f, u64 nf, int rest) {
    const u64 dim = u64(1) << n;
    const u64 total = dim * dim;
    for (u64 e = u64(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += u64(gridDim.x) * blockDim.x) {
        const u64 r = e >> n, c = e & (dim - 1);
        double2 v = make_double2(0.0, 0.0);
        if (r == c) {
            u64 lo = 0, hi = nf;
            while (lo < hi) {
                const u64 mid = (lo + hi) >> 1;
                if (f[mid] < r) lo = mid + 1; else hi = mid;
            }
            const bool listed = lo < nf && f[lo] == r;
            v = make_double2((listed != (rest != 0)) ? -1.0 : 1.0, 0.0);
        }
        m[e] = v;
    }
}

// dense_mvm: one thread per row, the row's sum in column order.  A warp owns 32 rows and walks
// the columns in 32-wide tiles staged through shared memory, so the matrix streams in coalesced
// 512-byte row segments while each thread's accumulation order stays the reference's.
constexpr int kRows = 32;
__global__ void __launch_bounds__(kRows) k_dense_mvm(const double2* __restrict__ m, const double2* __restrict__ x,
                                                    double2* __restrict__ out, int n) {
    __shared__ double2 tile[kRows][kRows + 1];
    __shared__ double2 xs[kRows];
    const u64 dim = u64(1) << n;
    const unsigned t = threadIdx.x;
    const u64 r0 = u64(blockIdx.x) * kRows;
    double2 acc = make_double2(0.0, 0.0);
    const u64 cols = dim < kRows ? dim : kRows;
    for (u64 c0 = 0; c0 < dim; c0 += cols) {
        for (unsigned i = 0; i < kRows && r0 + i < dim; ++i)
            if (t < cols) tile[i][t] = __ldcs(m + (r0 + i) * dim + c0 + t);
        if (t < cols) xs[t] = x[c0 + t];
        __syncwarp();
        if (r0 + t < dim)
            for (unsigned c = 0; c < cols; ++c) {
                const double2 p = cmul_rn(tile[t][c], xs[c]);
                acc = make_double2(__dadd_rn(acc.x, p.x), __dadd_rn(acc.y, p.y));
            }
        __syncwarp();
    }
    if (r0 + t < dim) out[r0 + t] = acc;
}

}  // namespace

void dense_build(double2* m, int n, const DenseFold& fold, cudaStream_t st) {
    const u64 total = (u64(1) << n) << n;
    const unsigned blocks = unsigned(total / 256 + 1 < 148ull * 32 ? total / 256 + 1 : 148ull * 32);
    TimedLaunch tl("dense_build", 16.0 * double(total), st);
    k_dense_build<<<blocks, 256, 0, st>>>(m, n, fold);
    check_launch("k_dense_build");
}

void dense_diag(double2* m, int n, const std::uint64_t* flipped_dev, std::uint64_t nf, int rest, cudaStream_t st) {
    const u64 total = (u64(1) << n) << n;
    const unsigned blocks = unsigned(total / 256 + 1 < 148ull * 32 ? total / 256 + 1 : 148ull * 32);
    TimedLaunch tl("dense_build", 16.0 * double(total), st);
    k_dense_diag<<<blocks, 256, 0, st>>>(m, n, flipped_dev, nf, rest);
    check_launch("k_dense_diag");
}

void dense_mvm(const double2* m, const double2* x, double2* out, int n, cudaStream_t st) {
    const u64 dim = u64(1) << n;
    TimedLaunch tl("dense_mvm", 16.0 * double(dim * dim) + 32.0 * double(dim), st);
    k_dense_mvm<<<unsigned((dim + kRows - 1) / kRows), kRows, 0, st>>>(m, x, out, n);
    check_launch("k_dense_mvm");
}

}  // namespace qcs
