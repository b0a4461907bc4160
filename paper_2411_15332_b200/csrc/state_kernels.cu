// state_kernels.cu -- diagonal sign steps, reductions and state initialisation (sm_100a).
//
// References: DiagSign steps (circuit.hpp:17-25, engine.cpp:62-80) and the StateVector
// helpers (core.cpp:22-40).  All kernels are HBM streams; grids are sized in multiples of the
// 148 SMs with grid-stride loops so reductions are deterministic for a given n.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "common.hpp"
#include "kernels.hpp"

namespace qcs {
namespace {

using u64 = std::uint64_t;
constexpr int kSMs = 148;

__device__ __forceinline__ double2 neg_exact(double2 x) {
    // 0 + (-1 + 0i) * x with dax_mvm's rounding: (-1*xr - 0*xi, -1*xi + 0*xr), then 0 + .
    const double pr = __dsub_rn(__dmul_rn(-1.0, x.x), __dmul_rn(0.0, x.y));
    const double pi = __dadd_rn(__dmul_rn(-1.0, x.y), __dmul_rn(0.0, x.x));
    return make_double2(__dadd_rn(0.0, pr), __dadd_rn(0.0, pi));
}

__device__ __forceinline__ bool listed(const u64* f, u64 nf, u64 i) {
    u64 lo = 0, hi = nf;
    while (lo < hi) {
        const u64 mid = (lo + hi) >> 1;
        if (__ldg(f + mid) < i) lo = mid + 1; else hi = mid;
    }
    return lo < nf && __ldg(f + lo) == i;
}

__global__ void k_diag_sign(double2* __restrict__ a, u64 dim, const u64* __restrict__ f, u64 nf, int rest) {
    const u64 stride = u64(gridDim.x) * blockDim.x;
    for (u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x; i < dim; i += stride) {
        if (listed(f, nf, i) != (rest != 0)) a[i] = neg_exact(__ldcs(a + i));
    }
}

__global__ void k_negate_listed(double2* __restrict__ a, const u64* __restrict__ idx, u64 count) {
    const u64 stride = u64(gridDim.x) * blockDim.x;
    for (u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride) {
        const u64 j = idx[i];
        if (i > 0 && idx[i - 1] == j) continue;  // duplicates flip once (binary-search semantics)
        a[j] = neg_exact(a[j]);
    }
}

// ---- reductions: fixed grid, per-block partials in scratch, final pass by block 0 of a
// second launch, so the summation order depends only on n.
constexpr int kRedThreads = 512;
constexpr int kRedBlocks = kSMs * 4;

__device__ __forceinline__ double block_sum(double v, double* sh) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    v = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
    if (threadIdx.x < 32)
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;
}

__global__ void k_norm2_partial(const double2* __restrict__ a, u64 dim, double* part) {
    __shared__ double sh[32];
    double acc = 0.0;
    const u64 stride = u64(gridDim.x) * blockDim.x;
    for (u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x; i < dim; i += stride) {
        const double2 x = __ldcs(a + i);
        acc += x.x * x.x + x.y * x.y;
    }
    acc = block_sum(acc, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

__global__ void k_sum_partials(double* part, int count) {
    __shared__ double sh[32];
    double acc = 0.0;
    for (int i = threadIdx.x; i < count; i += blockDim.x) acc += part[i];
    acc = block_sum(acc, sh);
    if (threadIdx.x == 0) part[count] = acc;
}

// distance between two states: per block max |a_i - b_i| and sum |a_i - b_i|^2 (fixed grid)
__global__ void k_distance_partial(const double2* __restrict__ a, const double2* __restrict__ b, u64 dim,
                                   double* part) {
    __shared__ double sh[32];
    __shared__ double shm[32];
    double acc = 0.0, mx = 0.0;
    const u64 stride = u64(gridDim.x) * blockDim.x;
    for (u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x; i < dim; i += stride) {
        const double2 x = __ldcs(a + i), y = __ldcs(b + i);
        const double dr = x.x - y.x, di = x.y - y.y;
        const double d2 = dr * dr + di * di;
        acc += d2;
        mx = fmax(mx, sqrt(d2));
    }
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_down_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) shm[threadIdx.x >> 5] = mx;
    acc = block_sum(acc, sh);
    if (threadIdx.x == 0) {
        for (int w = 1; w < int(blockDim.x >> 5); ++w) mx = fmax(mx, shm[w]);
        part[2 * blockIdx.x] = acc;
        part[2 * blockIdx.x + 1] = mx;
    }
}

__global__ void k_distance_final(double* part, int count) {
    __shared__ double sh[32];
    double acc = 0.0, mx = 0.0;
    for (int i = threadIdx.x; i < count; i += blockDim.x) {
        acc += part[2 * i];
        mx = fmax(mx, part[2 * i + 1]);
    }
    acc = block_sum(acc, sh);
    __syncthreads();
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_down_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < int(blockDim.x >> 5); ++w) mx = fmax(mx, sh[w]);
        part[2 * count] = acc;
        part[2 * count + 1] = mx;
    }
}

__global__ void k_probabilities(const double2* __restrict__ a, u64 dim, double* __restrict__ p) {
    const u64 stride = u64(gridDim.x) * blockDim.x;
    for (u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x; i < dim; i += stride) {
        const double2 x = __ldcs(a + i);
        p[i] = __dadd_rn(__dmul_rn(x.x, x.x), __dmul_rn(x.y, x.y));  // std::norm, core.cpp:38
    }
}

struct ArgMax {
    double p;
    u64 i;
};
__device__ __forceinline__ ArgMax better(ArgMax a, ArgMax b) {
    // larger probability wins; equal -> smaller index (std::max_element keeps the first)
    if (b.p > a.p || (b.p == a.p && b.i < a.i)) return b;
    return a;
}

__global__ void k_argmax_partial(const double2* __restrict__ a, u64 dim, ArgMax* part) {
    __shared__ ArgMax sh[32];
    ArgMax best{-1.0, ~u64(0)};
    const u64 stride = u64(gridDim.x) * blockDim.x;
    for (u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x; i < dim; i += stride) {
        const double2 x = __ldcs(a + i);
        best = better(best, ArgMax{__dadd_rn(__dmul_rn(x.x, x.x), __dmul_rn(x.y, x.y)), i});
    }
    for (int o = 16; o > 0; o >>= 1) {
        ArgMax other{__shfl_down_sync(0xffffffffu, best.p, o), __shfl_down_sync(0xffffffffu, best.i, o)};
        best = better(best, other);
    }
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = best;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < int(blockDim.x >> 5); ++w) best = better(best, sh[w]);
        part[blockIdx.x] = best;
    }
}

__global__ void k_argmax_final(ArgMax* part, int count) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        ArgMax best = part[0];
        for (int i = 1; i < count; ++i) best = better(best, part[i]);
        part[count] = best;
    }
}

__global__ void k_gather(const double2* __restrict__ a, const u64* __restrict__ idx, u64 count,
                         double2* __restrict__ out) {
    const u64 stride = u64(gridDim.x) * blockDim.x;
    for (u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride) out[i] = a[idx[i]];
}

__global__ void k_scale(double2* __restrict__ a, u64 dim, double s) {
    const u64 stride = u64(gridDim.x) * blockDim.x;
    for (u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x; i < dim; i += stride) {
        const double2 x = __ldcs(a + i);
        __stcs(a + i, make_double2(x.x * s, x.y * s));
    }
}

__global__ void k_fill_basis(double2* __restrict__ a, u64 dim, u64 index) {
    const u64 stride = u64(gridDim.x) * blockDim.x;
    for (u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x; i < dim; i += stride)
        __stcs(a + i, make_double2(i == index ? 1.0 : 0.0, 0.0));
}

// splitmix64 counter hash -> two uniforms -> Box-Muller: i.i.d. N(0,1) re and im per index.
__device__ __forceinline__ u64 mix64(u64 z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

__global__ void k_fill_random(double2* __restrict__ a, u64 dim, u64 seed) {
    const u64 stride = u64(gridDim.x) * blockDim.x;
    const u64 key = mix64(seed);
    for (u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x; i < dim; i += stride) {
        const u64 h1 = mix64(key ^ (2 * i)), h2 = mix64(key ^ (2 * i + 1));
        const double u1 = (double(h1 >> 11) + 1.0) * 0x1.0p-53;  // (0, 1]
        const double u2 = double(h2 >> 11) * 0x1.0p-53;          // [0, 1)
        const double r = sqrt(-2.0 * log(u1));
        double sn, cs;
        sincospi(2.0 * u2, &sn, &cs);
        __stcs(a + i, make_double2(r * cs, r * sn));
    }
}

// ---- top-k (k <= 16).  One pass at copy bandwidth: every warp keeps its 16 best so far in a
// shared-memory buffer together with the threshold tau they imply (its 16th best); an element
// that does not beat tau costs one comparison, the few that do are appended to the buffer with a
// ballot (no atomics) and the buffer is cut back to its 16 best (16 warp arg-max rounds) before
// the next batch of loads.  (The first version kept a sorted list of 16 per THREAD in registers:
// 138 registers, one resident block per SM, 23 ms for the 64 GiB state of n=32 against 9.9 ms
// for the norm alone.)  K candidates per block; the host merges the block candidates.
constexpr int kTopK = 16;
constexpr int kTopU = 8;                        // independent 16-byte loads per thread in flight
constexpr int kTopBuf = kTopK + 32 * kTopU;     // a warp's buffer: its best 16 plus one batch

// the 16 best of wb[0..cnt) (by `better`: larger p, ties to the lower index) to wb[0..min(cnt,16)),
// best first; returns the new count; tau = the 16th best once there are 16
__device__ __forceinline__ unsigned warp_prune(ArgMax* wb, unsigned cnt, ArgMax& tau, unsigned lane) {
    const ArgMax none{-1.0, ~u64(0)};
    ArgMax mine = none;
    __syncwarp();
    for (int r = 0; r < kTopK; ++r) {
        ArgMax best = none;
        for (unsigned j = lane; j < cnt; j += 32) {
            const ArgMax e = wb[j];
            if (e.p >= 0.0) best = better(best, e);
        }
        for (int o = 16; o > 0; o >>= 1) {
            ArgMax other{__shfl_xor_sync(0xffffffffu, best.p, o), __shfl_xor_sync(0xffffffffu, best.i, o)};
            best = better(best, other);
        }
        if (int(lane) == r) mine = best;
        if (best.i != ~u64(0))  // its owner retires the winner (indices are unique)
            for (unsigned j = lane; j < cnt; j += 32)
                if (wb[j].i == best.i) wb[j].p = -2.0;
        __syncwarp();
    }
    if (lane < unsigned(kTopK)) wb[lane] = mine;
    __syncwarp();
    const unsigned kept = cnt < unsigned(kTopK) ? cnt : unsigned(kTopK);
    tau = kept == unsigned(kTopK) ? wb[kTopK - 1] : none;
    return kept;
}

// psum (optional): per-block sums of the probabilities (the norm of a report, in the same pass)
__global__ void __launch_bounds__(256, 2) k_topk_partial(const double2* __restrict__ a, u64 dim, int k,
                                                         ArgMax* __restrict__ out, double* __restrict__ psum) {
    __shared__ ArgMax buf[8][kTopBuf];
    __shared__ ArgMax sh[8];
    __shared__ ArgMax win;
    __shared__ double shs[32];
    const unsigned lane = threadIdx.x & 31u, w = threadIdx.x >> 5;
    ArgMax* const wb = buf[w];
    const ArgMax none{-1.0, ~u64(0)};
    if (u64(blockIdx.x) * blockDim.x >= dim) {  // small states: this block has no element
        if (threadIdx.x < unsigned(k)) out[u64(blockIdx.x) * k + threadIdx.x] = none;
        if (psum && threadIdx.x == 0) psum[blockIdx.x] = 0.0;
        return;
    }
    unsigned cnt = 0;   // warp-uniform
    ArgMax tau = none;  // warp-uniform
    double acc = 0.0;
    const u64 stride = u64(gridDim.x) * blockDim.x;
    const u64 first = u64(blockIdx.x) * blockDim.x + threadIdx.x;
    // warp-uniform trip count (the ballots below need the whole warp): lanes past dim idle.  The
    // next batch's loads are issued before the current batch is examined.
    double2 x[kTopU], y[kTopU];
    auto fetch = [&](u64 i0, double2 (&v)[kTopU]) {
#pragma unroll
        for (int u = 0; u < kTopU; ++u) {
            const u64 i = i0 + lane + u64(u) * stride;
            v[u] = i < dim ? __ldcs(a + i) : make_double2(0.0, 0.0);
        }
    };
    auto examine = [&](u64 i0, const double2 (&v)[kTopU]) {
#pragma unroll
        for (int u = 0; u < kTopU; ++u) {
            const u64 i = i0 + lane + u64(u) * stride;
            const bool valid = i < dim;
            const ArgMax c{__dadd_rn(__dmul_rn(v[u].x, v[u].x), __dmul_rn(v[u].y, v[u].y)), i};
            if (valid) acc += c.p;
            const bool pass = valid && better(tau, c).i == c.i;
            const unsigned m = __ballot_sync(0xffffffffu, pass);
            if (m) {
                if (pass) wb[cnt + __popc(m & ((1u << lane) - 1u))] = c;
                cnt += __popc(m);
            }
        }
        if (cnt > unsigned(kTopK)) cnt = warp_prune(wb, cnt, tau, lane);
    };
    const u64 step = kTopU * stride;
    u64 i0 = first - lane;
    if (i0 < dim) fetch(i0, x);
    while (i0 < dim) {
        if (i0 + step < dim) fetch(i0 + step, y);
        examine(i0, x);
        i0 += step;
        if (i0 >= dim) break;
        if (i0 + step < dim) fetch(i0 + step, x);
        examine(i0, y);
        i0 += step;
    }
    cnt = warp_prune(wb, cnt, tau, lane);  // sorted, best first
    if (psum) {
        acc = block_sum(acc, shs);
        if (threadIdx.x == 0) psum[blockIdx.x] = acc;
    }
    __syncthreads();
    // the block's k best among the warps' lists: thread t < 128 holds entry t % 16 of warp t / 16
    ArgMax h = none;
    if (threadIdx.x < 8 * kTopK) h = buf[threadIdx.x / kTopK][threadIdx.x % kTopK];
    if (h.p < 0.0) h = none;
    for (int round = 0; round < k; ++round) {
        ArgMax best = h;
        for (int o = 16; o > 0; o >>= 1) {
            ArgMax other{__shfl_down_sync(0xffffffffu, best.p, o), __shfl_down_sync(0xffffffffu, best.i, o)};
            best = better(best, other);
        }
        if (lane == 0) sh[w] = best;
        __syncthreads();
        if (threadIdx.x == 0) {
            ArgMax b = sh[0];
            for (int v = 1; v < int(blockDim.x >> 5); ++v) b = better(b, sh[v]);
            win = b;
            out[u64(blockIdx.x) * k + round] = b;
        }
        __syncthreads();
        if (h.i == win.i && h.i != ~u64(0)) h = none;
        __syncthreads();
    }
}

inline unsigned grid_for(u64 work, int threads) {
    const u64 want = (work + threads - 1) / threads;
    const u64 cap = u64(kSMs) * 16;
    return unsigned(want < 1 ? 1 : (want > cap ? cap : want));
}

}  // namespace

void launch_diag_sign(double2* amps, int n, const std::uint64_t* f, std::uint64_t nf, int rest,
                      cudaStream_t st) {
    const u64 dim = u64(1) << n;
    TimedLaunch tl("diag_sign", 32.0 * double(dim), st);
    k_diag_sign<<<grid_for(dim, 256), 256, 0, st>>>(amps, dim, f, nf, rest);
    check_launch("k_diag_sign");
}

void launch_negate_listed(double2* amps, const std::uint64_t* idx, std::uint64_t count, cudaStream_t st) {
    if (!count) return;
    TimedLaunch tl("negate_listed", 64.0 * double(count), st);
    k_negate_listed<<<grid_for(count, 256), 256, 0, st>>>(amps, idx, count);
    check_launch("k_negate_listed");
}

double reduce_norm2(const double2* amps, int n, double* scratch, cudaStream_t st) {
    const u64 dim = u64(1) << n;
    k_norm2_partial<<<kRedBlocks, kRedThreads, 0, st>>>(amps, dim, scratch);
    check_launch("k_norm2_partial");
    k_sum_partials<<<1, 1024, 0, st>>>(scratch, kRedBlocks);
    check_launch("k_sum_partials");
    double h = 0.0;
    QCS_CUDA(cudaMemcpyAsync(&h, scratch + kRedBlocks, sizeof(double), cudaMemcpyDeviceToHost, st));
    QCS_CUDA(cudaStreamSynchronize(st));
    return h;
}

void distance(const double2* a, const double2* b, std::uint64_t dim, double* max_abs, double* l2,
              cudaStream_t st) {
    double* part = nullptr;
    QCS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&part), sizeof(double) * (2 * kRedBlocks + 2), st));
    k_distance_partial<<<kRedBlocks, kRedThreads, 0, st>>>(a, b, dim, part);
    check_launch("k_distance_partial");
    k_distance_final<<<1, 1024, 0, st>>>(part, kRedBlocks);
    check_launch("k_distance_final");
    double h[2];
    QCS_CUDA(cudaMemcpyAsync(h, part + 2 * kRedBlocks, sizeof(h), cudaMemcpyDeviceToHost, st));
    QCS_CUDA(cudaFreeAsync(part, st));
    QCS_CUDA(cudaStreamSynchronize(st));
    *l2 = std::sqrt(h[0]);
    *max_abs = h[1];
}

void probabilities(const double2* amps, std::uint64_t dim, double* out, cudaStream_t st) {
    k_probabilities<<<grid_for(dim, 256), 256, 0, st>>>(amps, dim, out);
    check_launch("k_probabilities");
}

void argmax(const double2* amps, std::uint64_t dim, std::uint64_t* idx, double* p, void* scratch,
            cudaStream_t st) {
    ArgMax* part = static_cast<ArgMax*>(scratch);
    k_argmax_partial<<<kRedBlocks, kRedThreads, 0, st>>>(amps, dim, part);
    check_launch("k_argmax_partial");
    k_argmax_final<<<1, 32, 0, st>>>(part, kRedBlocks);
    check_launch("k_argmax_final");
    ArgMax h;
    QCS_CUDA(cudaMemcpyAsync(&h, part + kRedBlocks, sizeof(ArgMax), cudaMemcpyDeviceToHost, st));
    QCS_CUDA(cudaStreamSynchronize(st));
    *idx = h.i;
    *p = h.p;
}

void gather(const double2* amps, const std::uint64_t* idx, std::uint64_t count, double2* out, cudaStream_t st) {
    if (!count) return;
    k_gather<<<grid_for(count, 256), 256, 0, st>>>(amps, idx, count, out);
    check_launch("k_gather");
}

void scale(double2* amps, std::uint64_t dim, double s, cudaStream_t st) {
    k_scale<<<grid_for(dim, 256), 256, 0, st>>>(amps, dim, s);
    check_launch("k_scale");
}

void fill_basis(double2* amps, std::uint64_t dim, std::uint64_t index, cudaStream_t st) {
    k_fill_basis<<<grid_for(dim, 256), 256, 0, st>>>(amps, dim, index);
    check_launch("k_fill_basis");
}

void fill_random(double2* amps, std::uint64_t dim, std::uint64_t seed, cudaStream_t st) {
    k_fill_random<<<grid_for(dim, 256), 256, 0, st>>>(amps, dim, seed);
    check_launch("k_fill_random");
}

// The one-pass summary in two halves, so a caller can keep the device busy meanwhile:
// topk_begin enqueues the reduction and the read-back of the block candidates (and block sums)
// into `host` (pinned, topk_host_bytes(k) bytes) on stream st; topk_finish merges them once the
// stream has reached that point.
std::size_t topk_host_bytes(int k) { return sizeof(ArgMax) * std::size_t(kSMs * 2) * std::size_t(k) + sizeof(double) * kSMs * 2; }

void topk_begin(const double2* amps, std::uint64_t dim, int k, bool with_norm, void* host, cudaStream_t st) {
    if (k < 1 || k > kTopK) raise(QCS_ERR_ARG, "top-k supports 1 <= k <= 16");
    const int blocks = kSMs * 2;
    ArgMax* part = nullptr;
    const std::size_t pbytes = sizeof(ArgMax) * blocks * k;
    QCS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&part), pbytes + sizeof(double) * blocks, st));
    double* psum = with_norm ? reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(part) + pbytes) : nullptr;
    k_topk_partial<<<blocks, 256, 0, st>>>(amps, dim, k, part, psum);
    check_launch("k_topk_partial");
    QCS_CUDA(cudaMemcpyAsync(host, part, pbytes + (with_norm ? sizeof(double) * blocks : 0), cudaMemcpyDeviceToHost, st));
    QCS_CUDA(cudaFreeAsync(part, st));
}

void topk_finish(const void* host, int k, bool with_norm, std::uint64_t* idx, double* p, double* norm) {
    const int blocks = kSMs * 2;
    const auto* h = static_cast<const ArgMax*>(host);
    if (with_norm && norm) {
        const auto* hs = reinterpret_cast<const double*>(static_cast<const unsigned char*>(host) + sizeof(ArgMax) * blocks * k);
        double acc = 0.0;
        for (int i = 0; i < blocks; ++i) acc += hs[i];  // fixed block order: deterministic for a given n
        *norm = std::sqrt(acc);
    }
    std::vector<ArgMax> c;
    for (int i = 0; i < blocks * k; ++i)
        if (h[i].i != ~u64(0)) c.push_back(h[i]);
    std::sort(c.begin(), c.end(), [](const ArgMax& x, const ArgMax& y) { return x.p != y.p ? x.p > y.p : x.i < y.i; });
    for (int j = 0; j < k; ++j) {
        idx[j] = j < int(c.size()) ? c[j].i : ~u64(0);
        p[j] = j < int(c.size()) ? c[j].p : 0.0;
    }
}

void topk(const double2* amps, std::uint64_t dim, int k, std::uint64_t* idx, double* p, cudaStream_t st,
          double* norm) {
    std::vector<unsigned char> host(topk_host_bytes(k));
    topk_begin(amps, dim, k, norm != nullptr, host.data(), st);
    QCS_CUDA(cudaStreamSynchronize(st));
    topk_finish(host.data(), k, norm != nullptr, idx, p, norm);
}

std::size_t reduce_scratch_bytes() { return sizeof(ArgMax) * (kRedBlocks + 1) + 64; }

}  // namespace qcs
