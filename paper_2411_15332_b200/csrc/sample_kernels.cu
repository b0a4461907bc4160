// sample_kernels.cu -- seeded sampling from |amplitude|^2 on the device, index-exact against the
// reference's render_report (circuit_io.cpp:114-128):
//
//     acc = 0.0; for i: acc += probs[i]; cdf[i] = acc;        // sequential, rounded per add
//     u = uniform_real_distribution<double>(0, acc)(mt19937_64(seed)); lower_bound(cdf, u)
//
// The sequential rounded prefix sum is the hard part: a parallel scan rounds differently, and a
// sample lands on a different index whenever a draw falls between the two roundings of a CDF
// boundary.  We reproduce the sequential chain exactly without running it serially:
//
//  * While the running sum s stays inside one binade [2^e, 2^(e+1)) its representable values are
//    the multiples of u = ulp(s).  fl(s + p) = u * RNE(s/u + p/u), so the chain is an integer
//    walk K -> K + inc(p, K) where inc = floor(p/u) + {0,1}; the only dependence on K is the
//    tie-to-even case (p/u has fraction exactly 1/2), which depends on the parity of K.
//  * An element is therefore a map parity -> increment (two int64s); maps compose associatively
//    (f then g: b -> f(b) + g((b + f(b)) & 1)), so a chunk of the array reduces to one map in
//    parallel (k_chunk_maps).
//  * The host walks the chunk maps in order.  The chunk in which s would leave its binade is
//    replayed serially in plain double arithmetic from its exact start value (the same adds the
//    reference executes), and the walk resumes with the new binade's maps.
//
// The result is cdf_start[c] = the reference's acc just before chunk c, exactly, for every chunk,
// plus the final acc.  A draw's lower_bound then lies in one chunk (host binary search over
// cdf_start), which k_sample_in_chunk replays serially from its exact start value.  Nothing of
// size 2^n leaves the device; device memory beyond the state is 16 B per chunk.
#include <cmath>
#include <cstring>
#include <random>
#include <vector>

#include "common.hpp"
#include "kernels.hpp"

namespace qcs {
namespace {

using u64 = std::uint64_t;
using i64 = std::int64_t;

constexpr int kChunkLog = 12;             // 4096 amplitudes per chunk
constexpr u64 kChunk = u64(1) << kChunkLog;
constexpr int kMapThreads = 256;          // 16 elements per thread
constexpr int kSMs = 148;
constexpr int kPerThread = int(kChunk / kMapThreads);

struct PMap {  // increment for incoming parity 0 and 1
    i64 a0, a1;
};

__device__ __forceinline__ PMap compose(PMap f, PMap g) {
    PMap h;
    h.a0 = f.a0 + ((f.a0 & 1) ? g.a1 : g.a0);
    h.a1 = f.a1 + (((1 + f.a1) & 1) ? g.a1 : g.a0);
    return h;
}

__device__ __forceinline__ double prob(double2 x) {  // std::norm (core.cpp:38), no contraction
    return __dadd_rn(__dmul_rn(x.x, x.x), __dmul_rn(x.y, x.y));
}

// p/u for u = 2^ue: exact (a power-of-two scale), then the RNE increment map.  Increments are
// clamped at 2^60: any element that large leaves the binade, and that chunk is replayed serially.
__device__ __forceinline__ PMap elem_map(double p, int ue) {
    const double x = ldexp(p, -ue);
    if (!(x < 1152921504606846976.0)) return PMap{i64(1) << 60, i64(1) << 60};
    const double fl = floor(x);
    const double fr = x - fl;  // exact
    const i64 f = i64(fl);
    if (fr > 0.5) return PMap{f + 1, f + 1};
    if (fr < 0.5) return PMap{f, f};
    // tie: the sum K + f + 1/2 rounds to the even one of K + f, K + f + 1
    const i64 odd = f & 1;  // parity of f
    return PMap{odd ? f + 1 : f, odd ? f : f + 1};
}

// One block per chunk in [c0, c0 + count): the chunk's composed map for ulp exponent ue.
__global__ void __launch_bounds__(kMapThreads) k_chunk_maps(const double2* __restrict__ a, u64 c0, int ue,
                                                           PMap* __restrict__ out) {
    __shared__ PMap sh[kMapThreads / 32];
    const u64 base = (c0 + blockIdx.x) * kChunk + u64(threadIdx.x) * kPerThread;
    PMap m{0, 0};
#pragma unroll 4
    for (int j = 0; j < kPerThread; ++j) m = compose(m, elem_map(prob(a[base + j]), ue));
    // ordered warp reduction: lane l composes with lane l + o (its right neighbour block)
    const int lane = threadIdx.x & 31;
    for (int o = 1; o < 32; o <<= 1) {
        PMap r{__shfl_down_sync(0xffffffffu, m.a0, o), __shfl_down_sync(0xffffffffu, m.a1, o)};
        if ((lane & (2 * o - 1)) == 0) m = compose(m, r);
    }
    if (lane == 0) sh[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        PMap t = sh[0];
        for (int w = 1; w < kMapThreads / 32; ++w) t = compose(t, sh[w]);
        out[blockIdx.x] = t;
    }
}

// Probabilities of one range (the chunks the host replays serially).
__global__ void k_probs_range(const double2* __restrict__ a, u64 first, u64 count, double* __restrict__ p) {
    for (u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += u64(gridDim.x) * blockDim.x)
        p[i] = prob(a[first + i]);
}

// First index >= first with a nonzero probability (or dim): the sum leaves 0.0 there.
__global__ void k_first_nonzero(const double2* __restrict__ a, u64 first, u64 dim,
                                unsigned long long* __restrict__ out) {
    for (u64 i = first + u64(blockIdx.x) * blockDim.x + threadIdx.x; i < dim; i += u64(gridDim.x) * blockDim.x)
        if (prob(a[i]) != 0.0) {
            atomicMin(out, static_cast<unsigned long long>(i));
            return;
        }
}

// One thread per draw: replay the reference's adds over the draw's chunk from its exact start
// value; the first index whose running sum is >= u is std::lower_bound's answer.
__global__ void k_sample_in_chunk(const double2* __restrict__ a, u64 dim, const double* __restrict__ u,
                                  const u64* __restrict__ chunk, const double* __restrict__ start, u64 count,
                                  u64* __restrict__ out) {
    const u64 t = u64(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= count) return;
    const u64 c = chunk[t];
    const double want = u[t];
    double s = start[t];
    const u64 lo = c * kChunk;
    const u64 hi = lo + kChunk < dim ? lo + kChunk : dim;
    u64 j = lo;
    for (; j < hi; ++j) {
        s = __dadd_rn(s, prob(a[j]));
        if (s >= want) break;
    }
    out[t] = j < hi ? j : hi - 1;  // the host guarantees the answer lies in the chunk
}

int ulp_exp(double s) {  // exponent of ulp(s) for s > 0 (subnormals: -1074)
    int e = 0;
    std::frexp(s, &e);  // s = m * 2^e, m in [0.5, 1)
    const int ue = e - 53;
    return ue < -1074 ? -1074 : ue;
}

}  // namespace

// The exact sequential CDF at chunk granularity (see the file comment).  cdf_start has
// ceil(dim / kChunk) + 1 entries: cdf_start[c] = acc before chunk c (cdf_start[0] = 0) and the
// last entry = the final acc.
void sample_cdf_index(const double2* amps, u64 dim, std::vector<double>& cdf_start, cudaStream_t st) {
    const u64 chunks = (dim + kChunk - 1) / kChunk;
    cdf_start.assign(chunks + 1, 0.0);
    std::vector<double> hp(kChunk);
    double* dp = nullptr;
    PMap* dmap = nullptr;
    unsigned long long* dfirst = nullptr;
    QCS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dp), kChunk * sizeof(double), st));
    QCS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dmap), chunks * sizeof(PMap), st));
    QCS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dfirst), sizeof(unsigned long long), st));
    std::vector<PMap> hmap;

    // replay chunk c serially from s in double arithmetic: the reference's own adds
    auto replay = [&](u64 c, double s) {
        const u64 lo = c * kChunk, cnt = (lo + kChunk <= dim ? kChunk : dim - lo);
        k_probs_range<<<16, 256, 0, st>>>(amps, lo, cnt, dp);
        check_launch("k_probs_range");
        QCS_CUDA(cudaMemcpyAsync(hp.data(), dp, cnt * sizeof(double), cudaMemcpyDeviceToHost, st));
        QCS_CUDA(cudaStreamSynchronize(st));
        volatile double acc = s;  // one rounded add per element, as circuit_io.cpp:120
        for (u64 j = 0; j < cnt; ++j) acc = acc + hp[j];
        return double(acc);
    };

    double s = 0.0;
    u64 c = 0;
    u64 prev_len = 0;  // chunks walked in the previous binade: the next map window is twice that
    while (c < chunks) {
        cdf_start[c] = s;
        if (s == 0.0) {
            // 0 + 0 = 0 until the first nonzero probability; find its chunk and replay that one
            const unsigned long long none = ~0ull;
            QCS_CUDA(cudaMemcpyAsync(dfirst, &none, sizeof(none), cudaMemcpyHostToDevice, st));
            k_first_nonzero<<<unsigned(kSMs) * 8, 256, 0, st>>>(amps, c * kChunk, dim, dfirst);
            check_launch("k_first_nonzero");
            unsigned long long f = none;
            QCS_CUDA(cudaMemcpyAsync(&f, dfirst, sizeof(f), cudaMemcpyDeviceToHost, st));
            QCS_CUDA(cudaStreamSynchronize(st));
            if (f == none) {  // all remaining probabilities are zero
                for (u64 k = c; k <= chunks; ++k) cdf_start[k] = 0.0;
                break;
            }
            const u64 fc = u64(f) / kChunk;
            for (u64 k = c; k <= fc; ++k) cdf_start[k] = 0.0;
            s = replay(fc, 0.0);
            c = fc + 1;
            continue;
        }
        // a binade: walk chunk maps from c while the sum stays below 2^(e+1)
        const int ue = ulp_exp(s);
        int e2 = 0;
        std::frexp(s, &e2);
        const double top = std::ldexp(1.0, e2);  // 2^(e+1): the binade's end
        i64 K = i64(std::ldexp(s, -ue));        // s / u, exact (< 2^53)
        const i64 Ktop = i64(std::ldexp(top, -ue));
        const u64 start_c = c;
        u64 window = prev_len * 2 < 64 ? 64 : prev_len * 2;
        bool left = false;
        while (c < chunks && !left) {
            const u64 cnt = c + window <= chunks ? window : chunks - c;
            // full chunks only; a partial last chunk is replayed serially
            const u64 full = (c + cnt) * kChunk <= dim ? cnt : cnt - 1;
            if (full) {
                k_chunk_maps<<<unsigned(full), kMapThreads, 0, st>>>(amps, c, ue, dmap);
                check_launch("k_chunk_maps");
                hmap.resize(full);
                QCS_CUDA(cudaMemcpyAsync(hmap.data(), dmap, full * sizeof(PMap), cudaMemcpyDeviceToHost, st));
                QCS_CUDA(cudaStreamSynchronize(st));
            }
            u64 k = 0;
            for (; k < full; ++k) {
                const i64 inc = (K & 1) ? hmap[k].a1 : hmap[k].a0;
                if (inc >= Ktop - K) {  // this chunk reaches 2^(e+1): replay it exactly
                    s = replay(c + k, std::ldexp(double(K), ue));
                    ++k;
                    left = true;
                    break;
                }
                K += inc;
                cdf_start[c + k + 1] = std::ldexp(double(K), ue);
            }
            if (!left && full < cnt) {  // the partial last chunk
                s = replay(c + k, std::ldexp(double(K), ue));
                ++k;
                left = true;
            }
            c += k;
            if (!left) {
                s = std::ldexp(double(K), ue);
                window *= 2;
            }
        }
        prev_len = c - start_c;
    }
    cdf_start[chunks] = s;
    QCS_CUDA(cudaFreeAsync(dp, st));
    QCS_CUDA(cudaFreeAsync(dmap, st));
    QCS_CUDA(cudaFreeAsync(dfirst, st));
    QCS_CUDA(cudaStreamSynchronize(st));
}

// render_report's sampling (circuit_io.cpp:114-128), bit-for-bit: std::mt19937_64(seed), one
// uniform_real_distribution<double>(0, acc) draw per sample, lower_bound on the sequential CDF.
void sample(const double2* amps, u64 dim, u64 seed, u64 count, u64* out, double* total, cudaStream_t st) {
    std::vector<double> cdf_start;
    sample_cdf_index(amps, dim, cdf_start, st);
    const u64 chunks = cdf_start.size() - 1;
    const double acc = cdf_start[chunks];
    if (total) *total = acc;
    if (!count) return;
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> dist(0.0, acc);
    std::vector<double> hu(count), hs(count);
    std::vector<u64> hc(count);
    for (u64 i = 0; i < count; ++i) {
        const double u = dist(rng);
        hu[i] = u;
        // chunk c: the last one whose start (the acc before it) is < u; chunk 0 when none is
        // (cdf[0] >= u already, or u <= 0)
        u64 lo = 0, hi = chunks;  // invariant: answer in [lo, hi)
        while (hi - lo > 1) {
            const u64 mid = (lo + hi) / 2;
            if (cdf_start[mid] < u) lo = mid;
            else hi = mid;
        }
        hc[i] = lo;
        hs[i] = cdf_start[lo];
    }
    double *du = nullptr, *ds = nullptr;
    u64 *dc = nullptr, *dout = nullptr;
    QCS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&du), count * sizeof(double), st));
    QCS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ds), count * sizeof(double), st));
    QCS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dc), count * sizeof(u64), st));
    QCS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dout), count * sizeof(u64), st));
    QCS_CUDA(cudaMemcpyAsync(du, hu.data(), count * sizeof(double), cudaMemcpyHostToDevice, st));
    QCS_CUDA(cudaMemcpyAsync(ds, hs.data(), count * sizeof(double), cudaMemcpyHostToDevice, st));
    QCS_CUDA(cudaMemcpyAsync(dc, hc.data(), count * sizeof(u64), cudaMemcpyHostToDevice, st));
    // chunk 0's start value is acc "before index 0": the replay starts from 0.0 there
    k_sample_in_chunk<<<unsigned((count + 127) / 128), 128, 0, st>>>(amps, dim, du, dc, ds, count, dout);
    check_launch("k_sample_in_chunk");
    QCS_CUDA(cudaMemcpyAsync(out, dout, count * sizeof(u64), cudaMemcpyDeviceToHost, st));
    QCS_CUDA(cudaFreeAsync(du, st));
    QCS_CUDA(cudaFreeAsync(ds, st));
    QCS_CUDA(cudaFreeAsync(dc, st));
    QCS_CUDA(cudaFreeAsync(dout, st));
    QCS_CUDA(cudaStreamSynchronize(st));
}

u64 sample_chunk() { return kChunk; }

}  // namespace qcs
