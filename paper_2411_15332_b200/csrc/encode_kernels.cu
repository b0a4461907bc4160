// encode_kernels.cu -- the device gate encoder and compressed MVMs (sm_100a).
//
// step_matrix_dax / step_matrix_das (engine.cpp:135-151) build the step operator as a left
// fold of dax_mtp / das_mtp over per-qubit-position factors (dax.cpp:58-94, das.cpp:83-129):
// 2^n x 2^n operators, serially.  Row r of that fold is known in closed form: the Cartesian
// product of each factor's nonzeros in the factor's own row of r, enumerated with the first
// factor outermost (which is ascending column order), each value the left fold of the factor
// values -- 2x2 identities included, because their (1+0i) products decide signed zeros --
// and exact-zero products dropped (dax.cpp:80-81).  So the encoder is one thread per row:
// a counting pass, an exclusive scan, and an emitting pass, byte-identical to the reference.
//
// dax_mvm / das_mvm (dax.cpp:96-103, das.cpp:131-150) on explicit entries: one thread per row
// accumulates that row's entries in stream order, the reference's order.  The DAS cursor scan
// is parallelised by prefix sums: row(e) = #row flags before e, col(e) = sum of (dis + 1)
// since the row start, minus one.
#include <cub/device/device_scan.cuh>

#include <cstdint>

#include "common.hpp"
#include "kernels.hpp"

namespace qcs {
namespace {

using u64 = std::uint64_t;

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                        __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}

// Enumerate the entries of row r; visit(col, value) for every nonzero product in
// enumeration order.  Returns the number visited.
template <class Visit>
__device__ u64 row_entries(const EncodeStep& st, u64 r, Visit&& visit) {
    const int np = st.np, n = st.n;
    int g[64], idx[64];
    for (int e = 0; e < np; ++e) {
        const int j = st.order[e];
        const EncodePlacement& p = st.p[j];
        int gg = 0;
        for (int i = 0; i < p.k; ++i) gg |= int((r >> p.pos[i]) & 1) << (p.k - 1 - i);
        g[j] = gg;
        idx[e] = 0;
        if (p.nnz[gg] == 0) return 0;
    }
    // placement j -> its slot in the enumeration order
    int slot[64];
    for (int e = 0; e < np; ++e) slot[st.order[e]] = e;
    const u64 base = r & ~st.gate_mask;
    u64 count = 0;
    for (;;) {
        u64 col = base;
        for (int e = 0; e < np; ++e) {
            const int j = st.order[e];
            const EncodePlacement& p = st.p[j];
            const int c = p.col[g[j]][idx[e]];
            for (int i = 0; i < p.k; ++i) col |= u64((c >> (p.k - 1 - i)) & 1) << p.pos[i];
        }
        double2 v = make_double2(1.0, 0.0);
        for (int f = 0; f < st.nfold; ++f) {
            const int j = st.fold_gate[f];
            if (j < 0) {
                // an identity factor (1 + 0i) returns v bit for bit unless a component is -0
                // (x - (-0*0) / (+0) + (-0) can turn -0 into +0): only then multiply
                const bool neg_zero = (v.x == 0.0 && signbit(v.x)) || (v.y == 0.0 && signbit(v.y));
                if (f > 0 && !neg_zero) continue;
                v = f == 0 ? make_double2(1.0, 0.0) : cmul(v, make_double2(1.0, 0.0));
                continue;
            }
            const double2 fv = st.p[j].val[g[j]][idx[slot[j]]];
            v = f == 0 ? fv : cmul(v, fv);
        }
        (void)n;
        if (v.x != 0.0 || v.y != 0.0) {
            visit(count, col, v);
            ++count;
        }
        int e = np - 1;
        while (e >= 0) {
            const int j = st.order[e];
            if (++idx[e] < st.p[j].nnz[g[j]]) break;
            idx[e] = 0;
            --e;
        }
        if (e < 0) break;
    }
    return count;
}

__global__ void k_encode_count(const EncodeStep* __restrict__ stp, u64 dim, u64* __restrict__ counts) {
    const EncodeStep& st = *stp;
    const u64 stride = u64(gridDim.x) * blockDim.x;
    for (u64 r = u64(blockIdx.x) * blockDim.x + threadIdx.x; r < dim; r += stride)
        counts[r] = row_entries(st, r, [](u64, u64, double2) {});
}

__global__ void k_encode_emit(const EncodeStep* __restrict__ stp, u64 dim, const u64* __restrict__ offsets,
                              u64* __restrict__ rows, u64* __restrict__ cols, double2* __restrict__ vals) {
    const EncodeStep& st = *stp;
    const u64 stride = u64(gridDim.x) * blockDim.x;
    for (u64 r = u64(blockIdx.x) * blockDim.x + threadIdx.x; r < dim; r += stride) {
        const u64 o = offsets[r];
        row_entries(st, r, [&](u64 i, u64 col, double2 v) {
            if (rows) rows[o + i] = r;
            cols[o + i] = col;
            vals[o + i] = v;
        });
    }
}

// Placements on interleaved bit positions enumerate out of column order: sort each row's
// segment (insertion sort; segments are short for such steps).
__global__ void k_sort_segments(u64 dim, const u64* __restrict__ offsets, u64* __restrict__ cols,
                                double2* __restrict__ vals) {
    const u64 stride = u64(gridDim.x) * blockDim.x;
    for (u64 r = u64(blockIdx.x) * blockDim.x + threadIdx.x; r < dim; r += stride) {
        const u64 b = offsets[r], e = offsets[r + 1];
        for (u64 i = b + 1; i < e; ++i) {
            const u64 c = cols[i];
            const double2 v = vals[i];
            u64 j = i;
            while (j > b && cols[j - 1] > c) {
                cols[j] = cols[j - 1];
                vals[j] = vals[j - 1];
                --j;
            }
            cols[j] = c;
            vals[j] = v;
        }
    }
}

// DAS stream from the row-sorted DAX entries (das.hpp:13-27).  err = 1 on an all-zero row.
__global__ void k_das_from_dax(u64 dim, const u64* __restrict__ offsets, const u64* __restrict__ cols,
                               u64* __restrict__ dis, std::uint8_t* __restrict__ last, int* err) {
    const u64 stride = u64(gridDim.x) * blockDim.x;
    for (u64 r = u64(blockIdx.x) * blockDim.x + threadIdx.x; r < dim; r += stride) {
        const u64 b = offsets[r], e = offsets[r + 1];
        if (b == e) {
            atomicExch(err, 1);
            continue;
        }
        u64 next = 0;
        for (u64 i = b; i < e; ++i) {
            dis[i] = cols[i] - next;
            next = cols[i] + 1;
            last[i] = i + 1 == e;
        }
    }
}

// ---- dax_mvm: row pointers by binary search over the sorted row array
__global__ void k_dax_check(const u64* __restrict__ rows, const u64* __restrict__ cols, u64 count, u64 dim,
                            int* err) {
    const u64 stride = u64(gridDim.x) * blockDim.x;
    for (u64 e = u64(blockIdx.x) * blockDim.x + threadIdx.x; e < count; e += stride) {
        if (rows[e] >= dim || cols[e] >= dim) atomicExch(err, 1);
        else if (e > 0 && rows[e - 1] > rows[e]) atomicExch(err, 2);
    }
}

__device__ __forceinline__ u64 lower_bound(const u64* a, u64 n, u64 key) {
    u64 lo = 0, hi = n;
    while (lo < hi) {
        const u64 mid = (lo + hi) >> 1;
        if (a[mid] < key) lo = mid + 1; else hi = mid;
    }
    return lo;
}

__global__ void k_dax_mvm(const u64* __restrict__ rows, const u64* __restrict__ cols, const double2* __restrict__ vals,
                          u64 count, const double2* __restrict__ in, double2* __restrict__ out, u64 dim) {
    const u64 stride = u64(gridDim.x) * blockDim.x;
    for (u64 r = u64(blockIdx.x) * blockDim.x + threadIdx.x; r < dim; r += stride) {
        u64 e = lower_bound(rows, count, r);
        double2 acc = make_double2(0.0, 0.0);
        for (; e < count && rows[e] == r; ++e) {
            const double2 p = cmul(vals[e], in[cols[e]]);
            acc = make_double2(__dadd_rn(acc.x, p.x), __dadd_rn(acc.y, p.y));
        }
        out[r] = acc;
    }
}

// ---- das_mvm: row ids and columns by prefix sums
__global__ void k_das_prep(const u64* __restrict__ dis, const std::uint8_t* __restrict__ last, u64 count,
                           u64* __restrict__ flag_u64, u64* __restrict__ step_u64) {
    const u64 stride = u64(gridDim.x) * blockDim.x;
    for (u64 e = u64(blockIdx.x) * blockDim.x + threadIdx.x; e < count; e += stride) {
        flag_u64[e] = last[e] ? 1 : 0;
        step_u64[e] = dis[e] + 1;
    }
}

// rowid = exclusive scan of flags; cum = inclusive scan of (dis+1) (stored exclusive, so
// cum_incl(e) = cum_excl(e) + dis[e] + 1).  The row of entry e starts at the entry after the
// previous flag; row_begin[row] records it.
__global__ void k_das_rows(const std::uint8_t* __restrict__ last, const u64* __restrict__ rowid, u64 count,
                           u64 dim, u64* __restrict__ row_begin, u64* __restrict__ row_end, int* err) {
    const u64 stride = u64(gridDim.x) * blockDim.x;
    for (u64 e = u64(blockIdx.x) * blockDim.x + threadIdx.x; e < count; e += stride) {
        const u64 row = rowid[e];
        if (row >= dim) {
            atomicExch(err, 1);
            continue;
        }
        if (e == 0 || last[e - 1]) row_begin[row] = e;
        if (last[e] || e + 1 == count) row_end[row] = e + 1;
    }
}

__global__ void k_das_mvm(const u64* __restrict__ dis, const double2* __restrict__ vals,
                          const u64* __restrict__ cum_excl, const u64* __restrict__ row_begin,
                          const u64* __restrict__ row_end, const double2* __restrict__ in,
                          double2* __restrict__ out, u64 dim, int* err) {
    const u64 stride = u64(gridDim.x) * blockDim.x;
    for (u64 r = u64(blockIdx.x) * blockDim.x + threadIdx.x; r < dim; r += stride) {
        const u64 b = row_begin[r], e_end = row_end[r];
        double2 acc = make_double2(0.0, 0.0);
        const u64 before = cum_excl[b < e_end ? b : 0];
        for (u64 e = b; e < e_end; ++e) {
            const u64 col = cum_excl[e] + dis[e] - before;
            if (col >= dim) {
                atomicExch(err, 1);
                break;
            }
            const double2 p = cmul(vals[e], in[col]);
            acc = make_double2(__dadd_rn(acc.x, p.x), __dadd_rn(acc.y, p.y));
        }
        out[r] = acc;
    }
}

inline unsigned grid_for(u64 work, int threads) {
    const u64 want = (work + threads - 1) / threads;
    const u64 cap = u64(148) * 32;
    return unsigned(want < 1 ? 1 : (want > cap ? cap : want));
}

// One memory pool per device for the encoder / MVM scratch; it keeps up to 8 GiB mapped
// between calls, so repeated encodes do not pay for mapping fresh memory.
cudaMemPool_t scratch_pool() {
    static cudaMemPool_t pools[64] = {};
    int dev = 0;
    QCS_CUDA(cudaGetDevice(&dev));
    if (dev >= 64) raise(QCS_ERR_ARG, "device index out of range");
    if (!pools[dev]) {
        cudaMemPoolProps props{};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        QCS_CUDA(cudaMemPoolCreate(&pools[dev], &props));
        std::uint64_t keep = std::uint64_t(8) << 30;
        QCS_CUDA(cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &keep));
    }
    return pools[dev];
}

template <class T>
struct DevBuf {  // stream-ordered scratch from scratch_pool(): no cudaMalloc / unmap per call
    T* p = nullptr;
    cudaStream_t s = nullptr;
    DevBuf(u64 n, cudaStream_t st) : s(st) {
        if (n) QCS_CUDA(cudaMallocFromPoolAsync(reinterpret_cast<void**>(&p), n * sizeof(T), scratch_pool(), s));
    }
    ~DevBuf() { if (p) cudaFreeAsync(p, s); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
};

void exclusive_scan(const u64* in, u64* out, u64 n, cudaStream_t s) {
    std::size_t bytes = 0;
    QCS_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, s));
    DevBuf<unsigned char> tmp(bytes, s);
    QCS_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, in, out, n, s));
    note_launch();
    QCS_CUDA(cudaStreamSynchronize(s));
}

}  // namespace

// Encode one step on the device.  Returns the entry count; fills outputs when capacity allows.
u64 encode_step(const EncodeStep& host_step, bool das, u64 capacity, u64* rows_out, u64* cols_out,
                double2* vals_out, u64* dis_out, std::uint8_t* last_out, bool out_on_device, cudaStream_t s) {
    const u64 dim = u64(1) << host_step.n;
    DevBuf<EncodeStep> st(1, s);
    QCS_CUDA(cudaMemcpyAsync(st.p, &host_step, sizeof(EncodeStep), cudaMemcpyHostToDevice, s));
    DevBuf<u64> counts(dim + 1, s), offsets(dim + 1, s);
    QCS_CUDA(cudaMemsetAsync(counts.p + dim, 0, sizeof(u64), s));
    k_encode_count<<<grid_for(dim, 128), 128, 0, s>>>(st.p, dim, counts.p);
    check_launch("k_encode_count");
    exclusive_scan(counts.p, offsets.p, dim + 1, s);
    u64 total = 0;
    QCS_CUDA(cudaMemcpyAsync(&total, offsets.p + dim, sizeof(u64), cudaMemcpyDeviceToHost, s));
    QCS_CUDA(cudaStreamSynchronize(s));
    if (total > capacity) return total;
    // scratch only where the outputs cannot take the entries directly (DAS needs no rows)
    const bool direct = out_on_device && !das;
    DevBuf<u64> rows(direct || das ? 0 : total, s), cols(direct ? 0 : total, s);
    DevBuf<double2> vals(out_on_device ? 0 : total, s);
    double2* v = out_on_device ? vals_out : vals.p;
    u64* rr = direct ? rows_out : rows.p;
    u64* cc = direct ? cols_out : cols.p;
    k_encode_emit<<<grid_for(dim, 128), 128, 0, s>>>(st.p, dim, offsets.p, rr, cc, v);
    check_launch("k_encode_emit");
    if (!host_step.sorted) {
        k_sort_segments<<<grid_for(dim, 128), 128, 0, s>>>(dim, offsets.p, cc, v);
        check_launch("k_sort_segments");
    }
    if (das) {
        DevBuf<int> err(1, s);
        QCS_CUDA(cudaMemsetAsync(err.p, 0, sizeof(int), s));
        DevBuf<u64> dis(out_on_device ? 0 : total, s);
        DevBuf<std::uint8_t> last(out_on_device ? 0 : total, s);
        u64* dd = out_on_device ? dis_out : dis.p;
        std::uint8_t* ll = out_on_device ? last_out : last.p;
        k_das_from_dax<<<grid_for(dim, 128), 128, 0, s>>>(dim, offsets.p, cc, dd, ll, err.p);
        check_launch("k_das_from_dax");
        int h = 0;
        QCS_CUDA(cudaMemcpyAsync(&h, err.p, sizeof(int), cudaMemcpyDeviceToHost, s));
        QCS_CUDA(cudaStreamSynchronize(s));
        if (h) raise(QCS_ERR_ENCODING, "DAS tensor product produced an all-zero row");  // das.cpp:124-125
        if (!out_on_device) {
            QCS_CUDA(cudaMemcpyAsync(dis_out, dd, total * sizeof(u64), cudaMemcpyDeviceToHost, s));
            QCS_CUDA(cudaMemcpyAsync(last_out, ll, total, cudaMemcpyDeviceToHost, s));
        }
    } else if (!out_on_device) {
        QCS_CUDA(cudaMemcpyAsync(rows_out, rr, total * sizeof(u64), cudaMemcpyDeviceToHost, s));
        QCS_CUDA(cudaMemcpyAsync(cols_out, cc, total * sizeof(u64), cudaMemcpyDeviceToHost, s));
    }
    if (!out_on_device) QCS_CUDA(cudaMemcpyAsync(vals_out, v, total * sizeof(double2), cudaMemcpyDeviceToHost, s));
    QCS_CUDA(cudaStreamSynchronize(s));
    return total;
}

void dax_mvm(const u64* rows, const u64* cols, const double2* vals, u64 count, const double2* in, double2* out,
             u64 dim, int* err_dev, cudaStream_t s) {
    QCS_CUDA(cudaMemsetAsync(err_dev, 0, sizeof(int), s));
    if (count) {
        k_dax_check<<<grid_for(count, 256), 256, 0, s>>>(rows, cols, count, dim, err_dev);
        check_launch("k_dax_check");
    }
    int h = 0;
    QCS_CUDA(cudaMemcpyAsync(&h, err_dev, sizeof(int), cudaMemcpyDeviceToHost, s));
    QCS_CUDA(cudaStreamSynchronize(s));
    if (h == 1) raise(QCS_ERR_ENCODING, "DAX entry out of range");
    if (h == 2) raise(QCS_ERR_ENCODING, "DAX entries must be sorted by row");
    k_dax_mvm<<<grid_for(dim, 256), 256, 0, s>>>(rows, cols, vals, count, in, out, dim);
    check_launch("k_dax_mvm");
}

void das_mvm(const u64* dis, const std::uint8_t* last, const double2* vals, u64 count, const double2* in,
             double2* out, u64 dim, int* err_dev, cudaStream_t s) {
    DevBuf<u64> flag(count + 1, s), step(count + 1, s), rowid(count + 1, s), cum(count + 1, s), rb(dim, s), re(dim, s);
    QCS_CUDA(cudaMemsetAsync(err_dev, 0, sizeof(int), s));
    QCS_CUDA(cudaMemsetAsync(rb.p, 0, dim * sizeof(u64), s));
    QCS_CUDA(cudaMemsetAsync(re.p, 0, dim * sizeof(u64), s));
    if (count) {
        k_das_prep<<<grid_for(count, 256), 256, 0, s>>>(dis, last, count, flag.p, step.p);
        check_launch("k_das_prep");
        exclusive_scan(flag.p, rowid.p, count, s);
        exclusive_scan(step.p, cum.p, count, s);
        k_das_rows<<<grid_for(count, 256), 256, 0, s>>>(last, rowid.p, count, dim, rb.p, re.p, err_dev);
        check_launch("k_das_rows");
    }
    k_das_mvm<<<grid_for(dim, 256), 256, 0, s>>>(dis, vals, cum.p, rb.p, re.p, in, out, dim, err_dev);
    check_launch("k_das_mvm");
    int h = 0;
    QCS_CUDA(cudaMemcpyAsync(&h, err_dev, sizeof(int), cudaMemcpyDeviceToHost, s));
    QCS_CUDA(cudaStreamSynchronize(s));
    if (h) raise(QCS_ERR_ENCODING, "malformed DAS stream");  // das.cpp:140
}

}  // namespace qcs
