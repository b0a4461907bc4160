// abi.cpp -- the extern "C" boundary (include/qcs_abi.h).  Every entry point converts the
// library's exceptions into status codes plus a thread-local message, mirroring how the
// reference surfaces SimError subclasses (core.hpp:13-36; the CLI prints them, qcsim_cli.cpp:435).
#include <cmath>
#include <cstring>
#include <new>
#include <string>

#include "engine.hpp"

namespace {

thread_local std::string g_last_error;

template <class F>
int guarded(F&& f) {
    try {
        f();
        g_last_error.clear();
        return QCS_OK;
    } catch (const qcs::Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "host allocation failed";
        return QCS_ERR_CAPACITY;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return QCS_ERR_SIM;
    }
}

void need(const void* p, const char* what) {
    if (!p) qcs::raise(QCS_ERR_ARG, std::string("null argument: ") + what);
}

}  // namespace

extern "C" {

const char* qcs_last_error(void) { return g_last_error.c_str(); }
const char* qcs_version(void) { return "qcs_b200 0.1 (sm_100a)"; }

int qcs_device_count(int* count) {
    return guarded([&] {
        need(count, "count");
        QCS_CUDA(cudaGetDeviceCount(count));
    });
}

int qcs_set_dense_cap(uint64_t cap) {
    qcs::set_dense_cap(cap);
    return QCS_OK;
}
uint64_t qcs_dense_cap(void) { return qcs::dense_cap(); }

// ---------------------------------------------------------------- catalog

int qcs_gate_catalog_size(void) { return qcs::catalog_size(); }

int qcs_gate_catalog_entry(int index, const char** name, int* arity, int* param_count, double* zero_ratio) {
    return guarded([&] {
        need(name, "name");
        need(arity, "arity");
        need(param_count, "param_count");
        need(zero_ratio, "zero_ratio");
        qcs::catalog_entry(index, name, arity, param_count, zero_ratio);
    });
}

int qcs_gate_lookup(const char* name, const double* params, int num_params, double* matrix_out, int* arity_out,
                    const char** canonical_name) {
    return guarded([&] {
        need(name, "name");
        need(matrix_out, "matrix_out");
        need(arity_out, "arity_out");
        if (num_params < 0 || (num_params > 0 && !params)) qcs::raise(QCS_ERR_ARG, "bad parameter list");
        std::vector<qcs::cplx> m;
        const char* canon = qcs::gate_lookup(name, std::vector<double>(params, params + num_params), m, arity_out);
        std::memcpy(matrix_out, m.data(), m.size() * sizeof(qcs::cplx));
        if (canonical_name) *canonical_name = canon;
    });
}

int qcs_canonical_params(const char* name, double* out, int* count) {
    return guarded([&] {
        need(name, "name");
        need(out, "out");
        need(count, "count");
        const auto p = qcs::canonical_params(name);
        *count = int(p.size());
        std::copy(p.begin(), p.end(), out);
    });
}

// ---------------------------------------------------------------- state

int qcs_state_create(int n, int device, uint64_t basis_index, qcs_state** out) {
    return guarded([&] {
        need(out, "out");
        *out = qcs::state_create(n, device, basis_index);
    });
}

int qcs_state_wrap(int n, int device, void* device_amps, void* cuda_stream, qcs_state** out) {
    return guarded([&] {
        need(out, "out");
        *out = qcs::state_wrap(n, device, device_amps, cuda_stream);
    });
}

int qcs_state_destroy(qcs_state* s) {
    delete s;
    return QCS_OK;
}

int qcs_state_info(const qcs_state* s, int* n, int* device, void** device_amps, void** stream) {
    return guarded([&] {
        need(s, "state");
        if (n) *n = s->n;
        if (device) *device = s->device;
        if (device_amps) *device_amps = s->amps;
        if (stream) *stream = s->stream;
    });
}

int qcs_state_set_basis(qcs_state* s, uint64_t basis_index) {
    return guarded([&] {
        need(s, "state");
        const uint64_t dim = uint64_t(1) << s->n;
        if (basis_index >= dim) qcs::raise(QCS_ERR_DIMENSION, "initial basis index out of range");
        qcs::DeviceGuard g(s->device);
        qcs::fill_basis(s->amps, dim, basis_index, s->stream);
    });
}

int qcs_state_random(qcs_state* s, uint64_t seed) {
    return guarded([&] {
        need(s, "state");
        qcs::DeviceGuard g(s->device);
        const uint64_t dim = uint64_t(1) << s->n;
        qcs::fill_random(s->amps, dim, seed, s->stream);
        const double n2 = qcs::reduce_norm2(s->amps, s->n, static_cast<double*>(s->scratch), s->stream);
        qcs::scale(s->amps, dim, 1.0 / std::sqrt(n2), s->stream);
    });
}

namespace {
void check_range(const qcs_state* s, uint64_t first, uint64_t count) {
    const uint64_t dim = uint64_t(1) << s->n;
    if (first > dim || count > dim - first) qcs::raise(QCS_ERR_DIMENSION, "amplitude range out of bounds");
}

// Work enqueued on s from now on starts after everything enqueued on `other` so far: an event on
// other's stream, waited on by s's stream (the host does not block).
void cross_wait(qcs_state* s, const qcs_state* other) {
    if (s == other || s->stream == other->stream) return;
    cudaEvent_t ev = nullptr;
    {
        qcs::DeviceGuard g(other->device);
        QCS_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        const cudaError_t e = cudaEventRecord(ev, other->stream);
        if (e != cudaSuccess) {
            cudaEventDestroy(ev);
            QCS_CUDA(e);
        }
    }
    qcs::DeviceGuard g(s->device);
    const cudaError_t e = cudaStreamWaitEvent(s->stream, ev, 0);
    cudaEventDestroy(ev);  // the wait stays valid (the event completes on its own)
    QCS_CUDA(e);
}
}  // namespace

int qcs_state_upload(qcs_state* s, const double* host, uint64_t first, uint64_t count) {
    return guarded([&] {
        need(s, "state");
        need(host, "host");
        check_range(s, first, count);
        qcs::DeviceGuard g(s->device);
        QCS_CUDA(cudaMemcpyAsync(s->amps + first, host, count * sizeof(double2), cudaMemcpyHostToDevice, s->stream));
    });
}

int qcs_state_download(qcs_state* s, double* host, uint64_t first, uint64_t count) {
    return guarded([&] {
        need(s, "state");
        need(host, "host");
        check_range(s, first, count);
        qcs::DeviceGuard g(s->device);
        QCS_CUDA(cudaMemcpyAsync(host, s->amps + first, count * sizeof(double2), cudaMemcpyDeviceToHost, s->stream));
        QCS_CUDA(cudaStreamSynchronize(s->stream));
    });
}

int qcs_state_download_async(qcs_state* s, double* host, uint64_t first, uint64_t count) {
    return guarded([&] {
        need(s, "state");
        need(host, "host");
        check_range(s, first, count);
        cudaPointerAttributes attr{};
        if (cudaPointerGetAttributes(&attr, host) != cudaSuccess || attr.type != cudaMemoryTypeHost) {
            cudaGetLastError();
            qcs::raise(QCS_ERR_ARG, "asynchronous download needs pinned host memory (qcs_host_alloc)");
        }
        qcs::DeviceGuard g(s->device);
        QCS_CUDA(cudaMemcpyAsync(host, s->amps + first, count * sizeof(double2), cudaMemcpyDeviceToHost, s->stream));
    });
}

int qcs_state_wait(qcs_state* s, const qcs_state* other) {
    return guarded([&] {
        need(s, "state");
        need(other, "other");
        cross_wait(s, other);
    });
}

int qcs_state_copy(qcs_state* dst, const qcs_state* src) {
    return guarded([&] {
        need(dst, "dst");
        need(src, "src");
        if (dst->n != src->n) qcs::raise(QCS_ERR_DIMENSION, "state copy qubit count mismatch");
        if (dst == src) return;
        // device-side ordering both ways, the host never blocks: the copy (on dst's stream)
        // starts after src's pending work, and src's later work starts after the copy has read it
        auto* s = const_cast<qcs_state*>(src);
        cross_wait(dst, s);
        {
            qcs::DeviceGuard g(dst->device);
            QCS_CUDA(cudaMemcpyAsync(dst->amps, src->amps, (sizeof(double2)) << src->n, cudaMemcpyDefault, dst->stream));
        }
        cross_wait(s, dst);
    });
}

int qcs_state_sync(qcs_state* s) {
    return guarded([&] {
        need(s, "state");
        qcs::DeviceGuard g(s->device);
        QCS_CUDA(cudaStreamSynchronize(s->stream));
        QCS_CUDA(cudaGetLastError());
    });
}

int qcs_host_alloc(size_t bytes, void** out) {
    return guarded([&] {
        need(out, "out");
        const cudaError_t e = cudaHostAlloc(out, bytes, cudaHostAllocPortable);
        if (e != cudaSuccess) {
            cudaGetLastError();
            qcs::raise(QCS_ERR_CAPACITY, std::string("pinned host allocation failed: ") + cudaGetErrorString(e));
        }
    });
}

int qcs_host_free(void* p) {
    return guarded([&] {
        if (p) QCS_CUDA(cudaFreeHost(p));
    });
}

// ---------------------------------------------------------------- steps

int qcs_apply_step(qcs_state* s, const qcs_placement* placements, int count) {
    return guarded([&] {
        need(s, "state");
        qcs::apply_step(s, placements, count);
    });
}

int qcs_apply_diag(qcs_state* s, const uint64_t* flipped, uint64_t count, int flip_rest) {
    return guarded([&] {
        need(s, "state");
        qcs::apply_diag(s, flipped, count, flip_rest);
    });
}

int qcs_apply_split(qcs_state* s, void* peer_amps, int self_bit, int num_sel, const int* sel_bits,
                    const double* blocks, uint32_t skip_mask) {
    return guarded([&] {
        need(s, "state");
        qcs::apply_split(s, peer_amps, self_bit, num_sel, sel_bits, blocks, skip_mask);
    });
}

int qcs_swap_peer(qcs_state* s, uint64_t offset, void* peer_amps, uint64_t count) {
    return guarded([&] {
        need(s, "state");
        if (count && !peer_amps) qcs::raise(QCS_ERR_ARG, "null peer block");
        check_range(s, offset, count);
        qcs::DeviceGuard g(s->device);
        qcs::TimerScope ts(s);
        qcs::launch_swap_peer(s->amps + offset, static_cast<double2*>(peer_amps), count, s->stream);
    });
}

int qcs_apply_rh(qcs_state* s) {
    return guarded([&] {
        need(s, "state");
        qcs::apply_rh(s);
    });
}

int qcs_rh_mvm(qcs_state* s, int n, double value, int sign_method, uint64_t block_size, uint64_t* sign_count,
               uint64_t* madd_count) {
    return guarded([&] {
        need(s, "state");
        qcs::rh_mvm(s, n, value, sign_method, block_size, sign_count, madd_count);
    });
}

// ---------------------------------------------------------------- reductions

int qcs_norm(qcs_state* s, double* out) {
    return guarded([&] {
        need(s, "state");
        need(out, "out");
        qcs::DeviceGuard g(s->device);
        *out = std::sqrt(qcs::reduce_norm2(s->amps, s->n, static_cast<double*>(s->scratch), s->stream));
    });
}

int qcs_probabilities(qcs_state* s, double* out, int mem) {
    return guarded([&] {
        need(s, "state");
        need(out, "out");
        qcs::DeviceGuard g(s->device);
        const uint64_t dim = uint64_t(1) << s->n;
        if (mem == QCS_MEM_DEVICE) {
            qcs::probabilities(s->amps, dim, out, s->stream);
            return;
        }
        double* tmp = nullptr;
        QCS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&tmp), dim * sizeof(double), s->stream));
        qcs::probabilities(s->amps, dim, tmp, s->stream);
        QCS_CUDA(cudaMemcpyAsync(out, tmp, dim * sizeof(double), cudaMemcpyDeviceToHost, s->stream));
        QCS_CUDA(cudaFreeAsync(tmp, s->stream));
        QCS_CUDA(cudaStreamSynchronize(s->stream));
    });
}

int qcs_state_distance(qcs_state* a, qcs_state* b, double* max_abs, double* l2) {
    return guarded([&] {
        need(a, "a");
        need(b, "b");
        need(max_abs, "max_abs");
        need(l2, "l2");
        if (a->n != b->n) qcs::raise(QCS_ERR_DIMENSION, "state distance qubit count mismatch");
        if (a->device != b->device) qcs::raise(QCS_ERR_ARG, "states on different devices");
        cross_wait(a, b);
        qcs::DeviceGuard g(a->device);
        qcs::distance(a->amps, b->amps, uint64_t(1) << a->n, max_abs, l2, a->stream);
        cross_wait(b, a);
    });
}

int qcs_argmax(qcs_state* s, uint64_t* index, double* probability) {
    return guarded([&] {
        need(s, "state");
        need(index, "index");
        need(probability, "probability");
        qcs::DeviceGuard g(s->device);
        qcs::argmax(s->amps, uint64_t(1) << s->n, index, probability, s->scratch, s->stream);
    });
}

int qcs_topk(qcs_state* s, int k, uint64_t* indices, double* probabilities) {
    return guarded([&] {
        need(s, "state");
        need(indices, "indices");
        need(probabilities, "probabilities");
        if (k < 1 || k > 16) qcs::raise(QCS_ERR_ARG, "top-k supports 1 <= k <= 16");
        if (s->summary_k) qcs::raise(QCS_ERR_ARG, "a summary of this state is pending");
        qcs::DeviceGuard g(s->device);
        if (!s->summary_host) QCS_CUDA(cudaHostAlloc(&s->summary_host, qcs::topk_host_bytes(16), cudaHostAllocDefault));
        qcs::topk_begin(s->amps, uint64_t(1) << s->n, k, false, s->summary_host, s->stream);
        QCS_CUDA(cudaStreamSynchronize(s->stream));
        qcs::topk_finish(s->summary_host, k, false, indices, probabilities, nullptr);
    });
}

int qcs_summary(qcs_state* s, int k, double* norm, uint64_t* indices, double* probabilities) {
    return guarded([&] {
        need(s, "state");
        need(norm, "norm");
        need(indices, "indices");
        need(probabilities, "probabilities");
        if (k < 1 || k > 16) qcs::raise(QCS_ERR_ARG, "top-k supports 1 <= k <= 16");
        if (s->summary_k) qcs::raise(QCS_ERR_ARG, "a summary of this state is already pending");
        qcs::DeviceGuard g(s->device);
        // the block candidates land in the state's pinned buffer (a pageable destination makes the
        // copy a staged, synchronous one: ~0.4 ms per call, more than a small circuit's passes)
        if (!s->summary_host) QCS_CUDA(cudaHostAlloc(&s->summary_host, qcs::topk_host_bytes(16), cudaHostAllocDefault));
        qcs::topk_begin(s->amps, uint64_t(1) << s->n, k, true, s->summary_host, s->stream);
        QCS_CUDA(cudaStreamSynchronize(s->stream));
        qcs::topk_finish(s->summary_host, k, true, indices, probabilities, norm);
    });
}

int qcs_sample(qcs_state* s, uint64_t seed, uint64_t count, uint64_t* out, double* total) {
    return guarded([&] {
        need(s, "state");
        if (count) need(out, "out");
        qcs::DeviceGuard g(s->device);
        qcs::sample(s->amps, uint64_t(1) << s->n, seed, count, out, total, s->stream);
    });
}

int qcs_summary_begin(qcs_state* s, int k) {
    return guarded([&] {
        need(s, "state");
        if (k < 1 || k > 16) qcs::raise(QCS_ERR_ARG, "top-k supports 1 <= k <= 16");
        if (s->summary_k) qcs::raise(QCS_ERR_ARG, "a summary of this state is already pending");
        qcs::DeviceGuard g(s->device);
        if (!s->summary_host) QCS_CUDA(cudaHostAlloc(&s->summary_host, qcs::topk_host_bytes(16), cudaHostAllocDefault));
        if (!s->summary_done) QCS_CUDA(cudaEventCreateWithFlags(&s->summary_done, cudaEventDisableTiming));
        qcs::topk_begin(s->amps, uint64_t(1) << s->n, k, true, s->summary_host, s->stream);
        QCS_CUDA(cudaEventRecord(s->summary_done, s->stream));
        s->summary_k = k;
    });
}

int qcs_summary_end(qcs_state* s, double* norm, uint64_t* indices, double* probabilities) {
    return guarded([&] {
        need(s, "state");
        need(norm, "norm");
        need(indices, "indices");
        need(probabilities, "probabilities");
        if (!s->summary_k) qcs::raise(QCS_ERR_ARG, "no summary of this state is pending");
        qcs::DeviceGuard g(s->device);
        const int k = s->summary_k;
        s->summary_k = 0;
        QCS_CUDA(cudaEventSynchronize(s->summary_done));
        qcs::topk_finish(s->summary_host, k, true, indices, probabilities, norm);
    });
}

int qcs_gather(qcs_state* s, const uint64_t* indices, uint64_t count, double* out) {
    return guarded([&] {
        need(s, "state");
        if (!count) return;
        need(indices, "indices");
        need(out, "out");
        const uint64_t dim = uint64_t(1) << s->n;
        for (uint64_t i = 0; i < count; ++i)
            if (indices[i] >= dim) qcs::raise(QCS_ERR_DIMENSION, "gather index out of range");
        qcs::DeviceGuard g(s->device);
        uint64_t* idx = nullptr;
        double2* buf = nullptr;
        QCS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&idx), count * sizeof(uint64_t), s->stream));
        QCS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&buf), count * sizeof(double2), s->stream));
        QCS_CUDA(cudaMemcpyAsync(idx, indices, count * sizeof(uint64_t), cudaMemcpyHostToDevice, s->stream));
        qcs::gather(s->amps, idx, count, buf, s->stream);
        QCS_CUDA(cudaMemcpyAsync(out, buf, count * sizeof(double2), cudaMemcpyDeviceToHost, s->stream));
        QCS_CUDA(cudaFreeAsync(idx, s->stream));
        QCS_CUDA(cudaFreeAsync(buf, s->stream));
        QCS_CUDA(cudaStreamSynchronize(s->stream));
    });
}

// ---------------------------------------------------------------- circuits

int qcs_simulate(qcs_state* s, const qcs_step* steps, int num_steps, int engine, const qcs_sim_options* opts,
                 qcs_step_report* reports) {
    return guarded([&] {
        need(s, "state");
        qcs::simulate(s, steps, num_steps, engine, opts, reports);
    });
}

int qcs_memory_report(int n, const qcs_step* steps, int num_steps, int engine, qcs_step_report* reports) {
    return guarded([&] {
        need(reports, "reports");
        qcs::memory_report(n, steps, num_steps, engine, reports);
    });
}

int qcs_plan_stats(int n, const qcs_step* steps, int num_steps, int engine, const qcs_sim_options* opts,
                   qcs_plan_info* out) {
    return guarded([&] {
        need(out, "out");
        qcs::plan_stats(n, steps, num_steps, engine, opts, out);
    });
}

int qcs_set_jit_mode(int mode) {
    return guarded([&] { qcs::set_jit_mode(mode); });
}
int qcs_get_jit_mode(void) { return qcs::jit_mode(); }
int qcs_set_pipeline_mode(int mode) {
    return guarded([&] { qcs::set_pipeline_mode(mode); });
}
int qcs_get_pipeline_mode(void) { return qcs::pipeline_mode(); }

int qcs_plan_compile(int n, const qcs_step* steps, int num_steps, int engine, const qcs_sim_options* opts,
                     int64_t* kernels, int64_t* cubin_bytes) {
    return guarded([&] {
        need(kernels, "kernels");
        need(cubin_bytes, "cubin_bytes");
        qcs::plan_compile(n, steps, num_steps, engine, opts, kernels, cubin_bytes);
    });
}

int qcs_plan_verify(int n, const qcs_step* steps, int num_steps, int engine, const qcs_sim_options* opts,
                    int64_t* passes) {
    return guarded([&] {
        need(passes, "passes");
        int64_t bytes = 0;
        qcs::plan_compile(n, steps, num_steps, engine, opts, passes, &bytes, true);
    });
}

// ---------------------------------------------------------------- compressed structures

int qcs_step_dax(int n, const qcs_placement* placements, int num_placements, int device, uint64_t* rows,
                 uint64_t* cols, double* values, uint64_t capacity, int mem, uint64_t* count) {
    return guarded([&] {
        need(count, "count");
        if (capacity) {
            need(rows, "rows");
            need(cols, "cols");
            need(values, "values");
        }
        *count = qcs::step_encode(n, placements, num_placements, device, false, capacity, rows, cols, values, nullptr,
                                  nullptr, mem == QCS_MEM_DEVICE);
        if (capacity && *count > capacity) qcs::raise(QCS_ERR_CAPACITY, "output capacity below the entry count");
    });
}

int qcs_step_das(int n, const qcs_placement* placements, int num_placements, int device, uint64_t* dis,
                 uint8_t* last_in_row, double* values, uint64_t capacity, int mem, uint64_t* count) {
    return guarded([&] {
        need(count, "count");
        if (capacity) {
            need(dis, "dis");
            need(last_in_row, "last_in_row");
            need(values, "values");
        }
        *count = qcs::step_encode(n, placements, num_placements, device, true, capacity, nullptr, nullptr, values, dis,
                                  last_in_row, mem == QCS_MEM_DEVICE);
        if (capacity && *count > capacity) qcs::raise(QCS_ERR_CAPACITY, "output capacity below the entry count");
    });
}

}  // extern "C"

namespace {

template <class T>
struct Staged {  // device view of a host or device array
    T* dev = nullptr;
    bool owned = false;
    cudaStream_t s;
    Staged(const T* p, uint64_t n, int mem, cudaStream_t st) : s(st) {
        if (mem == QCS_MEM_DEVICE || n == 0) {
            dev = const_cast<T*>(p);
            return;
        }
        QCS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dev), n * sizeof(T), s));
        owned = true;
        QCS_CUDA(cudaMemcpyAsync(dev, p, n * sizeof(T), cudaMemcpyHostToDevice, s));
    }
    ~Staged() {
        if (owned) cudaFreeAsync(dev, s);
    }
};

void mvm_prologue(const qcs_state* in, qcs_state* out) {
    need(in, "in");
    need(out, "out");
    if (in->n != out->n) qcs::raise(QCS_ERR_DIMENSION, "MVM shape mismatch");
    if (in->device != out->device) qcs::raise(QCS_ERR_ARG, "in/out states on different devices");
    if (in->amps == out->amps) qcs::raise(QCS_ERR_ARG, "MVM is out-of-place: in and out must differ");
}

}  // namespace

extern "C" {

int qcs_dax_mvm(const uint64_t* rows, const uint64_t* cols, const double* values, uint64_t count, int mem,
                const qcs_state* in, qcs_state* out) {
    return guarded([&] {
        mvm_prologue(in, out);
        if (count) {
            need(rows, "rows");
            need(cols, "cols");
            need(values, "values");
        }
        qcs::DeviceGuard g(out->device);
        QCS_CUDA(cudaStreamSynchronize(in->stream));
        Staged<uint64_t> r(rows, count, mem, out->stream), c(cols, count, mem, out->stream);
        Staged<double2> v(reinterpret_cast<const double2*>(values), count, mem, out->stream);
        qcs::dax_mvm(r.dev, c.dev, v.dev, count, in->amps, out->amps, uint64_t(1) << out->n,
                     static_cast<int*>(out->scratch), out->stream);
    });
}

int qcs_das_mvm(const uint64_t* dis, const uint8_t* last_in_row, const double* values, uint64_t count, int mem,
                const qcs_state* in, qcs_state* out) {
    return guarded([&] {
        mvm_prologue(in, out);
        if (count) {
            need(dis, "dis");
            need(last_in_row, "last_in_row");
            need(values, "values");
        }
        qcs::DeviceGuard g(out->device);
        QCS_CUDA(cudaStreamSynchronize(in->stream));
        Staged<uint64_t> d(dis, count, mem, out->stream);
        Staged<uint8_t> l(last_in_row, count, mem, out->stream);
        Staged<double2> v(reinterpret_cast<const double2*>(values), count, mem, out->stream);
        qcs::das_mvm(d.dev, l.dev, v.dev, count, in->amps, out->amps, uint64_t(1) << out->n,
                     static_cast<int*>(out->scratch), out->stream);
    });
}

// ---------------------------------------------------------------- profiling hooks

uint64_t qcs_kernel_launches(void) { return qcs::launches(); }

int qcs_timing_enable(qcs_state* s, int enable) {
    return guarded([&] {
        need(s, "state");
        qcs::DeviceGuard g(s->device);
        qcs::timing_enable(s, enable != 0);
    });
}

int qcs_timing_reset(qcs_state* s) {
    return guarded([&] {
        need(s, "state");
        qcs::DeviceGuard g(s->device);
        qcs::timing_reset(s);
    });
}

int qcs_timing_count(qcs_state* s, int* count) {
    return guarded([&] {
        need(s, "state");
        need(count, "count");
        qcs::DeviceGuard g(s->device);
        *count = qcs::timing_count(s);
    });
}

int qcs_timing_entry(qcs_state* s, int index, const char** kernel_class, uint64_t* launches, double* total_ms,
                     double* algorithmic_bytes) {
    return guarded([&] {
        need(s, "state");
        need(kernel_class, "kernel_class");
        need(launches, "launches");
        need(total_ms, "total_ms");
        need(algorithmic_bytes, "algorithmic_bytes");
        qcs::timing_entry(s, index, kernel_class, launches, total_ms, algorithmic_bytes);
    });
}

int qcs_event_record(qcs_state* s, int slot) {
    return guarded([&] {
        need(s, "state");
        if (slot < 0 || slot >= 8) qcs::raise(QCS_ERR_ARG, "event slot must be 0..7");
        qcs::DeviceGuard g(s->device);
        QCS_CUDA(cudaEventRecord(s->events[slot], s->stream));
    });
}

int qcs_event_elapsed_ms(qcs_state* s, int slot_begin, int slot_end, float* ms) {
    return guarded([&] {
        need(s, "state");
        need(ms, "ms");
        if (slot_begin < 0 || slot_begin >= 8 || slot_end < 0 || slot_end >= 8)
            qcs::raise(QCS_ERR_ARG, "event slot must be 0..7");
        qcs::DeviceGuard g(s->device);
        QCS_CUDA(cudaEventSynchronize(s->events[slot_end]));
        QCS_CUDA(cudaEventElapsedTime(ms, s->events[slot_begin], s->events[slot_end]));
    });
}

}  // extern "C"
