// engine.cpp -- device state handles, per-step dispatch and simulate() (host side).
//
// Mirrors the reference engine (proj/src/engine.cpp): the same per-step dispatch (RH for an
// all-Hadamard step under rh_dax, engine.cpp:167-175; otherwise the step operator), the same
// StepReport accounting (engine.cpp:82-95, :163-204), the same validation and errors
// (circuit.cpp:41-62).  What changes is where the work happens: operators are never built;
// each step becomes one or a few HBM passes over the device-resident state.
#include "engine.hpp"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>

namespace qcs {

namespace {
std::atomic<u64> g_launches{0};
std::atomic<u64> g_dense_cap{u64(1) << 26};  // kDefaultDenseCap, core.hpp:40
}  // namespace

void note_launch(int n) { g_launches.fetch_add(u64(n), std::memory_order_relaxed); }
u64 launches() { return g_launches.load(); }
u64 dense_cap() { return g_dense_cap.load(std::memory_order_relaxed); }
void set_dense_cap(u64 cap) { g_dense_cap.store(cap, std::memory_order_relaxed); }

DeviceGuard::DeviceGuard(int dev) {
    int cur = -1;
    cuda_check(cudaGetDevice(&cur), "cudaGetDevice (no CUDA device?)");
    if (cur != dev) {
        QCS_CUDA(cudaSetDevice(dev));
        prev = cur;
    }
}
DeviceGuard::~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
}

namespace {

void alloc_aux(qcs_state* s) {
    QCS_CUDA(cudaMalloc(&s->scratch, reduce_scratch_bytes()));
    for (auto& e : s->events) QCS_CUDA(cudaEventCreate(&e));
}

void ensure_flip(qcs_state* s, std::size_t count) {
    if (count <= s->flip_cap) return;
    if (s->flip_buf) QCS_CUDA(cudaFreeAsync(s->flip_buf, s->stream));
    const std::size_t cap = std::max<std::size_t>(count, 64);
    QCS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&s->flip_buf), cap * sizeof(u64), s->stream));
    s->flip_cap = cap;
}

void ensure_ops(qcs_state* s, std::size_t count) {
    if (count <= s->ops_cap) return;
    if (s->ops_buf) QCS_CUDA(cudaFreeAsync(s->ops_buf, s->stream));
    const std::size_t cap = std::max<std::size_t>(count, 16);
    QCS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&s->ops_buf), cap * sizeof(TileOp), s->stream));
    s->ops_cap = cap;
}

}  // namespace

qcs_state* state_create(int n, int device, u64 basis) {
    if (n < 1 || n > 62) raise(QCS_ERR_DIMENSION, "state vector needs 1 <= n <= 62 qubits");  // core.cpp:23
    const u64 dim = u64(1) << n;
    if (basis >= dim) raise(QCS_ERR_DIMENSION, "initial basis index out of range");            // core.cpp:25
    DeviceGuard g(device);
    auto* s = new qcs_state;
    s->n = n;
    s->device = device;
    try {
        QCS_CUDA(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
        s->owns_stream = true;
        if (n > 40) raise(QCS_ERR_CAPACITY, "state of 2^" + std::to_string(n) + " amplitudes exceeds device memory");
        const cudaError_t e = cudaMalloc(&s->amps, sizeof(double2) * dim);
        if (e != cudaSuccess) {
            cudaGetLastError();
            raise(QCS_ERR_CAPACITY, "state of 2^" + std::to_string(n) + " amplitudes (" +
                                        std::to_string(sizeof(double2) * dim) + " B) does not fit in device memory");
        }
        s->owns_mem = true;
        alloc_aux(s);
        fill_basis(s->amps, dim, basis, s->stream);
    } catch (...) {
        delete s;
        throw;
    }
    return s;
}

qcs_state* state_wrap(int n, int device, void* amps, void* stream) {
    if (n < 1 || n > 62) raise(QCS_ERR_DIMENSION, "state vector needs 1 <= n <= 62 qubits");
    if (!amps) raise(QCS_ERR_ARG, "null device pointer");
    DeviceGuard g(device);
    auto* s = new qcs_state;
    s->n = n;
    s->device = device;
    s->amps = static_cast<double2*>(amps);
    s->stream = static_cast<cudaStream_t>(stream);
    try {
        alloc_aux(s);
    } catch (...) {
        delete s;
        throw;
    }
    return s;
}

}  // namespace qcs

qcs_state::~qcs_state() {
    int cur = -1;
    if (cudaGetDevice(&cur) != cudaSuccess) return;
    cudaSetDevice(device);
    if (stream) cudaStreamSynchronize(stream);
    if (timer) qcs::destroy_timer(timer);
    if (flip_buf) cudaFree(flip_buf);
    if (ops_buf) cudaFree(ops_buf);
    if (scratch) cudaFree(scratch);
    for (auto& e : events)
        if (e) cudaEventDestroy(e);
    if (owns_mem && amps) cudaFree(amps);
    if (owns_stream && stream) cudaStreamDestroy(stream);
    cudaSetDevice(cur);
}

namespace qcs {

// ------------------------------------------------------------------ validation (circuit.cpp:41-62)

namespace {

void check_placements(int n, const qcs_placement* p, int count) {
    if (count < 0 || (count > 0 && !p)) raise(QCS_ERR_ARG, "null placement array");
    u64 covered = 0;
    for (int j = 0; j < count; ++j) {
        if (p[j].arity < 1) raise(QCS_ERR_ARG, "placement arity must be >= 1");
        if (p[j].arity > QCS_MAX_ARITY) raise(QCS_ERR_ARG, "placement arity above 3 is not supported");
        if (!p[j].qubits || !p[j].matrix) raise(QCS_ERR_ARG, "placement without qubits or matrix");
        for (int i = 0; i < p[j].arity; ++i) {
            const int q = p[j].qubits[i];
            if (q < 0 || q >= n) raise(QCS_ERR_DIMENSION, "gate placement out of range");
            const u64 bit = u64(1) << q;
            if (covered & bit) raise(QCS_ERR_DIMENSION, "overlapping gate placements in a step");
            covered |= bit;
        }
    }
}

}  // namespace

void validate_circuit(int n, const qcs_step* steps, int nsteps) {
    if (n < 1) raise(QCS_ERR_DIMENSION, "circuit needs n >= 1 qubits");
    if (nsteps < 0 || (nsteps > 0 && !steps)) raise(QCS_ERR_ARG, "null step array");
    const u64 dim = u64(1) << n;
    for (int i = 0; i < nsteps; ++i) {
        const qcs_step& st = steps[i];
        if (st.kind == QCS_STEP_DIAG) {
            if (st.num_flipped && !st.flipped) raise(QCS_ERR_ARG, "null flipped array");
            for (u64 k = 0; k < st.num_flipped; ++k)
                if (st.flipped[k] >= dim) raise(QCS_ERR_DIMENSION, "diagonal step index out of range");
        } else if (st.kind == QCS_STEP_GATES) {
            check_placements(n, st.placements, st.num_placements);
        } else {
            raise(QCS_ERR_ARG, "unknown step kind");
        }
    }
}

// ------------------------------------------------------------------ single steps

void apply_step(qcs_state* s, const qcs_placement* p, int count) {
    check_placements(s->n, p, count);
    DeviceGuard g(s->device);
    TimerScope ts(s);
    // Disjoint placements commute; one in-place pass each.  For one placement (and for steps
    // whose values are exact under products) this equals dax_mvm(step_matrix_dax) bit for bit.
    for (int j = 0; j < count; ++j) {
        const GateOp op = canonical_op(s->n, p[j]);
        GateDesc d;
        if (build_gate_desc(op, d)) launch_gate(s->amps, s->n, d, s->stream);
    }
}

void apply_diag(qcs_state* s, const u64* flipped, u64 count, int flip_rest) {
    const u64 dim = u64(1) << s->n;
    if (count && !flipped) raise(QCS_ERR_ARG, "null flipped array");
    std::vector<u64> f(flipped, flipped + count);
    for (u64 x : f)
        if (x >= dim) raise(QCS_ERR_DIMENSION, "diagonal step index out of range");
    std::sort(f.begin(), f.end());  // CircuitStep::of_diag sorts (circuit.cpp:25)
    f.erase(std::unique(f.begin(), f.end()), f.end());
    DeviceGuard g(s->device);
    TimerScope ts(s);
    if (!flip_rest && f.empty()) return;
    ensure_flip(s, f.size() + 1);
    if (!f.empty())
        QCS_CUDA(cudaMemcpyAsync(s->flip_buf, f.data(), f.size() * sizeof(u64), cudaMemcpyHostToDevice, s->stream));
    if (!flip_rest) launch_negate_listed(s->amps, s->flip_buf, f.size(), s->stream);
    else launch_diag_sign(s->amps, s->n, s->flip_buf, f.size(), 1, s->stream);
    // the host vector may be freed: pageable cudaMemcpyAsync has staged it before returning
}

namespace {

// Walsh-Hadamard plan: tiles of m bits; every tile after the first keeps the low `low` bits
// for coalescing and transforms up to m - low fresh bits.
void plan_rh(int n, std::vector<TilePass>& passes, std::vector<TileOp>& ops) {
    const int m = std::min(n, tile_max_bits());
    const int low = std::min(3, m);
    const double value = std::exp2(-0.5 * n);  // rh_build, rh.cpp:20
    int next = 0;
    while (next < n) {
        TilePass p{};
        p.op_begin = int(ops.size());
        int nb = 0;
        unsigned wmask = 0;
        if (next == 0) {
            for (int b = 0; b < m; ++b) p.bits[nb++] = b;
            wmask = (1u << m) - 1;
            next = m;
            TileOp sc{};
            sc.kind = TOP_SCALE;
            sc.scale = value;  // rh.cpp:99-100: scale first
            ops.push_back(sc);
        } else {
            const int cnt = std::min(m - low, n - next);
            for (int b = 0; b < low; ++b) p.bits[nb++] = b;
            for (int b = 0; b < cnt; ++b) {
                wmask |= 1u << nb;
                p.bits[nb++] = next + b;
            }
            next += cnt;
        }
        p.m = nb;
        TileOp w{};
        w.kind = TOP_WHT;
        w.wht_mask = wmask;
        ops.push_back(w);
        p.op_count = int(ops.size()) - p.op_begin;
        passes.push_back(p);
    }
}

void run_passes(qcs_state* s, const std::vector<TilePass>& passes, const std::vector<TileOp>& ops,
                const std::vector<u64>& flips) {
    ensure_ops(s, ops.size());
    QCS_CUDA(cudaMemcpyAsync(s->ops_buf, ops.data(), ops.size() * sizeof(TileOp), cudaMemcpyHostToDevice, s->stream));
    if (!flips.empty()) {
        ensure_flip(s, flips.size());
        QCS_CUDA(cudaMemcpyAsync(s->flip_buf, flips.data(), flips.size() * sizeof(u64), cudaMemcpyHostToDevice,
                                 s->stream));
    }
    for (const TilePass& p : passes) launch_tile_pass(s->amps, s->n, p, s->ops_buf, s->flip_buf, s->stream);
}

}  // namespace

void apply_rh(qcs_state* s) {
    DeviceGuard g(s->device);
    TimerScope ts(s);
    std::vector<TilePass> passes;
    std::vector<TileOp> ops;
    plan_rh(s->n, passes, ops);
    run_passes(s, passes, ops, {});
}

// ------------------------------------------------------------------ simulate

namespace {

u64 dense_step_bytes(int n) {  // engine.cpp:82-85
    if (2 * n + 4 >= 64) return UINT64_MAX;
    return u64(1) << (2 * n + 4);
}

int nonzeros(const qcs_placement& p) {
    const int dim = 1 << p.arity;
    int z = 0;
    for (int i = 0; i < dim * dim; ++i)
        if (p.matrix[2 * i] != 0.0 || p.matrix[2 * i + 1] != 0.0) ++z;
    return z;
}

// engine.cpp:89-95: product of per-factor nonzero counts (identity fill counts 2)
u64 step_nnz(const qcs_step& st, int n) {
    if (st.kind == QCS_STEP_DIAG) return u64(1) << n;
    u64 nnz = 1;
    int covered = 0;
    for (int j = 0; j < st.num_placements; ++j) {
        nnz *= u64(nonzeros(st.placements[j]));
        covered += st.placements[j].arity;
    }
    for (int q = covered; q < n; ++q) nnz *= 2;
    return nnz;
}

int num_factors(const qcs_step& st, int n) {
    int covered = 0;
    for (int j = 0; j < st.num_placements; ++j) covered += st.placements[j].arity;
    return st.num_placements + (n - covered);
}

bool is_hadamard_all(const qcs_step& st, int n) {  // circuit.cpp:31-39
    if (st.kind != QCS_STEP_GATES || st.num_placements != n) return false;
    u64 covered = 0;
    for (int j = 0; j < st.num_placements; ++j) {
        const qcs_placement& p = st.placements[j];
        if (!p.name || std::strcmp(p.name, "Hadamard") != 0 || p.arity != 1) return false;
        covered |= u64(1) << p.qubits[0];
    }
    return covered == ((n >= 64) ? ~u64(0) : (u64(1) << n) - 1);
}

u64 block_row_cost(int n, u64 b) {  // rh.cpp:51-54
    const u64 half = u64(1) << (n - 1);
    return half / b + b - 1;
}

u64 optimal_block_size(int n) {  // rh.cpp:68-75
    if (n < 2) raise(QCS_ERR_SIM, "block-size optimum needs n >= 2");
    const u64 half = u64(1) << (n - 1);
    u64 best = 1;
    for (u64 b = 1; b <= half; b <<= 1)
        if (block_row_cost(n, b) < block_row_cost(n, best)) best = b;
    return best;
}

// rh_mvm's sign counter totals per method (rh.cpp:110-154; the Table-2 formulas of
// qcsim_cli.cpp:109-118), with the reference's u64 arithmetic.
u64 rh_sign_count(int n, int method, u64 block) {
    const u64 half = u64(1) << (n - 1);
    switch (method) {
        case QCS_SIGN_NONOPT: return 4 * half * half;
        case QCS_SIGN_QUARTER: return half * half;
        case QCS_SIGN_BLOCK: {
            u64 b = block;
            if (b == 0) b = n >= 2 ? optimal_block_size(n) : 1;
            if (b == 0 || (b & (b - 1)) || b > half)
                raise(QCS_ERR_SIM, "block size must be a power of two within the row");  // rh.cpp:58
            return half * (half / b + b - 1);
        }
        case QCS_SIGN_LOGARITHM: return half * u64(n - 1);
        default: raise(QCS_ERR_ARG, "unknown sign method");
    }
}

}  // namespace

void simulate(qcs_state* s, const qcs_step* steps, int nsteps, int engine, const qcs_sim_options* opts,
              qcs_step_report* reports) {
    const int n = s->n;
    validate_circuit(n, steps, nsteps);
    if (engine < QCS_ENGINE_DENSE || engine > QCS_ENGINE_RH_DAX) raise(QCS_ERR_ARG, "unknown engine");
    qcs_sim_options o{QCS_SIGN_LOGARITHM, 0, 1};
    if (opts) o = *opts;
    const u64 dim = u64(1) << n;
    for (int i = 0; i < nsteps; ++i) {
        const qcs_step& st = steps[i];
        qcs_step_report r{};
        r.stage = st.stage;
        r.dense_bytes = dense_step_bytes(n);
        const bool use_rh = engine == QCS_ENGINE_RH_DAX && is_hadamard_all(st, n);
        if (use_rh) {
            r.structure = QCS_STRUCT_RH;
            r.matrix_bytes = 16;  // engine.cpp:173
            r.sign_count = rh_sign_count(n, o.sign_method, o.block_size);
            const u64 half = u64(1) << (n - 1);
            r.madd_count = 4 * half * half;  // rh.cpp:153
            apply_rh(s);
        } else {
            const u64 nnz = step_nnz(st, n);
            if (engine == QCS_ENGINE_DENSE) {
                // the Matrix method materialises 2^n x 2^n (core.cpp:58-60, engine.cpp:56)
                const bool too_big = dim > dense_cap() / dim;
                if (st.kind == QCS_STEP_DIAG && too_big) raise(QCS_ERR_CAPACITY, "diagonal step exceeds dense cap");
                if (st.kind == QCS_STEP_GATES && num_factors(st, n) > 1 && too_big)
                    raise(QCS_ERR_CAPACITY, "dense tensor product exceeds dense cap of " +
                                                std::to_string(dense_cap()) + " elements");
                r.structure = QCS_STRUCT_DENSE;
                r.entry_count = nnz;
                r.matrix_bytes = dim * dim * 16;
                r.madd_count = dim * dim;
            } else {
                r.structure = engine == QCS_ENGINE_DAS ? QCS_STRUCT_DAS : QCS_STRUCT_DAX;
                r.entry_count = nnz;
                r.matrix_bytes = 24 * nnz;  // dax.cpp:105, das.cpp:152
                r.madd_count = nnz;         // engine.cpp:191, :199
            }
            if (st.kind == QCS_STEP_DIAG) apply_diag(s, st.flipped, st.num_flipped, st.flip_rest);
            else apply_step(s, st.placements, st.num_placements);
        }
        if (reports) reports[i] = r;
    }
}

void memory_report(int n, const qcs_step* steps, int nsteps, int engine, qcs_step_report* reports) {
    validate_circuit(n, steps, nsteps);
    for (int i = 0; i < nsteps; ++i) {
        const qcs_step& st = steps[i];
        qcs_step_report r{};
        r.stage = st.stage;
        r.dense_bytes = dense_step_bytes(n);
        if (engine == QCS_ENGINE_RH_DAX && is_hadamard_all(st, n)) {
            r.structure = QCS_STRUCT_RH;
            r.matrix_bytes = 16;
        } else if (engine == QCS_ENGINE_DENSE) {
            r.structure = QCS_STRUCT_DENSE;
            r.matrix_bytes = r.dense_bytes;
            r.entry_count = step_nnz(st, n);
        } else {
            r.structure = engine == QCS_ENGINE_DAS ? QCS_STRUCT_DAS : QCS_STRUCT_DAX;
            r.entry_count = step_nnz(st, n);
            r.matrix_bytes = r.entry_count * 24;
        }
        reports[i] = r;
    }
}

// ------------------------------------------------------------------ device encoder

u64 step_encode(int n, const qcs_placement* p, int count, int device, bool das, u64 capacity, u64* rows, u64* cols,
                double* vals, u64* dis, std::uint8_t* last, bool on_device) {
    if (n < 1 || n > 62) raise(QCS_ERR_DIMENSION, "step needs 1 <= n <= 62 qubits");
    check_placements(n, p, count);
    if (count > 64) raise(QCS_ERR_ARG, "at most 64 placements per encoded step");
    auto st = std::make_unique<EncodeStep>();
    std::memset(st.get(), 0, sizeof(EncodeStep));
    st->n = n;
    st->np = count;
    st->sorted = 1;
    std::vector<int> first(count), carrier(count), contiguous(count);
    for (int j = 0; j < count; ++j) {
        const qcs_placement& pl = p[j];
        EncodePlacement& e = st->p[j];
        e.k = pl.arity;
        int mn = pl.qubits[0];
        contiguous[j] = 1;
        for (int i = 0; i < pl.arity; ++i) {
            e.pos[i] = n - 1 - pl.qubits[i];
            st->gate_mask |= u64(1) << e.pos[i];
            mn = std::min(mn, pl.qubits[i]);
            if (i > 0 && pl.qubits[i] != pl.qubits[i - 1] + 1) contiguous[j] = 0;
        }
        if (!contiguous[j]) st->sorted = 0;
        first[j] = mn;
        carrier[j] = contiguous[j] ? pl.qubits[0] : pl.qubits[pl.arity - 1];
        const int dim = 1 << pl.arity;
        for (int g = 0; g < dim; ++g) {
            int z = 0;
            for (int c = 0; c < dim; ++c) {
                const double re = pl.matrix[2 * (g * dim + c)], im = pl.matrix[2 * (g * dim + c) + 1];
                if (re == 0.0 && im == 0.0) continue;  // dax_encode (dax.cpp:42)
                e.col[g][z] = c;
                e.val[g][z] = make_double2(re, im);
                ++z;
            }
            e.nnz[g] = z;
        }
    }
    std::vector<int> ord(count);
    for (int j = 0; j < count; ++j) ord[j] = j;
    std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return first[a] < first[b]; });
    for (int j = 0; j < count; ++j) st->order[j] = ord[j];
    // fold items in position order (engine.cpp:40-51 for native placements; projector pieces
    // for the others, as oracle/ref_capi.cpp decomposes them)
    int q = 0;
    while (q < n) {
        int item = -1, step = 1;
        for (int j = 0; j < count; ++j)
            if (carrier[j] == q) {
                item = j;
                if (contiguous[j]) step = p[j].arity;
                break;
            }
        st->fold_gate[st->nfold++] = item;
        q += step;
    }
    DeviceGuard g(device);
    cudaStream_t s;
    QCS_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    u64 total = 0;
    try {
        total = encode_step(*st, das, capacity, rows, cols, reinterpret_cast<double2*>(vals), dis, last, on_device, s);
    } catch (...) {
        cudaStreamDestroy(s);
        throw;
    }
    cudaStreamDestroy(s);
    return total;
}

}  // namespace qcs
