// engine.cpp -- device state handles, per-step dispatch and simulate() (host side).
//
// Mirrors the reference engine (proj/src/engine.cpp): the same per-step dispatch (RH for an
// all-Hadamard step under rh_dax, engine.cpp:167-175; otherwise the step operator), the same
// StepReport accounting (engine.cpp:82-95, :163-204), the same validation and errors
// (circuit.cpp:41-62).  What changes is where the work happens: operators are never built;
// each step becomes one or a few HBM passes over the device-resident state.
#include "engine.hpp"
#include "planner.hpp"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <unordered_map>

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

// The library's short-lived device buffers (top-k candidates, gather lists, sampling tables) come
// from the device's default stream-ordered pool.  Its release threshold is 0 by default: every
// synchronisation hands the memory back to the driver and the next cudaMallocAsync is a real
// allocation (~0.2 ms each: a summary of a small state took 0.45 ms for a 27 us kernel).  Keep up
// to 64 MiB cached (once per device; a larger setting made by the application is left alone).
void keep_pool_warm(int device) {
    static std::atomic<unsigned long long> done{0};
    static const bool off = [] { const char* v = std::getenv("QCS_POOL_KEEP"); return v && std::atoi(v) == 0; }();  // A/B switch
    if (off || device < 0 || device >= 64 || (done.load() >> device & 1ull)) return;
    done.fetch_or(1ull << device);
    cudaMemPool_t pool = nullptr;
    if (cudaDeviceGetDefaultMemPool(&pool, device) != cudaSuccess) {
        cudaGetLastError();
        return;
    }
    std::uint64_t cur = 0;
    if (cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &cur) != cudaSuccess) cudaGetLastError();
    std::uint64_t want = std::uint64_t(64) << 20;
    if (cur < want && cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &want) != cudaSuccess) cudaGetLastError();
}

void alloc_aux(qcs_state* s) {
    keep_pool_warm(s->device);
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
    if (plan_buf) cudaFree(plan_buf);
    qcs::delete_plan_cache(plan_cache);
    for (auto& st : stage) {
        if (st.host) cudaFreeHost(st.host);
        if (st.done) cudaEventDestroy(st.done);
    }
    if (scratch) cudaFree(scratch);
    if (summary_host) cudaFreeHost(summary_host);
    if (summary_done) cudaEventDestroy(summary_done);
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

void apply_split(qcs_state* s, void* peer, int self_bit, int nsel, const int* sel, const double* blocks,
                 unsigned skip) {
    if (!peer) raise(QCS_ERR_ARG, "null peer shard");
    if (s->n < 1) raise(QCS_ERR_DIMENSION, "the shard needs a local qubit");
    if (self_bit != 0 && self_bit != 1) raise(QCS_ERR_ARG, "self_bit must be 0 or 1");
    if (nsel < 0 || nsel > 2) raise(QCS_ERR_ARG, "at most two selector bits");
    if (!blocks) raise(QCS_ERR_ARG, "null blocks");
    SplitParams p{};
    p.nl = s->n;
    p.self_bit = self_bit;
    p.nsel = nsel;
    p.skip = skip & ((1u << (1 << nsel)) - 1);
    for (int i = 0; i < nsel; ++i) {
        if (!sel || sel[i] < 0 || sel[i] >= s->n) raise(QCS_ERR_DIMENSION, "selector bit out of range");
        p.sel[i] = sel[i];
    }
    for (int v = 0; v < (1 << nsel); ++v)
        for (int k = 0; k < 4; ++k) {
            const double re = blocks[8 * v + 2 * k], im = blocks[8 * v + 2 * k + 1];
            p.m[v][k] = make_double2(re, im);
            if (re != 0.0 || im != 0.0) p.nz[v] = static_cast<unsigned char>(p.nz[v] | (1u << k));
        }
    DeviceGuard g(s->device);
    TimerScope ts(s);
    launch_split_pair(s->amps, static_cast<double2*>(peer), p, s->stream);
}

namespace {

void ensure_plan(qcs_state* s, std::size_t bytes) {
    if (bytes <= s->plan_cap) return;
    if (s->plan_buf) QCS_CUDA(cudaFreeAsync(s->plan_buf, s->stream));
    const std::size_t cap = std::max<std::size_t>(bytes, 1 << 16);
    QCS_CUDA(cudaMallocAsync(&s->plan_buf, cap, s->stream));
    s->plan_cap = cap;
}

// A single operation outside a tile pass: gates and diagonal gates run the gate kernel (it
// touches only the amplitudes they change), sign steps the diag-sign kernels.
void run_single(qcs_state* s, const FOp& f, const u64* flips_dev, u64 flip_cnt) {
    switch (f.kind) {
        case TOP_GATE:
        case TOP_DIAG: {
            GateDesc d;
            if (build_gate_desc(f.src, d)) launch_gate(s->amps, s->n, d, s->stream);
            return;
        }
        case TOP_WHT: {  // unnormalised butterfly [[1, 1], [1, -1]]: exact a + b, a - b
            GateOp op;
            op.k = 1;
            op.pos[0] = f.tpos[0];
            op.m = {1.0, 1.0, 1.0, -1.0};
            GateDesc d;
            build_gate_desc(op, d);
            launch_gate(s->amps, s->n, d, s->stream);
            return;
        }
        case TOP_SCALE:
            scale(s->amps, u64(1) << s->n, f.scale, s->stream);
            return;
        case TOP_SIGN:
            if (!f.flip_rest) launch_negate_listed(s->amps, flips_dev, flip_cnt, s->stream);
            else launch_diag_sign(s->amps, s->n, flips_dev, flip_cnt, 1, s->stream);
            return;
        default: return;
    }
}

void plan_fused_passes(int n, const std::vector<FOp>& ops, Lowered& low, std::int64_t init = -1);

// support: from a basis state, an amplitude can only become nonzero by flipping bits that
// non-diagonal operations target (gates, butterflies); diagonals and scales never do
void compute_reached(const std::vector<FOp>& ops, Lowered& low) {
    low.reached.assign(low.passes.size(), 0);
    u64 reached = 0;
    for (std::size_t i = 0; i < low.passes.size(); ++i) {
        low.reached[i] = reached;
        for (int idx : low.pass_ops[i]) {
            if (idx >= int(ops.size())) continue;  // a scale the planner added
            const FOp& f = ops[std::size_t(idx)];
            if (f.diagonal) continue;
            for (int k = 0; k < f.K; ++k) reached |= u64(1) << f.tpos[k];
        }
    }
}

void plan_fused(int n, const std::vector<FOp>& ops, Lowered& low, std::int64_t init = -1) {
    plan_fused_passes(n, ops, low, init);
    compute_reached(ops, low);
}

// Deferred qubits.  From a basis state, the amplitudes stay confined to the sub-cube spanned by
// the qubits that non-diagonal operations have targeted so far, and the passes skip every tile
// outside it (apply_support).  So the operations that can run before ANY non-diagonal operation
// on a set D of qubits -- everything outside D's light cone; operations on disjoint qubits and
// diagonal ones commute -- cost 2^-|D| of a sweep each when they run FIRST.  split_deferred
// partitions the list (order kept inside both parts); the two parts are planned separately so
// that no early pass pulls a gate on D in.
void split_deferred(const std::vector<FOp>& ops, u64 D, std::vector<int>& first, std::vector<int>& second) {
    u64 blocked_nd = 0, blocked_d = 0;
    for (std::size_t i = 0; i < ops.size(); ++i) {
        const FOp& f = ops[i];
        u64 targets = 0;
        if (!f.diagonal)
            for (int k = 0; k < f.K; ++k) targets |= u64(1) << f.tpos[k];
        const bool reaches = !f.diagonal && (f.kind == TOP_SIGN || (targets & D));
        const bool conflict = (f.touch & blocked_nd) || (!f.diagonal && (f.touch & blocked_d));
        if (reaches || conflict) {
            second.push_back(int(i));
            (f.diagonal ? blocked_d : blocked_nd) |= f.touch;
        } else {
            first.push_back(int(i));
        }
    }
}

// levels: deferred-qubit counts, decreasing (e.g. {4, 2}: what lies outside the cone of the top 4
// qubits runs first on 1/16 of the state, then what lies outside the cone of the top 2 on a
// quarter, then the rest)
Plan plan_with_levels(int n, const std::vector<FOp>& ops, const std::vector<int>& levels) {
    std::vector<std::vector<int>> parts;
    std::vector<int> rest(ops.size());
    for (std::size_t i = 0; i < ops.size(); ++i) rest[i] = int(i);
    for (int k : levels) {
        const u64 D = ((u64(1) << k) - 1) << (n - k);  // the k highest basis bits (reference qubits 0..k-1)
        std::vector<FOp> sub;
        sub.reserve(rest.size());
        for (int i : rest) sub.push_back(ops[std::size_t(i)]);
        std::vector<int> first, second;
        split_deferred(sub, D, first, second);
        if (first.empty()) continue;
        std::vector<int> a, b;
        for (int i : first) a.push_back(rest[std::size_t(i)]);
        for (int i : second) b.push_back(rest[std::size_t(i)]);
        parts.push_back(std::move(a));
        rest.swap(b);
    }
    if (!rest.empty()) parts.push_back(std::move(rest));
    if (parts.size() < 2) return plan_ops(n, ops, tile_max_bits());
    Plan out;
    for (const std::vector<int>& part : parts) {
        std::vector<FOp> sub;
        sub.reserve(part.size());
        for (int i : part) sub.push_back(ops[std::size_t(i)]);
        Plan p = plan_ops(n, sub, tile_max_bits());
        for (auto& pass : p.passes) {
            for (int& idx : pass.ops) idx = part[std::size_t(idx)];
            out.passes.push_back(std::move(pass));
        }
    }
    return out;
}
Plan plan_with_deferral(int n, const std::vector<FOp>& ops, int k) { return plan_with_levels(n, ops, {k}); }

// Estimated time of a plan run from a basis state (seconds): per pass, the larger of its FP64 time
// and its HBM time over the tiles that compute / load / store under the support masks
// apply_support will set (tiles outside the reached sub-cube are skipped), plus the launch and the
// scheduling of skipped tiles.  A model for choosing between plans, not a prediction: gates count
// 2.2 FP64 instructions per amplitude, other operations 0.4; the pipes run at the fractions the
// C4 passes reach (FP64 0.75 of 148 x 64 lanes at 1.8 GHz, HBM 0.8 of 6.5 TB/s).
double plan_cost_from_basis(int n, const std::vector<FOp>& ops, const Plan& plan) {
    const u64 full = n >= 64 ? ~u64(0) : (u64(1) << n) - 1;
    const std::size_t np = plan.passes.size();
    std::vector<u64> zmask(np + 1, 0);
    u64 reached = 0;
    for (std::size_t i = 0; i < np; ++i) {
        zmask[i] = full & ~plan.passes[i].tile & ~reached;
        for (int idx : plan.passes[i].ops) {
            const FOp& f = ops[std::size_t(idx)];
            if (f.diagonal) continue;
            if (f.kind == TOP_SIGN) reached = full;
            for (int k = 0; k < f.K; ++k) reached |= u64(1) << f.tpos[k];
        }
    }
    double total = 0.0;
    for (std::size_t i = 0; i < np; ++i) {
        const PlannedPass& p = plan.passes[i];
        const int m = __builtin_popcountll(p.tile);
        const double tiles = std::ldexp(1.0, n - m), amps = std::ldexp(1.0, n);
        const double active = std::ldexp(1.0, -__builtin_popcountll(zmask[i]));
        const double written = i + 1 < np ? std::ldexp(1.0, -__builtin_popcountll(zmask[i + 1] & ~p.tile)) : 1.0;
        double fp64_per_amp = 0.0;
        for (int idx : p.ops) {
            const FOp& f = ops[std::size_t(idx)];
            fp64_per_amp += (f.kind == TOP_GATE || f.kind == TOP_WHT) ? 2.2 : 0.4;
        }
        const double t_fp64 = fp64_per_amp * amps * active / (0.75 * 148.0 * 64.0 * 1.8e9);
        const double t_hbm = 16.0 * amps * ((i == 0 ? 0.0 : active) + std::max(written, active)) / (0.8 * 6.5e12);
        total += std::max(t_fp64, t_hbm) + 5e-6 + tiles * 1.4e-9;
    }
    return total;
}

// The plan of a circuit: plan_ops, or -- from a basis state, when the model says so -- the plan
// with 1..3 deferred qubits.  QCS_DEFER: -1 (default) choose by the model, 0 off, k forced.
// The model's choice depends on the circuit's structure only (which operations touch which qubits,
// which are diagonal), not on its angles: a variational loop that sends the same circuit with
// fresh angles pays for the candidate plans once (structure hash -> k; process-wide, bounded).
std::uint64_t structure_hash(int n, const std::vector<FOp>& ops) {
    std::uint64_t h = 1469598103934665603ull ^ std::uint64_t(n);
    auto mix = [&](std::uint64_t v) { h = (h ^ v) * 1099511628211ull; };
    for (const FOp& f : ops) {
        mix(std::uint64_t(f.kind) | (std::uint64_t(f.diagonal) << 8) | (std::uint64_t(f.K) << 16) | (std::uint64_t(f.dk) << 24));
        mix(f.touch);
        mix(f.ctrl_mask);
        for (int k = 0; k < f.K; ++k) mix(std::uint64_t(f.tpos[k]) + 0x9e37u);
    }
    return h;
}
std::mutex g_defer_mu;
std::unordered_map<std::uint64_t, int> g_defer_choice;

Plan choose_plan(int n, const std::vector<FOp>& ops, std::int64_t init, bool show) {
    static const int defer_env = [] { const char* v = std::getenv("QCS_DEFER"); return v ? std::atoi(v) : -1; }();
    if (init >= 0 && defer_env > 0) return plan_with_deferral(n, ops, std::min(defer_env, n - 4));
    if (!(init >= 0 && defer_env < 0 && n >= 20)) return plan_ops(n, ops, tile_max_bits());
    const std::uint64_t key = structure_hash(n, ops);
    {
        std::lock_guard<std::mutex> lk(g_defer_mu);
        auto it = g_defer_choice.find(key);
        if (it != g_defer_choice.end())
            return it->second > 0 ? plan_with_deferral(n, ops, it->second) : plan_ops(n, ops, tile_max_bits());
    }
    auto remember = [&](int k) {
        std::lock_guard<std::mutex> lk(g_defer_mu);
        if (g_defer_choice.size() >= 4096) g_defer_choice.clear();
        g_defer_choice[key] = k;
    };
    Plan plan = plan_ops(n, ops, tile_max_bits());
    if (plan.passes.size() < 3) {
        remember(0);
        return plan;
    }
    double best = plan_cost_from_basis(n, ops, plan);
    int gates = 0, best_k = 0;
    for (const FOp& f : ops) gates += !f.diagonal;
    for (int k = 1; k <= 3 && k <= n - 13; ++k) {
        // worth planning only when a good part of the circuit lies outside the light cone of the
        // deferred qubits (layered nearest-neighbour circuits; not random pairings, whose cones
        // cover everything after a few layers)
        std::vector<int> first, second;
        split_deferred(ops, ((u64(1) << k) - 1) << (n - k), first, second);
        int early = 0;
        for (int i : first) early += !ops[std::size_t(i)].diagonal;
        if (second.empty() || early * 10 < gates * 4) break;
        Plan cand = plan_with_deferral(n, ops, k);
        const double c = plan_cost_from_basis(n, ops, cand);
        if (show) std::fprintf(stderr, "defer %d: model %.1f ms (best so far %.1f ms)\n", k, 1e3 * c, 1e3 * best);
        if (c < 0.97 * best) {
            best = c;
            plan = std::move(cand);
            best_k = k;
        }
    }
    // (nested levels -- a wider set deferred first, e.g. {4, 2} or {6, 2} -- model within 3% of the
    // single level for C4 and cost two more plans: not searched; plan_with_levels takes them)
    remember(best_k);
    return plan;
}

void plan_fused_passes(int n, const std::vector<FOp>& ops, Lowered& low, std::int64_t init) {
    if (n >= 3) {
        static const bool show = std::getenv("QCS_PLAN_TIME") != nullptr;  // host planning cost, per stage
        const auto t0 = std::chrono::steady_clock::now();
        Plan plan = choose_plan(n, ops, init, show);
        const auto t1 = std::chrono::steady_clock::now();
        lower_plan(n, ops, plan, low);
        const auto t2 = std::chrono::steady_clock::now();
        if (show)
            std::fprintf(stderr, "plan_ops %.2f ms, lower_plan %.2f ms\n",
                         std::chrono::duration<double, std::milli>(t1 - t0).count(),
                         std::chrono::duration<double, std::milli>(t2 - t1).count());
        // (the pass kernels are compiled in execute_fused, once the support masks that decide
        // their form are known)
    } else {  // no 3-bit tile: one operation per pass
        for (std::size_t i = 0; i < ops.size(); ++i) {
            low.pass_ops.push_back({int(i)});
            low.single_flip_off.push_back(low.flips.size());
            low.single_flip_cnt.push_back(ops[i].flips.size());
            low.flips.insert(low.flips.end(), ops[i].flips.begin(), ops[i].flips.end());
            low.passes.emplace_back();
        }
    }
}

// Upload and launch a lowered plan on the state.  init (>= 0): the state is to start from the
// basis state |init>; consumed (set to -1) by folding it into the first pass when that pass
// writes every tile, else by a fill kernel first.  jit: per pass, the specialised kernel (kept by
// cached plans); cached: the cached plan's id (never reused, unlike its address), whose tables
// need no upload when plan_buf holds them; 0 for an uncached plan.
// Support tracking from a basis state |init> (init >= 0): tiles outside the support reached
// before a pass are zero (no load), tiles a pass leaves zero and the next reads as zero are not
// written, and the reset folds into the first pass.  Returns false when the reset could not be
// folded (the caller writes |init> first).  Shared by execute_fused and plan_stats.
bool apply_support(int n, Lowered& low, std::int64_t init) {
    bool folded = init < 0;
    if (!low.passes.empty()) low.passes[0].init = 0;
    // from a basis state: tiles outside the support reached before a pass are zero (no load)
    const u64 full = n >= 64 ? ~u64(0) : (u64(1) << n) - 1;
    for (std::size_t i = 0; i < low.passes.size() && n >= 3; ++i) {
        PassParams& P = low.passes[i];
        P.zmask = P.zval = 0;
        if (!(init >= 0) || low.pass_ops[i].size() < 2) continue;
        u64 tile = 0;
        for (int b = 0; b < P.m; ++b) tile |= u64(1) << P.bits[b];
        P.zmask = full & ~tile & ~low.reached[i];
        P.zval = u64(init) & P.zmask;
    }
    // a tile that is zero after this pass and that the next pass (running every tile) reads as
    // zero need not be written at all
    static const bool no_skip = std::getenv("QCS_NO_TILE_SKIP") != nullptr;  // A/B switch
    static const bool no_zero = std::getenv("QCS_NO_ZERO_INPUT") != nullptr;
    if (no_zero)
        for (auto& P : low.passes) P.zmask = P.zval = 0;
    for (std::size_t i = 0; i + 1 < low.passes.size() && n >= 3 && !no_skip; ++i) {
        PassParams& P = low.passes[i];
        const PassParams& Q = low.passes[i + 1];
        P.smask = P.sval = 0;
        if (!Q.zmask || low.pass_ops[i].size() < 2 || low.pass_ops[i + 1].size() < 2 || Q.list_cnt ||
            Q.alt_mode == ALT_SKIP)
            continue;
        u64 tile = 0;
        for (int b = 0; b < P.m; ++b) tile |= u64(1) << P.bits[b];
        P.smask = Q.zmask & ~tile;
        P.sval = Q.zval & ~tile;
    }
    if (!low.passes.empty()) low.passes.back().smask = low.passes.back().sval = 0;
    static const bool no_fold = std::getenv("QCS_NO_INIT_FOLD") != nullptr;  // A/B switch
    if (init >= 0) {
        const bool fold = !no_fold && !low.passes.empty() && low.pass_ops[0].size() >= 2 && n >= 3 && low.passes[0].list_cnt == 0 &&
                          low.passes[0].alt_mode != ALT_SKIP;
        if (fold) {
            low.passes[0].init = 1;
            low.passes[0].init_index = u64(init);
            folded = true;
        }
    }
    return folded;
}

void execute_fused(qcs_state* s, const std::vector<FOp>& ops, Lowered& low, std::int64_t* init,
                   std::vector<void*>* jit = nullptr, std::uint64_t cached = 0) {
    const int n = s->n;
    // plan buffer: [TileOps | flip lists | u64 tables], 256-byte aligned sections
    const std::size_t bb = low.big.size() * sizeof(TileOp);
    const std::size_t fb = low.flips.size() * sizeof(u64);
    const std::size_t tb = low.tables.size() * sizeof(u64);
    const std::size_t f_off = (bb + 255) & ~std::size_t(255);
    const std::size_t t_off = (f_off + fb + 255) & ~std::size_t(255);
    if ((bb + fb + tb) && !(cached && s->plan_loaded == cached)) {
        const std::size_t bytes = t_off + tb;
        ensure_plan(s, bytes + 8);
        // stream order keeps the upload behind the previous plan's kernels; the pinned slot is
        // reused only once its earlier upload has been read (four calls back: normally long ago)
        qcs_state::Stage& sg = s->stage[s->stage_next++ & 3];
        if (sg.done) QCS_CUDA(cudaEventSynchronize(sg.done));
        else QCS_CUDA(cudaEventCreateWithFlags(&sg.done, cudaEventDisableTiming));
        if (sg.cap < bytes) {
            if (sg.host) QCS_CUDA(cudaFreeHost(sg.host));
            sg.host = nullptr;
            sg.cap = 0;
            const std::size_t cap = std::max<std::size_t>(bytes, 1 << 16);
            QCS_CUDA(cudaHostAlloc(&sg.host, cap, cudaHostAllocDefault));
            sg.cap = cap;
        }
        auto* host = static_cast<unsigned char*>(sg.host);
        if (bb) std::memcpy(host, low.big.data(), bb);
        if (fb) std::memcpy(host + f_off, low.flips.data(), fb);
        if (tb) std::memcpy(host + t_off, low.tables.data(), tb);
        QCS_CUDA(cudaMemcpyAsync(s->plan_buf, host, bytes, cudaMemcpyHostToDevice, s->stream));
        QCS_CUDA(cudaEventRecord(sg.done, s->stream));
        s->plan_loaded = cached;
    }
    auto* base = static_cast<unsigned char*>(s->plan_buf);
    const auto* big_dev = reinterpret_cast<const TileOp*>(base);
    const auto* flips_dev = reinterpret_cast<const u64*>(base + f_off);
    const auto* tables_dev = reinterpret_cast<const u64*>(base + t_off);
    const std::int64_t init_index = init ? *init : -1;
    if (!apply_support(n, low, init_index)) fill_basis(s->amps, u64(1) << n, u64(init_index), s->stream);
    if (init) *init = -1;
    // compile the plan's missing pass kernels in parallel before its first launch (a kept plan's
    // later runs know their kernels and skip the source generation)
    const bool first_run = !jit || jit->size() != low.passes.size();
    if (jit && jit->size() != low.passes.size()) jit->assign(low.passes.size(), nullptr);
    if (first_run && n >= 3) jit_prepare(n, low.passes, low.pass_ops);
    for (std::size_t i = 0; i < low.passes.size(); ++i) {
        const auto& po = low.pass_ops[i];
        if (po.size() == 1) run_single(s, ops[std::size_t(po[0])], flips_dev + low.single_flip_off[i], low.single_flip_cnt[i]);
        else launch_tile_pass(s->amps, n, low.passes[i], big_dev, flips_dev, tables_dev, s->stream, jit ? &(*jit)[i] : nullptr);
    }
}

// Plan, lower, upload and launch a list of operations on the state.
void run_fused(qcs_state* s, const std::vector<FOp>& ops, std::int64_t* init = nullptr) {
    if (ops.empty()) return;
    Lowered low;
    plan_fused(s->n, ops, low, init ? *init : -1);
    s->plan_loaded = 0;
    execute_fused(s, ops, low, init);
}

std::vector<FOp> rh_ops(int n, double value) {
    std::vector<FOp> ops;
    ops.push_back(make_scale(value));  // rh_build's magnitude (rh.cpp:20), scale first (rh.cpp:99-100)
    for (int b = 0; b < n; ++b) ops.push_back(make_wht(b));
    return ops;
}

void append_step_ops(int n, const qcs_step& st, bool rh, std::vector<FOp>& ops) {
    if (rh) {
        auto r = rh_ops(n, std::exp2(-0.5 * n));
        ops.insert(ops.end(), r.begin(), r.end());
    } else if (st.kind == QCS_STEP_DIAG) {
        const bool any = st.flip_rest || st.num_flipped;
        if (any) ops.push_back(make_sign(n, std::vector<u64>(st.flipped, st.flipped + st.num_flipped), st.flip_rest));
    } else {
        for (int j = 0; j < st.num_placements; ++j) {
            FOp f;
            if (make_fop(canonical_op(n, st.placements[j]), f)) ops.push_back(std::move(f));
        }
    }
}

}  // namespace

void apply_rh(qcs_state* s) {
    DeviceGuard g(s->device);
    TimerScope ts(s);
    run_fused(s, rh_ops(s->n, std::exp2(-0.5 * s->n)));
}

u64 rh_sign_count(int n, int method, u64 block);

void rh_mvm(qcs_state* s, int n, double value, int method, u64 block, u64* sign_count, u64* madd_count) {
    // rh.cpp:92-96: the checks, in the reference's order
    if (n < 1) raise(QCS_ERR_DIMENSION, "RH MVM needs n >= 1");
    if (s->n != n) raise(QCS_ERR_DIMENSION, "RH MVM qubit count mismatch");
    const u64 half = u64(1) << (n - 1);
    const u64 signs = rh_sign_count(n, method, block);  // raises the block-size SimError (rh.cpp:58)
    DeviceGuard g(s->device);
    TimerScope ts(s);
    run_fused(s, rh_ops(n, value));
    if (sign_count) *sign_count = signs;
    if (madd_count) *madd_count = 4 * half * half;  // rh.cpp:153
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

}  // namespace

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

std::atomic<std::uint64_t> g_plan_ids{0};

struct CachedPlan {
    std::uint64_t id = ++g_plan_ids;        // identifies the plan's tables in plan_buf
    std::vector<unsigned char> key;
    std::vector<FOp> ops;
    Lowered low;
    std::vector<void*> jit;                 // per pass: its specialised kernel, once found
    std::vector<qcs_step_report> reports;
};

struct PlanCache {
    static constexpr std::size_t kEntries = 4;
    std::vector<std::unique_ptr<CachedPlan>> entries;  // most recently used last
    CachedPlan* find(const std::vector<unsigned char>& key) {
        for (std::size_t i = 0; i < entries.size(); ++i)
            if (entries[i]->key == key) {
                std::rotate(entries.begin() + std::ptrdiff_t(i), entries.begin() + std::ptrdiff_t(i) + 1, entries.end());
                return entries.back().get();
            }
        return nullptr;
    }
    CachedPlan& insert(std::unique_ptr<CachedPlan> p) {
        if (entries.size() >= kEntries) entries.erase(entries.begin());
        entries.push_back(std::move(p));
        return *entries.back();
    }
};

void delete_plan_cache(PlanCache* p) { delete p; }

namespace {
// everything the plan and the reports depend on, as bytes
void plan_key(int n, int engine, const qcs_sim_options& o, const qcs_step* steps, int nsteps,
              std::vector<unsigned char>& key) {
    auto put = [&](const void* p, std::size_t b) {
        const auto* c = static_cast<const unsigned char*>(p);
        key.insert(key.end(), c, c + b);
    };
    const std::int64_t head[] = {n, engine, o.sign_method, std::int64_t(o.block_size), o.fuse, jit_mode(),
                                 std::int64_t(dense_cap()), nsteps};
    put(head, sizeof(head));
    for (int i = 0; i < nsteps; ++i) {
        const qcs_step& st = steps[i];
        const std::int64_t sh[] = {st.kind, st.stage, st.flip_rest, std::int64_t(st.num_flipped), st.num_placements};
        put(sh, sizeof(sh));
        if (st.kind == QCS_STEP_DIAG) {
            if (st.num_flipped) put(st.flipped, st.num_flipped * sizeof(u64));
            continue;
        }
        for (int j = 0; j < st.num_placements; ++j) {
            const qcs_placement& p = st.placements[j];
            put(&p.arity, sizeof(p.arity));
            put(p.qubits, sizeof(int) * std::size_t(p.arity));
            put(p.matrix, sizeof(double) * 2 * (std::size_t(1) << (2 * p.arity)));
            // the name selects RH dispatch ("Hadamard", circuit.cpp:31-39)
            const std::size_t len = p.name ? std::strlen(p.name) : 0;
            put(&len, sizeof(len));
            if (len) put(p.name, len);
        }
    }
}
}  // namespace

namespace {

// The Matrix method (engine == dense): step_matrix_dense on the device, then dense_mvm into a
// scratch vector, copied back in place -- byte for byte the reference's dense engine
// (engine.cpp:126-133, :180-188; core.cpp:55-87).  Steps with a placement the reference cannot
// express (non-contiguous or reversed qubits) return false: the caller runs that step through
// the fused kernels (same operator; no reference bytes exist to match).
bool run_dense_step(qcs_state* s, const qcs_step& st) {
    const int n = s->n;
    const u64 dim = u64(1) << n;
    DenseFold fold{};
    if (st.kind == QCS_STEP_GATES) {
        std::vector<const qcs_placement*> at(std::size_t(n), nullptr);
        for (int j = 0; j < st.num_placements; ++j) {
            const qcs_placement& p = st.placements[j];
            for (int k = 1; k < p.arity; ++k)
                if (p.qubits[k] != p.qubits[0] + k) return false;
            at[std::size_t(p.qubits[0])] = &p;
        }
        int off = 0;
        for (int q = 0; q < n;) {
            if (fold.nfactors >= 32) raise(QCS_ERR_CAPACITY, "dense engine: too many factors");
            const qcs_placement* p = at[std::size_t(q)];
            const int k = p ? p->arity : 1;
            const int d = 1 << k;
            if (off + d * d > 512) raise(QCS_ERR_CAPACITY, "dense engine: factors too large");
            fold.arity[fold.nfactors] = k;
            fold.offset[fold.nfactors] = off;
            for (int e = 0; e < d * d; ++e)
                fold.mat[off + e] = p ? make_double2(p->matrix[2 * e], p->matrix[2 * e + 1])
                                      : make_double2((e == 0 || e == 3) ? 1.0 : 0.0, 0.0);
            off += d * d;
            ++fold.nfactors;
            q += k;
        }
    }
    double2* mat = nullptr;
    double2* out = nullptr;
    QCS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&mat), dim * dim * sizeof(double2), s->stream));
    QCS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&out), dim * sizeof(double2), s->stream));
    u64* flips = nullptr;
    if (st.kind == QCS_STEP_DIAG) {
        std::vector<u64> f(st.flipped, st.flipped + st.num_flipped);
        std::sort(f.begin(), f.end());
        f.erase(std::unique(f.begin(), f.end()), f.end());
        QCS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&flips), std::max<std::size_t>(1, f.size()) * sizeof(u64),
                                 s->stream));
        if (!f.empty())
            QCS_CUDA(cudaMemcpyAsync(flips, f.data(), f.size() * sizeof(u64), cudaMemcpyHostToDevice, s->stream));
        dense_diag(mat, n, flips, f.size(), st.flip_rest, s->stream);
        QCS_CUDA(cudaStreamSynchronize(s->stream));  // the host list must outlive the copy
    } else {
        dense_build(mat, n, fold, s->stream);
    }
    dense_mvm(mat, s->amps, out, n, s->stream);
    QCS_CUDA(cudaMemcpyAsync(s->amps, out, dim * sizeof(double2), cudaMemcpyDeviceToDevice, s->stream));
    QCS_CUDA(cudaFreeAsync(mat, s->stream));
    QCS_CUDA(cudaFreeAsync(out, s->stream));
    if (flips) QCS_CUDA(cudaFreeAsync(flips, s->stream));
    return true;
}

}  // namespace

void simulate(qcs_state* s, const qcs_step* steps, int nsteps, int engine, const qcs_sim_options* opts,
              qcs_step_report* reports) {
    const int n = s->n;
    validate_circuit(n, steps, nsteps);
    if (engine < QCS_ENGINE_DENSE || engine > QCS_ENGINE_RH_DAX) raise(QCS_ERR_ARG, "unknown engine");
    qcs_sim_options o{QCS_SIGN_LOGARITHM, 0, 1, 0, 0};
    if (opts) o = *opts;
    const u64 dim = u64(1) << n;
    if (o.reset && o.initial >= dim) raise(QCS_ERR_DIMENSION, "initial basis index out of range");  // circuit.cpp:41-62
    DeviceGuard g(s->device);
    TimerScope ts(s);
    std::int64_t init = o.reset ? std::int64_t(o.initial) : -1;
    // fused mode: a circuit simulated again on this state (same steps, engine, options) reuses
    // its plan -- operations, lowered passes, reports, specialised kernels -- and, when the
    // device plan buffer still holds its tables, their upload
    std::vector<unsigned char> key;
    static const bool no_cache = std::getenv("QCS_NO_PLAN_CACHE") != nullptr;  // A/B switch
    const bool matrix_method = engine == QCS_ENGINE_DENSE;
    if (o.fuse && !no_cache && !matrix_method) {
        plan_key(n, engine, o, steps, nsteps, key);
        if (!s->plan_cache) s->plan_cache = new PlanCache;
        if (CachedPlan* hit = s->plan_cache->find(key)) {
            if (reports) std::copy(hit->reports.begin(), hit->reports.end(), reports);
            execute_fused(s, hit->ops, hit->low, &init, &hit->jit, hit->id);
            if (init >= 0) fill_basis(s->amps, dim, u64(init), s->stream);
            return;
        }
    }
    std::vector<qcs_step_report> reps(static_cast<std::size_t>(nsteps));
    std::vector<FOp> ops;  // fused mode: the whole circuit; stepwise: one step at a time
    for (int i = 0; i < nsteps; ++i) {
        const qcs_step& st = steps[i];
        qcs_step_report r{};
        r.stage = st.stage;
        r.dense_bytes = dense_step_bytes(n);
        const bool use_rh = engine == QCS_ENGINE_RH_DAX && is_hadamard_all(st, n);
        if (!o.fuse || matrix_method) ops.clear();
        append_step_ops(n, st, use_rh, ops);
        if (use_rh) {
            r.structure = QCS_STRUCT_RH;
            r.matrix_bytes = 16;  // engine.cpp:173
            r.sign_count = rh_sign_count(n, o.sign_method, o.block_size);
            const u64 half = u64(1) << (n - 1);
            r.madd_count = 4 * half * half;  // rh.cpp:153
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
        }
        if (matrix_method) {
            if (init >= 0) {
                fill_basis(s->amps, dim, u64(init), s->stream);
                init = -1;
            }
            if (run_dense_step(s, st)) {
                ops.clear();
            } else {  // a placement the reference cannot place: this step through the fused kernels
                run_fused(s, ops, &init);
                ops.clear();
            }
        } else if (!o.fuse) {
            run_fused(s, ops, &init);  // one step: fused only within the step
        }
        reps[std::size_t(i)] = r;
    }
    if (reports) std::copy(reps.begin(), reps.end(), reports);
    if (o.fuse && !matrix_method) {
        merge_single_qubit(n, ops);
        split_phases(ops);
        if (!ops.empty() && no_cache) {
            run_fused(s, ops, &init);
        } else if (!ops.empty()) {
            auto cp = std::make_unique<CachedPlan>();
            cp->key = std::move(key);
            cp->ops = std::move(ops);
            cp->reports = std::move(reps);
            plan_fused(n, cp->ops, cp->low, init);
            CachedPlan& e = s->plan_cache->insert(std::move(cp));
            execute_fused(s, e.ops, e.low, &init, &e.jit, e.id);
        }
    }
    if (init >= 0) fill_basis(s->amps, dim, u64(init), s->stream);  // no operation at all
}

namespace {
void add_plan_stats(int n, const std::vector<FOp>& ops, qcs_plan_info* out, std::int64_t init = -1) {
    if (ops.empty()) return;
    out->ops += std::int64_t(ops.size());
    if (n < 3) {
        out->passes += std::int64_t(ops.size());
        out->single_passes += std::int64_t(ops.size());
        return;
    }
    Lowered low;
    plan_fused_passes(n, ops, low, init);  // the plan execute_fused would run
    compute_reached(ops, low);
    apply_support(n, low, init);  // from |init> (opts->reset), as execute_fused runs the plan
    const bool dump = std::getenv("QCS_PLAN_DUMP") != nullptr;  // planner debugging: rounds and ops
    for (std::size_t i = 0; i < low.passes.size(); ++i) {
        if (dump) dump_pass(stderr, low.passes[i], low.pass_ops[i].size());
        ++out->passes;
        if (low.pass_ops[i].size() == 1) {
            ++out->single_passes;
            continue;
        }
        const PassParams& p = low.passes[i];
        ++out->tile_passes;
        {  // the tiles that compute: the listed ones, one for a pass from |init>, a 2^-|zmask| share
            double tiles = p.list_cnt ? double(p.list_cnt) : std::ldexp(1.0, n - p.m);
            double moved = tiles;
            if (p.init) {
                tiles = 1.0;
                moved = p.smask ? moved * std::ldexp(1.0, -__builtin_popcountll(p.smask)) : moved;
                moved = 0.5 * moved;  // loads nothing; stores what the next pass reads
            } else if (p.zmask) {
                tiles *= std::ldexp(1.0, -__builtin_popcountll(p.zmask));
            }
            const double f = tiles * pass_fp64_per_tile(p);
            if (dump) std::fprintf(stderr, "  fp64/amp %.2f  tiles %.0f\n", f / std::ldexp(1.0, n), tiles);
            out->fp64_ops += std::int64_t(f);
            out->sweep_amps += std::int64_t(moved * std::ldexp(1.0, p.m));
        }
        if (p.alt_mode != ALT_NONE) ++out->alt_passes;
        if (p.alt_mode == ALT_SKIP) ++out->skip_passes;
        if (p.alt_mode == ALT_NONE && p.list_cnt) ++out->paired_passes;
        out->rounds += p.nrounds;
        for (int r = 0; r < p.nrounds; ++r)
            if (p.rounds[r].flags & RD_SMEM) ++out->smem_rounds;
            else out->reg_ops += p.rounds[r].op_count;
    }
}
}  // namespace

void plan_stats(int n, const qcs_step* steps, int nsteps, int engine, const qcs_sim_options* opts,
                qcs_plan_info* out) {
    validate_circuit(n, steps, nsteps);
    if (engine < QCS_ENGINE_DENSE || engine > QCS_ENGINE_RH_DAX) raise(QCS_ERR_ARG, "unknown engine");
    qcs_sim_options o{QCS_SIGN_LOGARITHM, 0, 1, 0, 0};
    if (opts) o = *opts;
    *out = qcs_plan_info{};
    out->max_tile_bits = std::min(tile_max_bits(), n);
    std::vector<FOp> ops;
    for (int i = 0; i < nsteps; ++i) {
        const bool use_rh = engine == QCS_ENGINE_RH_DAX && is_hadamard_all(steps[i], n);
        append_step_ops(n, steps[i], use_rh, ops);
        if (!o.fuse) {
            add_plan_stats(n, ops, out);
            ops.clear();
        }
    }
    if (o.fuse) {
        merge_single_qubit(n, ops);
        split_phases(ops);
        add_plan_stats(n, ops, out, o.reset ? std::int64_t(o.initial) : -1);
    }
}

void plan_compile(int n, const qcs_step* steps, int nsteps, int engine, const qcs_sim_options* opts,
                  std::int64_t* kernels, std::int64_t* cubin_bytes, bool verify_only) {
    validate_circuit(n, steps, nsteps);
    if (engine < QCS_ENGINE_DENSE || engine > QCS_ENGINE_RH_DAX) raise(QCS_ERR_ARG, "unknown engine");
    qcs_sim_options o{QCS_SIGN_LOGARITHM, 0, 1, 0, 0};
    if (opts) o = *opts;
    *kernels = 0;
    *cubin_bytes = 0;
    std::vector<FOp> ops;
    auto flush = [&] {
        if (ops.empty() || n < 3) return;
        Lowered low;
        lower_plan(n, ops, plan_ops(n, ops, tile_max_bits()), low);
        for (std::size_t i = 0; i < low.passes.size(); ++i) {
            if (low.pass_ops[i].size() == 1) continue;
            *cubin_bytes += std::int64_t(jit_compile_only(low.passes[i], verify_only));
            ++*kernels;
        }
        ops.clear();
    };
    for (int i = 0; i < nsteps; ++i) {
        append_step_ops(n, steps[i], engine == QCS_ENGINE_RH_DAX && is_hadamard_all(steps[i], n), ops);
        if (!o.fuse) flush();
    }
    if (o.fuse) {
        merge_single_qubit(n, ops);
        split_phases(ops);
        flush();
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
