// engine.hpp -- device state handle and the step engine (host side of libqcs_b200).
#pragma once

#include <cstdint>
#include <vector>

#include "common.hpp"
#include "kernels.hpp"

namespace qcs { struct LaunchTimer; struct PlanCache; }

struct qcs_state {
    int n = 0;
    int device = 0;
    double2* amps = nullptr;
    cudaStream_t stream = nullptr;
    bool owns_mem = false;
    bool owns_stream = false;
    void* scratch = nullptr;              // reduction scratch (device)
    std::uint64_t* flip_buf = nullptr;    // device copy of diag index lists
    std::size_t flip_cap = 0;
    void* plan_buf = nullptr;             // device copy of the current plan (rounds, ops, flips)
    std::size_t plan_cap = 0;
    // pinned host staging of plan uploads, a ring: a pageable copy would block the host until the
    // stream drains, so the next call's planning could not overlap the device's work
    struct Stage {
        void* host = nullptr;
        std::size_t cap = 0;
        cudaEvent_t done = nullptr;       // the upload from this slot has been read
    } stage[4];
    int stage_next = 0;
    qcs::PlanCache* plan_cache = nullptr;   // recently simulated circuits: their lowered plans (engine.cpp)
    std::uint64_t plan_loaded = 0;          // id of the cached plan whose tables plan_buf holds (0: none)
    cudaEvent_t events[8] = {};
    // qcs_summary_begin / _end: the pinned read-back of the summary's block candidates
    void* summary_host = nullptr;
    int summary_k = 0;              // k of the pending summary (0: none)
    cudaEvent_t summary_done = nullptr;
    qcs::LaunchTimer* timer = nullptr;   // per-launch timing (qcs_timing_enable)
    ~qcs_state();
};

namespace qcs {

using u64 = std::uint64_t;
void delete_plan_cache(PlanCache* p);

// Make `dev` current for the lifetime of the guard.
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev);
    ~DeviceGuard();
};

qcs_state* state_create(int n, int device, u64 basis);
qcs_state* state_wrap(int n, int device, void* amps, void* stream);

bool build_gate_desc(const GateOp& op, GateDesc& d);

void apply_step(qcs_state* s, const qcs_placement* p, int count);
void apply_diag(qcs_state* s, const u64* flipped, u64 count, int flip_rest);
void apply_rh(qcs_state* s);
void rh_mvm(qcs_state* s, int n, double value, int method, u64 block, u64* sign_count, u64* madd_count);

void simulate(qcs_state* s, const qcs_step* steps, int nsteps, int engine, const qcs_sim_options* opts,
              qcs_step_report* reports);
void apply_split(qcs_state* s, void* peer, int self_bit, int nsel, const int* sel, const double* blocks,
                 unsigned skip);
void plan_stats(int n, const qcs_step* steps, int nsteps, int engine, const qcs_sim_options* opts,
                qcs_plan_info* out);
void plan_compile(int n, const qcs_step* steps, int nsteps, int engine, const qcs_sim_options* opts,
                  std::int64_t* kernels, std::int64_t* cubin_bytes, bool verify_only = false);
void memory_report(int n, const qcs_step* steps, int nsteps, int engine, qcs_step_report* reports);
void validate_circuit(int n, const qcs_step* steps, int nsteps);

// device encoder entry (qcs_step_dax / qcs_step_das)
u64 step_encode(int n, const qcs_placement* p, int count, int device, bool das, u64 capacity, u64* rows,
                u64* cols, double* vals, u64* dis, std::uint8_t* last, bool on_device);

u64 dense_cap();
void set_dense_cap(u64 cap);

// catalog (gates.cpp)
int catalog_size();
void catalog_entry(int i, const char** name, int* arity, int* nparams, double* ratio);
const char* gate_lookup(const std::string& name, const std::vector<double>& params, std::vector<cplx>& out,
                        int* arity);
std::vector<double> canonical_params(const std::string& name);

std::size_t reduce_scratch_bytes();

// per-launch timing (timing.cpp)
struct TimerScope {
    LaunchTimer* prev;
    explicit TimerScope(qcs_state* s);
    ~TimerScope();
};
void timing_enable(qcs_state* s, bool on);
void timing_reset(qcs_state* s);
int timing_count(qcs_state* s);
void timing_entry(qcs_state* s, int i, const char** name, u64* launches, double* ms, double* bytes);
void destroy_timer(LaunchTimer* t);
u64 launches();

}  // namespace qcs
