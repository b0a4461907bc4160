// common.hpp -- shared types, error plumbing and arithmetic for libqcs_b200.
#pragma once

#include <cuda_runtime.h>

#include <complex>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "qcs_abi.h"

namespace qcs {

using u64 = std::uint64_t;
using cplx = std::complex<double>;

// Internal exception carrying an ABI status code; the C ABI layer converts it to a return
// value plus qcs_last_error() text.  Codes mirror the reference's SimError hierarchy.
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& what) : std::runtime_error(what), code(c) {}
};

[[noreturn]] inline void raise(int code, const std::string& what) { throw Error(code, what); }

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) raise(QCS_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define QCS_CUDA(call) ::qcs::cuda_check((call), #call)

// Launch bookkeeping: every kernel launch of the library goes through note_launch() so the
// bench can report how many of OUR kernels ran (bench.py "gpu_launches").
void note_launch(int n = 1);
inline void check_launch(const char* name) {
    note_launch();
    cuda_check(cudaGetLastError(), name);
}

// Optional per-launch timing (qcs_timing_enable): CUDA events around each launch on the
// launching stream, attributed to a kernel class with its algorithmic HBM bytes.  Active
// only while an entry point working on a timing-enabled state runs (thread-local sink).
struct LaunchTimer;
struct TimedLaunch {
    LaunchTimer* t = nullptr;
    int slot = -1;
    TimedLaunch(const char* cls, double algorithmic_bytes, cudaStream_t s);
    ~TimedLaunch();
    TimedLaunch(const TimedLaunch&) = delete;
    TimedLaunch& operator=(const TimedLaunch&) = delete;
};

// Canonical form of one placement: gate bits sorted by descending basis-bit position (the
// reference's MSB-first factor order), matrix permuted to match, so ascending local column
// equals ascending global column -- the order dax_mvm accumulates in (dax.cpp:101).
struct GateOp {
    int k = 0;                 // arity
    int pos[QCS_MAX_ARITY];    // basis-bit positions, pos[0] > pos[1] > ... (local bit k-1-i)
    std::vector<cplx> m;       // 2^k x 2^k row-major in canonical local order
    std::string name;          // catalog name, "" when unknown
};

// Validate reference-qubit placements and canonicalise them (circuit.cpp:41-62 rules).
GateOp canonical_op(int n, const qcs_placement& p);

}  // namespace qcs
