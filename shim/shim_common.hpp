// shim_common.hpp -- shared pieces of the link-substitute shims (engine_b200.cpp, mvm_b200.cpp):
// status -> reference exception mapping, and a per-thread pool of device states so repeated
// reference-API calls reuse one device allocation (and, for simulate, its plan cache) instead of
// allocating 2^n * 16 B and re-planning on every call.
#pragma once

#include <cstdint>
#include <string>

#include "qcs_abi.h"
#include "qcsim/core.hpp"

namespace qcsim::b200 {

[[noreturn]] inline void rethrow(int rc) {
    const std::string msg = qcs_last_error();
    switch (rc) {
        case QCS_ERR_CAPACITY: throw CapacityError(msg);
        case QCS_ERR_DIMENSION: throw DimensionError(msg);
        case QCS_ERR_ENCODING: throw EncodingError(msg);
        case QCS_ERR_PARSE: throw ParseError(msg);
        default: throw SimError(msg);
    }
}

inline void check(int rc) {
    if (rc != QCS_OK) rethrow(rc);
}

// Slots of the per-thread pool: one kept device state each, re-created only when the qubit count
// changes.  The reference API is reentrant and single-threaded per call (SURVEY.md section 8b
// "Threading"), so a thread-local pool keeps different threads on different handles.
enum Slot { kSimulate = 0, kMvmIn = 1, kMvmOut = 2, kSlots = 3 };

struct StatePool {
    qcs_state* s[kSlots] = {};
    int n[kSlots] = {};
    ~StatePool() {
        for (qcs_state*& p : s)
            if (p) qcs_state_destroy(p);
    }
    qcs_state* get(Slot slot, int qubits) {
        if (s[slot] && n[slot] == qubits) return s[slot];
        if (s[slot]) {
            qcs_state_destroy(s[slot]);
            s[slot] = nullptr;
        }
        check(qcs_state_create(qubits, 0, 0, &s[slot]));
        n[slot] = qubits;
        return s[slot];
    }
};

inline StatePool& pool() {
    thread_local StatePool p;
    return p;
}

// log2 of a StateVector's dimension (the device holds power-of-two states only)
inline int qubits_of(std::uint64_t dim) {
    int q = 0;
    while ((std::uint64_t(1) << q) < dim) ++q;
    if ((std::uint64_t(1) << q) != dim) throw SimError("B200 MVM needs a power-of-two dimension");
    return q;
}

}  // namespace qcsim::b200
