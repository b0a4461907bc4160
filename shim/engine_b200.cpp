// engine_b200.cpp -- drop-in replacement for the reference's src/engine.cpp that runs the hot
// path on a B200 through the C ABI (include/qcs_abi.h).
//
// Build it in place of engine.cpp and link libqcs_b200.so; every other reference source stays
// as it is.  The public API of engine.hpp is kept symbol for symbol:
//   engine_name / engine_from_name   (engine.hpp:12-13)
//   step_matrix_dense / dax / das    (engine.hpp:37-39)  -- dax/das by the device encoder
//   simulate                         (engine.hpp:46)     -- qcs_simulate on a device state
//   memory_report                    (engine.hpp:49)     -- qcs_memory_report
// Errors come back as the same exception classes (core.hpp:13-36) with the library's message.
// oracle/Makefile builds this against /root/reference/proj/include and links the reference's
// own tests/acceptance.cpp with it (oracle/_ref/acceptance_b200).
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "qcs_abi.h"
#include "qcsim/engine.hpp"
#include "shim_common.hpp"

namespace qcsim {

using b200::check;
using b200::rethrow;

namespace {

// CircuitStep list -> qcs_step list (the vectors keep the pointed-to storage alive)
struct Marshalled {
    std::vector<qcs_step> steps;
    std::vector<std::vector<qcs_placement>> placements;
    std::vector<std::vector<int>> qubits;
};

void marshal(const std::vector<const CircuitStep*>& in, Marshalled& m) {
    m.steps.resize(in.size());
    m.placements.resize(in.size());
    m.qubits.clear();
    std::size_t nq = 0;
    for (const CircuitStep* s : in) nq += s->placements.size();
    m.qubits.reserve(nq);
    for (std::size_t i = 0; i < in.size(); ++i) {
        const CircuitStep& s = *in[i];
        qcs_step& q = m.steps[i];
        q = qcs_step{};
        q.stage = s.stage;
        if (s.kind == CircuitStep::Kind::diag) {
            q.kind = QCS_STEP_DIAG;
            q.flipped = s.diag.flipped.data();
            q.num_flipped = s.diag.flipped.size();
            q.flip_rest = s.diag.flip_rest ? 1 : 0;
            continue;
        }
        q.kind = QCS_STEP_GATES;
        for (const Placement& p : s.placements) {
            std::vector<int> qs(std::size_t(p.gate.arity));
            for (int j = 0; j < p.gate.arity; ++j) qs[std::size_t(j)] = p.first_qubit + j;
            m.qubits.push_back(std::move(qs));
            qcs_placement pl{};
            pl.arity = p.gate.arity;
            pl.qubits = m.qubits.back().data();
            pl.matrix = reinterpret_cast<const double*>(p.gate.matrix.data.data());
            pl.name = p.gate.name.c_str();
            m.placements[i].push_back(pl);
        }
        q.placements = m.placements[i].data();
        q.num_placements = int(m.placements[i].size());
    }
}

const char* structure_name(int s) {
    switch (s) {
        case QCS_STRUCT_DENSE: return "dense";
        case QCS_STRUCT_DAX: return "dax";
        case QCS_STRUCT_DAS: return "das";
        default: return "rh";
    }
}

StepReport to_report(const qcs_step_report& r) {
    StepReport s;
    s.structure = structure_name(r.structure);
    s.stage = r.stage;
    s.matrix_bytes = r.matrix_bytes;
    s.dense_bytes = r.dense_bytes;
    s.entry_count = r.entry_count;
    s.sign_count = r.sign_count;
    s.madd_count = r.madd_count;
    return s;
}

struct Device {  // the state lives on device 0 of this process
    int id = 0;
};

}  // namespace

const char* engine_name(Engine e) {
    switch (e) {
        case Engine::dense: return "dense";
        case Engine::dax: return "dax";
        case Engine::das: return "das";
        case Engine::rh_dax: return "rh-dax";
    }
    return "?";
}

Engine engine_from_name(const std::string& name) {
    static const std::map<std::string, Engine> m = {
        {"dense", Engine::dense}, {"dax", Engine::dax}, {"das", Engine::das},
        {"rh-dax", Engine::rh_dax}, {"rh_dax", Engine::rh_dax}};
    auto it = m.find(name);
    if (it == m.end()) throw ParseError("unknown engine: " + name);
    return it->second;
}

// The Matrix method's operator, composed from the reference's public dense_tensor: the placed
// gates at their first qubit, 2x2 identities elsewhere, most significant qubit first.
DenseMatrix step_matrix_dense(const CircuitStep& step, int n) {
    const std::uint64_t dim = std::uint64_t(1) << n;
    if (step.kind == CircuitStep::Kind::diag) {
        if (dim > dense_cap() / dim) throw CapacityError("diagonal step exceeds dense cap");
        DenseMatrix m(dim, dim);
        for (std::uint64_t i = 0; i < dim; ++i) m.at(i, i) = step.diag.negated(i) ? -1.0 : 1.0;
        return m;
    }
    std::map<int, const Placement*> at;
    for (const Placement& p : step.placements) at[p.first_qubit] = &p;
    const DenseMatrix id2 = DenseMatrix::identity(2);
    DenseMatrix acc;
    bool first = true;
    for (int q = 0; q < n;) {
        auto it = at.find(q);
        const DenseMatrix& f = it != at.end() ? it->second->gate.matrix : id2;
        acc = first ? f : dense_tensor(acc, f);
        first = false;
        q += it != at.end() ? it->second->gate.arity : 1;
    }
    return acc;
}

namespace {

Marshalled one_step(const CircuitStep& step) {
    Marshalled m;
    marshal({&step}, m);
    return m;
}

}  // namespace

// step_matrix_dax (engine.cpp:135-142) materialised by the device encoder.
DaxMatrix step_matrix_dax(const CircuitStep& step, int n) {
    DaxMatrix out;
    out.rows = out.cols = std::uint64_t(1) << n;
    if (step.kind == CircuitStep::Kind::diag) {
        out.entries.reserve(out.rows);
        for (std::uint64_t i = 0; i < out.rows; ++i)
            out.entries.push_back({i, i, step.diag.negated(i) ? cplx{-1.0, 0.0} : cplx{1.0, 0.0}});
        return out;
    }
    Marshalled m = one_step(step);
    std::uint64_t count = 0;
    int rc = qcs_step_dax(n, m.steps[0].placements, m.steps[0].num_placements, Device{}.id, nullptr, nullptr,
                          nullptr, 0, QCS_MEM_HOST, &count);
    if (rc != QCS_OK && rc != QCS_ERR_CAPACITY) rethrow(rc);
    std::vector<std::uint64_t> rows(count), cols(count);
    std::vector<cplx> vals(count);
    check(qcs_step_dax(n, m.steps[0].placements, m.steps[0].num_placements, Device{}.id, rows.data(), cols.data(),
                       reinterpret_cast<double*>(vals.data()), count, QCS_MEM_HOST, &count));
    out.entries.resize(count);
    for (std::uint64_t i = 0; i < count; ++i) out.entries[i] = {rows[i], cols[i], vals[i]};
    return out;
}

// step_matrix_das (engine.cpp:144-151) materialised by the device encoder.
DasMatrix step_matrix_das(const CircuitStep& step, int n) {
    DasMatrix out;
    out.rows = out.cols = std::uint64_t(1) << n;
    if (step.kind == CircuitStep::Kind::diag) {
        out.entries.reserve(out.rows);
        for (std::uint64_t i = 0; i < out.rows; ++i)
            out.entries.push_back({i, true, step.diag.negated(i) ? cplx{-1.0, 0.0} : cplx{1.0, 0.0}});
        return out;
    }
    Marshalled m = one_step(step);
    std::uint64_t count = 0;
    int rc = qcs_step_das(n, m.steps[0].placements, m.steps[0].num_placements, Device{}.id, nullptr, nullptr,
                          nullptr, 0, QCS_MEM_HOST, &count);
    if (rc != QCS_OK && rc != QCS_ERR_CAPACITY) rethrow(rc);
    std::vector<std::uint64_t> dis(count);
    std::vector<std::uint8_t> last(count);
    std::vector<cplx> vals(count);
    check(qcs_step_das(n, m.steps[0].placements, m.steps[0].num_placements, Device{}.id, dis.data(), last.data(),
                       reinterpret_cast<double*>(vals.data()), count, QCS_MEM_HOST, &count));
    out.entries.resize(count);
    for (std::uint64_t i = 0; i < count; ++i) out.entries[i] = {dis[i], last[i] != 0, vals[i]};
    return out;
}

// simulate (engine.cpp:153-210) on the GPU: same dispatch, same StepReport accounting.  The
// device state is kept per thread and per qubit count between calls (shim_common.hpp), so a
// repeated circuit reuses its lowered plan, specialised kernels and uploaded tables (the state's
// plan cache) and no 2^n allocation happens per call; |initial> is written by the first pass.
SimReport simulate(const Circuit& c, Engine engine, const SimOptions& opts) {
    c.validate();
    std::vector<const CircuitStep*> ptrs;
    for (const CircuitStep& s : c.steps) ptrs.push_back(&s);
    Marshalled m;
    marshal(ptrs, m);
    SimReport report;
    {
        qcs_state* st = b200::pool().get(b200::kSimulate, c.n);
        qcs_sim_options o{};
        o.sign_method = int(opts.sign_method);
        o.block_size = opts.block_size;
        o.fuse = 1;
        o.reset = 1;
        o.initial = c.initial;
        std::vector<qcs_step_report> reps(c.steps.size());
        check(qcs_simulate(st, m.steps.data(), int(m.steps.size()), int(engine), &o, reps.data()));
        for (const qcs_step_report& r : reps) {
            report.steps.push_back(to_report(r));
            report.total_sign_count += r.sign_count;
            report.total_madd_count += r.madd_count;
        }
        // the value-initialised result vectors (the reference API's value semantics) are written
        // while the device still runs the circuit (qcs_simulate returns with the work queued)
        const std::uint64_t dim = std::uint64_t(1) << c.n;
        report.final.n = c.n;
        report.final.amps.resize(dim);
        report.probabilities.resize(dim);
        check(qcs_state_download(st, reinterpret_cast<double*>(report.final.amps.data()), 0, dim));
        check(qcs_probabilities(st, report.probabilities.data(), QCS_MEM_HOST));
    }
    return report;
}

// memory_report (engine.cpp:212-234)
std::vector<StepReport> memory_report(const Circuit& c, Engine engine) {
    c.validate();
    std::vector<const CircuitStep*> ptrs;
    for (const CircuitStep& s : c.steps) ptrs.push_back(&s);
    Marshalled m;
    marshal(ptrs, m);
    std::vector<qcs_step_report> reps(c.steps.size());
    check(qcs_memory_report(c.n, m.steps.data(), int(m.steps.size()), int(engine), reps.data()));
    std::vector<StepReport> out;
    for (const qcs_step_report& r : reps) out.push_back(to_report(r));
    return out;
}

}  // namespace qcsim
