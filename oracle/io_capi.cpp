// io_capi.cpp -- extern "C" access to the reference's front end (src/circuit_io.cpp) for the
// golden-fixture generator.  TEST INFRASTRUCTURE ONLY: marshalling around the unmodified
// reference functions parse_circuit_json, simulate and render_report.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "qcsim/circuit_io.hpp"

using namespace qcsim;

namespace {
thread_local std::string g_err;

int code_of(const std::exception& e) {
    if (dynamic_cast<const CapacityError*>(&e)) return 1;
    if (dynamic_cast<const DimensionError*>(&e)) return 2;
    if (dynamic_cast<const EncodingError*>(&e)) return 3;
    if (dynamic_cast<const ParseError*>(&e)) return 4;
    if (dynamic_cast<const SimError*>(&e)) return 5;
    return 9;
}

long emit(const std::string& s, char* out, long cap) {
    if (long(s.size()) + 1 > cap) return -long(s.size()) - 1;
    std::memcpy(out, s.data(), s.size());
    out[s.size()] = 0;
    return long(s.size());
}
}  // namespace

extern "C" {

const char* io_last_error() { return g_err.c_str(); }

// parse_circuit_json -> simulate(engine) -> render_report(format, samples, seed).
// Returns the report length, or -(code) on a reference exception (message: io_last_error).
long io_run(const char* json_text, const char* engine, const char* format, int samples, unsigned long long seed,
            char* out, long cap) {
    try {
        const Circuit c = parse_circuit_json(json_text);
        const Engine e = engine_from_name(engine);
        const SimReport r = simulate(c, e);
        ReportOptions o;
        o.format = format;
        o.samples = samples;
        o.seed = seed;
        o.engine = engine;
        const long len = emit(render_report(r, c.n, o), out, cap);
        if (len < 0) return -100;
        return len;
    } catch (const std::exception& ex) {
        g_err = ex.what();
        return -code_of(ex);
    }
}

// parse_gate_expression (circuit_io.cpp:85-107): dense product written to out (interleaved).
long io_gate_expression(const char* expr, double* out, long cap_doubles) {
    try {
        const DenseMatrix m = parse_gate_expression(expr);
        if (long(m.data.size()) * 2 > cap_doubles) return -100;
        std::memcpy(out, m.data.data(), sizeof(cplx) * m.data.size());
        return long(m.rows);
    } catch (const std::exception& ex) {
        g_err = ex.what();
        return -code_of(ex);
    }
}

// render_report's sampling (circuit_io.cpp:114-128) on a given state: the unmodified
// render_report (human format) runs on a report whose final state and probabilities are the
// given amplitudes, and its "samples (seed S): ..." line is parsed back into out.
// Returns the number of samples, or -(code) on a reference exception.
long io_sample(int n, const double* amps, int samples, unsigned long long seed, unsigned long long* out) {
    try {
        SimReport r;
        r.final = StateVector(n);
        std::memcpy(r.final.amps.data(), amps, sizeof(cplx) * r.final.amps.size());
        r.probabilities = r.final.probabilities();
        ReportOptions o;
        o.format = "human";
        o.samples = samples;
        o.seed = seed;
        o.engine = "dax";
        const std::string rep = render_report(r, n, o);
        const std::size_t at = rep.find("samples (seed ");
        if (at == std::string::npos) return 0;
        const char* p = rep.c_str() + rep.find("):", at) + 2;
        long k = 0;
        char* end = nullptr;
        for (; k < samples; ++k, p = end) {
            out[k] = std::strtoull(p, &end, 10);
            if (end == p) break;
        }
        return k;
    } catch (const std::exception& ex) {
        g_err = ex.what();
        return -code_of(ex);
    }
}

}  // extern "C"
