// shim_timing.cpp -- TEST INFRASTRUCTURE: times repeated qcsim::simulate calls made through the
// reference's own C++ API, linked against the B200 link-substitute (shim/engine_b200.cpp), on
// the C1 circuit (BASELINE configs[0], built with the reference's CircuitStep::of_gates and
// gate_catalog_lookup) and on Grover n=20 (build_grover).  Prints one JSON line: per-call
// wall-clock medians of the repeated calls, which reuse the shim's kept per-thread device state and
// its plan cache.  tests/test_shim_gpu.py compares them with qcs_simulate on a kept state.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "qcsim/circuit.hpp"
#include "qcsim/engine.hpp"

using namespace qcsim;

namespace {

Circuit c1_circuit(std::uint64_t seed) {
    const int n = 12;
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> ang(0.0, 2.0 * M_PI);
    Circuit c;
    c.n = n;
    std::vector<Placement> h;
    for (int q = 0; q < n; ++q) h.push_back({gate_catalog_lookup("Hadamard"), q});
    c.steps.push_back(CircuitStep::of_gates(h));
    for (int layer = 0; layer < 4; ++layer) {
        std::vector<Placement> ry, rz;
        for (int q = 0; q < n; ++q) ry.push_back({gate_catalog_lookup("RY", {ang(rng)}), q});
        c.steps.push_back(CircuitStep::of_gates(ry));
        for (int q = 0; q + 1 < n; ++q) c.steps.push_back(CircuitStep::of_gates({{gate_catalog_lookup("CNOT"), q}}));
        for (int q = 0; q < n; ++q) rz.push_back({gate_catalog_lookup("RZ", {ang(rng)}), q});
        c.steps.push_back(CircuitStep::of_gates(rz));
    }
    return c;
}

double median_ms(const Circuit& c, int reps) {
    std::vector<double> t;
    for (int i = 0; i < reps + 3; ++i) {
        const auto a = std::chrono::steady_clock::now();
        const SimReport r = simulate(c, Engine::rh_dax);
        const auto b = std::chrono::steady_clock::now();
        if (r.final.amps.empty()) std::abort();
        if (i >= 3) t.push_back(std::chrono::duration<double, std::milli>(b - a).count());
    }
    std::sort(t.begin(), t.end());
    return t[t.size() / 2];
}

}  // namespace

int main() {
    const Circuit c1 = c1_circuit(20241122);
    const Circuit g = build_grover(20, 12345, 8);
    const double t1 = median_ms(c1, 50);
    const double tg = median_ms(g, 20);
    std::printf("{\"c1_ms\": %.4f, \"grover20_ms\": %.4f}\n", t1, tg);
    return 0;
}
