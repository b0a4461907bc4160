// ref_capi.cpp -- extern "C" access to the UNMODIFIED reference library (qcsim) for tests and
// for the CPU baseline.  TEST INFRASTRUCTURE ONLY: compiled by oracle/Makefile against
// /root/reference/proj/include and linked with the reference's own src/*.cpp objects into
// oracle/_ref/libqcsim_ref.so.  Nothing in the product links this.
//
// Every function below calls reference routines; the only logic of our own is argument
// marshalling and the projector decomposition for placements the reference cannot express
// (non-contiguous / reversed multi-qubit gates), which is built
// exclusively from the reference's dax_encode / dax_mtp.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <random>
#include <cstdint>
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include "qcsim/circuit.hpp"
#include "qcsim/engine.hpp"
#include "qcsim/gates.hpp"
#include "qcsim/rh.hpp"

using namespace qcsim;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const CapacityError*>(&e)) return 1;
    if (dynamic_cast<const DimensionError*>(&e)) return 2;
    if (dynamic_cast<const EncodingError*>(&e)) return 3;
    if (dynamic_cast<const ParseError*>(&e)) return 4;
    if (dynamic_cast<const SimError*>(&e)) return 5;
    return 9;
}

DenseMatrix to_dense(int k, const double* m) {
    const std::uint64_t dim = std::uint64_t(1) << k;
    DenseMatrix d(dim, dim);
    for (std::uint64_t i = 0; i < dim * dim; ++i) d.data[i] = cplx{m[2 * i], m[2 * i + 1]};
    return d;
}

struct PlacementIn {
    int k;
    std::vector<int> q;
    DenseMatrix m;
    std::string name;
    bool contiguous;
};

std::vector<PlacementIn> read_placements(int np, const int* arity, const int* qubits,
                                         const double* mats, const char* const* names) {
    std::vector<PlacementIn> out;
    int qo = 0;
    std::size_t mo = 0;
    for (int j = 0; j < np; ++j) {
        PlacementIn p;
        p.k = arity[j];
        p.q.assign(qubits + qo, qubits + qo + p.k);
        p.m = to_dense(p.k, mats + mo);
        p.name = names && names[j] ? names[j] : "custom";
        p.contiguous = true;
        for (int i = 1; i < p.k; ++i)
            if (p.q[i] != p.q[i - 1] + 1) p.contiguous = false;
        qo += p.k;
        mo += std::size_t(2) << (2 * p.k);
        out.push_back(std::move(p));
    }
    return out;
}

GateSpec spec_of(const PlacementIn& p) {
    GateSpec g;
    g.name = p.name;
    g.arity = p.k;
    g.matrix = p.m;
    return g;
}

// Factor list for one projector term, positions MSB first (engine.cpp:31-52 ordering).
// choice[j] selects the (a,b) control assignment of non-contiguous placement j.
DaxMatrix fold_term(int n, const std::vector<PlacementIn>& ps, const std::vector<int>& choice,
                    bool& zero_term) {
    static const DenseMatrix id2 = DenseMatrix::identity(2);
    std::vector<DenseMatrix> factors;
    int q = 0;
    zero_term = false;
    while (q < n) {
        bool placed = false;
        for (std::size_t j = 0; j < ps.size() && !placed; ++j) {
            const PlacementIn& p = ps[j];
            if (p.contiguous) {
                if (p.q[0] == q) {
                    factors.push_back(p.m);
                    q += p.k;
                    placed = true;
                }
                continue;
            }
            for (int i = 0; i < p.k; ++i) {
                if (p.q[i] != q) continue;
                const int nc = p.k - 1;
                const int a = choice[j] >> nc, b = choice[j] & ((1 << nc) - 1);
                DenseMatrix f(2, 2);
                if (i < nc) {
                    const int ai = (a >> (nc - 1 - i)) & 1, bi = (b >> (nc - 1 - i)) & 1;
                    f.at(ai, bi) = cplx{1.0, 0.0};
                } else {
                    bool any = false;
                    for (int x = 0; x < 2; ++x)
                        for (int y = 0; y < 2; ++y) {
                            f.at(x, y) = p.m.at((std::uint64_t(a) << 1) | x, (std::uint64_t(b) << 1) | y);
                            if (f.at(x, y) != cplx{0.0, 0.0}) any = true;
                        }
                    if (!any) zero_term = true;
                }
                factors.push_back(f);
                q += 1;
                placed = true;
                break;
            }
        }
        if (!placed) {
            factors.push_back(id2);
            q += 1;
        }
    }
    DaxMatrix acc = dax_encode(factors[0]);
    for (std::size_t i = 1; i < factors.size(); ++i) acc = dax_mtp(acc, dax_encode(factors[i]));
    return acc;
}

DaxMatrix general_step_dax(int n, const std::vector<PlacementIn>& ps) {
    bool all_native = true;
    for (const auto& p : ps) all_native &= p.contiguous;
    if (all_native) {
        std::vector<Placement> pl;
        for (const auto& p : ps) pl.push_back({spec_of(p), p.q[0]});
        return step_matrix_dax(CircuitStep::of_gates(pl), n);
    }
    // projector decomposition: iterate every (a,b) control assignment of every
    // non-contiguous placement, fold each term with the reference, merge by (row, col).
    std::vector<int> choice(ps.size(), 0), limit(ps.size(), 1);
    for (std::size_t j = 0; j < ps.size(); ++j)
        if (!ps[j].contiguous) limit[j] = 1 << (2 * (ps[j].k - 1));
    DaxMatrix merged;
    merged.rows = merged.cols = std::uint64_t(1) << n;
    for (;;) {
        bool zero_term = false;
        DaxMatrix t = fold_term(n, ps, choice, zero_term);
        if (!zero_term) merged.entries.insert(merged.entries.end(), t.entries.begin(), t.entries.end());
        std::size_t j = 0;
        while (j < ps.size() && ++choice[j] == limit[j]) choice[j++] = 0;
        if (j == ps.size()) break;
    }
    std::sort(merged.entries.begin(), merged.entries.end(), [](const DaxEntry& a, const DaxEntry& b) {
        return a.row != b.row ? a.row < b.row : a.col < b.col;
    });
    return merged;
}

StateVector to_state(int n, const double* s) {
    StateVector v;
    v.n = n;
    v.amps.resize(std::size_t(1) << n);
    std::memcpy(v.amps.data(), s, sizeof(double) * 2 * v.amps.size());
    return v;
}

double seconds_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_catalog_size() { return int(gate_catalog().size()); }

int ref_catalog_entry(int i, char* name, int cap, int* arity, int* nparams, double* ratio) {
    const GateInfo& g = gate_catalog().at(std::size_t(i));
    std::snprintf(name, std::size_t(cap), "%s", g.name.c_str());
    *arity = g.arity;
    *nparams = g.param_count;
    *ratio = g.zero_ratio;
    return 0;
}

int ref_gate_lookup(const char* name, const double* params, int np, double* out, int* arity) {
    try {
        const GateSpec g = gate_catalog_lookup(name, std::vector<double>(params, params + np));
        *arity = g.arity;
        std::memcpy(out, g.matrix.data.data(), sizeof(cplx) * g.matrix.data.size());
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_canonical_params(const char* name, double* out, int* np) {
    try {
        const auto p = canonical_params(name);
        *np = int(p.size());
        std::copy(p.begin(), p.end(), out);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// step_matrix_dax (native placements) or the projector decomposition (general placements).
long ref_step_dax(int n, int np, const int* arity, const int* qubits, const double* mats,
                  std::uint64_t* rows, std::uint64_t* cols, double* vals, long cap) {
    try {
        const DaxMatrix m = general_step_dax(n, read_placements(np, arity, qubits, mats, nullptr));
        if (long(m.entries.size()) > cap) return -1;
        for (std::size_t i = 0; i < m.entries.size(); ++i) {
            rows[i] = m.entries[i].row;
            cols[i] = m.entries[i].col;
            vals[2 * i] = m.entries[i].value.real();
            vals[2 * i + 1] = m.entries[i].value.imag();
        }
        return long(m.entries.size());
    } catch (const std::exception& e) {
        return -10 - fail(e);
    }
}

// step_matrix_das; native placements only.
long ref_step_das(int n, int np, const int* arity, const int* qubits, const double* mats,
                  std::uint64_t* dis, std::uint8_t* last, double* vals, long cap) {
    try {
        const auto ps = read_placements(np, arity, qubits, mats, nullptr);
        std::vector<Placement> pl;
        for (const auto& p : ps) {
            if (!p.contiguous) throw SimError("DAS oracle needs contiguous placements");
            pl.push_back({spec_of(p), p.q[0]});
        }
        const DasMatrix m = step_matrix_das(CircuitStep::of_gates(pl), n);
        if (long(m.entries.size()) > cap) return -1;
        for (std::size_t i = 0; i < m.entries.size(); ++i) {
            dis[i] = m.entries[i].dis;
            last[i] = m.entries[i].last_in_row ? 1 : 0;
            vals[2 * i] = m.entries[i].value.real();
            vals[2 * i + 1] = m.entries[i].value.imag();
        }
        return long(m.entries.size());
    } catch (const std::exception& e) {
        return -10 - fail(e);
    }
}

// step_matrix_dax / step_matrix_das of native placements, serialised by the reference's own
// dax_dump / das_dump (dax.cpp:107-118, das.cpp:154-165).  das: 0 = DAX1, 1 = DAS1.  Returns the
// byte count (or -(bytes) when cap is too small).
long ref_step_dump(int n, int np, const int* arity, const int* qubits, const double* mats, int das,
                   unsigned char* out, long cap) {
    try {
        const auto ps = read_placements(np, arity, qubits, mats, nullptr);
        std::vector<Placement> pl;
        for (const auto& p : ps) {
            if (!p.contiguous) throw SimError("dump oracle needs contiguous placements");
            pl.push_back({spec_of(p), p.q[0]});
        }
        std::ostringstream os;
        if (das) das_dump(step_matrix_das(CircuitStep::of_gates(pl), n), os);
        else dax_dump(step_matrix_dax(CircuitStep::of_gates(pl), n), os);
        const std::string b = os.str();
        if (long(b.size()) > cap) return -long(b.size());
        std::memcpy(out, b.data(), b.size());
        return long(b.size());
    } catch (const std::exception& e) {
        return -10 - fail(e);
    }
}

// Reference single-step pipeline (engine.cpp:192-199): step_matrix_dax then dax_mvm, timed
// separately (build = the MTP fold, mvm = the compressed MVM).  engine: 1 = dax, 2 = das.
int ref_apply_step(int n, int np, const int* arity, const int* qubits, const double* mats, int engine,
                   const double* in, double* out, double* t_build, double* t_mvm) {
    try {
        const auto ps = read_placements(np, arity, qubits, mats, nullptr);
        const StateVector s = to_state(n, in);
        StateVector r;
        auto t0 = std::chrono::steady_clock::now();
        if (engine == 2) {
            std::vector<Placement> pl;
            for (const auto& p : ps) pl.push_back({spec_of(p), p.q[0]});
            const DasMatrix m = step_matrix_das(CircuitStep::of_gates(pl), n);
            *t_build = seconds_since(t0);
            t0 = std::chrono::steady_clock::now();
            r = das_mvm(m, s);
        } else {
            const DaxMatrix m = general_step_dax(n, ps);
            *t_build = seconds_since(t0);
            t0 = std::chrono::steady_clock::now();
            r = dax_mvm(m, s);
        }
        *t_mvm = seconds_since(t0);
        std::memcpy(out, r.amps.data(), sizeof(cplx) * r.amps.size());
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_dax_mvm(int n, const std::uint64_t* rows, const std::uint64_t* cols, const double* vals,
                long count, const double* in, double* out) {
    try {
        DaxMatrix m;
        m.rows = m.cols = std::uint64_t(1) << n;
        m.entries.resize(std::size_t(count));
        for (long i = 0; i < count; ++i) m.entries[i] = {rows[i], cols[i], cplx{vals[2 * i], vals[2 * i + 1]}};
        const StateVector r = dax_mvm(m, to_state(n, in));
        std::memcpy(out, r.amps.data(), sizeof(cplx) * r.amps.size());
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_das_mvm(int n, const std::uint64_t* dis, const std::uint8_t* last, const double* vals,
                long count, const double* in, double* out) {
    try {
        DasMatrix m;
        m.rows = m.cols = std::uint64_t(1) << n;
        m.entries.resize(std::size_t(count));
        for (long i = 0; i < count; ++i) m.entries[i] = {dis[i], last[i] != 0, cplx{vals[2 * i], vals[2 * i + 1]}};
        const StateVector r = das_mvm(m, to_state(n, in));
        std::memcpy(out, r.amps.data(), sizeof(cplx) * r.amps.size());
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_rh_mvm(int n, const double* in, double* out, int method, std::uint64_t* sign_count,
               std::uint64_t* madd_count) {
    try {
        RhMvmStats st;
        const StateVector r = rh_mvm(rh_build(n), to_state(n, in), SignMethod(method), &st);
        std::memcpy(out, r.amps.data(), sizeof(cplx) * r.amps.size());
        *sign_count = st.sign_count;
        *madd_count = st.madd_count;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Whole-circuit simulate (engine.cpp:153-210).  Steps are flattened:
//   kind[s] (0 gates, 1 diag), stage[s], nplace[s] placements taken in order from
//   (arity, qubits, mats, names); diag steps take nflip[s] indices from flipped and flip_rest[s].
// Only native (contiguous) placements: this is the reference's own API.
int ref_simulate(int n, std::uint64_t initial, int nsteps, const int* kind, const int* stage,
                 const int* nplace, const int* arity, const int* qubits, const double* mats,
                 const char* const* names, const std::uint64_t* nflip, const std::uint64_t* flipped,
                 const int* flip_rest, int engine, int sign_method, double* out_state,
                 std::uint64_t* rep /* per step: matrix_bytes, dense_bytes, entry_count, sign_count, madd_count, structure-code */,
                 double* seconds) {
    try {
        Circuit c;
        c.n = n;
        c.initial = initial;
        int pi = 0, qo = 0;
        std::size_t mo = 0, fo = 0;
        for (int s = 0; s < nsteps; ++s) {
            if (kind[s] == 1) {
                DiagSign d;
                d.flipped.assign(flipped + fo, flipped + fo + nflip[s]);
                d.flip_rest = flip_rest[s] != 0;
                fo += nflip[s];
                c.steps.push_back(CircuitStep::of_diag(std::move(d), stage[s]));
                continue;
            }
            std::vector<Placement> pl;
            for (int j = 0; j < nplace[s]; ++j, ++pi) {
                GateSpec g;
                g.name = names[pi];
                g.arity = arity[pi];
                g.matrix = to_dense(arity[pi], mats + mo);
                pl.push_back({g, qubits[qo]});
                qo += arity[pi];
                mo += std::size_t(2) << (2 * arity[pi]);
            }
            c.steps.push_back(CircuitStep::of_gates(std::move(pl), stage[s]));
        }
        SimOptions opt;
        opt.sign_method = SignMethod(sign_method);
        const auto t0 = std::chrono::steady_clock::now();
        const SimReport r = simulate(c, Engine(engine), opt);
        *seconds = seconds_since(t0);
        std::memcpy(out_state, r.final.amps.data(), sizeof(cplx) * r.final.amps.size());
        for (std::size_t s = 0; s < r.steps.size(); ++s) {
            const StepReport& sr = r.steps[s];
            rep[6 * s + 0] = sr.matrix_bytes;
            rep[6 * s + 1] = sr.dense_bytes;
            rep[6 * s + 2] = sr.entry_count;
            rep[6 * s + 3] = sr.sign_count;
            rep[6 * s + 4] = sr.madd_count;
            rep[6 * s + 5] = sr.structure == "dense" ? 0 : sr.structure == "dax" ? 1 : sr.structure == "das" ? 2 : 3;
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Reference circuit builders, simulated with the given engine (circuit.cpp:80-149).
int ref_grover(int n, std::uint64_t marked, int iterations, int engine, double* out_state,
               int* nsteps) {
    try {
        const Circuit c = build_grover(n, marked, iterations);
        *nsteps = int(c.steps.size());
        const SimReport r = simulate(c, Engine(engine));
        std::memcpy(out_state, r.final.amps.data(), sizeof(cplx) * r.final.amps.size());
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

std::uint64_t ref_grover_auto_iterations(int n) { return grover_auto_iterations(n); }

int ref_qnn(int inputs, const double* angles, const int* weights, int engine, double* out_state,
            int* n_out) {
    try {
        const Circuit c = build_qnn_neuron(inputs, std::vector<double>(angles, angles + inputs),
                                           std::vector<int>(weights, weights + inputs));
        *n_out = c.n;
        const SimReport r = simulate(c, Engine(engine));
        std::memcpy(out_state, r.final.amps.data(), sizeof(cplx) * r.final.amps.size());
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// test_util.hpp:23-35 random_unit_state (mt19937_64 + std::normal_distribution).
void ref_random_unit_state(int n, std::uint64_t seed, double* out) {
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> dist;
    StateVector s(n);
    double norm2 = 0.0;
    for (cplx& a : s.amps) {
        a = {dist(rng), dist(rng)};
        norm2 += std::norm(a);
    }
    const double inv = 1.0 / std::sqrt(norm2);
    for (cplx& a : s.amps) a *= inv;
    std::memcpy(out, s.amps.data(), sizeof(cplx) * s.amps.size());
}

int ref_quadrant_sign(std::uint64_t r, std::uint64_t c, int n) { return quadrant_sign(r, c, n); }

}  // extern "C"
