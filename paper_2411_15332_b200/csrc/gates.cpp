// gates.cpp -- the gate catalog on the host (reference: proj/src/gates.cpp, 38 gates).
//
// The device never evaluates trigonometry: matrices are built here with std::complex<double>
// and std::cos / std::sin exactly as the reference composes them (gates.cpp:14-160), so the
// bytes handed to the kernels -- signed zeros included -- equal GateSpec::matrix::data.  The
// golden test tests/test_gates.py pins every entry against bytes produced by the reference.
#include <cmath>
#include <cstring>
#include <map>
#include <numbers>

#include "common.hpp"

namespace qcs {
namespace {

using M = std::vector<cplx>;
using P = const std::vector<double>&;

const double kH = 1.0 / std::sqrt(2.0);  // gates.cpp:11
const cplx kI{0.0, 1.0};                 // gates.cpp:12

cplx ei(double t) { return {std::cos(t), std::sin(t)}; }

M ident(int dim) {
    M m(std::size_t(dim) * dim);
    for (int i = 0; i < dim; ++i) m[std::size_t(i) * dim + i] = 1.0;
    return m;
}

// Controlled-U with the control on the higher-order qubit: U in the lower-right block
// (gates.cpp:28-34).
M ctrl(const M& u) {
    M m = ident(4);
    for (int r = 0; r < 2; ++r)
        for (int c = 0; c < 2; ++c) m[std::size_t(2 + r) * 4 + 2 + c] = u[std::size_t(r) * 2 + c];
    return m;
}

M phase(double lam) { return {1, 0, 0, ei(lam)}; }

M u3(double t, double phi, double lam) {  // gates.cpp:69-72
    const double c = std::cos(t / 2), s = std::sin(t / 2);
    return {c, -ei(lam) * s, ei(phi) * s, ei(phi + lam) * c};
}

M rz(double t) { return {ei(-t / 2), 0, 0, ei(t / 2)}; }

struct Def {
    int arity;
    int nparams;
    double ratio;  // declared zero ratio of the canonical form
    M (*build)(P);
};

// Keyed by canonical name; listing order is kOrder below.
const std::map<std::string, Def>& defs() {
    static const std::map<std::string, Def> t = {
        {"Hadamard", {1, 0, 0.0, [](P) -> M { return {kH, kH, kH, -kH}; }}},
        {"SX", {1, 0, 0.0, [](P) -> M {
             const cplx a{0.5, 0.5}, b{0.5, -0.5};
             return {a, b, b, a};
         }}},
        {"SXdg", {1, 0, 0.0, [](P) -> M {
             const cplx a{0.5, -0.5}, b{0.5, 0.5};
             return {a, b, b, a};
         }}},
        {"R", {1, 2, 0.0, [](P p) -> M {
             const double c = std::cos(p[0] / 2), s = std::sin(p[0] / 2);
             return {c, -kI * ei(-p[1]) * s, -kI * ei(p[1]) * s, c};
         }}},
        {"RX", {1, 1, 0.0, [](P p) -> M {
             const double c = std::cos(p[0] / 2), s = std::sin(p[0] / 2);
             return {c, -kI * s, -kI * s, c};
         }}},
        {"RY", {1, 1, 0.0, [](P p) -> M {
             const double c = std::cos(p[0] / 2), s = std::sin(p[0] / 2);
             return {c, -s, s, c};
         }}},
        {"U", {1, 3, 0.0, [](P p) -> M { return u3(p[0], p[1], p[2]); }}},
        {"U2", {1, 2, 0.0, [](P p) -> M {
             return {kH, -ei(p[1]) * kH, ei(p[0]) * kH, ei(p[0] + p[1]) * kH};
         }}},
        {"Identity", {1, 0, 0.5, [](P) -> M { return ident(2); }}},
        {"Pauli-X", {1, 0, 0.5, [](P) -> M { return {0, 1, 1, 0}; }}},
        {"Pauli-Y", {1, 0, 0.5, [](P) -> M { return {0, -kI, kI, 0}; }}},
        {"Pauli-Z", {1, 0, 0.5, [](P) -> M { return {1, 0, 0, -1}; }}},
        {"S", {1, 0, 0.5, [](P) -> M { return {1, 0, 0, kI}; }}},
        {"T", {1, 0, 0.5, [](P) -> M { return phase(std::numbers::pi / 4); }}},
        {"T-adjoint", {1, 0, 0.5, [](P) -> M { return phase(-std::numbers::pi / 4); }}},
        {"Phase", {1, 1, 0.5, [](P p) -> M { return phase(p[0]); }}},
        {"RZ", {1, 1, 0.5, [](P p) -> M { return rz(p[0]); }}},
        {"U1", {1, 1, 0.5, [](P p) -> M { return phase(p[0]); }}},
        {"CCX", {3, 0, 0.875, [](P) -> M {
             M m = ident(8);
             m[6 * 8 + 6] = 0;
             m[7 * 8 + 7] = 0;
             m[6 * 8 + 7] = 1;
             m[7 * 8 + 6] = 1;
             return m;
         }}},
        {"CSwap", {3, 0, 0.875, [](P) -> M {
             M m = ident(8);
             m[5 * 8 + 5] = 0;
             m[6 * 8 + 6] = 0;
             m[5 * 8 + 6] = 1;
             m[6 * 8 + 5] = 1;
             return m;
         }}},
        {"RXX", {2, 1, 0.5, [](P p) -> M {
             const cplx c = std::cos(p[0] / 2), s = -kI * std::sin(p[0] / 2);
             return {c, 0, 0, s, 0, c, s, 0, 0, s, c, 0, s, 0, 0, c};
         }}},
        {"RYY", {2, 1, 0.5, [](P p) -> M {
             const cplx c = std::cos(p[0] / 2), s = kI * std::sin(p[0] / 2);
             return {c, 0, 0, s, 0, c, -s, 0, 0, -s, c, 0, s, 0, 0, c};
         }}},
        {"RZX", {2, 1, 0.5, [](P p) -> M {
             const cplx c = std::cos(p[0] / 2), s = -kI * std::sin(p[0] / 2);
             return {c, s, 0, 0, s, c, 0, 0, 0, 0, c, -s, 0, 0, -s, c};
         }}},
        {"ECR", {2, 0, 0.5, [](P) -> M {
             const cplx h = kH;
             return {0, h, 0, kI * h, h, 0, -kI * h, 0, 0, kI * h, 0, h, -kI * h, 0, h, 0};
         }}},
        {"CH", {2, 0, 0.625, [](P) -> M { return ctrl({kH, kH, kH, -kH}); }}},
        {"CSX", {2, 0, 0.625, [](P) -> M {
             const cplx a{0.5, 0.5}, b{0.5, -0.5};
             return ctrl({a, b, b, a});
         }}},
        {"CU", {2, 4, 0.625, [](P p) -> M {
             M u = u3(p[0], p[1], p[2]);
             for (cplx& v : u) v *= ei(p[3]);
             return ctrl(u);
         }}},
        {"CU3", {2, 3, 0.625, [](P p) -> M { return ctrl(u3(p[0], p[1], p[2])); }}},
        {"RZZ", {2, 1, 0.75, [](P p) -> M {
             M m(16);
             m[0] = ei(-p[0] / 2);
             m[5] = ei(p[0] / 2);
             m[10] = ei(p[0] / 2);
             m[15] = ei(-p[0] / 2);
             return m;
         }}},
        {"Swap", {2, 0, 0.75, [](P) -> M { return {1, 0, 0, 0, 0, 0, 1, 0, 0, 1, 0, 0, 0, 0, 0, 1}; }}},
        {"iSwap", {2, 0, 0.75, [](P) -> M { return {1, 0, 0, 0, 0, 0, kI, 0, 0, kI, 0, 0, 0, 0, 0, 1}; }}},
        {"Controlled-X", {2, 0, 0.75, [](P) -> M { return ctrl({0, 1, 1, 0}); }}},
        {"Controlled-Y", {2, 0, 0.75, [](P) -> M { return ctrl({0, -kI, kI, 0}); }}},
        {"Controlled-Z", {2, 0, 0.75, [](P) -> M { return ctrl({1, 0, 0, -1}); }}},
        {"DCX", {2, 0, 0.75, [](P) -> M { return {1, 0, 0, 0, 0, 0, 0, 1, 0, 1, 0, 0, 0, 0, 1, 0}; }}},
        {"CPhase", {2, 1, 0.75, [](P p) -> M { return ctrl(phase(p[0])); }}},
        {"CRZ", {2, 1, 0.75, [](P p) -> M { return ctrl(rz(p[0])); }}},
        {"CU1", {2, 1, 0.75, [](P p) -> M { return ctrl(phase(p[0])); }}},
    };
    return t;
}

// Listing order (gates.cpp:249-258): grouped by shape / zero-ratio class.
const char* const kOrder[] = {
    "Hadamard", "SX", "SXdg", "R", "RX", "RY", "U", "U2",
    "Identity", "Pauli-X", "Pauli-Y", "Pauli-Z", "S", "T", "T-adjoint", "Phase", "RZ", "U1",
    "CCX", "CSwap",
    "RXX", "RYY", "RZX", "ECR",
    "CH", "CSX", "CU", "CU3",
    "RZZ", "Swap", "iSwap", "Controlled-X", "Controlled-Y", "Controlled-Z", "DCX", "CPhase",
    "CRZ", "CU1",
};
constexpr int kCatalogSize = int(sizeof(kOrder) / sizeof(kOrder[0]));

// Alias names (gates.cpp:224-234).
const std::map<std::string, std::string>& alias_map() {
    static const std::map<std::string, std::string> a = {
        {"H", "Hadamard"}, {"I", "Identity"}, {"X", "Pauli-X"}, {"Y", "Pauli-Y"}, {"Z", "Pauli-Z"},
        {"Tdg", "T-adjoint"}, {"P", "Phase"}, {"CX", "Controlled-X"}, {"CNOT", "Controlled-X"},
        {"CY", "Controlled-Y"}, {"CZ", "Controlled-Z"}, {"SWAP", "Swap"}, {"Toffoli", "CCX"},
        {"Fredkin", "CSwap"}, {"square root of Pauli-X", "SX"},
    };
    return a;
}

const std::pair<const std::string, Def>& find(const std::string& name) {
    auto al = alias_map().find(name);
    const std::string& key = al == alias_map().end() ? name : al->second;
    auto it = defs().find(key);
    if (it == defs().end()) raise(QCS_ERR_SIM, "unknown gate: " + name);
    return *it;
}

}  // namespace

int catalog_size() { return kCatalogSize; }

void catalog_entry(int i, const char** name, int* arity, int* nparams, double* ratio) {
    if (i < 0 || i >= kCatalogSize) raise(QCS_ERR_ARG, "catalog index out of range");
    const Def& d = defs().at(kOrder[i]);
    *name = kOrder[i];
    *arity = d.arity;
    *nparams = d.nparams;
    *ratio = d.ratio;
}

// gate_catalog_lookup (gates.cpp:277-292).  Returns the canonical name's storage.
const char* gate_lookup(const std::string& name, const std::vector<double>& params, std::vector<cplx>& out,
                        int* arity) {
    const auto& kv = find(name);
    const Def& d = kv.second;
    if (int(params.size()) != d.nparams)
        raise(QCS_ERR_SIM, "gate " + kv.first + " takes " + std::to_string(d.nparams) +
                               " parameter(s), got " + std::to_string(params.size()));
    out = d.build(params);
    *arity = d.arity;
    return kv.first.c_str();
}

// canonical_params (gates.cpp:241-242, :271-275).
std::vector<double> canonical_params(const std::string& name) {
    static const double kAngles[4] = {1.1, 0.7, 0.3, 0.9};
    const Def& d = find(name).second;
    return std::vector<double>(kAngles, kAngles + d.nparams);
}

}  // namespace qcs
