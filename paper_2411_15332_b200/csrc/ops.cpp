// ops.cpp -- placement canonicalisation and the gate-pass descriptor builder (host side).
//
// The reference builds the whole 2^n x 2^n step operator (engine.cpp:135-151) and multiplies
// (dax.cpp:96-103).  Its rows are sparse and structured: row r of a single-placement step
// has the gate's nonzeros of local row g(r) at columns r with the gate bits replaced.  This
// file turns one placement into that row recipe (the implicit "DAX descriptor") and into
// the minimal sub-cube of the state a kernel has to touch.
#include <algorithm>
#include <cstring>

#include "common.hpp"
#include "kernels.hpp"

namespace qcs {

GateOp canonical_op(int n, const qcs_placement& p) {
    if (p.arity < 1 || p.arity > QCS_MAX_ARITY) raise(QCS_ERR_ARG, "placement arity must be 1..3");
    if (!p.qubits || !p.matrix) raise(QCS_ERR_ARG, "placement without qubits or matrix");
    const int k = p.arity;
    int q[QCS_MAX_ARITY];
    for (int i = 0; i < k; ++i) {
        q[i] = p.qubits[i];
        if (q[i] < 0 || q[i] >= n) raise(QCS_ERR_DIMENSION, "gate placement out of range");  // circuit.cpp:53-54
        for (int j = 0; j < i; ++j)
            if (q[j] == q[i]) raise(QCS_ERR_DIMENSION, "overlapping gate placements in a step");
    }
    // canonical order: ascending qubit index == descending basis-bit position
    int perm[QCS_MAX_ARITY];  // canonical slot s takes original slot perm[s]
    for (int i = 0; i < k; ++i) perm[i] = i;
    std::sort(perm, perm + k, [&](int a, int b) { return q[a] < q[b]; });
    GateOp op;
    op.k = k;
    op.name = p.name ? p.name : "";
    for (int s = 0; s < k; ++s) op.pos[s] = n - 1 - q[perm[s]];
    const int dim = 1 << k;
    // canonical local index -> original local index (bit k-1-s of canonical <-> slot perm[s])
    auto to_orig = [&](int c) {
        int o = 0;
        for (int s = 0; s < k; ++s)
            if (c & (1 << (k - 1 - s))) o |= 1 << (k - 1 - perm[s]);
        return o;
    };
    op.m.resize(std::size_t(dim) * dim);
    for (int r = 0; r < dim; ++r)
        for (int c = 0; c < dim; ++c) {
            const std::size_t src = std::size_t(to_orig(r)) * dim + to_orig(c);
            op.m[std::size_t(r) * dim + c] = cplx{p.matrix[2 * src], p.matrix[2 * src + 1]};
        }
    return op;
}

namespace {
inline bool is_zero(const cplx& v) { return v.real() == 0.0 && v.imag() == 0.0; }
inline bool is_one(const cplx& v) { return v.real() == 1.0 && v.imag() == 0.0; }
}  // namespace

// Row recipe of a canonical op restricted to its touched sub-cube.  Returns false when the
// op is the identity (nothing to do: every row is e_g with value exactly 1, which dax_mvm
// reproduces bit for bit up to the sign of zero).
bool build_gate_desc(const GateOp& op, GateDesc& d) {
    std::memset(&d, 0, sizeof(d));
    const int k = op.k, dim = 1 << k;
    bool touched[8] = {}, needed[8] = {};
    int nt = 0;
    for (int g = 0; g < dim; ++g) {
        int nz = 0, only = -1;
        for (int c = 0; c < dim; ++c)
            if (!is_zero(op.m[std::size_t(g) * dim + c])) { ++nz; only = c; }
        const bool ident = nz == 1 && only == g && is_one(op.m[std::size_t(g) * dim + g]);
        if (!ident) {
            touched[g] = needed[g] = true;
            ++nt;
            for (int c = 0; c < dim; ++c)
                if (!is_zero(op.m[std::size_t(g) * dim + c])) needed[c] = true;
        }
    }
    if (nt == 0) return false;
    // Sector completion: when basis bit 0 is a gate bit (canonical local bit 0), close the
    // touched set under its flip, so every 32-byte sector (amplitudes 2u, 2u+1) is read and
    // written whole instead of half.  An added row is an identity row, computed as
    // 0 + (1+0i) * x -- exactly what dax_mvm writes for it (the DAX step holds that entry).
    if (op.pos[k - 1] == 0) {
        for (int g = 0; g < dim; ++g)
            if (touched[g] && !touched[g ^ 1]) {
                touched[g ^ 1] = needed[g ^ 1] = true;
                ++nt;
            }
    }
    // local bits constant across the needed set are fixed: the kernel enumerates only the
    // sub-cube (e.g. a CNOT touches half the state, a CZ a quarter)
    int fixed_mask = 0, fixed_val = 0;
    for (int b = 0; b < k; ++b) {
        int seen = -1;
        bool constant = true;
        for (int g = 0; g < dim; ++g) {
            if (!needed[g]) continue;
            const int v = (g >> b) & 1;
            if (seen < 0) seen = v; else if (seen != v) constant = false;
        }
        if (constant) { fixed_mask |= 1 << b; fixed_val |= seen << b; }
    }
    int free_local[3], nfree = 0;
    for (int b = 0; b < k; ++b)
        if (!(fixed_mask & (1 << b))) free_local[nfree++] = b;
    d.k = k;
    d.nfree = nfree;
    // local bit b <-> canonical slot s = k-1-b <-> basis position op.pos[k-1-b]
    for (int i = 0; i < k; ++i) d.pos_asc[i] = op.pos[k - 1 - i];  // pos[] is descending
    d.fixed_val = 0;
    for (int b = 0; b < k; ++b)
        if (fixed_val & (1 << b)) d.fixed_val |= std::uint64_t(1) << op.pos[k - 1 - b];
    for (int i = 0; i < nfree; ++i) d.free_bit[i] = std::uint64_t(1) << op.pos[k - 1 - free_local[i]];
    for (int m = 0; m < (1 << nfree); ++m)
        for (int i = 0; i < nfree; ++i)
            if (m & (1 << i)) d.member_off[m] |= d.free_bit[i];
    auto member_of = [&](int g) {
        int m = 0;
        for (int i = 0; i < nfree; ++i)
            if (g & (1 << free_local[i])) m |= 1 << i;
        return m;
    };
    d.load_mask = 0;
    for (int g = 0; g < dim; ++g)
        if (needed[g]) d.load_mask |= 1u << member_of(g);
    d.nrows = 0;
    for (int g = 0; g < dim; ++g) {
        if (!touched[g]) continue;
        const int r = d.nrows++;
        d.row_member[r] = std::uint8_t(member_of(g));
        int z = 0;
        for (int c = 0; c < dim; ++c) {  // ascending canonical column == ascending global column
            const cplx v = op.m[std::size_t(g) * dim + c];
            if (is_zero(v)) continue;    // dax_encode skips exact zeros (dax.cpp:42)
            d.col_member[r][z] = std::uint8_t(member_of(c));
            d.val[r][z] = make_double2(v.real(), v.imag());
            d.vkind[r][z] = std::uint8_t(v.imag() == 0.0 ? 1 : (v.real() == 0.0 ? 2 : 0));
            ++z;
        }
        d.nnz[r] = std::uint8_t(z);
    }
    return true;
}

}  // namespace qcs
