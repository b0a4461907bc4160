// jit.cpp -- per-pass specialised tile kernels, generated and compiled at run time (NVRTC).
//
// The interpreter kernel k_tile (tile_kernels.cu) walks each pass's operation list from the
// kernel parameter space: every group of 8 amplitudes pays for the operation dispatch, the
// coefficient loads and -- because all operation kinds share one register assignment -- the
// register moves that reconcile the kinds' code paths.  Gate-heavy passes (C4, C5) are issue
// bound on exactly that overhead (profiles/r01_ncu_full_tile_c4.json).  Here the pass's
// STRUCTURE -- rounds, register bits, operation kinds, target bits, control masks, sign tables --
// becomes straight-line CUDA source built from the same device building blocks
// (tile_device.cuh), so the generated kernel does exactly the interpreter's arithmetic in the
// same order (bit-identical results) without any of the dispatch.  Coefficients stay in the
// kernel parameters, so one compiled kernel serves every pass of the same structure (the layers
// of a circuit, circuits with new angles).  Kernels are cached by their source text.
#include <cuda.h>
#include <nvrtc.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <string>
#include <thread>
#include <vector>

#include <unistd.h>

#include "common.hpp"
#include "kernels.hpp"

namespace qcs {

extern const char* const kJitSrcKernels;  // kernels.hpp and tile_device.cuh, embedded by build.py
extern const char* const kJitSrcDevice;

namespace {

struct Out {
    std::string s;
    void operator()(const char* fmt, ...) __attribute__((format(printf, 2, 3))) {
        char buf[1024];
        va_list ap;
        va_start(ap, fmt);
        const int k = std::vsnprintf(buf, sizeof(buf), fmt, ap);
        va_end(ap);
        if (k >= int(sizeof(buf))) raise(QCS_ERR_SIM, "internal: generated line too long");
        s += buf;
    }
};


// FP64 instructions (DFMA / DMUL / DADD, per thread) the generated code executes per group of 8
// amplitudes, accumulated while a pass's source is generated (pass_fp64_per_tile): the
// roofline's compute side for the FP64-bound passes (bench.py)
thread_local double g_fp64 = 0.0;
thread_local double g_fp64_groups = 1.0;  // groups per tile of the round being generated
void fp64(double k) { g_fp64 += k * g_fp64_groups; }

// Addressing proof (QCS_JIT_VERIFY=1 or qcs_plan_compile's verify mode): while a round is
// generated, its address arithmetic is also evaluated for every thread, group iteration and
// register, under every combination of the runtime relabelling terms, and must address each of
// the tile's 2^m shared-memory slots exactly once (in bounds, a permutation) -- and likewise
// the direct HBM stores of a relabelled last round.  compute-sanitizer is closed on this GPU
// pool; this checks the one place where a bad shared-memory index could come from.
bool verify_on() {
    static const bool on = [] { const char* v = std::getenv("QCS_JIT_VERIFY"); return v && std::atoi(v) != 0; }();
    return on;
}
thread_local bool g_verify = false;

bool knob_swaps() {
    static const bool on = [] { const char* v = std::getenv("QCS_JIT_SWAPS"); return !v || std::atoi(v) != 0; }();
    return on;
}

// a non-signed diagonal whose phase bits are all constant over a register group (dk <= 2)
bool group_const(const RegOp& op) {
    return op.dk >= 1 && op.dk <= 2 && op.dreg[0] == 0xff && (op.dk == 1 || op.dreg[1] == 0xff);
}

bool has_pivot(const PassParams& p) {  // pivoted gates or virtual permutations: specialised kernels only
    for (int i = 0; i < p.nops; ++i) {
        const int k = p.ops[i].kind & KF_KIND;
        if ((k == TOP_GATE && (p.ops[i].kind & KF_PIVOT)) || k == TOP_PERM) return true;
    }
    return false;
}

int knob_unroll() {
    static const int u = [] { const char* v = std::getenv("QCS_JIT_UNROLL"); return v ? std::atoi(v) : 1; }();
    return u;
}

bool knob_bankswap() {
    static const bool on = [] { const char* v = std::getenv("QCS_JIT_BANKSWAP"); return !v || std::atoi(v) != 0; }();
    return on;
}

// the cg (value of the group-constant phase bits) expression of a +-1 diagonal, as source
std::string const_bits(bool c0, bool c1, int dk, int p0, int p1) {
    std::string e = "0";
    char buf[128];
    if (c0) {
        std::snprintf(buf, sizeof(buf), " | (int((g0 >> %d) & 1) << %d)", p0, dk - 1);
        e += buf;
    }
    if (c1) {
        std::snprintf(buf, sizeof(buf), " | int((g0 >> %d) & 1)", p1);
        e += buf;
    }
    return e;
}

// Lazy +-1 sign flips (round 2).  The CZ ring between a round's two layers and the Z-like parts
// of gates leave registers negated; the interpreter (and round 1) xor-ed the sign bits of all
// eight registers before every later gate (~4 integer instructions per amplitude per flush).
// Here the pending signs are tracked while the round is generated -- a compile-time mask `ct`
// plus runtime terms that are linear in the register index (group-constant phase bits times a
// register bit: rs0..rs2, or all registers: rsc) -- and consumed for free where the arithmetic
// allows: a pivoted gate takes a pair's sign difference as the sign of its ratio (an operand
// negation in the DFMA; a runtime difference flips the ratio once per group) and passes the
// signs on to its outputs; the round's diagonal table takes them as signed entries.  Anything
// else (butterflies, non-pivoted gates, sign steps, the round's end) flushes them first.  Sign
// flips are exact, so the results are bit for bit those of flushing early.
// Measured on B200 (tools/gpu_r02p.sh, three alternating repetitions): C4 n=32 276.5 ms with the
// track, 268.5 ms without -- slower: the ratio flips and signed table entries sit on the FMA
// critical path where the xor flushes did not.  Kept as an option (QCS_JIT_LAZY_SIGNS=1).
bool knob_lazy_signs() {
    static const bool on = [] { const char* v = std::getenv("QCS_JIT_LAZY_SIGNS"); return v && std::atoi(v) != 0; }();
    return on;
}

struct SignTrack {
    unsigned ct = 0;           // compile-time: registers negated
    bool rt[4] = {};           // runtime terms pending in rs0, rs1, rs2 (registers with bit b set), rsc (all)
    bool any() const { return ct || rt[0] || rt[1] || rt[2] || rt[3]; }
};
const char* const kRs[4] = {"rs0", "rs1", "rs2", "rsc"};

// the runtime part of register q's sign as a source expression ("" when none)
std::string rt_parity(const SignTrack& st, int q) {
    std::string e;
    for (int b = 0; b < 4; ++b)
        if (st.rt[b] && (b == 3 || (q >> b & 1))) e += (e.empty() ? "" : " ^ ") + std::string(kRs[b]);
    return e;
}

void sign_reset_rt(Out& o, SignTrack& st) {
    for (int b = 0; b < 4; ++b)
        if (st.rt[b]) {
            o("      %s = 0u;\n", kRs[b]);
            st.rt[b] = false;
        }
}

// apply every pending sign to the registers (xor of sign bits) and clear the track
void sign_flush(Out& o, SignTrack& st) {
    if (!st.any()) return;
    std::string m = std::to_string(st.ct) + "u";
    static const unsigned pat[4] = {0xaau, 0xccu, 0xf0u, 0xffu};
    for (int b = 0; b < 4; ++b)
        if (st.rt[b]) m += " ^ ((0u - " + std::string(kRs[b]) + ") & " + std::to_string(pat[b]) + "u)";
    o("      flip_mask(v, %s);\n", m.c_str());
    st.ct = 0;
    sign_reset_rt(o, st);
}

// a +-1 diagonal whose flipped registers are byte cg of smask when the group-constant phase
// bits spell cg: the cg-independent part joins ct; each runtime part must be affine-linear in the
// register index (then it becomes rs terms); false (nothing emitted) otherwise
bool sign_add(Out& o, SignTrack& st, unsigned long long smask, bool c0, bool c1, int dk, int p0, int p1) {
    auto byte = [&](int cg) { return unsigned(smask >> (8 * cg)) & 0xffu; };
    std::string ue, we;  // cg bit 1 and bit 0 as runtime 0/1 expressions
    char buf[64];
    if (dk == 2 && c0) { std::snprintf(buf, sizeof(buf), "unsigned((g0 >> %d) & 1)", p0); ue = buf; }
    if (dk == 2 && c1) { std::snprintf(buf, sizeof(buf), "unsigned((g0 >> %d) & 1)", p1); we = buf; }
    if (dk == 1 && c0) { std::snprintf(buf, sizeof(buf), "unsigned((g0 >> %d) & 1)", p0); we = buf; }
    const unsigned f0 = byte(0);
    struct Term { unsigned m; std::string e; };
    std::vector<Term> terms;
    if (!we.empty()) terms.push_back({byte(1) ^ f0, we});
    if (!ue.empty()) terms.push_back({byte(2) ^ f0, ue});
    if (!we.empty() && !ue.empty()) terms.push_back({byte(3) ^ byte(2) ^ byte(1) ^ f0, "(" + ue + " & " + we + ")"});
    struct Lin { bool a0, a[3]; };
    std::vector<Lin> lins;
    for (const Term& t : terms) {
        Lin l{};
        l.a0 = t.m & 1u;
        for (int b = 0; b < 3; ++b) l.a[b] = ((t.m >> (1 << b)) & 1u) != l.a0;
        for (int q = 0; q < 8; ++q) {
            bool v = l.a0;
            for (int b = 0; b < 3; ++b) v ^= l.a[b] && (q >> b & 1);
            if (v != bool(t.m >> q & 1u)) return false;
        }
        lins.push_back(l);
    }
    st.ct ^= f0;
    for (std::size_t i = 0; i < terms.size(); ++i) {
        if (!terms[i].m) continue;
        for (int b = 0; b < 3; ++b)
            if (lins[i].a[b]) {
                o("      %s ^= %s;\n", kRs[b], terms[i].e.c_str());
                st.rt[b] = true;
            }
        if (lins[i].a0) {
            o("      rsc ^= %s;\n", terms[i].e.c_str());
            st.rt[3] = true;
        }
    }
    return true;
}

// A one-target gate on register bit t of the registers in `en` (a literal mask): X-like gates
// (exactly [[0, 1], [1, 0]]) are register swaps -- no arithmetic, value-identical to the
// interpreter's 0*x0 + 1*x1 up to the sign of an exact zero -- the others the real or complex
// 2x2 forms of tile_device.cuh.
void emit_gate(Out& o, int kb, int t, const double2* c, const std::string& coef, unsigned en, int G, unsigned piv,
               SignTrack* st = nullptr) {
    const unsigned all = (1u << G) - 1;
    // pending signs: a pivoted or swap gate on all registers consumes / permutes them; any other
    // gate needs them applied first
    auto swap_bits = [&](unsigned m) {  // exchange the sign bits of each pair along t
        unsigned r = m;
        for (int q = 0; q < G; ++q)
            if (!(q >> t & 1)) {
                const unsigned a = m >> q & 1u, b = m >> (q | (1 << t)) & 1u;
                r = (r & ~((1u << q) | (1u << (q | (1 << t))))) | (b << q) | (a << (q | (1 << t)));
            }
        return r;
    };
    auto pairs = [&](unsigned e) {
        int k = 0;
        for (int q = 0; q < G; ++q)
            if (!(q >> t & 1) && (e >> q & 1)) ++k;
        return k;
    };
    if (kb & KF_PIVOT) {  // piv: this bit's 4 pivot flags
        const int per_row = (kb & KF_REAL) ? 2 : 4;
        fp64(double(pairs(en & all)) * (((piv >> 2 & 1) ? 0 : per_row) + ((piv >> 3 & 1) ? 0 : per_row)));
        const int P0 = int(piv & 1), P1 = int(piv >> 1 & 1);
        if (st && st->any() && (en & all) != all && !(P0 == 0 && P1 == 1)) sign_flush(o, *st);
        unsigned neg = 0;
        std::string r0 = "(" + coef + ")[0]", r1 = "(" + coef + ")[1]";
        if (st && st->any()) {
            for (int q = 0; q < G; ++q)
                if (!(q >> t & 1) && ((st->ct >> q) ^ (st->ct >> (q | (1 << t)))) & 1u) neg |= 1u << q;
            if (st->rt[t]) {  // the runtime sign difference of every pair along t: flip the ratios
                r0 = "flipd2(" + r0 + ", " + kRs[t] + ")";
                r1 = "flipd2(" + r1 + ", " + kRs[t] + ")";
            }
        }
        if (en & all)
            o("      gate1p<%d, %d, %d, %d, %d, %d, 0x%xu, 0x%xu>(v, %s, %s);\n", t, P0, P1, int(piv >> 2 & 1),
              int(piv >> 3 & 1), (kb & KF_REAL) ? 1 : 0, en & all, neg, r0.c_str(), r1.c_str());
        if (st && st->any()) {  // the outputs carry the sign of their row's pivot input
            if (P0 == 1 && P1 == 0) {
                st->ct = swap_bits(st->ct);
                if (st->rt[t]) { o("      rsc ^= %s;\n", kRs[t]); st->rt[3] = true; }
            } else if (P0 == 0 && P1 == 0) {
                for (int q = 0; q < G; ++q)
                    if (!(q >> t & 1)) st->ct = (st->ct & ~(1u << (q | (1 << t)))) | ((st->ct >> q & 1u) << (q | (1 << t)));
                if (st->rt[t]) { o("      %s = 0u;\n", kRs[t]); st->rt[t] = false; }
            } else if (P0 == 1 && P1 == 1) {
                for (int q = 0; q < G; ++q)
                    if (!(q >> t & 1)) st->ct = (st->ct & ~(1u << q)) | ((st->ct >> (q | (1 << t)) & 1u) << q);
                if (st->rt[t]) {
                    o("      rsc ^= %s; %s = 0u;\n", kRs[t], kRs[t]);
                    st->rt[3] = true;
                    st->rt[t] = false;
                }
            }
        }
        return;
    }
    const bool swap = c[0].x == 0.0 && c[0].y == 0.0 && c[3].x == 0.0 && c[3].y == 0.0 && c[1].x == 1.0 &&
                      c[1].y == 0.0 && c[2].x == 1.0 && c[2].y == 0.0 && knob_swaps();
    if (st && st->any()) {
        if (swap && (en & all) == all) {  // a register swap permutes the pending signs
            st->ct = swap_bits(st->ct);
            if (st->rt[t]) { o("      rsc ^= %s;\n", kRs[t]); st->rt[3] = true; }
        } else {
            sign_flush(o, *st);
        }
    }
    if (swap) {
        for (int q = 0; q < G; ++q)
            if (!(q >> t & 1) && (en >> q & 1))
                o("      { const double2 x = v[%d]; v[%d] = v[%d]; v[%d] = x; }\n", q, q, q | (1 << t), q | (1 << t));
        return;
    }
    const char* g = (kb & KF_REAL) ? "gate1r" : "gate1";
    fp64(double(pairs(en & all)) * ((kb & KF_REAL) ? 8 : 16));
    if ((en & all) == all) o("      %s<%d, false>(v, %s, 0xffffu);\n", g, t, coef.c_str());
    else if (en) o("      %s<%d, true>(v, %s, 0x%xu);\n", g, t, coef.c_str(), en);
}

// The layout relabelling of the virtual permutations (TOP_PERM): an affine map over GF(2) on
// the local index bits, x -> A x ^ b (column i of A = the image of bit i).
// Gates controlled only outside the tile add a term to the offset on the tiles where their
// controls hold (a condition on the tile base, uniform over the CTA): `rt`.
struct Affine {
    unsigned col[16];
    unsigned b = 0;
    std::vector<std::pair<const RegOp*, unsigned>> rt;  // (op whose outside controls gate it, vector)
    explicit Affine(int m) {
        for (int i = 0; i < 16; ++i) col[i] = i < m ? 1u << i : 0u;
    }
    bool identity(int m) const {
        for (int i = 0; i < m; ++i)
            if (col[i] != 1u << i) return false;
        return b == 0 && rt.empty();
    }
    std::string offset_expr() const {  // b and the runtime terms, as source
        char buf[160];
        std::snprintf(buf, sizeof(buf), "%uu", b);
        std::string e = buf;
        for (const auto& [op, v] : rt) {
            std::snprintf(buf, sizeof(buf), " ^ (((base & 0x%llxull) == 0x%llxull) ? %uu : 0u)",
                          (unsigned long long)op->gctrl_mask, (unsigned long long)op->gctrl_val, v);
            e += buf;
        }
        return e;
    }
    unsigned apply(unsigned x) const {
        unsigned y = b;
        for (int i = 0; i < 16; ++i)
            if (x >> i & 1) y ^= col[i];
        return y;
    }
    // the permutation of an X-like gate: x -> x ^ (cond(x) ? e_t : 0), cond = (x & cm) == cv
    // (cm at most one bit): linear part M = I + e_t e_c^T (with a control c), offset d
    static void perm(const RegOp& op, unsigned& e_t, int& c, unsigned& d) {
        e_t = 1u << op.t;
        c = op.lctrl_mask ? __builtin_ctz(unsigned(op.lctrl_mask)) : -1;
        d = (c < 0 || !(op.lctrl_val >> c & 1)) ? e_t : 0u;
    }
    void compose_right(const RegOp& op) {  // this <- this o pi (loads after the permutation)
        unsigned e_t, d;
        int c;
        perm(op, e_t, c, d);
        const unsigned colt = apply(e_t) ^ b;  // A e_t
        if (op.gctrl_mask) {  // x ^ e_t on the tiles where the outside controls hold
            rt.push_back({&op, colt});
            return;
        }
        if (c >= 0) col[c] ^= colt;
        b ^= apply(d) ^ b;  // A d
    }
    void compose_left(const RegOp& op) {  // this <- pi o this (stores of the permuted result)
        unsigned e_t, d;
        int c;
        perm(op, e_t, c, d);
        if (op.gctrl_mask) {
            rt.push_back({&op, e_t});
            return;
        }
        auto mul = [&](unsigned v) { return c >= 0 && (v >> c & 1) ? v ^ e_t : v; };
        for (int i = 0; i < 16; ++i) col[i] = mul(col[i]);
        for (auto& term : rt) term.second = mul(term.second);
        b = mul(b) ^ d;
    }
};

// source of A x (no offset) for the local group index `var` whose register bits are zero
std::string affine_expr(const Affine& A, const char* var, unsigned regmask, int m) {
    unsigned idmask = 0;
    std::string e;
    for (int i = 0; i < m; ++i) {
        if (regmask >> i & 1) continue;
        if (A.col[i] == 1u << i) {
            idmask |= 1u << i;
            continue;
        }
        char buf[96];
        std::snprintf(buf, sizeof(buf), " ^ ((0u - ((%s >> %d) & 1u)) & %uu)", var, i, A.col[i]);
        e += buf;
    }
    char head[64];
    std::snprintf(head, sizeof(head), "(%s & %uu)", var, idmask);
    return head + e;
}

// A +-1 diagonal whose phase bits are register bits and/or bits constant over the group
// (c0 / c1: phase bit 0 / 1 is group-constant, at basis position p0 / p1).  sm holds, per value
// cg of the constant bits, the G-bit mask of registers that flip.  The flips that do not depend
// on the group (cg = 0) are returned for the round's pending mask `negacc`, which thereby stays a
// compile-time constant (flip_signs1 then touches only the flagged registers); the
// group-dependent rest is applied here, one conditional xor of the sign bit per affected
// register (flip_cond) -- merging it into negacc made every later flush a run-time mask over all
// registers (~5 integer instructions per register; 17% of a C4 pass's instructions).
unsigned long long emit_signed(Out& o, unsigned long long sm, bool c0, bool c1, int dk, int p0, int p1, int G) {
    const unsigned long long gmask = (1ull << G) - 1;
    auto field = [&](int cg) { return (sm >> (G * cg)) & gmask; };
    const unsigned long long m0 = field(0);
    if (!c0 && !c1) return m0;
    static const bool split = [] { const char* v = std::getenv("QCS_JIT_SPLIT_SIGNS"); return !v || std::atoi(v) != 0; }();
    if (!split) {  // A/B: the group-dependent flips into negacc as well
        o("      negacc ^= unsigned(0x%llxull >> (%d * (%s))) & 0x%llxu;\n", sm, G, const_bits(c0, c1, dk, p0, p1).c_str(), gmask);
        return 0;
    }
    for (int a = 0; a <= (c0 ? 1 : 0); ++a)
        for (int b = 0; b <= (c1 ? 1 : 0); ++b) {
            if (!a && !b) continue;
            const int cg = (a << (dk - 1)) | b;
            const unsigned long long d = field(cg) ^ m0;
            if (!d) continue;
            auto term = [](int pos, int want) {  // 1u when basis bit `pos` of the group equals `want`
                const std::string b = "(unsigned(g0 >> " + std::to_string(pos) + ") & 1u)";
                return want ? b : "(" + b + " ^ 1u)";
            };
            std::string cond;
            if (c0) cond = term(p0, a);
            if (c1) cond = cond.empty() ? term(p1, b) : "(" + cond + " & " + term(p1, b) + ")";
            o("      flip_cond<0x%llxu>(v, %s);\n", d, cond.c_str());
        }
    return m0;
}


// One register round: the interpreter's round loop (tile_kernels.cu) with every structural
// field of the operations as a literal.  (16-amplitude rounds -- 4 register bits, 22% fewer
// rounds for C4 -- were measured no faster at 2 resident tiles per SM and slower for C3.)
// `map`: the layout relabelling so far (updated by the round's leading TOP_PERM ops); `last`:
// the program's last round, which stores straight to HBM when the layout is not the identity
// or trailing TOP_PERM ops permute its result.  Returns true when it did.
bool emit_register_round(Out& o, const PassParams& P, int ri, unsigned threads, Affine& map, bool last) {
    const RoundDesc& R = P.rounds[ri];
    int ob = R.op_begin, oe = R.op_begin + R.op_count;
    while (ob < oe && (P.ops[ob].kind & KF_KIND) == TOP_PERM) map.compose_right(P.ops[ob++]);
    Affine store(P.m);  // trailing permutations: where the round's (last) results go
    int te = oe;
    while (te > ob && (P.ops[te - 1].kind & KF_KIND) == TOP_PERM) --te;
    for (int i = te; i < oe; ++i) store.compose_left(P.ops[i]);
    if (te < oe && !last) raise(QCS_ERR_SIM, "internal: trailing relabelling outside a pass's last round");
    const bool relabel = !map.identity(P.m);
    const bool direct = last && (relabel || te < oe);
    const int W = round_width(R), G = 1 << W;  // 3 or 4 register bits (RD_W4)
    const unsigned long long gmask = (1ull << G) - 1;
    const unsigned ngroups = (1u << P.m) >> W;
    g_fp64_groups = double(ngroups);
    unsigned off[16] = {};
    unsigned regmask = 0;
    for (int i = 0; i < W; ++i) regmask |= 1u << round_reg(R, i);
    for (int q = 0; q < G; ++q)
        for (int i = 0; i < W; ++i)
            if (q >> i & 1) off[q] |= 1u << round_reg(R, i);
    auto swz = [](unsigned j) { return j ^ ((j >> 3) & 7u); };
    o("  {  // round %d: register bits", ri);
    for (int i = 0; i < W; ++i) o(" %d", round_reg(R, i));
    o("\n");
    // Thread order: the 8 threads of one 16-byte shared-memory phase differ in gb's low 3 bits,
    // i.e. in the round's lowest 3 non-register tile bits.  Their bank group is bits 0..2 XOR
    // bits 3..5 of the (swizzled) position; when those three bits do not map to 8 distinct
    // groups, swap one of them with a higher non-register bit that does (same groups, another
    // thread order: the accesses become conflict-free).
    auto bank = [&](int b) { const unsigned v = map.col[b]; return (v & 7u) ^ ((v >> 3) & 7u); };
    auto independent = [&](int a, int b, int c) {
        const unsigned x = bank(a), y = bank(b), z = bank(c);
        return x && y && z && x != y && x != z && y != z && (x ^ y) != z;
    };
    std::vector<int> nonreg;
    for (int b = 0; b < P.m; ++b)
        if (!(regmask >> b & 1)) nonreg.push_back(b);
    int swap_a = -1, swap_b = -1;
    if (knob_bankswap() && nonreg.size() >= 4 && !independent(nonreg[0], nonreg[1], nonreg[2])) {
        for (int i = 0; i < 3 && swap_a < 0; ++i)
            for (std::size_t j = 3; j < nonreg.size() && swap_a < 0; ++j) {
                int c[3] = {nonreg[0], nonreg[1], nonreg[2]};
                c[i] = nonreg[j];
                if (independent(c[0], c[1], c[2])) {
                    swap_a = nonreg[std::size_t(i)];
                    swap_b = nonreg[j];
                }
            }
    }
    // The group index lb = S(D(gb)) (D: zeros inserted at the register bits, S: the swap) and
    // its relabelled position are linear in gb, and gb = t + k * threads: the thread's part is
    // computed once per round, each iteration adds a constant.
    auto deposit = [&](unsigned g) {
        for (int i = 0; i < W; ++i) g = ((g >> round_reg(R, i)) << (round_reg(R, i) + 1)) | (g & ((1u << round_reg(R, i)) - 1));
        if (swap_a >= 0 && ((g >> swap_a) ^ (g >> swap_b)) & 1u) g ^= (1u << swap_a) | (1u << swap_b);
        return g;
    };
    const unsigned iters = ngroups > threads ? ngroups / threads : 1u;
    std::vector<unsigned> lk, pk, sk;  // per bit j of k: lb, A lb and A_s lb of k = 2^j
    for (unsigned j = 0; (1u << j) < iters; ++j) {
        const unsigned l = deposit(threads << j);
        lk.push_back(l);
        pk.push_back(map.apply(l) ^ map.b);
        sk.push_back(store.apply(l) ^ store.b);
    }
    auto kexpr = [&](const std::vector<unsigned>& v) {
        std::string e = "0u";
        char buf[96];
        for (std::size_t j = 0; j < v.size(); ++j) {
            std::snprintf(buf, sizeof(buf), " ^ ((0u - ((k >> %zu) & 1u)) & %uu)", j, v[j]);
            e += buf;
        }
        return e;
    };
    if (g_verify || verify_on()) {
        const unsigned tsz = 1u << P.m;
        auto swz1 = [](unsigned j) { return j ^ ((j >> 3) & 7u); };
        auto sw = [&](unsigned g) {  // lb_t of thread t: zeros at the register bits, then the swap
            for (int i = 0; i < W; ++i) g = ((g >> round_reg(R, i)) << (round_reg(R, i) + 1)) | (g & ((1u << round_reg(R, i)) - 1));
            if (swap_a >= 0 && ((g >> swap_a) ^ (g >> swap_b)) & 1u) g ^= (1u << swap_a) | (1u << swap_b);
            return g;
        };
        auto kx = [](const std::vector<unsigned>& v, unsigned k) {
            unsigned x = 0;
            for (std::size_t j = 0; j < v.size(); ++j)
                if (k >> j & 1) x ^= v[j];
            return x;
        };
        // the runtime relabelling terms XOR a tile-uniform constant into every address: a
        // permutation of the tile stays one when each term lies inside the tile, so check that
        // and prove the rest with the terms off
        for (const auto& term : map.rt)
            if (term.second >= tsz) raise(QCS_ERR_SIM, "internal: a runtime relabelling term leaves the tile");
        for (const auto& term : store.rt)
            if (term.second >= tsz) raise(QCS_ERR_SIM, "internal: a runtime relabelling term leaves the tile");
        const std::size_t nrt = 0, nst = 0;
        const unsigned nthreads = threads > ngroups ? ngroups : threads;
        for (unsigned combo = 0; combo < (1u << nrt); ++combo) {
            unsigned rtv = 0;
            (void)combo;
            std::vector<unsigned char> seen(tsz, 0);
            for (unsigned t = 0; t < nthreads; ++t) {
                const unsigned lbt = sw(t);
                const unsigned plt = map.apply(lbt) ^ rtv;  // affine_expr(lb_t) ^ offset_expr
                for (unsigned k = 0; k < iters; ++k) {
                    const unsigned slb = swz1(plt ^ kx(pk, k));
                    for (int q = 0; q < G; ++q) {
                        const unsigned pos = slb ^ swz1(map.apply(off[q]) ^ map.b);
                        if (pos >= tsz || seen[pos]++)
                            raise(QCS_ERR_SIM, "internal: round " + std::to_string(ri) +
                                                   " addresses a shared-memory slot twice or out of the tile");
                    }
                }
            }
        }
        if (direct) {  // the last round's stores straight to HBM: a permutation of the tile too
            for (unsigned combo = 0; combo < (1u << nst); ++combo) {
                unsigned rtv = 0;
                (void)combo;
                std::vector<unsigned char> seen(tsz, 0);
                for (unsigned t = 0; t < nthreads; ++t) {
                    const unsigned sdt = store.apply(sw(t)) ^ rtv;
                    for (unsigned k = 0; k < iters; ++k) {
                        const unsigned sd = sdt ^ kx(sk, k);
                        for (int q = 0; q < G; ++q) {
                            const unsigned cq = store.apply(off[q]) ^ store.b;
                            const unsigned loc = ((sd ^ cq) & 7u) | ((sd >> 3) << 3 ^ (cq >> 3) << 3);
                            if (loc >= tsz || seen[loc]++)
                                raise(QCS_ERR_SIM, "internal: direct stores of round " + std::to_string(ri) +
                                                       " hit an amplitude twice or leave the tile");
                        }
                    }
                }
            }
        }
    }
    std::string lbx = "t";
    for (int i = 0; i < W; ++i) lbx = "insert_zero(" + lbx + ", " + std::to_string(round_reg(R, i)) + ")";
    o("    unsigned lb_t = %s;\n", lbx.c_str());
    if (swap_a >= 0)
        o("    { const unsigned d = ((lb_t >> %d) ^ (lb_t >> %d)) & 1u; lb_t ^= (d << %d) | (d << %d); }\n", swap_a,
          swap_b, swap_a, swap_b);
    if (relabel)
        o("    const unsigned pl_t = %s ^ %s;\n", affine_expr(map, "lb_t", regmask, P.m).c_str(),
          map.offset_expr().c_str());
    else
        o("    const unsigned pl_t = lb_t;\n");
    if (direct)
        o("    const unsigned sd_t = %s ^ %s;\n", affine_expr(store, "lb_t", regmask, P.m).c_str(),
          store.offset_expr().c_str());
    if (threads > ngroups) o("    if (t < %uu)\n", ngroups);
    o("#pragma unroll %d\n", knob_unroll());
    o("    for (unsigned k = 0; k < %uu; ++k) {\n", iters);
    o("      const unsigned lb = lb_t ^ %s;\n", kexpr(lk).c_str());
    o("      const unsigned slb = swz(pl_t ^ %s);  // physical position of the group's first amplitude\n",
      kexpr(pk).c_str());
    unsigned soff[16];
    for (int q = 0; q < G; ++q) soff[q] = swz(map.apply(off[q]) ^ map.b);  // A off[q]
    o("      double2 v[%d];\n", G);
    for (int q = 0; q < G; ++q) o("      v[%d] = sm[slb ^ %uu];\n", q, soff[q]);
    o("      const u64 g0 = base | (lb & 7u) | hi_tab[lb >> 3];\n");
    o("      unsigned negacc = 0;\n");
    // phases constant over a group (diagonals on bits outside the registers) multiply into one
    // scalar per group when a round has several -- passes that pivot their gates only (a
    // different rounding; the pivot-free passes stay value-identical to the interpreter)
    int nconst = 0;
    for (int oi = ob; oi < te; ++oi)
        if ((P.ops[oi].kind & KF_KIND) == TOP_DIAG && !(P.ops[oi].kind & KF_SIGNED) && group_const(P.ops[oi])) ++nconst;
    const bool accumulate = nconst >= 2 && has_pivot(P);
    if (accumulate) o("      double2 gs = make_double2(1.0, 0.0);\n");
    o("      (void)g0; (void)negacc;\n");
    const bool lazy = knob_lazy_signs() && W == 3;  // the track is written for 8 registers
    SignTrack st;
    SignTrack* stp = lazy ? &st : nullptr;
    if (lazy) o("      unsigned rs0 = 0u, rs1 = 0u, rs2 = 0u, rsc = 0u;\n      (void)rs0; (void)rs1; (void)rs2; (void)rsc;\n");
    for (int oi = ob; oi < te; ++oi) {
        const RegOp& op = P.ops[oi];
        const int kb = op.kind, kind = kb & KF_KIND;
        if (kind == TOP_PERM) raise(QCS_ERR_SIM, "internal: relabelling inside a round");
        if (!lazy && (kb & KF_FLUSH)) o("      flip_signs1(v, negacc);\n");
        // lazy signs: operations that neither commute with pending flips nor consume them
        if (lazy && (kind == TOP_WHT || kind == TOP_SIGN || (kind == TOP_GATE && (kb & KF_GCTRL)))) sign_flush(o, st);
        const bool gc = kb & KF_GCTRL;
        if (gc) o("      if ((base & 0x%llxull) == 0x%llxull) {\n", (unsigned long long)op.gctrl_mask,
                  (unsigned long long)op.gctrl_val);
        if (lazy && kind == TOP_DIAG && (kb & KF_SIGNED)) {
            // +-1 diagonals into the sign track; a pattern that is not affine in the register
            // index (never in the BASELINE circuits) is applied at once
            auto one = [&](unsigned long long sm, bool c0, bool c1, int dk, int p0, int p1) {
                if (sign_add(o, st, sm, c0, c1, dk, p0, p1)) return;
                o("      flip_mask(v, unsigned(0x%llxull >> (%d * (%s))) & 0x%llxu);\n", sm, G,
                  const_bits(c0, c1, dk, p0, p1).c_str(), gmask);
            };
            if (kb & KF_BUNDLE) {
                st.ct ^= unsigned(op.smask & gmask);
                for (int i = 0; i < op.t; ++i) {
                    SignEntry e;
                    std::memcpy(&e, &P.pool[op.ref + i], sizeof(e));
                    one(e.smask, e.cmask & 1u, e.cmask & 2u, e.dk, e.p0, e.p1);
                }
            } else {
                one(op.smask, op.dreg[0] == 0xff, op.dk == 2 && op.dreg[1] == 0xff, op.dk, op.dpos[0], op.dpos[1]);
            }
        } else if (kind == TOP_DIAG && (kb & KF_SIGNED) && (kb & KF_BUNDLE)) {
            unsigned long long acc = op.smask & gmask;
            for (int i = 0; i < op.t; ++i) {
                SignEntry e;
                std::memcpy(&e, &P.pool[op.ref + i], sizeof(e));
                acc ^= emit_signed(o, e.smask, e.cmask & 1u, e.cmask & 2u, e.dk, e.p0, e.p1, G);
            }
            if (acc) o("      negacc ^= 0x%llxu;\n", acc);
        } else if (kind == TOP_DIAG && (kb & KF_SIGNED)) {
            const bool c0 = op.dreg[0] == 0xff, c1 = op.dk == 2 && op.dreg[1] == 0xff;
            unsigned long long sm = op.smask;  // byte cg: the registers that flip when the constant bits spell cg
            if (W == 4) {  // 16 registers: the 16-bit masks from the phase bits (dskip = the -1 entries)
                sm = 0;
                for (int cg = 0; cg < 4; ++cg)
                    for (int q = 0; q < G; ++q) {
                        int g = 0;
                        for (int i = 0; i < op.dk; ++i) {
                            const int bit = op.dreg[i] < W ? (q >> op.dreg[i]) & 1
                                                           : (i == 0 && op.dk == 2 ? (cg >> 1) & 1 : cg & 1);
                            g |= bit << (op.dk - 1 - i);
                        }
                        if (op.dskip >> g & 1) sm |= 1ull << (16 * cg + q);
                    }
            }
            const unsigned long long acc = emit_signed(o, sm, c0, c1, op.dk, op.dpos[0], op.dpos[1], G);
            if (acc) o("      negacc ^= 0x%llxu;\n", acc);
        } else if (kind == TOP_WHT) {
            for (int b = 0; b < W; ++b)
                if (op.t >> b & 1) {
                    o("      butterfly<%d>(v);\n", b);
                    fp64(16);
                }
        } else if (kind == TOP_SCALE) {
            o("      { const double sc = P.ops[%d].c[0].x;\n", oi);
            o("        for (int q = 0; q < %d; ++q) v[q] = make_double2(v[q].x * sc, v[q].y * sc); }\n", G);
            fp64(2 * G);
        } else if (kind == TOP_GATE && (kb & KF_BUNDLE)) {
            for (int b = 0; b < W; ++b)
                if (op.t >> b & 1) emit_gate(o, kb, b, P.pool + op.ref + 4 * b, "P.pool + " + std::to_string(op.ref + 4 * b),
                                             (1u << G) - 1, G, (op.dtab >> (4 * b)) & 15u, stp);
        } else if (kind == TOP_GATE) {
            // controls on register bits select registers (a literal mask); controls on the other
            // tile bits are one condition per group
            const unsigned cmr = unsigned(op.lctrl_mask) & regmask, cvr = unsigned(op.lctrl_val) & regmask;
            const unsigned cmn = unsigned(op.lctrl_mask) & ~regmask, cvn = unsigned(op.lctrl_val) & ~regmask;
            unsigned en = 0;
            for (int q = 0; q < G; ++q)
                if ((off[q] & cmr) == cvr) en |= 1u << q;
            if (cmn && lazy) sign_flush(o, st);  // a per-group condition: the track cannot follow it
            if (cmn) o("      if ((lb & %uu) == %uu) {\n", cmn, cvn);
            emit_gate(o, kb, op.t, op.c, "P.ops[" + std::to_string(oi) + "].c", en, G, op.dtab & 15u, cmn ? nullptr : stp);
            if (cmn) o("      }\n");
        } else if (kind == TOP_DTAB && lazy && st.any()) {
            // the round's diagonal table takes the pending signs as signed entries
            for (int q = 0; q < G; ++q) {
                const bool cs = st.ct >> q & 1u;
                const std::string rp = rt_parity(st, q);
                if (op.dskip >> q & 1) {  // entry exactly 1: only the sign, if any
                    if (cs || !rp.empty())
                        o("      v[%d] = flipd2(v[%d], %s);\n", q, q, (std::string(cs ? "1u" : "0u") + (rp.empty() ? "" : " ^ " + rp)).c_str());
                    continue;
                }
                fp64(P.pool[op.ref + q].y == 0.0 ? 2 : 4);
                if (P.pool[op.ref + q].y == 0.0) {
                    std::string sx = std::string(cs ? "-" : "") + "P.pool[" + std::to_string(op.ref + q) + "].x";
                    if (!rp.empty()) sx = "flipd(" + sx + ", " + rp + ")";
                    o("      { const double s = %s; v[%d] = make_double2(v[%d].x * s, v[%d].y * s); }\n", sx.c_str(), q, q, q);
                } else {
                    std::string e = "P.pool[" + std::to_string(op.ref + q) + "]";
                    if (cs) e = "make_double2(-" + e + ".x, -" + e + ".y)";
                    if (!rp.empty()) e = "flipd2(" + e + ", " + rp + ")";
                    o("      v[%d] = cmul_f(%s, v[%d]);\n", q, e.c_str(), q);
                }
            }
            st.ct = 0;
            sign_reset_rt(o, st);
        } else if (kind == TOP_DTAB) {
            const unsigned skipm = W == 4 ? unsigned(op.smask) : unsigned(op.dskip);
            for (int q = 0; q < G; ++q) {
                if (skipm >> q & 1) continue;
                fp64(P.pool[op.ref + q].y == 0.0 ? 2 : 4);
                if (P.pool[op.ref + q].y == 0.0)  // real entry (e.g. only gate row scales): 2 FP64
                    o("      { const double s = P.pool[%d].x; v[%d] = make_double2(v[%d].x * s, v[%d].y * s); }\n", op.ref + q,
                      q, q, q);
                else
                    o("      v[%d] = cmul_f(P.pool[%d], v[%d]);\n", q, op.ref + q, q);
            }
        } else if (kind == TOP_DIAG && accumulate && group_const(op)) {
            // a phase constant over the group: into the group's scalar, applied once at the end
            fp64(4);
            if (op.dk == 1) {
                o("      { const int g = int((g0 >> %d) & 1);\n", op.dpos[0]);
                o("        if (!((%uu >> g) & 1u)) gs = cmul_f(g ? P.ops[%d].c[1] : P.ops[%d].c[0], gs); }\n",
                  unsigned(op.dskip), oi, oi);
            } else {
                o("      { const int g = (int((g0 >> %d) & 1) << 1) | int((g0 >> %d) & 1);\n", op.dpos[0], op.dpos[1]);
                o("        if (!((%uu >> g) & 1u)) { double2 d = P.ops[%d].c[0]; if (g == 1) d = P.ops[%d].c[1];\n",
                  unsigned(op.dskip), oi, oi);
                o("          if (g == 2) d = P.ops[%d].c[2]; if (g == 3) d = P.ops[%d].c[3]; gs = cmul_f(d, gs); } }\n", oi,
                  oi);
            }
        } else if (kind == TOP_DIAG) {
            fp64(4 * G);
            if (op.dk == 1 && op.dreg[0] == 0xff) {
                o("      { const int g = int((g0 >> %d) & 1);\n", op.dpos[0]);
                o("        if (!((%uu >> g) & 1u)) { const double2 d = g ? P.ops[%d].c[1] : P.ops[%d].c[0];\n",
                  unsigned(op.dskip), oi, oi);
                o("          for (int q = 0; q < %d; ++q) v[q] = cmul_f(d, v[q]); } }\n", G);
            } else if (op.dk == 1) {
                o("      diag_reg<%d>(v, P.ops[%d].c[0], P.ops[%d].c[1], %uu);\n", op.dreg[0], oi, oi, unsigned(op.dskip));
            } else if (op.dk == 2 && has_pivot(P) && ((op.dreg[0] == 0xff) != (op.dreg[1] == 0xff))) {
                // one register bit and one bit constant over the group: two entries per group, a
                // static choice per register (no per-register selection)
                const int ci = op.dreg[0] == 0xff ? 0 : 1, ri = 1 - ci, rb = op.dreg[ri];
                auto entry = [&](int rv, const char* cb) {  // source of the entry for register-bit value rv
                    char buf[96];
                    if (ri == 0) std::snprintf(buf, sizeof(buf), "P.ops[%d].c[%d | %s]", oi, rv << 1, cb);
                    else std::snprintf(buf, sizeof(buf), "P.ops[%d].c[(%s << 1) | %d]", oi, cb, rv);
                    return std::string(buf);
                };
                o("      { const int cb = int((g0 >> %d) & 1);\n", op.dpos[ci]);
                o("        const double2 e0 = %s, e1 = %s;\n", entry(0, "cb").c_str(), entry(1, "cb").c_str());
                for (int q = 0; q < G; ++q) o("        v[%d] = cmul_f(e%d, v[%d]);\n", q, (q >> rb) & 1, q);
                o("      }\n");
            } else if (W == 4) {  // 16 registers: the entry index per register, constant bits at run time
                std::string cgx = "0";
                for (int i = 0; i < op.dk; ++i)
                    if (op.dreg[i] >= W)
                        cgx += " | (int((g0 >> " + std::to_string(op.dpos[i]) + ") & 1) << " + std::to_string(op.dk - 1 - i) + ")";
                o("      { const int cg = %s; (void)cg;\n", cgx.c_str());
                for (int q = 0; q < G; ++q) {
                    int rp = 0;
                    for (int i = 0; i < op.dk; ++i)
                        if (op.dreg[i] < W) rp |= ((q >> op.dreg[i]) & 1) << (op.dk - 1 - i);
                    if (op.dk <= 2)
                        o("        { const int g = cg | %d; if (!((%uu >> g) & 1u)) v[%d] = cmul_f(P.ops[%d].c[g], v[%d]); }\n", rp,
                          unsigned(op.dskip), q, oi, q);
                    else
                        o("        { const int g = cg | %d; if (!((%uu >> g) & 1u)) v[%d] = cmul_f(big[%d].val[0][g], v[%d]); }\n",
                          rp, unsigned(op.dskip), q, op.ref, q);
                }
                o("      }\n");
            } else {
                o("      diag_op(v, P.ops[%d], big, g0);\n", oi);
            }
        } else if (kind == TOP_SIGN) {
            o("      { const TileOp& so = big[%d];\n", op.ref);
            o("        if (!(sign_hit >> %u & 1u)) {\n", unsigned(op.sidx) & 31u);
            o("          if (so.flip_rest) { for (int q = 0; q < %d; ++q) v[q] = neg_exact(v[q]); }\n", G);
            fp64(8 * G);
            o("        } else {\n");
            o("          const u64* f = flipped + so.flip_off;\n");
            for (int q = 0; q < G; ++q) {
                o("          { const unsigned j = lb | %uu; const u64 gi = base | (j & 7u) | hi_tab[j >> 3];\n", off[q]);
                o("            if (listed(f, so.flip_cnt, gi) != (so.flip_rest != 0)) v[%d] = neg_exact(v[%d]); }\n", q, q);
            }
            o("        } }\n");
        } else {
            raise(QCS_ERR_SIM, "internal: operation kind without a generated form");
        }
        if (gc) o("      }\n");
    }
    if (accumulate)
        for (int q = 0; q < G; ++q) o("      v[%d] = cmul_f(gs, v[%d]);\n", q, q);
    if (accumulate) fp64(4 * G);
    if (!lazy && (R.flags & RD_SIGNS)) o("      flip_signs1(v, negacc);\n");
    if (lazy) sign_flush(o, st);
    if (direct) {  // straight to HBM: logical index store(lb ^ off[q]) of the tile
        o("      { const unsigned sd = sd_t ^ %s;\n", kexpr(sk).c_str());
        o("        const u64 gs = base | hi_tab[sd >> 3];\n");
        for (int q = 0; q < G; ++q) {
            const unsigned cq = store.apply(off[q]) ^ store.b;  // A_s off[q]
            o("        __stcs(a + (gs ^ u64((sd ^ %uu) & 7u) ^ hi_tab[%u]), v[%d]);\n", cq, cq >> 3, q);
        }
        o("      }\n    }\n  }\n");
        return true;
    }
    for (int q = 0; q < G; ++q) o("      sm[slb ^ %uu] = v[%d];\n", soff[q], q);
    o("    }\n    QCS_SYNC();\n  }\n");
    return false;
}

void emit_smem_round(Out& o, const PassParams& P, int ri, unsigned threads) {
    const RoundDesc& R = P.rounds[ri];
    o("  {  // round %d: gates on 2-3 targets in shared memory\n", ri);
    for (int oi = R.op_begin; oi < R.op_begin + R.op_count; ++oi) {
        o("    { const TileOp& o = big[%d];\n", P.ops[oi].ref);
        o("      if (!(o.gctrl_mask && (base & o.gctrl_mask) != o.gctrl_val)) {\n");
        o("        if (o.gcase == 2) smem_gate<2>(sm, o, %d, %uu); else smem_gate<3>(sm, o, %d, %uu);\n", P.m, threads,
          P.m, threads);
        o("      }\n      QCS_SYNC(); }\n");
    }
    o("  }\n");
}

// one program (the main rounds or the missed-tile alternative), then the tile's write-back
bool emit_rounds(Out& o, const PassParams& P, int begin, int end, unsigned threads, bool persist = false) {
    Affine map(P.m);
    bool direct = false;
    for (int ri = begin; ri < end; ++ri) {
        if (P.rounds[ri].flags & RD_SMEM) {
            if (!map.identity(P.m)) raise(QCS_ERR_SIM, "internal: shared-memory round after a relabelling");
            emit_smem_round(o, P, ri, threads);
        } else {
            direct = emit_register_round(o, P, ri, threads, map, ri + 1 == end);
        }
    }
    if (persist) return direct;  // the caller emits the ring's write-back / refill
    if (!direct) o("  tile_end(a, P, tmap, c);\n");
    return direct;
}

// ---- persistent pipelined form (tile_device.cuh, "persistent pipelined passes")
// Which passes take it: plain gate/diagonal passes (no sign steps, shared-memory rounds, skip or
// support masks, tile lists) with enough tiles to fill the ring on every SM.  QCS_PERSIST /
// qcs_set_pipeline_mode: 0 off; 1 (default) passes with 16-register rounds whose tile moves as
// TMA boxes and is stored through shared memory (those run 2 CTAs per SM otherwise); 2 every
// eligible pass, including relabelled passes (direct stores) and cp.async-loaded tiles --
// measured slower for passes of 8-register rounds (profiles/r02_ab_round_scheduler.txt).
std::atomic<int> g_persist{[] { const char* e = std::getenv("QCS_PERSIST"); return e ? std::atoi(e) : 1; }()};
int persist_knob() { return g_persist.load(std::memory_order_relaxed); }
constexpr unsigned kPersistThreads = 512, kPersistRing = 196608;  // two groups of 256; bytes of ring
unsigned persist_slots(const PassParams& P) {
    static const int cap = [] { const char* e = std::getenv("QCS_PERSIST_SLOTS"); return e ? std::atoi(e) : 4; }();
    return std::min<unsigned>(unsigned(cap), kPersistRing / (16u << P.m));
}
int pass_state_bits(const PassParams& P) {
    int n = P.m;
    for (int i = 0; i < P.nruns; ++i) n += P.run_len[i];
    return n;
}
bool has_direct_store(const PassParams& P) {
    // the last round stores straight to HBM when a relabelling is live at it (emit_register_round)
    for (int i = 0; i < P.nops; ++i)
        if ((P.ops[i].kind & KF_KIND) == TOP_PERM) return true;
    return false;
}
bool persist_wanted(const PassParams& P, unsigned F) {
    const int knob = persist_knob();
    if (knob <= 0 || P.m < 10 || P.m > 12) return false;
    if ((F & (4u | 8u)) || P.alt_mode != ALT_NONE || P.list_cnt || P.init || P.zmask || P.smask) return false;
    bool w4 = false;
    for (int r = 0; r < P.nrounds; ++r) {
        if (P.rounds[r].flags & RD_SMEM) return false;
        w4 |= (P.rounds[r].flags & RD_W4) != 0;
    }
    const int n = pass_state_bits(P);
    if (n - P.m < 11) return false;  // >= 2048 tiles: several ring turns per SM
    if (persist_slots(P) < 3) return false;
    // the default: passes with 16-register rounds whose tile moves as TMA boxes and whose last
    // round stores through shared memory; mode 2 adds 8-register passes, relabelled passes (direct
    // stores) and tiles that load as per-thread cp.async copies
    if (knob == 1) return w4 && !has_direct_store(P) && tile_tma_iter(n, P) >= 0;
    return true;
}

std::string pass_source(const PassParams& P, unsigned F, unsigned threads, bool persist) {
    Out o;
    static const int minb_env = [] { const char* v = std::getenv("QCS_JIT_MINB"); return v ? std::atoi(v) : 0; }();
    static const int w4_minb = [] { const char* v = std::getenv("QCS_W4_MINB"); return v ? std::atoi(v) : 2; }();
    bool w4 = false;
    for (int r = 0; r < P.nrounds; ++r) w4 |= (P.rounds[r].flags & RD_W4) != 0;
    // resident tiles per SM: 3 (80 registers) for 8-register rounds; 16-register rounds need ~100
    const int minb = minb_env > 0 ? minb_env : w4 ? w4_minb : (F & 8u) ? 2 : 3;
    o("#include \"tile_device.cuh\"\n");
    o("using namespace qcs;\nusing namespace qcs::tile;\n");
    if (persist) {
        const unsigned S = persist_slots(P);
        o("#define QCS_SYNC() group_sync(grp)\n");
        o("extern \"C\" __global__ void __launch_bounds__(%u, 1)\n", kPersistThreads);
        o("qcs_pass(double2* __restrict__ a, const __grid_constant__ PassParams P, const TileOp* __restrict__ big,\n");
        o("         const u64* __restrict__ flipped, const u64* __restrict__ tables, const __grid_constant__ TmapParam tmap) {\n");
        o("  extern __shared__ __align__(1024) unsigned char smem_raw[];\n");
        o("  PersistCtx c;\n");
        o("  persist_begin<%uu>(a, P, tables, tmap, smem_raw, c);\n", S);
        o("  const u64* const hi_tab = c.hi_tab;\n");
        o("  const unsigned grp = threadIdx.x >> 8, t = threadIdx.x & 255u;\n");
        o("  const unsigned sign_hit = 0;\n  (void)sign_hit; (void)hi_tab; (void)big; (void)flipped; (void)a;\n");
        o("  unsigned slot = grp, use = 0;\n");
        o("#pragma unroll 1\n");
        o("  for (u64 tile = blockIdx.x + u64(grp) * gridDim.x; tile < c.ntiles; tile += 2ull * gridDim.x) {\n");
        o("  double2* const sm = c.sm0 + (slot << %d);\n", P.m);
        o("  const u64 base = tile_base_of(P, tile);\n");
        o("  mbar_wait(c.full + 2u * slot + (use & 1u), (use >> 1) & 1u);\n");
        const bool direct = emit_rounds(o, P, 0, P.nrounds, 256, true);
        o("  persist_end<%uu, %s>(a, P, tmap, c, grp, t, tile, base, sm, c.full + 2u * slot + ((use + 1u) & 1u));\n", S,
          direct ? "true" : "false");
        o("  slot += 2u;\n  if (slot >= %uu) { slot -= %uu; ++use; }\n", S, S);
        o("  }\n");
        o("  persist_finish();\n");
        o("}\n");
        return o.s;
    }
    o("#define QCS_SYNC() __syncthreads()\n");
    o("extern \"C\" __global__ void __launch_bounds__(%u, %d)\n", threads, minb);
    o("qcs_pass(double2* __restrict__ a, const __grid_constant__ PassParams P, const TileOp* __restrict__ big,\n");
    o("         const u64* __restrict__ flipped, const u64* __restrict__ tables, const __grid_constant__ TmapParam tmap) {\n");
    o("  extern __shared__ __align__(1024) unsigned char smem_raw[];\n");
    o("  TileCtx c;\n");
    o("  if (!tile_begin<%uu>(a, P, big, flipped, tables, tmap, smem_raw, c)) return;\n", F);
    o("  double2* const sm = c.sm;\n  const u64* const hi_tab = c.hi_tab;\n  const u64 base = c.base;\n");
    o("  const unsigned sign_hit = c.sign_hit;\n  const unsigned t = threadIdx.x;\n");
    o("  (void)sign_hit; (void)hi_tab;\n");
    if (P.alt_mode == ALT_ROUNDS) {
        o("  if (c.rb == 0 && c.re == %d) {\n", P.nrounds);
        emit_rounds(o, P, 0, P.nrounds, threads);
        o("  } else {\n");
        emit_rounds(o, P, P.alt_begin, P.alt_begin + P.alt_nrounds, threads);
        o("  }\n");
    } else {
        emit_rounds(o, P, 0, P.nrounds, threads);
    }
    o("}\n");
    return o.s;
}
std::string pass_source(const PassParams& P, unsigned F, unsigned threads) {
    return pass_source(P, F, threads, persist_wanted(P, F));
}

// FP64 instructions per tile of the pass's main program as its specialised kernel runs it
// (per thread, summed over the tile's 2^m / 8 groups)
double fp64_per_tile(const PassParams& P) {
    PassParams Q = P;
    if (Q.alt_mode == ALT_ROUNDS) Q.alt_mode = ALT_NONE;  // the main program only
    g_fp64 = 0.0;
    (void)pass_source(Q, 0xffu, 256);
    const double per_tile = g_fp64;  // each round's per-group counts times its groups per tile
    g_fp64 = 0.0;
    return per_tile;
}

void nvrtc_check(nvrtcResult r, const char* what) {
    if (r != NVRTC_SUCCESS) raise(QCS_ERR_SIM, std::string(what) + ": " + nvrtcGetErrorString(r));
}

struct JitKernel {
    cudaLibrary_t lib = nullptr;
    cudaKernel_t kernel = nullptr;
    bool persist = false;        // the persistent pipelined form: one CTA of 512 threads per SM
    std::size_t persist_smem = 0;
    std::set<int> attr_devices;  // devices whose dynamic shared-memory limit is raised
    std::map<int, CUfunction> fn;  // per device: the kernel's function in that device's context
};

// Driver entry points for launching the library kernels as CUfunctions (cuLaunchKernel).
struct Driver {
    CUresult (*kernel_get_function)(CUfunction*, CUkernel) = nullptr;
    CUresult (*func_set_attribute)(CUfunction, CUfunction_attribute, int) = nullptr;
    CUresult (*launch)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, CUstream,
                       void**, void**) = nullptr;
    bool ok = false;
};
const Driver& driver() {
    static const Driver d = [] {
        Driver r;
        auto get = [](const char* name, void** fn) {
            cudaDriverEntryPointQueryResult q{};
            if (cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess) {
                cudaGetLastError();
                *fn = nullptr;
            }
        };
        get("cuKernelGetFunction", reinterpret_cast<void**>(&r.kernel_get_function));
        get("cuFuncSetAttribute", reinterpret_cast<void**>(&r.func_set_attribute));
        get("cuLaunchKernel", reinterpret_cast<void**>(&r.launch));
        const char* v = std::getenv("QCS_JIT_LAUNCH");  // "rt": cudaLaunchKernel on the cudaKernel_t
        r.ok = r.kernel_get_function && r.func_set_attribute && r.launch && !(v && !std::strcmp(v, "rt"));
        return r;
    }();
    return d;
}
void cu_check(CUresult r, const char* what) {
    if (r != CUDA_SUCCESS) raise(QCS_ERR_CUDA, std::string(what) + " failed (CUresult " + std::to_string(int(r)) + ")");
}

std::mutex g_mu;
std::map<std::string, std::unique_ptr<JitKernel>> g_cache;
std::atomic<unsigned long long> g_compiles{0};

std::vector<char> nvrtc_cubin(const std::string& src);

// Optional on-disk cache of compiled pass kernels (QCS_JIT_CACHE=<directory>): a kernel's cubin
// is stored with its full source (the key is the complete text: headers, options, generated
// code), so a later process reuses it instead of compiling.  Off by default.
std::string full_key(const std::string& src) {
    int major = 0, minor = 0;
    nvrtcVersion(&major, &minor);
    return std::string(kJitSrcKernels) + kJitSrcDevice + "\n// nvrtc " + std::to_string(major) + "." +
           std::to_string(minor) + " sm_100a\n" + src;
}

std::vector<char> compile_cubin(const std::string& src) {
    static const char* dir = std::getenv("QCS_JIT_CACHE");
    if (!dir || !*dir) return nvrtc_cubin(src);
    const std::string key = full_key(src);
    std::uint64_t h = 1469598103934665603ull;  // FNV-1a
    for (unsigned char ch : key) h = (h ^ ch) * 1099511628211ull;
    char name[32];
    std::snprintf(name, sizeof(name), "%016llx", (unsigned long long)h);
    // one file per kernel: [u64 key bytes][key][u64 cubin bytes][u64 FNV-1a of the cubin][cubin],
    // written to a mkstemp() file in the same directory and renamed into place, so concurrent
    // processes (torchrun ranks sharing the directory) never see a torn or mismatched entry
    const std::string path = std::string(dir) + "/qcs_" + name + ".kc";
    auto fnv = [](const char* p, std::size_t n) {
        std::uint64_t x = 1469598103934665603ull;
        for (std::size_t i = 0; i < n; ++i) x = (x ^ static_cast<unsigned char>(p[i])) * 1099511628211ull;
        return x;
    };
    {
        std::FILE* f = std::fopen(path.c_str(), "rb");
        if (f) {
            std::string body;
            char buf[65536];
            std::size_t k;
            while ((k = std::fread(buf, 1, sizeof(buf), f)) > 0) body.append(buf, k);
            std::fclose(f);
            std::uint64_t kl = 0, cl = 0, ch = 0;
            if (body.size() >= 8) std::memcpy(&kl, body.data(), 8);
            if (body.size() >= 8 + kl + 16) {
                std::memcpy(&cl, body.data() + 8 + kl, 8);
                std::memcpy(&ch, body.data() + 16 + kl, 8);
                const char* cub = body.data() + 24 + kl;
                if (body.size() == 24 + kl + cl && cl > 0 && body.compare(8, kl, key) == 0 && fnv(cub, cl) == ch)
                    return std::vector<char>(cub, cub + cl);
            }
        }
    }
    std::vector<char> cubin = nvrtc_cubin(src);
    std::string tmpl = std::string(dir) + "/qcs_" + name + ".XXXXXX";
    const int fd = mkstemp(tmpl.data());
    if (fd < 0) return cubin;  // read-only cache directory: compile only
    std::FILE* f = fdopen(fd, "wb");
    if (!f) {
        close(fd);
        std::remove(tmpl.c_str());
        return cubin;
    }
    const std::uint64_t kl = key.size(), cl = cubin.size(), ch = fnv(cubin.data(), cubin.size());
    bool ok = std::fwrite(&kl, 8, 1, f) == 1 && std::fwrite(key.data(), 1, kl, f) == kl &&
              std::fwrite(&cl, 8, 1, f) == 1 && std::fwrite(&ch, 8, 1, f) == 1 &&
              std::fwrite(cubin.data(), 1, cl, f) == cl;
    ok = (std::fclose(f) == 0) && ok;
    if (ok) std::rename(tmpl.c_str(), path.c_str());
    else std::remove(tmpl.c_str());
    return cubin;
}

std::vector<char> nvrtc_cubin(const std::string& src) {
    if (std::getenv("QCS_JIT_DUMP")) std::fprintf(stderr, "---- qcs_pass\n%s", src.c_str());
    nvrtcProgram prog;
    const char* headers[] = {kJitSrcKernels, kJitSrcDevice};
    const char* names[] = {"kernels.hpp", "tile_device.cuh"};
    nvrtc_check(nvrtcCreateProgram(&prog, src.c_str(), "qcs_pass.cu", 2, headers, names), "nvrtcCreateProgram");
    static const bool verbose = std::getenv("QCS_JIT_VERBOSE") != nullptr;  // ptxas register / spill report
    const char* opts[] = {"-arch=sm_100a", "-std=c++17", "--fmad=false", "-lineinfo", "-default-device",
                          "--ptxas-options=-v"};
    const nvrtcResult rc = nvrtcCompileProgram(prog, verbose ? 6 : 5, opts);
    if (verbose && rc == NVRTC_SUCCESS) {
        std::size_t n = 0;
        nvrtcGetProgramLogSize(prog, &n);
        std::string log(n, '\0');
        nvrtcGetProgramLog(prog, log.data());
        std::fprintf(stderr, "%s", log.c_str());
    }
    if (rc != NVRTC_SUCCESS) {
        std::size_t n = 0;
        nvrtcGetProgramLogSize(prog, &n);
        std::string log(n, '\0');
        nvrtcGetProgramLog(prog, log.data());
        nvrtcDestroyProgram(&prog);
        raise(QCS_ERR_SIM, "pass kernel compilation failed: " + log.substr(0, 2000));
    }
    std::size_t n = 0;
    nvrtc_check(nvrtcGetCUBINSize(prog, &n), "nvrtcGetCUBINSize");
    std::vector<char> cubin(n);
    nvrtc_check(nvrtcGetCUBIN(prog, cubin.data()), "nvrtcGetCUBIN");
    nvrtcDestroyProgram(&prog);
    return cubin;
}

JitKernel& load(const std::string& src, const std::vector<char>& cubin) {
    // callers hold g_mu
    const std::size_t n = cubin.size();
    auto k = std::make_unique<JitKernel>();
    QCS_CUDA(cudaLibraryLoadData(&k->lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0));
    QCS_CUDA(cudaLibraryGetKernel(&k->kernel, k->lib, "qcs_pass"));
    ++g_compiles;
    k->persist = src.find("persist_begin<") != std::string::npos;
    auto& ref = *k;
    g_cache.emplace(src, std::move(k));
    return ref;
}

JitKernel& compile(const std::string& src) {
    // callers hold g_mu
    auto it = g_cache.find(src);
    if (it != g_cache.end()) return *it->second;
    return load(src, compile_cubin(src));
}


// worth a compile (~0.5 s, once per structure): enough tiles x rounds of work
bool has_w4(const PassParams& p) {
    for (int r = 0; r < p.nrounds; ++r)
        if (p.rounds[r].flags & RD_W4) return true;
    return false;
}

bool wanted(const PassParams& p, double tiles) {
    if (has_w4(p)) return true;  // 16-register rounds exist only in the specialised form
    const int mode = jit_mode();
    if (mode == 0) return false;
    return mode >= 2 || has_pivot(p) || (tiles * double(p.nrounds) >= 32768.0 && p.nrounds >= 2);
}

}  // namespace

namespace {
std::atomic<int> g_mode{[] {
    const char* v = std::getenv("QCS_JIT");
    if (!v || !*v) return 1;                 // default: passes with enough work
    if (!std::strcmp(v, "force")) return 2;  // every tile pass
    if (!std::strcmp(v, "pivot")) return 3;  // every tile pass, pivoted gates
    return std::atoi(v) != 0 ? 1 : 0;
}()};
}  // namespace

int pipeline_mode() { return persist_knob(); }
void set_pipeline_mode(int mode) {
    if (mode < 0 || mode > 2) raise(QCS_ERR_ARG, "pipeline mode must be 0, 1 or 2");
    g_persist.store(mode);
}
int jit_mode() { return g_mode.load(std::memory_order_relaxed); }
void set_jit_mode(int mode) {
    if (mode < 0 || mode > 3) raise(QCS_ERR_ARG, "jit mode must be 0, 1, 2 or 3");
    g_mode.store(mode);
}

bool jit_virtual(int n, int m, bool skip_pass) {
    static const bool perms = [] { const char* v = std::getenv("QCS_JIT_PERMS"); return !v || std::atoi(v) != 0; }();
    const int mode = jit_mode();
    if (m < 3 || !perms) return false;
    if (mode == 3) return true;
    return mode == 1 && !skip_pass && n - m >= 11;  // big passes (>= 2048 tiles): specialised anyway
}

bool jit_pivot(int n, const PassParams& p) {
    static const bool pivots = [] { const char* v = std::getenv("QCS_JIT_PIVOT"); return !v || std::atoi(v) != 0; }();
    const int mode = jit_mode();
    if (mode == 3) return true;
    if (mode != 1 || !pivots) return false;
    const double tiles = p.list_cnt ? double(p.list_cnt) : std::ldexp(1.0, n - p.m);
    return wanted(p, tiles);
}

unsigned long long jit_compiles() { return g_compiles.load(); }

void jit_prepare(int n, const std::vector<PassParams>& passes, const std::vector<std::vector<int>>& pass_ops) {
    std::vector<std::string> todo;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        std::set<std::string> seen;
        for (std::size_t i = 0; i < passes.size(); ++i) {
            const PassParams& p = passes[i];
            if (pass_ops[i].size() < 2 || p.m < 3 || p.m > n) continue;
            const double tiles = p.list_cnt ? double(p.list_cnt) : std::ldexp(1.0, n - p.m);
            if (!wanted(p, tiles)) continue;
            unsigned F = 0, threads = 0;
            tile_pass_shape(p, F, threads);
            std::string src = pass_source(p, F, threads);
            if (g_cache.count(src) || !seen.insert(src).second) continue;
            todo.push_back(std::move(src));
        }
    }
    if (todo.size() < 2) return;  // a single kernel compiles at its launch
    // NVRTC programs compile concurrently; modules load afterwards under the cache lock
    std::vector<std::vector<char>> cubins(todo.size());
    std::vector<std::string> errors(todo.size());
    std::atomic<std::size_t> next{0};
    auto worker = [&] {
        for (std::size_t i; (i = next.fetch_add(1)) < todo.size();) {
            try {
                cubins[i] = compile_cubin(todo[i]);
            } catch (const std::exception& e) {
                errors[i] = e.what();
            }
        }
    };
    static const unsigned threads_env = [] { const char* v = std::getenv("QCS_JIT_THREADS"); return v ? unsigned(std::atoi(v)) : 0u; }();
    const unsigned hw = threads_env ? threads_env : std::max(1u, std::thread::hardware_concurrency());
    const std::size_t nthreads = std::min<std::size_t>(todo.size(), std::min(hw, 32u));
    std::vector<std::thread> pool;
    for (std::size_t i = 1; i < nthreads; ++i) pool.emplace_back(worker);
    worker();
    for (auto& th : pool) th.join();
    for (const auto& e : errors)
        if (!e.empty()) raise(QCS_ERR_SIM, e);
    std::lock_guard<std::mutex> lk(g_mu);
    for (std::size_t i = 0; i < todo.size(); ++i)
        if (!g_cache.count(todo[i])) load(todo[i], cubins[i]);
}

std::size_t jit_compile_only(const PassParams& p, bool verify_only) {
    unsigned F = 0, threads = 0;
    tile_pass_shape(p, F, threads);
    if (verify_only) {  // generate with the addressing proof on, no NVRTC
        g_verify = true;
        try {
            const std::string src = pass_source(p, F, threads);
            if (std::getenv("QCS_JIT_DUMP")) std::fprintf(stderr, "---- qcs_pass (verify)\n%s", src.c_str());
        } catch (...) {
            g_verify = false;
            throw;
        }
        g_verify = false;
        return 0;
    }
    return compile_cubin(pass_source(p, F, threads)).size();
}

double pass_fp64_per_tile(const PassParams& p) { return fp64_per_tile(p); }

bool launch_tile_pass_jit(double2* amps, const PassParams& p, unsigned F, const TileOp* big_dev,
                          const std::uint64_t* flipped_dev, const std::uint64_t* tables_dev, const TmapParam& tmap,
                          unsigned tiles, unsigned threads, std::size_t smem, std::size_t smem_max, cudaStream_t st,
                          void** jit_slot) {
    if (!(jit_slot && *jit_slot) && !wanted(p, double(tiles))) return false;
    int dev = 0;
    QCS_CUDA(cudaGetDevice(&dev));
    cudaKernel_t kern;
    CUfunction fn = nullptr;
    const Driver& drv = driver();
    {
        std::lock_guard<std::mutex> lk(g_mu);
        // a plan the caller keeps remembers its kernel (no source generation on reuse)
        JitKernel& k = jit_slot && *jit_slot
                           ? *static_cast<JitKernel*>(*jit_slot)
                           : compile(pass_source(p, F, threads, persist_wanted(p, F)));
        if (jit_slot) *jit_slot = &k;
        if (k.persist) {  // one CTA per SM, the ring of tile slots in its shared memory
            static int sms[64] = {};
            if (dev < 64 && !sms[dev]) QCS_CUDA(cudaDeviceGetAttribute(&sms[dev], cudaDevAttrMultiProcessorCount, dev));
            const unsigned nsm = unsigned(dev < 64 && sms[dev] > 0 ? sms[dev] : 148);
            tiles = std::min(tiles, nsm);
            threads = kPersistThreads;
            smem = 1024 + std::size_t(persist_slots(p)) * (std::size_t(16) << p.m) + (std::size_t(8) << (p.m - 3)) + 128;
            smem_max = std::max(smem_max, smem);
        }
        if (drv.ok) {
            auto it = k.fn.find(dev);
            if (it == k.fn.end()) {
                cu_check(drv.kernel_get_function(&fn, reinterpret_cast<CUkernel>(k.kernel)), "cuKernelGetFunction");
                cu_check(drv.func_set_attribute(fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, int(smem_max)),
                         "cuFuncSetAttribute");
                cu_check(drv.func_set_attribute(fn, CU_FUNC_ATTRIBUTE_PREFERRED_SHARED_MEMORY_CARVEOUT, 100),
                         "cuFuncSetAttribute");
                it = k.fn.emplace(dev, fn).first;
            }
            fn = it->second;
        } else if (!k.attr_devices.count(dev)) {
            QCS_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(k.kernel),
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_max)));
            QCS_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(k.kernel),
                                          cudaFuncAttributePreferredSharedMemoryCarveout, 100));
            k.attr_devices.insert(dev);
        }
        kern = k.kernel;
    }
    void* a = amps;
    const void* b = big_dev;
    const void* f = flipped_dev;
    const void* tb = tables_dev;
    void* args[] = {&a, const_cast<PassParams*>(&p), &b, &f, &tb, const_cast<TmapParam*>(&tmap)};
    if (fn) cu_check(drv.launch(fn, tiles, 1, 1, threads, 1, 1, unsigned(smem), st, args, nullptr), "cuLaunchKernel");
    else QCS_CUDA(cudaLaunchKernel(reinterpret_cast<const void*>(kern), dim3(tiles), dim3(threads), args, smem, st));
    return true;
}

}  // namespace qcs
