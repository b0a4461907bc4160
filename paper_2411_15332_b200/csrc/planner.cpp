// planner.cpp -- fusion planner: circuit operations -> HBM passes -> register rounds.
//
// The reference applies every step as its own full operator-vector product (engine.cpp:162-205).
// On the GPU the cost of a step is one HBM round trip of the state, so consecutive operations
// are grouped into passes whose target bits fit one shared-memory tile (tile_kernels.cu).
// Operations may move earlier past unscheduled ones only when they commute: disjoint bit
// supports, or both diagonal.  A pass keeps basis bits 0..2 in its tile for coalescing.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "engine.hpp"
#include "planner.hpp"

namespace qcs {

namespace {
// planner A/B switches for measurements (host side, read once)
bool knob(const char* name) {
    const char* v = std::getenv(name);
    return v && *v && *v != '0';
}
const bool kNoTables = knob("QCS_NO_DTAB");
// 16-amplitude register rounds (4 register bits) in the specialised kernels: a third fewer rounds
// for C4 (59 -> 39), measured 265.8 -> 260.5 ms (tools/gpu_r02w.sh); QCS_JIT_W4=0 turns them off
bool knob_w4() {
    static const bool on = [] { const char* v = std::getenv("QCS_JIT_W4"); return !v || std::atoi(v) != 0; }();
    return on;
}
const bool kNoReal = knob("QCS_NO_REAL");
inline bool is_zero(const cplx& v) { return v.real() == 0.0 && v.imag() == 0.0; }
inline bool is_one(const cplx& v) { return v.real() == 1.0 && v.imag() == 0.0; }
}  // namespace

// One canonical placement -> one fused operation (nullopt-like: returns false for identity).
bool make_fop(const GateOp& op, FOp& f) {
    const int k = op.k, dim = 1 << k;
    f = FOp{};
    f.src = op;
    bool any = false, diag = true;
    for (int g = 0; g < dim; ++g)
        for (int c = 0; c < dim; ++c) {
            const cplx v = op.m[std::size_t(g) * dim + c];
            if (is_zero(v)) continue;
            if (c != g) diag = false;
            if (!(c == g && is_one(v))) any = true;
        }
    if (!any) return false;
    for (int i = 0; i < k; ++i) f.touch |= u64(1) << op.pos[i];
    if (diag) {
        f.kind = TOP_DIAG;
        f.diagonal = true;
        f.dk = k;
        for (int i = 0; i < k; ++i) f.dpos[i] = op.pos[i];
        for (int g = 0; g < dim; ++g) {
            const cplx v = op.m[std::size_t(g) * dim + g];
            f.dval[g] = make_double2(v.real(), v.imag());
            f.dskip[g] = is_one(v);
        }
        return true;
    }
    // peel controls: local bit b is a control (on 1) when every row with b = 0 is an identity
    // row and no row with b = 1 reads a column with b = 0
    std::vector<int> bits;  // remaining local bits (of the canonical k-bit index), ascending
    for (int b = 0; b < k; ++b) bits.push_back(b);
    int cmask = 0;
    for (int b = 0; b < k; ++b) {
        bool ctrl = true;
        for (int g = 0; g < dim && ctrl; ++g) {
            if ((cmask & g) != cmask) continue;  // rows already excluded by earlier controls
            for (int c = 0; c < dim; ++c) {
                const cplx v = op.m[std::size_t(g) * dim + c];
                if (is_zero(v)) continue;
                if (!(g >> b & 1)) {
                    if (!(c == g && is_one(v))) { ctrl = false; break; }
                } else if (!(c >> b & 1)) { ctrl = false; break; }
            }
        }
        if (ctrl && int(bits.size()) > 1) {
            cmask |= 1 << b;
            bits.erase(std::find(bits.begin(), bits.end(), b));
        }
    }
    const int K = int(bits.size());
    // targets, most significant first; local bit b <-> canonical slot k-1-b <-> op.pos[k-1-b]
    f.kind = TOP_GATE;
    f.K = K;
    for (int i = 0; i < K; ++i) f.tpos[i] = op.pos[k - 1 - bits[K - 1 - i]];
    for (int b = 0; b < k; ++b)
        if (cmask >> b & 1) {
            f.ctrl_mask |= u64(1) << op.pos[k - 1 - b];
            f.ctrl_val |= u64(1) << op.pos[k - 1 - b];
        }
    auto full = [&](int mm) {  // K-bit member -> canonical k-bit index with controls set
        int g = cmask;
        for (int i = 0; i < K; ++i)
            if (mm >> (K - 1 - i) & 1) g |= 1 << bits[K - 1 - i];
        return g;
    };
    f.nrows = 0;
    for (int r = 0; r < (1 << K); ++r) {
        const int g = full(r);
        int nz = 0, only = -1;
        for (int c = 0; c < dim; ++c)
            if (!is_zero(op.m[std::size_t(g) * dim + c])) { ++nz; only = c; }
        if (nz == 1 && only == g && is_one(op.m[std::size_t(g) * dim + g])) continue;  // identity row
        const int row = f.nrows++;
        f.row_member[row] = std::uint8_t(r);
        int z = 0;
        for (int mm = 0; mm < (1 << K); ++mm) {  // ascending member == ascending global column
            const cplx v = op.m[std::size_t(g) * dim + full(mm)];
            if (is_zero(v)) continue;
            f.col_member[row][z] = std::uint8_t(mm);
            f.val[row][z] = make_double2(v.real(), v.imag());
            ++z;
        }
        f.nnz[row] = std::uint8_t(z);
    }
    return true;
}

FOp make_sign(int n, std::vector<u64> flips, bool rest) {
    FOp f{};
    f.kind = TOP_SIGN;
    f.diagonal = true;
    f.touch = n >= 64 ? ~u64(0) : (u64(1) << n) - 1;
    std::sort(flips.begin(), flips.end());
    flips.erase(std::unique(flips.begin(), flips.end()), flips.end());
    f.flips = std::move(flips);
    f.flip_rest = rest;
    return f;
}

FOp make_scale(double s) {
    FOp f{};
    f.kind = TOP_SCALE;
    f.diagonal = true;
    f.scale = s;
    return f;
}

FOp make_wht(int bit) {
    FOp f{};
    f.kind = TOP_WHT;
    f.K = 1;
    f.tpos[0] = bit;
    f.touch = u64(1) << bit;
    return f;
}

namespace {

bool elementwise(const FOp& f) { return f.kind == TOP_DIAG || f.kind == TOP_SIGN || f.kind == TOP_SCALE; }

// one uncontrolled single-qubit gate or one-bit diagonal: returns its basis bit, else -1
int single_qubit_bit(const FOp& f) {
    if (f.src.k != 1) return -1;
    if (f.kind == TOP_GATE && f.K == 1 && f.ctrl_mask == 0) return f.tpos[0];
    if (f.kind == TOP_DIAG && f.dk == 1) return f.dpos[0];
    return -1;
}

}  // namespace

// Gate fusion for fused passes: a run of single-qubit operations on the same qubit, with no
// operation touching that qubit in between, becomes one 2x2 -- their product (later * earlier).
// Halves the FP64 work of layers like C4's RY-then-RZ; an identity product disappears.
void merge_single_qubit(int n, std::vector<FOp>& ops) {
    std::vector<int> open(std::size_t(n), -1);  // index in `out` of the chain head on each bit
    std::vector<FOp> out;
    out.reserve(ops.size());
    // a butterfly (RH's H^n, unnormalised [[1, 1], [1, -1]]) joins a one-qubit GATE next to it on
    // its bit (C4/C1: H^n then the RY layer): the product is one 2x2 of the gate's kind (real stays
    // real), and the butterfly no longer needs a register round of its own.  Butterflies do not
    // merge with each other or with diagonals, so the sign-step programs of Grover-like
    // circuits (butterfly pairs around sign steps, C3) keep their structure.
    static const cplx kB[4] = {cplx(1.0, 0.0), cplx(1.0, 0.0), cplx(1.0, 0.0), cplx(-1.0, 0.0)};
    static const bool no_wht_merge = knob("QCS_NO_WHT_MERGE");  // A/B switch
    auto is_wht = [](const FOp& x) { return x.kind == TOP_WHT; };
    auto is_gate1 = [](const FOp& x) { return x.kind == TOP_GATE && x.src.k == 1 && x.K == 1 && x.ctrl_mask == 0; };
    for (FOp& f : ops) {
        int bit = single_qubit_bit(f);
        if (bit < 0 && is_wht(f) && !no_wht_merge) bit = f.tpos[0];
        const int hi = bit >= 0 ? open[std::size_t(bit)] : -1;
        bool merge = hi >= 0;
        if (merge) {
            const FOp& head = out[std::size_t(hi)];
            if (is_wht(f) || is_wht(head)) merge = (is_wht(f) && is_gate1(head)) || (is_wht(head) && is_gate1(f));
        }
        if (merge) {
            FOp& head = out[std::size_t(hi)];
            const cplx* a = is_wht(f) ? kB : f.src.m.data();      // later
            const cplx* b = is_wht(head) ? kB : head.src.m.data();  // earlier
            GateOp g;
            g.k = 1;
            g.pos[0] = bit;
            g.m.resize(4);
            for (int r = 0; r < 2; ++r)
                for (int c = 0; c < 2; ++c)
                    g.m[std::size_t(r * 2 + c)] = a[r * 2] * b[c] + a[r * 2 + 1] * b[2 + c];
            FOp merged;
            if (make_fop(g, merged)) {
                head = std::move(merged);
            } else {  // the product is the identity
                head.kind = -1;
                open[std::size_t(bit)] = -1;
            }
            continue;
        }
        for (int b = 0; b < n; ++b)
            if (f.touch >> b & 1) open[std::size_t(b)] = -1;
        out.push_back(std::move(f));
        if (bit >= 0) open[std::size_t(bit)] = int(out.size()) - 1;
    }
    ops.clear();
    for (FOp& f : out)
        if (f.kind >= 0) ops.push_back(std::move(f));
}

// Phase splitting for fused passes: a one-qubit gate whose rows each carry one common phase is
// D_L * R with R real, one whose columns do is R * D_R.  The real factor costs half the FP64
// instructions of a complex 2x2 and the diagonal joins its round's diagonal table (lower_plan):
// C4's merged RZ * RY, Y = diag(-i, i) * X.  The factors reproduce the gate to ~1e-16; fused
// passes are held to 1e-12.
void split_phases(std::vector<FOp>& ops) {
    if (knob("QCS_NO_SPLIT")) return;
    std::vector<FOp> out;
    out.reserve(ops.size());
    auto one_qubit = [](int bit, const cplx (&m)[4], FOp& f) {
        GateOp g;
        g.k = 1;
        g.pos[0] = bit;
        g.m.assign(m, m + 4);
        return make_fop(g, f);
    };
    for (FOp& f : ops) {
        bool split = false;
        if (f.kind == TOP_GATE && f.src.k == 1 && f.K == 1 && f.ctrl_mask == 0) {
            const cplx* m = f.src.m.data();
            bool real = true;
            for (int i = 0; i < 4; ++i) real &= m[i].imag() == 0.0;
            // factor by rows (by_rows) or columns: entry (r, c) = d[line] * R(r, c), R real
            for (int by_rows = 1; !real && !split && by_rows >= 0; --by_rows) {
                cplx d[2];
                cplx R[4];
                bool ok = true;
                for (int l = 0; l < 2 && ok; ++l) {
                    const int i0 = by_rows ? 2 * l : l, i1 = by_rows ? 2 * l + 1 : l + 2;
                    const cplx big = std::abs(m[i0]) >= std::abs(m[i1]) ? m[i0] : m[i1];
                    if (std::abs(big) == 0.0) { ok = false; break; }
                    d[l] = big / std::abs(big);
                    for (int i : {i0, i1}) {
                        const cplx x = m[i] * std::conj(d[l]);
                        if (std::fabs(x.imag()) > 1e-15) ok = false;
                        R[i] = cplx(x.real(), 0.0);
                    }
                }
                if (!ok) continue;
                const cplx D[4] = {d[0], cplx(0.0, 0.0), cplx(0.0, 0.0), d[1]};
                cplx Rm[4] = {R[0], R[1], R[2], R[3]};
                FOp fr, fd;
                const bool has_r = one_qubit(f.tpos[0], Rm, fr), has_d = one_qubit(f.tpos[0], D, fd);
                if (by_rows) {  // D_L * R: R first
                    if (has_r) out.push_back(std::move(fr));
                    if (has_d) out.push_back(std::move(fd));
                } else {
                    if (has_d) out.push_back(std::move(fd));
                    if (has_r) out.push_back(std::move(fr));
                }
                split = true;
            }
        }
        if (!split) out.push_back(std::move(f));
    }
    ops.swap(out);
}

namespace {
// One greedy plan.  strict_dims: the tile search counts tensor-map dims the round-1 way (a dim per
// gap between tile runs as well) when it prefers tiles that move as one TMA box.
Plan plan_ops_policy(int n, const std::vector<FOp>& ops, int max_bits, bool strict_dims, std::size_t max_starts) {
    Plan plan;
    const int M = std::min(max_bits, n);
    static const bool no_seed = knob("QCS_NO_TILE_SEARCH");  // A/B switch
    std::vector<int> remaining(ops.size());
    for (std::size_t i = 0; i < ops.size(); ++i) remaining[i] = int(i);
    // One pass grown greedily in operation order from the tile bits `seed` (bits 0..2 always):
    // an operation joins when it commutes with everything skipped before it and its targets fit.
    struct Grown {
        u64 S = 0;
        std::vector<int> chosen, skipped;
        std::size_t stop = ~std::size_t(0);  // remaining[stop..] were not scanned (all skipped)
        int gates = 0;
        bool signs = false;
    };
    auto grow = [&](u64 seed) {
        Grown g;
        u64 S = seed;
        for (int b = 0; b < std::min(3, n); ++b) S |= u64(1) << b;
        int used = __builtin_popcountll(S);
        u64 nd_block = 0, d_block = 0;  // supports of skipped non-diagonal / diagonal ops
        // once a sign step is in the pass, later non-elementwise ops must target bits the pass
        // used before it: then on the tiles the sign step misses, the pass mirrors around it
        // and collapses (missed_tile_program), e.g. Grover's H..H Z0 H..H
        bool signed_pass = false;
        u64 pre_sign = 0;
        const u64 full = n >= 64 ? ~u64(0) : (u64(1) << n) - 1;
        for (std::size_t pos = 0; pos < remaining.size(); ++pos) {
            const int idx = remaining[pos];
            if ((nd_block & full) == full) {  // every bit waits on a skipped gate: nothing else can join
                g.stop = pos;  // the rest stays skipped (appended for the winner only)
                break;
            }
            const FOp& f = ops[std::size_t(idx)];
            const bool conflict = (f.touch & nd_block) || (!f.diagonal && (f.touch & d_block));
            bool take = false;
            if (!conflict) {
                if (elementwise(f)) {
                    take = true;
                } else {
                    u64 need = 0;
                    for (int i = 0; i < f.K; ++i) need |= u64(1) << f.tpos[i];
                    const u64 targets = need;
                    if (signed_pass && (need & ~pre_sign)) need = ~u64(0);  // not mirrored: later
                    need &= ~S;
                    const int add = __builtin_popcountll(need);
                    if (used + add <= M) {
                        S |= need;
                        used += add;
                        take = true;
                        if (!signed_pass) pre_sign |= targets;
                    }
                }
            }
            if (take && int(g.chosen.size()) >= kPassMaxOps - 4) take = false;
            if (take) {
                if (f.kind == TOP_SIGN) signed_pass = true;
                g.signs |= f.kind == TOP_SIGN;
                if (!elementwise(f)) ++g.gates;
                g.chosen.push_back(idx);
            } else {
                g.skipped.push_back(idx);
                (f.diagonal ? d_block : nd_block) |= f.touch;
            }
        }
        // pad the tile to M bits with the lowest unused positions (bigger tiles, same cost)
        for (int b = 0; b < n && used < M; ++b)
            if (!(S >> b & 1)) {
                S |= u64(1) << b;
                ++used;
            }
        g.S = S;
        return g;
    };
    // dims of the tile's TMA tensor map (tile_tensor_map): bits 0..2, then every run of tile bits
    // (split at 8 bits) and every run of other bits; > 5 falls back to per-thread cp.async tiles,
    // which cost the pass ~15% more instructions (address arithmetic per 16 bytes)
    auto tma_dims = [&](u64 S) { return tma_layout(S, n, nullptr, strict_dims || tma_gap_dims()); };
    static const double tma_weight = [] {
        const char* v = std::getenv("QCS_TILE_TMA_WEIGHT");
        return v ? std::atof(v) : 0.85;
    }();
    auto score = [&](const Grown& g) { return double(g.gates) * (tma_dims(g.S) > 5 ? tma_weight : 1.0); };
    while (!remaining.empty()) {
        Grown best = grow(0);
        // Tile search: the circuit-order tile fills with the first new bits it meets, which for a
        // layered circuit is a run of qubits whose light cone the neighbouring runs cut short.
        // Seeding the tile with the targets of a later ready gate instead (up to 48 candidates)
        // and keeping the pass with the most gates finds tiles whose light cones reach further
        // (fewer passes).  Passes with sign steps keep the circuit-order tile (their skip and
        // mirror programs depend on it).
        if (!no_seed && !best.signs && M >= 6) {
            // seed j: the first new target bits met from the j-th remaining gate on (as many as
            // the tile takes), i.e. the tile a pass starting at that gate would fill
            std::vector<u64> seeds;
            u64 low = 0;
            for (int b = 0; b < std::min(3, n); ++b) low |= u64(1) << b;
            std::vector<std::size_t> starts;
            for (std::size_t p = 0; p < remaining.size() && starts.size() < max_starts; ++p)
                if (!elementwise(ops[std::size_t(remaining[p])])) starts.push_back(p);
            for (std::size_t st : starts) {
                u64 seed = low;
                for (std::size_t p = st; p < remaining.size(); ++p) {
                    const FOp& f = ops[std::size_t(remaining[p])];
                    if (elementwise(f)) continue;
                    u64 t = 0;
                    for (int i = 0; i < f.K; ++i) t |= u64(1) << f.tpos[i];
                    if (__builtin_popcountll(seed | t) > M) break;
                    seed |= t;
                }
                if (std::find(seeds.begin(), seeds.end(), seed) == seeds.end()) seeds.push_back(seed);
                // and the gate's own targets alone (the rest filled in circuit order)
                const FOp& f = ops[std::size_t(remaining[st])];
                u64 t = low;
                for (int i = 0; i < f.K; ++i) t |= u64(1) << f.tpos[i];
                if (std::find(seeds.begin(), seeds.end(), t) == seeds.end()) seeds.push_back(t);
            }
            double best_score = score(best);
            for (u64 seed : seeds) {
                Grown g = grow(seed);
                const double sc = score(g);
                if (!g.signs && sc > best_score) {
                    best_score = sc;
                    best = std::move(g);
                }
            }
        }
        plan.passes.push_back(PlannedPass{best.S, best.chosen});
        if (best.stop < remaining.size())
            best.skipped.insert(best.skipped.end(), remaining.begin() + std::ptrdiff_t(best.stop), remaining.end());
        remaining.swap(best.skipped);
    }
    return plan;
}
}  // namespace

// The tile search is greedy (most gates per pass), so which tiles count as one TMA box steers
// where the passes of a layered circuit cut it, and one more pass is one more sweep of the state.
// Plan under both dim counts -- the layout the kernels use, and the stricter round-1 count --
// and keep the plan with fewer passes (ties: fewer tiles that need more than 5 dims, then the
// kernels' own count).  C4 n=32: 9 passes under the kernels' count alone, 8 under the strict one.
Plan plan_ops(int n, const std::vector<FOp>& ops, int max_bits) {
    static const bool one_policy = knob("QCS_PLAN_ONE_POLICY") || knob("QCS_NO_TILE_SEARCH");  // A/B switch
    static const std::size_t seeds = [] { const char* v = std::getenv("QCS_TILE_SEEDS"); return std::size_t(v ? std::atoi(v) : 48); }();
    static const std::size_t deep_seeds = [] { const char* v = std::getenv("QCS_TILE_DEEP_SEEDS"); return std::size_t(v ? std::atoi(v) : 400); }();
    Plan best = plan_ops_policy(n, ops, max_bits, false, seeds);
    if (one_policy || tma_gap_dims() || best.passes.size() < 3) return best;
    auto non_tma = [&](const Plan& p) {
        int c = 0;
        for (const auto& q : p.passes) c += tma_layout(q.tile, n, nullptr, false) > 5;
        return c;
    };
    auto consider = [&](Plan&& b) {
        if (b.passes.size() < best.passes.size() ||
            (b.passes.size() == best.passes.size() && non_tma(b) < non_tma(best)))
            best = std::move(b);
    };
    consider(plan_ops_policy(n, ops, max_bits, true, seeds));
    // Plans of many passes over big states (the C5 family: scattered CNOT pairs) also try a wider
    // seed window: a pass saved is ~30 ms at n=32, the wider search ~15 ms of planning (C5 family
    // n=32: 25 -> 23 passes; C4's 8-pass plans are left alone -- the wider window finds 9).
    if (n >= 26 && best.passes.size() >= 12 && deep_seeds > seeds) {
        consider(plan_ops_policy(n, ops, max_bits, false, deep_seeds));
        consider(plan_ops_policy(n, ops, max_bits, true, deep_seeds));
    }
    return best;
}

// The program a pass runs on tiles that none of its sign steps' listed indices fall in: each
// sign step is then the scalar -1 (flip_rest) or +1, scalars commute with everything, and a
// butterfly pair on one bit with nothing between them touching that bit is 2 I.  Returns false
// when the pass has no sign step; alt = the remaining operations (a leading scale if the
// scalar is not 1), empty when the pass is the identity on those tiles.  Exact: the scalars are
// +-1, the H^n scales 2^(-n/2) and the factors 2.
// Reduce an operation list with every sign step taken as its missed-tile scalar (-1 when
// flip_rest, else +1): scales and sign scalars multiply into s, and a butterfly pair on one bit
// with nothing between them touching that bit is 2 I.  keep = what remains, in order.
void reduce_scalar(const std::vector<FOp>& ops, const std::vector<int>& list, double& s, std::vector<int>& keep) {
    s = 1.0;
    keep.clear();
    for (int idx : list) {
        const FOp& f = ops[std::size_t(idx)];
        if (f.kind == TOP_SIGN) {
            if (f.flip_rest) s = -s;
            continue;
        }
        if (f.kind == TOP_SCALE) {
            s *= f.scale;
            continue;
        }
        if (f.kind == TOP_WHT) {
            const u64 bit = u64(1) << f.tpos[0];
            int j = int(keep.size()) - 1;
            while (j >= 0 && !(ops[std::size_t(keep[std::size_t(j)])].touch & bit)) --j;
            if (j >= 0 && ops[std::size_t(keep[std::size_t(j)])].kind == TOP_WHT &&
                ops[std::size_t(keep[std::size_t(j)])].tpos[0] == f.tpos[0]) {
                keep.erase(keep.begin() + j);
                s *= 2.0;
                continue;
            }
        }
        keep.push_back(idx);
    }
}

bool missed_tile_program(const std::vector<FOp>& ops, const std::vector<int>& list, std::vector<FOp>& alt) {
    bool any_sign = false;
    for (int idx : list) any_sign |= ops[std::size_t(idx)].kind == TOP_SIGN;
    if (!any_sign) return false;
    double s = 1.0;
    std::vector<int> keep;
    reduce_scalar(ops, list, s, keep);
    alt.clear();
    if (s != 1.0) alt.push_back(make_scale(s));
    for (int idx : keep) alt.push_back(ops[std::size_t(idx)]);
    return true;
}

// Lower planned passes to kernel descriptors: one PassParams (constant-bank operation list) per
// pass, plus the plan-wide TileOp array (shared-memory gates, sign steps, 3-bit diagonals).
namespace {

// Pivoted gates for the specialised kernels: a 2x2 row (a, b) with pivot a (its diagonal entry
// unless that one is zero or tiny) is
// a * (x_piv + (b / a) x_other) -- one fused multiply-add per component for a real ratio, two for
// a complex one, instead of two / four -- and the row scale a commutes to the end of the round
// when no later operation of the round targets the gate's bit, where it joins the round's
// diagonal table (created if the round has none).  Gates qualify without controls outside the
// registers; controls on register bits select which table entries take the scale.
void pivot_pass(PassParams& P, int& npool) {
    static const bool no_chain = knob("QCS_NO_SCALE_CHAIN");  // A/B switch
    const int nr = P.alt_mode == ALT_ROUNDS ? P.alt_begin + P.alt_nrounds : P.nrounds;
    std::vector<RegOp> ops;
    std::vector<RoundDesc> rounds(P.rounds, P.rounds + nr);
    for (int ri = 0; ri < nr; ++ri) {
        RoundDesc& R = rounds[std::size_t(ri)];
        const int b0 = R.op_begin, b1 = R.op_begin + R.op_count;
        R.op_begin = std::uint16_t(ops.size());
        std::vector<RegOp> rops(P.ops + b0, P.ops + b1);
        if (R.flags & RD_SMEM) {
            ops.insert(ops.end(), rops.begin(), rops.end());
            continue;
        }
        std::vector<RegOp> trailing;  // relabellings of the last round's stores stay last
        while (!rops.empty() && (rops.back().kind & KF_KIND) == TOP_PERM) {
            trailing.insert(trailing.begin(), rops.back());
            rops.pop_back();
        }
        const int W = round_width(R), G = 1 << W;
        unsigned regmask = 0;
        for (int i = 0; i < W; ++i) regmask |= 1u << round_reg(R, i);
        // the round's table: the existing one (the last operation) or a new one
        int tab = -1;
        if (!rops.empty() && (rops.back().kind & KF_KIND) == TOP_DTAB) tab = int(rops.size()) - 1;
        cplx table[16];
        for (int q = 0; q < G; ++q)
            table[q] = tab >= 0 ? cplx(P.pool[rops[std::size_t(tab)].ref + q].x, P.pool[rops[std::size_t(tab)].ref + q].y)
                                : cplx(1.0, 0.0);
        const bool room = tab >= 0 || (npool + G <= kPassPool && int(ops.size() + rops.size()) + 1 < kPassMaxOps);
        bool changed = false;
        for (std::size_t i = 0; i < rops.size() && room; ++i) {
            RegOp& o = rops[i];
            if ((o.kind & KF_KIND) != TOP_GATE || (o.kind & KF_GCTRL) || (o.lctrl_mask & ~regmask)) continue;

            const bool bundle = o.kind & KF_BUNDLE;
            const unsigned bits = bundle ? o.t : 1u << o.t;
            // the deferred scale is a diagonal on the target and the (register) control bits.  Per
            // target bit: no later operation of the round targets it -> the round's table; the
            // next one that does is an uncontrolled gate with only commuting operations between
            // (diagonals, controls) -> the scale folds into that gate's columns (scale chaining:
            // two layers of one qubit in one round, the round scheduler's light cones); else no pivot
            unsigned support = 0;
            for (int k = 0; k < W; ++k)
                if (o.lctrl_mask >> round_reg(R, k) & 1) support |= 1u << k;
            bool later = false;
            int chain[4] = {-1, -1, -1, -1};
            for (int b = 0; b < W && !later; ++b) {
                if (!(bits >> b & 1)) continue;
                for (std::size_t j = i + 1; j < rops.size(); ++j) {
                    const RegOp& g = rops[j];
                    const int k = g.kind & KF_KIND;
                    const unsigned tj = k == TOP_WHT || (g.kind & KF_BUNDLE) ? g.t : k == TOP_GATE ? 1u << g.t : 0u;
                    if (!((k == TOP_GATE || k == TOP_WHT) && (tj >> b & 1))) continue;
                    if (k == TOP_GATE && !g.lctrl_mask && !(g.kind & KF_GCTRL) && !(g.kind & KF_PIVOT) && !o.lctrl_mask &&
                        !no_chain)
                        chain[b] = int(j);
                    else
                        later = true;
                    break;
                }
            }
            for (std::size_t j = i + 1; j < rops.size() && !later; ++j) {  // register-bit controls
                const int k = rops[j].kind & KF_KIND;
                const unsigned tj = k == TOP_WHT || (rops[j].kind & KF_BUNDLE) ? rops[j].t
                                    : k == TOP_GATE ? 1u << rops[j].t : 0u;
                if ((k == TOP_GATE || k == TOP_WHT) && (tj & support)) later = true;
            }
            if (later) continue;
            // registers the gate acts on (register-bit controls)
            unsigned en = 0;
            for (int q = 0; q < G; ++q) {
                unsigned lq = 0;
                for (int k = 0; k < W; ++k)
                    if (q >> k & 1) lq |= 1u << round_reg(R, k);
                if ((lq & o.lctrl_mask) == o.lctrl_val) en |= 1u << q;
            }
            // every target bit must pivot (a zero row cannot)
            double2* cs[4] = {nullptr, nullptr, nullptr, nullptr};
            bool ok = true;
            for (int b = 0; b < W; ++b)
                if (bits >> b & 1) {
                    cs[b] = bundle ? P.pool + o.ref + 4 * b : o.c;
                    for (int r = 0; r < 2; ++r) ok &= std::abs(cplx(cs[b][2 * r].x, cs[b][2 * r].y)) +
                                                          std::abs(cplx(cs[b][2 * r + 1].x, cs[b][2 * r + 1].y)) > 0.0;
                }
            if (!ok) continue;
            unsigned piv = 0;
            for (int b = 0; b < W; ++b) {
                if (!(bits >> b & 1)) continue;
                double2* c = cs[b];
                const int fb = bundle ? b : 0;
                cplx scale[2], rho[2];
                for (int r = 0; r < 2; ++r) {
                    const cplx a0(c[2 * r].x, c[2 * r].y), a1(c[2 * r + 1].x, c[2 * r + 1].y);
                    // pivot on the diagonal entry (row r on column r) unless it is zero or tiny next
                    // to the other entry: with a fused multiply-add the row's error stays ~1 ulp of
                    // |a0 x0| + |a1 x1| whichever nonzero entry pivots, and a fixed orientation keeps
                    // the generated source -- and so the compiled kernel -- independent of the
                    // angles (a variational circuit with new angles reuses its kernels)
                    const double ad = std::abs(r ? a1 : a0), ao = std::abs(r ? a0 : a1);
                    static const bool larger = knob("QCS_PIVOT_LARGER");  // A/B: round-1 rule
                    const int pv = larger ? (std::abs(a1) > std::abs(a0) ? 1 : 0)
                                          : ((ad > 0.0 && ad >= 0x1p-20 * ao) ? r : 1 - r);
                    scale[r] = pv ? a1 : a0;
                    rho[r] = (pv ? a0 : a1) / scale[r];
                    piv |= unsigned(pv) << (4 * fb + r);
                    if (rho[r] == cplx(0.0, 0.0)) piv |= 1u << (4 * fb + 2 + r);
                }
                for (int r = 0; r < 2; ++r) c[r] = make_double2(rho[r].real(), rho[r].imag());
                c[2] = c[3] = make_double2(0.0, 0.0);
                const int rb = bundle ? b : o.t;
                if (chain[rb] >= 0) {  // G' = G diag(scale0, scale1): columns of the later gate
                    RegOp& g = rops[std::size_t(chain[rb])];
                    double2* gc = (g.kind & KF_BUNDLE) ? P.pool + g.ref + 4 * rb : g.c;
                    for (int e = 0; e < 4; ++e) {
                        const cplx v = cplx(gc[e].x, gc[e].y) * scale[e & 1];
                        gc[e] = make_double2(v.real(), v.imag());
                    }
                    bool real = true;  // the later gate's kind: real only if all its coefficients are
                    const unsigned gb = (g.kind & KF_BUNDLE) ? g.t : 1u;
                    for (int bb = 0; bb < W; ++bb) {
                        if (!(gb >> bb & 1)) continue;
                        const double2* x = (g.kind & KF_BUNDLE) ? P.pool + g.ref + 4 * bb : g.c;
                        for (int e = 0; e < 4; ++e) real &= x[e].y == 0.0;
                    }
                    g.kind = std::uint8_t(real ? (g.kind | KF_REAL) : (g.kind & ~KF_REAL));
                    continue;
                }
                for (int q = 0; q < G; ++q)
                    if (en >> q & 1) table[q] *= scale[q >> rb & 1];
            }
            bool real = true;
            for (int b = 0; b < W; ++b)
                if (bits >> b & 1) real &= cs[b][0].y == 0.0 && cs[b][1].y == 0.0;
            o.kind = std::uint8_t((o.kind & ~KF_REAL) | KF_PIVOT | (real ? KF_REAL : 0));
            o.dtab = std::uint16_t(piv);
            changed = true;
        }
        if (changed) {
            if (tab < 0) {
                RegOp t{};
                t.kind = TOP_DTAB;
                t.ref = std::uint16_t(npool);
                npool += G;
                rops.push_back(t);
                tab = int(rops.size()) - 1;
            }
            RegOp& t = rops[std::size_t(tab)];
            t.dskip = 0;
            t.smask = 0;
            for (int q = 0; q < G; ++q) {
                P.pool[t.ref + q] = make_double2(table[q].real(), table[q].imag());
                if (table[q] == cplx(1.0, 0.0)) {
                    if (q < 8) t.dskip = std::uint8_t(t.dskip | (1u << q));
                    t.smask |= 1u << q;
                }
            }
        }
        ops.insert(ops.end(), rops.begin(), rops.end());
        ops.insert(ops.end(), trailing.begin(), trailing.end());
        R.op_count = std::uint16_t(ops.size() - R.op_begin);
    }
    if (int(ops.size()) > kPassMaxOps) raise(QCS_ERR_SIM, "internal: too many operations in a pass");
    std::copy(ops.begin(), ops.end(), P.ops);
    std::copy(rounds.begin(), rounds.end(), P.rounds);
    P.nops = int(ops.size());
}

// Table normalisation (round 2): every round's diagonal table but the pass's last is divided by
// its entry 0 -- which becomes exactly 1 and is skipped (one complex multiply per 8 amplitudes
// less) -- and the product of those entries, a scalar that commutes with everything, joins the
// pass's last table.  Passes with sign-step programs or tile lists keep their tables.
void normalize_tables(PassParams& P) {
    static const bool off = knob("QCS_NO_TABLE_NORM");  // A/B switch
    if (off || P.alt_mode != ALT_NONE || P.list_cnt) return;
    std::vector<std::pair<int, int>> tabs;  // (op index, registers per group)
    for (int r = 0; r < P.nrounds; ++r) {
        const RoundDesc& R = P.rounds[r];
        if (R.flags & RD_SMEM) continue;
        for (int i = R.op_begin; i < R.op_begin + R.op_count; ++i)
            if ((P.ops[i].kind & KF_KIND) == TOP_DTAB) tabs.push_back({i, 1 << round_width(R)});
    }
    if (tabs.size() < 2) return;
    cplx carry(1.0, 0.0);
    auto entry = [&](const RegOp& t, int q) { return cplx(P.pool[t.ref + q].x, P.pool[t.ref + q].y); };
    auto store = [&](RegOp& t, int q, cplx v) {
        P.pool[t.ref + q] = make_double2(v.real(), v.imag());
        const bool one = v == cplx(1.0, 0.0);
        if (q < 8) t.dskip = std::uint8_t(one ? (t.dskip | (1u << q)) : (t.dskip & ~(1u << q)));
        t.smask = one ? (t.smask | (1u << q)) : (t.smask & ~(1u << q));
    };
    for (std::size_t k = 0; k + 1 < tabs.size(); ++k) {
        RegOp& t = P.ops[tabs[k].first];
        const int G = tabs[k].second;
        const cplx f = entry(t, 0);
        if (f == cplx(1.0, 0.0) || std::abs(f) == 0.0 || !std::isfinite(f.real()) || !std::isfinite(f.imag())) continue;
        const cplx nc = carry * f;
        if (!std::isfinite(nc.real()) || std::abs(nc) == 0.0) continue;
        for (int q = 1; q < G; ++q) store(t, q, entry(t, q) / f);
        store(t, 0, cplx(1.0, 0.0));
        carry = nc;
    }
    if (carry == cplx(1.0, 0.0)) return;
    RegOp& last = P.ops[tabs.back().first];
    for (int q = 0; q < tabs.back().second; ++q) store(last, q, entry(last, q) * carry);
}

}  // namespace

namespace {

// D' (y) = D (pi_k ( ... pi_1 (y))) for X-like relabellings pi_i (target t, controls in ctrl_mask:
// y -> y ^ (cond(y) ? e_t : 0)), as a diagonal on the bits D's bits depend on; false when those
// are more than three.
template <class At>
bool conjugate_diag(const FOp& d, const std::vector<int>& perms, At at, FOp& out) {
    u64 dep[64];  // bits of y that bit b of pi_k(...pi_1(y)) depends on
    for (int b = 0; b < 64; ++b) dep[b] = u64(1) << b;
    for (int idx : perms) {  // (controls outside the tile make the diagonal depend on them: fine)
        const FOp& p = at(idx);
        const int t = p.tpos[0];
        for (int b = 0; b < 64; ++b)
            if (p.ctrl_mask >> b & 1) dep[t] |= dep[b];
    }
    u64 sup = 0;
    for (int i = 0; i < d.dk; ++i) sup |= dep[d.dpos[i]];
    const int k = __builtin_popcountll(sup);
    if (k > 3 || k < 1) return false;
    int pos[3], np = 0;  // ascending support positions
    for (int b = 0; b < 64; ++b)
        if (sup >> b & 1) pos[np++] = b;
    GateOp g;
    g.k = k;
    for (int i = 0; i < k; ++i) g.pos[i] = pos[k - 1 - i];  // most significant first
    const int dim = 1 << k;
    g.m.assign(std::size_t(dim) * dim, cplx(0.0, 0.0));
    for (int a = 0; a < dim; ++a) {
        u64 y = 0;  // canonical local index a: bit k-1-i <-> pos[i] (most significant first)
        for (int i = 0; i < k; ++i)
            if (a >> (k - 1 - i) & 1) y |= u64(1) << g.pos[i];
        for (int idx : perms) {
            const FOp& p = at(idx);
            if ((y & p.ctrl_mask) == p.ctrl_val) y ^= u64(1) << p.tpos[0];
        }
        int e = 0;
        for (int i = 0; i < d.dk; ++i) e |= int((y >> d.dpos[i]) & 1) << (d.dk - 1 - i);
        g.m[std::size_t(a) * dim + a] = cplx(d.dval[e].x, d.dval[e].y);
    }
    return make_fop(g, out) && out.kind == TOP_DIAG;
}

// Round scheduling (light cones).  A pass's operations arrive in circuit order, so a layered
// circuit (C4: a gate on every qubit, then diagonals coupling neighbours) forms one register round
// per three qubits per layer.  But a layer-(L+1) gate on a bit only waits for the operations that
// do not commute with it -- the bit's own layer-L gate and the diagonals on it -- so once its
// diagonal partners have their layer-L gates, it can run in the SAME round as those (one
// shared-memory round trip for two layers).  This reorders the pass's list (only commuting
// operations swap places) into groups, each the ready operations on a set of three register
// bits chosen greedily for the most gates: +-1 diagonals (sign flips, CZ) run as soon as they
// are ready, phase diagonals wait for a group holding their bits.  A one-bit phase followed in
// its group by a gate on that bit, with only diagonals between, folds into the gate (G' = G D):
// one complex 2x2 instead of a multiply on every register.  Used when it saves rounds.
struct SchedOp {
    bool elem = false;        // commutes with every other elementwise operation
    bool gate = false;        // needs its target in the registers
    bool takeable_any = false;  // elementwise and cheap anywhere (+-1, scale)
    unsigned reg = 0;         // gate: local target bit mask; phase diagonal: local bits (0: outside)
    std::vector<int> succ;
    int npred = 0;
};

bool signed_diag(const FOp& f) {
    if (f.kind != TOP_DIAG) return false;
    for (int g = 0; g < (1 << f.dk); ++g)
        if (f.dval[g].y != 0.0 || (f.dval[g].x != 1.0 && f.dval[g].x != -1.0)) return false;
    return true;
}

int round_count(const std::vector<FOp>& ops, const std::vector<int>& list, const int* loc, int width) {
    int rounds = 0;
    unsigned cur = 0;
    bool open = false;
    for (int idx : list) {
        const FOp& f = ops[std::size_t(idx)];
        if (elementwise(f)) continue;
        const unsigned t = 1u << loc[f.tpos[0]];
        if (open && (__builtin_popcount(cur | t) <= width)) {
            cur |= t;
        } else {
            ++rounds;
            cur = t;
            open = true;
        }
    }
    return rounds;
}

bool schedule_rounds(int n, const int* loc, int m, const std::vector<FOp>& ops, const std::vector<int>& list,
                     std::vector<FOp>& out_ops, std::vector<int>& out_list, int width = 3) {
    static const bool off = knob("QCS_NO_ROUND_SCHED");  // A/B switch
    const int N = int(list.size());
    if (off || N < 4 || m < 4) return false;
    for (int idx : list) {
        const FOp& f = ops[std::size_t(idx)];
        const bool ok = f.kind == TOP_DIAG || f.kind == TOP_SCALE || (f.kind == TOP_WHT) ||
                        (f.kind == TOP_GATE && f.K == 1 && loc[f.tpos[0]] >= 0);
        if (!ok) return false;
    }
    std::vector<SchedOp> so(static_cast<std::size_t>(N));
    // dependencies through each basis bit: a non-elementwise operation waits for everything on
    // the bit since the previous one (and that one); an elementwise one for the previous one
    std::vector<int> last_nd(std::size_t(n), -1);
    std::vector<std::vector<int>> since(static_cast<std::size_t>(n));
    auto edge = [&](int a, int b) { so[std::size_t(a)].succ.push_back(b); ++so[std::size_t(b)].npred; };
    for (int i = 0; i < N; ++i) {
        const FOp& f = ops[std::size_t(list[std::size_t(i)])];
        SchedOp& o = so[std::size_t(i)];
        o.elem = elementwise(f);
        o.gate = !o.elem;
        if (o.gate) o.reg = 1u << loc[f.tpos[0]];
        if (f.kind == TOP_SCALE || signed_diag(f)) o.takeable_any = true;
        if (f.kind == TOP_DIAG && !o.takeable_any) {
            bool inside = true;
            for (int j = 0; j < f.dk; ++j) {
                if (loc[f.dpos[j]] < 0) inside = false;
                else o.reg |= 1u << loc[f.dpos[j]];
            }
            if (!inside) o.reg = 0;  // a bit outside the tile: never in the registers
        }
        std::vector<int> preds;
        for (int b = 0; b < n; ++b) {
            if (!(f.touch >> b & 1)) continue;
            if (o.elem) {
                if (last_nd[std::size_t(b)] >= 0) preds.push_back(last_nd[std::size_t(b)]);
                since[std::size_t(b)].push_back(i);
            } else {
                if (last_nd[std::size_t(b)] >= 0) preds.push_back(last_nd[std::size_t(b)]);
                for (int e : since[std::size_t(b)]) preds.push_back(e);
                since[std::size_t(b)].clear();
                last_nd[std::size_t(b)] = i;
            }
        }
        std::sort(preds.begin(), preds.end());
        preds.erase(std::unique(preds.begin(), preds.end()), preds.end());
        for (int p : preds) edge(p, i);
    }
    std::vector<int> cnt(static_cast<std::size_t>(N)), tmp(static_cast<std::size_t>(N));
    for (int i = 0; i < N; ++i) cnt[std::size_t(i)] = so[std::size_t(i)].npred;
    std::vector<char> done(std::size_t(N), 0);
    std::vector<int> order, group_of;
    order.reserve(std::size_t(N));
    int group = 0;
    auto takeable = [&](int i, unsigned T) {
        if (T == ~0u) return true;  // the final group: everything that is left
        const SchedOp& o = so[std::size_t(i)];
        if (o.gate) return (o.reg & ~T) == 0;
        if (o.takeable_any) return true;
        return o.reg != 0 && (o.reg & ~T) == 0;
    };
    // run the ready closure for register set T; commit: record the order, else count gates
    std::vector<int> stack, taken;
    auto closure = [&](unsigned T, bool commit, long& score) {
        tmp = cnt;
        stack.clear();
        taken.clear();
        for (int i = 0; i < N; ++i)
            if (!done[std::size_t(i)] && tmp[std::size_t(i)] == 0) stack.push_back(i);
        std::sort(stack.begin(), stack.end(), std::greater<int>());  // lowest index first
        int gates = 0;
        long early = 0;
        while (!stack.empty()) {
            const int i = stack.back();
            stack.pop_back();
            if (!takeable(i, T)) continue;
            taken.push_back(i);
            if (so[std::size_t(i)].gate) {
                ++gates;
                early += N - i;
            }
            for (int s2 : so[std::size_t(i)].succ)
                if (--tmp[std::size_t(s2)] == 0) stack.push_back(s2);
        }
        score = long(gates) * (1L << 32) + early;
        if (commit) {
            for (int i : taken) {
                done[std::size_t(i)] = 1;
                order.push_back(i);
                group_of.push_back(group);
            }
            cnt = tmp;
            ++group;
        }
        return gates;
    };
    static const long bank_penalty = [] {
        const char* v = std::getenv("QCS_BANK_PENALTY");  // in quarter gates
        return long((v ? std::atof(v) : 0.0) * double(1L << 30));  // default off: C4 n=32 has 4 such rounds of 39, and avoiding them costs a round
    }();
    while (int(order.size()) < N) {
        unsigned U = 0;  // bits with an unscheduled gate
        for (int i = 0; i < N; ++i)
            if (!done[std::size_t(i)] && so[std::size_t(i)].gate) U |= so[std::size_t(i)].reg;
        if (!U) {  // only diagonals left: the rest in list order
            long sc;
            closure(~0u, true, sc);
            continue;
        }
        std::vector<int> bits;
        for (int b = 0; b < m; ++b)
            if (U >> b & 1) bits.push_back(b);
        long best = -1;
        unsigned bestT = 0;
        const int nb = int(bits.size());
        // every subset of min(width, nb) of the bits with pending gates
        const int k = std::min(width, nb);
        std::vector<int> pick(static_cast<std::size_t>(k));
        for (int i = 0; i < k; ++i) pick[std::size_t(i)] = i;
        for (;;) {
            unsigned T = 0;
            for (int i : pick) T |= 1u << bits[std::size_t(i)];
            long sc;
            closure(T, false, sc);
            // register sets that hold local bits b and b + 3 (b < 3) leave no thread-index bit for
            // bank-group bit b of the swizzled tile (position j ^ ((j >> 3) & 7)): every 16-byte
            // access of the round is a 2-way bank conflict.  Cost: a fraction of a gate per pair.
            for (int b = 0; b < 3; ++b)
                if ((T >> b & 1u) && (T >> (b + 3) & 1u)) sc -= bank_penalty;
            if (sc > best) {
                best = sc;
                bestT = T;
            }
            int i = k - 1;
            while (i >= 0 && pick[std::size_t(i)] == nb - k + i) --i;
            if (i < 0) break;
            ++pick[std::size_t(i)];
            for (int j = i + 1; j < k; ++j) pick[std::size_t(j)] = pick[std::size_t(j - 1)] + 1;
        }
        long sc;
        if (closure(bestT, true, sc) == 0) return false;  // no progress: keep the circuit order
    }
    // fold one-bit phases into the next gate on their bit within their group
    out_ops.clear();
    out_list.clear();
    std::vector<char> gone(std::size_t(N), 0);
    std::vector<FOp> local(static_cast<std::size_t>(N));
    for (int i = 0; i < N; ++i) local[std::size_t(i)] = ops[std::size_t(list[std::size_t(i)])];
    for (std::size_t k = 0; k < order.size(); ++k) {
        const int i = order[k];
        const FOp& d = local[std::size_t(i)];
        if (d.kind != TOP_DIAG || d.dk != 1 || d.src.k != 1 || signed_diag(d)) continue;
        const int bit = d.dpos[0];
        for (std::size_t j = k + 1; j < order.size() && group_of[j] == group_of[k]; ++j) {
            const FOp& g = local[std::size_t(order[j])];
            if (!(g.touch >> bit & 1) || gone[std::size_t(order[j])]) continue;
            if (elementwise(g)) continue;  // diagonals commute with the phase
            if (g.kind == TOP_GATE && g.K == 1 && g.ctrl_mask == 0 && g.src.k == 1 && g.tpos[0] == bit) {
                GateOp p;
                p.k = 1;
                p.pos[0] = bit;
                p.m.resize(4);
                for (int r = 0; r < 2; ++r)
                    for (int c = 0; c < 2; ++c)
                        p.m[std::size_t(r * 2 + c)] = g.src.m[std::size_t(r * 2)] * d.src.m[std::size_t(c)] +
                                                      g.src.m[std::size_t(r * 2 + 1)] * d.src.m[std::size_t(2 + c)];
                FOp merged;
                if (make_fop(p, merged) && merged.kind == TOP_GATE) {
                    local[std::size_t(order[j])] = std::move(merged);
                    gone[std::size_t(i)] = 1;
                }
            }
            break;
        }
    }
    for (int i : order) {
        if (gone[std::size_t(i)]) continue;
        out_ops.push_back(local[std::size_t(i)]);
        out_list.push_back(int(out_ops.size()) - 1);
    }
    return round_count(out_ops, out_list, loc, width) < round_count(ops, list, loc, width);
}

}  // namespace

void lower_plan(int n, const std::vector<FOp>& ops_in, const Plan& plan, Lowered& out) {
    out = Lowered{};
    // Missed-tile programs (tile-kernel passes of >= 2 operations).  One that is only a scalar
    // s becomes a skip: the pass's tiles reached by a sign step get scale(1/s) appended, and the
    // product of the s moves to a pass that runs every tile (scalars commute with everything).
    const std::size_t np = plan.passes.size();
    std::vector<std::vector<int>> lists(np);
    std::vector<std::vector<FOp>> alts(np);
    std::vector<char> has_alt(np, 0);
    bool any_plain = false;  // a pass that runs every tile exists (it can carry the scalars)
    for (std::size_t i = 0; i < np; ++i) {
        lists[i] = plan.passes[i].ops;
        if (lists[i].size() >= 2) has_alt[i] = missed_tile_program(ops_in, lists[i], alts[i]);
        any_plain |= !has_alt[i];
    }
    std::vector<FOp> ext;  // ops_in plus the scales the deferral adds
    bool extended = false;
    auto add_op = [&](const FOp& f) {
        if (!extended) {
            ext = ops_in;
            extended = true;
        }
        ext.push_back(f);
        return int(ext.size()) - 1;
    };
    double carry = 1.0;
    std::vector<char> skip(np, 0);
    for (std::size_t i = 0; i < np && any_plain; ++i) {
        if (!has_alt[i] || alts[i].size() > 1 || (alts[i].size() == 1 && alts[i][0].kind != TOP_SCALE)) continue;
        const double sc = alts[i].empty() ? 1.0 : alts[i][0].scale;
        if (sc != 1.0) {
            if (std::fabs(std::log2(std::fabs(carry * sc))) > 400.0) continue;  // keep clear of under/overflow
            lists[i].push_back(add_op(make_scale(1.0 / sc)));
            carry *= sc;
        }
        alts[i].clear();
        skip[i] = 1;
    }
    // Pass pairs around a skip pass.  With Q a skip pass (the identity, after the carried scalar,
    // on every tile its sign steps miss) between passes P and P' on the same tile bits whose
    // programs compose to a scalar s (P' P = s I: e.g. the same butterflies twice, Grover's
    // H_low ... H_low), the triple P' Q P is s I on every P-tile that no tile Q reaches
    // intersects.  So P and P' run only on the P-tiles that do (one Q-tile meets 2^k P-tiles,
    // k = the Q-tile bits outside P's tile), s moves to the carrier, and P' appends 1/s on the
    // tiles it runs.  Exact: s is a power of two (butterfly pairs) times the pass scales.
    std::vector<std::vector<u64>> forced(np);
    for (std::size_t i = 0; i + 2 < np && any_plain; ++i) {
        const std::size_t j = i + 1, k = i + 2;
        if (!skip[j] || !forced[i].empty() || has_alt[i] || has_alt[k] || lists[i].size() < 2 || lists[k].size() < 2)
            continue;
        const u64 S = plan.passes[i].tile, SQ = plan.passes[j].tile;
        if (plan.passes[k].tile != S) continue;
        std::vector<int> both = lists[i];
        both.insert(both.end(), lists[k].begin(), lists[k].end());
        double s2 = 1.0;
        std::vector<int> rest;
        reduce_scalar(extended ? ext : ops_in, both, s2, rest);
        if (!rest.empty() || s2 == 0.0 || std::fabs(std::log2(std::fabs(carry * s2))) > 400.0) continue;
        // the P-tiles that the reached Q-tiles meet
        std::vector<u64> flips;
        for (int idx : lists[j]) {
            const FOp& f = (extended ? ext : ops_in)[std::size_t(idx)];
            if (f.kind == TOP_SIGN) flips.insert(flips.end(), f.flips.begin(), f.flips.end());
        }
        const u64 full = n >= 64 ? ~u64(0) : (u64(1) << n) - 1;
        const u64 outP = full & ~S, freeb = outP & SQ;  // P-tile bits a Q-tile leaves free
        const int nfree = __builtin_popcountll(freeb), nout = __builtin_popcountll(outP);
        if (flips.empty() || nfree > 16 || nout >= 63) continue;
        std::vector<u64> touched;
        for (u64 e : flips)
            for (u64 v = 0; v < (u64(1) << nfree); ++v) {
                u64 x = e & ~freeb, w = v;  // deposit v into the free bits
                for (int b = 0; b < n; ++b)
                    if (freeb >> b & 1) {
                        x = (x & ~(u64(1) << b)) | ((w & 1) << b);
                        w >>= 1;
                    }
                u64 tile = 0;  // x's bits outside P's tile, compressed
                for (int b = 0, c = 0; b < n; ++b)
                    if (outP >> b & 1) tile |= ((x >> b) & 1) << c++;
                touched.push_back(tile);
            }
        std::sort(touched.begin(), touched.end());
        touched.erase(std::unique(touched.begin(), touched.end()), touched.end());
        if (touched.size() > (u64(1) << nout) / 8) continue;  // not worth it
        if (s2 != 1.0) {
            lists[k].push_back(add_op(make_scale(1.0 / s2)));
            carry *= s2;
        }
        forced[i] = touched;
        forced[k] = touched;
        ++i;  // P' is used up
    }
    int carrier = -1;
    for (std::size_t i = 0; i < np && carrier < 0; ++i)
        if (!has_alt[i] && forced[i].empty()) carrier = int(i);
    if (carry != 1.0) {
        if (carrier < 0) raise(QCS_ERR_SIM, "internal: no pass to carry the deferred scalars");
        auto& cl = lists[std::size_t(carrier)];
        cl.insert(cl.begin(), add_op(make_scale(carry)));
    }
    // scalars commute with everything: one scale per pass (the planner pulls every H^n step's
    // 2^(-n/2) into the first pass, and the carried scalars join them)
    for (std::size_t i = 0; i < np; ++i) {
        int first = -1, count = 0;
        double prod = 1.0;
        for (std::size_t k = 0; k < lists[i].size(); ++k) {
            const FOp& f = (extended ? ext : ops_in)[std::size_t(lists[i][k])];
            if (f.kind != TOP_SCALE) continue;
            if (first < 0) first = int(k);
            prod *= f.scale;
            ++count;
        }
        // (a pass of scales only stays as it is: as one operation it would leave the tile kernels)
        if (count < 2 || count == int(lists[i].size()) || !std::isfinite(prod) || prod == 0.0) continue;
        std::vector<int> keep;
        for (std::size_t k = 0; k < lists[i].size(); ++k) {
            const int idx = lists[i][k];
            if (int(k) == first) keep.push_back(add_op(make_scale(prod)));
            else if ((extended ? ext : ops_in)[std::size_t(idx)].kind != TOP_SCALE) keep.push_back(idx);
        }
        lists[i].swap(keep);
    }
    const std::vector<FOp>& ops = extended ? ext : ops_in;
    for (std::size_t pi = 0; pi < np; ++pi) {
        const PlannedPass& pp = plan.passes[pi];
        PassParams P{};
        int loc[64];
        std::fill(loc, loc + 64, -1);
        for (int b = 0; b < n; ++b)
            if (pp.tile >> b & 1) {
                loc[b] = P.m;
                P.bits[P.m++] = b;
            }
        int nops = 0, nsign = 0, npool = 0;
        std::uint64_t flip_off = 0, flip_cnt = 0;
        const bool virt_pass = jit_virtual(n, P.m, has_alt[pi] && alts[pi].empty());
        // 16-amplitude register rounds (4 register bits) for passes the specialised kernels run
        // with pivots: gates and diagonals only (no sign steps, shared-memory gates, relabellings)
        int RW = 3;
        if (knob_w4() && !has_alt[pi] && forced[pi].empty() && P.m >= 8 && (jit_mode() == 1 || jit_mode() == 3)) {
            bool ok = true;
            for (int idx : lists[pi]) {
                const FOp& f = ops[std::size_t(idx)];
                if (f.kind == TOP_SIGN || (f.kind == TOP_GATE && f.K >= 2)) ok = false;
                static const bool w4_perms = [] { const char* v = std::getenv("QCS_W4_PERMS"); return v && std::atoi(v) != 0; }();
                if (f.kind == TOP_GATE && f.K == 1 && f.nrows == 2 && f.nnz[0] == 1 && f.nnz[1] == 1 && virt_pass && !w4_perms) ok = false;
            }
            // worth it only for passes with arithmetic to spare: a pass of a few butterflies is
            // HBM bound, and the 16-register kernels keep 2 tiles resident per SM instead of 3
            // (C3 n=30: 11.1 ms with them, 9.9 ms without)
            static const int w4_min_gates = [] { const char* v = std::getenv("QCS_W4_MIN_GATES"); return v ? std::atoi(v) : 16; }();
            int work = 0;
            for (int idx : lists[pi]) {
                const FOp& f = ops[std::size_t(idx)];
                work += (f.kind == TOP_GATE || f.kind == TOP_WHT) ? 1 : 0;
            }
            if (ok && work >= w4_min_gates) RW = 4;
        }
        const int RG = 1 << RW;  // registers per group
        // rounds of <= 3 register bits; gates on 2-3 targets get shared-memory rounds
        struct RoundPlan {
            bool smem;
            unsigned mask;
            std::vector<int> ops;
            std::vector<int> perms;  // virtual permutations at the round's start (TOP_PERM)
        };
        // Virtual permutations (specialised kernels only): an X-like gate with at most one
        // control, all in the tile, moves no data and needs no register bit -- it becomes a
        // relabelling of the shared-memory addresses of the following rounds (an affine map over
        // the local index bits), and at the pass end, if the layout is not the identity, the
        // last round stores straight to HBM at the relabelled indices.  The gate is placed at a
        // round boundary; operations after it join the current round only if they commute.
        auto is_perm = [&](const FOp& f) {
            if (f.kind != TOP_GATE || f.K != 1 || f.nrows != 2 || f.nnz[0] != 1 || f.nnz[1] != 1) return false;
            if (!(f.val[0][0].x == 1.0 && f.val[0][0].y == 0.0 && f.val[1][0].x == 1.0 && f.val[1][0].y == 0.0 &&
                  f.col_member[0][0] == 1 && f.col_member[1][0] == 0 && f.row_member[0] == 0 && f.row_member[1] == 1))
                return false;
            if (loc[f.tpos[0]] < 0) return false;
            int inside = 0, outside = 0;
            for (int b = 0; b < n; ++b)
                if (f.ctrl_mask >> b & 1) ++(loc[b] >= 0 ? inside : outside);
            // one control in the tile (a linear relabelling), or controls outside it only (a
            // relabelling offset on the tiles where they hold)
            return (inside <= 1 && outside == 0) || inside == 0;
        };
        auto lower_list = [&](const std::vector<FOp>& src, const std::vector<int>& list) {
        // diagonals moved ahead of pending relabellings (conjugated): indices past src
        std::vector<FOp> extra;
        extra.reserve(list.size());
        auto at = [&](int idx) -> const FOp& {
            return idx < int(src.size()) ? src[std::size_t(idx)] : extra[std::size_t(idx) - src.size()];
        };
        std::vector<RoundPlan> rounds;
        bool virt = virt_pass;
        for (int idx : list)  // shared-memory gate rounds address the tile directly: no relabelling
            if (at(idx).kind == TOP_GATE && at(idx).K >= 2) virt = false;
        std::vector<int> pending;  // virtual permutations after the current round's operations
        u64 pending_touch = 0;
        for (int idx : list) {
            const FOp& f = at(idx);
            if (virt && is_perm(f)) {
                pending.push_back(idx);
                pending_touch |= f.touch;
                continue;
            }
            static const bool no_conj = std::getenv("QCS_NO_CONJ") != nullptr;  // A/B switch
            if (!no_conj && !pending.empty() && f.kind == TOP_DIAG && (f.touch & pending_touch) && !rounds.empty() &&
                !rounds.back().smem) {
                // D after the pending relabellings pi_1..pi_k is D' = D o pi_k o ... o pi_1 before
                // them: still diagonal, on the bits D's bits depend on through the relabellings
                FOp g;
                if (conjugate_diag(f, pending, at, g)) {
                    extra.push_back(std::move(g));
                    const int nidx = int(src.size() + extra.size()) - 1;
                    rounds.back().ops.push_back(nidx);
                    continue;
                }
            }
            if (!pending.empty() && (f.kind == TOP_SIGN || (f.touch & pending_touch) || rounds.empty())) {
                // after the pending permutations: a new round whose loads apply them
                unsigned t0 = 0;
                if (!elementwise(f))
                    for (int i = 0; i < f.K; ++i) t0 |= 1u << loc[f.tpos[i]];
                rounds.push_back({false, t0, {idx}, pending});
                pending.clear();
                pending_touch = 0;
                continue;
            }
            const bool smem = f.kind == TOP_GATE && f.K >= 2;
            unsigned t = 0;
            if (!elementwise(f))
                for (int i = 0; i < f.K; ++i) t |= 1u << loc[f.tpos[i]];
            if (smem) {
                if (!rounds.empty() && rounds.back().smem) rounds.back().ops.push_back(idx);
                else rounds.push_back({true, 0u, {idx}});
                continue;
            }
            if (rounds.empty() || rounds.back().smem) {
                rounds.push_back({false, t, {idx}});
                continue;
            }
            auto& cur = rounds.back();
            if ((t & ~cur.mask) == 0) {
                cur.ops.push_back(idx);
            } else if (__builtin_popcount(cur.mask | t) <= RW) {
                cur.mask |= t;
                cur.ops.push_back(idx);
            } else {
                rounds.push_back({false, t, {idx}});
            }
        }
        if (!pending.empty()) {  // permutations after the last operation: the last round's stores
            if (rounds.empty()) rounds.push_back({false, 0u, {}, {}});
            for (int idx : pending) rounds.back().ops.push_back(idx);  // trailing TOP_PERM ops
        }
        for (auto& r : rounds) {
            if (P.nrounds >= kPassMaxOps) raise(QCS_ERR_SIM, "internal: too many rounds in a pass");
            unsigned mask = r.mask;
            // pad to RW register bits, preferring bits above 2: a round without bits 0..2 can
            // move its amplitudes to and from HBM directly (whole 128-byte runs per warp)
            const int rw = r.smem ? 3 : RW;
            for (int b = 3; b < P.m && __builtin_popcount(mask) < rw; ++b) mask |= 1u << b;
            for (int b = 0; b < P.m && __builtin_popcount(mask) < rw; ++b) mask |= 1u << b;
            RoundDesc& rd = P.rounds[P.nrounds++];
            rd.flags = r.smem ? RD_SMEM : 0;
            int c = 0;
            for (int b = 0; b < P.m; ++b)
                if (mask >> b & 1) {
                    if (c < 3) rd.r[c] = std::uint8_t(b);
                    else rd.flags = std::uint8_t(rd.flags | RD_W4 | (b << 4));
                    ++c;
                }
            auto reg = [&](int pos) -> int {
                const int l = loc[pos];
                for (int i = 0; i < round_width(rd); ++i)
                    if (round_reg(rd, i) == l) return i;
                return -1;
            };
            rd.op_begin = std::uint16_t(nops);
            // diagonals on the round's register bits that commute to the end of the round (no
            // later operation targets their bits) combine into one table of 8 entries (TOP_DTAB)
            std::vector<int> seq, tab;
            if (!r.smem) {
                for (std::size_t i = 0; i < r.ops.size(); ++i) {
                    const FOp& f = at(r.ops[i]);
                    bool movable = !kNoTables && f.kind == TOP_DIAG && npool + RG <= kPassPool - 4 * RW;
                    for (int j = 0; movable && j < f.dk; ++j) movable = loc[f.dpos[j]] >= 0 && reg(f.dpos[j]) >= 0;
                    if (movable) {  // +-1 diagonals stay pending sign flips (cheaper)
                        bool signed_only = true;
                        for (int g = 0; g < (1 << f.dk); ++g) {
                            const double2 d = f.dval[g];
                            if (d.y != 0.0 || (d.x != 1.0 && d.x != -1.0)) signed_only = false;
                        }
                        movable = !signed_only;
                    }
                    for (std::size_t j = i + 1; movable && j < r.ops.size(); ++j) {
                        const FOp& g = at(r.ops[j]);
                        if (g.kind != TOP_GATE && g.kind != TOP_WHT) continue;
                        u64 tg = 0;
                        for (int k = 0; k < g.K; ++k) tg |= u64(1) << g.tpos[k];
                        if (tg & f.touch) movable = false;
                    }
                    (movable ? tab : seq).push_back(r.ops[i]);
                }
            } else {
                seq = r.ops;
            }
            bool pending_signs = false;  // a +-1 diagonal since the last butterfly / gate
            auto perm_op = [&](const FOp& f) {  // virtual permutation: target / control as local bits
                if (nops >= kPassMaxOps) raise(QCS_ERR_SIM, "internal: too many operations in a pass");
                RegOp o{};
                o.kind = TOP_PERM;
                o.t = std::uint8_t(loc[f.tpos[0]]);
                for (int b = 0; b < n; ++b) {
                    if (!(f.ctrl_mask >> b & 1)) continue;
                    const bool want = f.ctrl_val >> b & 1;
                    if (loc[b] >= 0) {
                        o.lctrl_mask = std::uint16_t(o.lctrl_mask | (1u << loc[b]));
                        if (want) o.lctrl_val = std::uint16_t(o.lctrl_val | (1u << loc[b]));
                    } else {
                        o.gctrl_mask |= u64(1) << b;
                        if (want) o.gctrl_val |= u64(1) << b;
                    }
                }
                if (o.gctrl_mask) o.kind = std::uint8_t(o.kind | KF_GCTRL);
                P.ops[nops++] = o;
            };
            for (int idx : r.perms) perm_op(at(idx));  // before the round's loads
            std::vector<int> trailing;  // after the pass's last operations: the last round's stores
            for (int idx : seq) {
                const FOp& f = at(idx);
                if (virt && is_perm(f)) {
                    trailing.push_back(idx);
                    continue;
                }
                if (nops >= kPassMaxOps) raise(QCS_ERR_SIM, "internal: too many operations in a pass");
                RegOp o{};
                o.kind = std::uint8_t(f.kind);
                for (int b = 0; b < n; ++b) {  // controls: in the tile per group, outside per tile
                    if (!(f.ctrl_mask >> b & 1)) continue;
                    const bool want = f.ctrl_val >> b & 1;
                    if (loc[b] >= 0) {
                        o.lctrl_mask |= 1u << loc[b];
                        if (want) o.lctrl_val |= 1u << loc[b];
                    } else {
                        o.gctrl_mask |= u64(1) << b;
                        if (want) o.gctrl_val |= u64(1) << b;
                    }
                }
                TileOp big{};
                bool use_big = false;
                switch (f.kind) {
                    case TOP_GATE:
                        if (rd.flags & RD_SMEM) {
                            big.gcase = f.K;
                            for (int i = 0; i < f.K; ++i) big.tl[i] = loc[f.tpos[i]];
                            big.nrows = f.nrows;
                            big.lctrl_mask = o.lctrl_mask;
                            big.lctrl_val = o.lctrl_val;
                            big.gctrl_mask = o.gctrl_mask;
                            big.gctrl_val = o.gctrl_val;
                            std::memcpy(big.row_member, f.row_member, sizeof(big.row_member));
                            std::memcpy(big.nnz, f.nnz, sizeof(big.nnz));
                            std::memcpy(big.col_member, f.col_member, sizeof(big.col_member));
                            std::memcpy(big.val, f.val, sizeof(big.val));
                            use_big = true;
                        } else {
                            o.t = std::uint8_t(reg(f.tpos[0]));
                            // dense 2x2 (rows the gate leaves alone stay identity rows): the
                            // kernel's one straight-line form; zeros and ones are exact under fma
                            o.c[0] = o.c[3] = make_double2(1.0, 0.0);
                            o.c[1] = o.c[2] = make_double2(0.0, 0.0);
                            for (int row = 0; row < f.nrows; ++row) {
                                const int rm = f.row_member[row];
                                o.c[2 * rm] = o.c[2 * rm + 1] = make_double2(0.0, 0.0);
                                for (int z = 0; z < f.nnz[row]; ++z) o.c[2 * rm + f.col_member[row][z]] = f.val[row][z];
                            }
                            if (!kNoReal && o.c[0].y == 0.0 && o.c[1].y == 0.0 && o.c[2].y == 0.0 && o.c[3].y == 0.0)
                                o.kind = std::uint8_t(o.kind | KF_REAL);
                        }
                        break;
                    case TOP_WHT: {  // a run of single-bit butterflies becomes one masked op
                        const unsigned bit = 1u << reg(f.tpos[0]);
                        if (nops > rd.op_begin && (P.ops[nops - 1].kind & ~KF_FLUSH) == TOP_WHT && !(P.ops[nops - 1].t & bit)) {
                            P.ops[nops - 1].t = std::uint8_t(P.ops[nops - 1].t | bit);
                            continue;
                        }
                        o.t = std::uint8_t(bit);
                        break;
                    }
                    case TOP_DIAG:
                        o.dk = std::uint8_t(f.dk);
                        for (int i = 0; i < f.dk; ++i) {
                            o.dpos[i] = std::uint8_t(f.dpos[i]);
                            const int rb = loc[f.dpos[i]] >= 0 ? reg(f.dpos[i]) : -1;
                            o.dreg[i] = rb >= 0 ? std::uint8_t(rb) : 0xff;
                        }
                        for (int q = 0; q < 8 && f.dk <= 2; ++q) {  // register part of the entry index
                            unsigned rp = 0;
                            for (int i = 0; i < f.dk; ++i)
                                if (o.dreg[i] < 3) rp |= ((unsigned(q) >> o.dreg[i]) & 1u) << (f.dk - 1 - i);
                            o.dtab = std::uint16_t(o.dtab | (rp << (2 * q)));
                        }
                        for (int g = 0; g < (1 << f.dk); ++g) {
                            if (f.dskip[g]) o.dskip = std::uint8_t(o.dskip | (1u << g));
                            if (g < 4) o.c[g] = f.dval[g];
                            big.val[0][g] = f.dval[g];
                        }
                        use_big = f.dk == 3;
                        break;
                    case TOP_SIGN:
                        o.sidx = std::uint32_t(nsign++);
                        big.flip_off = out.flips.size();
                        big.flip_cnt = f.flips.size();
                        big.flip_rest = f.flip_rest;
                        flip_off = big.flip_off;
                        flip_cnt = big.flip_cnt;
                        out.flips.insert(out.flips.end(), f.flips.begin(), f.flips.end());
                        use_big = true;
                        break;
                    case TOP_SCALE:
                        o.c[0] = make_double2(f.scale, 0.0);
                        break;
                    default: break;
                }
                if (use_big) {
                    if (out.big.size() >= 0xffff) raise(QCS_ERR_SIM, "internal: plan too large");
                    o.ref = std::uint16_t(out.big.size());
                    out.big.push_back(big);
                }
                if (o.gctrl_mask) o.kind = std::uint8_t(o.kind | KF_GCTRL);
                if (f.kind == TOP_DIAG && f.dk <= 2) {  // +-1 diagonals (Z, CZ, sign parts): sign flips
                    bool signed_only = true;
                    unsigned neg = 0;
                    for (int g = 0; g < (1 << f.dk); ++g) {
                        const double2 d = f.dval[g];
                        if (d.y != 0.0 || (d.x != 1.0 && d.x != -1.0)) signed_only = false;
                        if (d.x == -1.0) neg |= 1u << g;
                    }
                    if (signed_only) {
                        o.kind = std::uint8_t(o.kind | KF_SIGNED);
                        o.dskip = std::uint8_t(neg);
                        // for each value cg of the group-constant bits: the registers that flip
                        for (int cg = 0; cg < 4; ++cg) {
                            unsigned byte = 0;
                            for (int q = 0; q < 8; ++q) {
                                const int g = cg | int((o.dtab >> (2 * q)) & 3u);
                                if (neg >> g & 1) byte |= 1u << q;
                            }
                            o.smask |= byte << (8 * cg);
                        }
                    }
                }
                if (o.kind & KF_SIGNED) pending_signs = true;
                if ((f.kind == TOP_WHT || f.kind == TOP_GATE) && pending_signs) {
                    o.kind = std::uint8_t(o.kind | KF_FLUSH);
                    pending_signs = false;
                }
                // consecutive +-1 diagonals (CZ rings, Z): one bundled operation; the ones with
                // no group-constant bit fold into one flip byte at plan time
                if (o.kind == (TOP_DIAG | KF_SIGNED) && nops > rd.op_begin && RW == 3) {
                    RegOp& prev = P.ops[nops - 1];
                    auto add_entry = [&](const RegOp& x, RegOp& b) {
                        const bool c0 = x.dreg[0] == 0xff, c1 = x.dk == 2 && x.dreg[1] == 0xff;
                        if (!c0 && !c1) {
                            b.smask ^= x.smask & 0xffu;
                            return;
                        }
                        SignEntry e{};
                        e.smask = x.smask;
                        e.dk = x.dk;
                        e.p0 = x.dpos[0];
                        e.p1 = x.dpos[1];
                        e.cmask = std::uint8_t((c0 ? 1u : 0u) | (c1 ? 2u : 0u));
                        std::memcpy(&P.pool[npool++], &e, sizeof(e));
                        b.t = std::uint8_t(b.t + 1);
                    };
                    const bool prev_sign = (prev.kind & ~KF_BUNDLE) == (TOP_DIAG | KF_SIGNED);
                    if (prev_sign && npool + 2 <= kPassPool && prev.t < 250) {
                        if (!(prev.kind & KF_BUNDLE)) {
                            RegOp b = prev;
                            b.kind = std::uint8_t(b.kind | KF_BUNDLE);
                            b.smask = 0;
                            b.t = 0;
                            b.ref = std::uint16_t(npool);
                            add_entry(prev, b);
                            prev = b;
                        }
                        add_entry(o, prev);
                        continue;
                    }
                }
                // consecutive uncontrolled one-qubit gates on different register bits: one
                // bundled operation (one dispatch per group instead of up to three)
                if (f.kind == TOP_GATE && !(rd.flags & RD_SMEM) && (o.kind & ~KF_REAL) == TOP_GATE && !o.lctrl_mask &&
                    nops > rd.op_begin) {
                    RegOp& prev = P.ops[nops - 1];
                    const bool prev_gate = (prev.kind & ~(KF_BUNDLE | KF_FLUSH | KF_REAL)) == TOP_GATE &&
                                           !prev.lctrl_mask && (prev.kind & KF_REAL) == (o.kind & KF_REAL);
                    const unsigned pmask = (prev.kind & KF_BUNDLE) ? prev.t : (1u << prev.t);
                    if (prev_gate && !(pmask & (1u << o.t)) && ((prev.kind & KF_BUNDLE) || npool + 4 * RW <= kPassPool)) {
                        if (!(prev.kind & KF_BUNDLE)) {
                            prev.ref = std::uint16_t(npool);
                            npool += 4 * RW;
                            for (int k = 0; k < 4; ++k) P.pool[prev.ref + 4 * prev.t + k] = prev.c[k];
                            prev.kind = std::uint8_t(prev.kind | KF_BUNDLE);
                            prev.t = std::uint8_t(1u << prev.t);
                        }
                        for (int k = 0; k < 4; ++k) P.pool[prev.ref + 4 * o.t + k] = o.c[k];
                        prev.t = std::uint8_t(prev.t | (1u << o.t));
                        continue;
                    }
                }
                P.ops[nops++] = o;
            }
            if (!tab.empty()) {
                if (nops >= kPassMaxOps) raise(QCS_ERR_SIM, "internal: too many operations in a pass");
                RegOp o{};
                o.kind = TOP_DTAB;
                o.ref = std::uint16_t(npool);
                for (int q = 0; q < RG; ++q) {
                    cplx t(1.0, 0.0);
                    for (int idx : tab) {
                        const FOp& f = at(idx);
                        int g = 0;
                        for (int i = 0; i < f.dk; ++i) g |= ((q >> reg(f.dpos[i])) & 1) << (f.dk - 1 - i);
                        if (!f.dskip[g]) t *= cplx(f.dval[g].x, f.dval[g].y);
                    }
                    P.pool[npool + q] = make_double2(t.real(), t.imag());
                    if (t == cplx(1.0, 0.0)) {
                        if (q < 8) o.dskip = std::uint8_t(o.dskip | (1u << q));
                        o.smask |= 1u << q;  // the skip mask of all RG entries (16-register rounds)
                    }
                }
                npool += RG;
                P.ops[nops++] = o;
            }
            for (int idx : trailing) perm_op(at(idx));
            rd.op_count = std::uint16_t(nops - rd.op_begin);
            if (pending_signs) rd.flags = std::uint8_t(rd.flags | RD_SIGNS);
        }
        };
        {
            std::vector<FOp> sched_ops;
            std::vector<int> sched_list;
            // passes whose X-like gates become virtual relabellings keep their order: the
            // relabellings need no register bits, and the scheduler's round count would not see that
            bool perms = false;
            if (virt_pass)
                for (int idx : lists[pi]) perms |= is_perm(ops[std::size_t(idx)]);
            if (!has_alt[pi] && !perms && schedule_rounds(n, loc, P.m, ops, lists[pi], sched_ops, sched_list, RW))
                lower_list(sched_ops, sched_list);
            else
                lower_list(ops, lists[pi]);
        }
        // tiles that no sign step's listed indices reach see every sign step as a scalar +-1;
        // there the pass often collapses (H_b H_b = 2 I for the unnormalised butterflies), so
        // such passes carry a second, simplified program for those tiles
        if (has_alt[pi]) {
            const std::vector<FOp>& alt = alts[pi];
            if (alt.empty()) {
                P.alt_mode = ALT_SKIP;
            } else if (nops + int(alt.size()) < kPassMaxOps && P.nrounds + int(alt.size()) < kPassMaxOps) {
                std::vector<int> idx(alt.size());
                for (std::size_t i = 0; i < alt.size(); ++i) idx[i] = int(i);
                P.alt_begin = std::uint16_t(P.nrounds);
                lower_list(alt, idx);
                P.alt_nrounds = std::uint16_t(P.nrounds - P.alt_begin);
                P.nrounds = P.alt_begin;  // the main program's rounds; the alternative follows
                P.alt_mode = ALT_ROUNDS;
            }
        }
        // the basis offset of each run of 8 (tile bits 3..m-1), copied into shared memory per tile
        for (int b = 0; b < n;) {  // runs of bits outside the tile
            if (pp.tile >> b & 1) {
                ++b;
                continue;
            }
            int e = b;
            while (e < n && !(pp.tile >> e & 1)) ++e;
            P.run_pos[P.nruns] = std::uint8_t(b);
            P.run_len[P.nruns++] = std::uint8_t(e - b);
            b = e;
        }
        if (out.tables.size() & 1) out.tables.push_back(0);  // 16-byte aligned (cp.async)
        P.hi_off = std::uint32_t(out.tables.size());
        for (unsigned k = 0; k < (1u << (P.m - 3)); ++k) {
            u64 v = 0;
            for (int b = 3; b < P.m; ++b)
                if (k >> (b - 3) & 1) v |= u64(1) << P.bits[b];
            out.tables.push_back(v);
        }
        if (P.alt_mode == ALT_SKIP) {  // launch only the tiles a sign step reaches
            std::vector<u64> hit;
            for (int idx : lists[pi]) {
                const FOp& f = ops[std::size_t(idx)];
                if (f.kind != TOP_SIGN) continue;
                for (u64 e : f.flips) {
                    u64 tile = 0;  // e's bits outside the tile, compressed
                    for (int b = 0, k = 0; b < n; ++b)
                        if (!(pp.tile >> b & 1)) tile |= ((e >> b) & 1) << k++;
                    hit.push_back(tile);
                }
            }
            std::sort(hit.begin(), hit.end());
            hit.erase(std::unique(hit.begin(), hit.end()), hit.end());
            const u64 ntiles = u64(1) << (n - P.m);
            if (!hit.empty() && hit.size() <= ntiles / 4) {
                P.list_off = std::uint32_t(out.tables.size());
                P.list_cnt = std::uint32_t(hit.size());
                out.tables.insert(out.tables.end(), hit.begin(), hit.end());
            }
        }
        if (!forced[pi].empty()) {  // one of a pass pair around a skip pass: only the tiles it reaches
            if (out.tables.size() & 1) out.tables.push_back(0);
            P.list_off = std::uint32_t(out.tables.size());
            P.list_cnt = std::uint32_t(forced[pi].size());
            out.tables.insert(out.tables.end(), forced[pi].begin(), forced[pi].end());
        }
        P.nops = nops;
        if (jit_pivot(n, P)) {
            pivot_pass(P, npool);
            normalize_tables(P);
        }
        out.passes.push_back(P);
        out.pass_ops.push_back(lists[pi]);
        out.single_flip_off.push_back(flip_off);
        out.single_flip_cnt.push_back(flip_cnt);
    }
}

void dump_pass(std::FILE* f, const PassParams& p, std::size_t nsrc) {
    std::fprintf(f, "pass m=%d src_ops=%zu rounds=%d ops=%d alt=%d list=%u bits=", p.m, nsrc, p.nrounds, p.nops,
                 int(p.alt_mode), p.list_cnt);
    for (int b = 0; b < p.m; ++b) std::fprintf(f, "%d%s", p.bits[b], b + 1 < p.m ? "," : "\n");
    if (nsrc == 1) return;
    const int nr = p.alt_mode == ALT_ROUNDS ? p.alt_begin + p.alt_nrounds : p.nrounds;
    for (int r = 0; r < nr; ++r) {
        const RoundDesc& R = p.rounds[r];
        std::fprintf(f, "  round%s%s regs=%d,%d,%d", (R.flags & RD_SMEM) ? " smem" : "", r >= p.nrounds ? " alt" : "",
                     R.r[0], R.r[1], R.r[2]);
        if (R.flags & RD_W4) std::fprintf(f, ",%d", round_reg(R, 3));
        std::fprintf(f, ":");
        for (int i = R.op_begin; i < R.op_begin + R.op_count; ++i) {
            const RegOp& o = p.ops[i];
            static const char* names[] = {"G", "D", "SIGN", "WHT", "SC", "DTAB", "PERM"};
            const int k = o.kind & KF_KIND;
            std::fprintf(f, " %s%s%s%s%s%s", k <= 6 ? names[k] : "?", (o.kind & KF_BUNDLE) ? "b" : "",
                         (o.kind & KF_SIGNED) ? "s" : "", (o.kind & KF_GCTRL) ? "g" : "", (o.kind & KF_FLUSH) ? "f" : "", (o.kind & KF_REAL) ? "r" : "");
            if (k == TOP_GATE || k == TOP_WHT) std::fprintf(f, "[t%d%s]", o.t, o.lctrl_mask ? " c" : "");
            if (k == TOP_DIAG) std::fprintf(f, "[dk%d r%d,%d]", o.dk, o.dreg[0] == 0xff ? -1 : o.dreg[0],
                                            o.dk > 1 ? (o.dreg[1] == 0xff ? -1 : o.dreg[1]) : -2);
        }
        std::fprintf(f, "\n");
    }
}

}  // namespace qcs
