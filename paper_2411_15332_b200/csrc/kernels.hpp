// kernels.hpp -- POD descriptors shared by host planning code and the sm_100a kernels, and
// the launch entry points of every kernel in this library.
#pragma once

#ifdef __CUDACC_RTC__  // NVRTC build of the per-pass specialised kernels (jit.cpp): no host headers
namespace std {
typedef unsigned char uint8_t;
typedef unsigned short uint16_t;
typedef unsigned int uint32_t;
typedef unsigned long uint64_t;
typedef int int32_t;
typedef unsigned long size_t;
}  // namespace std
typedef struct CUstream_st* cudaStream_t;
#else
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#endif

namespace qcs {

// ---------------------------------------------------------------- single-placement gate pass
// One canonical placement of arity k <= 3, reduced to the sub-cube of the state it touches.
// "Members" are the 2^nfree amplitudes of one group; free bit i of the member index selects
// free_bit[i] of the basis index.  Only `rows` (non-identity rows of the gate) are written;
// each row accumulates its nonzeros in ascending global column order from (0,0) with
// separately rounded multiply/add, i.e. exactly dax_mvm's per-row sum (dax.cpp:101).
struct GateDesc {
    int k;                    // gate bits (zero-inserted when enumerating groups)
    int nfree;                // enumerated bits per group (0..3)
    int nrows;                // rows written per group (<= 8)
    int pos_asc[3];           // gate bit positions, ascending (zero insertion order)
    std::uint64_t fixed_val;  // gate bits that are constant over the touched sub-cube
    std::uint64_t free_bit[3];
    std::uint64_t member_off[8];  // basis-index offset of each member (sum of its free bits)
    std::uint32_t load_mask;  // members that must be loaded
    std::uint8_t row_member[8];
    std::uint8_t nnz[8];
    std::uint8_t col_member[8][8];
    std::uint8_t vkind[8][8];     // coefficient kind: 0 complex, 1 real, 2 imaginary
    double2 val[8][8];
};

// Kernel classes chosen by the host from the descriptor (for launch shape / specialisation).
void launch_gate(double2* amps, int n, const GateDesc& d, cudaStream_t st);

// ---------------------------------------------------------------- the Matrix method (dense engine)
// step_matrix_dense's factors in fold order (most significant qubit first): factor f covers
// arity[f] index bits, its 2^k x 2^k row-major entries at mat[offset[f]].
struct DenseFold {
    int nfactors;
    int arity[32];
    int offset[32];
    double2 mat[512];
};
void dense_build(double2* m, int n, const DenseFold& fold, cudaStream_t st);
void dense_diag(double2* m, int n, const std::uint64_t* flipped_dev, std::uint64_t nf, int rest, cudaStream_t st);
void dense_mvm(const double2* m, const double2* x, double2* out, int n, cudaStream_t st);

// ---------------------------------------------------------------- diagonal sign step
// negate amplitudes whose index is (listed XOR flip_rest); `flipped` is a sorted device array.
void launch_diag_sign(double2* amps, int n, const std::uint64_t* flipped_dev, std::uint64_t nflip,
                      int flip_rest, cudaStream_t st);
// few listed indices, flip_rest = 0: touch only those amplitudes
void launch_negate_listed(double2* amps, const std::uint64_t* idx_dev, std::uint64_t count,
                          cudaStream_t st);

// ---------------------------------------------------------------- fused shared-memory passes
// A pass loads the 2^m amplitudes whose basis indices differ only in the tile bits, runs
// rounds of operations on register-held groups of 8 amplitudes, and writes the tile back:
// one HBM round trip for many gates (tile_kernels.cu).
enum TileOpKind : std::int32_t {
    TOP_GATE = 0,    // gate on <= 3 targets among the round bits (row tables as GateDesc)
    TOP_DIAG = 1,    // diagonal phase on up to 3 basis bits anywhere
    TOP_SIGN = 2,    // diag sign step: flipped list (global memory) XOR flip_rest
    TOP_WHT = 3,     // unnormalised butterflies (a+b, a-b) over round bits (wht_mask)
    TOP_SCALE = 4,   // multiply by a real scalar (the RH magnitude, rh.cpp:99-100)
    TOP_PERM = 6,    // specialised kernels only: a virtual X-like gate (target local bit t, at most one
                     // control in lctrl): leading ops of a round relabel its loads, trailing ops of the
                     // last round its stores
    TOP_DTAB = 5,    // register round: diagonal given per register, pool[ref + q] (q = 0..7); dskip bit q
                     // = entry q is exactly 1 (the round's diagonals on its register bits, combined)
};

struct TileOp {
    std::int32_t kind;
    std::int32_t gcase;          // TOP_GATE: register round: target register bit (K = 1);
                                 //           shared-memory round: K (2 or 3)
    std::int32_t tl[3];          // TOP_GATE shared-memory round: target local bits, most significant first
    std::int32_t nrows;          // TOP_GATE: touched rows
    std::uint32_t lctrl_mask;    // controls on tile bits (local index mask / required value)
    std::uint32_t lctrl_val;
    std::uint32_t wht_mask;      // TOP_WHT: register bits 0..2 to transform
    std::uint64_t gctrl_mask;    // controls outside the tile: required basis bits
    std::uint64_t gctrl_val;
    std::int32_t dk;             // TOP_DIAG: number of phase bits
    std::int32_t dpos[3];        // TOP_DIAG: basis-bit positions, most significant first
    std::uint64_t flip_off;      // TOP_SIGN: offset into the plan's flipped array
    std::uint64_t flip_cnt;
    std::int32_t flip_rest;
    double scale;                // TOP_SCALE
    std::uint8_t row_member[8];  // TOP_GATE: member index (gate-local) of each touched row
    std::uint8_t nnz[8];
    std::uint8_t col_member[8][8];
    double2 val[8][8];           // TOP_GATE rows / TOP_DIAG: val[0][g] = diagonal entry g
    std::uint8_t dskip[8];       // TOP_DIAG: entry g is exactly 1 (left untouched)
};

// RegOp::kind flags above the kind bits
constexpr int KF_KIND = 0x07;
constexpr int KF_REAL = 0x08;    // TOP_GATE (bundled or not): every coefficient is real (c[k].y == 0)
// KF_BUNDLE on a +-1 diagonal (KF_SIGNED): a run of them; smask low byte = the flips of the ones
// with no group-constant bit, pool[ref .. ref + t) = SignEntry for the others
struct SignEntry {
    std::uint32_t smask;      // byte cg = registers that flip when the constant bits spell cg
    std::uint8_t dk, p0, p1;  // phase bits; basis positions of the constant ones
    std::uint8_t cmask;       // bit 0: phase bit 0 is constant over a group, bit 1: phase bit 1
    std::uint64_t pad;
};
static_assert(sizeof(SignEntry) == 16, "one pool slot");
constexpr int KF_BUNDLE = 0x10;  // TOP_GATE: dense gates on the register bits of mask t, coefficients
                                 // in PassParams::pool[ref + 4 * bit] (m00 m01 m10 m11 per bit)
constexpr int KF_FLUSH = 0x20;   // apply the pending +-1 sign flips before this op (set by the planner)
constexpr int KF_SIGNED = 0x40;  // TOP_DIAG with entries in {+1, -1}: dskip holds the -1 entries
constexpr int KF_GCTRL = 0x80;   // has controls outside the tile (gctrl_mask / gctrl_val)
// KF_PIVOT on TOP_GATE (the KF_SIGNED bit; that one is TOP_DIAG-only): pivoted form, specialised
// kernels only.  Per target bit b (single gates: b = 0 in the fields), output row r is
// x[piv] + rho_r * x[other], with rho_r in coefficient slot r (c[r] / pool[ref + 4b + r]); dtab
// bits 4b..4b+3 = piv_0, piv_1 (1: the row's pivot is input 1), zero_0, zero_1 (rho_r == 0).  The
// rows' scales were folded into the round's diagonal table (TOP_DTAB).
constexpr int KF_PIVOT = KF_SIGNED;

// Compact register-round operation; a pass's list travels in the kernel parameter space.
struct RegOp {
    std::uint8_t kind;        // TOP_GATE (one target), TOP_DIAG, TOP_SIGN, TOP_WHT, TOP_SCALE | KF_* flags
    std::uint8_t t;           // TOP_GATE: target register bit; TOP_WHT: register-bit mask
    std::uint8_t dk;          // TOP_DIAG: phase bits (<= 3)
    std::uint8_t dskip;       // TOP_DIAG: bit g set = entry g is exactly 1 (untouched)
    std::uint8_t dreg[3];     // TOP_DIAG: register bit of phase bit i, 0xff = constant over a group
    std::uint8_t dpos[3];     // TOP_DIAG: basis-bit position of phase bit i (most significant first)
    std::uint16_t ref;        // TOP_SIGN / shared-memory gates / 3-bit diagonals: index into the plan's TileOp array
    std::uint32_t lctrl_mask; // controls on tile bits (local-index mask / required value)
    std::uint32_t lctrl_val;
    std::uint32_t sidx;       // TOP_SIGN: index among the pass's sign steps
    std::uint64_t gctrl_mask; // controls outside the tile (basis bits / required value)
    std::uint64_t gctrl_val;
    std::uint16_t dtab;       // TOP_DIAG (dk <= 2): register part of the entry index for q = 0..7, 2 bits each
    std::uint32_t smask;      // KF_SIGNED: byte cg = registers q that flip when the constant bits spell cg
    double2 c[4];             // TOP_GATE: the 2x2 matrix m00, m01, m10, m11; TOP_DIAG: entries; TOP_SCALE: c[0].x
};

constexpr int RD_SMEM = 1;    // gates on 2-3 targets, run straight on shared memory
constexpr int RD_SIGNS = 2;   // register round ending with pending +-1 sign flips
constexpr int RD_W4 = 4;      // specialised kernels only: 4 register bits (16 amplitudes per group),
                              // the fourth local bit in flags bits 4..7
struct RoundDesc {
    std::uint8_t flags;       // RD_* (bits 4..7: the fourth register bit of an RD_W4 round)
    std::uint8_t r[3];        // local tile bits held in registers (ascending)
    std::uint16_t op_begin, op_count;
};
// register bits of a round and their local tile bits (r[3] lives in the flags byte)
inline constexpr int round_width(const RoundDesc& R) { return (R.flags & RD_W4) ? 4 : 3; }
inline constexpr int round_reg(const RoundDesc& R, int i) { return i < 3 ? int(R.r[i]) : int(R.flags >> 4); }

#ifndef __CUDACC_RTC__  // host-side planning helpers
// The TMA tensor-map layout of a tile: its bit set S over an n-bit state (bits 0..2 included).
// Dim 0 is the tile's 8 contiguous amplitudes (16 doubles); every further dim is a run of <= 8
// tile bits starting at state bit `pos`.  The state bits above a run, up to the next tile bit,
// ride in the same dim as the high bits of its coordinate (extent 2^len, box 2^inlen), so only
// the tile's own runs cost dims; a gap too wide for a 31-bit coordinate gets dims of its own
// (inlen 0, box 1).  Coordinates: (base >> pos) & (2^len - 1), shifted left once for dim 0
// (whose unit is one double).  Returns the rank; `out` (16 entries, may be null) receives the dims.
// gap_dims = true: the round-1 layout, one dim per gap as well (A/B: QCS_TMA_GAP_DIMS=1).
struct TmaDim {
    int pos, len, inlen;
};
inline int tma_layout(std::uint64_t S, int n, TmaDim* out, bool gap_dims) {
    if ((S & 7u) != 7u) return 99;
    int rank = 0;
    auto push = [&](int pos, int len, int inlen) {
        if (out && rank < 16) out[rank] = TmaDim{pos, len, inlen};
        ++rank;
    };
    auto gap = [&](int from, int to) {  // dims of their own over state bits [from, to)
        for (int c = from; c < to; c += 31) push(c, to - c < 31 ? to - c : 31, 0);
    };
    int b = 3;
    while (b < n && !(S >> b & 1)) ++b;
    if (gap_dims || b > 30) {
        push(0, 3, 3);
        gap(3, b);
    } else {
        push(0, b, 3);
    }
    while (b < n) {
        int e = b, g;
        while (e < n && (S >> e & 1)) ++e;  // tile bits [b, e)
        for (g = e; g < n && !(S >> g & 1);) ++g;  // the gap [e, g) above them
        for (int c = b; c < e;) {
            const int len = e - c < 8 ? e - c : 8;
            if (c + len < e) {
                push(c, len, len);
            } else if (gap_dims || len + (g - e) > 31) {
                push(c, len, len);
                gap(e, g);
            } else {
                push(c, len + (g - e), len);
            }
            c += len;
        }
        b = g;
    }
    return rank;
}
inline bool tma_gap_dims() {
    static const bool on = [] { const char* v = std::getenv("QCS_TMA_GAP_DIMS"); return v && std::atoi(v) != 0; }();
    return on;
}
#endif

#ifndef QCS_PASS_MAX_OPS
#define QCS_PASS_MAX_OPS 200
#endif
constexpr int kPassMaxOps = QCS_PASS_MAX_OPS;
#ifndef QCS_PASS_POOL
#define QCS_PASS_POOL 512
#endif
constexpr int kPassPool = QCS_PASS_POOL;    // double2 slots for gate bundles (12 per bundle)
enum : std::uint8_t { ALT_NONE = 0, ALT_ROUNDS = 1, ALT_SKIP = 2 };
struct PassParams {           // <= 32 KB: the kernel parameter limit
    int m;                    // tile bits (3..12)
    int nrounds;
    int nops;
    int bits[16];             // basis-bit positions, ascending; bits[0..2] = 0, 1, 2
    // tiles that no sign step's listed index reaches (sign_hit == 0) run the alternative:
    // ALT_ROUNDS: rounds [alt_begin, alt_begin + alt_nrounds); ALT_SKIP: nothing (identity)
    std::uint8_t alt_mode;
    std::uint16_t alt_begin, alt_nrounds;
    std::uint32_t hi_off;     // this pass's table of run offsets (tile bits 3..m-1) in the plan's tables
    int tma_rank;             // > 0: the tile moves as TMA boxes of this rank (set at launch)
    std::uint8_t tma_iter;    // the top tma_iter local tile bits are iterated: 2^tma_iter boxes per tile
    std::uint8_t tma_gap_pos[5], tma_gap_len[5];  // per dim: the state bits its coordinate spans (tma_layout)
    int nruns;                // the basis bits outside the tile, as runs: a tile index deposits into them
    std::uint8_t run_pos[16], run_len[16];
    std::uint32_t list_off, list_cnt;  // list_cnt > 0: run only these tiles (ALT_SKIP passes)
    std::uint32_t init;       // 1: the pass starts from the basis state |init_index> instead of loading
    std::uint64_t init_index;
    std::uint64_t zmask, zval;  // tiles whose base bits under zmask differ from zval hold only zeros
                                // (outside the support the circuit has reached): nothing to load
    std::uint64_t smask, sval;  // tiles whose base bits under smask differ from sval are skipped: zero
                                // and read as zero by the next pass (its zmask), nothing to write
    std::uint64_t base_or;      // OR-ed into every tile's base: a launch that enumerates only the
                                // tiles smask keeps (its runs leave the smask bits out) sets sval here
    RoundDesc rounds[kPassMaxOps];
    RegOp ops[kPassMaxOps];
    double2 pool[kPassPool];
};
// the kernel's parameters: PassParams, four pointers and a 128-byte tensor map in 32764 bytes
static_assert(sizeof(PassParams) + 4 * 8 + 128 + 64 <= 32764, "kernel parameter space");

// The pass's TMA tensor map (a CUtensorMap, cuda.h) as opaque kernel-parameter bytes
struct alignas(64) TmapParam {
    unsigned long long w[16];
};

#ifndef __CUDACC_RTC__
// The pass as a kernel specialised to its operation list (jit.cpp); false when the pass is not
// worth a compile (or QCS_JIT=0), and the interpreter k_tile runs it.
bool launch_tile_pass_jit(double2* amps, const struct PassParams& p, unsigned F, const struct TileOp* big_dev,
                          const std::uint64_t* flipped_dev, const std::uint64_t* tables_dev, const TmapParam& tmap,
                          unsigned tiles, unsigned threads, std::size_t smem, std::size_t smem_max, cudaStream_t st,
                          void** jit_slot = nullptr);
double pass_fp64_per_tile(const struct PassParams& p);  // FP64 instructions per tile, specialised form (jit.cpp)
int jit_mode();                      // 0 off, 1 passes with enough work (default), 2 every tile pass, 3 = 2 + pivots
bool jit_pivot(int n, const struct PassParams& p);  // lower this pass's gates to the pivoted form
bool jit_virtual(int n, int m, bool skip_pass);      // lower this pass's X-like gates to relabellings
void set_jit_mode(int mode);
// persistent pipelined pass kernels (jit.cpp): 0 off, 1 passes with 16-register rounds (default), 2 every eligible pass
int pipeline_mode();
void set_pipeline_mode(int mode);
// NVRTC only (no device): cubin bytes; verify_only: generate with the addressing proof, no compile
std::size_t jit_compile_only(const struct PassParams& p, bool verify_only = false);
void tile_pass_shape(const struct PassParams& p, unsigned& F, unsigned& threads);  // kernel variant, CTA size
// host only: how many of the tile's top local bits its TMA boxes iterate (tile_tensor_map's
// choice), or -1 when the tile does not move as TMA boxes
int tile_tma_iter(int n, const struct PassParams& p);
unsigned long long jit_compiles();   // pass kernels compiled so far
#endif

// tables_dev: the plan's u64 tables (Lowered::tables): run offsets and tile lists
// sets p.tma_* for the launch
// jit_slot (optional): the pass's specialised kernel, found once and kept by the caller's plan
void launch_tile_pass(double2* amps, int n, PassParams& p, const TileOp* big_dev,
                      const std::uint64_t* flipped_dev, const std::uint64_t* tables_dev, cudaStream_t st,
                      void** jit_slot = nullptr);
int tile_max_bits();

// A gate on a shard-global qubit over peer memory (peer_kernels.cu): blocks v (selected by the
// local bits sel[0..nsel-1], most significant first) are 2x2 matrices m00 m01 m10 m11 on the
// global qubit; skip bit v = block v is the identity.
struct SplitParams {
    int nl;          // local qubits of the shard
    int self_bit;    // this rank's value of the global qubit
    int nsel;        // <= 2
    int sel[2];      // local basis-bit positions selecting the block
    unsigned skip;
    unsigned char nz[4];  // bit k: entry k of block v is nonzero
    double2 m[4][4];
};
void launch_swap_peer(double2* self, double2* peer, std::uint64_t count, cudaStream_t st);
void launch_split_pair(double2* self, double2* peer, const SplitParams& p, cudaStream_t st);

// ---------------------------------------------------------------- reductions
double reduce_norm2(const double2* amps, int n, double* scratch_dev, cudaStream_t st);
void probabilities(const double2* amps, std::uint64_t dim, double* out_dev, cudaStream_t st);
// max |a_i - b_i| and the L2 norm of a - b (synchronises st)
void distance(const double2* a, const double2* b, std::uint64_t dim, double* max_abs, double* l2,
              cudaStream_t st);
void argmax(const double2* amps, std::uint64_t dim, std::uint64_t* idx, double* p, void* scratch_dev,
            cudaStream_t st);
// k <= 16 largest probabilities, descending, ties to the lower index; norm (optional): the
// state's norm from the same pass (sqrt of the summed probabilities)
std::size_t topk_host_bytes(int k);
void topk_begin(const double2* amps, std::uint64_t dim, int k, bool with_norm, void* host, cudaStream_t st);
void topk_finish(const void* host, int k, bool with_norm, std::uint64_t* idx, double* p, double* norm);
void topk(const double2* amps, std::uint64_t dim, int k, std::uint64_t* idx, double* p, cudaStream_t st,
          double* norm = nullptr);
// seeded sampling with the reference's sequential CDF (sample_kernels.cu)
void sample(const double2* amps, std::uint64_t dim, std::uint64_t seed, std::uint64_t count, std::uint64_t* out,
            double* total, cudaStream_t st);
void gather(const double2* amps, const std::uint64_t* idx_dev, std::uint64_t count, double2* out_dev,
            cudaStream_t st);
void scale(double2* amps, std::uint64_t dim, double s, cudaStream_t st);
void fill_basis(double2* amps, std::uint64_t dim, std::uint64_t index, cudaStream_t st);
void fill_random(double2* amps, std::uint64_t dim, std::uint64_t seed, cudaStream_t st);

// ---------------------------------------------------------------- DAX / DAS encoder
// One step in the reference's left-fold order (engine.cpp:31-52, dax.cpp:58-94).
struct EncodePlacement {
    int k;
    int pos[3];               // basis-bit positions in gate-local order (local bit k-1-i <-> pos[i])
    int nnz[8];
    int col[8][8];            // nonzero local columns of each local row, ascending local column
    double2 val[8][8];
};
struct EncodeStep {
    int n;
    int np;
    int sorted;               // enumeration order yields ascending columns (no per-row sort)
    int order[64];            // placements in enumeration order
    int nfold;
    int fold_gate[64];        // fold items in position order: placement index, or -1 = identity
    std::uint64_t gate_mask;
    EncodePlacement p[64];
};
// Materialise one step (DAX rows/cols/vals, or the DAS stream when das = true) on the device.
// Returns the entry count; writes outputs only when it does not exceed capacity.
std::uint64_t encode_step(const EncodeStep& st, bool das, std::uint64_t capacity, std::uint64_t* rows,
                          std::uint64_t* cols, double2* vals, std::uint64_t* dis, std::uint8_t* last,
                          bool out_on_device, cudaStream_t s);
// dax_mvm from row-sorted entries
void dax_mvm(const std::uint64_t* rows, const std::uint64_t* cols, const double2* vals, std::uint64_t count,
             const double2* in, double2* out, std::uint64_t dim, int* err_dev, cudaStream_t s);
void das_mvm(const std::uint64_t* dis, const std::uint8_t* last, const double2* vals, std::uint64_t count,
             const double2* in, double2* out, std::uint64_t dim, int* err_dev, cudaStream_t s);

}  // namespace qcs
