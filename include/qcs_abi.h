/*
 * qcs_abi.h -- C ABI of the B200 state-vector engine (libqcs_b200.so).
 *
 * The reference (arXiv 2411.15332, /root/reference/proj) has no FFI: its hot path is a set of
 * free C++ functions in namespace qcsim.  Each entry point below replaces one of them; the
 * comment names the reference declaration (path:line under proj/).  Plain pointers and sizes
 * only: no torch or C++ types cross this boundary.
 *
 * Conventions
 *  - Complex numbers are interleaved (re, im) doubles, the byte layout of
 *    std::complex<double>; a state of n qubits is 2*2^n doubles (core.hpp:66-76).
 *  - Qubit q is bit (n-1-q) of the basis index: qubit 0 is the most significant bit
 *    (core.hpp:64-66).
 *  - A placement lists its qubits in gate-local order: local index bit (arity-1-i) is
 *    qubits[i].  Contiguous ascending lists are the reference's own placements
 *    (circuit.hpp:10-15); any other distinct list is accepted as well (a superset).
 *  - Every function returns QCS_OK or an error code mirroring the reference's exception
 *    hierarchy (core.hpp:13-36); qcs_last_error() gives the message (thread-local).  The
 *    library never falls back to the CPU: without a CUDA device calls fail with QCS_ERR_CUDA.
 *  - Calls on one state are asynchronous on that state's stream unless they return host data;
 *    qcs_state_sync surfaces deferred CUDA errors.  One state must not be used from two threads
 *    at once; distinct states may (the reference is reentrant).
 */
#ifndef QCS_ABI_H
#define QCS_ABI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QCS_MAX_ARITY 3 /* largest catalog gate (CCX, CSwap), gates.cpp:193-194 */

/* status codes -- SimError (core.hpp:13-16) and its subclasses (core.hpp:18-36) */
enum {
    QCS_OK = 0,
    QCS_ERR_CAPACITY = 1,  /* CapacityError  (core.hpp:18-21) */
    QCS_ERR_DIMENSION = 2, /* DimensionError (core.hpp:23-26) */
    QCS_ERR_ENCODING = 3,  /* EncodingError  (core.hpp:28-31) */
    QCS_ERR_PARSE = 4,     /* ParseError     (core.hpp:33-36) */
    QCS_ERR_SIM = 5,       /* SimError       (core.hpp:13-16) */
    QCS_ERR_CUDA = 6,      /* device failure or no device */
    QCS_ERR_NCCL = 7,      /* collective failure */
    QCS_ERR_ARG = 8        /* null pointer / malformed argument */
};

/* engines and sign methods -- engine.hpp:10, rh.hpp:22 */
enum { QCS_ENGINE_DENSE = 0, QCS_ENGINE_DAX = 1, QCS_ENGINE_DAS = 2, QCS_ENGINE_RH_DAX = 3 };
enum { QCS_SIGN_NONOPT = 0, QCS_SIGN_QUARTER = 1, QCS_SIGN_BLOCK = 2, QCS_SIGN_LOGARITHM = 3 };
enum { QCS_STEP_GATES = 0, QCS_STEP_DIAG = 1 };               /* CircuitStep::Kind, circuit.hpp:30 */
enum { QCS_STRUCT_DENSE = 0, QCS_STRUCT_DAX = 1, QCS_STRUCT_DAS = 2, QCS_STRUCT_RH = 3 };
enum { QCS_MEM_HOST = 0, QCS_MEM_DEVICE = 1 };

const char* qcs_last_error(void);
const char* qcs_version(void);
int qcs_device_count(int* count);

/* dense_cap / set_dense_cap (core.hpp:38-43): element cap of the Matrix (dense) engine,
 * default 2^26; QCS_ENGINE_DENSE raises QCS_ERR_CAPACITY where the reference would. */
int qcs_set_dense_cap(uint64_t cap);
uint64_t qcs_dense_cap(void);

/* ------------------------------------------------------------------ gate catalog
 * gates.hpp:29 gate_catalog, :31 gate_known, :36 gate_catalog_lookup, :41 canonical_params.
 * Matrices are computed on the host exactly as the reference computes them, so the device
 * receives identical bytes. */
int qcs_gate_catalog_size(void);
int qcs_gate_catalog_entry(int index, const char** name, int* arity, int* param_count,
                           double* zero_ratio);
int qcs_gate_lookup(const char* name, const double* params, int num_params,
                    double* matrix_out /* 2*4^arity doubles, capacity 2*64 */, int* arity_out,
                    const char** canonical_name);
int qcs_canonical_params(const char* name, double* out /* capacity 4 */, int* count);

/* ------------------------------------------------------------------ device state
 * StateVector (core.hpp:64-76), held in HBM as 2^n x 16 B. */
typedef struct qcs_state qcs_state;

/* StateVector(n, basis_index), core.cpp:22-28: 1 <= n <= 62, basis_index < 2^n. */
int qcs_state_create(int n, int device, uint64_t basis_index, qcs_state** out);
/* Borrow caller-owned device memory (2^n x 16 B on `device`) and a CUDA stream (NULL = the
 * legacy default stream).  The handle never frees borrowed memory. */
int qcs_state_wrap(int n, int device, void* device_amps, void* cuda_stream, qcs_state** out);
int qcs_state_destroy(qcs_state* s);
int qcs_state_info(const qcs_state* s, int* n, int* device, void** device_amps, void** stream);
int qcs_state_set_basis(qcs_state* s, uint64_t basis_index);
/* Copy amplitudes [first, first+count) from / to host memory (pinned memory is fastest). */
int qcs_state_upload(qcs_state* s, const double* host, uint64_t first, uint64_t count);
int qcs_state_download(qcs_state* s, double* host, uint64_t first, uint64_t count);
/* The same read-back enqueued on the state's stream without waiting: `host` must be pinned
 * (qcs_host_alloc) and is complete after qcs_state_sync.  Lets a caller keep several states
 * (requests) in flight, as bench.py's end-to-end arm does. */
int qcs_state_download_async(qcs_state* s, double* host, uint64_t first, uint64_t count);
int qcs_state_copy(qcs_state* dst, const qcs_state* src);
/* Order: work enqueued on `s` from now on starts only after everything enqueued on `other` so
 * far has finished (an event on other's stream, waited on by s's stream; the host does not
 * block).  A serving loop keeps its requests' sweeps back to back on the device while their
 * PCIe copies overlap (bench.py's end-to-end arm). */
int qcs_state_wait(qcs_state* s, const qcs_state* other);
int qcs_state_sync(qcs_state* s);
/* Seeded i.i.d. Gaussian re/im, L2-normalised (a synthetic-input generator on the device). */
int qcs_state_random(qcs_state* s, uint64_t seed);

/* Pinned host buffers for fast transfers (cudaHostAlloc / cudaFreeHost). */
int qcs_host_alloc(size_t bytes, void** out);
int qcs_host_free(void* p);

/* ------------------------------------------------------------------ one step at a time */
typedef struct {
    int arity;            /* 1..QCS_MAX_ARITY */
    const int* qubits;    /* arity distinct reference qubit indices, gate-local order */
    const double* matrix; /* row-major 2^arity x 2^arity, interleaved (re, im) */
    const char* name;     /* catalog name or NULL; used for the RH dispatch and reports */
} qcs_placement;

/* One gates step: s <- step_matrix(placements) * s, computed without materialising the
 * operator.  Replaces step_matrix_dax (engine.hpp:38) + dax_mvm (dax.hpp:37) and
 * step_matrix_das (engine.hpp:39) + das_mvm (das.hpp:39): the results are identical.
 * Bit-exact with the reference for single-placement steps and for steps whose values
 * are all in {0, +-1, +-i}; otherwise within 1e-12 per amplitude. */
int qcs_apply_step(qcs_state* s, const qcs_placement* placements, int count);

/* One diagonal sign step (circuit.hpp:20-25, engine.cpp:62-80): negate the amplitudes whose
 * index is listed XOR flip_rest.  Bit-exact. */
int qcs_apply_diag(qcs_state* s, const uint64_t* flipped, uint64_t count, int flip_rest);

/* A one-qubit gate (optionally controlled by local qubits) on a shard-GLOBAL qubit of a state
 * sharded by its top qubits, computed straight over peer memory: `s` is this rank's shard,
 * `peer_amps` the partner shard (the rank differing in that global bit), mapped into this
 * device's address space (NVLink P2P; on one device, another buffer).  This rank takes the
 * pairs whose local top bit equals self_bit (its own value of the global qubit), loads the
 * partner amplitude, and stores both outputs.  Blocks: 2^num_sel matrices of 2x2 complex
 * (interleaved, row-major m00 m01 m10 m11) on the global qubit, block v selected by the local
 * basis bits sel_bits[0..num_sel-1] (most significant first); skip_mask bit v = block v is the
 * identity and is not touched.  dax_mvm arithmetic: bit-exact with the unsharded gate.
 * Both ranks call it for the same gate; the caller orders it after the partner's previous
 * work on its shard and before the partner's next (a barrier on each side).  B200-specific:
 * the reference has no multi-device code. */
int qcs_apply_split(qcs_state* s, void* peer_amps, int self_bit, int num_sel, const int* sel_bits,
                    const double* blocks, uint32_t skip_mask);

/* Swap the amplitudes [offset, offset+count) of this shard with `count` amplitudes of peer
 * memory at `peer_amps` (a partner shard mapped into this device's address space: NVLink P2P,
 * or another buffer on one device).  The data movement of a global<->local qubit remap of a
 * sharded state (partition.py): the two ranks of a pair each swap one half of their block pair,
 * so nothing is staged and every amplitude crosses the link once each way.  The caller orders
 * it after the partner's earlier work and before its later work (a barrier on each side).
 * B200-specific (the reference has no multi-device code). */
int qcs_swap_peer(qcs_state* s, uint64_t offset, void* peer_amps, uint64_t count);

/* rh_mvm(rh_build(n), s) (rh.hpp:64-66): H^{(x)n} as a Walsh-Hadamard butterfly, scaled once
 * by exp2(-n/2) (rh.cpp:20).  Within 1e-12 of the reference (whose own error is larger). */
int qcs_apply_rh(qcs_state* s);
/* rh_mvm(RhMatrix{n, value}, s, method, stats, block_size) (rh.hpp:64-66, rh.cpp:92-156) in place:
 * s <- value * H^(x)n s (scale first, then the butterflies).  sign_count / madd_count (optional)
 * receive RhMvmStats as the reference's counters total them (madd = 4 * (2^(n-1))^2; signs per
 * method, the Table-2 formulas).  Errors as the reference: n < 1 or n != the state's qubit count
 * -> QCS_ERR_DIMENSION; an invalid block size for QCS_SIGN_BLOCK -> QCS_ERR_SIM (rh.cpp:58). */
int qcs_rh_mvm(qcs_state* s, int n, double value, int sign_method, uint64_t block_size, uint64_t* sign_count,
               uint64_t* madd_count);

/* ------------------------------------------------------------------ reductions
 * StateVector::norm / probabilities (core.cpp:30-40). */
int qcs_norm(qcs_state* s, double* out);
/* probabilities into host memory (mem = QCS_MEM_HOST) or device memory (QCS_MEM_DEVICE),
 * 2^n doubles, bit-exact (re*re + im*im). */
int qcs_probabilities(qcs_state* s, double* out, int mem);
/* argmax of the probabilities, first index on ties (std::max_element, circuit_io.cpp:111-112) */
int qcs_argmax(qcs_state* s, uint64_t* index, double* probability);
/* k largest probabilities, descending, ties to the lower index (circuit_io.cpp:140-147) */
int qcs_topk(qcs_state* s, int k, uint64_t* indices, double* probabilities);
/* max_i |a_i - b_i| and ||a - b||_2 over two states of the same size on one device, reduced
 * on the device (no download).  Ordered after both states' pending work.  B200-specific: the
 * BASELINE-size parity tests compare the fused engine with its per-gate kernels this way. */
int qcs_state_distance(qcs_state* a, qcs_state* b, double* max_abs, double* l2);
/* What a report needs from a state in ONE pass over it: the norm (sqrt of the summed
 * probabilities, core.cpp:30-34) and the k <= 16 largest probabilities as qcs_topk gives them
 * (indices[0] is the argmax).  Host outputs; synchronous. */
int qcs_summary(qcs_state* s, int k, double* norm, uint64_t* indices, double* probabilities);
/* qcs_summary in two halves: _begin enqueues the pass and its read-back on the state's stream
 * and returns at once; _end waits for it and returns the same values.  Lets a serving loop
 * queue request i+1 while request i's summary is still on the device.  One pending per state. */
int qcs_summary_begin(qcs_state* s, int k);
int qcs_summary_end(qcs_state* s, double* norm, uint64_t* indices, double* probabilities);
/* render_report's seeded sampling (circuit_io.cpp:114-128), index-exact: std::mt19937_64(seed),
 * `count` draws of uniform_real_distribution<double>(0, acc), each the std::lower_bound of the
 * draw in the SEQUENTIAL rounded prefix sum of the probabilities (acc += p_i).  The device
 * reproduces that rounded chain exactly (binade-wise integer walk + serial replay of the chunks
 * where the sum changes binade, csrc/sample_kernels.cu) without moving 2^n values to the host.
 * out: host, count indices; total (optional): the final acc.  Synchronous. */
int qcs_sample(qcs_state* s, uint64_t seed, uint64_t count, uint64_t* out, double* total);
/* amplitudes at arbitrary indices (host index list, host output 2*count doubles) */
int qcs_gather(qcs_state* s, const uint64_t* indices, uint64_t count, double* out);

/* ------------------------------------------------------------------ whole circuits */
typedef struct {
    int kind;  /* QCS_STEP_GATES or QCS_STEP_DIAG */
    int stage; /* builder annotation, surfaces in reports (circuit.hpp:34) */
    const qcs_placement* placements;
    int num_placements;
    const uint64_t* flipped; /* diag steps; sorted or not */
    uint64_t num_flipped;
    int flip_rest;
} qcs_step;

typedef struct {
    int sign_method;     /* SimOptions::sign_method (engine.hpp:42); reports only */
    uint64_t block_size; /* SimOptions::block_size (engine.hpp:43); 0 = optimal */
    int fuse;            /* 0: one pass per step in circuit order (bit-exact per step);
                            1: fuse consecutive operations into shared-memory passes
                               (within 1e-12); default 1 */
    int reset;           /* 1: start from the basis state |initial> (Circuit::initial) instead of
                            the state's content -- folded into the first pass when that pass
                            sweeps every tile (no separate write of the state); 0 (default): as is */
    uint64_t initial;
} qcs_sim_options;

typedef struct {             /* StepReport, engine.hpp:16-24 */
    int structure;           /* QCS_STRUCT_* */
    int stage;
    uint64_t matrix_bytes;   /* accounting bytes of the structure (24 B / entry, RH 16 B) */
    uint64_t dense_bytes;    /* 2^{2n} * 16, saturating */
    uint64_t entry_count;    /* stored nonzeros (0 for RH) */
    uint64_t sign_count;
    uint64_t madd_count;
} qcs_step_report;

/* simulate(Circuit, Engine, SimOptions) (engine.hpp:46, engine.cpp:153-210) applied to the
 * state `s` in place, from its current content or (opts->reset) from |opts->initial>.
 * reports: num_steps entries or NULL.  Circuit::validate rules apply (circuit.cpp:41-62). */
int qcs_simulate(qcs_state* s, const qcs_step* steps, int num_steps, int engine,
                 const qcs_sim_options* opts, qcs_step_report* reports);

/* memory_report (engine.hpp:49, engine.cpp:212-234): accounting without a state update. */
int qcs_memory_report(int n, const qcs_step* steps, int num_steps, int engine,
                      qcs_step_report* reports);

/* Fused-pass plan of a circuit, host only (no device needed): what qcs_simulate with the same
 * engine and options launches.  B200-specific (the reference has no planner); used by the
 * tests and the measurement tools to count HBM sweeps. */
typedef struct qcs_plan_info {
    int64_t ops;            /* state operations after single-qubit merging (fuse) */
    int64_t passes;         /* HBM sweeps over the state: tile passes + single-op launches */
    int64_t tile_passes;
    int64_t single_passes;  /* passes of one operation, run by the dedicated gate kernels */
    int64_t rounds;         /* register + shared-memory rounds over all tile passes */
    int64_t smem_rounds;
    int64_t reg_ops;        /* operations in the register rounds (after butterfly merging) */
    int64_t max_tile_bits;  /* tile size used (log2 amplitudes) */
    int64_t alt_passes;     /* tile passes with a simplified program for tiles no sign step reaches */
    int64_t skip_passes;    /* ... where that program is the identity: only the reached tiles move */
    int64_t paired_passes;  /* passes of a pair around a skip pass that composes to a scalar: they
                               run only on the tiles the skip pass reaches */
    int64_t fp64_ops;       /* FP64 instructions (DFMA/DMUL/DADD, per thread) the tile passes execute,
                               counted from their specialised kernels over the tiles that compute */
    int64_t sweep_amps;     /* amplitudes the tile passes load and store (HBM traffic / 32 B) */
} qcs_plan_info;
int qcs_plan_stats(int n, const qcs_step* steps, int num_steps, int engine, const qcs_sim_options* opts,
                   qcs_plan_info* out);
/* Generate and compile (NVRTC, host only) the specialised kernel of every tile pass of that
 * plan -- the kernels qcs_simulate runs for passes with enough work (QCS_JIT=force: all).
 * *kernels = passes compiled, *cubin_bytes = total code size.  B200-specific check/tool. */
/* Which tile passes run as specialised kernels: 0 none (the interpreter kernel runs every
 * pass), 1 passes with enough work (default), 2 all.  Initial value from QCS_JIT (0/1/force).
 * Both forms compute bit-identical results; process-wide. */
int qcs_set_jit_mode(int mode);
int qcs_get_jit_mode(void);
/* Which specialised pass kernels take the persistent pipelined form -- one CTA per SM walking its
 * tiles through a ring of shared-memory slots, the HBM round trip of a tile hidden behind the
 * arithmetic of its neighbours: 0 none, 1 passes with 16-amplitude register rounds (default), 2
 * every eligible pass.  Initial value from QCS_PERSIST.  Same arithmetic in the same order as the
 * one-tile-per-CTA form: bit-identical results; process-wide; plans already cached by a state
 * keep their kernels.  B200-specific. */
int qcs_set_pipeline_mode(int mode);
int qcs_get_pipeline_mode(void);
int qcs_plan_compile(int n, const qcs_step* steps, int num_steps, int engine, const qcs_sim_options* opts,
                     int64_t* kernels, int64_t* cubin_bytes);
/* Host-only addressing proof of that plan's specialised kernels (no compile): for every register
 * round, the shared-memory addresses of every thread, group iteration and register -- under
 * every combination of runtime relabelling terms -- must cover the tile's slots exactly once
 * (in bounds, a permutation), and a relabelled last round's direct HBM stores likewise.
 * QCS_ERR_SIM with the failing round on a violation; *passes = passes checked.  B200-specific
 * (compute-sanitizer is not available on the GPU pool; this replaces its memcheck for these
 * accesses). */
int qcs_plan_verify(int n, const qcs_step* steps, int num_steps, int engine, const qcs_sim_options* opts,
                    int64_t* passes);

/* ------------------------------------------------------------------ compressed structures
 * The device gate encoder: materialise step_matrix_dax / step_matrix_das (engine.hpp:38-39)
 * on the GPU, byte-identical to the reference, without ever forming dense operators.
 * Output arrays are host (QCS_MEM_HOST) or device (QCS_MEM_DEVICE) memory of `capacity`
 * entries; *count receives the entry count (also when capacity is too small, which returns
 * QCS_ERR_CAPACITY).  Passing capacity 0 queries the count. */
int qcs_step_dax(int n, const qcs_placement* placements, int num_placements, int device,
                 uint64_t* rows, uint64_t* cols, double* values, uint64_t capacity, int mem,
                 uint64_t* count);
/* DasEntry stream (das.hpp:13-27): dis, last_in_row (0/1 bytes), value. */
int qcs_step_das(int n, const qcs_placement* placements, int num_placements, int device,
                 uint64_t* dis, uint8_t* last_in_row, double* values, uint64_t capacity, int mem,
                 uint64_t* count);
/* dax_mvm (dax.hpp:37, dax.cpp:96-103) on explicit entries, out-of-place: out = M * in.
 * Entries must be sorted by row (the DaxMatrix invariant, dax.hpp:20-21). */
int qcs_dax_mvm(const uint64_t* rows, const uint64_t* cols, const double* values, uint64_t count,
                int mem, const qcs_state* in, qcs_state* out);
/* das_mvm (das.hpp:39, das.cpp:131-150) on an explicit stream, out-of-place. */
int qcs_das_mvm(const uint64_t* dis, const uint8_t* last_in_row, const double* values,
                uint64_t count, int mem, const qcs_state* in, qcs_state* out);

/* ------------------------------------------------------------------ profiling hooks */
/* Number of kernels this library launched since load (process-wide). */
uint64_t qcs_kernel_launches(void);
/* Record / read CUDA events on the state's stream (for timing kernels on the launching stream). */
int qcs_event_record(qcs_state* s, int slot);
int qcs_event_elapsed_ms(qcs_state* s, int slot_begin, int slot_end, float* ms);
/* Per-launch timing: when enabled, every kernel the library launches for this state is
 * bracketed by CUDA events on the state's stream and attributed to its kernel class together
 * with its algorithmic HBM bytes (32 B per touched amplitude, whole 32-byte sectors). */
int qcs_timing_enable(qcs_state* s, int enable);
int qcs_timing_reset(qcs_state* s);
int qcs_timing_count(qcs_state* s, int* count); /* synchronises; number of kernel classes */
int qcs_timing_entry(qcs_state* s, int index, const char** kernel_class, uint64_t* launches,
                     double* total_ms, double* algorithmic_bytes);

#ifdef __cplusplus
}
#endif
#endif /* QCS_ABI_H */
