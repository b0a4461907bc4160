/*
 * qcs_oracle.c -- CPU restatement of the reference hot path.  TEST INFRASTRUCTURE ONLY.
 *
 * This file is the parity checker for the B200 product in paper_2411_15332_b200/.  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
 * load it.  The product never links or calls it; the product fails loudly when its CUDA
 * library is missing.
 *
 * Each function restates one reference routine (paths relative to /root/reference/proj):
 *   orc_step_entries_row -> src/engine.cpp:31-52 (step_factors) + src/dax.cpp:58-94 (dax_mtp
 *                           left fold, zero-product drop at :80-81) evaluated one row at a time
 *   orc_apply_step       -> src/engine.cpp:135-142 + src/dax.cpp:96-103 (step_matrix_dax then
 *                           dax_mvm, fused into a row-streaming loop; identical accumulation order)
 *   orc_step_dax         -> src/engine.cpp:135-142 (materialised DAX entries)
 *   orc_step_das         -> src/engine.cpp:144-151, src/das.cpp:43-65,83-129 (DAS stream)
 *   orc_dax_mvm          -> src/dax.cpp:96-103
 *   orc_das_mvm          -> src/das.cpp:131-150
 *   orc_apply_diag       -> src/engine.cpp:62-70 + src/circuit.cpp:9-12 + src/dax.cpp:96-103
 *   orc_rh_mvm           -> src/rh.cpp:92-156 (quarter loop, O(4^n); signs = (-1)^popcount(r&c),
 *                           which every sign method yields: tests/test_rh.cpp:149-163)
 *   orc_wht              -> the butterfly form of the same operator (O(n 2^n)), pinned against
 *                           orc_rh_mvm within tolerance (the reference's own RH tolerance is 1e-10,
 *                           tests/acceptance.cpp:225)
 *   orc_norm / orc_probabilities -> src/core.cpp:30-40
 *
 * Generalised placements: the reference only places gates on contiguous ascending qubits
 * (include/qcsim/circuit.hpp:10-15).  BASELINE configs need arbitrary qubit lists (seeded
 * controls, the CZ ring wrap).  For those the oracle follows the projector decomposition
 * used by oracle/ref_capi.cpp: the gate's last listed qubit
 * carries a 2x2 block, every other listed qubit an elementary |a><b| factor (value 1), and the
 * entries are merged in ascending global column order.
 *
 * Arithmetic: complex products are (ar*br - ai*bi, ar*bi + ai*br) with separately rounded
 * operations, matching libstdc++/GCC on x86-64 without FMA; build with -ffp-contract=off.
 * Complex numbers are interleaved double pairs (re, im), the byte layout of
 * std::complex<double>.  Qubit q is bit (n-1-q) of the basis index (core.hpp:64-66).
 */
#include <pthread.h>
#include <unistd.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_MAX_PLACE 64
#define ORC_MAX_ARITY 6

enum { ORC_OK = 0, ORC_ERR_DIMENSION = 2, ORC_ERR_ENCODING = 3, ORC_ERR_CAPACITY = 1, ORC_ERR_ARG = 8 };

static inline void cmul(double ar, double ai, double br, double bi, double* rr, double* ri) {
    const double t1 = ar * br, t2 = ai * bi, t3 = ar * bi, t4 = ai * br;
    *rr = t1 - t2;
    *ri = t3 + t4;
}

/* ---------------------------------------------------------------- step description */

typedef struct {
    int k;                      /* arity */
    int q[ORC_MAX_ARITY];       /* qubits in gate-local order (local bit k-1-i <-> q[i]) */
    int contiguous;             /* q[i+1] == q[i]+1 for all i (reference-native placement) */
    int carrier;                /* qubit at which the gate value enters the fold */
    const double* m;            /* 2^k x 2^k interleaved, row-major */
} orc_place;

typedef struct {
    int n;
    int np;
    orc_place p[ORC_MAX_PLACE];
    int order[ORC_MAX_PLACE];   /* placements sorted by minimum qubit (enumeration order) */
    int fold[ORC_MAX_PLACE];    /* placements in fold order (position of their carrier) */
    int sorted_cols;            /* 1 when enumeration order already yields ascending columns */
    uint64_t gate_mask;         /* union of placement bits */
} orc_step;

static int build_step(int n, int np, const int* arity, const int* qubits, const double* mats,
                      orc_step* st) {
    if (n < 1 || n > 62 || np < 0 || np > ORC_MAX_PLACE) return ORC_ERR_ARG;
    st->n = n;
    st->np = np;
    st->gate_mask = 0;
    st->sorted_cols = 1;
    int qoff = 0;
    size_t moff = 0;
    for (int j = 0; j < np; ++j) {
        orc_place* p = &st->p[j];
        p->k = arity[j];
        if (p->k < 1 || p->k > ORC_MAX_ARITY) return ORC_ERR_ARG;
        p->contiguous = 1;
        for (int i = 0; i < p->k; ++i) {
            p->q[i] = qubits[qoff + i];
            if (p->q[i] < 0 || p->q[i] >= n) return ORC_ERR_DIMENSION;
            const uint64_t bit = (uint64_t)1 << (n - 1 - p->q[i]);
            if (st->gate_mask & bit) return ORC_ERR_DIMENSION; /* overlap: circuit.cpp:55-58 */
            st->gate_mask |= bit;
            if (i > 0 && p->q[i] != p->q[i - 1] + 1) p->contiguous = 0;
        }
        p->carrier = p->contiguous ? p->q[0] : p->q[p->k - 1];
        if (!p->contiguous) st->sorted_cols = 0;
        p->m = mats + moff;
        qoff += p->k;
        moff += (size_t)2 << (2 * p->k);
    }
    /* enumeration order: by minimum qubit; fold order: by carrier position */
    for (int j = 0; j < np; ++j) st->order[j] = st->fold[j] = j;
    for (int a = 1; a < np; ++a)
        for (int b = a; b > 0; --b) {
            int ja = st->order[b - 1], jb = st->order[b];
            int qa = st->p[ja].q[0], qb = st->p[jb].q[0];
            for (int i = 1; i < st->p[ja].k; ++i) if (st->p[ja].q[i] < qa) qa = st->p[ja].q[i];
            for (int i = 1; i < st->p[jb].k; ++i) if (st->p[jb].q[i] < qb) qb = st->p[jb].q[i];
            if (qa > qb) { st->order[b - 1] = jb; st->order[b] = ja; } else break;
        }
    for (int a = 1; a < np; ++a)
        for (int b = a; b > 0; --b) {
            int ja = st->fold[b - 1], jb = st->fold[b];
            if (st->p[ja].carrier > st->p[jb].carrier) { st->fold[b - 1] = jb; st->fold[b] = ja; } else break;
        }
    return ORC_OK;
}

static inline int local_row(const orc_place* p, int n, uint64_t r) {
    int g = 0;
    for (int i = 0; i < p->k; ++i) g |= (int)((r >> (n - 1 - p->q[i])) & 1u) << (p->k - 1 - i);
    return g;
}

static inline uint64_t col_bits(const orc_place* p, int n, int c) {
    uint64_t v = 0;
    for (int i = 0; i < p->k; ++i) v |= (uint64_t)((c >> (p->k - 1 - i)) & 1) << (n - 1 - p->q[i]);
    return v;
}

typedef struct { uint64_t col; double re, im; } orc_entry;

static int cmp_entry(const void* a, const void* b) {
    const uint64_t x = ((const orc_entry*)a)->col, y = ((const orc_entry*)b)->col;
    return x < y ? -1 : (x > y ? 1 : 0);
}

/*
 * All stored entries of row r of the step's operation matrix, in ascending column order,
 * zero products dropped.  The value of an entry is the left fold of dax_mtp over the per-position
 * factor list (engine.cpp:139-141): first factor's value, then multiply by each following
 * factor's value, identities (1+0i) included, so the bytes equal step_matrix_dax.
 * Returns the number of entries written to out (capacity cap) or -1 on overflow.
 */
static long row_entries(const orc_step* st, uint64_t r, orc_entry* out, long cap) {
    const int n = st->n, np = st->np;
    int g[ORC_MAX_PLACE];
    int nz_cnt[ORC_MAX_PLACE];
    int nz_col[ORC_MAX_PLACE][1 << ORC_MAX_ARITY];
    for (int e = 0; e < np; ++e) {
        const int j = st->order[e];
        const orc_place* p = &st->p[j];
        g[j] = local_row(p, n, r);
        const int dim = 1 << p->k;
        const double* row = p->m + (size_t)2 * dim * g[j];
        int c = 0;
        for (int col = 0; col < dim; ++col)
            if (row[2 * col] != 0.0 || row[2 * col + 1] != 0.0) nz_col[j][c++] = col; /* dax.cpp:42 */
        nz_cnt[j] = c;
        if (c == 0) return 0;
    }
    /* odometer over placements in enumeration order, last placement fastest */
    int idx[ORC_MAX_PLACE];
    memset(idx, 0, sizeof(idx));
    long count = 0;
    const uint64_t base = r & ~st->gate_mask;
    for (;;) {
        uint64_t col = base;
        for (int e = 0; e < np; ++e) {
            const int j = st->order[e];
            col |= col_bits(&st->p[j], n, nz_col[j][idx[e]]);
        }
        /* value fold in position order: identities at uncovered positions and at the
           non-carrier qubits of a generalised placement, the gate value at its carrier */
        double vr = 0.0, vi = 0.0;
        int started = 0;
        int fpos = 0; /* next placement in fold order */
        int q = 0;
        while (q < n) {
            const orc_place* p = NULL;
            int pj = -1;
            if (fpos < np && st->p[st->fold[fpos]].carrier == q) { pj = st->fold[fpos]; p = &st->p[pj]; }
            double fr = 1.0, fi = 0.0;
            int step = 1;
            if (p) {
                int e = 0;
                while (st->order[e] != pj) ++e;
                const int dim = 1 << p->k;
                const double* v = p->m + (size_t)2 * (dim * g[pj] + nz_col[pj][idx[e]]);
                fr = v[0];
                fi = v[1];
                if (p->contiguous) step = p->k;
                ++fpos;
            }
            if (!started) { vr = fr; vi = fi; started = 1; }
            else { double tr, ti; cmul(vr, vi, fr, fi, &tr, &ti); vr = tr; vi = ti; }
            q += step;
        }
        if (vr != 0.0 || vi != 0.0) { /* dax.cpp:80-81 */
            if (count >= cap) return -1;
            out[count].col = col;
            out[count].re = vr;
            out[count].im = vi;
            ++count;
        }
        int e = np - 1;
        while (e >= 0) {
            const int j = st->order[e];
            if (++idx[e] < nz_cnt[j]) break;
            idx[e] = 0;
            --e;
        }
        if (e < 0) break;
    }
    if (!st->sorted_cols && count > 1) qsort(out, (size_t)count, sizeof(orc_entry), cmp_entry);
    return count;
}

static long row_capacity(const orc_step* st) {
    long cap = 1;
    for (int j = 0; j < st->np; ++j) cap *= (long)1 << st->p[j].k;
    return cap;
}

/* ---------------------------------------------------------------- public entry points */

/* Number of entries of the step matrix (analytic upper bound used to size buffers). */
long orc_step_row_capacity(int n, int np, const int* arity, const int* qubits, const double* mats) {
    orc_step st;
    if (build_step(n, np, arity, qubits, mats, &st) != ORC_OK) return -1;
    return row_capacity(&st);
}

/*
 * step_matrix_dax + dax_mvm as one streaming pass: out[r] = sum over the row's entries in
 * ascending column order of value * in[col], accumulated from (0,0) (dax.cpp:98-101).
 * in/out are 2*2^n doubles and must not alias.
 */
struct apply_job {
    const orc_step* st;
    const double* in;
    double* out;
    uint64_t r0, r1;
    long cap;
    int rc;
};

static void* apply_rows(void* arg) {
    struct apply_job* j = (struct apply_job*)arg;
    orc_entry* buf = (orc_entry*)malloc(sizeof(orc_entry) * (size_t)j->cap);
    if (!buf) { j->rc = ORC_ERR_CAPACITY; return NULL; }
    for (uint64_t r = j->r0; r < j->r1; ++r) {
        const long cnt = row_entries(j->st, r, buf, j->cap);
        double ar = 0.0, ai = 0.0;
        for (long e = 0; e < cnt; ++e) {
            double pr, pi;
            cmul(buf[e].re, buf[e].im, j->in[2 * buf[e].col], j->in[2 * buf[e].col + 1], &pr, &pi);
            ar = ar + pr;
            ai = ai + pi;
        }
        j->out[2 * r] = ar;
        j->out[2 * r + 1] = ai;
    }
    free(buf);
    j->rc = ORC_OK;
    return NULL;
}

/* Worker threads for the row loop of orc_apply_step: ORC_THREADS, else the online cores (<= 64).
 * Rows are independent and each row's arithmetic is unchanged, so the result is the same bytes
 * at any thread count (the reference's per-row accumulation order, dax.cpp:98-101). */
static int apply_threads(uint64_t dim) {
    const char* v = getenv("ORC_THREADS");
    long t = v ? atol(v) : sysconf(_SC_NPROCESSORS_ONLN);
    if (t < 1) t = 1;
    if (t > 64) t = 64;
    if (dim < ((uint64_t)1 << 16)) t = 1;
    return (int)t;
}

int orc_apply_step(int n, int np, const int* arity, const int* qubits, const double* mats,
                   const double* in, double* out) {
    orc_step st;
    int rc = build_step(n, np, arity, qubits, mats, &st);
    if (rc != ORC_OK) return rc;
    const long cap = row_capacity(&st);
    const uint64_t dim = (uint64_t)1 << n;
    const int nt = apply_threads(dim);
    struct apply_job jobs[64];
    pthread_t tid[64];
    for (int t = 0; t < nt; ++t) {
        jobs[t].st = &st;
        jobs[t].in = in;
        jobs[t].out = out;
        jobs[t].r0 = dim / (uint64_t)nt * (uint64_t)t;
        jobs[t].r1 = t + 1 == nt ? dim : dim / (uint64_t)nt * (uint64_t)(t + 1);
        jobs[t].cap = cap;
        jobs[t].rc = ORC_OK;
    }
    if (nt == 1) {
        apply_rows(&jobs[0]);
        return jobs[0].rc;
    }
    int started = 0;
    for (; started < nt; ++started)
        if (pthread_create(&tid[started], NULL, apply_rows, &jobs[started]) != 0) break;
    for (int t = started; t < nt; ++t) apply_rows(&jobs[t]); /* could not start: run inline */
    for (int t = 0; t < started; ++t) pthread_join(tid[t], NULL);
    for (int t = 0; t < nt; ++t)
        if (jobs[t].rc != ORC_OK) return jobs[t].rc;
    return ORC_OK;
}

/*
 * Materialised DAX entries (row-major, strictly ascending linear index), engine.cpp:135-142.
 * Writes at most cap entries; returns the entry count, or -1 when cap is too small.
 */
long orc_step_dax(int n, int np, const int* arity, const int* qubits, const double* mats,
                  uint64_t* rows, uint64_t* cols, double* vals, long cap) {
    orc_step st;
    if (build_step(n, np, arity, qubits, mats, &st) != ORC_OK) return -2;
    const long rcap = row_capacity(&st);
    orc_entry* buf = (orc_entry*)malloc(sizeof(orc_entry) * (size_t)rcap);
    if (!buf) return -2;
    const uint64_t dim = (uint64_t)1 << n;
    long total = 0;
    for (uint64_t r = 0; r < dim; ++r) {
        const long cnt = row_entries(&st, r, buf, rcap);
        if (total + cnt > cap) { free(buf); return -1; }
        for (long e = 0; e < cnt; ++e) {
            rows[total] = r;
            cols[total] = buf[e].col;
            vals[2 * total] = buf[e].re;
            vals[2 * total + 1] = buf[e].im;
            ++total;
        }
    }
    free(buf);
    return total;
}

/*
 * Materialised DAS stream (das.hpp:13-27): dis = zeros since the previous stored entry of the
 * row (or the row start), last_in_row flags the row's final entry.  An all-zero row cannot be
 * encoded (das.cpp:59-61, :124-125): returns -3.  -1 = cap too small.
 */
long orc_step_das(int n, int np, const int* arity, const int* qubits, const double* mats,
                  uint64_t* dis, uint8_t* last, double* vals, long cap) {
    orc_step st;
    if (build_step(n, np, arity, qubits, mats, &st) != ORC_OK) return -2;
    const long rcap = row_capacity(&st);
    orc_entry* buf = (orc_entry*)malloc(sizeof(orc_entry) * (size_t)rcap);
    if (!buf) return -2;
    const uint64_t dim = (uint64_t)1 << n;
    long total = 0;
    for (uint64_t r = 0; r < dim; ++r) {
        const long cnt = row_entries(&st, r, buf, rcap);
        if (cnt == 0) { free(buf); return -3; }
        if (total + cnt > cap) { free(buf); return -1; }
        uint64_t next = 0;
        for (long e = 0; e < cnt; ++e) {
            dis[total] = buf[e].col - next;
            next = buf[e].col + 1;
            last[total] = (uint8_t)(e == cnt - 1);
            vals[2 * total] = buf[e].re;
            vals[2 * total + 1] = buf[e].im;
            ++total;
        }
    }
    free(buf);
    return total;
}

/* dax.cpp:96-103 on materialised entries. */
int orc_dax_mvm(int n, const uint64_t* rows, const uint64_t* cols, const double* vals, long count,
                const double* in, double* out) {
    const uint64_t dim = (uint64_t)1 << n;
    memset(out, 0, sizeof(double) * 2 * dim);
    for (long e = 0; e < count; ++e) {
        if (rows[e] >= dim || cols[e] >= dim) return ORC_ERR_ENCODING;
        double pr, pi;
        cmul(vals[2 * e], vals[2 * e + 1], in[2 * cols[e]], in[2 * cols[e] + 1], &pr, &pi);
        out[2 * rows[e]] = out[2 * rows[e]] + pr;
        out[2 * rows[e] + 1] = out[2 * rows[e] + 1] + pi;
    }
    return ORC_OK;
}

/* das.cpp:131-150: a forward scan with running (row, col) cursors. */
int orc_das_mvm(int n, const uint64_t* dis, const uint8_t* last, const double* vals, long count,
                const double* in, double* out) {
    const uint64_t dim = (uint64_t)1 << n;
    memset(out, 0, sizeof(double) * 2 * dim);
    uint64_t row = 0, col = 0;
    for (long e = 0; e < count; ++e) {
        col += dis[e];
        if (row >= dim || col >= dim) return ORC_ERR_ENCODING; /* "malformed DAS stream" */
        double pr, pi;
        cmul(vals[2 * e], vals[2 * e + 1], in[2 * col], in[2 * col + 1], &pr, &pi);
        out[2 * row] = out[2 * row] + pr;
        out[2 * row + 1] = out[2 * row + 1] + pi;
        if (last[e]) { ++row; col = 0; } else { col += 1; }
    }
    return ORC_OK;
}

/* Diagonal sign step: engine.cpp:62-70 (entries +-1) through dax_mvm; DiagSign::negated is
   circuit.cpp:9-12 (listed != flip_rest).  flipped must be sorted ascending. */
static int listed(const uint64_t* f, uint64_t nf, uint64_t i) {
    uint64_t lo = 0, hi = nf;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) / 2;
        if (f[mid] < i) lo = mid + 1; else hi = mid;
    }
    return lo < nf && f[lo] == i;
}

int orc_apply_diag(int n, const uint64_t* flipped, uint64_t nf, int flip_rest, const double* in,
                   double* out) {
    const uint64_t dim = (uint64_t)1 << n;
    for (uint64_t i = 0; i < nf; ++i) if (flipped[i] >= dim) return ORC_ERR_DIMENSION;
    for (uint64_t i = 0; i < dim; ++i) {
        const double d = (listed(flipped, nf, i) != (flip_rest != 0)) ? -1.0 : 1.0;
        double pr, pi;
        cmul(d, 0.0, in[2 * i], in[2 * i + 1], &pr, &pi);
        out[2 * i] = 0.0 + pr;
        out[2 * i + 1] = 0.0 + pi;
    }
    return ORC_OK;
}

/* rh.cpp:92-156, quarter loop.  O(4^n): intended for n <= 14. */
int orc_rh_mvm(int n, const double* in, double* out) {
    if (n < 1) return ORC_ERR_DIMENSION;
    const uint64_t dim = (uint64_t)1 << n, half = dim >> 1;
    const double value = exp2(-0.5 * n); /* rh.cpp:20 */
    double* sc = (double*)malloc(sizeof(double) * 2 * dim);
    if (!sc) return ORC_ERR_CAPACITY;
    for (uint64_t i = 0; i < 2 * dim; ++i) sc[i] = in[i] * value; /* rh.cpp:99-100 */
    memset(out, 0, sizeof(double) * 2 * dim);
    for (uint64_t r = 0; r < half; ++r)
        for (uint64_t c = 0; c < half; ++c) {
            const double sg = (__builtin_popcountll(r & c) & 1) ? -1.0 : 1.0;
            const double a0 = sg * sc[2 * c], a1 = sg * sc[2 * c + 1];
            const double b0 = sg * sc[2 * (c + half)], b1 = sg * sc[2 * (c + half) + 1];
            out[2 * r] = out[2 * r] + a0;
            out[2 * r + 1] = out[2 * r + 1] + a1;
            out[2 * r] = out[2 * r] + b0;
            out[2 * r + 1] = out[2 * r + 1] + b1;
            out[2 * (r + half)] = out[2 * (r + half)] + a0;
            out[2 * (r + half) + 1] = out[2 * (r + half) + 1] + a1;
            out[2 * (r + half)] = out[2 * (r + half)] - b0;
            out[2 * (r + half) + 1] = out[2 * (r + half) + 1] - b1;
        }
    free(sc);
    return ORC_OK;
}

/* The same operator as a radix-2 butterfly: scale by exp2(-n/2) first, then (a+b, a-b) per bit. */
int orc_wht(int n, const double* in, double* out) {
    if (n < 1) return ORC_ERR_DIMENSION;
    const uint64_t dim = (uint64_t)1 << n;
    const double value = exp2(-0.5 * n);
    for (uint64_t i = 0; i < 2 * dim; ++i) out[i] = in[i] * value;
    for (int b = 0; b < n; ++b) {
        const uint64_t h = (uint64_t)1 << b;
        for (uint64_t i = 0; i < dim; ++i) {
            if (i & h) continue;
            const uint64_t j = i | h;
            const double ar = out[2 * i], ai = out[2 * i + 1], br = out[2 * j], bi = out[2 * j + 1];
            out[2 * i] = ar + br;
            out[2 * i + 1] = ai + bi;
            out[2 * j] = ar - br;
            out[2 * j + 1] = ai - bi;
        }
    }
    return ORC_OK;
}

/* core.cpp:30-34: sequential sum of std::norm, then sqrt. */
double orc_norm(int n, const double* s) {
    const uint64_t dim = (uint64_t)1 << n;
    double acc = 0.0;
    for (uint64_t i = 0; i < dim; ++i) acc += s[2 * i] * s[2 * i] + s[2 * i + 1] * s[2 * i + 1];
    return sqrt(acc);
}

/* core.cpp:36-40 */
void orc_probabilities(int n, const double* s, double* p) {
    const uint64_t dim = (uint64_t)1 << n;
    for (uint64_t i = 0; i < dim; ++i) p[i] = s[2 * i] * s[2 * i] + s[2 * i + 1] * s[2 * i + 1];
}
