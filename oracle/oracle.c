/*
 * oracle.c -- CPU restatement of the reference MSBFM hot path, in plain C.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the *checker*: it may be loaded by
 * tests/, by __graft_entry__.smoke() and by bench.py's cpu_baseline leg, and by
 * nothing else.  The product (paper_2301_11828_b200/) never links or calls it.
 *
 * Every function restates the algorithm of the reference library `pdfast`
 * (header-only C++20 under /root/reference/proj/include/pdfast, cited below as
 * <file>:<line>).  The spectral product  f = A_hat u  that the reference
 * evaluates with zero-padded FFTs (convolution.hpp:249-259) is restated here as
 * the equivalent direct stencil sum over the lattice window (the reference's
 * own independent oracle, tests/support/oracles.hpp:72-96), which is exact
 * linear correlation; the two agree to round-off (the reference's own tests
 * pin this at 1e-10..1e-12, tests/test_convolution.cpp:129-155).
 *
 * Pinning: this restatement is checked in tests/test_oracle.py against
 *  - the reference's known-answer tests (alpha, s0, 22 nonzero K^xx at M=3,
 *    stretch sqrt(2)-1, inclusive threshold, crossing counts), and
 *  - golden vectors produced by the reference itself (its headers compiled
 *    unmodified against oracle/fftw_cpu, see oracle/Makefile and
 *    oracle/gen_golden.py) and committed under tests/golden/.
 *
 * No FMA contraction: build with -ffp-contract=off so operation order and
 * rounding follow the reference (g++ x86-64 default target has no FMA).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

typedef int64_t idx_t;

/* ------------------------------------------------------- row threading --
 * The row sweeps below (apply, corrections, dense force) compute every node
 * independently with the serial operation order, so splitting the node range
 * over threads is bit-identical to the serial sweep.  ORC_THREADS caps the
 * thread count (default: online cores, at most 64). */
typedef void (*orc_rows_fn)(void* ctx, idx_t p0, idx_t p1);
typedef struct {
    orc_rows_fn fn;
    void* ctx;
    idx_t p0, p1;
} orc_rows_job;

static void* orc_rows_thread(void* a) {
    orc_rows_job* j = (orc_rows_job*)a;
    j->fn(j->ctx, j->p0, j->p1);
    return NULL;
}

static void orc_par_rows(idx_t n, orc_rows_fn fn, void* ctx) {
    long t = sysconf(_SC_NPROCESSORS_ONLN);
    const char* env = getenv("ORC_THREADS");
    if (env && atoi(env) > 0) t = atoi(env);
    if (t > 64) t = 64;
    if (t < 1 || n < 65536) t = 1;
    if (t == 1) {
        fn(ctx, 0, n);
        return;
    }
    pthread_t th[64];
    orc_rows_job jobs[64];
    for (long i = 0; i < t; ++i) {
        jobs[i].fn = fn;
        jobs[i].ctx = ctx;
        jobs[i].p0 = n * i / t;
        jobs[i].p1 = n * (i + 1) / t;
    }
    for (long i = 1; i < t; ++i) pthread_create(&th[i], NULL, orc_rows_thread, &jobs[i]);
    orc_rows_thread(&jobs[0]);
    for (long i = 1; i < t; ++i) pthread_join(th[i], NULL);
}

typedef struct orc_t orc_t;
typedef struct {
    const orc_t* P;
    const double* u;
    double* f;
} orc_op_ctx;

/* ------------------------------------------------------------------ RNG --
 * std::mt19937 (32-bit Mersenne twister, init_genrand seeding) and the
 * libstdc++ uniform_real_distribution<double>: generate_canonical<double,53>
 * draws two 32-bit words, (w0 + w1*2^32) / 2^64, then x*(b-a)+a.
 * Used by tests/support/oracles.hpp:113-119 (random_field) and :99-110. */
typedef struct {
    uint32_t mt[624];
    int mti;
} orc_rng;

orc_rng* orc_rng_new(uint32_t seed) {
    orc_rng* r = (orc_rng*)malloc(sizeof(orc_rng));
    r->mt[0] = seed;
    for (int i = 1; i < 624; ++i)
        r->mt[i] = 1812433253u * (r->mt[i - 1] ^ (r->mt[i - 1] >> 30)) + (uint32_t)i;
    r->mti = 624;
    return r;
}

void orc_rng_free(orc_rng* r) { free(r); }

uint32_t orc_rng_next(orc_rng* r) {
    if (r->mti >= 624) {
        for (int k = 0; k < 624; ++k) {
            uint32_t y = (r->mt[k] & 0x80000000u) | (r->mt[(k + 1) % 624] & 0x7fffffffu);
            r->mt[k] = r->mt[(k + 397) % 624] ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
        }
        r->mti = 0;
    }
    uint32_t y = r->mt[r->mti++];
    y ^= (y >> 11);
    y ^= (y << 7) & 0x9d2c5680u;
    y ^= (y << 15) & 0xefc60000u;
    y ^= (y >> 18);
    return y;
}

double orc_rng_uniform(orc_rng* r, double a, double b) {
    const double w0 = (double)orc_rng_next(r);
    const double w1 = (double)orc_rng_next(r);
    const double two32 = 4294967296.0;
    double x = (w0 + w1 * two32) / (two32 * two32);
    if (x >= 1.0) x = nextafter(1.0, 0.0);
    return x * (b - a) + a;
}

void orc_rng_fill(orc_rng* r, idx_t n, double a, double b, double* out) {
    for (idx_t i = 0; i < n; ++i) out[i] = orc_rng_uniform(r, a, b);
}

/* ------------------------------------------------------------ geometry -- */
int orc_n_pairs(int dim) { return dim * (dim + 1) / 2; }

/* kernel.hpp:19-28 */
int orc_pair_index(int dim, int a, int b) {
    if (a > b) { int t = a; a = b; b = t; }
    if (dim == 2) return a + b;
    static const int row_start[3] = {0, 3, 5};
    return row_start[a] + b - a;
}

/* in-band off-centre offsets in for_each_offset order (kernel.hpp:71-89):
 * axis 0 outermost, keep 0 < |o|^2 <= M^2.  offs is n x 3 (unused axes 0). */
int orc_offsets(int dim, int M, int* offs) {
    int n = 0;
    const long M2 = (long)M * M;
    for (int a = -M; a <= M; ++a)
        for (int b = -M; b <= M; ++b)
            for (int c = (dim == 3 ? -M : 0); c <= (dim == 3 ? M : 0); ++c) {
                long n2 = (long)a * a + (long)b * b + (long)c * c;
                if (n2 == 0 || n2 > M2) continue;
                if (offs) { offs[3 * n] = a; offs[3 * n + 1] = b; offs[3 * n + 2] = c; }
                ++n;
            }
    return n;
}

/* kernel.hpp:50-54: axis Dim-1 slowest */
static idx_t stencil_index(int dim, int M, const int* o) {
    const int side = 2 * M + 1;
    idx_t idx = 0;
    for (int d = dim - 1; d >= 0; --d) idx = idx * side + (o[d] + M);
    return idx;
}

idx_t orc_stencil_size(int dim, int M) {
    idx_t s = 1;
    for (int d = 0; d < dim; ++d) s *= (2 * M + 1);
    return s;
}

/* material.hpp:15-24 */
double orc_alpha(double E, double delta, int dim, double thickness) {
    const double pi = 3.141592653589793238462643383279502884;
    if (dim == 2) return 9.0 * E / (pi * delta * delta * delta * thickness);
    return 12.0 * E / (pi * delta * delta * delta * delta);
}

/* material.hpp:27-31 (mode 0 = stress, 1 = strain) */
double orc_critical_stretch(double G0, double E, double delta, int mode) {
    const double pi = 3.141592653589793238462643383279502884;
    if (mode == 0) return sqrt(4.0 * pi * G0 / (9.0 * E * delta));
    return sqrt(5.0 * pi * G0 / (12.0 * E * delta));
}

/* grid.hpp:135-139 */
double orc_volume_correction(double dist, double delta, double h) {
    if (dist <= delta - 0.5 * h) return 1.0;
    if (dist <= delta) return 0.5 + (delta - dist) / h;
    return 0.0;
}

/* build_kernel, kernel.hpp:99-127.  K is n_pairs x (2M+1)^dim. */
void orc_build_kernel(int dim, double h, double delta, int M, double E, double thickness,
                      double* K) {
    const int np = orc_n_pairs(dim);
    const idx_t ss = orc_stencil_size(dim, M);
    memset(K, 0, sizeof(double) * (size_t)(np * ss));
    const double alpha = orc_alpha(E, delta, dim, thickness);
    const double vol = dim == 2 ? h * h * thickness : h * h * h;
    int nof = orc_offsets(dim, M, NULL);
    int* offs = (int*)malloc(sizeof(int) * 3 * (size_t)nof);
    orc_offsets(dim, M, offs);
    for (int k = 0; k < nof; ++k) {
        const int* o = offs + 3 * k;
        long n2 = 0;
        for (int d = 0; d < dim; ++d) n2 += (long)o[d] * o[d];
        const double dist = h * sqrt((double)n2);
        const double lam = orc_volume_correction(dist, delta, h);
        const double scale = alpha * lam * vol / (dist * dist * dist);
        for (int a = 0; a < dim; ++a)
            for (int b = a; b < dim; ++b)
                K[orc_pair_index(dim, a, b) * ss + stencil_index(dim, M, o)] =
                    scale * (o[a] * h) * (o[b] * h);
    }
    int zero[3] = {0, 0, 0};
    for (int a = 0; a < dim; ++a)
        for (int b = a; b < dim; ++b) {
            double sum = 0.0;
            double* Kp = K + orc_pair_index(dim, a, b) * ss;
            for (int k = 0; k < nof; ++k) sum += Kp[stencil_index(dim, M, offs + 3 * k)];
            Kp[stencil_index(dim, M, zero)] = -sum;
        }
    free(offs);
}

/* ------------------------------------------------------------- problem -- */
typedef struct {
    double box[6]; /* lo[0..dim), hi at [3..3+dim) */
    uint8_t dir_mask;
    int kind; /* 0 displacement, 1 velocity */
    double value;
} orc_constraint;

struct orc_t {
    int dim, dims[3];
    double h, origin[3], thickness, delta, E, rho;
    int M, nof, np, lw;
    idx_t n, ss;
    int* offs;          /* nof x 3, for_each_offset order */
    double* K;          /* np x ss */
    uint8_t* near_surface;
    uint8_t* cmask;
    double* De;         /* np x n, corrections.hpp:20-62 */
    uint32_t* ledger;   /* n x lw bit set over offsets (BondLedger, ledger.hpp:13-57) */
    idx_t total_broken;
    int n_cons;
    orc_constraint cons[16];
    double* body;       /* dim x n */
    /* VV state (timestepping.hpp:55-61) */
    double *u, *v, *f, *f_prev;
    double t, dt;
    idx_t step;
    int force_ready;
    int* sorted_off;    /* offsets sorted by linear displacement (partner order) */
    /* ADR state (AdrIntegrator, timestepping.hpp:79-145) */
    int integrator;     /* 0 velocity Verlet, 1 ADR */
    double* vh;         /* staggered velocity v_half (dim x n) */
    double mass[3];     /* adr_mass, timestepping.hpp:150-162 */
    int fixed;          /* fixed_damping given */
    double fixed_c, last_c;
};

static void pos_of(const orc_t* P, const int* c, double* x) {
    for (int d = 0; d < P->dim; ++d) x[d] = P->origin[d] + (c[d] + 0.5) * P->h;
}

static void coords_of(const orc_t* P, idx_t p, int* c) {
    c[0] = (int)(p % P->dims[0]);
    p /= P->dims[0];
    c[1] = (int)(p % P->dims[1]);
    c[2] = P->dim == 3 ? (int)(p / P->dims[1]) : 0;
}

static idx_t lin_of(const orc_t* P, const int* c) {
    if (P->dim == 2) return (idx_t)c[1] * P->dims[0] + c[0];
    return ((idx_t)c[2] * P->dims[1] + c[1]) * P->dims[0] + c[0];
}

static int in_lattice(const orc_t* P, const int* c) {
    for (int d = 0; d < P->dim; ++d)
        if (c[d] < 0 || c[d] >= P->dims[d]) return 0;
    return 1;
}

static int box_contains(const orc_t* P, const double* box, const double* x) {
    for (int d = 0; d < P->dim; ++d)
        if (x[d] < box[d] || x[d] > box[3 + d]) return 0;
    return 1;
}

static idx_t off_disp(const orc_t* P, const int* o) {
    return (idx_t)o[2] * P->dims[0] * P->dims[1] + (idx_t)o[1] * P->dims[0] + o[0];
}

static int cmp_disp_P_dims0, cmp_disp_P_dims1;
static const int* cmp_offs;
static int cmp_disp(const void* a, const void* b) {
    const int* oa = cmp_offs + 3 * *(const int*)a;
    const int* ob = cmp_offs + 3 * *(const int*)b;
    idx_t da = (idx_t)oa[2] * cmp_disp_P_dims0 * cmp_disp_P_dims1 + (idx_t)oa[1] * cmp_disp_P_dims0 + oa[0];
    idx_t db = (idx_t)ob[2] * cmp_disp_P_dims0 * cmp_disp_P_dims1 + (idx_t)ob[1] * cmp_disp_P_dims0 + ob[0];
    return da < db ? -1 : (da > db ? 1 : 0);
}

static void rebuild_regions(orc_t* P);

orc_t* orc_new(int dim, const int* dims, double h, const double* origin, double thickness,
               double delta, int M, double E, double rho) {
    orc_t* P = (orc_t*)calloc(1, sizeof(orc_t));
    P->dim = dim;
    P->dims[2] = 1;
    for (int d = 0; d < dim; ++d) {
        P->dims[d] = dims[d];
        P->origin[d] = origin ? origin[d] : 0.0;
    }
    P->h = h;
    P->thickness = thickness;
    P->delta = delta;
    P->M = M;
    P->E = E;
    P->rho = rho;
    P->n = (idx_t)P->dims[0] * P->dims[1] * P->dims[2];
    P->np = orc_n_pairs(dim);
    P->ss = orc_stencil_size(dim, M);
    P->nof = orc_offsets(dim, M, NULL);
    P->offs = (int*)malloc(sizeof(int) * 3 * (size_t)P->nof);
    orc_offsets(dim, M, P->offs);
    P->lw = (P->nof + 31) / 32;
    P->K = (double*)calloc((size_t)(P->np * P->ss), sizeof(double));
    orc_build_kernel(dim, h, delta, M, E, thickness, P->K);
    P->near_surface = (uint8_t*)calloc((size_t)P->n, 1);
    P->cmask = (uint8_t*)calloc((size_t)P->n, 1);
    P->De = (double*)calloc((size_t)(P->np * P->n), sizeof(double));
    P->ledger = (uint32_t*)calloc((size_t)(P->n * P->lw), sizeof(uint32_t));
    P->body = (double*)calloc((size_t)(dim * P->n), sizeof(double));
    P->sorted_off = (int*)malloc(sizeof(int) * (size_t)P->nof);
    for (int k = 0; k < P->nof; ++k) P->sorted_off[k] = k;
    cmp_disp_P_dims0 = P->dims[0];
    cmp_disp_P_dims1 = P->dims[1];
    cmp_offs = P->offs;
    qsort(P->sorted_off, (size_t)P->nof, sizeof(int), cmp_disp);
    rebuild_regions(P);
    return P;
}

void orc_free(orc_t* P) {
    if (!P) return;
    free(P->offs); free(P->K); free(P->near_surface); free(P->cmask); free(P->De);
    free(P->ledger); free(P->body); free(P->sorted_off);
    free(P->u); free(P->v); free(P->f); free(P->f_prev); free(P->vh);
    free(P);
}

idx_t orc_n_nodes(const orc_t* P) { return P->n; }
int orc_n_offsets(const orc_t* P) { return P->nof; }
void orc_get_offsets(const orc_t* P, int* out) { memcpy(out, P->offs, sizeof(int) * 3 * (size_t)P->nof); }
void orc_get_kernel(const orc_t* P, double* K) { memcpy(K, P->K, sizeof(double) * (size_t)(P->np * P->ss)); }
void orc_get_regions(const orc_t* P, uint8_t* near_surface, uint8_t* cmask) {
    if (near_surface) memcpy(near_surface, P->near_surface, (size_t)P->n);
    if (cmask) memcpy(cmask, P->cmask, (size_t)P->n);
}
void orc_get_de(const orc_t* P, double* De) { memcpy(De, P->De, sizeof(double) * (size_t)(P->np * P->n)); }

/* Regions ctor (grid.hpp:177-195) + SurfaceDiag ctor (corrections.hpp:24-42) */
static void rebuild_regions(orc_t* P) {
    const int dim = P->dim, M = P->M;
    memset(P->cmask, 0, (size_t)P->n);
    memset(P->De, 0, sizeof(double) * (size_t)(P->np * P->n));
    for (idx_t p = 0; p < P->n; ++p) {
        int c[3];
        coords_of(P, p, c);
        uint8_t ns = 0;
        for (int d = 0; d < dim; ++d)
            if (c[d] < M || c[d] >= P->dims[d] - M) { ns = 1; break; }
        P->near_surface[p] = ns;
    }
    for (int k = 0; k < P->n_cons; ++k)
        for (idx_t p = 0; p < P->n; ++p) {
            int c[3];
            double x[3];
            coords_of(P, p, c);
            pos_of(P, c, x);
            if (box_contains(P, P->cons[k].box, x)) P->cmask[p] |= P->cons[k].dir_mask;
        }
    for (idx_t p = 0; p < P->n; ++p) {
        if (!P->near_surface[p]) continue;
        int c[3];
        coords_of(P, p, c);
        for (int k = 0; k < P->nof; ++k) {
            const int* o = P->offs + 3 * k;
            int q[3] = {c[0] + o[0], c[1] + o[1], c[2] + o[2]};
            if (in_lattice(P, q)) continue;
            const idx_t si = stencil_index(dim, M, o);
            for (int a = 0; a < dim; ++a)
                for (int b = a; b < dim; ++b) {
                    const int pi = orc_pair_index(dim, a, b);
                    P->De[pi * P->n + p] += P->K[pi * P->ss + si];
                }
        }
    }
}

/* replace the stencils (e.g. tests/support/oracles.hpp:99-110 random kernels) */
void orc_set_kernel(orc_t* P, const double* K) {
    memcpy(P->K, K, sizeof(double) * (size_t)(P->np * P->ss));
    rebuild_regions(P);
}

/* kind 0 = displacement, 1 = velocity (grid.hpp:160-166) */
int orc_add_constraint(orc_t* P, const double* lo, const double* hi, int dir_mask, int kind,
                       double value) {
    if (P->n_cons >= 16) return -1;
    orc_constraint* c = &P->cons[P->n_cons++];
    memset(c, 0, sizeof(*c));
    for (int d = 0; d < P->dim; ++d) { c->box[d] = lo[d]; c->box[3 + d] = hi[d]; }
    c->dir_mask = (uint8_t)dir_mask;
    c->kind = kind;
    c->value = value;
    rebuild_regions(P);
    return 0;
}

/* Simulation ctor body-load fill, timestepping.hpp:192-196 */
void orc_add_load(orc_t* P, const double* lo, const double* hi, const double* value) {
    double box[6] = {0};
    for (int d = 0; d < P->dim; ++d) { box[d] = lo[d]; box[3 + d] = hi[d]; }
    for (idx_t p = 0; p < P->n; ++p) {
        int c[3];
        double x[3];
        coords_of(P, p, c);
        pos_of(P, c, x);
        if (box_contains(P, box, x))
            for (int d = 0; d < P->dim; ++d) P->body[d * P->n + p] += value[d];
    }
}

void orc_set_body(orc_t* P, const double* body) {
    memcpy(P->body, body, sizeof(double) * (size_t)(P->dim * P->n));
}

/* --------------------------------------------------------------- ledger -- */
static int find_offset(const orc_t* P, const int* o) {
    for (int k = 0; k < P->nof; ++k) {
        const int* s = P->offs + 3 * k;
        if (s[0] == o[0] && s[1] == o[1] && s[2] == o[2]) return k;
    }
    return -1;
}

/* BondLedger::break_bond (ledger.hpp:21-26).  1 = newly broken, 0 = already,
 * -1 = not an in-band lattice pair (the reference's apply_corrections would
 * throw LedgerOutOfBand for such an entry, corrections.hpp:99-100). */
int orc_break_bond(orc_t* P, idx_t p, idx_t q) {
    int cp[3], cq[3], o[3], no[3];
    coords_of(P, p, cp);
    coords_of(P, q, cq);
    for (int d = 0; d < 3; ++d) { o[d] = cq[d] - cp[d]; no[d] = -o[d]; }
    const int k = find_offset(P, o), kn = find_offset(P, no);
    if (k < 0 || kn < 0) return -1;
    uint32_t* wp = P->ledger + p * P->lw;
    if (wp[k >> 5] & (1u << (k & 31))) return 0;
    wp[k >> 5] |= 1u << (k & 31);
    P->ledger[q * P->lw + (kn >> 5)] |= 1u << (kn & 31);
    P->total_broken++;
    return 1;
}

int orc_is_broken_k(const orc_t* P, idx_t p, int k) {
    return (P->ledger[p * P->lw + (k >> 5)] >> (k & 31)) & 1u;
}

idx_t orc_total_broken(const orc_t* P) { return P->total_broken; }

/* all broken bonds as sorted (p, q) pairs with p < q */
idx_t orc_ledger_pairs(const orc_t* P, idx_t* out, idx_t cap) {
    idx_t cnt = 0;
    for (idx_t p = 0; p < P->n; ++p)
        for (int s = 0; s < P->nof; ++s) {
            const int k = P->sorted_off[s];
            if (!orc_is_broken_k(P, p, k)) continue;
            const idx_t q = p + off_disp(P, P->offs + 3 * k);
            if (q <= p) continue;
            if (out && cnt < cap) { out[2 * cnt] = p; out[2 * cnt + 1] = q; }
            ++cnt;
        }
    return cnt;
}

/* oracles.hpp:123-137 random_ledger (shares the caller's rng stream) */
void orc_random_ledger(orc_t* P, orc_rng* r, int tries) {
    for (int t = 0; t < tries; ++t) {
        const idx_t p = (idx_t)(orc_rng_next(r) % (uint64_t)P->n);
        int c[3];
        coords_of(P, p, c);
        const int* o = P->offs + 3 * (orc_rng_next(r) % (uint32_t)P->nof);
        for (int d = 0; d < 3; ++d) c[d] += o[d];
        if (!in_lattice(P, c)) continue;
        orc_break_bond(P, p, lin_of(P, c));
    }
}

/* oracles.hpp:99-110 random_kernel */
void orc_random_kernel(orc_t* P, orc_rng* r) {
    memset(P->K, 0, sizeof(double) * (size_t)(P->np * P->ss));
    for (int k = 0; k < P->nof; ++k)
        for (int a = 0; a < P->dim; ++a)
            for (int b = a; b < P->dim; ++b)
                P->K[orc_pair_index(P->dim, a, b) * P->ss + stencil_index(P->dim, P->M, P->offs + 3 * k)] =
                    orc_rng_uniform(r, -1.0, 1.0);
    int zero[3] = {0, 0, 0};
    for (int a = 0; a < P->dim; ++a)
        for (int b = a; b < P->dim; ++b)
            P->K[orc_pair_index(P->dim, a, b) * P->ss + stencil_index(P->dim, P->M, zero)] =
                orc_rng_uniform(r, -1.0, 1.0);
    rebuild_regions(P);
}

/* --------------------------------------------------------------- forces -- */
/* f = A_hat u, the translation-invariant operator generated by the stencils
 * with zero padding outside the lattice: FastForce::apply
 * (convolution.hpp:249-259) restated as oracles.hpp:72-96 tbt_apply_all. */
static void apply_fast_rows(void* vc, idx_t p0, idx_t p1) {
    const orc_op_ctx* X = (const orc_op_ctx*)vc;
    const orc_t* P = X->P;
    const double* u = X->u;
    double* f = X->f;
    const int dim = P->dim;
    const idx_t n = P->n;
    int zero[3] = {0, 0, 0};
    const idx_t c0 = stencil_index(dim, P->M, zero);
    for (idx_t p = p0; p < p1; ++p) {
        int c[3];
        coords_of(P, p, c);
        double acc[3];
        for (int a = 0; a < dim; ++a) {
            double s = 0.0;
            for (int b = 0; b < dim; ++b) s += P->K[orc_pair_index(dim, a, b) * P->ss + c0] * u[b * n + p];
            acc[a] = s;
        }
        for (int k = 0; k < P->nof; ++k) {
            const int* o = P->offs + 3 * k;
            int q[3] = {c[0] + o[0], c[1] + o[1], c[2] + o[2]};
            if (!in_lattice(P, q)) continue;
            const idx_t qi = lin_of(P, q);
            const idx_t si = stencil_index(dim, P->M, o);
            for (int a = 0; a < dim; ++a) {
                double s = 0.0;
                for (int b = 0; b < dim; ++b) s += P->K[orc_pair_index(dim, a, b) * P->ss + si] * u[b * n + qi];
                acc[a] += s;
            }
        }
        for (int a = 0; a < dim; ++a) f[a * n + p] = acc[a];
    }
}

void orc_apply_fast(const orc_t* P, const double* u, double* f) {
    orc_op_ctx X = {P, u, f};
    orc_par_rows(P->n, apply_fast_rows, &X);
}

/* apply_corrections, corrections.hpp:76-110: surface diagonal then the
 * fracture gather (partners in ascending q, as BondLedger stores them). */
static void corrections_rows(void* vc, idx_t p0, idx_t p1) {
    const orc_op_ctx* X = (const orc_op_ctx*)vc;
    const orc_t* P = X->P;
    const double* u = X->u;
    double* f = X->f;
    const int dim = P->dim;
    const idx_t n = P->n;
    for (idx_t p = p0; p < p1; ++p) {
        if (!P->near_surface[p]) continue;
        for (int a = 0; a < dim; ++a) {
            if ((P->cmask[p] >> a) & 1u) continue;
            double acc = 0.0;
            for (int b = 0; b < dim; ++b) acc += P->De[orc_pair_index(dim, a, b) * n + p] * u[b * n + p];
            f[a * n + p] += acc;
        }
    }
    if (P->total_broken == 0) return;
    for (idx_t p = p0; p < p1; ++p) {
        for (int s = 0; s < P->nof; ++s) {
            const int k = P->sorted_off[s];
            if (!orc_is_broken_k(P, p, k)) continue;
            const int* o = P->offs + 3 * k;
            const idx_t q = p + off_disp(P, o);
            const idx_t si = stencil_index(dim, P->M, o);
            for (int a = 0; a < dim; ++a) {
                if ((P->cmask[p] >> a) & 1u) continue;
                double acc = 0.0;
                for (int b = 0; b < dim; ++b)
                    acc += P->K[orc_pair_index(dim, a, b) * P->ss + si] * (u[b * n + p] - u[b * n + q]);
                f[a * n + p] += acc;
            }
        }
    }
}

/* apply_corrections, corrections.hpp:76-110: per row, the surface diagonal
 * first, then the fracture gather (partners in ascending q, as BondLedger
 * stores them).  Rows are independent (each row only writes its own f). */
void orc_apply_corrections(const orc_t* P, const double* u, double* f) {
    orc_op_ctx X = {P, u, f};
    orc_par_rows(P->n, corrections_rows, &X);
}

/* The corrected force the reference's tests compare:
 * FastForce::apply + apply_corrections (e.g. tests/test_corrections.cpp:107-110). */
void orc_matvec(const orc_t* P, const double* u, double* f) {
    orc_apply_fast(P, u, f);
    orc_apply_corrections(P, u, f);
}

/* dense_force, reference.hpp:100-127 (meshfree sum over present unbroken bonds) */
static void dense_rows(void* vc, idx_t p0, idx_t p1) {
    const orc_op_ctx* X = (const orc_op_ctx*)vc;
    const orc_t* P = X->P;
    const double* u = X->u;
    double* f = X->f;
    const int dim = P->dim;
    const idx_t n = P->n;
    const double alpha = orc_alpha(P->E, P->delta, dim, P->thickness);
    const double vol = dim == 2 ? P->h * P->h * P->thickness : P->h * P->h * P->h;
    const double h = P->h;
    for (idx_t p = p0; p < p1; ++p) {
        int c[3];
        coords_of(P, p, c);
        double acc[3] = {0, 0, 0};
        for (int k = 0; k < P->nof; ++k) {
            const int* o = P->offs + 3 * k;
            int q[3] = {c[0] + o[0], c[1] + o[1], c[2] + o[2]};
            if (!in_lattice(P, q)) continue;
            if (P->total_broken && orc_is_broken_k(P, p, k)) continue;
            const idx_t qi = lin_of(P, q);
            long n2 = 0;
            for (int d = 0; d < dim; ++d) n2 += (long)o[d] * o[d];
            const double dist = h * sqrt((double)n2);
            const double lam = orc_volume_correction(dist, P->delta, h);
            const double scale = alpha * lam * vol / (dist * dist * dist);
            for (int a = 0; a < dim; ++a) {
                double s = 0.0;
                for (int b = 0; b < dim; ++b) s += (o[a] * h) * (o[b] * h) * (u[b * n + qi] - u[b * n + p]);
                acc[a] += scale * s;
            }
        }
        for (int a = 0; a < dim; ++a) f[a * n + p] = acc[a];
    }
}

void orc_dense_force(const orc_t* P, const double* u, double* f) {
    orc_op_ctx X = {P, u, f};
    orc_par_rows(P->n, dense_rows, &X);
}

/* Simulation::evaluate_force, timestepping.hpp:295-310 */
void orc_evaluate_force(const orc_t* P, const double* u, double* f) {
    const idx_t n = P->n;
    orc_matvec(P, u, f);
    for (int d = 0; d < P->dim; ++d)
        for (idx_t p = 0; p < n; ++p) f[d * n + p] += P->body[d * n + p];
    for (int k = 0; k < P->n_cons; ++k)
        for (idx_t p = 0; p < n; ++p) {
            int c[3];
            double x[3];
            coords_of(P, p, c);
            pos_of(P, c, x);
            if (!box_contains(P, P->cons[k].box, x)) continue;
            for (int d = 0; d < P->dim; ++d)
                if ((P->cons[k].dir_mask >> d) & 1u) f[d * n + p] = 0.0;
        }
}

/* ------------------------------------------------------------------- CG --
 * The reference has no CG (SURVEY.md sec.0 finding 3).  Restated here as
 * plain Hestenes-Stiefel CG on the SPD operator K := -A restricted to free
 * DOFs, y = -mask .* A(mask .* v), A = FastForce::apply + apply_corrections,
 * rhs b_f = mask .* (b + A u_c), u_c = prescribed displacement values on
 * constrained DOFs (SURVEY.md sec.8a "Operator definition").  x0 = 0, stop at
 * ||r|| <= tol ||b_f||.  hist (optional) receives x_1..x_nhist. */
static double dotv(const double* a, const double* b, idx_t m) {
    double s = 0.0;
    for (idx_t i = 0; i < m; ++i) s += a[i] * b[i];
    return s;
}

void orc_constrained_values(const orc_t* P, double* uc) {
    const idx_t n = P->n;
    memset(uc, 0, sizeof(double) * (size_t)(P->dim * n));
    for (int k = 0; k < P->n_cons; ++k) {
        if (P->cons[k].kind != 0) continue;
        for (idx_t p = 0; p < n; ++p) {
            int c[3];
            double x[3];
            coords_of(P, p, c);
            pos_of(P, c, x);
            if (!box_contains(P, P->cons[k].box, x)) continue;
            for (int d = 0; d < P->dim; ++d)
                if ((P->cons[k].dir_mask >> d) & 1u) uc[d * n + p] = P->cons[k].value;
        }
    }
}

static void apply_K(const orc_t* P, const double* v, double* y) {
    const idx_t n = P->n;
    orc_matvec(P, v, y);
    for (int d = 0; d < P->dim; ++d)
        for (idx_t p = 0; p < n; ++p)
            y[d * n + p] = ((P->cmask[p] >> d) & 1u) ? 0.0 : -y[d * n + p];
}

void orc_cg_rhs(const orc_t* P, const double* b, double* bf) {
    const idx_t n = P->n, m = P->dim * n;
    double* uc = (double*)malloc(sizeof(double) * (size_t)m);
    double* Auc = (double*)malloc(sizeof(double) * (size_t)m);
    orc_constrained_values(P, uc);
    orc_matvec(P, uc, Auc);
    for (int d = 0; d < P->dim; ++d)
        for (idx_t p = 0; p < n; ++p)
            bf[d * n + p] = ((P->cmask[p] >> d) & 1u) ? 0.0 : b[d * n + p] + Auc[d * n + p];
    free(uc);
    free(Auc);
}

int orc_cg(const orc_t* P, const double* b, double* x, double tol, int maxit, int* iters,
           double* relres, double* hist, int nhist) {
    const idx_t n = P->n, m = P->dim * n;
    double* r = (double*)malloc(sizeof(double) * (size_t)m);
    double* p = (double*)malloc(sizeof(double) * (size_t)m);
    double* q = (double*)malloc(sizeof(double) * (size_t)m);
    orc_cg_rhs(P, b, r);
    memset(x, 0, sizeof(double) * (size_t)m);
    memcpy(p, r, sizeof(double) * (size_t)m);
    double rr = dotv(r, r, m);
    const double bnorm = sqrt(rr);
    int k = 0;
    double rel = bnorm > 0 ? 1.0 : 0.0;
    while (bnorm > 0 && k < maxit) {
        apply_K(P, p, q);
        const double pq = dotv(p, q, m);
        const double alpha = rr / pq;
        for (idx_t i = 0; i < m; ++i) { x[i] += alpha * p[i]; r[i] -= alpha * q[i]; }
        const double rr1 = dotv(r, r, m);
        ++k;
        if (hist && k <= nhist) memcpy(hist + (size_t)(k - 1) * m, x, sizeof(double) * (size_t)m);
        rel = sqrt(rr1) / bnorm;
        if (rel <= tol) break;
        const double beta = rr1 / rr;
        for (idx_t i = 0; i < m; ++i) p[i] = r[i] + beta * p[i];
        rr = rr1;
    }
    /* add the prescribed values back: full displacement */
    orc_constrained_values(P, q);
    for (idx_t i = 0; i < m; ++i) x[i] += q[i];
    if (iters) *iters = k;
    if (relres) *relres = rel;
    free(r); free(p); free(q);
    return 0;
}

/* relative residual of a full displacement x: ||mask (A x + b)|| / ||b_f|| */
double orc_static_residual(const orc_t* P, const double* b, const double* x) {
    const idx_t n = P->n, m = P->dim * n;
    double* f = (double*)malloc(sizeof(double) * (size_t)m);
    double* bf = (double*)malloc(sizeof(double) * (size_t)m);
    orc_matvec(P, x, f);
    orc_cg_rhs(P, b, bf);
    double num = 0, den = 0;
    for (int d = 0; d < P->dim; ++d)
        for (idx_t p = 0; p < n; ++p) {
            if ((P->cmask[p] >> d) & 1u) continue;
            const double rres = f[d * n + p] + b[d * n + p];
            num += rres * rres;
            den += bf[d * n + p] * bf[d * n + p];
        }
    free(f);
    free(bf);
    return den > 0 ? sqrt(num / den) : sqrt(num);
}

/* ------------------------------------------------------------- fracture -- */
/* bond_stretch, fracture.hpp:17-29 */
double orc_bond_stretch(int dim, const double* xp, const double* xq, const double* up,
                        const double* uq) {
    double len0 = 0.0, len1 = 0.0;
    for (int d = 0; d < dim; ++d) {
        const double r = xq[d] - xp[d];
        const double e = r + uq[d] - up[d];
        len0 += r * r;
        len1 += e * e;
    }
    len0 = sqrt(len0);
    len1 = sqrt(len1);
    return (len1 - len0) / len0;
}

/* update_bonds, fracture.hpp:204-231.  Returns the number of newly broken
 * bonds; out (cap pairs) receives them in (p, offset) visiting order. */
idx_t orc_update_bonds(orc_t* P, const double* u, double s0, const double* watch, idx_t* out,
                       idx_t cap) {
    const idx_t n = P->n;
    const int dim = P->dim;
    idx_t cnt = 0;
    for (idx_t p = 0; p < n; ++p) {
        int cp[3];
        double xp[3], up[3];
        coords_of(P, p, cp);
        pos_of(P, cp, xp);
        if (watch && !box_contains(P, watch, xp)) continue;
        for (int d = 0; d < dim; ++d) up[d] = u[d * n + p];
        for (int k = 0; k < P->nof; ++k) {
            const int* o = P->offs + 3 * k;
            int cq[3] = {cp[0] + o[0], cp[1] + o[1], cp[2] + o[2]};
            if (!in_lattice(P, cq)) continue;
            const idx_t q = lin_of(P, cq);
            if (q < p) continue;
            double xq[3], uq[3];
            pos_of(P, cq, xq);
            if (watch && !box_contains(P, watch, xq)) continue;
            if (orc_is_broken_k(P, p, k)) continue;
            for (int d = 0; d < dim; ++d) uq[d] = u[d * n + q];
            if (orc_bond_stretch(dim, xp, xq, up, uq) >= s0) {
                orc_break_bond(P, p, q);
                if (out && cnt < cap) { out[2 * cnt] = p; out[2 * cnt + 1] = q; }
                ++cnt;
            }
        }
    }
    return cnt;
}

/* orient2_sign / segments_cross, fracture.hpp:38-55 */
static int orient2_sign(const double* a, const double* b, const double* c) {
    const double t1 = (b[0] - a[0]) * (c[1] - a[1]);
    const double t2 = (b[1] - a[1]) * (c[0] - a[0]);
    const double det = t1 - t2;
    const double tol = 1e-10 * (fabs(t1) + fabs(t2));
    if (fabs(det) <= tol) return 0;
    return det > 0.0 ? 1 : -1;
}

static int segments_cross(const double* a, const double* b, const double* p, const double* q) {
    const int o1 = orient2_sign(a, b, p), o2 = orient2_sign(a, b, q);
    const int o3 = orient2_sign(p, q, a), o4 = orient2_sign(p, q, b);
    return o1 * o2 < 0 && o3 * o4 < 0;
}

/* CrackSpec<2>::bond_crosses for one segment (fracture.hpp:75-92) */
static int segment_crosses(const double* seg, const double* p, const double* q) {
    const double a[2] = {seg[0], seg[1]}, b[2] = {seg[2], seg[3]};
    const double width = seg[4];
    if (width <= 0.0) return segments_cross(a, b, p, q);
    const double t[2] = {b[0] - a[0], b[1] - a[1]};
    const double len = sqrt(t[0] * t[0] + t[1] * t[1]);
    if (len == 0.0) return 0;
    const double nrm[2] = {-t[1] / len, t[0] / len};
    const double sides[2] = {0.5 * width, -0.5 * width};
    for (int s = 0; s < 2; ++s) {
        const double side = sides[s];
        const double fa[2] = {a[0] + side * nrm[0], a[1] + side * nrm[1]};
        const double fb[2] = {b[0] + side * nrm[0], b[1] + side * nrm[1]};
        if (segments_cross(fa, fb, p, q)) return 1;
    }
    return 0;
}

/* CrackSpec<3>::bond_crosses for one notch (fracture.hpp:122-146).
 * notch = {axis, plane, width, lo0, lo1, lo2, hi0, hi1, hi2} */
static int notch_crosses(const double* nt, const double* p, const double* q) {
    const int axis = (int)nt[0];
    const double plane = nt[1], width = nt[2];
    const double faces[2] = {plane - 0.5 * width, plane + 0.5 * width};
    const int n_faces = width > 0.0 ? 2 : 1;
    for (int fi = 0; fi < n_faces; ++fi) {
        const double face = width > 0.0 ? faces[fi] : plane;
        const double dp = p[axis] - face, dq = q[axis] - face;
        const double tol = 1e-12 * (fabs(p[axis]) + fabs(q[axis]) + fabs(face));
        if (fabs(dp) <= tol || fabs(dq) <= tol) continue;
        if (!((dp > 0.0 && dq < 0.0) || (dp < 0.0 && dq > 0.0))) continue;
        const double t = dp / (dp - dq);
        int inside = 1;
        for (int d = 0; d < 3; ++d) {
            if (d == axis) continue;
            const double x = p[d] + t * (q[d] - p[d]);
            inside = inside && x >= nt[3 + d] && x <= nt[6 + d];
        }
        if (inside) return 1;
    }
    return 0;
}

/* seed_cracks, fracture.hpp:164-198, one crack element at a time (the
 * ledger is a set, so seeding the union equals seeding each element). */
static idx_t seed_generic(orc_t* P, const double* bb_lo, const double* bb_hi, const double* geom,
                          int is_notch) {
    int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    const double pad = P->delta + P->h;
    for (int d = 0; d < P->dim; ++d) {
        int l = (int)floor((bb_lo[d] - pad - P->origin[d]) / P->h);
        int u = (int)ceil((bb_hi[d] + pad - P->origin[d]) / P->h);
        lo[d] = l > 0 ? l : 0;
        hi[d] = u < P->dims[d] - 1 ? u : P->dims[d] - 1;
    }
    idx_t added = 0;
    int c[3];
    for (c[0] = lo[0]; c[0] <= hi[0]; ++c[0])
        for (c[1] = lo[1]; c[1] <= hi[1]; ++c[1])
            for (c[2] = lo[2]; c[2] <= hi[2]; ++c[2]) {
                const idx_t p = lin_of(P, c);
                double xp[3];
                pos_of(P, c, xp);
                for (int k = 0; k < P->nof; ++k) {
                    const int* o = P->offs + 3 * k;
                    int qc[3] = {c[0] + o[0], c[1] + o[1], c[2] + o[2]};
                    if (!in_lattice(P, qc)) continue;
                    const idx_t q = lin_of(P, qc);
                    if (q < p) continue;
                    double xq[3];
                    pos_of(P, qc, xq);
                    const int cross = is_notch ? notch_crosses(geom, xp, xq) : segment_crosses(geom, xp, xq);
                    if (cross && orc_break_bond(P, p, q) == 1) ++added;
                }
            }
    return added;
}

/* segment = {ax, ay, bx, by, width} (CrackSpec<2>::Segment) */
idx_t orc_seed_segment(orc_t* P, const double* seg) {
    double lo[3], hi[3];
    for (int d = 0; d < 2; ++d) {
        const double a = seg[d], b = seg[2 + d], w = seg[4];
        lo[d] = fmin(a - w, b - w);
        hi[d] = fmax(a + w, b + w);
    }
    return seed_generic(P, lo, hi, seg, 0);
}

/* notch = {axis, plane, width, lo0, lo1, lo2, hi0, hi1, hi2} (CrackSpec<3>::Notch) */
idx_t orc_seed_notch(orc_t* P, const double* nt) {
    double lo[3], hi[3];
    const int axis = (int)nt[0];
    for (int d = 0; d < 3; ++d) {
        lo[d] = d == axis ? nt[1] - nt[2] : nt[3 + d];
        hi[d] = d == axis ? nt[1] + nt[2] : nt[6 + d];
    }
    return seed_generic(P, lo, hi, nt, 1);
}

/* ------------------------------------------------------- velocity Verlet --
 * Simulation<Dim> with Integrator::Vv (timestepping.hpp:167-351). */
static void enforce_constraints(orc_t* P) {
    const idx_t n = P->n;
    for (int k = 0; k < P->n_cons; ++k) {
        const orc_constraint* cs = &P->cons[k];
        for (int d = 0; d < P->dim; ++d) {
            if (!((cs->dir_mask >> d) & 1u)) continue;
            for (idx_t p = 0; p < n; ++p) {
                int c[3];
                double x[3];
                coords_of(P, p, c);
                pos_of(P, c, x);
                if (!box_contains(P, cs->box, x)) continue;
                if (cs->kind == 0) { P->u[d * n + p] = cs->value; P->v[d * n + p] = 0.0; }
                else { P->u[d * n + p] = cs->value * P->t; P->v[d * n + p] = cs->value; }
            }
        }
    }
}

void orc_sim_init(orc_t* P, double dt) {
    const size_t m = (size_t)(P->dim * P->n);
    free(P->u); free(P->v); free(P->f); free(P->f_prev);
    P->u = (double*)calloc(m, sizeof(double));
    P->v = (double*)calloc(m, sizeof(double));
    P->f = (double*)calloc(m, sizeof(double));
    P->f_prev = (double*)calloc(m, sizeof(double));
    P->t = 0.0;
    P->dt = dt;
    P->step = 0;
    P->force_ready = 0;
    P->integrator = 0;
    enforce_constraints(P);
}

/* Simulation<Dim> with Integrator::Adr: adr_mass (timestepping.hpp:150-162)
 * over the in-band offsets in for_each_offset order (kernel.hpp:71-89);
 * fixed_damping NaN = adaptive (std::nullopt). */
void orc_sim_init_adr(orc_t* P, double dt, double fixed_damping) {
    orc_sim_init(P, dt);
    free(P->vh);
    P->vh = (double*)calloc((size_t)(P->dim * P->n), sizeof(double));
    P->integrator = 1;
    P->fixed = fixed_damping == fixed_damping;
    P->fixed_c = P->fixed ? fixed_damping : 0.0;
    P->last_c = 0.0;
    const int side = 2 * P->M + 1;
    for (int a = 0; a < P->dim; ++a) {
        double row = 0.0;
        for (int b = 0; b < P->dim; ++b) {
            double off_abs = 0.0;
            const int pr = orc_pair_index(P->dim, a, b);
            for (int k = 0; k < P->nof; ++k) {
                const int* o = &P->offs[3 * k];
                idx_t si = 0;
                for (int d = P->dim - 1; d >= 0; --d) si = si * side + (o[d] + P->M);
                off_abs += fabs(P->K[pr * P->ss + si]);
            }
            row += 2.0 * off_abs;
        }
        P->mass[a] = 0.25 * dt * dt * row;
    }
}

double orc_sim_adr_damping(const orc_t* P) { return P->last_c; }
void orc_sim_adr_mass(const orc_t* P, double* m) { for (int a = 0; a < P->dim; ++a) m[a] = P->mass[a]; }

/* AdrIntegrator::advance + estimate_damping, timestepping.hpp:86-139 */
static void adr_advance(orc_t* P) {
    const idx_t n = P->n;
    const double dt = P->dt;
    if (P->step == 0) {
        for (int a = 0; a < P->dim; ++a) {
            const double inv_m = 1.0 / P->mass[a];
            for (idx_t p = 0; p < n; ++p) {
                if ((P->cmask[p] >> a) & 1u) continue;
                P->vh[a * n + p] = 0.5 * dt * P->f[a * n + p] * inv_m;
            }
        }
    } else {
        double c;
        if (P->fixed) {
            c = P->fixed_c;
        } else {
            double num = 0.0, den = 0.0;
            for (int a = 0; a < P->dim; ++a)
                for (idx_t p = 0; p < n; ++p) {
                    if ((P->cmask[p] >> a) & 1u) continue;
                    const double up = P->u[a * n + p], vh = P->vh[a * n + p];
                    double k = 0.0;
                    if (vh != 0.0) k = -(P->f[a * n + p] - P->f_prev[a * n + p]) / (P->mass[a] * dt * vh);
                    if (k > 0.0) num += up * up * k;
                    den += up * up;
                }
            if (den <= 0.0 || num <= 0.0) c = 0.0;
            else {
                c = 2.0 * sqrt(num / den);
                if (1.9 / dt < c) c = 1.9 / dt;
            }
        }
        P->last_c = c;
        const double lead = 2.0 - c * dt, trail = 1.0 / (2.0 + c * dt);
        for (int a = 0; a < P->dim; ++a) {
            const double inv_m = 1.0 / P->mass[a];
            for (idx_t p = 0; p < n; ++p) {
                if ((P->cmask[p] >> a) & 1u) continue;
                P->vh[a * n + p] = (lead * P->vh[a * n + p] + 2.0 * dt * P->f[a * n + p] * inv_m) * trail;
            }
        }
    }
    for (int a = 0; a < P->dim; ++a)
        for (idx_t p = 0; p < n; ++p) {
            if ((P->cmask[p] >> a) & 1u) continue;
            P->u[a * n + p] += dt * P->vh[a * n + p];
        }
}

void orc_sim_set_velocity(orc_t* P, const double* v) {
    memcpy(P->v, v, sizeof(double) * (size_t)(P->dim * P->n));
}

/* Simulation::step, timestepping.hpp:209-241 (VV branch).  s0 < 0 disables
 * fracture.  Returns the number of newly broken bonds. */
idx_t orc_sim_step(orc_t* P, double s0, const double* watch) {
    const idx_t n = P->n;
    const int dim = P->dim;
    const double dt = P->dt, inv_rho = 1.0 / P->rho;
    if (!P->force_ready) { orc_evaluate_force(P, P->u, P->f); P->force_ready = 1; }
    if (P->integrator == 1) {  /* ADR branch, timestepping.hpp:215-220 */
        adr_advance(P);
        P->t += dt;
        enforce_constraints(P);
        double* tmp = P->f_prev; P->f_prev = P->f; P->f = tmp;
        orc_evaluate_force(P, P->u, P->f);
        idx_t nb = 0;
        if (s0 >= 0.0) nb = orc_update_bonds(P, P->u, s0, watch, NULL, 0);
        P->step++;
        return nb;
    }
    for (int a = 0; a < dim; ++a)   /* vv_drift :312-322 */
        for (idx_t p = 0; p < n; ++p) {
            if ((P->cmask[p] >> a) & 1u) continue;
            P->u[a * n + p] += dt * P->v[a * n + p] + 0.5 * dt * dt * P->f[a * n + p] * inv_rho;
        }
    P->t += dt;
    enforce_constraints(P);
    double* tmp = P->f_prev; P->f_prev = P->f; P->f = tmp;
    orc_evaluate_force(P, P->u, P->f);
    for (int a = 0; a < dim; ++a)   /* vv_kick :324-334 */
        for (idx_t p = 0; p < n; ++p) {
            if ((P->cmask[p] >> a) & 1u) continue;
            P->v[a * n + p] += 0.5 * dt * (P->f_prev[a * n + p] + P->f[a * n + p]) * inv_rho;
        }
    enforce_constraints(P);
    idx_t nb = 0;
    if (s0 >= 0.0) nb = orc_update_bonds(P, P->u, s0, watch, NULL, 0);
    P->step++;
    return nb;
}

void orc_sim_get(const orc_t* P, double* u, double* v, double* f, double* t) {
    const size_t m = sizeof(double) * (size_t)(P->dim * P->n);
    if (u) memcpy(u, P->u, m);
    if (v) memcpy(v, P->v, m);
    if (f) memcpy(f, P->f, m);
    if (t) *t = P->t;
}
