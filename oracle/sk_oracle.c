/*
 * sk_oracle.c -- CPU restatement of the reference hot path (see sk_oracle.h).
 * TEST INFRASTRUCTURE: the checker for the B200 library, never the product.
 *
 * Every function cites the reference file:line it restates. Compile with
 * -ffp-contract=off: the arithmetic order written here IS the contract.
 */
#define _GNU_SOURCE
#include "sk_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ------------------------------------------------------------------------- */
/* Contract constants                       */
/* ------------------------------------------------------------------------- */
#define R1_LANES 32
#define R1_LROWS 16
#define R1_SEG (R1_LANES * R1_LROWS) /* rows per segment */
#define R2_TILE 32
#define HH_RATIO 1e-6      /* sigma_min/sigma_max below this -> Householder path */

/* Golden-generation build (libsk_oracle_mt.so, -fopenmp): loops over independent
 * outputs run on all host threads. Every output keeps its own operation sequence,
 * so results are bitwise those of the serial build (tests/test_oracle_pins.py
 * checks both builds against the same fixtures). The default build (the CPU
 * baseline) has no OpenMP, like the reference (proj/CMakeLists.txt:3-15). */
#ifdef _OPENMP
#define SKO_STR(x) #x
#define SKO_PAR(cond) _Pragma(SKO_STR(omp parallel for schedule(static) if(cond)))
#else
#define SKO_PAR(cond)
#endif
#define PAR_MIN 4096 /* elements below which a loop stays serial */

/* Lean Lanczos storage (golden generation at configs whose bases exceed host RAM):
 * only the last LEAN_KEEP blocks are kept; a clean-up pass (which needs every block)
 * or a request for V fails loudly instead. */
#define LEAN_KEEP 3
static int g_lean = 0;
void sko_set_lean(int on) { g_lean = on; }

static __thread char g_err[512];
static void set_err(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
}
const char* sko_last_error(void) { return g_err; }

int sko_contract_constants(int64_t* out4) {
    out4[0] = R1_SEG;
    out4[1] = R1_LANES;
    out4[2] = R2_TILE;
    out4[3] = 0;
    return 0;
}

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

static void* xcalloc(size_t n, size_t sz) {
    void* p = calloc(n ? n : 1, sz ? sz : 1);
    if (!p) {
        fprintf(stderr, "sk_oracle: out of memory (%zu x %zu)\n", n, sz);
        abort();
    }
    return p;
}

/* ------------------------------------------------------------------------- */
/* Dense column-major matrices (dense_matrix.hpp:12-47)                       */
/* ------------------------------------------------------------------------- */
typedef struct {
    int64_t rows, cols;
    double* a;
} dmat;
#define AT(m, i, j) ((m).a[(size_t)(j) * (size_t)(m).rows + (size_t)(i)])

static dmat dm_new(int64_t r, int64_t c) {
    dmat m = {r, c, (double*)xcalloc((size_t)(r * c), sizeof(double))};
    return m;
}
static void dm_free(dmat* m) {
    free(m->a);
    m->a = NULL;
    m->rows = m->cols = 0;
}
static dmat dm_copy(const dmat* x) {
    dmat m = dm_new(x->rows, x->cols);
    memcpy(m.a, x->a, sizeof(double) * (size_t)(x->rows * x->cols));
    return m;
}
/* embed_to (factorized_solvers.cpp:26-33): zero-padded copy. */
static dmat dm_embed(const dmat* x, int64_t rows, int64_t cols) {
    dmat m = dm_new(rows, cols);
    for (int64_t j = 0; j < x->cols; ++j)
        memcpy(m.a + j * rows, x->a + j * x->rows, sizeof(double) * (size_t)x->rows);
    return m;
}
/* axpy (dense_matrix.cpp:105-108): y += alpha * x, mul then add per entry. */
static void dm_axpy(double alpha, const dmat* x, dmat* y) {
    const size_t n = (size_t)(x->rows * x->cols);
    SKO_PAR(n >= PAR_MIN)
    for (size_t i = 0; i < n; ++i) y->a[i] = y->a[i] + alpha * x->a[i];
}
/* matmul_a_bt (dense_matrix.cpp:124-129): out(i,j) = sum_t a(i,t) b(j,t). */
static dmat dm_a_bt(const dmat* a, const dmat* b) {
    dmat o = dm_new(a->rows, b->rows);
    for (int64_t j = 0; j < b->rows; ++j)
        for (int64_t i = 0; i < a->rows; ++i) {
            double acc = 0.0;
            for (int64_t t = 0; t < a->cols; ++t) acc = acc + AT(*a, i, t) * AT(*b, j, t);
            AT(o, i, j) = acc;
        }
    return o;
}

/* ------------------------------------------------------------------------- */
/* Reductions                                                                 */
/* ------------------------------------------------------------------------- */
static void butterfly32(double* lane) {
    double tmp[R1_LANES];
    for (int d = 16; d >= 1; d >>= 1) {
        for (int l = 0; l < R1_LANES; ++l) tmp[l] = lane[l] + lane[l ^ d];
        memcpy(lane, tmp, sizeof tmp);
    }
}
/* canonical pairwise tree: node(l,i) = node(l-1,2i) + node(l-1,2i+1) or node(l-1,2i) */
static double tree_reduce(double* a, int64_t count) {
    if (count <= 0) return 0.0;
    while (count > 1) {
        const int64_t half = (count + 1) / 2;
        for (int64_t i = 0; i < half; ++i)
            a[i] = (2 * i + 1 < count) ? a[2 * i] + a[2 * i + 1] : a[2 * i];
        count = half;
    }
    return a[0];
}

/* R1: sum_{row0 <= i < n} x[i]*y[i] by the segment contract. */
static double r1_dot(const double* x, const double* y, int64_t n, int64_t row0) {
    if (n <= 0) return 0.0;
    const int64_t S = (n + R1_SEG - 1) / R1_SEG;
    double* seg = (double*)xcalloc((size_t)S, sizeof(double));
    SKO_PAR(S >= 64)
    for (int64_t g = 0; g < S; ++g) {
        double lane[R1_LANES];
        for (int l = 0; l < R1_LANES; ++l) {
            double acc = 0.0;
            for (int m = 0; m < R1_LROWS; ++m) {
                const int64_t i = g * R1_SEG + l + R1_LANES * m;
                if (i < n && i >= row0) acc = acc + x[i] * y[i];
            }
            lane[l] = acc;
        }
        butterfly32(lane);
        seg[g] = lane[0];
    }
    const double r = tree_reduce(seg, S);
    free(seg);
    return r;
}
static double seq_dot(const double* x, const double* y, int64_t n, int64_t row0) {
    double acc = 0.0;
    for (int64_t i = row0; i < n; ++i) acc = acc + x[i] * y[i];
    return acc;
}
typedef double (*dot_fn)(const double*, const double*, int64_t, int64_t);

/* R2: sum over window rows x cols of a(i,j)*b(i,j) by the tile contract. */
static double r2_inner(const dmat* a, const dmat* b, int64_t rows, int64_t cols) {
    if (rows <= 0 || cols <= 0) return 0.0;
    const int64_t nti = (rows + R2_TILE - 1) / R2_TILE, ntj = (cols + R2_TILE - 1) / R2_TILE;
    double* colres = (double*)xcalloc((size_t)ntj, sizeof(double));
    double* tiles_all = (double*)xcalloc((size_t)(nti * ntj), sizeof(double));
    SKO_PAR(ntj >= 8)
    for (int64_t tj = 0; tj < ntj; ++tj) {
        double lane[R1_LANES];
        double* tiles = tiles_all + tj * nti;
        for (int64_t ti = 0; ti < nti; ++ti) {
            for (int l = 0; l < R1_LANES; ++l) {
                const int64_t i = ti * R2_TILE + l;
                double acc = 0.0;
                if (i < rows)
                    for (int c = 0; c < R2_TILE; ++c) {
                        const int64_t j = tj * R2_TILE + c;
                        if (j < cols) acc = acc + AT(*a, i, j) * AT(*b, i, j);
                    }
                lane[l] = acc;
            }
            butterfly32(lane);
            tiles[ti] = lane[0];
        }
        colres[tj] = tree_reduce(tiles, nti);
    }
    const double r = tree_reduce(colres, ntj);
    free(colres);
    free(tiles_all);
    return r;
}
/* frobenius_inner / windowed_inner (dense_matrix.cpp:131-152): sequential. */
static double seq_window_inner(const dmat* a, const dmat* b, int64_t rows, int64_t cols) {
    double acc = 0.0;
    for (int64_t j = 0; j < cols; ++j)
        for (int64_t i = 0; i < rows; ++i) acc = acc + AT(*a, i, j) * AT(*b, i, j);
    return acc;
}
static double win_inner(int mode, const dmat* a, const dmat* b, int64_t rows, int64_t cols) {
    return mode == SKO_REPRODUCIBLE ? r2_inner(a, b, rows, cols) : seq_window_inner(a, b, rows, cols);
}

/* ------------------------------------------------------------------------- */
/* RNG: mt19937_64 + Box-Muller (problems.cpp:65-96), libstdc++ uniform      */
/* ------------------------------------------------------------------------- */
typedef struct {
    uint64_t mt[312];
    int idx;
} mt64;
static void mt64_seed(mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
}
static uint64_t mt64_next(mt64* g) {
    if (g->idx >= 312) {
        const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
        for (int i = 0; i < 312; ++i) {
            const uint64_t x = (g->mt[i] & UM) | (g->mt[(i + 1) % 312] & LM);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
        }
        g->idx = 0;
    }
    uint64_t y = g->mt[g->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}
/* uniform_open_closed (problems.cpp:68-70) */
static double uniform_oc(mt64* g) { return ((double)(mt64_next(g) >> 11) + 1.0) * 0x1.0p-53; }
/* std::generate_canonical<double,53>(mt19937_64) as in libstdc++ (GCC 13) */
static double canonical(mt64* g) {
    double sum = (double)mt64_next(g);
    double r = sum / 18446744073709551616.0;
    if (r >= 1.0) r = nextafter(1.0, 0.0);
    return r;
}
/* uniform_real_distribution(a,b): canonical*(b-a)+a */
static double uniform_ab(mt64* g, double a, double b) { return canonical(g) * (b - a) + a; }

void sko_random_rhs(int64_t rows, int64_t s, uint64_t seed, double* out) {
    mt64 g;
    mt64_seed(&g, seed);
    double spare = 0.0;
    int have = 0;
    const int64_t count = rows * s;
    for (int64_t i = 0; i < count; ++i) {
        if (have) {
            out[i] = spare;
            have = 0;
        } else {
            const double u1 = uniform_oc(&g), u2 = uniform_oc(&g);
            const double radius = sqrt(-2.0 * log(u1));
            const double angle = 2.0 * M_PI * u2;
            out[i] = radius * cos(angle);
            spare = radius * sin(angle);
            have = 1;
        }
    }
}
/* oracles::random_dense (tests/oracles.hpp:39-46) */
void sko_random_dense(int64_t rows, int64_t cols, uint64_t seed, double* out) {
    mt64 g;
    mt64_seed(&g, seed);
    for (int64_t j = 0; j < cols; ++j)
        for (int64_t i = 0; i < rows; ++i) out[j * rows + i] = uniform_ab(&g, -1.0, 1.0);
}

/* ------------------------------------------------------------------------- */
/* CSR (sparse_matrix.cpp:12-132)                                             */
/* ------------------------------------------------------------------------- */
void sko_csr_free(sko_csr* a) {
    if (!a) return;
    free(a->row_ptr);
    free(a->col_idx);
    free(a->values);
    memset(a, 0, sizeof *a);
}
static int csr_validate(const sko_csr* a) { /* sparse_matrix.cpp:16-31 */
    if (a->n_rows < 0 || a->n_cols < 0) return set_err("SparseMatrix: negative dimension"), SKO_ERR_INVALID_MATRIX;
    if (a->row_ptr[0] != 0 || a->row_ptr[a->n_rows] != a->nnz)
        return set_err("SparseMatrix: row_ptr endpoints inconsistent with nnz"), SKO_ERR_INVALID_MATRIX;
    for (int64_t i = 0; i < a->n_rows; ++i) {
        if (a->row_ptr[i] > a->row_ptr[i + 1])
            return set_err("SparseMatrix: row_ptr not nondecreasing"), SKO_ERR_INVALID_MATRIX;
        for (int64_t k = a->row_ptr[i]; k < a->row_ptr[i + 1]; ++k) {
            if (a->col_idx[k] < 0 || a->col_idx[k] >= a->n_cols)
                return set_err("SparseMatrix: column index out of range"), SKO_ERR_INVALID_MATRIX;
            if (k > a->row_ptr[i] && a->col_idx[k] <= a->col_idx[k - 1])
                return set_err("SparseMatrix: column indices not strictly increasing in row"),
                       SKO_ERR_INVALID_MATRIX;
        }
    }
    return SKO_OK;
}

typedef struct {
    const int64_t* rows;
    const int64_t* cols;
} trip_ctx;
static __thread trip_ctx g_trip;
static int trip_cmp(const void* pa, const void* pb) {
    const int64_t a = *(const int64_t*)pa, b = *(const int64_t*)pb;
    if (g_trip.rows[a] != g_trip.rows[b]) return g_trip.rows[a] < g_trip.rows[b] ? -1 : 1;
    if (g_trip.cols[a] != g_trip.cols[b]) return g_trip.cols[a] < g_trip.cols[b] ? -1 : 1;
    return a < b ? -1 : (a > b); /* stable: duplicates summed in input order */
}
/* from_triplets (sparse_matrix.cpp:34-69) */
int sko_csr_from_triplets(int64_t n_rows, int64_t n_cols, int64_t count, const int64_t* rows,
                          const int64_t* cols, const double* vals, sko_csr* out) {
    for (int64_t k = 0; k < count; ++k)
        if (rows[k] < 0 || rows[k] >= n_rows || cols[k] < 0 || cols[k] >= n_cols)
            return set_err("from_triplets: index out of range"), SKO_ERR_INVALID_MATRIX;
    int64_t* order = (int64_t*)xcalloc((size_t)count, sizeof(int64_t));
    for (int64_t k = 0; k < count; ++k) order[k] = k;
    g_trip.rows = rows;
    g_trip.cols = cols;
    qsort(order, (size_t)count, sizeof(int64_t), trip_cmp);
    out->n_rows = n_rows;
    out->n_cols = n_cols;
    out->row_ptr = (int64_t*)xcalloc((size_t)n_rows + 1, sizeof(int64_t));
    out->col_idx = (int64_t*)xcalloc((size_t)count, sizeof(int64_t));
    out->values = (double*)xcalloc((size_t)count, sizeof(double));
    int64_t nz = 0, last_r = -1, last_c = -1;
    for (int64_t q = 0; q < count; ++q) {
        const int64_t idx = order[q];
        if (nz > 0 && rows[idx] == last_r && cols[idx] == last_c) {
            out->values[nz - 1] = out->values[nz - 1] + vals[idx];
        } else {
            out->row_ptr[rows[idx] + 1]++;
            out->col_idx[nz] = cols[idx];
            out->values[nz] = vals[idx];
            ++nz;
            last_r = rows[idx];
            last_c = cols[idx];
        }
    }
    for (int64_t i = 1; i <= n_rows; ++i) out->row_ptr[i] += out->row_ptr[i - 1];
    out->nnz = nz;
    free(order);
    return csr_validate(out);
}

/* transposed (sparse_matrix.cpp:80-95): rows of A^T in ascending source row. */
int sko_csr_transpose(const sko_csr* a, sko_csr* out) {
    out->n_rows = a->n_cols;
    out->n_cols = a->n_rows;
    out->nnz = a->nnz;
    out->row_ptr = (int64_t*)xcalloc((size_t)a->n_cols + 1, sizeof(int64_t));
    out->col_idx = (int64_t*)xcalloc((size_t)a->nnz, sizeof(int64_t));
    out->values = (double*)xcalloc((size_t)a->nnz, sizeof(double));
    for (int64_t k = 0; k < a->nnz; ++k) out->row_ptr[a->col_idx[k] + 1]++;
    for (int64_t i = 1; i <= a->n_cols; ++i) out->row_ptr[i] += out->row_ptr[i - 1];
    int64_t* next = (int64_t*)xcalloc((size_t)a->n_cols + 1, sizeof(int64_t));
    memcpy(next, out->row_ptr, sizeof(int64_t) * (size_t)a->n_cols);
    for (int64_t i = 0; i < a->n_rows; ++i)
        for (int64_t k = a->row_ptr[i]; k < a->row_ptr[i + 1]; ++k) {
            const int64_t pos = next[a->col_idx[k]]++;
            out->col_idx[pos] = i;
            out->values[pos] = a->values[k];
        }
    free(next);
    return SKO_OK;
}

static double csr_fro(const sko_csr* a) {
    double acc = 0.0;
    for (int64_t k = 0; k < a->nnz; ++k) acc = acc + a->values[k] * a->values[k];
    return sqrt(acc);
}
/* is_symmetric (sparse_matrix.cpp:109-132) */
int sko_csr_is_symmetric(const sko_csr* a, double tol) {
    if (a->n_rows != a->n_cols) return 0;
    sko_csr at;
    sko_csr_transpose(a, &at);
    double diff2 = 0.0;
    for (int64_t i = 0; i < a->n_rows; ++i) {
        int64_t ka = a->row_ptr[i], kb = at.row_ptr[i];
        const int64_t ea = a->row_ptr[i + 1], eb = at.row_ptr[i + 1];
        while (ka < ea || kb < eb) {
            const int64_t ca = ka < ea ? a->col_idx[ka] : a->n_cols;
            const int64_t cb = kb < eb ? at.col_idx[kb] : a->n_cols;
            double d;
            if (ca < cb)
                d = a->values[ka++];
            else if (cb < ca)
                d = -at.values[kb++];
            else
                d = a->values[ka++] - at.values[kb++];
            diff2 = diff2 + d * d;
        }
    }
    sko_csr_free(&at);
    const double fa = csr_fro(a);
    return sqrt(diff2) <= tol * (fa > 1e-300 ? fa : 1e-300);
}

/* Direct CSR emitters for the stencil generators: rows come out with columns in
 * ascending order, identical to from_triplets on the reference's triplet stream
 * (problems.cpp:10-60; no duplicates occur). */
static void csr_alloc(sko_csr* o, int64_t n, int64_t maxnnz) {
    o->n_rows = o->n_cols = n;
    o->row_ptr = (int64_t*)xcalloc((size_t)n + 1, sizeof(int64_t));
    o->col_idx = (int64_t*)xcalloc((size_t)maxnnz, sizeof(int64_t));
    o->values = (double*)xcalloc((size_t)maxnnz, sizeof(double));
}
/* laplacian_2d (problems.cpp:10-30) */
int sko_laplacian_2d(int64_t grid, sko_csr* out) {
    if (grid < 2) return set_err("laplacian_2d: grid must be >= 2"), SKO_ERR_DIMENSION;
    const int64_t n = grid * grid;
    csr_alloc(out, n, 5 * n);
    int64_t nz = 0;
    for (int64_t iy = 0; iy < grid; ++iy)
        for (int64_t ix = 0; ix < grid; ++ix) {
            const int64_t p = ix + grid * iy;
            if (iy > 0) out->col_idx[nz] = p - grid, out->values[nz++] = -1.0;
            if (ix > 0) out->col_idx[nz] = p - 1, out->values[nz++] = -1.0;
            out->col_idx[nz] = p, out->values[nz++] = 4.0;
            if (ix < grid - 1) out->col_idx[nz] = p + 1, out->values[nz++] = -1.0;
            if (iy < grid - 1) out->col_idx[nz] = p + grid, out->values[nz++] = -1.0;
            out->row_ptr[p + 1] = nz;
        }
    out->nnz = nz;
    return SKO_OK;
}
/* 2D sibling of convection_diffusion_3d (problems.cpp:32-60): diag 4,
 * couplings -1 -/+ w_d*h/2 with h = 1/(grid+1). */
int sko_convection_diffusion_2d(int64_t grid, double wx, double wy, sko_csr* out) {
    if (grid < 2) return set_err("convection_diffusion_2d: grid must be >= 2"), SKO_ERR_DIMENSION;
    const int64_t n = grid * grid;
    const double h = 1.0 / ((double)grid + 1.0);
    const double cx = wx * h / 2.0, cy = wy * h / 2.0;
    csr_alloc(out, n, 5 * n);
    int64_t nz = 0;
    for (int64_t iy = 0; iy < grid; ++iy)
        for (int64_t ix = 0; ix < grid; ++ix) {
            const int64_t p = ix + grid * iy;
            if (iy > 0) out->col_idx[nz] = p - grid, out->values[nz++] = -1.0 - cy;
            if (ix > 0) out->col_idx[nz] = p - 1, out->values[nz++] = -1.0 - cx;
            out->col_idx[nz] = p, out->values[nz++] = 4.0;
            if (ix < grid - 1) out->col_idx[nz] = p + 1, out->values[nz++] = -1.0 + cx;
            if (iy < grid - 1) out->col_idx[nz] = p + grid, out->values[nz++] = -1.0 + cy;
            out->row_ptr[p + 1] = nz;
        }
    out->nnz = nz;
    return SKO_OK;
}
/* convection_diffusion_3d (problems.cpp:32-60) */
int sko_convection_diffusion_3d(int64_t grid, double wx, double wy, double wz, sko_csr* out) {
    if (grid < 2) return set_err("convection_diffusion_3d: grid must be >= 2"), SKO_ERR_DIMENSION;
    const int64_t n = grid * grid * grid, g2 = grid * grid;
    const double h = 1.0 / ((double)grid + 1.0);
    const double c0 = wx * h / 2.0, c1 = wy * h / 2.0, c2 = wz * h / 2.0;
    csr_alloc(out, n, 7 * n);
    int64_t nz = 0;
    for (int64_t iz = 0; iz < grid; ++iz)
        for (int64_t iy = 0; iy < grid; ++iy)
            for (int64_t ix = 0; ix < grid; ++ix) {
                const int64_t p = ix + grid * (iy + grid * iz);
                if (iz > 0) out->col_idx[nz] = p - g2, out->values[nz++] = -1.0 - c2;
                if (iy > 0) out->col_idx[nz] = p - grid, out->values[nz++] = -1.0 - c1;
                if (ix > 0) out->col_idx[nz] = p - 1, out->values[nz++] = -1.0 - c0;
                out->col_idx[nz] = p, out->values[nz++] = 6.0;
                if (ix < grid - 1) out->col_idx[nz] = p + 1, out->values[nz++] = -1.0 + c0;
                if (iy < grid - 1) out->col_idx[nz] = p + grid, out->values[nz++] = -1.0 + c1;
                if (iz < grid - 1) out->col_idx[nz] = p + g2, out->values[nz++] = -1.0 + c2;
                out->row_ptr[p + 1] = nz;
            }
    out->nnz = nz;
    return SKO_OK;
}

/* tests/oracles.hpp:49-66 */
int sko_random_sparse(int64_t n, int64_t m, double density, uint64_t seed, double diag_shift,
                      sko_csr* out) {
    mt64 g;
    mt64_seed(&g, seed);
    int64_t cap = n * m, cnt = 0;
    int64_t* r = (int64_t*)xcalloc((size_t)cap, sizeof(int64_t));
    int64_t* c = (int64_t*)xcalloc((size_t)cap, sizeof(int64_t));
    double* v = (double*)xcalloc((size_t)cap, sizeof(double));
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j < m; ++j) {
            const int diag = (i == j && n == m);
            if (diag || canonical(&g) * (1.0 - 0.0) + 0.0 < density) {
                r[cnt] = i;
                c[cnt] = j;
                v[cnt] = uniform_ab(&g, -1.0, 1.0) + (diag ? diag_shift : 0.0);
                ++cnt;
            }
        }
    const int rc = sko_csr_from_triplets(n, m, cnt, r, c, v, out);
    free(r);
    free(c);
    free(v);
    return rc;
}
static int dense_to_csr_full(const double* d, int64_t n, sko_csr* out) {
    /* the reference pushes every (i,j) entry including zeros (oracles.hpp:77-85) */
    csr_alloc(out, n, n * n);
    int64_t nz = 0;
    for (int64_t i = 0; i < n; ++i) {
        for (int64_t j = 0; j < n; ++j) out->col_idx[nz] = j, out->values[nz++] = d[j * n + i];
        out->row_ptr[i + 1] = nz;
    }
    out->nnz = nz;
    return SKO_OK;
}
/* tests/oracles.hpp:70-87 */
int sko_random_spd(int64_t n, uint64_t seed, sko_csr* out) {
    mt64 g;
    mt64_seed(&g, seed);
    double* r = (double*)xcalloc((size_t)(n * n), sizeof(double));
    double* s = (double*)xcalloc((size_t)(n * n), sizeof(double));
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < n; ++i) r[j * n + i] = uniform_ab(&g, -1.0, 1.0);
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < n; ++i) s[j * n + i] = 0.5 * (r[j * n + i] + r[i * n + j]);
    double mx = -1.0;
    for (int64_t i = 0; i < n; ++i) {
        double acc = 0.0;
        for (int64_t j = 0; j < n; ++j) acc = acc + fabs(s[j * n + i]);
        if (acc > mx) mx = acc;
    }
    const double shift = mx + 1.0;
    for (int64_t i = 0; i < n; ++i) s[i * n + i] = s[i * n + i] + shift;
    dense_to_csr_full(s, n, out);
    free(r);
    free(s);
    return SKO_OK;
}
/* tests/oracles.hpp:90-106 */
int sko_random_diag_dominant(int64_t n, uint64_t seed, sko_csr* out) {
    mt64 g;
    mt64_seed(&g, seed);
    double* r = (double*)xcalloc((size_t)(n * n), sizeof(double));
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < n; ++i) r[j * n + i] = uniform_ab(&g, -1.0, 1.0);
    for (int64_t i = 0; i < n; ++i) {
        double acc = 0.0;
        for (int64_t j = 0; j < n; ++j) acc = acc + fabs(r[j * n + i]);
        r[i * n + i] = acc + 1.0;
    }
    dense_to_csr_full(r, n, out);
    free(r);
    return SKO_OK;
}

/* ------------------------------------------------------------------------- */
/* SpMM (sparse_matrix.cpp:142-200) with the parallel knob (parallel.cpp)      */
/* ------------------------------------------------------------------------- */
static int g_par_enabled = 0, g_par_threads = 1;
void sko_set_parallel(int enabled, int threads) {
    g_par_enabled = enabled;
    g_par_threads = enabled ? (threads > 0 ? threads : 1) : 1;
}
typedef struct {
    const sko_csr* a;
    const double* x;
    double* y;
    int64_t xr, yr, cols, lo, hi;
} spmm_job;
/* spmm_rows (sparse_matrix.cpp:142-158): acc += v*x in stored order. */
static void* spmm_rows(void* p) {
    spmm_job* j = (spmm_job*)p;
    for (int64_t c = 0; c < j->cols; ++c)
        for (int64_t i = j->lo; i < j->hi; ++i) {
            double acc = 0.0;
            for (int64_t k = j->a->row_ptr[i]; k < j->a->row_ptr[i + 1]; ++k)
                acc = acc + j->a->values[k] * j->x[c * j->xr + j->a->col_idx[k]];
            j->y[c * j->yr + i] = acc;
        }
    return NULL;
}
/* spmmt_cols (sparse_matrix.cpp:166-182): column-parallel ascending scatter. */
static void* spmmt_cols(void* p) {
    spmm_job* j = (spmm_job*)p;
    for (int64_t c = j->lo; c < j->hi; ++c)
        for (int64_t i = 0; i < j->a->n_rows; ++i) {
            const double xij = j->x[c * j->xr + i];
            if (xij == 0.0) continue;
            for (int64_t k = j->a->row_ptr[i]; k < j->a->row_ptr[i + 1]; ++k)
                j->y[c * j->yr + j->a->col_idx[k]] += j->a->values[k] * xij;
        }
    return NULL;
}
/* parallel_for_ranges (parallel.cpp:26-42) */
static void par_for(int64_t n, spmm_job base, void* (*fn)(void*)) {
    const int threads = g_par_enabled ? g_par_threads : 1;
    if (threads <= 1 || n < 256) {
        base.lo = 0;
        base.hi = n;
        fn(&base);
        return;
    }
    const int64_t chunk = (n + threads - 1) / threads;
    pthread_t tid[256];
    spmm_job jobs[256];
    int nt = 0;
    for (int t = 0; t < threads && t < 256; ++t) {
        const int64_t lo = (int64_t)t * chunk, hi = lo + chunk < n ? lo + chunk : n;
        if (lo >= hi) break;
        jobs[nt] = base;
        jobs[nt].lo = lo;
        jobs[nt].hi = hi;
        pthread_create(&tid[nt], NULL, fn, &jobs[nt]);
        ++nt;
    }
    for (int t = 0; t < nt; ++t) pthread_join(tid[t], NULL);
}
int sko_spmm(const sko_csr* a, const double* x, int64_t cols, double* y) {
    spmm_job j = {a, x, y, a->n_cols, a->n_rows, cols, 0, 0};
    par_for(a->n_rows, j, spmm_rows);
    return SKO_OK;
}
int sko_spmm_transpose(const sko_csr* a, const double* x, int64_t cols, double* y) {
    memset(y, 0, sizeof(double) * (size_t)(a->n_cols * cols));
    spmm_job j = {a, x, y, a->n_rows, a->n_cols, cols, 0, 0};
    par_for(cols, j, spmmt_cols);
    return SKO_OK;
}

/* ------------------------------------------------------------------------- */
/* Small dense kernels                                                        */
/* ------------------------------------------------------------------------- */
/* One-sided Jacobi singular values of a rows x cols matrix (stand-in for the
 * reference's Eigen JacobiSVD, decompositions.cpp:96-104; only the extremes
 * are consumed, block_krylov.cpp:19-23). The GPU runs the identical sequence. */
static void jacobi_extremes(const double* m, int64_t rows, int64_t cols, double* smax, double* smin) {
    double a[64 * 64];
    double* A = rows * cols <= 64 * 64 ? a : (double*)xcalloc((size_t)(rows * cols), sizeof(double));
    memcpy(A, m, sizeof(double) * (size_t)(rows * cols));
    for (int sweep = 0; sweep < 60; ++sweep) {
        int rotated = 0;
        for (int64_t p = 0; p < cols; ++p)
            for (int64_t q = p + 1; q < cols; ++q) {
                double al = 0.0, be = 0.0, ga = 0.0;
                for (int64_t i = 0; i < rows; ++i) {
                    const double ap = A[p * rows + i], aq = A[q * rows + i];
                    al = al + ap * ap;
                    be = be + aq * aq;
                    ga = ga + ap * aq;
                }
                if (ga == 0.0) continue;
                if (fabs(ga) <= 1e-15 * sqrt(al) * sqrt(be)) continue;
                const double zeta = (be - al) / (2.0 * ga);
                double t;
                if (fabs(zeta) > 1e150)
                    t = 1.0 / (2.0 * zeta);
                else
                    t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                const double c = 1.0 / sqrt(1.0 + t * t), sn = c * t;
                for (int64_t i = 0; i < rows; ++i) {
                    const double ap = A[p * rows + i], aq = A[q * rows + i];
                    A[p * rows + i] = c * ap - sn * aq;
                    A[q * rows + i] = sn * ap + c * aq;
                }
                rotated = 1;
            }
        if (!rotated) break;
    }
    const int64_t k = rows < cols ? rows : cols;
    double mx = 0.0, mn = INFINITY;
    /* singular values = the k largest column norms */
    double norms[4096];
    double* nv = cols <= 4096 ? norms : (double*)xcalloc((size_t)cols, sizeof(double));
    for (int64_t j = 0; j < cols; ++j) {
        double acc = 0.0;
        for (int64_t i = 0; i < rows; ++i) acc = acc + A[j * rows + i] * A[j * rows + i];
        nv[j] = sqrt(acc);
    }
    /* partial selection sort: descending */
    for (int64_t x = 0; x < k; ++x) {
        int64_t best = x;
        for (int64_t y = x + 1; y < cols; ++y)
            if (nv[y] > nv[best]) best = y;
        const double t = nv[x];
        nv[x] = nv[best];
        nv[best] = t;
    }
    if (k > 0) {
        mx = nv[0];
        mn = nv[k - 1];
    } else {
        mn = 0.0;
    }
    *smax = mx;
    *smin = mn;
    if (nv != norms) free(nv);
    if (A != a) free(A);
}
int sko_singular_extremes(const double* m, int64_t s, double* smax, double* smin) {
    jacobi_extremes(m, s, s, smax, smin);
    return SKO_OK;
}

/* Cholesky G = R^T R, R upper with positive diagonal. Returns 0 on failure. */
static int cholesky_upper(const double* G, int64_t s, double* R) {
    memset(R, 0, sizeof(double) * (size_t)(s * s));
    for (int64_t j = 0; j < s; ++j) {
        for (int64_t i = 0; i < j; ++i) {
            double acc = G[j * s + i];
            for (int64_t t = 0; t < i; ++t) acc = acc - R[i * s + t] * R[j * s + t];
            R[j * s + i] = acc / R[i * s + i];
        }
        double acc = G[j * s + j];
        for (int64_t t = 0; t < j; ++t) acc = acc - R[j * s + t] * R[j * s + t];
        if (!(acc > 0.0) || !isfinite(acc)) return 0;
        R[j * s + j] = sqrt(acc);
    }
    return 1;
}

/* compact_qr (decompositions.cpp:16-78) with a pluggable dot: sequential for
 * reference order, R1 for the reproducible contract. x: n x s column-major. */
static void householder_qr(const double* x, int64_t n, int64_t s, dot_fn dot, double* qout,
                           double* rout) {
    const int64_t p = n < s ? n : s;
    double* w = (double*)xcalloc((size_t)(n * s), sizeof(double));
    memcpy(w, x, sizeof(double) * (size_t)(n * s));
    double* tau = (double*)xcalloc((size_t)p, sizeof(double));
    double* proj = (double*)xcalloc((size_t)s, sizeof(double));
#define W(i, j) w[(size_t)(j) * (size_t)n + (size_t)(i)]
    for (int64_t j = 0; j < p; ++j) {
        const double norm = sqrt(dot(&W(0, j), &W(0, j), n, j));
        if (norm == 0.0) continue;
        const double alpha = W(j, j) >= 0.0 ? -norm : norm;
        const double v0 = W(j, j) - alpha;
        W(j, j) = alpha;
        const double t = -v0 / alpha;
        tau[j] = t;
        const int64_t tail = n - j - 1;
        if (tail > 0) {
            SKO_PAR(tail >= PAR_MIN)
            for (int64_t i = j + 1; i < n; ++i) W(i, j) = W(i, j) / v0;
        }
        const int64_t rest = s - j - 1;
        if (rest > 0) {
            SKO_PAR(rest > 1 && tail >= PAR_MIN)
            for (int64_t c = j + 1; c < s; ++c) {
                double pr = W(j, c);
                if (tail > 0) pr = pr + dot(&W(0, j), &W(0, c), n, j + 1);
                proj[c] = pr * t;
            }
            for (int64_t c = j + 1; c < s; ++c) W(j, c) = W(j, c) - proj[c];
            if (tail > 0) {
                SKO_PAR(tail >= PAR_MIN)
                for (int64_t i = j + 1; i < n; ++i)
                    for (int64_t c = j + 1; c < s; ++c) W(i, c) = W(i, c) - W(i, j) * proj[c];
            }
        }
    }
    double* q = qout;
    memset(q, 0, sizeof(double) * (size_t)(n * p));
#define Q(i, j) q[(size_t)(j) * (size_t)n + (size_t)(i)]
    for (int64_t j = 0; j < p; ++j) Q(j, j) = 1.0;
    for (int64_t j = p - 1; j >= 0; --j) {
        const double t = tau[j];
        if (t == 0.0) continue;
        const int64_t tail = n - j - 1;
        SKO_PAR(p - j > 1 && tail >= PAR_MIN)
        for (int64_t c = j; c < p; ++c) {
            double pr = Q(j, c);
            if (tail > 0) pr = pr + dot(&W(0, j), &Q(0, c), n, j + 1);
            proj[c] = pr * t;
        }
        for (int64_t c = j; c < p; ++c) Q(j, c) = Q(j, c) - proj[c];
        if (tail > 0) {
            SKO_PAR(tail >= PAR_MIN)
            for (int64_t i = j + 1; i < n; ++i)
                for (int64_t c = j; c < p; ++c) Q(i, c) = Q(i, c) - W(i, j) * proj[c];
        }
    }
    memset(rout, 0, sizeof(double) * (size_t)(p * s));
    for (int64_t j = 0; j < s; ++j)
        for (int64_t i = 0; i <= (j < p - 1 ? j : p - 1); ++i) rout[j * p + i] = W(i, j);
    for (int64_t j = 0; j < p; ++j)
        if (rout[j * p + j] < 0.0) {
            for (int64_t c = j; c < s; ++c) rout[c * p + j] = -rout[c * p + j];
            SKO_PAR(n >= PAR_MIN)
            for (int64_t i = 0; i < n; ++i) Q(i, j) = -Q(i, j);
        }
#undef W
#undef Q
    free(w);
    free(tau);
    free(proj);
}
int sko_thin_qr(const double* x, int64_t n, int64_t s, double* q, double* r) {
    if (n < s) return set_err("thin_qr: requires n_rows >= n_cols"), SKO_ERR_DIMENSION;
    householder_qr(x, n, s, seq_dot, q, r);
    return SKO_OK;
}

/* ------------------------------------------------------------------------- */
/* Block Krylov basis (block_krylov.cpp)                                      */
/* ------------------------------------------------------------------------- */
enum { PATH_DIRECT = 0, PATH_HOUSEHOLDER = 1, PATH_CLEANUP = 2, PATH_UNUSED = 3 };

struct sko_basis {
    const sko_csr* op;
    sko_csr opT; /* reproducible mode: gather over the transposed CSR */
    int has_opT;
    int transpose, arnoldi, full_reorth, mode;
    double tol;
    int64_t n, s, blocks, cap;
    double* v; /* n x cap*s, column-major, block b = columns [b*s, b*s+s) (orthonormal V) */
    double* u;  /* reproducible mode: raw blocks U_b with V_b = U_b N_b^{-1} */
    double* nf; /* reproducible mode: N_b (s x s, column-major) per block */
    double** hcol;
    int64_t* hrows;
    int64_t steps, hcap;
    double hfro2;
    int exhausted, broken;
    int lean; /* keep only the last LEAN_KEEP blocks (Lanczos, golden generation) */
    int64_t paths[4];
};

/* Reference order stores the orthonormal blocks V; the reproducible contract stores
 * only the raw blocks U_b and their factors N_b (V_b = U_b N_b^{-1} is formed on
 * output, bitwise the block the extension produced). */
static int64_t slot(const sko_basis* b, int64_t j) { return b->lean ? j % LEAN_KEEP : j; }
static double* blk(const sko_basis* b, int64_t j) { return b->v + (size_t)(slot(b, j) * b->s * b->n); }
static double* ublk(const sko_basis* b, int64_t j) { return b->u + (size_t)(slot(b, j) * b->s * b->n); }
static double* nfb(const sko_basis* b, int64_t j) { return b->nf + (size_t)(j * b->s * b->s); }

/* q: orthonormal block; u/N: its raw form and factor (reproducible mode only) */
static void basis_append(sko_basis* b, const double* q, const double* u, const double* N) {
    if (b->blocks == b->cap) {
        const int64_t ncap = b->cap ? 2 * b->cap : 8;
        const int64_t dcap = b->lean ? LEAN_KEEP : ncap; /* n x s data slots */
        if (b->mode == SKO_REFERENCE_ORDER) {
            b->v = (double*)realloc(b->v, sizeof(double) * (size_t)(dcap * b->s * b->n));
            if (!b->v) abort();
        } else {
            b->u = (double*)realloc(b->u, sizeof(double) * (size_t)(dcap * b->s * b->n));
            b->nf = (double*)realloc(b->nf, sizeof(double) * (size_t)(ncap * b->s * b->s));
            if (!b->u || !b->nf) abort();
        }
        b->cap = ncap;
    }
    if (b->mode == SKO_REFERENCE_ORDER) {
        memcpy(blk(b, b->blocks), q, sizeof(double) * (size_t)(b->s * b->n));
    } else {
        memcpy(ublk(b, b->blocks), u, sizeof(double) * (size_t)(b->s * b->n));
        memcpy(nfb(b, b->blocks), N, sizeof(double) * (size_t)(b->s * b->s));
    }
    b->blocks++;
}
static void basis_push_h(sko_basis* b, double* col, int64_t rows) {
    if (b->steps == b->hcap) {
        b->hcap = b->hcap ? 2 * b->hcap : 16;
        b->hcol = (double**)realloc(b->hcol, sizeof(double*) * (size_t)b->hcap);
        b->hrows = (int64_t*)realloc(b->hrows, sizeof(int64_t) * (size_t)b->hcap);
    }
    b->hcol[b->steps] = col;
    b->hrows[b->steps] = rows;
    b->steps++;
}

/* apply_operator (block_krylov.cpp:54-56) */
static void basis_apply(const sko_basis* b, const double* x, double* y) {
    if (!b->transpose)
        sko_spmm(b->op, x, b->s, y);
    else if (b->mode == SKO_REFERENCE_ORDER)
        sko_spmm_transpose(b->op, x, b->s, y);
    else
        sko_spmm(&b->opT, x, b->s, y); /* gather in ascending source row == scatter order */
}

/* X^T Y (s x s) with the mode's reduction: out[u*s+t] = sum_i X(i,t) Y(i,u).
 * Reference order: one sequential dot per entry. Reproducible: every entry's R1
 * sum (r1_dot), all entries formed segment by segment. */
static void gram(const sko_basis* b, const double* X, const double* Y, double* out) {
    const int64_t n = b->n, s = b->s, ss = s * s;
    if (b->mode != SKO_REPRODUCIBLE) {
        SKO_PAR(ss > 1 && n >= PAR_MIN)
        for (int64_t e = 0; e < ss; ++e) {
            const int64_t u = e / s, t = e % s;
            out[u * s + t] = seq_dot(X + t * n, Y + u * n, n, 0);
        }
        return;
    }
    const int64_t S = (n + R1_SEG - 1) / R1_SEG;
    double* seg = (double*)xcalloc((size_t)(S * ss), sizeof(double));
    SKO_PAR(S >= 16)
    for (int64_t g = 0; g < S; ++g) {
        double lane[R1_LANES];
        for (int64_t e = 0; e < ss; ++e) {
            const double* x = X + (e % s) * n;
            const double* y = Y + (e / s) * n;
            for (int l = 0; l < R1_LANES; ++l) {
                double acc = 0.0;
                for (int m = 0; m < R1_LROWS; ++m) {
                    const int64_t i = g * R1_SEG + l + R1_LANES * m;
                    if (i < n) acc = acc + x[i] * y[i];
                }
                lane[l] = acc;
            }
            butterfly32(lane);
            seg[e * S + g] = lane[0];
        }
    }
    for (int64_t e = 0; e < ss; ++e) out[(e / s) * s + (e % s)] = tree_reduce(seg + e * S, S);
    free(seg);
}
/* w -= V c per row: tmp = sum_t V(i,t) c(t,u) (sequential), w = w - tmp. */
static void sub_vc(const sko_basis* b, const double* V, const double* c, double* w) {
    const int64_t n = b->n, s = b->s;
    SKO_PAR(n >= PAR_MIN)
    for (int64_t i = 0; i < n; ++i)
        for (int64_t u = 0; u < s; ++u) {
            double tmp = 0.0;
            for (int64_t t = 0; t < s; ++t) tmp = tmp + V[t * n + i] * c[u * s + t];
            w[u * n + i] = w[u * n + i] - tmp;
        }
}
/* Normalisation contract: q = w N^{-1} by forward substitution per row with the
 * reciprocal diagonal, q_u = (w_u - sum_{t<u} q_t N(t,u)) * (1/N(u,u)). The GPU
 * stores blocks unnormalised with N and applies exactly this on every read. */
static void apply_norm(const sko_basis* b, const double* w, const double* N, double* q) {
    const int64_t n = b->n, s = b->s;
    double dinv[64];
    for (int64_t u = 0; u < s; ++u) dinv[u] = 1.0 / N[u * s + u];
    SKO_PAR(n >= PAR_MIN)
    for (int64_t i = 0; i < n; ++i)
        for (int64_t u = 0; u < s; ++u) {
            double acc = w[u * n + i];
            for (int64_t t = 0; t < u; ++t) acc = acc - q[t * n + i] * N[u * s + t];
            q[u * n + i] = acc * dinv[u];
        }
}

/* c = N^{-T} G (forward substitution, N^T lower): c(t,u) = (G(t,u) - sum_{r<t} N(r,t) c(r,u)) / N(t,t) */
static void tri_ntinv(const double* N, const double* G, int64_t s, double* c) {
    double dinv[64];
    for (int64_t t = 0; t < s; ++t) dinv[t] = 1.0 / N[t * s + t];
    for (int64_t u = 0; u < s; ++u)
        for (int64_t t = 0; t < s; ++t) {
            double acc = G[u * s + t];
            for (int64_t r = 0; r < t; ++r) acc = acc - N[t * s + r] * c[u * s + r];
            c[u * s + t] = acc * dinv[t];
        }
}
/* M = N^{-1} c (backward substitution): M(t,u) = (c(t,u) - sum_{r>t} N(t,r) M(r,u)) / N(t,t) */
static void tri_ninv(const double* N, const double* c, int64_t s, double* M) {
    double dinv[64];
    for (int64_t t = 0; t < s; ++t) dinv[t] = 1.0 / N[t * s + t];
    for (int64_t u = 0; u < s; ++u)
        for (int64_t t = s - 1; t >= 0; --t) {
            double acc = c[u * s + t];
            for (int64_t r = t + 1; r < s; ++r) acc = acc - N[r * s + t] * M[u * s + r];
            M[u * s + t] = acc * dinv[t];
        }
}
/* reproducible CGS pass against raw blocks [b0,b1): c_b = N_b^{-T} (U_b^T x) (R1);
 * then x <- x - sum_b U_b (N_b^{-1} c_b) */
static void cgs_raw(const sko_basis* b, int64_t b0, int64_t b1, double* x, double* c_out, int update) {
    const int64_t s = b->s, ss = s * s;
    double G[64 * 64], M[64 * 64];
    double* Ms = (double*)xcalloc((size_t)((b1 - b0 + 1) * ss), sizeof(double));
    for (int64_t jb = b0; jb < b1; ++jb) {
        gram(b, ublk(b, jb), x, G);
        tri_ntinv(nfb(b, jb), G, s, c_out + jb * ss);
        tri_ninv(nfb(b, jb), c_out + jb * ss, s, M);
        memcpy(Ms + (jb - b0) * ss, M, sizeof(double) * (size_t)ss);
    }
    if (update)
        for (int64_t jb = b0; jb < b1; ++jb) sub_vc(b, ublk(b, jb), Ms + (jb - b0) * ss, x);
    free(Ms);
}

/* Reproducible Lanczos pass (block_krylov.cpp:79-84 in CGS form) with RAW Grams:
 * Gamma_b = U_b^T z (R1) against the raw operator output z = op U_{k-1}, then
 * G_b = Gamma_b N_{k-1}^{-1} (each row of Gamma forward-substituted exactly like a
 * basis row, apply_norm), c_b = N_b^{-T} G_b, M_b = N_b^{-1} c_b, and
 * w <- w - sum_b U_b M_b with w = z N_{k-1}^{-1}. Raw Grams let the device form
 * the next extension's Grams in the same sweep that writes U_k, before N_k is
 * known. */
static void lanczos_pass_raw(const sko_basis* b, int64_t b0, int64_t b1, const double* z, double* w,
                             double* c_out) {
    const int64_t s = b->s, ss = s * s;
    const double* Nk = nfb(b, b1 - 1);
    double dinv[64];
    for (int64_t u = 0; u < s; ++u) dinv[u] = 1.0 / Nk[u * s + u];
    double* Ms = (double*)xcalloc((size_t)((b1 - b0 + 1) * ss), sizeof(double));
    for (int64_t jb = b0; jb < b1; ++jb) {
        double Gam[64 * 64], G[64 * 64];
        gram(b, ublk(b, jb), z, Gam);
        for (int64_t t = 0; t < s; ++t) /* row t of Gamma: (Gamma(t,u))_u */
            for (int64_t u = 0; u < s; ++u) {
                double acc = Gam[u * s + t];
                for (int64_t r = 0; r < u; ++r) acc = acc - G[r * s + t] * Nk[u * s + r];
                G[u * s + t] = acc * dinv[u];
            }
        tri_ntinv(nfb(b, jb), G, s, c_out + jb * ss);
        tri_ninv(nfb(b, jb), c_out + jb * ss, s, Ms + (jb - b0) * ss);
    }
    for (int64_t jb = b0; jb < b1; ++jb) sub_vc(b, ublk(b, jb), Ms + (jb - b0) * ss, w);
    free(Ms);
}

/* Normalisation of a materialised candidate wx under the reproducible contract:
 * direct R1 Gram -> Cholesky -> sigma extremes; Householder (with R1 dots) when
 * the Gram is not positive definite or sigma_min < 1e-6 sigma_max. */
typedef struct {
    double R[64 * 64];
    double N[64 * 64]; /* normalisation factor stored with the raw block */
    double smax, smin;
    int householder;
} norm_result;

/* Q: orthonormal block; U (optional): the raw block stored by the device */
static void norm_direct(const sko_basis* b, const double* wx, double* Q, norm_result* nr, double* U) {
    const int64_t s = b->s, n = b->n;
    double G[64 * 64];
    gram(b, wx, wx, G);
    int ok = cholesky_upper(G, s, nr->R);
    if (ok) {
        jacobi_extremes(nr->R, s, s, &nr->smax, &nr->smin);
        if (nr->smin < HH_RATIO * nr->smax) ok = 0;
    }
    if (ok) {
        if (U) memcpy(U, wx, sizeof(double) * (size_t)(n * s));
        memcpy(nr->N, nr->R, sizeof(double) * (size_t)(s * s));
        apply_norm(b, wx, nr->R, Q);
        nr->householder = 0;
    } else {
        double* qh = (double*)xcalloc((size_t)(n * s), sizeof(double));
        householder_qr(wx, n, s, r1_dot, qh, nr->R);
        jacobi_extremes(nr->R, s, s, &nr->smax, &nr->smin);
        memset(nr->N, 0, sizeof nr->N);
        for (int64_t u = 0; u < s; ++u) nr->N[u * s + u] = 1.0;
        if (U) memcpy(U, qh, sizeof(double) * (size_t)(n * s));
        apply_norm(b, qh, nr->N, Q); /* the device reads Q_h through an identity factor */
        free(qh);
        nr->householder = 1;
    }
}

/* init (block_krylov.cpp:27-52) */
int sko_basis_init(const sko_csr* op, const double* start, int64_t s, int arnoldi, int transpose,
                   double breakdown_tol, int lanczos_full_reorth, int mode, sko_basis** out,
                   double* r_out) {
    if (op->n_rows != op->n_cols) return set_err("basis init: operator must be square"), SKO_ERR_DIMENSION;
    if (s < 1 || s > op->n_rows)
        return set_err("basis init: block size must be in [1, n]"), SKO_ERR_DIMENSION;
    if (s > 64) return set_err("basis init: block size above 64 unsupported"), SKO_ERR_DIMENSION;
    sko_basis* b = (sko_basis*)xcalloc(1, sizeof(sko_basis));
    b->op = op;
    b->transpose = transpose;
    b->arnoldi = arnoldi;
    b->full_reorth = lanczos_full_reorth;
    b->mode = mode;
    b->tol = breakdown_tol;
    b->n = op->n_rows;
    b->s = s;
    b->lean = g_lean && !arnoldi && !lanczos_full_reorth;
    if (transpose && mode == SKO_REPRODUCIBLE) {
        sko_csr_transpose(op, &b->opT);
        b->has_opT = 1;
    }
    const int64_t n = b->n;
    double* q = (double*)xcalloc((size_t)(n * s), sizeof(double));
    double* ub = (double*)xcalloc((size_t)(n * s), sizeof(double));
    double R[64 * 64], N[64 * 64];
    double smax, smin;
    if (mode == SKO_REFERENCE_ORDER) {
        householder_qr(start, n, s, seq_dot, q, R);
        jacobi_extremes(R, s, s, &smax, &smin);
    } else {
        norm_result nr;
        memset(&nr, 0, sizeof nr);
        norm_direct(b, start, q, &nr, ub);
        memcpy(R, nr.R, sizeof(double) * (size_t)(s * s));
        memcpy(N, nr.N, sizeof(double) * (size_t)(s * s));
        smax = nr.smax;
        smin = nr.smin;
        b->paths[nr.householder ? PATH_HOUSEHOLDER : PATH_DIRECT]++;
    }
    if (smin < 1e-12 * smax || smax == 0.0) {
        free(q);
        free(ub);
        if (b->has_opT) sko_csr_free(&b->opT);
        free(b);
        return set_err("basis init: start block is numerically rank deficient"), SKO_ERR_RANK_DEFICIENT;
    }
    basis_append(b, q, ub, N);
    free(q);
    free(ub);
    if (r_out) memcpy(r_out, R, sizeof(double) * (size_t)(s * s));
    *out = b;
    return SKO_OK;
}

/* try_extend (block_krylov.cpp:63-145) */
int sko_basis_try_extend(sko_basis* b) {
    if (b->broken) return set_err("basis extend: basis already broke down"), SKO_ERR_BREAKDOWN;
    if (b->exhausted) return 1;
    const int64_t n = b->n, s = b->s, k = b->blocks, ss = s * s;
    const int64_t first = b->arnoldi ? 0 : (k - 2 > 0 ? k - 2 : 0);
    double* w = (double*)xcalloc((size_t)(n * s), sizeof(double));
    double* wr = NULL; /* reproducible: raw operator output z = op U_{k-1} */
    if (b->mode == SKO_REFERENCE_ORDER) {
        basis_apply(b, blk(b, k - 1), w);
    } else {
        /* w = (op U_{k-1}) N_{k-1}^{-1}: raw SpMM, then one row normalisation */
        wr = (double*)xcalloc((size_t)(n * s), sizeof(double));
        basis_apply(b, ublk(b, k - 1), wr);
        apply_norm(b, wr, nfb(b, k - 1), w);
    }
    double* hcoef = (double*)xcalloc((size_t)(k * ss), sizeof(double)); /* block jb at jb*ss */
    double* q = (double*)xcalloc((size_t)(n * s), sizeof(double));
    double* uk = (double*)xcalloc((size_t)(n * s), sizeof(double));
    double R[64 * 64], NK[64 * 64];
    double smax = 0, smin = 0;
    int path = PATH_DIRECT, hh = 0;

    if (b->mode == SKO_REFERENCE_ORDER) {
        double c[64 * 64];
        for (int64_t jb = first; jb < k; ++jb) { /* :79-84 */
            gram(b, blk(b, jb), w, c);
            sub_vc(b, blk(b, jb), c, w);
            memcpy(hcoef + jb * ss, c, sizeof(double) * (size_t)ss);
        }
        if (b->arnoldi) { /* :87-93 */
            for (int64_t jb = 0; jb < k; ++jb) {
                gram(b, blk(b, jb), w, c);
                sub_vc(b, blk(b, jb), c, w);
                for (int64_t e = 0; e < ss; ++e) hcoef[jb * ss + e] = hcoef[jb * ss + e] + c[e];
            }
        } else if (b->full_reorth) { /* :94-100 */
            for (int64_t jb = 0; jb < k; ++jb) {
                gram(b, blk(b, jb), w, c);
                sub_vc(b, blk(b, jb), c, w);
            }
        }
        householder_qr(w, n, s, seq_dot, q, R); /* :102-103 */
        jacobi_extremes(R, s, s, &smax, &smin);
        hh = 1;
    } else {
        /* reproducible contract: CGS pass(es) on the raw blocks, direct CholQR */
        double* cc = (double*)xcalloc((size_t)(k * ss), sizeof(double));
        if (b->arnoldi)
            cgs_raw(b, first, k, w, hcoef, 1); /* w <- w - V_J c_J */
        else
            lanczos_pass_raw(b, first, k, wr, w, hcoef);
        if (b->arnoldi || b->full_reorth) {
            /* second CGS pass (Arnoldi: recorded into H; full re-orth: not recorded) */
            cgs_raw(b, 0, k, w, cc, 1);
            if (b->arnoldi)
                for (int64_t e = 0; e < k * ss; ++e) hcoef[e] = hcoef[e] + cc[e];
        }
        norm_result nr;
        memset(&nr, 0, sizeof nr);
        norm_direct(b, w, q, &nr, uk);
        memcpy(R, nr.R, sizeof(double) * (size_t)ss);
        memcpy(NK, nr.N, sizeof(double) * (size_t)ss);
        smax = nr.smax;
        smin = nr.smin;
        path = nr.householder ? PATH_HOUSEHOLDER : PATH_DIRECT;
        hh = nr.householder;
        free(cc);
    }
    (void)hh;
    b->paths[b->mode == SKO_REPRODUCIBLE ? path : PATH_HOUSEHOLDER]++;

    /* scale (:105-111). Reproducible Arnoldi: per-block sums in the reference's
     * inner order, combined by the canonical pairwise tree over blocks. */
    double coeff2 = 0.0;
    if (b->mode == SKO_REPRODUCIBLE && b->arnoldi) {
        double* hsq = (double*)xcalloc((size_t)(k - first + 1), sizeof(double));
        for (int64_t jb = first; jb < k; ++jb) {
            double acc = 0.0;
            for (int64_t c = 0; c < s; ++c)
                for (int64_t r = 0; r < s; ++r) {
                    const double h = hcoef[jb * ss + c * s + r];
                    acc = acc + h * h;
                }
            hsq[jb - first] = acc;
        }
        coeff2 = tree_reduce(hsq, k - first);
        free(hsq);
    } else {
        for (int64_t jb = first; jb < k; ++jb)
            for (int64_t c = 0; c < s; ++c)
                for (int64_t r = 0; r < s; ++r) {
                    const double h = hcoef[jb * ss + c * s + r];
                    coeff2 = coeff2 + h * h;
                }
    }
    double r2 = 0.0;
    for (int64_t e = 0; e < ss; ++e) r2 = r2 + R[e] * R[e];
    const double scale = sqrt(b->hfro2 + coeff2 + r2);

    if (!b->arnoldi && smin < b->tol * scale) { /* :113-124 clean-up, not recorded in H */
        if (b->lean) {
            free(w); free(wr); free(hcoef); free(q); free(uk);
            return set_err("lean basis: a clean-up pass needs every block"), SKO_ERR_ALLOC;
        }
        if (b->mode == SKO_REFERENCE_ORDER) {
            double c[64 * 64];
            for (int64_t jb = 0; jb < k; ++jb) {
                gram(b, blk(b, jb), w, c);
                sub_vc(b, blk(b, jb), c, w);
            }
            householder_qr(w, n, s, seq_dot, q, R);
            jacobi_extremes(R, s, s, &smax, &smin);
        } else {
            double* d = (double*)xcalloc((size_t)(k * ss), sizeof(double));
            cgs_raw(b, 0, k, w, d, 1);
            norm_result nr;
            memset(&nr, 0, sizeof nr);
            norm_direct(b, w, q, &nr, uk);
            memcpy(R, nr.R, sizeof(double) * (size_t)ss);
            memcpy(NK, nr.N, sizeof(double) * (size_t)ss);
            smax = nr.smax;
            smin = nr.smin;
            b->paths[PATH_CLEANUP]++;
            free(d);
        }
    }

    int rc;
    if (smax <= b->tol * scale || scale == 0.0) { /* :126-133 exhausted */
        double* col = (double*)xcalloc((size_t)(k * s * s), sizeof(double));
        for (int64_t c = 0; c < s; ++c)
            for (int64_t jb = first; jb < k; ++jb)
                for (int64_t r = 0; r < s; ++r) col[c * (k * s) + jb * s + r] = hcoef[jb * ss + c * s + r];
        basis_push_h(b, col, k * s);
        b->hfro2 = b->hfro2 + coeff2;
        b->exhausted = 1;
        rc = 1;
    } else if (smin < b->tol * scale) { /* :134-137 hard breakdown */
        b->broken = 1;
        set_err("basis extend: candidate block is rank deficient (no deflation)");
        rc = SKO_ERR_BREAKDOWN;
    } else { /* :139-144 grown */
        const int64_t rows = (k + 1) * s;
        double* col = (double*)xcalloc((size_t)(rows * s), sizeof(double));
        for (int64_t c = 0; c < s; ++c) {
            for (int64_t jb = first; jb < k; ++jb)
                for (int64_t r = 0; r < s; ++r) col[c * rows + jb * s + r] = hcoef[jb * ss + c * s + r];
            for (int64_t r = 0; r < s; ++r) col[c * rows + k * s + r] = R[c * s + r];
        }
        basis_push_h(b, col, rows);
        b->hfro2 = b->hfro2 + coeff2 + r2;
        basis_append(b, q, uk, NK);
        rc = 0;
    }
    free(w);
    free(wr);
    free(hcoef);
    free(q);
    free(uk);
    return rc;
}

int64_t sko_basis_cols(const sko_basis* b) { return b->blocks * b->s; }
int64_t sko_basis_steps(const sko_basis* b) { return b->steps; }
int sko_basis_exhausted(const sko_basis* b) { return b->exhausted; }
/* the first `blocks` blocks of V, column-major (basis_prefix, block_krylov.cpp:152-157) */
static int basis_v_out(const sko_basis* b, int64_t blocks, double* out) {
    if (b->lean) return set_err("lean basis: V is not kept"), SKO_ERR_ALLOC;
    const size_t bs = (size_t)(b->s * b->n);
    for (int64_t j = 0; j < blocks; ++j) {
        if (b->mode == SKO_REFERENCE_ORDER)
            memcpy(out + j * bs, blk(b, j), sizeof(double) * bs);
        else
            apply_norm(b, ublk(b, j), nfb(b, j), out + j * bs);
    }
    return SKO_OK;
}
void sko_basis_matrix(const sko_basis* b, double* out) { basis_v_out(b, b->blocks, out); }
void sko_basis_path_counts(const sko_basis* b, int64_t* out4) { memcpy(out4, b->paths, sizeof b->paths); }
void sko_basis_free(sko_basis* b) {
    if (!b) return;
    free(b->v);
    free(b->u);
    free(b->nf);
    for (int64_t e = 0; e < b->steps; ++e) free(b->hcol[e]);
    free(b->hcol);
    free(b->hrows);
    if (b->has_opT) sko_csr_free(&b->opT);
    free(b);
}
/* hessenberg_top_left (block_krylov.cpp:159-171) */
int sko_basis_hessenberg(const sko_basis* b, int64_t rows, int64_t cols, double* out) {
    if (rows > sko_basis_cols(b) || cols > b->s * b->steps)
        return set_err("hessenberg_top_left: block exceeds recurrence matrix"), SKO_ERR_DIMENSION;
    memset(out, 0, sizeof(double) * (size_t)(rows * cols));
    for (int64_t e = 0; e * b->s < cols; ++e) {
        const int64_t rmax = rows < b->hrows[e] ? rows : b->hrows[e];
        const int64_t cmax = cols - e * b->s < b->s ? cols - e * b->s : b->s;
        for (int64_t c = 0; c < cmax; ++c)
            for (int64_t r = 0; r < rmax; ++r) out[(e * b->s + c) * rows + r] = b->hcol[e][c * b->hrows[e] + r];
    }
    return SKO_OK;
}
static double h_at(const sko_basis* b, int64_t i, int64_t l) {
    const int64_t e = l / b->s;
    if (i >= b->hrows[e]) return 0.0;
    return b->hcol[e][(l % b->s) * b->hrows[e] + i];
}

/* accumulate_h_times (block_krylov.cpp:173-192): c += H p, block by block,
 * each block's s-term dot formed first and then added (GEBP structure). */
/* (Every output entry c(i,j) receives its block terms in ascending jb; the loops
 * run output columns outermost so they can be spread over threads.) */
static void acc_h_times(const sko_basis* b, const dmat* p, dmat* c) {
    const int64_t s = b->s, jblocks = p->rows / s;
    SKO_PAR(p->cols > 1 && p->cols * c->rows >= PAR_MIN)
    for (int64_t j = 0; j < p->cols; ++j)
        for (int64_t jb = 0; jb < jblocks; ++jb) {
            const int64_t r0 = b->arnoldi ? 0 : ((jb - 1) * s > 0 ? (jb - 1) * s : 0);
            const int64_t r1 = b->hrows[jb] < c->rows ? b->hrows[jb] : c->rows;
            if (r1 <= r0) continue;
            const double* hb = b->hcol[jb];
            const int64_t hr = b->hrows[jb];
            for (int64_t i = r0; i < r1; ++i) {
                double d = 0.0;
                for (int64_t t = 0; t < s; ++t) d = d + hb[t * hr + i] * AT(*p, jb * s + t, j);
                AT(*c, i, j) = AT(*c, i, j) + d;
            }
        }
}
/* accumulate_times_ht (block_krylov.cpp:194-213): c += p H^T. */
static void acc_times_ht(const sko_basis* b, const dmat* p, dmat* c) {
    const int64_t s = b->s, jblocks = p->cols / s;
    SKO_PAR(c->cols > 1 && c->cols * p->rows >= PAR_MIN)
    for (int64_t jc = 0; jc < c->cols; ++jc)
        for (int64_t jb = 0; jb < jblocks; ++jb) {
            const int64_t r0 = b->arnoldi ? 0 : ((jb - 1) * s > 0 ? (jb - 1) * s : 0);
            const int64_t r1 = b->hrows[jb] < c->cols ? b->hrows[jb] : c->cols;
            if (jc < r0 || jc >= r1) continue;
            const double* hb = b->hcol[jb];
            const int64_t hr = b->hrows[jb];
            for (int64_t i = 0; i < p->rows; ++i) {
                double d = 0.0;
                for (int64_t t = 0; t < s; ++t) d = d + AT(*p, i, jb * s + t) * hb[t * hr + jc];
                AT(*c, i, jc) = AT(*c, i, jc) + d;
            }
        }
}
int sko_basis_accumulate_h_times(const sko_basis* b, const double* p, int64_t pr, int64_t pc,
                                 double* c, int64_t cr, int64_t cc) {
    if (pr % b->s != 0 || pr > b->s * b->steps)
        return set_err("accumulate_h_times: p rows incompatible with H"), SKO_ERR_DIMENSION;
    if (cc < pc || cr > sko_basis_cols(b)) return set_err("accumulate_h_times: bad output shape"), SKO_ERR_DIMENSION;
    dmat P = {pr, pc, (double*)p}, C = {cr, cc, c};
    acc_h_times(b, &P, &C);
    return SKO_OK;
}
int sko_basis_accumulate_times_ht(const sko_basis* b, const double* p, int64_t pr, int64_t pc,
                                  double* c, int64_t cr, int64_t cc) {
    if (pc % b->s != 0 || pc > b->s * b->steps)
        return set_err("accumulate_times_ht: p cols incompatible with H"), SKO_ERR_DIMENSION;
    if (cr < pr || cc > sko_basis_cols(b)) return set_err("accumulate_times_ht: bad output shape"), SKO_ERR_DIMENSION;
    dmat P = {pr, pc, (double*)p}, C = {cr, cc, c};
    acc_times_ht(b, &P, &C);
    return SKO_OK;
}

/* acc[i] = fma(x[i], a, acc[i]) for i < n (one rounding per term; hardware FMA
 * when the host has it -- bitwise the same result as libm's fma). */
#if defined(__x86_64__) && defined(__GNUC__)
__attribute__((target("avx2,fma"))) static void fma_axpy_hw(double* acc, const double* x, double a, int64_t n) {
    for (int64_t i = 0; i < n; ++i) acc[i] = __builtin_fma(x[i], a, acc[i]);
}
#endif
static void fma_axpy(double* acc, const double* x, double a, int64_t n) {
#if defined(__x86_64__) && defined(__GNUC__)
    static int hw = -1;
    if (hw < 0) hw = __builtin_cpu_supports("fma") && __builtin_cpu_supports("avx2");
    if (hw) {
        fma_axpy_hw(acc, x, a, n);
        return;
    }
#endif
    for (int64_t i = 0; i < n; ++i) acc[i] = fma(x[i], a, acc[i]);
}

/* ------------------------------------------------------------------------- */
/* Core image Q = [H P, 0] + [P G^T; 0] windowed to the basis sizes          */
/* (factorized_solvers.cpp:62-87 CG, :261-266 BiCGSTAB)                       */
/* ------------------------------------------------------------------------- */
static dmat image(const sko_basis* vb, const sko_basis* wb, const dmat* p, int64_t sched, int mode) {
    const int64_t rows = sched < sko_basis_cols(vb) ? sched : sko_basis_cols(vb);
    const int64_t cols = sched < sko_basis_cols(wb) ? sched : sko_basis_cols(wb);
    dmat q = dm_new(rows, cols);
    const int lyap = vb == wb;
    if (mode == SKO_REFERENCE_ORDER) {
        if (lyap) { /* :73-80, hp + hp^T */
            dmat hp = dm_new(rows, p->cols);
            acc_h_times(vb, p, &hp);
            for (int64_t j = 0; j < p->cols; ++j)
                for (int64_t i = 0; i < rows; ++i) AT(q, i, j) = AT(q, i, j) + AT(hp, i, j);
            for (int64_t j = 0; j < rows; ++j)
                for (int64_t i = 0; i < p->cols; ++i) AT(q, i, j) = AT(q, i, j) + AT(hp, j, i);
            dm_free(&hp);
        } else {
            acc_h_times(vb, p, &q);
            acc_times_ht(wb, p, &q);
        }
        return q;
    }
    /* reproducible: q = Hpart + Gpart, each part its own sum */
    dmat hpart = dm_new(rows, cols), gpart = dm_new(rows, cols);
    if (!vb->arnoldi) {
        acc_h_times(vb, p, &hpart);
        acc_times_ht(wb, p, &gpart);
    } else {
        /* hpart(i,j) = fma chain over l ascending of H(i,l) p(l,j), structural zeros
         * of the block Hessenberg skipped; gpart(i,j) likewise over p(i,l) G(j,l).
         * Each entry's chain is formed in its own accumulator (column j at a time). */
        const int64_t hc = p->cols < cols ? p->cols : cols;
        SKO_PAR(hc > 1)
        for (int64_t j = 0; j < hc; ++j) {
            double* acc = &AT(hpart, 0, j);
            for (int64_t l = 0; l < p->rows; ++l) {
                const int64_t e = l / vb->s, hr = vb->hrows[e];
                const int64_t lim = rows < hr ? rows : hr;
                fma_axpy(acc, vb->hcol[e] + (l % vb->s) * hr, AT(*p, l, j), lim);
            }
        }
        const int64_t gr = p->rows < rows ? p->rows : rows;
        SKO_PAR(cols > 1)
        for (int64_t j = 0; j < cols; ++j) {
            double* acc = &AT(gpart, 0, j);
            for (int64_t l = 0; l < p->cols; ++l) {
                if (j >= wb->hrows[l / wb->s]) continue;
                fma_axpy(acc, &AT(*p, 0, l), h_at(wb, j, l), gr);
            }
        }
    }
    for (int64_t j = 0; j < cols; ++j)
        for (int64_t i = 0; i < rows; ++i) {
            const int hj = j < p->cols, gi = i < p->rows;
            AT(q, i, j) = hj && gi ? AT(hpart, i, j) + AT(gpart, i, j)
                                   : (hj ? AT(hpart, i, j) : (gi ? AT(gpart, i, j) : 0.0));
        }
    dm_free(&hpart);
    dm_free(&gpart);
    return q;
}

/* ------------------------------------------------------------------------- */
/* Solvers (factorized_solvers.cpp:89-389)                                    */
/* ------------------------------------------------------------------------- */
struct sko_solution {
    int status;
    int64_t nrec, caprec;
    int64_t* iters;
    double *rel, *tb, *tk;
    double total;
    int64_t n, m, rv, rw;
    double *V, *core, *W;
    int64_t ncap;
    dmat* captured;
    int64_t paths[4];
};
static void push_rec(sko_solution* sol, int64_t it, double rel, double tb, double tk) {
    if (sol->nrec == sol->caprec) {
        sol->caprec = sol->caprec ? 2 * sol->caprec : 64;
        sol->iters = (int64_t*)realloc(sol->iters, sizeof(int64_t) * (size_t)sol->caprec);
        sol->rel = (double*)realloc(sol->rel, sizeof(double) * (size_t)sol->caprec);
        sol->tb = (double*)realloc(sol->tb, sizeof(double) * (size_t)sol->caprec);
        sol->tk = (double*)realloc(sol->tk, sizeof(double) * (size_t)sol->caprec);
    }
    sol->iters[sol->nrec] = it;
    sol->rel[sol->nrec] = rel;
    sol->tb[sol->nrec] = tb;
    sol->tk[sol->nrec] = tk;
    sol->nrec++;
}
static void capture(sko_solution* sol, const dmat* x) {
    sol->captured = (dmat*)realloc(sol->captured, sizeof(dmat) * (size_t)(sol->ncap + 1));
    sol->captured[sol->ncap++] = dm_copy(x);
}
/* resolve_max_iter (solver_types.cpp:34-38) */
static int64_t resolve_max_iter(const sko_config* c, int64_t n, int64_t m) {
    if (c->max_iter > 0) return c->max_iter;
    const double root = sqrt((double)n * (double)m);
    const int64_t v = 10 * (int64_t)ceil(root);
    return v < 10000 ? v : 10000;
}
static void finish_solution(sko_solution* sol, const sko_basis* vb, const sko_basis* wb, dmat* x) {
    sol->n = vb->n;
    sol->m = wb->n;
    sol->rv = x->rows;
    sol->rw = x->cols;
    if (!vb->lean) { /* lean runs keep the history and the core only */
        sol->V = (double*)xcalloc((size_t)(sol->n * sol->rv), sizeof(double));
        sol->W = (double*)xcalloc((size_t)(sol->m * sol->rw), sizeof(double));
        basis_v_out(vb, sol->rv / vb->s, sol->V);
        basis_v_out(wb, sol->rw / wb->s, sol->W);
    }
    sol->core = x->a;
    x->a = NULL;
    for (int i = 0; i < 4; ++i) sol->paths[i] = vb->paths[i] + (vb != wb ? wb->paths[i] : 0);
}

static int run_cg(const sko_csr* a, const double* c1, const sko_csr* b, const double* c2, int64_t s,
                  const sko_config* cfg, int mode, sko_solution** out) {
    const int lyap = b == NULL;
    const int64_t m = lyap ? a->n_rows : b->n_rows;
    const int64_t max_iter = resolve_max_iter(cfg, a->n_rows, m);
    sko_solution* sol = (sko_solution*)xcalloc(1, sizeof(sko_solution));
    const double t_start = now_s();
    double tk0 = 0, tb0 = 0, t0 = now_s();
    sko_basis *vb = NULL, *wb = NULL;
    dmat rl = dm_new(s, s), rr = dm_new(s, s);
    int rc = sko_basis_init(a, c1, s, 0, 0, cfg->breakdown_tol, cfg->lanczos_full_reorth, mode, &vb, rl.a);
    if (rc == SKO_OK && !lyap)
        rc = sko_basis_init(b, c2, s, 0, 1, cfg->breakdown_tol, cfg->lanczos_full_reorth, mode, &wb, rr.a);
    if (rc != SKO_OK) {
        sko_basis_free(vb);
        dm_free(&rl);
        dm_free(&rr);
        free(sol);
        return rc;
    }
    if (lyap) {
        wb = vb;
        memcpy(rr.a, rl.a, sizeof(double) * (size_t)(s * s));
    }
    tk0 = now_s() - t0;
    t0 = now_s();
    dmat r = dm_a_bt(&rl, &rr); /* :125 */
    dmat p = dm_copy(&r), x = {0, 0, NULL};
    double rho = win_inner(mode, &r, &r, r.rows, r.cols);
    const double norm_r0 = sqrt(rho);
    tb0 = now_s() - t0;
    push_rec(sol, 0, 1.0, tb0, tk0);
    sol->status = SKO_MAX_ITER;

    for (int64_t k = 0; k < max_iter; ++k) {
        double rel = sol->rel[sol->nrec - 1], tk = 0;
        t0 = now_s();
        int e = sko_basis_try_extend(vb);
        if (e >= 0 && !lyap) e = sko_basis_try_extend(wb);
        tk = now_s() - t0;
        if (e < 0) {
            sol->status = SKO_BREAKDOWN;
            push_rec(sol, k + 1, rel, 0, tk);
            break;
        }
        t0 = now_s();
        dmat q = image(vb, wb, &p, (k + 2) * s, mode);
        const double denom = win_inner(mode, &r, &q, r.rows, r.cols); /* :154 */
        if (fabs(denom) < cfg->breakdown_tol * rho) {
            sol->status = SKO_BREAKDOWN;
            push_rec(sol, k + 1, rel, now_s() - t0, tk);
            dm_free(&q);
            break;
        }
        const double alpha = rho / denom;
        dmat xn = dm_embed(&x, p.rows, p.cols);
        dm_free(&x);
        x = xn;
        dm_axpy(alpha, &p, &x);
        dmat rn = dm_embed(&r, q.rows, q.cols);
        dm_axpy(-alpha, &q, &rn);
        double rho_next = win_inner(mode, &rn, &rn, rn.rows, rn.cols);
        const double norm_r = sqrt(rho_next); /* frobenius_norm: same sum in both modes */
        rel = norm_r / norm_r0;
        if (cfg->capture_iterates) capture(sol, &x);
        if (norm_r <= norm_r0 * cfg->eps_tol) {
            sol->status = SKO_CONVERGED;
            push_rec(sol, k + 1, rel, now_s() - t0, tk);
            dm_free(&q);
            dm_free(&r);
            r = rn;
            break;
        }
        const double beta = rho_next / rho;
        dmat pn = dm_copy(&rn);
        dmat pp = dm_embed(&p, rn.rows, rn.cols);
        dm_axpy(beta, &pp, &pn);
        dm_free(&pp);
        dm_free(&p);
        dm_free(&r);
        dm_free(&q);
        p = pn;
        r = rn;
        rho = rho_next;
        push_rec(sol, k + 1, rel, now_s() - t0, tk);
    }
    finish_solution(sol, vb, wb, &x);
    sol->total = now_s() - t_start;
    dm_free(&r);
    dm_free(&p);
    dm_free(&rl);
    dm_free(&rr);
    sko_basis_free(vb);
    if (!lyap) sko_basis_free(wb);
    *out = sol;
    return SKO_OK;
}

static double window_norm(int mode, const dmat* big, int64_t rows, int64_t cols) {
    return sqrt(win_inner(mode, big, big, rows, cols));
}

static int run_bicgstab(const sko_csr* a, const sko_csr* b, const double* c1, const double* c2,
                        int64_t s, const sko_config* cfg, int mode, sko_solution** out) {
    const int64_t max_iter = resolve_max_iter(cfg, a->n_rows, b->n_rows);
    sko_solution* sol = (sko_solution*)xcalloc(1, sizeof(sko_solution));
    const double t_start = now_s();
    double t0 = now_s();
    sko_basis *vb = NULL, *wb = NULL;
    dmat rl = dm_new(s, s), rr = dm_new(s, s);
    int rc = sko_basis_init(a, c1, s, 1, 0, cfg->breakdown_tol, 0, mode, &vb, rl.a);
    if (rc == SKO_OK) rc = sko_basis_init(b, c2, s, 1, 1, cfg->breakdown_tol, 0, mode, &wb, rr.a);
    if (rc != SKO_OK) {
        sko_basis_free(vb);
        dm_free(&rl);
        dm_free(&rr);
        free(sol);
        return rc;
    }
    const double tk0 = now_s() - t0;
    t0 = now_s();
    dmat r = dm_a_bt(&rl, &rr);
    dmat rs = dm_copy(&r), p = dm_copy(&r), x = {0, 0, NULL};
    double rho = win_inner(mode, &rs, &r, r.rows, r.cols);
    const double norm_r0 = sqrt(win_inner(mode, &r, &r, r.rows, r.cols));
    const double norm_shadow = norm_r0;
    push_rec(sol, 0, 1.0, now_s() - t0, tk0);
    sol->status = SKO_MAX_ITER;

    for (int64_t k = 0; k < max_iter; ++k) {
        double rel = sol->rel[sol->nrec - 1], tk = 0, tb = 0;
        t0 = now_s();
        int e = sko_basis_try_extend(vb);
        if (e >= 0) e = sko_basis_try_extend(wb);
        tk += now_s() - t0;
        if (e < 0) {
            sol->status = SKO_BREAKDOWN;
            push_rec(sol, k + 1, rel, tb, tk);
            break;
        }
        t0 = now_s();
        dmat q = image(vb, wb, &p, (2 * k + 2) * s, mode);
        const double denom = win_inner(mode, &rs, &q, rs.rows, rs.cols);
        const double q_win = window_norm(mode, &q, rs.rows, rs.cols);
        if (fabs(denom) < cfg->breakdown_tol * norm_shadow * q_win) {
            tb += now_s() - t0;
            sol->status = SKO_BREAKDOWN;
            push_rec(sol, k + 1, rel, tb, tk);
            dm_free(&q);
            break;
        }
        const double alpha = rho / denom;
        dmat sm = dm_embed(&r, q.rows, q.cols);
        dm_axpy(-alpha, &q, &sm);
        tb += now_s() - t0;
        t0 = now_s();
        e = sko_basis_try_extend(vb);
        if (e >= 0) e = sko_basis_try_extend(wb);
        tk += now_s() - t0;
        if (e < 0) {
            sol->status = SKO_BREAKDOWN;
            push_rec(sol, k + 1, rel, tb, tk);
            dm_free(&q);
            dm_free(&sm);
            break;
        }
        t0 = now_s();
        dmat t = image(vb, wb, &sm, (2 * k + 3) * s, mode);
        const double tt = win_inner(mode, &t, &t, t.rows, t.cols);
        const double ssv = win_inner(mode, &sm, &sm, sm.rows, sm.cols);
        double omega;
        int broke = 0;
        if (sqrt(ssv) <= cfg->eps_tol * norm_r0)
            omega = 0.0;
        else if (tt < cfg->breakdown_tol * ssv)
            broke = 1, omega = 0.0;
        else
            omega = win_inner(mode, &sm, &t, sm.rows, sm.cols) / tt;
        if (broke) {
            tb += now_s() - t0;
            sol->status = SKO_BREAKDOWN;
            push_rec(sol, k + 1, rel, tb, tk);
            dm_free(&q);
            dm_free(&sm);
            dm_free(&t);
            break;
        }
        dmat xn = dm_embed(&x, sm.rows, sm.cols);
        dm_free(&x);
        x = xn;
        {
            dmat pp = dm_embed(&p, sm.rows, sm.cols);
            dm_axpy(alpha, &pp, &x);
            dm_free(&pp);
        }
        dm_axpy(omega, &sm, &x);
        dmat rn = dm_embed(&sm, t.rows, t.cols);
        dm_axpy(-omega, &t, &rn);
        const double norm_r = sqrt(win_inner(mode, &rn, &rn, rn.rows, rn.cols));
        rel = norm_r / norm_r0;
        if (cfg->capture_iterates) capture(sol, &x);
        if (norm_r <= norm_r0 * cfg->eps_tol) {
            tb += now_s() - t0;
            sol->status = SKO_CONVERGED;
            push_rec(sol, k + 1, rel, tb, tk);
            dm_free(&q);
            dm_free(&sm);
            dm_free(&t);
            dm_free(&rn);
            break;
        }
        const double rho_next = win_inner(mode, &rs, &rn, rs.rows, rs.cols);
        const double r_win = window_norm(mode, &rn, rs.rows, rs.cols);
        if (fabs(rho_next) < cfg->breakdown_tol * norm_shadow * r_win) {
            tb += now_s() - t0;
            sol->status = SKO_BREAKDOWN;
            push_rec(sol, k + 1, rel, tb, tk);
            dm_free(&q);
            dm_free(&sm);
            dm_free(&t);
            dm_free(&rn);
            break;
        }
        const double beta = (alpha / omega) * (rho_next / rho);
        dmat pn = dm_copy(&rn);
        {
            dmat pp = dm_embed(&p, rn.rows, rn.cols);
            dm_axpy(beta, &pp, &pn);
            dm_free(&pp);
            dmat qp = dm_embed(&q, rn.rows, rn.cols);
            dm_axpy(-beta * omega, &qp, &pn);
            dm_free(&qp);
        }
        dm_free(&p);
        dm_free(&r);
        dm_free(&q);
        dm_free(&sm);
        dm_free(&t);
        p = pn;
        r = rn;
        rho = rho_next;
        tb += now_s() - t0;
        push_rec(sol, k + 1, rel, tb, tk);
    }
    finish_solution(sol, vb, wb, &x);
    sol->total = now_s() - t_start;
    dm_free(&r);
    dm_free(&rs);
    dm_free(&p);
    dm_free(&rl);
    dm_free(&rr);
    sko_basis_free(vb);
    sko_basis_free(wb);
    *out = sol;
    return SKO_OK;
}

/* require_solver_inputs (factorized_solvers.cpp:50-58) + entry points :204-225 */
int sko_solve(int method, const sko_csr* a, const sko_csr* b, const double* c1, const double* c2,
              int64_t s, const sko_config* cfg, int mode, sko_solution** out) {
    *out = NULL;
    if (method == SKO_METHOD_CG_LYAPUNOV) {
        if (a->n_rows != a->n_cols) return set_err("factorized_cg_lyapunov: A must be square"), SKO_ERR_DIMENSION;
        if (!sko_csr_is_symmetric(a, 1e-12))
            return set_err("factorized_cg_lyapunov: A is not symmetric"), SKO_ERR_INVALID_MATRIX;
        return run_cg(a, c1, NULL, NULL, s, cfg, mode, out);
    }
    if (a->n_rows != a->n_cols || b->n_rows != b->n_cols)
        return set_err("solver: A and B must be square"), SKO_ERR_DIMENSION;
    if (s < 1) return set_err("solver: C1 and C2 must have the same positive column count"), SKO_ERR_DIMENSION;
    if (method == SKO_METHOD_CG) {
        if (!sko_csr_is_symmetric(a, 1e-12)) return set_err("factorized_cg: A is not symmetric"), SKO_ERR_INVALID_MATRIX;
        if (!sko_csr_is_symmetric(b, 1e-12)) return set_err("factorized_cg: B is not symmetric"), SKO_ERR_INVALID_MATRIX;
        return run_cg(a, c1, b, c2, s, cfg, mode, out);
    }
    return run_bicgstab(a, b, c1, c2, s, cfg, mode, out);
}

int sko_solution_status(const sko_solution* sol) { return sol->status; }
int64_t sko_solution_n_records(const sko_solution* sol) { return sol->nrec; }
void sko_solution_history(const sko_solution* sol, int64_t* iters, double* rel, double* t_basic,
                          double* t_krylov) {
    for (int64_t i = 0; i < sol->nrec; ++i) {
        if (iters) iters[i] = sol->iters[i];
        if (rel) rel[i] = sol->rel[i];
        if (t_basic) t_basic[i] = sol->tb[i];
        if (t_krylov) t_krylov[i] = sol->tk[i];
    }
}
void sko_solution_dims(const sko_solution* sol, int64_t* n, int64_t* rv, int64_t* m, int64_t* rw) {
    *n = sol->n;
    *rv = sol->rv;
    *m = sol->m;
    *rw = sol->rw;
}
void sko_solution_copy(const sko_solution* sol, double* v, double* core, double* w) {
    if (v && sol->V) memcpy(v, sol->V, sizeof(double) * (size_t)(sol->n * sol->rv));
    if (core && sol->core) memcpy(core, sol->core, sizeof(double) * (size_t)(sol->rv * sol->rw));
    if (w && sol->W) memcpy(w, sol->W, sizeof(double) * (size_t)(sol->m * sol->rw));
}
int64_t sko_solution_n_captured(const sko_solution* sol) { return sol->ncap; }
void sko_solution_captured(const sko_solution* sol, int64_t i, int64_t* rows, int64_t* cols, double* out) {
    *rows = sol->captured[i].rows;
    *cols = sol->captured[i].cols;
    if (out) memcpy(out, sol->captured[i].a, sizeof(double) * (size_t)(*rows * *cols));
}
double sko_solution_total_time(const sko_solution* sol) { return sol->total; }
void sko_solution_path_counts(const sko_solution* sol, int64_t* out4) { memcpy(out4, sol->paths, sizeof sol->paths); }
void sko_solution_free(sko_solution* sol) {
    if (!sol) return;
    free(sol->iters);
    free(sol->rel);
    free(sol->tb);
    free(sol->tk);
    free(sol->V);
    free(sol->W);
    free(sol->core);
    for (int64_t i = 0; i < sol->ncap; ++i) dm_free(&sol->captured[i]);
    free(sol->captured);
    free(sol);
}

/* small_sylvester_apply (factorized_solvers.cpp:37-46) */
int sko_small_sylvester_apply(const double* p, int64_t pr, int64_t pc, const double* h, int64_t hr,
                              const double* g, int64_t gr, double* out) {
    /* h: hr x pr, g: gr x pc */
    memset(out, 0, sizeof(double) * (size_t)(hr * gr));
    for (int64_t j = 0; j < pc; ++j)
        for (int64_t i = 0; i < hr; ++i) {
            double acc = 0.0;
            for (int64_t t = 0; t < pr; ++t) acc = acc + h[t * hr + i] * p[j * pr + t];
            out[j * hr + i] = acc;
        }
    for (int64_t j = 0; j < gr; ++j)
        for (int64_t i = 0; i < pr; ++i) {
            double acc = 0.0;
            for (int64_t t = 0; t < pc; ++t) acc = acc + p[t * pr + i] * g[t * gr + j];
            out[j * hr + i] = out[j * hr + i] + acc;
        }
    return SKO_OK;
}

/* true_residual_factors (factorized_solvers.cpp:391-439), reference order. */
double sko_true_residual_factors(const sko_csr* a, const sko_csr* b, const double* c1,
                                 const double* c2, int64_t s, const double* v, int64_t rv,
                                 const double* core, const double* w, int64_t rw) {
    const int64_t n = a->n_rows, m = b->n_rows, r = rw;
    /* denominator ||C1 C2^T|| via compact QRs */
    const int64_t p1 = n < s ? n : s, p2 = m < s ? m : s;
    double* q1 = (double*)xcalloc((size_t)(n * p1), sizeof(double));
    double* r1 = (double*)xcalloc((size_t)(p1 * s), sizeof(double));
    double* q2 = (double*)xcalloc((size_t)(m * p2), sizeof(double));
    double* r2 = (double*)xcalloc((size_t)(p2 * s), sizeof(double));
    householder_qr(c1, n, s, seq_dot, q1, r1);
    householder_qr(c2, m, s, seq_dot, q2, r2);
    dmat R1 = {p1, s, r1}, R2 = {p2, s, r2};
    dmat den = dm_a_bt(&R1, &R2);
    const double denom = sqrt(seq_window_inner(&den, &den, den.rows, den.cols));
    dm_free(&den);
    /* vc = V core (n x r), avc = A vc, btw = B^T W */
    double* vc = (double*)xcalloc((size_t)(n * r), sizeof(double));
    for (int64_t j = 0; j < r; ++j)
        for (int64_t i = 0; i < n; ++i) {
            double acc = 0.0;
            for (int64_t t = 0; t < rv; ++t) acc = acc + v[t * n + i] * core[j * rv + t];
            vc[j * n + i] = acc;
        }
    double* avc = (double*)xcalloc((size_t)(n * r), sizeof(double));
    double* btw = (double*)xcalloc((size_t)(m * r), sizeof(double));
    sko_spmm(a, vc, r, avc);
    sko_spmm_transpose(b, w, r, btw);
    const int64_t wdt = s + 2 * r;
    double* uf = (double*)xcalloc((size_t)(n * wdt), sizeof(double));
    double* vf = (double*)xcalloc((size_t)(m * wdt), sizeof(double));
    memcpy(uf, c1, sizeof(double) * (size_t)(n * s));
    memcpy(uf + n * s, avc, sizeof(double) * (size_t)(n * r));
    memcpy(uf + n * (s + r), vc, sizeof(double) * (size_t)(n * r));
    memcpy(vf, c2, sizeof(double) * (size_t)(m * s));
    memcpy(vf + m * s, w, sizeof(double) * (size_t)(m * r));
    memcpy(vf + m * (s + r), btw, sizeof(double) * (size_t)(m * r));
    const int64_t pu = n < wdt ? n : wdt, pv = m < wdt ? m : wdt;
    double* qu = (double*)xcalloc((size_t)(n * pu), sizeof(double));
    double* ru = (double*)xcalloc((size_t)(pu * wdt), sizeof(double));
    double* qv = (double*)xcalloc((size_t)(m * pv), sizeof(double));
    double* rvv = (double*)xcalloc((size_t)(pv * wdt), sizeof(double));
    householder_qr(uf, n, wdt, seq_dot, qu, ru);
    householder_qr(vf, m, wdt, seq_dot, qv, rvv);
    for (int64_t j = s; j < wdt; ++j)
        for (int64_t i = 0; i < pu; ++i) ru[j * pu + i] = -ru[j * pu + i];
    dmat RU = {pu, wdt, ru}, RV = {pv, wdt, rvv};
    dmat res = dm_a_bt(&RU, &RV);
    const double num = sqrt(seq_window_inner(&res, &res, res.rows, res.cols));
    dm_free(&res);
    free(q1); free(r1); free(q2); free(r2); free(vc); free(avc); free(btw);
    free(uf); free(vf); free(qu); free(ru); free(qv); free(rvv);
    return num / denom;
}

/* reductions exposed for tests */
double sko_frobenius_inner(const double* x, const double* y, int64_t rows, int64_t cols) {
    dmat a = {rows, cols, (double*)x}, b = {rows, cols, (double*)y};
    return seq_window_inner(&a, &b, rows, cols);
}
double sko_r1_dot(const double* x, const double* y, int64_t n) { return r1_dot(x, y, n, 0); }
double sko_r2_inner(const double* x, const double* y, int64_t rows, int64_t cols) {
    dmat a = {rows, cols, (double*)x}, b = {rows, cols, (double*)y};
    return r2_inner(&a, &b, rows, cols);
}
