/*
 * sk_oracle.h -- CPU restatement of the factorized-Krylov hot path of the
 * reference (`sylkrylov`, arXiv 2605.28274). TEST INFRASTRUCTURE ONLY: this
 * library is the checker that the B200 product path is compared against; it is
 * loaded by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg, never by the product path.
 *
 * Two arithmetic modes:
 *   SKO_REFERENCE_ORDER  -- follows the reference loop by loop: sequential sums
 *                           where it writes loops (dense_matrix.cpp:131-152,
 *                           factorized_solvers.cpp:17-22), plain sequential loops
 *                           where it calls Eigen, Householder thin_qr
 *                           (decompositions.cpp:16-78), block MGS
 *                           (block_krylov.cpp:79-100).
 *   SKO_REPRODUCIBLE     -- the reproducible-reduction contract the GPU executes
 *                           bit for bit: fixed
 *                           segment/tile reduction trees, CGS(2) + CholQR with a
 *                           Householder fallback, fma-chained dense Arnoldi image.
 *
 * The reference itself cannot be built here (Eigen3, GTest and its vendored
 * CLI11/json are absent -- SURVEY.md section 8c), so this restatement is pinned
 * against the reference's own known-answer tests (tests/test_oracle_*.py).
 */
#ifndef SK_ORACLE_H
#define SK_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* CSR with the reference's 64-bit index width (sparse_matrix.hpp:11-48). */
typedef struct {
    int64_t n_rows, n_cols, nnz;
    int64_t* row_ptr;
    int64_t* col_idx;
    double* values;
} sko_csr;

/* Mirrors SolverConfig (solver_types.hpp:36-45). */
typedef struct {
    double eps_tol;
    int64_t max_iter;
    double breakdown_tol;
    int32_t capture_iterates;
    int32_t lanczos_full_reorth;
} sko_config;

enum {
    SKO_OK = 0,
    SKO_ERR_DIMENSION = -1,      /* DimensionError          errors.hpp:9-13  */
    SKO_ERR_INVALID_MATRIX = -2, /* InvalidMatrixError      errors.hpp:18-21 */
    SKO_ERR_RANK_DEFICIENT = -3, /* RankDeficientStartError errors.hpp:24-27 */
    SKO_ERR_BREAKDOWN = -4,      /* BreakdownError (hard)   errors.hpp:32-40 */
    SKO_ERR_EXHAUSTED = -5,      /* BreakdownError(invariant_subspace=true)  */
    SKO_ERR_ALLOC = -6
};
enum { SKO_CONVERGED = 0, SKO_MAX_ITER = 1, SKO_BREAKDOWN = 2 }; /* SolveStatus */
enum { SKO_REPRODUCIBLE = 0, SKO_REFERENCE_ORDER = 1 };
enum { SKO_METHOD_CG = 0, SKO_METHOD_CG_LYAPUNOV = 1, SKO_METHOD_BICGSTAB = 2 };

const char* sko_last_error(void);
int sko_contract_constants(int64_t* out4); /* {R1 segment rows, lanes, R2 tile, pyth guard bits} */
void sko_set_lean(int on); /* golden generation: keep only the last Lanczos blocks (no V output) */

/* ---- CSR / problems (sparse_matrix.cpp, problems.cpp) ---- */
int sko_csr_from_triplets(int64_t n_rows, int64_t n_cols, int64_t count, const int64_t* rows,
                          const int64_t* cols, const double* vals, sko_csr* out);
int sko_csr_transpose(const sko_csr* a, sko_csr* out);
int sko_csr_is_symmetric(const sko_csr* a, double tol);
void sko_csr_free(sko_csr* a);
int sko_laplacian_2d(int64_t grid, sko_csr* out);
int sko_convection_diffusion_2d(int64_t grid, double wx, double wy, sko_csr* out);
int sko_convection_diffusion_3d(int64_t grid, double wx, double wy, double wz, sko_csr* out);
void sko_random_rhs(int64_t rows, int64_t s, uint64_t seed, double* out);
/* test-side generators of proj/tests/oracles.hpp:39-106 (column-major dense) */
void sko_random_dense(int64_t rows, int64_t cols, uint64_t seed, double* out);
int sko_random_sparse(int64_t n, int64_t m, double density, uint64_t seed, double diag_shift,
                      sko_csr* out);
int sko_random_spd(int64_t n, uint64_t seed, sko_csr* out);
int sko_random_diag_dominant(int64_t n, uint64_t seed, sko_csr* out);

/* ---- kernels (reference order) ---- */
void sko_set_parallel(int enabled, int threads); /* parallel.cpp:15-19 */
int sko_spmm(const sko_csr* a, const double* x, int64_t cols, double* y);
int sko_spmm_transpose(const sko_csr* a, const double* x, int64_t cols, double* y);
int sko_thin_qr(const double* x, int64_t n, int64_t s, double* q, double* r); /* Householder */
int sko_singular_extremes(const double* m, int64_t s, double* smax, double* smin);

/* ---- block Krylov basis (block_krylov.hpp) ---- */
typedef struct sko_basis sko_basis;
int sko_basis_init(const sko_csr* op, const double* start, int64_t s, int arnoldi, int transpose,
                   double breakdown_tol, int lanczos_full_reorth, int mode, sko_basis** out,
                   double* r_out);
int sko_basis_try_extend(sko_basis* b); /* 0 grown, 1 exhausted, <0 error */
int64_t sko_basis_cols(const sko_basis* b);
int64_t sko_basis_steps(const sko_basis* b);
int sko_basis_exhausted(const sko_basis* b);
void sko_basis_matrix(const sko_basis* b, double* out);
int sko_basis_hessenberg(const sko_basis* b, int64_t rows, int64_t cols, double* out);
int sko_basis_accumulate_h_times(const sko_basis* b, const double* p, int64_t pr, int64_t pc,
                                 double* c, int64_t cr, int64_t cc);
int sko_basis_accumulate_times_ht(const sko_basis* b, const double* p, int64_t pr, int64_t pc,
                                  double* c, int64_t cr, int64_t cc);
void sko_basis_path_counts(const sko_basis* b, int64_t* out4);
void sko_basis_free(sko_basis* b);

/* ---- solvers (factorized_solvers.hpp:39-61) ---- */
typedef struct sko_solution sko_solution;
int sko_solve(int method, const sko_csr* a, const sko_csr* b, const double* c1, const double* c2,
              int64_t s, const sko_config* cfg, int mode, sko_solution** out);
int sko_solution_status(const sko_solution* sol);
int64_t sko_solution_n_records(const sko_solution* sol);
void sko_solution_history(const sko_solution* sol, int64_t* iters, double* rel, double* t_basic,
                          double* t_krylov);
void sko_solution_dims(const sko_solution* sol, int64_t* n, int64_t* rv, int64_t* m, int64_t* rw);
void sko_solution_copy(const sko_solution* sol, double* v, double* core, double* w);
int64_t sko_solution_n_captured(const sko_solution* sol);
void sko_solution_captured(const sko_solution* sol, int64_t i, int64_t* rows, int64_t* cols,
                           double* out);
double sko_solution_total_time(const sko_solution* sol);
void sko_solution_path_counts(const sko_solution* sol, int64_t* out4);
void sko_solution_free(sko_solution* sol);

/* reductions exposed for tests: sequential (reference) and the two contracts */
double sko_frobenius_inner(const double* x, const double* y, int64_t rows, int64_t cols);
double sko_r1_dot(const double* x, const double* y, int64_t n);
double sko_r2_inner(const double* x, const double* y, int64_t rows, int64_t cols);

double sko_true_residual_factors(const sko_csr* a, const sko_csr* b, const double* c1,
                                 const double* c2, int64_t s, const double* v, int64_t rv,
                                 const double* core, const double* w, int64_t rw);
int sko_small_sylvester_apply(const double* p, int64_t pr, int64_t pc, const double* h,
                              int64_t hr, const double* g, int64_t gr, double* out);

#ifdef __cplusplus
}
#endif
#endif
