/*
 * sylkrylov_b200.h -- C-ABI of the B200-native factorized-Krylov hot path.
 *
 * Drop-in boundary for the reference's solver entry points
 * (proj/include/sylkrylov/factorized_solvers.hpp:39-61). Plain pointers and
 * sizes only; no C++ or torch types. The C++ shim
 * include/sylkrylov_b200/factorized_solvers.hpp rebuilds the reference's
 * `sylkrylov::FactorizedSolution` and re-throws its exception types
 * (errors.hpp:9-57) on top of these functions.
 *
 * Threading: one in-flight solve per device; calls are reentrant across
 * devices. Errors: negative sk_status, message via sk_last_error()
 * (thread-local), mirroring the reference's exception taxonomy.
 */
#ifndef SYLKRYLOV_B200_H
#define SYLKRYLOV_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* CSR operator, reference index width (sparse_matrix.hpp:11-48: 64-bit
 * index_t, strictly increasing columns per row). Host pointers unless
 * sk_gpu_options.inputs_on_device is set. */
typedef struct {
    int64_t n_rows, n_cols, nnz;
    const int64_t* row_ptr;
    const int64_t* col_idx;
    const double* values;
} sk_csr;

/* Field-for-field mirror of SolverConfig (solver_types.hpp:36-45). */
typedef struct {
    double eps_tol;              /* default 1e-8 */
    int64_t max_iter;            /* 0 -> min(10*ceil(sqrt(n*m)), 10000) (solver_types.cpp:34-38) */
    double breakdown_tol;        /* default 1e-12 */
    int32_t capture_iterates;    /* test hook: snapshot the core after every iteration */
    int32_t lanczos_full_reorth; /* forwarded to block Lanczos */
} sk_config;

/* Device-side options (no reference counterpart). Zero-initialise for defaults. */
typedef struct {
    int32_t device;              /* CUDA ordinal */
    int32_t profile;             /* 1: time every kernel class with CUDA events */
    int64_t capacity_bytes;      /* HBM budget for the bases (0: 90% of free memory) */
    int32_t reduction_mode;      /* SK_REDUCTION_* (0: the reproducible contract) */
    int32_t reserved[7];
} sk_gpu_options;

/* Arithmetic mode of the sums on the path.
 *  SK_REDUCTION_REPRODUCIBLE: fixed reduction trees; results are
 *    bit-identical across launches, grids and row partitions, and bit-identical to the
 *    oracle's SKO_REPRODUCIBLE mode. The only mode the device executes.
 *  SK_REDUCTION_REFERENCE_ORDER: the reference's single sequential sum per inner product
 *    (dense_matrix.cpp:131-152) is one dependent chain per output and cannot be laid out
 *    on the device; requesting it returns SK_ERR_UNSUPPORTED. The oracle's
 *    SKO_REFERENCE_ORDER mode is the CPU statement of it, and the distance between the two
 *    modes is pinned by tests (CG family <= 1e-10 over whole runs; BiCGSTAB inside the
 *    window the recurrence's own sensitivity allows, tests/test_bicgstab_sensitivity.py). */
enum { SK_REDUCTION_REPRODUCIBLE = 0, SK_REDUCTION_REFERENCE_ORDER = 1 };

typedef enum {
    SK_OK = 0,
    SK_ERR_DIMENSION = -1,       /* DimensionError         (errors.hpp:9-13)  */
    SK_ERR_INVALID_MATRIX = -2,  /* InvalidMatrixError     (errors.hpp:18-21) */
    SK_ERR_RANK_DEFICIENT = -3,  /* RankDeficientStartError(errors.hpp:24-27) */
    SK_ERR_CUDA = -10,           /* CUDA runtime failure, or no device       */
    SK_ERR_OUT_OF_MEMORY = -11,
    SK_ERR_CAPACITY = -12,       /* basis budget exceeded before max_iter    */
    SK_ERR_UNSUPPORTED = -13,    /* e.g. block size s > 8 on the device path */
    SK_ERR_IO = -14              /* IoError                (errors.hpp:48-51) */
} sk_status;

/* SolveStatus (solver_types.hpp:11) */
enum { SK_SOLVE_CONVERGED = 0, SK_SOLVE_MAX_ITER = 1, SK_SOLVE_BREAKDOWN = 2 };

/* IterationRecord (solver_types.hpp:15-23) */
typedef struct {
    int64_t iteration;
    double rel_residual;
    double t_basic_s;
    double t_krylov_s;
    double t_trunc_s;
} sk_iteration_record;

/* Execution statistics of one solve (device-timed). */
typedef struct {
    double device_time_s;        /* whole solve on the device (events) */
    double h2d_time_s, d2h_time_s;
    int64_t h2d_bytes, d2h_bytes;
    int64_t kernel_launches;
    int64_t iterations;
    /* per kernel class (profile=1): 0 spmm, 1 gram, 2 rare-path, 3 write-block,
     * 4 core-a, 5 core-b, 6 arnoldi-update, 7 dense-image, 8 other */
    double class_time_s[9];
    int64_t class_launches[9];
    double class_bytes[9];       /* algorithmic bytes */
    int64_t paths[4];            /* extension paths: direct, householder, clean-up, unused */
    double class_flops[9];       /* FP64 flops of compute-bound classes (7: dense image), else 0 */
} sk_solve_stats;

typedef struct sk_solution sk_solution;

/* factorized_cg (factorized_solvers.hpp:39-43; factorized_solvers.cpp:204-210) */
sk_status sk_factorized_cg(const sk_csr* a, const sk_csr* b, const double* c1, const double* c2,
                           int64_t s, const sk_config* cfg, const sk_gpu_options* gpu,
                           sk_solution** out);
/* factorized_cg_lyapunov (factorized_solvers.hpp:45-48; .cpp:212-218) */
sk_status sk_factorized_cg_lyapunov(const sk_csr* a, const double* c1, int64_t s,
                                    const sk_config* cfg, const sk_gpu_options* gpu,
                                    sk_solution** out);
/* factorized_bicgstab (factorized_solvers.hpp:50-53; .cpp:220-389) */
sk_status sk_factorized_bicgstab(const sk_csr* a, const sk_csr* b, const double* c1,
                                 const double* c2, int64_t s, const sk_config* cfg,
                                 const sk_gpu_options* gpu, sk_solution** out);

/* Resident problems: inputs uploaded once, solved many times (benchmarks). */
typedef struct sk_problem sk_problem;
enum { SK_METHOD_CG = 0, SK_METHOD_CG_LYAPUNOV = 1, SK_METHOD_BICGSTAB = 2 };
sk_status sk_problem_create(int32_t method, const sk_csr* a, const sk_csr* b, const double* c1,
                            const double* c2, int64_t s, const sk_gpu_options* gpu,
                            sk_problem** out);
sk_status sk_problem_solve(sk_problem* p, const sk_config* cfg, sk_solution** out);
void sk_problem_free(sk_problem* p);

/* FactorizedSolution accessors (factorized_solvers.hpp:14-23). V/core/W stay
 * in HBM until copied; copies are column-major like DenseMatrix. */
int32_t sk_solution_status(const sk_solution* sol);
void sk_solution_dims(const sk_solution* sol, int64_t* n, int64_t* rv, int64_t* m, int64_t* rw);
int64_t sk_solution_num_records(const sk_solution* sol);
sk_status sk_solution_history(const sk_solution* sol, sk_iteration_record* records, int64_t count);
double sk_solution_total_time(const sk_solution* sol);
sk_status sk_solution_copy_V(const sk_solution* sol, double* out);    /* n  x rv */
sk_status sk_solution_copy_core(const sk_solution* sol, double* out); /* rv x rw */
sk_status sk_solution_copy_W(const sk_solution* sol, double* out);    /* m  x rw */
/* Column ranges [col0, col0 + ncols) of V / W (n x ncols, m x ncols column-major):
 * only the basis blocks covering the range leave HBM. */
sk_status sk_solution_copy_V_cols(const sk_solution* sol, int64_t col0, int64_t ncols, double* out);
sk_status sk_solution_copy_W_cols(const sk_solution* sol, int64_t col0, int64_t ncols, double* out);
int64_t sk_solution_num_captured(const sk_solution* sol);
sk_status sk_solution_captured_core(const sk_solution* sol, int64_t i, int64_t* rows,
                                    int64_t* cols, double* out);
sk_status sk_solution_stats(const sk_solution* sol, sk_solve_stats* out);
void sk_solution_free(sk_solution* sol);

/* Row partition (the reference has no multi-GPU path -- this is
 * the north star's "A's rows and B's rows partitioned across GPUs"). Rows are
 * split on reduction chunks (aligned power-of-two groups of 512-row R1
 * segments), so every rank's history, cores and classification decisions are
 * bitwise those of the single-GPU solve. Per iteration: one all-gather of the
 * Gram chunk nodes per pass and one halo exchange of the newest basis block.
 * CG and Lyapunov CG with s <= 4. */
typedef struct sk_comm sk_comm;
typedef struct sk_partition {
  int64_t row0, rows;          /* this rank's global rows [row0, row0 + rows) */
  int64_t chunk_rows;          /* rows per reduction chunk */
  int64_t chunks, chunks_max, chunks_total;
  int64_t halo;                /* ghost rows per side (one grid line / plane, or the bandwidth) */
} sk_partition;
/* Pure host function: the plan every rank computes identically. */
sk_status sk_partition_plan(int64_t n, int64_t halo, int32_t world, int32_t rank, sk_partition* out);
/* NCCL transport (one process per GPU): rank 0 makes the id, the caller
 * broadcasts it (e.g. torch.distributed), every rank creates its communicator.
 * libnccl.so.2 is loaded at run time. */
sk_status sk_nccl_unique_id(uint8_t* out128);
sk_status sk_comm_create_nccl(const uint8_t* id128, int32_t nranks, int32_t rank, int32_t device,
                              sk_comm** out);
/* In-process group: nranks communicators whose ranks are host threads (one
 * solve per thread); collectives are device copies behind host barriers. */
sk_status sk_comm_create_local_group(int32_t nranks, sk_comm** out /* nranks entries */);
int32_t sk_comm_rank(const sk_comm* c);
int32_t sk_comm_size(const sk_comm* c);
void sk_comm_free(sk_comm* c);
/* Every rank passes the whole A, B, C1, C2 (host) and keeps only its rows. */
sk_status sk_problem_create_partitioned(int32_t method, const sk_csr* a, const sk_csr* b,
                                        const double* c1, const double* c2, int64_t s,
                                        const sk_gpu_options* gpu, sk_comm* comm, sk_problem** out);
/* Partitioned solutions hold this rank's rows of V and W (sk_solution_dims
 * then reports the local row counts). */
sk_status sk_solution_partition(const sk_solution* sol, int64_t* row0_v, int64_t* rows_v,
                                int64_t* row0_w, int64_t* rows_w);

const char* sk_last_error(void);
const char* sk_version(void);
int32_t sk_device_count(void);
/* FP64 peak of the device in TFLOP/s, measured (register-chain microbenchmark, CUDA
 * events): DFMA chains (fma = 2 flops) and mul-then-add chains (the arithmetic
 * contract's form). Denominator of the FP64 roofline (bench.py). */
sk_status sk_measure_fp64_peak(int32_t device, double* dfma_tflops, double* dmul_dadd_tflops);

/* True residual ||A X + X B - C1 C2^T||_F / ||C1 C2^T||_F of X = V core W^T on the
 * device (replaces true_residual / true_residual_factors, factorized_solvers.hpp:56-61,
 * factorized_solvers.cpp:391-444): the R factors of [C1, A V core, V core] and
 * [C2, W, B^T W] by a streaming TSQR (the stacked factors are never formed), the
 * residual core R_U diag(I, -I, -I) R_V^T reduced on the host. Floating point, not
 * the bitwise contract. Errors as the reference: SK_ERR_DIMENSION for shapes,
 * SK_ERR_INVALID_MATRIX for a zero right-hand side. sk_true_residual reads V, core
 * and W where the solution holds them (HBM); sk_true_residual_factors takes host
 * column-major factors (n x rv, rv x rw, m x rw); sk_problem_true_residual uses the
 * problem's resident operators and C1/C2 (Lyapunov: B = A, C2 = C1). */
sk_status sk_true_residual(const sk_csr* a, const sk_csr* b, const double* c1, const double* c2, int64_t s,
                           const sk_solution* sol, double* rel);
sk_status sk_true_residual_factors(const sk_csr* a, const sk_csr* b, const double* c1, const double* c2,
                                   int64_t s, const double* v, int64_t rv, const double* core,
                                   const double* w, int64_t rw, double* rel);
sk_status sk_problem_true_residual(const sk_problem* p, const sk_solution* sol, double* rel);

/* X-parity through factor products (the stacked-factor pattern of
 * true_residual_factors, factorized_solvers.cpp:410-438): r_out (column-major,
 * (r + ref_cols)^2, upper triangular) = the R factor of [V_sol, V_ref] (side 0) or
 * [W_sol, W_ref] (side 1), V_sol read where the solution holds it (HBM), V_ref a host
 * column-major rows x ref_cols matrix (e.g. the CPU oracle's factors). Then
 * ||X_sol - X_ref||_F = ||R_V diag(core_sol, -core_ref) R_W^T||_F. Streaming TSQR on the
 * device; floating point outside the bitwise contract. */
sk_status sk_solution_stacked_r(const sk_solution* sol, int32_t side, const double* ref, int64_t ref_cols,
                                double* r_out);

/* Kernel-level entry for parity tests: y = A x (reference spmm order) or
 * y = A^T x (spmm_transpose, via the transposed CSR) on the device. */
sk_status sk_spmm(const sk_csr* a, const double* x, int64_t s, int32_t transpose, double* y);

/* Problem generators (problems.cpp:10-96 restated, plus the 2D convection-
 * diffusion sibling): kind 0 = laplacian_2d, 1 = convection_diffusion_2d,
 * 2 = convection_diffusion_3d (wind = convection vector w; Peclet Pe with a
 * unit wind d is w = Pe*d). Caller allocates n+1 / nnz / nnz entries. */
int64_t sk_gen_stencil_nnz(int32_t kind, int64_t grid);
sk_status sk_gen_stencil(int32_t kind, int64_t grid, const double* wind, int64_t* row_ptr,
                         int64_t* col_idx, double* values);
/* random_rhs: rows x s column-major, std::mt19937_64 + Box-Muller (bitwise the reference's). */
sk_status sk_gen_random_rhs(int64_t rows, int64_t s, uint64_t seed, double* out);

/* Page-locked host buffers for inputs: C1 / C2 passed from such memory are copied
 * by DMA directly (pageable memory goes through the library's pinned staging lanes). */
sk_status sk_host_alloc(int64_t bytes, void** out);
void sk_host_free(void* p);

/* On-disk formats. Text is byte-identical to the reference's
 * writers (17 significant digits, "%.17g"); all return SK_ERR_IO on a failed
 * open or write, with the path in sk_last_error().
 *   sk_write_history_csv         -- write_history_csv   (bench.cpp:179-193)
 *   sk_write_matrix_market_csr   -- write_matrix_market(SparseMatrix) (matrix_market.cpp:148-161)
 *   sk_write_matrix_market_dense -- write_matrix_market(DenseMatrix)  (matrix_market.cpp:163-175)
 *   sk_solution_write_factors    -- the V.mtx / core.mtx / W.mtx triple of the CLI
 *     (main.cpp:182-184) into directory dir (which must exist), streamed from HBM
 *     block by block and formatted on all host threads; format SK_FORMAT_BINARY
 *     writes V.skb / core.skb / W.skb instead: the binary sidecar for solutions
 *     whose text form would not fit a disk (C5: ~170 GB of text), layout =
 *     8-byte magic "SKFACT01", int64 rows, int64 cols, rows*cols little-endian
 *     fp64 column-major. */
enum { SK_FORMAT_MATRIX_MARKET = 0, SK_FORMAT_BINARY = 1 };
sk_status sk_write_history_csv(const sk_solution* sol, const char* path);
sk_status sk_write_matrix_market_csr(const sk_csr* a, const char* path);
sk_status sk_write_matrix_market_dense(const double* a, int64_t rows, int64_t cols, const char* path);
sk_status sk_solution_write_factors(const sk_solution* sol, const char* dir, int32_t format);

#ifdef __cplusplus
}
#endif
#endif
