// C entry points over the reference's own Eigen-free sources (compiled from
// /root/reference/proj/src/{sparse_matrix,parallel,problems,matrix_market}.cpp by
// oracle/build_ref.sh into oracle/_ref/). TEST INFRASTRUCTURE: used only to pin
// the oracle's restatement of SpMM, CSR utilities and generators bitwise.
#include <cstring>
#include <vector>

#include "sylkrylov/dense_matrix.hpp"
#include "sylkrylov/errors.hpp"
#include "sylkrylov/matrix_market.hpp"
#include "sylkrylov/parallel.hpp"
#include "sylkrylov/problems.hpp"
#include "sylkrylov/sparse_matrix.hpp"

using namespace sylkrylov;

// The only DenseMatrix member the Eigen-free sources need (dense_matrix.hpp:17):
// a zero-initialised column-major buffer. Restated here because dense_matrix.cpp
// includes Eigen.
namespace sylkrylov {
DenseMatrix::DenseMatrix(index_t n_rows, index_t n_cols)
    : n_rows_(n_rows), n_cols_(n_cols), values_(static_cast<size_t>(n_rows * n_cols), 0.0) {
    if (n_rows < 0 || n_cols < 0) throw DimensionError("DenseMatrix: negative dimension");
}
}  // namespace sylkrylov

namespace {
int64_t export_csr(const SparseMatrix& a, int64_t* rp, int64_t* ci, double* v) {
    if (rp) std::memcpy(rp, a.row_ptr().data(), sizeof(int64_t) * a.row_ptr().size());
    if (ci) std::memcpy(ci, a.col_idx().data(), sizeof(int64_t) * a.col_idx().size());
    if (v) std::memcpy(v, a.values().data(), sizeof(double) * a.values().size());
    return a.nnz();
}
SparseMatrix import_csr(int64_t nr, int64_t nc, int64_t nnz, const int64_t* rp, const int64_t* ci,
                        const double* v) {
    return SparseMatrix(nr, nc, std::vector<index_t>(rp, rp + nr + 1), std::vector<index_t>(ci, ci + nnz),
                        std::vector<double>(v, v + nnz));
}
DenseMatrix import_dense(int64_t rows, int64_t cols, const double* x) {
    DenseMatrix m(rows, cols);
    std::memcpy(m.data(), x, sizeof(double) * rows * cols);
    return m;
}
}  // namespace

extern "C" {
int64_t ref_laplacian_2d(int64_t grid, int64_t* rp, int64_t* ci, double* v) {
    return export_csr(laplacian_2d(grid), rp, ci, v);
}
int64_t ref_convection_diffusion_3d(int64_t grid, double w0, double w1, double w2, int64_t* rp, int64_t* ci,
                                    double* v) {
    return export_csr(convection_diffusion_3d(grid, {w0, w1, w2}), rp, ci, v);
}
void ref_random_rhs(int64_t rows, int64_t s, uint64_t seed, double* out) {
    DenseMatrix m = random_rhs(rows, s, seed);
    std::memcpy(out, m.data(), sizeof(double) * rows * s);
}
void ref_spmm(int64_t nr, int64_t nc, int64_t nnz, const int64_t* rp, const int64_t* ci, const double* v,
              const double* x, int64_t cols, double* y) {
    DenseMatrix r = spmm(import_csr(nr, nc, nnz, rp, ci, v), import_dense(nc, cols, x));
    std::memcpy(y, r.data(), sizeof(double) * nr * cols);
}
void ref_spmm_transpose(int64_t nr, int64_t nc, int64_t nnz, const int64_t* rp, const int64_t* ci,
                        const double* v, const double* x, int64_t cols, double* y) {
    DenseMatrix r = spmm_transpose(import_csr(nr, nc, nnz, rp, ci, v), import_dense(nr, cols, x));
    std::memcpy(y, r.data(), sizeof(double) * nc * cols);
}
int64_t ref_transposed(int64_t nr, int64_t nc, int64_t nnz, const int64_t* rp, const int64_t* ci,
                       const double* v, int64_t* trp, int64_t* tci, double* tv) {
    return export_csr(import_csr(nr, nc, nnz, rp, ci, v).transposed(), trp, tci, tv);
}
int ref_is_symmetric(int64_t nr, int64_t nc, int64_t nnz, const int64_t* rp, const int64_t* ci, const double* v,
                     double tol) {
    return import_csr(nr, nc, nnz, rp, ci, v).is_symmetric(tol) ? 1 : 0;
}
void ref_set_parallel(int enabled, unsigned threads) { set_parallel_kernels(enabled != 0, threads); }
// Matrix Market writers / reader (matrix_market.cpp): 0 ok, -1 on any exception
int ref_write_mm_csr(int64_t nr, int64_t nc, int64_t nnz, const int64_t* rp, const int64_t* ci, const double* v,
                     const char* path) {
    try {
        write_matrix_market(import_csr(nr, nc, nnz, rp, ci, v), path);
        return 0;
    } catch (...) {
        return -1;
    }
}
int ref_write_mm_dense(int64_t rows, int64_t cols, const double* x, const char* path) {
    try {
        write_matrix_market(import_dense(rows, cols, x), path);
        return 0;
    } catch (...) {
        return -1;
    }
}
// sparse read: call with null buffers for the sizes (n_rows, n_cols, nnz), then with buffers
int64_t ref_read_mm_csr(const char* path, int64_t* dims, int64_t* rp, int64_t* ci, double* v) {
    try {
        SparseMatrix a = read_matrix_market_sparse(path);
        dims[0] = a.rows();
        dims[1] = a.cols();
        dims[2] = a.nnz();
        return export_csr(a, rp, ci, v);
    } catch (...) {
        return -1;
    }
}
}
