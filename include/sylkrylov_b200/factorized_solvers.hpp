// sylkrylov_b200/factorized_solvers.hpp -- C++ drop-in for the reference's
// solver API (proj/include/sylkrylov/factorized_solvers.hpp:14-61 and
// solver_types.hpp:11-47, errors.hpp:9-57) over the C-ABI sylkrylov_b200.h.
//
// Callers of sylkrylov::factorized_cg / factorized_cg_lyapunov /
// factorized_bicgstab compile unchanged against this header (namespace
// sylkrylov::b200 re-exported as sylkrylov with SYLKRYLOV_B200_AS_REFERENCE)
// and link libsk_b200.so; the solve runs on the B200 and the factors are copied
// back into column-major DenseMatrix values exactly like the reference returns
// them. Exceptions are the reference's types; numerical outcomes (breakdown,
// max_iter) are reported in FactorizedSolution::status as in the reference.
#pragma once

#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../sylkrylov_b200.h"

namespace sylkrylov {
namespace b200 {

using index_t = std::ptrdiff_t;

// ---- errors.hpp:9-57 ----
struct DimensionError : std::invalid_argument {
  explicit DimensionError(const std::string& w) : std::invalid_argument(w) {}
};
struct InvalidMatrixError : std::invalid_argument {
  explicit InvalidMatrixError(const std::string& w) : std::invalid_argument(w) {}
};
struct RankDeficientStartError : std::runtime_error {
  explicit RankDeficientStartError(const std::string& w) : std::runtime_error(w) {}
};
struct DeviceError : std::runtime_error {  // CUDA failure / no device / capacity
  explicit DeviceError(const std::string& w) : std::runtime_error(w) {}
};

// ---- dense_matrix.hpp:12-47 (column-major fp64) ----
class DenseMatrix {
 public:
  DenseMatrix() = default;
  DenseMatrix(index_t r, index_t c) : r_(r), c_(c), v_(static_cast<size_t>(r * c), 0.0) {
    if (r < 0 || c < 0) throw DimensionError("DenseMatrix: negative dimension");
  }
  index_t rows() const { return r_; }
  index_t cols() const { return c_; }
  double& operator()(index_t i, index_t j) { return v_[static_cast<size_t>(j * r_ + i)]; }
  double operator()(index_t i, index_t j) const { return v_[static_cast<size_t>(j * r_ + i)]; }
  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }
  const std::vector<double>& values() const { return v_; }

 private:
  index_t r_ = 0, c_ = 0;
  std::vector<double> v_;
};

// ---- sparse_matrix.hpp:11-48 (CSR, 64-bit indices) ----
class SparseMatrix {
 public:
  SparseMatrix() = default;
  SparseMatrix(index_t nr, index_t nc, std::vector<index_t> rp, std::vector<index_t> ci, std::vector<double> v)
      : nr_(nr), nc_(nc), rp_(std::move(rp)), ci_(std::move(ci)), v_(std::move(v)) {}
  index_t rows() const { return nr_; }
  index_t cols() const { return nc_; }
  index_t nnz() const { return static_cast<index_t>(v_.size()); }
  const std::vector<index_t>& row_ptr() const { return rp_; }
  const std::vector<index_t>& col_idx() const { return ci_; }
  const std::vector<double>& values() const { return v_; }
  sk_csr c_view() const {
    static_assert(sizeof(index_t) == sizeof(int64_t), "64-bit index_t expected");
    return sk_csr{nr_, nc_, nnz(), reinterpret_cast<const int64_t*>(rp_.data()),
                  reinterpret_cast<const int64_t*>(ci_.data()), v_.data()};
  }

 private:
  index_t nr_ = 0, nc_ = 0;
  std::vector<index_t> rp_{0}, ci_;
  std::vector<double> v_;
};

// ---- solver_types.hpp:11-47 ----
enum class SolveStatus { converged, max_iter, breakdown };
struct IterationRecord {
  index_t iteration = 0;
  double rel_residual = 0.0;
  double t_basic_s = 0.0, t_krylov_s = 0.0, t_trunc_s = 0.0;
};
struct ConvergenceHistory {
  std::vector<IterationRecord> records;
  double total_time_s = 0.0;
  index_t iterations() const { return records.empty() ? 0 : records.back().iteration; }
  double final_rel_residual() const { return records.empty() ? 1.0 : records.back().rel_residual; }
};
struct SolverConfig {
  double eps_tol = 1e-8;
  index_t max_iter = 0;
  double breakdown_tol = 1e-12;
  bool capture_iterates = false;
  bool lanczos_full_reorth = false;
};
struct FactorizedSolution {
  DenseMatrix V, core, W;
  ConvergenceHistory history;
  SolveStatus status = SolveStatus::max_iter;
  std::vector<DenseMatrix> captured_cores;
};

namespace detail {
inline void raise(sk_status rc) {
  const std::string msg = sk_last_error();
  switch (rc) {
    case SK_OK: return;
    case SK_ERR_DIMENSION: throw DimensionError(msg);
    case SK_ERR_INVALID_MATRIX: throw InvalidMatrixError(msg);
    case SK_ERR_RANK_DEFICIENT: throw RankDeficientStartError(msg);
    default: throw DeviceError(msg);
  }
}
inline sk_config cfg(const SolverConfig& c) {
  return sk_config{c.eps_tol, static_cast<int64_t>(c.max_iter), c.breakdown_tol, c.capture_iterates ? 1 : 0,
                   c.lanczos_full_reorth ? 1 : 0};
}
inline FactorizedSolution collect(sk_solution* h) {
  FactorizedSolution out;
  int64_t n, rv, m, rw;
  sk_solution_dims(h, &n, &rv, &m, &rw);
  out.V = DenseMatrix(n, rv);
  out.core = DenseMatrix(rv, rw);
  out.W = DenseMatrix(m, rw);
  raise(sk_solution_copy_V(h, out.V.data()));
  raise(sk_solution_copy_core(h, out.core.data()));
  raise(sk_solution_copy_W(h, out.W.data()));
  const int64_t nrec = sk_solution_num_records(h);
  std::vector<sk_iteration_record> rec(static_cast<size_t>(nrec));
  raise(sk_solution_history(h, rec.data(), nrec));
  for (const auto& r : rec)
    out.history.records.push_back({static_cast<index_t>(r.iteration), r.rel_residual, r.t_basic_s, r.t_krylov_s,
                                   r.t_trunc_s});
  out.history.total_time_s = sk_solution_total_time(h);
  const int32_t st = sk_solution_status(h);
  out.status = st == SK_SOLVE_CONVERGED ? SolveStatus::converged
                                        : (st == SK_SOLVE_BREAKDOWN ? SolveStatus::breakdown : SolveStatus::max_iter);
  for (int64_t i = 0; i < sk_solution_num_captured(h); ++i) {
    int64_t r, c;
    raise(sk_solution_captured_core(h, i, &r, &c, nullptr));
    DenseMatrix x(r, c);
    raise(sk_solution_captured_core(h, i, &r, &c, x.data()));
    out.captured_cores.push_back(std::move(x));
  }
  sk_solution_free(h);
  return out;
}
}  // namespace detail

// factorized_solvers.hpp:39-53
inline FactorizedSolution factorized_cg(const SparseMatrix& a, const SparseMatrix& b, const DenseMatrix& c1,
                                        const DenseMatrix& c2, const SolverConfig& cfg = {}) {
  if (c1.rows() != a.rows() || c2.rows() != b.rows()) throw DimensionError("solver: C1/C2 row counts must match A/B");
  if (c1.cols() != c2.cols() || c1.cols() < 1)
    throw DimensionError("solver: C1 and C2 must have the same positive column count");
  const sk_csr ca = a.c_view(), cb = b.c_view();
  const sk_config cc = detail::cfg(cfg);
  sk_solution* h = nullptr;
  detail::raise(sk_factorized_cg(&ca, &cb, c1.data(), c2.data(), c1.cols(), &cc, nullptr, &h));
  return detail::collect(h);
}
inline FactorizedSolution factorized_cg_lyapunov(const SparseMatrix& a, const DenseMatrix& c1,
                                                 const SolverConfig& cfg = {}) {
  if (c1.rows() != a.rows()) throw DimensionError("factorized_cg_lyapunov: C1 rows must match A");
  const sk_csr ca = a.c_view();
  const sk_config cc = detail::cfg(cfg);
  sk_solution* h = nullptr;
  detail::raise(sk_factorized_cg_lyapunov(&ca, c1.data(), c1.cols(), &cc, nullptr, &h));
  return detail::collect(h);
}
inline FactorizedSolution factorized_bicgstab(const SparseMatrix& a, const SparseMatrix& b, const DenseMatrix& c1,
                                              const DenseMatrix& c2, const SolverConfig& cfg = {}) {
  if (c1.rows() != a.rows() || c2.rows() != b.rows()) throw DimensionError("solver: C1/C2 row counts must match A/B");
  if (c1.cols() != c2.cols() || c1.cols() < 1)
    throw DimensionError("solver: C1 and C2 must have the same positive column count");
  const sk_csr ca = a.c_view(), cb = b.c_view();
  const sk_config cc = detail::cfg(cfg);
  sk_solution* h = nullptr;
  detail::raise(sk_factorized_bicgstab(&ca, &cb, c1.data(), c2.data(), c1.cols(), &cc, nullptr, &h));
  return detail::collect(h);
}

}  // namespace b200
}  // namespace sylkrylov

#ifdef SYLKRYLOV_B200_AS_REFERENCE
namespace sylkrylov {
using namespace b200;
}
#endif
