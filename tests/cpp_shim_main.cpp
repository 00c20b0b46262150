// Compiles against the C++ drop-in shim exactly like a reference caller would
// (test_factorized_solvers.cpp:22-33 identity pair; RankDeficientRhsRejected).
#define SYLKRYLOV_B200_AS_REFERENCE
#include "sylkrylov_b200/factorized_solvers.hpp"

#include <cmath>
#include <cstdio>

using namespace sylkrylov;

static SparseMatrix identity(index_t n) {
  std::vector<index_t> rp(n + 1), ci(n);
  for (index_t i = 0; i <= n; ++i) rp[i] = i;
  for (index_t i = 0; i < n; ++i) ci[i] = i;
  return SparseMatrix(n, n, rp, ci, std::vector<double>(n, 1.0));
}

int main() {
  const index_t n = 7, m = 5, s = 2;
  DenseMatrix c1(n, s), c2(m, s);
  for (index_t j = 0; j < s; ++j) {
    for (index_t i = 0; i < n; ++i) c1(i, j) = std::sin(1.0 + i + 3 * j);
    for (index_t i = 0; i < m; ++i) c2(i, j) = std::cos(2.0 + i - j);
  }
  FactorizedSolution sol = factorized_cg(identity(n), identity(m), c1, c2);
  double err = 0, nrm = 0;
  for (index_t i = 0; i < n; ++i)
    for (index_t j = 0; j < m; ++j) {
      double x = 0, e = 0;
      for (index_t a = 0; a < sol.core.rows(); ++a)
        for (index_t b = 0; b < sol.core.cols(); ++b) x += sol.V(i, a) * sol.core(a, b) * sol.W(j, b);
      for (index_t t = 0; t < s; ++t) e += 0.5 * c1(i, t) * c2(j, t);
      err += (x - e) * (x - e);
      nrm += e * e;
    }
  const bool ok1 = sol.status == SolveStatus::converged && sol.history.iterations() == 1 &&
                   std::sqrt(err) <= 1e-13 * std::sqrt(nrm);
  bool ok2 = false;
  DenseMatrix bad(8, 2);
  for (index_t i = 0; i < 8; ++i) bad(i, 0) = bad(i, 1) = static_cast<double>(i);
  try {
    factorized_cg_lyapunov(identity(8), bad);
  } catch (const RankDeficientStartError&) {
    ok2 = true;
  }
  std::printf("identity_pair=%d rank_deficient=%d\n", ok1, ok2);
  return (ok1 && ok2) ? 0 : 1;
}
