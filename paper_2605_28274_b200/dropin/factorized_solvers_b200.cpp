// Drop-in replacement for the reference's src/factorized_solvers.cpp.
//
// This translation unit is compiled INTO the reference build in place of
// proj/src/factorized_solvers.cpp: it includes the reference's OWN
// headers (proj/include/sylkrylov/*.hpp, unchanged) and defines every function that
// file defines -- factorized_solvers.hpp:25-61 -- on top of the C-ABI
// (include/sylkrylov_b200.h, libsk_b200.so). Callers (tools/main.cpp:165-185,
// src/bench.cpp:86-103, the reference's tests) compile and link unchanged; the solve
// runs on the B200.
//
//   factorized_cg / factorized_cg_lyapunov / factorized_bicgstab
//       -> sk_factorized_* (host CSR + column-major blocks in, solution handle out),
//          factors copied back into DenseMatrix values (the reference returns V, core, W
//          by value, factorized_solvers.cpp:194-195; Lyapunov: W is a copy of V)
//   true_residual / true_residual_factors -> sk_true_residual_factors (device TSQR)
//   embed / embed_to / small_sylvester_apply -> small host helpers (declared in the same
//          header, used by the reference's tests), written against DenseMatrix's accessors
//
// Errors: the C-ABI's negative codes are re-thrown as the reference's own exception types
// (errors.hpp:9-57) with the library's message; numerical outcomes are reported in
// FactorizedSolution::status exactly like the reference (converged / max_iter / breakdown).
// Environment: SYLKRYLOV_B200_DEVICE selects the CUDA ordinal (default 0).
#include <cstdint>
#include <cstdlib>
#include <string>
#include <vector>

#include "sylkrylov/errors.hpp"
#include "sylkrylov/factorized_solvers.hpp"
#include "sylkrylov_b200.h"

namespace sylkrylov {
namespace {

static_assert(sizeof(index_t) == sizeof(int64_t), "the C-ABI carries the reference's 64-bit index_t as int64_t");

[[noreturn]] void rethrow(sk_status rc) {
    const std::string msg = sk_last_error();
    switch (rc) {
        case SK_ERR_DIMENSION: throw DimensionError(msg);
        case SK_ERR_INVALID_MATRIX: throw InvalidMatrixError(msg);
        case SK_ERR_RANK_DEFICIENT: throw RankDeficientStartError(msg);
        case SK_ERR_IO: throw IoError(msg);
        default: throw std::runtime_error("sylkrylov-b200: " + msg);  // CUDA / memory / capacity
    }
}
inline void check(sk_status rc) {
    if (rc != SK_OK) rethrow(rc);
}

sk_csr view(const SparseMatrix& a) {
    return sk_csr{a.rows(), a.cols(), a.nnz(), reinterpret_cast<const int64_t*>(a.row_ptr().data()),
                  reinterpret_cast<const int64_t*>(a.col_idx().data()), a.values().data()};
}
sk_config view(const SolverConfig& c) {
    return sk_config{c.eps_tol, static_cast<int64_t>(c.max_iter), c.breakdown_tol, c.capture_iterates ? 1 : 0,
                     c.lanczos_full_reorth ? 1 : 0};
}
sk_gpu_options device_options() {
    sk_gpu_options g{};
    if (const char* e = std::getenv("SYLKRYLOV_B200_DEVICE")) g.device = std::atoi(e);
    return g;
}

struct Handle {  // frees the device-side solution on every exit path
    sk_solution* h = nullptr;
    ~Handle() { sk_solution_free(h); }
};

FactorizedSolution collect(sk_solution* h, bool lyapunov) {
    FactorizedSolution out;
    int64_t n = 0, rv = 0, m = 0, rw = 0;
    sk_solution_dims(h, &n, &rv, &m, &rw);
    out.V = DenseMatrix(n, rv);
    out.core = DenseMatrix(rv, rw);
    check(sk_solution_copy_V(h, out.V.data()));
    check(sk_solution_copy_core(h, out.core.data()));
    if (lyapunov) {
        out.W = out.V;  // factorized_solvers.cpp:195
    } else {
        out.W = DenseMatrix(m, rw);
        check(sk_solution_copy_W(h, out.W.data()));
    }
    const int64_t nrec = sk_solution_num_records(h);
    std::vector<sk_iteration_record> rec(static_cast<size_t>(nrec));
    check(sk_solution_history(h, rec.data(), nrec));
    out.history.records.reserve(rec.size());
    for (const sk_iteration_record& r : rec) {
        IterationRecord x;
        x.iteration = static_cast<index_t>(r.iteration);
        x.rel_residual = r.rel_residual;
        x.t_basic_s = r.t_basic_s;
        x.t_krylov_s = r.t_krylov_s;
        x.t_trunc_s = r.t_trunc_s;
        out.history.records.push_back(x);
    }
    out.history.total_time_s = sk_solution_total_time(h);
    switch (sk_solution_status(h)) {
        case SK_SOLVE_CONVERGED: out.status = SolveStatus::converged; break;
        case SK_SOLVE_BREAKDOWN: out.status = SolveStatus::breakdown; break;
        default: out.status = SolveStatus::max_iter; break;
    }
    const int64_t ncap = sk_solution_num_captured(h);
    for (int64_t i = 0; i < ncap; ++i) {
        int64_t r = 0, c = 0;
        check(sk_solution_captured_core(h, i, &r, &c, nullptr));
        DenseMatrix x(r, c);
        check(sk_solution_captured_core(h, i, &r, &c, x.data()));
        out.captured_cores.push_back(std::move(x));
    }
    return out;
}

void require_two_sided(const SparseMatrix& a, const SparseMatrix& b, const DenseMatrix& c1, const DenseMatrix& c2) {
    // the reference's messages (factorized_solvers.cpp:50-58); the library repeats the checks
    if (a.rows() != a.cols() || b.rows() != b.cols()) throw DimensionError("solver: A and B must be square");
    if (c1.rows() != a.rows() || c2.rows() != b.rows())
        throw DimensionError("solver: C1/C2 row counts must match A/B");
    if (c1.cols() != c2.cols() || c1.cols() < 1)
        throw DimensionError("solver: C1 and C2 must have the same positive column count");
}

}  // namespace

DenseMatrix embed_to(const DenseMatrix& m, index_t rows, index_t cols) {
    if (rows < m.rows() || cols < m.cols()) throw DimensionError("embed: target smaller than matrix");
    DenseMatrix out(rows, cols);
    for (index_t j = 0; j < m.cols(); ++j)
        for (index_t i = 0; i < m.rows(); ++i) out(i, j) = m(i, j);
    return out;
}

DenseMatrix embed(const DenseMatrix& m, index_t target) { return embed_to(m, target, target); }

DenseMatrix small_sylvester_apply(const DenseMatrix& p, const DenseMatrix& h, const DenseMatrix& g) {
    if (h.cols() != p.rows() || g.cols() != p.cols())
        throw DimensionError("small_sylvester_apply: shapes do not conform");
    DenseMatrix out(h.rows(), g.rows());
    // [H P, 0]: rows of H, the first p.cols() columns
    for (index_t j = 0; j < p.cols(); ++j)
        for (index_t l = 0; l < p.rows(); ++l) {
            const double plj = p(l, j);
            for (index_t i = 0; i < h.rows(); ++i) out(i, j) += h(i, l) * plj;
        }
    // [P G^T; 0]: the first p.rows() rows, all g.rows() columns
    for (index_t j = 0; j < g.rows(); ++j)
        for (index_t l = 0; l < p.cols(); ++l) {
            const double gjl = g(j, l);
            for (index_t i = 0; i < p.rows(); ++i) out(i, j) += p(i, l) * gjl;
        }
    return out;
}

FactorizedSolution factorized_cg(const SparseMatrix& a, const SparseMatrix& b, const DenseMatrix& c1,
                                 const DenseMatrix& c2, const SolverConfig& cfg) {
    require_two_sided(a, b, c1, c2);
    const sk_csr ca = view(a), cb = view(b);
    const sk_config cc = view(cfg);
    const sk_gpu_options g = device_options();
    Handle s;
    check(sk_factorized_cg(&ca, &cb, c1.data(), c2.data(), c1.cols(), &cc, &g, &s.h));
    return collect(s.h, false);
}

FactorizedSolution factorized_cg_lyapunov(const SparseMatrix& a, const DenseMatrix& c1, const SolverConfig& cfg) {
    if (a.rows() != a.cols()) throw DimensionError("factorized_cg_lyapunov: A must be square");
    if (c1.rows() != a.rows()) throw DimensionError("factorized_cg_lyapunov: C1 rows must match A");
    const sk_csr ca = view(a);
    const sk_config cc = view(cfg);
    const sk_gpu_options g = device_options();
    Handle s;
    check(sk_factorized_cg_lyapunov(&ca, c1.data(), c1.cols(), &cc, &g, &s.h));
    return collect(s.h, true);
}

FactorizedSolution factorized_bicgstab(const SparseMatrix& a, const SparseMatrix& b, const DenseMatrix& c1,
                                       const DenseMatrix& c2, const SolverConfig& cfg) {
    require_two_sided(a, b, c1, c2);
    const sk_csr ca = view(a), cb = view(b);
    const sk_config cc = view(cfg);
    const sk_gpu_options g = device_options();
    Handle s;
    check(sk_factorized_bicgstab(&ca, &cb, c1.data(), c2.data(), c1.cols(), &cc, &g, &s.h));
    return collect(s.h, false);
}

double true_residual_factors(const SparseMatrix& a, const SparseMatrix& b, const DenseMatrix& c1,
                             const DenseMatrix& c2, const DenseMatrix& v, const DenseMatrix& core,
                             const DenseMatrix& w) {
    // the reference's checks and messages (factorized_solvers.cpp:395-400)
    if (a.rows() != a.cols() || b.rows() != b.cols()) throw DimensionError("true_residual: A and B must be square");
    if (c1.rows() != a.rows() || c2.rows() != b.rows() || c1.cols() != c2.cols())
        throw DimensionError("true_residual: right-hand side shapes do not conform");
    if (v.rows() != a.rows() || w.rows() != b.rows() || core.rows() != v.cols() || core.cols() != w.cols())
        throw DimensionError("true_residual: factor shapes do not conform");
    const sk_csr ca = view(a), cb = view(b);
    double rel = 0.0;
    check(sk_true_residual_factors(&ca, &cb, c1.data(), c2.data(), c1.cols(), v.data(), v.cols(), core.data(),
                                   w.data(), w.cols(), &rel));
    return rel;
}

double true_residual(const SparseMatrix& a, const SparseMatrix& b, const DenseMatrix& c1, const DenseMatrix& c2,
                     const FactorizedSolution& sol) {
    return true_residual_factors(a, b, c1, c2, sol.V, sol.core, sol.W);
}

}  // namespace sylkrylov
