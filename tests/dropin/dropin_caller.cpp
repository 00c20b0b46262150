// A reference-style caller compiled against the reference's OWN headers (unchanged,
// /root/reference/proj/include) and linked with
//   - the reference's own Eigen-free sources (oracle/_ref/libsylkrylov_ref.so:
//     sparse_matrix.cpp, problems.cpp, matrix_market.cpp, parallel.cpp, solver_types.cpp),
//   - paper_2605_28274_b200/dropin/factorized_solvers_b200.cpp in place of the reference's
//     src/factorized_solvers.cpp,
//   - libsk_b200.so.
// It does what tools/main.cpp:96-185 does (Matrix Market in, solve, true residual) plus the
// reference's error cases, and prints the histories with 17 digits for the parity test.
// TEST CODE: built by oracle/build_ref.sh into oracle/_ref/dropin_caller (needs /root/reference
// to compile; the built binary travels to the GPU box).
#include <array>
#include <cstdio>
#include <string>

#include "sylkrylov/errors.hpp"
#include "sylkrylov/factorized_solvers.hpp"
#include "sylkrylov/matrix_market.hpp"
#include "sylkrylov/problems.hpp"
#include "sylkrylov/sparse_matrix.hpp"

using namespace sylkrylov;

static void print_solution(const char* name, const FactorizedSolution& sol, double tr) {
    std::printf("%s status=%s iterations=%td rv=%td rw=%td n=%td m=%td true_residual=%.6e\n", name,
                to_string(sol.status), sol.history.iterations(), sol.core.rows(), sol.core.cols(), sol.V.rows(),
                sol.W.rows(), tr);
    std::printf("%s history", name);
    for (const IterationRecord& r : sol.history.records) std::printf(" %.17g", r.rel_residual);
    std::printf("\n");
    double vsum = 0.0, csum = 0.0, wsum = 0.0;
    for (double x : sol.V.values()) vsum += x * x;
    for (double x : sol.core.values()) csum += x * x;
    for (double x : sol.W.values()) wsum += x * x;
    std::printf("%s fro2 V=%.17g core=%.17g W=%.17g\n", name, vsum, csum, wsum);
}

int main(int argc, char** argv) {
    const std::string dir = argc > 1 ? argv[1] : "/tmp";
    // Matrix Market round trip through the reference's own reader / writer (main.cpp:100-103)
    const SparseMatrix lap = laplacian_2d(24);
    write_matrix_market(lap, dir + "/A.mtx");
    const SparseMatrix a = read_matrix_market_sparse(dir + "/A.mtx");
    const DenseMatrix c1 = random_rhs(a.rows(), 2, 1234), c2 = random_rhs(a.rows(), 2, 1235);
    SolverConfig cfg;
    cfg.eps_tol = 1e-8;

    const FactorizedSolution cg = factorized_cg(a, a, c1, c2, cfg);
    print_solution("cg", cg, true_residual(a, a, c1, c2, cg));

    const FactorizedSolution ly = factorized_cg_lyapunov(a, c1, cfg);
    print_solution("lyapunov", ly, true_residual(a, a, c1, c1, ly));

    const SparseMatrix ca = convection_diffusion_3d(8, std::array<double, 3>{10.0, 10.0, 10.0});
    const DenseMatrix d1 = random_rhs(ca.rows(), 2, 99), d2 = random_rhs(ca.rows(), 2, 100);
    const FactorizedSolution bi = factorized_bicgstab(ca, ca, d1, d2, cfg);
    print_solution("bicgstab", bi, true_residual(ca, ca, d1, d2, bi));

    // error behaviour (factorized_solvers.cpp:50-58, 207-208; block_krylov.cpp:38-40)
    int ok = 0;
    try {
        factorized_cg(ca, ca, d1, d2, cfg);
    } catch (const InvalidMatrixError& e) {
        ok += 1;
        std::printf("nonsymmetric: InvalidMatrixError: %s\n", e.what());
    }
    try {
        factorized_cg(a, a, c1, d2, cfg);
    } catch (const DimensionError& e) {
        ok += 1;
        std::printf("shape: DimensionError: %s\n", e.what());
    }
    try {
        DenseMatrix z(a.rows(), 2);  // zero block: rank deficient start
        factorized_cg(a, a, z, c2, cfg);
    } catch (const RankDeficientStartError& e) {
        ok += 1;
        std::printf("rankdef: RankDeficientStartError: %s\n", e.what());
    }
    // embed / small_sylvester_apply (declared in the same header)
    DenseMatrix p(2, 2), h(3, 2), g(3, 2);
    p(0, 0) = 1; p(1, 1) = 2; h(0, 0) = 1; h(1, 1) = 1; h(2, 1) = 0.5; g(0, 0) = 2; g(1, 1) = 1; g(2, 0) = 3;
    const DenseMatrix q = small_sylvester_apply(p, h, g);
    std::printf("image %td x %td: q00=%.17g q11=%.17g q21=%.17g q02=%.17g\n", q.rows(), q.cols(), q(0, 0), q(1, 1),
                q(2, 1), q(0, 2));
    std::printf("errors_ok=%d\n", ok);
    return ok == 3 ? 0 : 1;
}
