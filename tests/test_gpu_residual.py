"""Device true residual (true_residual / true_residual_factors,
factorized_solvers.cpp:391-444) against the oracle's reference-order restatement
and dense numpy residuals. Floating point (Householder TSQR on the device against
the reference's sequential Householder QR): tolerances are written per test."""
import numpy as np
import pytest

from helpers import to_sk

pytestmark = pytest.mark.gpu


def fro(x):
    return float(np.sqrt(np.sum(x * x)))


def dense_residual(a, b, c1, c2, x):
    c = c1 @ c2.T
    return fro(c - a.dense() @ x - x @ b.dense()) / fro(c)


def test_known_answers(sk, po):
    """TrueResidual.* (test_factorized_kernels.cpp:99-154) through the device path."""
    a = po.from_triplets(1, 1, [0], [0], [3.0])
    b = po.from_triplets(1, 1, [0], [0], [2.0])
    r = sk.true_residual_factors(to_sk(sk, a), to_sk(sk, b), np.array([[10.0]]), np.array([[1.0]]),
                                 np.eye(1), np.array([[2.0]]), np.eye(1))
    assert r <= 1e-15
    a, b = po.random_spd(6, 70), po.random_spd(5, 71)
    c1, c2 = po.random_dense(6, 2, 72), po.random_dense(5, 2, 73)
    v = np.zeros((6, 3)); w = np.zeros((5, 3))
    v[0, 0] = v[1, 1] = v[2, 2] = 1.0; w[0, 0] = w[1, 1] = w[2, 2] = 1.0
    r = sk.true_residual_factors(to_sk(sk, a), to_sk(sk, b), c1, c2, v, np.zeros((3, 3)), w)
    assert abs(r - 1.0) <= 1e-14
    for (n, m, s, rk, sa, sb) in [(9, 7, 2, 4, 74, 75), (4, 4, 2, 3, 81, 82)]:
        a = po.random_sparse(n, n, 0.4, sa) if n == 9 else po.random_spd(n, sa)
        b = po.random_sparse(m, m, 0.4, sb) if n == 9 else po.random_spd(m, sb)
        c1, c2 = po.random_dense(n, s, sa + 2), po.random_dense(m, s, sa + 3)
        v, w, core = po.random_dense(n, rk, sa + 4), po.random_dense(m, rk, sa + 5), po.random_dense(rk, rk, sa + 6)
        e = dense_residual(a, b, c1, c2, v @ core @ w.T)
        got = sk.true_residual_factors(to_sk(sk, a), to_sk(sk, b), c1, c2, v, core, w)
        ref = po.true_residual_factors(a, b, c1, c2, v, core, w)
        assert abs(got - e) <= 1e-12 * e
        assert abs(got - ref) <= 1e-12 * ref


@pytest.mark.parametrize("chunk", [None, "333"])
def test_config1_solution_vs_oracle(sk, po, chunk, monkeypatch):
    """BASELINE config 1 converged solution: device residual (factors in HBM) vs the
    oracle on the downloaded factors; `chunk` forces a many-chunk TSQR."""
    if chunk:
        monkeypatch.setenv("SK_TR_CHUNK", chunk)
    a = po.laplacian_2d(64)
    c1 = po.random_rhs(4096, 1, 1234); c1 /= np.linalg.norm(c1)
    c2 = po.random_rhs(4096, 1, 1235); c2 /= np.linalg.norm(c2)
    A = to_sk(sk, a)
    sol = sk.factorized_cg(A, A, c1, c2, sk.SolverConfig(eps_tol=1e-8, max_iter=500))
    got = sk.true_residual(A, A, c1, c2, sol)
    ref = po.true_residual_factors(a, a, c1, c2, sol.V, sol.core, sol.W)
    assert ref < 1e-7
    assert abs(got - ref) <= 1e-6 * ref, (got, ref)
    # the factor-upload entry agrees with the resident one
    got2 = sk.true_residual_factors(A, A, c1, c2, sol.V, sol.core, sol.W)
    assert abs(got2 - ref) <= 1e-6 * ref


def test_lyapunov_resident_problem(sk, po):
    a = po.laplacian_2d(40)
    c1 = po.random_rhs(1600, 2, 9)
    prob = sk.ResidentProblem("cg_lyapunov", to_sk(sk, a), None, c1)
    sol = prob.solve(sk.SolverConfig(eps_tol=1e-8))
    got = prob.true_residual(sol)
    ref = po.true_residual_factors(a, a, c1, c1, sol.V, sol.core, sol.W)
    assert abs(got - ref) <= 1e-6 * ref, (got, ref)
    sol.free()
    prob.free()


@pytest.mark.parametrize("kind", ["stencil", "csr"])
def test_bicgstab_nonsymmetric(sk, po, kind):
    """Nonsymmetric B: B^T as a mirrored stencil or a transposed CSR (with a halo
    of the CSR bandwidth); a few iterations, the residual is O(1e-2 .. 1)."""
    if kind == "stencil":
        a = po.convection_diffusion_2d(24, (10.0, 10.0))
        b = po.convection_diffusion_2d(20, (10.0, -10.0))
    else:
        a = po.random_diag_dominant(300, 5)
        b = po.random_diag_dominant(250, 6)
    c1, c2 = po.random_rhs(a.n_rows, 2, 3), po.random_rhs(b.n_rows, 2, 4)
    A, B = to_sk(sk, a), to_sk(sk, b)
    sol = sk.factorized_bicgstab(A, B, c1, c2, sk.SolverConfig(eps_tol=1e-12, max_iter=6))
    got = sk.true_residual(A, B, c1, c2, sol)
    e = dense_residual(a, b, c1, c2, sol.V @ sol.core @ sol.W.T)
    assert abs(got - e) <= 1e-10 * e + 1e-14, (got, e)


def test_zero_rhs_and_shapes(sk, po):
    a = po.laplacian_2d(8)
    A = to_sk(sk, a)
    with pytest.raises(sk.InvalidMatrixError):
        sk.true_residual_factors(A, A, np.zeros((64, 1)), np.zeros((64, 1)), np.ones((64, 2)),
                                 np.ones((2, 2)), np.ones((64, 2)))
    with pytest.raises(sk.DimensionError):
        sk.true_residual_factors(A, A, np.ones((64, 1)), np.ones((64, 1)), np.ones((64, 2)),
                                 np.ones((3, 2)), np.ones((64, 2)))


def test_config5_true_residual_tracks_history(sk):
    """BASELINE config 5 at full size (n = m = 16.7M, r = 400: the stacked factors
    would be 107 GB and are streamed): the device true residual equals the
    recurrence's residual history to 1e-6 relative (size-independent property)."""
    from paper_2605_28274_b200.problems import baseline_config
    cfg = baseline_config(5)
    prob = sk.ResidentProblem(cfg.method, cfg.a, cfg.b, cfg.c1, cfg.c2)
    try:
        sol = prob.solve(sk.SolverConfig(eps_tol=cfg.eps_tol, max_iter=cfg.max_iter))
        r = prob.true_residual(sol)
        h = sol.history.final_rel_residual()
        assert abs(r - h) <= 1e-6 * h, (r, h)
        sol.free()
    finally:
        prob.free()


def test_fp64_peak_microbenchmark_is_sane(sk):
    """sk_measure_fp64_peak (the FP64 roofline denominator in bench.py): DFMA chains reach
    about twice the flop rate of mul-then-add chains, both in the B200's range."""
    dfma, dmuladd = sk.measure_fp64_peak(0)
    assert 15.0 < dfma < 90.0, dfma
    assert 8.0 < dmuladd < 45.0, dmuladd
    assert 1.5 < dfma / dmuladd < 2.5


def test_copy_factors_staged_equals_blockwise(sk, po):
    """sk_solution_copy_V/W (double-buffered export + multi-lane staged D2H) against the
    column-range accessor."""
    a = po.laplacian_2d(40)
    c1, c2 = po.random_rhs(a.n_rows, 2, 3), po.random_rhs(a.n_rows, 2, 4)
    sol = sk.factorized_cg(to_sk(sk, a), to_sk(sk, a), c1, c2, sk.SolverConfig(eps_tol=1e-6))
    v = sol.V
    ref = po.factorized_cg(a, a, c1, c2, po.Config(eps_tol=1e-6), po.REPRODUCIBLE)
    assert np.array_equal(v, ref.V) and np.array_equal(sol.W, ref.W)
    pv = sk.pinned_empty(v.shape)
    import ctypes as C
    from paper_2605_28274_b200 import _check, _p, lib
    _check(lib().sk_solution_copy_V(sol._h, _p(pv)))
    assert np.array_equal(pv, v)
