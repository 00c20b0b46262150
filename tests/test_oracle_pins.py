"""Pins the CPU oracle (oracle/) against the reference's own known-answer tests,
re-expressed from proj/tests/*.cpp (GTest is absent, so pytest + numpy dense
oracles stand in for oracles.hpp / Eigen). Every test runs in both arithmetic
modes where the reference test is mode-independent. CPU only."""
import json
import os

import numpy as np
import pytest

from oracle import pyoracle as po

MODES = [po.REPRODUCIBLE, po.REFERENCE_ORDER]
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def fro(x):
    return float(np.linalg.norm(x))


# ---------------------------------------------------------------- generators
def test_rng_matches_libstdcxx_golden():
    """problems.cpp:65-96 and oracles.hpp:39-46, pinned against g++'s <random>."""
    g = json.load(open(os.path.join(GOLDEN, "rng_golden.json")))
    rhs = po.random_rhs(7, 1, 1234)[:, 0]
    assert np.array_equal(rhs, np.array(g["random_rhs_7_1234"]))
    dense = po.random_dense(5, 2, 7)
    assert np.array_equal(dense.ravel(order="F"), np.array(g["random_dense_5x2_7"]))


def test_random_rhs_deterministic():
    """test_problems.cpp:47-53: bitwise re-runs."""
    assert np.array_equal(po.random_rhs(100, 3, 9), po.random_rhs(100, 3, 9))
    assert not np.array_equal(po.random_rhs(100, 3, 9), po.random_rhs(100, 3, 10))


@pytest.mark.parametrize("grid", [2, 3, 7])
def test_laplacian_emitter_equals_triplet_path(grid):
    """The direct CSR emitter equals from_triplets over the reference's stream (problems.cpp:10-30)."""
    a = po.laplacian_2d(grid)
    rows, cols, vals = [], [], []
    idx = lambda ix, iy: ix + grid * iy
    for iy in range(grid):
        for ix in range(grid):
            p = idx(ix, iy)
            rows.append(p); cols.append(p); vals.append(4.0)
            if ix > 0: rows.append(p); cols.append(idx(ix - 1, iy)); vals.append(-1.0)
            if ix < grid - 1: rows.append(p); cols.append(idx(ix + 1, iy)); vals.append(-1.0)
            if iy > 0: rows.append(p); cols.append(idx(ix, iy - 1)); vals.append(-1.0)
            if iy < grid - 1: rows.append(p); cols.append(idx(ix, iy + 1)); vals.append(-1.0)
    t = po.from_triplets(grid * grid, grid * grid, rows, cols, vals)
    assert np.array_equal(a.row_ptr, t.row_ptr) and np.array_equal(a.col_idx, t.col_idx)
    assert np.array_equal(a.values, t.values)


def test_convection_diffusion_3d_structure():
    """problems.cpp:32-60: -1 -/+ w h/2 couplings, diagonal 6, nonsymmetric with wind."""
    g = 4
    a = po.convection_diffusion_3d(g, (10.0, 10.0, 10.0))
    d = a.dense()
    h = 1.0 / (g + 1)
    assert d[0, 0] == 6.0
    assert d[0, 1] == -1.0 + 10.0 * h / 2.0
    assert d[1, 0] == -1.0 - 10.0 * h / 2.0
    assert not po.is_symmetric(a)
    assert po.is_symmetric(po.convection_diffusion_3d(g, (0.0, 0.0, 0.0)))
    b = po.convection_diffusion_2d(5, (10.0, -10.0))
    assert b.nnz == 5 * 25 - 4 * 5


def test_sparse_invariants_and_symmetry():
    """test_core_linalg.cpp:191-209."""
    with pytest.raises(po.OracleError):
        po.from_triplets(2, 2, [0], [2], [1.0])
    assert po.is_symmetric(po.from_triplets(2, 2, [0, 0, 1, 1], [0, 1, 0, 1], [2.0, -1.0, -1.0, 2.0]))
    assert not po.is_symmetric(po.from_triplets(2, 2, [0, 1], [1, 0], [1.0, 2.0]))


def test_duplicates_summed():
    t = po.from_triplets(2, 2, [0, 0, 1], [1, 1, 0], [1.0, 2.5, 4.0])
    assert t.nnz == 2 and t.values[0] == 3.5


# ---------------------------------------------------------------- SpMM
def test_spmm_identity_and_tridiagonal():
    """Spmm.IdentityPassesThrough / TridiagonalRowSums (test_core_linalg.cpp:11-27)."""
    x = po.random_dense(3, 2, 11)
    assert np.array_equal(po.spmm(po.Csr.identity(3), x), x)
    a = po.from_triplets(3, 3, [0, 0, 1, 1, 1, 2, 2], [0, 1, 0, 1, 2, 1, 2], [2, -1, -1, 2, -1, -1, 2])
    y = po.spmm(a, np.ones((3, 1)))
    assert list(y[:, 0]) == [1.0, 0.0, 1.0]


def test_spmm_matches_dense():
    """Spmm.MatchesDenseOracle (1e-14) and DistributesOverAddition (1e-13)."""
    a = po.random_sparse(50, 50, 0.1, 42)
    x = po.random_dense(50, 4, 43)
    e = a.dense() @ x
    assert fro(po.spmm(a, x) - e) <= 1e-14 * fro(e)
    b = po.random_sparse(40, 40, 0.15, 7)
    x, y = po.random_dense(40, 3, 8), po.random_dense(40, 3, 9)
    lhs = po.spmm(b, x + y)
    assert fro(lhs - po.spmm(b, x) - po.spmm(b, y)) <= 1e-13 * fro(lhs)


def test_spmm_transpose_known_answers():
    """SpmmTranspose.SingleEntry / MatchesDenseOracle (test_core_linalg.cpp:57-74)."""
    a = po.from_triplets(3, 3, [1], [0], [5.0])
    e2 = np.zeros((3, 1)); e2[1] = 1.0
    assert list(po.spmm_transpose(a, e2)[:, 0]) == [5.0, 0.0, 0.0]
    a = po.random_sparse(30, 40, 0.2, 44)
    x = po.random_dense(30, 5, 45)
    e = a.dense().T @ x
    assert fro(po.spmm_transpose(a, x) - e) <= 1e-14 * fro(e)


def test_spmm_transpose_equals_gather_on_transposed_csr():
    """The device's gather over transposed() reproduces the scatter order exactly."""
    a = po.random_sparse(64, 48, 0.2, 3)
    x = po.random_dense(64, 3, 4)
    assert np.array_equal(po.spmm_transpose(a, x), po.spmm(po.transpose(a), x))


# ---------------------------------------------------------------- inner products
def test_frobenius_inner_known_answers():
    """FrobeniusInner.* (test_core_linalg.cpp:84-107)."""
    assert po.frobenius_inner(np.eye(2), np.eye(2)) == 2.0
    x = np.array([[1.0, 2.0], [3.0, 4.0]])
    y = np.array([[5.0, 6.0], [7.0, 8.0]])
    assert po.frobenius_inner(x, y) == 70.0
    assert po.r2_inner(x, y) == 70.0
    x, y = po.random_dense(7, 5, 20), po.random_dense(7, 5, 21)
    flat = float(np.sum(x.ravel(order="F") * y.ravel(order="F")))
    assert abs(po.frobenius_inner(x, y) - flat) <= 1e-15 * abs(flat)
    assert abs(po.r2_inner(x, y) - flat) <= 1e-14 * abs(flat)


def test_reduction_contracts_are_accurate():
    """R1/R2 trees sum the same terms as the sequential loop, to rounding."""
    rng = np.random.default_rng(5)
    v = rng.standard_normal(100_003)
    w = rng.standard_normal(100_003)
    exact = float(np.dot(v.astype(np.longdouble), w.astype(np.longdouble)))
    assert abs(po.r1_dot(v, w) - exact) <= 1e-12 * np.abs(v * w).sum()
    m1 = rng.standard_normal((97, 131))
    m2 = rng.standard_normal((97, 131))
    assert abs(po.r2_inner(m1, m2) - float(np.sum(m1 * m2))) <= 1e-12 * np.abs(m1 * m2).sum()


# ---------------------------------------------------------------- QR / SVD
def test_thin_qr_known_answers():
    """ThinQr.* (test_core_linalg.cpp:113-153)."""
    q, r = po.thin_qr(np.eye(3))
    assert fro(q - np.eye(3)) <= 1e-15 and fro(r - np.eye(3)) <= 1e-15
    q, r = po.thin_qr(np.array([[3.0], [4.0]]))
    assert abs(q[0, 0] - 0.6) <= 1e-15 and abs(q[1, 0] - 0.8) <= 1e-15 and abs(r[0, 0] - 5.0) <= 1e-15
    x = po.random_dense(20, 3, 30)
    q, r = po.thin_qr(x)
    assert fro(q.T @ q - np.eye(3)) <= 1e-12
    assert fro(q @ r - x) <= 1e-12 * fro(x)
    assert np.all(np.diag(r) >= 0.0)
    for s in (8, 32, 64):
        q, _ = po.thin_qr(po.random_dense(200, s, 31 + s))
        assert fro(q.T @ q - np.eye(s)) <= 1e-12 * s
    x = np.zeros((6, 3)); x[:, 0] = np.arange(1, 7); x[:, 2] = 2 * np.arange(1, 7)
    q, r = po.thin_qr(x)
    assert fro(q @ r - x) <= 1e-12 * fro(x)
    with pytest.raises(po.OracleError):
        po.thin_qr(np.zeros((2, 4)))


def test_singular_extremes():
    """Svd.DiagonalValues / RankOneOuterProduct (test_core_linalg.cpp:167-189)."""
    smax, smin = po.singular_extremes(np.array([[3.0, 0.0], [0.0, 1.0]]))
    assert abs(smax - 3.0) <= 1e-14 and abs(smin - 1.0) <= 1e-14
    u = po.random_dense(4, 1, 50); u /= fro(u)
    v = po.random_dense(4, 1, 51); v /= fro(v)
    smax, smin = po.singular_extremes(u @ v.T)
    assert abs(smax - 1.0) <= 1e-13 and abs(smin) <= 1e-13
    m = po.random_dense(6, 6, 52)
    sv = np.linalg.svd(m, compute_uv=False)
    smax, smin = po.singular_extremes(m)
    assert abs(smax - sv[0]) <= 1e-13 * sv[0] and abs(smin - sv[-1]) <= 1e-12 * sv[0]


# ---------------------------------------------------------------- block Krylov basis
def recurrence_residual(op_dense, basis, transpose=False):
    v = basis.matrix()
    h = basis.hessenberg()
    vk = v[:, :h.shape[1]]
    av = (op_dense.T if transpose else op_dense) @ vk
    return fro(av - v @ h)


def orth_defect(basis):
    v = basis.matrix()
    return fro(v.T @ v - np.eye(v.shape[1]))


def brute_krylov_orthonormal(a, c, k, rank_tol=1e-12):
    """oracles.hpp:122-144."""
    n = a.shape[0]
    q = np.zeros((n, 0))
    block = c.copy()
    for _ in range(k):
        z = block / np.linalg.norm(block)
        for _p in range(2):
            if q.shape[1]:
                z = z - q @ (q.T @ z)
        u, sv, _ = np.linalg.svd(z, full_matrices=False)
        keep = int(np.sum(sv > rank_tol))
        if keep:
            q = np.hstack([q, u[:, :keep]])
        block = a @ block
    return q


@pytest.mark.parametrize("mode", MODES)
def test_basis_init_known_answers(mode):
    """BasisInit.* (test_block_krylov.cpp:38-65)."""
    e0 = np.zeros((5, 1)); e0[0] = 1.0
    b = po.Basis(po.Csr.identity(5), e0, True, False, mode=mode)
    assert b.cols == 1 and abs(b.r[0, 0] - 1.0) <= 1e-15 and abs(b.matrix()[0, 0] - 1.0) <= 1e-15
    b = po.Basis(po.Csr.identity(3), np.array([[3.0], [4.0], [0.0]]), False, False, mode=mode)
    v = b.matrix()
    assert abs(v[0, 0] - 0.6) <= 1e-15 and abs(v[1, 0] - 0.8) <= 1e-15 and abs(b.r[0, 0] - 5.0) <= 1e-15
    start = np.zeros((4, 2)); start[:, 0] = start[:, 1] = np.arange(1.0, 5.0)
    with pytest.raises(po.OracleError) as ei:
        po.Basis(po.Csr.identity(4), start, True, False, mode=mode)
    assert ei.value.code == -3


@pytest.mark.parametrize("mode", MODES)
def test_hand_computed_lanczos_step(mode):
    """BasisExtend.HandComputedLanczosStep (test_block_krylov.cpp:67-83)."""
    op = po.from_triplets(2, 2, [0, 1], [0, 1], [2.0, 3.0])
    start = np.full((2, 1), 1.0 / np.sqrt(2.0))
    b = po.Basis(op, start, False, False, mode=mode)
    assert b.try_extend() == "grown"
    h = b.hessenberg()
    assert h.shape == (2, 1)
    assert abs(h[0, 0] - 2.5) <= 1e-14 and abs(h[1, 0] - 0.5) <= 1e-14
    v = b.matrix()
    assert abs(v[0, 1] + 1 / np.sqrt(2)) <= 1e-14 and abs(v[1, 1] - 1 / np.sqrt(2)) <= 1e-14


@pytest.mark.parametrize("mode", MODES)
def test_exhaustion_vs_breakdown(mode):
    """IdentityOperatorBreaksDownImmediately / ExhaustionIsDistinguished /
    PartialRankDeficiencyIsHardBreakdown (test_block_krylov.cpp:85-124)."""
    b = po.Basis(po.Csr.identity(6), po.random_dense(6, 2, 5), True, False, mode=mode)
    with pytest.raises(po.OracleError) as ei:
        b.extend()
    assert ei.value.code == -5 and b.exhausted and b.cols == 2
    h = b.hessenberg()
    assert h.shape == (2, 2) and fro(h - np.eye(2)) <= 1e-12
    assert b.try_extend() == "exhausted"
    b = po.Basis(po.random_spd(4, 17), po.random_dense(4, 3, 18), True, False, mode=mode)
    with pytest.raises(po.OracleError) as ei:
        b.extend()
    assert ei.value.code == -4
    with pytest.raises(po.OracleError):
        b.try_extend()


@pytest.mark.parametrize("mode", MODES)
def test_tridiagonal_recurrence(mode):
    """TridiagonalRecurrenceResidual (test_block_krylov.cpp:126-133)."""
    op = po.laplacian_2d(10)
    b = po.Basis(op, po.random_dense(100, 2, 7), False, False, mode=mode)
    for _ in range(10):
        assert b.try_extend() == "grown"
    assert recurrence_residual(op.dense(), b) <= 1e-12 * fro(b.hessenberg())


@pytest.mark.parametrize("mode", MODES)
def test_arnoldi_orthogonality(mode):
    """ArnoldiOrthogonalityStaysTight + AtFiveHundredColumns (test_block_krylov.cpp:135-223)."""
    op = po.random_sparse(120, 120, 0.1, 23)
    b = po.Basis(op, po.random_dense(120, 4, 24), True, False, mode=mode)
    for _ in range(14):
        assert b.try_extend() == "grown"
    assert orth_defect(b) <= 1e-10 * np.sqrt(b.cols)
    op = po.random_sparse(640, 640, 0.02, 40, 2.0)
    b = po.Basis(op, po.random_dense(640, 4, 41), True, False, mode=mode)
    while b.cols < 512:
        assert b.try_extend() == "grown"
    assert orth_defect(b) <= 1e-10 * np.sqrt(512.0)


@pytest.mark.parametrize("mode", MODES)
def test_lanczos_tridiagonal_symmetric(mode):
    """LanczosTridiagonalAndSymmetric (test_block_krylov.cpp:144-159): off-band exactly 0."""
    op = po.random_spd(60, 25)
    s = 3
    b = po.Basis(op, po.random_dense(60, s, 26), False, False, mode=mode)
    for _ in range(8):
        assert b.try_extend() == "grown"
    h = b.hessenberg()
    off, asym = 0.0, 0.0
    for j in range(h.shape[1]):
        for i in range(h.shape[0]):
            if i // s > j // s + 1 or j // s > i // s + 1:
                off += h[i, j] ** 2
            if i < h.shape[1] and j < h.shape[0]:
                asym += (h[i, j] - h[j, i]) ** 2
    assert off == 0.0
    assert np.sqrt(asym) <= 1e-12 * fro(h)


@pytest.mark.parametrize("mode", MODES)
def test_transpose_flag(mode):
    """TransposeFlagUsesOperatorTranspose (test_block_krylov.cpp:161-168)."""
    op = po.random_sparse(40, 40, 0.15, 27)
    b = po.Basis(op, po.random_dense(40, 2, 28), True, True, mode=mode)
    for _ in range(6):
        assert b.try_extend() == "grown"
    assert recurrence_residual(op.dense(), b, transpose=True) <= 1e-12 * fro(b.hessenberg())


@pytest.mark.parametrize("mode", MODES)
def test_spans_brute_force_krylov(mode):
    """SpansBruteForceKrylovSpace (test_block_krylov.cpp:170-184)."""
    op = po.random_sparse(30, 30, 0.3, 29)
    start = po.random_dense(30, 2, 30)
    b = po.Basis(op, start, True, False, mode=mode)
    for _ in range(4):
        assert b.try_extend() == "grown"
    v = b.matrix()
    q = brute_krylov_orthonormal(op.dense(), start, 5)
    assert q.shape[1] == v.shape[1]
    assert fro(v - q @ (q.T @ v)) <= 1e-8


@pytest.mark.parametrize("mode", MODES)
def test_lanczos_agrees_with_arnoldi(mode):
    """LanczosAgreesWithArnoldiOnSymmetricOperators (test_block_krylov.cpp:186-214)."""
    op = po.random_spd(50, 31)
    start = po.random_dense(50, 2, 32)
    lan = po.Basis(op, start, False, False, mode=mode)
    arn = po.Basis(op, start, True, False, mode=mode)
    for _ in range(10):
        assert lan.try_extend() == "grown" and arn.try_extend() == "grown"
    vl, va = lan.matrix(), arn.matrix()
    for blk in range(lan.cols // 2):
        bl, ba = vl[:, 2 * blk:2 * blk + 2], va[:, 2 * blk:2 * blk + 2]
        assert fro(bl - ba @ (ba.T @ bl)) <= 1e-8
    hl, ha = lan.hessenberg(), arn.hessenberg()
    nl = np.sqrt((hl ** 2).sum(0))
    na = np.sqrt((ha ** 2).sum(0))
    assert np.all(np.abs(nl - na) <= 1e-8 * np.maximum(1.0, na))


@pytest.mark.parametrize("mode", MODES)
def test_lanczos_full_reorth(mode):
    """LanczosFullReorthKeepsGlobalOrthogonality (test_block_krylov.cpp:225-245)."""
    op = po.laplacian_2d(12)
    start = po.random_dense(144, 1, 42)
    plain = po.Basis(op, start, False, False, mode=mode)
    reo = po.Basis(op, start, False, False, lanczos_full_reorth=True, mode=mode)
    for _ in range(70):
        assert plain.try_extend() == "grown" and reo.try_extend() == "grown"
    assert orth_defect(reo) <= 1e-10 * np.sqrt(71.0)
    assert orth_defect(reo) <= orth_defect(plain)
    h = reo.hessenberg()
    for j in range(h.shape[1]):
        for i in range(h.shape[0]):
            if i > j + 1 or j > i + 1:
                assert h[i, j] == 0.0


@pytest.mark.parametrize("mode", MODES)
def test_banded_products(mode):
    """BandedProductsMatchAssembledHessenberg (test_block_krylov.cpp:247-264)."""
    op = po.laplacian_2d(8)
    s, j = 3, 4
    b = po.Basis(op, po.random_dense(64, s, 33), False, False, mode=mode)
    for _ in range(6):
        assert b.try_extend() == "grown"
    p = po.random_dense(j * s, j * s, 34)
    h = b.hessenberg((j + 1) * s, j * s)
    fast = np.zeros(((j + 1) * s, p.shape[1]), order="F")
    b.accumulate_h_times(p, fast)
    assert fro(fast - h @ p) <= 1e-13 * fro(h)
    fast2 = np.zeros((p.shape[0], (j + 1) * s), order="F")
    b.accumulate_times_ht(p, fast2)
    assert fro(fast2 - p @ h.T) <= 1e-13 * fro(h)


@pytest.mark.parametrize("mode", MODES)
def test_basis_invariants_random(mode):
    """acceptance criterion 6 (acceptance.cpp:217-266), 12 seeded operators."""
    rng = np.random.default_rng(6060)
    for inst in range(12):
        n = int(rng.integers(40, 201))
        s = int(rng.integers(1, 5))
        lanczos = inst % 2 == 1
        ks_limit = min(24 if lanczos else 60, ((n - s) // s) * s)
        ext = max(1, ks_limit // s - 1)
        seed = 7000 + inst
        a = po.random_spd(n, seed) if lanczos else po.random_sparse(n, n, 0.1, seed, 2.0)
        b = po.Basis(a, po.random_dense(n, s, seed + 500), not lanczos, False, mode=mode)
        for _ in range(ext):
            if b.try_extend() != "grown":
                break
        v, h = b.matrix(), b.hessenberg()
        assert orth_defect(b) / np.sqrt(v.shape[1]) <= 1e-10
        assert fro(a.dense() @ v[:, :h.shape[1]] - v @ h) / max(fro(h), 1e-300) <= 1e-12


# ---------------------------------------------------------------- factorized kernels
def test_small_sylvester_apply():
    """SmallSylvesterApply.ScalarFormula / ZeroInput (test_factorized_kernels.cpp:35-59)."""
    p, h1, h2, g1, g2 = 1.75, 2.0, -0.5, 3.0, 0.25
    out = po.small_sylvester_apply(np.array([[p]]), np.array([[h1], [h2]]), np.array([[g1], [g2]]))
    assert out[0, 0] == h1 * p + p * g1 and out[0, 1] == p * g2
    assert out[1, 0] == h2 * p and out[1, 1] == 0.0
    z = po.small_sylvester_apply(np.zeros((4, 4)), po.random_dense(6, 4, 5), po.random_dense(6, 4, 6))
    assert fro(z) == 0.0
    with pytest.raises(po.OracleError):
        po.small_sylvester_apply(np.zeros((2, 2)), np.zeros((3, 3)), np.zeros((3, 2)))


def test_small_sylvester_matches_dense_lift():
    """SmallSylvesterApply.MatchesDenseLift (test_factorized_kernels.cpp:61-92)."""
    n, s, j = 30, 2, 3
    a = po.random_sparse(n, n, 0.2, 60)
    b = po.random_sparse(n, n, 0.2, 61)
    c1, c2 = po.random_dense(n, s, 62), po.random_dense(n, s, 63)
    vb = po.Basis(a, c1, True, False)
    wb = po.Basis(b, c2, True, True)
    for _ in range(j):
        assert vb.try_extend() == "grown" and wb.try_extend() == "grown"
    p = po.random_dense(j * s, j * s, 64)
    h = vb.hessenberg((j + 1) * s, j * s)
    g = wb.hessenberg((j + 1) * s, j * s)
    img = po.small_sylvester_apply(p, h, g)
    v, w = vb.matrix()[:, :j * s], wb.matrix()[:, :j * s]
    vp, wp = vb.matrix()[:, :(j + 1) * s], wb.matrix()[:, :(j + 1) * s]
    x = v @ p @ w.T
    lhs = a.dense() @ x + x @ b.dense()
    assert fro(lhs - vp @ img @ wp.T) <= 1e-12 * fro(lhs)


def dense_residual(a, b, c1, c2, x):
    c = c1 @ c2.T
    return fro(c - a.dense() @ x - x @ b.dense()) / fro(c)


def test_true_residual_known_answers():
    """TrueResidual.* (test_factorized_kernels.cpp:99-154)."""
    a = po.from_triplets(1, 1, [0], [0], [3.0])
    b = po.from_triplets(1, 1, [0], [0], [2.0])
    r = po.true_residual_factors(a, b, np.array([[10.0]]), np.array([[1.0]]), np.eye(1), np.array([[2.0]]), np.eye(1))
    assert r <= 1e-15
    a, b = po.random_spd(6, 70), po.random_spd(5, 71)
    c1, c2 = po.random_dense(6, 2, 72), po.random_dense(5, 2, 73)
    v = np.zeros((6, 3)); w = np.zeros((5, 3))
    v[0, 0] = v[1, 1] = v[2, 2] = 1.0; w[0, 0] = w[1, 1] = w[2, 2] = 1.0
    assert abs(po.true_residual_factors(a, b, c1, c2, v, np.zeros((3, 3)), w) - 1.0) <= 1e-14
    for (n, m, s, r, sa, sb) in [(9, 7, 2, 4, 74, 75), (4, 4, 2, 3, 81, 82)]:
        a = po.random_sparse(n, n, 0.4, sa) if n == 9 else po.random_spd(n, sa)
        b = po.random_sparse(m, m, 0.4, sb) if n == 9 else po.random_spd(m, sb)
        c1, c2 = po.random_dense(n, s, sa + 2), po.random_dense(m, s, sa + 3)
        v, w, core = po.random_dense(n, r, sa + 4), po.random_dense(m, r, sa + 5), po.random_dense(r, r, sa + 6)
        e = dense_residual(a, b, c1, c2, v @ core @ w.T)
        assert abs(po.true_residual_factors(a, b, c1, c2, v, core, w) - e) <= 1e-12 * e


# ---------------------------------------------------------------- solvers
def kron_solve(a, b, c1, c2):
    """kron_solve (reference_solvers.cpp:392-429) via numpy."""
    n, m = a.n_rows, b.n_rows
    f = np.kron(np.eye(m), a.dense()) + np.kron(b.dense().T, np.eye(n))
    x = np.linalg.solve(f, (c1 @ c2.T).ravel(order="F"))
    return x.reshape((n, m), order="F")


def matrix_oriented_cg(a, b, c, eps, max_iter):
    """matrix_oriented_cg (reference_solvers.cpp:29-97) restated in numpy."""
    A, B = a.dense(), b.dense()
    x = np.zeros_like(c); r = c.copy(); p = r.copy()
    rho = float(np.sum(r * r)); n0 = np.sqrt(rho)
    hist = [1.0]
    for _ in range(max_iter):
        q = A @ p + p @ B
        alpha = rho / float(np.sum(r * q))
        x += alpha * p
        r -= alpha * q
        nr = np.linalg.norm(r)
        hist.append(nr / n0)
        if nr <= n0 * eps:
            break
        rn = float(np.sum(r * r))
        p = r + (rn / rho) * p
        rho = rn
    return np.array(hist)


def matrix_oriented_bicgstab(a, b, c, eps, max_iter):
    """matrix_oriented_bicgstab (reference_solvers.cpp:99-192) restated in numpy."""
    A, B = a.dense(), b.dense()
    op = lambda z: A @ z + z @ B
    x = np.zeros_like(c); r = c.copy(); rs = r.copy(); p = r.copy()
    rho = float(np.sum(r * rs)); n0 = np.sqrt(float(np.sum(r * r)))
    hist = [1.0]
    for _ in range(max_iter):
        q = op(p)
        alpha = rho / float(np.sum(rs * q))
        s = r - alpha * q
        t = op(s)
        tt, ss = float(np.sum(t * t)), float(np.sum(s * s))
        omega = 0.0 if np.sqrt(ss) <= eps * n0 else float(np.sum(t * s)) / tt
        x += alpha * p + omega * s
        r = s - omega * t
        nr = np.linalg.norm(r)
        hist.append(nr / n0)
        if nr <= n0 * eps:
            break
        rn = float(np.sum(r * rs))
        beta = (alpha / omega) * (rn / rho)
        p = r + beta * p - beta * omega * q
        rho = rn
    return np.array(hist)


def densified(sol):
    return sol.V @ sol.core @ sol.W.T


@pytest.mark.parametrize("mode", MODES)
def test_identity_pairs_converge_in_one_iteration(mode):
    """test_factorized_solvers.cpp:22-33, 76-85, 117-128."""
    c1, c2 = po.random_dense(7, 2, 1), po.random_dense(5, 2, 2)
    s = po.factorized_cg(po.Csr.identity(7), po.Csr.identity(5), c1, c2, None, mode)
    e = 0.5 * c1 @ c2.T
    assert s.status == "converged" and s.n_iterations == 1 and fro(densified(s) - e) <= 1e-13 * fro(e)
    c1 = po.random_dense(6, 2, 20)
    s = po.factorized_cg_lyapunov(po.Csr.identity(6), c1, None, mode)
    e = 0.5 * c1 @ c1.T
    assert s.status == "converged" and s.n_iterations == 1 and fro(densified(s) - e) <= 1e-13 * fro(e)
    c1, c2 = po.random_dense(6, 2, 30), po.random_dense(4, 2, 31)
    s = po.factorized_bicgstab(po.Csr.identity(6), po.Csr.identity(4), c1, c2, None, mode)
    e = 0.5 * c1 @ c2.T
    assert s.status == "converged" and s.n_iterations == 1 and fro(densified(s) - e) <= 1e-12 * fro(e)


@pytest.mark.parametrize("mode", MODES)
def test_cg_matches_kronecker(mode):
    """FactorizedCg.MatchesKroneckerOracle (1e-8) and BiCGSTAB (1e-7)."""
    a, b = po.random_spd(8, 10), po.random_spd(6, 11)
    c1, c2 = po.random_dense(8, 2, 12), po.random_dense(6, 2, 13)
    s = po.factorized_cg(a, b, c1, c2, po.Config(eps_tol=1e-10), mode)
    e = kron_solve(a, b, c1, c2)
    assert s.status == "converged" and fro(densified(s) - e) <= 1e-8 * fro(e)
    a, b = po.random_diag_dominant(9, 32), po.random_diag_dominant(7, 33)
    c1, c2 = po.random_dense(9, 1, 34), po.random_dense(7, 1, 35)
    s = po.factorized_bicgstab(a, b, c1, c2, po.Config(eps_tol=1e-9), mode)
    e = kron_solve(a, b, c1, c2)
    assert s.status == "converged" and fro(densified(s) - e) <= 1e-7 * fro(e)


@pytest.mark.parametrize("mode", MODES)
def test_acceptance_oracle_equivalence(mode):
    """acceptance criterion 1 (acceptance.cpp:54-96): 20 seeded instances vs Kronecker, 1e-7."""
    rng = np.random.default_rng(20240517)
    for inst in range(20):
        s = 1 + inst % 3
        n = int(rng.choice([v for v in range(4, 31) if v % s == 0]))
        m = int(rng.choice([v for v in range(4, 31) if v % s == 0]))
        seed = 1000 + 7 * inst
        cg = inst % 2 == 0
        a = po.random_spd(n, seed) if cg else po.random_diag_dominant(n, seed)
        b = po.random_spd(m, seed + 1) if cg else po.random_diag_dominant(m, seed + 1)
        c1, c2 = po.random_dense(n, s, seed + 2), po.random_dense(m, s, seed + 3)
        cfg = po.Config(eps_tol=1e-10)
        sol = po.factorized_cg(a, b, c1, c2, cfg, mode) if cg else po.factorized_bicgstab(a, b, c1, c2, cfg, mode)
        assert sol.status == "converged", (inst, sol.status)
        e = kron_solve(a, b, c1, c2)
        assert fro(densified(sol) - e) / fro(e) <= 1e-7, inst


@pytest.mark.parametrize("mode", MODES)
def test_rank_bookkeeping(mode):
    """RankBookkeepingIsExact (test_factorized_solvers.cpp:57-74, 146-162)."""
    a = po.laplacian_2d(9)
    s = po.factorized_cg_lyapunov(a, po.random_dense(81, 3, 17),
                                  po.Config(eps_tol=1e-30, max_iter=6, capture_iterates=True), mode)
    assert s.status == "max_iter" and len(s.captured) == 6
    for k, core in enumerate(s.captured):
        assert core.shape == ((k + 1) * 3, (k + 1) * 3)
    a = po.convection_diffusion_3d(4, (10.0, 10.0, 10.0))
    s = po.factorized_bicgstab(a, a, po.random_dense(64, 2, 36), po.random_dense(64, 2, 37),
                               po.Config(eps_tol=1e-30, max_iter=4, capture_iterates=True), mode)
    assert s.status == "max_iter" and len(s.captured) == 4
    for k, core in enumerate(s.captured):
        assert core.shape == ((2 * k + 2) * 2, (2 * k + 2) * 2)


@pytest.mark.parametrize("mode", MODES)
def test_lyapunov_agrees_with_sylvester(mode):
    """AgreesWithSylvesterRoute (test_factorized_solvers.cpp:87-101): 1e-10; bitwise in the
    reproducible contract."""
    a = po.laplacian_2d(10)
    c1 = po.random_dense(100, 2, 21)
    lyap = po.factorized_cg_lyapunov(a, c1, po.Config(eps_tol=1e-8), mode)
    sylv = po.factorized_cg(a, a, c1, c1, po.Config(eps_tol=1e-8), mode)
    assert lyap.status == "converged"
    assert lyap.rel_residual.size == sylv.rel_residual.size
    assert np.all(np.abs(lyap.rel_residual - sylv.rel_residual) <= 1e-10 * np.maximum(sylv.rel_residual, 1e-30))
    if mode == po.REPRODUCIBLE:
        assert np.array_equal(lyap.rel_residual, sylv.rel_residual)


@pytest.mark.parametrize("mode", MODES)
def test_lyapunov_core_symmetric(mode):
    """CoreStaysSymmetricEveryIteration (test_factorized_solvers.cpp:103-115)."""
    a = po.laplacian_2d(8)
    s = po.factorized_cg_lyapunov(a, po.random_dense(64, 2, 22), po.Config(eps_tol=1e-9, capture_iterates=True), mode)
    assert s.status == "converged"
    for core in s.captured:
        assert fro(core - core.T) <= 1e-12 * max(fro(core), 1e-300)


@pytest.mark.parametrize("mode", MODES)
def test_equivalence_to_matrix_oriented_cg(mode):
    """EquivalenceToMatrixOrientedCg (test_factorized_solvers.cpp:164-182): 1e-6 over 20 it."""
    a, b = po.random_spd(40, 40), po.random_spd(50, 41)
    c1, c2 = po.random_dense(40, 2, 42), po.random_dense(50, 2, 43)
    fac = po.factorized_cg(a, b, c1, c2, po.Config(eps_tol=1e-14, max_iter=20), mode)
    mo = matrix_oriented_cg(a, b, c1 @ c2.T, 1e-14, 20)
    cnt = min(fac.rel_residual.size, mo.size)
    assert cnt >= 10
    assert np.all(np.abs(fac.rel_residual[:cnt] - mo[:cnt]) <= 1e-6 * np.maximum(mo[:cnt], 1e-30))


@pytest.mark.parametrize("mode", MODES)
def test_acceptance_matrix_oriented_equivalence(mode):
    """acceptance criterion 2 (acceptance.cpp:100-145): CG 1e-6 over 20, BiCGSTAB 1e-4 over 10."""
    a = po.laplacian_2d(30)
    c1 = po.random_rhs(900, 3, 101)
    fac = po.factorized_cg_lyapunov(a, c1, po.Config(eps_tol=1e-13, max_iter=25), mode)
    mo = matrix_oriented_cg(a, a, c1 @ c1.T, 1e-13, 25)
    assert np.max(np.abs(fac.rel_residual[1:21] - mo[1:21]) / mo[1:21]) <= 1e-6
    a3 = po.convection_diffusion_3d(8, (10.0, 10.0, 10.0))
    d1, d2 = po.random_rhs(512, 3, 102), po.random_rhs(512, 3, 103)
    fb = po.factorized_bicgstab(a3, a3, d1, d2, po.Config(eps_tol=1e-13, max_iter=12), mode)
    mb = matrix_oriented_bicgstab(a3, a3, d1 @ d2.T, 1e-13, 12)
    assert np.max(np.abs(fb.rel_residual[1:11] - mb[1:11]) / mb[1:11]) <= 1e-4


@pytest.mark.parametrize("mode", MODES)
def test_reported_residual_tracks_true_residual(mode):
    """ReportedResidualTracksTrueResidual / BicgstabConvergedTrueResidualWithinContract /
    SolutionFactorsAreOrthonormal (test_factorized_solvers.cpp:184-219)."""
    a, b = po.random_spd(30, 44), po.random_spd(30, 45)
    c1, c2 = po.random_dense(30, 2, 46), po.random_dense(30, 2, 47)
    s = po.factorized_cg(a, b, c1, c2, po.Config(eps_tol=1e-6), mode)
    truth = po.true_residual(a, b, c1, c2, s)
    assert s.status == "converged" and abs(s.rel_residual[-1] - truth) <= 1e-6 and truth <= 1e-5
    a, b = po.random_diag_dominant(24, 48), po.random_diag_dominant(21, 49)
    c1, c2 = po.random_dense(24, 3, 50), po.random_dense(21, 3, 51)
    s = po.factorized_bicgstab(a, b, c1, c2, po.Config(eps_tol=1e-8), mode)
    assert s.status == "converged" and po.true_residual(a, b, c1, c2, s) <= 1e-7
    a, b = po.random_spd(24, 52), po.random_spd(18, 53)
    s = po.factorized_cg(a, b, po.random_dense(24, 3, 54), po.random_dense(18, 3, 55), po.Config(eps_tol=1e-10), mode)
    r = max(s.V.shape[1], 1)
    assert fro(s.V.T @ s.V - np.eye(s.V.shape[1])) <= 1e-10 * np.sqrt(r)
    assert fro(s.W.T @ s.W - np.eye(s.W.shape[1])) <= 1e-10 * np.sqrt(r)


@pytest.mark.parametrize("mode", MODES)
def test_input_errors(mode):
    """NonsymmetricOperatorRejected / RankDeficientRhsRejected (test_factorized_solvers.cpp:50-55, 221-226)."""
    with pytest.raises(po.OracleError) as ei:
        po.factorized_cg(po.random_diag_dominant(6, 14), po.random_spd(6, 15), po.random_dense(6, 1, 16),
                         po.random_dense(6, 1, 16), None, mode)
    assert ei.value.code == -2
    c1 = np.zeros((8, 2)); c1[:, 0] = c1[:, 1] = np.arange(8.0)
    with pytest.raises(po.OracleError) as ei:
        po.factorized_cg_lyapunov(po.random_spd(8, 56), c1, None, mode)
    assert ei.value.code == -3


@pytest.mark.parametrize("mode", MODES)
def test_subspace_structure(mode):
    """acceptance criterion 7 (acceptance.cpp:271-331)."""
    n = 25
    for cg, seed in [(True, 301), (False, 302)]:
        a = po.random_spd(n, seed) if cg else po.random_diag_dominant(n, seed)
        b = po.random_spd(n, seed + 1) if cg else po.random_diag_dominant(n, seed + 1)
        c1, c2 = po.random_dense(n, 1, seed + 2), po.random_dense(n, 1, seed + 3)
        cfg = po.Config(eps_tol=1e-30, max_iter=6, capture_iterates=True)
        sol = po.factorized_cg(a, b, c1, c2, cfg, mode) if cg else po.factorized_bicgstab(a, b, c1, c2, cfg, mode)
        for k, core in enumerate(sol.captured):
            depth = k + 1 if cg else 2 * k + 2
            qv = brute_krylov_orthonormal(a.dense(), c1, depth)
            qw = brute_krylov_orthonormal(b.dense().T, c2, depth)
            x = sol.V[:, :core.shape[0]] @ core @ sol.W[:, :core.shape[1]].T
            proj = fro(x - qv @ (qv.T @ x @ qw) @ qw.T)
            assert proj <= 1e-10 * fro(x)


def test_golden_histories_regenerate_bitwise():
    """The committed fixtures are what the oracle produces today (bitwise)."""
    g = json.load(open(os.path.join(GOLDEN, "histories.json")))
    a = po.laplacian_2d(64)
    c1 = po.random_rhs(4096, 1, 1234); c1 /= np.linalg.norm(c1)
    c2 = po.random_rhs(4096, 1, 1235); c2 /= np.linalg.norm(c2)
    s = po.factorized_cg(a, a, c1, c2, po.Config(eps_tol=1e-8, max_iter=500), po.REPRODUCIBLE)
    assert s.rel_residual.tolist() == g["config1_cg_reproducible"]["rel_residual"]
    s = po.factorized_cg(a, a, c1, c2, po.Config(eps_tol=1e-8, max_iter=500), po.REFERENCE_ORDER)
    assert s.rel_residual.tolist() == g["config1_cg_reference_order"]["rel_residual"]


def test_config1_modes_agree_early_and_iteration_count():
    """Faithfulness of the reproducible contract vs the reference order on config 1:
    same iteration count, histories agree to 1e-10 over the first 100 iterations."""
    g = json.load(open(os.path.join(GOLDEN, "histories.json")))
    r = np.array(g["config1_cg_reproducible"]["rel_residual"])
    f = np.array(g["config1_cg_reference_order"]["rel_residual"])
    assert abs(r.size - f.size) <= 1
    assert np.max(np.abs(r[:101] - f[:101]) / f[:101]) <= 1e-10
