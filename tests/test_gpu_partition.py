"""Row-partitioned CG / Lyapunov CG on one GPU.

The partitioned data path (local row blocks with ghost rows, per-chunk tree
nodes, all-gather, replicated finalisation, halo exchange, paused rare paths)
runs with `world` ranks as host threads of one process, each on its own stream
(sk_comm_create_local_group): collectives are host-mediated device copies, so
no kernel waits on another rank's kernel. Every rank's history, core and
classification counters must be bitwise those of the single-GPU solve, and the
ranks' rows of V and W must concatenate to the single-GPU factors bitwise.
"""
import numpy as np
import pytest
import scipy.sparse as sp

from helpers import bits_equal, max_rel, to_sk

pytestmark = pytest.mark.gpu


def _check(sols, ref):
    for s_ in sols:
        assert s_.status == ref.status
        h, hr = s_.history.rel_residuals(), ref.history.rel_residuals()
        assert h.size == hr.size
        assert bits_equal(h, hr), f"max rel diff {max_rel(h, hr)}"
        assert bits_equal(s_.core, ref.core)
        assert s_.stats["paths"] == ref.stats["paths"]
    sv = sorted(sols, key=lambda t: t.row0_v)
    assert bits_equal(np.vstack([t.V for t in sv]), ref.V)
    sw = sorted(sols, key=lambda t: t.row0_w)
    assert bits_equal(np.vstack([t.W for t in sw]), ref.W)


def _banded_spd(sk, n, offs, seed):
    rng = np.random.default_rng(seed)
    m = sp.csr_matrix((n, n))
    for o in offs:
        v = rng.uniform(-1.0, 1.0, n - o)
        m = m + sp.diags(v, o, shape=(n, n)) + sp.diags(v, -o, shape=(n, n))
    d = np.asarray(abs(m).sum(axis=1)).ravel() + 1.0
    m = (m + sp.diags(d, 0)).tocsr()
    m.sort_indices()
    return sk.SparseMatrix.from_scipy(m)


@pytest.mark.parametrize("world", [2, 4])
def test_partitioned_cg_stencil_s2(sk, po, world):
    a = to_sk(sk, po.laplacian_2d(256))
    n = a.n_rows
    c1, c2 = po.random_rhs(n, 2, 1234), po.random_rhs(n, 2, 1235)
    cfg = sk.SolverConfig(eps_tol=1e-8, max_iter=40)
    ref = sk.factorized_cg(a, a, c1, c2, cfg)
    _check(sk.solve_local_group("cg", a, a, c1, c2, world, cfg), ref)


def test_partitioned_cg_matches_oracle(sk, po):
    a = po.laplacian_2d(256)
    c1, c2 = po.random_rhs(65536, 1, 7), po.random_rhs(65536, 1, 8)
    ref = po.factorized_cg(a, a, c1, c2, po.Config(eps_tol=1e-8, max_iter=25), po.REPRODUCIBLE)
    sols = sk.solve_local_group("cg", to_sk(sk, a), to_sk(sk, a), c1, c2, 2,
                                sk.SolverConfig(eps_tol=1e-8, max_iter=25))
    for s_ in sols:
        assert bits_equal(s_.history.rel_residuals(), ref.rel_residual)
        assert bits_equal(s_.core, ref.core)
    assert bits_equal(np.vstack([t.V for t in sorted(sols, key=lambda t: t.row0_v)]), ref.V)


def test_partitioned_lyapunov_stencil(sk, po):
    a = to_sk(sk, po.laplacian_2d(256))
    c1 = po.random_rhs(a.n_rows, 1, 99)
    cfg = sk.SolverConfig(eps_tol=1e-8, max_iter=30)
    ref = sk.factorized_cg_lyapunov(a, c1, cfg)
    _check(sk.solve_local_group("cg_lyapunov", a, None, c1, None, 3, cfg), ref)


def test_partitioned_two_operators(sk, po):
    """Distinct A and B (both symmetric stencils): the two sides carry different operators."""
    a = po.laplacian_2d(256)
    rp, ci = np.asarray(a.row_ptr), np.asarray(a.col_idx)
    vb = 0.5 * np.asarray(a.values, dtype=np.float64)
    rows = np.repeat(np.arange(a.n_rows), np.diff(rp))
    vb[ci == rows] += 1.0  # B = A/2 + I: still one constant value per stencil offset
    b = sk.SparseMatrix(a.n_rows, a.n_cols, rp, ci, vb)
    c1, c2 = po.random_rhs(65536, 2, 3), po.random_rhs(65536, 2, 4)
    cfg = sk.SolverConfig(eps_tol=1e-8, max_iter=30)
    ref = sk.factorized_cg(to_sk(sk, a), b, c1, c2, cfg)
    _check(sk.solve_local_group("cg", to_sk(sk, a), b, c1, c2, 2, cfg), ref)


@pytest.mark.parametrize("world,s", [(2, 1), (3, 2)])
def test_partitioned_csr_banded(sk, po, world, s):
    """General CSR (no stencil): ghost rows = bandwidth, columns shifted per rank."""
    a = _banded_spd(sk, 65536, (1, 7, 300), 5)
    c1, c2 = po.random_rhs(65536, s, 11), po.random_rhs(65536, s, 12)
    cfg = sk.SolverConfig(eps_tol=1e-10, max_iter=30)
    ref = sk.factorized_cg(a, a, c1, c2, cfg)
    _check(sk.solve_local_group("cg", a, a, c1, c2, world, cfg), ref)


def test_partitioned_3d_stencil_lyapunov(sk, po):
    a = to_sk(sk, po.convection_diffusion_3d(32, (0.0, 0.0, 0.0)))  # 7-point Laplacian
    c1 = po.random_rhs(a.n_rows, 2, 5)
    cfg = sk.SolverConfig(eps_tol=1e-8, max_iter=25)
    ref = sk.factorized_cg_lyapunov(a, c1, cfg)
    _check(sk.solve_local_group("cg_lyapunov", a, None, c1, None, 2, cfg), ref)


def test_partitioned_identity_cleanup_path(sk, po):
    """Identity pair: the candidate is rounding noise, so classification asks for
    the Lanczos clean-up (Gram against every block, update, direct Gram), run
    while the ranks are paused, with partitioned reductions."""
    n = 65536
    i_n = sk.SparseMatrix.identity(n)
    c1, c2 = po.random_rhs(n, 2, 1), po.random_rhs(n, 2, 2)
    ref = sk.factorized_cg(i_n, i_n, c1, c2)
    assert ref.stats["paths"]["cleanup"] > 0
    sols = sk.solve_local_group("cg", i_n, i_n, c1, c2, 2)
    _check(sols, ref)
    assert sols[0].status == "converged" and sols[0].history.iterations() == 1


def test_partitioned_zero_operator_householder_path(sk, po):
    """A = 0, B = I: the V-side candidate is exactly zero, the direct Gram has no
    Cholesky factor and the Householder rare path runs on the gathered candidate."""
    n = 65536
    zero = sk.SparseMatrix(n, n, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int64), np.zeros(n))
    i_n = sk.SparseMatrix.identity(n)
    c1, c2 = po.random_rhs(n, 2, 5), po.random_rhs(n, 2, 6)
    ref = sk.factorized_cg(zero, i_n, c1, c2)
    assert ref.stats["paths"]["householder"] > 0
    _check(sk.solve_local_group("cg", zero, i_n, c1, c2, 2), ref)


def test_partitioned_rejects_bicgstab(sk, po):
    a = to_sk(sk, po.laplacian_2d(256))
    c = po.random_rhs(65536, 1, 1)
    comms = sk.Communicator.local_group(2)
    with pytest.raises(sk.UnsupportedError):
        sk.PartitionedProblem("bicgstab", a, a, c, c, comms[0])


@pytest.mark.parametrize("transport", ["local", "nccl"])
def test_partitioned_single_rank_transports(sk, po, transport):
    """One-rank communicator: the partitioned data path (chunk nodes, all-gather,
    replicated finalisation) through each transport, incl. NCCL loaded at run time."""
    a = to_sk(sk, po.laplacian_2d(128))
    c1, c2 = po.random_rhs(a.n_rows, 2, 31), po.random_rhs(a.n_rows, 2, 32)
    cfg = sk.SolverConfig(eps_tol=1e-8, max_iter=20)
    ref = sk.factorized_cg(a, a, c1, c2, cfg)
    if transport == "nccl":
        comm = sk.Communicator.nccl(sk.Communicator.nccl_unique_id(), 1, 0, 0)
    else:
        comm = sk.Communicator.local_group(1)[0]
    prob = sk.PartitionedProblem("cg", a, a, c1, c2, comm)
    sol = prob.solve(cfg)
    _check([sol], ref)
    sol.free()
    prob.free()
    comm.free()
