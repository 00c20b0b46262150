"""CPU-side checks of the product library: it loads, exports every C-ABI symbol
include/sylkrylov_b200.h declares, its host-side generators equal the oracle's
bitwise, and the solver fails loudly (no CPU fallback) without a CUDA device."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def skl():
    from paper_2605_28274_b200 import build
    build.build()
    import paper_2605_28274_b200 as sk
    sk.lib()
    return sk


def header_symbols():
    src = open(os.path.join(ROOT, "include", "sylkrylov_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sk_[A-Za-z0-9_]+)\s*\(", src)))


def test_exports_every_header_symbol(skl):
    syms = header_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(skl.lib(), s)]
    assert not missing, missing


def test_built_for_sm100a():
    lib = os.path.join(ROOT, "paper_2605_28274_b200", "libsk_b200.so")
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {lib} 2>/dev/null").read()
    assert "sm_100a" in out


@pytest.mark.parametrize("grid", [2, 5, 17])
def test_generators_match_oracle(skl, grid):
    from oracle import pyoracle as po
    from paper_2605_28274_b200 import problems as pr
    a, b = pr.laplacian_2d(grid), po.laplacian_2d(grid)
    assert np.array_equal(a.row_ptr, b.row_ptr) and np.array_equal(a.col_idx, b.col_idx)
    assert np.array_equal(a.values, b.values)
    a, b = pr.convection_diffusion_2d(grid, (10.0, -10.0)), po.convection_diffusion_2d(grid, (10.0, -10.0))
    assert np.array_equal(a.col_idx, b.col_idx) and np.array_equal(a.values, b.values)
    if grid <= 5:
        a, b = pr.convection_diffusion_3d(grid, (5.0, 2.5, 1.25)), po.convection_diffusion_3d(grid, (5.0, 2.5, 1.25))
        assert np.array_equal(a.row_ptr, b.row_ptr) and np.array_equal(a.values, b.values)
    assert np.array_equal(pr.random_rhs(101, 3, 77), po.random_rhs(101, 3, 77))


def test_large_laplacian_parallel_fill(skl):
    from oracle import pyoracle as po
    from paper_2605_28274_b200 import problems as pr
    a, b = pr.laplacian_2d(700), po.laplacian_2d(700)
    assert np.array_equal(a.row_ptr, b.row_ptr) and np.array_equal(a.col_idx, b.col_idx)


def test_no_cpu_fallback(skl):
    if skl.device_count() > 0:
        pytest.skip("a CUDA device is present")
    a = skl.SparseMatrix.identity(4)
    with pytest.raises(skl.CudaError):
        skl.factorized_cg(a, a, np.ones((4, 1)), np.ones((4, 1)))


def test_input_validation_before_device(skl):
    """Reference error taxonomy (errors.hpp) is raised by host validation."""
    bad = skl.SparseMatrix(2, 2, np.array([0, 1, 2]), np.array([0, 2]), np.array([1.0, 1.0]))
    with pytest.raises(skl.InvalidMatrixError):
        skl.factorized_cg(bad, bad, np.ones((2, 1)), np.ones((2, 1)))
    a = skl.SparseMatrix.identity(3)
    with pytest.raises(skl.DimensionError):
        skl.factorized_cg(a, a, np.ones((4, 1)), np.ones((3, 1)))


def _csr_from_dense(skl, d):
    import scipy.sparse as spx
    return skl.SparseMatrix.from_scipy(spx.csr_matrix(d))


@pytest.mark.parametrize("case", ["decreasing_rowptr", "col_out_of_range", "unsorted_cols"])
def test_validation_reports_lowest_bad_row(skl, case):
    """sparse_matrix.cpp:12-32: the parallel host scan reports the error a
    sequential scan would (lowest offending row), on a matrix large enough to be
    split across host threads."""
    n = 300_000
    rp = np.arange(n + 1, dtype=np.int64)
    ci = np.arange(n, dtype=np.int64)
    val = np.ones(n)
    if case == "decreasing_rowptr":
        rp = rp.copy(); rp[200_000] = rp[200_001] + 1
        msg = "not nondecreasing"
    elif case == "col_out_of_range":
        ci = ci.copy(); ci[250_000] = n; ci[10_000] = -1
        msg = "out of range"
    else:
        rp = np.concatenate([np.arange(0, 2 * 100, 2), 200 + np.arange(n - 100 + 1)]).astype(np.int64)
        ci = np.concatenate([np.stack([np.arange(100) + 1, np.arange(100)], 1).ravel(),
                             np.arange(100, n)]).astype(np.int64)
        val = np.ones(ci.size)
        msg = "strictly increasing"
    a = skl.SparseMatrix(n, n, rp, ci, val)
    with pytest.raises(skl.InvalidMatrixError, match=msg):
        skl.factorized_cg(a, a, np.ones((n, 1)), np.ones((n, 1)))


def test_symmetry_checks(skl):
    """Bitwise-symmetric operators skip the transpose; near-symmetric ones (within
    the reference's 1e-12 relative tolerance) still pass through the full check;
    nonsymmetric ones are rejected (factorized_solvers.cpp:207-216)."""
    rng = np.random.default_rng(3)
    d = rng.standard_normal((40, 40)) * (rng.random((40, 40)) < 0.2) + 10 * np.eye(40)
    sym = d + d.T
    near = sym.copy(); near[3, 5] *= 1 + 1e-15
    expect_cuda = skl.device_count() == 0
    for mat in (sym, near):
        a = _csr_from_dense(skl, mat)
        if expect_cuda:
            with pytest.raises(skl.CudaError):
                skl.factorized_cg(a, a, np.ones((40, 1)), np.ones((40, 1)))
            with pytest.raises(skl.CudaError):
                skl.factorized_cg_lyapunov(a, np.ones((40, 1)))
    a = _csr_from_dense(skl, d)
    with pytest.raises(skl.InvalidMatrixError, match="not symmetric"):
        skl.factorized_cg(a, a, np.ones((40, 1)), np.ones((40, 1)))
    with pytest.raises(skl.InvalidMatrixError, match="not symmetric"):
        skl.factorized_cg_lyapunov(a, np.ones((40, 1)))
    s = _csr_from_dense(skl, sym)
    with pytest.raises(skl.InvalidMatrixError, match="B is not symmetric"):
        skl.factorized_cg(s, a, np.ones((40, 1)), np.ones((40, 1)))


def test_true_residual_shape_checks_before_device(skl):
    """true_residual_factors shape checks (factorized_solvers.cpp:394-400) run on the host."""
    a = skl.SparseMatrix.identity(4)
    with pytest.raises(skl.DimensionError):
        skl.true_residual_factors(a, a, np.ones((4, 1)), np.ones((4, 1)), np.ones((4, 2)), np.ones((3, 2)),
                                  np.ones((4, 2)))
    with pytest.raises(skl.DimensionError):
        skl.true_residual_factors(a, a, np.ones((4, 1)), np.ones((4, 2)), np.ones((4, 2)), np.ones((2, 2)),
                                  np.ones((4, 2)))


def test_speculative_stencil_invalid_row_raises_without_device(skl):
    """The one-shot entry points check only a stencil's leading rows before the
    solve; an invalid later row must still raise the reference's error (here the
    speculative attempt fails without a device and the checked path reports)."""
    from paper_2605_28274_b200.problems import laplacian_2d
    a = laplacian_2d(40)
    n = a.n_rows
    ci = a.col_idx.copy()
    k0 = a.row_ptr[n - 1]
    ci[k0], ci[k0 + 1] = ci[k0 + 1], ci[k0]
    bad = skl.SparseMatrix(n, n, a.row_ptr, ci, a.values)
    with pytest.raises(skl.InvalidMatrixError, match="strictly increasing"):
        skl.factorized_cg(bad, bad, np.ones((n, 1)), np.ones((n, 1)))


@pytest.mark.parametrize("method", ["cg", "bicgstab", "lyapunov"])
def test_speculative_stencil_late_row_out_of_range(skl, method):
    """a nonsymmetric stencil whose LAST row holds an out-of-range
    column must raise InvalidMatrixError (sparse_matrix.cpp:12-32), not crash: the
    speculative stencil path may not let a host pass (symmetry, transpose) index the
    unvalidated rows. Runs without a device (host checks come first)."""
    from paper_2605_28274_b200 import problems as pr
    g = 64
    n = g * g
    for wind in ((10.0, 10.0), (0.0, 0.0)):
        c = pr.convection_diffusion_2d(g, wind)
        ci = np.array(c.col_idx, copy=True)
        ci[-1] = 5000  # n = 4096
        bad = skl.SparseMatrix(n, n, c.row_ptr, ci, c.values)
        good = skl.SparseMatrix(n, n, c.row_ptr, c.col_idx, c.values)
        c1, c2 = np.ones((n, 1)), np.ones((n, 1))
        with pytest.raises(skl.InvalidMatrixError):
            if method == "cg":
                skl.factorized_cg(bad, bad, c1, c2)
            elif method == "lyapunov":
                skl.factorized_cg_lyapunov(bad, c1)
            else:
                skl.factorized_bicgstab(good, bad, c1, c2)


def test_reference_order_reduction_mode_is_rejected(sk_host):
    """sk_gpu_options.reduction_mode: the device executes the reproducible
    contract only; asking for the reference's sequential sums fails loudly, never a fallback."""
    sk = sk_host
    from paper_2605_28274_b200 import problems as pr
    a = pr.laplacian_2d(8)
    c = pr.random_rhs(64, 1, 3)
    with pytest.raises(sk.UnsupportedError, match="reference_order"):
        sk.factorized_cg(a, a, c, c, sk.SolverConfig(), sk.GpuOptions(reduction_mode=1))
