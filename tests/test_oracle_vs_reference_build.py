"""Pins the oracle bitwise against the reference's OWN code where it compiles here
without Eigen: sparse_matrix.cpp (spmm, spmm_transpose, transposed, is_symmetric),
parallel.cpp and problems.cpp (laplacian_2d, convection_diffusion_3d, random_rhs),
built by oracle/build_ref.sh into oracle/_ref/. CPU only; skipped if the reference
library is unavailable (e.g. on a GPU box without a prebuilt copy)."""
import ctypes as C
import os

import numpy as np
import pytest

from oracle import pyoracle as po

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                   "libsylkrylov_ref.so")
i64p, f64p = C.POINTER(C.c_int64), C.POINTER(C.c_double)


@pytest.fixture(scope="module")
def ref():
    if not os.path.exists(REF):
        if os.path.isdir("/root/reference/proj/src"):
            os.system(os.path.join(os.path.dirname(REF), "..", "build_ref.sh") + " > /dev/null")
        if not os.path.exists(REF):
            pytest.skip("reference library not built (no /root/reference here)")
    lib = C.CDLL(REF)
    lib.ref_laplacian_2d.restype = C.c_int64
    lib.ref_convection_diffusion_3d.restype = C.c_int64
    lib.ref_transposed.restype = C.c_int64
    return lib


def P(a, t=f64p):
    return a.ctypes.data_as(t)


def ref_lap(lib, g):
    nnz = lib.ref_laplacian_2d(C.c_int64(g), None, None, None)
    rp = np.zeros(g * g + 1, dtype=np.int64)
    ci = np.zeros(nnz, dtype=np.int64)
    v = np.zeros(nnz)
    lib.ref_laplacian_2d(C.c_int64(g), P(rp, i64p), P(ci, i64p), P(v))
    return po.Csr(g * g, g * g, rp, ci, v)


def ref_cd3(lib, g, w):
    args = (C.c_int64(g), C.c_double(w[0]), C.c_double(w[1]), C.c_double(w[2]))
    nnz = lib.ref_convection_diffusion_3d(*args, None, None, None)
    rp = np.zeros(g ** 3 + 1, dtype=np.int64)
    ci = np.zeros(nnz, dtype=np.int64)
    v = np.zeros(nnz)
    lib.ref_convection_diffusion_3d(*args, P(rp, i64p), P(ci, i64p), P(v))
    return po.Csr(g ** 3, g ** 3, rp, ci, v)


@pytest.mark.parametrize("g", [2, 3, 8, 64])
def test_laplacian_bitwise(ref, g):
    r, o = ref_lap(ref, g), po.laplacian_2d(g)
    assert np.array_equal(r.row_ptr, o.row_ptr) and np.array_equal(r.col_idx, o.col_idx)
    assert np.array_equal(r.values.view(np.uint64), o.values.view(np.uint64))


@pytest.mark.parametrize("g,w", [(3, (10.0, 10.0, 10.0)), (6, (5.0, 2.5, 1.25)), (4, (0.0, 0.0, 0.0))])
def test_convdiff3d_bitwise(ref, g, w):
    r, o = ref_cd3(ref, g, w), po.convection_diffusion_3d(g, w)
    assert np.array_equal(r.row_ptr, o.row_ptr) and np.array_equal(r.col_idx, o.col_idx)
    assert np.array_equal(r.values.view(np.uint64), o.values.view(np.uint64))


@pytest.mark.parametrize("rows,s,seed", [(7, 1, 1234), (4096, 1, 1235), (1000, 3, 42), (333, 8, 7)])
def test_random_rhs_bitwise(ref, rows, s, seed):
    out = np.zeros((rows, s), order="F")
    ref.ref_random_rhs(C.c_int64(rows), C.c_int64(s), C.c_uint64(seed), P(out))
    assert np.array_equal(out.view(np.uint64), po.random_rhs(rows, s, seed).view(np.uint64))


def _args(a):
    return (C.c_int64(a.n_rows), C.c_int64(a.n_cols), C.c_int64(a.nnz), P(a.row_ptr, i64p), P(a.col_idx, i64p),
            P(a.values))


@pytest.mark.parametrize("threads", [0, 4])
def test_spmm_bitwise(ref, threads):
    ref.ref_set_parallel(C.c_int(1 if threads else 0), C.c_uint(threads))
    for a in [po.laplacian_2d(30), po.random_sparse(200, 150, 0.05, 3), po.convection_diffusion_3d(7, (5.0, 2.5, 1.25))]:
        for s in (1, 2, 5):
            x = np.asfortranarray(po.random_dense(a.n_cols, s, 11 + s))
            y = np.zeros((a.n_rows, s), order="F")
            ref.ref_spmm(*_args(a), P(x), C.c_int64(s), P(y))
            assert np.array_equal(y.view(np.uint64), po.spmm(a, x).view(np.uint64))
            xt = np.asfortranarray(po.random_dense(a.n_rows, s, 21 + s))
            yt = np.zeros((a.n_cols, s), order="F")
            ref.ref_spmm_transpose(*_args(a), P(xt), C.c_int64(s), P(yt))
            assert np.array_equal(yt.view(np.uint64), po.spmm_transpose(a, xt).view(np.uint64))
            # the device's gather over the transposed CSR reproduces the reference scatter
            assert np.array_equal(yt, po.spmm(po.transpose(a), xt))
    ref.ref_set_parallel(C.c_int(0), C.c_uint(1))


def test_transposed_and_symmetry_bitwise(ref):
    for a in [po.random_sparse(50, 40, 0.2, 9), po.laplacian_2d(9), po.convection_diffusion_3d(4, (10.0, 10.0, 10.0))]:
        nnz = a.nnz
        trp = np.zeros(a.n_cols + 1, dtype=np.int64)
        tci = np.zeros(nnz, dtype=np.int64)
        tv = np.zeros(nnz)
        ref.ref_transposed(*_args(a), P(trp, i64p), P(tci, i64p), P(tv))
        o = po.transpose(a)
        assert np.array_equal(trp, o.row_ptr) and np.array_equal(tci, o.col_idx) and np.array_equal(tv, o.values)
        if a.n_rows == a.n_cols:
            assert bool(ref.ref_is_symmetric(*_args(a), C.c_double(1e-12))) == po.is_symmetric(a)
