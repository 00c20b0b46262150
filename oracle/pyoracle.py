"""ctypes front of the CPU oracle (oracle/libsk_oracle.so).

TEST INFRASTRUCTURE ONLY. Imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference leg as the checker; the product
path (paper_2605_28274_b200) never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsk_oracle.so")

REPRODUCIBLE = 0
REFERENCE_ORDER = 1
CG, CG_LYAPUNOV, BICGSTAB = 0, 1, 2
STATUS = {0: "converged", 1: "max_iter", 2: "breakdown"}

i64p = C.POINTER(C.c_int64)
f64p = C.POINTER(C.c_double)


class _Csr(C.Structure):
    _fields_ = [("n_rows", C.c_int64), ("n_cols", C.c_int64), ("nnz", C.c_int64),
                ("row_ptr", i64p), ("col_idx", i64p), ("values", f64p)]


class _Cfg(C.Structure):
    _fields_ = [("eps_tol", C.c_double), ("max_iter", C.c_int64), ("breakdown_tol", C.c_double),
                ("capture_iterates", C.c_int32), ("lanczos_full_reorth", C.c_int32)]


def build(force: bool = False) -> str:
    src = max(os.path.getmtime(os.path.join(HERE, f)) for f in ("sk_oracle.c", "sk_oracle.h", "Makefile"))
    if force or any(not os.path.exists(p) or os.path.getmtime(p) < src
                    for p in (LIB_PATH, os.path.join(HERE, "libsk_oracle_mt.so"))):
        subprocess.check_call(["make", "-s", "-C", HERE])
    return LIB_PATH


_lib = None


def use_threads(threads: int) -> None:
    """Switch to the OpenMP build (bitwise equal to the serial one) with `threads`
    host threads for the oracle's loops and its SpMM (parallel.cpp's knob).
    Golden generation only: the CPU baseline times the serial reference flags."""
    global _lib, LIB_PATH
    build()
    os.environ["OMP_NUM_THREADS"] = str(threads)
    LIB_PATH = os.path.join(HERE, "libsk_oracle_mt.so")
    _lib = None
    lib().sko_set_parallel(1, int(threads))


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        L = _lib
        L.sko_last_error.restype = C.c_char_p
        L.sko_solution_total_time.restype = C.c_double
        L.sko_true_residual_factors.restype = C.c_double
        for name in ["sko_frobenius_inner", "sko_r1_dot", "sko_r2_inner"]:
            getattr(L, name).restype = C.c_double
        for name in ["sko_basis_cols", "sko_basis_steps", "sko_solution_n_records",
                     "sko_solution_n_captured"]:
            getattr(L, name).restype = C.c_int64
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


ERRORS = {-1: "DimensionError", -2: "InvalidMatrixError", -3: "RankDeficientStartError",
          -4: "BreakdownError", -5: "BreakdownError(invariant_subspace)", -6: "AllocError"}


def _check(rc: int):
    if rc < 0:
        raise OracleError(rc, f"{ERRORS.get(rc, rc)}: {lib().sko_last_error().decode()}")
    return rc


def _p(a, t=f64p):
    return a.ctypes.data_as(t)


@dataclass
class Csr:
    """CSR with the reference's int64 indices (sparse_matrix.hpp:11-48)."""
    n_rows: int
    n_cols: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.values.size)

    def c(self) -> _Csr:
        self.row_ptr = np.ascontiguousarray(self.row_ptr, dtype=np.int64)
        self.col_idx = np.ascontiguousarray(self.col_idx, dtype=np.int64)
        self.values = np.ascontiguousarray(self.values, dtype=np.float64)
        return _Csr(self.n_rows, self.n_cols, self.nnz, _p(self.row_ptr, i64p),
                    _p(self.col_idx, i64p), _p(self.values))

    def dense(self) -> np.ndarray:
        d = np.zeros((self.n_rows, self.n_cols))
        for i in range(self.n_rows):
            for k in range(self.row_ptr[i], self.row_ptr[i + 1]):
                d[i, self.col_idx[k]] = self.values[k]
        return d

    @staticmethod
    def from_c(c: _Csr) -> "Csr":
        n, nnz = c.n_rows, c.nnz
        rp = np.ctypeslib.as_array(c.row_ptr, shape=(n + 1,)).copy()
        ci = np.ctypeslib.as_array(c.col_idx, shape=(max(nnz, 1),))[:nnz].copy()
        va = np.ctypeslib.as_array(c.values, shape=(max(nnz, 1),))[:nnz].copy()
        out = Csr(int(c.n_rows), int(c.n_cols), rp, ci, va)
        lib().sko_csr_free(C.byref(c))
        return out

    @staticmethod
    def identity(n: int) -> "Csr":
        return Csr(n, n, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int64), np.ones(n))


def from_triplets(n_rows, n_cols, rows, cols, vals) -> Csr:
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    cols = np.ascontiguousarray(cols, dtype=np.int64)
    vals = np.ascontiguousarray(vals, dtype=np.float64)
    out = _Csr()
    _check(lib().sko_csr_from_triplets(C.c_int64(n_rows), C.c_int64(n_cols), C.c_int64(rows.size),
                                       _p(rows, i64p), _p(cols, i64p), _p(vals), C.byref(out)))
    return Csr.from_c(out)


def transpose(a: Csr) -> Csr:
    out = _Csr()
    ca = a.c()
    _check(lib().sko_csr_transpose(C.byref(ca), C.byref(out)))
    return Csr.from_c(out)


def is_symmetric(a: Csr, tol: float = 1e-12) -> bool:
    ca = a.c()
    return bool(lib().sko_csr_is_symmetric(C.byref(ca), C.c_double(tol)))


def _gen(fn, *args) -> Csr:
    out = _Csr()
    _check(fn(*args, C.byref(out)))
    return Csr.from_c(out)


def laplacian_2d(grid: int) -> Csr:
    return _gen(lib().sko_laplacian_2d, C.c_int64(grid))


def convection_diffusion_2d(grid: int, w) -> Csr:
    return _gen(lib().sko_convection_diffusion_2d, C.c_int64(grid), C.c_double(w[0]), C.c_double(w[1]))


def convection_diffusion_3d(grid: int, w) -> Csr:
    return _gen(lib().sko_convection_diffusion_3d, C.c_int64(grid), C.c_double(w[0]),
                C.c_double(w[1]), C.c_double(w[2]))


def random_rhs(rows: int, s: int, seed: int) -> np.ndarray:
    out = np.zeros((rows, s), order="F")
    lib().sko_random_rhs(C.c_int64(rows), C.c_int64(s), C.c_uint64(seed), _p(out))
    return out


def random_dense(rows: int, cols: int, seed: int) -> np.ndarray:
    out = np.zeros((rows, cols), order="F")
    lib().sko_random_dense(C.c_int64(rows), C.c_int64(cols), C.c_uint64(seed), _p(out))
    return out


def random_sparse(n, m, density, seed, diag_shift=0.0) -> Csr:
    return _gen(lib().sko_random_sparse, C.c_int64(n), C.c_int64(m), C.c_double(density),
                C.c_uint64(seed), C.c_double(diag_shift))


def random_spd(n, seed) -> Csr:
    return _gen(lib().sko_random_spd, C.c_int64(n), C.c_uint64(seed))


def random_diag_dominant(n, seed) -> Csr:
    return _gen(lib().sko_random_diag_dominant, C.c_int64(n), C.c_uint64(seed))


def set_parallel(enabled: bool, threads: int = 0):
    lib().sko_set_parallel(int(enabled), int(threads or os.cpu_count() or 1))


def spmm(a: Csr, x: np.ndarray) -> np.ndarray:
    x = np.asfortranarray(x, dtype=np.float64)
    y = np.zeros((a.n_rows, x.shape[1]), order="F")
    ca = a.c()
    lib().sko_spmm(C.byref(ca), _p(x), C.c_int64(x.shape[1]), _p(y))
    return y


def spmm_transpose(a: Csr, x: np.ndarray) -> np.ndarray:
    x = np.asfortranarray(x, dtype=np.float64)
    y = np.zeros((a.n_cols, x.shape[1]), order="F")
    ca = a.c()
    lib().sko_spmm_transpose(C.byref(ca), _p(x), C.c_int64(x.shape[1]), _p(y))
    return y


def thin_qr(x: np.ndarray):
    x = np.asfortranarray(x, dtype=np.float64)
    n, s = x.shape
    q = np.zeros((n, s), order="F")
    r = np.zeros((s, s), order="F")
    _check(lib().sko_thin_qr(_p(x), C.c_int64(n), C.c_int64(s), _p(q), _p(r)))
    return q, r


def singular_extremes(m: np.ndarray):
    m = np.asfortranarray(m, dtype=np.float64)
    a, b = C.c_double(), C.c_double()
    lib().sko_singular_extremes(_p(m), C.c_int64(m.shape[0]), C.byref(a), C.byref(b))
    return a.value, b.value


def contract_constants():
    out = np.zeros(4, dtype=np.int64)
    lib().sko_contract_constants(_p(out, i64p))
    return dict(seg_rows=int(out[0]), lanes=int(out[1]), tile=int(out[2]))


class Basis:
    """BlockKrylovBasis (block_krylov.hpp:31-100)."""

    def __init__(self, op: Csr, start: np.ndarray, arnoldi: bool, transpose: bool,
                 breakdown_tol: float = 1e-12, lanczos_full_reorth: bool = False,
                 mode: int = REPRODUCIBLE):
        self.op = op
        self._cop = op.c()
        start = np.asfortranarray(start, dtype=np.float64)
        self.n, self.s = start.shape
        self.r = np.zeros((self.s, self.s), order="F")
        h = C.c_void_p()
        _check(lib().sko_basis_init(C.byref(self._cop), _p(start), C.c_int64(self.s), int(arnoldi),
                                    int(transpose), C.c_double(breakdown_tol),
                                    int(lanczos_full_reorth), int(mode), C.byref(h), _p(self.r)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            lib().sko_basis_free(self.h)
            self.h = None

    def try_extend(self) -> str:
        rc = _check(lib().sko_basis_try_extend(self.h))
        return "grown" if rc == 0 else "exhausted"

    def extend(self):
        if self.try_extend() == "exhausted":
            raise OracleError(-5, "basis extend: Krylov subspace is invariant (exhausted)")

    @property
    def cols(self) -> int:
        return int(lib().sko_basis_cols(self.h))

    @property
    def steps(self) -> int:
        return int(lib().sko_basis_steps(self.h))

    @property
    def exhausted(self) -> bool:
        return bool(lib().sko_basis_exhausted(self.h))

    def matrix(self) -> np.ndarray:
        out = np.zeros((self.n, self.cols), order="F")
        lib().sko_basis_matrix(self.h, _p(out))
        return out

    def hessenberg(self, rows=None, cols=None) -> np.ndarray:
        rows = self.cols if rows is None else rows
        cols = self.s * self.steps if cols is None else cols
        out = np.zeros((rows, cols), order="F")
        _check(lib().sko_basis_hessenberg(self.h, C.c_int64(rows), C.c_int64(cols), _p(out)))
        return out

    def accumulate_h_times(self, p: np.ndarray, c: np.ndarray):
        p = np.asfortranarray(p, dtype=np.float64)
        assert c.flags.f_contiguous
        _check(lib().sko_basis_accumulate_h_times(self.h, _p(p), C.c_int64(p.shape[0]),
                                                  C.c_int64(p.shape[1]), _p(c),
                                                  C.c_int64(c.shape[0]), C.c_int64(c.shape[1])))

    def accumulate_times_ht(self, p: np.ndarray, c: np.ndarray):
        p = np.asfortranarray(p, dtype=np.float64)
        assert c.flags.f_contiguous
        _check(lib().sko_basis_accumulate_times_ht(self.h, _p(p), C.c_int64(p.shape[0]),
                                                   C.c_int64(p.shape[1]), _p(c),
                                                   C.c_int64(c.shape[0]), C.c_int64(c.shape[1])))

    def path_counts(self):
        out = np.zeros(4, dtype=np.int64)
        lib().sko_basis_path_counts(self.h, _p(out, i64p))
        return dict(zip(["direct", "householder", "cleanup", "unused"], out.tolist()))


@dataclass
class Solution:
    status: str
    iterations: np.ndarray
    rel_residual: np.ndarray
    t_basic: np.ndarray
    t_krylov: np.ndarray
    V: np.ndarray
    core: np.ndarray
    W: np.ndarray
    total_time_s: float
    captured: list = field(default_factory=list)
    paths: dict = field(default_factory=dict)

    @property
    def n_iterations(self) -> int:
        return int(self.iterations[-1]) if self.iterations.size else 0


@dataclass
class Config:
    """SolverConfig (solver_types.hpp:36-45)."""
    eps_tol: float = 1e-8
    max_iter: int = 0
    breakdown_tol: float = 1e-12
    capture_iterates: bool = False
    lanczos_full_reorth: bool = False

    def c(self) -> _Cfg:
        return _Cfg(self.eps_tol, self.max_iter, self.breakdown_tol, int(self.capture_iterates),
                    int(self.lanczos_full_reorth))


def solve(method: int, a: Csr, b: Csr | None, c1: np.ndarray, c2: np.ndarray | None,
          cfg: Config | None = None, mode: int = REPRODUCIBLE, lean: bool = False) -> Solution:
    """lean: Lanczos bases keep only their last blocks (history and core only; V, W
    are returned empty) -- golden generation at configs larger than host RAM."""
    cfg = cfg or Config()
    c1 = np.asfortranarray(c1, dtype=np.float64)
    s = c1.shape[1]
    ca = a.c()
    cb = b.c() if b is not None else None
    c2a = np.asfortranarray(c2, dtype=np.float64) if c2 is not None else None
    if method != CG_LYAPUNOV and (c2a is None or c2a.shape[1] != s or c1.shape[0] != a.n_rows
                                  or c2a.shape[0] != b.n_rows):
        raise OracleError(-1, "DimensionError: solver: C1/C2 shapes do not conform")
    if method == CG_LYAPUNOV and c1.shape[0] != a.n_rows:
        raise OracleError(-1, "DimensionError: factorized_cg_lyapunov: C1 rows must match A")
    h = C.c_void_p()
    cc = cfg.c()
    L = lib()
    if lean:
        L.sko_set_lean(1)
    try:
        _check(L.sko_solve(int(method), C.byref(ca), C.byref(cb) if cb is not None else None,
                           _p(c1), _p(c2a) if c2a is not None else None, C.c_int64(s),
                           C.byref(cc), int(mode), C.byref(h)))
    finally:
        if lean:
            L.sko_set_lean(0)
    try:
        nrec = int(L.sko_solution_n_records(h))
        it = np.zeros(nrec, dtype=np.int64)
        rel = np.zeros(nrec)
        tb = np.zeros(nrec)
        tk = np.zeros(nrec)
        L.sko_solution_history(h, _p(it, i64p), _p(rel), _p(tb), _p(tk))
        n, rv, m, rw = (C.c_int64() for _ in range(4))
        L.sko_solution_dims(h, C.byref(n), C.byref(rv), C.byref(m), C.byref(rw))
        V = np.zeros((n.value, 0 if lean else rv.value), order="F")
        core = np.zeros((rv.value, rw.value), order="F")
        W = np.zeros((m.value, 0 if lean else rw.value), order="F")
        L.sko_solution_copy(h, _p(V), _p(core), _p(W))
        caps = []
        for i in range(int(L.sko_solution_n_captured(h))):
            r_, c_ = C.c_int64(), C.c_int64()
            L.sko_solution_captured(h, C.c_int64(i), C.byref(r_), C.byref(c_), None)
            buf = np.zeros((r_.value, c_.value), order="F")
            L.sko_solution_captured(h, C.c_int64(i), C.byref(r_), C.byref(c_), _p(buf))
            caps.append(buf)
        paths = np.zeros(4, dtype=np.int64)
        L.sko_solution_path_counts(h, _p(paths, i64p))
        return Solution(STATUS[L.sko_solution_status(h)], it, rel, tb, tk, V, core, W,
                        float(L.sko_solution_total_time(h)), caps,
                        dict(zip(["direct", "householder", "cleanup", "unused"], paths.tolist())))
    finally:
        L.sko_solution_free(h)


def factorized_cg(a, b, c1, c2, cfg=None, mode=REPRODUCIBLE, lean=False):
    return solve(CG, a, b, c1, c2, cfg, mode, lean)


def factorized_cg_lyapunov(a, c1, cfg=None, mode=REPRODUCIBLE, lean=False):
    return solve(CG_LYAPUNOV, a, None, c1, None, cfg, mode, lean)


def factorized_bicgstab(a, b, c1, c2, cfg=None, mode=REPRODUCIBLE):
    return solve(BICGSTAB, a, b, c1, c2, cfg, mode)


def true_residual_factors(a: Csr, b: Csr, c1, c2, v, core, w) -> float:
    c1 = np.asfortranarray(c1, dtype=np.float64)
    c2 = np.asfortranarray(c2, dtype=np.float64)
    v = np.asfortranarray(v, dtype=np.float64)
    core = np.asfortranarray(core, dtype=np.float64)
    w = np.asfortranarray(w, dtype=np.float64)
    ca, cb = a.c(), b.c()
    return float(lib().sko_true_residual_factors(C.byref(ca), C.byref(cb), _p(c1), _p(c2),
                                                C.c_int64(c1.shape[1]), _p(v), C.c_int64(v.shape[1]),
                                                _p(core), _p(w), C.c_int64(w.shape[1])))


def true_residual(a, b, c1, c2, sol: Solution) -> float:
    return true_residual_factors(a, b, c1, c2, sol.V, sol.core, sol.W)


def small_sylvester_apply(p, h, g) -> np.ndarray:
    p = np.asfortranarray(p, dtype=np.float64)
    h = np.asfortranarray(h, dtype=np.float64)
    g = np.asfortranarray(g, dtype=np.float64)
    if h.shape[1] != p.shape[0] or g.shape[1] != p.shape[1]:
        raise OracleError(-1, "DimensionError: small_sylvester_apply: shapes do not conform")
    out = np.zeros((h.shape[0], g.shape[0]), order="F")
    lib().sko_small_sylvester_apply(_p(p), C.c_int64(p.shape[0]), C.c_int64(p.shape[1]), _p(h),
                                    C.c_int64(h.shape[0]), _p(g), C.c_int64(g.shape[0]), _p(out))
    return out


def frobenius_inner(x, y) -> float:
    """frobenius_inner (dense_matrix.cpp:131-139): sequential column-major."""
    x = np.asfortranarray(x, dtype=np.float64)
    y = np.asfortranarray(y, dtype=np.float64)
    if x.shape != y.shape:
        raise OracleError(-1, "DimensionError: frobenius_inner: shapes differ")
    return float(lib().sko_frobenius_inner(_p(x), _p(y), C.c_int64(x.shape[0]), C.c_int64(x.shape[1])))


def r1_dot(x, y) -> float:
    x = np.ascontiguousarray(x, dtype=np.float64).ravel()
    y = np.ascontiguousarray(y, dtype=np.float64).ravel()
    return float(lib().sko_r1_dot(_p(x), _p(y), C.c_int64(x.size)))


def r2_inner(x, y) -> float:
    x = np.asfortranarray(x, dtype=np.float64)
    y = np.asfortranarray(y, dtype=np.float64)
    return float(lib().sko_r2_inner(_p(x), _p(y), C.c_int64(x.shape[0]), C.c_int64(x.shape[1])))
