"""sylkrylov-b200: B200-native factorized Krylov solvers for AX + XB = C1 C2^T.

Python mirror of the reference interface (proj/include/sylkrylov/
factorized_solvers.hpp:39-61, solver_types.hpp:11-47, errors.hpp:9-57) over the
C-ABI in include/sylkrylov_b200.h. The compute path is libsk_b200.so (sm_100a
kernels); there is no CPU fallback -- loading fails loudly when the library or
a CUDA device is missing.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsk_b200.so")
LIB_PATH = os.environ.get("SK_LIB_PATH", LIB_PATH)  # experiment variants (build.py SK_VARIANT)

i64p = C.POINTER(C.c_int64)
f64p = C.POINTER(C.c_double)


# ---- errors (errors.hpp:9-57) ----
class SylkrylovError(RuntimeError):
    code = 0


class DimensionError(SylkrylovError, ValueError):
    code = -1


class InvalidMatrixError(SylkrylovError, ValueError):
    code = -2


class RankDeficientStartError(SylkrylovError):
    code = -3


class CudaError(SylkrylovError):
    code = -10


class OutOfMemoryError(SylkrylovError, MemoryError):
    code = -11


class CapacityError(SylkrylovError):
    code = -12


class UnsupportedError(SylkrylovError):
    code = -13


class IoError(SylkrylovError, OSError):
    """errors.hpp:48-51 (a failed open or write of an output file)."""
    code = -14


class ParseError(SylkrylovError, ValueError):
    """errors.hpp:54-57 (malformed Matrix Market input)."""


_ERRORS = {e.code: e for e in [DimensionError, InvalidMatrixError, RankDeficientStartError,
                                CudaError, OutOfMemoryError, CapacityError, UnsupportedError, IoError]}


class _Csr(C.Structure):
    _fields_ = [("n_rows", C.c_int64), ("n_cols", C.c_int64), ("nnz", C.c_int64),
                ("row_ptr", i64p), ("col_idx", i64p), ("values", f64p)]


class _Cfg(C.Structure):
    _fields_ = [("eps_tol", C.c_double), ("max_iter", C.c_int64), ("breakdown_tol", C.c_double),
                ("capture_iterates", C.c_int32), ("lanczos_full_reorth", C.c_int32)]


class _Gpu(C.Structure):
    _fields_ = [("device", C.c_int32), ("profile", C.c_int32), ("capacity_bytes", C.c_int64),
                ("reduction_mode", C.c_int32), ("reserved", C.c_int32 * 7)]


class _Rec(C.Structure):
    _fields_ = [("iteration", C.c_int64), ("rel_residual", C.c_double), ("t_basic_s", C.c_double),
                ("t_krylov_s", C.c_double), ("t_trunc_s", C.c_double)]


class _Stats(C.Structure):
    _fields_ = [("device_time_s", C.c_double), ("h2d_time_s", C.c_double), ("d2h_time_s", C.c_double),
                ("h2d_bytes", C.c_int64), ("d2h_bytes", C.c_int64), ("kernel_launches", C.c_int64),
                ("iterations", C.c_int64), ("class_time_s", C.c_double * 9),
                ("class_launches", C.c_int64 * 9), ("class_bytes", C.c_double * 9),
                ("paths", C.c_int64 * 4), ("class_flops", C.c_double * 9)]


KERNEL_CLASSES = ["spmm", "gram", "rare_path", "update", "core_a", "core_b",
                  "arnoldi_update", "dense_image", "other"]

_lib = None


def lib() -> C.CDLL:
    """Loads libsk_b200.so (build it with `python paper_2605_28274_b200/build.py`)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run paper_2605_28274_b200/build.py "
                              "(the B200 path has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        L.sk_last_error.restype = C.c_char_p
        L.sk_version.restype = C.c_char_p
        L.sk_solution_total_time.restype = C.c_double
        for f in ["sk_solution_num_records", "sk_solution_num_captured"]:
            getattr(L, f).restype = C.c_int64
        L.sk_solution_status.restype = C.c_int32
        L.sk_device_count.restype = C.c_int32
        _lib = L
    return _lib


def _check(rc: int):
    if rc != 0:
        raise _ERRORS.get(rc, SylkrylovError)(lib().sk_last_error().decode())


def _p(a, t=f64p):
    return a.ctypes.data_as(t)


def device_count() -> int:
    return int(lib().sk_device_count())


# ---- types (sparse_matrix.hpp, solver_types.hpp) ----
@dataclass
class SparseMatrix:
    """CSR with 64-bit indices and strictly increasing columns per row."""
    n_rows: int
    n_cols: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.values.size)

    def rows(self) -> int:
        return self.n_rows

    def cols(self) -> int:
        return self.n_cols

    def _c(self) -> _Csr:
        self.row_ptr = np.ascontiguousarray(self.row_ptr, dtype=np.int64)
        self.col_idx = np.ascontiguousarray(self.col_idx, dtype=np.int64)
        self.values = np.ascontiguousarray(self.values, dtype=np.float64)
        return _Csr(self.n_rows, self.n_cols, self.nnz, _p(self.row_ptr, i64p),
                    _p(self.col_idx, i64p), _p(self.values))

    @staticmethod
    def from_scipy(m) -> "SparseMatrix":
        m = m.tocsr()
        m.sort_indices()
        return SparseMatrix(m.shape[0], m.shape[1], m.indptr.astype(np.int64),
                            m.indices.astype(np.int64), m.data.astype(np.float64))

    @staticmethod
    def identity(n: int) -> "SparseMatrix":
        return SparseMatrix(n, n, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int64),
                            np.ones(n))


@dataclass
class SolverConfig:
    eps_tol: float = 1e-8
    max_iter: int = 0
    breakdown_tol: float = 1e-12
    capture_iterates: bool = False
    lanczos_full_reorth: bool = False

    def _c(self) -> _Cfg:
        return _Cfg(self.eps_tol, self.max_iter, self.breakdown_tol, int(self.capture_iterates),
                    int(self.lanczos_full_reorth))


@dataclass
class GpuOptions:
    device: int = 0
    profile: bool = False
    capacity_bytes: int = 0
    reduction_mode: int = 0  # SK_REDUCTION_REPRODUCIBLE; 1 = reference_order (unsupported on the device)

    def _c(self) -> _Gpu:
        return _Gpu(self.device, int(self.profile), self.capacity_bytes, int(self.reduction_mode))


@dataclass
class IterationRecord:
    iteration: int
    rel_residual: float
    t_basic_s: float = 0.0
    t_krylov_s: float = 0.0
    t_trunc_s: float = 0.0


@dataclass
class ConvergenceHistory:
    records: List[IterationRecord] = field(default_factory=list)
    total_time_s: float = 0.0

    def iterations(self) -> int:
        return self.records[-1].iteration if self.records else 0

    def final_rel_residual(self) -> float:
        return self.records[-1].rel_residual if self.records else 1.0

    def rel_residuals(self) -> np.ndarray:
        return np.array([r.rel_residual for r in self.records])


STATUS = {0: "converged", 1: "max_iter", 2: "breakdown"}


class FactorizedSolution:
    """X = V core W^T (factorized_solvers.hpp:14-23). V, core, W are fetched from
    HBM lazily (V/W can be tens of GB at the large configs)."""

    def __init__(self, handle):
        self._h = handle
        L = lib()
        self.status = STATUS[int(L.sk_solution_status(handle))]
        n, rv, m, rw = (C.c_int64() for _ in range(4))
        L.sk_solution_dims(handle, C.byref(n), C.byref(rv), C.byref(m), C.byref(rw))
        self.n, self.rv, self.m, self.rw = n.value, rv.value, m.value, rw.value
        cnt = int(L.sk_solution_num_records(handle))
        recs = (_Rec * max(cnt, 1))()
        _check(L.sk_solution_history(handle, recs, C.c_int64(cnt)))
        self.history = ConvergenceHistory(
            [IterationRecord(r.iteration, r.rel_residual, r.t_basic_s, r.t_krylov_s, r.t_trunc_s)
             for r in recs[:cnt]], float(L.sk_solution_total_time(handle)))
        st = _Stats()
        _check(L.sk_solution_stats(handle, C.byref(st)))
        self.stats = {
            "device_time_s": st.device_time_s, "h2d_time_s": st.h2d_time_s,
            "h2d_bytes": st.h2d_bytes, "d2h_bytes": st.d2h_bytes,
            "kernel_launches": st.kernel_launches, "iterations": st.iterations,
            "classes": {KERNEL_CLASSES[i]: {"time_s": st.class_time_s[i],
                                             "launches": st.class_launches[i],
                                             "bytes": st.class_bytes[i],
                                             "flops": st.class_flops[i]} for i in range(9)},
            "paths": dict(zip(["direct", "householder", "cleanup", "unused"], list(st.paths))),
        }
        self.captured_cores = []
        for i in range(int(L.sk_solution_num_captured(handle))):
            r_, c_ = C.c_int64(), C.c_int64()
            _check(L.sk_solution_captured_core(handle, C.c_int64(i), C.byref(r_), C.byref(c_), None))
            buf = np.zeros((r_.value, c_.value), order="F")
            _check(L.sk_solution_captured_core(handle, C.c_int64(i), C.byref(r_), C.byref(c_), _p(buf)))
            self.captured_cores.append(buf)
        # row partition: this rank's global row offsets of V and W (0 on one GPU)
        r0v, r0w = C.c_int64(), C.c_int64()
        _check(L.sk_solution_partition(handle, C.byref(r0v), None, C.byref(r0w), None))
        self.row0_v, self.row0_w = r0v.value, r0w.value
        self._V = self._W = self._core = None

    @property
    def V(self) -> np.ndarray:
        if self._V is None:
            self._V = np.zeros((self.n, self.rv), order="F")
            _check(lib().sk_solution_copy_V(self._h, _p(self._V)))
        return self._V

    @property
    def W(self) -> np.ndarray:
        if self._W is None:
            self._W = np.zeros((self.m, self.rw), order="F")
            _check(lib().sk_solution_copy_W(self._h, _p(self._W)))
        return self._W

    @property
    def core(self) -> np.ndarray:
        if self._core is None:
            self._core = np.zeros((self.rv, self.rw), order="F")
            _check(lib().sk_solution_copy_core(self._h, _p(self._core)))
        return self._core

    def write_factors(self, out_dir: str, fmt: str = "mtx") -> None:
        """V / core / W files of the CLI (main.cpp:182-184), streamed from HBM:
        fmt "mtx" = Matrix Market text (V.mtx, core.mtx, W.mtx), "binary" = the
        binary sidecar (V.skb, core.skb, W.skb; read back with read_factor)."""
        os.makedirs(out_dir, exist_ok=True)
        code = {"mtx": 0, "binary": 1}[fmt]
        _check(lib().sk_solution_write_factors(self._h, os.fsencode(out_dir), C.c_int32(code)))

    def write_history_csv(self, path: str) -> None:
        """write_history_csv (bench.cpp:179-193), byte-identical format."""
        _check(lib().sk_write_history_csv(self._h, os.fsencode(path)))

    def free(self):
        if getattr(self, "_h", None):
            lib().sk_solution_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def _mat(c, rows, name) -> np.ndarray:
    c = np.asfortranarray(np.asarray(c, dtype=np.float64))
    if c.ndim != 2 or c.shape[0] != rows:
        raise DimensionError(f"solver: {name} row count must match the operator")
    return c


def factorized_cg(a: SparseMatrix, b: SparseMatrix, c1, c2, cfg: Optional[SolverConfig] = None,
                  gpu: Optional[GpuOptions] = None) -> FactorizedSolution:
    """factorized_cg (factorized_solvers.hpp:39-43)."""
    c1 = _mat(c1, a.n_rows, "C1")
    c2 = _mat(c2, b.n_rows, "C2")
    if c1.shape[1] != c2.shape[1] or c1.shape[1] < 1:
        raise DimensionError("solver: C1 and C2 must have the same positive column count")
    ca, cb = a._c(), b._c()
    h = C.c_void_p()
    cfg_c = (cfg or SolverConfig())._c()
    gpu_c = (gpu or GpuOptions())._c()
    _check(lib().sk_factorized_cg(C.byref(ca), C.byref(cb), _p(c1), _p(c2), C.c_int64(c1.shape[1]),
                                  C.byref(cfg_c), C.byref(gpu_c), C.byref(h)))
    return FactorizedSolution(h)


def factorized_cg_lyapunov(a: SparseMatrix, c1, cfg: Optional[SolverConfig] = None,
                           gpu: Optional[GpuOptions] = None) -> FactorizedSolution:
    """factorized_cg_lyapunov (factorized_solvers.hpp:45-48)."""
    if a.n_rows != a.n_cols:
        raise DimensionError("factorized_cg_lyapunov: A must be square")
    c1 = _mat(c1, a.n_rows, "C1")
    ca = a._c()
    h = C.c_void_p()
    cfg_c = (cfg or SolverConfig())._c()
    gpu_c = (gpu or GpuOptions())._c()
    _check(lib().sk_factorized_cg_lyapunov(C.byref(ca), _p(c1), C.c_int64(c1.shape[1]),
                                           C.byref(cfg_c), C.byref(gpu_c), C.byref(h)))
    return FactorizedSolution(h)


def factorized_bicgstab(a: SparseMatrix, b: SparseMatrix, c1, c2,
                        cfg: Optional[SolverConfig] = None,
                        gpu: Optional[GpuOptions] = None) -> FactorizedSolution:
    """factorized_bicgstab (factorized_solvers.hpp:50-53)."""
    c1 = _mat(c1, a.n_rows, "C1")
    c2 = _mat(c2, b.n_rows, "C2")
    if c1.shape[1] != c2.shape[1] or c1.shape[1] < 1:
        raise DimensionError("solver: C1 and C2 must have the same positive column count")
    ca, cb = a._c(), b._c()
    h = C.c_void_p()
    cfg_c = (cfg or SolverConfig())._c()
    gpu_c = (gpu or GpuOptions())._c()
    _check(lib().sk_factorized_bicgstab(C.byref(ca), C.byref(cb), _p(c1), _p(c2),
                                        C.c_int64(c1.shape[1]), C.byref(cfg_c), C.byref(gpu_c),
                                        C.byref(h)))
    return FactorizedSolution(h)


METHODS = {"cg": 0, "cg_lyapunov": 1, "bicgstab": 2}


class ResidentProblem:
    """Inputs uploaded once to HBM (sk_problem_create), solved repeatedly."""

    def __init__(self, method: str, a: SparseMatrix, b: Optional[SparseMatrix], c1, c2=None,
                 gpu: Optional[GpuOptions] = None):
        c1 = _mat(c1, a.n_rows, "C1")
        self._keep = [c1]
        ca = a._c()
        cb = b._c() if b is not None else None
        c2a = _mat(c2, b.n_rows, "C2") if c2 is not None else None
        self._keep.append(c2a)
        gpu_c = (gpu or GpuOptions())._c()
        h = C.c_void_p()
        _check(lib().sk_problem_create(C.c_int32(METHODS[method]), C.byref(ca),
                                       C.byref(cb) if cb is not None else None, _p(c1),
                                       _p(c2a) if c2a is not None else None,
                                       C.c_int64(c1.shape[1]), C.byref(gpu_c), C.byref(h)))
        self._h = h

    def solve(self, cfg: Optional[SolverConfig] = None) -> FactorizedSolution:
        h = C.c_void_p()
        cfg_c = (cfg or SolverConfig())._c()
        _check(lib().sk_problem_solve(self._h, C.byref(cfg_c), C.byref(h)))
        return FactorizedSolution(h)

    def true_residual(self, sol: FactorizedSolution) -> float:
        """Device true residual of `sol` against this problem's resident operators and
        right-hand side (factorized_solvers.cpp:441-444; sk_problem_true_residual)."""
        out = C.c_double()
        _check(lib().sk_problem_true_residual(self._h, sol._h, C.byref(out)))
        return out.value

    def free(self):
        if getattr(self, "_h", None):
            lib().sk_problem_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def true_residual(a: SparseMatrix, b: SparseMatrix, c1, c2, sol: FactorizedSolution) -> float:
    """true_residual (factorized_solvers.hpp:56-57) on the device: the solution's V,
    core and W are read where they live (HBM)."""
    c1 = _mat(c1, a.n_rows, "C1")
    c2 = _mat(c2, b.n_rows, "C2")
    if c1.shape[1] != c2.shape[1]:
        raise DimensionError("true_residual: right-hand side shapes do not conform")
    ca, cb = a._c(), b._c()
    out = C.c_double()
    _check(lib().sk_true_residual(C.byref(ca), C.byref(cb), _p(c1), _p(c2), C.c_int64(c1.shape[1]),
                                  sol._h, C.byref(out)))
    return out.value


def true_residual_factors(a: SparseMatrix, b: SparseMatrix, c1, c2, v, core, w) -> float:
    """true_residual_factors (factorized_solvers.hpp:59-61) on the device for host factors."""
    c1 = _mat(c1, a.n_rows, "C1")
    c2 = _mat(c2, b.n_rows, "C2")
    v = np.asfortranarray(np.asarray(v, dtype=np.float64))
    core = np.asfortranarray(np.asarray(core, dtype=np.float64))
    w = np.asfortranarray(np.asarray(w, dtype=np.float64))
    if c1.shape[1] != c2.shape[1]:
        raise DimensionError("true_residual: right-hand side shapes do not conform")
    if (v.ndim != 2 or core.ndim != 2 or w.ndim != 2 or v.shape[0] != a.n_rows or w.shape[0] != b.n_rows
            or core.shape != (v.shape[1], w.shape[1])):
        raise DimensionError("true_residual: factor shapes do not conform")
    ca, cb = a._c(), b._c()
    out = C.c_double()
    _check(lib().sk_true_residual_factors(C.byref(ca), C.byref(cb), _p(c1), _p(c2), C.c_int64(c1.shape[1]),
                                          _p(v), C.c_int64(v.shape[1]), _p(core), _p(w),
                                          C.c_int64(w.shape[1]), C.byref(out)))
    return out.value


def x_distance(sol: FactorizedSolution, v_ref, core_ref, w_ref, lyapunov: bool = False):
    """||X_sol - X_ref||_F / ||X_ref||_F with X = V core W^T on both sides, through factor
    products only (the stacked-factor QR of factorized_solvers.cpp:410-438):
    R_V = qr([V_sol, V_ref]).R and R_W = qr([W_sol, W_ref]).R by the device's streaming TSQR
    (sk_solution_stacked_r: V_sol, W_sol never leave HBM), then the small product
    R_V diag(core_sol, -core_ref) R_W^T on the host. Returns (relative distance, ||X_ref||_F)."""
    v_ref = np.asfortranarray(np.asarray(v_ref, dtype=np.float64))
    w_ref = v_ref if lyapunov else np.asfortranarray(np.asarray(w_ref, dtype=np.float64))
    core_ref = np.asarray(core_ref, dtype=np.float64)
    if v_ref.shape[0] != sol.n or w_ref.shape[0] != sol.m or core_ref.shape != (v_ref.shape[1], w_ref.shape[1]):
        raise DimensionError("x_distance: reference factor shapes do not conform")

    def stacked(side, ref, r_own):
        wdt = r_own + ref.shape[1]
        out = np.zeros((wdt, wdt), order="F")
        _check(lib().sk_solution_stacked_r(sol._h, C.c_int32(side), _p(ref), C.c_int64(ref.shape[1]), _p(out)))
        return np.triu(out)

    rv = stacked(0, v_ref, sol.rv)
    rw = rv if (lyapunov and sol.rw == sol.rv) else stacked(1, w_ref, sol.rw)
    core = sol.core
    mid = np.zeros((rv.shape[0], rw.shape[0]))
    mid[:sol.rv, :sol.rw] = core
    mid[sol.rv:, sol.rw:] = -core_ref
    diff = np.linalg.norm(rv @ mid @ rw.T)
    ref_norm = np.linalg.norm(rv[:, sol.rv:] @ core_ref @ rw[:, sol.rw:].T)
    return float(diff / ref_norm), float(ref_norm)


def spmm(a: SparseMatrix, x, transpose: bool = False) -> np.ndarray:
    """Device SpMM (K1) in the reference's per-row order (sparse_matrix.cpp:142-200)."""
    x = np.asfortranarray(np.asarray(x, dtype=np.float64))
    rows = a.n_cols if transpose else a.n_rows
    y = np.zeros((rows, x.shape[1]), order="F")
    ca = a._c()
    _check(lib().sk_spmm(C.byref(ca), _p(x), C.c_int64(x.shape[1]), C.c_int32(int(transpose)), _p(y)))
    return y


# ---------------------------------------------------------------------------
# Row partition: multi-GPU CG / Lyapunov CG
# ---------------------------------------------------------------------------
class _Partition(C.Structure):
    _fields_ = [(f, C.c_int64) for f in
                ("row0", "rows", "chunk_rows", "chunks", "chunks_max", "chunks_total", "halo")]


def partition_plan(n: int, halo: int, world: int, rank: int) -> dict:
    """The row split every rank computes identically (sk_partition_plan; host only)."""
    out = _Partition()
    _check(lib().sk_partition_plan(C.c_int64(n), C.c_int64(halo), C.c_int32(world), C.c_int32(rank),
                                   C.byref(out)))
    return {f: getattr(out, f) for f, _ in _Partition._fields_}


class Communicator:
    """Collectives of the row-partitioned solve: NCCL (one process per GPU) or an
    in-process group whose ranks are host threads (sk_comm)."""

    def __init__(self, handle):
        self._h = handle
        self.rank = int(lib().sk_comm_rank(handle))
        self.size = int(lib().sk_comm_size(handle))

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        _check(lib().sk_nccl_unique_id(buf))
        return bytes(buf)

    @classmethod
    def nccl(cls, uid: bytes, nranks: int, rank: int, device: int) -> "Communicator":
        if len(uid) != 128:
            raise DimensionError("NCCL unique id must be 128 bytes")
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        h = C.c_void_p()
        _check(lib().sk_comm_create_nccl(buf, C.c_int32(nranks), C.c_int32(rank), C.c_int32(device),
                                         C.byref(h)))
        return cls(h)

    @classmethod
    def local_group(cls, nranks: int) -> list:
        hs = (C.c_void_p * nranks)()
        _check(lib().sk_comm_create_local_group(C.c_int32(nranks), hs))
        return [cls(C.c_void_p(h)) for h in hs]

    def free(self):
        if getattr(self, "_h", None):
            lib().sk_comm_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class PartitionedProblem(ResidentProblem):
    """This rank's rows of a CG / Lyapunov CG problem (sk_problem_create_partitioned).
    Every rank passes the whole operators and right-hand sides; solve() must be
    called by all ranks of the communicator together."""

    def __init__(self, method: str, a: SparseMatrix, b: Optional[SparseMatrix], c1, c2,
                 comm: Communicator, gpu: Optional[GpuOptions] = None):
        c1 = _mat(c1, a.n_rows, "C1")
        c2a = _mat(c2, b.n_rows, "C2") if c2 is not None else None
        self._keep = [c1, c2a, comm]
        ca = a._c()
        cb = b._c() if b is not None else None
        gpu_c = (gpu or GpuOptions())._c()
        h = C.c_void_p()
        _check(lib().sk_problem_create_partitioned(
            C.c_int32(METHODS[method]), C.byref(ca), C.byref(cb) if cb is not None else None, _p(c1),
            _p(c2a) if c2a is not None else None, C.c_int64(c1.shape[1]), C.byref(gpu_c), comm._h,
            C.byref(h)))
        self._h = h


def solve_local_group(method: str, a: SparseMatrix, b: Optional[SparseMatrix], c1, c2, world: int,
                      cfg: Optional[SolverConfig] = None, gpu: Optional[GpuOptions] = None) -> list:
    """Runs the row-partitioned solve with `world` ranks as host threads of this
    process (sk_comm_create_local_group); returns every rank's solution."""
    import threading

    comms = Communicator.local_group(world)
    sols, errs = [None] * world, [None] * world
    probs = [None] * world

    def run(r):
        try:
            probs[r] = PartitionedProblem(method, a, b, c1, c2, comms[r], gpu)
            sols[r] = probs[r].solve(cfg)
        except BaseException as e:  # surfaced after join
            errs[r] = e

    ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for e in errs:
        if e is not None:
            raise e
    for p in probs:
        p.free()
    return sols


# ---- page-locked host arrays ----
class _Pinned:
    def __init__(self, ptr):
        self.ptr = ptr

    def __del__(self):
        try:
            lib().sk_host_free(self.ptr)
        except Exception:
            pass


def measure_fp64_peak(device: int = 0):
    """(DFMA TFLOP/s, mul-then-add TFLOP/s) of the device, measured (sk_measure_fp64_peak)."""
    f, m = C.c_double(), C.c_double()
    _check(lib().sk_measure_fp64_peak(C.c_int32(device), C.byref(f), C.byref(m)))
    return f.value, m.value


def pinned_empty(shape, dtype=np.float64, order: str = "F") -> np.ndarray:
    """A numpy array in page-locked host memory (sk_host_alloc): solver inputs in
    such memory reach HBM by direct DMA instead of through the staging lanes."""
    dt = np.dtype(dtype)
    nbytes = int(np.prod(shape)) * dt.itemsize
    p = C.c_void_p()
    _check(lib().sk_host_alloc(C.c_int64(nbytes), C.byref(p)))
    owner = _Pinned(p)
    buf = (C.c_char * max(nbytes, 1)).from_address(p.value)
    buf.owner = owner  # freed when the last view of the buffer goes away
    return np.ndarray(shape, dtype=dt, buffer=buf, order=order)


# ---- on-disk formats (matrix_market.cpp, bench.cpp:179-193, main.cpp:146-239) ----
def write_matrix_market(m, path: str) -> None:
    """write_matrix_market (matrix_market.cpp:148-175): a SparseMatrix as
    "coordinate real general", a 2-D array as "array real general" (column-major),
    17 significant digits. Formatting runs natively on all host threads."""
    if isinstance(m, SparseMatrix):
        cm = m._c()
        _check(lib().sk_write_matrix_market_csr(C.byref(cm), os.fsencode(path)))
        return
    a = np.asfortranarray(np.asarray(m, dtype=np.float64))
    if a.ndim != 2:
        raise DimensionError("write_matrix_market: a 2-D array is required")
    _check(lib().sk_write_matrix_market_dense(_p(a), C.c_int64(a.shape[0]), C.c_int64(a.shape[1]),
                                              os.fsencode(path)))


def read_matrix_market(path: str):
    """read_matrix_market (matrix_market.cpp:1-138 restated): coordinate real
    general/symmetric -> SparseMatrix (symmetric storage expanded, duplicates
    summed, columns sorted as from_triplets, sparse_matrix.cpp:34-69); array real
    general -> column-major ndarray. Anything else raises ParseError."""
    with open(path) as f:
        header = f.readline()
        tok = header.split()
        if len(tok) < 5 or tok[0].lower() != "%%matrixmarket" or tok[1].lower() != "matrix":
            raise ParseError(f"{path}: malformed MatrixMarket header: {header.rstrip()}")
        fmt, field, sym = tok[2].lower(), tok[3].lower(), tok[4].lower()
        if fmt not in ("coordinate", "array"):
            raise ParseError(f"{path}: unsupported format '{tok[2]}'")
        if field != "real":
            raise ParseError(f"{path}: unsupported field '{tok[3]}' (real required)")
        if sym not in ("general", "symmetric"):
            raise ParseError(f"{path}: unsupported symmetry '{tok[4]}'")
        if fmt == "array" and sym == "symmetric":
            raise ParseError(f"{path}: array symmetric storage not supported")
        lines = [ln for ln in f.read().splitlines() if ln.strip() and not ln.lstrip().startswith("%")]
    if not lines:
        raise ParseError(f"{path}: missing size line")
    size = lines[0].split()
    try:
        if fmt == "array":
            rows, cols = int(size[0]), int(size[1])
            vals = np.array([float(x) for x in lines[1:]], dtype=np.float64)
            if vals.size != rows * cols:
                raise ParseError(f"{path}: expected {rows * cols} values, found {vals.size}")
            return vals.reshape((rows, cols), order="F")
        rows, cols, nnz = int(size[0]), int(size[1]), int(size[2])
        ent = np.array([ln.split()[:3] for ln in lines[1:]], dtype=np.float64).reshape(-1, 3)
    except (ValueError, IndexError) as e:
        raise ParseError(f"{path}: {e}") from None
    if ent.shape[0] != nnz:
        raise ParseError(f"{path}: expected {nnz} entries, found {ent.shape[0]}")
    i = ent[:, 0].astype(np.int64) - 1
    j = ent[:, 1].astype(np.int64) - 1
    v = ent[:, 2]
    if ((i < 0) | (i >= rows) | (j < 0) | (j >= cols)).any():
        raise ParseError(f"{path}: entry index out of range")
    if sym == "symmetric":
        off = i != j
        i, j, v = np.concatenate([i, j[off]]), np.concatenate([j, i[off]]), np.concatenate([v, v[off]])
    order = np.lexsort((j, i))
    i, j, v = i[order], j[order], v[order]
    key = i * cols + j
    first = np.ones(key.size, dtype=bool)
    first[1:] = key[1:] != key[:-1]
    # duplicates summed (from_triplets; the reference's std::sort leaves their order unspecified)
    vs = np.add.reduceat(v, np.flatnonzero(first)) if v.size else v.copy()
    ii, jj = i[first], j[first]
    row_ptr = np.zeros(rows + 1, dtype=np.int64)
    np.add.at(row_ptr, ii + 1, 1)
    return SparseMatrix(rows, cols, np.cumsum(row_ptr), jj.astype(np.int64), vs)


def read_factor(path: str) -> np.ndarray:
    """Reads a binary sidecar written by FactorizedSolution.write_factors(fmt="binary")."""
    with open(path, "rb") as f:
        if f.read(8) != b"SKFACT01":
            raise ParseError(f"{path}: not a factor sidecar")
        rows, cols = np.frombuffer(f.read(16), dtype="<i8")
        data = np.frombuffer(f.read(), dtype="<f8")
    if data.size != rows * cols:
        raise ParseError(f"{path}: truncated ({data.size} of {rows * cols} values)")
    return data.reshape((int(rows), int(cols)), order="F")


def write_solution(out_dir: str, method: str, sol: FactorizedSolution, a: SparseMatrix, b: SparseMatrix,
                   c1, c2, cfg: Optional["SolverConfig"] = None, inputs: Optional[dict] = None,
                   seed: Optional[int] = None, fmt: str = "mtx", lyapunov: bool = False) -> dict:
    """The output directory of `sylkrylov solve` for the factorized methods
    (main.cpp:146-239): V/core/W, history.csv and meta.json with the same keys
    (the true residual is computed on the device). Returns the meta dict."""
    import json
    import math
    cfg = cfg or SolverConfig()
    os.makedirs(out_dir, exist_ok=True)
    residual = true_residual(a, b, c1, c2, sol)
    sol.write_factors(out_dir, fmt)
    sol.write_history_csv(os.path.join(out_dir, "history.csv"))
    recs = sol.history.records
    # resolve_max_iter (solver_types.cpp:34-38)
    max_iter = cfg.max_iter if cfg.max_iter > 0 else min(10 * math.ceil(math.sqrt(float(a.n_rows) * float(b.n_rows))),
                                                         10000)
    meta = {"method": method, "eps_tol": cfg.eps_tol, "max_iter": max_iter,
            "lyapunov": lyapunov, "inputs": inputs or {},
            "format": "factored", "status": sol.status, "iterations": sol.history.iterations(),
            "final_true_residual": residual,
            "ranks": {"rank": min(sol.rv, sol.rw), "v_cols": sol.rv, "w_cols": sol.rw},
            "timings": {"total_s": sol.history.total_time_s,
                        "basic_s": sum(r.t_basic_s for r in recs),
                        "krylov_s": sum(r.t_krylov_s for r in recs),
                        "trunc_s": sum(r.t_trunc_s for r in recs)}}
    if seed is not None:
        meta["seed"] = seed
    with open(os.path.join(out_dir, "meta.json"), "w") as f:
        f.write(json.dumps(meta, indent=2, sort_keys=True) + "\n")
    return meta
