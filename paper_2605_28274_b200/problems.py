"""Problem generators and the BASELINE.json configurations.

Generators restate proj/src/problems.cpp:10-96 in the product library
(sk_gen_* in include/sylkrylov_b200.h): 5-point / 7-point stencils with
Dirichlet boundaries, centred convection couplings -1 -/+ w h/2 (h = 1/(g+1)),
and random_rhs from std::mt19937_64 + Box-Muller. Peclet convention: w = Pe x wind.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import SparseMatrix, _check, _p, i64p, lib

LAPLACIAN_2D, CONVDIFF_2D, CONVDIFF_3D = 0, 1, 2


def _stencil(kind: int, grid: int, wind=(0.0, 0.0, 0.0)) -> SparseMatrix:
    L = lib()
    L.sk_gen_stencil_nnz.restype = C.c_int64
    nnz = int(L.sk_gen_stencil_nnz(C.c_int32(kind), C.c_int64(grid)))
    if nnz < 0:
        raise ValueError("grid must be >= 2")
    n = grid ** 3 if kind == CONVDIFF_3D else grid * grid
    rp = np.zeros(n + 1, dtype=np.int64)
    ci = np.zeros(nnz, dtype=np.int64)
    va = np.zeros(nnz, dtype=np.float64)
    w = np.array([float(x) for x in (list(wind) + [0.0, 0.0, 0.0])[:3]])
    _check(L.sk_gen_stencil(C.c_int32(kind), C.c_int64(grid), _p(w), _p(rp, i64p), _p(ci, i64p), _p(va)))
    return SparseMatrix(n, n, rp, ci, va)


def laplacian_2d(grid: int) -> SparseMatrix:
    """laplacian_2d (problems.cpp:10-30)."""
    return _stencil(LAPLACIAN_2D, grid)


def convection_diffusion_2d(grid: int, wind) -> SparseMatrix:
    """2D analogue of convection_diffusion_3d."""
    return _stencil(CONVDIFF_2D, grid, wind)


def convection_diffusion_3d(grid: int, wind) -> SparseMatrix:
    """convection_diffusion_3d (problems.cpp:32-60)."""
    return _stencil(CONVDIFF_3D, grid, wind)


def random_rhs(rows: int, s: int, seed: int) -> np.ndarray:
    """random_rhs (problems.cpp:71-96): column-major rows x s, N(0,1)."""
    out = np.zeros((rows, s), order="F")
    _check(lib().sk_gen_random_rhs(C.c_int64(rows), C.c_int64(s), C.c_uint64(seed), _p(out)))
    return out


@dataclass
class Config:
    name: str
    method: str               # "cg" | "cg_lyapunov" | "bicgstab"
    a: SparseMatrix
    b: Optional[SparseMatrix]
    c1: np.ndarray
    c2: Optional[np.ndarray]
    eps_tol: float
    max_iter: int
    description: str


def baseline_config(idx: int, seed: int = 1234) -> Config:
    """BASELINE.json configs[idx-1] with the SURVEY 8d conventions (C2 seed = seed + 1)."""
    if idx == 1:
        a = laplacian_2d(64)
        c1 = random_rhs(4096, 1, seed)
        c1 /= np.linalg.norm(c1)
        c2 = random_rhs(4096, 1, seed + 1)
        c2 /= np.linalg.norm(c2)
        return Config("C1", "cg", a, a, c1, c2, 1e-8, 500,
                      "factorized CG, 2D Laplacian 64x64 (n=m=4096), s=1, unit-norm columns")
    if idx == 2:
        a = convection_diffusion_2d(256, (10.0, 10.0))
        b = convection_diffusion_2d(256, (10.0, -10.0))
        return Config("C2", "bicgstab", a, b, random_rhs(65536, 4, seed), random_rhs(65536, 4, seed + 1),
                      1e-8, 0, "factorized BiCGSTAB, 2D conv-diff 256^2, Pe 10, winds (1,1)/(1,-1), s=4")
    if idx == 3:
        a = laplacian_2d(1024)
        return Config("C3", "cg_lyapunov", a, None, random_rhs(1 << 20, 1, seed), None, 1e-8, 0,
                      "factorized CG Lyapunov, 2D Laplacian 1024^2 (n=1,048,576), s=1")
    if idx == 4:
        a = convection_diffusion_3d(128, (5.0, 2.5, 1.25))
        b = convection_diffusion_3d(64, (0.0, 0.0, 0.0))
        return Config("C4", "bicgstab", a, b, random_rhs(128 ** 3, 8, seed), random_rhs(64 ** 3, 8, seed + 1),
                      1e-8, 0, "factorized BiCGSTAB, 3D conv-diff 128^3 (Pe 5) x 3D Laplacian 64^3, s=8")
    if idx == 5:
        a = laplacian_2d(4096)
        return Config("C5", "cg", a, a, random_rhs(1 << 24, 2, seed), random_rhs(1 << 24, 2, seed + 1),
                      1e-8, 200, "factorized CG, 2D Laplacian 4096^2 (n=m=16,777,216), s=2, 200 iterations")
    raise ValueError(idx)
