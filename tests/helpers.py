"""Shared helpers: convert oracle CSR to the product's SparseMatrix, bitwise compares."""
import numpy as np


def to_sk(sk, csr):
    return sk.SparseMatrix(csr.n_rows, csr.n_cols, csr.row_ptr, csr.col_idx, csr.values)


def bits_equal(a, b) -> bool:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.shape != b.shape:
        return False
    return bool(np.array_equal(a.view(np.uint64), b.view(np.uint64)) or np.array_equal(a, b))


def max_rel(a, b) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300))) if a.size else 0.0
