"""File formats on the path's input side (gmfkit/io.py:96-139).

The reference reads coordinate MatrixMarket with scipy and densifies it
(io.py:104-109), so a 1.3M x 500 count matrix becomes 5.2 GB of float64
before the fit even starts.  ``read_matrix_market_csr`` parses the file in
native code (``gmf_mm_header`` / ``gmf_mm_read_csr``) straight into the CSR
the device path uploads; ``read_matrix_market`` keeps the reference's dense
return for drop-in callers.  Duplicate coordinates are summed and symmetric
files mirrored, as scipy's ``mmread`` + ``todense`` do; values must be counts
(nonnegative integers), the device path's input.  ``read_mask_file`` and
``write_matrix_market`` mirror the reference's (mask lists are 1-based
'row col' lines of unobserved entries).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _lib
from .exceptions import ConfigError
from .model import ResponseMatrix

__all__ = ["read_matrix_market_csr", "read_matrix_market", "write_matrix_market",
           "read_mask_file"]


def _read_csr(path):
    lib = _lib.lib()
    p = os.fsencode(os.fspath(path))
    n, m, cap = C.c_int64(), C.c_int64(), C.c_int64()
    _lib.check(lib.gmf_mm_header(p, C.byref(n), C.byref(m), C.byref(cap)), "gmf_mm_header")
    indptr = np.zeros(n.value + 1, dtype=np.int64)
    indices = np.zeros(max(cap.value, 1), dtype=np.int32)
    counts = np.zeros(max(cap.value, 1), dtype=np.int32)
    nnz = C.c_int64()
    _lib.check(lib.gmf_mm_read_csr(p, cap.value, indptr.ctypes.data, indices.ctypes.data,
                                   counts.ctypes.data, C.byref(nnz)), "gmf_mm_read_csr")
    k = nnz.value
    return (n.value, m.value), indptr, indices[:k].copy(), counts[:k].copy()


def read_matrix_market_csr(path) -> ResponseMatrix:
    """Coordinate MatrixMarket counts -> a CSR ResponseMatrix (no densification)."""
    shape, indptr, indices, counts = _read_csr(path)
    return ResponseMatrix(csr=(indptr, indices, counts), shape=shape)


def read_matrix_market(path) -> np.ndarray:
    """Dense float64 array, the reference's return (io.py:104-109)."""
    (n, m), indptr, indices, counts = _read_csr(path)
    out = np.zeros((n, m))
    rows = np.repeat(np.arange(n), np.diff(indptr))
    out[rows, indices] = counts
    return out


def write_matrix_market(path, values, mask=None) -> None:
    """Coordinate MatrixMarket of the observed nonzeros (io.py:96-101)."""
    from scipy import io as spio
    from scipy import sparse
    values = np.asarray(values, dtype=float)
    filled = np.where(mask, values, 0.0) if mask is not None else values
    filled = np.where(np.isfinite(filled), filled, 0.0)
    spio.mmwrite(str(path), sparse.coo_matrix(filled), precision=17)


def read_mask_file(path, shape):
    """Boolean observation mask from a 1-based unobserved-entry list (io.py:121-139)."""
    mask = np.ones(shape, dtype=bool)
    with open(path) as fh:
        for lineno, line in enumerate(fh, start=1):
            line = line.strip()
            if not line or line.startswith(("%", "#")):
                continue
            parts = line.split()
            if len(parts) != 2:
                raise ConfigError(f"{path}: line {lineno}: expected 'row col'")
            try:
                i, j = int(parts[0]) - 1, int(parts[1]) - 1
            except ValueError:
                raise ConfigError(f"{path}: line {lineno}: indices must be integers") from None
            if not (0 <= i < shape[0] and 0 <= j < shape[1]):
                raise ConfigError(f"{path}: line {lineno}: index out of range")
            mask[i, j] = False
    return mask
