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
           "read_mask_file", "write_mask_file", "write_dense_csv", "read_dense_csv",
           "write_json", "read_json", "Manifest"]


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


# ---------------------------------------------------------------------------
# dense CSV, mask lists, JSON reports and run manifests (io.py:42-95,
# 111-118, 142-200): the output side of the CLI, byte-compatible with the
# reference's files (17 significant digits round-trip float64; NaN = missing)
# ---------------------------------------------------------------------------

def _num(v: float) -> str:
    return "NaN" if v != v else format(float(v), ".17g")


def write_dense_csv(path, values, row_names=None, col_names=None) -> None:
    """Header row of column names, a leading label column, one line per row."""
    a = np.asarray(values, dtype=float)
    if a.ndim != 2:
        raise ConfigError("write_dense_csv expects a 2-D array")
    n, m = a.shape
    rn = row_names or [f"r{i + 1}" for i in range(n)]
    cn = col_names or [f"c{j + 1}" for j in range(m)]
    lines = ["," + ",".join(cn)]
    lines += [rn[i] + "," + ",".join(_num(v) for v in a[i]) for i in range(n)]
    with open(path, "w") as fh:
        fh.write("\n".join(lines) + "\n")


def read_dense_csv(path):
    """(values, row_names, col_names); a malformed field reports line and column."""
    with open(path) as fh:
        head = fh.readline().rstrip("\n")
        if not head:
            raise ConfigError(f"{path}: line 1: empty header")
        cn = head.split(",")[1:]
        vals, rn = [], []
        for lineno, line in enumerate(fh, start=2):
            line = line.rstrip("\n")
            if not line:
                continue
            f = line.split(",")
            if len(f) != len(cn) + 1:
                raise ConfigError(f"{path}: line {lineno}: expected {len(cn) + 1} fields, "
                                  f"got {len(f)}")
            row = []
            for col, tok in enumerate(f[1:], start=2):
                try:
                    row.append(float(tok))
                except ValueError:
                    raise ConfigError(f"{path}: line {lineno}: column {col}: not a number") from None
            rn.append(f[0])
            vals.append(row)
    if not vals:
        raise ConfigError(f"{path}: no data rows")
    return np.asarray(vals), rn, cn


def write_mask_file(path, mask) -> None:
    """1-based 'row col' lines of the unobserved positions, row-major."""
    holes = np.argwhere(~np.asarray(mask, dtype=bool))
    with open(path, "w") as fh:
        fh.write("% unobserved entries, 1-based 'row col'\n")
        fh.writelines(f"{i + 1} {j + 1}\n" for i, j in holes)


def _plain(obj):
    """numpy scalars / arrays inside a report -> JSON-native values."""
    if isinstance(obj, (np.floating, np.integer, np.bool_)):
        return obj.item()
    if isinstance(obj, np.ndarray):
        return obj.tolist()
    if isinstance(obj, dict):
        return {k: _plain(v) for k, v in obj.items()}
    if isinstance(obj, (list, tuple)):
        return [_plain(v) for v in obj]
    return obj


def write_json(path, obj) -> None:
    """Sorted keys, 2-space indent, trailing newline (byte-stable across reruns)."""
    import json
    with open(path, "w") as fh:
        json.dump(_plain(obj), fh, indent=2, sort_keys=True)
        fh.write("\n")


def read_json(path):
    import json
    with open(path) as fh:
        return json.load(fh)


def sha256_of(path) -> str:
    import hashlib
    h = hashlib.sha256()
    with open(path, "rb") as fh:
        while True:
            block = fh.read(1 << 20)
            if not block:
                break
            h.update(block)
    return h.hexdigest()


class Manifest:
    """Run metadata (io.py:165-195): command, merged config, seed, input
    checksums, versions; wall clock and peak RSS are added by finish(), so
    every other output file stays byte-stable across reruns."""

    def __init__(self, command: str, config: dict, seed, inputs=None):
        import sys
        import time
        from . import __version__
        self._t0 = time.perf_counter()
        self.payload = {"command": command, "config": _plain(config), "seed": seed,
                        "input_checksums": {str(p): sha256_of(p) for p in (inputs or [])},
                        "gmfkit_version": __version__,
                        "python_version": sys.version.split()[0]}

    def finish(self, path, elapsed_extra: dict | None = None) -> None:
        import resource
        import time
        self.payload["wall_clock_seconds"] = time.perf_counter() - self._t0
        self.payload["peak_rss_mb"] = resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1024.0
        if elapsed_extra:
            self.payload.update(_plain(elapsed_extra))
        write_json(path, self.payload)
