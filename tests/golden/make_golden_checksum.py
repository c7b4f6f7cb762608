"""Checksum of a regenerated count matrix (shared by make_golden.py and the
tests; no reference import)."""
import numpy as np


def y_checksum(y_int):
    """Order-sensitive checksum of a count matrix (guards the regenerated c2 input)."""
    y = np.asarray(y_int, dtype=np.int64)
    cols = np.arange(y.shape[1], dtype=np.int64)
    rows = np.arange(y.shape[0], dtype=np.int64)
    return np.asarray([y.sum(), np.count_nonzero(y), (y * cols[None, :]).sum() % (2**61 - 1),
                       (y * rows[:, None]).sum() % (2**61 - 1)], dtype=np.int64)
