"""Minibatch gradient / Fisher-diagonal estimates on the device
(gmfkit/gradients.py:35-141): the standalone face of the fused K1 kernel."""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .exceptions import ConfigError

__all__ = ["Minibatch", "GradientPair", "minibatch_gradients", "full_gradients",
           "penalty_vectors"]


@dataclass
class Minibatch:
    """Row index set I and column index set J (gradients.py:35-53)."""

    row_idx: np.ndarray
    col_idx: np.ndarray

    def __post_init__(self):
        self.row_idx = np.asarray(self.row_idx, dtype=np.intp)
        self.col_idx = np.asarray(self.col_idx, dtype=np.intp)
        if self.row_idx.size == 0 or self.col_idx.size == 0:
            raise ConfigError("minibatch index sets must be nonempty")
        for name, idx in (("row", self.row_idx), ("col", self.col_idx)):
            if idx.min() < 0 or np.unique(idx).size != idx.size:
                raise ConfigError(f"minibatch {name} indices must be unique and nonnegative")

    @classmethod
    def full(cls, n: int, m: int) -> "Minibatch":
        return cls(np.arange(n), np.arange(m))


@dataclass
class GradientPair:
    """Gradients and Fisher Hessian diagonals for [Gamma, U] and [B, V] rows."""

    g_rowside: np.ndarray
    h_rowside: np.ndarray
    g_colside: np.ndarray
    h_colside: np.ndarray


def penalty_vectors(covs, d, penalty):
    """Per-coordinate ridge weights (gradients.py:91-99)."""
    return (np.concatenate([np.full(covs.q, penalty.lam_gamma), np.full(d, penalty.lam_u)]),
            np.concatenate([np.full(covs.p, penalty.lam_b), np.full(d, penalty.lam_v)]))


def _complement(idx, size):
    keep = np.ones(size, dtype=bool)
    keep[idx] = False
    return np.flatnonzero(keep)


def minibatch_gradients(state, data, covs, fam, lnk, penalty, mb, y_block=None, *,
                        offset=None, dtype="f64", device=None, return_nb_sums=False,
                        k1_impl="auto"):
    """Unbiased block estimates of the full gradients (gradients.py:116-132),
    computed by the fused K1 kernel through gmf_minibatch_grad."""
    from .engine import DeviceFit, Schedule
    from .optim import SgdConfig
    n, m = state.n, state.m
    I, J = mb.row_idx, mb.col_idx
    if I.max() >= n or J.max() >= m:
        raise ConfigError("minibatch indices out of range")
    if y_block is not None:
        raise ConfigError("y_block (pre-imputed working block) is not supported on the device path")
    state.check_shapes(data, covs)
    rows = [I] + ([_complement(I, n)] if I.size < n else [])
    cols = [J] + ([_complement(J, m)] if J.size < m else [])
    sched = Schedule(n, m, SgdConfig(max_epochs=1), row_blocks=rows, col_blocks=cols, n_steps=0)
    fit = DeviceFit(data, covs, fam, lnk, penalty, SgdConfig(max_epochs=1), state,
                    schedule=sched, offset=offset, dtype=dtype, device=device, k1_impl=k1_impl)
    try:
        alpha = getattr(fam, "nb_shape", 1.0)
        g_row, h_row, g_col, h_col, nb = fit.minibatch_grad(0, 0, alpha)
        cv = lambda t: t.double().cpu().numpy()
        gp = GradientPair(cv(g_row), cv(h_row), cv(g_col), cv(h_col))
        if return_nb_sums:
            return gp, tuple(nb.cpu().numpy().tolist())
        return gp
    finally:
        fit.close()


def full_gradients(state, data, covs, fam, lnk, penalty, y_work=None, **kw):
    """Exact gradients over all rows and columns (gradients.py:135-141)."""
    state.check_shapes(data, covs)
    return minibatch_gradients(state, data, covs, fam, lnk, penalty,
                               Minibatch.full(state.n, state.m), y_work, **kw)
