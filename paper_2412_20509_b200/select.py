"""Model-selection consumers of the deviance kernels (gmfkit/select.py).

``information_criteria`` (select.py:81-96) needs the deviance of a fitted
state over every observed entry plus, for the negative binomial, the
dispersion constant of select.py:57-78; both come from ONE streaming pass
over the resident counts (``gmf_loglik_full``: dense or CSR, zeros handled
analytically).  ``mu_at`` (select.py:141-145) and ``heldout_scores`` (the
cross-validation scoring of select.py:201-213: ``_mu_at`` then
``metrics.rel_deviance``) evaluate the predictor at listed entries on the
GPU (``gmf_entries_eval``), fused with the four metric sums so the
held-out means never round-trip through host memory.

The per-entry predictor follows the fit's own: ``U V' + X B' + Gamma Z'``
(+ the optional per-row ``offset``, the SURVEY §8c shim applied to
``_mu_at`` as well); the device path implements Poisson and negative
binomial with the log link, like the fit.
"""
from __future__ import annotations

import numpy as np

from . import _lib
from .engine import DeviceFit, Schedule
from .exceptions import ConfigError
from .families import Poisson
from .metrics import EvalResult, ratios
from .model import CovariateSet, FactorizationState, PenaltyConfig, ResponseMatrix, parameter_count

__all__ = ["information_criteria", "loglik_terms", "mu_at", "heldout_scores"]


def _state_fit(state, data, covs, fam, lnk, offset, dtype, device):
    """A zero-step device handle holding ``state`` over ``data`` (one row block)."""
    from .optim import SgdConfig
    cfg = SgdConfig(max_epochs=1)
    sched = Schedule(state.n, state.m, cfg, row_blocks=[np.arange(state.n)],
                     col_blocks=[np.arange(state.m)], n_steps=0)
    fit = DeviceFit(data, covs, fam, lnk, PenaltyConfig(), cfg, state, schedule=sched,
                    offset=offset, dtype=dtype, device=device)
    fit.reset(fam.nb_shape if fam.kind == "neg_binomial" else 1.0)
    return fit


def loglik_terms(state: FactorizationState, data: ResponseMatrix, covs: CovariateSet, fam, lnk,
                 *, offset=None, dtype="f64", device=None):
    """(sum w D(y, mu), dispersion constant c) over all observed entries, one
    pass on the GPU; c = -2 sum w (sat + y log y) for the negative binomial
    (select.py:71-78), 0 for Poisson (select.py:79)."""
    state.check_shapes(data, covs)
    fit = _state_fit(state, data, covs, fam, lnk, offset, dtype, device)
    try:
        dev, const = fit.loglik_full()
    finally:
        fit.close()
    return dev, const


def information_criteria(state: FactorizationState, data: ResponseMatrix, covs: CovariateSet,
                         fam, lnk, *, offset=None, dtype="f64", device=None):
    """(AIC, BIC) of a fitted state (select.py:81-96):
    AIC = D/phi + c(phi) + 2k, BIC = D/phi + c(phi) + k log|Omega|,
    k = pm + qn + d(n+m) + 1."""
    dev, const = loglik_terms(state, data, covs, fam, lnk, offset=offset, dtype=dtype,
                              device=device)
    val = dev / state.phi + const
    k = parameter_count(data.n, data.m, covs.p, covs.q, state.rank)
    return val + 2.0 * k, val + k * np.log(data.n_observed)


def _entries(fit: DeviceFit, rows, cols):
    torch = fit.torch
    rows = np.asarray(rows, dtype=np.int64).ravel()
    cols = np.asarray(cols, dtype=np.int64).ravel()
    if rows.shape != cols.shape:
        raise ConfigError("rows and cols must have the same length")
    if rows.size and (rows.min() < 0 or rows.max() >= fit.n or cols.min() < 0
                      or cols.max() >= fit.m):
        raise ConfigError("entry index out of range")
    inv = np.empty(fit.n, dtype=np.int64)
    inv[fit.order] = np.arange(fit.n, dtype=np.int64)
    r = torch.from_numpy(inv[rows]).to(fit.device)
    c = torch.from_numpy(cols.astype(np.int32)).to(fit.device)
    return r, c


def mu_at(state: FactorizationState, covs: CovariateSet, lnk, rows, cols, *, offset=None,
          dtype="f64", device=None) -> np.ndarray:
    """g^{-1}(eta) at the listed entries (select.py:141-145), on the GPU."""
    empty = ResponseMatrix(csr=(np.zeros(state.n + 1, np.int64), np.zeros(0, np.int32),
                                np.zeros(0, np.int32)), shape=(state.n, state.m))
    fit = _state_fit(state, empty, covs, Poisson(), lnk, offset, dtype, device)
    try:
        r, c = _entries(fit, rows, cols)
        out = fit.torch.empty(r.numel(), dtype=fit.torch.float64, device=fit.device)
        _lib.check(fit.lib.gmf_entries_eval(fit.h, _lib.ptr(r), _lib.ptr(c), None, r.numel(), 0.0,
                                            _lib.ptr(out), None, fit.stream()),
                   "gmf_entries_eval")
        return out.cpu().numpy()
    finally:
        fit.close()


def heldout_scores(state: FactorizationState, covs: CovariateSet, fam, lnk, rows, cols, y_test,
                   ybar_train: float, *, offset=None, dtype="f64", device=None) -> EvalResult:
    """Held-out scoring of cv_rank_select (select.py:206-208 with
    metrics.py:35-55): mu at (rows, cols), then rel_deviance and rel_log_rmse
    against the train mean, fused in one kernel."""
    y = np.asarray(y_test, dtype=float).ravel()
    if y.size == 0:
        raise ConfigError("test set is empty")
    if y.size != np.asarray(rows).size:
        raise ConfigError("y_test and mu_hat must have the same length")
    if fam.kind not in ("poisson", "neg_binomial"):
        raise _lib.UnsupportedError(f"device scoring implements poisson/neg_binomial, got {fam.kind}")
    empty = ResponseMatrix(csr=(np.zeros(state.n + 1, np.int64), np.zeros(0, np.int32),
                                np.zeros(0, np.int32)), shape=(state.n, state.m))
    fit = _state_fit(state, empty, covs, fam if fam.kind == "neg_binomial" else Poisson(), lnk,
                     offset, dtype, device)
    try:
        torch = fit.torch
        r, c = _entries(fit, rows, cols)
        yd = torch.from_numpy(y).to(fit.device)
        sums = torch.zeros(4, dtype=torch.float64, device=fit.device)
        _lib.check(fit.lib.gmf_entries_eval(fit.h, _lib.ptr(r), _lib.ptr(c), _lib.ptr(yd),
                                            r.numel(), float(ybar_train), None, _lib.ptr(sums),
                                            fit.stream()), "gmf_entries_eval")
        s = sums.cpu().numpy()
    finally:
        fit.close()
    dev, lr = ratios(s)
    return EvalResult(rel_log_rmse=lr, rel_deviance=dev, n_test=int(y.size))

