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

__all__ = ["information_criteria", "loglik_terms", "mu_at", "heldout_scores", "RankSelectionReport",
           "holdout_mask", "cv_rank_select", "scree_eigenvalues", "residual_scores", "elbow_pick"]


def _state_fit(state, data, covs, fam, lnk, offset, dtype, device, eval_only=False):
    """A zero-step device handle holding ``state`` over ``data`` (one row block)."""
    from .optim import SgdConfig
    cfg = SgdConfig(max_epochs=1)
    sched = Schedule(state.n, state.m, cfg, row_blocks=[np.arange(state.n)],
                     col_blocks=[np.arange(state.m)], n_steps=0)
    fit = DeviceFit(data, covs, fam, lnk, PenaltyConfig(), cfg, state, schedule=sched,
                    offset=offset, dtype=dtype, device=device, eval_only=eval_only)
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
        if fit.general:
            const = _general_constant(fit, data, fam, state.phi)
    finally:
        fit.close()
    return dev, const


def _general_constant(fit, data, fam, phi):
    """c(phi) of select.py:57-79 for a general-mode fit, over the observed
    entries: n_obs log phi (Gaussian, inverse Gaussian), 2 sum(lgamma(s) -
    s log s + s) with s = w / phi (Gamma), the NB saturated terms for a
    non-log link, else 0."""
    torch = fit.torch
    n_obs = int(data.n_observed)
    # unobserved entries carry the hole marker (last mantissa bit) in y_work
    obs = None
    if not data.fully_observed:
        idt = torch.int64 if fit.y_work.dtype == torch.float64 else torch.int32
        obs = (fit.y_work.view(idt) & 1) == 0
    kind = fam.kind
    if kind in ("gaussian", "inverse_gaussian"):
        return float(n_obs * np.log(phi))
    if kind == "gamma":
        if fit.weights is None:
            s = 1.0 / phi
            from math import lgamma
            return float(2.0 * n_obs * (lgamma(s) - s * np.log(s) + s))
        s = fit.weights.double() / phi
        t = 2.0 * (torch.lgamma(s) - s * torch.log(s) + s)
        return float((t if obs is None else torch.where(obs, t, torch.zeros_like(t))).sum().item())
    if kind == "neg_binomial":
        a = float(fam.nb_shape)
        y = fit.y_work.double()
        if obs is not None:
            y = torch.where(obs, y, torch.zeros_like(y))
        w = 1.0 if fit.weights is None else fit.weights.double()
        sat = (torch.lgamma(y + a) - torch.lgamma(torch.tensor(a, device=y.device, dtype=y.dtype))
               - torch.lgamma(y + 1.0) - (y + a) * torch.log(y + a) + a * np.log(a))
        ylogy = torch.where(y > 0, y * torch.log(torch.where(y > 0, y, torch.ones_like(y))),
                            torch.zeros_like(y))
        t = -2.0 * (w * (sat + ylogy))
        return float((t if obs is None else torch.where(obs, t, torch.zeros_like(t))).sum().item())
    return 0.0


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
    fit = _state_fit(state, empty, covs, Poisson(), lnk, offset, dtype, device, eval_only=True)
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
    empty = ResponseMatrix(csr=(np.zeros(state.n + 1, np.int64), np.zeros(0, np.int32),
                                np.zeros(0, np.int32)), shape=(state.n, state.m))
    fit = _state_fit(state, empty, covs, fam, lnk, offset, dtype, device, eval_only=True)
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



# ---------------------------------------------------------------------------
# repeated-holdout CV over ranks, scree (select.py:99-138, 148-294)
# ---------------------------------------------------------------------------

from dataclasses import dataclass, field   # noqa: E402


@dataclass
class RankSelectionReport:
    """select.py:45-53."""
    ranks: list
    aic: list = field(default_factory=list)
    bic: list = field(default_factory=list)
    cv_deviance: list = field(default_factory=list)   # per-rank lists, one per fold
    scree_eigenvalues: list = field(default_factory=list)
    chosen: dict = field(default_factory=dict)
    failures: list = field(default_factory=list)       # (rank, fold, message)


def holdout_mask(data: ResponseMatrix, fraction: float, seed: int = 0):
    """Mask floor(fraction |Omega|) observed entries uniformly at random
    (select.py:99-121); returns (train ResponseMatrix, (rows, cols))."""
    if not 0.0 < fraction < 1.0:
        raise ConfigError("holdout fraction must lie strictly between 0 and 1")
    if data.csr is not None:
        data = ResponseMatrix(data.dense(), weights=data.weights)
    rows, cols = np.nonzero(data.mask)
    n_test = int(np.floor(fraction * rows.size))
    rng = np.random.default_rng(seed)
    if n_test == 0:
        return data, (rows[:0], cols[:0])
    for _ in range(100):
        pick = np.sort(rng.choice(rows.size, size=n_test, replace=False))
        mask = data.mask.copy()
        mask[rows[pick], cols[pick]] = False
        if mask.any(axis=1).all() and mask.any(axis=0).all():
            train = ResponseMatrix(data.values, mask, data.weights)
            return train, (rows[pick], cols[pick])
    raise ConfigError("could not draw a holdout leaving every row and column observed")


def _nan_safe_mean(values) -> float:
    arr = np.asarray(values, dtype=float)
    finite = arr[np.isfinite(arr)]
    return float(finite.mean()) if finite.size else float("nan")


def _pad_state(state: FactorizationState, d: int, rng) -> FactorizationState:
    """Grow a projected state to rank d with small random columns (select.py:130-138)."""
    add = d - state.rank
    if add <= 0:
        return state.copy()
    u = np.hstack([state.u, 1e-3 * rng.standard_normal((state.n, add))])
    v = np.hstack([state.v, 1e-3 * rng.standard_normal((state.m, add))])
    return FactorizationState(state.b.copy(), state.gamma.copy(), u, v, state.phi, state.nb_shape)


def _ols_residual(data: ResponseMatrix, covs: CovariateSet, device=None):
    """log1p observed data minus its OLS fit on the covariates (select.py:240-251),
    a dense device array."""
    import torch
    from .initialization import _dense_inputs, _ols_stage_dense
    _lib.require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else
                       int(str(device).split(":")[-1]))
    Y, mask, W = _dense_inputs(data, dev)
    y_log = torch.log1p(torch.clamp(torch.where(mask, Y, torch.zeros_like(Y)), min=-0.5))
    X = torch.from_numpy(np.ascontiguousarray(covs.x, dtype=float)).to(dev)
    Z = torch.from_numpy(np.ascontiguousarray(covs.z, dtype=float)).to(dev)
    b = _ols_stage_dense(y_log, W, X, None)
    eta = X @ b.T
    gamma = _ols_stage_dense(y_log.T, W.T, Z, eta.T)
    if Z.shape[1]:
        eta = eta + gamma @ Z.T
    return torch.where(mask, y_log - eta, torch.zeros_like(Y))


def scree_eigenvalues(data: ResponseMatrix, covs: CovariateSet, max_rank: int, seed: int = 0,
                      *, device=None) -> np.ndarray:
    """Descending squared singular values of the log1p OLS residual (select.py:254-261)."""
    from .initialization import randomized_svd_dense
    if max_rank > min(data.shape):
        raise ConfigError("max_rank cannot exceed min(n, m)")
    _, sing, _ = randomized_svd_dense(_ols_residual(data, covs, device), max_rank, seed=seed)
    return np.sort(sing.cpu().numpy() ** 2)[::-1]


def residual_scores(data: ResponseMatrix, covs: CovariateSet, d: int, seed: int = 0,
                    *, device=None) -> np.ndarray:
    """Row scores of the log1p OLS residual (select.py:264-269)."""
    from .initialization import randomized_svd_dense
    left, sing, _ = randomized_svd_dense(_ols_residual(data, covs, device), d, seed=seed)
    return (left * sing).cpu().numpy()


def elbow_pick(eigenvalues):
    """Rank at the largest consecutive eigenvalue gap ratio (select.py:272-294)."""
    vals = np.asarray(list(eigenvalues), dtype=float)
    if vals.size == 0:
        raise ConfigError("eigenvalue list is empty")
    if np.any(np.diff(vals) > 1e-12):
        raise ConfigError("eigenvalues must be sorted in decreasing order")
    if vals.size == 1:
        return 1, {"warning": "single eigenvalue; rank 1 by default"}
    with np.errstate(divide="ignore", invalid="ignore"):
        r = vals[:-1] / vals[1:]
    r = np.where(np.isnan(r), 1.0, r)
    best = int(np.argmax(r))
    flags = {}
    others = np.delete(r, best)
    if others.size and np.max(r) <= 2.0 * np.max(others):
        flags["ambiguous"] = True
        if np.allclose(r, r[0], rtol=1e-8, atol=1e-12):
            return 1, flags
    return best + 1, flags


def cv_rank_select(data: ResponseMatrix, covs: CovariateSet, fam, lnk, ranks, folds: int = 5,
                   cfg=None, penalty: PenaltyConfig | None = None, algorithm: str = "asgd",
                   holdout_fraction: float = 0.3, seed: int = 0, threads: int = 1,
                   include_scree: bool = True, *, dtype="f64", devices=None):
    """Repeated-holdout CV over a rank grid plus AIC/BIC and the scree pick
    (select.py:148-237).  Every (fold, rank) cell is a device fit of the train
    matrix (the holdout as unobserved entries, imputed on the device), ranks
    fitted in increasing order, each warm-started from the previous rank's
    projected state padded with a small random column (the first rank from
    init_glm_svd).  ``devices``: CUDA devices the folds are spread over, one
    host thread per device (folds are independent replicas); the default is
    the current device, folds in turn.  Results are seed-deterministic."""
    from concurrent.futures import ThreadPoolExecutor

    from .exceptions import GmfError
    from .optim import SgdConfig, fit_asgd
    if folds < 2:
        raise ConfigError("need at least 2 folds")
    ranks = sorted(set(int(d) for d in ranks))
    if any(d < 0 for d in ranks):
        raise ConfigError("ranks must be nonnegative")
    if algorithm != "asgd":
        raise _lib.UnsupportedError(f"the device fitter is aSGD; algorithm {algorithm!r} "
                                    "(quasi-Newton / AIRWLS) is not on the device path")
    cfg = cfg or SgdConfig()
    penalty = penalty or PenaltyConfig()
    if data.csr is not None:
        data = ResponseMatrix(data.dense(), weights=data.weights)
    splits = [holdout_mask(data, holdout_fraction, seed=seed + 1000 * f) for f in range(folds)]
    rngs = [np.random.default_rng(seed + 7919 + f) for f in range(folds)]
    ybars = [float(np.mean(train.values[train.mask])) for train, _ in splits]
    report = RankSelectionReport(ranks=list(ranks))
    warm = [None] * folds
    import torch
    devs = list(devices) if devices else [torch.cuda.current_device()]

    def cell(f, d):
        train, _ = splits[f]
        dev = devs[f % len(devs)]
        try:
            with torch.cuda.device(dev):
                init = _pad_state(warm[f], d, rngs[f]) if warm[f] is not None else None
                return fit_asgd(train, covs, fam, lnk, penalty, cfg, init_state=init, rank=d,
                                identify_mode="B1", dtype=dtype, device=dev)
        except GmfError as err:   # a failed cell must not poison the grid
            return err

    for d in ranks:
        aics, bics, dvs = [], [], []
        if len(devs) > 1:
            with ThreadPoolExecutor(max_workers=len(devs)) as pool:
                results = list(pool.map(lambda f: cell(f, d), range(folds)))
        else:
            results = [cell(f, d) for f in range(folds)]
        for f, res in enumerate(results):
            if isinstance(res, GmfError):
                report.failures.append((d, f, str(res)))
                dvs.append(np.nan); aics.append(np.nan); bics.append(np.nan)
                continue
            state, _ = res
            train, (trows, tcols) = splits[f]
            dev = devs[f % len(devs)]
            try:
                aic, bic = information_criteria(state, train, covs, fam, lnk, dtype=dtype, device=dev)
                sc = heldout_scores(state, covs, fam, lnk, trows, tcols,
                                    data.values[trows, tcols], ybars[f], dtype=dtype, device=dev)
                dv = sc.rel_deviance
            except GmfError as err:
                report.failures.append((d, f, str(err)))
                dvs.append(np.nan); aics.append(np.nan); bics.append(np.nan)
                continue
            warm[f] = state
            aics.append(aic)
            bics.append(bic)
            dvs.append(dv)
        report.aic.append(_nan_safe_mean(aics))
        report.bic.append(_nan_safe_mean(bics))
        report.cv_deviance.append(dvs)
    cv_means = [_nan_safe_mean(v) for v in report.cv_deviance]
    report.chosen["cv"] = ranks[int(np.argmin(np.nan_to_num(cv_means, nan=np.inf)))]
    report.chosen["aic"] = ranks[int(np.argmin(np.nan_to_num(report.aic, nan=np.inf)))]
    report.chosen["bic"] = ranks[int(np.argmin(np.nan_to_num(report.bic, nan=np.inf)))]
    if include_scree:
        max_rank = min(max(ranks) + 1, min(data.shape))
        report.scree_eigenvalues = list(scree_eigenvalues(data, covs, max_rank))
        pick, _ = elbow_pick(report.scree_eigenvalues)
        report.chosen["scree"] = pick
    return report
