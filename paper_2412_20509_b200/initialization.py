"""OLS-SVD starting values on the GPU (gmfkit/initialization.py:143-169).

The reference builds the dense n x m link-transformed response, its OLS
residual and a randomized SVD of it (initialization.py:62-82) -- 5.2 GB of
fp64 per copy at 1.3M x 500.  Here nothing n x m is materialised.  With a
fully observed count matrix and the log link,

    Y_eps = log(Y + eps) = log(eps) 1 1' + S,   S sparse like Y,
    A     = Y_eps - X B' - Gamma Z' = S + L R',
    L = [1 | X | Gamma],  R = [log(eps) 1 | -B | -Z],

so every product of the initialization is one sparse product with S
(``gmf_csr_spmm`` over the CSR for S P, over the CSC for S' Q) plus
rank-(1+p+q) corrections.  The OLS stages solve the reference's damped normal
equations (glm.py:36-64 with the Gaussian/identity single Fisher step:
(D'D + 1e-8 I) c = D'(y - offset)); the range finder replays the reference's
probe (numpy ``default_rng(seed).standard_normal``) so the sketched subspace
is the reference's; the NB shape moment (initialization.py:93-100) is one
pass over all entries (``gmf_init_moments``).  Dense QR/SVD of the
(k + 10)-column sketches run in cuSOLVER through torch (library calls on
tall-skinny matrices).

Scope: Poisson / negative binomial with the log link, fully observed
responses, unit prior weights (the fit's own device scope).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .engine import _counts_int32
from .exceptions import ConfigError
from .model import CovariateSet, FactorizationState, ResponseMatrix

__all__ = ["InitMethod", "init_ols_svd", "init_glm_svd", "fit_glm_batched", "randomized_svd_sparse",
           "randomized_svd_dense"]


class _Laps:
    """GMF_VERBOSE=1: per-stage wall clock (device synchronised) to stderr."""

    def __init__(self):
        import os
        import time
        self.on = bool(os.environ.get("GMF_VERBOSE"))
        self.time = time
        self.t0 = time.perf_counter()

    def __call__(self, what):
        if self.on:
            import sys
            import torch
            torch.cuda.synchronize()
            print(f"[gmf] init_ols_svd {what}: {1e3 * (self.time.perf_counter() - self.t0):.1f} ms",
                  file=sys.stderr)


_LINK_EPS = {"log": 0.1, "logit": 0.01, "inverse": 0.1, "inverse_squared": 0.1}
_DAMPING = 1e-8            # glm.py:68 fit_glm_batched default
_ETA_CLIP_LOG = (-700.0, 700.0)   # initialization.py:217-220


@dataclass
class InitMethod:
    """Residual kind and g_eps perturbation (initialization.py:29-45)."""

    residual_kind: str = "deviance"
    link_epsilon: float | None = None

    def __post_init__(self):
        if self.residual_kind not in ("deviance", "pearson"):
            raise ConfigError("residual_kind must be 'deviance' or 'pearson'")
        if self.link_epsilon is not None and self.link_epsilon <= 0:
            raise ConfigError("link_epsilon must be positive")

    def eps_for(self, lnk) -> float:
        if self.link_epsilon is not None:
            return self.link_epsilon
        return _LINK_EPS.get(lnk.kind, 0.1)


class _SparseCounts:
    """Y on the device as CSR and CSC (int64 pointers, int32 indices/counts)."""

    def __init__(self, data: ResponseMatrix, dev):
        import torch
        n, m = data.shape
        if data.csr is not None:
            indptr, indices, vals = data.csr
        else:
            r, c = np.nonzero(data.values)
            indptr = np.zeros(n + 1, np.int64)
            np.cumsum(np.bincount(r, minlength=n), out=indptr[1:])
            indices, vals = c.astype(np.int32), data.values[r, c]
        counts = _counts_int32(np.asarray(vals), "response")
        self.n, self.m = n, m
        self.ptr = torch.from_numpy(np.asarray(indptr, np.int64)).to(dev)
        self.col = torch.from_numpy(np.asarray(indices, np.int32)).to(dev)
        self.val = torch.from_numpy(counts).to(dev)
        lens = self.ptr[1:] - self.ptr[:-1]
        self.max_row = int(lens.max().item()) if n else 0
        # CSC by a stable sort on the column index (row order kept within a column)
        order = torch.argsort(self.col.long(), stable=True)
        rows = torch.repeat_interleave(torch.arange(n, device=dev, dtype=torch.int32), lens)
        self.cptr = torch.zeros(m + 1, dtype=torch.int64, device=dev)
        self.cptr[1:] = torch.cumsum(torch.bincount(self.col.long(), minlength=m), 0)
        self.crow = rows[order].contiguous()
        self.cval = self.val[order].contiguous()
        clens = self.cptr[1:] - self.cptr[:-1]
        self.max_col = int(clens.max().item()) if m else 0

    def _spmm(self, transpose, P, eps):
        import torch
        lib = _lib.lib()
        P = P.contiguous()
        r = P.shape[1]
        nrows = self.m if transpose else self.n
        ptr, idx, val, mx = ((self.cptr, self.crow, self.cval, self.max_col) if transpose
                             else (self.ptr, self.col, self.val, self.max_row))
        out = torch.empty((nrows, r), dtype=torch.float64, device=P.device)
        wb = int(lib.gmf_spmm_work_bytes(nrows, mx, r))
        work = torch.empty(max(wb, 1), dtype=torch.uint8, device=P.device)
        stream = torch.cuda.current_stream(P.device).cuda_stream
        _lib.check(lib.gmf_csr_spmm(nrows, _lib.ptr(ptr), _lib.ptr(idx), _lib.ptr(val), mx,
                                    float(eps), _lib.ptr(P), r, _lib.ptr(out), _lib.ptr(work),
                                    stream), "gmf_csr_spmm")
        return out

    def s_mul(self, P, eps):
        """S P, P (m x r)."""
        return self._spmm(False, P, eps)

    def st_mul(self, Q, eps):
        """S' Q, Q (n x r)."""
        return self._spmm(True, Q, eps)

    def dense_s(self, eps):
        import torch
        out = torch.zeros((self.n, self.m), dtype=torch.float64, device=self.ptr.device)
        rows = torch.repeat_interleave(torch.arange(self.n, device=out.device),
                                       self.ptr[1:] - self.ptr[:-1])
        out[rows, self.col.long()] = torch.log(self.val.double() + eps) - math.log(eps)
        return out


def _damped_solve(design, rhs):
    """(D'D + 1e-8 I)^{-1} rhs (glm.py:49-53, Gaussian/identity Fisher step)."""
    import torch
    p = design.shape[1]
    G = design.T @ design + _DAMPING * torch.eye(p, dtype=torch.float64, device=design.device)
    return torch.linalg.solve(G, rhs)


def randomized_svd_sparse(Y: _SparseCounts, eps, L, R, k, oversample=10, n_power=2, seed=0):
    """randomized_svd (initialization.py:62-82) of A = S + L R' on the GPU."""
    import torch
    n, m = Y.n, Y.m
    dev = L.device
    k = min(k, min(n, m))
    if k == 0:
        z = lambda *s: torch.zeros(s, dtype=torch.float64, device=dev)
        return z(n, 0), z(0), z(m, 0)
    if k + oversample >= min(n, m):
        A = Y.dense_s(eps) + L @ R.T
        u, s, vt = torch.linalg.svd(A, full_matrices=False)
        return u[:, :k], s[:k], vt[:k].T
    rng = np.random.default_rng(seed)
    probe = torch.from_numpy(rng.standard_normal((m, k + oversample))).to(dev)
    a_mul = lambda P: Y.s_mul(P, eps) + L @ (R.T @ P)
    at_mul = lambda Q: Y.st_mul(Q, eps) + R @ (L.T @ Q)
    sketch = a_mul(probe)
    for _ in range(n_power):
        q, _ = torch.linalg.qr(sketch)
        sketch = a_mul(at_mul(q))
    q, _ = torch.linalg.qr(sketch)
    u_small, s, vt = torch.linalg.svd(at_mul(q).T, full_matrices=False)
    return (q @ u_small)[:, :k], s[:k], vt[:k].T


def init_ols_svd(data: ResponseMatrix, covs: CovariateSet, fam, lnk, d: int,
                 method: InitMethod | None = None, seed: int = 0, return_info: bool = False,
                 *, device=None):
    """Least-squares initialization on the link-transformed response
    (initialization.py:143-169), computed on the GPU; returns a host state."""
    import torch
    method = method or InitMethod()
    n, m = data.shape
    if d > min(n, m):
        raise ConfigError("rank d cannot exceed min(n, m)")
    if fam.kind not in ("poisson", "neg_binomial") or lnk.kind != "log":
        raise _lib.UnsupportedError(
            f"device initialization implements poisson/neg_binomial with log link, "
            f"got {fam.kind}+{lnk.kind}")
    if not data.fully_observed or data.weights is not None:
        raise _lib.UnsupportedError("device initialization needs a fully observed, unweighted "
                                    "response")
    _lib.require_cuda()
    _lib.lib()
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else
                       int(str(device).split(":")[-1]))
    eps = method.eps_for(lnk)
    leps = math.log(eps)
    lap = _Laps()
    Y = _SparseCounts(data, dev)
    lap("upload + CSC")
    f64 = dict(dtype=torch.float64, device=dev)
    X = torch.from_numpy(np.ascontiguousarray(covs.x, dtype=float)).to(dev)
    Z = torch.from_numpy(np.ascontiguousarray(covs.z, dtype=float)).to(dev)
    p, q = X.shape[1], Z.shape[1]
    ones_n, ones_m = torch.ones((n, 1), **f64), torch.ones((m, 1), **f64)

    # B stage: columns regress y_eps on X (initialization.py:154)
    if p:
        rhs = leps * X.sum(0)[:, None] * ones_m.T + Y.st_mul(X, eps).T      # X' Y_eps
        B = _damped_solve(X, rhs).T.contiguous()
    else:
        B = torch.zeros((m, 0), **f64)
    # Gamma stage: rows regress y_eps - X B' on Z (initialization.py:155-156)
    if q:
        rhs = leps * Z.sum(0)[None, :] + Y.s_mul(Z, eps) - X @ (B.T @ Z)    # rows of Z'(y_eps - off)
        Gm = _damped_solve(Z, rhs.T).T.contiguous()
    else:
        Gm = torch.zeros((n, 0), **f64)

    lap("OLS stages")
    # residual SVD (initialization.py:159-162)
    L = torch.cat([ones_n, X, Gm], 1)
    R = torch.cat([leps * ones_m, -B, -Z], 1)
    left, sing, right = randomized_svd_sparse(Y, eps, L, R, d, seed=seed)
    U = left * sing
    V = right
    lap("randomized SVD")

    nb_shape = 1.0
    if fam.kind == "neg_binomial":    # initialization.py:93-100 at mu0 (164-166)
        lib = _lib.lib()
        out = torch.zeros(2, **f64)
        work = torch.empty(int(lib.gmf_moments_work_bytes()), dtype=torch.uint8, device=dev)
        stream = torch.cuda.current_stream(dev).cuda_stream
        _lib.check(lib.gmf_init_moments(n, m, _lib.ptr(Y.ptr), _lib.ptr(Y.col), _lib.ptr(Y.val),
                                        _lib.ptr(X), _lib.ptr(B), p, _lib.ptr(Gm), _lib.ptr(Z), q,
                                        _ETA_CLIP_LOG[0], _ETA_CLIP_LOG[1], _lib.ptr(out),
                                        _lib.ptr(work), stream), "gmf_init_moments")
        num, den = (float(v) for v in out.cpu().numpy())
        nb_shape = 1e8 if den <= 0 else float(np.clip(num / den, 1e-4, 1e8))
    lap("NB moments")
    host = lambda t: t.cpu().numpy()
    state = FactorizationState(host(B), host(Gm), host(U), host(V), 1.0, nb_shape)
    lap("download")
    info = {"method": "ols_svd"}
    return (state, info) if return_info else state


# ---------------------------------------------------------------------------
# GLM-SVD (the reference's default initialization, initialization.py:172-214)
# ---------------------------------------------------------------------------

def _dense_inputs(data: ResponseMatrix, dev):
    """Y, observation mask and effective weights as dense fp64 device arrays."""
    import torch
    n, m = data.shape
    if data.csr is not None:
        indptr, indices, vals = data.csr
        Y = torch.zeros((n, m), dtype=torch.float64, device=dev)
        rows = np.repeat(np.arange(n), np.diff(np.asarray(indptr)))
        Y[torch.from_numpy(rows).to(dev), torch.from_numpy(np.asarray(indices, np.int64)).to(dev)] = \
            torch.from_numpy(np.asarray(vals, dtype=float)).to(dev)
        mask = torch.ones((n, m), dtype=torch.bool, device=dev)
    else:
        mask_h = data.mask if data.mask is not None else np.ones((n, m), bool)
        Y = torch.from_numpy(np.where(mask_h, data.values, 0.0)).to(dev)
        mask = torch.from_numpy(np.asarray(mask_h)).to(dev)
    W = (torch.ones((n, m), dtype=torch.float64, device=dev) if data.weights is None
         else torch.from_numpy(np.asarray(data.weights, dtype=float)).to(dev))
    return Y, mask, torch.where(mask, W, torch.zeros_like(W))


def _xlogy_ratio(y, mu):
    import torch
    return torch.where(y == 0, torch.zeros_like(y), y * torch.log(y / mu))


def _dev0(kind, alpha, y, mu):
    """Unit deviance without weights (families.py:267-425, every family)."""
    import torch
    if kind == "poisson":
        return 2.0 * (_xlogy_ratio(y, mu) - (y - mu))
    if kind == "neg_binomial":
        return 2.0 * (_xlogy_ratio(y, mu) - (y + alpha) * torch.log1p((y - mu) / (mu + alpha)))
    if kind == "gaussian":
        return (y - mu) ** 2
    if kind == "gamma":
        return 2.0 * ((y - mu) / mu - torch.log(y / mu))
    if kind == "inverse_gaussian":
        return (y - mu) ** 2 / (y * mu ** 2)
    mc = torch.clamp(mu, 1e-10, 1.0 - 1e-10)          # bernoulli (families.py:389-391)
    return 2.0 * (_xlogy_ratio(y, mc) + _xlogy_ratio(1.0 - y, 1.0 - mc))


def _mean(link, eta):
    """g^{-1}(eta) (kernels/_ref.py:21-32)."""
    import torch
    if link == "identity":
        return eta
    if link == "log":
        return torch.exp(eta)
    if link == "logit":
        return torch.sigmoid(eta)
    if link == "inverse":
        return 1.0 / eta
    return 1.0 / torch.sqrt(eta)


def _variance(kind, alpha, mu):
    if kind == "gaussian":
        return mu * 0 + 1.0
    if kind == "gamma":
        return mu * mu
    if kind == "inverse_gaussian":
        return mu * mu * mu
    if kind == "poisson":
        return mu
    if kind == "bernoulli":
        return mu * (1.0 - mu)
    return mu * (1.0 + mu / alpha)


def _derivs(kind, alpha, y, eta, w, link="log"):
    """dotD / ddotD with phi = 1: the canonical pairs' simplified forms, else
    -w r / (nu g'), w / (nu g'^2) (kernels/_ref.py:96-117)."""
    import torch
    mu = _mean(link, eta)
    r = y - mu
    pair = (kind, link)
    if pair == ("poisson", "log"):
        return -w * r, w * mu
    if pair == ("neg_binomial", "log"):
        inv = 1.0 / (1.0 + mu / alpha)
        return -w * r * inv, w * mu * inv
    if pair == ("bernoulli", "logit"):
        return -w * r, w * mu * (1.0 - mu)
    if pair == ("gaussian", "identity"):
        return -w * r, w * torch.ones_like(mu)
    if pair == ("gamma", "inverse"):
        return w * r, w * mu * mu
    if pair == ("inverse_gaussian", "inverse_squared"):
        return w * r / 2.0, w * mu ** 3 / 4.0
    nu = _variance(kind, alpha, mu)
    g1 = {"identity": lambda: torch.ones_like(mu), "log": lambda: 1.0 / mu,
          "logit": lambda: 1.0 / (mu * (1.0 - mu)), "inverse": lambda: -1.0 / (mu * mu),
          "inverse_squared": lambda: -2.0 / mu ** 3}[link]()
    return -w * r / (nu * g1), w / (nu * g1 * g1)


def _batched_deviance(kind, alpha, y, w, eta, link="log"):
    """Per-problem weighted deviance (glm.py:27-33): NaN-safe at dropped entries."""
    import torch
    dev = _dev0(kind, alpha, y, _mean(link, eta))
    return torch.where(w > 0, w * dev, torch.zeros_like(dev)).sum(0)


def _perturbed_transform(link, y, eps):
    """g_eps(y) (initialization.py:47-59)."""
    import torch
    if link == "identity":
        return y.clone()
    if link == "log":
        return torch.log(y + eps)
    if link == "logit":
        c = torch.clamp(y, eps, 1.0 - eps)
        return torch.log(c / (1.0 - c))
    c = torch.clamp(y, min=eps)
    return 1.0 / c if link == "inverse" else 1.0 / (c * c)


_ETA_CLIP = {"log": (-700.0, 700.0), "logit": (-700.0, 700.0), "inverse": (1e-8, float("inf")),
             "inverse_squared": (1e-8, float("inf")),
             "identity": (-float("inf"), float("inf"))}   # initialization.py:217-225
_SAFE_FILL = {"bernoulli": 0.5, "gaussian": 0.0}           # initialization.py:117-120, else 1.0


def fit_glm_batched(y, w, design, kind, alpha, offset=None, coef0=None, damping=1e-8,
                    max_iter=50, tol=1e-10, max_halvings=12, link="log"):
    """Batched penalized Fisher scoring for the m column GLMs of y (n x m) on a
    shared design (glm.py:68-133; lam = 0), all problems on the GPU at once:
    eta, the derivatives and the deviances are n x m device arrays, the m
    (p x p) Fisher systems one batched solve.  Returns (coef (m, p), converged)."""
    import torch
    n, m = y.shape
    p = design.shape[1]
    dev_ = y.device
    if p == 0:
        return torch.zeros((m, 0), dtype=torch.float64, device=dev_), torch.ones(m, dtype=torch.bool, device=dev_)
    off = torch.zeros_like(y) if offset is None else offset
    coef = torch.zeros((m, p), dtype=torch.float64, device=dev_) if coef0 is None else coef0.clone()
    eye = damping * torch.eye(p, dtype=torch.float64, device=dev_)
    keep = w > 0

    def deviance(c):
        return _batched_deviance(kind, alpha, y, w, design @ c.T + off, link)

    dev = deviance(coef)
    active = torch.ones(m, dtype=torch.bool, device=dev_)
    converged = torch.zeros(m, dtype=torch.bool, device=dev_)
    for _ in range(max_iter):
        eta = design @ coef.T + off
        dotd, ddotd = _derivs(kind, alpha, y, eta, w, link)
        dotd = torch.where(keep, dotd, torch.zeros_like(dotd))
        ddotd = torch.where(keep, ddotd, torch.zeros_like(ddotd))
        grad = dotd.T @ design
        hess = torch.einsum("ip,ij,iq->jpq", design, ddotd, design) + eye
        delta = -torch.linalg.solve(hess, grad[:, :, None])[:, :, 0]
        delta[~active] = 0.0
        step = torch.ones(m, dtype=torch.float64, device=dev_)
        cand = coef + step[:, None] * delta
        dev_new = deviance(cand)
        for _ in range(max_halvings):
            bad = active & (~torch.isfinite(dev_new) | (dev_new > dev + 1e-8))
            if not bool(bad.any()):
                break
            step = torch.where(bad, step * 0.5, step)
            cand = torch.where(bad[:, None], coef + step[:, None] * delta, cand)
            dev_new = torch.where(bad, deviance(cand), dev_new)
        still_bad = active & ~torch.isfinite(dev_new)
        if bool(still_bad.any()):
            cand = torch.where(still_bad[:, None], coef, cand)
            dev_new = torch.where(still_bad, dev, dev_new)
            active = active & ~still_bad
        moved = (cand - coef).abs().amax(1)
        scale = 1.0 + coef.abs().amax(1)
        coef = cand
        done = active & (moved < tol * scale)
        converged = converged | done
        active = active & ~done
        dev = torch.where(torch.isfinite(dev_new), dev_new, dev)
        if not bool(active.any()):
            break
    return coef, converged


def _ols_stage_dense(y_eps, w, design, offset):
    """One exact Gaussian/identity Fisher step (initialization.py:137-141)."""
    import torch
    p = design.shape[1]
    if p == 0:
        return torch.zeros((y_eps.shape[1], 0), dtype=torch.float64, device=y_eps.device)
    r = y_eps - (0.0 if offset is None else offset)
    grad = -(w * r).T @ design
    hess = torch.einsum("ip,ij,iq->jpq", design, w, design) + \
        _DAMPING * torch.eye(p, dtype=torch.float64, device=y_eps.device)
    return -torch.linalg.solve(hess, grad[:, :, None])[:, :, 0]


def _glm_or_fallback(y, w, design, kind, alpha, offset, coef_fallback, info, label, link="log"):
    """initialization.py:123-134: non-converged problems keep the OLS seed."""
    import torch
    coef, conv = fit_glm_batched(y, w, design, kind, alpha, offset=offset, coef0=coef_fallback,
                                 link=link)
    bad = ~conv
    if bool(bad.any()):
        coef = torch.where(bad[:, None], coef_fallback, coef)
        info.setdefault("glm_fallbacks", {})[label] = int(bad.sum().item())
    return coef


def randomized_svd_dense(a, k, oversample=10, n_power=2, seed=0):
    """randomized_svd (initialization.py:62-82) of a dense device matrix, the
    reference's probe replayed from numpy's generator."""
    import torch
    n, m = a.shape
    k = min(k, min(n, m))
    dev_ = a.device
    if k == 0:
        z = lambda *s: torch.zeros(s, dtype=torch.float64, device=dev_)
        return z(n, 0), z(0), z(m, 0)
    if k + oversample >= min(n, m):
        u, s, vt = torch.linalg.svd(a, full_matrices=False)
        return u[:, :k], s[:k], vt[:k].T
    rng = np.random.default_rng(seed)
    probe = torch.from_numpy(rng.standard_normal((m, k + oversample))).to(dev_)
    sketch = a @ probe
    for _ in range(n_power):
        q, _ = torch.linalg.qr(sketch)
        sketch = a @ (a.T @ q)
    q, _ = torch.linalg.qr(sketch)
    u_small, s, vt = torch.linalg.svd(q.T @ a, full_matrices=False)
    return (q @ u_small)[:, :k], s[:k], vt[:k].T


def init_glm_svd(data: ResponseMatrix, covs: CovariateSet, fam, lnk, d: int,
                 method: InitMethod | None = None, seed: int = 0, return_info: bool = False,
                 *, device=None):
    """GLM-based initialization (initialization.py:172-214) on the GPU: column
    GLMs for B, row GLMs for Gamma given the column effects, the deviance (or
    Pearson) residual SVD for U, column GLMs on U for V -- every batched GLM a
    set of n x m device arrays and one batched (p x p) solve per Fisher step;
    non-converged problems fall back to their OLS seeds as in the reference.
    Handles unobserved entries and prior weights (zero weight at holes), every
    family and link of the reference, and the Pearson start of phi for the
    free-dispersion families (initialization.py:85-90); returns a host state."""
    import torch
    method = method or InitMethod()
    n, m = data.shape
    if d > min(n, m):
        raise ConfigError("rank d cannot exceed min(n, m)")
    _lib.require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else
                       int(str(device).split(":")[-1]))
    kind, link = fam.kind, lnk.kind
    alpha = float(getattr(fam, "nb_shape", 1.0))
    eps = method.eps_for(lnk)
    Y, mask, W = _dense_inputs(data, dev)
    y_safe = torch.where(mask, Y, torch.full_like(Y, _SAFE_FILL.get(kind, 1.0)))   # _safe_y
    y_eps = _perturbed_transform(link, y_safe, eps)
    X = torch.from_numpy(np.ascontiguousarray(covs.x, dtype=float)).to(dev)
    Z = torch.from_numpy(np.ascontiguousarray(covs.z, dtype=float)).to(dev)
    p, q = X.shape[1], Z.shape[1]
    info = {"method": "glm_svd"}

    # stage 1: column regressions for B
    b = _ols_stage_dense(y_eps, W, X, None)
    if p:
        b = _glm_or_fallback(y_safe, W, X, kind, alpha, None, b, info, "b", link)
    offset = X @ b.T
    # stage 2: row regressions for Gamma given the column effects
    gamma = _ols_stage_dense(y_eps.T, W.T, Z, offset.T)
    if q:
        gamma = _glm_or_fallback(y_safe.T.contiguous(), W.T.contiguous(), Z, kind, alpha,
                                 offset.T.contiguous(), gamma, info, "gamma", link)
    eta0 = offset + (gamma @ Z.T if q else 0.0)
    mu0 = _mean(link, torch.clamp(eta0, *_ETA_CLIP[link]))
    # stage 3: residual SVD for the latent scores (initialization.py:103-114)
    if method.residual_kind == "pearson":
        r = (Y - mu0) * torch.sqrt(W / _variance(kind, alpha, mu0))
    else:
        ud = W * _dev0(kind, alpha, Y, mu0)
        r = torch.sign(Y - mu0) * torch.sqrt(torch.clamp(ud, min=0.0))
    resid = torch.where(mask, r, torch.zeros_like(r))
    left, sing, right = randomized_svd_dense(resid, d, seed=seed)
    u = left * sing
    # stage 4: column regressions for V with U as the design
    if d > 0:
        v0 = _ols_stage_dense(torch.where(mask, y_eps - eta0, torch.zeros_like(Y)), W, u, None)
        v = _glm_or_fallback(y_safe, W, u, kind, alpha, eta0, v0, info, "v", link)
    else:
        v = torch.zeros((m, 0), dtype=torch.float64, device=dev)
    nb_shape = 1.0
    if kind == "neg_binomial":      # initialization.py:93-100 at mu0
        num = float((torch.where(mask, W * mu0 ** 2, torch.zeros_like(Y))).sum().item())
        den = float((torch.where(mask, W * ((Y - mu0) ** 2 - mu0), torch.zeros_like(Y))).sum().item())
        nb_shape = 1e8 if den <= 0 else float(np.clip(num / den, 1e-4, 1e8))
    phi = 1.0
    if fam.has_free_dispersion:     # initialization.py:85-90 at mu0
        r2 = torch.where(mask, W * (Y - mu0) ** 2 / _variance(kind, alpha, mu0), torch.zeros_like(Y))
        dof = max(int(mask.sum().item()) - (p * m + q * n + (n + m) * d + 1), 1)
        phi = float(r2.sum().item()) / dof
    host = lambda t: t.cpu().numpy()
    state = FactorizationState(host(b), host(gamma), host(u), host(v), phi, nb_shape)
    return (state, info) if return_info else state
