"""(A) + (B1)/(B2)/(B3) identifiability projection on the device
(gmfkit/identify.py:59-138).

O(n d^2) work -- Gram matrices and design cross products over the n rows,
and applying small transforms to every row -- runs in the C ABI
(gmf_cross_rows / gmf_rows_affine, fp64 accumulation).  The p x p solves,
the d x d factorizations and the m x d column side (V, small) are host
linear algebra, exactly the scale at which the reference uses LAPACK
(identify.py:29-45).  U's thin QR is CholeskyQR2 on the device Gram matrix,
with an eigen pseudo-inverse for numerically rank-deficient U.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .exceptions import ConfigError, SingularSystemError

_SIGN_EPS = 1e-12


class _Dev:
    """Row-side device arrays of a projection problem."""

    def __init__(self, torch, device, tdt, theta_row, theta_col, x, z, p, q, d):
        self.torch, self.device, self.tdt = torch, device, tdt
        self.theta_row, self.theta_col, self.x, self.z = theta_row, theta_col, x, z
        self.p, self.q, self.d = p, q, d
        self.dt = _lib.F64 if tdt == torch.float64 else _lib.F32
        self.lib = _lib.lib()

    def stream(self):
        return C.c_void_p(self.torch.cuda.current_stream(self.device).cuda_stream)

    def cross(self, A, a0, a, B, b0, b):
        """A[:, a0:a0+a]' B[:, b0:b0+b] over all rows (fp64)."""
        torch = self.torch
        rows = A.shape[0]
        out = torch.zeros(a * b, device=self.device, dtype=torch.float64)
        if rows == 0 or a == 0 or b == 0:
            return np.zeros((a, b))
        work = torch.empty(int(self.lib.gmf_cross_work_bytes(a, b)), device=self.device,
                           dtype=torch.uint8)
        _lib.check(self.lib.gmf_cross_rows(self.dt, rows, _lib.ptr(A), A.shape[1], a0, a,
                                           _lib.ptr(B), B.shape[1], b0, b, _lib.ptr(out),
                                           _lib.ptr(work), self.stream()), "gmf_cross_rows")
        return out.cpu().numpy().reshape(a, b)

    def affine(self, Y, y0, c, beta, A, a0, a, M):
        """Y[:, y0:y0+c] <- beta Y[:, y0:y0+c] + A[:, a0:a0+a] @ M."""
        if Y.shape[0] == 0 or c == 0:
            return
        Mt = self.torch.as_tensor(np.ascontiguousarray(M, dtype=np.float64).reshape(a, c),
                                  device=self.device)
        _lib.check(self.lib.gmf_rows_affine(self.dt, Y.shape[0], _lib.ptr(Y), Y.shape[1], y0, c,
                                            float(beta), _lib.ptr(A), A.shape[1] if A.dim() > 1 else 1,
                                            a0, a, _lib.ptr(Mt), self.stream()), "gmf_rows_affine")


def _solve(gram, rhs, what):
    try:
        return np.linalg.solve(gram, rhs)
    except np.linalg.LinAlgError:
        raise SingularSystemError(
            f"rank-deficient design while removing the covariate span from {what}") from None


def _eig_factor(G, n, m):
    """R with R'R = G (rows of dropped directions zero) and its pseudo-inverse."""
    lam, E = np.linalg.eigh(G)
    lmax = max(lam.max(), 0.0)
    keep = lam > max(n, m) * np.finfo(float).eps * lmax
    s = np.zeros_like(lam)
    s[keep] = np.sqrt(lam[keep])
    inv = np.zeros_like(lam)
    inv[keep] = 1.0 / s[keep]
    return (E * s).T, E * inv


def _u_factor(dev: _Dev, n, m):
    """(R_U, P) with U_orig = Q R_U, where P is the d x d map that, applied to
    the CURRENT device U, yields Q (CholeskyQR2; eigen fallback)."""
    q, d = dev.q, dev.d
    G = dev.cross(dev.theta_row, q, d, dev.theta_row, q, d)
    G = 0.5 * (G + G.T)
    try:
        L1 = np.linalg.cholesky(G)
        dg = np.diag(L1)
        if dg.min() <= 1e-7 * dg.max():
            raise np.linalg.LinAlgError
    except np.linalg.LinAlgError:
        return _eig_factor(G, n, m)       # device U untouched
    # CholeskyQR2: Q1 = U R1^-1 on the device, then R2 from Q1'Q1
    R1 = L1.T
    dev.affine(dev.theta_row, q, d, 0.0, dev.theta_row, q, d, np.linalg.inv(R1))
    # from here on the device holds Q1: every factor is taken of Q1 itself
    G2 = dev.cross(dev.theta_row, q, d, dev.theta_row, q, d)
    G2 = 0.5 * (G2 + G2.T)
    try:
        R2 = np.linalg.cholesky(G2).T
        P2 = np.linalg.inv(R2)
    except np.linalg.LinAlgError:
        R2, P2 = _eig_factor(G2, n, m)
    return R2 @ R1, P2


def project_on_device(dev: _Dev, n, m, mode="B1"):
    """In-place projection of the device state; returns the info dict."""
    mode = mode.upper()
    if mode not in ("B1", "B2", "B3"):
        raise ConfigError(f"unknown identifiability mode {mode!r}")
    p, q, d = dev.p, dev.q, dev.d
    info = {"mode": mode, "effective_rank": d, "rank_deficient": False}
    tr, tc, x, z = dev.theta_row, dev.theta_col, dev.x, dev.z
    # ---- (A) identify.py:78-89 ----
    if p:
        xtx = dev.cross(x, 0, p, x, 0, p)
    if q:
        ztz = dev.cross(z, 0, q, z, 0, q)
    if p and q:
        dg = _solve(xtx, dev.cross(x, 0, p, tr, 0, q), "Gamma")        # (p, q)
        dev.affine(tr, 0, q, 1.0, x, 0, p, -dg)                          # Gamma -= X D
        dev.affine(tc, 0, p, 1.0, z, 0, q, dg.T)                         # B += Z D'
    if p and d:
        du = _solve(xtx, dev.cross(x, 0, p, tr, q, d), "U")            # (p, d)
        dev.affine(tr, q, d, 1.0, x, 0, p, -du)                          # U -= X D
        dev.affine(tc, 0, p, 1.0, tc, p, d, du.T)                        # B += V D'
    if q and d:
        dv = _solve(ztz, dev.cross(z, 0, q, tc, p, d), "V")            # (q, d)
        dev.affine(tc, p, d, 1.0, z, 0, q, -dv)                          # V -= Z D
        dev.affine(tr, 0, q, 1.0, tr, q, d, dv.T)                        # Gamma += U D'
    if d == 0:
        return info
    if mode == "B3":
        _b3(dev, info)
        return info
    # ---- B1/B2 thin-QR SVD of U V' (identify.py:40-45, 93-110) ----
    v = tc[:, p:].double().cpu().numpy()
    R_u, Rpinv = _u_factor(dev, n, m)
    qv, rv = np.linalg.qr(v)
    cu, sig, cvt = np.linalg.svd(R_u @ rv.T)
    cut = max(n, m) * np.finfo(float).eps * (sig[0] if sig.size else 0.0)
    eff = int(np.sum(sig > cut))
    if eff < d:
        sig = np.where(sig > cut, sig, 0.0)
        info["effective_rank"] = eff
        info["rank_deficient"] = True
    right = qv @ cvt.T
    Mu = Rpinv @ cu                               # U_cur @ Mu = left factor
    if mode == "B1":
        Mu = Mu * sig
        v_new = right
    else:
        v_new = right * sig
    # sign rule on V's columns (identify.py:48-56), applied to both factors
    signs = np.ones(d)
    for k in range(d):
        col = v_new[:, k]
        nz = np.flatnonzero(np.abs(col) > _SIGN_EPS)
        if nz.size and col[nz[0]] < 0:
            signs[k] = -1.0
    Mu = Mu * signs
    v_new = v_new * signs
    if info["rank_deficient"]:
        Mu[:, eff:] = 0.0
        v_new[:, eff:] = 0.0
    dev.affine(tr, q, d, 0.0, tr, q, d, Mu)
    tc[:, p:] = dev.torch.as_tensor(v_new, device=dev.device, dtype=dev.tdt)
    return info


def _b3(dev: _Dev, info):
    """B3 (identify.py:111-135): whiten U's column covariance, then rotate so
    V's leading d x d block is lower triangular with a positive diagonal.
    Column sums and the Gram matrix of U come from the device (fixed-order
    fp64); the d x d algebra and V (m x d) are host work; U is updated by one
    row-local affine map U <- U S^{-1/2} Q diag(signs)."""
    torch, tr, tc, p, q, d = dev.torch, dev.theta_row, dev.theta_col, dev.p, dev.q, dev.d
    rows = tr.shape[0]
    ones = torch.ones((rows, 1), device=dev.device, dtype=dev.tdt)
    mean = dev.cross(ones, 0, 1, tr, q, d) / rows                      # (1, d)
    G = dev.cross(tr, q, d, tr, q, d)
    S = (G - rows * mean.T @ mean) / rows
    S = 0.5 * (S + S.T)
    try:
        evals, evecs = np.linalg.eigh(S)
    except np.linalg.LinAlgError:
        raise SingularSystemError("whitening of U failed") from None
    if evals.min() <= rows * np.finfo(float).eps * max(evals.max(), 1.0):
        info["rank_deficient"] = True
        info["effective_rank"] = int(np.sum(evals > 0))
        raise SingularSystemError("U has a degenerate column covariance; B3 whitening undefined")
    s_inv_half = evecs @ np.diag(evals ** -0.5) @ evecs.T
    s_half = evecs @ np.diag(evals ** 0.5) @ evecs.T
    v = tc[:, p:].double().cpu().numpy() @ s_half
    q_rot, r = np.linalg.qr(v.T)
    v_new = r.T
    signs = np.sign(np.diag(v_new[:d, :d]))
    signs[signs == 0] = 1.0
    dev.affine(tr, q, d, 0.0, tr, q, d, (s_inv_half @ q_rot) * signs)
    tc[:, p:] = torch.as_tensor(v_new * signs, device=dev.device, dtype=dev.tdt)


def project_constraints(state, covs, mode="B1", return_info=False, dtype="f64", device=None):
    """Drop-in for gmfkit.identify.project_constraints on a host state."""
    import torch
    from .model import FactorizationState
    mode_u = mode.upper()
    if mode_u not in ("B1", "B2", "B3"):
        raise ConfigError(f"unknown identifiability mode {mode!r}")
    _lib.require_cuda()
    dev_t = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    tdt = torch.float64 if dtype == "f64" else torch.float32
    p, q, d = covs.p, covs.q, state.rank
    up = lambda a: torch.as_tensor(np.ascontiguousarray(a), device=dev_t, dtype=tdt)
    tr = up(np.hstack([state.gamma, state.u]))
    tc = up(np.hstack([state.b, state.v]))
    dev = _Dev(torch, dev_t, tdt, tr, tc, up(covs.x), up(covs.z), p, q, d)
    info = project_on_device(dev, state.n, state.m, mode_u)
    trh = tr.double().cpu().numpy()
    tch = tc.double().cpu().numpy()
    out = FactorizationState(tch[:, :p].copy(), trh[:, :q].copy(), trh[:, q:].copy(),
                             tch[:, p:].copy(), state.phi, state.nb_shape)
    return (out, info) if return_info else out


def check_constraints(state, covs, mode="B1") -> dict:
    """Max absolute violations of (A) and the normalization (identify.py:141-188)."""
    mode = mode.upper()
    x, z, d = covs.x, covs.z, state.rank

    def mx(a):
        return float(np.abs(a).max()) if a.size else 0.0

    rep = {"xt_gamma": mx(x.T @ state.gamma), "xt_u": mx(x.T @ state.u), "zt_v": mx(z.T @ state.v)}
    if d == 0:
        rep["normalization"] = 0.0
        return rep
    utu, vtv = state.u.T @ state.u, state.v.T @ state.v
    off = ~np.eye(d, dtype=bool)
    if mode == "B1":
        a, b, nm = vtv, utu, ("v_orthonormality", "u_off_diagonal")
    elif mode == "B2":
        a, b, nm = utu, vtv, ("u_orthonormality", "v_off_diagonal")
    elif mode == "B3":
        n = state.n
        mean = state.u.mean(axis=0, keepdims=True)
        rep["u_standardized"] = mx((utu - n * mean.T @ mean) / n - np.eye(d))
        top = state.v[:d, :d]
        rep["v_upper_triangle"] = mx(top[np.triu_indices(d, k=1)]) if d > 1 else 0.0
        rep["v_diag_positive"] = float(max(0.0, -np.min(np.diag(top))))
        rep["normalization"] = max(rep["u_standardized"], rep["v_upper_triangle"],
                                   rep["v_diag_positive"])
        return rep
    else:
        raise ConfigError(f"unknown identifiability mode {mode!r}")
    rep[nm[0]] = mx(a - np.eye(d))
    rep[nm[1]] = mx(b[off])
    rep["sigma_sorted"] = float(max(0.0, np.max(np.diff(np.diag(b)), initial=0.0)))
    rep["normalization"] = max(rep[nm[0]], rep[nm[1]], rep["sigma_sorted"])
    return rep
