"""CPU oracle for the aSGD hot path -- TEST INFRASTRUCTURE ONLY.

This module is the parity checker for the CUDA path in
``paper_2412_20509_b200``.  It is a plain-numpy restatement of the
reference (`gmfkit`, /root/reference/pkg/src/gmfkit) algorithm for the
hot path named in BASELINE.json: the block-wise adaptive SGD step, the
stochastic negative-binomial shape update, the tracked objective, and the
(A)+(B1) identifiability projection.  Every function cites the reference
file:line it restates.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg (``--impl reference`` / ``cpu_baseline``) may import this module.  The
product path never calls it; the package fails loudly without its CUDA
library instead.

Parity of this restatement is PINNED against golden vectors produced by
running the reference itself (tests/golden/make_golden.py imports gmfkit
from /root/reference and writes tests/golden/*.npz); see
tests/test_oracle_golden.py.

Extension over the reference: an optional per-row
``offset`` enters the linear predictor, eta = offset_i + x_i.b_j +
gamma_i.z_j + u_i.v_j.  With ``offset=None`` the oracle is exactly the
reference model.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# family / link integer codes: gmfkit/kernels/_ref.py:15-16
GAUSSIAN, GAMMA, INV_GAUSSIAN, POISSON, BERNOULLI, NEG_BINOMIAL = range(6)
IDENTITY, LOG, LOGIT, INVERSE, INVERSE_SQUARED = range(5)
FAMILY_CODES = {"gaussian": GAUSSIAN, "gamma": GAMMA, "inverse_gaussian": INV_GAUSSIAN,
                "poisson": POISSON, "bernoulli": BERNOULLI, "neg_binomial": NEG_BINOMIAL}
LINK_CODES = {"identity": IDENTITY, "log": LOG, "logit": LOGIT, "inverse": INVERSE,
              "inverse_squared": INVERSE_SQUARED}

NB_SHAPE_FLOOR = 1e-4     # gmfkit/optim.py:57
NB_SHAPE_CEILING = 1e8    # gmfkit/optim.py:58
SNAPSHOT_STRIDE = 4       # gmfkit/optim.py:309
BERNOULLI_EPS = 1e-10     # gmfkit/kernels/_ref.py:18


class OracleDivergence(ArithmeticError):
    """Non-finite tracked objective (gmfkit/optim.py:319-331)."""

    def __init__(self, msg, state=None):
        super().__init__(msg)
        self.state = state


# ---------------------------------------------------------------------------
# scalar schedule (gmfkit/optim.py:130-148)
# ---------------------------------------------------------------------------

def learning_rate(t, k0, k1, tau):
    """rho_t = k0 / (1 + k0 k1 t)^tau  -- optim.py:130-134."""
    return k0 / (1.0 + k0 * k1 * t) ** tau


def bias_correction(t, a1, a2):
    """(1 - a2^t)/(1 - a1^t), 1 when a1 == a2 -- optim.py:142-148."""
    if a1 == a2:
        return 1.0
    return (1.0 - a2 ** t) / (1.0 - a1 ** t)


# ---------------------------------------------------------------------------
# per-entry algebra (gmfkit/kernels/_ref.py:21-108, _core.pyx:58-111)
# ---------------------------------------------------------------------------

def mean_of_eta(lcode, eta):
    """Inverse link -- kernels/_ref.py:21-32."""
    if lcode == IDENTITY:
        return np.array(eta, dtype=float)
    if lcode == LOG:
        return np.exp(eta)
    if lcode == LOGIT:
        return 1.0 / (1.0 + np.exp(-eta))
    if lcode == INVERSE:
        return 1.0 / eta
    if lcode == INVERSE_SQUARED:
        return 1.0 / np.sqrt(eta)
    raise ValueError(lcode)


def _variance(fcode, mu, alpha):
    # kernels/_ref.py:35-48
    return {GAUSSIAN: lambda: np.ones_like(mu), GAMMA: lambda: mu * mu,
            INV_GAUSSIAN: lambda: mu ** 3, POISSON: lambda: mu,
            BERNOULLI: lambda: mu * (1.0 - mu),
            NEG_BINOMIAL: lambda: mu * (1.0 + mu / alpha)}[fcode]()


def _link_d1(lcode, mu):
    # kernels/_ref.py:51-62
    return {IDENTITY: lambda: np.ones_like(mu), LOG: lambda: 1.0 / mu,
            LOGIT: lambda: 1.0 / (mu * (1.0 - mu)), INVERSE: lambda: -1.0 / (mu * mu),
            INVERSE_SQUARED: lambda: -2.0 / mu ** 3}[lcode]()


def derivs_from_mu(fcode, lcode, y, mu, w, phi, alpha):
    """(dotD, ddotD Fisher) -- kernels/_ref.py:65-88 (canonical shortcuts 71-85)."""
    r = y - mu
    if fcode == POISSON and lcode == LOG:
        return -w * r / phi, w * mu / phi
    if fcode == NEG_BINOMIAL and lcode == LOG:
        den = 1.0 + mu / alpha
        return -w * r / (phi * den), w * mu / (phi * den)
    if fcode == BERNOULLI and lcode == LOGIT:
        return -w * r / phi, w * mu * (1.0 - mu) / phi
    if fcode == GAUSSIAN and lcode == IDENTITY:
        return -w * r / phi, w / phi * np.ones_like(mu)
    if fcode == GAMMA and lcode == INVERSE:
        return w * r / phi, w * mu * mu / phi
    if fcode == INV_GAUSSIAN and lcode == INVERSE_SQUARED:
        return w * r / (2.0 * phi), w * mu ** 3 / (4.0 * phi)
    nu = _variance(fcode, mu, alpha)
    g1 = _link_d1(lcode, mu)
    return -w * r / (phi * nu * g1), w / (phi * nu * g1 * g1)


def _xlogy_ratio(y, mu):
    """y * log(y / mu) with the 0 * log 0 = 0 convention of scipy xlogy."""
    y = np.asarray(y, dtype=float)
    out = np.zeros(np.broadcast(y, mu).shape)
    pos = np.broadcast_to(y != 0, out.shape)
    yb = np.broadcast_to(y, out.shape)
    mb = np.broadcast_to(mu, out.shape)
    out[pos] = yb[pos] * np.log(yb[pos] / mb[pos])
    return out


def unit_deviance(fcode, y, mu, alpha):
    """Unit deviance D(y, mu) -- kernels/_ref.py:91-108."""
    if fcode == POISSON:
        return 2.0 * (_xlogy_ratio(y, mu) - (y - mu))
    if fcode == NEG_BINOMIAL:
        return 2.0 * (_xlogy_ratio(y, mu) - (y + alpha) * np.log1p((y - mu) / (mu + alpha)))
    if fcode == GAUSSIAN:
        return (y - mu) ** 2
    if fcode == GAMMA:
        return 2.0 * ((y - mu) / mu - np.log(y / mu))
    if fcode == INV_GAUSSIAN:
        return (y - mu) ** 2 / (y * mu * mu)
    if fcode == BERNOULLI:
        mu = np.clip(mu, BERNOULLI_EPS, 1.0 - BERNOULLI_EPS)
        return 2.0 * (_xlogy_ratio(y, mu) + _xlogy_ratio(1.0 - y, 1.0 - mu))
    raise ValueError(fcode)


def deviance_from_mu(fcode, y, mu, w, alpha):
    """Sum of weighted unit deviances -- kernels/_ref.py:91-108."""
    return float(np.sum(w * unit_deviance(fcode, y, mu, alpha)))


# ---------------------------------------------------------------------------
# model algebra (gmfkit/model.py:229-283, gradients.py:91-132)
# ---------------------------------------------------------------------------

@dataclass
class OState:
    """Mirror of FactorizationState (model.py:139-190): b (m,p) gamma (n,q) u (n,d) v (m,d)."""
    b: np.ndarray
    gamma: np.ndarray
    u: np.ndarray
    v: np.ndarray
    phi: float = 1.0
    nb_shape: float = 1.0

    def copy(self):
        return OState(self.b.copy(), self.gamma.copy(), self.u.copy(), self.v.copy(),
                      self.phi, self.nb_shape)


class CsrRows:
    """Read-only CSR-backed response that indexes like the dense (n, m) float
    array the reference stores (model.py:46-98): ``y[I]`` densifies rows I,
    ``y[rows, cols]`` gathers entries.  Lets the oracle run configs whose dense
    matrix does not fit in host RAM (c4: 1.3M x 500) on exactly the same
    arithmetic, since every step only touches the drawn block's rows."""

    def __init__(self, indptr, indices, data, shape):
        self.indptr = np.asarray(indptr, dtype=np.int64)
        self.indices = np.asarray(indices, dtype=np.int64)
        self.data = np.asarray(data, dtype=np.float64)
        self.shape = (int(shape[0]), int(shape[1]))

    def __getitem__(self, key):
        if isinstance(key, tuple):
            rows, cols = (np.asarray(k, dtype=np.int64) for k in key)
            if not hasattr(self, "_keys"):   # row-major linear index of every nonzero
                r = np.repeat(np.arange(self.shape[0], dtype=np.int64), np.diff(self.indptr))
                self._keys = r * self.shape[1] + self.indices
            q = rows * self.shape[1] + cols
            pos = np.minimum(np.searchsorted(self._keys, q), max(self._keys.size - 1, 0))
            hit = (self._keys.size > 0) & (self._keys[pos] == q) if self._keys.size else np.zeros(q.size, bool)
            return np.where(hit, self.data[pos] if self._keys.size else 0.0, 0.0)
        rows = np.asarray(key, dtype=np.int64)
        out = np.zeros((rows.size, self.shape[1]))
        lo, hi = self.indptr[rows], self.indptr[rows + 1]
        lens = hi - lo
        r = np.repeat(np.arange(rows.size), lens)
        src = np.repeat(lo - np.concatenate([[0], np.cumsum(lens)[:-1]]), lens) + np.arange(lens.sum())
        out[r, self.indices[src]] = self.data[src]
        return out


@dataclass
class OProblem:
    """Dense fully observed response plus designs (model.py:46-136)."""
    y: np.ndarray                  # (n, m) float64
    x: np.ndarray                  # (n, p)
    z: np.ndarray                  # (m, q)
    w: np.ndarray | None = None    # (n, m) weights, None == ones
    offset: np.ndarray | None = None   # (n,) extension (SURVEY §8c shim)

    @property
    def n(self):
        return self.y.shape[0]

    @property
    def m(self):
        return self.y.shape[1]

    def weights(self, rows=None, cols=None):
        if self.w is None:
            shape = (self.n if rows is None else len(rows), self.m if cols is None else len(cols))
            return np.ones(shape)
        w = self.w if rows is None else self.w[rows]
        return w if cols is None else w[:, cols]


def linear_predictor(st: OState, pb: OProblem, rows=None, cols=None):
    """eta block, BLAS order UV' then XB' then GammaZ' -- model.py:229-256 (+offset)."""
    u = st.u if rows is None else st.u[rows]
    x = pb.x if rows is None else pb.x[rows]
    g = st.gamma if rows is None else st.gamma[rows]
    v = st.v if cols is None else st.v[cols]
    b = st.b if cols is None else st.b[cols]
    z = pb.z if cols is None else pb.z[cols]
    eta = u @ v.T
    if x.shape[1]:
        eta += x @ b.T
    if z.shape[1]:
        eta += g @ z.T
    if pb.offset is not None:
        off = pb.offset if rows is None else pb.offset[rows]
        eta += off[:, None]
    return eta


def penalty_value(st: OState, lam):
    """0.5 sum lam_X ||X||_F^2 over (B, Gamma, U, V) -- model.py:259-265."""
    lb, lg, lu, lv = lam
    return 0.5 * (lb * float(np.sum(st.b ** 2)) + lg * float(np.sum(st.gamma ** 2))
                  + lu * float(np.sum(st.u ** 2)) + lv * float(np.sum(st.v ** 2)))


def penalized_objective(st, pb, fcode, lcode, lam):
    """Full half-deviance / phi + penalty -- model.py:268-276."""
    if isinstance(pb.y, CsrRows):   # row chunks, same per-entry arithmetic
        dev = 0.0
        step = max(1, 2_000_000 // pb.m)
        for lo in range(0, pb.n, step):
            rows = np.arange(lo, min(pb.n, lo + step))
            mu = mean_of_eta(lcode, linear_predictor(st, pb, rows))
            dev += deviance_from_mu(fcode, pb.y[rows], mu, pb.weights(rows), st.nb_shape)
        return dev / (2.0 * st.phi) + penalty_value(st, lam)
    mu = mean_of_eta(lcode, linear_predictor(st, pb))
    dev = deviance_from_mu(fcode, pb.y, mu, pb.weights(), st.nb_shape)
    return dev / (2.0 * st.phi) + penalty_value(st, lam)


# ---------------------------------------------------------------------------
# model selection and held-out metrics (gmfkit/select.py, gmfkit/metrics.py)
# ---------------------------------------------------------------------------

def dispersion_constant(fcode, y, w, phi, alpha):
    """phi/alpha part of -2 log-likelihood beyond D/phi -- select.py:57-79."""
    from scipy.special import gammaln
    if fcode in (GAUSSIAN, INV_GAUSSIAN):
        return float(y.size * np.log(phi))
    if fcode == GAMMA:
        shape = w / phi
        return float(2.0 * np.sum(gammaln(shape) - shape * np.log(shape) + shape))
    if fcode == NEG_BINOMIAL:
        a = alpha
        sat = (gammaln(y + a) - gammaln(a) - gammaln(y + 1.0)
               - (y + a) * np.log(y + a) + a * np.log(a))
        ylogy = np.where(y > 0, y * np.log(np.where(y > 0, y, 1.0)), 0.0)
        return float(-2.0 * np.sum(w * (sat + ylogy)))
    return 0.0


def information_criteria(st, pb, fcode, lcode, alpha):
    """(AIC, BIC) = D/phi + c(phi) + (2 | log n_obs) k -- select.py:81-96
    (fully observed; k = pm + qn + d(n+m) + 1, model.py:279-283)."""
    mu = mean_of_eta(lcode, linear_predictor(st, pb))
    y, w = pb.y.ravel(), pb.weights().ravel()
    dev = float(np.sum(w * unit_deviance(fcode, y, mu.ravel(), alpha))) / st.phi
    dev += dispersion_constant(fcode, y, w, st.phi, alpha)
    n, m = pb.y.shape
    k = pb.x.shape[1] * m + pb.z.shape[1] * n + st.u.shape[1] * (n + m) + 1
    return dev + 2.0 * k, dev + k * np.log(n * m)


def mu_at(st, pb, lcode, rows, cols):
    """g^{-1}(eta) at listed entries -- select.py:141-145 (+ offset shim)."""
    eta = np.einsum("ik,ik->i", st.u[rows], st.v[cols])
    if pb.x.shape[1]:
        eta = eta + np.einsum("ik,ik->i", pb.x[rows], st.b[cols])
    if pb.z.shape[1]:
        eta = eta + np.einsum("ik,ik->i", st.gamma[rows], pb.z[cols])
    if pb.offset is not None:
        eta = eta + pb.offset[rows]
    return mean_of_eta(lcode, eta)


def rel_log_rmse(y, mu, ybar):
    """metrics.py:35-45."""
    num = np.sum(np.log((1.0 + y) / (1.0 + mu)) ** 2)
    den = np.sum(np.log((1.0 + y) / (1.0 + ybar)) ** 2)
    return float(num / den)


def rel_deviance(fcode, y, mu, ybar, alpha):
    """metrics.py:48-55 (unit weights)."""
    num = np.sum(unit_deviance(fcode, y, mu, alpha))
    den = np.sum(unit_deviance(fcode, y, np.full_like(y, float(ybar)), alpha))
    return float(num / den)


# ---------------------------------------------------------------------------
# OLS-SVD initialization (gmfkit/initialization.py:62-82, 93-100, 143-169)
# ---------------------------------------------------------------------------

def randomized_svd(a, k, oversample=10, n_power=2, seed=0):
    """Truncated SVD by a randomized range finder -- initialization.py:62-82."""
    n, m = a.shape
    k = min(k, min(n, m))
    if k == 0:
        return np.zeros((n, 0)), np.zeros(0), np.zeros((m, 0))
    if k + oversample >= min(n, m):
        u, s, vt = np.linalg.svd(a, full_matrices=False)
        return u[:, :k], s[:k], vt[:k].T
    rng = np.random.default_rng(seed)
    probe = rng.standard_normal((m, k + oversample))
    sketch = a @ probe
    for _ in range(n_power):
        q, _ = np.linalg.qr(sketch)
        sketch = a @ (a.T @ q)
    q, _ = np.linalg.qr(sketch)
    u_small, s, vt = np.linalg.svd(q.T @ a, full_matrices=False)
    return (q @ u_small)[:, :k], s[:k], vt[:k].T


def _ols(y, design, offset=None, damping=1e-8):
    """Single Gaussian/identity Fisher step from zero = damped least squares,
    per column of y -- glm.py:36-64 via initialization.py:136-140."""
    p = design.shape[1]
    if p == 0:
        return np.zeros((y.shape[1], 0))
    r = y if offset is None else y - offset
    return np.linalg.solve(design.T @ design + damping * np.eye(p), design.T @ r).T


def init_ols_svd(pb: OProblem, d, fcode, eps=0.1, seed=0):
    """Fully observed, unit-weight, log-link init_ols_svd -- initialization.py:143-169."""
    y_eps = np.log(pb.y + eps)
    b = _ols(y_eps, pb.x)
    offset = pb.x @ b.T
    gamma = _ols(y_eps.T, pb.z, offset.T)
    eta0 = offset + (gamma @ pb.z.T if pb.z.shape[1] else 0.0)
    left, sing, right = randomized_svd(y_eps - eta0, d, seed=seed)
    mu0 = np.exp(np.clip(eta0, -700.0, 700.0))
    nb = 1.0
    if fcode == NEG_BINOMIAL:
        num = float(np.sum(mu0 ** 2))
        den = float(np.sum((pb.y - mu0) ** 2 - mu0))
        nb = 1e8 if den <= 0 else float(np.clip(num / den, 1e-4, 1e8))
    return OState(b, gamma, left * sing, right, 1.0, nb)


def penalty_vectors(p, q, d, lam):
    """Per-coordinate ridge weights [Gamma,U] and [B,V] -- gradients.py:91-99."""
    lb, lg, lu, lv = lam
    return (np.concatenate([np.full(q, lg), np.full(d, lu)]),
            np.concatenate([np.full(p, lb), np.full(d, lv)]))


@dataclass
class OGrad:
    """Mirror of GradientPair (gradients.py:56-63)."""
    g_row: np.ndarray
    h_row: np.ndarray
    g_col: np.ndarray
    h_col: np.ndarray


def block_derivs(st, pb, I, J, fcode, lcode):
    """eta -> mu -> (dotD, ddotD) on the block I x J (optim.py:427-440)."""
    eta = linear_predictor(st, pb, I, J)
    mu = mean_of_eta(lcode, eta)
    y = pb.y[I][:, J]
    w = pb.weights(I, J)
    with np.errstate(all="ignore"):
        dd, hh = derivs_from_mu(fcode, lcode, y, mu, w, st.phi, st.nb_shape)
    return y, w, mu, dd, hh


def minibatch_gradients(st, pb, I, J, fcode, lcode, lam):
    """Unbiased block gradient / Fisher-diagonal estimates -- gradients.py:102-132."""
    n, m = pb.n, pb.m
    _, _, _, dd, hh = block_derivs(st, pb, I, J, fcode, lcode)
    a_row = np.hstack([pb.z[J], st.v[J]])
    a_col = np.hstack([pb.x[I], st.u[I]])
    th_row = np.hstack([st.gamma[I], st.u[I]])
    th_col = np.hstack([st.b[J], st.v[J]])
    lr, lc = penalty_vectors(pb.x.shape[1], pb.z.shape[1], st.u.shape[1], lam)
    s_row, s_col = m / len(J), n / len(I)
    return OGrad(s_row * (dd @ a_row) + lr * th_row,
                 s_row * (hh @ (a_row * a_row)) + lr,
                 s_col * (dd.T @ a_col) + lc * th_col,
                 s_col * (hh.T @ (a_col * a_col)) + lc)


def nb_moment_sums(y, mu, w):
    """(sum w mu^2, sum w((y-mu)^2 - mu)) -- optim.py:225-226."""
    return float(np.sum(w * mu ** 2)), float(np.sum(w * ((y - mu) ** 2 - mu)))


def pearson_phi_update(phi_bar, rho, y, mu, w, fcode, alpha, n, m, n_i, n_j, p, q, d):
    """Smoothed stochastic Pearson update of phi -- optim.py:175-202:
    phi_hat = sum_B w (y - mu)^2 / nu(mu) * (nm / n* m*) / N with
    N = nm - mp - nq - (n + m) d - 1 (optim.py:171-172, model.py:279-283)."""
    dof = n * m - (p * m + q * n + d * (n + m) + 1)
    if dof <= 0:
        raise ValueError("model is over-parameterized: nonpositive residual dof")
    with np.errstate(all="ignore"):
        s = float(np.sum(w * (y - mu) ** 2 / _variance(fcode, mu, alpha)))
    return (1.0 - rho) * phi_bar + rho * (s * (n * m) / (n_i * n_j) / dof)


def nb_shape_update(alpha_bar, rho, num, den, floor=NB_SHAPE_FLOOR, ceiling=NB_SHAPE_CEILING):
    """Smoothed moment update of the NB shape -- optim.py:205-229."""
    a_hat = num / den if den > 0 else ceiling
    a_hat = min(max(floor, a_hat), ceiling)
    return (1.0 - rho) * alpha_bar + rho * a_hat


# ---------------------------------------------------------------------------
# partitions, eval sample, tracked objective (optim.py:253-338)
# ---------------------------------------------------------------------------

def partition(rng, size, block):
    """Sorted near-equal chunks of a random permutation -- optim.py:253-257."""
    perm = rng.permutation(size)
    k = int(math.ceil(size / block))
    return [np.sort(c) for c in np.array_split(perm, k)]


def eval_entries_full(n, m, cap, rng):
    """_eval_entries for a fully observed n x m matrix -- optim.py:260-271.

    np.nonzero of an all-True mask enumerates row-major linear indices, so
    the chosen pairs are pick // m, pick % m with identical RNG consumption.
    """
    total = n * m
    if total <= cap:
        lin = np.arange(total)
        return lin // m, lin % m, 1.0
    pick = np.sort(rng.choice(total, size=cap, replace=False))
    return pick // m, pick % m, total / cap


def entrywise_eta(st, pb, rows, cols):
    """eta at (row, col) pairs -- optim.py:274-280 (+offset)."""
    eta = np.einsum("ik,ik->i", st.u[rows], st.v[cols])
    if pb.x.shape[1]:
        eta += np.einsum("ik,ik->i", pb.x[rows], st.b[cols])
    if pb.z.shape[1]:
        eta += np.einsum("ik,ik->i", st.gamma[rows], pb.z[cols])
    if pb.offset is not None:
        eta += pb.offset[rows]
    return eta


def tracked_objective(st, pb, fcode, lcode, lam, entries):
    """Sampled deviance (inflated) / (2 phi) + penalty -- optim.py:283-290."""
    rows, cols, scale = entries
    eta = entrywise_eta(st, pb, rows, cols)
    with np.errstate(all="ignore"):
        mu = mean_of_eta(lcode, eta)
        w = np.ones(rows.size) if pb.w is None else pb.w[rows, cols]
        dev = deviance_from_mu(fcode, pb.y[rows, cols], mu, w, st.nb_shape)
    return scale * dev / (2.0 * st.phi) + penalty_value(st, lam)


# ---------------------------------------------------------------------------
# (A) + (B1) identifiability projection (identify.py:29-110)
# ---------------------------------------------------------------------------

def _proj(design, target):
    # identify.py:29-37
    return np.linalg.solve(design.T @ design, design.T @ target)


def project_b1(st: OState, x, z):
    """(A) covariate-span removal, then thin-QR SVD with sign fix -- identify.py:59-110."""
    b, g, u, v = st.b.copy(), st.gamma.copy(), st.u.copy(), st.v.copy()
    p, q, d = x.shape[1], z.shape[1], u.shape[1]
    if p and q:
        dg = _proj(x, g)
        g -= x @ dg
        b += z @ dg.T
    if p and d:
        du = _proj(x, u)
        u -= x @ du
        b += v @ du.T
    if q and d:
        dv = _proj(z, v)
        v -= z @ dv
        g += u @ dv.T
    info = {"effective_rank": d, "rank_deficient": False}
    if d:
        qu, ru = np.linalg.qr(u)
        qv, rv = np.linalg.qr(v)
        cu, sig, cvt = np.linalg.svd(ru @ rv.T)
        left, right = qu @ cu, qv @ cvt.T
        cut = max(u.shape[0], v.shape[0]) * np.finfo(float).eps * (sig[0] if sig.size else 0.0)
        eff = int(np.sum(sig > cut))
        if eff < d:
            sig = np.where(sig > cut, sig, 0.0)
            info.update(effective_rank=eff, rank_deficient=True)
        u, v = left * sig, right
        for k in range(d):   # identify.py:48-56
            col = v[:, k]
            nz = np.flatnonzero(np.abs(col) > 1e-12)
            if nz.size and col[nz[0]] < 0:
                v[:, k] = -col
                u[:, k] = -u[:, k]
        if info["rank_deficient"]:
            u[:, eff:] = 0.0
            v[:, eff:] = 0.0
    return OState(b, g, u, v, st.phi, st.nb_shape), info


# ---------------------------------------------------------------------------
# the aSGD driver (optim.py:383-489)
# ---------------------------------------------------------------------------

@dataclass
class OConfig:
    """Mirror of SgdConfig defaults (optim.py:61-106)."""
    max_epochs: int = 500
    rate_k0: float = 0.01
    rate_k1: float = 0.01
    rate_tau: float = 0.75
    mb_rows: int = 100
    mb_cols: int = 20
    smooth_a1: float = 0.1
    smooth_a2: float = 0.01
    damping: float = 1e-3
    tol: float = 1e-5
    seed: int = 0
    max_eval_entries: int = 100_000


@dataclass
class OReport:
    final_objective: float = float("nan")
    objective_trace: list = field(default_factory=list)
    nb_shape_trace: list = field(default_factory=list)
    phi_trace: list = field(default_factory=list)
    epochs_run: int = 0
    converged: bool = False
    iterations: int = 0
    row_blocks: list = field(default_factory=list)
    col_blocks: list = field(default_factory=list)
    block_sequence: list = field(default_factory=list)


def replay_schedule(n, m, cfg: OConfig, n_steps=None):
    """Host RNG replay of (row_blocks, col_blocks, eval entries, I draws) -- optim.py:404-423."""
    rng = np.random.default_rng(cfg.seed)
    rb = partition(rng, n, min(cfg.mb_rows, n))
    cb = partition(rng, m, min(cfg.mb_cols, m))
    ent = eval_entries_full(n, m, cfg.max_eval_entries, rng)
    steps = cfg.max_epochs * len(cb) if n_steps is None else n_steps
    seq = [int(rng.integers(len(rb))) for _ in range(steps)]
    return rb, cb, ent, seq


def fit_asgd(pb: OProblem, fcode, lcode, lam, cfg: OConfig, init: OState, *,
             identify=True, est_alpha=None, est_phi=None, callback=None, final_objective=True):
    """Restatement of fit_asgd for fully observed data -- optim.py:383-489.

    ``est_alpha`` / ``est_phi`` default to the 'auto' policy (optim.py:156-168):
    NB estimates its shape, the free-dispersion families (Gaussian, Gamma,
    inverse Gaussian) estimate phi, Poisson and Bernoulli estimate nothing.
    """
    if est_alpha is None:
        est_alpha = fcode == NEG_BINOMIAL
    if est_phi is None:
        est_phi = fcode in (GAUSSIAN, GAMMA, INV_GAUSSIAN)
    st = init.copy()
    n, m = pb.n, pb.m
    p, q, d = pb.x.shape[1], pb.z.shape[1], st.u.shape[1]
    rng = np.random.default_rng(cfg.seed)
    rb = partition(rng, n, min(cfg.mb_rows, n))
    cb = partition(rng, m, min(cfg.mb_cols, m))
    ent = eval_entries_full(n, m, cfg.max_eval_entries, rng)
    lr, lc = penalty_vectors(p, q, d, lam)
    gbr, hbr = np.zeros((n, q + d)), np.zeros((n, q + d))
    gbc, hbc = np.zeros((m, p + d)), np.zeros((m, p + d))
    rep = OReport(row_blocks=rb, col_blocks=cb)
    obj0 = tracked_objective(st, pb, fcode, lcode, lam, ent)
    rep.objective_trace.append(obj0)
    rep.nb_shape_trace.append(st.nb_shape)
    rep.phi_trace.append(st.phi)
    snapshot = st.copy()
    if not np.isfinite(obj0):
        raise OracleDivergence("objective is non-finite at the initial state")
    a1, a2 = cfg.smooth_a1, cfg.smooth_a2
    t, streak = 0, 0
    for epoch in range(cfg.max_epochs):
        for J in cb:
            bi = int(rng.integers(len(rb)))
            I = rb[bi]
            rep.block_sequence.append(bi)
            rho = learning_rate(t, cfg.rate_k0, cfg.rate_k1, cfg.rate_tau)
            alpha_t = bias_correction(t + 1, a1, a2)
            y, w, mu, dd, hh = block_derivs(st, pb, I, J, fcode, lcode)
            a_row = np.hstack([pb.z[J], st.v[J]])
            a_col = np.hstack([pb.x[I], st.u[I]])
            th_row = np.hstack([st.gamma[I], st.u[I]])
            th_col = np.hstack([st.b[J], st.v[J]])
            s_row, s_col = m / len(J), n / len(I)
            g_row = s_row * (dd @ a_row) + lr * th_row
            h_row = s_row * (hh @ (a_row * a_row)) + lr
            g_col = s_col * (dd.T @ a_col) + lc * th_col
            h_col = s_col * (hh.T @ (a_col * a_col)) + lc
            gbc[J] = (1 - a1) * gbc[J] + a1 * g_col
            hbc[J] = (1 - a2) * hbc[J] + a2 * h_col
            gbr[I] = (1 - a1) * gbr[I] + a1 * g_row
            hbr[I] = (1 - a2) * hbr[I] + a2 * h_row
            dc = -alpha_t * gbc[J] / (hbc[J] + cfg.damping)
            st.b[J] += rho * dc[:, :p]
            st.v[J] += rho * dc[:, p:]
            dr = -alpha_t * gbr[I] / (hbr[I] + cfg.damping)
            st.gamma[I] += rho * dr[:, :q]
            st.u[I] += rho * dr[:, q:]
            if est_phi:
                st.phi = pearson_phi_update(st.phi, rho, y, mu, w, fcode, st.nb_shape, n, m,
                                            len(I), len(J), p, q, d)
            if est_alpha:
                num, den = nb_moment_sums(y, mu, w)
                st.nb_shape = nb_shape_update(st.nb_shape, rho, num, den)
            if callback is not None:
                callback(t, st)
            t += 1
        rep.epochs_run = epoch + 1
        obj = tracked_objective(st, pb, fcode, lcode, lam, ent)
        prev = rep.objective_trace[-1]
        rep.objective_trace.append(obj)
        rep.nb_shape_trace.append(st.nb_shape)
        rep.phi_trace.append(st.phi)
        if not np.isfinite(obj):
            raise OracleDivergence("objective became non-finite", state=snapshot)
        if len(rep.objective_trace) % SNAPSHOT_STRIDE == 0:
            snapshot = st.copy()
        rel = abs(obj - prev) / (abs(prev) + 1e-12)
        streak = streak + 1 if rel < cfg.tol else 0
        if streak >= 2:
            rep.converged = True
            break
    rep.iterations = t
    final = project_b1(st, pb.x, pb.z)[0] if identify else st.copy()
    if final_objective:
        rep.final_objective = penalized_objective(final, pb, fcode, lcode, lam)
    return final, rep
