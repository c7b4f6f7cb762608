"""Seeded synthetic inputs standing in for BASELINE.json configs c1-c5.

The paper's datasets (Arigoni 26,472x500; TENxBrainData 1.23M x 500) are
not available here; these generators reproduce the SHAPES and value
distributions BASELINE.json names, never their contents.

Counts are drawn as Poisson or as the Gamma-Poisson negative binomial with
per-gene dispersion phi_j (lambda ~ Gamma(phi_j, mu/phi_j),
y ~ Poisson(lambda)).  The gene-intercept mean is calibrated analytically
(expected zero fraction, bisection) to hit the stated sparsity.

Large configs (c3/c4) can draw the counts on a CUDA device through torch's
RNG (input generation is benchmark plumbing, not the measured path); the
host generator is used for every parity case.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class WorkloadSpec:
    name: str
    n: int
    m: int
    d: int
    family: str            # "poisson" | "neg_binomial"
    dtype: str             # "f32" | "f64"
    y_format: str          # "dense" | "csr"
    mb_rows: int
    epochs: int
    p: int = 1             # X = [1, batch...]
    q: int = 0             # Z = ones when q == 1
    offset: bool = False
    groups: int = 1
    u_sd: float = 0.5
    v_sd: float = 0.5
    zero_frac: float | None = None   # calibrate intercept mean to this
    b_mean: float = 1.0
    b_sd: float = 0.3
    gamma_sd: float = 0.3
    lib_mean: float = 5000.0
    lib_sd: float = 0.6
    seed: int = 0


SPECS = {
    # BASELINE.json configs[0]
    "c1": WorkloadSpec("c1", 1000, 100, 5, "poisson", "f64", "dense", 100, 50,
                       p=1, q=1, u_sd=0.5, v_sd=0.5, b_mean=1.0, b_sd=0.3, gamma_sd=0.3),
    # configs[1]: offset = centred log library size
    "c2": WorkloadSpec("c2", 26472, 500, 15, "neg_binomial", "f64", "dense", 2000, 500,
                       p=1, q=0, offset=True, groups=7, u_sd=0.3, v_sd=0.3,
                       zero_frac=0.85, b_sd=1.0, lib_mean=5000.0, lib_sd=0.6),
    # configs[2]
    "c3": WorkloadSpec("c3", 100000, 1000, 10, "neg_binomial", "f32", "csr", 5000, 20,
                       p=2, q=1, groups=12, u_sd=0.5, v_sd=0.5, zero_frac=0.90),
    # configs[3]: the north-star headline workload
    "c4": WorkloadSpec("c4", 1300000, 500, 10, "neg_binomial", "f32", "csr", 10000, 10,
                       p=1, q=0, offset=True, groups=10, u_sd=0.3, v_sd=0.3,
                       zero_frac=0.92, b_sd=1.0, lib_mean=3000.0, lib_sd=0.7),
}


@dataclass
class Workload:
    spec: WorkloadSpec
    x: np.ndarray
    z: np.ndarray
    offset: np.ndarray | None
    truth: dict
    phi_gene: np.ndarray | None
    y_dense: np.ndarray | None = None          # (n, m) int32
    csr: tuple | None = None                   # (indptr int64, indices int32, data int32)
    meta: dict = field(default_factory=dict)

    def init_state(self, seed=1, noise=0.05):
        """Deterministic perturbation of the truth (SURVEY §8d 'init_state')."""
        rng = np.random.default_rng(seed)
        t = self.truth
        pert = lambda a: a + noise * rng.standard_normal(a.shape)
        return dict(b=pert(t["b"]), gamma=pert(t["gamma"]), u=pert(t["u"]), v=pert(t["v"]),
                    phi=1.0, nb_shape=2.0 if self.spec.family == "neg_binomial" else 1.0)

    def dense_f64(self, rows=None):
        if self.y_dense is not None:
            y = self.y_dense if rows is None else self.y_dense[rows]
            return y.astype(np.float64)
        indptr, idx, val = self.csr
        rows = np.arange(self.spec.n) if rows is None else np.asarray(rows)
        out = np.zeros((rows.size, self.spec.m))
        for k, r in enumerate(rows):
            a, b = indptr[r], indptr[r + 1]
            out[k, idx[a:b]] = val[a:b]
        return out


def _zero_prob(eta, phi_gene, family):
    mu = np.exp(eta)
    if family == "poisson":
        return np.exp(-mu)
    return np.exp(phi_gene * (np.log(phi_gene) - np.log(phi_gene + mu)))


def _calibrate_shift(eta_sub, phi_gene, family, target):
    lo, hi = -20.0, 20.0
    for _ in range(60):
        mid = 0.5 * (lo + hi)
        z = _zero_prob(eta_sub + mid, phi_gene, family).mean()
        if z > target:
            lo = mid
        else:
            hi = mid
    return 0.5 * (lo + hi)


def _params(spec: WorkloadSpec, n_rows=None):
    """Model parameters and designs; n_rows truncates to the first rows."""
    rng = np.random.default_rng(spec.seed)
    n, m, d = spec.n, spec.m, spec.d
    if spec.groups > 1:
        probs = rng.dirichlet(np.full(spec.groups, 5.0))
        groups = rng.choice(spec.groups, size=n, p=probs)
        cent = rng.standard_normal((spec.groups, d))
        u = cent[groups] + spec.u_sd * rng.standard_normal((n, d))
    else:
        u = spec.u_sd * rng.standard_normal((n, d))
    v = spec.v_sd * rng.standard_normal((m, d))
    x = np.ones((n, spec.p))
    if spec.p > 1:
        x[:, 1:] = (rng.uniform(size=(n, spec.p - 1)) < 0.5).astype(float)
    z = np.ones((m, spec.q))
    b = np.empty((m, spec.p))
    b[:, 0] = spec.b_mean + spec.b_sd * rng.standard_normal(m)
    if spec.p > 1:
        b[:, 1:] = 0.3 * rng.standard_normal((m, spec.p - 1))
    gamma = spec.gamma_sd * rng.standard_normal((n, spec.q))
    offset = None
    if spec.offset:
        lib = np.exp(np.log(spec.lib_mean) + spec.lib_sd * rng.standard_normal(n))
        offset = np.log(lib) - np.log(spec.lib_mean)
    phi_gene = rng.gamma(2.0, 2.5, size=m) if spec.family == "neg_binomial" else None
    if spec.family == "neg_binomial":
        phi_gene = np.maximum(phi_gene, 1e-2)
    meta = {}
    if spec.zero_frac is not None:
        sub = np.random.default_rng(spec.seed + 7).choice(n, size=min(n, 4000), replace=False)
        eta_sub = u[sub] @ v.T + x[sub] @ b.T + (gamma[sub] @ z.T if spec.q else 0.0)
        if offset is not None:
            eta_sub = eta_sub + offset[sub, None]
        shift = _calibrate_shift(eta_sub, phi_gene, spec.family, spec.zero_frac)
        b[:, 0] += shift
        meta["intercept_mean"] = float(spec.b_mean + shift)
    if n_rows is not None:
        u, x, gamma = u[:n_rows], x[:n_rows], gamma[:n_rows]
        offset = None if offset is None else offset[:n_rows]
    truth = dict(b=b, gamma=gamma, u=u, v=v)
    return x, z, offset, truth, phi_gene, meta


def _eta_rows(truth, x, z, offset, lo, hi):
    eta = truth["u"][lo:hi] @ truth["v"].T + x[lo:hi] @ truth["b"].T
    if z.shape[1]:
        eta += truth["gamma"][lo:hi] @ z.T
    if offset is not None:
        eta += offset[lo:hi, None]
    return np.minimum(eta, 12.0)


def generate(name_or_spec, n_rows=None, device=None, **overrides) -> Workload:
    """Build a workload.  ``n_rows`` keeps the first rows of the full-size
    parameter draw (same distribution, smaller n); ``device='cuda'`` draws
    counts with torch on the GPU (used for c3/c4 in bench.py)."""
    spec = SPECS[name_or_spec] if isinstance(name_or_spec, str) else name_or_spec
    if overrides:
        spec = WorkloadSpec(**{**spec.__dict__, **overrides})
    x, z, offset, truth, phi_gene, meta = _params(spec, n_rows)
    n = x.shape[0]
    m = spec.m
    spec_eff = WorkloadSpec(**{**spec.__dict__, "n": n})
    wl = Workload(spec_eff, x, z, offset, truth, phi_gene, meta=meta)
    chunk = max(1, 4_000_000 // m)
    if device is not None and str(device).startswith("cuda"):
        _draw_torch(wl, chunk, device)
    else:
        _draw_numpy(wl, chunk)
    if spec.y_format == "csr" and wl.csr is None:
        wl.csr = dense_to_csr(wl.y_dense)
        wl.y_dense = None
    nnz = int(wl.csr[0][-1]) if wl.csr is not None else int(np.count_nonzero(wl.y_dense))
    wl.meta.update(nnz=nnz, zero_frac=1.0 - nnz / (n * m))
    return wl


def _draw_numpy(wl, chunk):
    spec = wl.spec
    rng = np.random.default_rng(spec.seed + 1)
    y = np.empty((spec.n, spec.m), dtype=np.int32)
    for lo in range(0, spec.n, chunk):
        hi = min(spec.n, lo + chunk)
        mu = np.exp(_eta_rows(wl.truth, wl.x, wl.z, wl.offset, lo, hi))
        if spec.family == "neg_binomial":
            lam = rng.gamma(wl.phi_gene[None, :], mu / wl.phi_gene[None, :])
        else:
            lam = mu
        y[lo:hi] = np.minimum(rng.poisson(lam), 2**31 - 1).astype(np.int32)
    wl.y_dense = y


def _draw_torch(wl, chunk, device):
    import torch
    spec = wl.spec
    gen = torch.Generator(device=device)
    gen.manual_seed(spec.seed + 1)
    v = torch.as_tensor(wl.truth["v"], device=device)
    b = torch.as_tensor(wl.truth["b"], device=device)
    zt = torch.as_tensor(wl.z, device=device)
    phi = None if wl.phi_gene is None else torch.as_tensor(wl.phi_gene, device=device)
    indptr = [np.zeros(1, dtype=np.int64)]
    idx_parts, val_parts, dense_parts = [], [], []
    base = 0
    for lo in range(0, spec.n, chunk):
        hi = min(spec.n, lo + chunk)
        u = torch.as_tensor(wl.truth["u"][lo:hi], device=device)
        xr = torch.as_tensor(wl.x[lo:hi], device=device)
        eta = u @ v.T + xr @ b.T
        if spec.q:
            eta += torch.as_tensor(wl.truth["gamma"][lo:hi], device=device) @ zt.T
        if wl.offset is not None:
            eta += torch.as_tensor(wl.offset[lo:hi], device=device)[:, None]
        mu = torch.exp(torch.clamp(eta, max=12.0))
        if phi is not None:
            conc = phi[None, :].expand_as(mu).contiguous()
            g = torch._standard_gamma(conc, generator=gen) if _std_gamma_has_gen() else \
                torch._standard_gamma(conc)
            lam = g * (mu / phi[None, :])
        else:
            lam = mu
        y = torch.poisson(lam, generator=gen).clamp_(max=2**31 - 1).to(torch.int32)
        if spec.y_format == "csr":
            nzr, nzc = torch.nonzero(y, as_tuple=True)
            counts = torch.bincount(nzr, minlength=hi - lo).cpu().numpy().astype(np.int64)
            indptr.append(base + np.cumsum(counts))
            base += int(counts.sum())
            idx_parts.append(nzc.to(torch.int32).cpu().numpy())
            val_parts.append(y[nzr, nzc].cpu().numpy())
        else:
            dense_parts.append(y.cpu().numpy())
    if spec.y_format == "csr":
        wl.csr = (np.concatenate(indptr), np.concatenate(idx_parts), np.concatenate(val_parts))
    else:
        wl.y_dense = np.concatenate(dense_parts)


def _std_gamma_has_gen():
    import inspect
    import torch
    try:
        torch._standard_gamma(torch.ones(1), generator=None)
        return True
    except TypeError:
        return False


def dense_to_csr(y):
    y = np.asarray(y)
    rows, cols = np.nonzero(y)
    counts = np.bincount(rows, minlength=y.shape[0]).astype(np.int64)
    indptr = np.zeros(y.shape[0] + 1, dtype=np.int64)
    np.cumsum(counts, out=indptr[1:])
    return indptr, cols.astype(np.int32), y[rows, cols].astype(np.int32)
