"""Generate golden vectors by running the REFERENCE (gmfkit) itself.

Run in the build container only (needs /root/reference):

    python tests/golden/make_golden.py

The reference package is imported from /root/reference/pkg/src (its
pure-numpy kernel backend is selected; gmfkit's own tests pin it to the
compiled backend at 1e-13, kernels/test_kernels.py:43-55).  Outputs are
small .npz fixtures committed under tests/golden/; nothing at test time
reads /root/reference.

Fixtures:
  c1.npz          BASELINE config 1 exactly (Poisson, 1000x100, k=5, X=Z=1,
                  mb 100 x all columns, 50 epochs): per-step states at
                  checkpoints, step-0 gradients, trace, final state/objective.
  nb_offset.npz   NB with a per-row offset (SURVEY §8c shim), p=1, q=0.
  nb_cov_s3.npz   NB, p=2, q=1, mb_cols < m (S = 3 column blocks per epoch).
  converge.npz    Poisson with the default-style tol: converged flag/epochs.
  diverge.npz     rate_k0=1.2, damping=0: DivergenceError after 4 epochs; the
                  snapshot is the state after epoch 3 (not the init).
  seam.npz        derivs_from_mu / deviance / mean_of_eta vectors, all families.
  project.npz     (A)+(B1) projections incl. a rank-deficient case.
  weighted.npz    minibatch gradients with non-unit prior weights.
  c2.npz          BASELINE config 2 at full size (26,472 x 500 NB fp64, k=15,
                  offset), 20 epochs: traces, final objective, V/B at check
                  steps, projected V/B and U at a row sample (make_c2).
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)
sys.path.insert(0, HERE)
os.environ.setdefault("GMFKIT_PURE_PYTHON", "1")

import gmfkit as gk                      # noqa: E402
import gmfkit.model as gmodel            # noqa: E402
import gmfkit.optim as goptim            # noqa: E402
from gmfkit.kernels import _ref as gref  # noqa: E402

from paper_2412_20509_b200 import workloads  # noqa: E402

CHECK_STEPS = (0, 1, 4, 9, 19, 49)


def _state_arrays(prefix, st):
    return {f"{prefix}_b": st.b.copy(), f"{prefix}_gamma": st.gamma.copy(),
            f"{prefix}_u": st.u.copy(), f"{prefix}_v": st.v.copy(),
            f"{prefix}_nb": np.float64(st.nb_shape), f"{prefix}_phi": np.float64(st.phi)}


class OffsetShim:
    """Add a per-row offset to every eta entry point of the reference."""

    def __init__(self, offset):
        self.offset = offset
        self.saved = {}

    def __enter__(self):
        off = self.offset
        orig_lp = gmodel.linear_predictor
        orig_ent = goptim._entrywise_eta

        def lp(state, covs, rows=None, cols=None):
            eta = orig_lp(state, covs, rows, cols)
            o = off if rows is None else off[np.asarray(rows)]
            return eta + o[:, None]

        def ent(state, covs, rows, cols):
            return orig_ent(state, covs, rows, cols) + off[rows]

        self.saved = {"m": orig_lp, "o": goptim.linear_predictor, "e": orig_ent}
        gmodel.linear_predictor = lp
        goptim.linear_predictor = lp
        goptim._entrywise_eta = ent
        return self

    def __exit__(self, *exc):
        gmodel.linear_predictor = self.saved["m"]
        goptim.linear_predictor = self.saved["o"]
        goptim._entrywise_eta = self.saved["e"]


def _run_fit(y, x, z, init, fam, cfg, offset=None, lam=None, weights=None, mask=None):
    pen = lam or gk.PenaltyConfig()
    yv = y.astype(float)
    if mask is not None:
        yv = np.where(mask, yv, np.nan)
    data = gk.ResponseMatrix(yv, mask=mask, weights=weights)
    covs = gk.CovariateSet(x=x if x.shape[1] else None, z=z if z.shape[1] else None,
                           n=y.shape[0], m=y.shape[1])
    steps = {}

    def cb(t, st):
        if t in CHECK_STEPS:
            steps[t] = st.copy()

    init_st = gk.FactorizationState(init["b"], init["gamma"], init["u"], init["v"],
                                    init.get("phi", 1.0), init.get("nb_shape", 1.0))
    ctx = OffsetShim(offset) if offset is not None else None
    if ctx:
        ctx.__enter__()
    try:
        # step-0 gradient on the replayed first block
        rng = np.random.default_rng(cfg.seed)
        rb = goptim._partition(rng, y.shape[0], min(cfg.mb_rows, y.shape[0]))
        cb_ = goptim._partition(rng, y.shape[1], min(cfg.mb_cols, y.shape[1]))
        goptim._eval_entries(data, cfg.max_eval_entries, rng)
        first = int(rng.integers(len(rb)))
        fam_live = gk.NegBinomial(init_st.nb_shape) if fam.kind == "neg_binomial" else fam
        g0 = gk.minibatch_gradients(init_st, data, covs, fam_live, gk.Log(), pen,
                                    gk.Minibatch(rb[first], cb_[0]))
        final, rep = gk.fit_asgd(data, covs, fam, gk.Log(), pen, cfg, init_st, callback=cb)
        unproj, _ = gk.fit_asgd(data, covs, fam, gk.Log(), pen, cfg, init_st,
                                identify_mode=None)
    finally:
        if ctx:
            ctx.__exit__()
    out = {"y": y.astype(np.int32), "x": x, "z": z, "first_block": np.int64(first),
           "g0_g_row": g0.g_rowside, "g0_h_row": g0.h_rowside,
           "g0_g_col": g0.g_colside, "g0_h_col": g0.h_colside,
           "trace": np.asarray(rep.objective_trace), "nb_trace": np.asarray(rep.nb_shape_trace),
           "final_objective": np.float64(rep.final_objective),
           "epochs_run": np.int64(rep.epochs_run), "converged": np.bool_(rep.converged),
           "iterations": np.int64(rep.diagnostics["iterations"]),
           "check_steps": np.asarray(sorted(steps), dtype=np.int64),
           "cfg": np.asarray([cfg.max_epochs, cfg.mb_rows, cfg.mb_cols, cfg.seed,
                              cfg.max_eval_entries], dtype=np.int64),
           "cfg_f": np.asarray([cfg.rate_k0, cfg.rate_k1, cfg.rate_tau, cfg.smooth_a1,
                                cfg.smooth_a2, cfg.damping, cfg.tol]),
           "lam": np.asarray([pen.lam_b, pen.lam_gamma, pen.lam_u, pen.lam_v]),
           "family": np.asarray(fam.kind)}
    if offset is not None:
        out["offset"] = offset
    if weights is not None:
        out["w"] = weights
    if mask is not None:
        out["mask"] = mask
        out["nafill"] = np.int64(cfg.nafill_every)
    out.update(_state_arrays("init", init_st))
    out.update(_state_arrays("final", final))
    out.update(_state_arrays("unproj", unproj))
    for t, st in steps.items():
        out.update(_state_arrays(f"step{t}", st))
    return out


def make_c1():
    wl = workloads.generate("c1")
    y = wl.y_dense
    data = gk.ResponseMatrix(y.astype(float))
    covs = gk.CovariateSet(x=wl.x, z=wl.z)
    init = gk.init_glm_svd(data, covs, gk.Poisson(), gk.Log(), 5, seed=0)
    init_d = dict(b=init.b, gamma=init.gamma, u=init.u, v=init.v, phi=init.phi,
                  nb_shape=init.nb_shape)
    cfg = gk.SgdConfig(max_epochs=50, mb_rows=100, mb_cols=100, tol=1e-30, seed=0)
    return _run_fit(y, wl.x, wl.z, init_d, gk.Poisson(), cfg)


C2_EPOCHS = 20
C2_CHECK = (0, 1, 4, 9, 19)


from make_golden_checksum import y_checksum  # noqa: E402


def make_c2():
    """BASELINE config 2 at FULL size (26,472 x 500 NB, k=15, fp64, centred
    log-library offset through the SURVEY 8c shim, mb 2,000 rows x all
    columns) run by gmfkit itself for C2_EPOCHS epochs (tol 1e-30).  The
    counts and init are regenerated from the seeded workload generator at
    test time (checksum stored); the fixture keeps the traces, the final
    objective, V/B at check steps and the projected state's V, B and U at a
    fixed row sample."""
    wl = workloads.generate("c2")
    y = wl.y_dense
    init = wl.init_state()
    cfg = gk.SgdConfig(max_epochs=C2_EPOCHS, mb_rows=2000, mb_cols=500, tol=1e-30, seed=0)
    data = gk.ResponseMatrix(y.astype(float))
    covs = gk.CovariateSet(x=wl.x, z=None, n=y.shape[0], m=y.shape[1])
    st0 = gk.FactorizationState(init["b"], init["gamma"], init["u"], init["v"], 1.0,
                                init["nb_shape"])
    steps = {}

    def cb(t, st):
        if t in C2_CHECK:
            steps[t] = (st.b.copy(), st.v.copy(), float(st.nb_shape))

    with OffsetShim(wl.offset):
        final, rep = gk.fit_asgd(data, covs, gk.NegBinomial(init["nb_shape"]), gk.Log(),
                                 gk.PenaltyConfig(), cfg, st0, callback=cb)
    rows = np.sort(np.random.default_rng(11).choice(y.shape[0], 600, replace=False))
    out = {"y_checksum": y_checksum(y), "trace": np.asarray(rep.objective_trace),
           "nb_trace": np.asarray(rep.nb_shape_trace),
           "final_objective": np.float64(rep.final_objective),
           "epochs_run": np.int64(rep.epochs_run),
           "iterations": np.int64(rep.diagnostics["iterations"]),
           "final_b": final.b, "final_v": final.v, "final_nb": np.float64(final.nb_shape),
           "sample_rows": rows, "final_u_rows": final.u[rows],
           "check_steps": np.asarray(sorted(steps), dtype=np.int64)}
    for t, (b, v, nb) in steps.items():
        out[f"step{t}_b"], out[f"step{t}_v"], out[f"step{t}_nb"] = b, v, np.float64(nb)
    return out


def _nb_problem(n, m, p, q, d, seed, offset):
    rng = np.random.default_rng(seed)
    x = np.ones((n, p))
    if p > 1:
        x[:, 1:] = (rng.uniform(size=(n, p - 1)) < 0.5)
    z = np.ones((m, q))
    u = rng.normal(0, 0.4, (n, d))
    v = rng.normal(0, 0.4, (m, d))
    b = rng.normal(0.3, 0.4, (m, p))
    g = rng.normal(0, 0.3, (n, q))
    off = rng.normal(0, 0.6, n) if offset else None
    eta = u @ v.T + x @ b.T + (g @ z.T if q else 0) + (off[:, None] if offset else 0)
    mu = np.exp(eta)
    lam_ = rng.gamma(2.0, mu / 2.0)
    y = rng.poisson(lam_).astype(np.int32)
    init = dict(b=b + rng.normal(0, 0.05, b.shape), gamma=g + rng.normal(0, 0.05, g.shape),
                u=u + rng.normal(0, 0.05, u.shape), v=v + rng.normal(0, 0.05, v.shape),
                phi=1.0, nb_shape=1.5)
    return y, x, z, off, init


def make_nb_offset():
    y, x, z, off, init = _nb_problem(1200, 150, 1, 0, 6, 11, True)
    cfg = gk.SgdConfig(max_epochs=30, mb_rows=200, mb_cols=150, tol=1e-30, seed=3)
    return _run_fit(y, x, z, init, gk.NegBinomial(1.5), cfg, offset=off)


def make_nb_cov_s3():
    y, x, z, _, init = _nb_problem(900, 120, 2, 1, 4, 12, False)
    cfg = gk.SgdConfig(max_epochs=12, mb_rows=150, mb_cols=40, tol=1e-30, seed=5)
    pen = gk.PenaltyConfig(lam=0.7, blocks=(0.1, 0.2, 1.0, 0.5))
    return _run_fit(y, x, z, init, gk.NegBinomial(1.5), cfg, lam=pen)


def make_converge():
    rng = np.random.default_rng(21)
    n, m, d = 120, 30, 2
    u = rng.normal(0, 0.5, (n, d))
    v = rng.normal(0, 0.5, (m, d))
    b = rng.normal(1.0, 0.3, (m, 1))
    y = rng.poisson(np.exp(u @ v.T + b.T)).astype(np.int32)
    x = np.ones((n, 1))
    z = np.ones((m, 0))
    data = gk.ResponseMatrix(y.astype(float))
    covs = gk.CovariateSet(x=x, m=m)
    init = gk.init_glm_svd(data, covs, gk.Poisson(), gk.Log(), d, seed=0)
    init_d = dict(b=init.b, gamma=init.gamma, u=init.u, v=init.v)
    cfg = gk.SgdConfig(max_epochs=2000, seed=0, tol=1e-4, mb_rows=60, mb_cols=30,
                       rate_k0=0.05)
    return _run_fit(y, x, z, init_d, gk.Poisson(), cfg)


def make_diverge():
    rng = np.random.default_rng(22)
    n, m, d = 60, 12, 1
    u = rng.normal(0, 0.5, (n, d))
    v = rng.normal(0, 0.5, (m, d))
    b = rng.normal(1.0, 0.3, (m, 1))
    y = rng.poisson(np.exp(u @ v.T + b.T)).astype(np.int32)
    x = np.ones((n, 1))
    data = gk.ResponseMatrix(y.astype(float))
    covs = gk.CovariateSet(x=x, m=m)
    init = gk.init_glm_svd(data, covs, gk.Poisson(), gk.Log(), d, seed=0)
    cfg = gk.SgdConfig(max_epochs=200, seed=0, rate_k0=1.2, rate_k1=0.0, damping=0.0,
                       mb_rows=20, mb_cols=12)
    count = []
    try:
        gk.fit_asgd(data, covs, gk.Poisson(), gk.Log(), gk.PenaltyConfig(), cfg, init,
                    callback=lambda t, s: count.append(t))
        raise RuntimeError("expected divergence")
    except gk.DivergenceError as err:
        snap = err.state
    out = {"y": y, "x": x, "z": np.ones((m, 0)), "steps_before": np.int64(len(count)),
           "cfg": np.asarray([cfg.max_epochs, cfg.mb_rows, cfg.mb_cols, cfg.seed,
                              cfg.max_eval_entries], dtype=np.int64),
           "cfg_f": np.asarray([cfg.rate_k0, cfg.rate_k1, cfg.rate_tau, cfg.smooth_a1,
                                cfg.smooth_a2, cfg.damping, cfg.tol])}
    out.update(_state_arrays("init", init))
    out.update(_state_arrays("snap", snap))
    return out


def make_seam():
    rng = np.random.default_rng(31)
    out = {}
    pairs = [("poisson", "log", gk.Poisson()), ("neg_binomial", "log", gk.NegBinomial(2.3)),
             ("gaussian", "identity", gk.Gaussian()), ("gamma", "inverse", gk.Gamma()),
             ("inverse_gaussian", "inverse_squared", gk.InverseGaussian()),
             ("bernoulli", "logit", gk.Bernoulli()), ("gamma", "log", gk.Gamma()),
             ("gaussian", "log", gk.Gaussian()), ("inverse_gaussian", "log", gk.InverseGaussian())]
    for fk, lk, fam in pairs:
        n = 257
        if fk == "bernoulli":
            mu = rng.uniform(0.15, 0.85, n)
        elif fk == "gaussian" and lk == "identity":
            mu = rng.normal(0, 2, n)
        else:
            mu = rng.uniform(0.5, 5.0, n)
        y = fam.sample(mu, rng=rng)
        if fk in ("gamma", "inverse_gaussian"):
            y = np.maximum(y, 1e-3)
        if fk in ("poisson", "neg_binomial"):
            y[:20] = 0.0
        w = rng.uniform(0.5, 2.0, n)
        lnk = gk.link(lk)
        eta = lnk.eval(mu)
        fc, lc = gk.kernels.FAMILY_CODES[fk], gk.kernels.LINK_CODES[lk]
        alpha = getattr(fam, "nb_shape", 1.0)
        mu_k = gref.mean_of_eta(lc, eta)
        dd, hh = gref.derivs_from_mu(fc, lc, y, mu_k, w, 1.3, alpha)
        dev = gref.deviance_from_mu(fc, y, mu_k, w, alpha)
        key = f"{fk}+{lk}"
        out[f"{key}|y"] = y
        out[f"{key}|eta"] = eta
        out[f"{key}|w"] = w
        out[f"{key}|mu"] = mu_k
        out[f"{key}|dotd"] = dd
        out[f"{key}|ddotd"] = hh
        out[f"{key}|dev"] = np.float64(dev)
        out[f"{key}|codes"] = np.asarray([fc, lc], dtype=np.int64)
        out[f"{key}|alpha"] = np.float64(alpha)
    return out


def make_project():
    rng = np.random.default_rng(41)
    out = {}
    for k in range(3):
        n, m, d, p, q = 25 + 5 * k, 10, 3, 2, 1
        x = np.hstack([np.ones((n, 1)), rng.normal(size=(n, p - 1))])
        z = np.ones((m, q))
        covs = gk.CovariateSet(x=x, z=z)
        st = gk.FactorizationState(b=rng.normal(size=(m, p)), gamma=rng.normal(size=(n, q)),
                                   u=rng.normal(size=(n, d)), v=rng.normal(size=(m, d)))
        pr = gk.project_constraints(st, covs, "B1")
        out.update({f"{k}|x": x, f"{k}|z": z})
        out.update(_state_arrays(f"{k}|in", st))
        out.update(_state_arrays(f"{k}|out", pr))
    n, m = 10, 6
    u = rng.normal(size=(n, 2))
    v = rng.normal(size=(m, 2))
    st = gk.FactorizationState(np.zeros((m, 0)), np.zeros((n, 0)),
                               np.hstack([u, u[:, :1]]), np.hstack([v, np.zeros((m, 1))]))
    pr, info = gk.project_constraints(st, gk.CovariateSet.empty(n, m), "B1", return_info=True)
    out.update(_state_arrays("rd|in", st))
    out.update(_state_arrays("rd|out", pr))
    out["rd|eff"] = np.int64(info["effective_rank"])
    return out


def make_weighted():
    rng = np.random.default_rng(51)
    n, m, d = 40, 16, 3
    y, x, z, off, init = _nb_problem(n, m, 1, 1, d, 52, False)
    w = rng.uniform(0.5, 2.0, (n, m))
    data = gk.ResponseMatrix(y.astype(float), weights=w)
    covs = gk.CovariateSet(x=x, z=z)
    st = gk.FactorizationState(init["b"], init["gamma"], init["u"], init["v"], 1.0, 1.7)
    pen = gk.PenaltyConfig(lam=0.8, blocks=(0.2, 0.1, 1.0, 0.6))
    I = np.array([1, 4, 5, 9, 17, 30])
    J = np.arange(m)
    gp = gk.minibatch_gradients(st, data, covs, gk.NegBinomial(1.7), gk.Log(), pen,
                                gk.Minibatch(I, J))
    obj = gk.penalized_objective(st, data, covs, gk.NegBinomial(1.7), gk.Log(), pen)
    out = {"y": y, "x": x, "z": z, "w": w, "I": I, "g_row": gp.g_rowside,
           "h_row": gp.h_rowside, "g_col": gp.g_colside, "h_col": gp.h_colside,
           "objective": np.float64(obj), "lam": np.asarray([0.16, 0.08, 0.8, 0.48])}
    out.update(_state_arrays("st", st))
    return out


def make_select():
    """information_criteria / _mu_at / rel_deviance / rel_log_rmse of the
    reference (select.py:57-96, 141-145; metrics.py:35-55)."""
    import gmfkit.select as gsel
    import gmfkit.metrics as gmet
    rng = np.random.default_rng(61)
    out = {}
    cases = [("pois", gk.Poisson(), 1.3, False, 2, 1), ("nb", gk.NegBinomial(1.7), 1.0, False, 2, 1),
             ("nbw", gk.NegBinomial(0.6), 1.0, True, 1, 0), ("nb50", gk.NegBinomial(50.0), 1.0, False, 1, 1)]
    for k, (key, fam, phi, weighted, p, q) in enumerate(cases):
        n, m, d = 60, 24, 3
        y, x, z, off, init = _nb_problem(n, m, p, q, d, 62 + k, False)
        w = rng.uniform(0.5, 2.0, (n, m)) if weighted else None
        data = gk.ResponseMatrix(y.astype(float), weights=w)
        covs = gk.CovariateSet(x=x, z=z)
        st = gk.FactorizationState(init["b"], init["gamma"], init["u"], init["v"], phi,
                                   getattr(fam, "nb_shape", 1.0))
        aic, bic = gsel.information_criteria(st, data, covs, fam, gk.Log())
        rows = rng.integers(0, n, 50)
        cols = rng.integers(0, m, 50)
        ybar = float(np.mean(y))
        mu_t = gsel._mu_at(st, covs, gk.Log(), rows, cols)
        yt = y[rows, cols].astype(float)
        out[f"{key}|y"] = y
        out[f"{key}|x"] = covs.x
        out[f"{key}|z"] = covs.z
        if w is not None:
            out[f"{key}|w"] = w
        out.update(_state_arrays(f"{key}|st", st))
        out[f"{key}|alpha"] = np.float64(getattr(fam, "nb_shape", 1.0))
        out[f"{key}|aic"] = np.float64(aic)
        out[f"{key}|bic"] = np.float64(bic)
        out[f"{key}|rows"] = rows
        out[f"{key}|cols"] = cols
        out[f"{key}|ybar"] = np.float64(ybar)
        out[f"{key}|mu_test"] = mu_t
        out[f"{key}|rel_dev"] = np.float64(gmet.rel_deviance(yt, mu_t, ybar, fam))
        out[f"{key}|rel_lrmse"] = np.float64(gmet.rel_log_rmse(yt, mu_t, ybar))
    return out


def make_init():
    """init_ols_svd of the reference (initialization.py:143-169), Poisson and
    NB, randomized range finder and the exact-SVD fallback."""
    out = {}
    cases = [("pois", gk.Poisson(), 300, 80, 1, 1, 4), ("nb", gk.NegBinomial(2.0), 400, 60, 2, 1, 5),
             ("small", gk.NegBinomial(1.0), 30, 12, 1, 0, 3), ("noz", gk.Poisson(), 200, 50, 0, 0, 2)]
    for k, (key, fam, n, m, p, q, d) in enumerate(cases):
        y, x, z, off, init = _nb_problem(n, m, max(p, 1), q, d, 81 + k, False)
        x = x[:, :p]
        data = gk.ResponseMatrix(y.astype(float))
        covs = gk.CovariateSet(x=x, z=z)
        st = gk.init_ols_svd(data, covs, fam, gk.Log(), d, seed=3)
        out[f"{key}|y"] = y
        out[f"{key}|x"] = x
        out[f"{key}|z"] = z
        out[f"{key}|d"] = np.int64(d)
        out[f"{key}|nbfam"] = np.int64(fam.kind == "neg_binomial")
        out[f"{key}|b"] = st.b
        out[f"{key}|gamma"] = st.gamma
        out[f"{key}|uv"] = st.u @ st.v.T
        out[f"{key}|s"] = np.linalg.norm(st.u, axis=0)
        out[f"{key}|nb_shape"] = np.float64(st.nb_shape)
        out[f"{key}|phi"] = np.float64(st.phi)
    return out


def make_init_glm():
    """init_glm_svd of the reference (initialization.py:172-214): Poisson / NB,
    covariates on both sides, a masked and weighted case, the Pearson residual
    kind, and the exact-SVD fallback."""
    out = {}
    cases = [("pois", gk.Poisson(), 300, 80, 2, 1, 4, False, False, "deviance"),
             ("nb", gk.NegBinomial(2.0), 400, 60, 1, 1, 5, False, False, "deviance"),
             ("masked", gk.NegBinomial(1.3), 350, 70, 2, 0, 3, True, True, "deviance"),
             ("pearson", gk.Poisson(), 250, 50, 1, 0, 3, False, False, "pearson"),
             ("small", gk.NegBinomial(1.0), 30, 12, 1, 0, 3, False, False, "deviance")]
    for k, (key, fam, n, m, p, q, d, masked, weighted, rk) in enumerate(cases):
        y, x, z, off, init = _nb_problem(n, m, max(p, 1), q, d, 91 + k, False)
        x = x[:, :p]
        rng = np.random.default_rng(191 + k)
        mask = rng.uniform(size=y.shape) > 0.15 if masked else None
        w = rng.uniform(0.5, 2.0, size=y.shape) if weighted else None
        yv = y.astype(float) if mask is None else np.where(mask, y, np.nan)
        data = gk.ResponseMatrix(yv, mask=mask, weights=w)
        covs = gk.CovariateSet(x=x, z=z)
        st, info = gk.init_glm_svd(data, covs, fam, gk.Log(), d, seed=3, return_info=True,
                                   method=gk.InitMethod(residual_kind=rk))
        out[f"{key}|y"] = y
        out[f"{key}|x"] = x
        out[f"{key}|z"] = z
        out[f"{key}|d"] = np.int64(d)
        out[f"{key}|fam"] = np.asarray(fam.kind)
        out[f"{key}|alpha"] = np.float64(getattr(fam, "nb_shape", 1.0))
        out[f"{key}|rk"] = np.asarray(rk)
        if mask is not None:
            out[f"{key}|mask"] = mask
        if w is not None:
            out[f"{key}|w"] = w
        out[f"{key}|b"] = st.b
        out[f"{key}|gamma"] = st.gamma
        out[f"{key}|uv"] = st.u @ st.v.T
        out[f"{key}|nb_shape"] = np.float64(st.nb_shape)
        out[f"{key}|fallbacks"] = np.asarray(str(info.get("glm_fallbacks", {})))
    return out


def make_cv():
    """cv_rank_select of the reference (select.py:148-237): two folds of 30 %
    holdouts fitted (imputed holes, GLM-SVD start, warm starts over ranks),
    AIC/BIC, held-out relative deviance, the scree pick (select.py:240-294)."""
    y, x, z, _, _ = _nb_problem(240, 50, 1, 0, 2, 131, False)
    data = gk.ResponseMatrix(y.astype(float))
    covs = gk.CovariateSet(x=x, m=50)
    cfg = gk.SgdConfig(max_epochs=20, mb_rows=60, mb_cols=50, tol=1e-30, seed=1)
    rep = gk.cv_rank_select(data, covs, gk.NegBinomial(1.5), gk.Log(), [1, 2, 3], folds=2, cfg=cfg,
                            seed=5)
    scree = gk.scree_eigenvalues(data, covs, 4)
    return {"y": y, "x": x, "aic": np.asarray(rep.aic), "bic": np.asarray(rep.bic),
            "cv": np.asarray(rep.cv_deviance), "scree": np.asarray(rep.scree_eigenvalues),
            "scree4": np.asarray(scree), "failures": np.asarray(str(rep.failures)),
            "chosen": np.asarray([rep.chosen["cv"], rep.chosen["aic"], rep.chosen["bic"],
                                  rep.chosen["scree"]])}


def make_cv_gamma():
    """cv_rank_select of the reference for a non-count family (Gamma / log,
    estimated dispersion): masked train fits, GLM-SVD starts, AIC/BIC with the
    Gamma dispersion constant, held-out relative deviance."""
    y, x, z, _ = _general_problem("gamma", "log", 200, 40, 1, 0, 2, 141)
    data = gk.ResponseMatrix(y)
    covs = gk.CovariateSet(x=x, m=40)
    cfg = gk.SgdConfig(max_epochs=16, mb_rows=50, mb_cols=40, tol=1e-30, seed=2)
    rep = gk.cv_rank_select(data, covs, gk.Gamma(), gk.Log(), [1, 2, 3], folds=2, cfg=cfg, seed=6)
    return {"y": y, "x": x, "aic": np.asarray(rep.aic), "bic": np.asarray(rep.bic),
            "cv": np.asarray(rep.cv_deviance), "failures": np.asarray(str(rep.failures)),
            "chosen": np.asarray([rep.chosen["cv"], rep.chosen["aic"], rep.chosen["bic"],
                                  rep.chosen["scree"]])}


def make_cv_gauss():
    """cv_rank_select of the reference on Gaussian / identity data (matrix
    completion with an estimated variance): masked train fits, AIC/BIC with
    n_obs log phi, held-out relative deviance."""
    y, x, z, _ = _general_problem("gaussian", "identity", 200, 40, 1, 0, 2, 151)
    data = gk.ResponseMatrix(y)
    covs = gk.CovariateSet(x=x, m=40)
    cfg = gk.SgdConfig(max_epochs=16, mb_rows=50, mb_cols=40, tol=1e-30, seed=2)
    rep = gk.cv_rank_select(data, covs, gk.Gaussian(), gk.Identity(), [1, 2, 3], folds=2, cfg=cfg,
                            seed=6)
    return {"y": y, "x": x, "aic": np.asarray(rep.aic), "bic": np.asarray(rep.bic),
            "cv": np.asarray(rep.cv_deviance), "failures": np.asarray(str(rep.failures)),
            "chosen": np.asarray([rep.chosen["cv"], rep.chosen["aic"], rep.chosen["bic"],
                                  rep.chosen["scree"]])}


def make_api():
    """Block helpers of the public API: linear_predictor (model.py:229-256),
    impute_block (optim.py:232-245), update_nb_shape_stochastic (205-229)."""
    y, x, z, _, init = _nb_problem(120, 30, 2, 1, 3, 141, False)
    mask = np.random.default_rng(142).uniform(size=y.shape) > 0.2
    w = np.random.default_rng(143).uniform(0.5, 2.0, size=y.shape)
    data = gk.ResponseMatrix(np.where(mask, y, np.nan), mask=mask, weights=w)
    covs = gk.CovariateSet(x=x, z=z)
    st = gk.FactorizationState(init["b"], init["gamma"], init["u"], init["v"], 1.0, 1.5)
    I, J = np.array([3, 7, 8, 50, 99]), np.array([0, 4, 5, 29])
    mb = gk.Minibatch(I, J)
    eta = gk.linear_predictor(st, covs, I, J)
    eta_all = gk.linear_predictor(st, covs)
    blk = gk.impute_block(st, data, covs, gk.Log(), mb)
    nb = gk.update_nb_shape_stochastic(st, data, mb, 0.3, covs=covs, lnk=gk.Log())
    return {"y": y, "x": x, "z": z, "mask": mask, "w": w, "I": I, "J": J, "eta": eta,
            "eta_all": eta_all, "block": blk, "nb": np.float64(nb),
            **_state_arrays("st", st)}


def make_cli():
    """The reference CLI end to end (cli.py:151-201, 204-253): `fit` (GLM-SVD
    start, aSGD, B1) and `cv --criterion scree` on a small CSV."""
    import tempfile
    from gmfkit import cli as gcli
    from gmfkit import io as gio
    y, x, z, _, _ = _nb_problem(160, 40, 1, 0, 2, 151, False)
    out = {"y": y}
    with tempfile.TemporaryDirectory() as tmp:
        ycsv = os.path.join(tmp, "y.csv")
        gio.write_dense_csv(ycsv, y.astype(float))
        rc = gcli.main(["fit", "--y", ycsv, "--rank", "2", "--family", "neg_binomial",
                        "--nb-shape", "1.5", "--max-epochs", "15", "--mb-rows", "40",
                        "--mb-cols", "40", "--tol", "1e-30", "--out", os.path.join(tmp, "fit")])
        out["fit_rc"] = np.int64(rc)
        for name in ("U", "V"):
            out[name] = gio.read_dense_csv(os.path.join(tmp, "fit", f"{name}.csv"))[0]
        rep = gio.read_json(os.path.join(tmp, "fit", "fit_report.json"))
        out["trace"] = np.asarray(rep["objective_trace"])
        out["final_objective"] = np.float64(rep["final_objective"])
        rc = gcli.main(["cv", "--y", ycsv, "--ranks", "1:3", "--criterion", "scree",
                        "--out", os.path.join(tmp, "cv")])
        out["cv_rc"] = np.int64(rc)
        rr = gio.read_json(os.path.join(tmp, "cv", "rank_report.json"))
        out["scree"] = np.asarray(rr["scree_eigenvalues"])
        out["scree_pick"] = np.int64(rr["chosen"]["scree"])
    return out


def make_mm():
    """MatrixMarket files and the reference's dense reads of them
    (io.py:96-109); the files themselves are fixtures under golden/mm/."""
    import gmfkit.io as gio
    d = os.path.join(HERE, "mm")
    os.makedirs(d, exist_ok=True)
    rng = np.random.default_rng(91)
    y = rng.poisson(rng.gamma(0.5, 2.0, (50, 20))).astype(float)
    y[3] = 0.0                                         # an empty row
    gio.write_matrix_market(os.path.join(d, "counts.mtx"), y)
    with open(os.path.join(d, "sym_pattern.mtx"), "w") as fh:
        fh.write("%%MatrixMarket matrix coordinate pattern symmetric\n% a comment\n"
                 "5 5 4\n1 1\n3 1\n5 2\n4 4\n")
    with open(os.path.join(d, "dups.mtx"), "w") as fh:
        fh.write("%%MatrixMarket matrix coordinate integer general\n%\n% comments\n"
                 "4 6 7\n2 3 4\n1 6 1\n2 3 5\n4 1 0\n\n4 2 7\n3 5 2\n1 1 3\n")
    out = {}
    for name in ("counts", "sym_pattern", "dups"):
        out[name] = gio.read_matrix_market(os.path.join(d, f"{name}.mtx"))
    return out


def make_project_b23():
    """project_constraints in the B2 and B3 modes (identify.py:59-138)."""
    rng = np.random.default_rng(43)
    out = {}
    for k in range(3):
        n, m, d, p, q = 40 + 7 * k, 12, 3, 2, 1
        x = np.hstack([np.ones((n, 1)), rng.normal(size=(n, p - 1))])
        z = np.ones((m, q)) if k != 1 else rng.normal(size=(m, q))
        covs = gk.CovariateSet(x=x, z=z)
        st = gk.FactorizationState(b=rng.normal(size=(m, p)), gamma=rng.normal(size=(n, q)),
                                   u=rng.normal(size=(n, d)), v=rng.normal(size=(m, d)))
        out.update({f"{k}|x": x, f"{k}|z": z})
        out.update(_state_arrays(f"{k}|in", st))
        for mode in ("B2", "B3"):
            pr = gk.project_constraints(st, covs, mode)
            out.update(_state_arrays(f"{k}|{mode}", pr))
    return out


def make_masked():
    """Unobserved entries (~15 %): imputation at the initial state and every
    nafill_every steps (optim.py:368-374, 430-436), NB with an offset."""
    y, x, z, off, init = _nb_problem(700, 90, 1, 0, 4, 21, True)
    mask = np.random.default_rng(22).uniform(size=y.shape) > 0.15
    cfg = gk.SgdConfig(max_epochs=25, mb_rows=140, mb_cols=90, tol=1e-30, seed=4, nafill_every=1)
    return _run_fit(y, x, z, init, gk.NegBinomial(1.5), cfg, offset=off, mask=mask)


def make_masked_p3():
    """Poisson with covariates, holes refilled every third step, S = 2."""
    y, x, z, _, init = _nb_problem(600, 80, 2, 1, 3, 23, False)
    mask = np.random.default_rng(24).uniform(size=y.shape) > 0.2
    cfg = gk.SgdConfig(max_epochs=10, mb_rows=120, mb_cols=40, tol=1e-30, seed=6, nafill_every=3)
    return _run_fit(y, x, z, init, gk.Poisson(), cfg, mask=mask)


GENERAL_CASES = (
    # name, family, link, dispersion policy, (p, q, d), seed
    ("gauss_id", "gaussian", "identity", "auto", (1, 1, 3), 31),
    ("gamma_log", "gamma", "log", "auto", (1, 0, 3), 32),
    ("bern_logit", "bernoulli", "logit", "auto", (1, 1, 2), 33),
    ("ig_log", "inverse_gaussian", "log", "auto", (1, 0, 2), 34),
    ("qpois", "poisson", "log", "estimate", (2, 1, 3), 35),
    ("gamma_inv", "gamma", "inverse", "fixed", (1, 0, 2), 36),
    ("pois_id", "poisson", "identity", "auto", (1, 0, 2), 37),
)


def _general_problem(fam_kind, lnk_kind, n, m, p, q, d, seed):
    """Real-valued (or count) responses simulated by gmfkit's own family
    samplers at a known state; the init is the truth perturbed."""
    rng = np.random.default_rng(seed)
    x = np.hstack([np.ones((n, 1)), rng.normal(0, 1, (n, p - 1))]) if p else np.zeros((n, 0))
    z = rng.normal(0, 0.3, (m, q)) if q else np.zeros((m, 0))
    u = rng.normal(0, 0.25, (n, d))
    v = rng.normal(0, 0.25, (m, d))
    gamma = rng.normal(0, 0.2, (n, q))
    b = rng.normal(0, 0.15, (m, p))
    if p:
        # the intercept places eta inside the link's domain with margin
        b[:, 0] += {"identity": 3.0, "log": 0.8, "logit": 0.0, "inverse": 1.5,
                    "inverse_squared": 1.5}[lnk_kind]
    eta = u @ v.T + x @ b.T + gamma @ z.T
    lnk = gk.link(lnk_kind)
    fam = gk.family(fam_kind)
    mu = lnk.inverse(eta)
    y = fam.sample(mu, phi=0.4 if fam.has_free_dispersion else 1.0, rng=rng)
    init = {"b": b + 0.03 * rng.normal(size=b.shape), "gamma": gamma * 0.8,
            "u": u + 0.05 * rng.normal(size=u.shape), "v": v + 0.05 * rng.normal(size=v.shape),
            "phi": 1.0, "nb_shape": 1.0}
    return y, x, z, init


def make_general():
    """Families and links beyond Poisson/NB+log, and the Pearson dispersion
    update (families.py:267-441, optim.py:175-202, 465-468): whole fits of the
    reference, per-step states, phi traces, step-0 gradients."""
    out = {"cases": np.asarray([c[0] for c in GENERAL_CASES])}
    for name, fk, lk, disp, (p, q, d), seed in GENERAL_CASES:
        n, m = 360, 48
        y, x, z, init = _general_problem(fk, lk, n, m, p, q, d, seed)
        data = gk.ResponseMatrix(y.astype(float))
        covs = gk.CovariateSet(x=x if p else None, z=z if q else None, n=n, m=m)
        fam, lnk = gk.family(fk), gk.link(lk)
        cfg = gk.SgdConfig(max_epochs=24, mb_rows=90, mb_cols=m, tol=1e-30, seed=seed,
                           rate_k0=0.01, rate_k1=0.01)
        pen = gk.PenaltyConfig()
        st0 = gk.FactorizationState(init["b"], init["gamma"], init["u"], init["v"], 1.0, 1.0)
        steps = {}

        def cb(t, st, steps=steps):
            if t in CHECK_STEPS:
                steps[t] = st.copy()

        rng = np.random.default_rng(cfg.seed)
        rb = goptim._partition(rng, n, cfg.mb_rows)
        cb_ = goptim._partition(rng, m, m)
        goptim._eval_entries(data, cfg.max_eval_entries, rng)
        first = int(rng.integers(len(rb)))
        g0 = gk.minibatch_gradients(st0, data, covs, fam, lnk, pen, gk.Minibatch(rb[first], cb_[0]))
        final, rep = gk.fit_asgd(data, covs, fam, lnk, pen, cfg, st0, dispersion=disp, callback=cb)
        unproj, _ = gk.fit_asgd(data, covs, fam, lnk, pen, cfg, st0, dispersion=disp,
                                identify_mode=None)
        arrs = {"y": y, "x": x, "z": z, "family": np.asarray(fk), "link": np.asarray(lk),
                "dispersion": np.asarray(disp), "first_block": np.int64(first),
                "g0_g_row": g0.g_rowside, "g0_h_row": g0.h_rowside,
                "g0_g_col": g0.g_colside, "g0_h_col": g0.h_colside,
                "trace": np.asarray(rep.objective_trace), "phi_trace": np.asarray(rep.phi_trace),
                "final_objective": np.float64(rep.final_objective),
                "epochs_run": np.int64(rep.epochs_run),
                "cfg": np.asarray([cfg.max_epochs, cfg.mb_rows, cfg.mb_cols, cfg.seed],
                                  dtype=np.int64),
                "check_steps": np.asarray(sorted(steps), dtype=np.int64)}
        arrs.update(_state_arrays("init", st0))
        arrs.update(_state_arrays("final", final))
        arrs.update(_state_arrays("unproj", unproj))
        for t, st in steps.items():
            arrs.update(_state_arrays(f"step{t}", st))
        assert np.all(np.isfinite(rep.objective_trace)), name
        out.update({f"{name}__{k}": v for k, v in arrs.items()})
    return out


def make_general_masked():
    """Unobserved entries under non-count families, Gaussian included
    (optim.py:368-374, 430-436 with families.py:267-396): whole fits of the
    reference on ~15 % masked responses, nafill_every = 2."""
    out = {"cases": np.asarray(["gauss_id", "gamma_log", "bern_logit", "ig_log"])}
    for name, fk, lk, disp, (p, q, d), seed in GENERAL_CASES:
        if name not in ("gauss_id", "gamma_log", "bern_logit", "ig_log"):
            continue
        n, m = 300, 40
        y, x, z, init = _general_problem(fk, lk, n, m, p, q, d, seed + 200)
        mask = np.random.default_rng(seed + 300).uniform(size=y.shape) > 0.15
        data = gk.ResponseMatrix(np.where(mask, y, np.nan), mask=mask)
        covs = gk.CovariateSet(x=x if p else None, z=z if q else None, n=n, m=m)
        fam, lnk = gk.family(fk), gk.link(lk)
        cfg = gk.SgdConfig(max_epochs=20, mb_rows=75, mb_cols=m, tol=1e-30, seed=seed,
                           nafill_every=2)
        st0 = gk.FactorizationState(init["b"], init["gamma"], init["u"], init["v"], 1.0, 1.0)
        final, rep = gk.fit_asgd(data, covs, fam, lnk, gk.PenaltyConfig(), cfg, st0,
                                 dispersion=disp, identify_mode=None)
        arrs = {"y": y, "mask": mask, "x": x, "z": z, "family": np.asarray(fk),
                "link": np.asarray(lk), "dispersion": np.asarray(disp),
                "trace": np.asarray(rep.objective_trace), "phi_trace": np.asarray(rep.phi_trace),
                "final_objective": np.float64(rep.final_objective),
                "cfg": np.asarray([cfg.max_epochs, cfg.mb_rows, cfg.mb_cols, cfg.seed,
                                   cfg.nafill_every], dtype=np.int64)}
        arrs.update(_state_arrays("init", st0))
        arrs.update(_state_arrays("final", final))
        assert np.all(np.isfinite(rep.objective_trace)), name
        out.update({f"{name}__{k}": v for k, v in arrs.items()})
    return out


def make_init_general():
    """init_glm_svd of the reference for the general families / links, incl.
    the Pearson start of phi (initialization.py:85-90, 172-214)."""
    out = {"cases": np.asarray([c[0] for c in GENERAL_CASES])}
    for name, fk, lk, disp, (p, q, d), seed in GENERAL_CASES:
        n, m = 240, 40
        y, x, z, _ = _general_problem(fk, lk, n, m, p, q, d, seed + 100)
        data = gk.ResponseMatrix(y.astype(float))
        covs = gk.CovariateSet(x=x if p else None, z=z if q else None, n=n, m=m)
        st, info = gk.init_glm_svd(data, covs, gk.family(fk), gk.link(lk), d, seed=5,
                                   return_info=True)
        out.update({f"{name}__y": y, f"{name}__x": x, f"{name}__z": z, f"{name}__d": np.int64(d),
                    f"{name}__family": np.asarray(fk), f"{name}__link": np.asarray(lk),
                    f"{name}__b": st.b, f"{name}__gamma": st.gamma, f"{name}__uv": st.u @ st.v.T,
                    f"{name}__phi": np.float64(st.phi),
                    f"{name}__fallbacks": np.asarray(str(info.get("glm_fallbacks", {})))})
    return out


def main():
    makers = {"general": make_general, "init_general": make_init_general,
              "general_masked": make_general_masked, "cv_gamma": make_cv_gamma, "cv_gauss": make_cv_gauss, "c1": make_c1, "nb_offset": make_nb_offset, "nb_cov_s3": make_nb_cov_s3,
              "converge": make_converge, "diverge": make_diverge, "seam": make_seam,
              "project": make_project, "weighted": make_weighted,
              "select": make_select, "init": make_init, "mm": make_mm,
              "project_b23": make_project_b23, "c2": make_c2, "masked": make_masked,
              "masked_p3": make_masked_p3, "init_glm": make_init_glm, "cv": make_cv,
              "api": make_api, "cli": make_cli}
    only = sys.argv[1:] or list(makers)
    for name in only:
        arrs = makers[name]()
        path = os.path.join(HERE, f"{name}.npz")
        np.savez_compressed(path, **arrs)
        print(f"wrote {path} ({os.path.getsize(path) / 1024:.0f} KiB)")


if __name__ == "__main__":
    main()
