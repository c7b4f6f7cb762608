"""GPU parity of general mode -- any family / link at run time on the
CUDA-core K1, real-valued responses, the Pearson dispersion update -- against
the reference's own fits (tests/golden/general.npz from gmfkit) and the
oracle.  fp64: trajectories to 1e-9; fp32: north-star tolerances."""
import numpy as np
import pytest

from conftest import golden, normwise
from oracle import asgd_oracle as orc
from test_general_oracle import CASES, case

pytestmark = pytest.mark.gpu

gk = pytest.importorskip("paper_2412_20509_b200")


@pytest.fixture(autouse=True)
def _gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _setup(c):
    n, m = c["y"].shape
    data = gk.ResponseMatrix(c["y"].astype(float))
    covs = gk.CovariateSet(x=c["x"] if c["x"].shape[1] else None,
                           z=c["z"] if c["z"].shape[1] else None, n=n, m=m)
    fam, lnk = gk.family(str(c["family"])), gk.link(str(c["link"]))
    me, mr, mc, seed = (int(v) for v in c["cfg"])
    cfg = gk.SgdConfig(max_epochs=me, mb_rows=mr, mb_cols=mc, tol=1e-30, seed=seed)
    init = gk.FactorizationState(c["init_b"], c["init_gamma"], c["init_u"], c["init_v"], 1.0, 1.0)
    return data, covs, fam, lnk, cfg, init


@pytest.mark.parametrize("name", CASES)
def test_general_fit_fp64_matches_reference(name):
    c = case(golden("general"), name)
    data, covs, fam, lnk, cfg, init = _setup(c)
    seen = {}

    def cb(t, st):
        if t in set(c["check_steps"].tolist()):
            seen[t] = st.copy()

    final, rep = gk.fit_asgd(data, covs, fam, lnk, gk.PenaltyConfig(), cfg, init,
                             dispersion=str(c["dispersion"]), callback=cb, dtype="f64")
    assert rep.epochs_run == int(c["epochs_run"])
    assert normwise(rep.objective_trace, c["trace"]) < 1e-9
    assert normwise(rep.phi_trace, c["phi_trace"]) < 1e-9
    assert seen
    for t, st in seen.items():
        for blk in ("b", "gamma", "u", "v"):
            assert normwise(getattr(st, blk), c[f"step{t}_{blk}"]) < 1e-8, (t, blk)
        assert abs(st.phi - float(c[f"step{t}_phi"])) < 1e-9 * float(c[f"step{t}_phi"])
    assert abs(final.phi - float(c["final_phi"])) < 1e-9 * float(c["final_phi"])
    assert normwise(final.u @ final.v.T, c["final_u"] @ c["final_v"].T) < 1e-7
    fo = float(c["final_objective"])
    assert abs(rep.final_objective - fo) < 1e-9 * abs(fo)
    assert rep.diagnostics["algorithm"] == "asgd"


@pytest.mark.parametrize("name", CASES)
def test_general_fit_fp32(name):
    c = case(golden("general"), name)
    data, covs, fam, lnk, cfg, init = _setup(c)
    final, rep = gk.fit_asgd(data, covs, fam, lnk, gk.PenaltyConfig(), cfg, init,
                             dispersion=str(c["dispersion"]), dtype="f32")
    assert normwise(rep.objective_trace, c["trace"]) < 1e-3
    assert normwise(rep.phi_trace, c["phi_trace"]) < 1e-3
    assert normwise(final.u @ final.v.T, c["final_u"] @ c["final_v"].T) < 1e-3
    fo = float(c["final_objective"])
    assert abs(rep.final_objective - fo) < 1e-3 * abs(fo)


@pytest.mark.parametrize("name", ["gauss_id", "gamma_inv", "pois_id"])
@pytest.mark.parametrize("dtype,tol", [("f64", 1e-10), ("f32", 1e-4)])
def test_general_step0_gradient(name, dtype, tol):
    c = case(golden("general"), name)
    data, covs, fam, lnk, cfg, init = _setup(c)
    from paper_2412_20509_b200.engine import Schedule
    sch = Schedule(*c["y"].shape, cfg)
    mb = gk.Minibatch(sch.row_blocks[int(c["first_block"])], sch.col_blocks[0])
    g = gk.minibatch_gradients(init, data, covs, fam, lnk, gk.PenaltyConfig(), mb, dtype=dtype)
    for mine, key in ((g.g_rowside, "g0_g_row"), (g.h_rowside, "g0_h_row"),
                      (g.g_colside, "g0_g_col"), (g.h_colside, "g0_h_col")):
        assert normwise(mine, c[key]) < tol, key


def test_general_wide_bucket_and_objective():
    """K = p+q+d in (16, 32] runs the second general bucket; penalized_objective
    of a non-count family on the GPU against the oracle."""
    rng = np.random.default_rng(5)
    n, m, d = 300, 40, 18
    x = np.ones((n, 1))
    u, v = rng.normal(0, 0.15, (n, d)), rng.normal(0, 0.15, (m, d))
    b = rng.normal(2.0, 0.1, (m, 1))
    y = u @ v.T + x @ b.T + rng.normal(0, 0.5, (n, m))
    st = gk.FactorizationState(b, np.zeros((n, 0)), u, v, 0.7, 1.0)
    data, covs = gk.ResponseMatrix(y), gk.CovariateSet(x=x, m=m)
    pen = gk.PenaltyConfig()
    got = gk.penalized_objective(st, data, covs, gk.Gaussian(), gk.Identity(), pen)
    pb = orc.OProblem(y, x, np.zeros((m, 0)))
    ost = orc.OState(b, np.zeros((n, 0)), u, v, 0.7, 1.0)
    want = orc.penalized_objective(ost, pb, orc.GAUSSIAN, orc.IDENTITY, (0.0, 0.0, 1.0, 0.0))
    assert abs(got - want) < 1e-10 * abs(want)
    cfg = gk.SgdConfig(max_epochs=6, mb_rows=100, mb_cols=m, tol=1e-30, seed=2)
    final, rep = gk.fit_asgd(data, covs, gk.Gaussian(), gk.Identity(), pen, cfg, st, dtype="f64")
    ocfg = orc.OConfig(max_epochs=6, mb_rows=100, mb_cols=m, tol=1e-30, seed=2)
    ofinal, orep = orc.fit_asgd(pb, orc.GAUSSIAN, orc.IDENTITY, (0.0, 0.0, 1.0, 0.0), ocfg, ost)
    assert normwise(rep.objective_trace, orep.objective_trace) < 1e-9
    assert normwise(rep.phi_trace, orep.phi_trace) < 1e-9
    assert normwise(final.u @ final.v.T, ofinal.u @ ofinal.v.T) < 1e-7


def test_general_mode_limits():
    """What general mode refuses, with the reference's error taxonomy."""
    from paper_2412_20509_b200 import _lib
    rng = np.random.default_rng(0)
    n, m, d = 60, 12, 2
    y = rng.gamma(2.0, 1.0, (n, m))
    st = gk.FactorizationState(np.zeros((m, 1)), np.zeros((n, 0)), rng.normal(0, .1, (n, d)),
                               rng.normal(0, .1, (m, d)), 1.0, 1.0)
    covs = gk.CovariateSet(x=np.ones((n, 1)), m=m)
    cfg = gk.SgdConfig(max_epochs=2, mb_rows=30, mb_cols=m)
    bad = y.copy()
    bad[3, 4] = -1.0
    with pytest.raises(gk.DomainError):      # gamma responses must be positive
        gk.fit_asgd(gk.ResponseMatrix(bad), covs, gk.Gamma(), gk.Log(), gk.PenaltyConfig(), cfg, st)
    from paper_2412_20509_b200.workloads import dense_to_csr
    yc = rng.poisson(2.0, (n, m))
    with pytest.raises(_lib.UnsupportedError):   # general mode needs a dense response
        gk.fit_asgd(gk.ResponseMatrix(csr=dense_to_csr(yc), shape=yc.shape), covs, gk.Poisson(),
                    gk.Identity(), gk.PenaltyConfig(), cfg, st)


def test_update_dispersion_stochastic_matches_oracle():
    c = case(golden("general"), "gamma_log")
    data, covs, fam, lnk, cfg, init = _setup(c)
    from paper_2412_20509_b200.engine import Schedule
    sch = Schedule(*c["y"].shape, cfg)
    I, J = sch.row_blocks[0], sch.col_blocks[0]
    got = gk.update_dispersion_stochastic(init, data, covs, fam, gk.Minibatch(I, J), 0.3, lnk)
    pb = orc.OProblem(c["y"].astype(float), c["x"], c["z"])
    ost = orc.OState(c["init_b"], c["init_gamma"], c["init_u"], c["init_v"], 1.0, 1.0)
    y, w, mu, _, _ = orc.block_derivs(ost, pb, I, J, orc.GAMMA, orc.LOG)
    n, m = c["y"].shape
    want = orc.pearson_phi_update(1.0, 0.3, y, mu, w, orc.GAMMA, 1.0, n, m, len(I), len(J),
                                  c["x"].shape[1], c["z"].shape[1], c["init_u"].shape[1])
    assert abs(got - want) < 1e-12 * abs(want)


@pytest.mark.parametrize("name", CASES)
def test_init_glm_svd_general_matches_reference(name):
    """The reference's default start for every family / link, with the Pearson
    start of phi (initialization.py:85-90, 172-214)."""
    c = case(golden("init_general"), name)
    n, m = c["y"].shape
    data = gk.ResponseMatrix(c["y"].astype(float))
    covs = gk.CovariateSet(x=c["x"] if c["x"].shape[1] else None,
                           z=c["z"] if c["z"].shape[1] else None, n=n, m=m)
    st, info = gk.init_glm_svd(data, covs, gk.family(str(c["family"])), gk.link(str(c["link"])),
                               int(c["d"]), seed=5, return_info=True)
    assert str(info.get("glm_fallbacks", {})) == str(c["fallbacks"])
    assert normwise(st.b, c["b"]) < 1e-7
    if c["gamma"].size:
        assert normwise(st.gamma, c["gamma"]) < 1e-7
    assert normwise(st.u @ st.v.T, c["uv"]) < 1e-6
    assert st.phi == pytest.approx(float(c["phi"]), rel=1e-8)


def test_fit_asgd_rank_only_general_family():
    """fit_asgd(rank=d) for a non-count family: GLM-SVD start, then general mode."""
    c = case(golden("init_general"), "gamma_log")
    n, m = c["y"].shape
    data = gk.ResponseMatrix(c["y"].astype(float))
    covs = gk.CovariateSet(x=c["x"], n=n, m=m)
    cfg = gk.SgdConfig(max_epochs=6, mb_rows=80, mb_cols=m, tol=1e-30, seed=5)
    final, rep = gk.fit_asgd(data, covs, gk.Gamma(), gk.Log(), gk.PenaltyConfig(), cfg,
                             rank=int(c["d"]))
    assert rep.epochs_run == 6 and np.all(np.isfinite(rep.objective_trace))
    assert rep.phi_trace[0] == pytest.approx(float(c["phi"]), rel=1e-8)
    assert rep.phi_trace[-1] != rep.phi_trace[0]


@pytest.mark.parametrize("name", ["gauss_id", "gamma_log", "bern_logit", "gamma_inv", "ig_log"])
def test_model_selection_general_family(name):
    """information_criteria (with the family's dispersion constant), mu_at and
    held-out scores for non-count families / links (select.py:57-96, 141-145;
    metrics.py:35-55) against the oracle."""
    from paper_2412_20509_b200.select import heldout_scores, information_criteria, mu_at
    c = case(golden("general"), name)
    data, covs, fam, lnk, cfg, _ = _setup(c)
    st = gk.FactorizationState(c["unproj_b"], c["unproj_gamma"], c["unproj_u"], c["unproj_v"],
                               float(c["unproj_phi"]), 1.0)
    pb = orc.OProblem(c["y"].astype(float), c["x"], c["z"])
    ost = orc.OState(st.b, st.gamma, st.u, st.v, st.phi, 1.0)
    fc, lc = orc.FAMILY_CODES[fam.kind], orc.LINK_CODES[lnk.kind]
    aic, bic = information_criteria(st, data, covs, fam, lnk)
    oaic, obic = orc.information_criteria(ost, pb, fc, lc, 1.0)
    assert abs(aic - oaic) < 1e-10 * abs(oaic) and abs(bic - obic) < 1e-10 * abs(obic)
    rng = np.random.default_rng(9)
    rows, cols = rng.integers(0, c["y"].shape[0], 500), rng.integers(0, c["y"].shape[1], 500)
    mu = mu_at(st, covs, lnk, rows, cols)
    omu = orc.mu_at(ost, pb, lc, rows, cols)
    assert normwise(mu, omu) < 1e-12
    y_test = c["y"][rows, cols].astype(float)
    ybar = float(c["y"].mean())
    res = heldout_scores(st, covs, fam, lnk, rows, cols, y_test, ybar)
    assert res.rel_deviance == pytest.approx(orc.rel_deviance(fc, y_test, omu, ybar, 1.0), rel=1e-10)
    assert gk.rel_deviance(y_test, omu, ybar, fam) == pytest.approx(res.rel_deviance, rel=1e-10)


@pytest.mark.parametrize("name", ["gauss_id", "gamma_log", "bern_logit", "ig_log"])
@pytest.mark.parametrize("dtype,tol", [("f64", 1e-9), ("f32", 1e-3)])
def test_general_fit_with_unobserved_entries(name, dtype, tol):
    """General mode on a masked response (a hole is its imputed mean with the
    last mantissa bit set, refilled on the device every nafill_every steps;
    optim.py:368-374, 430-436) against the reference's own fits
    (make_golden.py general_masked)."""
    c = case(golden("general_masked"), name)
    n, m = c["y"].shape
    mask = c["mask"]
    data = gk.ResponseMatrix(np.where(mask, c["y"], np.nan), mask=mask)
    covs = gk.CovariateSet(x=c["x"] if c["x"].shape[1] else None,
                           z=c["z"] if c["z"].shape[1] else None, n=n, m=m)
    me, mr, mc, seed, nafill = (int(v) for v in c["cfg"])
    cfg = gk.SgdConfig(max_epochs=me, mb_rows=mr, mb_cols=mc, tol=1e-30, seed=seed,
                       nafill_every=nafill)
    st = gk.FactorizationState(c["init_b"], c["init_gamma"], c["init_u"], c["init_v"], 1.0, 1.0)
    final, rep = gk.fit_asgd(data, covs, gk.family(str(c["family"])), gk.link(str(c["link"])),
                             gk.PenaltyConfig(), cfg, st, dispersion=str(c["dispersion"]),
                             identify_mode=None, dtype=dtype)
    assert normwise(rep.objective_trace, c["trace"]) < tol
    assert normwise(rep.phi_trace, c["phi_trace"]) < tol
    assert normwise(final.u @ final.v.T, c["final_u"] @ c["final_v"].T) < 100 * tol
    fo = float(c["final_objective"])
    assert abs(rep.final_objective - fo) < tol * abs(fo)


@pytest.mark.parametrize("gold,fam,lnk", [("cv_gamma", "gamma", "log"),
                                          ("cv_gauss", "gaussian", "identity")])
def test_cv_rank_select_general_matches_reference(gold, fam, lnk):
    """cv_rank_select for non-count families: masked general-mode train fits
    with GLM-SVD starts, AIC/BIC with the family's dispersion constant over
    the observed entries, held-out deviance."""
    from paper_2412_20509_b200.select import cv_rank_select
    g = golden(gold)
    data = gk.ResponseMatrix(g["y"].astype(float))
    covs = gk.CovariateSet(x=g["x"], m=40)
    cfg = gk.SgdConfig(max_epochs=16, mb_rows=50, mb_cols=40, tol=1e-30, seed=2)
    rep = cv_rank_select(data, covs, gk.family(fam), gk.link(lnk), [1, 2, 3], folds=2, cfg=cfg,
                         seed=6)
    assert str(rep.failures) == str(g["failures"])
    assert normwise(rep.aic, g["aic"]) < 1e-6
    assert normwise(rep.bic, g["bic"]) < 1e-6
    assert normwise(np.asarray(rep.cv_deviance), g["cv"]) < 1e-5
    assert [rep.chosen[k] for k in ("cv", "aic", "bic", "scree")] == g["chosen"].tolist()
