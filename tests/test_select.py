"""Model selection on the deviance kernels:
information_criteria (select.py:81-96), _mu_at (select.py:141-145),
rel_deviance / rel_log_rmse (metrics.py:35-55).

CPU: the oracle restatement against the reference's own outputs
(tests/golden/select.npz).  GPU: the CUDA path through the C ABI against the
golden values and the oracle, dense and CSR, fp64 (1e-10 relative) and fp32
(1e-4 relative, the north star's fp32 bound)."""
import numpy as np
import pytest

from conftest import golden
from oracle import asgd_oracle as orc

CASES = ["pois", "nb", "nbw", "nb50"]


def _ostate(g, key):
    p = f"{key}|st"
    return orc.OState(g[f"{p}_b"], g[f"{p}_gamma"], g[f"{p}_u"], g[f"{p}_v"],
                      float(g[f"{p}_phi"]), float(g[f"{p}_nb"]))


def _oproblem(g, key):
    w = g[f"{key}|w"] if f"{key}|w" in g.files else None
    return orc.OProblem(g[f"{key}|y"].astype(float), g[f"{key}|x"], g[f"{key}|z"], w=w)


def _fcode(key):
    return orc.POISSON if key == "pois" else orc.NEG_BINOMIAL


def _rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


@pytest.mark.parametrize("key", CASES)
def test_oracle_information_criteria_matches_reference(key):
    g = golden("select")
    st, pb = _ostate(g, key), _oproblem(g, key)
    aic, bic = orc.information_criteria(st, pb, _fcode(key), orc.LOG, float(g[f"{key}|alpha"]))
    assert _rel(aic, float(g[f"{key}|aic"])) < 1e-12
    assert _rel(bic, float(g[f"{key}|bic"])) < 1e-12


@pytest.mark.parametrize("key", CASES)
def test_oracle_heldout_metrics_match_reference(key):
    g = golden("select")
    st, pb = _ostate(g, key), _oproblem(g, key)
    rows, cols = g[f"{key}|rows"], g[f"{key}|cols"]
    mu = orc.mu_at(st, pb, orc.LOG, rows, cols)
    np.testing.assert_allclose(mu, g[f"{key}|mu_test"], rtol=1e-13)
    yt = pb.y[rows, cols]
    ybar = float(g[f"{key}|ybar"])
    alpha = float(g[f"{key}|alpha"])
    assert _rel(orc.rel_deviance(_fcode(key), yt, mu, ybar, alpha), float(g[f"{key}|rel_dev"])) < 1e-12
    assert _rel(orc.rel_log_rmse(yt, mu, ybar), float(g[f"{key}|rel_lrmse"])) < 1e-12


def test_select_api_exports():
    gk = pytest.importorskip("paper_2412_20509_b200")
    from paper_2412_20509_b200 import metrics, select
    for name in ("information_criteria", "loglik_terms", "mu_at", "heldout_scores"):
        assert callable(getattr(select, name))
    for name in ("rel_deviance", "rel_log_rmse", "score_sums"):
        assert callable(getattr(metrics, name))
    with pytest.raises(gk.ConfigError):
        metrics._check_args(np.zeros(0), np.zeros(0))
    with pytest.raises(gk.ConfigError):
        metrics._check_args(np.zeros(3), np.zeros(2))
    with pytest.raises(gk.DegenerateError):
        metrics.ratios(np.array([1.0, 0.0, 1.0, 1.0]))


# ------------------------------------------------------------------- GPU --

def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _gk_case(g, key, csr=False):
    import paper_2412_20509_b200 as gk
    import scipy.sparse as sp
    y = g[f"{key}|y"]
    n, m = y.shape
    w = g[f"{key}|w"] if f"{key}|w" in g.files else None
    if csr:
        data = gk.ResponseMatrix(csr=sp.csr_matrix(y), shape=(n, m))
    else:
        data = gk.ResponseMatrix(y.astype(float), weights=w)
    x, z = g[f"{key}|x"], g[f"{key}|z"]
    covs = gk.CovariateSet(x=x if x.shape[1] else None, z=z if z.shape[1] else None, n=n, m=m)
    p = f"{key}|st"
    st = gk.FactorizationState(g[f"{p}_b"], g[f"{p}_gamma"], g[f"{p}_u"], g[f"{p}_v"],
                               float(g[f"{p}_phi"]), float(g[f"{p}_nb"]))
    fam = gk.Poisson() if key == "pois" else gk.NegBinomial(float(g[f"{key}|alpha"]))
    return gk, data, covs, st, fam


@pytest.mark.gpu
@pytest.mark.parametrize("key", CASES)
@pytest.mark.parametrize("dtype,tol", [("f64", 1e-10), ("f32", 1e-4)])
def test_gpu_information_criteria(key, dtype, tol):
    _need_gpu()
    from paper_2412_20509_b200 import select
    g = golden("select")
    gk, data, covs, st, fam = _gk_case(g, key)
    aic, bic = select.information_criteria(st, data, covs, fam, gk.Log(), dtype=dtype)
    assert _rel(aic, float(g[f"{key}|aic"])) < tol
    assert _rel(bic, float(g[f"{key}|bic"])) < tol


@pytest.mark.gpu
@pytest.mark.parametrize("key", ["pois", "nb", "nb50"])
def test_gpu_information_criteria_csr_equals_dense(key):
    _need_gpu()
    from paper_2412_20509_b200 import select
    g = golden("select")
    gk, data, covs, st, fam = _gk_case(g, key)
    _, cdata, _, _, _ = _gk_case(g, key, csr=True)
    d1, c1 = select.loglik_terms(st, data, covs, fam, gk.Log())
    d2, c2 = select.loglik_terms(st, cdata, covs, fam, gk.Log())
    assert _rel(d2, d1) < 1e-12
    assert (c1 == 0.0 and c2 == 0.0) if key == "pois" else _rel(c2, c1) < 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("key", CASES)
@pytest.mark.parametrize("dtype,tol", [("f64", 1e-10), ("f32", 1e-4)])
def test_gpu_heldout_scores(key, dtype, tol):
    _need_gpu()
    from paper_2412_20509_b200 import metrics, select
    g = golden("select")
    gk, data, covs, st, fam = _gk_case(g, key)
    rows, cols = g[f"{key}|rows"], g[f"{key}|cols"]
    mu = select.mu_at(st, covs, gk.Log(), rows, cols, dtype=dtype)
    ref_mu = g[f"{key}|mu_test"]
    assert np.max(np.abs(mu - ref_mu)) / np.max(np.abs(ref_mu)) < tol
    yt = g[f"{key}|y"][rows, cols].astype(float)
    ybar = float(g[f"{key}|ybar"])
    res = select.heldout_scores(st, covs, fam, gk.Log(), rows, cols, yt, ybar, dtype=dtype)
    assert res.n_test == rows.size
    assert _rel(res.rel_deviance, float(g[f"{key}|rel_dev"])) < tol
    assert _rel(res.rel_log_rmse, float(g[f"{key}|rel_lrmse"])) < tol
    # metrics on device arrays (the seam form of metrics.py)
    assert _rel(metrics.rel_deviance(yt, ref_mu, ybar, fam), float(g[f"{key}|rel_dev"])) < 1e-12
    assert _rel(metrics.rel_log_rmse(yt, ref_mu, ybar), float(g[f"{key}|rel_lrmse"])) < 1e-12


@pytest.mark.gpu
def test_gpu_heldout_errors():
    _need_gpu()
    from paper_2412_20509_b200 import metrics, select
    g = golden("select")
    gk, data, covs, st, fam = _gk_case(g, "nb")
    with pytest.raises(gk.ConfigError):
        select.heldout_scores(st, covs, fam, gk.Log(), [], [], [], 1.0)
    with pytest.raises(gk.ConfigError):
        select.mu_at(st, covs, gk.Log(), [0, 1], [0])
    with pytest.raises(gk.ConfigError):
        select.mu_at(st, covs, gk.Log(), [st.n], [0])
    y = np.full(5, 2.0)
    with pytest.raises(gk.DegenerateError):
        metrics.rel_deviance(y, y + 1.0, 2.0, fam)


@pytest.mark.gpu
def test_gpu_information_criteria_c3_scale_against_oracle():
    """A c3-shaped (NB, p=2, q=1, d=10, CSR ~90 % zeros) 20,000 x 1,000 state:
    AIC/BIC through one streaming pass vs the oracle in fp64."""
    _need_gpu()
    import paper_2412_20509_b200 as gk
    from paper_2412_20509_b200 import select
    import scipy.sparse as sp
    rng = np.random.default_rng(7)
    n, m, d = 20_000, 1_000, 10
    x = np.hstack([np.ones((n, 1)), rng.integers(0, 2, (n, 1)).astype(float)])
    z = np.ones((m, 1))
    u, v = rng.normal(0, 0.5, (n, d)), rng.normal(0, 0.5, (m, d))
    b = np.column_stack([rng.normal(-3.2, 0.5, m), rng.normal(0, 0.3, m)])
    gam = rng.normal(0, 0.2, (n, 1))
    eta = u @ v.T + x @ b.T + gam @ z.T
    alpha = 2.5
    y = rng.poisson(rng.gamma(alpha, np.exp(eta) / alpha)).astype(np.int32)
    st = gk.FactorizationState(b, gam, u, v, 1.0, alpha)
    covs = gk.CovariateSet(x=x, z=z)
    data = gk.ResponseMatrix(csr=sp.csr_matrix(y), shape=(n, m))
    fam = gk.NegBinomial(alpha)
    aic, bic = select.information_criteria(st, data, covs, fam, gk.Log())
    ost = orc.OState(b, gam, u, v, 1.0, alpha)
    oaic, obic = orc.information_criteria(ost, orc.OProblem(y.astype(float), x, z),
                                          orc.NEG_BINOMIAL, orc.LOG, alpha)
    assert _rel(aic, oaic) < 1e-10 and _rel(bic, obic) < 1e-10


@pytest.mark.gpu
@pytest.mark.parametrize("dtype,tol", [("f64", 1e-10), ("f32", 1e-4)])
def test_gpu_selection_with_offset_against_oracle(dtype, tol):
    """c4-style model (intercept-only X, per-row log-library offset, CSR),
    the SURVEY §8c offset shim on both sides; large counts with a small NB
    shape stress the zero-grid identity D(0, mu) = 2 alpha log1p(mu / alpha)."""
    _need_gpu()
    import scipy.sparse as sp
    import paper_2412_20509_b200 as gk
    from paper_2412_20509_b200 import select
    rng = np.random.default_rng(17)
    n, m, d, alpha = 3_000, 500, 10, 0.4
    x = np.ones((n, 1))
    off = rng.normal(0, 0.7, n)
    u, v = rng.normal(0, 0.3, (n, d)), rng.normal(0, 0.3, (m, d))
    b = rng.normal(-1.0, 1.0, (m, 1))
    eta = u @ v.T + x @ b.T + off[:, None]
    y = rng.poisson(rng.gamma(alpha, np.exp(eta) / alpha)).astype(np.int32)
    st = gk.FactorizationState(b, np.zeros((n, 0)), u, v, 1.0, alpha)
    covs = gk.CovariateSet(x=x, m=m)
    data = gk.ResponseMatrix(csr=sp.csr_matrix(y), shape=(n, m))
    fam = gk.NegBinomial(alpha)
    pb = orc.OProblem(y.astype(float), x, np.zeros((m, 0)), offset=off)
    ost = orc.OState(b, np.zeros((n, 0)), u, v, 1.0, alpha)
    aic, bic = select.information_criteria(st, data, covs, fam, gk.Log(), offset=off, dtype=dtype)
    oaic, obic = orc.information_criteria(ost, pb, orc.NEG_BINOMIAL, orc.LOG, alpha)
    assert _rel(aic, oaic) < tol and _rel(bic, obic) < tol
    rows, cols = rng.integers(0, n, 20_000), rng.integers(0, m, 20_000)
    mu_o = orc.mu_at(ost, pb, orc.LOG, rows, cols)
    mu_g = select.mu_at(st, covs, gk.Log(), rows, cols, offset=off, dtype=dtype)
    assert np.max(np.abs(mu_g - mu_o)) / np.max(mu_o) < tol
    yt = y[rows, cols].astype(float)
    ybar = float(y.mean())
    res = select.heldout_scores(st, covs, fam, gk.Log(), rows, cols, yt, ybar, offset=off,
                                dtype=dtype)
    assert _rel(res.rel_deviance, orc.rel_deviance(orc.NEG_BINOMIAL, yt, mu_o, ybar, alpha)) < tol
    assert _rel(res.rel_log_rmse, orc.rel_log_rmse(yt, mu_o, ybar)) < tol
