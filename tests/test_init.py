"""OLS-SVD initialization (initialization.py:143-169).

CPU: the oracle restatement against the reference's own init_ols_svd
(tests/golden/init.npz).  GPU: the sparse, residual-free device path
(gmf_csr_spmm + gmf_init_moments behind paper_2412_20509_b200.initialization)
against the golden values and the oracle: B, Gamma and the NB shape to
1e-10 relative, U V' (the basis-free product; singular-vector signs are not
unique) to 1e-8 normwise."""
import numpy as np
import pytest

from conftest import golden, normwise
from oracle import asgd_oracle as orc

CASES = ["pois", "nb", "small", "noz"]


def _rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


def _nrm(a, b):
    if b.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


@pytest.mark.parametrize("key", CASES)
def test_oracle_init_matches_reference(key):
    g = golden("init")
    pb = orc.OProblem(g[f"{key}|y"].astype(float), g[f"{key}|x"], g[f"{key}|z"])
    fc = orc.NEG_BINOMIAL if int(g[f"{key}|nbfam"]) else orc.POISSON
    st = orc.init_ols_svd(pb, int(g[f"{key}|d"]), fc, seed=3)
    assert _nrm(st.b, g[f"{key}|b"]) < 1e-12
    assert _nrm(st.gamma, g[f"{key}|gamma"]) < 1e-12
    assert _nrm(st.u @ st.v.T, g[f"{key}|uv"]) < 1e-10
    assert _rel(st.nb_shape, float(g[f"{key}|nb_shape"])) < 1e-12


def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.gpu
@pytest.mark.parametrize("key", CASES)
@pytest.mark.parametrize("fmt", ["dense", "csr"])
def test_gpu_init_matches_reference(key, fmt):
    _need_gpu()
    import scipy.sparse as sp
    import paper_2412_20509_b200 as gk
    from paper_2412_20509_b200.initialization import init_ols_svd
    g = golden("init")
    y = g[f"{key}|y"]
    n, m = y.shape
    data = (gk.ResponseMatrix(y.astype(float)) if fmt == "dense"
            else gk.ResponseMatrix(csr=sp.csr_matrix(y), shape=(n, m)))
    x, z = g[f"{key}|x"], g[f"{key}|z"]
    covs = gk.CovariateSet(x=x if x.shape[1] else None, z=z if z.shape[1] else None, n=n, m=m)
    fam = gk.NegBinomial(1.0) if int(g[f"{key}|nbfam"]) else gk.Poisson()
    st = init_ols_svd(data, covs, fam, gk.Log(), int(g[f"{key}|d"]), seed=3)
    assert _nrm(st.b, g[f"{key}|b"]) < 1e-10
    assert _nrm(st.gamma, g[f"{key}|gamma"]) < 1e-10
    assert _nrm(st.u @ st.v.T, g[f"{key}|uv"]) < 1e-8
    np.testing.assert_allclose(np.linalg.norm(st.u, axis=0), g[f"{key}|s"], rtol=1e-9)
    assert _rel(st.nb_shape, float(g[f"{key}|nb_shape"])) < 1e-10
    assert st.phi == float(g[f"{key}|phi"])


@pytest.mark.gpu
def test_gpu_init_long_columns_against_oracle():
    """c3-shaped counts (20,000 x 1,000, p=2, q=1, d=10, ~90 % zeros): CSC
    columns of ~2,000 nonzeros exercise the segmented S' Q path."""
    _need_gpu()
    import scipy.sparse as sp
    import paper_2412_20509_b200 as gk
    from paper_2412_20509_b200.initialization import init_ols_svd
    rng = np.random.default_rng(11)
    n, m, d = 20_000, 1_000, 10
    x = np.hstack([np.ones((n, 1)), rng.integers(0, 2, (n, 1)).astype(float)])
    z = np.ones((m, 1))
    eta = (rng.normal(0, 0.5, (n, d)) @ rng.normal(0, 0.5, (m, d)).T
           + x @ np.column_stack([rng.normal(-3.2, 0.5, m), rng.normal(0, 0.3, m)]).T)
    y = rng.poisson(rng.gamma(2.0, np.exp(eta) / 2.0)).astype(np.int32)
    data = gk.ResponseMatrix(csr=sp.csr_matrix(y), shape=(n, m))
    st = init_ols_svd(data, gk.CovariateSet(x=x, z=z), gk.NegBinomial(1.0), gk.Log(), d, seed=0)
    ost = orc.init_ols_svd(orc.OProblem(y.astype(float), x, z), d, orc.NEG_BINOMIAL, seed=0)
    assert _nrm(st.b, ost.b) < 1e-10
    assert _nrm(st.gamma, ost.gamma) < 1e-10
    assert _nrm(st.u @ st.v.T, ost.u @ ost.v.T) < 1e-8
    assert _rel(st.nb_shape, ost.nb_shape) < 1e-10


@pytest.mark.gpu
def test_gpu_init_feeds_fit():
    """init -> fit_asgd on the device, the reference's usual pipeline."""
    _need_gpu()
    import paper_2412_20509_b200 as gk
    from paper_2412_20509_b200.initialization import init_ols_svd
    g = golden("init")
    y = g["nb|y"]
    data = gk.ResponseMatrix(y.astype(float))
    covs = gk.CovariateSet(x=g["nb|x"], z=g["nb|z"])
    fam = gk.NegBinomial(1.0)
    st0 = init_ols_svd(data, covs, fam, gk.Log(), 5, seed=3)
    cfg = gk.SgdConfig(max_epochs=20, mb_rows=100, mb_cols=60, tol=1e-30, seed=0)
    st, rep = gk.fit_asgd(data, covs, gk.NegBinomial(st0.nb_shape), gk.Log(), gk.PenaltyConfig(),
                          cfg, init_state=st0)
    assert np.isfinite(rep.objective_trace).all()
    assert rep.objective_trace[-1] < rep.objective_trace[0]


def test_init_rejects_out_of_scope():
    import paper_2412_20509_b200 as gk
    from paper_2412_20509_b200.initialization import InitMethod, init_ols_svd
    y = np.ones((4, 3))
    covs = gk.CovariateSet(n=4, m=3)
    with pytest.raises(gk.ConfigError):
        init_ols_svd(gk.ResponseMatrix(y), covs, gk.Poisson(), gk.Log(), 5)
    with pytest.raises(gk.ConfigError):
        InitMethod(residual_kind="bogus")
    with pytest.raises(NotImplementedError):
        init_ols_svd(gk.ResponseMatrix(y), covs, gk.Gaussian(), gk.Identity(), 1)


@pytest.mark.gpu
def test_gpu_init_wide_sketch_against_oracle():
    """d = 25: the sketch has k + 10 = 35 > 32 columns, so every sparse
    product takes two lane passes; Poisson, dense input, q = 1."""
    _need_gpu()
    import paper_2412_20509_b200 as gk
    from paper_2412_20509_b200.initialization import init_ols_svd
    rng = np.random.default_rng(23)
    n, m, d = 3_000, 200, 25
    x = np.ones((n, 1))
    z = rng.normal(0, 1, (m, 1))
    eta = rng.normal(0, 0.3, (n, 4)) @ rng.normal(0, 0.3, (m, 4)).T + rng.normal(0.2, 0.5, m)
    y = rng.poisson(np.exp(eta)).astype(np.int32)
    st = init_ols_svd(gk.ResponseMatrix(y.astype(float)), gk.CovariateSet(x=x, z=z),
                      gk.Poisson(), gk.Log(), d, seed=5)
    ost = orc.init_ols_svd(orc.OProblem(y.astype(float), x, z), d, orc.POISSON, seed=5)
    assert _nrm(st.b, ost.b) < 1e-10
    assert _nrm(st.gamma, ost.gamma) < 1e-10
    assert _nrm(st.u @ st.v.T, ost.u @ ost.v.T) < 1e-8
    assert st.nb_shape == 1.0
