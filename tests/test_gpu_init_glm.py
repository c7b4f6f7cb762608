"""init_glm_svd on the GPU (gmfkit initialization.py:172-214, glm.py:68-133)
against the reference's own outputs (make_golden.py init_glm): batched Fisher
scoring with step halving for B, Gamma and V, the deviance / Pearson
residual SVD, masked and weighted responses; and fit_asgd(rank=d) taking it
as its start (optim.py:359-366)."""
import numpy as np
import pytest

from conftest import golden, normwise

pytestmark = pytest.mark.gpu

gk = pytest.importorskip("paper_2412_20509_b200")


@pytest.fixture(autouse=True)
def _gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _case(g, key):
    y = g[f"{key}|y"]
    mask = g[f"{key}|mask"] if f"{key}|mask" in g.files else None
    w = g[f"{key}|w"] if f"{key}|w" in g.files else None
    yv = y.astype(float) if mask is None else np.where(mask, y, np.nan)
    data = gk.ResponseMatrix(yv, mask=mask, weights=w)
    covs = gk.CovariateSet(x=g[f"{key}|x"], z=g[f"{key}|z"])
    fam = gk.Poisson() if str(g[f"{key}|fam"]) == "poisson" else gk.NegBinomial(float(g[f"{key}|alpha"]))
    return data, covs, fam, int(g[f"{key}|d"]), str(g[f"{key}|rk"])


@pytest.mark.parametrize("key", ["pois", "nb", "masked", "pearson", "small"])
def test_init_glm_svd_matches_reference(key):
    from paper_2412_20509_b200.initialization import InitMethod, init_glm_svd
    g = golden("init_glm")
    data, covs, fam, d, rk = _case(g, key)
    st, info = init_glm_svd(data, covs, fam, gk.Log(), d, seed=3, return_info=True,
                            method=InitMethod(residual_kind=rk))
    assert str(info.get("glm_fallbacks", {})) == str(g[f"{key}|fallbacks"])
    assert normwise(st.b, g[f"{key}|b"]) < 1e-8
    assert normwise(st.gamma, g[f"{key}|gamma"]) < 1e-8
    assert normwise(st.u @ st.v.T, g[f"{key}|uv"]) < 1e-7
    assert st.nb_shape == pytest.approx(float(g[f"{key}|nb_shape"]), rel=1e-9)


def test_fit_asgd_rank_only_starts_from_glm_svd():
    """fit_asgd(rank=d) = fit_asgd(init_glm_svd(..., seed=cfg.seed)) (optim.py:359-366)."""
    from paper_2412_20509_b200.initialization import init_glm_svd
    g = golden("init_glm")
    data, covs, fam, d, _ = _case(g, "nb")
    cfg = gk.SgdConfig(max_epochs=8, mb_rows=100, mb_cols=data.m, tol=1e-30, seed=2)
    a, ra = gk.fit_asgd(data, covs, fam, gk.Log(), gk.PenaltyConfig(), cfg, rank=d)
    init = init_glm_svd(data, covs, fam, gk.Log(), d, seed=cfg.seed)
    b, rb = gk.fit_asgd(data, covs, fam, gk.Log(), gk.PenaltyConfig(), cfg, init)
    assert ra.objective_trace == rb.objective_trace
    np.testing.assert_array_equal(a.u @ a.v.T, b.u @ b.v.T)
