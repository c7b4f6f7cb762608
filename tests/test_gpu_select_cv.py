"""cv_rank_select on the GPU (gmfkit select.py:148-237): holdout masks,
device fits of the train matrices (holes imputed on the device, GLM-SVD start,
warm starts over ranks), AIC/BIC and held-out relative deviance, the scree
pick -- against the reference's own run (make_golden.py cv)."""
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


def test_cv_rank_select_matches_reference():
    from paper_2412_20509_b200.select import cv_rank_select, scree_eigenvalues
    g = golden("cv")
    data = gk.ResponseMatrix(g["y"].astype(float))
    covs = gk.CovariateSet(x=g["x"], m=50)
    cfg = gk.SgdConfig(max_epochs=20, mb_rows=60, mb_cols=50, tol=1e-30, seed=1)
    rep = cv_rank_select(data, covs, gk.NegBinomial(1.5), gk.Log(), [1, 2, 3], folds=2, cfg=cfg,
                         seed=5)
    assert str(rep.failures) == str(g["failures"])
    assert normwise(rep.aic, g["aic"]) < 1e-7
    assert normwise(rep.bic, g["bic"]) < 1e-7
    assert normwise(np.asarray(rep.cv_deviance), g["cv"]) < 1e-6
    assert [rep.chosen[k] for k in ("cv", "aic", "bic", "scree")] == g["chosen"].tolist()
    assert normwise(rep.scree_eigenvalues, g["scree"]) < 1e-9
    assert normwise(scree_eigenvalues(data, covs, 4), g["scree4"]) < 1e-9


def test_holdout_mask_is_the_references():
    from paper_2412_20509_b200.select import holdout_mask
    g = golden("cv")
    data = gk.ResponseMatrix(g["y"].astype(float))
    train, (r, c) = holdout_mask(data, 0.3, seed=5)
    assert r.size == int(np.floor(0.3 * data.n * data.m))
    assert not train.mask[r, c].any() and train.mask.sum() == data.n * data.m - r.size


def test_block_helpers_match_reference():
    """linear_predictor, impute_block, update_nb_shape_stochastic (model.py:229-256,
    optim.py:205-245) against the reference's outputs (make_golden.py api)."""
    g = golden("api")
    data = gk.ResponseMatrix(np.where(g["mask"], g["y"], np.nan), mask=g["mask"], weights=g["w"])
    covs = gk.CovariateSet(x=g["x"], z=g["z"])
    st = gk.FactorizationState(g["st_b"], g["st_gamma"], g["st_u"], g["st_v"], 1.0, 1.5)
    mb = gk.Minibatch(g["I"], g["J"])
    assert normwise(gk.linear_predictor(st, covs, g["I"], g["J"]), g["eta"]) < 1e-14
    assert normwise(gk.linear_predictor(st, covs), g["eta_all"]) < 1e-14
    assert normwise(gk.impute_block(st, data, covs, gk.Log(), mb), g["block"]) < 1e-14
    nb = gk.update_nb_shape_stochastic(st, data, mb, 0.3, covs=covs, lnk=gk.Log())
    assert nb == pytest.approx(float(g["nb"]), rel=1e-12)
