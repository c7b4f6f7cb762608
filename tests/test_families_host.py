"""families.py mirrors gmfkit/families.py: domain checks, variance / deviance
/ link algebra against the oracle's restated formulas (pinned to the
reference by test_oracle_golden.py::seam and test_general_oracle.py)."""
import numpy as np
import pytest

import paper_2412_20509_b200 as gk
from oracle import asgd_oracle as orc


@pytest.mark.parametrize("kind", ["gaussian", "gamma", "inverse_gaussian", "poisson",
                                  "bernoulli", "neg_binomial"])
def test_family_algebra(kind):
    rng = np.random.default_rng(1)
    fam = gk.family(kind, nb_shape=1.7)
    fc = orc.FAMILY_CODES[kind]
    mu = rng.uniform(0.05, 0.95, 50)
    y = {"gaussian": rng.normal(0, 1, 50), "gamma": rng.gamma(2, 1, 50),
         "inverse_gaussian": rng.wald(1.0, 2.0, 50), "poisson": rng.poisson(2, 50).astype(float),
         "bernoulli": rng.integers(0, 2, 50).astype(float),
         "neg_binomial": rng.poisson(3, 50).astype(float)}[kind]
    np.testing.assert_allclose(fam.variance(mu), orc._variance(fc, mu, 1.7), rtol=1e-14)
    np.testing.assert_allclose(fam.unit_deviance(y, mu, 2.0),
                               2.0 * orc.unit_deviance(fc, y, mu, 1.7), rtol=1e-12, atol=1e-14)
    h = 1e-6
    num = (fam.variance(mu + h) - fam.variance(mu - h)) / (2 * h)
    np.testing.assert_allclose(fam.dvariance(mu), num, rtol=1e-6, atol=1e-8)
    s = fam.sample(np.full(2000, 0.5), phi=0.5, rng=np.random.default_rng(0))
    assert abs(s.mean() - 0.5) < 0.1
    assert fam == gk.family(kind, nb_shape=1.7) and hash(fam) == hash(gk.family(kind, nb_shape=1.7))


@pytest.mark.parametrize("kind", ["identity", "log", "logit", "inverse", "inverse_squared"])
def test_link_algebra(kind):
    lnk = gk.link(kind)
    lc = orc.LINK_CODES[kind]
    mu = np.random.default_rng(2).uniform(0.05, 0.95, 40)
    eta = lnk.eval(mu)
    np.testing.assert_allclose(lnk.inverse(eta), mu, rtol=1e-12)
    np.testing.assert_allclose(lnk.inverse(eta), orc.mean_of_eta(lc, eta), rtol=1e-12)
    np.testing.assert_allclose(lnk.deriv1(mu), orc._link_d1(lc, mu), rtol=1e-13)
    h = 1e-6
    np.testing.assert_allclose(lnk.deriv2(mu), (lnk.deriv1(mu + h) - lnk.deriv1(mu - h)) / (2 * h),
                               rtol=1e-5, atol=1e-6)


def test_domain_errors_and_canonical_links():
    with pytest.raises(gk.DomainError):
        gk.Gamma().check_y(np.array([1.0, 0.0]))
    with pytest.raises(gk.DomainError):
        gk.Bernoulli().check_mu(np.array([0.2, 1.0]))
    with pytest.raises(gk.DomainError):
        gk.Log().eval(np.array([-1.0]))
    with pytest.raises(gk.DomainError):
        gk.InverseSquared().inverse(np.array([0.0]))
    with pytest.raises(gk.DomainError):
        gk.family("tweedie")
    with pytest.raises(gk.DomainError):
        gk.Poisson().unit_deviance(np.array([1.0]), np.array([1.0]), w=0.0)
    pairs = {"gaussian": "identity", "gamma": "inverse", "inverse_gaussian": "inverse_squared",
             "poisson": "log", "bernoulli": "logit", "neg_binomial": "log"}
    for f, l in pairs.items():
        assert gk.canonical_link(gk.family(f)).kind == l
