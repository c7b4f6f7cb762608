"""check_constraints (identify.py:141-188) on the reference's own B2/B3
projections (tests/golden/project_b23.npz): host-only, CPU."""
import pytest

from conftest import golden

gk = pytest.importorskip("paper_2412_20509_b200")


@pytest.mark.parametrize("mode", ["B2", "B3"])
def test_check_constraints_on_reference_projections(mode):
    g = golden("project_b23")
    for k in range(3):
        p = f"{k}|{mode}"
        st = gk.FactorizationState(g[f"{p}_b"], g[f"{p}_gamma"], g[f"{p}_u"], g[f"{p}_v"])
        covs = gk.CovariateSet(x=g[f"{k}|x"], z=g[f"{k}|z"])
        rep = gk.check_constraints(st, covs, mode)
        assert rep["normalization"] < 1e-8, rep
        assert max(rep.values()) < 1e-8, rep
        st_in = gk.FactorizationState(g[f"{k}|in_b"], g[f"{k}|in_gamma"], g[f"{k}|in_u"],
                                      g[f"{k}|in_v"])
        assert gk.check_constraints(st_in, covs, mode)["normalization"] > 1e-3


def test_check_constraints_unknown_mode():
    g = golden("project_b23")
    st = gk.FactorizationState(g["0|B3_b"], g["0|B3_gamma"], g["0|B3_u"], g["0|B3_v"])
    with pytest.raises(gk.ConfigError):
        gk.check_constraints(st, gk.CovariateSet(x=g["0|x"], z=g["0|z"]), "B4")
