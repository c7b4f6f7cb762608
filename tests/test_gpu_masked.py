"""GPU parity with unobserved entries: the working response is imputed at the
initial state and refilled with the step's mean every nafill_every steps
(gmfkit optim.py:368-374, 430-436), the tracked objective and the final
deviance skip the holes, and a standalone minibatch gradient masks them
(gradients.py:66-88).  Goldens: the reference itself (make_golden.py
masked, masked_p3)."""
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


def _setup(g):
    me, mr, mc, seed, cap = (int(v) for v in g["cfg"])
    k0, k1, tau, a1, a2, damp, tol = (float(v) for v in g["cfg_f"])
    cfg = gk.SgdConfig(max_epochs=me, rate_k0=k0, rate_k1=k1, rate_tau=tau, mb_rows=mr,
                       mb_cols=mc, smooth_a1=a1, smooth_a2=a2, damping=damp, tol=tol,
                       seed=seed, max_eval_entries=cap, nafill_every=int(g["nafill"]))
    mask = g["mask"]
    y = np.where(mask, g["y"].astype(float), np.nan)
    data = gk.ResponseMatrix(y, mask=mask)
    n, m = y.shape
    covs = gk.CovariateSet(x=g["x"] if g["x"].shape[1] else None,
                           z=g["z"] if g["z"].shape[1] else None, n=n, m=m)
    off = g["offset"] if "offset" in g.files else None
    fam = (gk.NegBinomial(float(g["init_nb"])) if str(g["family"]) == "neg_binomial"
           else gk.Poisson())
    st = gk.FactorizationState(g["init_b"], g["init_gamma"], g["init_u"], g["init_v"],
                               float(g["init_phi"]), float(g["init_nb"]))
    pen = gk.PenaltyConfig(lam=1.0, blocks=tuple(float(v) for v in g["lam"]))
    return data, covs, off, fam, st, pen, cfg


@pytest.mark.parametrize("name", ["masked", "masked_p3"])
def test_masked_fit_trajectory_fp64(name):
    g = golden(name)
    data, covs, off, fam, st, pen, cfg = _setup(g)
    seen = {}
    checks = set(g["check_steps"].tolist())

    def cb(t, s):
        if t in checks:
            seen[t] = s.copy()

    final, rep = gk.fit_asgd(data, covs, fam, gk.Log(), pen, cfg, st, callback=cb, offset=off,
                             dtype="f64")
    assert rep.diagnostics["iterations"] == int(g["iterations"])
    assert normwise(rep.objective_trace, g["trace"]) < 1e-11
    assert normwise(rep.nb_shape_trace, g["nb_trace"]) < 1e-11
    assert seen.keys() == checks
    for t, s in seen.items():
        for blk in ("b", "gamma", "u", "v"):
            assert normwise(getattr(s, blk), g[f"step{t}_{blk}"]) < 1e-9, (t, blk)
    ref_uv = g["final_u"] @ g["final_v"].T
    assert normwise(final.u @ final.v.T, ref_uv) < 1e-9
    assert rep.final_objective == pytest.approx(float(g["final_objective"]), rel=1e-10)


@pytest.mark.parametrize("name", ["masked", "masked_p3"])
def test_masked_fit_fp32_within_north_star(name):
    g = golden(name)
    data, covs, off, fam, st, pen, cfg = _setup(g)
    final, rep = gk.fit_asgd(data, covs, fam, gk.Log(), pen, cfg, st, offset=off, dtype="f32")
    assert normwise(rep.objective_trace, g["trace"]) < 1e-4
    ref_uv = g["final_u"] @ g["final_v"].T
    assert normwise(final.u @ final.v.T, ref_uv) < 1e-3
    assert rep.final_objective == pytest.approx(float(g["final_objective"]), rel=1e-3)


@pytest.mark.parametrize("dtype,tol", [("f64", 1e-10), ("f32", 1e-4)])
def test_masked_standalone_gradient_drops_holes(dtype, tol):
    """minibatch_gradients on a masked response: unobserved entries carry no
    weight (gradients.py:66-88), the reference's own step-0 gradient."""
    from paper_2412_20509_b200.engine import Schedule
    g = golden("masked")
    data, covs, off, fam, st, pen, cfg = _setup(g)
    sch = Schedule(data.n, data.m, cfg, mask=data.mask, n_steps=1)
    assert int(sch.block_seq[0]) == int(g["first_block"])
    mb = gk.Minibatch(sch.row_blocks[sch.block_seq[0]], sch.col_blocks[0])
    gp = gk.minibatch_gradients(st, data, covs, fam, gk.Log(), pen, mb, offset=off, dtype=dtype)
    for mine, key in ((gp.g_rowside, "g0_g_row"), (gp.h_rowside, "g0_h_row"),
                      (gp.g_colside, "g0_g_col"), (gp.h_colside, "g0_h_col")):
        assert normwise(mine, g[key]) < tol, (key, normwise(mine, g[key]))
