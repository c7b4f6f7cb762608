"""Pin the oracle's general families / links and its Pearson dispersion update
against the reference's own fits (tests/golden/general.npz, written by
make_golden.py::make_general from gmfkit: families.py:267-441 with the links
of :98-210, optim.py:175-202).  CPU only."""
import numpy as np
import pytest

from conftest import golden, normwise
from oracle import asgd_oracle as orc

CASES = ["gauss_id", "gamma_log", "bern_logit", "ig_log", "qpois", "gamma_inv", "pois_id"]


def case(g, name):
    pre = f"{name}__"
    return {k[len(pre):]: g[k] for k in g.files if k.startswith(pre)}


def est_phi_of(c):
    fam, disp = str(c["family"]), str(c["dispersion"])
    if disp == "fixed":
        return False
    if disp == "estimate":
        return fam != "neg_binomial"
    return fam in ("gaussian", "gamma", "inverse_gaussian")


def test_cases_listed():
    assert sorted(golden("general")["cases"].tolist()) == sorted(CASES)


@pytest.mark.parametrize("name", CASES)
def test_oracle_general_fit_matches_reference(name):
    c = case(golden("general"), name)
    pb = orc.OProblem(c["y"].astype(float), c["x"], c["z"])
    fc, lc = orc.FAMILY_CODES[str(c["family"])], orc.LINK_CODES[str(c["link"])]
    me, mr, mc, seed = (int(v) for v in c["cfg"])
    cfg = orc.OConfig(max_epochs=me, mb_rows=mr, mb_cols=mc, tol=1e-30, seed=seed)
    init = orc.OState(c["init_b"].copy(), c["init_gamma"].copy(), c["init_u"].copy(),
                      c["init_v"].copy(), 1.0, 1.0)
    seen = {}

    def cb(t, st):
        if t in set(c["check_steps"].tolist()):
            seen[t] = st.copy()

    lam = (0.0, 0.0, 1.0, 0.0)   # PenaltyConfig() defaults (model.py:193-226)
    final, rep = orc.fit_asgd(pb, fc, lc, lam, cfg, init, est_alpha=False,
                              est_phi=est_phi_of(c), callback=cb)
    assert rep.epochs_run == int(c["epochs_run"])
    assert normwise(rep.objective_trace, c["trace"]) < 1e-11
    assert normwise(rep.phi_trace, c["phi_trace"]) < 1e-11
    assert seen
    for t, st in seen.items():
        for blk in ("b", "gamma", "u", "v"):
            assert normwise(getattr(st, blk), c[f"step{t}_{blk}"]) < 1e-10, (t, blk)
        assert abs(st.phi - float(c[f"step{t}_phi"])) < 1e-11 * float(c[f"step{t}_phi"])
    assert normwise(final.u @ final.v.T, c["final_u"] @ c["final_v"].T) < 1e-9
    assert abs(rep.final_objective - float(c["final_objective"])) < 1e-10 * abs(float(c["final_objective"]))


@pytest.mark.parametrize("name", CASES)
def test_oracle_general_step0_gradient(name):
    c = case(golden("general"), name)
    pb = orc.OProblem(c["y"].astype(float), c["x"], c["z"])
    fc, lc = orc.FAMILY_CODES[str(c["family"])], orc.LINK_CODES[str(c["link"])]
    me, mr, mc, seed = (int(v) for v in c["cfg"])
    cfg = orc.OConfig(max_epochs=me, mb_rows=mr, mb_cols=mc, tol=1e-30, seed=seed)
    rb, cb, _, seq = orc.replay_schedule(pb.n, pb.m, cfg, n_steps=1)
    assert seq[0] == int(c["first_block"])
    init = orc.OState(c["init_b"], c["init_gamma"], c["init_u"], c["init_v"], 1.0, 1.0)
    gp = orc.minibatch_gradients(init, pb, rb[seq[0]], cb[0], fc, lc, (0.0, 0.0, 1.0, 0.0))
    for mine, key in ((gp.g_row, "g0_g_row"), (gp.h_row, "g0_h_row"),
                      (gp.g_col, "g0_g_col"), (gp.h_col, "g0_h_col")):
        assert normwise(mine, c[key]) < 1e-12, key
