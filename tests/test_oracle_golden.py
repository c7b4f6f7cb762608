"""Pin the CPU oracle (oracle/asgd_oracle.py) against the reference's own
outputs (tests/golden/*.npz, written by tests/golden/make_golden.py from
gmfkit).  CPU only."""
import numpy as np
import pytest

from conftest import golden, normwise
from oracle import asgd_oracle as orc


def _cfg(g):
    me, mr, mc, seed, cap = (int(v) for v in g["cfg"])
    k0, k1, tau, a1, a2, damp, tol = (float(v) for v in g["cfg_f"])
    return orc.OConfig(max_epochs=me, rate_k0=k0, rate_k1=k1, rate_tau=tau, mb_rows=mr,
                       mb_cols=mc, smooth_a1=a1, smooth_a2=a2, damping=damp, tol=tol,
                       seed=seed, max_eval_entries=cap)


def _state(g, prefix):
    return orc.OState(g[f"{prefix}_b"].copy(), g[f"{prefix}_gamma"].copy(),
                      g[f"{prefix}_u"].copy(), g[f"{prefix}_v"].copy(),
                      float(g[f"{prefix}_phi"]), float(g[f"{prefix}_nb"]))


def _problem(g):
    off = g["offset"] if "offset" in g.files else None
    w = g["w"] if "w" in g.files else None
    return orc.OProblem(g["y"].astype(float), g["x"], g["z"], w=w, offset=off)


FITS = ["c1", "nb_offset", "nb_cov_s3", "converge"]


@pytest.mark.parametrize("name", FITS)
def test_oracle_fit_matches_reference(name):
    g = golden(name)
    pb = _problem(g)
    fc = orc.FAMILY_CODES[str(g["family"])]
    lam = tuple(float(v) for v in g["lam"])
    seen = {}

    def cb(t, st):
        if t in set(g["check_steps"].tolist()):
            seen[t] = st.copy()

    final, rep = orc.fit_asgd(pb, fc, orc.LOG, lam, _cfg(g), _state(g, "init"), callback=cb)
    # fp64 restatement of the same algorithm: agreement to rounding
    assert rep.epochs_run == int(g["epochs_run"])
    assert rep.converged == bool(g["converged"])
    assert rep.iterations == int(g["iterations"])
    assert normwise(rep.objective_trace, g["trace"]) < 1e-12
    assert normwise(rep.nb_shape_trace, g["nb_trace"]) < 1e-12
    for t, st in seen.items():
        ref = _state(g, f"step{t}")
        for blk in ("b", "gamma", "u", "v"):
            assert normwise(getattr(st, blk), getattr(ref, blk)) < 1e-11, (t, blk)
        assert abs(st.nb_shape - ref.nb_shape) <= 1e-12 * abs(ref.nb_shape)
    ref_final = _state(g, "final")
    assert normwise(final.u @ final.v.T, ref_final.u @ ref_final.v.T) < 1e-10
    for blk in ("b", "gamma", "u", "v"):
        assert normwise(getattr(final, blk), getattr(ref_final, blk)) < 1e-8, blk
    assert abs(rep.final_objective - float(g["final_objective"])) < 1e-10 * abs(float(g["final_objective"]))


@pytest.mark.parametrize("name", ["c1", "nb_offset", "nb_cov_s3"])
def test_oracle_step0_gradient(name):
    g = golden(name)
    pb = _problem(g)
    cfg = _cfg(g)
    rb, cb, _, seq = orc.replay_schedule(pb.n, pb.m, cfg, n_steps=1)
    assert seq[0] == int(g["first_block"])
    fc = orc.FAMILY_CODES[str(g["family"])]
    gp = orc.minibatch_gradients(_state(g, "init"), pb, rb[seq[0]], cb[0], fc, orc.LOG,
                                 tuple(float(v) for v in g["lam"]))
    for mine, key in ((gp.g_row, "g0_g_row"), (gp.h_row, "g0_h_row"),
                      (gp.g_col, "g0_g_col"), (gp.h_col, "g0_h_col")):
        assert normwise(mine, g[key]) < 1e-13, key


def test_oracle_divergence_snapshot():
    g = golden("diverge")
    pb = _problem(g)
    steps = []
    with pytest.raises(orc.OracleDivergence) as err:
        orc.fit_asgd(pb, orc.POISSON, orc.LOG, (0.0, 0.0, 1.0, 0.0), _cfg(g), _state(g, "init"),
                     callback=lambda t, s: steps.append(t))
    assert len(steps) == int(g["steps_before"])
    snap = err.value.state
    ref = _state(g, "snap")
    for blk in ("b", "u", "v"):
        assert normwise(getattr(snap, blk), getattr(ref, blk)) < 1e-12


def test_oracle_seam_formulas():
    g = golden("seam")
    keys = sorted({k.split("|")[0] for k in g.files})
    assert len(keys) == 9
    for key in keys:
        fc, lc = (int(v) for v in g[f"{key}|codes"])
        alpha = float(g[f"{key}|alpha"])
        mu = orc.mean_of_eta(lc, g[f"{key}|eta"])
        assert normwise(mu, g[f"{key}|mu"]) < 1e-14, key
        dd, hh = orc.derivs_from_mu(fc, lc, g[f"{key}|y"], mu, g[f"{key}|w"], 1.3, alpha)
        assert normwise(dd, g[f"{key}|dotd"]) < 1e-13, key
        assert normwise(hh, g[f"{key}|ddotd"]) < 1e-13, key
        dev = orc.deviance_from_mu(fc, g[f"{key}|y"], mu, g[f"{key}|w"], alpha)
        assert dev == pytest.approx(float(g[f"{key}|dev"]), rel=1e-12), key


def test_oracle_projection():
    g = golden("project")
    for k in range(3):
        st = _state(g, f"{k}|in")
        out, _ = orc.project_b1(st, g[f"{k}|x"], g[f"{k}|z"])
        ref = _state(g, f"{k}|out")
        for blk in ("b", "gamma", "u", "v"):
            assert normwise(getattr(out, blk), getattr(ref, blk)) < 1e-10, (k, blk)
    st = _state(g, "rd|in")
    out, info = orc.project_b1(st, np.zeros((10, 0)), np.zeros((6, 0)))
    assert info["effective_rank"] == int(g["rd|eff"])
    assert normwise(out.u @ out.v.T, g["rd|out_u"] @ g["rd|out_v"].T) < 1e-12


def test_oracle_weighted_gradient_and_objective():
    g = golden("weighted")
    pb = _problem(g)
    st = _state(g, "st")
    lam = tuple(float(v) for v in g["lam"])
    gp = orc.minibatch_gradients(st, pb, g["I"], np.arange(pb.m), orc.NEG_BINOMIAL, orc.LOG, lam)
    for mine, key in ((gp.g_row, "g_row"), (gp.h_row, "h_row"), (gp.g_col, "g_col"),
                      (gp.h_col, "h_col")):
        assert normwise(mine, g[key]) < 1e-13, key
    obj = orc.penalized_objective(st, pb, orc.NEG_BINOMIAL, orc.LOG, lam)
    assert obj == pytest.approx(float(g["objective"]), rel=1e-12)


def test_known_answers():
    # gmfkit tests/test_optim.py:17-46 known-answer constants
    assert orc.learning_rate(0, 0.03, 0.01, 0.75) == 0.03
    assert orc.learning_rate(100, 0.01, 1.0, 1.0) == pytest.approx(0.005)
    assert orc.bias_correction(1, 0.1, 0.01) == pytest.approx(1.1)
    assert orc.bias_correction(5, 0.3, 0.3) == 1.0
    # Poisson deviance D(2, 1) = 2(2 ln 2 - 1), tests/test_families.py:42-44
    d = orc.unit_deviance(orc.POISSON, np.array([2.0]), np.array([1.0]), 1.0)[0]
    assert d == pytest.approx(2 * (2 * np.log(2) - 1))


def _c2_oracle(callback=None, csr=False):
    from paper_2412_20509_b200 import workloads
    wl = workloads.generate("c2")
    init = wl.init_state()
    y = wl.y_dense
    yy = orc.CsrRows(*workloads.dense_to_csr(y), y.shape) if csr else y.astype(float)
    pb = orc.OProblem(yy, wl.x, np.zeros((y.shape[1], 0)), offset=wl.offset)
    st = orc.OState(init["b"], init["gamma"], init["u"], init["v"], 1.0, init["nb_shape"])
    cfg = orc.OConfig(max_epochs=20, mb_rows=2000, mb_cols=500, tol=1e-30, seed=0)
    return wl, orc.fit_asgd(pb, orc.NEG_BINOMIAL, orc.LOG, (0.0, 0.0, 1.0, 0.0), cfg, st,
                            callback=callback)


@pytest.mark.parametrize("csr", [False, True])
def test_oracle_c2_full_size_matches_reference(csr):
    """BASELINE config 2 at full size (26,472 x 500 NB fp64, k=15, offset):
    the oracle against gmfkit's own 20-epoch run (tests/golden/c2.npz); the
    CSR-backed response (used for configs too large to densify) is the same
    arithmetic."""
    import sys, os
    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
    from make_golden_checksum import y_checksum
    g = golden("c2")
    seen = {}
    checks = set(g["check_steps"].tolist())

    def cb(t, st):
        if t in checks:
            seen[t] = (st.b.copy(), st.v.copy(), st.nb_shape)

    wl, (final, rep) = _c2_oracle(cb, csr)
    assert np.array_equal(y_checksum(wl.y_dense), g["y_checksum"])
    assert rep.iterations == int(g["iterations"])
    assert normwise(rep.objective_trace, g["trace"]) < 1e-12
    assert normwise(rep.nb_shape_trace, g["nb_trace"]) < 1e-12
    for t, (b, v, nb) in seen.items():
        assert normwise(v, g[f"step{t}_v"]) < 1e-10, t
        assert normwise(b, g[f"step{t}_b"]) < 1e-10, t
    rows = g["sample_rows"]
    assert normwise(final.u[rows] @ final.v.T, g["final_u_rows"] @ g["final_v"].T) < 1e-9
    assert rep.final_objective == pytest.approx(float(g["final_objective"]), rel=1e-11)
