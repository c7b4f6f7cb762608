"""GPU parity: the CUDA path (through the C ABI) against the reference's
golden vectors and the CPU oracle.  Tolerances are the north star's:
per-step gradients 1e-10 relative (fp64) / 1e-4 (fp32), final deviance and
U V' within 1e-3 relative; fp64 trajectories are held much tighter."""
import ctypes as C

import numpy as np
import pytest

from conftest import golden, normwise
from oracle import asgd_oracle as orc

pytestmark = pytest.mark.gpu

gk = pytest.importorskip("paper_2412_20509_b200")


def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.fixture(autouse=True)
def _gpu():
    _need_gpu()


def _cfg(g):
    me, mr, mc, seed, cap = (int(v) for v in g["cfg"])
    k0, k1, tau, a1, a2, damp, tol = (float(v) for v in g["cfg_f"])
    return gk.SgdConfig(max_epochs=me, rate_k0=k0, rate_k1=k1, rate_tau=tau, mb_rows=mr,
                        mb_cols=mc, smooth_a1=a1, smooth_a2=a2, damping=damp, tol=tol,
                        seed=seed, max_eval_entries=cap)


def _state(g, prefix):
    return gk.FactorizationState(g[f"{prefix}_b"], g[f"{prefix}_gamma"], g[f"{prefix}_u"],
                                 g[f"{prefix}_v"], float(g[f"{prefix}_phi"]),
                                 float(g[f"{prefix}_nb"]))


def _problem(g):
    data = gk.ResponseMatrix(g["y"].astype(float),
                             weights=g["w"] if "w" in g.files else None)
    n, m = g["y"].shape
    covs = gk.CovariateSet(x=g["x"] if g["x"].shape[1] else None,
                           z=g["z"] if g["z"].shape[1] else None, n=n, m=m)
    off = g["offset"] if "offset" in g.files else None
    return data, covs, off


def _fam(g, nb=None):
    kind = str(g["family"])
    if kind == "neg_binomial":
        return gk.NegBinomial(float(g["init_nb"]) if nb is None else nb)
    return gk.Poisson()


def _pen(g):
    lam = [float(v) for v in g["lam"]]
    # lam_b, lam_gamma, lam_u, lam_v = lam * blocks with lam = 1
    return gk.PenaltyConfig(lam=1.0, blocks=tuple(lam))


# ---------------------------------------------------------------- level 1 seam

@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_seam_kernels_match_reference(dtype):
    import torch
    from paper_2412_20509_b200 import _lib
    lib = _lib.lib()
    g = golden("seam")
    tdt = torch.float64 if dtype == "f64" else torch.float32
    code = _lib.F64 if dtype == "f64" else _lib.F32
    tol = 1e-12 if dtype == "f64" else 2e-5
    keys = sorted({k.split("|")[0] for k in g.files})
    for key in keys:
        fc, lc = (int(v) for v in g[f"{key}|codes"])
        alpha = float(g[f"{key}|alpha"])
        t = lambda a: torch.as_tensor(np.asarray(a), device="cuda", dtype=tdt)
        eta, y, w = t(g[f"{key}|eta"]), t(g[f"{key}|y"]), t(g[f"{key}|w"])
        mu = torch.empty_like(eta)
        _lib.check(lib.gmf_mean_of_eta(lc, code, _lib.ptr(eta), _lib.ptr(mu), eta.numel(), None))
        dd, hh = torch.empty_like(eta), torch.empty_like(eta)
        _lib.check(lib.gmf_derivs_from_mu(fc, lc, code, _lib.ptr(y), _lib.ptr(mu), _lib.ptr(w),
                                          eta.numel(), 1.3, alpha, _lib.ptr(dd), _lib.ptr(hh), None))
        work = torch.empty(int(lib.gmf_reduce_work_bytes(eta.numel())), dtype=torch.uint8, device="cuda")
        dev = torch.zeros(1, dtype=torch.float64, device="cuda")
        _lib.check(lib.gmf_deviance_from_mu(fc, code, _lib.ptr(y), _lib.ptr(mu), _lib.ptr(w),
                                            eta.numel(), alpha, _lib.ptr(dev), _lib.ptr(work), None))
        torch.cuda.synchronize()
        assert normwise(mu.cpu().numpy(), g[f"{key}|mu"]) < tol, key
        assert normwise(dd.cpu().numpy(), g[f"{key}|dotd"]) < 50 * tol, key
        assert normwise(hh.cpu().numpy(), g[f"{key}|ddotd"]) < 50 * tol, key
        assert abs(dev.item() - float(g[f"{key}|dev"])) <= 50 * tol * abs(float(g[f"{key}|dev"])), key


# ---------------------------------------------------------------- K1 gradients

@pytest.mark.parametrize("name", ["c1", "nb_offset", "nb_cov_s3"])
@pytest.mark.parametrize("dtype,tol", [("f64", 1e-10), ("f32", 1e-4)])
def test_step0_gradient_matches_reference(name, dtype, tol):
    g = golden(name)
    data, covs, off = _problem(g)
    cfg = _cfg(g)
    from paper_2412_20509_b200.engine import Schedule
    sch = Schedule(data.n, data.m, cfg, n_steps=1)
    assert int(sch.block_seq[0]) == int(g["first_block"])
    mb = gk.Minibatch(sch.row_blocks[sch.block_seq[0]], sch.col_blocks[0])
    gp = gk.minibatch_gradients(_state(g, "init"), data, covs, _fam(g), gk.Log(), _pen(g), mb,
                                offset=off, dtype=dtype)
    for mine, key in ((gp.g_rowside, "g0_g_row"), (gp.h_rowside, "g0_h_row"),
                      (gp.g_colside, "g0_g_col"), (gp.h_colside, "g0_h_col")):
        assert normwise(mine, g[key]) < tol, (key, normwise(mine, g[key]))


def test_weighted_gradient_matches_reference():
    g = golden("weighted")
    data = gk.ResponseMatrix(g["y"].astype(float), weights=g["w"])
    covs = gk.CovariateSet(x=g["x"], z=g["z"])
    st = _state(g, "st")
    pen = gk.PenaltyConfig(lam=1.0, blocks=tuple(float(v) for v in g["lam"]))
    gp = gk.minibatch_gradients(st, data, covs, gk.NegBinomial(1.7), gk.Log(), pen,
                                gk.Minibatch(g["I"], np.arange(data.m)))
    for mine, key in ((gp.g_rowside, "g_row"), (gp.h_rowside, "h_row"),
                      (gp.g_colside, "g_col"), (gp.h_colside, "h_col")):
        assert normwise(mine, g[key]) < 1e-10, key
    obj = gk.penalized_objective(st, data, covs, gk.NegBinomial(1.7), gk.Log(), pen)
    assert obj == pytest.approx(float(g["objective"]), rel=1e-10)


def test_minibatch_hand_computed():
    # gmfkit tests/test_gradients.py:110-130
    y = np.array([[3.0, 1.0], [2.0, 5.0]])
    u = np.array([[0.2], [0.4]])
    v = np.array([[0.3], [0.1]])
    st = gk.FactorizationState(np.zeros((2, 0)), np.zeros((2, 0)), u, v)
    data = gk.ResponseMatrix(y)
    covs = gk.CovariateSet.empty(2, 2)
    pen = gk.PenaltyConfig(lam=0.5, blocks=(0, 0, 1, 1))
    gp = gk.minibatch_gradients(st, data, covs, gk.Poisson(), gk.Log(), pen, gk.Minibatch([1], [0]))
    mu = np.exp(0.4 * 0.3)
    dd = -(y[1, 0] - mu)
    assert gp.g_rowside[0, 0] == pytest.approx(2 * dd * 0.3 + 0.5 * 0.4, rel=1e-12)
    assert gp.g_colside[0, 0] == pytest.approx(2 * dd * 0.4 + 0.5 * 0.3, rel=1e-12)
    assert gp.h_rowside[0, 0] == pytest.approx(2 * mu * 0.3 ** 2 + 0.5, rel=1e-12)
    assert gp.h_colside[0, 0] == pytest.approx(2 * mu * 0.4 ** 2 + 0.5, rel=1e-12)


# ---------------------------------------------------------------- fit trajectories

@pytest.mark.parametrize("name", ["c1", "nb_offset", "nb_cov_s3"])
def test_fit_trajectory_fp64(name):
    g = golden(name)
    data, covs, off = _problem(g)
    seen = {}
    checks = set(g["check_steps"].tolist())

    def cb(t, st):
        if t in checks:
            seen[t] = st.copy()

    final, rep = gk.fit_asgd(data, covs, _fam(g), gk.Log(), _pen(g), _cfg(g), _state(g, "init"),
                             callback=cb, offset=off, dtype="f64")
    assert rep.epochs_run == int(g["epochs_run"])
    assert rep.converged == bool(g["converged"])
    assert rep.diagnostics["iterations"] == int(g["iterations"])
    assert normwise(rep.objective_trace, g["trace"]) < 1e-11
    assert normwise(rep.nb_shape_trace, g["nb_trace"]) < 1e-11
    assert seen.keys() == checks
    for t, st in seen.items():
        ref = _state(g, f"step{t}")
        for blk in ("b", "gamma", "u", "v"):
            assert normwise(getattr(st, blk), getattr(ref, blk)) < 1e-9, (t, blk)
    ref = _state(g, "final")
    assert normwise(final.u @ final.v.T, ref.u @ ref.v.T) < 1e-9
    for blk in ("b", "gamma", "u", "v"):
        assert normwise(getattr(final, blk), getattr(ref, blk)) < 1e-7, blk
    assert rep.final_objective == pytest.approx(float(g["final_objective"]), rel=1e-10)


@pytest.mark.parametrize("name", ["c1", "nb_offset", "nb_cov_s3"])
def test_fit_fp32_within_north_star(name):
    g = golden(name)
    data, covs, off = _problem(g)
    final, rep = gk.fit_asgd(data, covs, _fam(g), gk.Log(), _pen(g), _cfg(g), _state(g, "init"),
                             offset=off, dtype="f32")
    ref = _state(g, "final")
    assert normwise(final.u @ final.v.T, ref.u @ ref.v.T) < 1e-3
    assert rep.final_objective == pytest.approx(float(g["final_objective"]), rel=1e-3)
    assert normwise(rep.objective_trace, g["trace"]) < 1e-4


def test_fit_no_callback_equals_callback_path():
    g = golden("nb_offset")
    data, covs, off = _problem(g)
    a, ra = gk.fit_asgd(data, covs, _fam(g), gk.Log(), _pen(g), _cfg(g), _state(g, "init"),
                        offset=off)
    b, rb = gk.fit_asgd(data, covs, _fam(g), gk.Log(), _pen(g), _cfg(g), _state(g, "init"),
                        offset=off, callback=lambda t, s: None)
    assert ra.objective_trace == rb.objective_trace      # bitwise: fixed-order reductions
    assert np.array_equal(a.u, b.u)


def test_convergence_decision_matches_reference():
    g = golden("converge")
    data, covs, off = _problem(g)
    final, rep = gk.fit_asgd(data, covs, gk.Poisson(), gk.Log(), _pen(g), _cfg(g),
                             _state(g, "init"))
    assert rep.converged and bool(g["converged"])
    assert rep.epochs_run == int(g["epochs_run"])
    assert normwise(rep.objective_trace, g["trace"]) < 1e-10


def test_divergence_carries_snapshot():
    g = golden("diverge")
    data = gk.ResponseMatrix(g["y"].astype(float))
    covs = gk.CovariateSet(x=g["x"], m=g["y"].shape[1])
    steps = []
    with pytest.raises(gk.DivergenceError) as err:
        gk.fit_asgd(data, covs, gk.Poisson(), gk.Log(), gk.PenaltyConfig(), _cfg(g),
                    _state(g, "init"), callback=lambda t, s: steps.append(t))
    assert len(steps) == int(g["steps_before"])
    snap = err.value.state
    assert snap is not None and np.isfinite(snap.u).all()
    ref = _state(g, "snap")
    for blk in ("b", "u", "v"):
        assert normwise(getattr(snap, blk), getattr(ref, blk)) < 1e-10, blk


def test_seed_determinism_bitwise():
    g = golden("nb_cov_s3")
    data, covs, off = _problem(g)
    _, r1 = gk.fit_asgd(data, covs, _fam(g), gk.Log(), _pen(g), _cfg(g), _state(g, "init"))
    _, r2 = gk.fit_asgd(data, covs, _fam(g), gk.Log(), _pen(g), _cfg(g), _state(g, "init"))
    assert r1.objective_trace == r2.objective_trace


def test_csr_equals_dense_bitwise():
    from paper_2412_20509_b200.workloads import dense_to_csr
    g = golden("nb_offset")
    data, covs, off = _problem(g)
    csr = gk.ResponseMatrix(csr=dense_to_csr(g["y"]), shape=g["y"].shape)
    for dtype in ("f64", "f32"):
        a, ra = gk.fit_asgd(data, covs, _fam(g), gk.Log(), _pen(g), _cfg(g), _state(g, "init"),
                            offset=off, dtype=dtype)
        b, rb = gk.fit_asgd(csr, covs, _fam(g), gk.Log(), _pen(g), _cfg(g), _state(g, "init"),
                            offset=off, dtype=dtype)
        assert ra.objective_trace[:-1] == rb.objective_trace[:-1]
        assert np.array_equal(a.u, b.u) and np.array_equal(a.v, b.v)


# ---------------------------------------------------------------- K4 projection

def test_projection_matches_reference():
    g = golden("project")
    for k in range(3):
        st = _state(g, f"{k}|in")
        covs = gk.CovariateSet(x=g[f"{k}|x"], z=g[f"{k}|z"])
        out = gk.project_constraints(st, covs, "B1")
        ref = _state(g, f"{k}|out")
        for blk in ("b", "gamma", "u", "v"):
            assert normwise(getattr(out, blk), getattr(ref, blk)) < 1e-9, (k, blk)
        twice = gk.project_constraints(out, covs, "B1")
        for blk in ("b", "gamma", "u", "v"):
            assert np.allclose(getattr(out, blk), getattr(twice, blk), atol=1e-9)
        rep = gk.check_constraints(out, covs, "B1")
        assert max(rep.values()) < 1e-8
    st = _state(g, "rd|in")
    out, info = gk.project_constraints(st, gk.CovariateSet.empty(10, 6), "B1", return_info=True)
    assert info["rank_deficient"] and info["effective_rank"] == int(g["rd|eff"])
    assert np.allclose(out.u[:, 2], 0.0)
    assert normwise(out.u @ out.v.T, g["rd|out_u"] @ g["rd|out_v"].T) < 1e-10


def test_projection_uniqueness_across_reparameterizations(rng):
    n, m, d, p, q = 25, 10, 3, 2, 1
    x = np.hstack([np.ones((n, 1)), rng.normal(size=(n, p - 1))])
    z = np.ones((m, q))
    covs = gk.CovariateSet(x=x, z=z)
    st = gk.FactorizationState(rng.normal(size=(m, p)), rng.normal(size=(n, q)),
                               rng.normal(size=(n, d)), rng.normal(size=(m, d)))
    mix = rng.normal(size=(3, 3)) + 3 * np.eye(3)
    other = st.copy()
    other.u = st.u @ mix
    other.v = st.v @ np.linalg.inv(mix).T
    shift = rng.normal(size=(p, q))
    other.gamma = other.gamma + x @ shift
    other.b = other.b - z @ shift.T
    a = gk.project_constraints(st, covs, "B1")
    b = gk.project_constraints(other, covs, "B1")
    for blk in ("b", "gamma", "u", "v"):
        assert np.allclose(getattr(a, blk), getattr(b, blk), atol=1e-8), blk


# ---------------------------------------------------------------- full-size property

def test_c4_full_size_block_gradient_against_oracle():
    """BASELINE config 4 at full size (1.3M x 500 CSR, fp32): one drawn block's
    gradient against the fp64 oracle on that block, plus bitwise determinism."""
    from paper_2412_20509_b200 import workloads
    from paper_2412_20509_b200.engine import DeviceFit, Schedule
    wl = workloads.generate("c4", device="cuda")
    sp = wl.spec
    data = gk.ResponseMatrix(csr=wl.csr, shape=(sp.n, sp.m))
    covs = gk.CovariateSet(x=wl.x, z=None, m=sp.m)
    init = wl.init_state()
    st = gk.FactorizationState(**init)
    cfg = gk.SgdConfig(max_epochs=sp.epochs, mb_rows=sp.mb_rows, mb_cols=sp.m)
    sch = Schedule(sp.n, sp.m, cfg)
    fit = DeviceFit(data, covs, gk.NegBinomial(2.0), gk.Log(), gk.PenaltyConfig(), cfg, st,
                    schedule=sch, offset=wl.offset, dtype="f32", est_alpha=True)
    try:
        blk = int(sch.block_seq[0])
        out1 = [t.double().cpu().numpy() for t in fit.minibatch_grad(blk, 0, 2.0)[:4]]
        out2 = [t.double().cpu().numpy() for t in fit.minibatch_grad(blk, 0, 2.0)[:4]]
    finally:
        fit.close()
    for a, b in zip(out1, out2):
        assert np.array_equal(a, b)
    I = sch.row_blocks[blk]
    pb = orc.OProblem(wl.dense_f64(I), wl.x[I], np.zeros((sp.m, 0)), offset=wl.offset[I])
    ost = orc.OState(init["b"], init["gamma"][I], init["u"][I], init["v"], 1.0, 2.0)
    ref = orc.minibatch_gradients(ost, pb, np.arange(I.size), np.arange(sp.m),
                                  orc.NEG_BINOMIAL, orc.LOG, (0.0, 0.0, 1.0, 0.0))
    # the oracle on the block alone has s_col = |I|/|I| = 1; rescale to n/|I|
    s = sp.n / I.size
    ref_gc = (ref.g_col - 0.0) * s
    ref_hc = ref.h_col * s
    assert normwise(out1[0], ref.g_row) < 1e-4
    assert normwise(out1[1], ref.h_row) < 1e-4
    assert normwise(out1[2], ref_gc) < 1e-4
    assert normwise(out1[3], ref_hc) < 1e-4


@pytest.mark.parametrize("mode", ["B2", "B3"])
@pytest.mark.parametrize("dtype,tol", [("f64", 1e-9), ("f32", 1e-4)])
def test_projection_b2_b3_match_reference(mode, dtype, tol):
    """B2 and B3 normalizations (identify.py:93-135) on the device against the
    reference's own projections (tests/golden/project_b23.npz)."""
    g = golden("project_b23")
    for k in range(3):
        st = _state(g, f"{k}|in")
        covs = gk.CovariateSet(x=g[f"{k}|x"], z=g[f"{k}|z"])
        out = gk.project_constraints(st, covs, mode, dtype=dtype)
        ref = _state(g, f"{k}|{mode}")
        for blk in ("b", "gamma", "u", "v"):
            assert normwise(getattr(out, blk), getattr(ref, blk)) < tol, (k, mode, blk)
        if dtype == "f64":
            rep = gk.check_constraints(out, covs, mode)
            assert rep["normalization"] < 1e-8 and max(rep.values()) < 1e-8, rep
