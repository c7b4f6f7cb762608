"""Tensor-core K1 (tcgen05, bf16-split operands, fp32 accumulation in TMEM)
against the CPU oracle and against the CUDA-core K1.

Shapes cover the tensor path's edges: partial 128-column tiles, row ranges
that are not multiples of the 32-row chunk, column blocks that are not the
identity (mb_cols < m), offsets, Poisson and NB, K = p+q+d above 16 (two
GEMM1 k-steps) and the largest row/column feature widths (q+d = p+d = 16).
Tolerance: the north star's fp32 gradient bound, 1e-4 normwise."""
import numpy as np
import pytest

from conftest import normwise
from oracle import asgd_oracle as orc

pytestmark = pytest.mark.gpu

gk = pytest.importorskip("paper_2412_20509_b200")

TOL = 1e-4


@pytest.fixture(autouse=True)
def _gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _problem(seed, n, m, d, p, q, family, offset):
    rng = np.random.default_rng(seed)
    x = np.hstack([np.ones((n, 1)), rng.normal(size=(n, p - 1))]) if p else np.zeros((n, 0))
    z = np.hstack([np.ones((m, 1)), rng.normal(size=(m, q - 1))]) if q else np.zeros((m, 0))
    b = rng.normal(0.5, 0.3, size=(m, p))
    gamma = rng.normal(0, 0.2, size=(n, q))
    u = rng.normal(0, 0.4, size=(n, d))
    v = rng.normal(0, 0.4, size=(m, d))
    off = rng.normal(0, 0.5, size=n) if offset else None
    eta = x @ b.T + gamma @ z.T + u @ v.T + (off[:, None] if offset else 0.0)
    mu = np.exp(np.clip(eta, -10, 6))
    if family == "nb":
        lam = rng.gamma(2.0, mu / 2.0)
        y = rng.poisson(lam)
    else:
        y = rng.poisson(mu)
    noisy = lambda a: a + rng.normal(0, 0.05, size=a.shape)
    st = gk.FactorizationState(noisy(b), noisy(gamma), noisy(u), noisy(v), 1.0, 2.0)
    return y.astype(float), x, z, off, st


CASES = [
    # (n, m, d, p, q, family, offset, mb_rows, mb_cols)
    (300, 200, 5, 1, 1, "poisson", False, 137, 200),     # partial 2nd tile, ragged chunks
    (517, 300, 10, 1, 0, "nb", True, 517, 300),          # c4-like features, offset, all rows
    (400, 260, 12, 4, 4, "nb", False, 150, 130),         # KA = 20: two GEMM1 k-steps; column blocks
    (150, 128, 15, 1, 1, "nb", True, 97, 128),           # Kr = Kc = 16 (widest), one full tile
    (64, 40, 3, 2, 0, "poisson", True, 33, 17),          # tiny: one partial tile, mostly-empty chunks
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"n{c[0]}m{c[1]}d{c[2]}p{c[3]}q{c[4]}{c[5]}")
@pytest.mark.parametrize("impl", ["tensor", "cuda_cores"])
def test_k1_block_gradient_matches_oracle(case, impl, k1_generation):
    n, m, d, p, q, family, offset, mbr, mbc = case
    y, x, z, off, st = _problem(7, n, m, d, p, q, family, offset)
    rng = np.random.default_rng(11)
    I = np.sort(rng.choice(n, size=mbr, replace=False))
    J = np.sort(rng.choice(m, size=mbc, replace=False))
    data = gk.ResponseMatrix(y)
    covs = gk.CovariateSet(x=x if p else None, z=z if q else None, n=n, m=m)
    lam = (0.3, 0.2, 1.0, 0.7)
    pen = gk.PenaltyConfig(lam=1.0, blocks=lam)
    fam = gk.NegBinomial(2.0) if family == "nb" else gk.Poisson()
    gp, nbs = gk.minibatch_gradients(st, data, covs, fam, gk.Log(), pen, gk.Minibatch(I, J),
                                     offset=off, dtype="f32", k1_impl=impl, return_nb_sums=True)
    pb = orc.OProblem(y, x, z, offset=off)
    ost = orc.OState(st.b, st.gamma, st.u, st.v, 1.0, 2.0)
    fcode = orc.NEG_BINOMIAL if family == "nb" else orc.POISSON
    ref = orc.minibatch_gradients(ost, pb, I, J, fcode, orc.LOG, lam)
    errs = {k: normwise(mine, r) for k, mine, r in (
        ("g_row", gp.g_rowside, ref.g_row), ("h_row", gp.h_rowside, ref.h_row),
        ("g_col", gp.g_colside, ref.g_col), ("h_col", gp.h_colside, ref.h_col))}
    assert max(errs.values()) < TOL, errs
    if family == "nb":
        _, w, mu, _, _ = orc.block_derivs(ost, pb, I, J, fcode, orc.LOG)
        num, den = orc.nb_moment_sums(y[I][:, J], mu, w)
        assert abs(nbs[0] - num) < TOL * abs(num) and abs(nbs[1] - den) < TOL * (abs(num) + abs(den))


@pytest.mark.parametrize("case", CASES[:3], ids=lambda c: f"n{c[0]}m{c[1]}")
def test_k1_tensor_close_to_cuda_cores(case, k1_generation):
    n, m, d, p, q, family, offset, mbr, mbc = case
    y, x, z, off, st = _problem(3, n, m, d, p, q, family, offset)
    I = np.arange(0, n, 2)
    J = np.arange(m)
    data = gk.ResponseMatrix(y)
    covs = gk.CovariateSet(x=x if p else None, z=z if q else None, n=n, m=m)
    fam = gk.NegBinomial(2.0) if family == "nb" else gk.Poisson()
    out = {}
    for impl in ("tensor", "cuda_cores"):
        out[impl] = gk.minibatch_gradients(st, data, covs, fam, gk.Log(), gk.PenaltyConfig(),
                                           gk.Minibatch(I, J), offset=off, dtype="f32", k1_impl=impl)
    a, b = out["tensor"], out["cuda_cores"]
    for f in ("g_rowside", "h_rowside", "g_colside", "h_colside"):
        assert normwise(getattr(a, f), getattr(b, f)) < TOL, f


def test_k1_tensor_csr_equals_dense_bitwise(k1_generation):
    from paper_2412_20509_b200.workloads import dense_to_csr
    y, x, z, off, st = _problem(5, 300, 200, 10, 1, 0, "nb", True)
    I, J = np.arange(7, 250), np.arange(200)
    covs = gk.CovariateSet(x=x, n=300, m=200)
    outs = []
    for data in (gk.ResponseMatrix(y), gk.ResponseMatrix(csr=dense_to_csr(y), shape=y.shape)):
        outs.append(gk.minibatch_gradients(st, data, covs, gk.NegBinomial(2.0), gk.Log(),
                                           gk.PenaltyConfig(), gk.Minibatch(I, J), offset=off,
                                           dtype="f32", k1_impl="tensor"))
    for f in ("g_rowside", "h_rowside", "g_colside", "h_colside"):
        assert np.array_equal(getattr(outs[0], f), getattr(outs[1], f)), f


def test_k1_tensor_rejects_ineligible_problems():
    from paper_2412_20509_b200 import _lib
    y, x, z, off, st = _problem(1, 50, 30, 3, 1, 0, "nb", False)
    covs = gk.CovariateSet(x=x, n=50, m=30)
    mb = gk.Minibatch(np.arange(50), np.arange(30))
    with pytest.raises(_lib.UnsupportedError):      # fp64 runs on the CUDA cores only
        gk.minibatch_gradients(st, gk.ResponseMatrix(y), covs, gk.NegBinomial(2.0), gk.Log(),
                               gk.PenaltyConfig(), mb, dtype="f64", k1_impl="tensor")
    with pytest.raises(_lib.UnsupportedError):      # prior weights
        gk.minibatch_gradients(st, gk.ResponseMatrix(y, weights=np.ones_like(y)), covs,
                               gk.NegBinomial(2.0), gk.Log(), gk.PenaltyConfig(), mb,
                               dtype="f32", k1_impl="tensor")


@pytest.mark.parametrize("impl", ["tensor", "cuda_cores"])
def test_fit_fp32_trajectory_per_impl(impl, k1_generation):
    from conftest import golden
    g = golden("nb_cov_s3")
    data = gk.ResponseMatrix(g["y"].astype(float))
    covs = gk.CovariateSet(x=g["x"], z=g["z"])
    st = gk.FactorizationState(g["init_b"], g["init_gamma"], g["init_u"], g["init_v"], 1.0,
                               float(g["init_nb"]))
    me, mr, mc, seed, cap = (int(v) for v in g["cfg"])
    k0, k1, tau, a1, a2, damp, tol = (float(v) for v in g["cfg_f"])
    cfg = gk.SgdConfig(max_epochs=me, rate_k0=k0, rate_k1=k1, rate_tau=tau, mb_rows=mr,
                       mb_cols=mc, smooth_a1=a1, smooth_a2=a2, damping=damp, tol=tol, seed=seed,
                       max_eval_entries=cap)
    pen = gk.PenaltyConfig(lam=1.0, blocks=tuple(float(v) for v in g["lam"]))
    final, rep = gk.fit_asgd(data, covs, gk.NegBinomial(st.nb_shape), gk.Log(), pen, cfg, st,
                             dtype="f32", k1_impl=impl)
    assert normwise(rep.objective_trace, g["trace"]) < TOL
    assert normwise(final.u @ final.v.T, g["final_u"] @ g["final_v"].T) < 1e-3


def test_packed_csr_equals_csr32_bitwise(k1_generation):
    """Packed CSR (one uint32 per nonzero) and int32 CSR hold the same counts:
    identical trajectories on both K1 implementations."""
    from conftest import golden
    from paper_2412_20509_b200.workloads import dense_to_csr
    g = golden("nb_offset")
    y = g["y"]
    data = gk.ResponseMatrix(csr=dense_to_csr(y), shape=y.shape)
    covs = gk.CovariateSet(x=g["x"], z=g["z"] if g["z"].shape[1] else None, n=y.shape[0], m=y.shape[1])
    st = gk.FactorizationState(g["init_b"], g["init_gamma"], g["init_u"], g["init_v"], 1.0,
                               float(g["init_nb"]))
    me, mr, mc, seed, cap = (int(v) for v in g["cfg"])
    cfg = gk.SgdConfig(max_epochs=me, mb_rows=mr, mb_cols=mc, seed=seed, tol=1e-30)
    pen = gk.PenaltyConfig(lam=1.0, blocks=tuple(float(v) for v in g["lam"]))
    for impl in ("tensor", "cuda_cores"):
        out = []
        for yf in ("csr32", "packed"):
            _, rep = gk.fit_asgd(data, covs, gk.NegBinomial(st.nb_shape), gk.Log(), pen, cfg, st,
                                 offset=g["offset"], dtype="f32", k1_impl=impl, y_format=yf)
            out.append(rep.objective_trace)
        assert out[0] == out[1], impl


def test_streaming_run_equals_resident_run_bitwise(k1_generation):
    """gmf_run_stream (one launch; each step waits for its row block's ready
    signal, statuses written to pinned host memory) reproduces gmf_run."""
    import torch
    from paper_2412_20509_b200 import _lib, workloads
    from paper_2412_20509_b200.engine import DeviceFit, Schedule
    y, x, z, off, st = _problem(9, 600, 140, 6, 1, 0, "nb", True)
    from paper_2412_20509_b200.workloads import dense_to_csr
    data = gk.ResponseMatrix(csr=dense_to_csr(y), shape=y.shape)
    covs = gk.CovariateSet(x=x, n=600, m=140)
    cfg = gk.SgdConfig(max_epochs=40, mb_rows=100, mb_cols=140, tol=1e-30, seed=2)
    sch = Schedule(600, 140, cfg)
    out = []
    for stream in (False, True):
        fit = DeviceFit(data, covs, gk.NegBinomial(2.0), gk.Log(), gk.PenaltyConfig(), cfg, st,
                        schedule=sch, offset=off, dtype="f32", est_alpha=True)
        try:
            fit.reset()
            if not stream:
                fit.run(30)
            else:
                sb = int(fit.lib.gmf_status_raw_bytes())
                host = torch.zeros(30 * sb, dtype=torch.uint8).pin_memory()
                cs = torch.cuda.Stream()
                fit.run_stream(30, host)
                for t in range(30):          # blocks are resident: signal each step
                    fit.stream_signal(t + 1, cs)
                torch.cuda.synchronize()
                st_last = _lib.GmfStatus()
                import ctypes as C
                fit.lib.gmf_status_decode(C.c_void_p(host.data_ptr() + 29 * sb), C.byref(st_last))
                assert st_last.t == 30
            status = fit.status()
            assert status.t == 30
            out.append((fit.trace(int(status.trace_len))[0], fit.theta_col.cpu().numpy().copy()))
        finally:
            fit.close()
    assert np.array_equal(out[0][0], out[1][0])
    assert np.array_equal(out[0][1], out[1][1])


@pytest.mark.parametrize("dtype,tol", [("f64", 1e-10), ("f32", 1e-4)])
def test_per_step_path_matches_persistent(monkeypatch, dtype, tol):
    """The per-step kernels (k_obj / k_grad / k_colrec / k_apply -- the path
    every rank of a multi-rank fit runs) reproduce the persistent k_fit: same
    objective trace and final factors, with the per-step objective read from
    the row-slot / padded-column caches that k_apply keeps current."""
    from paper_2412_20509_b200.engine import DeviceFit, Schedule
    from paper_2412_20509_b200.workloads import dense_to_csr
    y, x, z, off, st = _problem(13, 500, 150, 6, 2, 1, "nb", True)
    data = gk.ResponseMatrix(csr=dense_to_csr(y), shape=y.shape)
    covs = gk.CovariateSet(x=x, z=z, n=500, m=150)
    cfg = gk.SgdConfig(max_epochs=40, mb_rows=90, mb_cols=150, tol=1e-30, seed=4)
    sch = Schedule(500, 150, cfg)
    out = []
    for per_step in (False, True):
        if per_step:
            monkeypatch.setenv("GMF_NO_PERSISTENT", "1")
        fit = DeviceFit(data, covs, gk.NegBinomial(2.0), gk.Log(), gk.PenaltyConfig(), cfg, st,
                        schedule=sch, offset=off, dtype=dtype, est_alpha=True)
        try:
            fit.reset()
            fit.run(40)
            status = fit.status()
            out.append((fit.trace(int(status.trace_len))[0],
                        fit.theta_row.cpu().numpy().copy(), fit.theta_col.cpu().numpy().copy()))
        finally:
            fit.close()
        monkeypatch.delenv("GMF_NO_PERSISTENT", raising=False)
    assert len(out[0][0]) == len(out[1][0]) > 3
    assert np.allclose(out[0][0], out[1][0], rtol=tol, atol=0)
    for a, b in zip(out[0][1:], out[1][1:]):
        assert normwise(b, a) < tol


@pytest.mark.gpu
@pytest.mark.parametrize("gen", [1, 2])
def test_k1_generation_is_the_one_requested(gen, monkeypatch):
    """GMF_TC_VERSION selects the tensor-core K1 generation the handle runs
    (gmf_k1_version), so the parametrized parity tests exercise both."""
    import torch
    from paper_2412_20509_b200.engine import DeviceFit, Schedule
    monkeypatch.setenv("GMF_TC_VERSION", str(gen))
    rng = np.random.default_rng(5)
    n, m, d = 3000, 300, 4
    y = rng.poisson(1.5, (n, m)).astype(float)
    st = gk.FactorizationState(rng.normal(0, .1, (m, 1)), np.zeros((n, 0)), rng.normal(0, .3, (n, d)),
                               rng.normal(0, .3, (m, d)), 1.0, 2.0)
    cfg = gk.SgdConfig(max_epochs=3, mb_rows=1000, mb_cols=m, tol=1e-30, seed=0)
    fit = DeviceFit(gk.ResponseMatrix(y), gk.CovariateSet(x=np.ones((n, 1)), m=m), gk.Poisson(),
                    gk.Log(), gk.PenaltyConfig(), cfg, st, schedule=Schedule(n, m, cfg), dtype="f32",
                    k1_impl="tensor")
    try:
        assert fit.k1_version == gen
    finally:
        fit.close()
        torch.cuda.synchronize()


def _grad_vs_oracle(y, x, z, off, st, I, J, family, data):
    n, m = y.shape
    covs = gk.CovariateSet(x=x if x.shape[1] else None, z=z if z.shape[1] else None, n=n, m=m)
    lam = (0.3, 0.2, 1.0, 0.7)
    fam = gk.NegBinomial(2.0) if family == "nb" else gk.Poisson()
    gp = gk.minibatch_gradients(st, data, covs, fam, gk.Log(), gk.PenaltyConfig(lam=1.0, blocks=lam),
                                gk.Minibatch(I, J), offset=off, dtype="f32", k1_impl="tensor")
    pb = orc.OProblem(y, x, z, offset=off)
    ost = orc.OState(st.b, st.gamma, st.u, st.v, 1.0, 2.0)
    ref = orc.minibatch_gradients(ost, pb, I, J, orc.NEG_BINOMIAL if family == "nb" else orc.POISSON,
                                  orc.LOG, lam)
    errs = {k: normwise(mine, r) for k, mine, r in (
        ("g_row", gp.g_rowside, ref.g_row), ("h_row", gp.h_rowside, ref.h_row),
        ("g_col", gp.g_colside, ref.g_col), ("h_col", gp.h_colside, ref.h_col))}
    return gp, errs


@pytest.mark.parametrize("family", ["poisson", "nb"])
def test_k1_v2_csr_with_32_feature_operands(family, monkeypatch):
    """K1 v2 on a CSR response with K = p+q+d + sentinels in (16, 32]: shared
    memory then holds a single A1 buffer, whose second chunk can only be
    staged once GEMM1 of the first has run (a c5 sweep cell, 65,536 x 500
    d = 15 CSR, found the prologue waiting for it before the MMA warp ran)."""
    from paper_2412_20509_b200.workloads import dense_to_csr
    monkeypatch.setenv("GMF_TC_VERSION", "2")
    y, x, z, off, st = _problem(21, 900, 200, 15, 1, 1, family, False)
    I, J = np.arange(13, 880), np.arange(200)
    data = gk.ResponseMatrix(csr=dense_to_csr(y), shape=y.shape)
    _, errs = _grad_vs_oracle(y, x, z, off, st, I, J, family, data)
    assert max(errs.values()) < TOL, errs


@pytest.mark.parametrize("fmt", ["dense", "csr"])
def test_k1_v2_wide_matrix_two_units_per_cta(fmt, monkeypatch):
    """Wide matrix on K1 v2: 8 column tiles x 37 row ranges = two units per CTA
    (the per-unit prologue / drain and the mbarrier phases carried across
    units), 24 chunks per unit."""
    from paper_2412_20509_b200.workloads import dense_to_csr
    monkeypatch.setenv("GMF_TC_VERSION", "2")
    y, x, z, off, st = _problem(22, 1500, 1000, 5, 1, 1, "nb", True)
    I, J = np.arange(1500), np.arange(1000)
    data = gk.ResponseMatrix(y) if fmt == "dense" else gk.ResponseMatrix(csr=dense_to_csr(y),
                                                                         shape=y.shape)
    _, errs = _grad_vs_oracle(y, x, z, off, st, I, J, "nb", data)
    assert max(errs.values()) < TOL, errs
