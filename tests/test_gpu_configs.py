"""GPU parity at the BASELINE.json fit configurations, full size.

c2 (26,472 x 500 NB fp64, k=15, offset) against gmfkit's own 20-epoch run
(tests/golden/c2.npz) and in fp32 within the north-star tolerances; c3
(100,000 x 1,000 CSR fp32, p=2, q=1) over its 20 epochs and c4 (1.3M x 500
CSR fp32, the bench workload) over its 10 epochs through the persistent fit
kernel the bench times, both against the fp64 oracle on the identical
inputs and replayed minibatch sequence (oracle.CsrRows: the oracle reads the
drawn block's rows from the CSR, same arithmetic as the dense restatement).
Tolerances are the north star's: fp32 per-step quantities 1e-4 normwise,
final deviance and U V' 1e-3 relative; fp64 is held far tighter."""
import os
import sys

import numpy as np
import pytest

from conftest import GOLDEN, golden, normwise
from oracle import asgd_oracle as orc

pytestmark = pytest.mark.gpu

gk = pytest.importorskip("paper_2412_20509_b200")
sys.path.insert(0, GOLDEN)
from make_golden_checksum import y_checksum  # noqa: E402


@pytest.fixture(autouse=True)
def _gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _uv_rows(st, rows):
    return st.u[rows] @ st.v.T


# ---------------------------------------------------------------- c2 (fp64 = the reference's precision)

def _c2():
    from paper_2412_20509_b200 import workloads
    wl = workloads.generate("c2")
    g = golden("c2")
    assert np.array_equal(y_checksum(wl.y_dense), g["y_checksum"]), "regenerated c2 input differs"
    data = gk.ResponseMatrix(wl.y_dense.astype(float))
    covs = gk.CovariateSet(x=wl.x, z=None, m=wl.spec.m)
    st = gk.FactorizationState(**wl.init_state())
    cfg = gk.SgdConfig(max_epochs=20, mb_rows=2000, mb_cols=500, tol=1e-30, seed=0)
    return wl, g, data, covs, st, cfg


def test_c2_full_size_fp64_matches_reference():
    wl, g, data, covs, st, cfg = _c2()
    seen = {}
    checks = set(g["check_steps"].tolist())

    def cb(t, s):
        if t in checks:
            seen[t] = (s.b.copy(), s.v.copy(), s.nb_shape)

    final, rep = gk.fit_asgd(data, covs, gk.NegBinomial(st.nb_shape), gk.Log(),
                             gk.PenaltyConfig(), cfg, st, offset=wl.offset, dtype="f64",
                             callback=cb)
    assert rep.diagnostics["iterations"] == int(g["iterations"])
    assert normwise(rep.objective_trace, g["trace"]) < 1e-11
    assert normwise(rep.nb_shape_trace, g["nb_trace"]) < 1e-11
    assert seen.keys() == checks
    for t, (b, v, nb) in seen.items():
        assert normwise(v, g[f"step{t}_v"]) < 1e-9, t
        assert normwise(b, g[f"step{t}_b"]) < 1e-9, t
        assert nb == pytest.approx(float(g[f"step{t}_nb"]), rel=1e-11)
    rows = g["sample_rows"]
    assert normwise(_uv_rows(final, rows), g["final_u_rows"] @ g["final_v"].T) < 1e-9
    assert normwise(final.b, g["final_b"]) < 1e-8
    assert rep.final_objective == pytest.approx(float(g["final_objective"]), rel=1e-10)


def test_c2_full_size_fp64_persistent_equals_callback_path():
    """The persistent launch (no callback) and the one-step-per-launch path are bitwise equal."""
    wl, g, data, covs, st, cfg = _c2()
    fam = gk.NegBinomial(st.nb_shape)
    a, ra = gk.fit_asgd(data, covs, fam, gk.Log(), gk.PenaltyConfig(), cfg, st,
                        offset=wl.offset, dtype="f64")
    assert normwise(ra.objective_trace, g["trace"]) < 1e-11
    assert ra.final_objective == pytest.approx(float(g["final_objective"]), rel=1e-10)


def test_c2_full_size_fp32_within_north_star():
    wl, g, data, covs, st, cfg = _c2()
    final, rep = gk.fit_asgd(data, covs, gk.NegBinomial(st.nb_shape), gk.Log(),
                             gk.PenaltyConfig(), cfg, st, offset=wl.offset, dtype="f32")
    rows = g["sample_rows"]
    assert normwise(rep.objective_trace, g["trace"]) < 1e-4
    assert normwise(rep.nb_shape_trace, g["nb_trace"]) < 1e-4
    assert normwise(_uv_rows(final, rows), g["final_u_rows"] @ g["final_v"].T) < 1e-3
    assert rep.final_objective == pytest.approx(float(g["final_objective"]), rel=1e-3)


# ---------------------------------------------------------------- c3, c4 (fp32 CSR) vs the oracle

def _csr_problem(name, epochs):
    from paper_2412_20509_b200 import workloads
    wl = workloads.generate(name, device="cuda")
    sp = wl.spec
    data = gk.ResponseMatrix(csr=wl.csr, shape=(sp.n, sp.m))
    covs = gk.CovariateSet(x=wl.x, z=wl.z if sp.q else None, m=sp.m)
    st = gk.FactorizationState(**wl.init_state())
    cfg = gk.SgdConfig(max_epochs=epochs, mb_rows=sp.mb_rows, mb_cols=sp.m, tol=1e-30, seed=0)
    init = wl.init_state()
    pb = orc.OProblem(orc.CsrRows(*wl.csr, (sp.n, sp.m)), wl.x,
                      wl.z if sp.q else np.zeros((sp.m, 0)), offset=wl.offset)
    ost = orc.OState(init["b"], init["gamma"], init["u"], init["v"], 1.0, init["nb_shape"])
    ocfg = orc.OConfig(max_epochs=epochs, mb_rows=sp.mb_rows, mb_cols=sp.m, tol=1e-30, seed=0)
    return wl, data, covs, st, cfg, pb, ost, ocfg


def _oracle_fit(pb, ost, ocfg, callback=None):
    return orc.fit_asgd(pb, orc.NEG_BINOMIAL, orc.LOG, (0.0, 0.0, 1.0, 0.0), ocfg, ost,
                        callback=callback)


def _compare_final(final, rep, ofinal, orep, n, seed=5):
    rows = np.sort(np.random.default_rng(seed).choice(n, min(n, 20000), replace=False))
    assert normwise(rep.objective_trace, orep.objective_trace) < 1e-4
    assert normwise(rep.nb_shape_trace, orep.nb_shape_trace) < 1e-4
    assert normwise(_uv_rows(final, rows), _uv_rows(ofinal, rows)) < 1e-3
    assert normwise(final.b, ofinal.b) < 1e-3
    assert rep.final_objective == pytest.approx(orep.final_objective, rel=1e-3)


def test_c3_full_size_fp32_csr_matches_oracle(k1_generation):
    wl, data, covs, st, cfg, pb, ost, ocfg = _csr_problem("c3", 20)
    final, rep = gk.fit_asgd(data, covs, gk.NegBinomial(st.nb_shape), gk.Log(),
                             gk.PenaltyConfig(), cfg, st, dtype="f32")
    ofinal, orep = _oracle_fit(pb, ost, ocfg)
    assert rep.diagnostics["iterations"] == orep.iterations == 20
    _compare_final(final, rep, ofinal, orep, wl.spec.n)


def test_c4_full_size_persistent_fit_matches_oracle(k1_generation):
    """The headline workload through the persistent k_fit the bench times
    (one launch, no callback): 10 epochs vs the oracle, and the per-step states
    of steps 0..9 (one k_fit launch per step through the callback path: V, B,
    the drawn block's U rows, the NB shape) -- every step's gradient and update
    enter these."""
    wl, data, covs, st, cfg, pb, ost, ocfg = _csr_problem("c4", 10)
    fam = gk.NegBinomial(st.nb_shape)
    final, rep = gk.fit_asgd(data, covs, fam, gk.Log(), gk.PenaltyConfig(), cfg, st,
                             offset=wl.offset, dtype="f32")
    ref_steps = {}
    from paper_2412_20509_b200.engine import Schedule
    seq = Schedule(wl.spec.n, wl.spec.m, cfg).block_seq
    blocks = Schedule(wl.spec.n, wl.spec.m, cfg).row_blocks

    def ocb(t, s):
        I = blocks[int(seq[t])]
        ref_steps[t] = (s.b.copy(), s.v.copy(), s.u[I].copy(), s.nb_shape)

    ofinal, orep = _oracle_fit(pb, ost, ocfg, ocb)
    assert rep.diagnostics["iterations"] == orep.iterations == 10
    _compare_final(final, rep, ofinal, orep, wl.spec.n)

    got = {}

    def cb(t, s):
        I = blocks[int(seq[t])]
        got[t] = (s.b.copy(), s.v.copy(), s.u[I].copy(), s.nb_shape)

    _, rep2 = gk.fit_asgd(data, covs, fam, gk.Log(), gk.PenaltyConfig(), cfg, st,
                          offset=wl.offset, dtype="f32", callback=cb, identify_mode=None)
    assert rep2.objective_trace == rep.objective_trace     # same kernels, same order
    assert sorted(got) == list(range(10))
    for t in range(10):
        b, v, uI, nb = got[t]
        ob, ov, ouI, onb = ref_steps[t]
        assert normwise(v, ov) < 1e-4, t
        assert normwise(b, ob) < 1e-4, t
        assert normwise(uI, ouI) < 1e-4, t
        assert nb == pytest.approx(onb, rel=1e-4)


# ---------------------------------------------------------------- c5 sweep cells (gradient + update step)

C5_CELLS = [
    # (n*, m, d, family, dtype, k1_impl, y_format)
    (4096, 500, 5, "nb", "f32", "tensor", "csr"),
    (4096, 2000, 15, "nb", "f32", "tensor", "dense"),
    (4096, 5000, 5, "poisson", "f32", "tensor", "dense"),
    (4096, 5000, 50, "nb", "f32", "cuda_cores", "csr"),
    (4096, 500, 50, "poisson", "f32", "auto", "dense"),
    (4096, 2000, 15, "nb", "f64", "auto", "csr"),
    (4096, 5000, 5, "poisson", "f64", "auto", "dense"),
    (4096, 500, 50, "nb", "f64", "auto", "dense"),
    (256, 5000, 15, "nb", "f32", "tensor", "csr"),
]


@pytest.mark.parametrize("cell", C5_CELLS, ids=lambda c: "-".join(str(v) for v in c))
def test_c5_cell_gradient_matches_oracle(cell, k1_generation):
    """BASELINE config 5 cells: one block of n* rows x all m columns from a
    c1-style matrix (dense, or CSR at ~90% zeros), the fused block gradient and
    NB moment sums against the fp64 oracle (1e-10 fp64, 1e-4 fp32)."""
    from paper_2412_20509_b200.workloads import dense_to_csr
    nI, m, d, family, dtype, impl, yfmt = cell
    n = 2 * nI
    rng = np.random.default_rng(nI + m + d)
    u = rng.normal(0, 0.5 / np.sqrt(d / 5), (n, d))
    v = rng.normal(0, 0.5 / np.sqrt(d / 5), (m, d))
    b = rng.normal(1.0 if yfmt == "dense" else -2.6, 0.3, (m, 1))
    gamma = rng.normal(0, 0.3, (n, 1))
    eta = np.clip(u @ v.T + b.T + gamma, -15, 8)
    mu = np.exp(eta)
    y = rng.poisson(rng.gamma(2.0, mu / 2.0) if family == "nb" else mu)
    x, z = np.ones((n, 1)), np.ones((m, 1))
    noisy = lambda a: a + rng.normal(0, 0.05, a.shape)
    st = gk.FactorizationState(noisy(b), noisy(gamma), noisy(u), noisy(v), 1.0, 2.0)
    data = (gk.ResponseMatrix(csr=dense_to_csr(y), shape=y.shape) if yfmt == "csr"
            else gk.ResponseMatrix(y.astype(float)))
    covs = gk.CovariateSet(x=x, z=z, n=n, m=m)
    fam = gk.NegBinomial(2.0) if family == "nb" else gk.Poisson()
    I = np.sort(rng.choice(n, nI, replace=False))
    J = np.arange(m)
    gp, nbs = gk.minibatch_gradients(st, data, covs, fam, gk.Log(), gk.PenaltyConfig(),
                                     gk.Minibatch(I, J), dtype=dtype, k1_impl=impl,
                                     return_nb_sums=True)
    pb = orc.OProblem(y.astype(float), x, z)
    ost = orc.OState(st.b, st.gamma, st.u, st.v, 1.0, 2.0)
    fcode = orc.NEG_BINOMIAL if family == "nb" else orc.POISSON
    ref = orc.minibatch_gradients(ost, pb, I, J, fcode, orc.LOG, (0.0, 0.0, 1.0, 0.0))
    tol = 1e-10 if dtype == "f64" else 1e-4
    errs = {k: normwise(mine, r) for k, mine, r in (
        ("g_row", gp.g_rowside, ref.g_row), ("h_row", gp.h_rowside, ref.h_row),
        ("g_col", gp.g_colside, ref.g_col), ("h_col", gp.h_colside, ref.h_col))}
    assert max(errs.values()) < tol, errs
    if family == "nb":
        _, w, mu_b, _, _ = orc.block_derivs(ost, pb, I, J, fcode, orc.LOG)
        num, den = orc.nb_moment_sums(y[I].astype(float), mu_b, w)
        assert abs(nbs[0] - num) < tol * abs(num)
        assert abs(nbs[1] - den) < tol * (abs(num) + abs(den))
