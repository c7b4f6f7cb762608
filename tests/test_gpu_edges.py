"""Edge cases of the block gradient (K1) and the fit kernel on the GPU,
against the CPU oracle: empty and full responses, the CSR staging overflow
path, counts past the packed-CSR limit, degenerate shapes, and a fit whose
row blocks are ragged.  Tolerances: the north star's (fp64 1e-10, fp32
gradients 1e-4 normwise)."""
import numpy as np
import pytest

from conftest import normwise
from oracle import asgd_oracle as orc

pytestmark = pytest.mark.gpu

gk = pytest.importorskip("paper_2412_20509_b200")


@pytest.fixture(autouse=True)
def _gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _state(rng, n, m, d, p, q):
    return gk.FactorizationState(rng.normal(0.3, 0.2, (m, p)), rng.normal(0, 0.2, (n, q)),
                                 rng.normal(0, 0.3, (n, d)), rng.normal(0, 0.3, (m, d)), 1.0, 2.0)


def _check(y, st, x, z, off, I, J, family, dtype, impl, csr):
    from paper_2412_20509_b200.workloads import dense_to_csr
    n, m = y.shape
    data = gk.ResponseMatrix(csr=dense_to_csr(y), shape=y.shape) if csr else gk.ResponseMatrix(y)
    covs = gk.CovariateSet(x=x, z=z, n=n, m=m)
    fam = gk.NegBinomial(2.0) if family == "nb" else gk.Poisson()
    lam = (0.3, 0.2, 1.0, 0.7)
    gp = gk.minibatch_gradients(st, data, covs, fam, gk.Log(), gk.PenaltyConfig(lam=1.0, blocks=lam),
                                gk.Minibatch(I, J), offset=off, dtype=dtype, k1_impl=impl)
    pb = orc.OProblem(y, x if x is not None else np.zeros((n, 0)),
                      z if z is not None else np.zeros((m, 0)), offset=off)
    ost = orc.OState(st.b, st.gamma, st.u, st.v, 1.0, 2.0)
    fcode = orc.NEG_BINOMIAL if family == "nb" else orc.POISSON
    ref = orc.minibatch_gradients(ost, pb, I, J, fcode, orc.LOG, lam)
    errs = {k: normwise(mine, r) for k, mine, r in (
        ("g_row", gp.g_rowside, ref.g_row), ("h_row", gp.h_rowside, ref.h_row),
        ("g_col", gp.g_colside, ref.g_col), ("h_col", gp.h_colside, ref.h_col))}
    return errs


IMPLS = [("f32", "tensor", 1e-4), ("f32", "cuda_cores", 1e-4), ("f64", "cuda_cores", 1e-10)]


@pytest.mark.parametrize("dtype,impl,tol", IMPLS, ids=lambda v: str(v))
def test_all_zero_response(dtype, impl, tol):
    """An all-zero Y (CSR with no nonzeros): only the mu terms remain."""
    rng = np.random.default_rng(1)
    n, m = 140, 90
    st = _state(rng, n, m, 4, 1, 0)
    x = np.ones((n, 1))
    y = np.zeros((n, m))
    errs = _check(y, st, x, None, None, np.arange(5, 120), np.arange(m), "nb", dtype, impl, True)
    assert max(errs.values()) < tol, errs


@pytest.mark.parametrize("dtype,impl,tol", IMPLS, ids=lambda v: str(v))
def test_fully_dense_csr_overflows_staging(dtype, impl, tol):
    """Every entry nonzero: a 32-row chunk holds 32 * 300 > kStageCap (2048)
    nonzeros, so the K1 reads the CSR range directly instead of staging it."""
    rng = np.random.default_rng(2)
    n, m = 96, 300
    st = _state(rng, n, m, 5, 1, 1)
    x = np.ones((n, 1))
    z = np.ones((m, 1))
    y = rng.poisson(3.0, (n, m)) + 1.0
    errs = _check(y, st, x, z, None, np.arange(n), np.arange(m), "poisson", dtype, impl, True)
    assert max(errs.values()) < tol, errs


def test_counts_past_packed_limit_use_csr32():
    """Counts above 65535 cannot be packed (count << 16 | col): the automatic
    format falls back to 32-bit CSR and the gradient still matches."""
    from paper_2412_20509_b200.engine import packable
    rng = np.random.default_rng(3)
    n, m = 64, 50
    st = _state(rng, n, m, 3, 1, 0)
    x = np.ones((n, 1))
    y = rng.poisson(2.0, (n, m)).astype(float)
    y[5, 7] = 70000.0
    y[40, 49] = 65536.0
    assert not packable(m, y[y > 0])
    errs = _check(y, st, x, None, None, np.arange(n), np.arange(m), "nb", "f32", "tensor", True)
    assert max(errs.values()) < 1e-4, errs


@pytest.mark.parametrize("dtype,impl,tol", IMPLS, ids=lambda v: str(v))
def test_degenerate_shapes(dtype, impl, tol):
    """One row, one column block of 3 columns, d = 1, no covariates."""
    rng = np.random.default_rng(4)
    n, m = 5, 3
    st = _state(rng, n, m, 1, 0, 0)
    y = rng.poisson(1.5, (n, m)).astype(float)
    errs = _check(y, st, None, None, None, np.array([2]), np.arange(m), "poisson", dtype, impl, False)
    assert max(errs.values()) < tol, errs


@pytest.mark.parametrize("dtype,tol", [("f64", 1e-9), ("f32", 1e-3)])
def test_fit_with_ragged_blocks_matches_oracle(dtype, tol):
    """mb_rows / mb_cols that do not divide n / m (short last row and column
    blocks), NB with its shape estimated: the objective trace, NB shape trace
    and final U V' follow the oracle's fit."""
    rng = np.random.default_rng(5)
    n, m, d = 211, 77, 3
    st = _state(rng, n, m, d, 1, 0)
    x = np.ones((n, 1))
    y = rng.poisson(2.0, (n, m)).astype(float)
    cfg = gk.SgdConfig(max_epochs=6, mb_rows=50, mb_cols=30, tol=1e-30, seed=8)
    final, rep = gk.fit_asgd(gk.ResponseMatrix(y), gk.CovariateSet(x=x, n=n, m=m),
                             gk.NegBinomial(2.0), gk.Log(), gk.PenaltyConfig(), cfg, st, dtype=dtype)
    pb = orc.OProblem(y, x, np.zeros((m, 0)))
    ost = orc.OState(st.b, st.gamma, st.u, st.v, 1.0, 2.0)
    ocfg = orc.OConfig(max_epochs=6, mb_rows=50, mb_cols=30, tol=1e-30, seed=8)
    lam = (0.0, 0.0, 1.0, 0.0)   # PenaltyConfig() defaults: lam 1, blocks (0, 0, 1, 0)
    ofinal, orep = orc.fit_asgd(pb, orc.NEG_BINOMIAL, orc.LOG, lam, ocfg, ost)
    assert len(rep.objective_trace) == len(orep.objective_trace) > 3
    assert normwise(rep.objective_trace, orep.objective_trace) < tol
    assert normwise(rep.nb_shape_trace, orep.nb_shape_trace) < tol
    assert normwise(final.u @ final.v.T, ofinal.u @ ofinal.v.T) < tol


@pytest.mark.parametrize("dtype,tol", [("f32", 1e-4), ("f64", 1e-10)])
def test_rank50_gradient_uses_64_feature_bucket(dtype, tol):
    """c5's largest rank: K = p + q + d = 52 > 32 runs the CUDA-core K1 in the
    64-feature bucket (fp32: 64-column tiles; fp64: 32-column tiles with the
    row-side reduction in two feature halves; the tensor path is limited to
    q+d, p+d <= 16)."""
    rng = np.random.default_rng(6)
    n, m, d = 300, 180, 50
    st = _state(rng, n, m, d, 1, 1)
    st.u *= 0.3
    st.v *= 0.3
    x = np.ones((n, 1))
    z = np.ones((m, 1))
    y = rng.poisson(2.0, (n, m)).astype(float)
    errs = _check(y, st, x, z, None, np.arange(20, 260), np.arange(m), "nb", dtype, "auto", True)
    assert max(errs.values()) < tol, errs


def test_oversize_k1_tile_is_rejected_cleanly():
    """fp64 with prior weights at K = 64: the K1 tile exceeds the 227 KB of
    shared memory a CTA may use -> UnsupportedError, not a CUDA error."""
    from paper_2412_20509_b200 import _lib
    rng = np.random.default_rng(8)
    n, m, d = 80, 40, 62
    st = _state(rng, n, m, d, 1, 1)
    y = rng.poisson(2.0, (n, m)).astype(float)
    w = rng.uniform(0.5, 2.0, (n, m))
    with pytest.raises(_lib.UnsupportedError):
        gk.minibatch_gradients(st, gk.ResponseMatrix(y, weights=w),
                               gk.CovariateSet(x=np.ones((n, 1)), z=np.ones((m, 1))),
                               gk.Poisson(), gk.Log(), gk.PenaltyConfig(),
                               gk.Minibatch(np.arange(n), np.arange(m)), dtype="f64")


@pytest.mark.parametrize("y_format", ["dense", "csr"])
def test_rank50_fp64_fit_matches_oracle(y_format):
    """fp64 at rank 50 (persistent kernel, split row reduction) follows the
    oracle's fit at fp64 tolerance, dense and CSR."""
    rng = np.random.default_rng(17)
    n, m, d = 160, 90, 50
    st = _state(rng, n, m, d, 1, 0)
    st.u *= 0.2
    st.v *= 0.2
    x = np.ones((n, 1))
    y = rng.poisson(2.0, (n, m)).astype(float)
    cfg = gk.SgdConfig(max_epochs=5, mb_rows=40, mb_cols=m, tol=1e-30, seed=3)
    if y_format == "csr":
        import scipy.sparse as sp
        data = gk.ResponseMatrix(csr=sp.csr_matrix(y.astype(np.int32)), shape=(n, m))
    else:
        data = gk.ResponseMatrix(y)
    final, rep = gk.fit_asgd(data, gk.CovariateSet(x=x, n=n, m=m), gk.NegBinomial(2.0),
                             gk.Log(), gk.PenaltyConfig(), cfg, st, dtype="f64")
    pb = orc.OProblem(y, x, np.zeros((m, 0)))
    ost = orc.OState(st.b, st.gamma, st.u, st.v, 1.0, 2.0)
    ocfg = orc.OConfig(max_epochs=5, mb_rows=40, mb_cols=m, tol=1e-30, seed=3)
    ofinal, orep = orc.fit_asgd(pb, orc.NEG_BINOMIAL, orc.LOG, (0.0, 0.0, 1.0, 0.0), ocfg, ost)
    assert len(rep.objective_trace) == len(orep.objective_trace)
    assert normwise(rep.objective_trace, orep.objective_trace) < 1e-10
    assert normwise(final.u @ final.v.T, ofinal.u @ ofinal.v.T) < 1e-9


def test_rank50_fit_matches_oracle():
    """A short fp32 fit at rank 50 (64-feature bucket, persistent kernel and
    cached objective) follows the oracle's trace within the fp32 bounds."""
    rng = np.random.default_rng(7)
    n, m, d = 160, 90, 50
    st = _state(rng, n, m, d, 1, 0)
    st.u *= 0.2
    st.v *= 0.2
    x = np.ones((n, 1))
    y = rng.poisson(2.0, (n, m)).astype(float)
    cfg = gk.SgdConfig(max_epochs=5, mb_rows=40, mb_cols=m, tol=1e-30, seed=3)
    final, rep = gk.fit_asgd(gk.ResponseMatrix(y), gk.CovariateSet(x=x, n=n, m=m), gk.Poisson(),
                             gk.Log(), gk.PenaltyConfig(), cfg, st, dtype="f32")
    pb = orc.OProblem(y, x, np.zeros((m, 0)))
    ost = orc.OState(st.b, st.gamma, st.u, st.v, 1.0, 2.0)
    ocfg = orc.OConfig(max_epochs=5, mb_rows=40, mb_cols=m, tol=1e-30, seed=3)
    ofinal, orep = orc.fit_asgd(pb, orc.POISSON, orc.LOG, (0.0, 0.0, 1.0, 0.0), ocfg, ost)
    assert len(rep.objective_trace) == len(orep.objective_trace)
    assert normwise(rep.objective_trace, orep.objective_trace) < 1e-4
    assert normwise(final.u @ final.v.T, ofinal.u @ ofinal.v.T) < 1e-3
