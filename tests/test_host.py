"""CPU-only tests: the C-ABI library loads and exports every declared
symbol, and the host logic (schedule replay, sharding, layouts, config
validation, error mapping) agrees with the oracle / reference contracts."""
import os
import re

import numpy as np
import pytest

from conftest import REPO
from oracle import asgd_oracle as orc

import paper_2412_20509_b200 as gk
from paper_2412_20509_b200 import _lib
from paper_2412_20509_b200.engine import Schedule, eval_entries, permute_csr, shard_rows
from paper_2412_20509_b200.workloads import dense_to_csr


def _declared_symbols():
    hdr = open(os.path.join(REPO, "include", "gmf_asgd.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(gmf_[a-z_0-9]+)\s*\(", hdr)))


def test_library_exports_every_declared_symbol():
    so = _lib.lib()
    declared = _declared_symbols()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(so, name), name
        assert name in _lib.SIGNATURES, name
    assert b"sm_100a" in so.gmf_version()


def test_library_error_plumbing_without_gpu():
    so = _lib.lib()
    rc = so.gmf_mean_of_eta(99, _lib.F64, None, None, 0, None)
    assert rc == _lib.GMF_ERR_DOMAIN
    assert "link" in _lib.last_error()
    with pytest.raises(gk.DomainError):
        _lib.check(rc)
    assert so.gmf_cross_work_bytes(3, 4) > 0


def test_device_entry_points_refuse_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    data = gk.ResponseMatrix(np.ones((4, 3)))
    covs = gk.CovariateSet.empty(4, 3)
    st = gk.FactorizationState.zeros(4, 3, d=1)
    with pytest.raises(_lib.CudaError):
        gk.fit_asgd(data, covs, gk.Poisson(), gk.Log(), gk.PenaltyConfig(), gk.SgdConfig(), st)


@pytest.mark.parametrize("n,m,mbr,mbc,epochs,cap", [
    (1000, 100, 100, 100, 50, 100_000),     # c1: eval = everything
    (1200, 150, 200, 150, 30, 100_000),     # sample drawn
    (900, 120, 150, 40, 12, 100_000),       # S = 3
    (26472, 500, 2000, 500, 5, 100_000),    # c2 shape: 14 blocks of 1890-1891
])
def test_schedule_replays_reference_rng(n, m, mbr, mbc, epochs, cap):
    cfg = gk.SgdConfig(max_epochs=epochs, mb_rows=mbr, mb_cols=mbc, seed=3, max_eval_entries=cap)
    s = Schedule(n, m, cfg)
    ocfg = orc.OConfig(max_epochs=epochs, mb_rows=mbr, mb_cols=mbc, seed=3, max_eval_entries=cap)
    rb, cb, ent, seq = orc.replay_schedule(n, m, ocfg)
    assert len(s.row_blocks) == len(rb) and all(np.array_equal(a, b) for a, b in zip(s.row_blocks, rb))
    assert all(np.array_equal(a, b) for a, b in zip(s.col_blocks, cb))
    assert np.array_equal(s.eval_rows, ent[0]) and np.array_equal(s.eval_cols, ent[1])
    assert s.eval_scale == ent[2]
    assert s.block_seq.tolist() == seq


def test_eval_entries_fast_path_equals_nonzero_path():
    rng1, rng2 = np.random.default_rng(5), np.random.default_rng(5)
    mask = np.ones((300, 70), dtype=bool)
    a = eval_entries(300, 70, 1000, rng1)
    b = eval_entries(300, 70, 1000, rng2, mask=mask)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and a[2] == b[2]
    assert rng1.integers(1 << 30) == rng2.integers(1 << 30)


def test_c2_block_sizes_match_survey():
    s = Schedule(26472, 500, gk.SgdConfig(max_epochs=1, mb_rows=2000, mb_cols=500))
    sizes = sorted({b.size for b in s.row_blocks})
    assert len(s.row_blocks) == 14 and sizes == [1890, 1891]


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_rows_partitions_every_block(world):
    s = Schedule(1003, 20, gk.SgdConfig(max_epochs=1, mb_rows=97, mb_cols=20))
    seen = []
    for r in range(world):
        order, ptr, scale = shard_rows(s, world, r)
        assert ptr[-1] == order.size
        for k, blk in enumerate(s.row_blocks):
            part = order[ptr[k]:ptr[k + 1]]
            assert np.isin(part, blk).all()
            assert scale[k] == pytest.approx(1003 / blk.size)
        seen.append(order)
    allrows = np.sort(np.concatenate(seen))
    assert np.array_equal(allrows, np.arange(1003))


def test_permute_csr_matches_dense(rng):
    y = rng.poisson(0.3, size=(57, 23)).astype(np.int32)
    ptr, idx, val = dense_to_csr(y)
    order = rng.permutation(57)
    p2, i2, v2 = permute_csr(ptr, idx, val, order)
    dense = np.zeros_like(y)
    for r in range(57):
        dense[r, i2[p2[r]:p2[r + 1]]] = v2[p2[r]:p2[r + 1]]
    assert np.array_equal(dense, y[order])


def test_config_validation_mirrors_reference():
    with pytest.raises(gk.ConfigError):
        gk.SgdConfig(rate_tau=0.4)
    with pytest.raises(gk.ConfigError):
        gk.SgdConfig(smooth_a1=0.0)
    with pytest.raises(gk.ConfigError):
        gk.SgdConfig(rate_k0=0.0)
    gk.SgdConfig(rate_k1=0.0)
    assert gk.learning_rate(0, gk.SgdConfig(rate_k0=0.03)) == 0.03
    assert gk.learning_rate(100, gk.SgdConfig(rate_k0=0.01, rate_k1=1.0, rate_tau=1.0)) == pytest.approx(0.005)
    assert gk.bias_correction(1, 0.1, 0.01) == pytest.approx(1.1)
    with pytest.raises(gk.ConfigError):
        gk.bias_correction(0, 0.1, 0.01)
    g, h = gk.smooth_update(0.0, 0.0, 10.0, 4.0, 0.1, 0.5)
    assert g == pytest.approx(1.0) and h == pytest.approx(2.0)
    assert gk.parameter_count(5000, 500, 3, 1, 5) == 34001


def test_minibatch_and_response_validation():
    with pytest.raises(gk.ConfigError):
        gk.Minibatch([], [1])
    with pytest.raises(gk.ConfigError):
        gk.Minibatch([1, 1], [0])
    with pytest.raises(gk.ConfigError):
        gk.ResponseMatrix(csr=(np.array([0, 1]), np.array([5]), np.array([1])), shape=(1, 3))
    with pytest.raises(gk.ConfigError):
        gk.ResponseMatrix(np.ones((2, 2)), weights=np.zeros((2, 2)))
    r = gk.ResponseMatrix(csr=dense_to_csr(np.eye(3, dtype=np.int32)), shape=(3, 3))
    assert r.fully_observed and r.n_observed == 9


def test_fit_requires_init_state():
    data = gk.ResponseMatrix(np.ones((4, 3)))
    covs = gk.CovariateSet.empty(4, 3)
    with pytest.raises(gk.ConfigError):
        gk.fit_asgd(data, covs, gk.Poisson(), gk.Log(), gk.PenaltyConfig(), gk.SgdConfig())


def test_exception_taxonomy_matches_reference():
    assert issubclass(gk.ConfigError, ValueError) and issubclass(gk.ConfigError, gk.GmfError)
    assert issubclass(gk.DivergenceError, ArithmeticError)
    e = gk.DivergenceError("x", state=1)
    assert e.state == 1


def test_packed_csr_round_trip():
    from paper_2412_20509_b200.engine import pack_csr, packable, unpack_csr
    rng = np.random.default_rng(4)
    cols = rng.integers(0, 65536, size=1000)
    counts = rng.integers(0, 65536, size=1000)
    w = pack_csr(cols, counts)
    assert w.dtype == np.int32 and w.size == 1000
    c2, v2 = unpack_csr(w)
    assert np.array_equal(c2, cols) and np.array_equal(v2, counts)
    assert packable(65536, counts) and not packable(65537, counts)
    assert not packable(10, np.array([0, 65536])) and packable(10, np.array([], dtype=int))


def test_csr_input_is_canonicalized():
    """Unsorted rows, duplicate coordinates and explicit zeros are rewritten
    to the canonical CSR of the dense matrix the reference sees (duplicates
    summed, as scipy's densify does; io.py:104-109)."""
    import scipy.sparse as sp
    rng = np.random.default_rng(3)
    n, m, nnz = 40, 17, 300
    r = rng.integers(0, n, nnz)
    c = rng.integers(0, m, nnz)
    v = rng.integers(0, 4, nnz)            # includes explicit zeros
    coo = sp.coo_matrix((v, (r, c)), shape=(n, m))
    dense = coo.toarray()
    # a deliberately non-canonical CSR: rows grouped, columns shuffled inside rows
    order = np.lexsort((rng.random(nnz), r))
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(r, minlength=n), out=indptr[1:])
    data = gk.ResponseMatrix(csr=(indptr, c[order], v[order]), shape=(n, m))
    ip, ix, dv = data.csr
    assert np.all(dv != 0)
    for i in range(n):
        cols = ix[ip[i]:ip[i + 1]]
        assert np.all(np.diff(cols) > 0)
    back = sp.csr_matrix((dv, ix, ip), shape=(n, m)).toarray()
    np.testing.assert_array_equal(back, dense)
    # canonical input passes through unchanged (no copy)
    canon = sp.csr_matrix(dense)
    canon.eliminate_zeros()
    d2 = gk.ResponseMatrix(csr=canon, shape=(n, m))
    assert d2.csr[1] is not None and np.array_equal(d2.csr[1], canon.indices)
