"""The multi-rank step on NCCL: per step the objective / K1 kernels write the
rank record, NCCL all-gathers it and every rank applies the fixed-order sum
(optim._Exchange, exchange='device').  32 steps at a time are captured as one
CUDA graph (no per-step host loop).

On one GPU: a one-rank NCCL group drives the exchange path (optim's
_FORCE_EXCHANGE test hook) -- the graph-captured steps equal the eager steps
bitwise and both reproduce the reference's trajectory.  With >= 2 GPUs: two
ranks, one GPU each, reproduce the single-rank fit."""
import os
import socket

import numpy as np
import pytest

from conftest import REPO, golden, normwise

pytestmark = pytest.mark.gpu

gk = pytest.importorskip("paper_2412_20509_b200")


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem():
    g = golden("nb_offset")
    n, m = g["y"].shape
    data = gk.ResponseMatrix(g["y"].astype(float))
    covs = gk.CovariateSet(x=g["x"], m=m)
    st = gk.FactorizationState(g["init_b"], g["init_gamma"], g["init_u"], g["init_v"], 1.0,
                               float(g["init_nb"]))
    cfg = gk.SgdConfig(max_epochs=30, mb_rows=200, mb_cols=m, tol=1e-30, seed=3)
    return g, data, covs, st, cfg


@pytest.fixture
def nccl_group():
    import torch
    import torch.distributed as dist
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_port()}", rank=0,
                            world_size=1, device_id=torch.device("cuda", 0))
    try:
        yield dist.group.WORLD
    finally:
        dist.destroy_process_group()


def test_graph_captured_exchange_equals_eager_and_reference(nccl_group, monkeypatch):
    from paper_2412_20509_b200 import optim
    g, data, covs, st, cfg = _problem()
    monkeypatch.setattr(optim, "_FORCE_EXCHANGE", True)
    runs = {}
    for graph in (False, True):
        monkeypatch.setattr(optim, "_GRAPH_EXCHANGE", graph)
        final, rep = gk.fit_asgd(data, covs, gk.NegBinomial(1.5), gk.Log(), gk.PenaltyConfig(), cfg,
                                 st, offset=g["offset"], dtype="f64", process_group=nccl_group,
                                 exchange="device", identify_mode=None)
        runs[graph] = (final, rep)
    (a, ra), (b, rb) = runs[False], runs[True]
    assert ra.objective_trace == rb.objective_trace
    np.testing.assert_array_equal(a.u, b.u)
    np.testing.assert_array_equal(a.v, b.v)
    assert normwise(rb.objective_trace, g["trace"]) < 1e-10
    assert normwise(b.u @ b.v.T, g["unproj_u"] @ g["unproj_v"].T) < 1e-8


def _two_gpu_worker(rank, port, out):
    import sys
    sys.path.insert(0, REPO)
    import torch
    import torch.distributed as dist
    import paper_2412_20509_b200 as gk2
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=2, device_id=torch.device("cuda", rank))
    g, data, covs, st, cfg = _problem()
    final, rep = gk2.fit_asgd(data, covs, gk2.NegBinomial(1.5), gk2.Log(), gk2.PenaltyConfig(),
                              cfg, st, offset=g["offset"], dtype="f64", device=rank,
                              process_group=dist.group.WORLD, exchange="device",
                              identify_mode=None)
    if rank == 0:
        np.savez(out, trace=np.asarray(rep.objective_trace), uv=final.u @ final.v.T)
    dist.destroy_process_group()


def test_two_gpus_nccl_exchange_matches_single_rank(tmp_path):
    import torch
    import torch.multiprocessing as mp
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    out = str(tmp_path / "r0.npz")
    mp.spawn(_two_gpu_worker, args=(_port(), out), nprocs=2, join=True)
    r = np.load(out)
    g = golden("nb_offset")
    assert normwise(r["trace"], g["trace"]) < 1e-10
    assert normwise(r["uv"], g["unproj_u"] @ g["unproj_v"].T) < 1e-8


def test_general_mode_through_the_exchange_path(nccl_group, monkeypatch):
    """General mode (Gamma / log with the Pearson dispersion update) on the
    per-step kernels of the multi-rank path, eager and graph-captured: the
    Pearson sums ride in the rank record and phi advances in k_apply."""
    from paper_2412_20509_b200 import optim
    from test_general_oracle import case
    c = case(golden("general"), "gamma_log")
    n, m = c["y"].shape
    data = gk.ResponseMatrix(c["y"].astype(float))
    covs = gk.CovariateSet(x=c["x"], n=n, m=m)
    me, mr, mc, seed = (int(v) for v in c["cfg"])
    cfg = gk.SgdConfig(max_epochs=me, mb_rows=mr, mb_cols=mc, tol=1e-30, seed=seed)
    st = gk.FactorizationState(c["init_b"], c["init_gamma"], c["init_u"], c["init_v"], 1.0, 1.0)
    monkeypatch.setattr(optim, "_FORCE_EXCHANGE", True)
    for graph in (False, True):
        monkeypatch.setattr(optim, "_GRAPH_EXCHANGE", graph)
        final, rep = gk.fit_asgd(data, covs, gk.Gamma(), gk.Log(), gk.PenaltyConfig(), cfg, st,
                                 dtype="f64", process_group=nccl_group, exchange="device",
                                 identify_mode=None)
        assert normwise(rep.objective_trace, c["trace"]) < 1e-9, graph
        assert normwise(rep.phi_trace, c["phi_trace"]) < 1e-9, graph
        assert normwise(final.u @ final.v.T, c["unproj_u"] @ c["unproj_v"].T) < 1e-7, graph
        assert abs(final.phi - float(c["unproj_phi"])) < 1e-9 * float(c["unproj_phi"])
