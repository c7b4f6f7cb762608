"""Multi-rank path.

CPU (gloo, world size 2): the row-sharded decomposition the device engine
uses -- each rank owns a slice of every row block, computes column-side
partials, NB moment sums and objective partials for its rows, all-gathers
the records and sums them in rank order -- reproduces the single-process
oracle step exactly (host logic of engine.shard_rows / optim._Exchange).

GPU (gloo host exchange, 2 processes on one device): the C-ABI per-step
kernels (gmf_step_local / gmf_step_apply) across 2 ranks reproduce the
single-rank fit.  No kernel waits on another rank: records cross ranks
through host memory between kernel launches.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import REPO, golden, normwise


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


# ---------------------------------------------------------------- CPU, gloo

def _cpu_worker(rank, world, port, out):
    import sys
    sys.path.insert(0, REPO)
    from oracle import asgd_oracle as orc
    from paper_2412_20509_b200 import SgdConfig
    from paper_2412_20509_b200.engine import Schedule, shard_rows
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = golden("nb_offset")
    y = g["y"].astype(float)
    n, m = y.shape
    pb = orc.OProblem(y, g["x"], g["z"], offset=g["offset"])
    st = orc.OState(g["init_b"], g["init_gamma"], g["init_u"], g["init_v"], 1.0,
                    float(g["init_nb"]))
    cfg = SgdConfig(max_epochs=3, mb_rows=200, mb_cols=m, seed=3)
    sch = Schedule(n, m, cfg)
    blk = int(sch.block_seq[0])
    order, ptr, scale = shard_rows(sch, world, rank)
    rows = order[ptr[blk]:ptr[blk + 1]]          # this rank's slice of block I
    I = sch.row_blocks[blk]
    J = np.arange(m)
    # rank-local record: unscaled column partials + NB sums
    _, w, mu, dd, hh = orc.block_derivs(st, pb, rows, J, orc.NEG_BINOMIAL, orc.LOG)
    a_col = np.hstack([pb.x[rows], st.u[rows]])
    rec = np.concatenate([(dd.T @ a_col).ravel(), (hh.T @ (a_col ** 2)).ravel(),
                          np.array(orc.nb_moment_sums(y[rows][:, J], mu, w))])
    t = torch.from_numpy(rec)
    gathered = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(gathered, t)
    tot = sum(x.numpy() for x in gathered)        # fixed rank order
    kc = pb.x.shape[1] + st.u.shape[1]
    s_col = n / I.size
    g_col = s_col * tot[:m * kc].reshape(m, kc)
    h_col = s_col * tot[m * kc:2 * m * kc].reshape(m, kc) + 0.0
    ref = orc.minibatch_gradients(st, pb, I, J, orc.NEG_BINOMIAL, orc.LOG, (0.0, 0.0, 1.0, 0.0))
    _, w2, mu2, _, _ = orc.block_derivs(st, pb, I, J, orc.NEG_BINOMIAL, orc.LOG)
    num, den = orc.nb_moment_sums(y[I][:, J], mu2, w2)
    out[rank] = (normwise(g_col, ref.g_col), normwise(h_col, ref.h_col),
                 abs(tot[-2] - num) / abs(num), abs(tot[-1] - den) / abs(den))
    dist.destroy_process_group()


def test_row_sharded_records_sum_to_single_rank_gradient():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_cpu_worker, args=(world, port, out), nprocs=world, join=True)
    for r in range(world):
        gc, hc, dn, dd = out[r]
        assert gc < 1e-12 and hc < 1e-12 and dn < 1e-12 and dd < 1e-12, out[r]


# ---------------------------------------------------------------- GPU, 2 ranks

def _gpu_worker(rank, world, port, out, dtype):
    import sys
    sys.path.insert(0, REPO)
    import paper_2412_20509_b200 as gk
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    g = golden("nb_cov_s3")
    data = gk.ResponseMatrix(g["y"].astype(float))
    covs = gk.CovariateSet(x=g["x"], z=g["z"])
    st = gk.FactorizationState(g["init_b"], g["init_gamma"], g["init_u"], g["init_v"], 1.0,
                               float(g["init_nb"]))
    me, mr, mc, seed, cap = (int(v) for v in g["cfg"])
    cfg = gk.SgdConfig(max_epochs=me, mb_rows=mr, mb_cols=mc, seed=seed, tol=1e-30)
    pen = gk.PenaltyConfig(lam=1.0, blocks=tuple(float(v) for v in g["lam"]))
    final, rep = gk.fit_asgd(data, covs, gk.NegBinomial(st.nb_shape), gk.Log(), pen, cfg, st,
                             dtype=dtype, process_group=dist.group.WORLD, exchange="host")
    out[rank] = (np.asarray(rep.objective_trace), final.u @ final.v.T, rep.epochs_run,
                 rep.final_objective)
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_two_ranks_match_single_rank_fit(dtype):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2412_20509_b200 as gk
    g = golden("nb_cov_s3")
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_gpu_worker, args=(r, world, port, out, dtype)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    data = gk.ResponseMatrix(g["y"].astype(float))
    covs = gk.CovariateSet(x=g["x"], z=g["z"])
    st = gk.FactorizationState(g["init_b"], g["init_gamma"], g["init_u"], g["init_v"], 1.0,
                               float(g["init_nb"]))
    me, mr, mc, seed, cap = (int(v) for v in g["cfg"])
    cfg = gk.SgdConfig(max_epochs=me, mb_rows=mr, mb_cols=mc, seed=seed, tol=1e-30)
    pen = gk.PenaltyConfig(lam=1.0, blocks=tuple(float(v) for v in g["lam"]))
    final, rep = gk.fit_asgd(data, covs, gk.NegBinomial(st.nb_shape), gk.Log(), pen, cfg, st,
                             dtype=dtype)
    tol = 1e-10 if dtype == "f64" else 1e-4
    for r in range(world):
        trace, uv, epochs, fobj = out[r]
        assert epochs == rep.epochs_run
        assert normwise(trace, rep.objective_trace) < tol
        assert normwise(uv, final.u @ final.v.T) < (1e-8 if dtype == "f64" else 1e-3)
        assert abs(fobj - rep.final_objective) < tol * abs(rep.final_objective) * 10
    # reference trajectory too
    assert normwise(out[0][0], g["trace"]) < tol
