"""Time the §8f consumers at the c4 shape (1.3M x 500 NB, CSR ~92 % zeros):
the one-pass log-likelihood behind information_criteria (k_objfull with the
NB dispersion constant), held-out scoring of 1M entries (k_entries), and
init_ols_svd (gmf_csr_spmm / gmf_init_moments + cuSOLVER on the sketches).
CUDA events on the launching stream, after a warm-up call; prints one JSON
object.  Usage: python tools/aux_bench.py [--config c4] [--reps 5]"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_20509_b200 as gk  # noqa: E402
from paper_2412_20509_b200 import _lib, workloads  # noqa: E402
from paper_2412_20509_b200.initialization import init_ols_svd  # noqa: E402
from paper_2412_20509_b200.select import _entries, _state_fit  # noqa: E402


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--dtype", default=None)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    wl = workloads.generate(a.config, device="cuda:0")
    sp = wl.spec
    data = gk.ResponseMatrix(csr=wl.csr, shape=(sp.n, sp.m))
    covs = gk.CovariateSet(x=wl.x, z=wl.z if sp.q else None, m=sp.m)
    st = gk.FactorizationState(**wl.init_state())
    fam = gk.NegBinomial(st.nb_shape)
    dtype = a.dtype or sp.dtype
    nnz = int(wl.csr[0][-1])
    out = {"config": sp.name, "n": sp.n, "m": sp.m, "d": sp.d, "nnz": nnz, "dtype": dtype}

    fit = _state_fit(st, data, covs, fam, gk.Log(), wl.offset, dtype, 0)
    res = torch.zeros(2, dtype=torch.float64, device=dev)
    call = lambda: _lib.check(fit.lib.gmf_loglik_full(fit.h, _lib.ptr(res), fit.stream()), "ll")
    ms = timed(call, a.reps)
    e = 4 if dtype == "f32" else 8
    ll_bytes = nnz * 4 + (sp.n + 1) * 8 + sp.n * e * (sp.d + sp.p + 1) + sp.m * e * (sp.d + sp.p)
    out["loglik_full"] = {"ms": ms, "entries_per_s": sp.n * sp.m / (ms * 1e-3),
                          "algorithmic_bytes": ll_bytes, "GB_s": ll_bytes / (ms * 1e-3) / 1e9,
                          "note": "predictor + exp/log1p per entry over all n*m entries "
                                  "(fp32 transcendentals on the f32 path, fp64 on f64), lgamma "
                                  "at the nonzeros; instruction-issue bound (ncu)"}
    rng = np.random.default_rng(0)
    nt = 1_000_000
    rows, cols = rng.integers(0, sp.n, nt), rng.integers(0, sp.m, nt)
    r, c = _entries(fit, rows, cols)
    yd = torch.from_numpy(rng.integers(0, 5, nt).astype(float)).to(dev)
    sums = torch.zeros(4, dtype=torch.float64, device=dev)
    call = lambda: _lib.check(fit.lib.gmf_entries_eval(fit.h, _lib.ptr(r), _lib.ptr(c),
                                                       _lib.ptr(yd), nt, 1.0, None,
                                                       _lib.ptr(sums), fit.stream()), "ent")
    ms = timed(call, a.reps)
    out["heldout_scores"] = {"ms": ms, "entries": nt, "entries_per_s": nt / (ms * 1e-3)}
    fit.close()

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    init_ols_svd(data, covs, fam, gk.Log(), sp.d, seed=0)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    init_ols_svd(data, covs, fam, gk.Log(), sp.d, seed=0)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    out["init_ols_svd"] = {"s_first": t1 - t0, "s_second": t2 - t1,
                           "note": "wall clock incl. host->device CSR upload and CSC build; "
                                   "no n x m array is formed (reference: dense f64 n x m)"}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
