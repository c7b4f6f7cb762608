"""BASELINE config 5 / SURVEY §8d c5: the isolated gradient + update step
swept over block rows n* in {256, 4096, 65536} x columns m in {500, 2000,
5000} x rank d in {5, 15, 50}, Poisson and NB, fp32 and fp64, dense and CSR
(~90 % zeros) counts.

Counts are drawn as c1 (Poisson, X = Z = ones) from an n = 65,536-row matrix
per (m, format) on the GPU (seeded synthetic data; the CSR variant's
intercept is calibrated to 90 % zeros).  Each cell builds a device fit with
mb_rows = n*, mb_cols = m and a 1,024-entry tracked sample (so the step is
the gradient + update with a negligible objective), runs W warm-up steps,
then times K steps of one persistent launch with CUDA events, and, as a
second figure, the block gradient K1 alone (per-step kernel, gmf_time_grad).
Reported per cell: step and K1 time, entries/s (n* m per step), algorithmic
bytes per step (bench._step_bytes) and the achieved fraction of
the measured HBM bandwidth.  fp64 at K = p+q+d > 32 (d = 50) runs the
fp64 64-feature bucket (32-column tiles, row-side reduction in two feature
halves).

usage: python tools/sweep_c5.py [--steps K] [--warmup W] [--quick] > out.jsonl
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--quick", action="store_true", help="m = 500 only")
    ap.add_argument("--only-d", type=int, default=None, help="one rank only")
    ap.add_argument("--only-dtype", default=None, help="f32 or f64 only")
    ap.add_argument("--only-m", type=int, default=None, help="one column count only")
    ap.add_argument("--only-family", default=None, help="poisson or nb only")
    ap.add_argument("--only-nstar", type=int, default=None, help="one block size only")
    ap.add_argument("--only-format", default=None, help="dense or csr only")
    args = ap.parse_args()
    import torch
    import paper_2412_20509_b200 as gk
    from paper_2412_20509_b200 import _lib, workloads
    from paper_2412_20509_b200.engine import DeviceFit, Schedule
    import bench

    peak, peak_src = bench._peak_hbm()
    N = 65536
    ms_list = [500] if args.quick else [500, 2000, 5000]
    if args.only_m:
        ms_list = [args.only_m]
    for m in ms_list:
        for fmt in ((args.only_format,) if args.only_format else ("dense", "csr")):
            spec = workloads.WorkloadSpec("c5", N, m, 5, "poisson", "f32", fmt, 256, 1, p=1, q=1,
                                          zero_frac=0.90 if fmt == "csr" else None)
            t0 = time.perf_counter()
            wl = workloads.generate(spec, device="cuda")
            gen_s = time.perf_counter() - t0
            if fmt == "csr":
                data = gk.ResponseMatrix(csr=wl.csr, shape=(N, m))
            else:
                data = gk.ResponseMatrix(wl.y_dense.astype(float))
            covs = gk.CovariateSet(x=wl.x, z=wl.z, m=m)
            print(json.dumps({"gen": {"m": m, "format": fmt, "seconds": round(gen_s, 1),
                                      "zero_frac": round(wl.meta["zero_frac"], 4)}}), flush=True)
            rng = np.random.default_rng(0)
            for d in ((args.only_d,) if args.only_d else (5, 15, 50)):
                st = gk.FactorizationState(wl.truth["b"], wl.truth["gamma"],
                                           0.3 * rng.standard_normal((N, d)),
                                           0.3 * rng.standard_normal((m, d)), 1.0, 2.0)
                for family in ((args.only_family,) if args.only_family else ("poisson", "nb")):
                    for dtype in ((args.only_dtype,) if args.only_dtype else ("f32", "f64")):
                        for nstar in ((args.only_nstar,) if args.only_nstar else (256, 4096, 65536)):
                            cell = {"nstar": nstar, "m": m, "d": d, "family": family,
                                    "dtype": dtype, "format": fmt}
                            try:
                                cell.update(_cell(gk, _lib, DeviceFit, Schedule, bench, torch, data,
                                                  covs, st, family, dtype, nstar, m, d, fmt,
                                                  args, peak))
                            except _lib.UnsupportedError as e:
                                cell["unsupported"] = str(e).split(": ", 1)[-1][:120]
                            print(json.dumps(cell), flush=True)
            del data, wl
            torch.cuda.empty_cache()
    print(json.dumps({"peak_hbm_gbs": peak, "peak_source": peak_src}), flush=True)


def _cell(gk, _lib, DeviceFit, Schedule, bench, torch, data, covs, st, family, dtype, nstar, m,
          d, fmt, args, peak):
    N = st.u.shape[0]
    W, K = args.warmup, args.steps
    cfg = gk.SgdConfig(max_epochs=W + K + 4, mb_rows=nstar, mb_cols=m, tol=1e-30, seed=0,
                       max_eval_entries=1024)
    sch = Schedule(N, m, cfg)
    fam = gk.NegBinomial(2.0) if family == "nb" else gk.Poisson()
    fit = DeviceFit(data, covs, fam, gk.Log(), gk.PenaltyConfig(), cfg, st, schedule=sch,
                    dtype=dtype, est_alpha=family == "nb")
    try:
        fit.reset()
        fit.run(W)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fit.run(K)
        e1.record()
        torch.cuda.synchronize()
        step_ms = e0.elapsed_time(e1) / K
        status = fit.status()
        assert status.t == W + K and not status.stopped, (status.t, status.stopped)
        avg = C.c_double()
        _lib.check(fit.lib.gmf_time_grad(fit.h, int(sch.block_seq[0]), 20, C.byref(avg),
                                         fit.stream()), "gmf_time_grad")
        k1_ms = avg.value
        impl = fit.k1_impl
        packed = fit.y_format == "packed"
        # the timed steps' blocks: rows and nonzeros (block-major layout)
        rbp = fit.rbp.cpu().numpy()
        seq = np.asarray(sch.block_seq[W:W + K])
        rows = (rbp[seq + 1] - rbp[seq]).astype(float)
        if fit.csr_ptr is not None:
            cptr = fit.csr_ptr.cpu().numpy()
            nnz = (cptr[rbp[seq + 1]] - cptr[rbp[seq]]).astype(float)
        else:
            nnz = np.zeros_like(rows)
    finally:
        fit.close()
    nI, nnz_I = float(rows.mean()), float(nnz.mean())

    class _S:
        pass
    sp = _S()
    sp.p, sp.q, sp.d, sp.m, sp.y_format, sp.offset = 1, 1, d, m, fmt, False
    e = 4 if dtype == "f32" else 8
    byts = bench._step_bytes(sp, nI, nnz_I, e, 4 if packed else 8)
    achieved = byts / (step_ms * 1e-3) / 1e9
    return {"impl": impl, "y_format": "packed" if packed else ("csr32" if fmt == "csr" else "dense"),
            "step_us": round(step_ms * 1e3, 2), "k1_us": round(k1_ms * 1e3, 2),
            "entries_per_s": nI * m / (step_ms * 1e-3),
            "bytes_per_step": int(byts), "hbm_gbs": round(achieved, 1),
            "hbm_frac": round(achieved / peak, 4)}


if __name__ == "__main__":
    main()
