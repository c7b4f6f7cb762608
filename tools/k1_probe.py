"""K1 timing probe on the c4 workload: per-step k_grad launches through
gmf_time_grad for each K1 implementation, plus the persistent-kernel geometry.
Usage: python tools/k1_probe.py [--impl tensor|cuda_cores|both] [--iters N]"""
import argparse
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--impl", default="both")
    ap.add_argument("--iters", type=int, default=200)
    ap.add_argument("--config", default="c4")
    args = ap.parse_args()
    import torch
    import paper_2412_20509_b200 as gk
    from paper_2412_20509_b200 import _lib, workloads
    from paper_2412_20509_b200.engine import DeviceFit, Schedule
    wl = workloads.generate(args.config, device="cuda")
    sp = wl.spec
    data = gk.ResponseMatrix(csr=wl.csr, shape=(sp.n, sp.m)) if sp.y_format == "csr" else \
        gk.ResponseMatrix(wl.y_dense.astype(float))
    covs = gk.CovariateSet(x=wl.x, z=wl.z if sp.q else None, m=sp.m)
    st = gk.FactorizationState(**wl.init_state())
    cfg = gk.SgdConfig(max_epochs=50, mb_rows=sp.mb_rows, mb_cols=sp.m, tol=1e-30)
    sch = Schedule(sp.n, sp.m, cfg)
    impls = ["tensor", "cuda_cores"] if args.impl == "both" else [args.impl]
    for impl in impls:
        fit = DeviceFit(data, covs, gk.NegBinomial(2.0), gk.Log(), gk.PenaltyConfig(), cfg, st,
                        schedule=sch, offset=wl.offset, dtype=sp.dtype, est_alpha=True, k1_impl=impl)
        fit.reset()
        geo = (C.c_int64 * 8)()
        fit.lib.gmf_geometry(fit.h, geo)
        avg = C.c_double()
        _lib.check(fit.lib.gmf_time_grad(fit.h, int(sch.block_seq[0]), args.iters, C.byref(avg),
                                         fit.stream()), "time_grad")
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        fit.run(20)
        e0.record()
        fit.run(200)
        e1.record()
        torch.cuda.synchronize()
        print(json.dumps({"impl": fit.k1_impl, "k1_us": avg.value * 1e3,
                          "step_us": e0.elapsed_time(e1) / 200 * 1e3,
                          "geometry": [int(v) for v in geo]}), flush=True)
        fit.close()


if __name__ == "__main__":
    main()
