"""Copy-stream probe for the streaming e2e leg on c4: how long the per-step
host -> device copies (packed-CSR slice, row pointers, ready signal) take on
their own, without the fit kernel running.
usage: python tools/e2e_probe.py [--steps E]"""
import argparse
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=400)
    args = ap.parse_args()
    import numpy as np
    import torch
    import paper_2412_20509_b200 as gk
    from paper_2412_20509_b200 import workloads
    from paper_2412_20509_b200.engine import DeviceFit, Schedule
    wl = workloads.generate("c4", device="cuda")
    sp = wl.spec
    data = gk.ResponseMatrix(csr=wl.csr, shape=(sp.n, sp.m))
    covs = gk.CovariateSet(x=wl.x, z=None, m=sp.m)
    st = gk.FactorizationState(**wl.init_state())
    E = args.steps
    cfg = gk.SgdConfig(max_epochs=E + 8, mb_rows=sp.mb_rows, mb_cols=sp.m, tol=1e-30, seed=0)
    sched = Schedule(sp.n, sp.m, cfg)
    fit = DeviceFit(data, covs, gk.NegBinomial(2.0), gk.Log(), gk.PenaltyConfig(), cfg, st,
                    schedule=sched, offset=wl.offset, dtype="f32", est_alpha=True)
    fit.reset()
    rbp = fit.rbp.cpu().numpy()
    h_col = fit.csr_col.cpu().pin_memory()
    h_ptr = fit.csr_ptr.cpu().pin_memory()
    cptr = h_ptr.numpy()
    seq = sched.block_seq
    cs = torch.cuda.Stream()
    for variant in ("col+ptr+signal", "col+signal", "col only"):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        import time
        w0 = time.perf_counter()
        with torch.cuda.stream(cs):
            e0.record(cs)
            for k in range(E):
                b = int(seq[k])
                r0, r1 = int(rbp[b]), int(rbp[b + 1])
                a0, a1 = int(cptr[r0]), int(cptr[r1])
                fit.csr_col[a0:a1].copy_(h_col[a0:a1], non_blocking=True)
                if variant == "col+ptr+signal":
                    fit.csr_ptr[r0:r1 + 1].copy_(h_ptr[r0:r1 + 1], non_blocking=True)
                if variant != "col only":
                    fit.stream_signal(k + 1, cs)
            e1.record(cs)
        w1 = time.perf_counter()
        torch.cuda.synchronize()
        print(f"{variant}: copy stream {e0.elapsed_time(e1) / E * 1e3:.1f} us/step, "
              f"host enqueue {(w1 - w0) / E * 1e6:.1f} us/step", flush=True)
    fit.close()


if __name__ == "__main__":
    main()
