#!/usr/bin/env python
"""bench.py -- aSGD matrix entries/s on BASELINE.json config 4 (the north
star's headline workload): negative-binomial GMF, 1,300,000 x 500, rank 10,
intercept + centred log-library-size offset, CSR int32 counts (~92% zeros),
minibatch 10,000 rows x all 500 columns, fp32.

A "step" is one aSGD step of the reference semantics (optim.py:421-476):
one drawn row block x all columns (= one epoch, S = 1), including the tracked
objective.  ``value`` = sum_t |I_t| * m / device time with inputs resident
in HBM; ``e2e`` streams each step's block from pinned host memory and reads
the step's objective back.  Run:

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

N > 1 is launched by torchrun (one process per GPU, NCCL); every rank
processes its slice of the same drawn block each step (row sharding with a
per-step all-gather of the column-side partials), timed as max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "aSGD matrix entries/sec"
UNIT = "entries/s"


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20000)
    ap.add_argument("--warmup", type=int, default=200)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4", choices=["c1", "c2", "c3", "c4"])
    ap.add_argument("--e2e-steps", type=int, default=400)
    ap.add_argument("--cpu-steps", type=int, default=12)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--phases", type=int, default=0)
    ap.add_argument("--no-aux", action="store_true",
                    help="skip the model-selection / initialization legs (SURVEY 8f)")
    ap.add_argument("--k1-impl", default="auto", choices=["auto", "tensor", "cuda_cores"])
    return ap.parse_args()


def _peak_hbm():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md recipe)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.samples = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-i", str(self.idx), "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append((time.perf_counter(), line.strip()))

    def stop(self, t0, t1):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(2)
        except Exception:
            self.proc.kill()
        rows = [s for (ts, s) in self.samples if t0 - 0.1 <= ts <= t1 + 0.15] or \
               [s for _, s in self.samples[-2:]]
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            f = [x.strip() for x in r.split(",")]
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except Exception:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws == 1 and not os.environ.get("GMF_BENCH_FORCE_EXCHANGE"):
        return 1, 0, 0, None
    import torch
    import torch.distributed as dist
    lr = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(lr)
    if ws == 1:   # test hook: the multi-rank code path on a one-rank NCCL group
        dist.init_process_group("nccl", init_method="tcp://127.0.0.1:29581", rank=0, world_size=1,
                                device_id=torch.device("cuda", lr))
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", lr))
    return ws, dist.get_rank(), lr, dist.group.WORLD


def _k1_bytes(spec, nI, nnz_I, e, nnz_bytes=8):
    """Algorithmic HBM bytes of one K1 launch: the block's
    counts (nnz_bytes per stored nonzero: 8 CSR int32, 4 packed), row
    features and offset read once, column features read once, row-side and
    column-side gradient partials written once."""
    p, q, d, m = spec.p, spec.q, spec.d, spec.m
    y = nnz_bytes * nnz_I + 8 * (nI + 1) if spec.y_format == "csr" else 4 * nI * m
    rows = nI * e * (p + q + d + (1 if spec.offset else 0)) + nI * e * 2 * (q + d)
    cols = m * e * (p + q + d) + m * e * 2 * (p + d)
    return y + rows + cols


def _step_bytes(spec, nI, nnz_I, e, nnz_bytes=8):
    """Algorithmic bytes of a whole step: K1 + the EMA/update
    traffic (read gbar, hbar, theta; write them back) of rows I and columns J."""
    kr, kc = spec.q + spec.d, spec.p + spec.d
    return _k1_bytes(spec, nI, nnz_I, e, nnz_bytes) + nI * e * 6 * kr + spec.m * e * 6 * kc


def _cpu_baseline(wl, steps, time_budget=25.0):
    """The oracle port (oracle/asgd_oracle.py, numpy + OpenBLAS) on a bounded
    row sample of the same workload: 13 row blocks of mb_rows, same block
    shape, fully dense fp64 as the reference stores it (model.py:46-98)."""
    from oracle import asgd_oracle as orc
    sp = wl.spec
    nsub = min(sp.n, 13 * sp.mb_rows)
    rows = np.arange(nsub)
    y = wl.dense_f64(rows)
    off = None if wl.offset is None else wl.offset[rows]
    pb = orc.OProblem(y, wl.x[rows], wl.z, offset=off)
    init = wl.init_state()
    st = orc.OState(init["b"], init["gamma"][rows], init["u"][rows], init["v"], 1.0,
                    init["nb_shape"])
    cfg = orc.OConfig(max_epochs=steps, mb_rows=sp.mb_rows, mb_cols=sp.m, tol=1e-30, seed=0)
    stamps = [time.perf_counter()]
    fam = orc.NEG_BINOMIAL if sp.family == "neg_binomial" else orc.POISSON

    class _Stop(Exception):
        pass

    def cb(t, s):
        stamps.append(time.perf_counter())
        if stamps[-1] - stamps[0] > time_budget:
            raise _Stop()

    try:
        orc.fit_asgd(pb, fam, orc.LOG, (0.0, 0.0, 1.0, 0.0), cfg, st, identify=False,
                     callback=cb, final_objective=False)
    except _Stop:
        pass
    dts = np.diff(stamps)[2:] if len(stamps) > 4 else np.diff(stamps)
    step_s = float(np.median(dts))
    try:
        import threadpoolctl
        threads = max((p.get("num_threads", 1) for p in threadpoolctl.threadpool_info()), default=1)
    except Exception:
        threads = os.cpu_count()
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    return {"value": sp.mb_rows * sp.m / step_s, "unit": UNIT, "cores": int(min(cores, threads)),
            "kind": "port",
            "sample": (f"oracle/asgd_oracle.py fit_asgd on rows 0..{nsub} of {sp.name} "
                       f"({nsub // sp.mb_rows} blocks of {sp.mb_rows} x {sp.m}, dense fp64, "
                       f"tracked objective every step), median of {len(dts)} steps"),
            "ms_per_step": step_s * 1e3}


def _gmfkit_timing(wl, steps, time_budget=150.0):
    """The UNMODIFIED reference (gmfkit, installed into baseline/_ref with its
    compiled Cython kernel) through its own public fit_asgd on a bounded row
    sample of the workload (13 row blocks of mb_rows x all columns, dense fp64
    as gmfkit stores it), per-step wall time from callback timestamps exactly
    as the reference's own timing test does (test_acceptance.py:359-368).
    The per-row offset of c2/c4 enters through a runtime wrapper of gmfkit's
    three eta entry points (SURVEY 8c shim; the installed files are untouched).
    Returns None when baseline/_ref is missing."""
    ref = os.path.join(REPO, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "gmfkit")):
        return None
    if ref not in sys.path:
        sys.path.insert(0, ref)
    import gmfkit as G
    import gmfkit.kernels as GK
    import gmfkit.model as GM
    import gmfkit.optim as GO
    sp = wl.spec
    nsub = min(sp.n, 13 * sp.mb_rows)
    rows = np.arange(nsub)
    y = wl.dense_f64(rows)
    init = wl.init_state()
    st = G.FactorizationState(init["b"], init["gamma"][rows], init["u"][rows], init["v"], 1.0,
                              init["nb_shape"])
    data = G.ResponseMatrix(y)
    covs = G.CovariateSet(x=wl.x[rows], z=wl.z if sp.q else None, n=nsub, m=sp.m)
    fam = G.NegBinomial(init["nb_shape"]) if sp.family == "neg_binomial" else G.Poisson()
    cfg = G.SgdConfig(max_epochs=steps, mb_rows=sp.mb_rows, mb_cols=sp.m, tol=1e-30, seed=0)
    saved = (GM.linear_predictor, GO.linear_predictor, GO._entrywise_eta)
    if wl.offset is not None:
        off = wl.offset[rows]

        def lp(state, cv, r=None, c=None):
            eta = saved[0](state, cv, r, c)
            return eta + (off if r is None else off[np.asarray(r)])[:, None]

        def ent(state, cv, r, c):
            return saved[2](state, cv, r, c) + off[r]
        GM.linear_predictor = GO.linear_predictor = lp
        GO._entrywise_eta = ent
    stamps = [time.perf_counter()]

    class _Stop(Exception):
        pass

    def cb(t, s):
        stamps.append(time.perf_counter())
        if stamps[-1] - stamps[0] > time_budget:
            raise _Stop()

    try:
        G.fit_asgd(data, covs, fam, G.Log(), G.PenaltyConfig(), cfg, st, identify_mode=None,
                   callback=cb)
    except _Stop:
        pass
    finally:
        GM.linear_predictor, GO.linear_predictor, GO._entrywise_eta = saved
    dts = np.diff(stamps)[3:] if len(stamps) > 6 else np.diff(stamps)
    step_s = float(np.median(dts))
    try:
        import threadpoolctl
        threads = max((p.get("num_threads", 1) for p in threadpoolctl.threadpool_info()), default=1)
    except Exception:
        threads = os.cpu_count()
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    return {"value": sp.mb_rows * sp.m / step_s, "unit": UNIT, "cores": int(min(cores, threads)),
            "kind": "reference",
            "sample": (f"gmfkit {getattr(G, '__version__', '')} (baseline/_ref, kernels.IMPL="
                       f"{GK.IMPL}) fit_asgd on rows 0..{nsub} of {sp.name} ({nsub // sp.mb_rows} "
                       f"blocks of {sp.mb_rows} x {sp.m}, dense fp64, tracked objective every "
                       f"step), median of {len(dts)} callback-to-callback steps"),
            "ms_per_step": step_s * 1e3}


def run_reference(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if ws > 1 and rank != 0:
        return
    from paper_2412_20509_b200 import workloads
    wl = workloads.generate(args.config, n_rows=13 * workloads.SPECS[args.config].mb_rows)
    steps = max(3, min(args.steps, 60))
    warm = min(args.warmup, 3)
    cb = _gmfkit_timing(wl, steps + warm + 1, time_budget=150.0)
    if cb is None:   # reference not installed: the oracle port stands in
        cb = _cpu_baseline(wl, steps + warm, time_budget=150.0)
    sp = wl.spec
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT,
            "n_gpus": 0, "steps": steps, "warmup": warm,
            "ms_per_step": cb["ms_per_step"], "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": _workload_desc(args.config), "n_sample_rows": sp.n,
                       "mb_rows": sp.mb_rows, "m": sp.m, "d": sp.d},
            "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _aux_legs(wl, data, covs, st, fam, dev, reps=3):
    """SURVEY 8f rows on the same workload: the one-pass log-likelihood behind
    information_criteria (k_objfull + NB constant, all n*m entries) and
    init_ols_svd (sparse products, no n x m residual).  CUDA events for the
    kernel, wall clock for the init call (it includes the CSR upload)."""
    import torch
    import paper_2412_20509_b200 as gk
    from paper_2412_20509_b200 import _lib
    from paper_2412_20509_b200.initialization import init_ols_svd
    from paper_2412_20509_b200.select import _state_fit
    sp = wl.spec
    fit = _state_fit(st, data, covs, fam, gk.Log(), wl.offset, sp.dtype, dev.index)
    try:
        res = torch.zeros(2, dtype=torch.float64, device=dev)
        call = lambda: _lib.check(fit.lib.gmf_loglik_full(fit.h, _lib.ptr(res), fit.stream()),
                                  "gmf_loglik_full")
        call()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(torch.cuda.current_stream(dev))
        for _ in range(reps):
            call()
        e1.record(torch.cuda.current_stream(dev))
        torch.cuda.synchronize(dev)
        ll_ms = e0.elapsed_time(e1) / reps
    finally:
        fit.close()
    init_ols_svd(data, covs, fam, gk.Log(), sp.d, seed=0)
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    init_ols_svd(data, covs, fam, gk.Log(), sp.d, seed=0)
    torch.cuda.synchronize(dev)
    init_s = time.perf_counter() - t0
    return {"loglik_full": {"kernel": "k_objfull (deviance + NB dispersion constant, all n*m "
                                      "entries; information_criteria)",
                            "ms": ll_ms, "entries_per_s": sp.n * sp.m / (ll_ms * 1e-3)},
            "init_ols_svd": {"s": init_s, "path": "gmf_csr_spmm / gmf_init_moments + cuSOLVER "
                                                  "sketches; host CSR upload included"}}


def _fp64_c2_leg(dev, steps=2000, warmup=50):
    """The reference's own precision beside the fp32 headline: BASELINE config
    2 (26,472 x 500 NB, k = 15, offset, dense, mb 2,000 rows) in fp64 on the
    CUDA-core K1, one persistent launch of `steps` aSGD steps, CUDA events."""
    import torch
    import paper_2412_20509_b200 as gk
    from paper_2412_20509_b200 import workloads
    from paper_2412_20509_b200.engine import DeviceFit, Schedule
    wl = workloads.generate("c2", device=str(dev))
    sp = wl.spec
    data = gk.ResponseMatrix(wl.y_dense.astype(float))
    covs = gk.CovariateSet(x=wl.x, z=wl.z if sp.q else None, m=sp.m)
    st = gk.FactorizationState(**wl.init_state())
    cfg = gk.SgdConfig(max_epochs=warmup + steps + 8, mb_rows=sp.mb_rows, mb_cols=sp.m,
                       tol=1e-30, seed=0)
    sched = Schedule(sp.n, sp.m, cfg)
    fit = DeviceFit(data, covs, gk.NegBinomial(st.nb_shape), gk.Log(), gk.PenaltyConfig(), cfg, st,
                    schedule=sched, offset=wl.offset, dtype="f64", device=dev.index,
                    est_alpha=True)
    try:
        fit.reset()
        fit.run(warmup)
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fit.run(steps)
        e1.record()
        torch.cuda.synchronize(dev)
        ms = e0.elapsed_time(e1)
        status = fit.status()
        assert status.t == warmup + steps and not status.stopped
        sizes = np.array([b.size for b in sched.row_blocks])
        entries = float(sizes[sched.block_seq[warmup:warmup + steps]].sum()) * sp.m
    finally:
        fit.close()
    return {"workload": _workload_desc("c2"), "dtype": "f64", "k1_impl": fit.k1_impl,
            "steps": steps, "warmup": warmup, "ms_per_step": ms / steps,
            "value": entries / (ms / 1e3), "unit": UNIT}


def _workload_desc(name):
    return {
        "c1": "c1: Poisson GMF 1,000 x 100, k=5, X=Z=1, dense int32, mb 100 rows x all columns, fp64",
        "c2": "c2: NB GMF 26,472 x 500, k=15, 7-group mixture, log-library offset, dense int32, mb 2,000 rows, fp64",
        "c3": "c3: NB GMF 100,000 x 1,000, k=10, X=[1,batch], Z=1, CSR int32 ~90% zeros, mb 5,000 rows, fp32",
        "c4": "c4: NB GMF 1,300,000 x 500, k=10, intercept + log-library offset, CSR ~92% zeros, mb 10,000 rows x all 500 columns, fp32",
    }[name]


def main():
    args = _args()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import paper_2412_20509_b200 as gk
    from paper_2412_20509_b200 import _lib, workloads
    from paper_2412_20509_b200.engine import DeviceFit, Schedule
    from paper_2412_20509_b200.optim import _Exchange

    world, rank, local, group = _dist()
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    wl = workloads.generate(args.config, device=str(dev))
    sp = wl.spec
    if sp.y_format == "csr":
        data = gk.ResponseMatrix(csr=wl.csr, shape=(sp.n, sp.m))
    else:
        data = gk.ResponseMatrix(wl.y_dense.astype(float))
    covs = gk.CovariateSet(x=wl.x, z=wl.z if sp.q else None, m=sp.m)
    st = gk.FactorizationState(**wl.init_state())
    fam = gk.NegBinomial(st.nb_shape) if sp.family == "neg_binomial" else gk.Poisson()
    W, K, E = args.warmup, args.steps, args.e2e_steps
    cfg = gk.SgdConfig(max_epochs=W + K + E + args.phases + 8, mb_rows=sp.mb_rows, mb_cols=sp.m, tol=1e-30,
                       seed=0)
    sched = Schedule(sp.n, sp.m, cfg)
    fit = DeviceFit(data, covs, fam, gk.Log(), gk.PenaltyConfig(), cfg, st, schedule=sched,
                    offset=wl.offset, dtype=sp.dtype, device=local, world=world, rank=rank,
                    est_alpha=sp.family == "neg_binomial", k1_impl=args.k1_impl)
    fit.reset()
    ex = _Exchange(fit, group, "device") if group is not None else None

    state = {"eager_done": False}

    def steps(k):
        # N = 1: one persistent launch.  N > 1: the rank step (objective, K1,
        # record copy, NCCL all-gather, fixed-order apply) replayed as CUDA
        # graphs of 32 steps, as fit_asgd drives it (optim._Exchange.graph);
        # one eager step first warms the communicator, the remainder is eager
        if ex is None:
            fit.run(k)
            return
        if not state["eager_done"] and k > 0:
            n0 = fit.launch_count()
            ex.step()
            state["per_step"] = fit.launch_count() - n0   # kernels of one rank step
            state["eager_done"] = True
            k -= 1
        while k >= 32:
            ex.graph(32)
            k -= 32
        for _ in range(k):
            ex.step()

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            torch.distributed.barrier()

    # ---- warm-up ----
    steps(W)
    barrier()
    # ---- timed region: K steps, inputs resident in HBM ----
    props = torch.cuda.get_device_properties(dev)
    bus = "%08X:%02X:%02X.0" % (getattr(props, "pci_domain_id", 0), getattr(props, "pci_bus_id", 0),
                                getattr(props, "pci_device_id", 0))
    clk = Clocks(bus)
    clk.start()
    time.sleep(0.3)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = fit.launch_count()
    w0 = time.perf_counter()
    e0.record()
    steps(K)
    e1.record()
    barrier()
    timed_launches = fit.launch_count() - launches0
    if ex is not None:   # graph replays launch their captured kernels without the host counter
        timed_launches = state.get("per_step", 0) * K
    w1 = time.perf_counter()
    ms = e0.elapsed_time(e1)
    clocks = clk.stop(w0, w1)
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    status = fit.status()
    assert status.t == W + K and not status.stopped, (status.t, status.stopped)
    import ctypes as C
    geo = (C.c_int64 * 8)()
    _lib.check(fit.lib.gmf_geometry(fit.h, geo), "gmf_geometry")
    geometry = dict(zip(["fit_ctas", "fit_row_splits", "col_tiles", "tile_cols",
                         "step_row_splits", "feature_bucket", "k1_smem_bytes", "max_block_rows"],
                        [int(v) for v in geo]))
    phases = None
    if args.phases and world == 1 and geometry["fit_ctas"] > 0:   # persistent k_fit only
        import ctypes as C
        nprof = int(fit.lib.gmf_profile_len(fit.h))
        buf = (C.c_double * nprof)()
        _lib.check(fit.lib.gmf_profile(fit.h, 1, None, fit.stream()), "gmf_profile")
        fit.run(args.phases)
        _lib.check(fit.lib.gmf_profile(fit.h, 0, buf, fit.stream()), "gmf_profile")
        nst = max(buf[5], 1.0)
        names = ["objective_partials", "k1_tiles", "barrier1", "phase2_update", "barrier2"]
        phases = {nm: buf[i] / nst / 1e3 for i, nm in enumerate(names)}
        for i, nm in ((6, "p2_totals"), (7, "p2_rows"), (8, "p2_cols"), (9, "p2_rest"), (10, "p2_norms")):
            phases[nm + "_cum"] = buf[i] / nst / 1e3
        per = np.array(buf[16:16 + 32 * geometry["fit_ctas"]]).reshape(-1, 32)
        tl = np.array(buf[16 + 32 * geometry["fit_ctas"]:]).reshape(16, 32)
        if tl.any():   # K1 v2 event timeline of CTA 0, last step (us from its first event)
            t0 = tl[tl > 0].min()
            evn = ["ld_issue_start", "ld_issue_end", "ld_scatter_start", "-", "mma_gemm1", "mma_gemm23",
                   "ew_eta_ready", "ew_computed", "ew_p_free", "ew_p_full", "-", "unit_start",
                   "ew_drained", "-", "-", "mma_gemm1_committed"]
            phases["k1_timeline_cta0_us"] = {
                evn[e]: [round((v - t0) / 1e3, 2) if v > 0 else None for v in tl[e][:8]]
                for e in range(16) if tl[e].any()}
        st_ = per[:, :5]
        oc = per[:, 5:7] / nst    # objective sub-phase clocks per step
        phases["objective_subphases_us(mean over CTAs)"] = {
            "loop": float(oc[:, 0].mean() / 1965.0), "block_reduce": float(oc[:, 1].mean() / 1965.0)}
        phases["p2_totals_us(mean over CTAs, SM clocks)"] = float((per[:, 7] / nst).mean() / 1965.0)
        kc = per[:, 8:16] / nst   # K1 sub-phase clocks per step (tensor path)
        if kc.any():
            names_k = ["col_operands", "staging_wait", "y_a1_gemm1", "d2_readout_b3", "barrier",
                       "next_stage_rowside", "elementwise_gemm23", "drain_d3"]
            if int(fit.lib.gmf_k1_version(fit.h)) == 2:   # warp-specialized K1 (gmf_tc2.cuh)
                kc = per[:, 8:24] / nst
                names_k = ["ew_unit_prologue", "ew_wait_eta", "-", "ew_wait_y",
                           "ew_elementwise", "ew_wait_p_free", "ew_d2_readout_p_store",
                           "ew_unit_drain", "mma_wait_operands", "mma_wait_eta_free", "mma_issue",
                           "mma_wait_p_full", "ld_staging_issue", "ld_wait_staged",
                           "ld_wait_y_free", "ld_scatter"]
            phases["k1_subphases_us(mean over CTAs)"] = {
                nm: float(kc[:, i].mean() / 1965.0) for i, nm in enumerate(names_k)}
        t0 = st_[:, 0].min()
        rel = (st_ - t0) / 1e3
        phases["last_step_per_cta_us"] = {
            "obj_end(min/mean/max)": [rel[:, 1].min(), rel[:, 1].mean(), rel[:, 1].max()],
            "k1_end(min/mean/max)": [rel[:, 2].min(), rel[:, 2].mean(), rel[:, 2].max()],
            "k1_dur(min/mean/max)": [(rel[:, 2] - rel[:, 1]).min(), (rel[:, 2] - rel[:, 1]).mean(),
                                     (rel[:, 2] - rel[:, 1]).max()],
            "barrier1_release(min/max)": [rel[:, 3].min(), rel[:, 3].max()],
            "phase2_end(min/mean/max)": [rel[:, 4].min(), rel[:, 4].mean(), rel[:, 4].max()],
        }
        phases["unit"] = "us/step (CTA 0 globaltimer)"
        print(json.dumps({"phases": phases}), file=sys.stderr, flush=True)
        K2 = args.phases
    else:
        K2 = 0
    sizes = np.array([b.size for b in sched.row_blocks])
    seq = sched.block_seq
    entries = float(sizes[seq[W:W + K]].sum()) * sp.m
    value = entries / (ms / 1e3)

    # ---- roofline of the dominant kernel ----
    # The timed region is ONE launch of the persistent fit kernel k_fit (every
    # phase of every step), so the roofline is k_fit's: algorithmic bytes of
    # one step (_step_bytes: the drawn block's CSR + row state in and out, all
    # columns' state, the tracked sample) over the device time per step.  The
    # per-step K1 kernel timed alone (gmf_time_grad, per-step path) is kept
    # as a secondary figure.
    e_sz = 8 if sp.dtype == "f64" else 4
    blk = int(seq[W + K - 1])
    rbp = fit.rbp.cpu().numpy()
    if fit.csr_ptr is not None:
        cptr = fit.csr_ptr.cpu().numpy()
        nnz_blk = int(cptr[rbp[blk + 1]] - cptr[rbp[blk]])
    else:
        nnz_blk = 0
    nI_loc = int(rbp[blk + 1] - rbp[blk])
    import ctypes as C
    avg = C.c_double()
    _lib.check(fit.lib.gmf_time_grad(fit.h, blk, 200, C.byref(avg), fit.stream()), "gmf_time_grad")
    k1_ms = avg.value
    nnzb = 4 if fit.y_format == "packed" else 8
    k1_bytes = _k1_bytes(workloads.WorkloadSpec(**{**sp.__dict__}), nI_loc, nnz_blk, e_sz, nnzb)
    peak, peak_src = _peak_hbm()
    ms_step = ms / K
    step_bytes = _step_bytes(sp, nI_loc, nnz_blk, e_sz, nnzb)
    achieved = step_bytes / (ms_step / 1e3) / 1e9
    traffic = None
    tpath = os.path.join(REPO, "profiles", f"kfit_traffic_{args.config}.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get("dram_bytes_per_step")
        except Exception:
            traffic = None
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic,
                "kernel": "k_fit (persistent fit kernel: tracked objective, K1 fused gradient, "
                          "EMA/adaptive updates, two grid barriers per step)",
                "algorithmic_bytes_per_step": step_bytes, "peak_source": peak_src,
                "k1_impl": fit.k1_impl,
                "k1_standalone": {"kernel": "k_grad (K1 alone, per-step path)", "ms": k1_ms,
                                  "bytes": k1_bytes,
                                  "GB_s": k1_bytes / (k1_ms / 1e3) / 1e9}}

    # ---- e2e: stream each step's block from pinned host memory ----
    # ONE persistent launch (C-ABI gmf_run_stream) runs the E steps; step t
    # waits, before its gradient, for its drawn row block (CSR slice, or
    # dense rows) to be copied host -> device on a copy stream, which then
    # bumps the ready counter (gmf_stream_signal).  Each step's status word is
    # written by the kernel into pinned host memory (device -> host per step).
    e2e = None
    if E > 0 and world == 1:
        packed = fit.csr_ptr is not None and fit.csr_val is None
        if fit.csr_ptr is not None:
            h_col = fit.csr_col.cpu().pin_memory()
            h_val = None if packed else fit.csr_val.cpu().pin_memory()
            h_ptr = fit.csr_ptr.cpu().pin_memory()
            cptr = h_ptr.numpy()
        else:
            h_y = fit.y_dense.cpu().pin_memory()
        sbytes = int(fit.lib.gmf_status_raw_bytes())
        status_h = torch.zeros(E * sbytes, dtype=torch.uint8).pin_memory()
        cs = torch.cuda.Stream(dev)
        main = torch.cuda.current_stream(dev)
        t_first = W + K + K2
        h2d = 0
        barrier()
        launches0 = fit.launch_count()
        e0.record(main)
        cs.wait_event(e0)
        fit.run_stream(E, status_h)
        with torch.cuda.stream(cs):
            for k in range(E):
                b = int(seq[t_first + k])
                r0, r1 = int(rbp[b]), int(rbp[b + 1])
                if fit.csr_ptr is not None:
                    a0, a1 = int(cptr[r0]), int(cptr[r1])
                    fit.csr_col[a0:a1].copy_(h_col[a0:a1], non_blocking=True)
                    if not packed:
                        fit.csr_val[a0:a1].copy_(h_val[a0:a1], non_blocking=True)
                    fit.csr_ptr[r0:r1 + 1].copy_(h_ptr[r0:r1 + 1], non_blocking=True)
                    h2d += (a1 - a0) * (4 if packed else 8) + (r1 - r0 + 1) * 8
                else:
                    fit.y_dense[r0:r1].copy_(h_y[r0:r1], non_blocking=True)
                    h2d += (r1 - r0) * sp.m * 4
                fit.stream_signal(t_first + k + 1, cs)
                h2d += 8
        e1.record(main)
        barrier()
        e_launches = fit.launch_count() - launches0
        e_ms = e0.elapsed_time(e1)
        st_e = _lib.GmfStatus()
        import ctypes as C
        fit.lib.gmf_status_decode(C.c_void_p(status_h.data_ptr() + (E - 1) * sbytes), C.byref(st_e))
        try:
            streamed_ok = fit.status().t == W + K + K2 + E and st_e.t == W + K + K2 + E
        except _lib.GmfError:   # a profiler serialising the copy stream: blocks never arrived
            streamed_ok = False
        if not streamed_ok:
            print(json.dumps({"warning": "streaming e2e aborted (copy stream not concurrent, e.g. "
                              "under a profiler); e2e not reported"}), file=sys.stderr)
            E = 0
    if E > 0 and world == 1:
        e_entries = float(sizes[seq[t_first:t_first + E]].sum()) * sp.m
        e2e = {"value": e_entries / (e_ms / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d // E), "d2h_bytes_per_step": sbytes,
               "steps": E, "ms_per_step": e_ms / E, "gpu_launches": int(e_launches),
               "path": "C-ABI gmf_run_stream: one persistent launch; step t's row block copied from "
                       "pinned host memory on a copy stream, then gmf_stream_signal(t+1); the kernel "
                       "waits for the signal before step t's gradient and writes each step's status "
                       "word to pinned host memory"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = _cpu_baseline(wl, max(4, args.cpu_steps))
        cpu = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")}
    fit.close()
    aux = None
    if rank == 0 and world == 1 and not args.no_aux:
        try:
            aux = _aux_legs(wl, data, covs, st, fam, dev)
        except Exception as err:   # reported, never fatal to the headline line
            aux = {"error": f"{type(err).__name__}: {err}"}
    fp64_c2 = None
    if rank == 0 and world == 1 and not args.no_aux and args.config == "c4":
        try:
            fp64_c2 = _fp64_c2_leg(dev)
        except Exception as err:
            fp64_c2 = {"error": f"{type(err).__name__}: {err}"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": W, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": sp.dtype,
            "data": "synthetic (seeded Gamma-Poisson NB counts with BASELINE shapes)",
            "config": {"workload": _workload_desc(args.config), "n": sp.n, "m": sp.m,
                       "d": sp.d, "p": sp.p, "q": sp.q, "mb_rows": sp.mb_rows,
                       "nnz": wl.meta.get("nnz"), "zero_frac": round(wl.meta.get("zero_frac", 0), 4),
                       "y_format": sp.y_format,
                       "l2": "inputs (CSR %.0f MB + factors) exceed the 126 MB L2; each step draws "
                             "a random row block" % (wl.meta.get("nnz", 0) * (4 if fit.y_format == "packed" else 8) / 1e6),
                       "parallelism": f"rows of each block split x{world}" if world > 1 else "1 GPU",
                       "geometry": geometry, "k1_impl": fit.k1_impl, "y_storage": fit.y_format},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(timed_launches), "clocks": clocks, "aux": aux,
            "fp64_c2": fp64_c2,
        }
        print(json.dumps(line), flush=True)
    if group is not None:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
