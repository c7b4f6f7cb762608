"""Block-wise adaptive SGD (aSGD) on the B200: the drop-in ``fit_asgd``.

Signature, defaults, return types and error behaviour mirror
gmfkit/optim.py:383-489; the step loop runs as CUDA kernels behind the C ABI
(include/gmf_asgd.h):

    per step t  (one CUDA graph node triple, no host sync):
      K3  tracked objective of the current state at epoch boundaries
          (optim.py:283-290, 477-480)
      K1  fused eta -> mu -> dotD/ddotD -> row/column gradient contractions
          for the drawn block I x J (optim.py:427-448)
      K2  tracker decision (optim.py:301-338), EMA + adaptive update of rows I
          and columns J (optim.py:450-462), NB shape update (optim.py:469-473)

The host replays the reference RNG stream once (partitions, tracked sample,
row-block draws), so device and reference trajectories coincide step for
step.  The host only polls a status word between graph launches.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .engine import DeviceFit, Schedule
from .exceptions import ConfigError, DivergenceError
from .identify import _Dev, project_on_device
from .model import FactorizationState, parameter_count, penalty_value

__all__ = ["SgdConfig", "FitReport", "learning_rate", "smooth_update", "bias_correction",
           "fit_asgd"]


@dataclass
class SgdConfig:
    """Optimizer hyperparameters (optim.py:61-106)."""

    max_epochs: int = 500
    rate_k0: float = 0.01
    rate_k1: float = 0.01
    rate_tau: float = 0.75
    mb_rows: int = 100
    mb_cols: int = 20
    smooth_a1: float = 0.1
    smooth_a2: float = 0.01
    damping: float = 1e-3
    tol: float = 1e-5
    nafill_every: int = 1
    seed: int = 0
    stepsize: float = 0.2
    nsteps: int = 1
    max_eval_entries: int = 100_000

    def __post_init__(self):
        if self.max_epochs < 1:
            raise ConfigError("max_epochs must be at least 1")
        if self.rate_k0 <= 0 or self.rate_k1 < 0:
            raise ConfigError("need rate_k0 > 0 and rate_k1 >= 0")
        if not 0.5 < self.rate_tau <= 1.0:
            raise ConfigError("rate_tau must lie in (1/2, 1]")
        if self.mb_rows < 1 or self.mb_cols < 1:
            raise ConfigError("minibatch sizes must be positive")
        for name in ("smooth_a1", "smooth_a2"):
            a = getattr(self, name)
            if not 0.0 < a <= 1.0:
                raise ConfigError(f"{name} must lie in (0, 1]")
        if self.damping < 0 or self.tol <= 0:
            raise ConfigError("need damping >= 0 and tol > 0")
        if self.nafill_every < 1 or self.nsteps < 1:
            raise ConfigError("nafill_every and nsteps must be >= 1")
        if self.stepsize <= 0:
            raise ConfigError("stepsize must be positive")
        if self.max_eval_entries < 1:
            raise ConfigError("max_eval_entries must be positive")


@dataclass
class FitReport:
    """Convergence and diagnostic output of a fit (optim.py:109-127)."""

    final_objective: float = np.nan
    objective_trace: list = field(default_factory=list)
    epochs_run: int = 0
    converged: bool = False
    elapsed_seconds: float = 0.0
    phi_trace: list = field(default_factory=list)
    nb_shape_trace: list = field(default_factory=list)
    diagnostics: dict = field(default_factory=dict)


def learning_rate(t: int, cfg: SgdConfig) -> float:
    """rho_t = k0 / (1 + k0 k1 t)^tau (optim.py:130-134)."""
    if t < 0:
        raise ConfigError("iteration index must be nonnegative")
    return cfg.rate_k0 / (1.0 + cfg.rate_k0 * cfg.rate_k1 * t) ** cfg.rate_tau


def smooth_update(prev_g, prev_h, hat_g, hat_h, a1: float, a2: float):
    """EMA of gradient and Hessian estimates (optim.py:137-139)."""
    return (1.0 - a1) * prev_g + a1 * hat_g, (1.0 - a2) * prev_h + a2 * hat_h


def bias_correction(t: int, a1: float, a2: float) -> float:
    """(1 - a2^t) / (1 - a1^t); 1 when a1 == a2 (optim.py:142-148)."""
    if t < 1:
        raise ConfigError("bias correction is undefined at t = 0")
    if a1 == a2:
        return 1.0
    return (1.0 - a2 ** t) / (1.0 - a1 ** t)


def _resolve_dispersion(fam, dispersion: str):
    """(estimate_phi, estimate_nb_shape) (optim.py:156-168)."""
    if dispersion == "fixed":
        return False, False
    if dispersion == "estimate":
        return (False, True) if fam.kind == "neg_binomial" else (True, False)
    if dispersion == "auto":
        return (False, True) if fam.kind == "neg_binomial" else (fam.has_free_dispersion, False)
    raise ConfigError(f"dispersion must be auto, fixed or estimate, got {dispersion!r}")


def _dist_info(process_group):
    if process_group is None:
        return 1, 0
    import torch.distributed as dist
    return dist.get_world_size(process_group), dist.get_rank(process_group)


class _Exchange:
    """Per-step all-gather of the rank records (column-side partials, NB sums,
    objective partials).  ``mode='device'`` gathers device tensors (NCCL over
    NVLink); ``mode='host'`` stages through host memory (gloo), which lets
    several ranks share one GPU without any kernel waiting on another."""

    def __init__(self, fit: DeviceFit, group, mode):
        import torch
        self.torch, self.fit, self.group, self.mode = torch, fit, group, mode
        w = fit.world
        nb = fit.rec_bytes
        self.rec = torch.empty(nb, dtype=torch.uint8, device=fit.device)
        self.gathered = torch.empty(w * nb, dtype=torch.uint8, device=fit.device)
        if mode == "host":
            self.h_rec = torch.empty(nb, dtype=torch.uint8)
            self.h_gat = torch.empty(w * nb, dtype=torch.uint8)

    def step(self):
        import torch.distributed as dist
        fit = self.fit
        fit.step_local()
        _lib.check(fit.lib.gmf_record_copy(fit.h, _lib.ptr(self.rec), fit.stream()),
                   "gmf_record_copy")
        if self.mode == "host":
            self.h_rec.copy_(self.rec)
            dist.all_gather_into_tensor(self.h_gat, self.h_rec, group=self.group)
            self.gathered.copy_(self.h_gat)
        else:
            dist.all_gather_into_tensor(self.gathered, self.rec, group=self.group)
        fit.step_apply(self.gathered)

    def graph(self, k):
        """k steps (objective, K1, record copy, NCCL all-gather, fixed-order
        apply) captured as ONE CUDA graph, replayed without a per-step host
        loop; the kernels read the step index from the device control block,
        so replays advance the fit and turn into no-ops once it stopped.
        Device (NCCL) exchange only; built on first use, after one eager step
        has warmed the communicator."""
        torch = self.torch
        g = self.graphs.get(k) if hasattr(self, "graphs") else None
        if g is None:
            if not hasattr(self, "graphs"):
                self.graphs = {}
            side = torch.cuda.Stream(self.fit.device)
            side.wait_stream(torch.cuda.current_stream(self.fit.device))
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(side), torch.cuda.graph(g, stream=side):
                for _ in range(k):
                    self.step()
            torch.cuda.current_stream(self.fit.device).wait_stream(side)
            self.graphs[k] = g
        g.replay()


def _gather_rows(fit: DeviceFit, tensor, group, mode):
    """Global (n x k) host array of a row-sharded device tensor, original order."""
    import torch
    import torch.distributed as dist
    w = fit.world
    loc = tensor.double().cpu()
    sizes = [None] * w
    dist.all_gather_object(sizes, (int(loc.shape[0]), fit.order.tolist()), group=group)
    width = loc.shape[1]
    nmax = max(s[0] for s in sizes)
    pad = torch.zeros((nmax, width), dtype=torch.float64)
    pad[:loc.shape[0]] = loc
    outs = [torch.zeros_like(pad) for _ in range(w)]
    dist.all_gather(outs, pad, group=group)
    full = np.empty((fit.n, width))
    for (cnt, order), o in zip(sizes, outs):
        full[np.asarray(order, dtype=np.int64)] = o[:cnt].numpy()
    return full


def fit_asgd(data, covs, fam, lnk, penalty, cfg: SgdConfig, init_state=None, *, rank=None,
             identify_mode="B1", dispersion="auto", callback=None, offset=None, dtype="f64",
             device=None, process_group=None, exchange="device", k1_impl="auto", y_format="auto"):
    """Block-wise adaptive stochastic quasi-Newton descent on the GPU.

    Drop-in for gmfkit.fit_asgd (optim.py:383-489); returns ``(state,
    FitReport)`` with the state projected onto the identifiability constraints
    (``identify_mode=None`` skips it).  Extensions: ``offset`` (per-row term
    in eta), ``dtype`` ('f64' | 'f32'), ``device``, and ``process_group``
    (rows of every block split across the group's ranks, one GPU each), and
    ``k1_impl`` ('auto' | 'tensor' | 'cuda_cores'): the fused-gradient kernel
    (tensor cores for fp32 when eligible), ``y_format`` ('auto' | 'csr32' |
    'packed') for a sparse response: packed CSR (one uint32 per nonzero) is
    used when m <= 65536 and counts <= 65535.
    """
    started = time.perf_counter()
    if init_state is None:   # optim.py:359-366: the GLM-SVD start
        if rank is None:
            raise ConfigError("pass init_state or rank")
        from .initialization import init_glm_svd
        init_state = init_glm_svd(data, covs, fam, lnk, rank, seed=cfg.seed, device=device)
    init_state.check_shapes(data, covs)
    est_phi, est_alpha = _resolve_dispersion(fam, dispersion)
    if offset is not None and np.asarray(offset).shape != (data.n,):
        raise ConfigError("offset must have one entry per row")
    n, m = data.shape
    world, my_rank = _dist_info(process_group)
    mask = None if data.fully_observed else data.mask
    sched = Schedule(n, m, cfg, mask=mask)
    fit = DeviceFit(data, covs, fam, lnk, penalty, cfg, init_state, schedule=sched,
                    offset=offset, dtype=dtype, device=device, world=world, rank=my_rank,
                    est_alpha=est_alpha, est_phi=est_phi, k1_impl=k1_impl, y_format=y_format)
    try:
        fit.reset()
        _drive(fit, callback, process_group, exchange)
        st = fit.status()
        trace, nb_trace = fit.trace(int(st.trace_len))
        phi_trace = fit.phi_trace(int(st.trace_len))
        if st.diverged_init:
            raise DivergenceError("objective is non-finite at the initial state")

        def host_state(snapshot, nb, phi):
            if world == 1:
                return fit.download_state(snapshot=snapshot, nb_shape=nb, phi=phi)
            got = _gathered_state(fit, process_group, exchange, nb, snapshot)
            got.phi = float(phi)
            return got

        if st.diverged:
            k_snap = max(int(st.snapshot_trace_len) - 1, 0)
            raise DivergenceError("objective became non-finite; carrying the last finite state",
                                  state=host_state(True, float(nb_trace[k_snap]),
                                                   float(phi_trace[k_snap])))
        info = None
        if identify_mode and world == 1:
            dev = _Dev(fit.torch, fit.device, fit.tdt, fit.theta_row, fit.theta_col, fit.x,
                       fit.z, covs.p, covs.q, init_state.rank)
            info = project_on_device(dev, n, m, identify_mode)
            dev_sum = fit.objective_dev()
            final = fit.download_state(nb_shape=st.nb_shape, phi=st.phi)
        else:
            final = host_state(False, st.nb_shape, st.phi)
            if identify_mode:
                from .identify import project_constraints
                final, info = project_constraints(final, covs, identify_mode, return_info=True,
                                                  dtype=dtype, device=fit.device.index)
            dev_sum = None
        if dev_sum is None:
            # the live family: NB shape as fitted (optim.py:293-298, 401)
            live = type(fam)(final.nb_shape) if fam.kind == "neg_binomial" else fam
            final_obj = _full_objective(final, data, covs, live, lnk, penalty, offset, dtype,
                                        fit.device.index)
        else:
            final_obj = dev_sum / (2.0 * final.phi) + penalty_value(final, penalty)
        if world > 1:
            import torch.distributed as dist
            vals = [None] * world
            dist.all_gather_object(vals, final_obj, group=process_group)
            final_obj = float(vals[0])
        report = FitReport(
            final_objective=float(final_obj),
            objective_trace=[float(v) for v in trace],
            epochs_run=int(st.trace_len) - 1,
            converged=bool(st.converged),
            elapsed_seconds=time.perf_counter() - started,
            phi_trace=[float(v) for v in phi_trace],
            nb_shape_trace=[float(v) for v in nb_trace],
            diagnostics={"iterations": int(st.t),
                         "row_blocks": [b.tolist() for b in sched.row_blocks],
                         "col_blocks": [b.tolist() for b in sched.col_blocks],
                         "algorithm": "asgd", "device": str(fit.device), "dtype": dtype,
                         "world_size": world, "identify_info": info})
        return final, report
    finally:
        fit.close()


def _gathered_state(fit: DeviceFit, group, exchange, nb_shape, snapshot=False):
    """Host FactorizationState of a row-sharded fit (collective over the group)."""
    tr = _gather_rows(fit, fit.snapshot_rows() if snapshot else fit.theta_row, group, exchange)
    tc = (fit.snap_col if snapshot else fit.theta_col).double().cpu().numpy()
    p, q = fit.p, fit.q
    return FactorizationState(tc[:, :p].copy(), tr[:, :q].copy(), tr[:, q:].copy(),
                              tc[:, p:].copy(), fit.phi, nb_shape)


# multi-rank driver knobs: per-step records exchanged inside captured CUDA
# graphs of _GRAPH_STEPS steps (device / NCCL exchange); _FORCE_EXCHANGE runs
# the exchange path for a one-rank group too (tests of the multi-rank path on
# a single GPU)
_GRAPH_EXCHANGE = True
_GRAPH_STEPS = 32
_FORCE_EXCHANGE = False


def _drive(fit: DeviceFit, callback, group, exchange):
    """Run steps until the device tracker stops (converged / diverged /
    max_epochs); the host only polls the status word between chunks."""
    total = fit.schedule.max_steps + 1          # + the final tracking pass
    if fit.world > 1 or (_FORCE_EXCHANGE and group is not None):
        ex = _Exchange(fit, group, exchange)
        t = 0
        use_graph = exchange == "device" and callback is None and _GRAPH_EXCHANGE
        while True:
            prev = t
            if use_graph and t > 0 and t + _GRAPH_STEPS <= total:
                ex.graph(_GRAPH_STEPS)   # 32 steps per launch, status polled between
                t += _GRAPH_STEPS
            else:
                ex.step()
                t += 1
            if callback is not None or t % 32 == 0 or t >= total:
                st = fit.status()
                if callback is not None and st.t > prev:
                    # collective: every rank gathers the live state (optim.py:474-475)
                    live = _gathered_state(fit, group, exchange, st.nb_shape)
                    live.phi = float(st.phi)
                    callback(int(st.t) - 1, live)
                if st.stopped:
                    return
        return
    if callback is not None:
        while True:
            st0 = fit.status()
            fit.run(1)
            st = fit.status()
            if st.t > st0.t:
                callback(int(st.t) - 1, fit.download_state(nb_shape=st.nb_shape, phi=st.phi))
            if st.stopped:
                return
    chunk = 16
    while True:
        fit.run(chunk)
        st = fit.status()
        if st.stopped:
            return
        chunk = min(chunk * 2, 1024)


def _full_objective(state, data, covs, fam, lnk, penalty, offset, dtype, device):
    from .engine import Schedule as _S
    sched = _S(state.n, state.m, SgdConfig(max_epochs=1), row_blocks=[np.arange(state.n)],
               col_blocks=[np.arange(state.m)], n_steps=0)
    fit = DeviceFit(data, covs, fam, lnk, penalty, SgdConfig(max_epochs=1), state,
                    schedule=sched, offset=offset, dtype=dtype, device=device)
    try:
        fit.reset(getattr(fam, "nb_shape", state.nb_shape) if fam.kind == "neg_binomial"
                  else 1.0)
        dev = fit.objective_dev()
    finally:
        fit.close()
    return dev / (2.0 * state.phi) + penalty_value(state, penalty)


def penalized_objective(state, data, covs, fam, lnk, penalty, *, offset=None, dtype="f64",
                        device=None):
    """Masked half-deviance + penalty (model.py:268-276), deviance on the GPU."""
    state.check_shapes(data, covs)
    return _full_objective(state, data, covs, fam, lnk, penalty, offset, dtype, device)


# ---------------------------------------------------------------------------
# block helpers of the reference's public API (model.py:229-256,
# optim.py:205-245), evaluated on the GPU
# ---------------------------------------------------------------------------

def _dev_index(device):
    import torch
    _lib.require_cuda()
    return torch.device("cuda", torch.cuda.current_device() if device is None else
                        int(str(device).split(":")[-1]))


def _eta_block_device(state, covs, rows, cols, dev, offset=None):
    """eta for rows x cols as a device fp64 array, U V' first (BLAS order of
    model.py:251-255), then X B', then Gamma Z'."""
    import torch
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=float)).to(dev)
    ri = slice(None) if rows is None else np.asarray(rows)
    ci = slice(None) if cols is None else np.asarray(cols)
    eta = t(state.u[ri]) @ t(state.v[ci]).T
    if covs.p:
        eta = eta + t(covs.x[ri]) @ t(state.b[ci]).T
    if covs.q:
        eta = eta + t(state.gamma[ri]) @ t(covs.z[ci]).T
    if offset is not None:
        eta = eta + t(np.asarray(offset, dtype=float)[ri])[:, None]
    return eta


def linear_predictor(state: FactorizationState, covs, rows=None, cols=None, *, offset=None,
                     device=None) -> np.ndarray:
    """eta block for the requested rows x cols (model.py:229-256), on the GPU."""
    n, m = state.n, state.m
    if rows is not None:
        rows = np.asarray(rows)
        if rows.size and (rows.min() < -n or rows.max() >= n):
            raise IndexError(f"row index out of range for n={n}")
    if cols is not None:
        cols = np.asarray(cols)
        if cols.size and (cols.min() < -m or cols.max() >= m):
            raise IndexError(f"column index out of range for m={m}")
    return _eta_block_device(state, covs, rows, cols, _dev_index(device), offset).cpu().numpy()


def impute_block(state: FactorizationState, data, covs, lnk, mb, *, offset=None,
                 device=None) -> np.ndarray:
    """Working copy of the Y block with unobserved entries set to mu
    (optim.py:232-245); observed entries untouched."""
    import torch
    if lnk.kind != "log":
        raise _lib.UnsupportedError(f"device imputation implements the log link, got {lnk.kind}")
    I, J = np.asarray(mb.row_idx), np.asarray(mb.col_idx)
    ix = np.ix_(I, J)
    block = np.array(data.dense()[ix], copy=True)
    if data.csr is None:
        miss = ~data.mask[ix]
        if miss.any():
            dev = _dev_index(device)
            mu = torch.exp(_eta_block_device(state, covs, I, J, dev, offset)).cpu().numpy()
            block[miss] = mu[miss]
    return block


def _mean_device(lnk, eta):
    """mu = g^{-1}(eta) on the device through the C ABI seam (kernels/_ref.py:21-32)."""
    import torch
    mu = torch.empty_like(eta)
    st = torch.cuda.current_stream(eta.device).cuda_stream
    _lib.check(_lib.lib().gmf_mean_of_eta(_lib.LINK_CODES[lnk.kind], _lib.F64, _lib.ptr(eta),
                                          _lib.ptr(mu), eta.numel(), st), "gmf_mean_of_eta")
    return mu


def _variance_device(fam, mu):
    kind = fam.kind
    if kind == "gaussian":
        return mu * 0 + 1.0
    if kind == "gamma":
        return mu * mu
    if kind == "inverse_gaussian":
        return mu * mu * mu
    if kind == "poisson":
        return mu
    if kind == "bernoulli":
        return mu * (1.0 - mu)
    return mu * (1.0 + mu / float(fam.nb_shape))


def update_dispersion_stochastic(state: FactorizationState, data, covs, fam, mb, rate: float,
                                 lnk=None, y_block=None, mu_block=None, *, offset=None,
                                 device=None) -> float:
    """Smoothed stochastic Pearson update of phi (optim.py:175-202):
    phi_hat = (1/N) (nm / n* m*) sum_B w (y - mu)^2 / nu(mu) with
    N = nm - mp - nq - (n+m)d - 1; the block sums run on the GPU in fp64
    (inside a fit the same sum is fused into K1)."""
    import torch
    n, m = data.shape
    dof = n * m - parameter_count(n, m, covs.p, covs.q, state.rank)
    if dof <= 0:
        raise ConfigError("model is over-parameterized: nonpositive residual dof")
    I, J = np.asarray(mb.row_idx), np.asarray(mb.col_idx)
    ix = np.ix_(I, J)
    dev = _dev_index(device)
    if mu_block is None:
        if lnk is None:
            raise ConfigError("mu_block or lnk needed")
        mu = _mean_device(lnk, _eta_block_device(state, covs, I, J, dev, offset).contiguous())
    else:
        mu = torch.from_numpy(np.asarray(mu_block, dtype=float)).to(dev)
    if y_block is None:
        vals = data.dense()[ix]
        y_np = vals if data.csr is not None else np.where(data.mask[ix], vals, np.nan)
        y = torch.from_numpy(np.asarray(y_np, dtype=float)).to(dev)
        y = torch.where(torch.isnan(y), mu, y)
    else:
        y = torch.from_numpy(np.asarray(y_block, dtype=float)).to(dev)
    w = (torch.ones_like(mu) if data.weights is None else
         torch.from_numpy(np.asarray(data.weights[ix], dtype=float)).to(dev))
    s = float((w * (y - mu) ** 2 / _variance_device(fam, mu)).sum().item())
    return (1.0 - rate) * state.phi + rate * (s * (n * m) / (I.size * J.size) / dof)


def update_nb_shape_stochastic(state: FactorizationState, data, mb, rate: float,
                               floor: float = 1e-4, covs=None, lnk=None, y_block=None,
                               mu_block=None, ceiling: float = 1e8, *, offset=None,
                               device=None) -> float:
    """Smoothed stochastic moment update of the NB shape (optim.py:205-229):
    alpha_hat = sum w mu^2 / sum w ((y - mu)^2 - mu) on the block (ceiling when
    the denominator is not positive), clipped to [floor, ceiling]; the sums
    run on the GPU in fp64."""
    import torch
    I, J = np.asarray(mb.row_idx), np.asarray(mb.col_idx)
    ix = np.ix_(I, J)
    dev = _dev_index(device)
    if mu_block is None:
        if lnk is None or covs is None:
            raise ConfigError("mu_block or (covs, lnk) needed")
        mu = torch.exp(_eta_block_device(state, covs, I, J, dev, offset))
    else:
        mu = torch.from_numpy(np.asarray(mu_block, dtype=float)).to(dev)
    if y_block is None:
        vals = data.dense()[ix]
        y_np = vals if data.csr is not None else np.where(data.mask[ix], vals, np.nan)
        y = torch.from_numpy(np.asarray(y_np, dtype=float)).to(dev)
        y = torch.where(torch.isnan(y), mu, y)
    else:
        y = torch.from_numpy(np.asarray(y_block, dtype=float)).to(dev)
    w = (torch.ones_like(mu) if data.weights is None else
         torch.from_numpy(np.asarray(data.weights[ix], dtype=float)).to(dev))
    num = float((w * mu ** 2).sum().item())
    den = float((w * ((y - mu) ** 2 - mu)).sum().item())
    ah = num / den if den > 0 else ceiling
    ah = min(max(floor, ah), ceiling)
    return (1.0 - rate) * state.nb_shape + rate * ah
