"""Device session of one aSGD fit: host schedule replay, block-major upload,
the C-ABI handle, and state read-back.

Layout in HBM (one process per GPU; rows of every block optionally split
across ranks):
  * rows are stored BLOCK-MAJOR: the fixed random row partition of
    optim.py:406 is concatenated, so row block r is the contiguous range
    [row_block_ptr[r], row_block_ptr[r+1]) and every K1 CTA streams
    contiguous rows;
  * Y is dense int32 (n x m) or CSR int32 (row_ptr int64, col int32, val int32);
  * theta_row = [Gamma | U] (n x (q+d)), theta_col = [B | V] (m x (p+d)) in the
    compute dtype, plus their EMA buffers and divergence snapshots;
  * the schedule (row-block draws, column blocks, tracked-objective sample,
    learning-rate tables) is replayed on the host from the shared seed, so
    device and reference trajectories are directly comparable.
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _lib
from .exceptions import ConfigError
from .model import FactorizationState


# ---------------------------------------------------------------------------
# host schedule replay (optim.py:253-271, 404-408, 423)
# ---------------------------------------------------------------------------

def partition(rng, size, block):
    """Sorted near-equal chunks of a random permutation (optim.py:253-257)."""
    perm = rng.permutation(size)
    k = int(math.ceil(size / block))
    return [np.sort(c) for c in np.array_split(perm, k)]


def eval_entries(n, m, cap, rng, mask=None):
    """Fixed objective sample (optim.py:260-271).  For a fully observed matrix
    the row-major enumeration of np.nonzero is implicit, so the picks map to
    (pick // m, pick % m) with identical RNG consumption."""
    if mask is None:
        total = n * m
        if total <= cap:
            lin = np.arange(total, dtype=np.int64)
            return lin // m, lin % m, 1.0
        pick = np.sort(rng.choice(total, size=cap, replace=False))
        return pick // m, pick % m, total / cap
    rows, cols = np.nonzero(mask)
    total = rows.size
    if total <= cap:
        return rows, cols, 1.0
    pick = np.sort(rng.choice(total, size=cap, replace=False))
    return rows[pick], cols[pick], total / cap


class Schedule:
    """Everything fit_asgd draws from ``default_rng(cfg.seed)``, in order."""

    def __init__(self, n, m, cfg, mask=None, row_blocks=None, col_blocks=None, n_steps=None):
        rng = np.random.default_rng(cfg.seed)
        if row_blocks is None:
            self.row_blocks = partition(rng, n, min(cfg.mb_rows, n))
            self.col_blocks = partition(rng, m, min(cfg.mb_cols, m))
            self.eval_rows, self.eval_cols, self.eval_scale = eval_entries(
                n, m, cfg.max_eval_entries, rng, mask)
        else:   # explicit blocks (standalone minibatch / objective calls)
            self.row_blocks = [np.asarray(b, dtype=np.int64) for b in row_blocks]
            self.col_blocks = [np.asarray(b, dtype=np.int64) for b in col_blocks]
            self.eval_rows = np.zeros(0, dtype=np.int64)
            self.eval_cols = np.zeros(0, dtype=np.int64)
            self.eval_scale = 1.0
        R = len(self.row_blocks)
        self.steps_per_epoch = len(self.col_blocks)
        steps = cfg.max_epochs * self.steps_per_epoch if n_steps is None else n_steps
        if row_blocks is None:
            self.block_seq = np.fromiter((rng.integers(R) for _ in range(steps)),
                                         dtype=np.int32, count=steps)
        else:
            self.block_seq = np.zeros(steps, dtype=np.int32)
        self.max_steps = steps


def shard_rows(schedule: Schedule, world: int, rank: int):
    """Rows of every block split across ranks: rank k owns the k-th contiguous
    slice of each (sorted) block, so all ranks work on the same drawn block
    each step.  Returns (local original-row order, local block
    pointer, per-block s_col = n / |I_r|)."""
    parts, sizes, scales = [], [], []
    n = sum(b.size for b in schedule.row_blocks)
    for blk in schedule.row_blocks:
        chunk = -(-blk.size // world)
        sl = blk[rank * chunk:(rank + 1) * chunk]
        parts.append(sl)
        sizes.append(sl.size)
        scales.append(n / blk.size)
    order = np.concatenate(parts) if parts else np.zeros(0, dtype=np.int64)
    ptr = np.zeros(len(sizes) + 1, dtype=np.int64)
    np.cumsum(sizes, out=ptr[1:])
    return order.astype(np.int64), ptr, np.asarray(scales, dtype=np.float64)


def permute_csr(indptr, indices, data, order):
    """Rows of a CSR matrix in ``order`` (vectorized gather)."""
    starts = indptr[order]
    lens = indptr[order + 1] - starts
    new_ptr = np.zeros(order.size + 1, dtype=np.int64)
    np.cumsum(lens, out=new_ptr[1:])
    nnz = int(new_ptr[-1])
    if nnz == 0:
        return new_ptr, np.zeros(0, np.int32), np.zeros(0, np.int32)
    src = np.repeat(starts - new_ptr[:-1], lens) + np.arange(nnz, dtype=np.int64)
    return new_ptr, np.asarray(indices)[src].astype(np.int32), np.asarray(data)[src]


def _mean_of_eta(kind, eta):
    """g^{-1}(eta) without domain checks (kernels/_ref.py:21-32), for seeding
    the working response at unobserved entries."""
    with np.errstate(all="ignore"):
        if kind == "identity":
            return np.asarray(eta, dtype=float)
        if kind == "log":
            return np.exp(eta)
        if kind == "logit":
            return 1.0 / (1.0 + np.exp(-eta))
        if kind == "inverse":
            return 1.0 / eta
        return 1.0 / np.sqrt(eta)


def _counts_int32(vals, what):
    v = np.asarray(vals)
    if v.dtype.kind in "iu":
        if v.size and (v.min() < 0 or v.max() > 2**31 - 1):
            raise ConfigError(f"{what}: counts must lie in [0, 2^31)")
        return v.astype(np.int32)
    if v.size and (np.any(v < 0) or np.any(v != np.round(v)) or np.any(v > 2**31 - 1)):
        raise _lib.UnsupportedError(
            f"{what}: the device path stores responses as int32 counts; "
            "non-integer or negative values are not supported")
    return v.astype(np.int32)


# ---------------------------------------------------------------------------
# packed CSR (GMF_Y_CSR_PACK32): one uint32 per nonzero, (count << 16) | column
# ---------------------------------------------------------------------------

def packable(m, counts):
    """Packed CSR holds columns < 65536 and counts <= 65535."""
    counts = np.asarray(counts)
    return m <= 65536 and (counts.size == 0 or (int(counts.min()) >= 0 and int(counts.max()) <= 65535))


def pack_csr(cols, counts):
    """int32 view of the packed words (the C ABI's csr_col for PACK32)."""
    w = (np.asarray(counts).astype(np.uint32) << np.uint32(16)) | np.asarray(cols).astype(np.uint32)
    return w.view(np.int32)


def unpack_csr(words):
    """(columns, counts) of packed words (test/debug helper)."""
    w = np.asarray(words).view(np.uint32)
    return (w & np.uint32(0xFFFF)).astype(np.int32), (w >> np.uint32(16)).astype(np.int32)


# ---------------------------------------------------------------------------
# the device fit
# ---------------------------------------------------------------------------

class DeviceFit:
    """Uploads one problem in block-major layout and owns its gmf_handle."""

    def __init__(self, data, covs, fam, lnk, penalty, cfg, state: FactorizationState, *,
                 schedule: Schedule, offset=None, dtype="f64", device=None, world=1, rank=0,
                 est_alpha=False, est_phi=False, k1_impl="auto", y_format="auto",
                 eval_only=False):
        import torch
        _lib.require_cuda()
        lib = _lib.lib()
        # the fused count kernels cover poisson / neg_binomial with the log
        # link; every other family / link pair, and any fit that estimates phi
        # (optim.py:175-202), runs in general mode: real-valued dense response,
        # family and link chosen at run time on the CUDA-core K1
        general = (est_phi or fam.kind not in ("poisson", "neg_binomial")
                   or lnk.kind != "log") and not eval_only
        holes = not data.fully_observed
        if holes and data.csr is not None:
            raise _lib.UnsupportedError("unobserved entries need a dense response")
        if general:
            if data.csr is not None:
                raise _lib.UnsupportedError(
                    f"{fam.kind}+{lnk.kind}"
                    f"{' with an estimated dispersion' if est_phi else ''} runs in general mode, "
                    "which needs a dense response")
            if k1_impl == "tensor":
                raise _lib.UnsupportedError("general mode runs K1 on the CUDA cores")
            fam.check_y(data.values[data.mask] if holes else data.values)   # DomainError (families.py:239-241)
        if dtype not in ("f32", "f64"):
            raise ConfigError(f"dtype must be 'f32' or 'f64', got {dtype!r}")
        if k1_impl not in _lib.K1_IMPL_CODES:
            raise ConfigError(f"k1_impl must be one of {sorted(_lib.K1_IMPL_CODES)}, got {k1_impl!r}")
        self.torch = torch
        dev_index = torch.cuda.current_device() if device is None else int(
            str(device).split(":")[-1] if isinstance(device, str) else device)
        self.device = torch.device("cuda", dev_index)
        self.tdt = torch.float64 if dtype == "f64" else torch.float32
        self.dtype = dtype
        self.n, self.m = data.shape
        self.p, self.q, self.d = covs.p, covs.q, state.rank
        self.world, self.rank = world, rank
        self.schedule = schedule
        order, rbp, rbscale = shard_rows(schedule, world, rank)
        self.order = order                       # local row k <- original row order[k]
        self.n_local = order.size
        dev, tdt = self.device, self.tdt

        def up(a, dt=None):
            a = np.ascontiguousarray(a)
            t = torch.from_numpy(a)
            return t.to(device=dev, dtype=dt if dt is not None else t.dtype)

        def up_padded(a, dt=None):
            # 16 bytes of readable tail slack (gmf_desc.flags: the tensor-core
            # K1 stages row ranges with TMA bulk copies of 16-byte aligned supersets)
            a = np.ascontiguousarray(a)
            t = torch.from_numpy(a)
            dt = dt if dt is not None else t.dtype
            buf = torch.zeros(t.numel() + 16, device=dev, dtype=dt)
            buf[:t.numel()].copy_(t.reshape(-1).to(dtype=dt))
            return buf[:t.numel()].view(t.shape)

        # ---- response ----
        if data.csr is not None:
            indptr, indices, vals = data.csr
            p2, c2, v2 = permute_csr(indptr, indices, vals, order)
            self.y_dense = None
            self.csr_ptr = up(p2)
            counts = _counts_int32(v2, "response")
            if y_format not in ("auto", "csr32", "packed"):
                raise ConfigError(f"y_format must be 'auto', 'csr32' or 'packed', got {y_format!r}")
            fits = packable(self.m, counts)
            if y_format == "packed" and not fits:
                raise ConfigError("packed CSR needs m <= 65536 and counts <= 65535")
            if y_format != "csr32" and fits:
                self.csr_col = up_padded(pack_csr(c2, counts))
                self.csr_val = None
                y_format_code = _lib.Y_CSR_PACK32
            else:
                self.csr_col = up_padded(c2.astype(np.int32))
                self.csr_val = up_padded(counts)
                y_format_code = _lib.Y_CSR_I32
        elif general:
            self.y_dense = None
            self.csr_ptr = self.csr_col = self.csr_val = None
            y_format_code = _lib.Y_DENSE_I32
        else:
            vals = data.values[order]
            if holes:   # observed counts; the working response below carries the holes
                vals = np.where(data.mask[order], vals, 0.0)
            self.y_dense = up(_counts_int32(vals, "response"))
            self.csr_ptr = self.csr_col = self.csr_val = None
            y_format_code = _lib.Y_DENSE_I32
        self.y_work = None
        self.general = general
        if general and not holes:   # the real-valued response itself (GMF_DESC_REAL_RESPONSE)
            self.y_work = up(data.values[order], self.tdt)
        elif holes:
            # working response (optim.py:368-374): observed counts, and at every
            # unobserved entry minus its mean at the initial state,
            # -g^{-1}(eta0) -- the sign marks the hole, the kernel refills it
            mo = data.mask[order]
            eta0 = state.u[order] @ state.v.T
            if covs.p:
                eta0 = eta0 + covs.x[order] @ state.b.T
            if covs.q:
                eta0 = eta0 + state.gamma[order] @ covs.z.T
            if offset is not None:
                eta0 = eta0 + np.asarray(offset, dtype=float)[order][:, None]
            mean0 = _mean_of_eta(lnk.kind, eta0)
            if general:
                # general mode: the hole marker is the last mantissa bit (set on
                # the imputed mean, cleared -- at most one ulp -- on the
                # observed values), since real-valued responses take the sign
                ndt, idt = (np.float64, np.int64) if dtype == "f64" else (np.float32, np.int32)
                yw = np.where(mo, data.values[order], mean0).astype(ndt)
                bits = yw.view(idt)
                bits[:] = np.where(mo, bits & ~idt(1), bits | idt(1))
            else:
                with np.errstate(all="ignore"):
                    yw = np.where(mo, data.values[order], -mean0)
            self.y_work = up(yw, self.tdt)
        self.weights = None
        if data.weights is not None:
            if data.csr is not None:
                raise _lib.UnsupportedError("prior weights need a dense response")
            self.weights = up(data.weights[order], tdt)
        # ---- designs, offset, parameters ----
        self.x = up_padded(covs.x[order], tdt)
        self.z = up(covs.z, tdt)
        self.offset = None if offset is None else up_padded(np.asarray(offset, dtype=float)[order], tdt)
        self.theta_row = up_padded(np.hstack([state.gamma, state.u])[order], tdt)
        self.theta_col = up(np.hstack([state.b, state.v]), tdt)
        Kr, Kc = self.q + self.d, self.p + self.d
        z = lambda r, c: torch.zeros((r, c), device=dev, dtype=tdt)
        self.gbar_row, self.hbar_row = z(self.n_local, Kr), z(self.n_local, Kr)
        self.gbar_col, self.hbar_col = z(self.m, Kc), z(self.m, Kc)
        self.snap_row, self.snap_col = z(self.n_local, Kr), z(self.m, Kc)
        # ---- schedule ----
        cb = schedule.col_blocks
        col_idx = np.concatenate(cb).astype(np.int32)
        cbp = np.zeros(len(cb) + 1, dtype=np.int64)
        np.cumsum([b.size for b in cb], out=cbp[1:])
        col_pos = np.zeros(self.m, dtype=np.int32)
        col_of = np.zeros(self.m, dtype=np.int32)
        for s, b in enumerate(cb):
            col_pos[b] = np.arange(b.size, dtype=np.int32)
            col_of[b] = s
        self.rbp = up(rbp)
        self.rbscale = up(rbscale)
        self.col_idx = up(col_idx)
        self.cbp = up(cbp)
        self.col_pos = up(col_pos)
        self.col_of = up(col_of)
        self.block_seq = up(schedule.block_seq if schedule.block_seq.size else np.zeros(1, np.int32))
        inv = np.full(self.n, -1, dtype=np.int64)
        inv[order] = np.arange(order.size, dtype=np.int64)
        er = inv[schedule.eval_rows] if schedule.eval_rows.size else np.zeros(0, np.int64)
        keep = er >= 0
        self.eval_row = up(er[keep].astype(np.int64)) if keep.any() else None
        self.eval_col = up(schedule.eval_cols[keep].astype(np.int32)) if keep.any() else None
        n_eval = int(keep.sum())

        self.y_format = {_lib.Y_DENSE_I32: "dense", _lib.Y_CSR_I32: "csr32",
                         _lib.Y_CSR_PACK32: "packed"}[y_format_code]
        self.desc = _lib.GmfDesc(n=self.n_local, m=self.m, p=self.p, q=self.q, d=self.d,
                                 dtype=_lib.F64 if dtype == "f64" else _lib.F32,
                                 family=_lib.FAMILY_CODES[fam.kind], link=_lib.LINK_CODES[lnk.kind],
                                 y_format=y_format_code, has_offset=int(offset is not None),
                                 has_weights=int(self.weights is not None), world_size=world,
                                 rank=rank, device=dev_index,
                                 flags=_lib.DESC_TAIL_PADDED |
                                 (_lib.DESC_REAL_RESPONSE if general else 0) |
                                 (_lib.DESC_REAL_HOLES if general and holes else 0) |
                                 (_lib.DESC_EVAL_ONLY if eval_only else 0))
        dof = self.n * self.m - (self.p * self.m + self.q * self.n + self.d * (self.n + self.m) + 1)
        if est_phi and dof <= 0:
            raise ConfigError("model is over-parameterized: nonpositive residual dof")
        self.cfg = _lib.GmfConfig(
            rate_k0=cfg.rate_k0, rate_k1=cfg.rate_k1, rate_tau=cfg.rate_tau,
            smooth_a1=cfg.smooth_a1, smooth_a2=cfg.smooth_a2, damping=cfg.damping, tol=cfg.tol,
            lam_b=penalty.lam_b, lam_gamma=penalty.lam_gamma, lam_u=penalty.lam_u,
            lam_v=penalty.lam_v, nb_floor=1e-4, nb_ceiling=1e8, phi=float(state.phi),
            eval_scale=float(schedule.eval_scale), max_epochs=cfg.max_epochs,
            est_alpha=int(bool(est_alpha)), snapshot_stride=4,
            k1_impl=_lib.K1_IMPL_CODES[k1_impl], nafill_every=int(cfg.nafill_every),
            est_phi=int(bool(est_phi)), inv_resid_dof=(1.0 / dof if dof > 0 else 0.0))
        P = _lib.ptr
        self.bufs = _lib.GmfBuffers(
            y_dense=P(self.y_dense), csr_ptr=P(self.csr_ptr), csr_col=P(self.csr_col),
            csr_val=P(self.csr_val), weights=P(self.weights), x=P(self.x), z=P(self.z),
            offset=P(self.offset), theta_row=P(self.theta_row), theta_col=P(self.theta_col),
            gbar_row=P(self.gbar_row), hbar_row=P(self.hbar_row), gbar_col=P(self.gbar_col),
            hbar_col=P(self.hbar_col), snap_row=P(self.snap_row), snap_col=P(self.snap_col),
            row_block_ptr=P(self.rbp), row_block_scale=P(self.rbscale),
            n_row_blocks=len(schedule.row_blocks), col_idx=P(self.col_idx),
            col_block_ptr=P(self.cbp), col_pos=P(self.col_pos), col_block_of=P(self.col_of),
            n_col_blocks=len(cb), block_seq=P(self.block_seq), max_steps=schedule.max_steps,
            eval_row=P(self.eval_row), eval_col=P(self.eval_col), n_eval=n_eval,
            y_work=P(self.y_work))
        self.phi = float(state.phi)
        self.init_nb_shape = float(state.nb_shape)
        h = C.c_void_p()
        torch.cuda.synchronize(dev)
        _lib.check(lib.gmf_create(C.byref(self.desc), C.byref(self.cfg), C.byref(self.bufs),
                                  C.byref(h)), "gmf_create")
        self.h = h
        self.lib = lib
        self.rec_bytes = int(lib.gmf_record_bytes(h))
        self.k1_impl = _lib.K1_IMPL_NAMES[int(lib.gmf_k1_impl(h))]
        self.k1_version = int(lib.gmf_k1_version(h))   # 0 CUDA cores, 1/2 tensor-core K1 v1/v2

    def ready_ptr(self):
        """Device address of the streaming ready counter (gmf_stream_ready_ptr)."""
        return int(self.lib.gmf_stream_ready_ptr(self.h))

    def run_stream(self, n_steps, host_status=None):
        """One launch of n_steps steps, each waiting for its block's ready flag
        (gmf_run_stream); host_status: pinned uint8 tensor of n_steps status words."""
        hs = C.c_void_p(host_status.data_ptr()) if host_status is not None else None
        _lib.check(self.lib.gmf_run_stream(self.h, int(n_steps), hs, self.stream()), "gmf_run_stream")

    def stream_signal(self, value, stream):
        """Enqueue ready = value on `stream` (a torch.cuda.Stream): step value-1's block is there."""
        _lib.check(self.lib.gmf_stream_signal(self.h, int(value), C.c_void_p(stream.cuda_stream)),
                   "gmf_stream_signal")

    def launch_count(self):
        """Kernels this handle has launched so far (C-ABI gmf_launch_count)."""
        return int(self.lib.gmf_launch_count(self.h))

    # ------------------------------------------------------------------
    def stream(self):
        return C.c_void_p(self.torch.cuda.current_stream(self.device).cuda_stream)

    def reset(self, nb_shape=None):
        nb = self.init_nb_shape if nb_shape is None else float(nb_shape)
        _lib.check(self.lib.gmf_reset(self.h, nb, self.stream()), "gmf_reset")

    def run(self, n_steps):
        _lib.check(self.lib.gmf_run(self.h, int(n_steps), self.stream()), "gmf_run")

    def step_local(self):
        _lib.check(self.lib.gmf_step_local(self.h, self.stream()), "gmf_step_local")

    def step_apply(self, gathered=None):
        g = None if gathered is None else C.c_void_p(gathered.data_ptr())
        _lib.check(self.lib.gmf_step_apply(self.h, g, self.stream()), "gmf_step_apply")

    def record_ptr(self):
        return self.lib.gmf_record_ptr(self.h)

    def status(self):
        st = _lib.GmfStatus()
        _lib.check(self.lib.gmf_status_read(self.h, C.byref(st), self.stream()), "gmf_status_read")
        return st

    def trace(self, n):
        obj = np.zeros(max(n, 1))
        nb = np.zeros(max(n, 1))
        _lib.check(self.lib.gmf_trace_read(
            self.h, obj.ctypes.data_as(C.POINTER(C.c_double)),
            nb.ctypes.data_as(C.POINTER(C.c_double)), n, self.stream()), "gmf_trace_read")
        return obj[:n], nb[:n]

    def phi_trace(self, n):
        phi = np.zeros(max(n, 1))
        _lib.check(self.lib.gmf_trace_phi_read(
            self.h, phi.ctypes.data_as(C.POINTER(C.c_double)), n, self.stream()),
            "gmf_trace_phi_read")
        return phi[:n]

    def minibatch_grad(self, row_block, col_block, nb_shape):
        torch = self.torch
        rb = self.schedule.row_blocks[row_block]
        cb = self.schedule.col_blocks[col_block]
        nI = int(self.rbp[row_block + 1] - self.rbp[row_block]) if self.world > 1 else rb.size
        Kr, Kc = self.q + self.d, self.p + self.d
        z = lambda r, c: torch.zeros((r, c), device=self.device, dtype=self.tdt)
        g_row, h_row, g_col, h_col = z(nI, Kr), z(nI, Kr), z(cb.size, Kc), z(cb.size, Kc)
        nb_sums = torch.zeros(2, device=self.device, dtype=torch.float64)
        P = _lib.ptr
        _lib.check(self.lib.gmf_minibatch_grad(self.h, row_block, col_block, float(nb_shape),
                                               P(g_row), P(h_row), P(g_col), P(h_col),
                                               P(nb_sums), self.stream()), "gmf_minibatch_grad")
        return g_row, h_row, g_col, h_col, nb_sums

    def objective_dev(self):
        out = self.torch.zeros(1, device=self.device, dtype=self.torch.float64)
        _lib.check(self.lib.gmf_objective_full(self.h, _lib.ptr(out), self.stream()),
                   "gmf_objective_full")
        return float(out.item())

    def loglik_full(self):
        """(sum w D over all local entries, NB dispersion constant) in one pass."""
        out = self.torch.zeros(2, device=self.device, dtype=self.torch.float64)
        _lib.check(self.lib.gmf_loglik_full(self.h, _lib.ptr(out), self.stream()),
                   "gmf_loglik_full")
        dev, const = out.cpu().numpy()
        return float(dev), float(const)

    def snapshot_rows(self):
        """Local rows of the divergence snapshot (copy-on-write reconstruction:
        blocks saved during the current snapshot period come from snap_row,
        the others are unchanged since the snapshot point)."""
        R = len(self.schedule.row_blocks)
        ver = (C.c_int64 * R)()
        period = C.c_int64()
        _lib.check(self.lib.gmf_snapshot_blocks(self.h, ver, C.byref(period), self.stream()),
                   "gmf_snapshot_blocks")
        rows = self.theta_row.clone()
        rbp = self.rbp.cpu().numpy()
        for r in range(R):
            if ver[r] == period.value and rbp[r + 1] > rbp[r]:
                rows[rbp[r]:rbp[r + 1]] = self.snap_row[rbp[r]:rbp[r + 1]]
        return rows

    def download_state(self, snapshot=False, phi=None, nb_shape=None) -> FactorizationState:
        """Host FactorizationState in the original row order (single rank)."""
        tr = (self.snapshot_rows() if snapshot else self.theta_row).double().cpu().numpy()
        tc = (self.snap_col if snapshot else self.theta_col).double().cpu().numpy()
        rows = np.empty((self.n, tr.shape[1]))
        rows[self.order] = tr
        return FactorizationState(tc[:, :self.p].copy(), rows[:, :self.q].copy(),
                                  rows[:, self.q:].copy(), tc[:, self.p:].copy(),
                                  self.phi if phi is None else phi,
                                  self.init_nb_shape if nb_shape is None else nb_shape)

    def close(self):
        if getattr(self, "h", None):
            self.lib.gmf_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
