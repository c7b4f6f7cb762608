"""ctypes binding of the C ABI in include/gmf_asgd.h (libgmf_asgd.so).

The library is the product: there is no fallback.  ``lib()`` raises
``LibraryMissingError`` when the in-tree shared library is absent, and every
device entry point raises when CUDA is unavailable.
"""
from __future__ import annotations

import ctypes as C
import os

from .exceptions import ConfigError, DomainError, GmfError

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GMF_LIB_PATH") or os.path.join(PKG, "libgmf_asgd.so")   # override: experiments

GMF_OK = 0
GMF_ERR_CONFIG = -1
GMF_ERR_DOMAIN = -2
GMF_ERR_CUDA = -3
GMF_ERR_UNSUPPORTED = -4
GMF_ERR_STATE = -5

F32, F64 = 0, 1
Y_DENSE_I32, Y_CSR_I32, Y_CSR_PACK32 = 0, 1, 2
K1_IMPL_CODES = {"auto": 0, "cuda_cores": 1, "tensor": 2}
K1_IMPL_NAMES = {v: k for k, v in K1_IMPL_CODES.items()}
FAMILY_CODES = {"gaussian": 0, "gamma": 1, "inverse_gaussian": 2, "poisson": 3,
                "bernoulli": 4, "neg_binomial": 5}
LINK_CODES = {"identity": 0, "log": 1, "logit": 2, "inverse": 3, "inverse_squared": 4}


class LibraryMissingError(ImportError):
    pass


class CudaError(GmfError, RuntimeError):
    pass


class UnsupportedError(GmfError, NotImplementedError):
    pass


class GmfDesc(C.Structure):
    _fields_ = [("n", C.c_int64), ("m", C.c_int64), ("p", C.c_int32), ("q", C.c_int32),
                ("d", C.c_int32), ("dtype", C.c_int32), ("family", C.c_int32),
                ("link", C.c_int32), ("y_format", C.c_int32), ("has_offset", C.c_int32),
                ("has_weights", C.c_int32), ("world_size", C.c_int32), ("rank", C.c_int32),
                ("device", C.c_int32), ("flags", C.c_int32)]


# gmf_desc.flags bit: row and CSR buffers readable 16 bytes past their end
DESC_TAIL_PADDED = 1
# general mode: real-valued response in y_work, family / link at run time
DESC_REAL_RESPONSE = 2
# evaluation-only handle (gmf_entries_eval under any family / link)
DESC_EVAL_ONLY = 4
# general mode with unobserved entries marked by sign (nonnegative responses)
DESC_REAL_HOLES = 8


class GmfConfig(C.Structure):
    _fields_ = [("rate_k0", C.c_double), ("rate_k1", C.c_double), ("rate_tau", C.c_double),
                ("smooth_a1", C.c_double), ("smooth_a2", C.c_double), ("damping", C.c_double),
                ("tol", C.c_double), ("lam_b", C.c_double), ("lam_gamma", C.c_double),
                ("lam_u", C.c_double), ("lam_v", C.c_double), ("nb_floor", C.c_double),
                ("nb_ceiling", C.c_double), ("phi", C.c_double), ("eval_scale", C.c_double),
                ("max_epochs", C.c_int64), ("est_alpha", C.c_int32),
                ("snapshot_stride", C.c_int32), ("k1_impl", C.c_int32), ("nafill_every", C.c_int32),
                ("est_phi", C.c_int32), ("reserved0", C.c_int32), ("inv_resid_dof", C.c_double)]


_P = C.c_void_p


class GmfBuffers(C.Structure):
    _fields_ = [("y_dense", _P), ("csr_ptr", _P), ("csr_col", _P), ("csr_val", _P),
                ("weights", _P), ("x", _P), ("z", _P), ("offset", _P),
                ("theta_row", _P), ("theta_col", _P), ("gbar_row", _P), ("hbar_row", _P),
                ("gbar_col", _P), ("hbar_col", _P), ("snap_row", _P), ("snap_col", _P),
                ("row_block_ptr", _P), ("row_block_scale", _P), ("n_row_blocks", C.c_int64),
                ("col_idx", _P), ("col_block_ptr", _P), ("col_pos", _P), ("col_block_of", _P),
                ("n_col_blocks", C.c_int64), ("block_seq", _P), ("max_steps", C.c_int64),
                ("eval_row", _P), ("eval_col", _P), ("n_eval", C.c_int64), ("y_work", _P)]


class GmfStatus(C.Structure):
    _fields_ = [("t", C.c_int64), ("trace_len", C.c_int64), ("snapshot_trace_len", C.c_int64),
                ("nb_shape", C.c_double), ("phi", C.c_double), ("last_objective", C.c_double),
                ("converged", C.c_int32), ("diverged", C.c_int32), ("diverged_init", C.c_int32),
                ("stopped", C.c_int32)]


# every symbol include/gmf_asgd.h declares: (name, restype, argtypes)
_i64, _i32, _d, _pd = C.c_int64, C.c_int32, C.c_double, C.POINTER(C.c_double)
SIGNATURES = {
    "gmf_mean_of_eta": (C.c_int, [C.c_int, C.c_int, _P, _P, _i64, _P]),
    "gmf_derivs_from_mu": (C.c_int, [C.c_int, C.c_int, C.c_int, _P, _P, _P, _i64, _d, _d, _P, _P, _P]),
    "gmf_reduce_work_bytes": (_i64, [_i64]),
    "gmf_deviance_from_mu": (C.c_int, [C.c_int, C.c_int, _P, _P, _P, _i64, _d, _P, _P, _P]),
    "gmf_create": (C.c_int, [C.POINTER(GmfDesc), C.POINTER(GmfConfig), C.POINTER(GmfBuffers),
                             C.POINTER(C.c_void_p)]),
    "gmf_destroy": (C.c_int, [_P]),
    "gmf_reset": (C.c_int, [_P, _d, _P]),
    "gmf_minibatch_grad": (C.c_int, [_P, _i64, _i64, _d, _P, _P, _P, _P, _P, _P]),
    "gmf_step_local": (C.c_int, [_P, _P]),
    "gmf_step_apply": (C.c_int, [_P, _P, _P]),
    "gmf_record_ptr": (_P, [_P]),
    "gmf_record_bytes": (_i64, [_P]),
    "gmf_record_copy": (C.c_int, [_P, _P, _P]),
    "gmf_run": (C.c_int, [_P, _i64, _P]),
    "gmf_status_read": (C.c_int, [_P, C.POINTER(GmfStatus), _P]),
    "gmf_trace_read": (C.c_int, [_P, _pd, _pd, _i64, _P]),
    "gmf_trace_phi_read": (C.c_int, [_P, _pd, _i64, _P]),
    "gmf_status_raw_bytes": (_i64, []),
    "gmf_snapshot_blocks": (C.c_int, [_P, C.POINTER(C.c_int64), C.POINTER(C.c_int64), _P]),
    "gmf_status_copy_async": (C.c_int, [_P, _P, _P]),
    "gmf_status_decode": (C.c_int, [_P, C.POINTER(GmfStatus)]),
    "gmf_time_grad": (C.c_int, [_P, _i64, _i32, _pd, _P]),
    "gmf_profile": (C.c_int, [_P, C.c_int, _pd, _P]),
    "gmf_profile_len": (_i64, [_P]),
    "gmf_geometry": (C.c_int, [_P, C.POINTER(C.c_int64)]),
    "gmf_k1_impl": (C.c_int, [_P]),
    "gmf_k1_version": (C.c_int, [_P]),
    "gmf_stream_ready_ptr": (_P, [_P]),
    "gmf_run_stream": (C.c_int, [_P, _i64, _P, _P]),
    "gmf_stream_signal": (C.c_int, [_P, _i64, _P]),
    "gmf_launch_count": (_i64, [_P]),
    "gmf_objective_full": (C.c_int, [_P, _P, _P]),
    "gmf_loglik_full": (C.c_int, [_P, _P, _P]),
    "gmf_entries_eval": (C.c_int, [_P, _P, _P, _P, _i64, _d, _P, _P, _P]),
    "gmf_score_work_bytes": (_i64, []),
    "gmf_score_pairs": (C.c_int, [C.c_int, C.c_int, _P, _P, _i64, _d, _d, _P, _P, _P]),
    "gmf_cross_work_bytes": (_i64, [_i32, _i32]),
    "gmf_cross_rows": (C.c_int, [C.c_int, _i64, _P, _i64, _i32, _i32, _P, _i64, _i32, _i32,
                                 _P, _P, _P]),
    "gmf_rows_affine": (C.c_int, [C.c_int, _i64, _P, _i64, _i32, _i32, _d, _P, _i64, _i32, _i32,
                                  _P, _P]),
    "gmf_spmm_work_bytes": (_i64, [_i64, _i64, _i32]),
    "gmf_csr_spmm": (C.c_int, [_i64, _P, _P, _P, _i64, _d, _P, _i32, _P, _P, _P]),
    "gmf_moments_work_bytes": (_i64, []),
    "gmf_init_moments": (C.c_int, [_i64, _i64, _P, _P, _P, _P, _P, _i32, _P, _P, _i32, _d, _d,
                                   _P, _P, _P]),
    "gmf_mm_header": (C.c_int, [C.c_char_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                C.POINTER(C.c_int64)]),
    "gmf_mm_read_csr": (C.c_int, [C.c_char_p, _i64, _P, _P, _P, C.POINTER(C.c_int64)]),
    "gmf_last_error": (C.c_char_p, []),
    "gmf_version": (C.c_char_p, []),
}

_LIB = None


def lib():
    """Load libgmf_asgd.so (once).  Raises when it has not been built."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise LibraryMissingError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2412_20509_b200.build` "
                "(the aSGD path has no CPU fallback)")
        so = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(so, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = so
    return _LIB


def last_error() -> str:
    return lib().gmf_last_error().decode(errors="replace")


def check(rc: int, what: str = ""):
    """Map a C ABI return code onto the gmfkit exception taxonomy."""
    if rc == GMF_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if rc == GMF_ERR_CONFIG:
        raise ConfigError(msg)
    if rc == GMF_ERR_DOMAIN:
        raise DomainError(msg)
    if rc == GMF_ERR_UNSUPPORTED:
        raise UnsupportedError(msg)
    if rc == GMF_ERR_CUDA:
        raise CudaError(msg)
    raise GmfError(msg)


def ptr(t):
    """Raw device pointer of a torch tensor (None -> NULL)."""
    return None if t is None else C.c_void_p(t.data_ptr())


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise CudaError("the B200 aSGD path needs a CUDA device; none is visible "
                        "(there is no CPU fallback)")
