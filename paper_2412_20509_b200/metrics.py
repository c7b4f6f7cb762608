"""Out-of-sample evaluation metrics on the GPU (gmfkit/metrics.py:1-55).

Both are ratios against the constant train-mean predictor: values below 1
mean the model beats that baseline on the held-out entries.  The four sums
(model and baseline deviance, model and baseline squared log ratios) come
from one fixed-order reduction kernel (``gmf_score_pairs``); argument
checks and error types follow the reference (``ConfigError`` for an empty
or mismatched test set, ``DegenerateError`` for a zero baseline).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .exceptions import ConfigError, DegenerateError
from .families import FamilySpec

__all__ = ["EvalResult", "rel_log_rmse", "rel_deviance", "score_sums"]


@dataclass
class EvalResult:
    rel_log_rmse: float
    rel_deviance: float
    n_test: int


def _as_device(a, device):
    import torch
    if isinstance(a, torch.Tensor):
        return a.to(device=device, dtype=torch.float64).reshape(-1).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=float).ravel())).to(device)


def _check_args(y_test, mu_hat):
    """metrics.py:25-32: flatten, refuse an empty or mismatched pair."""
    ny = int(y_test.numel()) if hasattr(y_test, "numel") else np.asarray(y_test).size
    nm = int(mu_hat.numel()) if hasattr(mu_hat, "numel") else np.asarray(mu_hat).size
    if ny == 0:
        raise ConfigError("test set is empty")
    if ny != nm:
        raise ConfigError("y_test and mu_hat must have the same length")


def score_sums(y_test, mu_hat, ybar_train: float, fam: FamilySpec | None = None, *,
               device=None) -> np.ndarray:
    """[sum D(y, mu), sum D(y, ybar), sum log^2((1+y)/(1+mu)),
    sum log^2((1+y)/(1+ybar))] of the pairs, computed on the GPU."""
    import torch
    _lib.require_cuda()
    _check_args(y_test, mu_hat)
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else
                       int(str(device).split(":")[-1]))
    y, mu = _as_device(y_test, dev), _as_device(mu_hat, dev)
    lib = _lib.lib()
    work = torch.empty(int(lib.gmf_score_work_bytes()), dtype=torch.uint8, device=dev)
    out = torch.zeros(4, dtype=torch.float64, device=dev)
    fcode = _lib.FAMILY_CODES["poisson" if fam is None else fam.kind]
    alpha = fam.nb_shape if fam is not None and fam.kind == "neg_binomial" else 1.0
    stream = torch.cuda.current_stream(dev).cuda_stream
    _lib.check(lib.gmf_score_pairs(fcode, _lib.F64, _lib.ptr(y), _lib.ptr(mu), y.numel(),
                                   float(ybar_train), alpha, _lib.ptr(out), _lib.ptr(work),
                                   stream), "gmf_score_pairs")
    return out.cpu().numpy()


def ratios(sums) -> tuple[float, float]:
    """(rel_deviance, rel_log_rmse) from score sums; DegenerateError on a zero
    baseline (metrics.py:44-45, 53-54)."""
    if sums[3] == 0.0 or sums[1] == 0.0:
        raise DegenerateError("all test responses equal the train mean baseline")
    return float(sums[0] / sums[1]), float(sums[2] / sums[3])


def rel_log_rmse(y_test, mu_hat, ybar_train: float, *, device=None) -> float:
    """sum log^2{(1+y)/(1+mu_hat)} / sum log^2{(1+y)/(1+ybar_train)} (metrics.py:35-45)."""
    s = score_sums(y_test, mu_hat, ybar_train, None, device=device)
    if s[3] == 0.0:
        raise DegenerateError("all test responses equal the train mean baseline")
    return float(s[2] / s[3])


def rel_deviance(y_test, mu_hat, ybar_train: float, fam: FamilySpec, *, device=None) -> float:
    """sum D(y, mu_hat) / sum D(y, ybar_train) over the test entries (metrics.py:48-55)."""
    s = score_sums(y_test, mu_hat, ybar_train, fam, device=device)
    if s[1] == 0.0:
        raise DegenerateError("all test responses equal the train mean baseline")
    return float(s[0] / s[1])
