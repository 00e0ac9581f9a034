"""Data-parallel Newton-Raphson over individuals (§8(f) f3).

The log-likelihood, gradient and Hessian are sums over individuals (P:348-351, P:435-443,
P:462-476), so each rank owns a contiguous slice of the individuals and calls the library's
data-parallel fit (`mnl_newton_fit_dp`, include/mnl.h) on it. The Newton-Raphson driver itself is
the library's (csrc/nr_driver.h, the same code as the single-GPU fit); at each exchange step it calls
back into an all-reduce that sums a DEVICE buffer across ranks:
  after every pass-1 evaluation   [l, bad-choice flag, g]        n_p + 2 doubles
  after every Hessian             packed upper triangle of -H    n_p (n_p + 1) / 2 doubles
All-reduce results are identical on every rank, so every rank factors the same -H and takes the
same step; the iterates stay bitwise identical without broadcasting the coefficients.

This module is argument marshalling only: the shard range, a torch.distributed (NCCL) all-reduce
callback over a raw device pointer, and the binding of the host-callback build of the same driver
(libnrhost.so) that tests/test_distributed.py runs on CPU with gloo.
"""
from __future__ import annotations

import ctypes
import os

from . import ALLREDUCE_FN, LIB_PATH, load, mnl_newton_fit_dp  # noqa: F401

HOST_LIB = os.path.join(os.path.dirname(LIB_PATH), "libnrhost.so")


def shard_range(N: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced slice [lo, hi) of the N individuals for `rank`."""
    base, rem = divmod(N, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


class _CudaArray:
    """A raw device pointer as a __cuda_array_interface__ object (torch.as_tensor wraps it, no copy)."""

    def __init__(self, ptr: int, count: int):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": "<f8", "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def device_view(ptr: int, count: int):
    """The library's device buffer [count] float64 as a torch tensor (shares memory)."""
    import torch
    return torch.as_tensor(_CudaArray(ptr, count), device="cuda")


def torch_stream(stream_ptr):
    import torch
    return torch.cuda.ExternalStream(stream_ptr) if stream_ptr else torch.cuda.default_stream()


def torch_allreduce(group=None):
    """ALLREDUCE_FN summing the buffer over `group` with torch.distributed (NCCL), ordered on the
    library's stream. Keep the returned object alive for the duration of the fit."""
    import torch
    import torch.distributed as dist

    def cb(buf, count, stream, ctx):
        try:
            t = device_view(buf, count)
            with torch.cuda.stream(torch_stream(stream)):
                dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
            return 0
        except Exception:  # noqa: BLE001 -- reported to the library as a failed exchange
            return 1

    return ALLREDUCE_FN(cb)


def newton_fit_dp(prob_local, group=None, **kw):
    """mnl_newton_fit_dp on this rank's shard with the torch.distributed all-reduce."""
    fn = torch_allreduce(group)
    return mnl_newton_fit_dp(prob_local, fn, **kw)


# ---- the same driver over host callbacks (libnrhost.so; CPU tests) ------------------------------

EVAL_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_double),
                           ctypes.POINTER(ctypes.c_double))
DIR_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_int))
TRIAL_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                            ctypes.POINTER(ctypes.c_double))
ACCEPT_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p)


class HostOps(ctypes.Structure):
    _fields_ = [("ctx", ctypes.c_void_p), ("eval_theta", EVAL_FN), ("direction", DIR_FN),
                ("eval_trial", TRIAL_FN), ("accept", ACCEPT_FN)]


class HostReport(ctypes.Structure):
    _fields_ = [("iters", ctypes.c_int32), ("halvings", ctypes.c_int32), ("evals", ctypes.c_int32),
                ("status", ctypes.c_int32), ("stop_reason", ctypes.c_int32),
                ("halvings_per_iter", ctypes.c_int32 * 64), ("loglik", ctypes.c_double),
                ("grad_norm", ctypes.c_double), ("delta_loglik", ctypes.c_double), ("min_margin", ctypes.c_double),
                ("loglik_per_iter", ctypes.c_double * 64), ("grad_norm_per_iter", ctypes.c_double * 64)]


_host = None


def _host_lib():
    global _host
    if _host is None:
        if not os.path.exists(HOST_LIB):
            from . import build as _b
            _b.build_host()
        _host = ctypes.CDLL(HOST_LIB)
        _host.nr_fit_host.argtypes = [ctypes.POINTER(HostOps), ctypes.c_double, ctypes.c_double, ctypes.c_int32,
                                      ctypes.POINTER(HostReport)]
        _host.nr_fit_host.restype = ctypes.c_int
    return _host


def run_host_driver(eval_theta, direction, eval_trial, accept, gtol=1e-6, ftol=0.0, max_iter=50) -> dict:
    """The library's Newton-Raphson driver (nr_driver.h) over Python callables:
      eval_theta() -> (status, l, ||g||^2)        at the current iterate
      direction() -> (status, not_spd)            the Newton direction there
      eval_trial(j) -> (status, l, ||g||^2)       at theta + delta / 2^j
      accept()                                    theta <- the last trial
    Returns the driver's report as a dict."""

    def _e(ctx, l, g2):
        rc, lv, gv = eval_theta()
        l[0], g2[0] = lv, gv
        return rc

    def _d(ctx, ns):
        rc, bad = direction()
        ns[0] = int(bool(bad))
        return rc

    def _t(ctx, j, l, g2):
        rc, lv, gv = eval_trial(j)
        l[0], g2[0] = lv, gv
        return rc

    def _a(ctx):
        accept()

    ops = HostOps(None, EVAL_FN(_e), DIR_FN(_d), TRIAL_FN(_t), ACCEPT_FN(_a))
    rep = HostReport()
    rc = _host_lib().nr_fit_host(ctypes.byref(ops), gtol, ftol, max_iter, ctypes.byref(rep))
    per_iter = ("halvings_per_iter", "loglik_per_iter", "grad_norm_per_iter")
    out = {k: getattr(rep, k) for k, _ in HostReport._fields_ if k not in per_iter}
    for k in per_iter:
        out[k] = list(getattr(rep, k)[:min(rep.iters, 64)])
    out["rc"] = rc
    return out
