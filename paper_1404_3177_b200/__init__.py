"""B200-native (sm_100a, FP64) Newton-Raphson hot path for multinomial logit (arXiv:1404.3177).

Thin ctypes binding over the C ABI in include/mnl.h (libmnl.so, built in-tree by build.py).
Argument marshalling only: every step of the path runs in the library's CUDA kernels.  There is
no CPU fallback: if the library or a CUDA device is missing, the calls raise.

Letters follow the ABI (include/mnl.h): X[N,p] (beta_k + implicit intercept), Y[N,K,f] (generic
gamma), Z[N,K,d] (alternative-specific alpha_k, base included), choice[N] int32 (0 = base).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libmnl.so")

MNL_OK, MNL_ERR_ARG, MNL_ERR_CUDA, MNL_ERR_NOT_SPD, MNL_ERR_LINESEARCH, MNL_ERR_NONFINITE, MNL_MAXITER = range(7)

EXPORTED = ("mnl_num_params", "mnl_eval", "mnl_newton_fit", "mnl_newton_fit_ex", "mnl_eval_host",
            "mnl_newton_fit_host", "mnl_cholesky", "mnl_cholesky_solve", "mnl_last_launch_count",
            "mnl_status_string", "mnl_release", "mnl_last_hessian_times", "mnl_newton_fit_opts", "mnl_hessvec",
            "mnl_std_errors", "mnl_predict", "mnl_last_eval_ms", "mnl_eval_async", "mnl_sym_pack",
            "mnl_sym_unpack", "mnl_check_shape", "mnl_newton_fit_dp")

MNL_STOP_NONE, MNL_STOP_GTOL, MNL_STOP_FTOL, MNL_STOP_MAXITER = range(4)
MNL_METHOD_NEWTON, MNL_METHOD_CG = 0, 1


class MnlError(RuntimeError):
    def __init__(self, code: int, where: str):
        super().__init__(f"{where}: {status_string(code)} ({code})")
        self.code = code


class FitOptions(ctypes.Structure):
    """mnl_fit_options (include/mnl.h)."""
    _fields_ = [("gtol", ctypes.c_double), ("ftol", ctypes.c_double), ("max_iter", ctypes.c_int32),
                ("method", ctypes.c_int32), ("cg_max_iter", ctypes.c_int32), ("cg_rtol", ctypes.c_double)]


class FitStats(ctypes.Structure):
    _fields_ = [("iters", ctypes.c_int32), ("halvings", ctypes.c_int32), ("evals", ctypes.c_int32),
                ("status", ctypes.c_int32), ("grad_norm", ctypes.c_double), ("loglik", ctypes.c_double),
                ("hess_ms", ctypes.c_double), ("chol_ms", ctypes.c_double), ("eval_ms", ctypes.c_double),
                ("total_ms", ctypes.c_double), ("gemm_ms", ctypes.c_double),
                ("halvings_per_iter", ctypes.c_int32 * 64), ("delta_loglik", ctypes.c_double),
                ("stop_reason", ctypes.c_int32), ("cg_iters", ctypes.c_int32), ("min_margin", ctypes.c_double),
                ("loglik_per_iter", ctypes.c_double * 64), ("grad_norm_per_iter", ctypes.c_double * 64)]

    def as_dict(self) -> dict:
        per_iter = ("halvings_per_iter", "loglik_per_iter", "grad_norm_per_iter")
        d = {k: getattr(self, k) for k, _ in self._fields_ if k not in per_iter}
        for k in per_iter:
            d[k] = list(getattr(self, k)[: min(self.iters, 64)])
        return d


# int (*)(double* buf, int64_t count, void* stream, void* ctx): in-place sum across ranks (mnl.h)
ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p)

_lib = None


def load(build_if_missing: bool = False):
    """Load libmnl.so (raises if absent, unless build_if_missing)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        if not build_if_missing:
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_1404_3177_b200.build` "
                              "(or __graft_entry__.build()); there is no CPU fallback")
        from . import build as _b
        _b.build()
    lib = ctypes.CDLL(LIB_PATH)
    V, I32, I64, D = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    lib.mnl_num_params.argtypes = [I32, I32, I32, I32]
    lib.mnl_num_params.restype = I64
    lib.mnl_eval.argtypes = [I64, I32, I32, I32, I32, V, V, V, V, V, V, V, V, V]
    lib.mnl_eval.restype = ctypes.c_int
    lib.mnl_newton_fit.argtypes = [I64, I32, I32, I32, I32, V, V, V, V, V, D, I32, V,
                                   ctypes.POINTER(I32), ctypes.POINTER(D), V]
    lib.mnl_newton_fit.restype = ctypes.c_int
    lib.mnl_newton_fit_ex.argtypes = [I64, I32, I32, I32, I32, V, V, V, V, V, D, I32, V,
                                      ctypes.POINTER(I32), ctypes.POINTER(D), ctypes.POINTER(FitStats), V]
    lib.mnl_newton_fit_ex.restype = ctypes.c_int
    lib.mnl_newton_fit_opts.argtypes = [I64, I32, I32, I32, I32, V, V, V, V, V, ctypes.POINTER(FitOptions), V,
                                        ctypes.POINTER(I32), ctypes.POINTER(D), ctypes.POINTER(FitStats), V]
    lib.mnl_newton_fit_opts.restype = ctypes.c_int
    lib.mnl_newton_fit_dp.argtypes = [I64, I32, I32, I32, I32, V, V, V, V, V, ctypes.POINTER(FitOptions),
                                      ALLREDUCE_FN, V, V, ctypes.POINTER(I32), ctypes.POINTER(D),
                                      ctypes.POINTER(FitStats), V]
    lib.mnl_newton_fit_dp.restype = ctypes.c_int
    lib.mnl_hessvec.argtypes = [I64, I32, I32, I32, I32, V, V, V, V, V, V, V, V]
    lib.mnl_hessvec.restype = ctypes.c_int
    lib.mnl_check_shape.argtypes = [I64, I32, I32, I32, I32]
    lib.mnl_check_shape.restype = ctypes.c_int
    lib.mnl_sym_pack.argtypes = [I32, V, V, V]
    lib.mnl_sym_pack.restype = ctypes.c_int
    lib.mnl_sym_unpack.argtypes = [I32, V, V, V]
    lib.mnl_sym_unpack.restype = ctypes.c_int
    lib.mnl_eval_async.argtypes = [I64, I32, I32, I32, I32, V, V, V, V, V, V, V, V, V, V]
    lib.mnl_eval_async.restype = ctypes.c_int
    lib.mnl_last_eval_ms.argtypes = [ctypes.POINTER(D)]
    lib.mnl_last_eval_ms.restype = ctypes.c_int
    lib.mnl_std_errors.argtypes = [I64, I32, I32, I32, I32, V, V, V, V, V, V, V]
    lib.mnl_std_errors.restype = ctypes.c_int
    lib.mnl_predict.argtypes = [I64, I32, I32, I32, I32, V, V, V, V, V, V]
    lib.mnl_predict.restype = ctypes.c_int
    lib.mnl_eval_host.argtypes = [I64, I32, I32, I32, I32, V, V, V, V, V, V, V, V]
    lib.mnl_eval_host.restype = ctypes.c_int
    lib.mnl_newton_fit_host.argtypes = [I64, I32, I32, I32, I32, V, V, V, V, V, D, I32, V,
                                        ctypes.POINTER(I32), ctypes.POINTER(D)]
    lib.mnl_newton_fit_host.restype = ctypes.c_int
    lib.mnl_cholesky.argtypes = [I32, V, V]
    lib.mnl_cholesky.restype = ctypes.c_int
    lib.mnl_cholesky_solve.argtypes = [I32, V, V, V, V]
    lib.mnl_cholesky_solve.restype = ctypes.c_int
    lib.mnl_spd_solve.argtypes = [I32, V, V, V, V]
    lib.mnl_spd_solve.restype = ctypes.c_int
    lib.mnl_last_launch_count.argtypes = []
    lib.mnl_last_launch_count.restype = I64
    lib.mnl_status_string.argtypes = [ctypes.c_int]
    lib.mnl_status_string.restype = ctypes.c_char_p
    lib.mnl_last_hessian_times.argtypes = [ctypes.POINTER(D)]
    lib.mnl_last_hessian_times.restype = ctypes.c_int
    lib.mnl_release.argtypes = []
    lib.mnl_release.restype = None
    _lib = lib
    return lib


def status_string(code: int) -> str:
    return load().mnl_status_string(code).decode()


def shape_supported(N: int, K: int, p: int, f: int = 0, d: int = 0) -> bool:
    """True if this build supports the shape (mnl_check_shape; no device needed)."""
    return load().mnl_check_shape(N, K, p, f, d) == MNL_OK


def num_params(K: int, p: int, f: int = 0, d: int = 0) -> int:
    return int(load().mnl_num_params(K, p, f, d))


def last_launch_count() -> int:
    """Kernel launches made by the last library call (counted by the library)."""
    return int(load().mnl_last_launch_count())


def last_eval_ms() -> float:
    """Device time (ms) of the last pass-1 kernel."""
    v = ctypes.c_double(0.0)
    rc = load().mnl_last_eval_ms(ctypes.byref(v))
    if rc != MNL_OK:
        raise MnlError(rc, "mnl_last_eval_ms")
    return v.value


def last_hessian_times() -> dict:
    """Device ms of the last Hessian assembly phases (CUDA events inside the library)."""
    out = (ctypes.c_double * 7)()
    load().mnl_last_hessian_times(out)
    return dict(j1_gemm=out[0], j1_reduce=out[1], j1_tail=out[2], j1_tail_reduce=out[3], j2_and_arrow=out[4],
                assemble=out[5], j1_operands=out[6])


def release() -> None:
    load().mnl_release()


# ---------------------------------------------------------------------------------------------
# torch (device) entry points
# ---------------------------------------------------------------------------------------------

def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1404_3177_b200 needs a CUDA device (no CPU fallback)")
    return torch


@dataclass
class Problem:
    """Device-resident inputs in the ABI layout (validated once)."""
    X: "object"
    Y: "object"
    Z: "object"
    choice: "object"
    N: int
    K: int
    p: int
    f: int
    d: int

    @property
    def n_p(self) -> int:
        return (self.K - 1) * (self.p + 1) + self.K * self.d + self.f

    def ptrs(self):
        return (self.X.data_ptr() if self.p else None, self.Y.data_ptr() if self.f else None,
                self.Z.data_ptr() if self.d else None, self.choice.data_ptr())


def problem(X, Y, Z, choice, K: int | None = None) -> Problem:
    """Wrap CUDA tensors X[N,p], Y[N,K,f], Z[N,K,d] (float64) and choice[N] (int32)."""
    torch = _torch()
    N = choice.shape[0]
    if K is None:
        K = Y.shape[1] if Y is not None and Y.dim() == 3 and Y.shape[1] else Z.shape[1]
    for name, t in (("X", X), ("Y", Y), ("Z", Z)):
        if t is not None and t.numel():
            if t.dtype != torch.float64 or not t.is_cuda or not t.is_contiguous():
                raise ValueError(f"{name} must be a contiguous CUDA float64 tensor")
    if choice.dtype != torch.int32 or not choice.is_cuda or not choice.is_contiguous():
        raise ValueError("choice must be a contiguous CUDA int32 tensor")
    p = X.shape[1] if X is not None and X.dim() == 2 else 0
    f = Y.shape[2] if Y is not None and Y.dim() == 3 else 0
    d = Z.shape[2] if Z is not None and Z.dim() == 3 else 0
    return Problem(X, Y, Z, choice, int(N), int(K), int(p), int(f), int(d))


def _stream(stream):
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def mnl_eval(prob: Problem, coef, grad: bool = True, hess: bool = False, stream=None):
    """(loglik[1], grad[n_p] | None, hess[n_p, n_p] | None) at coef (CUDA float64 [n_p])."""
    torch = _torch()
    dev = prob.choice.device
    ll = torch.empty(1, dtype=torch.float64, device=dev)
    g = torch.empty(prob.n_p, dtype=torch.float64, device=dev) if grad else None
    H = torch.empty(prob.n_p, prob.n_p, dtype=torch.float64, device=dev) if hess else None
    X, Y, Z, ch = prob.ptrs()
    rc = load().mnl_eval(prob.N, prob.K, prob.p, prob.f, prob.d, X, Y, Z, ch, coef.data_ptr(), ll.data_ptr(),
                         g.data_ptr() if grad else None, H.data_ptr() if hess else None, _stream(stream))
    if rc != MNL_OK:
        raise MnlError(rc, "mnl_eval")
    return ll, g, H


def mnl_eval_async(prob: Problem, coef, grad: bool = True, hess: bool = False, stream=None):
    """Enqueue an evaluation without synchronising: returns (loglik[1], grad | None, hess | None,
    status[1] int32) device tensors, valid once the stream has passed the work."""
    torch = _torch()
    dev = prob.choice.device
    ll = torch.empty(1, dtype=torch.float64, device=dev)
    st = torch.empty(1, dtype=torch.int32, device=dev)
    g = torch.empty(prob.n_p, dtype=torch.float64, device=dev) if grad else None
    H = torch.empty(prob.n_p, prob.n_p, dtype=torch.float64, device=dev) if hess else None
    X, Y, Z, ch = prob.ptrs()
    rc = load().mnl_eval_async(prob.N, prob.K, prob.p, prob.f, prob.d, X, Y, Z, ch, coef.data_ptr(), ll.data_ptr(),
                               g.data_ptr() if grad else None, H.data_ptr() if hess else None, st.data_ptr(),
                               _stream(stream))
    if rc != MNL_OK:
        raise MnlError(rc, "mnl_eval_async")
    return ll, g, H, st


@dataclass
class FitResult:
    coef: "object"
    iters: int
    loglik: float
    status: int
    stats: dict


def mnl_newton_fit(prob: Problem, coef0=None, tol: float = 1e-6, max_iter: int = 50, stream=None,
                   raise_on_error: bool = True, ftol: float = 0.0, method: str = "newton",
                   cg_max_iter: int = 0, cg_rtol: float = 0.0) -> FitResult:
    """Newton-Raphson fit (mnl_newton_fit_opts): gtol = tol, ftol (0 = off), method "newton" (exact
    Hessian + Cholesky) or "cg" (truncated Newton on Hessian-vector products)."""
    torch = _torch()
    coef = torch.empty(prob.n_p, dtype=torch.float64, device=prob.choice.device)
    it = ctypes.c_int32(0)
    ll = ctypes.c_double(0.0)
    st = FitStats()
    opts = FitOptions(tol, ftol, max_iter, {"newton": MNL_METHOD_NEWTON, "cg": MNL_METHOD_CG}[method],
                      cg_max_iter, cg_rtol)
    X, Y, Z, ch = prob.ptrs()
    rc = load().mnl_newton_fit_opts(prob.N, prob.K, prob.p, prob.f, prob.d, X, Y, Z, ch,
                                    coef0.data_ptr() if coef0 is not None else None, ctypes.byref(opts),
                                    coef.data_ptr(), ctypes.byref(it), ctypes.byref(ll), ctypes.byref(st),
                                    _stream(stream))
    if raise_on_error and rc not in (MNL_OK, MNL_MAXITER):
        raise MnlError(rc, "mnl_newton_fit")
    return FitResult(coef, it.value, ll.value, rc, st.as_dict())


def mnl_newton_fit_dp(prob: Problem, allreduce, coef0=None, tol: float = 1e-6, max_iter: int = 50, stream=None,
                      raise_on_error: bool = True, ftol: float = 0.0, method: str = "newton",
                      cg_max_iter: int = 0, cg_rtol: float = 0.0) -> FitResult:
    """Data-parallel fit (mnl_newton_fit_dp): `prob` holds THIS rank's individuals; `allreduce` is an
    ALLREDUCE_FN (e.g. distributed.torch_allreduce()) that sums a device buffer across ranks."""
    torch = _torch()
    coef = torch.empty(prob.n_p, dtype=torch.float64, device=prob.choice.device)
    it = ctypes.c_int32(0)
    ll = ctypes.c_double(0.0)
    st = FitStats()
    opts = FitOptions(tol, ftol, max_iter, {"newton": MNL_METHOD_NEWTON, "cg": MNL_METHOD_CG}[method],
                      cg_max_iter, cg_rtol)
    X, Y, Z, ch = prob.ptrs()
    rc = load().mnl_newton_fit_dp(prob.N, prob.K, prob.p, prob.f, prob.d, X, Y, Z, ch,
                                  coef0.data_ptr() if coef0 is not None else None, ctypes.byref(opts), allreduce,
                                  None, coef.data_ptr(), ctypes.byref(it), ctypes.byref(ll), ctypes.byref(st),
                                  _stream(stream))
    if raise_on_error and rc not in (MNL_OK, MNL_MAXITER):
        raise MnlError(rc, "mnl_newton_fit_dp")
    return FitResult(coef, it.value, ll.value, rc, st.as_dict())


def mnl_hessvec(prob: Problem, coef, v, stream=None):
    """H v at coef (CUDA float64 [n_p] each), without forming H."""
    torch = _torch()
    hv = torch.empty(prob.n_p, dtype=torch.float64, device=prob.choice.device)
    X, Y, Z, ch = prob.ptrs()
    rc = load().mnl_hessvec(prob.N, prob.K, prob.p, prob.f, prob.d, X, Y, Z, ch, coef.data_ptr(), v.data_ptr(),
                            hv.data_ptr(), _stream(stream))
    if rc != MNL_OK:
        raise MnlError(rc, "mnl_hessvec")
    return hv


def mnl_std_errors(prob: Problem, coef, stream=None):
    """sqrt(diag((-H)^{-1})) at coef (CUDA float64 [n_p]); the asymptotic standard errors at the MLE."""
    torch = _torch()
    se = torch.empty(prob.n_p, dtype=torch.float64, device=prob.choice.device)
    X, Y, Z, ch = prob.ptrs()
    rc = load().mnl_std_errors(prob.N, prob.K, prob.p, prob.f, prob.d, X, Y, Z, ch, coef.data_ptr(), se.data_ptr(),
                               _stream(stream))
    if rc != MNL_OK:
        raise MnlError(rc, "mnl_std_errors")
    return se


def mnl_predict(prob: Problem, coef, stream=None):
    """Choice probabilities P[N, K] at coef (CUDA float64 [n_p])."""
    torch = _torch()
    P = torch.empty(prob.N, prob.K, dtype=torch.float64, device=prob.choice.device)
    X, Y, Z, _ = prob.ptrs()
    rc = load().mnl_predict(prob.N, prob.K, prob.p, prob.f, prob.d, X, Y, Z, coef.data_ptr(), P.data_ptr(),
                            _stream(stream))
    if rc != MNL_OK:
        raise MnlError(rc, "mnl_predict")
    return P


def mnl_sym_pack(H, out=None, stream=None):
    """Upper triangle of the symmetric CUDA float64 [n, n] H, packed row by row (n(n+1)/2)."""
    torch = _torch()
    n = H.shape[0]
    if out is None:
        out = torch.empty(n * (n + 1) // 2, dtype=torch.float64, device=H.device)
    rc = load().mnl_sym_pack(n, H.data_ptr(), out.data_ptr(), _stream(stream))
    if rc != MNL_OK:
        raise MnlError(rc, "mnl_sym_pack")
    return out


def mnl_sym_unpack(packed, n: int, out=None, stream=None):
    """The symmetric [n, n] matrix from its packed upper triangle (both triangles written)."""
    torch = _torch()
    if out is None:
        out = torch.empty(n, n, dtype=torch.float64, device=packed.device)
    rc = load().mnl_sym_unpack(n, packed.data_ptr(), out.data_ptr(), _stream(stream))
    if rc != MNL_OK:
        raise MnlError(rc, "mnl_sym_unpack")
    return out


def mnl_cholesky(A, stream=None):
    """In-place lower Cholesky of the SPD CUDA float64 [n, n] tensor A; returns the status."""
    return load().mnl_cholesky(A.shape[0], A.data_ptr(), _stream(stream))


def mnl_cholesky_solve(L, b, stream=None):
    torch = _torch()
    x = torch.empty_like(b)
    rc = load().mnl_cholesky_solve(L.shape[0], L.data_ptr(), b.data_ptr(), x.data_ptr(), _stream(stream))
    if rc != MNL_OK:
        raise MnlError(rc, "mnl_cholesky_solve")
    return x


def mnl_spd_solve(A, b, stream=None):
    """x = A^{-1} b for the SPD CUDA float64 [n, n] tensor A (not modified): the Newton step's fused
    factor + solve path. Raises MnlError (MNL_ERR_NOT_SPD) if A is not positive definite."""
    torch = _torch()
    x = torch.empty_like(b)
    rc = load().mnl_spd_solve(A.shape[0], A.data_ptr(), b.data_ptr(), x.data_ptr(), _stream(stream))
    if rc != MNL_OK:
        raise MnlError(rc, "mnl_spd_solve")
    return x


# ---------------------------------------------------------------------------------------------
# host-buffer entry points (numpy); the library copies in and out inside the call
# ---------------------------------------------------------------------------------------------

def _np_ptr(a):
    return a.ctypes.data if a is not None and a.size else None


def mnl_eval_host(X, Y, Z, choice, coef, K: int, grad: bool = True, hess: bool = False):
    X = np.ascontiguousarray(X, dtype=np.float64)
    N = choice.shape[0]
    p = X.shape[1] if X.ndim == 2 else 0
    f = Y.shape[2] if Y is not None and Y.ndim == 3 else 0
    d = Z.shape[2] if Z is not None and Z.ndim == 3 else 0
    n_p = (K - 1) * (p + 1) + K * d + f
    ll = np.zeros(1)
    g = np.empty(n_p) if grad else None
    H = np.empty((n_p, n_p)) if hess else None
    Yc = np.ascontiguousarray(Y, dtype=np.float64) if f else None
    Zc = np.ascontiguousarray(Z, dtype=np.float64) if d else None
    ch = np.ascontiguousarray(choice, dtype=np.int32)
    cf = np.ascontiguousarray(coef, dtype=np.float64)
    rc = load().mnl_eval_host(N, K, p, f, d, _np_ptr(X), _np_ptr(Yc), _np_ptr(Zc), ch.ctypes.data,
                              cf.ctypes.data, ll.ctypes.data, _np_ptr(g), _np_ptr(H))
    if rc != MNL_OK:
        raise MnlError(rc, "mnl_eval_host")
    return float(ll[0]), g, H


def mnl_newton_fit_host(X, Y, Z, choice, K: int, coef0=None, tol: float = 1e-6, max_iter: int = 50):
    X = np.ascontiguousarray(X, dtype=np.float64)
    N = choice.shape[0]
    p = X.shape[1] if X.ndim == 2 else 0
    f = Y.shape[2] if Y is not None and Y.ndim == 3 else 0
    d = Z.shape[2] if Z is not None and Z.ndim == 3 else 0
    n_p = (K - 1) * (p + 1) + K * d + f
    Yc = np.ascontiguousarray(Y, dtype=np.float64) if f else None
    Zc = np.ascontiguousarray(Z, dtype=np.float64) if d else None
    ch = np.ascontiguousarray(choice, dtype=np.int32)
    c0 = np.ascontiguousarray(coef0, dtype=np.float64) if coef0 is not None else None
    coef = np.empty(n_p)
    it = ctypes.c_int32(0)
    ll = ctypes.c_double(0.0)
    rc = load().mnl_newton_fit_host(N, K, p, f, d, _np_ptr(X), _np_ptr(Yc), _np_ptr(Zc), ch.ctypes.data,
                                    _np_ptr(c0), tol, max_iter, coef.ctypes.data, ctypes.byref(it),
                                    ctypes.byref(ll))
    if rc not in (MNL_OK, MNL_MAXITER):
        raise MnlError(rc, "mnl_newton_fit_host")
    return coef, it.value, ll.value, rc
