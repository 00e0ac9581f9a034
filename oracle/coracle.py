"""ctypes adapter for liboracle.so (oracle/oracle.c): the plain CPU C oracle with the same Python
API as oracle/mnl_oracle.py (numpy), so every pin in tests/test_oracle_pins.py runs against both.

TEST INFRASTRUCTURE ONLY (tests/, __graft_entry__.smoke(), bench.py's cpu_baseline and
--impl reference legs). Shares no code with paper_1404_3177_b200/.

Functions the C library does not implement are formed here from its outputs by their definitions
only (H v = H @ v from the C Hessian; entries of H read from it; standard errors = numpy's inverse of
-H, the library step of the numpy oracle too). The truncated-Newton fit is numpy-oracle only.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from .mnl_oracle import (Data, FitLog, MAX_HALVINGS, MNL_ERR_ARG, MNL_ERR_LINESEARCH,  # noqa: F401
                         MNL_ERR_NONFINITE, MNL_ERR_NOT_SPD, MNL_MAXITER, MNL_OK, TAU_REL, make_data,
                         num_params)

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_HDR = os.path.join(_HERE, "oracle.h")
SO = os.path.join(_HERE, "liboracle.so")
_lib = None
KIND = "c"


def build(force: bool = False) -> str:
    """gcc -O3 -fopenmp (plain C; no -ffast-math: IEEE fp64 arithmetic in source order)."""
    stale = not os.path.exists(SO) or any(os.path.getmtime(s) > os.path.getmtime(SO) for s in (_SRC, _HDR))
    if force or stale:
        tmp = SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O3", "-std=c11", "-fopenmp", "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, SO)
    return SO


class IterLog(ctypes.Structure):
    _fields_ = [("loglik", ctypes.c_double), ("grad_norm", ctypes.c_double), ("loglik_new", ctypes.c_double),
                ("margin", ctypes.c_double), ("rejected_margin", ctypes.c_double), ("halvings", ctypes.c_int32),
                ("pad_", ctypes.c_int32)]


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(SO)
        P, I64, I32, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double
        dims = [I64, I32, I32, I32, I32]
        L.oracle_set_threads.argtypes = [I32]
        L.oracle_mnl_utilities.argtypes = dims + [P, P, P, P, P]
        L.oracle_mnl_softmax.argtypes = [I64, I32, P, P, P]
        L.oracle_mnl_eval.argtypes = dims + [P] * 8
        L.oracle_mnl_newton_fit.argtypes = dims + [P] * 5 + [D, I32, P, P, P]
        L.oracle_mnl_newton_fit_log.argtypes = dims + [P] * 5 + [D, I32, D, P, P, P, P, P, P, I32]
        L.oracle_cholesky.argtypes = [I32, P]
        L.oracle_cholesky_solve.argtypes = [I32, P, P, P]
        _lib = L
    return _lib


def set_threads(n: int = 0) -> int:
    return lib().oracle_set_threads(int(n))


def _ptr(a):
    return None if a is None or a.size == 0 else a.ctypes.data


def _args(D: Data):
    X = np.ascontiguousarray(D.X) if D.p else None
    Y = np.ascontiguousarray(D.Y) if D.f else None
    Z = np.ascontiguousarray(D.Z) if D.d else None
    ch = np.ascontiguousarray(D.choice, dtype=np.int32)
    return (X, Y, Z, ch)


def _dims(D: Data):
    return (D.N, D.K, D.p, D.f, D.d)


def utilities(D: Data, theta) -> np.ndarray:
    th = np.ascontiguousarray(theta, dtype=np.float64)
    X, Y, Z, _ = _args(D)
    V = np.empty((D.N, D.K))
    rc = lib().oracle_mnl_utilities(*_dims(D), _ptr(X), _ptr(Y), _ptr(Z), th.ctypes.data, V.ctypes.data)
    assert rc == MNL_OK, rc
    return V


def _softmax(V):
    V = np.ascontiguousarray(V, dtype=np.float64)
    P = np.empty_like(V)
    lse = np.empty(V.shape[0])
    rc = lib().oracle_mnl_softmax(V.shape[0], V.shape[1], V.ctypes.data, P.ctypes.data, lse.ctypes.data)
    assert rc == MNL_OK, rc
    return P, lse


def probabilities(V) -> np.ndarray:
    return _softmax(V)[0]


def loglik_terms(V, choice) -> np.ndarray:
    V = np.asarray(V, dtype=np.float64)
    return V[np.arange(V.shape[0]), np.asarray(choice)] - _softmax(V)[1]


def mnl_eval(D: Data, theta, want_grad=True, want_hess=True, status=False):
    th = np.ascontiguousarray(theta, dtype=np.float64)
    X, Y, Z, ch = _args(D)
    l = ctypes.c_double()
    g = np.empty(D.n_p) if want_grad else None
    H = np.empty((D.n_p, D.n_p)) if want_hess else None
    rc = lib().oracle_mnl_eval(*_dims(D), _ptr(X), _ptr(Y), _ptr(Z), ch.ctypes.data, th.ctypes.data,
                               ctypes.byref(l), _ptr(g), _ptr(H))
    if status:
        return rc, l.value, g, H
    assert rc in (MNL_OK, MNL_ERR_NONFINITE), rc
    return l.value, g, H


def loglik(D: Data, theta) -> float:
    return mnl_eval(D, theta, False, False)[0]


def gradient(D: Data, theta, P=None) -> np.ndarray:
    return mnl_eval(D, theta, True, False)[1]


def hessian(D: Data, theta, P=None) -> np.ndarray:
    return mnl_eval(D, theta, False, True)[2]


def hessian_entries(D: Data, theta, rows, cols, P=None) -> np.ndarray:
    H = hessian(D, theta)
    return H[np.asarray(rows, dtype=np.int64), np.asarray(cols, dtype=np.int64)]


def hessvec(D: Data, theta, v, P=None) -> np.ndarray:
    return hessian(D, theta) @ np.asarray(v, dtype=np.float64)


def std_errors(D: Data, theta) -> np.ndarray:
    return np.sqrt(np.diag(np.linalg.inv(-hessian(D, theta))))


def predict(D: Data, theta) -> np.ndarray:
    return probabilities(utilities(D, theta))


def cholesky(A) -> np.ndarray:
    L = np.array(A, dtype=np.float64, order="C")
    rc = lib().oracle_cholesky(L.shape[0], L.ctypes.data)
    if rc != MNL_OK:
        raise np.linalg.LinAlgError("not SPD")
    return L


def newton_fit(D: Data, coef0=None, tol: float = 1e-6, max_iter: int = 50, hess_fn=None, ftol: float = 0.0,
               step_fn=None) -> FitLog:
    """oracle_mnl_newton_fit_log; history entries carry l, gnorm, halvings, l_new and the R7 margins
    (margin = (l_new - (l - tau)) / max(1,|l|) of the accepted trial, rejected_margin of the last
    rejected one)."""
    assert hess_fn is None and step_fn is None, "the C oracle has one Newton step (Cholesky of -H)"
    X, Y, Z, ch = _args(D)
    c0 = None if coef0 is None else np.ascontiguousarray(coef0, dtype=np.float64)
    coef = np.empty(D.n_p)
    it, l, gn, stop = ctypes.c_int32(), ctypes.c_double(), ctypes.c_double(), ctypes.c_int32()
    cap = max(int(max_iter), 0) + 1
    logs = (IterLog * cap)()
    rc = lib().oracle_mnl_newton_fit_log(*_dims(D), _ptr(X), _ptr(Y), _ptr(Z), ch.ctypes.data, _ptr(c0), tol,
                                          int(max_iter), ftol, coef.ctypes.data, ctypes.byref(it), ctypes.byref(l),
                                          ctypes.byref(gn), ctypes.byref(stop), logs, cap)
    out = FitLog()
    out.status, out.iters, out.loglik, out.coef = rc, it.value, l.value, coef
    out.grad_norm, out.stop_reason = gn.value, stop.value
    out.history = [dict(l=e.loglik, gnorm=e.grad_norm, halvings=e.halvings, l_new=e.loglik_new,
                        margin=e.margin, rejected_margin=e.rejected_margin)
                   for e in list(logs)[:min(it.value, cap)]]
    if out.history:
        out.delta_loglik = abs(out.history[-1]["l_new"] - out.history[-1]["l"])
    return out
