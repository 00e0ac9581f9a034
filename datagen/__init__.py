"""Seeded synthetic inputs for the five BASELINE.json configs.

Shared by the oracle tests, the GPU parity tests and bench.py.  Holds none of
the estimator's arithmetic: it only draws arrays and samples choices from the
paper's random-utility model (see gen.c).  Shapes and distributions follow
BASELINE.json `configs` with the readings SURVEY.md §8(c) R15-R18:

  c1 tiny mixed : N=1000,   K=4,   p=3,  f=2,  d=1; X,Y~N(0,1), Z~U(-1,1), coefs~N(0,0.5)
  c2 X-only     : N=20000,  K=10,  p=20;            X~N(0,1), coefs~N(0,0.3)
  c3 X-only     : N=100000, K=20,  p=50;  X~N(0,1), columns j%10==9 ~ Bernoulli(0.3), coefs~N(0,0.2)
  c4 X-only     : N=500000, K=100, p=50;  X~N(0,1), beta~N(0,0.1), intercepts xi~N(0,1)
  c5 mixed+fit  : N=200000, K=50,  p=30, f=10, d=5; X,Y~N(0,1), Z~U(-1,1), coefs~N(0,0.1)

Letters are the ABI's: Y[N,K,f] has the generic coefficient
gamma, Z[N,K,d] the alternative-specific alpha_k (k = 0..K-1), X[N,p] the
individual-specific beta_k with an implicit intercept xi_k first in each chunk.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libmnlgen.so")
_lib = None


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "gen.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", _SO, src, "-lm"])
    return _SO


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        P = ctypes.c_void_p
        lib.gen_fill.argtypes = [P, ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, ctypes.c_double]
        lib.gen_fill_col.argtypes = [P, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64,
                                     ctypes.c_uint64, ctypes.c_int, ctypes.c_double]
        lib.gen_choices.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                    P, P, P, P, ctypes.c_uint64, ctypes.c_uint64, P]
        _lib = lib
    return _lib


NORMAL, UNIFORM, BERNOULLI = 0, 1, 2
# array ids inside a config's stream space
_S_X, _S_Y, _S_Z, _S_COEF, _S_CHOICE, _S_XI, _S_PERTURB, _S_START = 1, 2, 3, 4, 5, 6, 7, 8
_S_BERN = 64  # + column index


@dataclass(frozen=True)
class Spec:
    name: str
    N: int
    K: int
    p: int
    f: int = 0
    d: int = 0
    coef_sd: float = 0.5          # sd of every coefficient (R15: "N(0,s)" = sd s)
    xi_sd: float | None = None    # sd of the intercepts if different (c4, R17)
    bern_cols: tuple = ()         # X columns drawn Bernoulli(bern_p) instead of N(0,1) (c3, R16)
    bern_p: float = 0.3
    stream_base: int = 0          # separates the configs' RNG streams

    @property
    def n_params(self) -> int:
        return num_params(self.K, self.p, self.f, self.d)


CONFIGS = {
    "c1": Spec("c1", 1000, 4, 3, 2, 1, coef_sd=0.5, stream_base=1 << 20),
    "c2": Spec("c2", 20000, 10, 20, coef_sd=0.3, stream_base=2 << 20),
    "c3": Spec("c3", 100000, 20, 50, coef_sd=0.2, bern_cols=(9, 19, 29, 39, 49), stream_base=3 << 20),
    "c4": Spec("c4", 500000, 100, 50, coef_sd=0.1, xi_sd=1.0, stream_base=4 << 20),
    "c5": Spec("c5", 200000, 50, 30, 10, 5, coef_sd=0.1, stream_base=5 << 20),
}


def num_params(K: int, p: int, f: int, d: int) -> int:
    """n_p = (K-1)(p+1) + K*d + f  (layout SURVEY.md §0.3)."""
    return (K - 1) * (p + 1) + K * d + f


@dataclass
class Problem:
    spec: Spec
    seed: int
    X: np.ndarray            # [N, p] float64 (C-contiguous)
    Y: np.ndarray            # [N, K, f]
    Z: np.ndarray            # [N, K, d]
    choice: np.ndarray       # [N] int32 in [0, K)
    theta_true: np.ndarray   # [n_p]
    counts: np.ndarray = field(default=None)

    @property
    def dims(self):
        s = self.spec
        return s.N, s.K, s.p, s.f, s.d


def _arr(n):
    return np.empty(n, dtype=np.float64)


def draw(n: int, seed: int, stream: int, dist: int = NORMAL, scale: float = 1.0) -> np.ndarray:
    out = _arr(n)
    if n:
        _load().gen_fill(out.ctypes.data, n, seed, stream, dist, scale)
    return out


def make(spec: Spec | str, seed: int = 0, require_all_classes: bool = True) -> Problem:
    """Draw one problem instance. Deterministic in (spec, seed)."""
    if isinstance(spec, str):
        spec = CONFIGS[spec]
    lib = _load()
    N, K, p, f, d = spec.N, spec.K, spec.p, spec.f, spec.d
    sb = spec.stream_base
    X = draw(N * p, seed, sb + _S_X, NORMAL, 1.0).reshape(N, p)
    for c in spec.bern_cols:
        if c < p:
            lib.gen_fill_col(X.ctypes.data, N, p, c, seed, sb + _S_BERN + c, BERNOULLI, spec.bern_p)
    Y = draw(N * K * f, seed, sb + _S_Y, NORMAL, 1.0).reshape(N, K, f)
    Z = draw(N * K * d, seed, sb + _S_Z, UNIFORM, 1.0).reshape(N, K, d)
    n_p = spec.n_params
    theta = draw(n_p, seed, sb + _S_COEF, NORMAL, spec.coef_sd)
    if spec.xi_sd is not None:
        xi = draw(K - 1, seed, sb + _S_XI, NORMAL, spec.xi_sd)
        theta[(np.arange(K - 1) * (p + 1))] = xi
    choice = np.empty(N, dtype=np.int32)
    lib.gen_choices(N, K, p, f, d, X.ctypes.data, Y.ctypes.data, Z.ctypes.data, theta.ctypes.data,
                    seed, sb + _S_CHOICE, choice.ctypes.data)
    counts = np.bincount(choice, minlength=K)
    if require_all_classes and counts.min() < 1:
        # an empty class puts the MLE at -inf; never generate one.
        raise ValueError(f"{spec.name} seed {seed}: empty class (counts.min()=0)")
    return Problem(spec, seed, X, Y, Z, choice, theta, counts)


def custom(N: int, K: int, p: int, f: int = 0, d: int = 0, seed: int = 0, coef_sd: float = 0.5,
           xi_sd: float | None = None, name: str = "custom", require_all_classes: bool = True) -> Problem:
    """A small instance with the c1 distributions at arbitrary shape (tests)."""
    sb = (hash((N, K, p, f, d)) & 0xFFFF) << 24 | 7 << 40
    return make(Spec(name, N, K, p, f, d, coef_sd=coef_sd, xi_sd=xi_sd, stream_base=sb), seed,
                require_all_classes=require_all_classes)


def perturbed_theta(prob: Problem, sd: float = 0.05) -> np.ndarray:
    """theta_true + N(0, sd) (SURVEY.md §8(c) parity points)."""
    return prob.theta_true + draw(prob.theta_true.size, prob.seed, prob.spec.stream_base + _S_PERTURB, NORMAL, sd)


def random_start(prob: Problem, sd: float = 0.1) -> np.ndarray:
    return draw(prob.theta_true.size, prob.seed, prob.spec.stream_base + _S_START, NORMAL, sd)
