"""Plain fp64 CPU oracle of the mnlogit Newton-Raphson hot path.

TEST INFRASTRUCTURE ONLY.  Importable from tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs; never from the product path.
Shares no code with paper_1404_3177_b200/ (the CUDA path).

Citations: `P:n` = /root/reference/PAPER.md line n (not present on the GPU box;
the citations are for the reader).  Letters follow the ABI,
which swaps the paper's Y and Z:

  ABI X[N,p]   <-> paper X      (individual-specific data, coefs beta_k, k=1..K-1,
                                 intercept xi_k = first entry of each chunk)
  ABI Z[N,K,d] <-> paper Y_k    (alternative-varying data, alternative-specific
                                 coefs alpha_k for k = 0..K-1 incl. the base)
  ABI Y[N,K,f] <-> paper Z_k    (alternative-varying data, one generic coef gamma,
                                 differenced against the base)

theta layout (Eq. "theta vec"):
  [beta_1 | ... | beta_{K-1} | alpha_0 | ... | alpha_{K-1} | gamma],
  beta_k = [xi_k, beta_k1 .. beta_kp].

WHAT IS COMPUTED.  The paper's block method (Eq. "hessian block")
reaches exactly (up to rounding order) the plain definition of the
log-likelihood derivatives, so this oracle is that definition written out:

  V_ik  = normalized utility, Eq. "normalized utility"; V_i0 = 0
  P_ik  = softmax with base, Eqs. "probability"/"base probability"
  l     = sum_i [ -log(1 + sum_{k>=1} e^{V_ik}) + sum_{k>=1} V_ik I(y_i=k) ]
  J_i   = K x n_p Jacobian, J_i[k, r] = dV_ik / dtheta_r  (row 0 is zero)
  g     = sum_i J_i^T (e_{y_i} - p_i)                                       (App. A)
  H     = -sum_i J_i^T (diag p_i - p_i p_i^T) J_i                          ("old Hessian formula",
                                                                            App. B)
        = -[ sum_k J_(k)^T D(P_k) J_(k) - U^T U ],  U = sum_k D(P_k) J_(k)
          (the same sum with the matrix product expanded; J_(k) = the N x n_p
          matrix whose row i is row k of J_i; numpy matmul is the library step)

and the Newton iteration is Eq. "NR update" step by step, with the
readings of DESIGN.md §Readings (R7 roundoff floor, R8 30 halvings, R9 start 0,
R10 Euclidean gtol, R11 stop-before-Hessian).  The Cholesky factorisation of -H
is a library routine (numpy.linalg.cholesky / LAPACK).

Pins (tests/test_oracle_pins.py): closed forms at theta=0 (P:874 printed value),
K=2 textbook logistic regression, central finite differences, the
textbook dense X~^T W~ X~ of P:383-403, the paper's block formula
written independently, intercept-only closed-form MLE, invariants; standard
errors against the intercept-only closed-form variance (1/N)(1/p_k + 1/p_0).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
from scipy.linalg import solve_triangular

KIND = "numpy"
MNL_OK, MNL_ERR_ARG, MNL_ERR_CUDA, MNL_ERR_NOT_SPD, MNL_ERR_LINESEARCH, MNL_ERR_NONFINITE, MNL_MAXITER = range(7)
MAX_HALVINGS = 30          # R8
TAU_REL = 1e-12            # R7: accept l_j >= l - TAU_REL * max(1, |l|)


def num_params(K: int, p: int, f: int, d: int) -> int:
    """n_p = (K-1)(p+1) + K d + f  ((K-1) beta/xi sets, K alt-specific sets, 1 generic)."""
    return (K - 1) * (p + 1) + K * d + f


class Data:
    """One problem: X[N,p], Y[N,K,f], Z[N,K,d], choice[N] (0 = base alternative)."""

    def __init__(self, X, Y, Z, choice, K: int):
        X = np.asarray(X, dtype=np.float64)
        self.N = N = X.shape[0]
        self.K = K
        self.X = np.ascontiguousarray(X.reshape(N, -1))
        self.p = self.X.shape[1]
        self.Y = np.ascontiguousarray(np.asarray(Y, dtype=np.float64).reshape(N, K, -1)) if np.size(Y) else np.zeros((N, K, 0))
        self.Z = np.ascontiguousarray(np.asarray(Z, dtype=np.float64).reshape(N, K, -1)) if np.size(Z) else np.zeros((N, K, 0))
        self.f = self.Y.shape[2]
        self.d = self.Z.shape[2]
        self.choice = np.asarray(choice, dtype=np.int64).reshape(N)

    @property
    def n_p(self) -> int:
        return num_params(self.K, self.p, self.f, self.d)

    @property
    def off_alpha(self) -> int:
        return (self.K - 1) * (self.p + 1)

    @property
    def off_gamma(self) -> int:
        return self.off_alpha + self.K * self.d


def make_data(X, Y, Z, choice, K: int) -> Data:
    return Data(X, Y, Z, choice, K)


# ---------------------------------------------------------------------------
# Model: utilities and probabilities
# ---------------------------------------------------------------------------

def utilities(D: Data, theta: np.ndarray) -> np.ndarray:
    """V[N, K], Eq. "normalized utility" in ABI letters, V[:,0] = 0:
    V_ik = xi_k + x_i.beta_k + z_ik.alpha_k - z_i0.alpha_0 + (y_ik - y_i0).gamma,  k >= 1.
    (The generic data are differenced against the base.)"""
    N, K, p, f, d = D.N, D.K, D.p, D.f, D.d
    q = p + 1
    theta = np.asarray(theta, dtype=np.float64)
    V = np.zeros((N, K))
    alpha = theta[D.off_alpha:D.off_gamma].reshape(K, d)
    gamma = theta[D.off_gamma:]
    for k in range(1, K):
        b = theta[(k - 1) * q:k * q]
        v = b[0] + D.X @ b[1:]
        if d:
            v = v + D.Z[:, k, :] @ alpha[k] - D.Z[:, 0, :] @ alpha[0]
        if f:
            v = v + (D.Y[:, k, :] - D.Y[:, 0, :]) @ gamma
        V[:, k] = v
    return V


def probabilities(V: np.ndarray) -> np.ndarray:
    """P_ik = P_i0 e^{V_ik}, P_i0 = 1/(1 + sum_{k>=1} e^{V_ik}),
    evaluated with the overflow-safe shift m_i = max(0, max_k V_ik) (R12; V_i0 = 0
    is column 0 of V so the shift is the row max)."""
    m = V.max(axis=1, keepdims=True)
    E = np.exp(V - m)
    return E / E.sum(axis=1, keepdims=True)


def loglik_terms(V: np.ndarray, choice: np.ndarray) -> np.ndarray:
    """Per-individual terms of Eq. "log-lik function":
    -log(1 + sum_{k>=1} e^{V_ik}) + sum_{k>=1} V_ik I(y_i = k), with the same shift."""
    m = V.max(axis=1)
    lse = m + np.log(np.exp(V - m[:, None]).sum(axis=1))
    return V[np.arange(V.shape[0]), choice] - lse


def loglik(D: Data, theta) -> float:
    """l(theta); the sum over individuals is exactly rounded (math.fsum)."""
    return math.fsum(loglik_terms(utilities(D, theta), D.choice))


# ---------------------------------------------------------------------------
# The Jacobian J_i[k, r] = dV_ik / dtheta_r, column by column
# ---------------------------------------------------------------------------

def jac_column(D: Data, r: int):
    """Column r of every J_i, as (ks, vals): J_i[k, r] = vals[i, j] for k = ks[j], 0 elsewhere.

    From Eq. "normalized utility" (ABI letters):
      r in beta_k  (entry a of chunk k):  dV_ik/dtheta_r = x~_ia (x~_i0 = 1, the intercept P:340); only row k
      r in alpha_k, k >= 1 (entry c):      z_ikc; only row k
      r in alpha_0 (entry c):              -z_i0c in every row k >= 1
      r in gamma (entry e):                y_ike - y_i0e in every row k >= 1
    """
    N, K, p, d = D.N, D.K, D.p, D.d
    q = p + 1
    if r < D.off_alpha:
        k, a = r // q + 1, r % q
        col = np.ones(N) if a == 0 else D.X[:, a - 1]
        return [k], col[:, None]
    if r < D.off_gamma:
        k, c = divmod(r - D.off_alpha, d)
        if k >= 1:
            return [k], D.Z[:, k, c][:, None]
        return list(range(1, K)), np.repeat(-D.Z[:, 0, c][:, None], K - 1, axis=1)
    e = r - D.off_gamma
    return list(range(1, K)), D.Y[:, 1:, e] - D.Y[:, 0, e][:, None]


def jac_row_support(D: Data, k: int) -> list[int]:
    """Columns r where row k (k >= 1) of J_i can be nonzero: beta_k, alpha_k, alpha_0, gamma."""
    q = D.p + 1
    cols = list(range((k - 1) * q, k * q))
    cols += list(range(D.off_alpha + k * D.d, D.off_alpha + (k + 1) * D.d))
    cols += list(range(D.off_alpha, D.off_alpha + D.d))
    cols += list(range(D.off_gamma, D.n_p))
    return cols


def jac_row_block(D: Data, k: int, cols: list[int], cache: dict | None = None) -> np.ndarray:
    """J_(k)[:, cols]: the N x |cols| matrix of J_i[k, c] (columns from jac_column, optionally cached)."""
    out = np.zeros((D.N, len(cols)))
    for j, c in enumerate(cols):
        ks, vals = cache[c] if cache is not None and c in cache else jac_column(D, c)
        if k in ks:
            out[:, j] = vals[:, ks.index(k)]
    return out


# ---------------------------------------------------------------------------
# Gradient and Hessian (plain definition)
# ---------------------------------------------------------------------------

def gradient(D: Data, theta, P: np.ndarray | None = None) -> np.ndarray:
    """g = sum_i J_i^T (e_{y_i} - p_i)   (App. A)."""
    if P is None:
        P = probabilities(utilities(D, theta))
    R = -P.copy()
    R[np.arange(D.N), D.choice] += 1.0
    g = np.empty(D.n_p)
    for r in range(D.n_p):
        ks, vals = jac_column(D, r)
        g[r] = np.sum(vals * R[:, ks])
    return g


def U_column(D: Data, P: np.ndarray, r: int) -> np.ndarray:
    """U[:, r] = sum_k P_ik J_i[k, r]  (= (J_i^T p_i)_r)."""
    ks, vals = jac_column(D, r)
    return np.sum(vals * P[:, ks], axis=1)


def hessian(D: Data, theta, P: np.ndarray | None = None) -> np.ndarray:
    """H = -sum_i J_i^T (diag p_i - p_i p_i^T) J_i   (App. B), expanded as
    H = -[ sum_k J_(k)^T D(P_k) J_(k) - U^T U ]; matmul is the library step.
    Memory: U is N x n_p doubles (c5: 2.8 GB); use hessian_entries() for c4."""
    if P is None:
        P = probabilities(utilities(D, theta))
    n_p = D.n_p
    U = np.empty((D.N, n_p))
    for r in range(n_p):
        U[:, r] = U_column(D, P, r)
    A = U.T @ U
    del U
    S = np.zeros((n_p, n_p))
    shared = {c: jac_column(D, c) for c in range(D.off_alpha, D.off_alpha + D.d)}   # alpha_0: every row
    shared.update({c: jac_column(D, c) for c in range(D.off_gamma, n_p)})          # gamma: every row
    for k in range(1, D.K):
        cols = jac_row_support(D, k)
        Jk = jac_row_block(D, k, cols, shared)
        S[np.ix_(cols, cols)] += Jk.T @ (P[:, k][:, None] * Jk)
    H = -(S - A)
    return 0.5 * (H + H.T)   # exact symmetry; both halves are the same sum up to rounding order


def hessian_entries(D: Data, theta, rows, cols, P: np.ndarray | None = None) -> np.ndarray:
    """H[r, c] for the listed pairs, each straight from the definition
    H_rc = -sum_i [ sum_k p_ik J_i[k,r] J_i[k,c] - (sum_k p_ik J_i[k,r])(sum_k p_ik J_i[k,c]) ],
    the k-sums running over each column's nonzero rows only (the other J entries are zero)."""
    if P is None:
        P = probabilities(utilities(D, theta))
    out = np.empty(len(rows))
    for t, (r, c) in enumerate(zip(rows, cols)):
        kr, vr = jac_column(D, int(r))
        kc, vc = jac_column(D, int(c))
        ur = np.sum(vr * P[:, kr], axis=1)
        uc = np.sum(vc * P[:, kc], axis=1)
        common = sorted(set(kr) & set(kc))
        diag = np.zeros(D.N)
        for k in common:
            diag += P[:, k] * vr[:, kr.index(k)] * vc[:, kc.index(k)]
        out[t] = -np.sum(diag - ur * uc)
    return out


def hessvec(D: Data, theta, v, P: np.ndarray | None = None) -> np.ndarray:
    """H v = -sum_i J_i^T (diag p_i - p_i p_i^T) (J_i v)  (applied to v; the product form of
    the paper's Hessian-free extension): s_i = J_i v, w_ik = p_ik (s_ik - p_i.s_i),
    (Hv)_r = -sum_i sum_k J_i[k, r] w_ik. Never forms H."""
    if P is None:
        P = probabilities(utilities(D, theta))
    v = np.asarray(v, dtype=np.float64)
    S = np.zeros((D.N, D.K))
    cols = [jac_column(D, r) for r in range(D.n_p)]
    for r, (ks, vals) in enumerate(cols):
        S[:, ks] += vals * v[r]
    W = P * (S - np.sum(P * S, axis=1, keepdims=True))
    out = np.empty(D.n_p)
    for r, (ks, vals) in enumerate(cols):
        out[r] = -np.sum(vals * W[:, ks])
    return out


def std_errors(D: Data, theta) -> np.ndarray:
    """se_j = sqrt([(-H)^{-1}]_jj) at theta: the square roots of the diagonal of the inverse observed
    information (the paper's estimation summary). numpy.linalg.inv is the library step."""
    H = hessian(D, theta)
    return np.sqrt(np.diag(np.linalg.inv(-H)))


def predict(D: Data, theta) -> np.ndarray:
    """P[N, K]: the choice probabilities of Eqs. "probability" / "base probability"."""
    return probabilities(utilities(D, np.asarray(theta, dtype=np.float64)))


def mnl_eval(D: Data, theta, want_grad=True, want_hess=True):
    """(loglik, grad, hess) at theta -- the oracle twin of the ABI's mnl_eval."""
    theta = np.asarray(theta, dtype=np.float64)
    V = utilities(D, theta)
    P = probabilities(V)
    l = math.fsum(loglik_terms(V, D.choice))
    g = gradient(D, theta, P) if want_grad else None
    H = hessian(D, theta, P) if want_hess else None
    return l, g, H


# ---------------------------------------------------------------------------
# Newton-Raphson with step halving (stopping P:219-220)
# ---------------------------------------------------------------------------

@dataclass
class FitLog:
    status: int = MNL_OK
    iters: int = 0
    loglik: float = float("nan")
    coef: np.ndarray | None = None
    history: list = field(default_factory=list)   # per iteration: dict(l, gnorm, halvings, margin)
    grad_norm: float = float("nan")
    stop_reason: int = 0       # 0 error, 1 gtol, 2 ftol, 3 maxiter (the ABI's mnl_stop_reason)
    delta_loglik: float = 0.0  # |l_t - l_(t-1)| of the last accepted update
    cg_iters: int = 0          # newton_cg_fit only


def newton_fit(D: Data, coef0=None, tol: float = 1e-6, max_iter: int = 50, hess_fn=None,
               ftol: float = 0.0, step_fn=None) -> FitLog:
    """theta_new = theta_old - H^{-1} dl/dtheta (Eq. "NR update"), with step halving
    until the log-likelihood is "not lower than" at theta_old (R7 floor tau). Stops at
    the first of the paper's conditions met: ||g||_2 < tol tested before
    forming H (R10, R11), |l_t - l_(t-1)| < ftol after an accepted update (ftol = 0: off), or
    iters == max_iter. step_fn(theta, P, g, l) -> (status, delta) replaces the Cholesky solve of
    (-H) delta = g (newton_cg_fit)."""
    theta = np.zeros(D.n_p) if coef0 is None else np.array(coef0, dtype=np.float64)
    log = FitLog()
    hess_fn = hess_fn or hessian
    ftol_met = False
    while True:
        V = utilities(D, theta)
        P = probabilities(V)
        l = math.fsum(loglik_terms(V, D.choice))
        if not np.isfinite(l):
            log.status = MNL_ERR_NONFINITE
            break
        g = gradient(D, theta, P)
        gnorm = float(np.sqrt(np.sum(g * g)))
        log.loglik, log.grad_norm = l, gnorm
        if gnorm < tol:
            log.status, log.stop_reason = MNL_OK, 1
            break
        if ftol_met:
            log.status, log.stop_reason = MNL_OK, 2
            break
        if log.iters == max_iter:
            log.status, log.stop_reason = MNL_MAXITER, 3
            break
        if step_fn is not None:
            status, delta = step_fn(theta, P, g, l)
            if status != MNL_OK:
                log.status = status
                break
        else:
            H = hess_fn(D, theta, P)
            try:
                L = np.linalg.cholesky(-H)
            except np.linalg.LinAlgError:
                log.status = MNL_ERR_NOT_SPD
                break
            delta = solve_triangular(L.T, solve_triangular(L, g, lower=True), lower=False)  # (-H) delta = g
        tau = TAU_REL * max(1.0, abs(l))
        accepted = False
        for j in range(MAX_HALVINGS + 1):
            theta_j = theta + np.ldexp(delta, -j)
            l_j = loglik(D, theta_j)
            if np.isfinite(l_j) and l_j >= l - tau:
                accepted = True
                break
        if not accepted:
            log.status = MNL_ERR_LINESEARCH
            break
        log.history.append(dict(l=l, gnorm=gnorm, halvings=j, l_new=l_j,
                                margin=(l_j - l) / max(1.0, abs(l))))
        log.delta_loglik = abs(l_j - l)
        ftol_met = ftol > 0.0 and log.delta_loglik < ftol
        theta = theta_j
        log.iters += 1
    log.coef = theta
    return log


def newton_cg_fit(D: Data, coef0=None, tol: float = 1e-6, max_iter: int = 50, ftol: float = 0.0,
                  cg_max_iter: int = 0, cg_rtol: float = 0.0) -> FitLog:
    """Truncated Newton (the paper's Hessian-free extension): the Newton system
    (-H) delta = g is solved approximately by conjugate gradients from delta = 0 using only products
    H p (hessvec), stopping at ||r|| <= eta ||g||, eta = cg_rtol or min(0.5, sqrt(||g||))
    (Eisenstat-Walker forcing), or after cg_max_iter (0: n_p) iterations, or at non-positive
    curvature (an error before the first step); then the same line search and stopping set as
    newton_fit."""
    counter = {"cg": 0}

    def step(theta, P, g, l):
        gn = float(np.sqrt(g @ g))
        eta = cg_rtol if cg_rtol > 0 else min(0.5, math.sqrt(gn))
        cmax = cg_max_iter if cg_max_iter > 0 else D.n_p
        delta = np.zeros(D.n_p)
        r = g.copy()
        pv = g.copy()
        rr = float(r @ r)
        for it in range(cmax):
            ap = -hessvec(D, theta, pv, P)
            pap = float(pv @ ap)
            if not (pap > 0 and np.isfinite(pap)):
                if it == 0:
                    return MNL_ERR_NOT_SPD, None
                break
            alpha = rr / pap
            delta = delta + alpha * pv
            r = r - alpha * ap
            rr_new = float(r @ r)
            counter["cg"] += 1
            if math.sqrt(rr_new) <= eta * gn:
                break
            pv = r + (rr_new / rr) * pv
            rr = rr_new
        return MNL_OK, delta

    log = newton_fit(D, coef0, tol, max_iter, ftol=ftol, step_fn=step)
    log.cg_iters = counter["cg"]
    return log
