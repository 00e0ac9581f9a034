"""Data-parallel Newton-Raphson over individuals (NEXT item f3).

The log-likelihood, gradient and Hessian are sums over individuals, so
each rank owns a contiguous slice of the individuals, evaluates its partial (l_r, g_r, H_r) with the
single-GPU kernels, and ONE all-reduce (sum) of [l, g, packed upper triangle of H] per iteration
forms (l, g, H) on every rank.  Every
rank then factors the same -H and takes the same step (all-reduce results are identical on all
ranks), so the iterates stay bitwise identical without broadcasting the coefficients.  Each
line-search trial needs one scalar all-reduce.

The driver is written against three callables so the host logic is testable on CPU with gloo:
  evaluate(theta, want_grad, want_hess) -> (l, g, H)   local sums (tensors; g, H may be None)
  all_reduce(tensor)                                    in-place sum over ranks
  solve(A, g) -> (status, delta)                        delta = A^{-1} g for the SPD A = -H
The step control is the same as mnl_newton_fit (include/mnl.h, readings R7-R11).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

MNL_OK, MNL_ERR_ARG, MNL_ERR_CUDA, MNL_ERR_NOT_SPD, MNL_ERR_LINESEARCH, MNL_ERR_NONFINITE, MNL_MAXITER = range(7)
MAX_HALVINGS = 30
TAU_REL = 1e-12


def shard_range(N: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced slice [lo, hi) of the N individuals for `rank`."""
    base, rem = divmod(N, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


@dataclass
class DPFit:
    status: int = MNL_OK
    iters: int = 0
    loglik: float = float("nan")
    grad_norm: float = float("nan")
    coef: object = None
    halvings: list = field(default_factory=list)


def torch_packer():
    """(pack, unpack) of the upper triangle with torch indexing (host-logic tests on CPU)."""
    import torch

    cache = {}

    def idx(n, dev):
        if (n, dev) not in cache:
            cache[(n, dev)] = torch.triu_indices(n, n, device=dev)
        return cache[(n, dev)]

    def pack(H):
        iu = idx(H.shape[0], H.device)
        return H[iu[0], iu[1]]

    def unpack(v, n):
        iu = idx(n, v.device)
        H = torch.empty(n, n, dtype=v.dtype, device=v.device)
        H[iu[0], iu[1]] = v
        H[iu[1], iu[0]] = v
        return H

    return pack, unpack


def newton_fit_dp(evaluate, all_reduce, solve, theta0, tol: float = 1e-6, max_iter: int = 50,
                  packer=None) -> DPFit:
    """Newton-Raphson with step halving on data sharded over ranks (identical on every rank).
    With `packer` = (pack, unpack) the Hessian evaluation exchanges ONE buffer [l, g, upper
    triangle of H] (n_p + 1 + n_p (n_p + 1) / 2 doubles, half the bytes of the full matrix);
    without it, [l, g] and the full H in two all-reduces."""
    import torch

    theta = theta0.clone()
    fit = DPFit()

    def reduced(th, want_hess):
        l, g, H = evaluate(th, True, want_hess)
        n = g.shape[0]
        if H is not None and packer is not None:
            buf = torch.cat([l.reshape(1).to(g.dtype), g, packer[0](H)])
            all_reduce(buf)
            return float(buf[0].item()), buf[1:n + 1], packer[1](buf[n + 1:], n)
        lg = torch.cat([l.reshape(1).to(g.dtype), g])
        all_reduce(lg)
        if H is not None:
            all_reduce(H)
        return float(lg[0].item()), lg[1:], H

    l, g, _ = reduced(theta, False)
    while True:
        if not math.isfinite(l):
            fit.status = MNL_ERR_NONFINITE
            break
        gnorm = float(torch.sqrt(torch.sum(g * g)).item())
        fit.loglik, fit.grad_norm = l, gnorm
        if gnorm < tol:
            fit.status = MNL_OK
            break
        if fit.iters == max_iter:
            fit.status = MNL_MAXITER
            break
        _, _, H = reduced(theta, True)   # the Hessian of the summed problem at theta
        status, delta = solve(-H, g)
        if status != MNL_OK:
            fit.status = status
            break
        tau = TAU_REL * max(1.0, abs(l))
        accepted = False
        for j in range(MAX_HALVINGS + 1):
            trial = theta + torch.ldexp(delta, torch.tensor(-j, dtype=torch.int32, device=delta.device))
            lj, gj, _ = reduced(trial, False)
            if math.isfinite(lj) and lj >= l - tau:
                accepted = True
                break
        if not accepted:
            fit.status = MNL_ERR_LINESEARCH
            break
        fit.halvings.append(j)
        theta, l, g = trial, lj, gj
        fit.iters += 1
    fit.coef = theta
    return fit


def cuda_evaluator(prob):
    """evaluate() over this rank's device-resident slice, through the C ABI (mnl_eval)."""
    from . import mnl_eval

    def evaluate(theta, want_grad, want_hess):
        return mnl_eval(prob, theta, grad=True, hess=want_hess)

    return evaluate


def cuda_packer():
    """(pack, unpack) with the library's kernels (mnl_sym_pack / mnl_sym_unpack)."""
    from . import mnl_sym_pack, mnl_sym_unpack

    def unpack(v, n):
        return mnl_sym_unpack(v.contiguous(), n)

    return (lambda H: mnl_sym_pack(H.contiguous())), unpack


def cuda_solver():
    """solve() with the library's Cholesky factor and triangular solves (mnl_cholesky[_solve])."""
    from . import MNL_OK as OK, mnl_cholesky, mnl_cholesky_solve

    def solve(A, g):
        A = A.contiguous()
        rc = mnl_cholesky(A)
        if rc != OK:
            return rc, None
        return OK, mnl_cholesky_solve(A, g.contiguous())

    return solve
