"""Data-parallel Newton-Raphson on CPU with gloo, world size 2.

The driver is the library's own (csrc/nr_driver.h, built over host callbacks as libnrhost.so): each
rank evaluates its slice of the individuals with the oracle and exchanges exactly what the device
path exchanges -- [l, bad-choice flag, g] after every evaluation and the packed upper triangle of
-H after every Hessian (include/mnl.h, mnl_newton_fit_dp) -- through one gloo all-reduce each. The
fit must equal the single-process oracle fit: same iterations and halvings, coefficients 1e-9."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import datagen
import oracle as O
from paper_1404_3177_b200 import distributed as DP

OK, ERR_ARG, ERR_NOT_SPD = 0, 1, 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def pack_upper(A):
    iu = np.triu_indices(A.shape[0])
    return A[iu]


def unpack_upper(v, n):
    A = np.empty((n, n))
    iu = np.triu_indices(n)
    A[iu] = v
    A[(iu[1], iu[0])] = v
    return A


class ShardOps:
    """The exchange of mnl_newton_fit_dp over gloo, with the oracle as this rank's evaluator."""

    def __init__(self, D, theta0, nan_first_trial_at_iter=None, bad_choice=False):
        self.D, self.theta, self.n = D, np.array(theta0, dtype=np.float64), D.n_p
        self.g = self.g_trial = self.trial = self.delta = None
        self.iter = 0
        self.nan_at = nan_first_trial_at_iter
        self.bad = 1.0 if bad_choice else 0.0

    def _eval(self, theta, poison=False):
        l, g, _ = O.mnl_eval(self.D, theta, want_grad=True, want_hess=False)
        if poison:
            l = float("nan")   # this shard overflowed: the summed l is non-finite on every rank
        buf = torch.tensor(np.concatenate([[l, self.bad], g]), dtype=torch.float64)
        dist.all_reduce(buf)
        b = buf.numpy()
        if b[1] != 0.0:
            return ERR_ARG, b[0], 0.0, b[2:]
        return OK, float(b[0]), float(np.sum(b[2:] ** 2)), b[2:].copy()

    def eval_theta(self):
        rc, l, g2, self.g = self._eval(self.theta)
        return rc, l, g2

    def direction(self):
        H = O.hessian(self.D, self.theta)
        buf = torch.from_numpy(pack_upper(-H).copy())
        dist.all_reduce(buf)
        A = unpack_upper(buf.numpy(), self.n)
        try:
            L = np.linalg.cholesky(A)
        except np.linalg.LinAlgError:
            return OK, True
        self.delta = np.linalg.solve(L.T, np.linalg.solve(L, self.g))
        return OK, False

    def eval_trial(self, j):
        self.trial = self.theta + np.ldexp(self.delta, -j)
        poison = self.nan_at is not None and self.iter == self.nan_at and j == 0
        rc, l, g2, self.g_trial = self._eval(self.trial, poison)
        return rc, l, g2

    def accept(self):
        self.theta, self.g = self.trial, self.g_trial
        self.iter += 1


def _worker(rank, world, port, shape, start_scale, out_path, nan_rank=None, bad_rank=None):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    N, K, p, f, d = shape
    prob = datagen.custom(N, K, p, f, d, seed=51, coef_sd=0.5)
    lo, hi = DP.shard_range(N, world, rank)
    D = O.Data(prob.X[lo:hi], prob.Y[lo:hi], prob.Z[lo:hi], prob.choice[lo:hi], K)
    ops = ShardOps(D, np.full(prob.spec.n_params, start_scale),
                   nan_first_trial_at_iter=0 if rank == nan_rank else None, bad_choice=rank == bad_rank)
    rep = DP.run_host_driver(ops.eval_theta, ops.direction, ops.eval_trial, ops.accept, gtol=1e-8)
    coef = torch.from_numpy(ops.theta)
    coefs = [torch.zeros_like(coef) for _ in range(world)]
    dist.all_gather(coefs, coef)
    if rank == 0:
        np.savez(out_path, coef=ops.theta, iters=rep["iters"], status=rep["rc"],
                 halvings=np.array(rep["halvings_per_iter"]), same=all(torch.equal(c, coefs[0]) for c in coefs),
                 min_margin=rep["min_margin"], lpi=np.array(rep["loglik_per_iter"]),
                 gpi=np.array(rep["grad_norm_per_iter"]))
    dist.destroy_process_group()


def _run(tmp_path, shape, start, **kw):
    out = str(tmp_path / "fit.npz")
    mp.spawn(_worker, args=(2, _free_port(), shape, start, out, kw.get("nan_rank"), kw.get("bad_rank")),
             nprocs=2, join=True)
    return np.load(out)


def _oracle_fit(shape, start):
    N, K, p, f, d = shape
    prob = datagen.custom(N, K, p, f, d, seed=51, coef_sd=0.5)
    return O.newton_fit(O.Data(prob.X, prob.Y, prob.Z, prob.choice, K), coef0=np.full(prob.spec.n_params, start),
                        tol=1e-8)


@pytest.mark.parametrize("shape,start", [((301, 4, 2, 1, 1), 0.0), ((250, 3, 3, 0, 2), 2.0)])
def test_data_parallel_fit_equals_single_process_oracle(tmp_path, shape, start):
    r = _run(tmp_path, shape, start)
    ref = _oracle_fit(shape, start)
    assert int(r["status"]) == OK and ref.status == O.MNL_OK
    assert bool(r["same"])                       # every rank holds the same iterate
    assert int(r["iters"]) == ref.iters
    assert list(r["halvings"]) == [h["halvings"] for h in ref.history]
    assert np.linalg.norm(r["coef"] - ref.coef) <= 1e-9 * np.linalg.norm(ref.coef)
    assert float(r["min_margin"]) > 1e-13       # R7 audit of the driver's decisions
    # the per-iteration report (l, ||g|| at the iterate starting each iteration) vs the oracle's log
    assert np.allclose(r["lpi"], [h["l"] for h in ref.history], rtol=1e-12, atol=0)
    assert np.allclose(r["gpi"], [h["gnorm"] for h in ref.history], rtol=1e-8, atol=1e-12)


def test_data_parallel_nonfinite_shard_rejects_on_every_rank(tmp_path):
    """A trial whose loglik is non-finite on ONE shard: the summed l is non-finite on every rank, so
    every rank rejects it and halves (no rank raises, none blocks in the collective)."""
    shape = (301, 4, 2, 1, 1)
    r = _run(tmp_path, shape, 0.0, nan_rank=1)
    ref = _oracle_fit(shape, 0.0)
    assert int(r["status"]) == OK and bool(r["same"])
    assert int(r["halvings"][0]) >= 1
    assert np.linalg.norm(r["coef"] - ref.coef) <= 1e-8 * np.linalg.norm(ref.coef)   # the unique MLE


def test_data_parallel_bad_choice_on_one_rank_is_an_error_everywhere(tmp_path):
    r = _run(tmp_path, (120, 3, 2, 0, 0), 0.0, bad_rank=1)
    assert int(r["status"]) == ERR_ARG and bool(r["same"])


def test_host_driver_single_process_matches_oracle_fit():
    """world size 1: the library's driver over the oracle reproduces the oracle's own Newton loop."""
    prob = datagen.custom(400, 5, 3, 2, 1, seed=14, coef_sd=0.5)
    D = O.Data(prob.X, prob.Y, prob.Z, prob.choice, prob.spec.K)
    st = {"theta": np.zeros(D.n_p)}

    def ev(theta):
        l, g, _ = O.mnl_eval(D, theta, want_hess=False)
        return l, g

    def eval_theta():
        st["l"], st["g"] = ev(st["theta"])
        return OK, st["l"], float(st["g"] @ st["g"])

    def direction():
        H = O.hessian(D, st["theta"])
        st["delta"] = np.linalg.solve(-H, st["g"])
        return OK, False

    def eval_trial(j):
        st["trial"] = st["theta"] + math.ldexp(1.0, -j) * st["delta"]
        st["lt"], st["gt"] = ev(st["trial"])
        return OK, st["lt"], float(st["gt"] @ st["gt"])

    def accept():
        st["theta"], st["g"] = st["trial"], st["gt"]

    rep = DP.run_host_driver(eval_theta, direction, eval_trial, accept, gtol=1e-9)
    ref = O.newton_fit(D, tol=1e-9)
    assert rep["rc"] == OK and rep["iters"] == ref.iters and rep["stop_reason"] == 1
    assert np.linalg.norm(st["theta"] - ref.coef) <= 1e-10 * np.linalg.norm(ref.coef)
    # max_iter and ftol through the same driver
    st["theta"] = np.zeros(D.n_p)
    rep1 = DP.run_host_driver(eval_theta, direction, eval_trial, accept, gtol=1e-12, max_iter=2)
    assert rep1["rc"] == 6 and rep1["iters"] == 2 and rep1["stop_reason"] == 3


def test_shard_range_partitions():
    for N in (1, 7, 100, 1001):
        for world in (1, 2, 3, 8):
            parts = [DP.shard_range(N, world, r) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == N
            assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1


def test_packed_exchange_layout_round_trip():
    # the layout of mnl_sym_pack / the packed -H of mnl_newton_fit_dp: row i holds columns i..n-1
    A = np.random.default_rng(1).standard_normal((7, 7))
    S = A + A.T
    v = pack_upper(S)
    assert v.size == 28 and np.array_equal(v[:7], S[0]) and np.array_equal(v[7:13], S[1, 1:])
    assert np.array_equal(unpack_upper(v, 7), S)
