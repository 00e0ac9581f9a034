"""Data-parallel Newton driver (paper_1404_3177_b200/distributed.py) on CPU with gloo, world size 2:
each rank evaluates its slice of the individuals with the oracle, one all-reduce per evaluation, and
the fit must equal the single-process oracle fit (same iterations and halvings, coefficients 1e-9)."""
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


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, shape, start_scale, out_path, packed=True):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    N, K, p, f, d = shape
    prob = datagen.custom(N, K, p, f, d, seed=51, coef_sd=0.5)
    lo, hi = DP.shard_range(N, world, rank)
    D = O.Data(prob.X[lo:hi], prob.Y[lo:hi], prob.Z[lo:hi], prob.choice[lo:hi], K)

    def evaluate(theta, want_grad, want_hess):
        l, g, H = O.mnl_eval(D, theta.numpy(), want_grad=True, want_hess=want_hess)
        return (torch.tensor(l, dtype=torch.float64), torch.from_numpy(g),
                torch.from_numpy(H) if want_hess else None)

    def all_reduce(t):
        dist.all_reduce(t)

    def solve(A, g):
        try:
            L = torch.linalg.cholesky(A)
        except RuntimeError:
            return DP.MNL_ERR_NOT_SPD, None
        return DP.MNL_OK, torch.cholesky_solve(g.reshape(-1, 1), L).reshape(-1)

    theta0 = torch.full((prob.spec.n_params,), start_scale, dtype=torch.float64)
    fit = DP.newton_fit_dp(evaluate, all_reduce, solve, theta0, tol=1e-8, packer=DP.torch_packer() if packed else None)
    coefs = [torch.zeros_like(fit.coef) for _ in range(world)]
    dist.all_gather(coefs, fit.coef)
    if rank == 0:
        np.savez(out_path, coef=fit.coef.numpy(), iters=fit.iters, status=fit.status,
                 halvings=np.array(fit.halvings), same=all(torch.equal(c, coefs[0]) for c in coefs))
    dist.destroy_process_group()


@pytest.mark.parametrize("shape,start,packed", [((301, 4, 2, 1, 1), 0.0, True), ((250, 3, 3, 0, 2), 2.0, True),
                                                ((301, 4, 2, 1, 1), 0.0, False)])
def test_data_parallel_fit_equals_single_process_oracle(tmp_path, shape, start, packed):
    out = str(tmp_path / "fit.npz")
    mp.spawn(_worker, args=(2, _free_port(), shape, start, out, packed), nprocs=2, join=True)
    r = np.load(out)
    N, K, p, f, d = shape
    prob = datagen.custom(N, K, p, f, d, seed=51, coef_sd=0.5)
    ref = O.newton_fit(O.Data(prob.X, prob.Y, prob.Z, prob.choice, K),
                       coef0=np.full(prob.spec.n_params, start), tol=1e-8)
    assert int(r["status"]) == DP.MNL_OK and ref.status == O.MNL_OK
    assert bool(r["same"])                       # every rank holds the same iterate
    assert int(r["iters"]) == ref.iters
    assert list(r["halvings"]) == [h["halvings"] for h in ref.history]
    assert np.linalg.norm(r["coef"] - ref.coef) <= 1e-9 * np.linalg.norm(ref.coef)


def test_shard_range_partitions():
    for N in (1, 7, 100, 1001):
        for world in (1, 2, 3, 8):
            parts = [DP.shard_range(N, world, r) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == N
            assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1


def test_torch_packer_round_trip():
    pack, unpack = DP.torch_packer()
    A = torch.randn(7, 7, dtype=torch.float64)
    S = A + A.T
    v = pack(S)
    assert v.numel() == 28 and torch.equal(v[:7], S[0]) and torch.equal(v[7:13], S[1, 1:])
    assert torch.equal(unpack(v, 7), S)
