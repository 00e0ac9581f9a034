#!/usr/bin/env python
"""Stress the Newton-step solve (mnl_spd_solve) and mnl_cholesky on random SPD matrices of random n
(seeded), against LAPACK: python tools/stress_spd.py COUNT SEED NMAX"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_1404_3177_b200 as M
    count, seed, nmax = (int(a) for a in sys.argv[1:4]) if len(sys.argv) > 3 else (200, 1, 3000)
    rng = np.random.default_rng(seed)
    worst = 0.0
    for t in range(count):
        n = int(rng.integers(1, nmax + 1))
        B = rng.standard_normal((n, n + int(rng.integers(1, 20))))
        A = B @ B.T / n + np.eye(n) * float(rng.choice([0.01, 0.1, 1.0]))
        b = rng.standard_normal(n)
        x_ref = np.linalg.solve(A, b)
        Ad = torch.from_numpy(A).cuda()
        x = M.mnl_spd_solve(Ad, torch.from_numpy(b).cuda()).cpu().numpy()
        err = np.linalg.norm(x - x_ref) / np.linalg.norm(x_ref)
        assert np.array_equal(Ad.cpu().numpy(), A), n
        if t % 4 == 0:
            assert M.mnl_cholesky(Ad) == M.MNL_OK
            L = np.tril(Ad.cpu().numpy())
            Lr = np.linalg.cholesky(A)
            el = np.max(np.abs(L - Lr)) / np.max(np.abs(Lr))
            assert el <= 1e-10, (n, el)
        worst = max(worst, err)
        assert err <= 1e-8, (n, err)
    print(f"{count} solves, n <= {nmax}: worst relative error {worst:.2e}")


if __name__ == "__main__":
    main()
