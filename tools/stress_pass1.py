#!/usr/bin/env python
"""Stress sweep of the pass-1 kernels: random shapes through the team mapping / the two-group X-only
kernel (forced) against k_eval.cu's paths (MNL_NO_YZW, MNL_NO_XG): loglik, gradient, H v, and the
whole Hessian (i.e. the probability rows and ybar) for the smaller n_p.
python tools/stress_pass1.py [count] [seed]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_1404_3177_b200 as M  # noqa: E402


def ev(dp, th, v, hess, env):
    for k in ("MNL_FORCE_YZW", "MNL_FORCE_XG", "MNL_NO_YZW", "MNL_NO_XG"):
        os.environ.pop(k, None)
    for k in env:
        os.environ[k] = "1"
    try:
        l, g, H = M.mnl_eval(dp, th, grad=True, hess=hess)
        hv = M.mnl_hessvec(dp, th, v)
        torch.cuda.synchronize()
        return l.item(), g.cpu().numpy(), (H.cpu().numpy() if hess else None), hv.cpu().numpy()
    finally:
        for k in env:
            os.environ.pop(k, None)


def main():
    count = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
    worst = 0.0
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    for it in range(count):
        xonly = rng.random() < 0.35
        if xonly:
            K, p, f, d = int(rng.integers(2, 129)), int(rng.integers(0, 64)), 0, 0
        else:
            K, p = int(rng.integers(2, 65)), int(rng.integers(0, 33))
            f, d = 2 * int(rng.integers(0, 9)), int(rng.integers(0, 9))
            if f + d == 0:
                f = 2
            if (K * d) % 2:
                K += 1 if K < 64 else -1
        N = int(rng.choice([8, 9, 31, 64, 100, 257, 1000, 4097, 12000, 40001]))
        if (N % 8) and ((N - 8) * p) % 2:
            N += 1
        prob = datagen.custom(N, K, p, f, d, seed=int(rng.integers(1 << 30)), coef_sd=0.3, require_all_classes=False)
        dp = M.problem(t(prob.X) if p else None, t(prob.Y) if f else None, t(prob.Z) if d else None,
                       t(prob.choice.astype(np.int32)), K=K)
        th = t(datagen.perturbed_theta(prob, 0.2))
        n_p = prob.spec.n_params
        v = t(rng.standard_normal(n_p))
        hess = n_p <= 700
        a = ev(dp, th, v, hess, ["MNL_FORCE_YZW", "MNL_FORCE_XG"])
        b = ev(dp, th, v, hess, ["MNL_NO_YZW", "MNL_NO_XG"])
        errs = [abs(a[0] - b[0]) / abs(b[0]), np.linalg.norm(a[1] - b[1]) / np.linalg.norm(b[1]),
                np.linalg.norm(a[3] - b[3]) / np.linalg.norm(b[3])]
        if hess:
            errs.append(np.linalg.norm(a[2] - b[2]) / np.linalg.norm(b[2]))
        worst = max(worst, max(errs))
        if max(errs) > 1e-11:
            print("MISMATCH", (N, K, p, f, d), errs, flush=True)
            sys.exit(1)
    print(f"{count} shapes, worst relative difference {worst:.2e}")


if __name__ == "__main__":
    main()
