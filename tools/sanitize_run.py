#!/usr/bin/env python
"""Small end-to-end run for compute-sanitizer: eval (l, g, H) + fit on c1 and a ragged shape."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402


def main():
    import torch
    import paper_1404_3177_b200 as M
    for prob in (datagen.make("c1"), datagen.custom(77, 5, 3, 2, 2, seed=9), datagen.custom(330, 33, 2, 0, 1, seed=4, require_all_classes=False)):
        s = prob.spec
        dev = torch.device("cuda", 0)
        dp = M.problem(torch.from_numpy(prob.X).to(dev), torch.from_numpy(prob.Y).to(dev) if s.f else None,
                       torch.from_numpy(prob.Z).to(dev) if s.d else None,
                       torch.from_numpy(prob.choice.astype(np.int32)).to(dev), K=s.K)
        ll, g, H = M.mnl_eval(dp, torch.from_numpy(prob.theta_true).to(dev), grad=True, hess=True)
        f = M.mnl_newton_fit(dp, tol=1e-8)
        torch.cuda.synchronize()
        print(s.name, s.N, s.K, ll.item(), f.iters, f.status, flush=True)


if __name__ == "__main__":
    main()
