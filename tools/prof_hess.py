#!/usr/bin/env python
"""Small driver for ncu: `reps` evaluations (loglik + gradient + Hessian) of one config through the C ABI."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402


def main():
    import torch
    import paper_1404_3177_b200 as M
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    mode = sys.argv[3] if len(sys.argv) > 3 else "eval"
    prob = datagen.make(cfg)
    s = prob.spec
    dev = torch.device("cuda", 0)
    dp = M.problem(torch.from_numpy(prob.X).to(dev), torch.from_numpy(prob.Y).to(dev) if s.f else None,
                   torch.from_numpy(prob.Z).to(dev) if s.d else None,
                   torch.from_numpy(prob.choice.astype(np.int32)).to(dev), K=s.K)
    th = torch.from_numpy(prob.theta_true).to(dev)
    for r in range(reps):
        if mode in ("fit", "fitcg"):
            f = M.mnl_newton_fit(dp, tol=1e-6, method="cg" if mode == "fitcg" else "newton")
            print(cfg, mode, f.iters, f.loglik, f.stats, flush=True)
        elif mode == "se":
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            se = M.mnl_std_errors(dp, th)
            e1.record()
            torch.cuda.synchronize()
            print(cfg, "std_errors ms %.3f" % e0.elapsed_time(e1), "se[:3]", se[:3].tolist(), flush=True)
        elif mode == "hv":
            v = th.clone()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            M.mnl_eval(dp, th, grad=True, hess=False)
            e0.record()
            hv = M.mnl_hessvec(dp, th, v)
            e1.record()
            torch.cuda.synchronize()
            print(cfg, "hessvec ms %.3f" % e0.elapsed_time(e1), flush=True)
        else:
            ll, g, H = M.mnl_eval(dp, th, grad=True, hess=True)
            torch.cuda.synchronize()
            print(cfg, r, ll.item(), M.last_hessian_times(), M.last_launch_count(), flush=True)


if __name__ == "__main__":
    main()
