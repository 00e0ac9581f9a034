#!/usr/bin/env python
"""Driver for pass-1 timing / ncu: `reps` evaluations (loglik + gradient, no Hessian) of one config
through the C ABI; prints the CUDA-event time of each call."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402


def main():
    import torch
    import paper_1404_3177_b200 as M
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    prob = datagen.make(cfg)
    s = prob.spec
    dev = torch.device("cuda", 0)
    dp = M.problem(torch.from_numpy(prob.X).to(dev), torch.from_numpy(prob.Y).to(dev) if s.f else None,
                   torch.from_numpy(prob.Z).to(dev) if s.d else None,
                   torch.from_numpy(prob.choice.astype(np.int32)).to(dev), K=s.K)
    th = torch.from_numpy(prob.theta_true).to(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts, tk = [], []
    for r in range(reps):
        e0.record()
        ll, g, _ = M.mnl_eval(dp, th, grad=True, hess=False)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
        tk.append(M.last_eval_ms())
    nbytes = 8 * s.N * (s.p + s.K * (s.f + s.d)) + 4 * s.N
    best = min(ts)
    print(cfg, "eval ms", ["%.3f" % t for t in ts], "best %.3f ms, input %.3f GB -> %.0f GB/s" %
          (best, nbytes / 1e9, nbytes / best / 1e6), "| kernel median %.4f ms -> %.0f GB/s" %
          (float(np.median(tk[1:] or tk)), nbytes / float(np.median(tk[1:] or tk)) / 1e6), flush=True)


if __name__ == "__main__":
    main()
