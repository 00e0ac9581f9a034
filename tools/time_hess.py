#!/usr/bin/env python
"""Quick GPU timing: per config, the median of `reps` mnl_eval calls with the Hessian (CUDA events
around the call, which includes pass 1) and the library's Hessian phase times, then one Newton fit.
Usage: python tools/time_hess.py c5 [c4 ...]"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402


def main():
    import torch
    import paper_1404_3177_b200 as M
    reps = int(os.environ.get("REPS", "7"))
    for cfg in sys.argv[1:] or ["c5"]:
        prob = datagen.make(cfg)
        s = prob.spec
        dev = torch.device("cuda", 0)
        dp = M.problem(torch.from_numpy(prob.X).to(dev), torch.from_numpy(prob.Y).to(dev) if s.f else None,
                       torch.from_numpy(prob.Z).to(dev) if s.d else None,
                       torch.from_numpy(prob.choice.astype(np.int32)).to(dev), K=s.K)
        th = torch.from_numpy(prob.theta_true).to(dev)
        ts, ph = [], []
        for r in range(reps + 2):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            M.mnl_eval(dp, th, grad=True, hess=True)
            e1.record()
            torch.cuda.synchronize()
            if r >= 2:
                ts.append(e0.elapsed_time(e1))
                ph.append(list(M.last_hessian_times().values()))
        print(cfg, "eval+hess ms median %.3f min %.3f" % (float(np.median(ts)), min(ts)),
              "phases", dict(zip(M.last_hessian_times().keys(), [round(x, 3) for x in np.median(np.array(ph), axis=0)])), flush=True)
        if cfg != "c4" or os.environ.get("FIT_C4"):
            fs = []
            for r in range(3):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                f = M.mnl_newton_fit(dp, tol=1e-6)
                torch.cuda.synchronize()
                fs.append(time.perf_counter() - t0)
            print(cfg, "fit s", [round(x, 4) for x in fs], "iters", f.iters, "hess_ms", round(f.stats["hess_ms"], 2),
                  "chol_ms", round(f.stats["chol_ms"], 2), flush=True)


if __name__ == "__main__":
    main()
