#!/usr/bin/env python
"""Context run shaped like the paper's Table 1 problem X (individual-specific data only,
50 variables incl. the intercept, K = 100, N = 100 000, n_p = 4950) -- EXTRA, not a BASELINE.json
config. Synthetic: X ~ N(0,1), coefficients ~ N(0, 0.1), choices drawn from the
model (the paper's makeModel data is not available). Prints one Hessian evaluation, one Newton
iteration and the full fits (Newton, truncated Newton) on this GPU; the paper's single-core numbers
(2.6 GHz Xeon, MKL; Table 1: Hessian 1074.1 s, NR 1125.5 s, total 1226.7 s) are context only."""
import json
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
    prob = datagen.custom(100000, 100, 49, 0, 0, seed=0, coef_sd=0.1, name="paper-table1-X")
    s = prob.spec
    dev = torch.device("cuda", 0)
    dp = M.problem(torch.from_numpy(prob.X).to(dev), None, None,
                   torch.from_numpy(prob.choice.astype(np.int32)).to(dev), K=s.K)
    th = torch.zeros(s.n_params, dtype=torch.float64, device=dev)
    M.mnl_eval(dp, th, grad=True, hess=True)
    hs = []
    for _ in range(3):
        M.mnl_eval(dp, th, grad=True, hess=True)
        t = M.last_hessian_times()
        hs.append(sum(t.values()))
    out = {"config": f"paper Table 1 problem X shape: N={s.N} K={s.K} p={s.p} (+intercept) n_p={s.n_params}",
           "hessian_ms": float(np.median(hs))}
    for method in ("newton", "cg"):
        M.mnl_newton_fit(dp, tol=1e-6, method=method)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f = M.mnl_newton_fit(dp, tol=1e-6, method=method)
        out[f"{method}_fit_s"] = time.perf_counter() - t0
        out[f"{method}_iters"] = f.iters
        out[f"{method}_status"] = f.status
    out["paper_single_core_s"] = {"hessian_total": 1074.1, "nr": 1125.5, "total": 1226.7,
                                  "hardware": "Intel 2.6 GHz, 1 core, MKL 11.0 (P:502-503, Table 1 P:535)"}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
