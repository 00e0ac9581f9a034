#!/usr/bin/env python
"""Context runs shaped like the paper's Table 1 problems (N = 100 000, K = 100): X (50
individual-specific variables incl. the intercept, n_p = 4950), Y (50 alternative-varying variables
with alternative-specific coefficients) and YZ (45 alternative-specific + 5 generic) -- EXTRA, not
BASELINE.json configs. Synthetic: data ~ N(0,1) / U(-1,1), coefficients ~ N(0, 0.1),
choices drawn from the model (the paper's makeModel data is not available). Prints one Hessian
evaluation and the full fits (Newton, truncated Newton) on this GPU next to the paper's single-core
numbers (2.6 GHz Xeon, MKL 11.0) -- context only."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402


PAPER = {  # Table 1: single core, seconds
    "X": {"hessian_total": 1074.1, "nr": 1125.5, "total": 1226.7},
    "Y": {"hessian_total": 1122.4, "nr": 1361.5, "total": 1511.8},
    "YZ": {"hessian_total": 1053.1, "nr": 1247.4, "total": 1417.5},
}
# shapes in ABI letters: X = individual-specific (p), Z = alternative-specific coefficients (d),
# Y = generic (f); intercepts always on (reading R3), so n_p exceeds the paper's by K - 1 for Y / YZ
SHAPES = {"X": (100000, 100, 49, 0, 0), "Y": (100000, 100, 0, 0, 50), "YZ": (100000, 100, 0, 5, 45)}


def run(name):
    import torch
    import paper_1404_3177_b200 as M
    N, K, p, f, d = SHAPES[name]
    prob = datagen.custom(N, K, p, f, d, seed=0, coef_sd=0.1, name="paper-table1-" + name)
    s = prob.spec
    dev = torch.device("cuda", 0)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    dp = M.problem(t(prob.X) if p else None, t(prob.Y) if f else None, t(prob.Z) if d else None,
                   t(prob.choice.astype(np.int32)), K=K)
    th = torch.zeros(s.n_params, dtype=torch.float64, device=dev)
    M.mnl_eval(dp, th, grad=True, hess=True)
    hs = []
    for _ in range(3):
        M.mnl_eval(dp, th, grad=True, hess=True)
        hs.append(sum(M.last_hessian_times().values()))
    out = {"problem": name, "config": f"N={N} K={K} p={p} f={f} d={d} n_p={s.n_params}",
           "hessian_ms": float(np.median(hs))}
    for method in ("newton", "cg"):
        M.mnl_newton_fit(dp, tol=1e-6, method=method)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fit = M.mnl_newton_fit(dp, tol=1e-6, method=method)
        out[f"{method}_fit_s"] = time.perf_counter() - t0
        out[f"{method}_iters"] = fit.iters
        out[f"{method}_status"] = fit.status
    out["paper_single_core_s"] = dict(PAPER[name], hardware="Intel 2.6 GHz, 1 core, MKL 11.0 (P:502-503)")
    M.release()
    return out


def main():
    names = sys.argv[1:] or ["X", "Y", "YZ"]
    for n in names:
        print(json.dumps(run(n)), flush=True)


if __name__ == "__main__":
    main()
