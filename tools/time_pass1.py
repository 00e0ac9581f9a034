#!/usr/bin/env python
"""Pass-1 kernel device time for an arbitrary shape: python tools/time_pass1.py N K p f d"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_1404_3177_b200 as M  # noqa: E402

N, K, p, f, d = map(int, sys.argv[1:6])
prob = datagen.custom(N, K, p, f, d, seed=0, coef_sd=0.1, require_all_classes=False)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
dp = M.problem(t(prob.X) if p else None, t(prob.Y) if f else None, t(prob.Z) if d else None,
               t(prob.choice.astype(np.int32)), K=K)
th = t(prob.theta_true)
ts = []
for _ in range(8):
    M.mnl_eval(dp, th, grad=True, hess=False)
    ts.append(M.last_eval_ms())
ms = float(np.median(ts[2:]))
nbytes = 8 * N * (p + K * (f + d)) + 4 * N
print(f"N={N} K={K} p={p} f={f} d={d}: pass 1 {ms:.3f} ms, {nbytes / ms / 1e6:.0f} GB/s")
