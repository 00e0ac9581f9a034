#!/usr/bin/env python
"""Hessian evaluation of one shape against the oracle (debugging aid): python tools/check_hess.py N K p f d"""
import os
import sys

import numpy as np

N, K, p, f, d = map(int, sys.argv[1:6])
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import datagen  # noqa: E402
import oracle as O  # noqa: E402
import paper_1404_3177_b200 as M  # noqa: E402

prob = datagen.custom(N, K, p, f, d, seed=N + K, coef_sd=0.3, require_all_classes=False)
D = O.Data(prob.X, prob.Y, prob.Z, prob.choice, K)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
dp = M.problem(t(prob.X) if p else None, t(prob.Y) if f else None, t(prob.Z) if d else None,
               t(prob.choice.astype(np.int32)), K=K)
th = datagen.perturbed_theta(prob, 0.2)
try:
    ll, g, H = M.mnl_eval(dp, t(th), grad=True, hess=True)
    torch.cuda.synchronize()
except Exception as e:  # noqa: BLE001
    print((N, K, p, f, d), "ERROR", e)
    sys.exit(0)
_, _, H_o = O.mnl_eval(D, th)
print((N, K, p, f, d), "hess rel %.3e" % (np.linalg.norm(H.cpu().numpy() - H_o) / np.linalg.norm(H_o)))
