#!/usr/bin/env python
"""Evaluate one shape on the GPU against the oracle (debugging aid): python tools/check_shape.py N K p f d [repo_root]"""
import os
import sys

import numpy as np

N, K, p, f, d = map(int, sys.argv[1:6])
root = sys.argv[6] if len(sys.argv) > 6 else os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, root)
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch  # noqa: E402

import datagen  # noqa: E402
import oracle as O  # noqa: E402
import paper_1404_3177_b200 as M  # noqa: E402

print("lib", M.LIB_PATH)
prob = datagen.custom(N, K, p, f, d, seed=N + K, coef_sd=0.3, require_all_classes=False)
D = O.Data(prob.X, prob.Y, prob.Z, prob.choice, K)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
dp = M.problem(t(prob.X) if p else None, t(prob.Y) if f else None, t(prob.Z) if d else None,
               t(prob.choice.astype(np.int32)), K=K)
th = datagen.perturbed_theta(prob, 0.2)
l_o, g_o, _ = O.mnl_eval(D, th, want_hess=False)
ll, g, _ = M.mnl_eval(dp, t(th), grad=True, hess=False)
gg = g.cpu().numpy()
print("loglik gpu %.12f oracle %.12f  grad rel %.3e" % (ll.item(), l_o, np.linalg.norm(gg - g_o) / np.linalg.norm(g_o)))
if os.environ.get("DETAIL"):
    q = p + 1
    err = np.abs(gg - g_o)
    bad = np.nonzero(err > 1e-8 * np.abs(g_o).max())[0]
    print("bad grad entries", bad.size, "first", bad[:10], "alternatives", sorted(set((bad[bad < (K - 1) * q] // q + 1).tolist()))[:40])
    P_o = O.probabilities(O.utilities(D, th))
    Pg = M.mnl_predict(dp, t(th)).cpu().numpy()
    rows = np.nonzero(np.abs(Pg - P_o).max(axis=1) > 1e-12)[0]
    cols = np.nonzero(np.abs(Pg - P_o).max(axis=0) > 1e-12)[0]
    print("P bad rows", rows.size, rows[:20], "bad cols", cols[:40])
    if f == 0 and d == 0:  # direct numpy check of the X-only utilities
        B = th.reshape(K - 1, q)
        V = np.zeros((N, K))
        V[:, 1:] = B[:, 0][None, :] + prob.X @ B[:, 1:].T
        V -= V.max(axis=1, keepdims=True)
        Pd = np.exp(V) / np.exp(V).sum(axis=1, keepdims=True)
        print("direct vs oracle max", np.abs(Pd - P_o).max(), "direct vs gpu max", np.abs(Pd - Pg).max())
