import os, sys
import numpy as np
sys.path.insert(0, os.getcwd())
import torch, datagen
import paper_1404_3177_b200 as M
N, K, p, f, d = 300, 4, 3, 2, 1
prob = datagen.custom(N, K, p, f, d, seed=71, coef_sd=0.4, require_all_classes=False)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
dp = M.problem(t(prob.X), t(prob.Y), t(prob.Z), t(prob.choice.astype(np.int32)), K=K)
th = t(prob.theta_true)
print("clean", M.mnl_eval(dp, th, grad=True, hess=False, raise_on_error=False)[0] if 'raise_on_error' in M.mnl_eval.__code__.co_varnames else M.mnl_eval(dp, th, grad=True, hess=False)[0])
for (i, k, e) in [(150, 2, 0), (150, 2, 1), (0, 0, 0), (299, 3, 1), (150, 0, 0), (150, 1, 0), (150, 3, 0), (151, 2, 0), (149,2,0)]:
    Y = dp.Y.clone(); Y[i, k, e] = float("nan")
    dY = M.problem(dp.X, Y, dp.Z, dp.choice, K=K)
    try:
        r = M.mnl_eval(dY, th, grad=True, hess=False)
        print(i, k, e, "no raise", float(r[0]), bool(torch.isnan(r[1]).any()))
    except M.MnlError as ex:
        print(i, k, e, "raised", ex.code)
