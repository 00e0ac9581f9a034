import os, sys
import numpy as np
sys.path.insert(0, os.getcwd())
import torch, datagen
import paper_1404_3177_b200 as M
os.environ["MNL_FORCE_YZW"] = "1"
for shape in [(1000, 4, 3, 2, 1), (334, 50, 5, 10, 5), (30000, 12, 9, 4, 3)]:
    N, K, p, f, d = shape
    prob = datagen.custom(N, K, p, f, d, seed=11, coef_sd=0.3, require_all_classes=False)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    dp = M.problem(t(prob.X) if p else None, t(prob.Y) if f else None, t(prob.Z) if d else None, t(prob.choice.astype(np.int32)), K=K)
    th = t(datagen.perturbed_theta(prob, 0.2))
    a = M.mnl_eval(dp, th, grad=True, hess=False); ga = a[1].cpu().numpy().copy()
    b = M.mnl_eval(dp, th, grad=True, hess=False); gb = b[1].cpu().numpy().copy()
    c = M.mnl_eval(dp, th, grad=True, hess=True); gc = c[1].cpu().numpy().copy()
    e = M.mnl_eval(dp, th, grad=True, hess=True); ge = e[1].cpu().numpy().copy()
    q = p + 1
    print(shape, "nohess twice equal:", np.array_equal(ga, gb), "hess twice equal:", np.array_equal(gc, ge), "hess vs nohess:", np.array_equal(ga, gc))
    dif = np.nonzero(ga != gc)[0]
    print("  differing idx", dif[:20], "n_beta", (K - 1) * q, "n_alpha", K * d, "max rel", (np.abs(ga - gc) / np.abs(ga)).max())
