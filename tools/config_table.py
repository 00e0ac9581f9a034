#!/usr/bin/env python
"""Per-config measurement table (BASELINE.md §4 / SURVEY.md §8(d)): GPU pass-1 time and GB/s,
Hessian time and TFLOP/s, Newton iteration and full-fit time, next to the CPU oracle on this host.

GPU times: CUDA events (library-internal for the Hessian phases), median of `reps` after warm-up.
Oracle: the plain C oracle the tests use (oracle/oracle.c), full-size where it finishes in about a minute,
otherwise a leading sample of the individuals with the time scaled by N / sample (all costs are
linear in N); the sample is printed with each number.
"""
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402


def flops_bytes(spec):
    N, K, p, f, d = spec.N, spec.K, spec.p, spec.f, spec.d
    q = p + 1
    pairs, vech = (K - 1) * K // 2, q * (q + 1) // 2
    j1 = 2.0 * N * pairs * vech
    nb, na = (K - 1) * q, K * d
    j2 = 2.0 * N * (nb + na + f) * (na + f) if (d + f) else 0.0
    ar = 2.0 * N * K * (q + d + f) * (d + f) if (d + f) else 0.0
    pass1_bytes = 8.0 * N * (p + K * (f + d)) + 4.0 * N  # gradient pass: X, Y, Z, choice read once
    return j1 + j2 + ar, pass1_bytes


def gpu_row(cfg, reps=5):
    import torch
    import paper_1404_3177_b200 as M
    prob = datagen.make(cfg)
    s = prob.spec
    dev = torch.device("cuda", 0)
    dp = M.problem(torch.from_numpy(prob.X).to(dev), torch.from_numpy(prob.Y).to(dev) if s.f else None,
                   torch.from_numpy(prob.Z).to(dev) if s.d else None,
                   torch.from_numpy(prob.choice.astype(np.int32)).to(dev), K=s.K)
    th = torch.from_numpy(prob.theta_true).to(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p1, hs, ev = [], [], []
    for r in range(reps + 2):
        M.mnl_eval(dp, th, grad=True, hess=False)
        p1.append(M.last_eval_ms())  # the pass-1 kernel's device time (events inside the library)
        e0.record()
        M.mnl_eval(dp, th, grad=True, hess=True)
        e1.record()
        torch.cuda.synchronize()
        ev.append(e0.elapsed_time(e1))
        t = M.last_hessian_times()
        hs.append(t["j1_gemm"] + t["j1_reduce"] + t["j1_tail"] + t["j1_tail_reduce"] + t["j2_and_arrow"] + t["assemble"] + t["j1_operands"])
    p1, hs, ev = [statistics.median(x[2:]) for x in (p1, hs, ev)]
    M.mnl_newton_fit(dp, tol=1e-6)  # warm-up
    fits = []
    for r in range(3):
        t0 = time.perf_counter()
        f = M.mnl_newton_fit(dp, tol=1e-6)
        fits.append((time.perf_counter() - t0, f))
    fit_s, f = sorted(fits, key=lambda x: x[0])[1]
    M.mnl_newton_fit(dp, tol=1e-6, method="cg")
    t0 = time.perf_counter()
    fcg = M.mnl_newton_fit(dp, tol=1e-6, method="cg")
    cg_s = time.perf_counter() - t0
    fc = torch.from_numpy(np.ascontiguousarray(prob.theta_true)).to(dev)
    M.mnl_std_errors(dp, fc)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    M.mnl_std_errors(dp, fc)
    se_s = time.perf_counter() - t0
    F, B = flops_bytes(s)
    return dict(cfg=cfg, N=s.N, K=s.K, n_p=s.n_params, pass1_ms=p1, pass1_GBs=B / (p1 / 1e3) / 1e9,
                hess_ms=hs, hess_evals_s=1e3 / hs, hess_tflops=F / (hs / 1e3) / 1e12, eval_with_hess_ms=ev,
                fit_s=fit_s, iters=f.iters, halvings=f.stats["halvings"], s_per_iter=fit_s / max(f.iters, 1),
                hess_ms_in_fit=f.stats["hess_ms"], chol_ms_in_fit=f.stats["chol_ms"], status=f.status,
                cg_fit_s=cg_s, cg_iters=fcg.iters, cg_inner=fcg.stats["cg_iters"], std_errors_s=se_s)


def oracle_row(cfg, budget_s=60.0):
    import oracle as O
    from oracle import coracle as OC  # the plain C oracle (liboracle.so), every host core
    prob = datagen.make(cfg)
    s = prob.spec
    n = s.N
    # pick a sample so one evaluation (l, g, H) takes roughly budget/4
    for cand in (s.N, 100000, 20000, 5000, 2000, 1000):
        if cand <= s.N:
            n = cand
            D = O.Data(prob.X[:n], prob.Y[:n], prob.Z[:n], prob.choice[:n], s.K)
            t0 = time.perf_counter()
            OC.mnl_eval(D, prob.theta_true)
            te = time.perf_counter() - t0
            if te < budget_s / 4 or cand == 1000:
                break
    scale = s.N / n
    t0 = time.perf_counter()
    OC.newton_fit(D, coef0=None, tol=1e-300, max_iter=1)
    t_iter = time.perf_counter() - t0
    return dict(cfg=cfg, oracle="C (oracle/oracle.c)", oracle_sample=n, oracle_eval_s=te * scale,
                oracle_s_per_iter=t_iter * scale, oracle_threads=OC.set_threads(0))


if __name__ == "__main__":
    cfgs = sys.argv[1:] or ["c1", "c2", "c3", "c4", "c5"]
    rows = []
    for c in cfgs:
        r = gpu_row(c)
        r.update(oracle_row(c))
        rows.append(r)
        print(json.dumps(r), flush=True)
    json.dump(rows, open(os.path.join(ROOT, "gpurun_out", "config_table.json"), "w"), indent=1)
