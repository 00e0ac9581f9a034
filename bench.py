#!/usr/bin/env python
"""Benchmark of the mnlogit Newton-Raphson hot path on B200 (one JSON line on rank 0).

A "step" is one full Newton-Raphson iteration through the C ABI (mnl_newton_fit with
max_iter = 1 from a fixed start): pass-1 evaluation (utilities, softmax, loglik, gradient, P
rows), Hessian assembly, Cholesky factor + solves, the step-halving line search (>= 1 more
evaluation) and the stopping test — every row of SURVEY.md §8(a).  Each iteration forms exactly
one Hessian, so the metric "Hessian evals/s" = Newton iterations/s.

Workload: BASELINE.json configs[3] ("c4", N=500000, K=100, p=50, n_p=5049), the largest single-GPU
config the metric is quoted on; inputs are synthetic (datagen, seed 0), resident in HBM and larger
than L2 (X 200 MB, probability rows 416 MB), so no L2 flush is needed between steps.

--gpus N > 1: data-parallel over individuals (mnl_newton_fit_dp; paper_1404_3177_b200/distributed.py):
rank r owns a contiguous slice of the c4 individuals; NCCL all-reduces [l, flag, g] after every
evaluation and the packed upper triangle of -H after the Hessian; every rank factors the same -H
(strong scaling: the total work is fixed).
--impl reference: the plain C oracle (oracle/oracle.c) as it stands, timed on this host's cores, one
full-size Newton iteration per step (the only other place bench.py executes oracle/).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402

METRIC = "Hessian evals/s (Newton iterations/s), FP64"
UNIT = "hessian_evals/s"


def load_peaks():
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    fp64 = None
    try:
        fp64 = json.load(open(os.path.join(ROOT, "profiles", "fp64_peak_r1.json")))
    except Exception:
        pass
    return peaks, fp64


def fp64_peak_tflops():
    """Roofline denominator for the DMMA kernel: the larger of
    (a) the measured DMMA.8x8x4 sustained peak (tools/fp64_peak.cu -> profiles/fp64_peak_r1.json) and
    (b) MEASURED_PEAKS bf16 x the guide's nominal FP64-tensor/BF16 ratio (45 / 2250)."""
    peaks, fp64 = load_peaks()
    cands = []
    if fp64 and fp64.get("dmma_tflops"):
        cands.append((float(fp64["dmma_tflops"]), "measured DMMA.8x8x4 sustained (profiles/fp64_peak_r1.json)"))
    if peaks.get("bf16_tflops"):
        cands.append((float(peaks["bf16_tflops"]) * 45.0 / 2250.0,
                      "MEASURED_PEAKS bf16_tflops x nominal FP64/BF16 ratio 45/2250"))
    if not cands:
        cands.append((37.0, "fallback: nominal 148 SM x 64 FMA/clk x 1.965 GHz"))
    return max(cands)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = os.path.join("/tmp", f"bench_clocks_{os.getpid()}.csv")

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        try:
            for line in open(self.path):
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 7 and parts[0].isdigit():
                    rows.append(parts)
        except Exception:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [int(r[0]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[j] for r in rows for j in range(4) if r[3 + j].lower() == "active"})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": int(rows[0][1]), "reasons": reasons,
                "samples": len(rows)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def hess_flops(spec):
    """Algorithmic flops of one Hessian assembly:
    F_min: the beta-beta pairs x vech GEMM (2 N (K-1)K/2 q(q+1)/2) + the Z/Y blocks;
    F_H:   the paper's method (every upper-triangular chunk-pair block as a full DGEMM)."""
    N, K, q, d, f = spec.N, spec.K, spec.p + 1, spec.d, spec.f
    pairs = (K - 1) * K // 2
    vech = q * (q + 1) // 2
    j1 = 2.0 * N * pairs * vech
    rem = vech % 128  # the library's split: whole 128-column tiles + a narrow tail launch (k_hess.cu)
    n1a = vech - rem if (vech > 128 and 0 < rem <= 96) else vech
    j1_main = 2.0 * N * pairs * n1a
    n_b, n_a = (K - 1) * q, K * d
    j2 = 2.0 * N * (n_b + n_a + f) * (n_a + f) if (d + f) else 0.0
    ar = 2.0 * N * K * (q + d + f) * (d + f) if (d + f) else 0.0
    # paper method: upper chunk pairs as full DGEMMs
    chunks = [q] * (K - 1) + [d] * K if d else [q] * (K - 1)
    s = sum(chunks)
    # sum over upper chunk pairs (incl. diagonal) of 2 N c_i c_j = N (S^2 + sum c_i^2); generic part O(K)
    F_H = N * (s * s + sum(c * c for c in chunks)) + (2.0 * N * K * f * (s + f) if f else 0.0)
    return dict(j1=j1, j1_main=j1_main, j2=j2, arrow=ar, f_min=j1 + j2 + ar, f_paper=F_H)


def run_dp(args):
    """N > 1: data-parallel Newton step over the ranks' slices (strong scaling)."""
    import torch
    import torch.distributed as dist
    import paper_1404_3177_b200 as M
    from paper_1404_3177_b200 import distributed as DP

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    M.load()
    prob = datagen.make(args.config, seed=args.seed)
    spec = prob.spec
    lo, hi = DP.shard_range(spec.N, ws, rank)
    X = torch.from_numpy(np.ascontiguousarray(prob.X[lo:hi])).to(dev)
    Y = torch.from_numpy(np.ascontiguousarray(prob.Y[lo:hi])).to(dev) if spec.f else None
    Z = torch.from_numpy(np.ascontiguousarray(prob.Z[lo:hi])).to(dev) if spec.d else None
    ch = torch.from_numpy(prob.choice[lo:hi].astype(np.int32)).to(dev)
    dp = M.problem(X, Y, Z, ch, K=spec.K)
    launches = [0]
    theta0 = torch.zeros(spec.n_params, dtype=torch.float64, device=dev)
    allreduce = DP.torch_allreduce()   # NCCL, ordered on the library's stream

    def step():
        # one Newton iteration of the library's data-parallel driver (mnl_newton_fit_dp): exchanges
        # [l, flag, g] per evaluation and the packed upper triangle of -H per Hessian
        f = M.mnl_newton_fit_dp(dp, allreduce, coef0=theta0, tol=1e-300, max_iter=1)
        launches[0] += M.last_launch_count()
        return f

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    launches[0] = 0
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record()
        for _ in range(args.steps):
            step()
        e1.record()
        torch.cuda.synchronize()
    dist.barrier()
    hts = M.last_hessian_times()  # the last Hessian of the last step (this rank's slice)
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    # e2e: each rank copies its slice from pinned host memory every step, result back to the host
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
    hX, hch = pin(prob.X[lo:hi]), pin(prob.choice[lo:hi].astype(np.int32))
    hY = pin(prob.Y[lo:hi]) if spec.f else None
    hZ = pin(prob.Z[lo:hi]) if spec.d else None
    n_e2e = max(1, min(args.steps, 3))
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(n_e2e):
        X.copy_(hX, non_blocking=True)
        ch.copy_(hch, non_blocking=True)
        if hY is not None:
            Y.copy_(hY, non_blocking=True)
        if hZ is not None:
            Z.copy_(hZ, non_blocking=True)
        f = step()
        f.coef.cpu()
    torch.cuda.synchronize()
    te = torch.tensor([(time.perf_counter() - t0) / n_e2e], dtype=torch.float64, device=dev)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    result = None
    if rank == 0:
        fl = hess_flops(spec)
        peak, peak_src = fp64_peak_tflops()
        j1_rank = fl["j1_main"] * (hi - lo) / spec.N
        j1_ms = hts["j1_gemm"]
        roof = {"kernel": "J1 main launch (k_pipe_gemm<128,32,3>) on rank 0's slice", "bound": "tensor",
                "achieved": j1_rank / (j1_ms / 1e3) / 1e12 if j1_ms else None,
                "peak": peak, "peak_source": peak_src, "unit": "TFLOP/s", "traffic": None,
                "algorithmic_flops_per_launch": j1_rank, "avg_launch_ms": j1_ms}
        roof["frac"] = roof["achieved"] / peak if roof["achieved"] else None
        bi = hX.numel() * 8 + hch.numel() * 4 + (hY.numel() * 8 if hY is not None else 0) + \
            (hZ.numel() * 8 if hZ is not None else 0)
        result = {
            "metric": METRIC, "value": args.steps / (ms / 1e3), "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (datagen seed %d)" % args.seed,
            "config": {"workload": f"{args.config}: N={spec.N} K={spec.K} p={spec.p} f={spec.f} d={spec.d} "
                                   f"n_p={spec.n_params}, one Newton iteration from theta=0 per step",
                       "l2": "inputs larger than L2 (no flush)",
                       "parallelism": f"data-parallel over individuals, {ws} ranks (mnl_newton_fit_dp): NCCL "
                                      f"all-reduce of [l, flag, g] per evaluation and of the packed -H per Hessian"},
            "s_per_newton_iter": ms / args.steps / 1e3,
            "roofline": roof,
            "gpu_launches": int(launches[0]),
            "clocks": clk.summary(),
            "e2e": {"value": 1.0 / float(te.item()), "unit": UNIT, "h2d_bytes_per_step": int(bi),
                    "d2h_bytes_per_step": int(spec.n_params * 8), "steps": n_e2e, "per_rank_bytes": True},
        }
    dist.barrier()
    dist.destroy_process_group()
    return result, prob


def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_1404_3177_b200 as M

    ws, rank, local = dist_env()
    if ws > 1 or os.environ.get("BENCH_FORCE_DP"):
        return run_dp(args)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    M.load()

    prob = datagen.make(args.config, seed=args.seed)
    spec = prob.spec
    X = torch.from_numpy(prob.X).to(dev)
    Y = torch.from_numpy(prob.Y).to(dev) if spec.f else None
    Z = torch.from_numpy(prob.Z).to(dev) if spec.d else None
    ch = torch.from_numpy(prob.choice.astype(np.int32)).to(dev)
    dp = M.problem(X, Y, Z, ch, K=spec.K)
    coef0 = torch.zeros(spec.n_params, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream()

    def step():
        return M.mnl_newton_fit(dp, coef0=coef0, tol=1e-300, max_iter=1)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches = 0
    gemm_ms, hess_ms, chol_ms = [], [], []
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            r = step()
            launches += M.last_launch_count()
            gemm_ms.append(M.last_hessian_times()["j1_gemm"])  # the dominant launch (CUDA events, its stream)
            hess_ms.append(r.stats["hess_ms"])
            chol_ms.append(r.stats["chol_ms"])
        e1.record(stream)
        torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    if ws > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = ws * args.steps / (ms / 1e3)

    result = None
    if rank == 0:
        fl = hess_flops(spec)
        peak, peak_src = fp64_peak_tflops()
        gemm_avg = float(np.mean(gemm_ms))
        achieved = fl["j1_main"] / (gemm_avg / 1e3) / 1e12
        traffic = None
        try:
            traffic = json.load(open(os.path.join(ROOT, "profiles", "traffic_r2.json"))).get(args.config)
        except Exception:
            pass
        # e2e: the same step through the host-buffer C ABI (H2D of inputs + D2H of the result inside)
        e2e = None
        if not args.no_e2e:
            pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
            hX, hY, hZ = pin(prob.X), pin(prob.Y), pin(prob.Z)
            hch = pin(prob.choice.astype(np.int32))
            hc0 = pin(np.zeros(spec.n_params))
            M.mnl_newton_fit_host(hX, hY if spec.f else None, hZ if spec.d else None, hch, spec.K, coef0=hc0,
                                  tol=1e-300, max_iter=1)
            n_e2e = max(1, min(args.steps, 5))
            t0 = time.perf_counter()
            for _ in range(n_e2e):
                M.mnl_newton_fit_host(hX, hY if spec.f else None, hZ if spec.d else None, hch, spec.K,
                                      coef0=hc0, tol=1e-300, max_iter=1)
            dt = (time.perf_counter() - t0) / n_e2e
            bi = hX.nbytes + (hY.nbytes if spec.f else 0) + (hZ.nbytes if spec.d else 0) + hch.nbytes + hc0.nbytes
            e2e = {"value": 1.0 / dt, "unit": UNIT, "h2d_bytes_per_step": int(bi),
                   "d2h_bytes_per_step": int(spec.n_params * 8 + 8), "steps": n_e2e}
        result = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (datagen seed %d)" % args.seed,
            "config": {"workload": f"{args.config}: N={spec.N} K={spec.K} p={spec.p} f={spec.f} d={spec.d} "
                                   f"n_p={spec.n_params}, one Newton iteration from theta=0 per step",
                       "l2": "inputs larger than L2 (no flush)",
                       "parallelism": "replicas" if ws > 1 else "single-gpu"},
            "s_per_newton_iter": ms_step / 1e3,
            "hessian_ms": float(np.mean(hess_ms)), "cholesky_solve_ms": float(np.mean(chol_ms)),
            "roofline": {"kernel": "J1 main launch: beta-beta pairs x vech DMMA GEMM over whole 128-column tiles "
                                   "(k_pipe_gemm<128,32,3> when both operands are materialised, else k_gen_gemm)",
                         "bound": "tensor", "achieved": achieved, "peak": peak, "peak_source": peak_src,
                         "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
                         "algorithmic_flops_per_launch": fl["j1_main"], "avg_launch_ms": gemm_avg,
                         "hessian_f_min_tflops": fl["f_min"] / (float(np.mean(hess_ms)) / 1e3) / 1e12,
                         "hessian_paper_method_equiv_tflops": fl["f_paper"] / (float(np.mean(hess_ms)) / 1e3) / 1e12},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "e2e": e2e,
        }
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()
    return result, prob


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _oracle_data(prob, n=None):
    import oracle as O
    n = prob.spec.N if n is None else n
    return O.Data(prob.X[:n], prob.Y[:n], prob.Z[:n], prob.choice[:n], prob.spec.K)


def oracle_iteration_seconds(prob, n=None, threads=0):
    """One Newton iteration of the plain C oracle (oracle/oracle.c, as it stands) from theta = 0 on the
    first n individuals (all by default): l and g, H, Cholesky of -H, the step-halving line search and
    l, g at the new iterate -- the same work as one bench step."""
    from oracle import coracle as OC
    n0 = OC.set_threads(0)
    try:
        OC.set_threads(threads)
        D = _oracle_data(prob, n)
        t0 = time.perf_counter()
        OC.newton_fit(D, coef0=None, tol=1e-300, max_iter=1)
        return time.perf_counter() - t0
    finally:
        OC.set_threads(n0)


def cpu_baseline(prob, n_sample):
    """The C oracle on a bounded sample: its N-proportional phases (pass 1, gradient,
    Hessian, line-search passes) timed on the first n_sample individuals and scaled by N / n_sample,
    plus its N-independent phase (the Cholesky factor + solves of the full n_p x n_p -H, timed at full
    size); then the single-thread context of c1-c3 (the paper timed one core)."""
    from oracle import coracle as OC
    s = prob.spec
    D = _oracle_data(prob, n_sample)
    th = np.zeros(s.n_params)
    t0 = time.perf_counter()
    _, g, H = OC.mnl_eval(D, th)              # l, g, H at theta = 0
    t_eval = time.perf_counter() - t0
    A = -H
    t0 = time.perf_counter()
    L = OC.cholesky(A)                        # n_p^3 / 3: independent of N
    t_chol = time.perf_counter() - t0
    t0 = time.perf_counter()
    for _ in range(4):                        # the c4 step's line-search passes + the new iterate's l, g
        OC.loglik(D, th)
    t_ls = time.perf_counter() - t0
    del L
    scale = s.N / n_sample
    per_iter = (t_eval + t_ls) * scale + t_chol
    ctx = {}
    for c in ("c1", "c2", "c3"):
        pc = datagen.make(c)
        ctx[c] = {"s_per_newton_iter_1_thread": oracle_iteration_seconds(pc, threads=1)}
    return {"value": 1.0 / per_iter, "unit": UNIT, "cores": OC.set_threads(0), "kind": "oracle",
            "cpu_model": cpu_model(),
            "sample": f"C oracle (oracle/oracle.c): l, g, H and 4 loglik passes on the first {n_sample} of {s.N} "
                      f"individuals of {s.name} ({t_eval + t_ls:.2f} s, scaled x{scale:.0f}: linear in N) + the "
                      f"Cholesky of the full {s.n_params}x{s.n_params} -H ({t_chol:.2f} s, not scaled)",
            "single_thread_context": ctx}


def run_reference(args):
    """The reference arm: the plain C oracle as it stands, one FULL-size Newton iteration per step (no
    sampling, no scaling), on every host core. A step takes about a minute on c4, so the run stops
    after --ref-budget seconds of timed steps (at least one) and reports the steps it actually ran."""
    ws, rank, local = dist_env()
    if rank != 0:
        return None
    from oracle import coracle as OC
    prob = datagen.make(args.config, seed=args.seed)
    times = []
    t_start = time.perf_counter()
    while len(times) < args.steps and (not times or time.perf_counter() - t_start < args.ref_budget):
        times.append(oracle_iteration_seconds(prob))
    per_step = float(np.mean(times))
    value = 1.0 / per_step
    spec = prob.spec
    cb = {"value": value, "unit": UNIT, "cores": OC.set_threads(0), "kind": "oracle", "cpu_model": cpu_model(),
          "sample": f"none: each step is one full-size C-oracle Newton iteration ({spec.N} individuals); "
                    f"{len(times)} timed steps, no warm-up (a CPU program without caches to warm)"}
    return {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
            "steps": len(times), "warmup": 0, "ms_per_step": per_step * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (datagen seed %d)" % args.seed,
            "config": {"workload": f"{args.config}: N={spec.N} K={spec.K} p={spec.p} f={spec.f} d={spec.d} "
                                   f"n_p={spec.n_params}, one Newton iteration from theta=0 per step",
                       "l2": "n/a (CPU)", "parallelism": "host cores (OpenMP)"},
            "step_s": times, "requested_steps": args.steps, "requested_warmup": args.warmup,
            "cpu_baseline": cb,
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def full_fit_extra(cfg: str, seed: int):
    """North-star context numbers in the same run: the full Newton fit of `cfg` to ||g|| < 1e-6
    (BASELINE.json configs[4] is the fit config), median of 3 after a warm-up fit."""
    import torch
    import paper_1404_3177_b200 as M
    prob = datagen.make(cfg, seed=seed)
    s = prob.spec
    dev = torch.device("cuda", torch.cuda.current_device())
    dp = M.problem(torch.from_numpy(prob.X).to(dev), torch.from_numpy(prob.Y).to(dev) if s.f else None,
                   torch.from_numpy(prob.Z).to(dev) if s.d else None,
                   torch.from_numpy(prob.choice.astype(np.int32)).to(dev), K=s.K)
    M.mnl_newton_fit(dp, tol=1e-6)
    runs = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f = M.mnl_newton_fit(dp, tol=1e-6)
        runs.append((time.perf_counter() - t0, f))
    t, f = sorted(runs, key=lambda r: r[0])[1]
    return {"config": f"{cfg}: N={s.N} K={s.K} p={s.p} f={s.f} d={s.d} n_p={s.n_params}", "fit_s": t,
            "iters": f.iters, "halvings": f.stats["halvings"], "s_per_newton_iter": t / max(1, f.iters),
            "hessian_ms_per_iter": f.stats["hess_ms"] / max(1, f.iters),
            "hessian_evals_per_s": 1e3 * max(1, f.iters) / f.stats["hess_ms"], "status": f.status,
            "grad_norm": f.stats["grad_norm"]}


def pass1_extra(cfg: str, seed: int, reps: int = 20):
    """Pass 1 (a1-a4: utilities, softmax, loglik, gradient; no Hessian, no P write) of `cfg` at
    theta_true: the kernel's device time (CUDA events around the launch, inside the library) and
    its algorithmic HBM bytes 8N(p + K(f + d)) + 4N (X, Y, Z, choice read once) against the HBM
    peak; plus the truncated-Newton (CG) fit of the same config."""
    import torch
    import paper_1404_3177_b200 as M
    prob = datagen.make(cfg, seed=seed)
    s = prob.spec
    dev = torch.device("cuda", torch.cuda.current_device())
    dp = M.problem(torch.from_numpy(prob.X).to(dev), torch.from_numpy(prob.Y).to(dev) if s.f else None,
                   torch.from_numpy(prob.Z).to(dev) if s.d else None,
                   torch.from_numpy(prob.choice.astype(np.int32)).to(dev), K=s.K)
    th = torch.from_numpy(prob.theta_true).to(dev)
    for _ in range(3):
        M.mnl_eval(dp, th, grad=True, hess=False)
    ts = []
    for _ in range(reps):
        M.mnl_eval(dp, th, grad=True, hess=False)
        ts.append(M.last_eval_ms())
    ms = float(np.median(ts))
    nbytes = 8 * s.N * (s.p + s.K * (s.f + s.d)) + 4 * s.N
    peaks, _ = load_peaks()
    hbm = float(peaks.get("hbm_gbs") or 6542.1)  # measured copy bandwidth (MEASURED_PEAKS.json)
    gbs = nbytes / (ms / 1e3) / 1e9
    M.mnl_newton_fit(dp, tol=1e-6, method="cg")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f = M.mnl_newton_fit(dp, tol=1e-6, method="cg")
    t_cg = time.perf_counter() - t0
    return {"config": f"{cfg}: N={s.N} K={s.K} p={s.p} f={s.f} d={s.d} n_p={s.n_params}",
            "pass1_roofline": {"kernel": "k_eval_w (fused a1-a4 pass, team mapping; gradient, no Hessian)", "bound": "hbm",
                               "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm,
                               "algorithmic_bytes_per_launch": nbytes, "avg_launch_ms": ms},
            "cg_fit": {"fit_s": t_cg, "iters": f.iters, "cg_iters": f.stats["cg_iters"], "status": f.status,
                       "grad_norm": f.stats["grad_norm"], "loglik": f.loglik}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4", choices=list(datagen.CONFIGS))
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--oracle-sample", type=int, default=50000)
    ap.add_argument("--ref-budget", type=float, default=240.0, help="reference arm: seconds of timed steps")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extra", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        res = run_reference(args)
        if res is not None:
            print(json.dumps(res), flush=True)
        return
    res, prob = run_ours(args)
    if res is None:
        return
    single = res.get("n_gpus", 1) == 1 and "data-parallel" not in res["config"]["parallelism"]
    if single and not args.no_extra and args.config != "c5":
        res["extra_full_fit"] = full_fit_extra("c5", args.seed)
        res["extra_full_fit"].update(pass1_extra("c5", args.seed))
    if not args.no_cpu_baseline and single:
        res["cpu_baseline"] = cpu_baseline(prob, args.oracle_sample)
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
