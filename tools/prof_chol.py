#!/usr/bin/env python
"""Time mnl_cholesky / mnl_cholesky_solve on a random SPD matrix (CUDA events)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_1404_3177_b200 as M
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 5049
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    g = torch.Generator(device="cuda").manual_seed(0)
    B = torch.randn(n, n + 16, dtype=torch.float64, device="cuda", generator=g)
    A0 = B @ B.T / n + torch.eye(n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    for r in range(reps):
        A = A0.clone()
        torch.cuda.synchronize()
        e[0].record()
        rc = M.mnl_cholesky(A)
        e[1].record()
        x = M.mnl_cholesky_solve(A, b)
        e[2].record()
        torch.cuda.synchronize()
        res = (A0 @ x - b).norm().item() / b.norm().item()
        print(f"n={n} rc={rc} chol_ms={e[0].elapsed_time(e[1]):.3f} solve_ms={e[1].elapsed_time(e[2]):.3f} "
              f"relres={res:.2e} launches={M.last_launch_count()}", flush=True)


if __name__ == "__main__":
    main()
