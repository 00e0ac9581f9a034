#!/usr/bin/env python
"""Time the Newton-step solve (mnl_spd_solve: tile-DAG factor + fused forward solve + backward
wavefront) and mnl_cholesky on random SPD matrices, CUDA events around the call (includes the
call's host overhead; the kernel-only times come from the ncu launch list)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_1404_3177_b200 as M
    ns = [int(a) for a in sys.argv[1].split(",")] if len(sys.argv) > 1 else [18, 189, 969, 1779, 5049]
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    for n in ns:
        g = torch.Generator(device="cuda").manual_seed(n)
        B = torch.randn(n, n + 16, dtype=torch.float64, device="cuda", generator=g)
        A0 = B @ B.T / n + torch.eye(n, dtype=torch.float64, device="cuda")
        b = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ts, tc = [], []
        for r in range(reps):
            torch.cuda.synchronize()
            e[0].record()
            x = M.mnl_spd_solve(A0, b)
            e[1].record()
            torch.cuda.synchronize()
            ts.append(e[0].elapsed_time(e[1]))
        for r in range(max(2, reps // 3)):
            A = A0.clone()
            torch.cuda.synchronize()
            e[0].record()
            M.mnl_cholesky(A)
            e[1].record()
            torch.cuda.synchronize()
            tc.append(e[0].elapsed_time(e[1]))
        res = (A0 @ x - b).norm().item() / b.norm().item()
        ts.sort(), tc.sort()
        print(f"n={n} spd_solve_ms min {ts[0]:.4f} med {ts[len(ts) // 2]:.4f}  cholesky_ms min {tc[0]:.4f}  "
              f"relres={res:.2e} launches={M.last_launch_count()}", flush=True)


if __name__ == "__main__":
    main()
