import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_1404_3177_b200 as M
for n in (8000, 12345, 16384):
    g = torch.Generator(device="cuda").manual_seed(n)
    B = torch.randn(n, n + 7, dtype=torch.float64, device="cuda", generator=g)
    A = B @ B.T / n + 0.1 * torch.eye(n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    x = M.mnl_spd_solve(A, b); torch.cuda.synchronize()
    e0.record(); x = M.mnl_spd_solve(A, b); e1.record(); torch.cuda.synchronize()
    res = ((A @ x - b).norm() / b.norm()).item()
    print(n, f"{e0.elapsed_time(e1):.2f} ms", f"relres {res:.2e}", flush=True)
