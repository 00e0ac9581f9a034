"""Shared test helpers (seeded inputs -> device problem / oracle data; sampled Hessian entries)."""
import numpy as np

import datagen
import oracle as O


def oracle_data(prob):
    return O.Data(prob.X, prob.Y, prob.Z, prob.choice, prob.spec.K)


def device_problem(prob, device="cuda"):
    import torch
    import paper_1404_3177_b200 as M
    s = prob.spec
    X = torch.from_numpy(np.ascontiguousarray(prob.X)).to(device)
    Y = torch.from_numpy(np.ascontiguousarray(prob.Y)).to(device)
    Z = torch.from_numpy(np.ascontiguousarray(prob.Z)).to(device)
    ch = torch.from_numpy(prob.choice.astype(np.int32)).to(device)
    return M.problem(X, Y if s.f else None, Z if s.d else None, ch, K=s.K)
