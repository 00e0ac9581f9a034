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


def sample_entries(D, n_random=256, seed=0):
    """Hessian entries covering every block kind (beta-beta within / across alternatives, beta-alpha,
    alpha-alpha, beta-gamma, alpha-gamma, gamma-gamma, diagonal, first/last) plus random ones."""
    n = D.n_p
    q = D.p + 1
    rs, cs = [], []

    def add(r, c):
        if 0 <= r < n and 0 <= c < n:
            rs.append(r); cs.append(c)

    for r in (0, 1, q - 1, q, n - 1, n // 2):
        add(r, r)
    add(0, q - 1); add(0, q); add(1, 2 * q + 1); add(q - 1, n - 1)
    nb = D.off_alpha
    if D.d:
        add(0, nb); add(0, nb + D.d); add(q, nb + D.d); add(nb, nb); add(nb, nb + D.d); add(nb + 1, nb + 2 * D.d - 1)
        add(n - 1 - D.f, nb)
    if D.f:
        g = D.off_gamma
        add(0, g); add(q + 1, g + D.f - 1); add(g, g); add(g, n - 1)
        if D.d:
            add(nb, g); add(nb + D.d, g + 1)
    rng = np.random.default_rng(seed)
    r = rng.integers(0, n, n_random)
    c = rng.integers(0, n, n_random)
    rs += list(r); cs += list(c)
    return np.array(rs), np.array(cs)
