"""GPU: the data-parallel fit (mnl_newton_fit_dp) and the library's
reentrancy across streams (§8(b)).

R ranks are emulated in ONE process on one GPU: R threads, each with its own CUDA stream (so its
own library workspace), each fitting ITS shard of the individuals through the CUDA path; the
exchange callback sums the R device buffers in rank order and hands the sum back to every rank
(what an NCCL all-reduce does). The fit must equal the single-process ORACLE fit of the whole
problem: identical iterations and halvings, coefficients within 1e-8, loglik within 1e-10
(l, g and H are sums over individuals: P:348-351)."""
import threading

import numpy as np
import pytest

import datagen
import oracle as O
from oracle import coracle as OC
from helpers import oracle_data

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1404_3177_b200 as M  # noqa: E402
from paper_1404_3177_b200 import distributed as DP  # noqa: E402


class ThreadGroup:
    """An in-process 'process group' of R threads: all-reduce = sum in rank order, result to all."""

    def __init__(self, R):
        self.R = R
        self.bar = threading.Barrier(R, timeout=300)
        self.bufs = [None] * R
        self.calls = [0] * R
        self.counts = [[] for _ in range(R)]

    def fn(self, rank):
        def cb(buf, count, stream, ctx):
            try:
                t = DP.device_view(buf, count)
                DP.torch_stream(stream).synchronize()   # this rank's contribution is final
                self.bufs[rank] = t
                self.calls[rank] += 1
                self.counts[rank].append(int(count))
                self.bar.wait()
                if rank == 0:
                    total = self.bufs[0].clone()
                    for r in range(1, self.R):
                        total += self.bufs[r]
                    for r in range(self.R):
                        self.bufs[r].copy_(total)
                    torch.cuda.synchronize()
                self.bar.wait()
                return 0
            except Exception:  # noqa: BLE001
                self.bar.abort()
                return 1

        return M.ALLREDUCE_FN(cb)


def run_dp(prob, R, coef0=None, **kw):
    s = prob.spec
    group = ThreadGroup(R)
    fns = [group.fn(r) for r in range(R)]
    results = [None] * R
    errors = []

    def work(r):
        try:
            lo, hi = DP.shard_range(s.N, R, r)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                dp = M.problem(torch.from_numpy(np.ascontiguousarray(prob.X[lo:hi])).cuda(),
                               torch.from_numpy(np.ascontiguousarray(prob.Y[lo:hi])).cuda(),
                               torch.from_numpy(np.ascontiguousarray(prob.Z[lo:hi])).cuda(),
                               torch.from_numpy(prob.choice[lo:hi].astype(np.int32)).cuda(), K=s.K)
                c0 = None if coef0 is None else torch.from_numpy(np.asarray(coef0, dtype=np.float64)).cuda()
                st.synchronize()
                results[r] = M.mnl_newton_fit_dp(dp, fns[r], coef0=c0, stream=st, raise_on_error=False, **kw)
                st.synchronize()
        except Exception as e:  # noqa: BLE001
            errors.append(e)
            group.bar.abort()

    th = [threading.Thread(target=work, args=(r,)) for r in range(R)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    return results, group


def check_against_oracle(results, ref, n_p):
    r0 = results[0]
    assert r0.status == M.MNL_OK and ref.status == O.MNL_OK
    for r in results[1:]:   # every rank holds the same iterate (the same sums, the same decisions)
        assert r.iters == r0.iters and r.loglik == r0.loglik and torch.equal(r.coef, r0.coef)
    assert r0.iters == ref.iters
    assert r0.stats["halvings_per_iter"] == [h["halvings"] for h in ref.history]
    coef = r0.coef.cpu().numpy()
    assert np.linalg.norm(coef - ref.coef) <= 1e-8 * np.linalg.norm(ref.coef)
    assert abs(r0.loglik - ref.loglik) <= 1e-10 * abs(ref.loglik)
    assert r0.stats["min_margin"] > 1e-13


@pytest.mark.parametrize("case,R", [("c2", 3), ((3000, 6, 5, 2, 1), 4), ((2500, 12, 20, 0, 0), 2),
                                    ((4000, 20, 6, 4, 3), 3)],
                         ids=["c2-R3", "mixed-R4", "xonly-R2", "yzs-R3"])
def test_dp_fit_equals_oracle(case, R):
    prob = datagen.make(case) if isinstance(case, str) else datagen.custom(*case, seed=61, coef_sd=0.4)
    ref = OC.newton_fit(oracle_data(prob), tol=1e-6)
    results, group = run_dp(prob, R, tol=1e-6)
    check_against_oracle(results, ref, prob.spec.n_params)
    n = prob.spec.n_params
    # exchange sizes: [l, flag, g] per evaluation, the packed -H per Newton step
    assert set(group.counts[0]) == {n + 2, n * (n + 1) // 2}
    assert group.counts[0].count(n * (n + 1) // 2) == results[0].iters


def test_dp_fit_with_halvings_equals_oracle():
    prob = datagen.custom(2000, 4, 2, 1, 1, seed=40, coef_sd=0.5)
    start = np.full(prob.spec.n_params, 3.0)
    ref = OC.newton_fit(oracle_data(prob), coef0=start, tol=1e-8)
    assert sum(h["halvings"] for h in ref.history) >= 1
    results, _ = run_dp(prob, 3, coef0=start, tol=1e-8)
    check_against_oracle(results, ref, prob.spec.n_params)


def test_dp_world1_equals_single_gpu_fit():
    prob = datagen.make("c1")
    results, _ = run_dp(prob, 1, tol=1e-8)
    dp = M.problem(torch.from_numpy(prob.X).cuda(), torch.from_numpy(prob.Y).cuda(), torch.from_numpy(prob.Z).cuda(),
                   torch.from_numpy(prob.choice.astype(np.int32)).cuda(), K=prob.spec.K)
    ref = M.mnl_newton_fit(dp, tol=1e-8)
    assert results[0].iters == ref.iters and torch.equal(results[0].coef, ref.coef)


def test_dp_cg_reaches_the_oracle_mle():
    prob = datagen.custom(6000, 8, 6, 2, 1, seed=62, coef_sd=0.4)
    ref = OC.newton_fit(oracle_data(prob), tol=1e-9)
    results, group = run_dp(prob, 2, tol=1e-9, method="cg")
    r0 = results[0]
    assert r0.status == M.MNL_OK and torch.equal(results[1].coef, r0.coef)
    assert np.linalg.norm(r0.coef.cpu().numpy() - ref.coef) <= 1e-8 * np.linalg.norm(ref.coef)
    assert prob.spec.n_params in group.counts[0]   # H v products exchanged


def test_concurrent_calls_on_distinct_streams_are_independent():
    """Reentrancy (§8(b)): threads evaluating different problems on their own streams at the same time
    get exactly the results of the same calls made one after another."""
    probs = [datagen.custom(3000, 7, 4, 2, 1, seed=70 + i, coef_sd=0.4) for i in range(3)]
    dps = [M.problem(torch.from_numpy(p.X).cuda(), torch.from_numpy(p.Y).cuda(), torch.from_numpy(p.Z).cuda(),
                     torch.from_numpy(p.choice.astype(np.int32)).cuda(), K=p.spec.K) for p in probs]
    ths = [torch.from_numpy(p.theta_true).cuda() for p in probs]
    seq = [M.mnl_eval(dp, th, grad=True, hess=True) for dp, th in zip(dps, ths)]
    seq_fit = [M.mnl_newton_fit(dp, tol=1e-8) for dp in dps]
    torch.cuda.synchronize()
    out, fits, errs = [None] * 3, [None] * 3, []

    def work(i):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                for _ in range(3):
                    out[i] = M.mnl_eval(dps[i], ths[i], grad=True, hess=True, stream=st)
                    fits[i] = M.mnl_newton_fit(dps[i], tol=1e-8, stream=st)
                st.synchronize()
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=work, args=(i,)) for i in range(3)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for (l0, g0, H0), (l1, g1, H1), f0, f1 in zip(seq, out, seq_fit, fits):
        assert torch.equal(l0, l1) and torch.equal(g0, g1) and torch.equal(H0, H1)
        assert f0.iters == f1.iters and torch.equal(f0.coef, f1.coef)
