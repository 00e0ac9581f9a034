"""Pins for the two CPU oracles -- oracle/mnl_oracle.py (numpy) and oracle/oracle.c (plain C,
liboracle.so, through oracle/coracle.py) -- against what the paper and the mathematics fix, never
against an oracle itself. Every test runs once per oracle (fixture `O`). `P:n` = PAPER.md line n."""
import math

import numpy as np
import pytest
from scipy.special import expit, log_expit

import datagen
import oracle.coracle as OC
import oracle.mnl_oracle as ON


@pytest.fixture(params=["numpy", "c"])
def O(request):
    return ON if request.param == "numpy" else OC


def numpy_only(O, why):
    if O is OC:
        pytest.skip(f"numpy oracle only: {why}")


def data_of(prob):
    return ON.Data(prob.X, prob.Y, prob.Z, prob.choice, prob.spec.K)


def tiny(N=200, K=4, p=3, f=2, d=1, seed=1, coef_sd=0.5):
    return datagen.custom(N, K, p, f, d, seed=seed, coef_sd=coef_sd)


# --- parameter counting (Table 1) -------------------------------------

def test_num_params_paper_counts(O):
    # Fish: income + intercept (X, p=1), catch alt-specific (ABI Z, d=1), price generic (ABI Y, f=1): 11
    assert O.num_params(K=4, p=1, f=1, d=1) == 11
    # Table 1 problem X: 50 variables incl. intercept, K=100 -> 4950
    assert O.num_params(K=100, p=49, f=0, d=0) == 4950
    # BASELINE configs
    assert [datagen.CONFIGS[c].n_params for c in ("c1", "c2", "c3", "c4", "c5")] == [18, 189, 969, 5049, 1779]


# --- closed forms at theta = 0 ------------------------------------------------------------

def test_loglik_at_zero_is_minus_N_log_K(O):
    D = data_of(datagen.make("c1"))
    assert O.loglik(D, np.zeros(D.n_p)) == pytest.approx(-1386.29436112, abs=1e-8)
    # nnet's printed initial value for N=10^4, K=10: 23025.850930 = N ln K
    pr = datagen.custom(10000, 10, 5, seed=3)
    D2 = data_of(pr)
    assert round(-O.loglik(D2, np.zeros(D2.n_p)), 6) == 23025.850930


def test_probabilities_uniform_at_zero_and_rows_sum_to_one(O):
    D = data_of(tiny())
    P = O.probabilities(O.utilities(D, np.zeros(D.n_p)))
    assert np.all(P == 0.25)
    th = datagen.draw(D.n_p, 5, 99, datagen.NORMAL, 2.0)
    P = O.probabilities(O.utilities(D, th))
    assert np.max(np.abs(P.sum(axis=1) - 1.0)) < 1e-15 * 4


def test_probabilities_overflow_safe(O):
    V = np.array([[0.0, 1000.0, 0.0], [0.0, -1000.0, -999.0]])
    P = O.probabilities(V)
    assert np.all(np.isfinite(P))
    assert P[0, 1] == 1.0 and P[0, 0] == 0.0
    assert P[1, 0] == pytest.approx(1.0)
    t = O.loglik_terms(V, np.array([1, 0]))
    assert np.all(np.isfinite(t)) and t[0] == 0.0


def test_gradient_at_zero_intercepts_is_count_minus_N_over_K(O):
    pr = tiny(N=300, K=5, p=2, f=0, d=0, seed=4)
    D = data_of(pr)
    g = O.gradient(D, np.zeros(D.n_p))
    q = D.p + 1
    n = np.bincount(D.choice, minlength=D.K)
    for k in range(1, D.K):
        assert g[(k - 1) * q] == pytest.approx(n[k] - D.N / D.K, abs=1e-10)


def test_intercept_only_hessian_closed_form(O):
    # N=100, K=4, theta=0: diagonal -N(1/K)(1-1/K) = -18.75, off-diagonal N/K^2 = 6.25
    pr = datagen.custom(100, 4, 0, seed=2)
    D = data_of(pr)
    H = O.hessian(D, np.zeros(D.n_p))
    assert np.allclose(np.diag(H), -18.75, atol=1e-12, rtol=0)
    off = H[~np.eye(3, dtype=bool)]
    assert np.allclose(off, 6.25, atol=1e-12, rtol=0)
    assert np.array_equal(O.hessian_entries(D, np.zeros(3), [0, 0], [0, 1]), np.array([-18.75, 6.25]))


# --- K = 2 is binary logistic regression ------------------------------------------

def test_K2_reduces_to_logistic_regression(O):
    pr = datagen.custom(400, 2, 3, f=2, d=2, seed=7, coef_sd=0.7)
    D = data_of(pr)
    th = datagen.draw(D.n_p, 11, 1, datagen.NORMAL, 0.5)
    # textbook design row in theta order: [1, x_i | -z_i0 | z_i1 | y_i1 - y_i0]
    W = np.hstack([np.ones((D.N, 1)), D.X, -D.Z[:, 0, :], D.Z[:, 1, :], D.Y[:, 1, :] - D.Y[:, 0, :]])
    eta = W @ th
    y = (D.choice == 1).astype(float)
    s = expit(eta)
    l_ref = np.sum(y * log_expit(eta) + (1 - y) * log_expit(-eta))
    g_ref = W.T @ (y - s)
    H_ref = -(W.T * (s * (1 - s))) @ W
    l, g, H = O.mnl_eval(D, th)
    assert l == pytest.approx(l_ref, rel=1e-13)
    assert np.max(np.abs(g - g_ref)) <= 1e-11 * np.max(np.abs(g_ref))
    assert np.max(np.abs(H - H_ref)) <= 1e-12 * np.max(np.abs(H_ref))


# --- finite differences -------------------------------------------------------------------

@pytest.mark.parametrize("shape", [(150, 4, 3, 2, 1), (120, 3, 2, 0, 2), (100, 5, 2, 3, 0), (90, 4, 0, 2, 0)])
def test_gradient_matches_central_fd(O, shape):
    N, K, p, f, d = shape
    D = data_of(tiny(N, K, p, f, d, seed=8))
    th = datagen.draw(D.n_p, 12, 2, datagen.NORMAL, 0.4)
    g = O.gradient(D, th)
    fd = np.empty_like(g)
    for r in range(D.n_p):
        h = 1e-5 * max(1.0, abs(th[r]))
        e = np.zeros(D.n_p); e[r] = h
        fd[r] = (O.loglik(D, th + e) - O.loglik(D, th - e)) / (2 * h)
    assert np.linalg.norm(fd - g) <= 1e-6 * np.linalg.norm(g)


@pytest.mark.parametrize("shape", [(150, 4, 3, 2, 1), (120, 3, 2, 0, 2), (100, 5, 2, 3, 0)])
def test_hessian_matches_central_fd_of_gradient(O, shape):
    N, K, p, f, d = shape
    D = data_of(tiny(N, K, p, f, d, seed=9))
    th = datagen.draw(D.n_p, 13, 3, datagen.NORMAL, 0.4)
    H = O.hessian(D, th)
    fd = np.empty_like(H)
    for r in range(D.n_p):
        h = 1e-5 * max(1.0, abs(th[r]))
        e = np.zeros(D.n_p); e[r] = h
        fd[:, r] = (O.gradient(D, th + e) - O.gradient(D, th - e)) / (2 * h)
    assert np.linalg.norm(fd - H) <= 1e-5 * np.linalg.norm(H)


# --- the textbook dense form and the paper's block form ---

def test_hessian_equals_textbook_dense_Xt_W_Xt_for_X_only(O):
    pr = tiny(N=60, K=5, p=3, f=0, d=0, seed=10)
    D = data_of(pr)
    th = datagen.draw(D.n_p, 14, 4, datagen.NORMAL, 0.5)
    P = O.probabilities(O.utilities(D, th))
    N, K, q = D.N, D.K, D.p + 1
    Xt1 = np.hstack([np.ones((N, 1)), D.X])
    Xtil = np.kron(np.eye(K - 1), Xt1)                       # block-diagonal, (K-1)N x (K-1)q
    Wtil = np.zeros(((K - 1) * N, (K - 1) * N))
    for k in range(1, K):
        for t in range(1, K):
            w = P[:, k] * ((k == t) - P[:, t])               # diag(W_kt)_i = P_ik(delta_kt - P_it)
            Wtil[(k - 1) * N:k * N, (t - 1) * N:t * N] = np.diag(w)
    H_ref = -Xtil.T @ Wtil @ Xtil
    yv = np.concatenate([(D.choice == k).astype(float) for k in range(1, K)])
    Pv = np.concatenate([P[:, k] for k in range(1, K)])
    g_ref = Xtil.T @ (yv - Pv)
    l, g, H = O.mnl_eval(D, th)
    assert np.max(np.abs(H - H_ref)) <= 1e-12 * np.max(np.abs(H_ref))
    assert np.max(np.abs(g - g_ref)) <= 1e-12 * np.max(np.abs(g_ref))


def block_form(O, D, th):
    """Eq. "loglik gradient" and Eq. "hessian block", paper's chunks in
    ABI letters: M = X~ for beta_k (k>=1), M = Z_k for alpha_k (k>=0), generic data Y~_k = Y_k - Y_0."""
    P = O.probabilities(O.utilities(D, th))
    N, K, p, f, d = D.N, D.K, D.p, D.f, D.d
    Xt1 = np.hstack([np.ones((N, 1)), D.X])
    chunks = [(k, Xt1) for k in range(1, K)] + [(k, D.Z[:, k, :]) for k in range(K)]
    Yt = [None] + [D.Y[:, k, :] - D.Y[:, 0, :] for k in range(1, K)]
    Yind = np.stack([(D.choice == k).astype(float) for k in range(K)], axis=1)
    W = lambda n, m: P[:, n] * ((n == m) - P[:, m])
    g_parts = [M.T @ (Yind[:, k] - P[:, k]) for k, M in chunks]
    g_parts.append(sum(Yt[k].T @ (Yind[:, k] - P[:, k]) for k in range(1, K)) if f else np.zeros(0))
    g = np.concatenate(g_parts)
    rows = []
    for n, Mn in chunks:
        row = [-(Mn.T * W(n, m)) @ Mm for m, Mm in chunks]
        row.append(-sum((Mn.T * W(n, k)) @ Yt[k] for k in range(1, K)) if f else np.zeros((Mn.shape[1], 0)))
        rows.append(np.hstack(row))
    if f:
        last = [-sum((Yt[k].T * W(k, m)) @ Mm for k in range(1, K)) for m, Mm in chunks]
        last.append(-sum((Yt[k].T * W(k, t)) @ Yt[t] for k in range(1, K) for t in range(1, K)))
        rows.append(np.hstack(last))
    return g, np.vstack(rows)


@pytest.mark.parametrize("shape", [(80, 4, 3, 2, 1), (70, 3, 1, 1, 2), (50, 5, 0, 2, 2), (64, 6, 4, 0, 0)])
def test_oracle_equals_paper_block_formulas(O, shape):
    N, K, p, f, d = shape
    D = data_of(tiny(N, K, p, f, d, seed=15))
    th = datagen.draw(D.n_p, 16, 5, datagen.NORMAL, 0.5)
    g_ref, H_ref = block_form(O, D, th)
    _, g, H = O.mnl_eval(D, th)
    assert np.max(np.abs(H - H_ref)) <= 1e-12 * np.max(np.abs(H_ref))
    assert np.max(np.abs(g - g_ref)) <= 1e-12 * np.max(np.abs(g_ref))
    rows = np.array([0, D.n_p - 1, D.n_p // 2, 1])
    cols = np.array([D.n_p - 1, D.n_p - 1, 0, D.n_p // 3])
    e = O.hessian_entries(D, th, rows, cols)
    assert np.max(np.abs(e - H_ref[rows, cols])) <= 1e-12 * np.max(np.abs(H_ref))


# --- structure and invariants ---------------------------------------------------------------

def test_hessian_symmetric_negative_definite_and_choice_independent(O):
    pr = datagen.make("c1")
    D = data_of(pr)
    H = O.hessian(D, pr.theta_true)
    assert np.array_equal(H, H.T)
    assert np.linalg.eigvalsh(-H).min() > 0
    D2 = ON.Data(pr.X, pr.Y, pr.Z, (pr.choice + 1) % pr.spec.K, pr.spec.K)
    assert np.array_equal(O.hessian(D2, pr.theta_true), H)


def test_duplicating_individuals_doubles_everything(O):
    pr = tiny(N=90, seed=17)
    D = data_of(pr)
    D2 = ON.Data(np.vstack([pr.X, pr.X]), np.vstack([pr.Y, pr.Y]), np.vstack([pr.Z, pr.Z]),
                np.concatenate([pr.choice, pr.choice]), pr.spec.K)
    th = datagen.draw(D.n_p, 18, 6, datagen.NORMAL, 0.5)
    l, g, H = O.mnl_eval(D, th)
    l2, g2, H2 = O.mnl_eval(D2, th)
    assert l2 == pytest.approx(2 * l, rel=1e-14)
    assert np.allclose(g2, 2 * g, rtol=1e-12, atol=1e-12)
    assert np.allclose(H2, 2 * H, rtol=1e-12, atol=1e-12)


def test_generic_data_shift_invariance(O):
    # Only differences against the base matter: y_ik -> y_ik + c_i leaves l, g, H unchanged
    pr = tiny(N=90, seed=19)
    D = data_of(pr)
    c = datagen.draw(pr.spec.N * pr.spec.f, 20, 7, datagen.NORMAL, 3.0).reshape(pr.spec.N, 1, pr.spec.f)
    D2 = ON.Data(pr.X, pr.Y + c, pr.Z, pr.choice, pr.spec.K)
    th = datagen.draw(D.n_p, 21, 8, datagen.NORMAL, 0.5)
    l, g, H = O.mnl_eval(D, th)
    l2, g2, H2 = O.mnl_eval(D2, th)
    assert l2 == pytest.approx(l, rel=1e-12)
    assert np.allclose(g2, g, rtol=1e-9, atol=1e-10)
    assert np.allclose(H2, H, rtol=1e-9, atol=1e-10)


def test_concavity(O):
    D = data_of(tiny(N=120, seed=22))
    a = datagen.draw(D.n_p, 23, 9, datagen.NORMAL, 1.0)
    b = datagen.draw(D.n_p, 24, 9, datagen.NORMAL, 1.0)
    for lam in (0.1, 0.5, 0.8):
        assert O.loglik(D, lam * a + (1 - lam) * b) >= lam * O.loglik(D, a) + (1 - lam) * O.loglik(D, b) - 1e-9


# --- Newton-Raphson ------------------------------------------------------------------------

def test_intercept_only_fit_closed_form(O):
    # xi_k = ln(n_k / n_0), l = sum_k n_k ln(n_k / N)
    pr = datagen.custom(500, 5, 0, seed=25, coef_sd=0.8)
    D = data_of(pr)
    fit = O.newton_fit(D, tol=1e-10)
    n = np.bincount(D.choice, minlength=D.K).astype(float)
    assert fit.status == O.MNL_OK
    assert np.allclose(fit.coef, np.log(n[1:] / n[0]), rtol=0, atol=1e-8)
    assert fit.loglik == pytest.approx(np.sum(n * np.log(n / D.N)), rel=1e-12)


def test_fit_properties_moment_condition_monotone_and_unique(O):
    pr = datagen.make("c1")
    D = data_of(pr)
    fit = O.newton_fit(D, tol=1e-9)
    assert fit.status == O.MNL_OK and fit.grad_norm < 1e-9
    ls = [h["l"] for h in fit.history] + [fit.loglik]
    assert all(b >= a for a, b in zip(ls, ls[1:]))
    # moment condition at the MLE with an intercept: sum_i P_ik = n_k
    P = O.probabilities(O.utilities(D, fit.coef))
    assert np.allclose(P.sum(axis=0), np.bincount(D.choice, minlength=D.K), atol=1e-7)
    # global concavity: a second start reaches the same optimum
    fit2 = O.newton_fit(D, coef0=datagen.random_start(pr), tol=1e-9)
    assert np.linalg.norm(fit2.coef - fit.coef) <= 1e-8 * np.linalg.norm(fit.coef)


def test_K2_fit_equals_independent_irls(O):
    pr = datagen.custom(600, 2, 3, f=1, d=1, seed=26, coef_sd=0.6)
    D = data_of(pr)
    fit = O.newton_fit(D, tol=1e-10)
    W = np.hstack([np.ones((D.N, 1)), D.X, -D.Z[:, 0, :], D.Z[:, 1, :], D.Y[:, 1, :] - D.Y[:, 0, :]])
    y = (D.choice == 1).astype(float)
    b = np.zeros(W.shape[1])
    for _ in range(50):   # textbook IRLS (weighted least squares on the working response)
        eta = W @ b
        s = expit(eta)
        w = s * (1 - s)
        zr = eta + (y - s) / w
        b_new = np.linalg.solve((W.T * w) @ W, (W.T * w) @ zr)
        if np.max(np.abs(b_new - b)) < 1e-14:
            b = b_new
            break
        b = b_new
    assert np.linalg.norm(fit.coef - b) <= 1e-8 * np.linalg.norm(b)


def test_line_search_halves_on_overshoot(O):
    # A start far out on a flat ridge makes the full Newton step overshoot; halving must kick in
    # and every accepted iterate must not lower l.
    pr = datagen.custom(200, 3, 1, seed=27, coef_sd=0.5)
    D = data_of(pr)
    start = np.full(D.n_p, 6.0)
    fit = O.newton_fit(D, coef0=start, tol=1e-8)
    assert fit.status == O.MNL_OK
    assert sum(h["halvings"] for h in fit.history) >= 1
    assert all(h["l_new"] >= h["l"] - 1e-12 * abs(h["l"]) for h in fit.history)


def test_maxiter_and_zero_iter(O):
    D = data_of(tiny(seed=28))
    fit = O.newton_fit(D, tol=1e-12, max_iter=1)
    assert fit.status == O.MNL_MAXITER and fit.iters == 1
    fit0 = O.newton_fit(D, tol=1e-12, max_iter=0)
    assert fit0.status == O.MNL_MAXITER and fit0.iters == 0 and np.all(fit0.coef == 0)


def test_recovery_of_true_coefficients_c2(O):
    # statistical pin (north_star "recovery of the true coefficients"): z = (theta_hat - theta_true)/se
    pr = datagen.make("c2")
    D = data_of(pr)
    fit = O.newton_fit(D, tol=1e-6)
    assert fit.status == O.MNL_OK
    H = O.hessian(D, fit.coef)
    se = np.sqrt(np.diag(np.linalg.inv(-H)))
    z = (fit.coef - pr.theta_true) / se
    assert np.max(np.abs(z)) < 5.0
    assert 0.85 < np.sqrt(np.mean(z * z)) < 1.15


# --- Hessian-vector products and truncated Newton --------------

@pytest.mark.parametrize("shape", [(150, 4, 3, 2, 1), (120, 3, 2, 0, 2), (100, 5, 2, 3, 0), (90, 4, 0, 2, 0)])
def test_hessvec_equals_hessian_times_v(O, shape):
    numpy_only(O, "H v products / truncated Newton")
    N, K, p, f, d = shape
    prob = tiny(N, K, p, f, d, seed=11)
    D = data_of(prob)
    rng = np.random.default_rng(3)
    th = prob.theta_true + 0.1 * rng.standard_normal(D.n_p)
    H = O.hessian(D, th)
    for _ in range(3):
        v = rng.standard_normal(D.n_p)
        hv = O.hessvec(D, th, v)
        assert np.linalg.norm(hv - H @ v) <= 1e-12 * np.linalg.norm(H @ v)


def test_hessvec_matches_central_fd_of_gradient(O):
    numpy_only(O, "H v products / truncated Newton")
    prob = tiny(150, 4, 3, 2, 1, seed=12)
    D = data_of(prob)
    rng = np.random.default_rng(4)
    th = prob.theta_true
    v = rng.standard_normal(D.n_p)
    v /= np.linalg.norm(v)
    eps = 1e-5
    fd = (O.gradient(D, th + eps * v) - O.gradient(D, th - eps * v)) / (2 * eps)
    hv = O.hessvec(D, th, v)
    assert np.linalg.norm(fd - hv) <= 1e-6 * np.linalg.norm(hv)


def test_ftol_stop_first_met_semantics(O):
    """P:219-221 / P:282-283: the fit ends at the first of gtol, ftol, maxiter; ftol compares
    successive log-likelihood values after an accepted update."""
    prob = tiny(400, 4, 3, 2, 1, seed=13)
    D = data_of(prob)
    full = O.newton_fit(D, tol=1e-10)
    assert full.status == O.MNL_OK and full.stop_reason == 1
    dls = [abs(h["l_new"] - h["l"]) for h in full.history]
    ftol = 0.5 * (dls[1] + dls[2]) if dls[1] > dls[2] else dls[2] * 1.01   # between the 2nd and 3rd changes
    fit = O.newton_fit(D, tol=1e-10, ftol=ftol)
    assert fit.status == O.MNL_OK and fit.stop_reason == 2
    k = fit.iters
    assert abs(fit.history[-1]["l_new"] - fit.history[-1]["l"]) < ftol
    assert all(abs(h["l_new"] - h["l"]) >= ftol for h in fit.history[:-1])
    assert k < full.iters and np.allclose(fit.coef, O.newton_fit(D, tol=1e-10, max_iter=k).coef, rtol=0, atol=0)
    assert fit.delta_loglik == pytest.approx(dls[k - 1], rel=0, abs=0)


def test_newton_cg_fit_reaches_the_mle(O):
    numpy_only(O, "H v products / truncated Newton")
    prob = tiny(400, 5, 3, 2, 1, seed=14)
    D = data_of(prob)
    exact = O.newton_fit(D, tol=1e-10)
    cg = O.newton_cg_fit(D, tol=1e-10)
    assert cg.status == O.MNL_OK and cg.cg_iters > 0
    assert np.linalg.norm(cg.coef - exact.coef) <= 1e-8 * np.linalg.norm(exact.coef)
    assert O.np.linalg.norm(O.gradient(D, cg.coef)) < 1e-10


def test_newton_cg_with_exhaustive_cg_is_the_newton_step(O):
    numpy_only(O, "H v products / truncated Newton")
    """CG run to a tiny residual solves (-H) delta = g: the iterates equal exact Newton's."""
    prob = tiny(300, 4, 2, 1, 1, seed=15)
    D = data_of(prob)
    exact = O.newton_fit(D, tol=1e-9)
    cg = O.newton_cg_fit(D, tol=1e-9, cg_rtol=1e-14)
    assert cg.iters == exact.iters
    assert [h["halvings"] for h in cg.history] == [h["halvings"] for h in exact.history]
    assert np.linalg.norm(cg.coef - exact.coef) <= 1e-10 * np.linalg.norm(exact.coef)


# --- standard errors and prediction ----------------

def test_std_errors_intercept_only_closed_form(O):
    # At the intercept-only MLE p_k = n_k / N and -H = N (diag(p) - p p^T) over k = 1..K-1, whose
    # inverse is (1/N)(diag(1/p_k) + (1/p_0) 1 1^T): se_k^2 = (1/N)(1/p_k + 1/p_0).
    pr = datagen.custom(700, 6, 0, seed=41, coef_sd=0.7)
    D = data_of(pr)
    n = np.bincount(D.choice, minlength=D.K).astype(float)
    th = np.log(n[1:] / n[0])
    se = O.std_errors(D, th)
    ph = n / D.N
    assert np.allclose(se, np.sqrt((1.0 / ph[1:] + 1.0 / ph[0]) / D.N), rtol=1e-12, atol=0)


def test_std_errors_K2_equal_logistic_regression(O):
    # K = 2: the inverse information of binary logistic regression on the textbook design
    pr = datagen.custom(300, 2, 2, f=1, d=1, seed=43, coef_sd=0.6)
    D = data_of(pr)
    th = datagen.draw(D.n_p, 13, 1, datagen.NORMAL, 0.4)
    W = np.hstack([np.ones((D.N, 1)), D.X, -D.Z[:, 0, :], D.Z[:, 1, :], D.Y[:, 1, :] - D.Y[:, 0, :]])
    s = expit(W @ th)
    info = (W.T * (s * (1 - s))) @ W
    assert np.allclose(O.std_errors(D, th), np.sqrt(np.diag(np.linalg.inv(info))), rtol=1e-11, atol=0)


def test_predict_rows_uniform_and_logistic(O):
    pr = tiny(N=120, K=5)
    D = data_of(pr)
    assert np.allclose(O.predict(D, np.zeros(D.n_p)), 1.0 / D.K, rtol=0, atol=1e-15)
    P = O.predict(D, pr.theta_true)
    assert np.allclose(P.sum(axis=1), 1.0, rtol=0, atol=1e-14) and P.min() > 0
    pr2 = datagen.custom(100, 2, 3, f=1, d=1, seed=44, coef_sd=0.6)
    D2 = data_of(pr2)
    W = np.hstack([np.ones((D2.N, 1)), D2.X, -D2.Z[:, 0, :], D2.Z[:, 1, :], D2.Y[:, 1, :] - D2.Y[:, 0, :]])
    assert np.allclose(O.predict(D2, pr2.theta_true)[:, 1], expit(W @ pr2.theta_true), rtol=1e-13, atol=0)


# --- the C oracle's own pieces (liboracle.so) ----------------------------------------------------

def test_c_cholesky_is_the_textbook_factor():
    # A = L L^T with L lower triangular and a positive diagonal is unique: equal to LAPACK's factor
    rng = np.random.default_rng(5)
    for n in (1, 7, 64, 131):
        B = rng.standard_normal((n, n))
        A = B @ B.T + n * np.eye(n)
        L = OC.cholesky(A)
        assert np.array_equal(L, np.tril(L)) and np.all(np.diag(L) > 0)
        assert np.linalg.norm(L @ L.T - A) <= 1e-14 * n * np.linalg.norm(A)
        assert np.linalg.norm(L - np.linalg.cholesky(A)) <= 1e-13 * np.linalg.norm(L)
    with pytest.raises(np.linalg.LinAlgError):
        OC.cholesky(np.array([[1.0, 2.0], [2.0, 1.0]]))


def test_c_oracle_line_search_margins_logged():
    # every accepted trial clears l - tau (margin >= 0), every rejected one is
    # below it (rejected_margin < 0); an overshooting start forces rejections
    pr = datagen.custom(200, 3, 1, seed=27, coef_sd=0.5)
    D = data_of(pr)
    fit = OC.newton_fit(D, coef0=np.full(D.n_p, 6.0), tol=1e-8)
    assert fit.status == OC.MNL_OK
    assert all(h["margin"] >= 0 for h in fit.history)
    rej = [h["rejected_margin"] for h in fit.history if h["halvings"] > 0]
    assert rej and all(m < 0 for m in rej)
    assert all(h["rejected_margin"] == np.inf for h in fit.history if h["halvings"] == 0)


def test_c_oracle_thread_count_does_not_change_results():
    pr = tiny(N=300, K=5, p=3, f=2, d=2, seed=31)
    D = data_of(pr)
    th = pr.theta_true
    n0 = OC.set_threads(0)
    try:
        OC.set_threads(1)
        a = OC.mnl_eval(D, th)
        OC.set_threads(3)
        b = OC.mnl_eval(D, th)
    finally:
        OC.set_threads(n0)
    assert a[0] == b[0] and np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])


@pytest.mark.parametrize("shape", [(300, 4, 3, 2, 1), (200, 7, 2, 3, 2), (250, 3, 5, 0, 0), (180, 5, 0, 2, 3)])
def test_numpy_and_c_oracles_agree(shape):
    # cross-check of two independent codings of the same definition (not a pin by itself)
    N, K, p, f, d = shape
    pr = tiny(N, K, p, f, d, seed=33)
    D = data_of(pr)
    th = datagen.perturbed_theta(pr, 0.3)
    l1, g1, H1 = ON.mnl_eval(D, th)
    l2, g2, H2 = OC.mnl_eval(D, th)
    assert abs(l1 - l2) <= 1e-14 * abs(l1)
    assert np.linalg.norm(g1 - g2) <= 1e-13 * np.linalg.norm(g1)
    assert np.linalg.norm(H1 - H2) <= 1e-13 * np.linalg.norm(H1)
    f1, f2 = ON.newton_fit(D, tol=1e-9), OC.newton_fit(D, tol=1e-9)
    assert f1.iters == f2.iters and [h["halvings"] for h in f1.history] == [h["halvings"] for h in f2.history]
    assert np.linalg.norm(f1.coef - f2.coef) <= 1e-12 * np.linalg.norm(f1.coef)


@pytest.mark.parametrize("cfg", ["c1", "c2", "c3", "c5"])
def test_golden_fit_r7_margins_and_oracles_agree(cfg):
    """R7 audit of the committed golden fits ("not lower than"): every
    accepted trial of the C oracle's fit clears l - tau by more than 1e-13 |l| and every rejected one
    misses it by more than that, so no accept/reject decision is a rounding tie; where the numpy
    oracle's golden fit also exists, both oracles took the same iterations and halvings and reached
    the same coefficients (1e-8)."""
    import json
    import os
    gdir = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    g = json.load(open(os.path.join(gdir, f"{cfg}_fit_c.json")))
    assert g["status"] == 0 and g["iters"] == len(g["history"])
    for h in g["history"]:
        assert h["margin"] > 1e-13, (cfg, h)
        if h["halvings"] > 0:
            assert h["rejected_margin"] < -1e-13, (cfg, h)
    pn = os.path.join(gdir, f"{cfg}_fit.json")
    if os.path.exists(pn):
        n = json.load(open(pn))
        assert n["iters"] == g["iters"] and n["halvings"] == g["halvings"]
        cn, cc = np.array(n["coef"]), np.array(g["coef"])
        assert np.linalg.norm(cn - cc) <= 1e-8 * np.linalg.norm(cc)
        assert abs(n["loglik"] - g["loglik"]) <= 1e-10 * abs(g["loglik"])
