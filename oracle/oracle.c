/* liboracle.so -- plain, slow, obviously correct CPU C oracle of the mnlogit Newton-Raphson hot
 * path: log-likelihood, gradient, Hessian and the Newton iteration of arXiv:1404.3177.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h). Shares no code with the CUDA path.
 *
 * Citations: P:n = PAPER.md line n (the paper's text; not present on the GPU box), S:n = SPEC.md,
 * R<n> = the readings of SURVEY.md §8(c) / DESIGN.md §3. Letters are the ABI's.
 *
 * WHAT IS COMPUTED. The paper's block method (Eq. "hessian block") reaches exactly, up to
 * rounding order, the plain definition of the derivatives of the log-likelihood, so this oracle is
 * that definition written out:
 *
 *   V_ik = normalized utility, V_i0 = 0:
 *          V_ik = xi_k + x_i.beta_k + z_ik.alpha_k - z_i0.alpha_0 + (y_ik - y_i0).gamma,  k >= 1
 *   P_ik = e^{V_ik} / sum_t e^{V_it}                                  (shift R12)
 *   l    = sum_i (V_{i,y_i} - log sum_k e^{V_ik})                     (Neumaier sum, R7)
 *   J_i  = the K x n_p Jacobian, J_i[k][r] = dV_ik / dtheta_r (row 0 is zero)
 *   g    = sum_i J_i^T (e_{y_i} - p_i)                                (App. A)
 *   H    = -sum_i J_i^T (diag p_i - p_i p_i^T) J_i                    (App. B)
 *   i.e. H[r][c] = sum_i ( u_ir u_ic - sum_k p_ik J_i[k][r] J_i[k][c] ),  u_i = J_i^T p_i,
 *
 * with the k-sums running over the nonzero entries of J_i only (every other term is a product with
 * an exact zero). Loops: rows r of H in parallel (OpenMP), individuals i in order, columns c >= r;
 * the lower triangle is the mirror. Memory is O(N (K + d + f) + n_p^2): P and the entries of u_i for
 * the columns with several nonzero J rows are stored per individual; no N x n_p array is formed.
 *
 * The Newton iteration follows the paper step by step with readings R7 (accept the
 * first l_j >= l - tau, tau = 1e-12 max(1,|l|)), R8 (at most 30 halvings), R9 (start 0), R10
 * (Euclidean ||g||_2 < tol), R11 (the stop test precedes forming H); the linear solve is the
 * textbook Cholesky-Banachiewicz factorisation of -H followed by two triangular solves.
 */
#include "oracle.h"

#include <math.h>
#include <omp.h>
#include <stdlib.h>
#include <string.h>

#define MAX_HALVINGS 30   /* R8 */
#define TAU_REL 1e-12     /* R7 */

typedef struct {
  int64_t N;
  int K, p, f, d, q, n_p, off_a, off_g;
  const double *X, *Y, *Z;
} prob_t;

static int make_prob(prob_t* D, int64_t N, int32_t K, int32_t p, int32_t f, int32_t d, const double* X,
                     const double* Y, const double* Z) {
  if (N < 1 || K < 2 || p < 0 || f < 0 || d < 0) return 0;
  if ((p > 0) != (X != NULL) || (f > 0) != (Y != NULL) || (d > 0) != (Z != NULL)) return 0;
  D->N = N; D->K = K; D->p = p; D->f = f; D->d = d;
  D->q = p + 1;
  D->off_a = (K - 1) * D->q;
  D->off_g = D->off_a + K * d;
  D->n_p = D->off_g + f;
  D->X = X; D->Y = Y; D->Z = Z;
  return 1;
}

/* ---- the model ------------------------------------------------------------------------------ */

/* Row i of V: Eq. "normalized utility" in ABI letters; the generic data are
 * differenced against the base, the base's alternative-specific term enters every V_ik. */
static void utility_row(const prob_t* D, int64_t i, const double* th, double* V) {
  const int K = D->K, p = D->p, f = D->f, d = D->d, q = D->q;
  const double* x = D->X ? D->X + i * p : NULL;
  const double* y = D->Y ? D->Y + i * K * f : NULL;
  const double* z = D->Z ? D->Z + i * K * d : NULL;
  V[0] = 0.0;
  for (int k = 1; k < K; ++k) {
    const double* b = th + (k - 1) * q;
    double v = b[0];                                           /* xi_k, the intercept */
    for (int a = 0; a < p; ++a) v += x[a] * b[1 + a];          /* x_i . beta_k */
    for (int c = 0; c < d; ++c)                                /* z_ik . alpha_k - z_i0 . alpha_0 */
      v += z[k * d + c] * th[D->off_a + k * d + c] - z[c] * th[D->off_a + c];
    for (int e = 0; e < f; ++e)                                /* (y_ik - y_i0) . gamma */
      v += (y[k * f + e] - y[e]) * th[D->off_g + e];
    V[k] = v;
  }
}

/* Softmax with the base alternative, shifted by m = max_k V_k (V_0 = 0 is included,
 * R12); returns log sum_k e^{V_k}. */
static double softmax_row(int K, const double* V, double* P) {
  double m = V[0];
  for (int k = 1; k < K; ++k) m = V[k] > m ? V[k] : m;
  double s = 0.0;
  for (int k = 0; k < K; ++k) s += exp(V[k] - m);
  for (int k = 0; k < K; ++k) P[k] = exp(V[k] - m) / s;
  return m + log(s);
}

/* Column r of J_i as its nonzero rows: J_i[ks[j]][r] = vals[j], j < return value.
 *   r in beta_k  (entry a of chunk k):  x~_ia (x~_i0 = 1, the intercept), row k only
 *   r in alpha_k, k >= 1 (entry c):     z_ikc, row k only
 *   r in alpha_0 (entry c):             -z_i0c in every row k >= 1
 *   r in gamma (entry e):               y_ike - y_i0e in every row k >= 1 */
static int jac_col(const prob_t* D, int64_t i, int r, int* ks, double* vals) {
  const int K = D->K, q = D->q, d = D->d, f = D->f;
  if (r < D->off_a) {
    const int k = r / q + 1, a = r % q;
    ks[0] = k;
    vals[0] = a == 0 ? 1.0 : D->X[i * D->p + a - 1];
    return 1;
  }
  if (r < D->off_g) {
    const int k = (r - D->off_a) / d, c = (r - D->off_a) % d;
    const double* z = D->Z + i * K * d;
    if (k >= 1) {
      ks[0] = k;
      vals[0] = z[k * d + c];
      return 1;
    }
    for (int t = 1; t < K; ++t) { ks[t - 1] = t; vals[t - 1] = -z[c]; }
    return K - 1;
  }
  const int e = r - D->off_g;
  const double* y = D->Y + i * K * f;
  for (int t = 1; t < K; ++t) { ks[t - 1] = t; vals[t - 1] = y[t * f + e] - y[e]; }
  return K - 1;
}

/* Neumaier-compensated sum of t[0..n) in index order (R7). */
static double neumaier(const double* t, int64_t n) {
  double s = 0.0, c = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double v = s + t[i];
    c += fabs(s) >= fabs(t[i]) ? (s - v) + t[i] : (t[i] - v) + s;
    s = v;
  }
  return s + c;
}

/* P[N][K] at theta and l (Neumaier over the per-individual terms, in order). Returns 0 if a
 * choice is out of range. */
static int probs_and_loglik(const prob_t* D, const int32_t* choice, const double* th, double* P,
                            double* l_out) {
  const int64_t N = D->N;
  const int K = D->K;
  double* term = (double*)malloc(sizeof(double) * N);
  int bad = 0;
#pragma omp parallel
  {
    double* V = (double*)malloc(sizeof(double) * K);
    double* Pl = (double*)malloc(sizeof(double) * K);
#pragma omp for schedule(static) reduction(| : bad)
    for (int64_t i = 0; i < N; ++i) {
      utility_row(D, i, th, V);
      double* Pi = P ? P + i * K : Pl;
      const double lse = softmax_row(K, V, Pi);
      const int y = choice[i];
      if (y < 0 || y >= K) { bad |= 1; term[i] = 0.0; continue; }
      term[i] = V[y] - lse;                       /* Eq. "log-lik function" */
    }
    free(V);
    free(Pl);
  }
  *l_out = neumaier(term, N);
  free(term);
  return !bad;
}

/* g_r = sum_i sum_k J_i[k][r] ([y_i = k] - P_ik), rows r in parallel, i in order. */
static void gradient(const prob_t* D, const int32_t* choice, const double* P, double* g) {
  const int K = D->K;
#pragma omp parallel
  {
    int* ks = (int*)malloc(sizeof(int) * K);
    double* vals = (double*)malloc(sizeof(double) * K);
#pragma omp for schedule(dynamic, 1)
    for (int r = 0; r < D->n_p; ++r) {
      double s = 0.0;
      for (int64_t i = 0; i < D->N; ++i) {
        const int nz = jac_col(D, i, r, ks, vals);
        for (int j = 0; j < nz; ++j) s += vals[j] * ((choice[i] == ks[j] ? 1.0 : 0.0) - P[i * K + ks[j]]);
      }
      g[r] = s;
    }
    free(ks);
    free(vals);
  }
}

/* Row r of H, columns c >= r, summed over the individuals in order:
 *   H[r][c] = sum_i ( u_ir u_ic - sum_k P_ik J_i[k][r] J_i[k][c] ),  u_ic = sum_k P_ik J_i[k][c].
 * Column blocks in theta order, each with the nonzero rows of its J columns (jac_col):
 *   beta_l / alpha_l (l >= 1): one nonzero row l with value m_b (x~_i or z_il), so
 *       u_ic = P_il m_b  and  sum_k P_ik J[k][r] J[k][c] = P_il J[l][r] m_b
 *       -> H[r][c] += P_il (u_ir - J[l][r]) m_b
 *   alpha_0 / gamma (rows 1..K-1): u_ic is read from Ug (formed by its definition per individual,
 *       below) and the k-sum runs over the nonzero rows of column r.
 * Compiled for AVX-512 / AVX2 / baseline, chosen at load time -- only the instruction set differs,
 * not the arithmetic or its order (no contraction: -std=c11). */
__attribute__((target_clones("arch=x86-64-v4", "arch=x86-64-v3", "default")))
static void hessian_row(const prob_t* D, const double* P, const double* Ug, int r, double* acc, double* Jr,
                        double* xt, int* ks, double* vals) {
  const int K = D->K, q = D->q, d = D->d, f = D->f, n = D->n_p, ng = d + f;
  for (int c = r; c < n; ++c) acc[c] = 0.0;
  for (int64_t i = 0; i < D->N; ++i) {
    const double* Pi = P + i * K;
    const double* z = d ? D->Z + i * K * d : NULL;
    const double* y = f ? D->Y + i * K * f : NULL;
    const double* ug = Ug + i * ng;   /* u_ic for c in alpha_0 (d), then gamma (f) */
    xt[0] = 1.0;
    for (int a = 1; a < q; ++a) xt[a] = D->X[i * D->p + a - 1];
    for (int k = 0; k < K; ++k) Jr[k] = 0.0;
    const int nz = jac_col(D, i, r, ks, vals);
    double ur = 0.0;
    for (int j = 0; j < nz; ++j) { Jr[ks[j]] = vals[j]; ur += Pi[ks[j]] * vals[j]; }
    /* beta_l blocks: columns (l-1)q .. lq-1 */
    for (int l = 1; l < K; ++l) {
      const int c0 = (l - 1) * q;
      if (c0 + q <= r) continue;
      const double t = Pi[l] * (ur - Jr[l]);
      double* a = acc + c0;
      for (int b = r > c0 ? r - c0 : 0; b < q; ++b) a[b] += t * xt[b];
    }
    if (d) {
      /* alpha_0 block: J[k][c] = -z_i0c for every k >= 1 */
      for (int c = 0; c < d; ++c) {
        const int col = D->off_a + c;
        if (col < r) continue;
        double s = 0.0;
        for (int j = 0; j < nz; ++j) s += Pi[ks[j]] * vals[j] * (-z[c]);
        acc[col] += ur * ug[c] - s;
      }
      /* alpha_l blocks, l >= 1 */
      for (int l = 1; l < K; ++l) {
        const int c0 = D->off_a + l * d;
        if (c0 + d <= r) continue;
        const double t = Pi[l] * (ur - Jr[l]);
        const double* m = z + l * d;
        double* a = acc + c0;
        for (int b = r > c0 ? r - c0 : 0; b < d; ++b) a[b] += t * m[b];
      }
    }
    /* gamma block: J[k][c] = y_ike - y_i0e for every k >= 1 */
    for (int e = 0; e < f; ++e) {
      const int col = D->off_g + e;
      if (col < r) continue;
      double s = 0.0;
      for (int j = 0; j < nz; ++j) s += Pi[ks[j]] * vals[j] * (y[ks[j] * f + e] - y[e]);
      acc[col] += ur * ug[d + e] - s;
    }
  }
}

/* H (full, exactly symmetric): rows in parallel, then the lower triangle mirrored. */
static void hessian(const prob_t* D, const double* P, double* H) {
  const int K = D->K, d = D->d, f = D->f, n = D->n_p, ng = d + f;
  /* u_ic = sum_{k>=1} P_ik J_i[k][c] for the columns with several nonzero rows (alpha_0, gamma) */
  double* Ug = (double*)malloc(sizeof(double) * (D->N * ng + 1));
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < D->N; ++i) {
    const double* Pi = P + i * K;
    for (int c = 0; c < d; ++c) {
      double u = 0.0;
      for (int k = 1; k < K; ++k) u += Pi[k] * (-D->Z[i * K * d + c]);
      Ug[i * ng + c] = u;
    }
    for (int e = 0; e < f; ++e) {
      const double* y = D->Y + i * K * f;
      double u = 0.0;
      for (int k = 1; k < K; ++k) u += Pi[k] * (y[k * f + e] - y[e]);
      Ug[i * ng + d + e] = u;
    }
  }
#pragma omp parallel
  {
    double* acc = (double*)malloc(sizeof(double) * n);
    double* Jr = (double*)malloc(sizeof(double) * K);   /* column r of J_i, dense over k */
    double* xt = (double*)malloc(sizeof(double) * D->q); /* x~_i = [1, x_i] */
    int* ks = (int*)malloc(sizeof(int) * K);
    double* vals = (double*)malloc(sizeof(double) * K);
#pragma omp for schedule(dynamic, 1)
    for (int r = 0; r < n; ++r) {
      hessian_row(D, P, Ug, r, acc, Jr, xt, ks, vals);
      for (int c = r; c < n; ++c) H[(int64_t)r * n + c] = acc[c];
    }
    free(acc); free(Jr); free(xt); free(ks); free(vals);
  }
  free(Ug);
  for (int r = 0; r < n; ++r)
    for (int c = 0; c < r; ++c) H[(int64_t)r * n + c] = H[(int64_t)c * n + r];
}

/* ---- linear algebra (textbook) ---------------------------------------------------------------- */

int oracle_cholesky(int32_t n, double* A) {
  if (n < 1 || !A) return ORACLE_ERR_ARG;
  /* Cholesky-Banachiewicz, row-major lower: L_jj = sqrt(A_jj - sum_k L_jk^2),
   * L_ij = (A_ij - sum_k L_ik L_jk) / L_jj for i > j (the i loop in parallel). */
  for (int j = 0; j < n; ++j) {
    double* Lj = A + (int64_t)j * n;
    double s = Lj[j];
    for (int k = 0; k < j; ++k) s -= Lj[k] * Lj[k];
    if (!(s > 0.0) || !isfinite(s)) return ORACLE_ERR_NOT_SPD;
    const double ljj = sqrt(s);
    Lj[j] = ljj;
#pragma omp parallel for schedule(static)
    for (int i = j + 1; i < n; ++i) {
      double* Li = A + (int64_t)i * n;
      double t = Li[j];
      for (int k = 0; k < j; ++k) t -= Li[k] * Lj[k];
      Li[j] = t / ljj;
    }
  }
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j) A[(int64_t)i * n + j] = 0.0;
  return ORACLE_OK;
}

int oracle_cholesky_solve(int32_t n, const double* L, const double* b, double* x) {
  if (n < 1 || !L || !b || !x) return ORACLE_ERR_ARG;
  double* y = (double*)malloc(sizeof(double) * n);
  for (int i = 0; i < n; ++i) {          /* L y = b */
    double s = b[i];
    for (int k = 0; k < i; ++k) s -= L[(int64_t)i * n + k] * y[k];
    y[i] = s / L[(int64_t)i * n + i];
  }
  for (int i = n - 1; i >= 0; --i) {     /* L^T x = y */
    double s = y[i];
    for (int k = i + 1; k < n; ++k) s -= L[(int64_t)k * n + i] * x[k];
    x[i] = s / L[(int64_t)i * n + i];
  }
  free(y);
  return ORACLE_OK;
}

/* ---- exported evaluation ---------------------------------------------------------------------- */

int oracle_set_threads(int32_t n) {
  if (n > 0) omp_set_num_threads(n);
  return omp_get_max_threads();
}

int oracle_num_threads(void) { return omp_get_max_threads(); }

int oracle_mnl_utilities(int64_t N, int32_t K, int32_t p, int32_t f, int32_t d, const double* X,
                         const double* Y, const double* Z, const double* coef, double* V) {
  prob_t D;
  if (!make_prob(&D, N, K, p, f, d, X, Y, Z) || !coef || !V) return ORACLE_ERR_ARG;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < N; ++i) utility_row(&D, i, coef, V + i * K);
  return ORACLE_OK;
}

int oracle_mnl_softmax(int64_t N, int32_t K, const double* V, double* P, double* lse) {
  if (N < 1 || K < 1 || !V || !P) return ORACLE_ERR_ARG;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < N; ++i) {
    const double l = softmax_row(K, V + i * K, P + i * K);
    if (lse) lse[i] = l;
  }
  return ORACLE_OK;
}

int oracle_mnl_eval(int64_t N, int32_t K, int32_t p, int32_t f, int32_t d, const double* X,
                    const double* Y, const double* Z, const int32_t* choice, const double* coef,
                    double* loglik, double* grad, double* hess) {
  prob_t D;
  if (!make_prob(&D, N, K, p, f, d, X, Y, Z) || !choice || !coef || !loglik) return ORACLE_ERR_ARG;
  double* P = (double*)malloc(sizeof(double) * N * K);
  if (!P) return ORACLE_ERR_ARG;
  double l = 0.0;
  if (!probs_and_loglik(&D, choice, coef, P, &l)) { free(P); return ORACLE_ERR_ARG; }
  *loglik = l;
  if (grad) gradient(&D, choice, P, grad);
  if (hess) hessian(&D, P, hess);
  free(P);
  return isfinite(l) ? ORACLE_OK : ORACLE_ERR_NONFINITE;
}

/* ---- Newton-Raphson ----------------------------------------------------------------- */

int oracle_mnl_newton_fit_log(int64_t N, int32_t K, int32_t p, int32_t f, int32_t d, const double* X,
                              const double* Y, const double* Z, const int32_t* choice, const double* coef0,
                              double tol, int32_t max_iter, double ftol, double* coef, int32_t* iters_out,
                              double* loglik_out, double* grad_norm_out, int32_t* stop_out, oracle_iter_log* log,
                              int32_t log_cap) {
  prob_t D;
  if (!make_prob(&D, N, K, p, f, d, X, Y, Z) || !choice || !coef || !iters_out || !loglik_out || !(tol > 0.0) ||
      max_iter < 0 || !(ftol >= 0.0))
    return ORACLE_ERR_ARG;
  const int n = D.n_p;
  double* theta = (double*)malloc(sizeof(double) * n);
  double* trial = (double*)malloc(sizeof(double) * n);
  double* g = (double*)malloc(sizeof(double) * n);
  double* delta = (double*)malloc(sizeof(double) * n);
  double* A = (double*)malloc(sizeof(double) * n * n);
  double* P = (double*)malloc(sizeof(double) * N * K);
  for (int r = 0; r < n; ++r) theta[r] = coef0 ? coef0[r] : 0.0;   /* R9 */
  int status = ORACLE_OK, stop = 0, iters = 0, ftol_met = 0;
  double l = 0.0, gnorm = NAN;
  for (;;) {
    if (!probs_and_loglik(&D, choice, theta, P, &l)) { status = ORACLE_ERR_ARG; break; }
    if (!isfinite(l)) { status = ORACLE_ERR_NONFINITE; break; }
    gradient(&D, choice, P, g);
    double g2 = 0.0;
    for (int r = 0; r < n; ++r) g2 += g[r] * g[r];
    gnorm = sqrt(g2);
    /* stopping set, first met: gtol before forming H (R10, R11), ftol after
     * an accepted update, then max_iter */
    if (gnorm < tol) { stop = 1; break; }
    if (ftol_met) { stop = 2; break; }
    if (iters == max_iter) { status = ORACLE_MAXITER; stop = 3; break; }
    hessian(&D, P, A);
    for (int64_t e = 0; e < (int64_t)n * n; ++e) A[e] = -A[e];     /* -H, SPD by concavity */
    if (oracle_cholesky(n, A) != ORACLE_OK) { status = ORACLE_ERR_NOT_SPD; break; }
    oracle_cholesky_solve(n, A, g, delta);                        /* (-H) delta = g */
    /* step halving: the first theta + delta / 2^j with l_j "not lower than" l (R7, R8) */
    const double tau = TAU_REL * (fabs(l) > 1.0 ? fabs(l) : 1.0);
    const double scale = fabs(l) > 1.0 ? fabs(l) : 1.0;
    double lj = 0.0, rej = INFINITY;
    int j, accepted = 0;
    for (j = 0; j <= MAX_HALVINGS; ++j) {
      for (int r = 0; r < n; ++r) trial[r] = theta[r] + ldexp(delta[r], -j);
      probs_and_loglik(&D, choice, trial, NULL, &lj);
      if (isfinite(lj) && lj >= l - tau) { accepted = 1; break; }
      rej = isfinite(lj) ? (lj - (l - tau)) / scale : -INFINITY;
    }
    if (!accepted) { status = ORACLE_ERR_LINESEARCH; break; }
    if (log && iters < log_cap) {
      oracle_iter_log* e = log + iters;
      e->loglik = l; e->grad_norm = gnorm; e->loglik_new = lj; e->halvings = j;
      e->margin = (lj - (l - tau)) / scale;
      e->rejected_margin = rej;
      e->pad_ = 0;
    }
    ftol_met = ftol > 0.0 && fabs(lj - l) < ftol;
    memcpy(theta, trial, sizeof(double) * n);
    l = lj;
    ++iters;
  }
  memcpy(coef, theta, sizeof(double) * n);
  *iters_out = iters;
  *loglik_out = l;
  if (grad_norm_out) *grad_norm_out = gnorm;
  if (stop_out) *stop_out = stop;
  free(theta); free(trial); free(g); free(delta); free(A); free(P);
  return status;
}

int oracle_mnl_newton_fit(int64_t N, int32_t K, int32_t p, int32_t f, int32_t d, const double* X,
                          const double* Y, const double* Z, const int32_t* choice, const double* coef0,
                          double tol, int32_t max_iter, double* coef, int32_t* iters, double* loglik) {
  return oracle_mnl_newton_fit_log(N, K, p, f, d, X, Y, Z, choice, coef0, tol, max_iter, 0.0, coef, iters, loglik,
                                   NULL, NULL, NULL, 0);
}
