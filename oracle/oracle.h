/* liboracle.so -- plain CPU C oracle of the mnlogit Newton-Raphson hot path.
 *
 * TEST INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs load it; the product path (paper_1404_3177_b200/) never does. It shares no
 * code, header, table or constant with libmnl.so (the CUDA path); the status numbers below are
 * restated from SURVEY.md §8(b), not included from include/mnl.h.
 *
 * Every pointer is a HOST pointer; arrays are row-major and caller-owned:
 *   X [N][p]      individual-specific data (intercept implicit)          NULL iff p == 0
 *   Y [N][K][f]   alternative-varying data, one generic coefficient gamma NULL iff f == 0
 *   Z [N][K][d]   alternative-varying data, alternative-specific alpha_k  NULL iff d == 0
 *   choice [N]    0..K-1, 0 = the base alternative
 *   coef [n_p]    [beta_1 | ... | beta_{K-1} | alpha_0 | ... | alpha_{K-1} | gamma],
 *                 beta_k = [xi_k, beta_k1 .. beta_kp]  (Eq. "theta vec")
 * n_p = (K-1)(p+1) + K d + f.  Letters are the ABI's (the paper's Y and Z swapped).
 *
 * Threads: OpenMP (OMP_NUM_THREADS, or oracle_set_threads). Results do not depend on the thread
 * count: every reduction runs in a fixed order. */
#ifndef MNL_ORACLE_H
#define MNL_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORACLE_OK = 0, ORACLE_ERR_ARG = 1, ORACLE_ERR_NOT_SPD = 3, ORACLE_ERR_LINESEARCH = 4,
       ORACLE_ERR_NONFINITE = 5, ORACLE_MAXITER = 6 };

/* One accepted Newton update (the parity audit of SURVEY.md §8(c) R7): loglik and ||g||_2 before
 * the update, halvings j, loglik after, margin = (l_new - (l - tau)) / max(1,|l|), i.e. how far the
 * accepted trial cleared the acceptance threshold; rejected_margin = the same for the last rejected
 * trial (j > 0), else +inf. */
typedef struct {
  double loglik, grad_norm, loglik_new, margin, rejected_margin;
  int32_t halvings;
  int32_t pad_;
} oracle_iter_log;

int oracle_set_threads(int32_t n);   /* 0 -> OpenMP default; returns the count in effect */
int oracle_num_threads(void);

/* V[N][K] (V_i0 = 0): Eq. "normalized utility". */
int oracle_mnl_utilities(int64_t N, int32_t K, int32_t p, int32_t f, int32_t d, const double* X,
                         const double* Y, const double* Z, const double* coef, double* V);
/* P[N][K] from V[N][K]: Eqs. "probability"/"base probability", PAPER.md:140-152 (shifted, R12);
 * lse[N] (may be NULL) = log sum_k e^{V_ik}. */
int oracle_mnl_softmax(int64_t N, int32_t K, const double* V, double* P, double* lse);

/* loglik, grad (NULL or [n_p]), hess (NULL or [n_p][n_p],
 * PAPER.md:380, App. B 731-776), all at coef. Returns ORACLE_ERR_ARG on bad sizes/pointers or a
 * choice outside [0,K), ORACLE_ERR_NONFINITE if l is not finite (outputs still written). */
int oracle_mnl_eval(int64_t N, int32_t K, int32_t p, int32_t f, int32_t d, const double* X,
                    const double* Y, const double* Z, const int32_t* choice, const double* coef,
                    double* loglik, double* grad, double* hess);

/* Newton-Raphson with step halving from coef0 (NULL -> 0), stopping at
 * ||g||_2 < tol (tested before forming H), |l_t - l_(t-1)| < ftol after an accepted update
 * (ftol = 0: off), or iters == max_iter (ORACLE_MAXITER). Outputs coef [n_p], iters, loglik. */
int oracle_mnl_newton_fit(int64_t N, int32_t K, int32_t p, int32_t f, int32_t d, const double* X,
                          const double* Y, const double* Z, const int32_t* choice, const double* coef0,
                          double tol, int32_t max_iter, double* coef, int32_t* iters, double* loglik);
/* The same with ftol, the final ||g||_2 and stop reason (1 gtol, 2 ftol, 3 maxiter, 0 error), and
 * the per-iteration log (up to log_cap entries; NULL allowed). */
int oracle_mnl_newton_fit_log(int64_t N, int32_t K, int32_t p, int32_t f, int32_t d, const double* X,
                              const double* Y, const double* Z, const int32_t* choice, const double* coef0,
                              double tol, int32_t max_iter, double ftol, double* coef, int32_t* iters,
                              double* loglik, double* grad_norm, int32_t* stop_reason, oracle_iter_log* log,
                              int32_t log_cap);

/* In-place lower Cholesky A = L L^T of the SPD n x n row-major matrix (upper triangle zeroed);
 * ORACLE_ERR_NOT_SPD on a non-positive pivot. Then x = (L L^T)^{-1} b. */
int oracle_cholesky(int32_t n, double* A);
int oracle_cholesky_solve(int32_t n, const double* L, const double* b, double* x);

#ifdef __cplusplus
}
#endif
#endif
