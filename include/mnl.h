/* mnl.h — C ABI of the B200 (sm_100a) multinomial-logit Newton-Raphson hot path.
 *
 * The operations follow the paper's statement of the problem (arXiv:1404.3177,
 * `P:n` = PAPER.md line n; section / equation named beside each):
 *   utility          Eq. "unormalized utility" P:104-107 and "normalized utility" P:129-138
 *   probabilities    Eqs. "probability" / "base probability" P:140-152
 *   log-likelihood   Eq. "log-lik function" P:348-351
 *   gradient         Eq. "loglik gradient" P:433-443 (App. A)
 *   Hessian          Eq. "hessian block" P:462-476 (App. A), symmetry P:484
 *   Newton step      Eq. "NR update" P:361-367, step halving P:367-371, stopping P:219-220
 *
 * LETTERS (SURVEY.md §0.3 — the ABI swaps the paper's Y and Z):
 *   U_ik = xi_k + x_i.beta_k + y_ik.gamma + z_ik.alpha_k        (alternative 0 is the base:
 *                                                                xi_0 = 0, beta_0 = 0)
 *   X[N][p]     individual-specific data, alternative-specific coefs beta_k (k = 1..K-1) plus an
 *               implicit intercept xi_k (a unity-valued column), never stored in X
 *   Y[N][K][f]  alternative-varying data with ONE generic coefficient vector gamma (paper's Z/alpha)
 *   Z[N][K][d]  alternative-varying data with alternative-specific coefficients alpha_k,
 *               k = 0..K-1, the base included (paper's Y/gamma_k)
 *
 * COEFFICIENT LAYOUT (Eq. "theta vec"), n_p = (K-1)(p+1) + K d + f:
 *   theta = [ beta_1 | ... | beta_{K-1} | alpha_0 | ... | alpha_{K-1} | gamma ]
 *   beta_k = [ xi_k, beta_k1 .. beta_kp ]
 *   off_beta(k) = (k-1)(p+1),  off_alpha(k) = (K-1)(p+1) + k d,  off_gamma = (K-1)(p+1) + K d
 *
 * CONVENTIONS. All arrays are row-major and C-contiguous. Floating point is IEEE fp64 end to end.
 * `grad` and `hess` are derivatives of l itself (hess is negative definite).
 * `hess` is the full symmetric n_p x n_p matrix, exactly symmetric (mirrored).
 * Results are deterministic run to run (fixed-order reductions, no floating-point atomics).
 *
 * OWNERSHIP. The caller owns every buffer passed in. Device pointers must be 16-byte aligned
 * (torch allocations are). The library owns its scratch (probabilities, packed design rows,
 * split-N partial tiles, Cholesky workspace), cached per (device, stream) and freed by
 * mnl_release().
 *
 * SYNCHRONISATION. Every call enqueues on `stream` (a cudaStream_t; NULL = legacy default
 * stream) of the CURRENT device, synchronises that stream before returning (mnl_eval_async
 * excepted), and returns a final status code.
 *
 * THREADING. Reentrant across distinct streams: each (device, stream) pair has its own scratch
 * and lock, so calls on different streams (from any threads, on any devices) run concurrently;
 * calls on the same stream are serialised. The host-buffer entry points share one internal
 * stream per device. mnl_release() must not overlap any other call.
 *
 * SIZE LIMITS OF THIS BUILD (MNL_ERR_ARG beyond them): 2 <= K <= 256, 0 <= d <= 64, 0 <= f <= 64,
 * 1 <= N < 2^31, n_p <= 16384, and p bounded by the pass-1 kernel's register-resident beta-gradient
 * accumulators: p + 1 <= 128 for K <= 32, <= 64 for K <= 128, <= 32 for K <= 256; plus its per-CTA
 * shared memory (<= 227 KB; the gradient partials of many alternative-varying variables move to
 * global scratch). mnl_check_shape() tells whether a shape is supported without touching a device.
 */
#ifndef MNL_H_
#define MNL_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  MNL_OK = 0,             /* success */
  MNL_ERR_ARG = 1,        /* bad argument: sizes, NULL pointer, misalignment, tol <= 0,
                             max_iter < 0, a choice outside [0, K) (checked on device) */
  MNL_ERR_CUDA = 2,       /* a CUDA runtime error (allocation, launch) */
  MNL_ERR_NOT_SPD = 3,    /* Cholesky of -H failed: the singular-design case of P:777-790;
                             the paper advises relaxing tolerances */
  MNL_ERR_LINESEARCH = 4, /* more than 30 step halvings without a non-decreasing loglik */
  MNL_ERR_NONFINITE = 5,  /* non-finite coefficient or log-likelihood */
  MNL_MAXITER = 6         /* warning class: max_iter Newton updates taken; outputs are valid */
} mnl_status;

/* n_p = (K-1)(p+1) + K*d + f, or -1 for K < 2 or negative sizes. */
int64_t mnl_num_params(int32_t K, int32_t p, int32_t f, int32_t d);

/* MNL_OK if every entry point supports the shape (N, K, p, f, d) in this build, else MNL_ERR_ARG
 * (the size limits above, including the pass-1 shared-memory bound). No device is needed. */
int mnl_check_shape(int64_t N, int32_t K, int32_t p, int32_t f, int32_t d);

/* One evaluation at `coef`: log-likelihood, gradient and, when
 * `hess` != NULL, the full Hessian.
 *   X      dev [N][p]     NULL iff p == 0
 *   Y      dev [N][K][f]  NULL iff f == 0
 *   Z      dev [N][K][d]  NULL iff d == 0
 *   choice dev [N]        int32 in [0, K), 0 = base alternative
 *   coef   dev [n_p]
 *   loglik dev [1]        out
 *   grad   dev [n_p]      out, or NULL
 *   hess   dev [n_p*n_p]  out, or NULL
 * Errors: MNL_ERR_ARG, MNL_ERR_CUDA, MNL_ERR_NONFINITE (non-finite loglik). */
int mnl_eval(int64_t N, int32_t K, int32_t p, int32_t f, int32_t d,
             const double* X, const double* Y, const double* Z, const int32_t* choice,
             const double* coef, double* loglik, double* grad, double* hess, void* stream);

/* Asynchronous mnl_eval: enqueues the same kernels on `stream` and returns without synchronising.
 *   status  dev int32 [1] out, written on the stream after the pass: MNL_OK, MNL_ERR_ARG (a choice
 *           outside [0, K)) or MNL_ERR_NONFINITE (non-finite loglik)
 * Host-side argument errors (sizes, NULL pointers, misalignment) are returned immediately; the
 * return value MNL_OK means "enqueued". The first call for a problem shape allocates library
 * scratch (which synchronises); later calls of the same shape launch only. The scratch belongs to
 * `stream`'s workspace, so asynchronous calls on different streams may overlap; consecutive calls
 * on one stream are ordered by the stream. */
int mnl_eval_async(int64_t N, int32_t K, int32_t p, int32_t f, int32_t d,
                   const double* X, const double* Y, const double* Z, const int32_t* choice,
                   const double* coef, double* loglik, double* grad, double* hess, int32_t* status,
                   void* stream);

/* Newton-Raphson maximum-likelihood fit.
 *   coef0   dev [n_p] start, or NULL => zeros (reading R9)
 *   tol     ||grad||_2 threshold (gtol; reading R10), > 0
 *   max_iter >= 0 Newton updates; 0 => evaluate only
 *   coef    dev [n_p] out (may alias coef0)
 *   iters   host out: accepted Newton updates
 *   loglik  host out: l at the returned coef
 * Each iteration: (l, g) at theta; stop if ||g|| < tol (before forming H, reading R11) or if
 * iters == max_iter (MNL_MAXITER); H; Cholesky of -H (MNL_ERR_NOT_SPD); delta = (-H)^{-1} g;
 * accept the first theta + delta/2^j, j = 0..30, with l_j >= l - 1e-12 max(1,|l|) (reading R7);
 * else MNL_ERR_LINESEARCH. */
int mnl_newton_fit(int64_t N, int32_t K, int32_t p, int32_t f, int32_t d,
                   const double* X, const double* Y, const double* Z, const int32_t* choice,
                   const double* coef0, double tol, int32_t max_iter,
                   double* coef, int32_t* iters, double* loglik, void* stream);

/* Per-fit report (the paper's est.stat). */
typedef struct {
  int32_t iters;            /* accepted Newton updates */
  int32_t halvings;         /* total step halvings (the paper's "linesearch iterations") */
  int32_t evals;            /* log-likelihood evaluations */
  int32_t status;
  double grad_norm;         /* ||g||_2 at the returned coef */
  double loglik;
  double hess_ms;           /* device time in Hessian assembly, summed over iterations */
  double chol_ms;           /* device time in Cholesky factor + solves */
  double eval_ms;           /* device time in log-likelihood / gradient passes */
  double total_ms;          /* wall time of the call */
  double gemm_ms;           /* device time of the beta-beta DMMA GEMMs (J1 + tail), summed */
  int32_t halvings_per_iter[64];  /* first 64 iterations */
  double delta_loglik;      /* |l_t - l_(t-1)| of the last accepted update (0 without one) */
  int32_t stop_reason;      /* mnl_stop_reason */
  int32_t cg_iters;         /* total conjugate-gradient iterations (method MNL_METHOD_CG) */
  double min_margin;        /* R7 audit: min over every line-search decision (accepted or rejected) of
                               |l_j - (l - tau)| / max(1,|l|); a decision closer than ~1e-13 to its
                               threshold could flip under a different summation order (+inf if none) */
  double loglik_per_iter[64];     /* l at the iterate that starts Newton iteration t (t < min(iters, 64)) */
  double grad_norm_per_iter[64];  /* ||g||_2 at that iterate (before its Hessian is formed) */
} mnl_fit_stats;

/* Why a fit stopped: the first of the paper's three conditions met. */
typedef enum {
  MNL_STOP_NONE = 0,        /* an error status ended the fit */
  MNL_STOP_GTOL = 1,        /* ||g||_2 < gtol */
  MNL_STOP_FTOL = 2,        /* |l_t - l_(t-1)| < ftol after an accepted update */
  MNL_STOP_MAXITER = 3      /* max_iter updates taken (status MNL_MAXITER) */
} mnl_stop_reason;

typedef enum {
  MNL_METHOD_NEWTON = 0,    /* exact Hessian + Cholesky (the paper's method) */
  MNL_METHOD_CG = 1         /* truncated Newton: conjugate gradients on Hessian-vector products,
                               H never formed (the paper's stated extension) */
} mnl_method;

/* Options of mnl_newton_fit_opts. */
typedef struct {
  double gtol;              /* ||g||_2 threshold, > 0 (reading R10) */
  double ftol;              /* |l_t - l_(t-1)| threshold tested after each accepted update; 0 = off */
  int32_t max_iter;         /* >= 0 Newton updates */
  int32_t method;           /* mnl_method */
  int32_t cg_max_iter;      /* MNL_METHOD_CG: CG iterations per Newton step; 0 => n_p */
  double cg_rtol;           /* MNL_METHOD_CG: stop CG at ||r|| <= cg_rtol ||g||; 0 => min(0.5, sqrt(||g||)) */
} mnl_fit_options;

/* mnl_newton_fit plus the report (stats may be NULL). */
int mnl_newton_fit_ex(int64_t N, int32_t K, int32_t p, int32_t f, int32_t d,
                      const double* X, const double* Y, const double* Z, const int32_t* choice,
                      const double* coef0, double tol, int32_t max_iter,
                      double* coef, int32_t* iters, double* loglik, mnl_fit_stats* stats,
                      void* stream);

/* The fit with the paper's full stopping set (gtol, ftol, maxiter: the first met ends it) and a
 * choice of Newton step (mnl_method). With MNL_METHOD_NEWTON and ftol = 0 it is mnl_newton_fit_ex.
 * MNL_METHOD_CG solves (-H) delta = g approximately by conjugate gradients with one
 * mnl_hessvec-style product per CG iteration (never forming H; memory O(N (K + f) + n_p)), then
 * takes the same step-halving line search; MNL_ERR_NOT_SPD if a CG curvature p'(-H)p <= 0 occurs
 * before any progress. opts must be non-NULL. */
int mnl_newton_fit_opts(int64_t N, int32_t K, int32_t p, int32_t f, int32_t d,
                        const double* X, const double* Y, const double* Z, const int32_t* choice,
                        const double* coef0, const mnl_fit_options* opts,
                        double* coef, int32_t* iters, double* loglik, mnl_fit_stats* stats, void* stream);

/* Element-wise sum of `count` doubles of the DEVICE buffer `buf` across all ranks of the caller's
 * process group, in place, ordered on `stream` (a cudaStream_t) -- e.g. ncclAllReduce(ncclSum) or
 * torch.distributed.all_reduce. Every rank must receive bitwise-identical sums (true of NCCL and of
 * any reduction that computes once and broadcasts). Return 0 on success. */
typedef int (*mnl_allreduce_fn)(double* buf, int64_t count, void* stream, void* ctx);

/* Data-parallel Newton-Raphson fit over individuals: l, g and H are
 * sums over individuals, so each rank passes ITS OWN individuals
 * (N, X, Y, Z, choice: a shard, N >= 1) and the same coef0 / options; the library runs the same
 * driver as mnl_newton_fit_opts and calls `allreduce` at each exchange step:
 *   after every pass-1 evaluation  [l, bad-choice flag, g]          (n_p + 2 doubles)
 *   after every Hessian            packed upper triangle of -H      (n_p (n_p + 1) / 2 doubles)
 *   (MNL_METHOD_CG: after every H v product, n_p doubles, instead of the Hessian)
 * Every rank therefore takes the same decisions (stop tests, Cholesky of the same -H, line-search
 * accept / reject on the same summed l) and returns the same coef, iters and loglik. A bad choice
 * on any rank is MNL_ERR_ARG on every rank; a non-finite l on any rank makes the summed l non-finite
 * (the trial is rejected everywhere). A CUDA error or a failed `allreduce` (non-zero return) ends
 * the call on that rank only: the caller must then abort the group. */
int mnl_newton_fit_dp(int64_t N, int32_t K, int32_t p, int32_t f, int32_t d,
                      const double* X, const double* Y, const double* Z, const int32_t* choice,
                      const double* coef0, const mnl_fit_options* opts,
                      mnl_allreduce_fn allreduce, void* allreduce_ctx,
                      double* coef, int32_t* iters, double* loglik, mnl_fit_stats* stats, void* stream);

/* Hessian-vector product at `coef`: hv = H v (P:462-476 applied to v without forming H):
 *   hv = -sum_i J_i^T (diag(P_i) - P_i P_i^T) J_i v,  J_i = d u_i / d theta
 * (u_i the K utilities of individual i). v, hv: dev [n_p] (may not alias). Same inputs and errors
 * as mnl_eval. */
int mnl_hessvec(int64_t N, int32_t K, int32_t p, int32_t f, int32_t d,
                const double* X, const double* Y, const double* Z, const int32_t* choice,
                const double* coef, const double* v, double* hv, void* stream);

/* Standard errors at `coef` (the paper's summary statistics):
 *   se_j = sqrt( [(-H)^{-1}]_jj ),  H the Hessian of P:462-476 at coef
 * (the inverse observed information; at the MLE the usual asymptotic standard errors).
 *   se  dev [n_p] out
 * Forms H, factors -H = L L^T (as the Newton step does) and sums the squares of the columns of
 * L^{-1} (blocked triangular inverse on DMMA, one CTA per 64-column block).
 * Errors: as mnl_eval, plus MNL_ERR_NOT_SPD when -H is not positive definite (singular design). */
int mnl_std_errors(int64_t N, int32_t K, int32_t p, int32_t f, int32_t d,
                   const double* X, const double* Y, const double* Z, const int32_t* choice,
                   const double* coef, double* se, void* stream);

/* Choice probabilities at `coef` (Eqs. "probability" / "base probability"):
 *   P  dev [N][K] out, row-major, 16-byte aligned; P[i][k] = e^{U_ik} / sum_l e^{U_il}
 * Same X, Y, Z conventions as mnl_eval; no choices are needed. Errors: MNL_ERR_ARG, MNL_ERR_CUDA,
 * MNL_ERR_NONFINITE. */
int mnl_predict(int64_t N, int32_t K, int32_t p, int32_t f, int32_t d,
                const double* X, const double* Y, const double* Z, const double* coef, double* P,
                void* stream);

/* Host-buffer variants: every pointer is HOST memory (pinned or pageable). The call copies the
 * inputs to the device, runs the same path and copies the outputs back, all inside the call. */
int mnl_eval_host(int64_t N, int32_t K, int32_t p, int32_t f, int32_t d,
                  const double* X, const double* Y, const double* Z, const int32_t* choice,
                  const double* coef, double* loglik, double* grad, double* hess);
int mnl_newton_fit_host(int64_t N, int32_t K, int32_t p, int32_t f, int32_t d,
                        const double* X, const double* Y, const double* Z, const int32_t* choice,
                        const double* coef0, double tol, int32_t max_iter,
                        double* coef, int32_t* iters, double* loglik);

/* Device-side pieces of the Newton step, exposed for tests and benchmarks. */
/* Cholesky A = L L^T of the SPD dev [n][n] row-major A, in place (lower triangle holds L;
 * the strict upper triangle is left undefined). MNL_ERR_NOT_SPD if a pivot is <= 0 or NaN. */
int mnl_cholesky(int32_t n, double* A, void* stream);
/* Solve (L L^T) x = b given the factor from mnl_cholesky; b and x dev [n], may alias. */
int mnl_cholesky_solve(int32_t n, const double* L, const double* b, double* x, void* stream);
/* Solve A x = b for the SPD dev [n][n] row-major A (lower triangle read; A is NOT modified) by the
 * Newton step's own path (row a6): the tile-DAG factorisation with the forward solve
 * fused into its diagonal tiles, then the backward wavefront (one kernel for n <= 64). b and x dev
 * [n], may alias. MNL_ERR_NOT_SPD if a pivot is <= 0 or NaN (x is then undefined). */
int mnl_spd_solve(int32_t n, const double* A, const double* b, double* x, void* stream);

/* Packed upper triangle of a symmetric dev [n][n] row-major matrix: packed[off(i) + j - i] =
 * H[i][j] for j >= i, off(i) = i n - i (i - 1) / 2 (n (n + 1) / 2 doubles), and back (both
 * triangles written, exactly symmetric). The data-parallel fit all-reduces the packed -H (written
 * straight by the Hessian assembly) -- half the bytes of the full matrix. */
int mnl_sym_pack(int32_t n, const double* H, double* packed, void* stream);
int mnl_sym_unpack(int32_t n, const double* packed, double* H, void* stream);

/* Device times (ms, CUDA events on the call's stream) of the last Hessian assembly:
 * out[0] beta-beta DMMA GEMM over whole 128-column tiles (J1), out[1] its split-N reduction,
 * out[2] the narrow tail GEMM of the remaining vech columns (J1b; 0 if none), out[3] its reduction,
 * out[4] the Z/Y blocks (J2 GEMM + reduction + same-alternative terms),
 * out[5] the symmetric assembly, out[6] the J1 operand materialisation that precedes out[0]
 * (weights every evaluation, design products once per packed design; 0 when generated in-kernel). */
int mnl_last_hessian_times(double out[7]);

/* Device time (ms, CUDA events on the call's stream) of the last pass-1 kernel (a1-a4, the fused
 * utility / softmax / loglik / gradient pass) launched by any call. */
int mnl_last_eval_ms(double* ms);

/* Kernel launches made by the last call on this thread (for the bench's gpu_launches).
 * mnl_last_eval_ms / mnl_last_hessian_times refer to the workspace of this thread's last call. */
int64_t mnl_last_launch_count(void);

const char* mnl_status_string(int code);

/* Free the library's cached device scratch. */
void mnl_release(void);

#ifdef __cplusplus
}
#endif
#endif /* MNL_H_ */
