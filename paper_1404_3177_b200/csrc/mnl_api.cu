// C ABI (include/mnl.h) and the Newton-Raphson driver.
//
// The driver runs on the host and keeps every array on the device; per evaluation only three
// scalars cross to the host (loglik, ||g||^2, the bad-choice flag) for step control.
#include <cuda_runtime.h>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/mnl.h"
#include "internal.h"

namespace mnl {

static thread_local int64_t g_launches = 0;
void count_launch(int n) { g_launches += n; }

namespace {

std::mutex g_mu;

template <class T>
bool grow(T** p, size_t* cap, size_t n) {
  if (n <= *cap && *p) return true;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *cap = 0;
  if (cudaMalloc(p, n * sizeof(T)) != cudaSuccess) return false;
  *cap = n;
  return true;
}

struct Workspace {
  int device = -1;
  int sms = 0;
  // packed rows
  double *Xp = nullptr, *Zp = nullptr, *Pr = nullptr;
  size_t cXp = 0, cZp = 0, cPr = 0;
  // eval partials / scalars
  double* part = nullptr;
  size_t cpart = 0;
  double* scal = nullptr;  // [4]
  int* err = nullptr;
  int* info = nullptr;
  unsigned* counter = nullptr;
  // Newton vectors / matrix
  double *theta = nullptr, *trial = nullptr, *grad = nullptr, *delta = nullptr, *A = nullptr;
  size_t ctheta = 0, ctrial = 0, cgrad = 0, cdelta = 0, cA = 0;
  double* cg = nullptr;  // truncated Newton: r, p, Hp, Ap [4][n_p] + 2 scalars
  size_t ccg = 0;
  // cached hessian plan
  HessPlan* hp = nullptr;
  Dims hp_dims{};
  Packed hp_pk{};
  // host-mode device copies
  double *hX = nullptr, *hY = nullptr, *hZ = nullptr, *hcoef = nullptr, *hout = nullptr, *hH = nullptr;
  int32_t* hch = nullptr;
  int32_t* zch = nullptr;  // all-zero choices for mnl_predict
  size_t czch = 0;
  size_t chX = 0, chY = 0, chZ = 0, chcoef = 0, chout = 0, chH = 0, chch = 0;
  cudaStream_t hstream = nullptr;
  cudaEvent_t ev_eval[2] = {nullptr, nullptr};  // around the last pass-1 kernel
};

Workspace g_ws;

const char* kStatus[] = {"MNL_OK", "MNL_ERR_ARG", "MNL_ERR_CUDA", "MNL_ERR_NOT_SPD",
                         "MNL_ERR_LINESEARCH", "MNL_ERR_NONFINITE", "MNL_MAXITER"};

bool dims_of(int64_t N, int32_t K, int32_t p, int32_t f, int32_t d, Dims* D) {
  if (N < 1 || N >= (int64_t(1) << 31) || K < 2 || K > 256 || p < 0 || p > 255 || f < 0 || f > 64 || d < 0 ||
      d > 64)
    return false;
  D->N = N; D->K = K; D->p = p; D->f = f; D->d = d;
  D->q = p + 1;
  D->n_beta = (K - 1) * D->q;
  D->n_alpha = K * d;
  D->n_p = D->n_beta + D->n_alpha + f;
  D->off_alpha = D->n_beta;
  D->off_gamma = D->n_beta + D->n_alpha;
  return D->n_p <= 16384;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int init_device(Workspace& W) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return MNL_ERR_CUDA;
  if (W.device != dev) {
    if (W.device >= 0) return MNL_ERR_CUDA;  // one device per process in this build
    W.device = dev;
    cudaDeviceGetAttribute(&W.sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaMalloc(&W.scal, 4 * sizeof(double)) != cudaSuccess) return MNL_ERR_CUDA;
    if (cudaMalloc(&W.err, sizeof(int)) != cudaSuccess) return MNL_ERR_CUDA;
    if (cudaMalloc(&W.info, sizeof(int)) != cudaSuccess) return MNL_ERR_CUDA;
    if (cudaMalloc(&W.counter, sizeof(unsigned)) != cudaSuccess) return MNL_ERR_CUDA;
    cudaMemset(W.counter, 0, sizeof(unsigned));
    cudaMemset(W.err, 0, sizeof(int));
  }
  return MNL_OK;
}

bool ensure_packed(Workspace& W, const Dims& D, Packed* pk) {
  pk->Npad = (D.N + kRowPad - 1) / kRowPad * kRowPad;
  pk->ldX = pad4mod16(D.q);
  pk->ldZ = pad4mod16(std::max(D.K * D.d, 1));
  pk->ldP = pad4mod16(D.K + D.f);
  const size_t nX = pk->Npad * pk->ldX, nZ = D.d ? pk->Npad * pk->ldZ : 2, nP = pk->Npad * pk->ldP;
  const bool newP = !(nP <= W.cPr && W.Pr);
  if (!grow(&W.Xp, &W.cXp, nX) || !grow(&W.Zp, &W.cZp, nZ) || !grow(&W.Pr, &W.cPr, nP)) return false;
  (void)newP;
  pk->Xp = W.Xp;
  pk->Zp = W.Zp;
  pk->Pr = W.Pr;
  return true;
}

HessPlan* get_hess_plan(Workspace& W, const Dims& D, const Packed& pk) {
  if (W.hp && memcmp(&W.hp_dims, &D, sizeof(Dims)) == 0 && W.hp_pk.Npad == pk.Npad && W.hp_pk.ldX == pk.ldX &&
      W.hp_pk.ldZ == pk.ldZ && W.hp_pk.ldP == pk.ldP)
    return W.hp;
  hess_plan_destroy(W.hp);
  W.hp = hess_plan_create(D, pk, W.sms);
  W.hp_dims = D;
  W.hp_pk = pk;
  return W.hp;
}

// One pass-1 evaluation; reads back [l, ||g||^2, err] into scal_h. grad may be null.
int run_eval(Workspace& W, const Dims& D, const EvalPlan& ep, const double* X, const double* Y, const double* Z,
             const int32_t* choice, const double* coef, const Packed* pk, bool writeP, double* grad,
             double* loglik_dev, double* scal_h, cudaStream_t st) {
  if (!grow(&W.part, &W.cpart, eval_part_doubles(ep))) return MNL_ERR_CUDA;
  cudaMemsetAsync(W.err, 0, sizeof(int), st);
  if (!W.ev_eval[0]) {
    cudaEventCreate(&W.ev_eval[0]);
    cudaEventCreate(&W.ev_eval[1]);
  }
  cudaEventRecord(W.ev_eval[0], st);
  cudaError_t e = launch_eval(D, ep, X, Y, Z, choice, coef, pk, grad != nullptr, writeP, W.part, W.err, st);
  if (e != cudaSuccess) return MNL_ERR_CUDA;
  cudaEventRecord(W.ev_eval[1], st);
  e = launch_eval_finalize(D, ep, W.part, grad != nullptr, grad, loglik_dev, W.scal, W.err, W.counter, st);
  if (e != cudaSuccess) return MNL_ERR_CUDA;
  if (cudaMemcpyAsync(scal_h, W.scal, 3 * sizeof(double), cudaMemcpyDeviceToHost, st) != cudaSuccess)
    return MNL_ERR_CUDA;
  if (cudaStreamSynchronize(st) != cudaSuccess) return MNL_ERR_CUDA;
  if (scal_h[2] != 0.0) return MNL_ERR_ARG;
  return MNL_OK;
}

// H v at the coefficients of the last evaluation with writeP (P_i in pk->Pr); hv dev [n_p].
int run_hessvec(Workspace& W, const Dims& D, const EvalPlan& ep, const double* X, const double* Y, const double* Z,
                const int32_t* choice, const double* v, const Packed* pk, double* hv, cudaStream_t st) {
  if (!grow(&W.part, &W.cpart, eval_part_doubles(ep))) return MNL_ERR_CUDA;
  cudaError_t e = launch_hessvec(D, ep, X, Y, Z, choice, v, pk, W.part, W.err, st);
  if (e != cudaSuccess) return MNL_ERR_CUDA;
  e = launch_eval_finalize(D, ep, W.part, true, hv, nullptr, W.scal, W.err, W.counter, st);
  return e == cudaSuccess ? MNL_OK : MNL_ERR_CUDA;
}

bool check_inputs(const Dims& D, const double* X, const double* Y, const double* Z, const int32_t* choice) {
  if ((D.p > 0) != (X != nullptr) || (D.f > 0) != (Y != nullptr) || (D.d > 0) != (Z != nullptr) || !choice)
    return false;
  if ((X && !aligned16(X)) || (Y && !aligned16(Y)) || (Z && !aligned16(Z)) || !aligned16(choice)) return false;
  return true;
}

int eval_impl(int64_t N, int32_t K, int32_t p, int32_t f, int32_t d, const double* X, const double* Y,
              const double* Z, const int32_t* choice, const double* coef, double* loglik, double* grad,
              double* hess, cudaStream_t st) {
  Dims D;
  if (!dims_of(N, K, p, f, d, &D) || !check_inputs(D, X, Y, Z, choice) || !coef || !loglik) return MNL_ERR_ARG;
  Workspace& W = g_ws;
  int rc = init_device(W);
  if (rc) return rc;
  EvalPlan ep;
  if (!eval_plan(D, &ep, W.sms)) return MNL_ERR_ARG;
  Packed pk{};
  const bool want_h = hess != nullptr;
  if (want_h) {
    if (!ensure_packed(W, D, &pk)) return MNL_ERR_CUDA;
    if (launch_pack(D, pk, X, Z, st) != cudaSuccess) return MNL_ERR_CUDA;
    if (W.hp) hess_plan_design_changed(W.hp);
  }
  double* g = grad;
  double scal[3];
  rc = run_eval(W, D, ep, X, Y, Z, choice, coef, want_h ? &pk : nullptr, want_h, g, loglik, scal, st);
  if (rc) return rc;
  if (!std::isfinite(scal[0])) return MNL_ERR_NONFINITE;
  if (want_h) {
    HessPlan* hp = get_hess_plan(W, D, pk);
    if (!hp) return MNL_ERR_CUDA;
    if (launch_hessian(hp, D, pk, Y, hess, D.n_p, +1.0, st) != cudaSuccess) return MNL_ERR_CUDA;
    if (cudaStreamSynchronize(st) != cudaSuccess) return MNL_ERR_CUDA;
  }
  return MNL_OK;
}

float elapsed(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

mnl_fit_options default_options(double tol, int32_t max_iter) {
  mnl_fit_options o;
  o.gtol = tol;
  o.ftol = 0.0;
  o.max_iter = max_iter;
  o.method = MNL_METHOD_NEWTON;
  o.cg_max_iter = 0;
  o.cg_rtol = 0.0;
  return o;
}

int fit_impl(int64_t N, int32_t K, int32_t p, int32_t f, int32_t d, const double* X, const double* Y,
             const double* Z, const int32_t* choice, const double* coef0, const mnl_fit_options& o,
             double* coef, int32_t* iters_out, double* loglik_out, mnl_fit_stats* stats, cudaStream_t st) {
  const auto t0 = std::chrono::steady_clock::now();
  Dims D;
  const double tol = o.gtol;
  const int32_t max_iter = o.max_iter;
  const bool use_cg = o.method == MNL_METHOD_CG;
  if (!dims_of(N, K, p, f, d, &D) || !check_inputs(D, X, Y, Z, choice) || !coef || !iters_out || !loglik_out ||
      !(tol > 0.0) || max_iter < 0 || !(o.ftol >= 0.0) || (o.method != MNL_METHOD_NEWTON && !use_cg) ||
      o.cg_max_iter < 0 || !(o.cg_rtol >= 0.0) || !(o.cg_rtol < 1.0))
    return MNL_ERR_ARG;
  Workspace& W = g_ws;
  int rc = init_device(W);
  if (rc) return rc;
  EvalPlan ep;
  if (!eval_plan(D, &ep, W.sms)) return MNL_ERR_ARG;
  Packed pk{};
  if (!ensure_packed(W, D, &pk)) return MNL_ERR_CUDA;
  const int n = D.n_p;
  if (!grow(&W.theta, &W.ctheta, n) || !grow(&W.trial, &W.ctrial, n) || !grow(&W.grad, &W.cgrad, n) ||
      !grow(&W.delta, &W.cdelta, n))
    return MNL_ERR_CUDA;
  if (!use_cg && !grow(&W.A, &W.cA, (size_t)n * n)) return MNL_ERR_CUDA;
  if (use_cg && !grow(&W.cg, &W.ccg, (size_t)4 * n + 2)) return MNL_ERR_CUDA;
  HessPlan* hp = use_cg ? nullptr : get_hess_plan(W, D, pk);
  if (!use_cg && !hp) return MNL_ERR_CUDA;
  if (launch_pack(D, pk, X, Z, st) != cudaSuccess) return MNL_ERR_CUDA;
  if (hp) hess_plan_design_changed(hp);
  if (coef0) cudaMemcpyAsync(W.theta, coef0, n * sizeof(double), cudaMemcpyDeviceToDevice, st);
  else cudaMemsetAsync(W.theta, 0, n * sizeof(double), st);

  cudaEvent_t ev[4];
  for (auto& e : ev) cudaEventCreate(&e);
  mnl_fit_stats S;
  memset(&S, 0, sizeof(S));
  double scal[3];
  rc = run_eval(W, D, ep, X, Y, Z, choice, W.theta, &pk, true, W.grad, nullptr, scal, st);
  S.evals = 1;
  int status = MNL_OK;
  int iters = 0;
  double l = scal[0], g2 = scal[1];
  bool ftol_met = false;
  while (rc == MNL_OK) {
    if (!std::isfinite(l)) { status = MNL_ERR_NONFINITE; break; }
    // the paper's stopping set, first met ends the fit: gtol is tested
    // before forming H (R11), ftol after an accepted update, then max_iter
    if (std::sqrt(g2) < tol) { status = MNL_OK; S.stop_reason = MNL_STOP_GTOL; break; }
    if (ftol_met) { status = MNL_OK; S.stop_reason = MNL_STOP_FTOL; break; }
    if (iters == max_iter) { status = MNL_MAXITER; S.stop_reason = MNL_STOP_MAXITER; break; }
    if (use_cg) {
      // truncated Newton: CG on (-H) delta = g with H v products, never forming H
      cudaEventRecord(ev[0], st);
      double* r = W.cg;
      double* pv = W.cg + n;
      double* hpv = W.cg + 2 * n;
      double* apv = W.cg + 3 * n;
      double* sc = W.cg + 4 * n;
      cudaMemsetAsync(W.delta, 0, n * sizeof(double), st);
      cudaMemcpyAsync(r, W.grad, n * sizeof(double), cudaMemcpyDeviceToDevice, st);
      cudaMemcpyAsync(pv, W.grad, n * sizeof(double), cudaMemcpyDeviceToDevice, st);
      const double gn = std::sqrt(g2);
      const double eta = o.cg_rtol > 0.0 ? o.cg_rtol : std::min(0.5, std::sqrt(gn));
      const int cg_max = o.cg_max_iter > 0 ? o.cg_max_iter : n;
      double rr = g2;
      bool fail = false;
      for (int it = 0; it < cg_max; ++it) {
        rc = run_hessvec(W, D, ep, X, Y, Z, choice, pv, &pk, hpv, st);
        if (rc) break;
        double h2[2];
        if (launch_cg_curv(n, pv, hpv, apv, sc, st) != cudaSuccess) { rc = MNL_ERR_CUDA; break; }
        cudaMemcpyAsync(h2, sc, sizeof(double), cudaMemcpyDeviceToHost, st);
        if (cudaStreamSynchronize(st) != cudaSuccess) { rc = MNL_ERR_CUDA; break; }
        const double pAp = h2[0];
        if (!(pAp > 0.0) || !std::isfinite(pAp)) { fail = it == 0; break; }  // negative curvature
        const double alpha = rr / pAp;
        if (launch_cg_update(n, alpha, pv, apv, W.delta, r, sc + 1, st) != cudaSuccess) { rc = MNL_ERR_CUDA; break; }
        cudaMemcpyAsync(h2 + 1, sc + 1, sizeof(double), cudaMemcpyDeviceToHost, st);
        if (cudaStreamSynchronize(st) != cudaSuccess) { rc = MNL_ERR_CUDA; break; }
        ++S.cg_iters;
        const double rr_new = h2[1];
        if (std::sqrt(rr_new) <= eta * gn) break;
        if (launch_cg_dir(n, rr_new / rr, r, pv, st) != cudaSuccess) { rc = MNL_ERR_CUDA; break; }
        rr = rr_new;
      }
      cudaEventRecord(ev[1], st);
      if (cudaStreamSynchronize(st) != cudaSuccess) rc = MNL_ERR_CUDA;
      if (rc) break;
      S.hess_ms += elapsed(ev[0], ev[1]);
      if (fail) { status = MNL_ERR_NOT_SPD; break; }
    } else {
    cudaEventRecord(ev[0], st);
    if (launch_hessian(hp, D, pk, Y, W.A, n, -1.0, st) != cudaSuccess) { rc = MNL_ERR_CUDA; break; }  // A = -H
    cudaEventRecord(ev[1], st);
    if (launch_cholesky_solve_fused(n, W.A, n, W.info, W.grad, W.delta, st) != cudaSuccess) {
      rc = MNL_ERR_CUDA;
      break;
    }
    cudaEventRecord(ev[2], st);
    int info = 0;
    cudaMemcpyAsync(&info, W.info, sizeof(int), cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) { rc = MNL_ERR_CUDA; break; }
    S.hess_ms += elapsed(ev[0], ev[1]);
    S.chol_ms += elapsed(ev[1], ev[2]);
    {
      double ht[7];
      hess_last_times(hp, ht);
      S.gemm_ms += ht[0] + ht[2];  // the beta-beta GEMM: whole tiles + narrow tail
    }
    if (info != 0) { status = MNL_ERR_NOT_SPD; break; }
    }
    // a7: step halving, accept the first l_j >= l - tau (R7, R8)
    const double tau = 1e-12 * std::max(1.0, std::fabs(l));
    bool accepted = false;
    int j = 0;
    double lt = 0.0, g2t = 0.0;
    for (j = 0; j <= 30; ++j) {
      if (launch_axpy_pow2(n, W.theta, W.delta, j, W.trial, st) != cudaSuccess) { rc = MNL_ERR_CUDA; break; }
      rc = run_eval(W, D, ep, X, Y, Z, choice, W.trial, &pk, true, W.grad, nullptr, scal, st);
      ++S.evals;
      if (rc) break;
      lt = scal[0];
      g2t = scal[1];
      if (std::isfinite(lt) && lt >= l - tau) { accepted = true; break; }
    }
    if (rc) break;
    if (!accepted) { status = MNL_ERR_LINESEARCH; break; }
    if (iters < 64) S.halvings_per_iter[iters] = j;
    S.halvings += j;
    std::swap(W.theta, W.trial);
    std::swap(W.ctheta, W.ctrial);
    S.delta_loglik = std::fabs(lt - l);
    ftol_met = o.ftol > 0.0 && S.delta_loglik < o.ftol;
    l = lt;
    g2 = g2t;
    ++iters;
  }
  for (auto& e : ev) cudaEventDestroy(e);
  if (rc) return rc;
  cudaMemcpyAsync(coef, W.theta, n * sizeof(double), cudaMemcpyDeviceToDevice, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return MNL_ERR_CUDA;
  *iters_out = iters;
  *loglik_out = l;
  if (stats) {
    S.iters = iters;
    S.status = status;
    S.grad_norm = std::sqrt(g2);
    S.loglik = l;
    S.total_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    S.eval_ms = S.total_ms - S.hess_ms - S.chol_ms;
    *stats = S;
  }
  return status;
}

cudaStream_t host_stream(Workspace& W) {
  if (!W.hstream) cudaStreamCreateWithFlags(&W.hstream, cudaStreamNonBlocking);
  return W.hstream;
}

}  // namespace
}  // namespace mnl

using namespace mnl;

extern "C" {

int64_t mnl_num_params(int32_t K, int32_t p, int32_t f, int32_t d) {
  if (K < 2 || p < 0 || f < 0 || d < 0) return -1;
  return (int64_t)(K - 1) * (p + 1) + (int64_t)K * d + f;
}

const char* mnl_status_string(int code) {
  if (code < 0 || code > 6) return "MNL_UNKNOWN";
  return kStatus[code];
}

int64_t mnl_last_launch_count(void) { return g_launches; }

int mnl_check_shape(int64_t N, int32_t K, int32_t p, int32_t f, int32_t d) {
  Dims D;
  if (!dims_of(N, K, p, f, d, &D)) return MNL_ERR_ARG;
  EvalPlan ep;
  return eval_plan(D, &ep, 148) ? MNL_OK : MNL_ERR_ARG;  // the pass-1 shared-memory bound
}

int mnl_last_eval_ms(double* ms) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!ms || !g_ws.ev_eval[0]) return MNL_ERR_ARG;
  float t = 0.f;
  if (cudaEventSynchronize(g_ws.ev_eval[1]) != cudaSuccess ||
      cudaEventElapsedTime(&t, g_ws.ev_eval[0], g_ws.ev_eval[1]) != cudaSuccess)
    return MNL_ERR_CUDA;
  *ms = t;
  return MNL_OK;
}

int mnl_last_hessian_times(double out[7]) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!out) return MNL_ERR_ARG;
  hess_last_times(g_ws.hp, out);
  return g_ws.hp ? MNL_OK : MNL_ERR_ARG;
}

int mnl_eval(int64_t N, int32_t K, int32_t p, int32_t f, int32_t d, const double* X, const double* Y,
             const double* Z, const int32_t* choice, const double* coef, double* loglik, double* grad, double* hess,
             void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_launches = 0;
  return eval_impl(N, K, p, f, d, X, Y, Z, choice, coef, loglik, grad, hess, (cudaStream_t)stream);
}

int mnl_newton_fit_ex(int64_t N, int32_t K, int32_t p, int32_t f, int32_t d, const double* X, const double* Y,
                      const double* Z, const int32_t* choice, const double* coef0, double tol, int32_t max_iter,
                      double* coef, int32_t* iters, double* loglik, mnl_fit_stats* stats, void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_launches = 0;
  return fit_impl(N, K, p, f, d, X, Y, Z, choice, coef0, default_options(tol, max_iter), coef, iters, loglik, stats,
                  (cudaStream_t)stream);
}

int mnl_newton_fit_opts(int64_t N, int32_t K, int32_t p, int32_t f, int32_t d, const double* X, const double* Y,
                        const double* Z, const int32_t* choice, const double* coef0, const mnl_fit_options* opts,
                        double* coef, int32_t* iters, double* loglik, mnl_fit_stats* stats, void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_launches = 0;
  if (!opts) return MNL_ERR_ARG;
  return fit_impl(N, K, p, f, d, X, Y, Z, choice, coef0, *opts, coef, iters, loglik, stats, (cudaStream_t)stream);
}

int mnl_hessvec(int64_t N, int32_t K, int32_t p, int32_t f, int32_t d, const double* X, const double* Y,
                const double* Z, const int32_t* choice, const double* coef, const double* v, double* hv,
                void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_launches = 0;
  Dims D;
  if (!dims_of(N, K, p, f, d, &D) || !check_inputs(D, X, Y, Z, choice) || !coef || !v || !hv || v == hv)
    return MNL_ERR_ARG;
  Workspace& W = g_ws;
  int rc = init_device(W);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  EvalPlan ep;
  if (!eval_plan(D, &ep, W.sms)) return MNL_ERR_ARG;
  Packed pk{};
  if (!ensure_packed(W, D, &pk)) return MNL_ERR_CUDA;  // for Pr
  double scal[3];
  rc = run_eval(W, D, ep, X, Y, Z, choice, coef, &pk, true, nullptr, nullptr, scal, st);  // P_i at coef
  if (rc) return rc;
  if (!std::isfinite(scal[0])) return MNL_ERR_NONFINITE;
  rc = run_hessvec(W, D, ep, X, Y, Z, choice, v, &pk, hv, st);
  if (rc) return rc;
  return cudaStreamSynchronize(st) == cudaSuccess ? MNL_OK : MNL_ERR_CUDA;
}

int mnl_eval_async(int64_t N, int32_t K, int32_t p, int32_t f, int32_t d, const double* X, const double* Y,
                   const double* Z, const int32_t* choice, const double* coef, double* loglik, double* grad,
                   double* hess, int32_t* status, void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_launches = 0;
  Dims D;
  if (!dims_of(N, K, p, f, d, &D) || !check_inputs(D, X, Y, Z, choice) || !coef || !loglik || !status)
    return MNL_ERR_ARG;
  Workspace& W = g_ws;
  int rc = init_device(W);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  EvalPlan ep;
  if (!eval_plan(D, &ep, W.sms)) return MNL_ERR_ARG;
  Packed pk{};
  const bool want_h = hess != nullptr;
  if (want_h) {
    if (!ensure_packed(W, D, &pk)) return MNL_ERR_CUDA;
    if (launch_pack(D, pk, X, Z, st) != cudaSuccess) return MNL_ERR_CUDA;
    if (W.hp) hess_plan_design_changed(W.hp);
  }
  if (!grow(&W.part, &W.cpart, eval_part_doubles(ep))) return MNL_ERR_CUDA;
  HessPlan* hp = want_h ? get_hess_plan(W, D, pk) : nullptr;  // (first use of a shape allocates)
  if (want_h && !hp) return MNL_ERR_CUDA;
  cudaMemsetAsync(W.err, 0, sizeof(int), st);
  if (launch_eval(D, ep, X, Y, Z, choice, coef, want_h ? &pk : nullptr, grad != nullptr, want_h, W.part, W.err, st) !=
      cudaSuccess)
    return MNL_ERR_CUDA;
  if (launch_eval_finalize(D, ep, W.part, grad != nullptr, grad, loglik, W.scal, W.err, W.counter, st, status) !=
      cudaSuccess)
    return MNL_ERR_CUDA;
  if (want_h && launch_hessian(hp, D, pk, Y, hess, D.n_p, +1.0, st) != cudaSuccess) return MNL_ERR_CUDA;
  return MNL_OK;
}

int mnl_std_errors(int64_t N, int32_t K, int32_t p, int32_t f, int32_t d, const double* X, const double* Y,
                   const double* Z, const int32_t* choice, const double* coef, double* se, void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_launches = 0;
  Dims D;
  if (!dims_of(N, K, p, f, d, &D) || !check_inputs(D, X, Y, Z, choice) || !coef || !se) return MNL_ERR_ARG;
  Workspace& W = g_ws;
  int rc = init_device(W);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  EvalPlan ep;
  if (!eval_plan(D, &ep, W.sms)) return MNL_ERR_ARG;
  Packed pk{};
  if (!ensure_packed(W, D, &pk)) return MNL_ERR_CUDA;
  if (launch_pack(D, pk, X, Z, st) != cudaSuccess) return MNL_ERR_CUDA;
  if (W.hp) hess_plan_design_changed(W.hp);
  double scal[3];
  rc = run_eval(W, D, ep, X, Y, Z, choice, coef, &pk, true, nullptr, nullptr, scal, st);  // P_i at coef
  if (rc) return rc;
  if (!std::isfinite(scal[0])) return MNL_ERR_NONFINITE;
  HessPlan* hp = get_hess_plan(W, D, pk);
  const int n = D.n_p;
  if (!hp || !grow(&W.A, &W.cA, (size_t)n * n)) return MNL_ERR_CUDA;
  if (launch_hessian(hp, D, pk, Y, W.A, n, -1.0, st) != cudaSuccess) return MNL_ERR_CUDA;  // A = -H
  if (launch_cholesky(n, W.A, n, W.info, st) != cudaSuccess) return MNL_ERR_CUDA;
  int info = 0;
  cudaMemcpyAsync(&info, W.info, sizeof(int), cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return MNL_ERR_CUDA;
  if (info) return MNL_ERR_NOT_SPD;
  if (launch_inv_diag_sqrt(n, W.A, n, se, st) != cudaSuccess) return MNL_ERR_CUDA;
  return cudaStreamSynchronize(st) == cudaSuccess ? MNL_OK : MNL_ERR_CUDA;
}

int mnl_predict(int64_t N, int32_t K, int32_t p, int32_t f, int32_t d, const double* X, const double* Y,
                const double* Z, const double* coef, double* P, void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_launches = 0;
  Dims D;
  if (!dims_of(N, K, p, f, d, &D) || !coef || !P || !aligned16(P)) return MNL_ERR_ARG;
  Workspace& W = g_ws;
  int rc = init_device(W);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  if (!grow(&W.zch, &W.czch, (size_t)N)) return MNL_ERR_CUDA;  // pass 1 reads a choice per row
  cudaMemsetAsync(W.zch, 0, (size_t)N * sizeof(int32_t), st);
  if (!check_inputs(D, X, Y, Z, W.zch)) return MNL_ERR_ARG;
  EvalPlan ep;
  if (!eval_plan(D, &ep, W.sms)) return MNL_ERR_ARG;
  Packed pk{};
  if (!ensure_packed(W, D, &pk)) return MNL_ERR_CUDA;
  double scal[3];
  rc = run_eval(W, D, ep, X, Y, Z, W.zch, coef, &pk, true, nullptr, nullptr, scal, st);
  if (rc) return rc;
  if (!std::isfinite(scal[0])) return MNL_ERR_NONFINITE;
  if (cudaMemcpy2DAsync(P, (size_t)K * sizeof(double), pk.Pr, (size_t)pk.ldP * sizeof(double),
                        (size_t)K * sizeof(double), (size_t)N, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
    return MNL_ERR_CUDA;
  return cudaStreamSynchronize(st) == cudaSuccess ? MNL_OK : MNL_ERR_CUDA;
}

int mnl_newton_fit(int64_t N, int32_t K, int32_t p, int32_t f, int32_t d, const double* X, const double* Y,
                   const double* Z, const int32_t* choice, const double* coef0, double tol, int32_t max_iter,
                   double* coef, int32_t* iters, double* loglik, void* stream) {
  return mnl_newton_fit_ex(N, K, p, f, d, X, Y, Z, choice, coef0, tol, max_iter, coef, iters, loglik, nullptr,
                           stream);
}

static bool h2d(double** dst, size_t* cap, const double* src, size_t n, cudaStream_t st) {
  if (!n) { return true; }
  if (!grow(dst, cap, n)) return false;
  return cudaMemcpyAsync(*dst, src, n * sizeof(double), cudaMemcpyHostToDevice, st) == cudaSuccess;
}

int mnl_eval_host(int64_t N, int32_t K, int32_t p, int32_t f, int32_t d, const double* X, const double* Y,
                  const double* Z, const int32_t* choice, const double* coef, double* loglik, double* grad,
                  double* hess) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_launches = 0;
  Dims D;
  if (!dims_of(N, K, p, f, d, &D) || !choice || !coef || !loglik) return MNL_ERR_ARG;
  Workspace& W = g_ws;
  int rc = init_device(W);
  if (rc) return rc;
  cudaStream_t st = host_stream(W);
  const int n = D.n_p;
  if (!h2d(&W.hX, &W.chX, X, (size_t)N * p, st) || !h2d(&W.hY, &W.chY, Y, (size_t)N * K * f, st) ||
      !h2d(&W.hZ, &W.chZ, Z, (size_t)N * K * d, st) || !h2d(&W.hcoef, &W.chcoef, coef, n, st))
    return MNL_ERR_CUDA;
  if (!grow(&W.hch, &W.chch, (size_t)N)) return MNL_ERR_CUDA;
  cudaMemcpyAsync(W.hch, choice, N * sizeof(int32_t), cudaMemcpyHostToDevice, st);
  if (!grow(&W.hout, &W.chout, (size_t)n + 2)) return MNL_ERR_CUDA;
  if (hess && !grow(&W.hH, &W.chH, (size_t)n * n)) return MNL_ERR_CUDA;
  rc = eval_impl(N, K, p, f, d, p ? W.hX : nullptr, f ? W.hY : nullptr, d ? W.hZ : nullptr, W.hch, W.hcoef,
                 W.hout + n, grad ? W.hout : nullptr, hess ? W.hH : nullptr, st);
  if (rc && rc != MNL_ERR_NONFINITE) return rc;
  cudaMemcpyAsync(loglik, W.hout + n, sizeof(double), cudaMemcpyDeviceToHost, st);
  if (grad) cudaMemcpyAsync(grad, W.hout, n * sizeof(double), cudaMemcpyDeviceToHost, st);
  if (hess) cudaMemcpyAsync(hess, W.hH, (size_t)n * n * sizeof(double), cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return MNL_ERR_CUDA;
  return rc;
}

int mnl_newton_fit_host(int64_t N, int32_t K, int32_t p, int32_t f, int32_t d, const double* X, const double* Y,
                        const double* Z, const int32_t* choice, const double* coef0, double tol, int32_t max_iter,
                        double* coef, int32_t* iters, double* loglik) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_launches = 0;
  Dims D;
  if (!dims_of(N, K, p, f, d, &D) || !choice || !coef || !iters || !loglik) return MNL_ERR_ARG;
  Workspace& W = g_ws;
  int rc = init_device(W);
  if (rc) return rc;
  cudaStream_t st = host_stream(W);
  const int n = D.n_p;
  if (!h2d(&W.hX, &W.chX, X, (size_t)N * p, st) || !h2d(&W.hY, &W.chY, Y, (size_t)N * K * f, st) ||
      !h2d(&W.hZ, &W.chZ, Z, (size_t)N * K * d, st))
    return MNL_ERR_CUDA;
  if (!grow(&W.hch, &W.chch, (size_t)N) || !grow(&W.hcoef, &W.chcoef, (size_t)n)) return MNL_ERR_CUDA;
  cudaMemcpyAsync(W.hch, choice, N * sizeof(int32_t), cudaMemcpyHostToDevice, st);
  if (coef0) cudaMemcpyAsync(W.hcoef, coef0, n * sizeof(double), cudaMemcpyHostToDevice, st);
  rc = fit_impl(N, K, p, f, d, p ? W.hX : nullptr, f ? W.hY : nullptr, d ? W.hZ : nullptr, W.hch,
                coef0 ? W.hcoef : nullptr, default_options(tol, max_iter), W.hcoef, iters, loglik, nullptr, st);
  if (rc != MNL_OK && rc != MNL_MAXITER) return rc;
  cudaMemcpyAsync(coef, W.hcoef, n * sizeof(double), cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return MNL_ERR_CUDA;
  return rc;
}

int mnl_cholesky(int32_t n, double* A, void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_launches = 0;
  if (n < 1 || !A) return MNL_ERR_ARG;
  Workspace& W = g_ws;
  int rc = init_device(W);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  if (launch_cholesky(n, A, n, W.info, st) != cudaSuccess) return MNL_ERR_CUDA;
  int info = 0;
  cudaMemcpyAsync(&info, W.info, sizeof(int), cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return MNL_ERR_CUDA;
  return info ? MNL_ERR_NOT_SPD : MNL_OK;
}

int mnl_cholesky_solve(int32_t n, const double* L, const double* b, double* x, void* stream) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_launches = 0;
  if (n < 1 || !L || !b || !x) return MNL_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  if (launch_chol_solve(n, L, n, b, x, st) != cudaSuccess) return MNL_ERR_CUDA;
  if (cudaStreamSynchronize(st) != cudaSuccess) return MNL_ERR_CUDA;
  return MNL_OK;
}

int mnl_sym_pack(int32_t n, const double* H, double* packed, void* stream) {
  g_launches = 0;
  if (n < 1 || !H || !packed) return MNL_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  if (launch_sym_pack(n, H, packed, st) != cudaSuccess) return MNL_ERR_CUDA;
  return cudaStreamSynchronize(st) == cudaSuccess ? MNL_OK : MNL_ERR_CUDA;
}

int mnl_sym_unpack(int32_t n, const double* packed, double* H, void* stream) {
  g_launches = 0;
  if (n < 1 || !H || !packed) return MNL_ERR_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  if (launch_sym_unpack(n, packed, H, st) != cudaSuccess) return MNL_ERR_CUDA;
  return cudaStreamSynchronize(st) == cudaSuccess ? MNL_OK : MNL_ERR_CUDA;
}

void mnl_release(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  Workspace& W = g_ws;
  hess_plan_destroy(W.hp);
  W.hp = nullptr;
  double* ds[] = {W.Xp, W.Zp, W.Pr, W.part, W.scal, W.theta, W.trial, W.grad, W.delta, W.A, W.cg,
                  W.hX, W.hY, W.hZ, W.hcoef, W.hout, W.hH};
  for (double* p : ds) cudaFree(p);
  cudaFree(W.err);
  cudaFree(W.info);
  cudaFree(W.counter);
  cudaFree(W.hch);
  cudaFree(W.zch);
  if (W.hstream) cudaStreamDestroy(W.hstream);
  for (cudaEvent_t ev : W.ev_eval)
    if (ev) cudaEventDestroy(ev);
  W = Workspace();
}

}  // extern "C"
