// The Newton-Raphson driver: control flow only (SURVEY.md §8(a) rows a7 step control, a8 stop;
// Eq. "NR update" P:361-367 and the step halving of P:367-371; stopping set P:219-221).
//
// One source for every caller: libmnl.so instantiates it with its device operations (single GPU,
// and data parallel with an all-reduce exchange inside the operations), and libnrhost.so with
// host callbacks so the same control flow is exercised on CPU (tests/test_distributed.py, gloo).
// Pure C++17: no CUDA types.
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>

namespace mnl {

enum : int { kOK = 0, kErrArg = 1, kErrCuda = 2, kErrNotSpd = 3, kErrLinesearch = 4, kErrNonfinite = 5,
             kMaxIter = 6 };
enum : int { kStopNone = 0, kStopGtol = 1, kStopFtol = 2, kStopMaxIter = 3 };

constexpr int kMaxHalvings = 30;   // reading R8
constexpr double kTauRel = 1e-12;  // reading R7: accept l_j >= l - 1e-12 max(1, |l|)

struct NrOptions {
  double gtol = 1e-6;   // ||g||_2 < gtol (reading R10), tested before forming H (R11)
  double ftol = 0.0;    // |l_t - l_(t-1)| < ftol after an accepted update; 0 = off
  int32_t max_iter = 50;
};

struct NrReport {
  int32_t iters = 0, halvings = 0, evals = 0, status = 0, stop_reason = kStopNone;
  int32_t halvings_per_iter[64] = {};
  double loglik = 0.0, grad_norm = 0.0, delta_loglik = 0.0;
  double min_margin = INFINITY;  // R7 audit: min |l_j - (l - tau)| / max(1,|l|) over every decision
  // l and ||g||_2 at the iterate that starts Newton iteration t (before its Hessian), t < 64
  double loglik_per_iter[64] = {}, grad_norm_per_iter[64] = {};
};

// Ops must provide (all values global, i.e. after any exchange across ranks):
//   int eval_theta(double* l, double* g2)      l(theta), ||g||^2 at the current iterate
//   int direction(bool* not_spd)               Newton direction delta at the current iterate
//   int eval_trial(int j, double* l, double* g2)  l, ||g||^2 at theta + delta / 2^j
//   void accept()                              theta <- the last trial (its gradient / P rows too)
// Each returns kOK or an error status (which ends the fit as is).
template <class Ops>
int nr_fit(Ops& ops, const NrOptions& o, NrReport* S) {
  int rc = ops.eval_theta(&S->loglik, &S->grad_norm);  // grad_norm holds ||g||^2 until the end
  S->evals = 1;
  int status = kOK;
  double& l = S->loglik;
  double g2 = S->grad_norm;
  bool ftol_met = false;
  while (rc == kOK) {
    if (!std::isfinite(l)) { status = kErrNonfinite; break; }
    // the first condition met ends the fit: gtol before forming H, ftol after an accepted update,
    // then max_iter
    if (std::sqrt(g2) < o.gtol) { S->stop_reason = kStopGtol; break; }
    if (ftol_met) { S->stop_reason = kStopFtol; break; }
    if (S->iters == o.max_iter) { status = kMaxIter; S->stop_reason = kStopMaxIter; break; }
    if (S->iters < 64) {
      S->loglik_per_iter[S->iters] = l;
      S->grad_norm_per_iter[S->iters] = std::sqrt(g2);
    }
    bool not_spd = false;
    rc = ops.direction(&not_spd);
    if (rc) break;
    if (not_spd) { status = kErrNotSpd; break; }
    // step halving: the first theta + delta / 2^j whose l_j is "not lower than" l (R7)
    const double scale = std::max(1.0, std::fabs(l));
    const double tau = kTauRel * scale;
    bool accepted = false;
    int j = 0;
    double lt = 0.0, g2t = 0.0;
    for (j = 0; j <= kMaxHalvings; ++j) {
      rc = ops.eval_trial(j, &lt, &g2t);
      ++S->evals;
      if (rc) break;
      if (std::isfinite(lt)) S->min_margin = std::min(S->min_margin, std::fabs(lt - (l - tau)) / scale);
      if (std::isfinite(lt) && lt >= l - tau) { accepted = true; break; }
    }
    if (rc) break;
    if (!accepted) { status = kErrLinesearch; break; }
    if (S->iters < 64) S->halvings_per_iter[S->iters] = j;
    S->halvings += j;
    ops.accept();
    S->delta_loglik = std::fabs(lt - l);
    ftol_met = o.ftol > 0.0 && S->delta_loglik < o.ftol;
    l = lt;
    g2 = g2t;
    ++S->iters;
  }
  S->grad_norm = std::sqrt(g2);
  S->status = rc ? rc : status;
  return S->status;
}

}  // namespace mnl
