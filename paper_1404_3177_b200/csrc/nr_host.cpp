// libnrhost.so: the Newton-Raphson driver of libmnl.so (nr_driver.h, the same source) over host
// callbacks, so its control flow -- stopping set, step halving, the R7 acceptance floor -- runs on
// CPU with any evaluator and exchange (tests/test_distributed.py: two gloo ranks, oracle shards).
// No CUDA. Not used by the product path (libmnl.so instantiates the driver with device operations).
#include "nr_driver.h"

extern "C" {

typedef struct {
  void* ctx;
  int (*eval_theta)(void* ctx, double* l, double* g2);
  int (*direction)(void* ctx, int* not_spd);
  int (*eval_trial)(void* ctx, int j, double* l, double* g2);
  void (*accept)(void* ctx);
} nr_host_ops;

typedef struct {
  int32_t iters, halvings, evals, status, stop_reason;
  int32_t halvings_per_iter[64];
  double loglik, grad_norm, delta_loglik, min_margin;
  double loglik_per_iter[64], grad_norm_per_iter[64];  // at the iterate starting each iteration
} nr_host_report;

int nr_fit_host(const nr_host_ops* ops, double gtol, double ftol, int32_t max_iter, nr_host_report* out) {
  if (!ops || !out || !ops->eval_theta || !ops->direction || !ops->eval_trial || !ops->accept || !(gtol > 0.0) ||
      !(ftol >= 0.0) || max_iter < 0)
    return mnl::kErrArg;
  struct Ops {
    const nr_host_ops* h;
    int eval_theta(double* l, double* g2) { return h->eval_theta(h->ctx, l, g2); }
    int direction(bool* not_spd) {
      int ns = 0;
      const int rc = h->direction(h->ctx, &ns);
      *not_spd = ns != 0;
      return rc;
    }
    int eval_trial(int j, double* l, double* g2) { return h->eval_trial(h->ctx, j, l, g2); }
    void accept() { h->accept(h->ctx); }
  } ops_{ops};
  mnl::NrOptions o;
  o.gtol = gtol;
  o.ftol = ftol;
  o.max_iter = max_iter;
  mnl::NrReport R;
  const int st = mnl::nr_fit(ops_, o, &R);
  out->iters = R.iters;
  out->halvings = R.halvings;
  out->evals = R.evals;
  out->status = R.status;
  out->stop_reason = R.stop_reason;
  for (int i = 0; i < 64; ++i) out->halvings_per_iter[i] = R.halvings_per_iter[i];
  out->loglik = R.loglik;
  out->grad_norm = R.grad_norm;
  out->delta_loglik = R.delta_loglik;
  out->min_margin = R.min_margin;
  for (int i = 0; i < 64; ++i) {
    out->loglik_per_iter[i] = R.loglik_per_iter[i];
    out->grad_norm_per_iter[i] = R.grad_norm_per_iter[i];
  }
  return st;
}

}  // extern "C"
