// Internal declarations shared by the CUDA translation units of libmnl.so.
// (Not part of the ABI; see include/mnl.h.)
#pragma once
#include <cstdint>
#include <mutex>
#include <cuda_runtime.h>

namespace mnl {

// ---- one-time per-device setup (thread-safe) ----------------------------------------------
// Kernel attributes set with cudaFuncSetAttribute are per device; f runs once per device for each
// `mask` (one per call site), under a process-wide lock so no launch can overtake the setter.
std::mutex& attr_mutex();
template <class F>
cudaError_t set_once_per_device(uint64_t& mask, F&& f) {
  std::lock_guard<std::mutex> lk(attr_mutex());
  int dev = 0;
  cudaGetDevice(&dev);
  if ((mask >> dev) & 1u) return cudaSuccess;
  const cudaError_t e = f();
  if (e == cudaSuccess) mask |= uint64_t(1) << dev;
  return e;
}

// Problem dimensions and the layout constants derived from them.
struct Dims {
  int64_t N;      // individuals
  int K, p, f, d; // alternatives, X cols, Y (generic) cols, Z (alt-specific) cols
  int q;          // p + 1 (intercept first)
  int n_beta;     // (K-1) q
  int n_alpha;    // K d
  int n_p;        // n_beta + n_alpha + f
  int off_alpha;  // = n_beta
  int off_gamma;  // = n_beta + n_alpha
};

// Packed per-individual rows in library scratch.
// Row strides are even (16-byte rows for bulk copies) and = 4 (mod 16) doubles, which makes
// the 4-row x 8-column fragment gathers of the Hessian generator bank-conflict-free (64-bit
// shared loads are served per half-warp: 4 rows x 4 columns must hit 16 distinct bank pairs).
struct Packed {
  int64_t Npad;   // N rounded up to a multiple of kRowPad; rows >= N are zero
  int ldX;        // Xp [Npad][ldX]: 1, x_i1..x_ip, 0...
  int ldZ;        // Zp [Npad][ldZ]: z_i (K*d), 0...
  int ldP;        // Pr [Npad][ldP]: P_i0..P_i,K-1, ybar_i1..ybar_if, 0...
  double* Xp;
  double* Zp;
  double* Pr;
};

constexpr int kRowPad = 64;   // Npad multiple (>= the largest chunk KC)

inline int pad4mod16(int n) {  // smallest m >= n with m % 16 == 4
  int m = n;
  while (m % 16 != 4) ++m;
  return m;
}

// ---- launch accounting --------------------------------------------------------------
void count_launch(int n = 1);

// ---- k_eval.cu -------------------------------------------------------------------------
// Per-CTA partials layout: [2 + n_p] doubles: l_sum, l_comp, grad[n_p].
// Shared-memory layout (in doubles) of the group mapping (k_eval_w.cu); nwk = 0: not in use.
struct EvalWLayout {
  int T, S, NBW;            // teams per CTA (0: not in use), warps per team, alternative blocks per warp
  int KS, RS, YS, ZS, XH;   // strides: beta table rows, residual rows, Y / Z ring slots, x block of a group
  int off_gam, off_team, team_sz;
  size_t smem;
};
struct EvalPlan {
  int grid, block, kpl, cm;
  int yzs, ns;  // alternative-varying rows staged per warp (bulk copies into an ns-slot ring)
  int stream;   // alpha / gamma gradients by k_yz_grad from residual rows (rg doubles of scratch)
  int64_t rg;
  int ti;       // individuals per tile
  size_t smem;
  int n_part;  // 2 + n_p
  // the group mapping (k_eval_w.cu), used by launch_eval and launch_hessvec when w.T > 0
  EvalWLayout w;
  int w_grid;
  // the two-group X-only kernel (k_eval_x.cu), used when x_grid > 0
  int x_grid, x_cm, x_scr, x_hv;  // x_hv: also for launch_hessvec
  size_t x_smem;
};
bool eval_plan(const Dims& D, EvalPlan* plan, int device_sms);
void eval_plan_w(const Dims& D, EvalPlan* plan, int device_sms);
void eval_plan_x(const Dims& D, EvalPlan* plan, int device_sms);
// The two-group X-only kernel (k_eval_x.cu): evaluation (hv = false) or Hessian-vector product.
cudaError_t launch_eval_x(const Dims& D, const EvalPlan& plan, const double* X, const int32_t* choice,
                          const double* coef, const Packed* pk, bool want_grad, bool writeP, bool hv, double* part,
                          int* err, cudaStream_t st);
// CTA partial rows written by launch_eval / launch_hessvec with this plan
inline int eval_nblk(const EvalPlan& ep, bool hv) {
  return ep.w.T ? ep.w_grid : ((ep.x_grid && (!hv || ep.x_hv)) ? ep.x_grid : ep.grid);
}
// doubles of the `part` scratch a launch with this plan needs (CTA partials + stream-mode residual rows)
inline size_t eval_part_doubles(const EvalPlan& ep) {
  const int g = ep.grid > ep.w_grid ? ep.grid : ep.w_grid;
  return (size_t)(g > ep.x_grid ? g : ep.x_grid) * ep.n_part + ep.rg;
}
// Pass 1 (a1-a4): utilities, softmax, loglik partials, gradient partials (if want_grad),
// and the probability rows Pr (if writeP). part: [grid][n_part].
cudaError_t launch_eval(const Dims& D, const EvalPlan& plan, const double* X, const double* Y,
                        const double* Z, const int32_t* choice, const double* coef,
                        const Packed* pk, bool want_grad, bool writeP, double* part, int* err,
                        cudaStream_t st);
// Fixed-order reduction of the CTA partials -> loglik, grad (optional); scal[0] = l,
// scal[1] = ||g||^2, scal[2] = err flag (as double), *status_out (if given) = the mnl_status of the
// evaluation (MNL_ERR_ARG for a bad choice, MNL_ERR_NONFINITE). `counter` is a zeroed int.
// Hessian-vector product pass: part receives H v (gradient slots) from P_i in pk->Pr (written by the
// last evaluation with writeP) and s_i = J_i v.
cudaError_t launch_hessvec(const Dims& D, const EvalPlan& plan, const double* X, const double* Y, const double* Z,
                           const int32_t* choice, const double* v, const Packed* pk, double* part, int* err,
                           cudaStream_t st);
// CG vector steps (single CTA, n <= 16384, deterministic): Ap = -Hp & out = p.Ap;
// delta += alpha p, r -= alpha Ap & out = r.r; p = r + beta p
cudaError_t launch_cg_curv(int n, const double* p, const double* hp, double* ap, double* out, cudaStream_t st);
cudaError_t launch_cg_update(int n, double alpha, const double* p, const double* ap, double* delta, double* r,
                             double* out, cudaStream_t st);
cudaError_t launch_cg_dir(int n, double beta, const double* r, double* p, cudaStream_t st);
cudaError_t launch_eval_finalize(const Dims& D, const EvalPlan& plan, const double* part,
                                 bool want_grad, double* grad, double* loglik_out, double* scal,
                                 const int* err, unsigned* counter, cudaStream_t st,
                                 int* status_out = nullptr, bool hv = false);
// The team mapping (k_eval_w.cu; its instantiations are split over three translation units by f).
cudaError_t launch_eval_w(const Dims& D, const EvalPlan& plan, const double* X, const double* Y, const double* Z,
                          const int32_t* choice, const double* coef, const Packed* pk, bool want_grad, bool writeP,
                          bool hv, double* part, int* err, cudaStream_t st);
cudaError_t launch_eval_w_part0(const Dims& D, const EvalPlan& plan, const double* X, const double* Y, const double* Z,
                          const int32_t* choice, const double* coef, const Packed* pk, bool want_grad, bool writeP,
                          bool hv, double* part, int* err, cudaStream_t st);
cudaError_t launch_eval_w_part1(const Dims& D, const EvalPlan& plan, const double* X, const double* Y, const double* Z,
                          const int32_t* choice, const double* coef, const Packed* pk, bool want_grad, bool writeP,
                          bool hv, double* part, int* err, cudaStream_t st);
cudaError_t launch_eval_w_part2(const Dims& D, const EvalPlan& plan, const double* X, const double* Y, const double* Z,
                          const int32_t* choice, const double* coef, const Packed* pk, bool want_grad, bool writeP,
                          bool hv, double* part, int* err, cudaStream_t st);
// Data-parallel exchange of one evaluation: xbuf [2 + n] = [l, bad-choice flag, g] from the
// finalised scalars [l, ||g||^2, flag] (+ g, or zeros if grad is null); after the all-reduce,
// grad (if not null) <- the summed g and scal <- [l, ||g||^2, flag] of the sums.
cudaError_t launch_dp_gather(int n, const double* scal, const double* grad, double* xbuf, cudaStream_t st);
cudaError_t launch_dp_scatter(int n, const double* xbuf, double* grad, double* scal, cudaStream_t st);
cudaError_t launch_pack(const Dims& D, const Packed& pk, const double* X, const double* Z,
                        cudaStream_t st);
cudaError_t launch_axpy_pow2(int n, const double* theta, const double* delta, int j,
                             double* out, cudaStream_t st);

// ---- k_hess.cu -------------------------------------------------------------------------
struct HessPlan;
HessPlan* hess_plan_create(const Dims& D, const Packed& pk, int device_sms);
void hess_plan_destroy(HessPlan*);
size_t hess_plan_bytes(const HessPlan*);
// Assemble the Hessian from Pr/Xp/Zp (+ Y for the arrow part). sign = +1 writes H,
// sign = -1 writes -H (the Newton system matrix). out: [n_p][ld_out], or with ld_out < 0 the packed
// upper triangle (row r: columns r..n_p-1 at r n_p - r (r - 1) / 2), the data-parallel exchange.
cudaError_t launch_hessian(HessPlan* hp, const Dims& D, const Packed& pk, const double* Y,
                           double* out, int ld_out, double sign, cudaStream_t st);
// Call after re-packing the design rows (Xp / Zp): invalidates data the plan derived from them.
void hess_plan_design_changed(HessPlan* hp);
// Phase times of the last launch_hessian (valid once the stream has passed it).
void hess_last_times(HessPlan* hp, double out[7]);

// Packed upper triangle of a symmetric dev [n][n] matrix (row i: columns i..n-1) and back (mirrored).
cudaError_t launch_sym_pack(int n, const double* H, double* out, cudaStream_t st);
cudaError_t launch_sym_unpack(int n, const double* in, double* H, cudaStream_t st);

// ---- k_chol.cu -------------------------------------------------------------------------
// Factorisation state (tile-major factor, inverse diagonal blocks, tile / block flags, the forward
// solution): one per workspace.
struct CholCtx;
CholCtx* chol_ctx_create();
void chol_ctx_destroy(CholCtx*);
// Lower Cholesky of the SPD n x n matrix A (lda) written into A's lower triangle (the tile-DAG
// factorisation, then a tile-major -> row-major copy); info: device int, set != 0 on failure.
cudaError_t launch_cholesky(CholCtx* cc, int n, double* A, int lda, int* info, cudaStream_t st);
// Solve A x = b: the tile-DAG factorisation of A (A itself is only read; the factor stays in the
// context's tile-major copy) with the forward solve fused into its diagonal tiles, then the
// backward solve (one kernel; nothing more for n <= 64). x may alias b.
cudaError_t launch_cholesky_solve_fused(CholCtx* cc, int n, double* A, int lda, int* info, const double* b,
                                        double* x, cudaStream_t st);
// se_j = sqrt([(L L^T)^{-1}]_jj) for the factor L in the lower triangle of L (lda); the strict upper
// triangle of L is overwritten (workspace for the blocks of L^{-1}).
cudaError_t launch_inv_diag_sqrt(CholCtx* cc, int n, double* L, int lda, double* se, cudaStream_t st);
// The Linv blocks of the last factor are reused by launch_chol_solve / launch_inv_diag_sqrt when the
// same pointer and n come back; chol_forget_factor() drops that association (a caller-supplied L).
void chol_forget_factor(CholCtx* cc);
// x = (L L^T)^{-1} b ; x may alias b.
cudaError_t launch_chol_solve(CholCtx* cc, int n, const double* L, int lda, const double* b, double* x,
                              cudaStream_t st);

}  // namespace mnl
