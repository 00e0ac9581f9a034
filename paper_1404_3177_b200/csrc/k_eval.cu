// Pass 1 of the Newton iteration, one fused streaming kernel:
//   a1 utilities   u_ik = xi_k + x_i.beta_k + z_ik.alpha_k + y_ik.gamma   (u_i0 carries
//                  only z_i0.alpha_0 + y_i0.gamma — the base normalisation of P:129-138 is the
//                  softmax's shift invariance: V_ik = u_ik - u_i0)
//   a2 softmax     P_ik = e^{u_ik - m_i} / s_i, m_i = max_k u_ik            (R12)
//   a3 loglik      l = sum_i (u_{i,y_i} - m_i - log s_i)
//   a4 gradient    g[beta_k]  = sum_i x~_i r_ik,  g[alpha_k] = sum_i z_ik r_ik,
//                  g[gamma]   = sum_i sum_k y_ik r_ik,  r_ik = I(y_i=k) - P_ik
//                  (raw y is exact: sum_k r_ik = 0 makes the base differencing of P:138 cancel)
// and, for the Hessian pass, the probability rows Pr[i] = [P_i0..P_i,K-1, ybar_i] with
// ybar_i = sum_k P_ik y_ik (the O(K) regrouping of the generic blocks).
//
// Layout: CTA = 8 warps, persistent over tiles of 32 individuals; a warp owns 4 individuals and
// its lanes the alternatives k = lane + 32*kk.  The utility GEMM X~ B uses B = [beta_k] staged
// transposed in shared memory; the beta-gradient X~^T R accumulates in registers per tile and
// in CTA-owned shared memory across tiles.  CTA partials are reduced in a fixed order by
// k_eval_finalize, so results are deterministic.
#include <algorithm>
#include <cmath>
#include <cstdio>

#include "internal.h"

namespace mnl {

namespace {

constexpr int TI = 32;   // individuals per tile
constexpr int NW = 8;    // warps per CTA
constexpr int IPW = 4;   // individuals per warp per tile

struct EvalArgs {
  int64_t N;
  int K, p, f, d, q, n_p, off_alpha, off_gamma;
  const double* X;
  const double* Y;
  const double* Z;
  const int32_t* choice;
  const double* coef;
  double* Pr;
  int ldP;
  int want_grad;
  int writeP;
  double* part;
  int n_part;
  int* err;
};

__device__ __forceinline__ void neu_add(double& s, double& c, double x) {
  // Neumaier compensated summation (a3: R7 requires compensated loglik sums).
  double t = s + x;
  if (fabs(s) >= fabs(x)) c += (s - t) + x;
  else c += (x - t) + s;
  s = t;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int KPL>
__global__ void __launch_bounds__(NW * 32) k_eval_kernel(const EvalArgs A) {
  extern __shared__ __align__(16) double sm[];
  constexpr int KP = 32 * KPL;
  const int K = A.K, q = A.q, d = A.d, f = A.f, p = A.p;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  double* Bs = sm;                        // [q][KP]   Bs[a][k] = beta_k[a], 0 for k = 0 / k >= K
  double* Gs = Bs + q * KP;               // [q][KP]   beta-gradient accumulators (CTA-owned)
  double* Xs = Gs + q * KP;               // [TI][q]   x~ rows of the tile
  double* Rs = Xs + TI * q;               // [TI][KP]  residuals r_ik
  double* Wa = Rs + TI * KP;              // [NW][KPL][d][32] alpha-gradient, lane-private
  double* Wg = Wa + NW * KPL * d * 32;    // [NW][f][32]      gamma-gradient, lane-private
  double* Cf = Wg + NW * f * 32;          // [K*d + f]        alpha_0..alpha_{K-1}, gamma

  for (int idx = tid; idx < q * KP; idx += blockDim.x) {
    int a = idx / KP, k = idx - a * KP;
    Bs[idx] = (k >= 1 && k < K) ? A.coef[(k - 1) * q + a] : 0.0;
    Gs[idx] = 0.0;
  }
  for (int idx = tid; idx < NW * KPL * d * 32 + NW * f * 32; idx += blockDim.x) Wa[idx] = 0.0;
  for (int idx = tid; idx < K * d + f; idx += blockDim.x) Cf[idx] = A.coef[A.off_alpha + idx];
  const double* alpha = Cf;
  const double* gamma = Cf + K * d;

  double l_s = 0.0, l_c = 0.0;  // this warp's loglik (Neumaier), identical on all lanes
  const int64_t ntiles = (A.N + TI - 1) / TI;

  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t i0 = tile * TI;
    const int nt = (int)(A.N - i0 < TI ? A.N - i0 : TI);
    __syncthreads();  // previous tile's phase C done with Xs / Rs; setup above visible
    for (int e = tid; e < TI * q; e += blockDim.x) {
      int i = e / q, a = e - i * q;
      double v = 0.0;
      if (i < nt) v = (a == 0) ? 1.0 : A.X[(i0 + i) * p + (a - 1)];
      Xs[e] = v;
    }
    __syncthreads();

    // ---- phase B: a1 + a2 + a3 (+ residuals, alpha/gamma gradients, P rows) ----
    double u[IPW][KPL];
#pragma unroll
    for (int j = 0; j < IPW; ++j)
#pragma unroll
      for (int kk = 0; kk < KPL; ++kk) u[j][kk] = 0.0;
    for (int a = 0; a < q; ++a) {
      double xv[IPW];
#pragma unroll
      for (int j = 0; j < IPW; ++j) xv[j] = Xs[(w * IPW + j) * q + a];
#pragma unroll
      for (int kk = 0; kk < KPL; ++kk) {
        double b = Bs[a * KP + lane + 32 * kk];
#pragma unroll
        for (int j = 0; j < IPW; ++j) u[j][kk] = fma(xv[j], b, u[j][kk]);
      }
    }
#pragma unroll
    for (int j = 0; j < IPW; ++j) {
      const int il = w * IPW + j;
      double* Rrow = Rs + il * KP;
      if (il >= nt) {  // ragged tail: no contribution
        if (A.want_grad)
#pragma unroll
          for (int kk = 0; kk < KPL; ++kk) Rrow[lane + 32 * kk] = 0.0;
        continue;
      }
      const int64_t i = i0 + il;
#pragma unroll
      for (int kk = 0; kk < KPL; ++kk) {
        const int k = lane + 32 * kk;
        if (k < K) {
          double v = u[j][kk];
          const double* zr = A.Z + (i * K + k) * d;
          for (int c = 0; c < d; ++c) v = fma(zr[c], alpha[k * d + c], v);
          const double* yr = A.Y + (i * K + k) * f;
          for (int e = 0; e < f; ++e) v = fma(yr[e], gamma[e], v);
          u[j][kk] = v;
        } else {
          u[j][kk] = -INFINITY;
        }
      }
      double m = u[j][0];
#pragma unroll
      for (int kk = 1; kk < KPL; ++kk) m = fmax(m, u[j][kk]);
      m = warp_max(m);
      double ex[KPL], s = 0.0;
#pragma unroll
      for (int kk = 0; kk < KPL; ++kk) {
        ex[kk] = (lane + 32 * kk < K) ? exp(u[j][kk] - m) : 0.0;
        s += ex[kk];
      }
      s = warp_sum(s);
      const double inv_s = 1.0 / s;
      int y = A.choice[i];
      if (y < 0 || y >= K) {
        if (lane == 0) atomicOr(A.err, 1);
        y = 0;
      }
      double uy_l = 0.0;
#pragma unroll
      for (int kk = 0; kk < KPL; ++kk)
        if (kk == (y >> 5)) uy_l = u[j][kk];
      const double uy = __shfl_sync(0xffffffffu, uy_l, y & 31);
      neu_add(l_s, l_c, uy - (m + log(s)));

      double P[KPL];
#pragma unroll
      for (int kk = 0; kk < KPL; ++kk) P[kk] = ex[kk] * inv_s;
      if (A.writeP) {
        double* pr = A.Pr + i * A.ldP;
#pragma unroll
        for (int kk = 0; kk < KPL; ++kk)
          if (lane + 32 * kk < K) pr[lane + 32 * kk] = P[kk];
        for (int e = 0; e < f; ++e) {
          double v = 0.0;
#pragma unroll
          for (int kk = 0; kk < KPL; ++kk) {
            const int k = lane + 32 * kk;
            if (k < K) v = fma(P[kk], A.Y[(i * K + k) * f + e], v);
          }
          v = warp_sum(v);
          if (lane == 0) pr[K + e] = v;
        }
      }
      if (A.want_grad) {
#pragma unroll
        for (int kk = 0; kk < KPL; ++kk) {
          const int k = lane + 32 * kk;
          const double r = (k < K) ? ((k == y ? 1.0 : 0.0) - P[kk]) : 0.0;
          Rrow[k] = r;
          if (k < K) {
            const double* zr = A.Z + (i * K + k) * d;
            for (int c = 0; c < d; ++c) Wa[((w * KPL + kk) * d + c) * 32 + lane] += zr[c] * r;
          }
        }
        for (int e = 0; e < f; ++e) {
          double v = 0.0;
#pragma unroll
          for (int kk = 0; kk < KPL; ++kk) {
            const int k = lane + 32 * kk;
            if (k < K) v = fma(A.Y[(i * K + k) * f + e], (k == y ? 1.0 : 0.0) - P[kk], v);
          }
          Wg[(w * f + e) * 32 + lane] += v;
        }
      }
    }
    if (!A.want_grad) continue;
    __syncthreads();

    // ---- phase C: beta gradient  G[a][k] += sum_i x~_ia r_ik  (a4, X~^T R) ----
    for (int ma0 = 0; ma0 * 8 < q; ma0 += 4) {
      double acc[4][KPL];
#pragma unroll
      for (int m4 = 0; m4 < 4; ++m4)
#pragma unroll
        for (int kk = 0; kk < KPL; ++kk) acc[m4][kk] = 0.0;
      for (int i = 0; i < TI; ++i) {
        double r[KPL];
#pragma unroll
        for (int kk = 0; kk < KPL; ++kk) r[kk] = Rs[i * KP + lane + 32 * kk];
#pragma unroll
        for (int m4 = 0; m4 < 4; ++m4) {
          const int a = w + 8 * (ma0 + m4);
          const double x = (a < q) ? Xs[i * q + a] : 0.0;
#pragma unroll
          for (int kk = 0; kk < KPL; ++kk) acc[m4][kk] = fma(x, r[kk], acc[m4][kk]);
        }
      }
#pragma unroll
      for (int m4 = 0; m4 < 4; ++m4) {
        const int a = w + 8 * (ma0 + m4);
        if (a < q)
#pragma unroll
          for (int kk = 0; kk < KPL; ++kk) Gs[a * KP + lane + 32 * kk] += acc[m4][kk];
      }
    }
  }

  // ---- CTA partials (fixed order) ----
  __syncthreads();
  double* out = A.part + (size_t)blockIdx.x * A.n_part;
  double* wl = Rs;  // reuse: per-warp loglik pairs
  if (lane == 0) { wl[2 * w] = l_s; wl[2 * w + 1] = l_c; }
  __syncthreads();
  if (tid == 0) {
    double s = 0.0, c = 0.0;
    for (int ww = 0; ww < NW; ++ww) { neu_add(s, c, wl[2 * ww]); neu_add(s, c, wl[2 * ww + 1]); }
    out[0] = s;
    out[1] = c;
  }
  if (!A.want_grad) return;
  for (int idx = tid; idx < (K - 1) * q; idx += blockDim.x) {
    int k = idx / q + 1, a = idx - (k - 1) * q;
    out[2 + idx] = Gs[a * KP + k];
  }
  for (int idx = tid; idx < K * d; idx += blockDim.x) {
    int k = idx / d, c = idx - k * d, kk = k >> 5, ln = k & 31;
    double v = 0.0;
    for (int ww = 0; ww < NW; ++ww) v += Wa[((ww * KPL + kk) * d + c) * 32 + ln];
    out[2 + A.off_alpha + idx] = v;
  }
  for (int e = tid; e < f; e += blockDim.x) {
    double v = 0.0;
    for (int ww = 0; ww < NW; ++ww)
      for (int ln = 0; ln < 32; ++ln) v += Wg[(ww * f + e) * 32 + ln];
    out[2 + A.off_gamma + e] = v;
  }
}

__global__ void __launch_bounds__(256) k_eval_finalize(const double* __restrict__ part, int n_part,
                                                      int nblk, int n_p, int want_grad,
                                                      double* grad, double* loglik_out,
                                                      double* scal, const int* err,
                                                      unsigned* counter) {
  __shared__ double red[256];
  __shared__ bool last;
  const int tid = threadIdx.x;
  const int r = blockIdx.x * 256 + tid;
  if (want_grad && r < n_p) {
    double s = 0.0, c = 0.0;
    for (int b = 0; b < nblk; ++b) neu_add(s, c, part[(size_t)b * n_part + 2 + r]);
    grad[r] = s + c;
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  double g2 = 0.0;
  if (want_grad)
    for (int j = tid; j < n_p; j += 256) {
      double v = __ldcg(grad + j);
      g2 = fma(v, v, g2);
    }
  red[tid] = g2;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (tid < o) red[tid] += red[tid + o];
    __syncthreads();
  }
  if (tid == 0) {
    double s = 0.0, c = 0.0;
    for (int b = 0; b < nblk; ++b) {
      neu_add(s, c, part[(size_t)b * n_part]);
      neu_add(s, c, part[(size_t)b * n_part + 1]);
    }
    const double l = s + c;
    scal[0] = l;
    scal[1] = red[0];
    scal[2] = (double)(*err);
    if (loglik_out) *loglik_out = l;
    *counter = 0u;
  }
}

__global__ void k_pack(int64_t N, int64_t Npad, int p, int Kd, const double* __restrict__ X,
                       const double* __restrict__ Z, double* Xp, int ldX, double* Zp, int ldZ) {
  const int64_t nx = Npad * ldX, nz = Zp ? Npad * ldZ : 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nx + nz;
       e += (int64_t)gridDim.x * blockDim.x) {
    if (e < nx) {
      const int64_t i = e / ldX;
      const int a = (int)(e - i * ldX);
      double v = 0.0;
      if (i < N) v = (a == 0) ? 1.0 : (a <= p ? X[i * p + a - 1] : 0.0);
      Xp[e] = v;
    } else {
      const int64_t t = e - nx, i = t / ldZ;
      const int j = (int)(t - i * ldZ);
      Zp[t] = (i < N && j < Kd) ? Z[i * Kd + j] : 0.0;
    }
  }
}

__global__ void k_axpy_pow2(int n, const double* theta, const double* delta, int j, double* out) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) out[r] = theta[r] + ldexp(delta[r], -j);  // a7: theta + delta / 2^j, exact scaling
}

template <int KPL>
cudaError_t launch_k(const EvalPlan& plan, const EvalArgs& a, cudaStream_t st) {
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(k_eval_kernel<KPL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         200 * 1024);
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  k_eval_kernel<KPL><<<plan.grid, plan.block, plan.smem, st>>>(a);
  count_launch();
  return cudaGetLastError();
}

}  // namespace

static size_t eval_smem(const Dims& D, int kpl) {
  const int KP = 32 * kpl;
  size_t n = 2 * (size_t)D.q * KP + (size_t)TI * D.q + (size_t)TI * KP + (size_t)NW * kpl * D.d * 32 +
             (size_t)NW * D.f * 32 + (size_t)D.K * D.d + D.f;
  return n * sizeof(double);
}

bool eval_plan(const Dims& D, EvalPlan* plan, int sms) {
  int kpl = 1;
  while (32 * kpl < D.K) kpl *= 2;
  if (kpl > 8) return false;
  size_t smem = eval_smem(D, kpl);
  if (smem > 200 * 1024) return false;
  plan->kpl = kpl;
  plan->smem = smem;
  plan->block = NW * 32;
  int per_sm = (int)((227 * 1024) / (smem + 1024));
  if (per_sm < 1) per_sm = 1;
  if (per_sm > 4) per_sm = 4;
  const int64_t ntiles = (D.N + TI - 1) / TI;
  int64_t grid = (int64_t)sms * per_sm;
  if (grid > ntiles) grid = ntiles;
  plan->grid = (int)grid;
  plan->n_part = 2 + D.n_p;
  return true;
}

cudaError_t launch_eval(const Dims& D, const EvalPlan& plan, const double* X, const double* Y,
                        const double* Z, const int32_t* choice, const double* coef,
                        const Packed* pk, bool want_grad, bool writeP, double* part, int* err,
                        cudaStream_t st) {
  EvalArgs a;
  a.N = D.N; a.K = D.K; a.p = D.p; a.f = D.f; a.d = D.d; a.q = D.q; a.n_p = D.n_p;
  a.off_alpha = D.off_alpha; a.off_gamma = D.off_gamma;
  a.X = X; a.Y = Y; a.Z = Z; a.choice = choice; a.coef = coef;
  a.Pr = writeP ? pk->Pr : nullptr;
  a.ldP = writeP ? pk->ldP : 0;
  a.want_grad = want_grad; a.writeP = writeP;
  a.part = part; a.n_part = plan.n_part; a.err = err;
  switch (plan.kpl) {
    case 1: return launch_k<1>(plan, a, st);
    case 2: return launch_k<2>(plan, a, st);
    case 4: return launch_k<4>(plan, a, st);
    case 8: return launch_k<8>(plan, a, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_eval_finalize(const Dims& D, const EvalPlan& plan, const double* part,
                                 bool want_grad, double* grad, double* loglik_out, double* scal,
                                 const int* err, unsigned* counter, cudaStream_t st) {
  int blocks = want_grad ? (D.n_p + 255) / 256 : 1;
  k_eval_finalize<<<blocks, 256, 0, st>>>(part, plan.n_part, plan.grid, D.n_p, want_grad, grad,
                                          loglik_out, scal, err, counter);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_pack(const Dims& D, const Packed& pk, const double* X, const double* Z,
                        cudaStream_t st) {
  int64_t total = pk.Npad * pk.ldX + (D.d ? pk.Npad * pk.ldZ : 0);
  int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
  k_pack<<<blocks, 256, 0, st>>>(D.N, pk.Npad, D.p, D.K * D.d, X, Z, pk.Xp, pk.ldX,
                                 D.d ? pk.Zp : nullptr, pk.ldZ);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_axpy_pow2(int n, const double* theta, const double* delta, int j, double* out,
                             cudaStream_t st) {
  k_axpy_pow2<<<(n + 255) / 256, 256, 0, st>>>(n, theta, delta, j, out);
  count_launch();
  return cudaGetLastError();
}

}  // namespace mnl
