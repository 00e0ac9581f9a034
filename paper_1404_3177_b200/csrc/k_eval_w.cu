// Pass 1 for models with alternative-varying data, "group" mapping
// (k_eval_w): the same quantities as k_eval.cu —
//   a1 u_ik = xi_k + x_i.beta_k + z_ik.alpha_k + y_ik.gamma      (base: P:129-138)
//   a2 P_ik = e^{u_ik - m_i} / s_i                                (R12)
//   a3 l    = sum_i (u_{i,y_i} - m_i - log s_i)
//   a4 g    = X~^T R, Z_k^T r_k, sum_k Y_k^T r_k, r_ik = I(y_i = k) - P_ik
// and, for the Hessian pass, the rows Pr[i] = [P_i0..P_i,K-1, ybar_i] —
// with a mapping that issues about a third of the instructions per individual.
//
// Every WARP works alone (no CTA barrier in the main loop) on groups of 8 consecutive individuals,
// the 8 rows of one DMMA m-block:
//   * lane 0..16 bulk-copy the group's 8 Y rows, 8 Z rows and its 8 x p block of X into the warp's
//     own ring (two halves of 8 slots, one mbarrier each): while group n is computed, group n + 1
//     is already in flight (whole rows, 16-byte multiples, DRAM bytes = algorithmic bytes);
//   * X~ B on the FP64 tensor pipe (mma.sync m8n8k4): the C fragment leaves lane (c8, r4) with
//     individual c8's alternatives 8 nb + 2 r4 + {0, 1} — four lanes per individual, every lane a
//     fixed set of alternatives — so the Y / Z contributions are 16-byte shared loads of two
//     adjacent alternatives' rows and plain FMAs in that same register layout, the row softmax is a
//     lane-local reduction plus two shuffles, and all 32 lanes carry live alternatives
//     (K = 50: 56 slots per individual instead of 64);
//   * the gamma gradient stays in that layout (lane-private partials); the residual rows go to
//     shared memory once, from where X~^T R runs on DMMA (accumulators in registers for the whole
//     kernel) and the alpha gradient is formed with lanes over the K d elements of the Z row;
//   * ybar_i = y_{i,y_i} - sum_k r_ik y_ik (the same FMAs as the gamma gradient: sum_k r_ik = 0
//     regrouped), reduced over the individual's four lanes.
// CTA partials are combined over the warps in warp order, then over the CTAs by k_eval_finalize
// (deterministic). Conditions (eval_plan_w): K <= 64, p <= 31, f even <= 16, d <= 8, K d even,
// N >= 8, K d <= 256, two warps' rings fit in shared memory. Anything else takes k_eval.cu's paths.
#include <algorithm>
#include <cstdlib>

#include "eval_common.h"

namespace mnl {
namespace {

constexpr int GR = 8;                  // individuals per group (one DMMA m-block)
constexpr int WNS = 2 * GR;            // ring slots per warp (two halves)
constexpr int W_F = 16, W_D = 8;       // capacity: generic variables, alternative-specific variables
constexpr int W_MB = 4;                // m-blocks of x~ columns (q <= 32)
constexpr int W_AJ = 8;                // alpha-gradient elements per lane (K d <= 256)

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ void bulk_g2s(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

template <int NB, bool WP>
__global__ void __launch_bounds__(256, 1) k_eval_w(const EvalArgs A, const EvalWLayout L) {
  extern __shared__ __align__(16) double sm[];
  const int K = A.K, q = A.q, d = A.d, f = A.f, p = A.p, QP = A.QP, Kd = K * d;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, nwk = blockDim.x >> 5;
  const int r4 = lane & 3, c8 = lane >> 2;
  const int KS = L.KS, RS = L.RS, YS = L.YS, ZS = L.ZS, XH = L.XH;
  double* Bs = sm;                                  // [QP][KS]  Bs[a][k] = beta_k[a] (column 0: base)
  double* Cf = sm + L.off_cf;                       // alpha [K d], gamma [f]
  double* Wb = sm + L.off_warp + (size_t)w * L.warp_sz;
  uint64_t* bars = reinterpret_cast<uint64_t*>(Wb);  // [2]
  double* Xb = Wb + 2;                              // [2][XH]  the group's x rows [8][p]
  double* Rw = Xb + 2 * XH;                         // [8][RS]  residual rows of the group
  double* Yr = Rw + GR * RS;                        // [16][YS]
  double* Zr = Yr + WNS * YS;                       // [16][ZS]
  for (int idx = tid; idx < QP * KS; idx += blockDim.x) {
    const int a = idx / KS, k = idx - a * KS;
    Bs[idx] = (a < q && k >= 1 && k < K) ? A.coef[(k - 1) * q + a] : 0.0;
  }
  for (int idx = tid; idx < Kd + f; idx += blockDim.x) Cf[idx] = A.coef[A.off_alpha + idx];
  const double* alpha = Cf;
  const double* gamma = Cf + Kd;
  if (lane == 0) {
    mbar_init(bars, 1);
    mbar_init(bars + 1, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const unsigned bar_s = static_cast<unsigned>(__cvta_generic_to_shared(bars));
  const unsigned xb_s = static_cast<unsigned>(__cvta_generic_to_shared(Xb));
  const unsigned yr_s = static_cast<unsigned>(__cvta_generic_to_shared(Yr));
  const unsigned zr_s = static_cast<unsigned>(__cvta_generic_to_shared(Zr));
  const unsigned by = (unsigned)(K * f) * 8u, bz = (unsigned)Kd * 8u, bx = (unsigned)(GR * p) * 8u;
  const int64_t ngroups = (A.N + GR - 1) / GR;
  const int64_t wg = (int64_t)blockIdx.x * nwk + w, wstride = (int64_t)gridDim.x * nwk;
  // stage group g into ring half `half` (all lanes call). A ragged last group is read as the last
  // 8 rows of the data; its rows below g * 8 are masked where they are used.
  auto issue = [&](int64_t g, int half) {
    int64_t i0 = g * GR;
    if (i0 + GR > A.N) i0 = A.N - GR;
    const unsigned bar = bar_s + 8u * half;
    if (lane == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the half's previous generic reads
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(GR * (by + bz) + bx)
                   : "memory");
    }
    __syncwarp();
    if (lane < GR) {
      if (by) bulk_g2s(yr_s + 8u * (unsigned)((half * GR + lane) * YS), A.Y + (i0 + lane) * (int64_t)(K * f), by, bar);
    } else if (lane < 2 * GR) {
      if (bz) bulk_g2s(zr_s + 8u * (unsigned)((half * GR + lane - GR) * ZS), A.Z + (i0 + lane - GR) * (int64_t)Kd, bz, bar);
    } else if (lane == 2 * GR) {
      if (bx) bulk_g2s(xb_s + 8u * (unsigned)(half * XH), A.X + i0 * p, bx, bar);
    }
  };
  if (wg < ngroups) issue(wg, 0);
  if (wg + wstride < ngroups) issue(wg + wstride, 1);

  double G[W_MB][NB][2];  // beta gradient: x~ columns 8 mb + c8, alternatives 8 nb + 2 r4 + {0, 1}
#pragma unroll
  for (int mb = 0; mb < W_MB; ++mb)
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) G[mb][nb][0] = G[mb][nb][1] = 0.0;
  double gam[W_F];  // gamma gradient, lane-private partials
#pragma unroll
  for (int e = 0; e < W_F; ++e) gam[e] = 0.0;
  double acc[W_AJ];  // alpha gradient of the Z-row elements lane + 32 j
  int ke[W_AJ];      // ... and the alternative each belongs to
#pragma unroll
  for (int j = 0; j < W_AJ; ++j) {
    acc[j] = 0.0;
    const int e = lane + 32 * j;
    ke[j] = (d > 0 && e < Kd) ? e / d : 0;
  }
  double l_s = 0.0, l_c = 0.0;
  const int MBr = (QP + 7) / 8;
  // the last alternative block may hold alternatives >= K: their loads are clamped to K - 1
  // (finite data) and their utilities set to -inf
  constexpr int KL = 8 * (NB - 1);
  const bool ok_l0 = KL + 2 * r4 < K, ok_l1 = KL + 2 * r4 + 1 < K;
  const int kl0 = ok_l0 ? KL + 2 * r4 : K - 1, kl1 = ok_l1 ? KL + 2 * r4 + 1 : K - 1;
  auto alt = [&](int nb, int h) { return nb < NB - 1 ? 8 * nb + 2 * r4 + h : (h ? kl1 : kl0); };

  int n = 0;
  for (int64_t g = wg; g < ngroups; g += wstride, ++n) {
    const int half = n & 1;
    const int64_t i0t = g * GR;
    const int64_t i0 = i0t + GR > A.N ? A.N - GR : i0t;
    const int64_t gi = i0 + c8;          // this lane's individual
    const bool valid = gi >= i0t;        // (rows of a ragged last group seen by the previous one)
    int y = __ldg(A.choice + gi);
    if (y < 0 || y >= K) {
      if (valid && r4 == 0) atomicOr(A.err, 1);
      y = 0;
    }
    mbar_wait(bar_s + 8u * half, (unsigned)((n >> 1) & 1));
    const double* xb = Xb + half * XH;
    const double* yb = Yr + (half * GR + c8) * YS;
    const double* zb = Zr + (half * GR + c8) * ZS;

    // ---- a1: u = X~ B on DMMA (rows = the group's individuals) ----
    double u[NB][2];
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) u[nb][0] = u[nb][1] = 0.0;
    for (int a0 = 0; a0 < QP; a0 += 4) {
      const int a = a0 + r4;
      const double av = a == 0 ? 1.0 : (a <= p ? xb[c8 * p + a - 1] : 0.0);
#pragma unroll
      for (int nb = 0; nb < NB; ++nb) dmma884(u[nb][0], u[nb][1], av, Bs[a * KS + nb * 8 + c8]);
    }
    // ---- a1: + y_k . gamma (pairs of components, 16-byte loads) ----
#pragma unroll
    for (int e2 = 0; e2 < W_F / 2; ++e2) {
      if (2 * e2 < f) {
        const double2 g2 = *reinterpret_cast<const double2*>(gamma + 2 * e2);
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) {
          const double2 v0 = *reinterpret_cast<const double2*>(yb + alt(nb, 0) * f + 2 * e2);
          const double2 v1 = *reinterpret_cast<const double2*>(yb + alt(nb, 1) * f + 2 * e2);
          u[nb][0] = fma(v0.y, g2.y, fma(v0.x, g2.x, u[nb][0]));
          u[nb][1] = fma(v1.y, g2.y, fma(v1.x, g2.x, u[nb][1]));
        }
      }
    }
    // ---- a1: + z_k . alpha_k (alpha is laid out like the Z row) ----
#pragma unroll
    for (int c = 0; c < W_D; ++c) {
      if (c < d) {
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) {
          const int o0 = alt(nb, 0) * d + c, o1 = alt(nb, 1) * d + c;
          u[nb][0] = fma(zb[o0], alpha[o0], u[nb][0]);
          u[nb][1] = fma(zb[o1], alpha[o1], u[nb][1]);
        }
      }
    }
    // ---- a2 / a3: softmax over the individual's four lanes, loglik ----
    if (!ok_l0) u[NB - 1][0] = -INFINITY;
    if (!ok_l1) u[NB - 1][1] = -INFINITY;
    // shift by the (fp32-rounded) maximum: any shift is exact for the softmax; it only has to keep
    // e^{u - m} <= ~1 (R12)
    float mf = -INFINITY;
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) mf = fmaxf(mf, fmaxf((float)u[nb][0], (float)u[nb][1]));
    mf = fmaxf(mf, __shfl_xor_sync(0xffffffffu, mf, 1));
    mf = fmaxf(mf, __shfl_xor_sync(0xffffffffu, mf, 2));
    const double m = (double)mf;
    double ssum = 0.0, uyl = 0.0;
#pragma unroll
    for (int nb = 0; nb < NB; ++nb)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (8 * nb + 2 * r4 + h == y) uyl = u[nb][h];
        const double e = exp_shifted(u[nb][h] - m);
        u[nb][h] = e;
        ssum += e;
      }
    ssum += __shfl_xor_sync(0xffffffffu, ssum, 1);
    ssum += __shfl_xor_sync(0xffffffffu, ssum, 2);
    const double uy = __shfl_sync(0xffffffffu, uyl, (lane & ~3) | ((y & 7) >> 1));
    if (valid && r4 == 0) neu_add(l_s, l_c, (uy - m) - log(ssum));
    const double inv_s = recip_ge1(ssum);
    double r[NB][2];
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) {
      const int k = 8 * nb + 2 * r4;
      const double P0 = u[nb][0] * inv_s, P1 = u[nb][1] * inv_s;
      r[nb][0] = valid ? ((k == y ? 1.0 : 0.0) - P0) : 0.0;
      r[nb][1] = valid ? ((k + 1 == y ? 1.0 : 0.0) - P1) : 0.0;
      if (WP && valid) {
        double* pr = A.Pr + gi * A.ldP + k;
        if (nb < NB - 1 || ok_l1) *reinterpret_cast<double2*>(pr) = make_double2(P0, P1);
        else if (ok_l0) pr[0] = P0;
      }
    }
    if (A.want_grad || WP) {
      // ---- a4: gamma gradient sum_k y_ke r_k in the same layout; WP: ybar_e = y_{y,e} - that sum ----
      double gp[WP ? W_F : 1];
#pragma unroll
      for (int e2 = 0; e2 < W_F / 2; ++e2) {
        if (2 * e2 < f) {
          double a0 = 0.0, a1 = 0.0;
#pragma unroll
          for (int nb = 0; nb < NB; ++nb) {
            const double2 v0 = *reinterpret_cast<const double2*>(yb + alt(nb, 0) * f + 2 * e2);
            const double2 v1 = *reinterpret_cast<const double2*>(yb + alt(nb, 1) * f + 2 * e2);
            a0 = fma(v1.x, r[nb][1], fma(v0.x, r[nb][0], a0));
            a1 = fma(v1.y, r[nb][1], fma(v0.y, r[nb][0], a1));
          }
          gam[2 * e2] += a0;
          gam[2 * e2 + 1] += a1;
          if constexpr (WP) {
            gp[2 * e2] = a0;
            gp[2 * e2 + 1] = a1;
          }
        }
      }
      if constexpr (WP) {
#pragma unroll
        for (int e = 0; e < W_F; ++e) {
          if (e < f) {
            double s = gp[e];
            s += __shfl_xor_sync(0xffffffffu, s, 1);
            s += __shfl_xor_sync(0xffffffffu, s, 2);
            if (valid && (e & 3) == r4) A.Pr[gi * A.ldP + K + e] = yb[y * f + e] - s;
          }
        }
      }
    }
    if (A.want_grad) {
      // ---- residual rows to shared memory ----
#pragma unroll
      for (int nb = 0; nb < NB; ++nb)
        *reinterpret_cast<double2*>(Rw + c8 * RS + 8 * nb + 2 * r4) = make_double2(r[nb][0], r[nb][1]);
      __syncwarp();
      // ---- a4: alpha gradient, lanes over the K d elements of the Z row ----
      if (d > 0) {
        const double* zg = Zr + (half * GR) * ZS;
#pragma unroll
        for (int j = 0; j < W_AJ; ++j) {
          if (32 * j < Kd) {
            const int e = lane + 32 * j;
            if (e < Kd) {
              double a = acc[j];
#pragma unroll
              for (int i = 0; i < GR; ++i) a = fma(zg[i * ZS + e], Rw[i * RS + ke[j]], a);
              acc[j] = a;
            }
          }
        }
      }
      // ---- a4: beta gradient G += X~^T R on DMMA (k = the group's individuals) ----
#pragma unroll
      for (int ks = 0; ks < GR / 4; ++ks) {
        double bf[NB];
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) bf[nb] = Rw[(4 * ks + r4) * RS + nb * 8 + c8];
#pragma unroll
        for (int mb = 0; mb < W_MB; ++mb) {
          if (mb < MBr) {
            const int a = mb * 8 + c8;
            const double af = a == 0 ? 1.0 : (a <= p ? xb[(4 * ks + r4) * p + a - 1] : 0.0);
#pragma unroll
            for (int nb = 0; nb < NB; ++nb) dmma884(G[mb][nb][0], G[mb][nb][1], af, bf[nb]);
          }
        }
      }
    }
    __syncwarp();  // every lane is done with this half (ring, x block, residual rows)
    if (g + 2 * wstride < ngroups) issue(g + 2 * wstride, half);
  }

  // ---------------- CTA partials (fixed order) ----------------
  __syncthreads();  // every warp has consumed all it staged: the warp regions are free
  double* out = A.part + (size_t)blockIdx.x * A.n_part;
  double* V = sm + L.off_warp;                // [nwk][n_p]
  double* LL = V + (size_t)nwk * A.n_p;      // [nwk 32][2]
  LL[2 * tid] = l_s;
  LL[2 * tid + 1] = l_c;
  if (A.want_grad) {
    double* Vw = V + (size_t)w * A.n_p;
#pragma unroll
    for (int mb = 0; mb < W_MB; ++mb)
#pragma unroll
      for (int nb = 0; nb < NB; ++nb)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int a = mb * 8 + c8, k = 8 * nb + 2 * r4 + h;
          if (a < q && k >= 1 && k < K) Vw[(k - 1) * q + a] = G[mb][nb][h];
        }
#pragma unroll
    for (int j = 0; j < W_AJ; ++j) {
      const int e = lane + 32 * j;
      if (e < Kd) Vw[A.off_alpha + e] = acc[j];
    }
#pragma unroll
    for (int e = 0; e < W_F; ++e) {
      if (e < f) {
        const double s = warp_sum(gam[e]);
        if (lane == 0) Vw[A.off_gamma + e] = s;
      }
    }
  }
  __syncthreads();
  if (tid == 0) {
    double s = 0.0, c = 0.0;
    for (int t = 0; t < nwk * 32; t += 4) {
      neu_add(s, c, LL[2 * t]);
      neu_add(s, c, LL[2 * t + 1]);
    }
    out[0] = s;
    out[1] = c;
  }
  if (!A.want_grad) return;
  for (int idx = tid; idx < A.n_p; idx += blockDim.x) {
    double v = 0.0;
    for (int ww = 0; ww < nwk; ++ww) v += V[(size_t)ww * A.n_p + idx];
    out[2 + idx] = v;
  }
}

template <int NB, bool WP>
cudaError_t launch_w(const EvalPlan& plan, const EvalArgs& a, cudaStream_t st) {
  static uint64_t attr_mask = 0;
  cudaError_t e = set_once_per_device(attr_mask, [] {
    return cudaFuncSetAttribute(k_eval_w<NB, WP>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  });
  if (e != cudaSuccess) return e;
  k_eval_w<NB, WP><<<plan.w_grid, plan.w.nwk * 32, plan.w_smem, st>>>(a, plan.w);
  count_launch();
  return cudaGetLastError();
}

}  // namespace

// The group mapping's plan: layout of the shared memory and the grid; plan->w.nwk = 0 when the
// shape does not qualify.
void eval_plan_w(const Dims& D, EvalPlan* plan, int sms) {
  plan->w.nwk = 0;
  plan->w_grid = 0;
  plan->w_smem = 0;
  const int Kd = D.K * D.d, Kf = D.K * D.f;
  if ((D.d + D.f) == 0 || D.K > 64 || D.K < 2 || D.q > 8 * W_MB || D.f % 2 || D.f > W_F || D.d > W_D || Kd % 2 ||
      Kd > 32 * W_AJ || D.N < GR || getenv("MNL_NO_YZW"))
    return;
  // bulk copies need 16-byte-aligned sources: the x block of a ragged last group starts at row N - 8
  if ((D.N % GR) && ((D.N - GR) * D.p) % 2) return;
  EvalWLayout& L = plan->w;
  const int NB = (D.K + 7) / 8, QP = (D.q + 3) / 4 * 4;
  L.KS = pad4mod16(8 * NB);
  L.RS = pad4mod16(8 * NB);
  L.YS = Kf;
  while (L.YS % 4 != 2) ++L.YS;  // slot stride = 16 (mod 32) bytes: the 16-byte loads of two individuals' lanes
                                 // (4 x 16 bytes at a 2 f 8-byte pitch each) interleave without bank conflicts
  if (Kf == 0) L.YS = 0;
  L.ZS = Kd + (Kd & 1);
  L.XH = GR * D.p;
  L.off_cf = QP * L.KS;
  L.off_warp = L.off_cf + ((Kd + D.f + 1) & ~1);
  L.warp_sz = 2 + 2 * L.XH + GR * L.RS + WNS * L.YS + WNS * L.ZS;
  if (L.warp_sz < D.n_p + 64 + 2) return;  // the final partials reuse the warp regions
  L.warp_sz = (L.warp_sz + 1) & ~1;
  int nwk = 8;
  while (nwk >= 2 && (size_t)(L.off_warp + (size_t)nwk * L.warp_sz) * sizeof(double) > 227 * 1024) --nwk;
  if (nwk < 2) return;
  const int64_t ngroups = (D.N + GR - 1) / GR;
  int64_t grid = sms;
  if (grid * nwk > ngroups) grid = (ngroups + nwk - 1) / nwk;
  L.nwk = nwk;
  plan->w_grid = (int)grid;
  plan->w_smem = (size_t)(L.off_warp + (size_t)nwk * L.warp_sz) * sizeof(double);
}

cudaError_t launch_eval_w(const Dims& D, const EvalPlan& plan, const double* X, const double* Y, const double* Z,
                          const int32_t* choice, const double* coef, const Packed* pk, bool want_grad, bool writeP,
                          double* part, int* err, cudaStream_t st) {
  EvalArgs a{};
  a.N = D.N; a.K = D.K; a.p = D.p; a.f = D.f; a.d = D.d; a.q = D.q; a.n_p = D.n_p;
  a.off_alpha = D.off_alpha; a.off_gamma = D.off_gamma;
  a.QP = (D.q + 3) / 4 * 4;
  a.X = X; a.Y = Y; a.Z = Z; a.choice = choice; a.coef = coef;
  a.Pr = writeP ? pk->Pr : nullptr;
  a.ldP = writeP ? pk->ldP : 0;
  a.want_grad = want_grad; a.writeP = writeP;
  a.part = part; a.n_part = plan.n_part; a.err = err;
  const int NB = (D.K + 7) / 8;
#define MNL_W_CASE(NB_)                                                    \
  case NB_:                                                                \
    return writeP ? launch_w<NB_, true>(plan, a, st) : launch_w<NB_, false>(plan, a, st);
  switch (NB) {
    MNL_W_CASE(1)
    MNL_W_CASE(2)
    MNL_W_CASE(3)
    MNL_W_CASE(4)
    MNL_W_CASE(5)
    MNL_W_CASE(6)
    MNL_W_CASE(7)
    MNL_W_CASE(8)
  }
#undef MNL_W_CASE
  return cudaErrorInvalidValue;
}

}  // namespace mnl
