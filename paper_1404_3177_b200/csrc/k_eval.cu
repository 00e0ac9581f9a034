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
// Layout: CTA = 8 warps, persistent over tiles of individuals (X tiles prefetched with
// cp.async, double-buffered).  The two dense contractions run on the FP64 tensor pipe
// (mma.sync m8n8k4, SASS DMMA.8x8x4):
//   phase B  U = X~ B   (warp w: individuals 8w..8w+7 x all alternatives; the C fragment gives
//            each lane 2 alternatives per 8-block of one individual, so the row softmax is a
//            local reduction plus two shuffles);
//   phase C  G += X~^T R (the beta gradient; CTA-persistent accumulators in registers).
// Phase E (only with Y or Z) folds the alpha/gamma gradients and ybar with lanes over
// alternatives. Three variants: YZS (16-row tiles; every warp bulk-copies the Y/Z rows of its own
// individuals into a 2-4 slot shared-memory ring and computes them in pairs; see phase_e_smem),
// the register path (direct L1 loads, values held in registers) and the general direct path.
// CTA partials are reduced in a fixed order by k_eval_finalize (deterministic).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "eval_common.h"

namespace mnl {

namespace {

constexpr int NW = 8;    // warps per CTA
// individuals per tile: 8 warps x 8 rows, halved for K > 128 or with alternative-varying data
// (whose per-warp row staging needs the shared memory)
// (K > 128, KPL = 8: 16 rows, utilities stashed in shared memory like the Y/Z paths -- holding the
// 32 alternative blocks of a row in registers spilled)
__host__ __device__ constexpr int tile_rows(int kpl, bool yz) { return kpl >= 8 ? 16 : (yz ? 32 : 64); }


// Phase E (only with Y or Z): per individual, lanes over alternatives (k = lane + 32 kk). Lane k
// reads its alternative's y_ik (f contiguous doubles) and z_ik (d) straight from the caller's
// arrays: a warp-wide load touches one 32-byte sector per lane and the following components hit
// the same sectors in L1 (the tile's Y and Z blocks were prefetched into L2). Pass 1: corr =
// z.alpha + y.gamma, softmax, loglik, P (global Pr) and r (Rs); pass 2 (L1 hits): ybar and the
// gamma / alpha gradients. This general version handles any f, d; phase_e_reg below keeps an
// individual's values in registers when they fit.
template <int KPL>
__host__ __device__ constexpr int gam_regs() { return KPL <= 2 ? 16 : 8; }  // gamma-gradient partials held in registers

template <int KPL, bool HV>
__device__ __forceinline__ void phase_e(const EvalArgs& A, const double* Us, double* Rs, const int* ch_t, double* red,
                                        const double* alpha, const double* gamma, double* Wa, double (&gam)[gam_regs<KPL>()],
                                        double& l_s, double& l_c, int64_t i0, int nt, int KPS, int w, int lane) {
  const int K = A.K, d = A.d, f = A.f;
  const int rows = (A.TI + NW - 1) / NW;  // individuals per warp per tile
  const int ib = w * rows;
  const int n_mine = min(rows, nt - ib);
  for (int ii = ib + max(n_mine, 0); ii < ib + rows; ++ii)  // ragged tail: zero residual rows
    for (int k = lane; k < KPS; k += 32) Rs[ii * KPS + k] = 0.0;
  bool kok[KPL];  // this lane's alternatives exist
#pragma unroll
  for (int kk = 0; kk < KPL; ++kk) kok[kk] = lane + 32 * kk < K;
  for (int jj = 0; jj < n_mine; ++jj) {
    const int ii = ib + jj;
    const int64_t gi = i0 + ii;
    const double* yl = A.Y + (gi * K + lane) * f;  // y_{i,lane+32kk,e} = yl[32 kk f + e]
    const double* zl = A.Z + (gi * K + lane) * d;  // z_{i,lane+32kk,c} = zl[32 kk d + c]
    int y = ch_t[ii];
    if (y < 0 || y >= K) {
      if (lane == 0) atomicOr(A.err, 1);
      y = 0;
    }
    // ---- pass 1: u_k += y_k . gamma + z_k . alpha_k (two accumulation chains per alternative) ----
    double ua[KPL], ub[KPL];
#pragma unroll
    for (int kk = 0; kk < KPL; ++kk) {
      ua[kk] = kok[kk] ? Us[ii * KPS + lane + 32 * kk] : 0.0;
      ub[kk] = 0.0;
    }
    {
      constexpr int JB4 = KPL >= 4 ? 2 : 4;  // components per batch of loads
      int j = 0;
      for (; j + JB4 <= f; j += JB4) {
        double v[JB4][KPL];
#pragma unroll
        for (int t = 0; t < JB4; ++t)
#pragma unroll
          for (int kk = 0; kk < KPL; ++kk) v[t][kk] = kok[kk] ? __ldg(yl + 32 * kk * f + j + t) : 0.0;
#pragma unroll
        for (int t = 0; t < JB4; ++t) {
          const double g = gamma[j + t];
#pragma unroll
          for (int kk = 0; kk < KPL; ++kk) {
            if (t & 1) ub[kk] = fma(v[t][kk], g, ub[kk]);
            else ua[kk] = fma(v[t][kk], g, ua[kk]);
          }
        }
      }
      for (; j < f; ++j) {
        const double g = gamma[j];
#pragma unroll
        for (int kk = 0; kk < KPL; ++kk)
          if (kok[kk]) ua[kk] = fma(__ldg(yl + 32 * kk * f + j), g, ua[kk]);
      }
      for (int c = 0; c < d; ++c) {
#pragma unroll
        for (int kk = 0; kk < KPL; ++kk)
          if (kok[kk]) ((c & 1) ? ub : ua)[kk] = fma(__ldg(zl + 32 * kk * d + c), alpha[(lane + 32 * kk) * d + c],
                                                   ((c & 1) ? ub : ua)[kk]);
      }
    }
    double u[KPL], r[KPL];
    if constexpr (HV) {  // Hessian-vector product: s_k = ua + ub, r_k = -P_k (s_k - sum_l P_l s_l)
      double ps = 0.0;
#pragma unroll
      for (int kk = 0; kk < KPL; ++kk) {
        u[kk] = kok[kk] ? __ldg(A.Pr + gi * A.ldP + lane + 32 * kk) : 0.0;
        ps = fma(u[kk], ua[kk] + ub[kk], ps);
      }
      ps = warp_sum(ps);
#pragma unroll
      for (int kk = 0; kk < KPL; ++kk) {
        const int k = lane + 32 * kk;
        r[kk] = kok[kk] ? -u[kk] * ((ua[kk] + ub[kk]) - ps) : 0.0;
        if (k < KPS) Rs[ii * KPS + k] = r[kk];
      }
    } else {
      double m = -INFINITY, uy_l = 0.0;
  #pragma unroll
      for (int kk = 0; kk < KPL; ++kk) {
        const int k = lane + 32 * kk;
        u[kk] = kok[kk] ? ua[kk] + ub[kk] : -INFINITY;
        if (k == y) uy_l = u[kk];
        m = fmax(m, u[kk]);
      }
      m = warp_max(m);
      double ssum = 0.0;
  #pragma unroll
      for (int kk = 0; kk < KPL; ++kk) {
        const double e = exp_shifted(u[kk] - m);  // (u = -inf where the alternative does not exist: 0)
        ssum += e;
        u[kk] = e;
      }
      ssum = warp_sum(ssum);
      const double uy = __shfl_sync(0xffffffffu, uy_l, y & 31);
      if (lane == 0) neu_add(l_s, l_c, uy - (m + log(ssum)));  // one lane per individual
      const double inv_s = recip_ge1(ssum);
  #pragma unroll
      for (int kk = 0; kk < KPL; ++kk) {
        const int k = lane + 32 * kk;
        const double P = u[kk] * inv_s;
        u[kk] = P;
        r[kk] = kok[kk] ? ((k == y ? 1.0 : 0.0) - P) : 0.0;
        if (k < KPS) Rs[ii * KPS + k] = r[kk];
        if (A.writeP && kok[kk]) A.Pr[gi * A.ldP + k] = P;
      }
    }
    if (A.Rg)  // stream mode: the alpha / gamma gradients come from k_yz_grad
#pragma unroll
      for (int kk = 0; kk < KPL; ++kk)
        if (kok[kk]) A.Rg[gi * K + lane + 32 * kk] = r[kk];
    if (A.Rg && !A.writeP) continue;  // nothing left for this individual
    // ---- pass 2 (L1 hits): ybar_e = sum_k P_k y_ke, gamma and alpha gradients ----
    // 8 components per batch; the cross-lane ybar sums go through red[8][33] (lane 4e'+j adds 8 of
    // the 32 partials, then two shuffles). The first 16 gamma partials stay in registers.
    auto ybar_batch = [&](int e0, double (&yb)[8], double (&gg)[8]) {
      constexpr int TB = KPL >= 4 ? 2 : 4;
#pragma unroll
      for (int t0 = 0; t0 < 8; t0 += TB) {
        double v[TB][KPL];
#pragma unroll
        for (int t = 0; t < TB; ++t)
#pragma unroll
          for (int kk = 0; kk < KPL; ++kk)
            v[t][kk] = (kok[kk] && e0 + t0 + t < f) ? __ldg(yl + 32 * kk * f + e0 + t0 + t) : 0.0;
#pragma unroll
        for (int t = 0; t < TB; ++t) {
          double ybt = 0.0, g = 0.0;
#pragma unroll
          for (int kk = 0; kk < KPL; ++kk) {
            ybt = fma(u[kk], v[t][kk], ybt);
            g = fma(v[t][kk], r[kk], g);
          }
          yb[t0 + t] = ybt;
          gg[t0 + t] = g;
        }
      }
      if (A.writeP) {
#pragma unroll
        for (int t = 0; t < 8; ++t) red[t * 33 + lane] = yb[t];
        __syncwarp();
        const int t = lane >> 2, j = lane & 3;
        double sacc = 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q) sacc += red[t * 33 + j * 8 + q];
        sacc += __shfl_xor_sync(0xffffffffu, sacc, 1);
        sacc += __shfl_xor_sync(0xffffffffu, sacc, 2);
        if (j == 0 && e0 + t < f) A.Pr[gi * A.ldP + K + e0 + t] = sacc;
        __syncwarp();
      }
    };
#pragma unroll
    for (int h = 0; h < gam_regs<KPL>() / 8; ++h) {
      if (8 * h < f) {
        double yb[8], gg[8];
        ybar_batch(8 * h, yb, gg);
        if (!A.Rg)
#pragma unroll
          for (int t = 0; t < 8; ++t) gam[8 * h + t] += gg[t];  // components >= f add exact zeros
      }
    }
    for (int e0 = gam_regs<KPL>(); e0 < f; e0 += 8) {
      double yb[8], gg[8];
      ybar_batch(e0, yb, gg);
      if (A.want_grad && !A.Rg)
#pragma unroll
        for (int t = 0; t < 8; ++t)
          if (e0 + t < f) Wa[NW * KPL * d * 32 + (w * f + e0 + t) * 32 + lane] += gg[t];
    }
    if (A.want_grad && d && !A.Rg) {
      for (int c = 0; c < d; ++c)
#pragma unroll
        for (int kk = 0; kk < KPL; ++kk)
          if (kok[kk]) {
            double* acc = Wa + ((w * KPL + kk) * d + c) * 32 + lane;
            *acc = fma(__ldg(zl + 32 * kk * d + c), r[kk], *acc);
          }
    }
  }
}

// Phase E when all (f + d) x KPL values of an individual fit in 32 registers per lane (c5: 15 x 2):
// one batch of independent loads per individual, issued while the previous individual computes
// (two register sets, ping-pong); both passes (utilities, then ybar and the gradients) read the
// registers. JR = 32 / KPL component slots; slots >= f + d hold zeros.
template <int KPL, bool HV>
__device__ __forceinline__ void phase_e_reg(const EvalArgs& A, const double* Us, double* Rs, const int* ch_t,
                                            double* red, const double* alpha, const double* gamma, double* Wa,
                                            double (&gam)[gam_regs<KPL>()], double& l_s, double& l_c, int64_t i0, int nt,
                                            int KPS, int w, int lane) {
  constexpr int JR = 32 / KPL;
  const int K = A.K, d = A.d, f = A.f, J = f + d;
  const int rows = (A.TI + NW - 1) / NW;  // individuals per warp per tile
  const int ib = w * rows;
  const int n_mine = min(rows, nt - ib);
  for (int ii = ib + max(n_mine, 0); ii < ib + rows; ++ii)  // ragged tail: zero residual rows
    for (int k = lane; k < KPS; k += 32) Rs[ii * KPS + k] = 0.0;
  if (n_mine <= 0) return;
  bool kok[KPL];
#pragma unroll
  for (int kk = 0; kk < KPL; ++kk) kok[kk] = lane + 32 * kk < K;
  auto load = [&](int64_t gi, double (&v)[JR][KPL]) {  // slots t < f: y_ike; f <= t < f + d: z_ik,t-f
    const double* yl = A.Y + (gi * K + lane) * f;
    const double* zl = A.Z + (gi * K + lane) * d;
#pragma unroll
    for (int t = 0; t < JR; ++t)
#pragma unroll
      for (int kk = 0; kk < KPL; ++kk)
        v[t][kk] = !kok[kk] ? 0.0 : (t < f ? __ldg(yl + 32 * kk * f + t) : (t < J ? __ldg(zl + 32 * kk * d + (t - f)) : 0.0));
  };
  auto process = [&](int ii, const double (&v)[JR][KPL]) {
    const int64_t gi = i0 + ii;
    int y = ch_t[ii];
    if (y < 0 || y >= K) {
      if (lane == 0) atomicOr(A.err, 1);
      y = 0;
    }
    double ua[KPL], ub[KPL];
#pragma unroll
    for (int kk = 0; kk < KPL; ++kk) {
      ua[kk] = kok[kk] ? Us[ii * KPS + lane + 32 * kk] : 0.0;
      ub[kk] = 0.0;
    }
#pragma unroll
    for (int t = 0; t < JR; ++t) {
      if (t < f) {
        const double g = gamma[t];
#pragma unroll
        for (int kk = 0; kk < KPL; ++kk) {
          if (t & 1) ub[kk] = fma(v[t][kk], g, ub[kk]);
          else ua[kk] = fma(v[t][kk], g, ua[kk]);
        }
      } else if (t < J) {
#pragma unroll
        for (int kk = 0; kk < KPL; ++kk) {
          const double a = kok[kk] ? alpha[(lane + 32 * kk) * d + (t - f)] : 0.0;
          if (t & 1) ub[kk] = fma(v[t][kk], a, ub[kk]);
          else ua[kk] = fma(v[t][kk], a, ua[kk]);
        }
      }
    }
    double u[KPL], r[KPL];
    if constexpr (HV) {  // Hessian-vector product: s_k = ua + ub, r_k = -P_k (s_k - sum_l P_l s_l)
      double ps = 0.0;
#pragma unroll
      for (int kk = 0; kk < KPL; ++kk) {
        u[kk] = kok[kk] ? __ldg(A.Pr + gi * A.ldP + lane + 32 * kk) : 0.0;
        ps = fma(u[kk], ua[kk] + ub[kk], ps);
      }
      ps = warp_sum(ps);
#pragma unroll
      for (int kk = 0; kk < KPL; ++kk) {
        const int k = lane + 32 * kk;
        r[kk] = kok[kk] ? -u[kk] * ((ua[kk] + ub[kk]) - ps) : 0.0;
        if (k < KPS) Rs[ii * KPS + k] = r[kk];
      }
    } else {
      double m = -INFINITY, uy_l = 0.0;
  #pragma unroll
      for (int kk = 0; kk < KPL; ++kk) {
        const int k = lane + 32 * kk;
        u[kk] = kok[kk] ? ua[kk] + ub[kk] : -INFINITY;
        if (k == y) uy_l = u[kk];
        m = fmax(m, u[kk]);
      }
      m = warp_max(m);
      double ssum = 0.0;
  #pragma unroll
      for (int kk = 0; kk < KPL; ++kk) {
        const double e = exp_shifted(u[kk] - m);  // (u = -inf where the alternative does not exist: 0)
        ssum += e;
        u[kk] = e;
      }
      ssum = warp_sum(ssum);
      const double uy = __shfl_sync(0xffffffffu, uy_l, y & 31);
      if (lane == 0) neu_add(l_s, l_c, uy - (m + log(ssum)));  // one lane per individual
      const double inv_s = recip_ge1(ssum);
  #pragma unroll
      for (int kk = 0; kk < KPL; ++kk) {
        const int k = lane + 32 * kk;
        const double P = u[kk] * inv_s;
        u[kk] = P;
        r[kk] = kok[kk] ? ((k == y ? 1.0 : 0.0) - P) : 0.0;
        if (k < KPS) Rs[ii * KPS + k] = r[kk];
        if (A.writeP && kok[kk]) A.Pr[gi * A.ldP + k] = P;
      }
    }
    // ybar (writeP) in groups of 8 components through red[8][33]; gamma partials (first 16 in
    // registers); alpha partials read-modify-write in this warp's private Wa slots
#pragma unroll
    for (int t0 = 0; t0 < JR; t0 += 8) {
      if (t0 < f) {
        double yb[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          double ybt = 0.0, g = 0.0;
          if (t0 + t < JR) {
#pragma unroll
            for (int kk = 0; kk < KPL; ++kk) {
              ybt = fma(u[kk], v[t0 + t][kk], ybt);
              g = fma(v[t0 + t][kk], r[kk], g);
            }
          }
          yb[t] = ybt;
          if (t0 + t < f) {
            if (t0 + t < 16) gam[(t0 + t) & 15] += g;
            else Wa[NW * KPL * d * 32 + (w * f + t0 + t) * 32 + lane] += g;
          }
        }
        if (A.writeP) {
#pragma unroll
          for (int t = 0; t < 8; ++t) red[t * 33 + lane] = yb[t];
          __syncwarp();
          const int t = lane >> 2, j = lane & 3;
          double sacc = 0.0;
#pragma unroll
          for (int q = 0; q < 8; ++q) sacc += red[t * 33 + j * 8 + q];
          sacc += __shfl_xor_sync(0xffffffffu, sacc, 1);
          sacc += __shfl_xor_sync(0xffffffffu, sacc, 2);
          if (j == 0 && t0 + t < f) A.Pr[gi * A.ldP + K + t0 + t] = sacc;
          __syncwarp();
        }
      }
    }
    if (A.want_grad) {
#pragma unroll
      for (int t = 0; t < JR; ++t)
        if (t >= f && t < J) {
#pragma unroll
          for (int kk = 0; kk < KPL; ++kk)
            if (kok[kk]) {
              double* acc = Wa + ((w * KPL + kk) * d + (t - f)) * 32 + lane;
              *acc = fma(v[t][kk], r[kk], *acc);
            }
        }
    }
  };
  double va[JR][KPL], vb[JR][KPL];
  load(i0 + ib, va);
  for (int jj = 0; jj < n_mine; jj += 2) {
    if (jj + 1 < n_mine) load(i0 + ib + jj + 1, vb);
    process(ib + jj, va);
    if (jj + 1 < n_mine) {
      if (jj + 2 < n_mine) load(i0 + ib + jj + 2, va);
      process(ib + jj + 1, vb);
    }
  }
}

// ---- Phase E with the alternative-varying rows staged in shared memory (YZS path) -----------
// Every warp streams the Y and Z rows of ITS OWN individuals (one contiguous K f and K d block
// each) into a private ring of NS slots with cp.async.bulk (mbarrier complete_tx), NS - 1
// individuals ahead of the one it computes: the reads from HBM are whole 16-byte-multiple blocks
// and lane k then reads alternative k's f (16-byte pairs) and d values from shared memory.
// Conditions (eval_plan): KPL <= 2, f even <= 16, d <= 8, K f and K d even.
// Per-warp state of the YZS pipeline: this warp's rows in tile order form a sequence s = 0, 1, ...
// (YZS_R = YZS_TI / NW rows per tile); position s lives in ring slot s mod NS.
constexpr int NWY = 8;  // warps per CTA of the YZS kernel
constexpr int YZS_TI = 16, YZS_R = YZS_TI / NWY;
struct YzsState {
  unsigned ring_s, bar_s;  // shared addresses of this warp's ring and mbarriers
  int slot, par;           // consume pointer: slot and phase parity of the next row
  int s_cur;               // sequence position of the next row to compute
  int s_issue, slot_i;     // next position to stage and its slot (lane 0 only)
  int lg_cnt;              // deferred logs: lane lg_cnt receives the next individual's (uy - m, s)
  double lg_a, lg_s;
  // lane 0's issue cursor: the next row to stage, its Y and Z rows, and the strides to the next one
  int64_t gi;
  const char *py, *pz;
  unsigned by, bz;  // bytes of one Y / Z row (K f 8, K d 8)
};
// lane 0: stage the next position of this warp's sequence (rows w R .. w R + R - 1 of every tile
// this CTA visits); false if it does not exist. The cursor advances by one row inside a tile and
// by gridDim.x * TI - (R - 1) rows to the next tile (no 64-bit products per row).
__device__ __forceinline__ bool yzs_issue(const EvalArgs& A, YzsState& st) {
  if (st.gi >= A.N) return false;
  const unsigned bar = st.bar_s + 8u * st.slot_i;
  const unsigned dst = st.ring_s + 8u * (unsigned)(st.slot_i * A.SLOT);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the slot's previous generic accesses
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(st.by + st.bz) : "memory");
  if (st.by)
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(st.py), "r"(st.by), "r"(bar)
                 : "memory");
  if (st.bz)
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     dst + st.by),
                 "l"(st.pz), "r"(st.bz), "r"(bar)
                 : "memory");
  const int s = st.s_issue++;
  const int64_t step = (s % YZS_R == YZS_R - 1) ? (int64_t)gridDim.x * YZS_TI - (YZS_R - 1) : 1;
  st.gi += step;
  st.py += step * st.by;
  st.pz += step * st.bz;
  st.slot_i = (st.slot_i + 1 == A.NS) ? 0 : st.slot_i + 1;
  return true;
}

constexpr int YZS_F = 16, YZS_D = 8;  // register capacity of the YZS path (gamma, alpha partials)

// NI consecutive rows of this warp (ii0 ..), computed together so that their dependency chains
// (loads -> utilities -> max / sum shuffles -> exp -> gradient sums) interleave. Lane k holds
// alternatives k + 32 kk. Reads its rows' staged Y [K][f] and Z [K][d] from the ring.
template <int KPL, bool HV, int NI, bool WP>
__device__ __forceinline__ void yzs_rows(const EvalArgs& A, double* Rs, const int* ch_t,
                                         const double* alpha, const double* gamma,
                                         double (&gam)[YZS_F], double (&alp)[KPL][YZS_D], double& l_s, double& l_c,
                                         int64_t i0, int ii0, int KPS, int w, int lane, const double* ring_w,
                                         YzsState& st) {
  const int K = A.K, d = A.d, f = A.f;
  bool kok[KPL];  // lane's alternatives exist (always for kk < KPL - 1: K > 32 (KPL - 1))
#pragma unroll
  for (int kk = 0; kk < KPL; ++kk) kok[kk] = (kk < KPL - 1) || (lane + 32 * kk < K);
  // the row offsets this lane reads: alternative lane + 32 kk, clamped to K - 1 where it does not
  // exist (finite data; those lanes' utilities are -inf and their residuals 0, so the values drop
  // out) -- the shared loads need no predicate
  int ky[KPL], kz[KPL];
#pragma unroll
  for (int kk = 0; kk < KPL; ++kk) {
    const int k = kok[kk] ? lane + 32 * kk : K - 1;
    ky[kk] = k * f;
    kz[kk] = k * d;
  }
  __syncwarp();
  if (lane == 0)  // stage ahead into the slots released by the previous rows
    while (st.s_issue <= st.s_cur + A.NS - 1 && yzs_issue(A, st)) {
    }
  int y[NI];
  int64_t gi[NI];
  double ua[NI][KPL], ub[NI][KPL];
  const double* ys[NI];
  const double* zs[NI];
#pragma unroll
  for (int j = 0; j < NI; ++j) {
    const int ii = ii0 + j;
    gi[j] = i0 + ii;
    y[j] = ch_t[ii];
    if (y[j] < 0 || y[j] >= K) {
      if (lane == 0) atomicOr(A.err, 1);
      y[j] = 0;
    }
#pragma unroll
    for (int kk = 0; kk < KPL; ++kk) {
      ua[j][kk] = kok[kk] ? Rs[ii * KPS + lane + 32 * kk] : 0.0;
      ub[j][kk] = 0.0;
    }
  }
#pragma unroll
  for (int j = 0; j < NI; ++j) {
    mbar_wait(st.bar_s + 8u * st.slot, (unsigned)st.par);
    ys[j] = ring_w + st.slot * A.SLOT;  // [K][f]
    zs[j] = ys[j] + K * f;              // [K][d]
    if (++st.slot == A.NS) {
      st.slot = 0;
      st.par ^= 1;
    }
  }
  st.s_cur += NI;
  // ---- u_k += y_k . gamma + z_k . alpha_k (components in chunks of 4: all loads of a chunk first) ----
#pragma unroll
  for (int e = 0; e < YZS_F; e += 4) {
    if (e + 4 <= f) {
      double2 v[2][NI][KPL];
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int j = 0; j < NI; ++j)
#pragma unroll
          for (int kk = 0; kk < KPL; ++kk)
            v[h][j][kk] = *reinterpret_cast<const double2*>(ys[j] + ky[kk] + e + 2 * h);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const double g0 = gamma[e + 2 * h], g1 = gamma[e + 2 * h + 1];
#pragma unroll
        for (int j = 0; j < NI; ++j)
#pragma unroll
          for (int kk = 0; kk < KPL; ++kk) {
            ua[j][kk] = fma(v[h][j][kk].x, g0, ua[j][kk]);
            ub[j][kk] = fma(v[h][j][kk].y, g1, ub[j][kk]);
          }
      }
    } else if (e < f) {  // the last 2 (f even)
      const double g0 = gamma[e], g1 = gamma[e + 1];
#pragma unroll
      for (int j = 0; j < NI; ++j)
#pragma unroll
        for (int kk = 0; kk < KPL; ++kk) {
          const double2 v = *reinterpret_cast<const double2*>(ys[j] + ky[kk] + e);
          ua[j][kk] = fma(v.x, g0, ua[j][kk]);
          ub[j][kk] = fma(v.y, g1, ub[j][kk]);
        }
    }
  }
#pragma unroll
  for (int c0 = 0; c0 < YZS_D; c0 += 4) {
    if (c0 + 4 <= d) {
      double z[4][NI][KPL], ac[4][KPL];
#pragma unroll
      for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int kk = 0; kk < KPL; ++kk) {
          ac[t][kk] = alpha[kz[kk] + c0 + t];
#pragma unroll
          for (int j = 0; j < NI; ++j) z[t][j][kk] = zs[j][kz[kk] + c0 + t];
        }
#pragma unroll
      for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int j = 0; j < NI; ++j)
#pragma unroll
          for (int kk = 0; kk < KPL; ++kk) {
            if (t & 1) ub[j][kk] = fma(z[t][j][kk], ac[t][kk], ub[j][kk]);
            else ua[j][kk] = fma(z[t][j][kk], ac[t][kk], ua[j][kk]);
          }
    } else {
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        if (c0 + t < d) {
#pragma unroll
          for (int j = 0; j < NI; ++j)
#pragma unroll
            for (int kk = 0; kk < KPL; ++kk) {
              const double z = zs[j][kz[kk] + c0 + t];
              const double ac = alpha[kz[kk] + c0 + t];
              if (t & 1) ub[j][kk] = fma(z, ac, ub[j][kk]);
              else ua[j][kk] = fma(z, ac, ua[j][kk]);
            }
        }
      }
    }
  }
  double u[NI][KPL], r[NI][KPL];
  if constexpr (HV) {  // Hessian-vector product: s_k = ua + ub, r_k = -P_k (s_k - sum_l P_l s_l)
    double ps[NI];
#pragma unroll
    for (int j = 0; j < NI; ++j) {
      ps[j] = 0.0;
#pragma unroll
      for (int kk = 0; kk < KPL; ++kk) {
        u[j][kk] = kok[kk] ? __ldg(A.Pr + gi[j] * A.ldP + lane + 32 * kk) : 0.0;
        ps[j] = fma(u[j][kk], ua[j][kk] + ub[j][kk], ps[j]);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int j = 0; j < NI; ++j) ps[j] += __shfl_xor_sync(0xffffffffu, ps[j], o);
#pragma unroll
    for (int j = 0; j < NI; ++j)
#pragma unroll
      for (int kk = 0; kk < KPL; ++kk) {
        const int k = lane + 32 * kk;
        r[j][kk] = kok[kk] ? -u[j][kk] * ((ua[j][kk] + ub[j][kk]) - ps[j]) : 0.0;
        if (k < KPS) Rs[(ii0 + j) * KPS + k] = r[j][kk];
      }
  } else {
    // shift by the (fp32-rounded) maximum: any shift is exact for the softmax; this one only has
    // to keep e^{u - m} <= ~1 (R12), so the cross-lane max runs on 32-bit shuffles
    float mf[NI];
    double uy_l[NI], ssum[NI];
#pragma unroll
    for (int j = 0; j < NI; ++j) {
      mf[j] = -INFINITY;
      uy_l[j] = 0.0;
#pragma unroll
      for (int kk = 0; kk < KPL; ++kk) {
        const int k = lane + 32 * kk;
        u[j][kk] = kok[kk] ? ua[j][kk] + ub[j][kk] : -INFINITY;
        if (k == y[j]) uy_l[j] = u[j][kk];
        mf[j] = fmaxf(mf[j], (float)u[j][kk]);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int j = 0; j < NI; ++j) mf[j] = fmaxf(mf[j], __shfl_xor_sync(0xffffffffu, mf[j], o));
#pragma unroll
    for (int j = 0; j < NI; ++j) {
      const double m = (double)mf[j];
      ssum[j] = 0.0;
#pragma unroll
      for (int kk = 0; kk < KPL; ++kk) {
        const double e = exp_shifted(u[j][kk] - m);  // (u = -inf where the alternative does not exist: 0)
        ssum[j] += e;
        u[j][kk] = e;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int j = 0; j < NI; ++j) ssum[j] += __shfl_xor_sync(0xffffffffu, ssum[j], o);
#pragma unroll
    for (int j = 0; j < NI; ++j) {
      const double uy = __shfl_sync(0xffffffffu, uy_l[j], y[j] & 31);
      // l_i = uy - m - log s: lane lg_cnt keeps (uy - m, s); every 32 individuals each lane takes one log
      if (lane == st.lg_cnt) {
        st.lg_a = uy - (double)mf[j];
        st.lg_s = ssum[j];
      }
      if (++st.lg_cnt == 32) {
        neu_add(l_s, l_c, st.lg_a - log(st.lg_s));
        st.lg_cnt = 0;
      }
      const double inv_s = recip_ge1(ssum[j]);
#pragma unroll
      for (int kk = 0; kk < KPL; ++kk) {
        const int k = lane + 32 * kk;
        const double P = u[j][kk] * inv_s;
        u[j][kk] = P;
        r[j][kk] = kok[kk] ? ((k == y[j] ? 1.0 : 0.0) - P) : 0.0;
        if (k < KPS) Rs[(ii0 + j) * KPS + k] = r[j][kk];
        if (WP && kok[kk]) A.Pr[gi[j] * A.ldP + k] = P;
      }
    }
  }
  // ---- ybar_e = sum_k P_k y_ke (writeP), gamma partials sum_k y_ke r_k, alpha partials z_kc r_k ----
  // in halves of 8 components: gamma partials, then (writeP) the cross-lane ybar sums by a
  // reduce-scatter over shuffles (warp_sum8)
#pragma unroll
  for (int e8 = 0; e8 < YZS_F; e8 += 8) {
    if (e8 < f) {
      double yb[NI][8];
#pragma unroll
      for (int e = e8; e < e8 + 8; e += 4) {
#pragma unroll
        for (int j = 0; j < NI; ++j) yb[j][e - e8] = yb[j][e - e8 + 1] = yb[j][e - e8 + 2] = yb[j][e - e8 + 3] = 0.0;
        if (e < f) {
          const int nh = (e + 4 <= f) ? 2 : 1;  // pairs in this chunk (f even)
          double2 v[2][NI][KPL];
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int j = 0; j < NI; ++j)
#pragma unroll
              for (int kk = 0; kk < KPL; ++kk)
                v[h][j][kk] = h < nh ? *reinterpret_cast<const double2*>(ys[j] + ky[kk] + e + 2 * h)
                                      : make_double2(0.0, 0.0);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            double g0 = 0.0, g1 = 0.0;
#pragma unroll
            for (int j = 0; j < NI; ++j)
#pragma unroll
              for (int kk = 0; kk < KPL; ++kk) {
                if constexpr (WP) {  // ybar only for the Hessian pass
                  yb[j][e - e8 + 2 * h] = fma(u[j][kk], v[h][j][kk].x, yb[j][e - e8 + 2 * h]);
                  yb[j][e - e8 + 2 * h + 1] = fma(u[j][kk], v[h][j][kk].y, yb[j][e - e8 + 2 * h + 1]);
                }
                g0 = fma(v[h][j][kk].x, r[j][kk], g0);
                g1 = fma(v[h][j][kk].y, r[j][kk], g1);
              }
            gam[e + 2 * h] += g0;  // components >= f collect exact zeros (never output)
            gam[e + 2 * h + 1] += g1;
          }
        }
      }
      if constexpr (!HV && WP) {
#pragma unroll
        for (int j = 0; j < NI; ++j) {
          const int t = (lane >> 2) & 7;  // the component warp_sum8 leaves in this lane
          const double sacc = warp_sum8(yb[j], lane);
          if ((lane & 3) == 0 && e8 + t < f) A.Pr[gi[j] * A.ldP + K + e8 + t] = sacc;
        }
      }
    }
  }
#pragma unroll
  for (int c0 = 0; c0 < YZS_D; c0 += 4) {
    if (c0 + 4 <= d) {  // a whole chunk of 4 components: all loads first
      double z[4][NI][KPL];
#pragma unroll
      for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int j = 0; j < NI; ++j)
#pragma unroll
          for (int kk = 0; kk < KPL; ++kk) z[t][j][kk] = zs[j][kz[kk] + c0 + t];
#pragma unroll
      for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int kk = 0; kk < KPL; ++kk) {
          double a = alp[kk][c0 + t];
#pragma unroll
          for (int j = 0; j < NI; ++j) a = fma(z[t][j][kk], r[j][kk], a);
          alp[kk][c0 + t] = a;
        }
    } else {
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        if (c0 + t < d) {
#pragma unroll
          for (int kk = 0; kk < KPL; ++kk) {
            double a = alp[kk][c0 + t];
#pragma unroll
            for (int j = 0; j < NI; ++j) a = fma(zs[j][kz[kk] + c0 + t], r[j][kk], a);
            alp[kk][c0 + t] = a;
          }
        }
      }
    }
  }
}

// Phase E of one tile for warp w (rows w YZS_R .. + YZS_R - 1): pairs of rows, a single ragged one
template <int KPL, bool HV>
__device__ __forceinline__ void phase_e_smem(const EvalArgs& A, double* Rs, const int* ch_t,
                                             const double* alpha, const double* gamma,
                                             double (&gam)[YZS_F], double (&alp)[KPL][YZS_D], double& l_s, double& l_c,
                                             int64_t i0, int nt, int KPS, int w, int lane, const double* ring_w,
                                             YzsState& st) {
  const int ib = w * YZS_R;
  const int n_mine = min(YZS_R, nt - ib);
  for (int ii = ib + max(n_mine, 0); ii < ib + YZS_R; ++ii)  // ragged tail: zero residual rows
    for (int k = lane; k < KPS; k += 32) Rs[ii * KPS + k] = 0.0;
  int jj = 0;
  if constexpr (YZS_R >= 2)
    for (; jj + 2 <= n_mine; jj += 2) {
      if (!HV && A.writeP) yzs_rows<KPL, HV, 2, true>(A, Rs, ch_t, alpha, gamma, gam, alp, l_s, l_c, i0, ib + jj, KPS, w, lane, ring_w, st);
      else yzs_rows<KPL, HV, 2, false>(A, Rs, ch_t, alpha, gamma, gam, alp, l_s, l_c, i0, ib + jj, KPS, w, lane, ring_w, st);
    }
  if (jj < n_mine) {
    if (!HV && A.writeP) yzs_rows<KPL, HV, 1, true>(A, Rs, ch_t, alpha, gamma, gam, alp, l_s, l_c, i0, ib + jj, KPS, w, lane, ring_w, st);
    else yzs_rows<KPL, HV, 1, false>(A, Rs, ch_t, alpha, gamma, gam, alp, l_s, l_c, i0, ib + jj, KPS, w, lane, ring_w, st);
  }
}

template <int KPL, int CM_MAX, bool HV, bool YZS>
__global__ void __launch_bounds__((YZS ? NWY : NW) * 32, 1) k_eval_kernel(const EvalArgs A) {
  constexpr int NWK = YZS ? NWY : NW;           // warps per CTA
  extern __shared__ __align__(16) double sm[];
  constexpr int KP = 32 * KPL, KPS = KP + 4;   // alternatives padded; smem row stride = 4 (mod 16)
  constexpr int NBN = KP / 8;                   // 8-wide alternative blocks
  const int TI = YZS ? YZS_TI : A.TI;
  const int K = A.K, q = A.q, d = A.d, f = A.f, p = A.p;
  const int QP = A.QP, XS = A.XS;              // q padded to 4; X tile row stride (= 4 mod 16)
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int r4 = lane & 3, c8 = lane >> 2;
  double* Bs = sm;                              // [QP][KPS]  Bs[a][k] = beta_k[a]
  double* Xs = Bs + QP * KPS;                   // [2][TI][XS] x~ tiles (col 0 = 1)
  double* Rs = Xs + 2 * TI * XS;                // [TI][KPS]  residuals
  // [TI][KPS] utilities from phase B (YZS: in place in Rs, each lane overwrites its own u by r)
  double* Ps = YZS ? Rs : Rs + TI * KPS;
  constexpr bool SPLITB = YZS || KPL >= 8;  // phase B split over row blocks x alternative groups, u stashed
  // [NWK][KPL][d][32] alpha-gradient, lane-private, then [NWK][f][32] gamma-gradient (e >= 8);
  // absent in stream mode (A.Rg: k_yz_grad forms those gradients) and in the YZS path (registers)
  double* Wa_s = Rs + (((d + f) || KPL >= 8) && !YZS ? 2 * TI * KPS : TI * KPS);
  double* Wa = Wa_s;
  double* Cf = Wa_s + (YZS || A.Rg ? 0 : NWK * KPL * d * 32 + NWK * f * 32);  // [K*d + f]  alpha, gamma
  int* chs = reinterpret_cast<int*>(Cf + K * d + f + 1);  // [2][TI] choices
  double* Red = Cf + K * d + f + 1 + TI;                  // [NWK][8][33] ybar reductions
  // YZS: per-warp mbarriers [NWK][NS] and rings [NWK][NS][SLOT] (16-byte aligned); the ybar scratch
  // is the row's own slot when it holds 8 x 33 doubles
  const int red_end = (int)(Red - sm) + ((d + f) && !YZS ? NWK * 8 * 33 : 0);
  uint64_t* Bar = reinterpret_cast<uint64_t*>(sm + ((red_end + 1) & ~1));
  double* Ring = sm + ((red_end + 1) & ~1) + NWK * A.NS;

  for (int idx = tid; idx < QP * KPS; idx += blockDim.x) {
    const int a = idx / KPS, k = idx - a * KPS;
    Bs[idx] = (a < q && k >= 1 && k < K) ? A.coef[(k - 1) * q + a] : 0.0;
  }
  for (int idx = tid; idx < 2 * TI * XS; idx += blockDim.x) Xs[idx] = ((idx % XS) == 0) ? 1.0 : 0.0;
  if (!YZS)
    for (int idx = tid; idx < (A.Rg ? 0 : NWK * KPL * d * 32 + NWK * f * 32); idx += blockDim.x) Wa[idx] = 0.0;
  for (int idx = tid; idx < K * d + f; idx += blockDim.x) Cf[idx] = A.coef[A.off_alpha + idx];
  const double* alpha = Cf;
  const double* gamma = Cf + K * d;
  // YZS: this lane's alpha_k coefficients and alpha / gamma gradient partials live in registers
  double alp[YZS ? KPL : 1][YZS_D], gamz[YZS_F];
  YzsState yst;
  if constexpr (YZS) {
    yst.ring_s = static_cast<unsigned>(__cvta_generic_to_shared(Ring + (size_t)w * A.NS * A.SLOT));
    yst.bar_s = static_cast<unsigned>(__cvta_generic_to_shared(Bar + w * A.NS));
    yst.slot = yst.par = yst.s_cur = yst.s_issue = yst.slot_i = yst.lg_cnt = 0;
    yst.lg_a = 0.0;
    yst.lg_s = 1.0;
    yst.by = (unsigned)A.K * A.f * 8u;
    yst.bz = (unsigned)A.K * A.d * 8u;
    yst.gi = (int64_t)blockIdx.x * YZS_TI + w * YZS_R;
    yst.py = reinterpret_cast<const char*>(A.Y) + yst.gi * yst.by;
    yst.pz = reinterpret_cast<const char*>(A.Z) + yst.gi * yst.bz;
#pragma unroll
    for (int kk = 0; kk < KPL; ++kk)
#pragma unroll
      for (int c = 0; c < YZS_D; ++c) alp[kk][c] = 0.0;
#pragma unroll
    for (int e = 0; e < YZS_F; ++e) gamz[e] = 0.0;
    if (lane == 0) {
      for (int j = 0; j < A.NS; ++j) mbar_init(Bar + w * A.NS + j, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    if (lane == 0)  // only lane 0 tracks the issue pointer
      while (yst.s_issue < A.NS && yzs_issue(A, yst)) {
      }
  }

  // phase-C warp grid over (m-blocks of a, n-blocks of k)
  const int MB = QP / 8 + ((QP & 7) ? 1 : 0);
  constexpr int WN = NBN < 8 ? NBN : 8;
  constexpr int WM = NWK / WN;
  const int cwm = w / WN, cwn = w % WN;
  constexpr int CN = NBN / WN;                 // n-blocks per warp (CM_MAX m-blocks per warp)
  double G[CM_MAX][CN][2];
#pragma unroll
  for (int i = 0; i < CM_MAX; ++i)
#pragma unroll
    for (int j = 0; j < CN; ++j) G[i][j][0] = G[i][j][1] = 0.0;
  double gam[gam_regs<KPL>()];  // gamma-gradient lane partials (the first 8 or 16; the rest in Wa)
#pragma unroll
  for (int e = 0; e < gam_regs<KPL>(); ++e) gam[e] = 0.0;


  double l_s = 0.0, l_c = 0.0;  // Neumaier loglik of this lane's rows (lanes with r4 == 0)
  const int64_t ntiles = (A.N + TI - 1) / TI;
  const unsigned xs_s = static_cast<unsigned>(__cvta_generic_to_shared(Xs));
  const int x_i0 = p ? tid / p : 0, x_a0 = p ? tid - x_i0 * p : 0;                    // tid = x_i0 p + x_a0
  const int x_di = p ? (int)blockDim.x / p : 0, x_da = p ? (int)blockDim.x - x_di * p : 0;  // blockDim likewise
  auto prefetch = [&](int64_t tile, int buf) {
    const int64_t i0 = tile * TI;
    const int nt = (int)(A.N - i0 < TI ? A.N - i0 : TI);
    const unsigned dst = xs_s + 8u * (unsigned)(buf * TI * XS);
    const double* src = A.X + i0 * p;
    int i = x_i0, a = x_a0;  // element e = tid + j blockDim = i p + a, advanced without divisions
    for (int e = tid; e < nt * p; e += blockDim.x) {
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst + 8u * (unsigned)(i * XS + a + 1)),
                   "l"(src + e)
                   : "memory");
      i += x_di;
      a += x_da;
      if (a >= p) {
        a -= p;
        ++i;
      }
    }
    for (int i = tid; i < nt; i += blockDim.x)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                       static_cast<unsigned>(__cvta_generic_to_shared(chs + buf * TI + i))),
                   "l"(A.choice + i0 + i)
                   : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
    if (!YZS && tid == 0) {  // warm L2 with the tile's alternative-varying rows (contiguous blocks)
      const double* blk[2] = {f ? A.Y + i0 * K * f : nullptr, d ? A.Z + i0 * K * d : nullptr};
      const int64_t len[2] = {(int64_t)nt * K * f * 8, (int64_t)nt * K * d * 8};
      for (int b = 0; b < 2; ++b) {
        if (!blk[b]) continue;
        const char* b0 = reinterpret_cast<const char*>(blk[b]);
        for (int64_t o = 0; o < len[b]; o += (1 << 20)) {  // <= 1 MB pieces, 16-byte multiples
          const unsigned bytes = (unsigned)((len[b] - o < (1 << 20) ? len[b] - o : (1 << 20)) & ~int64_t(15));
          if (bytes) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(b0 + o), "r"(bytes) : "memory");
        }
      }
    }
  };

  int buf = 0;
  __syncthreads();  // the shared-memory initialisation (Xs ones / zeros, Bs, Cf) is complete before any
                    // cp.async of the first tile can land in Xs
  if ((int64_t)blockIdx.x < ntiles) prefetch(blockIdx.x, 0);
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, buf ^= 1) {
    const int64_t i0 = tile * TI;
    const int nt = (int)(A.N - i0 < TI ? A.N - i0 : TI);
    __syncthreads();  // everyone done with the previous tile (buffers, Rs, Ps)
    if (tile + gridDim.x < ntiles) prefetch(tile + gridDim.x, buf ^ 1);
    else asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncthreads();
    const double* X_t = Xs + buf * TI * XS;
    const int* ch_t = chs + buf * TI;

    // ---------------- phase B: u = X~ B on DMMA, then softmax / loglik / residuals ----------------
    // YZS (16-row tiles): the warps split 2 row blocks x NG groups of alternative blocks (groups
    // beyond NBN idle)
    constexpr int RB = YZS_TI / 8;  // SPLITB (16-row tiles): 8-row blocks of the tile
    constexpr int NG = NWK / RB;
    constexpr int NBW = SPLITB ? (NBN >= NG ? NBN / NG : 1) : NBN;  // alternative blocks per warp
    const int il = SPLITB ? 8 * (w % RB) + c8 : (8 * w + c8) % TI;  // this lane's individual (C-fragment row)
    const int nb0 = SPLITB ? (w / RB) * NBW : 0;
    const bool in_b = SPLITB ? nb0 < NBN : 8 * w < TI;  // warps without a block skip phase B
    double u[NBW][2];
#pragma unroll
    for (int nb = 0; nb < NBW; ++nb) u[nb][0] = u[nb][1] = 0.0;
    for (int a0 = 0; a0 < (in_b ? QP : 0); a0 += 4) {
      const double av = X_t[il * XS + a0 + r4];
#pragma unroll
      for (int nb = 0; nb < NBW; ++nb) {
        const double bv = Bs[(a0 + r4) * KPS + (nb0 + nb) * 8 + c8];
        asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
            : "+d"(u[nb][0]), "+d"(u[nb][1])
            : "d"(av), "d"(bv));
      }
    }
    const bool valid = in_b && il < nt;
    const int64_t i = i0 + il;
    if (SPLITB || (d + f)) {
      // ---- alternative-varying data present (or K > 128): stash u, then phase E (lanes over
      // alternatives) ----
      if (in_b) {
#pragma unroll
        for (int nb = 0; nb < NBW; ++nb)
          *reinterpret_cast<double2*>(Ps + il * KPS + (nb0 + nb) * 8 + 2 * r4) = make_double2(u[nb][0], u[nb][1]);
      }
      __syncthreads();
      bool done = false;
      if constexpr (YZS) {
        phase_e_smem<KPL, HV>(A, Rs, ch_t, alpha, gamma, gamz, alp, l_s, l_c, i0, nt, KPS, w,
                              lane, Ring + (size_t)w * A.NS * A.SLOT, yst);
        done = true;
      } else if constexpr (KPL <= 2) {  // register path (the larger KPL would spill)
        if ((f + d) * KPL <= 32 && !A.Rg) {
          phase_e_reg<KPL, HV>(A, Ps, Rs, ch_t, Red + w * (8 * 33), alpha, gamma, Wa, gam, l_s, l_c, i0, nt, KPS, w, lane);
          done = true;
        }
      }
      if constexpr (!YZS)
        if (!done) phase_e<KPL, HV>(A, Ps, Rs, ch_t, Red + w * (8 * 33), alpha, gamma, Wa, gam, l_s, l_c, i0, nt, KPS, w, lane);
    } else if constexpr (!SPLITB) {
    if constexpr (HV) {
      // Hessian-vector product: u holds s_ik = (J_i v)_k; with P_i from the last evaluation
      // (Pr), r_ik = -P_ik (s_ik - sum_l P_il s_il), so that the gradient contractions below
      // accumulate H v (P:462-476 applied to v)
      double pk[NBN][2], ps = 0.0;
#pragma unroll
      for (int nb = 0; nb < NBN; ++nb)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int k = nb * 8 + 2 * r4 + h;
          pk[nb][h] = (valid && k < K) ? __ldg(A.Pr + i * A.ldP + k) : 0.0;
          ps = fma(pk[nb][h], u[nb][h], ps);
        }
      ps += __shfl_xor_sync(0xffffffffu, ps, 1);
      ps += __shfl_xor_sync(0xffffffffu, ps, 2);
      double* Rrow = Rs + il * KPS;
#pragma unroll
      for (int nb = 0; nb < NBN; ++nb) {
        const int k = nb * 8 + 2 * r4;
        double2 R2;
        R2.x = -pk[nb][0] * (u[nb][0] - ps);
        R2.y = -pk[nb][1] * (u[nb][1] - ps);
        if (in_b) *reinterpret_cast<double2*>(Rrow + k) = R2;
      }
    } else {
    int y = valid ? ch_t[il] : -1;  // -1 (a row beyond N): no alternative matches, residuals 0
    if (valid && (y < 0 || y >= K)) {
      atomicOr(A.err, 1);
      y = 0;
    }
    // shift by the (fp32-rounded) maximum: any shift is exact for the softmax, it only has to keep
    // e^{u - m} <= ~1 (R12); the fp32 maximum costs two instructions per alternative off the FP64
    // pipe, which the DMMAs of the other warps need
    float mf = -INFINITY;
#pragma unroll
    for (int nb = 0; nb < NBN; ++nb)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int k = nb * 8 + 2 * r4 + h;
        if (k >= K) u[nb][h] = -INFINITY;
        mf = fmaxf(mf, (float)u[nb][h]);
      }
    mf = fmaxf(mf, __shfl_xor_sync(0xffffffffu, mf, 1));
    mf = fmaxf(mf, __shfl_xor_sync(0xffffffffu, mf, 2));
    const double m = (double)mf;
    double ssum = 0.0, uy = 0.0;
#pragma unroll
    for (int nb = 0; nb < NBN; ++nb)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int k = nb * 8 + 2 * r4 + h;
        if (k == y) uy = u[nb][h];
        const double e = exp_shifted(u[nb][h] - m);  // (u = -inf for k >= K: 0)
        u[nb][h] = e;
        ssum += e;
      }
    ssum += __shfl_xor_sync(0xffffffffu, ssum, 1);
    ssum += __shfl_xor_sync(0xffffffffu, ssum, 2);
    uy += __shfl_xor_sync(0xffffffffu, uy, 1);
    uy += __shfl_xor_sync(0xffffffffu, uy, 2);
    if (valid && r4 == 0) neu_add(l_s, l_c, uy - (m + log(ssum)));
    // a row beyond N: P = 0 and (y = -1) r = 0; an alternative >= K: e = 0, so P = r = 0
    const double inv_s = valid ? recip_ge1(ssum) : 0.0;
    double* Rrow = Rs + il * KPS;
#pragma unroll
    for (int nb = 0; nb < NBN; ++nb) {
      const int k = nb * 8 + 2 * r4;
      double2 P2, R2;
      P2.x = __dmul_rn(u[nb][0], inv_s);  // (rounded products: the same r with and without the P rows)
      P2.y = __dmul_rn(u[nb][1], inv_s);
      R2.x = (k == y ? 1.0 : 0.0) - P2.x;
      R2.y = (k + 1 == y ? 1.0 : 0.0) - P2.y;
      if (in_b) *reinterpret_cast<double2*>(Rrow + k) = R2;
      if (A.writeP && valid) {
        double* pr = A.Pr + i * A.ldP + k;
        if (k + 1 < K) *reinterpret_cast<double2*>(pr) = P2;
        else if (k < K) pr[0] = P2.x;
      }
    }
    }  // !HV
    }
    __syncthreads();  // Rs complete

    // ---------------- phase C: beta gradient G[a][k] += sum_i x~_ia r_ik on DMMA ----------------
    if (A.want_grad) {
      for (int ks = 0; ks < TI / 4; ++ks) {
        double bf[CN];
#pragma unroll
        for (int j = 0; j < CN; ++j) bf[j] = Rs[(4 * ks + r4) * KPS + (cwn + WN * j) * 8 + c8];
#pragma unroll
        for (int mi = 0; mi < CM_MAX; ++mi) {
          const int mb = cwm + WM * mi;
          if (mb < MB) {
            const double af = X_t[(4 * ks + r4) * XS + mb * 8 + c8];
#pragma unroll
            for (int j = 0; j < CN; ++j)
              asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                  : "+d"(G[mi][j][0]), "+d"(G[mi][j][1])
                  : "d"(af), "d"(bf[j]));
          }
        }
      }
    }

  }

  // ---------------- CTA partials (fixed order) ----------------
  if constexpr (YZS)
    if (lane < yst.lg_cnt) neu_add(l_s, l_c, yst.lg_a - log(yst.lg_s));  // the deferred logs left over
  __syncthreads();
  double* out = A.part + (size_t)blockIdx.x * A.n_part;
  // finalisation scratch: the dead Bs .. Ps regions when they hold [NWK 32][8] doubles (they do
  // whenever the tile was shrunk for a large p), else Rs and what follows it; YZS: the drained rings
  double* fin = (Wa_s - sm >= NWK * 32 * 8) ? sm : Rs;
  double* scratch = YZS ? Ring : fin;
  // loglik: lanes with r4 == 0 hold rows; combine in (warp, lane) order
  scratch[2 * tid] = l_s;
  scratch[2 * tid + 1] = l_c;
  __syncthreads();
  if (tid == 0) {
    double s = 0.0, c = 0.0;
    for (int t = 0; t < NWK * 32; t += (YZS ? 1 : 4)) { neu_add(s, c, scratch[2 * t]); neu_add(s, c, scratch[2 * t + 1]); }
    out[0] = s;
    out[1] = c;
  }
  if (!A.want_grad) return;
  // beta gradient straight from the G fragments: G[a][k] -> out[2 + (k-1) q + a]
#pragma unroll
  for (int mi = 0; mi < CM_MAX; ++mi) {
    const int mb = cwm + WM * mi;
    if (mb < MB) {
      const int a = mb * 8 + c8;
#pragma unroll
      for (int j = 0; j < CN; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int k = (cwn + WN * j) * 8 + 2 * r4 + h;
          if (a < q && k >= 1 && k < K) out[2 + (k - 1) * q + a] = G[mi][j][h];
        }
    }
  }
  if constexpr (YZS) {
    // alpha / gamma register partials -> the (drained) rings as [NWK][KPL][d][32] + [NWK][f][32],
    // then fixed-order sums over warps and lanes
    __syncthreads();  // the loglik partials in the rings have been summed
    double* sa = Ring;
    double* sg = Ring + NWK * KPL * d * 32;
#pragma unroll
    for (int kk = 0; kk < KPL; ++kk)
#pragma unroll
      for (int c = 0; c < YZS_D; ++c)
        if (c < d) sa[((w * KPL + kk) * d + c) * 32 + lane] = alp[kk][c];
#pragma unroll
    for (int e = 0; e < YZS_F; ++e)
      if (e < f) sg[(w * f + e) * 32 + lane] = gamz[e];
    __syncthreads();
    for (int idx = tid; idx < K * d; idx += blockDim.x) {
      const int k = idx / d, c = idx - k * d, kk = k >> 5, ln = k & 31;
      double v = 0.0;
      for (int ww = 0; ww < NWK; ++ww) v += sa[((ww * KPL + kk) * d + c) * 32 + ln];
      out[2 + A.off_alpha + idx] = v;
    }
    for (int e = tid; e < f; e += blockDim.x) {
      double v = 0.0;
      for (int ww = 0; ww < NWK; ++ww)
        for (int ln = 0; ln < 32; ++ln) v += sg[(ww * f + e) * 32 + ln];
      out[2 + A.off_gamma + e] = v;
    }
    return;
  }
  if (A.Rg) return;  // stream mode: k_yz_grad writes this CTA's alpha / gamma slots
  // register partials of gamma components 8..15 into Wa (each (warp, lane) slot is private)
#pragma unroll
  for (int e = 8; e < gam_regs<KPL>(); ++e)
    if (e < f) Wa[NWK * KPL * d * 32 + (w * f + e) * 32 + lane] += gam[e];
  __syncthreads();
  // gamma partials: registers (e < 8) -> smem, then fixed-order sums
  double* gsc = fin;  // [NWK*32][8]
  for (int e = 0; e < 8; ++e) gsc[tid * 8 + e] = gam[e];
  __syncthreads();
  for (int idx = tid; idx < K * d; idx += blockDim.x) {
    const int k = idx / d, c = idx - k * d, kk = k >> 5, ln = k & 31;
    double v = 0.0;
    for (int ww = 0; ww < NWK; ++ww) v += Wa[((ww * KPL + kk) * d + c) * 32 + ln];
    out[2 + A.off_alpha + idx] = v;
  }
  for (int e = tid; e < f; e += blockDim.x) {
    double v = 0.0;
    if (e < 8) {
      for (int t = 0; t < NWK * 32; ++t) v += gsc[t * 8 + e];
    } else {
      for (int ww = 0; ww < NWK; ++ww)
        for (int ln = 0; ln < 32; ++ln) v += Wa[NWK * KPL * d * 32 + (ww * f + e) * 32 + ln];
    }
    out[2 + A.off_gamma + e] = v;
  }
}

// Stream mode (many alternative-varying variables): the alpha / gamma gradient partials of CTA b
// over the same contiguous share of the individuals, from the residual rows r_i (Rg) written by
// pass 1:  g[alpha_k,c] = sum_i z_ikc r_ik,  g[gamma_e] = sum_i sum_k y_ike r_ik.
// Threads own elements t of the K d (K f) row, 256 x YG_CH per chunk, in registers; Z and Y rows
// are read once, coalesced; the gamma sums over k go through shared memory in a fixed order.
constexpr int YG_CH = 8;
__global__ void __launch_bounds__(256) k_yz_grad(int64_t N, int K, int d, int f, const double* __restrict__ Y,
                                                const double* __restrict__ Z, const double* __restrict__ Rg,
                                                double* part, int n_part, int off_alpha, int off_gamma) {
  __shared__ double sred[256 * YG_CH];
  __shared__ double gsum[64];
  const int tid = threadIdx.x;
  const int64_t G = gridDim.x, b = blockIdx.x;
  const int64_t i_lo = b * N / G, i_hi = (b + 1) * N / G;
  double* out = part + b * (int64_t)n_part;
  // blockIdx.y: alpha chunk y (of 256 YG_CH elements); the y == 0 CTAs also do the gamma pass
  for (int pass = 0; pass < 2; ++pass) {
    const int W = pass == 0 ? d : f;  // values per alternative
    if (W == 0 || (pass == 1 && blockIdx.y != 0)) continue;
    const double* D = pass == 0 ? Z : Y;
    const int L = K * W;
    if (pass == 1) {
      if (tid < f) gsum[tid] = 0.0;
      __syncthreads();
    }
    const int t_begin = pass == 0 ? (int)blockIdx.y * 256 * YG_CH : 0;
    const int t_end = pass == 0 ? min(L, t_begin + 256 * YG_CH) : L;
    for (int t0 = t_begin; t0 < t_end; t0 += 256 * YG_CH) {
      double acc[YG_CH];
      int kt[YG_CH];
#pragma unroll
      for (int j = 0; j < YG_CH; ++j) {
        const int t = t0 + tid + 256 * j;
        kt[j] = t < L ? t / W : -1;
        acc[j] = 0.0;
      }
#pragma unroll 4
      for (int64_t i = i_lo; i < i_hi; ++i) {
        const double* row = D + i * L + t0 + tid;
        const double* rr = Rg + i * K;
#pragma unroll
        for (int j = 0; j < YG_CH; ++j)
          if (kt[j] >= 0) acc[j] = fma(__ldg(row + 256 * j), __ldg(rr + kt[j]), acc[j]);
      }
      if (pass == 0) {
#pragma unroll
        for (int j = 0; j < YG_CH; ++j)
          if (kt[j] >= 0) out[2 + off_alpha + t0 + tid + 256 * j] = acc[j];
      } else {
#pragma unroll
        for (int j = 0; j < YG_CH; ++j) sred[tid + 256 * j] = kt[j] >= 0 ? acc[j] : 0.0;
        __syncthreads();
        if (tid < f) {  // elements t = t0 + idx with t mod f == tid, in increasing idx order
          const int n = min(256 * YG_CH, L - t0);
          double v = gsum[tid];
          for (int idx = ((tid - t0) % f + f) % f; idx < n; idx += f) v += sred[idx];
          gsum[tid] = v;
        }
        __syncthreads();
      }
    }
    if (pass == 1 && tid < f) out[2 + off_gamma + tid] = gsum[tid];
  }
}

__global__ void __launch_bounds__(256) k_eval_finalize(const double* __restrict__ part, int n_part,
                                                      int nblk, int n_p, int want_grad,
                                                      double* grad, double* loglik_out,
                                                      double* scal, const int* err,
                                                      unsigned* counter, int* status_out) {
  __shared__ double red[256];
  __shared__ bool last;
  const int tid = threadIdx.x;
  const int r = blockIdx.x * 256 + tid;
  if (want_grad && r < n_p) {
    // fixed block order; the loads of 8 blocks are issued together (the partials sit in L2)
    double s = 0.0, c = 0.0;
    int b = 0;
    for (; b + 16 <= nblk; b += 16) {
      double v[16];
#pragma unroll
      for (int t = 0; t < 16; ++t) v[t] = __ldcg(part + (size_t)(b + t) * n_part + 2 + r);
#pragma unroll
      for (int t = 0; t < 16; ++t) neu_add(s, c, v[t]);
    }
    for (; b < nblk; ++b) neu_add(s, c, __ldcg(part + (size_t)b * n_part + 2 + r));
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
  double s = 0.0, c = 0.0;
  if (tid < 32) {
    // loglik: lane l sums blocks l, l + 32, ... (Neumaier), then lane 0 folds the 32 lane sums in
    // lane order (fixed order: deterministic)
    for (int b = tid; b < nblk; b += 32) {
      neu_add(s, c, __ldcg(part + (size_t)b * n_part));
      neu_add(s, c, __ldcg(part + (size_t)b * n_part + 1));
    }
    double S = 0.0, C = 0.0;
    for (int l = 0; l < 32; ++l) {
      const double sl = __shfl_sync(0xffffffffu, s, l), cl = __shfl_sync(0xffffffffu, c, l);
      neu_add(S, C, sl);
      neu_add(S, C, cl);
    }
    s = S;
    c = C;
  }
  if (tid == 0) {
    const double l = s + c;
    scal[0] = l;
    scal[1] = red[0];
    scal[2] = (double)(*err);
    if (loglik_out) *loglik_out = l;
    if (status_out) *status_out = *err ? 1 /* MNL_ERR_ARG */ : (isfinite(l) ? 0 : 5 /* MNL_ERR_NONFINITE */);
    *counter = 0u;
  }
}

__global__ void k_pack(int64_t N, int64_t Npad, int p, int Kd, const double* __restrict__ X,
                       const double* __restrict__ Z, double* Xp, int ldX, double* Zp, int ldZ, double* Pr,
                       int ldP) {
  // Xp / Zp rows (zero padding rows and columns) and the zero padding rows of Pr (rows >= N are
  // never written by pass 1; the Hessian kernels rely on them being exactly zero)
  const int64_t nx = Npad * ldX, nz = Zp ? Npad * ldZ : 0, npr = (Npad - N) * ldP;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nx + nz + npr;
       e += (int64_t)gridDim.x * blockDim.x) {
    if (e >= nx + nz) {
      Pr[N * ldP + (e - nx - nz)] = 0.0;
    } else if (e < nx) {
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

template <int KPL, int CM, bool HV, bool YZS>
cudaError_t launch_k(const EvalPlan& plan, const EvalArgs& a, cudaStream_t st) {
  static uint64_t attr_mask = 0;
  cudaError_t e = set_once_per_device(attr_mask, [] {
    return cudaFuncSetAttribute(k_eval_kernel<KPL, CM, HV, YZS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                227 * 1024);
  });
  if (e != cudaSuccess) return e;
  k_eval_kernel<KPL, CM, HV, YZS><<<plan.grid, plan.block, plan.smem, st>>>(a);
  count_launch();
  return cudaGetLastError();
}

// ---- small single-CTA vector kernels of the truncated-Newton (CG) step (n <= 16384) ----------
// Every reduction runs in one CTA in a fixed order (deterministic).
__device__ __forceinline__ double cta_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
  return t;  // valid in thread 0
}

// Ap = -Hp, out[0] = p . Ap
__global__ void __launch_bounds__(1024) k_cg_curv(int n, const double* p, const double* hp, double* ap, double* out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double a = -hp[i];
    ap[i] = a;
    s = fma(p[i], a, s);
  }
  s = cta_sum(s, red);
  if (threadIdx.x == 0) out[0] = s;
}

// delta += alpha p, r -= alpha Ap, out[0] = r . r
__global__ void __launch_bounds__(1024) k_cg_update(int n, double alpha, const double* p, const double* ap,
                                                   double* delta, double* r, double* out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    delta[i] = fma(alpha, p[i], delta[i]);
    const double ri = fma(-alpha, ap[i], r[i]);
    r[i] = ri;
    s = fma(ri, ri, s);
  }
  s = cta_sum(s, red);
  if (threadIdx.x == 0) out[0] = s;
}

// p = r + beta p
__global__ void __launch_bounds__(1024) k_cg_dir(int n, double beta, const double* r, double* p) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) p[i] = fma(beta, p[i], r[i]);
}

// ---- the data-parallel exchange of one evaluation ----------------------------
// xbuf = [l, bad-choice flag, g (n)] from this rank's finalised scalars [l, ||g||^2, flag] and g
__global__ void __launch_bounds__(1024) k_dp_gather(int n, const double* scal, const double* grad, double* xbuf) {
  if (threadIdx.x == 0) {
    xbuf[0] = scal[0];
    xbuf[1] = scal[2];
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) xbuf[2 + i] = grad ? grad[i] : 0.0;
}

// after the all-reduce (sums over ranks): g <- xbuf[2..], scal <- [l, ||g||^2 (fixed order), flag]
__global__ void __launch_bounds__(1024) k_dp_scatter(int n, const double* xbuf, double* grad, double* scal) {
  __shared__ double red[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double g = xbuf[2 + i];
    if (grad) grad[i] = g;
    s = fma(g, g, s);
  }
  s = cta_sum(s, red);
  if (threadIdx.x == 0) {
    scal[0] = xbuf[0];
    scal[1] = s;
    scal[2] = xbuf[1];
  }
}

}  // namespace

cudaError_t launch_dp_gather(int n, const double* scal, const double* grad, double* xbuf, cudaStream_t st) {
  k_dp_gather<<<1, 1024, 0, st>>>(n, scal, grad, xbuf);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_dp_scatter(int n, const double* xbuf, double* grad, double* scal, cudaStream_t st) {
  k_dp_scatter<<<1, 1024, 0, st>>>(n, xbuf, grad, scal);
  count_launch();
  return cudaGetLastError();
}

static int eval_qp(const Dims& D) { return (D.q + 3) / 4 * 4; }
static int eval_xs(const Dims& D) { return pad4mod16(eval_qp(D)); }

static size_t eval_smem(const Dims& D, int kpl, bool yzs, int ns, bool stream = false, int ti = 0) {
  const int KP = 32 * kpl, KPS = KP + 4, TI = yzs ? YZS_TI : (ti ? ti : tile_rows(kpl, (D.d + D.f) > 0));
  const int slot = D.K * (D.f + D.d);
  const int nw = yzs ? NWY : NW;
  size_t n = (size_t)eval_qp(D) * KPS + 2 * (size_t)TI * eval_xs(D) + (size_t)TI * KPS +
             (((D.d + D.f) || kpl >= 8) && !yzs ? (size_t)TI * KPS : 0) +
             (yzs || stream ? 0 : (size_t)nw * kpl * D.d * 32 + (size_t)nw * D.f * 32) +
             (size_t)D.K * D.d + D.f + 1 + TI +  // + 2*TI ints
             ((D.d + D.f) && !yzs ? (size_t)nw * 8 * 33 : 0);
  if (yzs) {
    n = (n + 1) & ~(size_t)1;
    const size_t ring = (size_t)nw * ns * slot;
    size_t scr = (size_t)nw * kpl * D.d * 32 + (size_t)nw * D.f * 32;  // finalisation scratch
    if (scr < (size_t)2 * nw * 32) scr = (size_t)2 * nw * 32;          // (and the loglik partials)
    n += (size_t)nw * ns + (ring > scr ? ring : scr);
  }
  return n * sizeof(double);
}

bool eval_plan(const Dims& D, EvalPlan* plan, int sms) {
  int kpl = 1;
  while (32 * kpl < D.K) kpl *= 2;
  if (kpl > 8) return false;

  // YZS (alternative-varying rows staged per warp with bulk copies): f even <= 16, d <= 8, whole
  // 16-byte rows (K f, K d even), K <= 64; 3 ring slots if they fit, else 2
  plan->yzs = 0;
  plan->ns = 0;
  const bool yzs_ok = (D.d + D.f) > 0 && kpl <= 2 && D.f % 2 == 0 && D.f <= YZS_F && D.d <= YZS_D &&
                      (D.K * D.f) % 2 == 0 && (D.K * D.d) % 2 == 0 && !getenv("MNL_NO_YZS");
  size_t smem = eval_smem(D, kpl, false, 0);
  if (yzs_ok) {
    for (int ns = 4; ns >= 2; --ns) {  // 4: two rows computed while the next two land
      const size_t sz = eval_smem(D, kpl, true, ns);
      if (sz <= 227 * 1024) {
        plan->yzs = 1;
        plan->ns = ns;
        smem = sz;
        break;
      }
    }
  }
  plan->ti = plan->yzs ? YZS_TI : tile_rows(kpl, (D.d + D.f) > 0);
  plan->stream = 0;
  if (smem > 227 * 1024 && !plan->yzs && (D.d + D.f) > 0) {
    // many alternative-specific / generic variables: no gradient partials in shared memory; pass 1
    // writes the residual rows and k_yz_grad streams Z and Y for the alpha / gamma gradients
    smem = eval_smem(D, kpl, false, 0, true);
    plan->stream = 1;
  }
  plan->rg = plan->stream ? D.N * (int64_t)D.K : 0;
  if (smem > 227 * 1024) return false;  // sm_100a opt-in maximum (232448 bytes)
  // register budget: phase-C accumulators (cm x cn blocks) + the phase-B row (nbn blocks)
  const int nwarps = plan->yzs ? NWY : NW;
  const int nbn = 4 * kpl, wn = nbn < 8 ? nbn : 8, wm = nwarps / wn, cn = nbn / wn;
  const int mb = (eval_qp(D) + 7) / 8;
  int cm = 2;
  while (cm < (mb + wm - 1) / wm) cm *= 2;
  if (cm > 8 || 2 * cm * cn + 2 * nbn > 96) return false;
  plan->cm = cm;
  plan->kpl = kpl;
  plan->smem = smem;
  plan->block = nwarps * 32;
  const int ti = plan->ti;
  const int64_t ntiles = (D.N + ti - 1) / ti;
  int64_t grid = sms;
  if (grid > ntiles) grid = ntiles;
  plan->grid = (int)grid;
  plan->n_part = 2 + D.n_p;
  eval_plan_w(D, plan, sms);
  eval_plan_x(D, plan, sms);
  return true;
}

static cudaError_t launch_eval_core(const Dims& D, const EvalPlan& plan, const double* X, const double* Y,
                                    const double* Z, const int32_t* choice, const double* coef, const Packed* pk,
                                    bool want_grad, bool writeP, bool hv, double* part, int* err, cudaStream_t st) {
  EvalArgs a;
  a.N = D.N; a.K = D.K; a.p = D.p; a.f = D.f; a.d = D.d; a.q = D.q; a.n_p = D.n_p;
  a.off_alpha = D.off_alpha; a.off_gamma = D.off_gamma;
  a.QP = eval_qp(D); a.XS = eval_xs(D);
  a.TI = plan.ti; a.SCR = 0;
  a.X = X; a.Y = Y; a.Z = Z; a.choice = choice; a.coef = coef;
  a.Pr = (writeP || hv) ? pk->Pr : nullptr;
  a.ldP = (writeP || hv) ? pk->ldP : 0;
  a.want_grad = want_grad; a.writeP = writeP && !hv;
  a.part = part; a.n_part = plan.n_part; a.err = err;
  a.Rg = plan.stream ? part + (size_t)plan.grid * plan.n_part : nullptr;
  a.NS = plan.ns;
  a.SLOT = D.K * (D.f + D.d);
#define MNL_EVAL_CM(KPL_, HV_, YZS_)                                                         \
  if (plan.cm == 2) return launch_k<KPL_, 2, HV_, YZS_>(plan, a, st);                        \
  if (plan.cm == 4) return launch_k<KPL_, 4, HV_, YZS_>(plan, a, st);                        \
  return launch_k<KPL_, 8, HV_, YZS_>(plan, a, st);
#define MNL_EVAL_CASE(KPL_)                                                                  \
  case KPL_:                                                                                 \
    if (hv) { MNL_EVAL_CM(KPL_, true, false) }                                               \
    MNL_EVAL_CM(KPL_, false, false)
  if (plan.yzs) {
    if (plan.kpl == 1) {
      if (hv) { MNL_EVAL_CM(1, true, true) }
      MNL_EVAL_CM(1, false, true)
    }
    if (plan.kpl == 2) {
      if (hv) { MNL_EVAL_CM(2, true, true) }
      MNL_EVAL_CM(2, false, true)
    }
    return cudaErrorInvalidValue;
  }
  switch (plan.kpl) {
    MNL_EVAL_CASE(1)
    MNL_EVAL_CASE(2)
    MNL_EVAL_CASE(4)
    case 8:  // eval_plan never picks cm = 8 for K > 128 (its register rule), so it is not instantiated
      if (hv) return plan.cm == 2 ? launch_k<8, 2, true, false>(plan, a, st) : launch_k<8, 4, true, false>(plan, a, st);
      return plan.cm == 2 ? launch_k<8, 2, false, false>(plan, a, st) : launch_k<8, 4, false, false>(plan, a, st);
  }
#undef MNL_EVAL_CM
#undef MNL_EVAL_CASE
  return cudaErrorInvalidValue;
}

static cudaError_t launch_eval_impl(const Dims& D, const EvalPlan& plan, const double* X, const double* Y,
                                    const double* Z, const int32_t* choice, const double* coef, const Packed* pk,
                                    bool want_grad, bool writeP, bool hv, double* part, int* err, cudaStream_t st) {
  cudaError_t e = launch_eval_core(D, plan, X, Y, Z, choice, coef, pk, want_grad, writeP, hv, part, err, st);
  if (e != cudaSuccess || !plan.stream || !want_grad) return e;
  double* Rg = part + (size_t)plan.grid * plan.n_part;
  const int ny = std::max(1, (D.K * D.d + 256 * YG_CH - 1) / (256 * YG_CH));  // alpha chunks
  k_yz_grad<<<dim3(plan.grid, ny), 256, 0, st>>>(D.N, D.K, D.d, D.f, Y, Z, Rg, part, plan.n_part, D.off_alpha,
                                                 D.off_gamma);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_eval(const Dims& D, const EvalPlan& plan, const double* X, const double* Y,
                        const double* Z, const int32_t* choice, const double* coef,
                        const Packed* pk, bool want_grad, bool writeP, double* part, int* err,
                        cudaStream_t st) {
  if (plan.w.T) return launch_eval_w(D, plan, X, Y, Z, choice, coef, pk, want_grad, writeP, false, part, err, st);
  if (plan.x_grid) return launch_eval_x(D, plan, X, choice, coef, pk, want_grad, writeP, false, part, err, st);
  return launch_eval_impl(D, plan, X, Y, Z, choice, coef, pk, want_grad, writeP, false, part, err, st);
}

cudaError_t launch_hessvec(const Dims& D, const EvalPlan& plan, const double* X, const double* Y, const double* Z,
                           const int32_t* choice, const double* v, const Packed* pk, double* part, int* err,
                           cudaStream_t st) {
  if (plan.w.T) return launch_eval_w(D, plan, X, Y, Z, choice, v, pk, true, false, true, part, err, st);
  if (plan.x_grid && plan.x_hv) return launch_eval_x(D, plan, X, choice, v, pk, true, false, true, part, err, st);
  return launch_eval_impl(D, plan, X, Y, Z, choice, v, pk, true, false, true, part, err, st);
}

cudaError_t launch_cg_curv(int n, const double* p, const double* hp, double* ap, double* out, cudaStream_t st) {
  k_cg_curv<<<1, 1024, 0, st>>>(n, p, hp, ap, out);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_cg_update(int n, double alpha, const double* p, const double* ap, double* delta, double* r,
                             double* out, cudaStream_t st) {
  k_cg_update<<<1, 1024, 0, st>>>(n, alpha, p, ap, delta, r, out);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_cg_dir(int n, double beta, const double* r, double* p, cudaStream_t st) {
  k_cg_dir<<<1, 1024, 0, st>>>(n, beta, r, p);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_eval_finalize(const Dims& D, const EvalPlan& plan, const double* part,
                                 bool want_grad, double* grad, double* loglik_out, double* scal,
                                 const int* err, unsigned* counter, cudaStream_t st, int* status_out, bool hv) {
  int blocks = want_grad ? (D.n_p + 255) / 256 : 1;
  k_eval_finalize<<<blocks, 256, 0, st>>>(part, plan.n_part, eval_nblk(plan, hv), D.n_p, want_grad, grad,
                                          loglik_out, scal, err, counter, status_out);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_pack(const Dims& D, const Packed& pk, const double* X, const double* Z,
                        cudaStream_t st) {
  int64_t total = pk.Npad * pk.ldX + (D.d ? pk.Npad * pk.ldZ : 0) + (pk.Npad - D.N) * pk.ldP;
  int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
  k_pack<<<blocks, 256, 0, st>>>(D.N, pk.Npad, D.p, D.K * D.d, X, Z, pk.Xp, pk.ldX,
                                 D.d ? pk.Zp : nullptr, pk.ldZ, pk.Pr, pk.ldP);
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
