// Pass 1 for models with alternative-varying data, "team" mapping
// (k_eval_w): the same quantities as k_eval.cu —
//   a1 u_ik = xi_k + x_i.beta_k + z_ik.alpha_k + y_ik.gamma      (base: P:129-138)
//   a2 P_ik = e^{u_ik - m_i} / s_i                                (R12)
//   a3 l    = sum_i (u_{i,y_i} - m_i - log s_i)
//   a4 g    = X~^T R, Z_k^T r_k, sum_k Y_k^T r_k, r_ik = I(y_i = k) - P_ik
// and, for the Hessian pass, the rows Pr[i] = [P_i0..P_i,K-1, ybar_i] —
// with a mapping that issues less than half the instructions per individual of the YZS path.
//
// A TEAM of S warps works on groups of 8 consecutive individuals, the 8 rows of one DMMA m-block;
// warp t of the team owns the alternative blocks t NBW .. t NBW + NBW - 1 (8 alternatives each).
// There is no CTA barrier in the main loop:
//   * the team's last warp bulk-copies the group's 8 Y rows, 8 Z rows and its 8 x p block of X
//     into the team's ring (two halves of 8 slots; a "full" mbarrier with the byte count and an
//     "empty" mbarrier the S warps arrive on per half): while group n is computed, group n + 1 is
//     in flight (whole rows, 16-byte multiples, DRAM bytes = algorithmic bytes);
//   * X~ B on the FP64 tensor pipe (mma.sync m8n8k4): the C fragment leaves lane (c8, r4) with
//     individual c8's alternatives 8 nb + 2 r4 + {0, 1} — four lanes per individual, every lane a
//     fixed set of alternatives — so the Y / Z contributions are shared loads of two adjacent
//     alternatives' rows and FMAs in that same register layout, and every lane carries live
//     alternatives (K = 50: 64 slots over 4 warps, none of the 32 lanes idle);
//   * softmax across the team with ONE exchange: warp t shifts by n_t ln 2, n_t = round(max_t /
//     ln 2) (any shift is exact for the softmax, R12), i.e. it forms e^{u} 2^{-n_t}; the warps
//     publish (n_t, s_t) per individual, meet on a named barrier, and rescale by the exact powers
//     of two 2^{n_t - n}, n = max_t n_t;
//   * the gamma / alpha gradients stay in that layout (lane-private partials; the z values of a
//     lane's alternatives are kept in registers from the utility step); the residual rows go to
//     shared memory once, from where X~^T R runs on DMMA (accumulators in registers);
//   * ybar_i = y_{i,y_i} - sum_k r_ik y_ik (the same FMAs as the gamma gradient: sum_k r_ik = 0
//     regrouped), summed over the team through shared memory (Hessian pass only).
// CTA partials are combined in a fixed order, then over the CTAs by k_eval_finalize
// (deterministic). Conditions (eval_plan_w): K <= 64, p <= 31, f even <= 16, d <= 8, K d even,
// N >= 8, two teams' rings fit in shared memory. Anything else takes k_eval.cu's paths.
#include <algorithm>
#include <cstdlib>

#include "eval_common.h"

namespace mnl {
namespace {

constexpr int GR = 8;                  // individuals per group (one DMMA m-block)
constexpr int WNS = 2 * GR;            // ring slots per team (two halves)
constexpr int W_F = 16, W_D = 8;       // capacity: generic variables, alternative-specific variables
constexpr int W_MB = 4;                // m-blocks of x columns (p <= 32)
// The kernel is instantiated for every (f / 2, d) with f even <= 16, d <= 8; the instantiations are
// split over three translation units (this file as part 0; k_eval_w1.cu and k_eval_w2.cu include it
// as parts 1 and 2) so that they compile in parallel: part P holds f / 2 = 3 P .. 3 P + 2.
#ifndef MNL_W_PART
#define MNL_W_PART 0
#endif
#define MNL_W_ROW(X, F2_) X(F2_, 0) X(F2_, 1) X(F2_, 2) X(F2_, 3) X(F2_, 4) X(F2_, 5) X(F2_, 6) X(F2_, 7) X(F2_, 8)
#if MNL_W_PART == 0
#define MNL_W_SHAPES(X) MNL_W_ROW(X, 0) MNL_W_ROW(X, 1) MNL_W_ROW(X, 2)
#define MNL_W_PART_FN launch_eval_w_part0
#elif MNL_W_PART == 1
#define MNL_W_SHAPES(X) MNL_W_ROW(X, 3) MNL_W_ROW(X, 4) MNL_W_ROW(X, 5)
#define MNL_W_PART_FN launch_eval_w_part1
#else
#define MNL_W_SHAPES(X) MNL_W_ROW(X, 6) MNL_W_ROW(X, 7) MNL_W_ROW(X, 8)
#define MNL_W_PART_FN launch_eval_w_part2
#endif
constexpr int W_S = 8;                 // warps per team at most (K <= 64, one alternative block per warp)

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

// 2^j for an integer-valued double (the conversion saturates; NaN gives 2^0)
__device__ __forceinline__ double pow2_nonpos(double j) { return pow2_int(min(__double2int_rn(j), 1000)); }

// e^u 2^{-n} for an integer-valued double n with u - n ln 2 <= ~1 and finite u: u = t ln2 + r
// (|r| <= ln2/2, Cody-Waite with fdlibm's split ln2), e^r by exp_poly, times 2^{t - n} built in the
// exponent field (0 below the normal range). Branch-free, so that the calls of a lane's
// alternatives interleave. NaN and +-inf give NaN. live = false (an alternative >= K): times 0.
__device__ __forceinline__ double exp_scaled(double u, double n, bool live) {
  const double t = rint(u * c_exp[0]);
  double r = fma(t, c_exp[1], u);
  r = fma(t, c_exp[2], r);
  // t - n is exact (integers below 2^53); the conversion saturates; NaN converts to 0
  const int ji = live ? min(__double2int_rn(t - n), 1000) : -2000;
  return exp_poly(r) * pow2_int(ji);
}

template <int NBW, int F2, int D, bool WP, bool HV>
__global__ void __launch_bounds__(NBW == 1 ? 448 : 256, 1) k_eval_w(const EvalArgs A, const EvalWLayout L) {
  extern __shared__ __align__(16) double sm[];
  constexpr int f = 2 * F2;
  const int K = A.K, q = A.q, p = A.p, PP = (A.p + 3) & ~3, Kd = K * D;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int r4 = lane & 3, c8 = lane >> 2;
  const int S = L.S, team = w / S, wt = w - team * S, nteams = L.T;
  // the team's last warp stages the ring and sums the loglik: it is the one whose alternative
  // blocks may lie (partly) beyond K, i.e. the one with the least other work
  const int lead = S - 1;
  const int KS = L.KS, RS = L.RS, YS = L.YS, ZS = L.ZS, XH = L.XH;
  double* Bs = sm;                                  // [PP][KS]  Bs[a][k] = beta_k[1 + a], x column a (column 0: base)
  double* gamma_s = sm + L.off_gam;                 // [f]
  double* Tb = sm + L.off_team + (size_t)team * L.team_sz;
  uint64_t* bars = reinterpret_cast<uint64_t*>(Tb);  // full[2], empty[2]
  double* Ex = Tb + 4;                              // [2][S][8][2]  (n_t, s_t)
  double* Uy = Ex + 2 * S * GR * 2;                 // [2][8]        u_{i, y_i} (written by its owner)
  double* Gx = Uy + 2 * GR;                         // [S][8][f]     ybar partials (Hessian pass only)
  double* Xb = Gx + S * GR * f;                     // [2][XH]  the group's x rows [8][p]
  double* Rw = Xb + 2 * XH;                         // [8][RS]  residual rows of the group
  double* Yr = Rw + GR * RS;                        // [16][YS]
  double* Zr = Yr + WNS * YS;                       // [16][ZS]
  for (int idx = tid; idx < PP * KS + 8; idx += blockDim.x) {  // (+ 8: the last row's reads beyond K)
    const int a = idx / KS, k = idx - a * KS;
    Bs[idx] = (a < p && k >= 1 && k < K) ? A.coef[(k - 1) * q + a + 1] : 0.0;
  }
  for (int idx = tid; idx < f; idx += blockDim.x) gamma_s[idx] = A.coef[A.off_gamma + idx];
  if (wt == lead && lane == 0) {
    mbar_init(bars, 1);
    mbar_init(bars + 1, 1);
    mbar_init(bars + 2, S);
    mbar_init(bars + 3, S);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const unsigned bar_s = static_cast<unsigned>(__cvta_generic_to_shared(bars));
  const unsigned xb_s = static_cast<unsigned>(__cvta_generic_to_shared(Xb));
  const unsigned yr_s = static_cast<unsigned>(__cvta_generic_to_shared(Yr));
  const unsigned zr_s = static_cast<unsigned>(__cvta_generic_to_shared(Zr));
  const unsigned by = (unsigned)(K * f) * 8u, bz = (unsigned)Kd * 8u, bx = (unsigned)(GR * p) * 8u;
  const int64_t ngroups = (A.N + GR - 1) / GR;
  const int64_t tg = (int64_t)blockIdx.x * nteams + team, tstride = (int64_t)gridDim.x * nteams;
  // the team's lead warp stages group g into ring half `half`. A ragged last group is read as the
  // last 8 rows of the data; its rows below g * 8 are masked where they are used.
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
  if (wt == lead) {
    if (tg < ngroups) issue(tg, 0);
    if (tg + tstride < ngroups) issue(tg + tstride, 1);
  }

  // this lane's alternatives: block nbg = wt NBW + nb, k = 8 nbg + 2 r4 + h; those >= K are read at
  // K - 1 (finite data) and their utilities set to -inf
  const int krel = K - 8 * wt * NBW - 2 * r4;  // alternative (nb, h) exists iff 8 nb + h < krel
  auto ok = [&](int nb, int h) { return 8 * nb + h < krel; };
  int oy[NBW][2], oz[NBW][2];
#pragma unroll
  for (int nb = 0; nb < NBW; ++nb)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int kc = min(8 * (wt * NBW + nb) + 2 * r4 + h, K - 1);
      oy[nb][h] = kc * f;
      oz[nb][h] = kc * D;
    }
  double xi[NBW][2];       // this lane's intercepts (0 for the base alternative)
  double gxi[NBW][2];      // ... and their gradient, lane-private over the lane's individual
#pragma unroll
  for (int nb = 0; nb < NBW; ++nb)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int k = 8 * (wt * NBW + nb) + 2 * r4 + h;
      xi[nb][h] = (k >= 1 && k < K) ? A.coef[(k - 1) * q] : 0.0;
      gxi[nb][h] = 0.0;
    }
  double G[W_MB][NBW][2];  // beta gradient: x columns 8 mb + c8, this lane's alternatives
#pragma unroll
  for (int mb = 0; mb < W_MB; ++mb)
#pragma unroll
    for (int nb = 0; nb < NBW; ++nb) G[mb][nb][0] = G[mb][nb][1] = 0.0;
  double gam[f ? f : 1];  // gamma gradient, lane-private partials
#pragma unroll
  for (int e = 0; e < f; ++e) gam[e] = 0.0;
  double ga[NBW][2][D ? D : 1];  // alpha gradient of this lane's alternatives
#pragma unroll
  for (int nb = 0; nb < NBW; ++nb)
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int c = 0; c < D; ++c) ga[nb][h][c] = 0.0;
  const double* alpha_g = A.coef + A.off_alpha;  // [K][D], laid out like the Z row
  double l_s = 0.0, l_c = 0.0;
  const int MBr = (p + 7) / 8;
  const bool xlast_ok = 8 * (MBr - 1) + c8 < p;  // this lane's x column of the last m-block exists
  const int bar_id = 1 + team, bar_n = 32 * S;

  // the lane's choice y_i, loaded one group ahead
  const int32_t* ch_lane = A.choice + c8;
  auto choice_of = [&](int64_t g) {
    const int64_t i0 = min(g * GR, A.N - GR);
    return g < ngroups ? __ldg(ch_lane + i0) : 0;
  };
  int y_next = choice_of(tg);
  int n = 0;
  for (int64_t g = tg; g < ngroups; g += tstride, ++n) {
    const int half = n & 1;
    const unsigned upar = (unsigned)((n >> 1) & 1);
    const int64_t i0t = g * GR;
    const int64_t i0 = i0t + GR > A.N ? A.N - GR : i0t;
    const int64_t gi = i0 + c8;          // this lane's individual
    const bool valid = gi >= i0t;        // (rows of a ragged last group seen by the previous one)
    int y = y_next;
    y_next = choice_of(g + tstride);
    if (y < 0 || y >= K) {
      if (valid && r4 == 0 && wt == lead) atomicOr(A.err, 1);
      y = 0;
    }
    // Hessian-vector product: P_i of the last evaluation (its loads land behind the wait)
    double pk[NBW][2];
    if constexpr (HV) {
#pragma unroll
      for (int nb = 0; nb < NBW; ++nb) {
        const double* pr = A.Pr + gi * A.ldP + 8 * (wt * NBW + nb) + 2 * r4;
        double2 P2 = make_double2(0.0, 0.0);
        if (ok(nb, 1)) P2 = __ldg(reinterpret_cast<const double2*>(pr));
        else if (ok(nb, 0)) P2.x = __ldg(pr);
        pk[nb][0] = P2.x;
        pk[nb][1] = P2.y;
      }
    }
    mbar_wait(bar_s + 8u * half, upar);
    const double* xb = Xb + half * XH;
    const double* yb = Yr + (half * GR + c8) * YS;
    const double* zb = Zr + (half * GR + c8) * ZS;

    // ---- a1: z_k . alpha_k first (its loads land while the DMMAs run; z is kept in registers
    // for the alpha gradient) ----
    double zv[NBW][2][D ? D : 1], zu[NBW][2];
#pragma unroll
    for (int nb = 0; nb < NBW; ++nb)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        zu[nb][h] = 0.0;
#pragma unroll
        for (int c = 0; c < D; ++c) zv[nb][h][c] = zb[oz[nb][h] + c];
      }
#pragma unroll
    for (int c = 0; c < D; ++c)
#pragma unroll
      for (int nb = 0; nb < NBW; ++nb)
#pragma unroll
        for (int h = 0; h < 2; ++h) zu[nb][h] = fma(zv[nb][h][c], __ldg(alpha_g + oz[nb][h] + c), zu[nb][h]);
    // ---- a1: u = X~ B on DMMA (rows = the group's individuals) ----
    double u[NBW][2];
#pragma unroll
    for (int nb = 0; nb < NBW; ++nb) u[nb][0] = xi[nb][0] + zu[nb][0], u[nb][1] = xi[nb][1] + zu[nb][1];
    {
      const double* xa = xb + c8 * p + r4;                       // A fragment: x_{c8, a0 + r4}
      const double* ba = Bs + r4 * KS + wt * NBW * 8 + c8;        // B fragment: Bs[a0 + r4][8 nbg + c8]
      int a0 = 0;
      double ub[NBW][2];  // a second accumulator set: two DMMA chains per block
#pragma unroll
      for (int nb = 0; nb < NBW; ++nb) ub[nb][0] = ub[nb][1] = 0.0;
#pragma unroll 2
      for (; a0 + 8 <= p; a0 += 8) {
        const double av = xa[a0], aw = xa[a0 + 4];
#pragma unroll
        for (int nb = 0; nb < NBW; ++nb) {
          dmma884(u[nb][0], u[nb][1], av, ba[a0 * KS + nb * 8]);
          dmma884(ub[nb][0], ub[nb][1], aw, ba[(a0 + 4) * KS + nb * 8]);
        }
      }
      for (; a0 + 4 <= p; a0 += 4) {
        const double av = xa[a0];
#pragma unroll
        for (int nb = 0; nb < NBW; ++nb) dmma884(ub[nb][0], ub[nb][1], av, ba[a0 * KS + nb * 8]);
      }
#pragma unroll
      for (int nb = 0; nb < NBW; ++nb) u[nb][0] += ub[nb][0], u[nb][1] += ub[nb][1];
      if (a0 < p) {  // ragged last step: columns >= p read column p - 1 against zero rows of Bs
        const double av = xb[c8 * p + min(a0 + r4, p - 1)];
#pragma unroll
        for (int nb = 0; nb < NBW; ++nb) dmma884(u[nb][0], u[nb][1], av, ba[a0 * KS + nb * 8]);
      }
    }
    // ---- a1: + y_k . gamma (pairs of components, 16-byte loads) ----
#pragma unroll
    for (int e2 = 0; e2 < F2; ++e2) {
      {
        const double2 g2 = *reinterpret_cast<const double2*>(gamma_s + 2 * e2);
#pragma unroll
        for (int nb = 0; nb < NBW; ++nb)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const double2 v = *reinterpret_cast<const double2*>(yb + oy[nb][h] + 2 * e2);
            u[nb][h] = fma(v.y, g2.y, fma(v.x, g2.x, u[nb][h]));
          }
      }
    }
    double r[NBW][2];
    const int yl = y - 8 * wt * NBW;  // y relative to this warp's alternatives
    if constexpr (HV) {
      // ---- Hessian-vector product: u holds s_ik = (J_i v)_k; r_ik = -P_ik (s_ik - sum_l P_il s_il), so
      // that the gradient contractions below accumulate H v (P:462-476 applied to v); one exchange
      // of the partial sums over the team ----
      double ps = 0.0;
#pragma unroll
      for (int nb = 0; nb < NBW; ++nb) ps = fma(pk[nb][1], u[nb][1], fma(pk[nb][0], u[nb][0], ps));
      ps += __shfl_xor_sync(0xffffffffu, ps, 1);
      ps += __shfl_xor_sync(0xffffffffu, ps, 2);
      if (r4 == 0) Ex[((half * S + wt) * GR + c8) * 2] = ps;
      asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(bar_n) : "memory");
      const double* ex = Ex + (half * S * GR + c8) * 2;
      double pt = (r4 < S ? ex[r4 * GR * 2] : 0.0) + (r4 + 4 < S ? ex[(r4 + 4) * GR * 2] : 0.0);
      pt += __shfl_xor_sync(0xffffffffu, pt, 1);
      pt += __shfl_xor_sync(0xffffffffu, pt, 2);
#pragma unroll
      for (int nb = 0; nb < NBW; ++nb)
#pragma unroll
        for (int h = 0; h < 2; ++h) r[nb][h] = valid ? -pk[nb][h] * (u[nb][h] - pt) : 0.0;
    } else {
    // ---- a2 / a3: softmax over the team, loglik ----
    float mf = -INFINITY;
#pragma unroll
    for (int nb = 0; nb < NBW; ++nb)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        mf = ok(nb, h) ? fmaxf(mf, (float)u[nb][h]) : mf;
      }
    mf = fmaxf(mf, __shfl_xor_sync(0xffffffffu, mf, 1));
    mf = fmaxf(mf, __shfl_xor_sync(0xffffffffu, mf, 2));
    // this warp's shift n_t ln 2 (a warp whose alternatives of a ragged last block are all >= K
    // cannot occur: its first block starts below K)
    const double nt = rint((double)mf * 1.4426950408889634);
    double ssum = 0.0;
#pragma unroll
    for (int nb = 0; nb < NBW; ++nb)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (8 * nb + 2 * r4 + h == yl) Uy[half * GR + c8] = u[nb][h];
        const double e = exp_scaled(u[nb][h], nt, ok(nb, h));  // 0 for an alternative >= K
        u[nb][h] = e;
        ssum += e;
      }
    ssum += __shfl_xor_sync(0xffffffffu, ssum, 1);
    ssum += __shfl_xor_sync(0xffffffffu, ssum, 2);
    if (r4 == 0) *reinterpret_cast<double2*>(Ex + ((half * S + wt) * GR + c8) * 2) = make_double2(nt, ssum);
    asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(bar_n) : "memory");
    // lane r4 of the individual's quad folds warps r4 and r4 + 4 (S <= 8), then the quad combines
    double nmax, stot;
    {
      const double* ex = Ex + (half * S * GR + c8) * 2;
      const double2 none = make_double2(-1e300, 0.0);
      const double2 na = r4 < S ? *reinterpret_cast<const double2*>(ex + r4 * GR * 2) : none;
      const double2 nb2 = r4 + 4 < S ? *reinterpret_cast<const double2*>(ex + (r4 + 4) * GR * 2) : none;
      nmax = na.x > nb2.x ? na.x : nb2.x;
      double o = __shfl_xor_sync(0xffffffffu, nmax, 1);
      nmax = o > nmax ? o : nmax;
      o = __shfl_xor_sync(0xffffffffu, nmax, 2);
      nmax = o > nmax ? o : nmax;
      stot = fma(nb2.y, pow2_nonpos(nb2.x - nmax), na.y * pow2_nonpos(na.x - nmax));
      stot += __shfl_xor_sync(0xffffffffu, stot, 1);
      stot += __shfl_xor_sync(0xffffffffu, stot, 2);
    }
    if (valid && r4 == 0 && wt == lead) {
      const double uy = Uy[half * GR + c8];
      // l_i = u_y - n ln2 - log s (ln2 split as in exp_scaled)
      neu_add(l_s, l_c, fma(nmax, -1.90821492927058770002e-10, fma(nmax, -6.93147180369123816490e-01, uy)) - log(stot));
    }
    const double cs = pow2_nonpos(nt - nmax) * recip_ge1(stot);
#pragma unroll
    for (int nb = 0; nb < NBW; ++nb) {
      const int k = 8 * nb + 2 * r4;
      // (explicitly rounded products: the gradient pass must not contract them into r where the
      // Hessian pass, which also stores P, cannot -- both passes give bit-identical l and g)
      const double P0 = __dmul_rn(u[nb][0], cs), P1 = __dmul_rn(u[nb][1], cs);
      r[nb][0] = valid ? ((k == yl ? 1.0 : 0.0) - P0) : 0.0;
      r[nb][1] = valid ? ((k + 1 == yl ? 1.0 : 0.0) - P1) : 0.0;
      if (WP && valid) {
        double* pr = A.Pr + gi * A.ldP + 8 * wt * NBW + k;
        if (ok(nb, 1)) *reinterpret_cast<double2*>(pr) = make_double2(P0, P1);
        else if (ok(nb, 0)) pr[0] = P0;
      }
    }
    }  // !HV
    if (A.want_grad || WP) {
      // ---- a4: gamma gradient sum_k y_ke r_k in the same layout; WP: ybar_e = y_{y,e} - that sum ----
#pragma unroll
      for (int e2 = 0; e2 < F2; ++e2) {
        {
          double a0 = 0.0, a1 = 0.0;
#pragma unroll
          for (int nb = 0; nb < NBW; ++nb)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const double2 v = *reinterpret_cast<const double2*>(yb + oy[nb][h] + 2 * e2);
              a0 = fma(v.x, r[nb][h], a0);
              a1 = fma(v.y, r[nb][h], a1);
            }
          gam[2 * e2] += a0;
          gam[2 * e2 + 1] += a1;
          if constexpr (WP) {  // the individual's sum over this warp's alternatives -> Gx
            a0 += __shfl_xor_sync(0xffffffffu, a0, 1);
            a1 += __shfl_xor_sync(0xffffffffu, a1, 1);
            a0 += __shfl_xor_sync(0xffffffffu, a0, 2);
            a1 += __shfl_xor_sync(0xffffffffu, a1, 2);
            if (r4 == 0) *reinterpret_cast<double2*>(Gx + (wt * GR + c8) * f + 2 * e2) = make_double2(a0, a1);
          }
        }
      }
      if constexpr (WP) {
        asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(bar_n) : "memory");
        // warp t writes components e = lane-quad slot r4 + 4 t, + 4 S, ... of its 8 individuals
        for (int e = r4 + 4 * wt; e < f; e += 4 * S) {
          double s = 0.0;
          for (int t = 0; t < S; ++t) s += Gx[(t * GR + c8) * f + e];
          if (valid) A.Pr[gi * A.ldP + K + e] = yb[y * f + e] - s;
        }
      }
    }
    if (A.want_grad) {
      // ---- residual rows (this warp's columns) to shared memory; intercept gradient ----
#pragma unroll
      for (int nb = 0; nb < NBW; ++nb) {
        if (8 * (wt * NBW + nb) < K)
          *reinterpret_cast<double2*>(Rw + c8 * RS + 8 * (wt * NBW + nb) + 2 * r4) = make_double2(r[nb][0], r[nb][1]);
        gxi[nb][0] += r[nb][0];
        gxi[nb][1] += r[nb][1];
      }
      // ---- a4: alpha gradient from the kept z values ----
#pragma unroll
      for (int nb = 0; nb < NBW; ++nb)
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int c = 0; c < D; ++c)  // (one block per warp: z re-read, its registers are needed)
            ga[nb][h][c] = fma(NBW == 1 ? zb[oz[nb][h] + c] : zv[nb][h][c], r[nb][h], ga[nb][h][c]);
      __syncwarp();
      // ---- a4: beta gradient G += X~^T R on DMMA (k = the group's individuals) ----
#pragma unroll
      for (int ks = 0; ks < GR / 4; ++ks) {
        double bf[NBW];
#pragma unroll
        for (int nb = 0; nb < NBW; ++nb) bf[nb] = Rw[(4 * ks + r4) * RS + (wt * NBW + nb) * 8 + c8];
        const double* xr = xb + (4 * ks + r4) * p;  // A fragment: x_{4 ks + r4, 8 mb + c8}
#pragma unroll
        for (int mb = 0; mb < W_MB; ++mb) {
          if (mb < MBr - 1) {
            const double af = xr[mb * 8 + c8];
#pragma unroll
            for (int nb = 0; nb < NBW; ++nb) dmma884(G[mb][nb][0], G[mb][nb][1], af, bf[nb]);
          } else if (mb == MBr - 1) {  // the last block: columns >= p contribute zeros
            const double af = xlast_ok ? xr[mb * 8 + c8] : 0.0;
#pragma unroll
            for (int nb = 0; nb < NBW; ++nb) dmma884(G[mb][nb][0], G[mb][nb][1], af, bf[nb]);
          }
        }
      }
    }
    __syncwarp();  // every lane is done with this half (ring, x block) and with the residual rows
    if (lane == 0)
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar_s + 8u * (2 + half)) : "memory");
    if (wt == lead && g + 2 * tstride < ngroups) {
      mbar_wait(bar_s + 8u * (2 + half), upar);  // all S warps have left the half
      issue(g + 2 * tstride, half);
    }
  }

  // ---------------- CTA partials (fixed order) ----------------
  __syncthreads();  // every team has consumed all it staged: the team regions are free
  const int nw = blockDim.x >> 5;
  double* out = A.part + (size_t)blockIdx.x * A.n_part;
  double* V = sm + L.off_team;                          // [T][n_p]   beta / alpha entries per team
  double* Vg = V + (size_t)nteams * A.n_p;             // [nw][W_F]  gamma partial per warp
  double* LL = Vg + nw * W_F;                          // [T 8][2]   loglik partials
  if (wt == lead && r4 == 0) {
    LL[2 * (team * GR + c8)] = l_s;
    LL[2 * (team * GR + c8) + 1] = l_c;
  }
  if (A.want_grad) {
    double* Vt = V + (size_t)team * A.n_p;
#pragma unroll
    for (int mb = 0; mb < W_MB; ++mb)
#pragma unroll
      for (int nb = 0; nb < NBW; ++nb)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int a = mb * 8 + c8, k = 8 * (wt * NBW + nb) + 2 * r4 + h;
          if (a < p && k >= 1 && k < K) Vt[(k - 1) * q + a + 1] = G[mb][nb][h];
        }
    // intercepts and alpha: the lane's partial is over its own individual (c8): sum the 8 lanes
    // with equal r4
#pragma unroll
    for (int nb = 0; nb < NBW; ++nb)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int k = 8 * (wt * NBW + nb) + 2 * r4 + h;
        double s = gxi[nb][h];
        s += __shfl_xor_sync(0xffffffffu, s, 4);
        s += __shfl_xor_sync(0xffffffffu, s, 8);
        s += __shfl_xor_sync(0xffffffffu, s, 16);
        if (c8 == 0 && k >= 1 && k < K) Vt[(k - 1) * q] = s;
      }
#pragma unroll
    for (int nb = 0; nb < NBW; ++nb)
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int c = 0; c < D; ++c) {
          double s = ga[nb][h][c];
          s += __shfl_xor_sync(0xffffffffu, s, 4);
          s += __shfl_xor_sync(0xffffffffu, s, 8);
          s += __shfl_xor_sync(0xffffffffu, s, 16);
          if (c8 == 0 && ok(nb, h)) Vt[A.off_alpha + oz[nb][h] + c] = s;
        }
#pragma unroll
    for (int e = 0; e < f; ++e) {
      {
        const double s = warp_sum(gam[e]);
        if (lane == 0) Vg[w * W_F + e] = s;
      }
    }
  }
  __syncthreads();
  if (tid == 0) {
    double s = 0.0, c = 0.0;
    for (int t = 0; t < nteams * GR; ++t) {
      neu_add(s, c, LL[2 * t]);
      neu_add(s, c, LL[2 * t + 1]);
    }
    out[0] = s;
    out[1] = c;
  }
  if (!A.want_grad) return;
  for (int idx = tid; idx < A.off_gamma; idx += blockDim.x) {
    double v = 0.0;
    for (int t = 0; t < nteams; ++t) v += V[(size_t)t * A.n_p + idx];
    out[2 + idx] = v;
  }
  for (int e = tid; e < f; e += blockDim.x) {
    double v = 0.0;
    for (int ww = 0; ww < nw; ++ww) v += Vg[ww * W_F + e];
    out[2 + A.off_gamma + e] = v;
  }
}

template <int NBW, int F2, int D, bool WP, bool HV>
cudaError_t launch_w(const EvalPlan& plan, const EvalArgs& a, cudaStream_t st) {
  static uint64_t attr_mask = 0;
  cudaError_t e = set_once_per_device(attr_mask, [] {
    return cudaFuncSetAttribute(k_eval_w<NBW, F2, D, WP, HV>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  });
  if (e != cudaSuccess) return e;
  const EvalWLayout& L = plan.w;
  k_eval_w<NBW, F2, D, WP, HV><<<plan.w_grid, L.S * L.T * 32, L.smem, st>>>(a, L);
  count_launch();
  return cudaGetLastError();
}

}  // namespace

#if MNL_W_PART == 0
// The team mapping's layout, one for the gradient pass and the Hessian pass (which also exchanges
// the ybar partials): the same teams and groups, hence bit-identical loglik and gradient from both.
// L->T = 0 when the shape does not qualify.
static void plan_w_layout(const Dims& D, EvalWLayout* out) {
  out->T = 0;
  const int Kd = D.K * D.d, Kf = D.K * D.f;
  const int NB = (D.K + 7) / 8, PP = (D.p + 3) / 4 * 4;
  const int64_t ngroups = (D.N + GR - 1) / GR;
  // two alternative blocks per warp (one block per warp puts 14 warps of 128 registers on the SM
  // instead of 8 of 255, but was slower: its per-warp fixed work and the 7-warp exchange outweigh
  // the extra warps; c5: 0.356 vs 0.320 ms)
  int best = 0;
  for (int nbw = 2; nbw <= 2; ++nbw) {
    EvalWLayout L;
    L.NBW = nbw;
    L.S = (NB + nbw - 1) / nbw;
    if (L.S > W_S) continue;
    // row stride of the beta table and of the residual rows: the K alternatives' blocks; a warp
    // whose second block lies wholly beyond K reads (finite, unused) values of the next row there
    L.KS = 8 * NB;
    while (L.KS % 16 != 4 && L.KS % 16 != 12) ++L.KS;  // conflict-free 4 x 8 fragment gathers
    L.RS = L.KS;
    L.YS = Kf;
    // slot stride = 16 (mod 32) bytes: the 16-byte loads of two individuals' lanes interleave
    while (Kf && L.YS % 4 != 2) ++L.YS;
    L.ZS = Kd + (Kd & 1);
    L.XH = GR * D.p;
    L.off_gam = PP * L.KS + 8;  // (+ 8: the last row's reads beyond K)
    L.off_team = L.off_gam + ((D.f + 1) & ~1);
    L.team_sz = 4 + 2 * L.S * GR * 2 + 2 * GR + L.S * GR * D.f + 2 * L.XH + GR * L.RS + WNS * L.YS +
                WNS * L.ZS;
    L.team_sz = (L.team_sz + 1) & ~1;
    int T = std::min(15, (nbw == 1 ? 14 : 8) / L.S);  // 448 / 256 threads; named barriers 1..15
    while (T >= 1 && (size_t)(L.off_team + (size_t)T * L.team_sz) * sizeof(double) > 227 * 1024) --T;
    if ((int64_t)T > ngroups) T = (int)ngroups;
    if (T < 1) continue;
    // the final partials reuse the team regions
    if ((size_t)T * L.team_sz < (size_t)T * D.n_p + (size_t)T * L.S * W_F + (size_t)T * GR * 2) continue;
    if (T * L.S <= best) continue;
    best = T * L.S;
    L.T = T;
    L.smem = (size_t)(L.off_team + (size_t)T * L.team_sz) * sizeof(double);
    *out = L;
  }
  // fewer than 8 warps per SM (large rows: one team's ring only): the YZS path hides latency
  // better (K = 64, f = 10, d = 5: 0.37 vs 0.54 ms); small problems: the YZS path's latency is
  // lower. MNL_FORCE_YZW (tests) lifts both rules.
  if ((best < 8 || D.N < 4096) && !getenv("MNL_FORCE_YZW")) out->T = 0;
}

// The team mapping's plan (layout and grid); plan->w.T = 0 when the shape does not qualify.
void eval_plan_w(const Dims& D, EvalPlan* plan, int sms) {
  plan->w.T = 0;
  plan->w_grid = 0;
  const int Kd = D.K * D.d;
  if ((D.d + D.f) == 0 || D.K > 64 || D.K < 2 || D.p > 8 * W_MB || D.f % 2 || D.f > W_F || D.d > W_D || Kd % 2 ||
      D.N < GR || getenv("MNL_NO_YZW"))
    return;
  // bulk copies need 16-byte-aligned sources: the x block of a ragged last group starts at row N - 8
  if ((D.N % GR) && ((D.N - GR) * D.p) % 2) return;
  plan_w_layout(D, &plan->w);
  if (!plan->w.T) return;
  const int64_t ngroups = (D.N + GR - 1) / GR;
  int64_t grid = sms;
  if (grid * plan->w.T > ngroups) grid = (ngroups + plan->w.T - 1) / plan->w.T;
  plan->w_grid = (int)grid;
}

#endif  // MNL_W_PART == 0

cudaError_t MNL_W_PART_FN(const Dims& D, const EvalPlan& plan, const double* X, const double* Y, const double* Z,
                          const int32_t* choice, const double* coef, const Packed* pk, bool want_grad, bool writeP,
                          bool hv, double* part, int* err, cudaStream_t st) {
  EvalArgs a{};
  a.N = D.N; a.K = D.K; a.p = D.p; a.f = D.f; a.d = D.d; a.q = D.q; a.n_p = D.n_p;
  a.off_alpha = D.off_alpha; a.off_gamma = D.off_gamma;
  a.X = X; a.Y = Y; a.Z = Z; a.choice = choice; a.coef = coef;
  a.Pr = (writeP || hv) ? pk->Pr : nullptr;
  a.ldP = (writeP || hv) ? pk->ldP : 0;
  a.want_grad = want_grad; a.writeP = writeP && !hv;
  a.part = part; a.n_part = plan.n_part; a.err = err;
#define MNL_W_LAUNCH(F2_, D_)                                                      \
  if (D.f == 2 * F2_ && D.d == D_)                                                  \
    return hv ? launch_w<2, F2_, D_, false, true>(plan, a, st)                       \
              : (writeP ? launch_w<2, F2_, D_, true, false>(plan, a, st) : launch_w<2, F2_, D_, false, false>(plan, a, st));
  MNL_W_SHAPES(MNL_W_LAUNCH)
#undef MNL_W_LAUNCH
  return cudaErrorInvalidValue;
}

#if MNL_W_PART == 0
cudaError_t launch_eval_w(const Dims& D, const EvalPlan& plan, const double* X, const double* Y, const double* Z,
                          const int32_t* choice, const double* coef, const Packed* pk, bool want_grad, bool writeP,
                          bool hv, double* part, int* err, cudaStream_t st) {
  auto fn = D.f < 6 ? launch_eval_w_part0 : (D.f < 12 ? launch_eval_w_part1 : launch_eval_w_part2);
  return fn(D, plan, X, Y, Z, choice, coef, pk, want_grad, writeP, hv, part, err, st);
}
#endif

}  // namespace mnl
