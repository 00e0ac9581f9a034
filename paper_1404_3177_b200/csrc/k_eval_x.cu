// Pass 1 for X-only models (f = d = 0, K <= 128), two warp groups
// per CTA (k_eval_x): the same quantities as k_eval.cu's X-only path —
//   a1 u_ik = xi_k + x_i.beta_k  (u_i0 = 0: the base), as U = X~ B on the FP64 tensor pipe
//   a2 P_ik = e^{u_ik - m_i} / s_i                                (R12)
//   a3 l    = sum_i (u_{i,y_i} - m_i - log s_i)
//   a4 g[beta_k] = sum_i x~_i r_ik = X~^T R on the tensor pipe, r_ik = I(y_i = k) - P_ik
// and the probability rows Pr[i] for the Hessian pass, or (HV) the Hessian-vector product with
// r_ik = -P_ik (s_ik - sum_l P_il s_il).
//
// In k_eval.cu the CTA's eight warps walk through a 64-row tile together: X~ B (DMMA), the row
// softmax (FP64 ALU: 2 K exps per lane), a CTA barrier, X~^T R (DMMA), a CTA barrier — so the tensor
// pipe idles while every warp is in the softmax (c4: 59 % active). Here the CTA holds TWO groups of
// four warps, each with its own 32-row tiles, staging buffers and named barrier; nothing ties the
// groups together, so one group's softmax overlaps the other's DMMAs (every scheduler hosts one
// warp of each group). Warp w of a group owns rows 8 w .. 8 w + 7 of the tile in X~ B (all
// alternative blocks; the C fragment leaves a lane with 2 alternatives per 8-block of one
// individual, so the row softmax is lane-local plus two shuffles) and a quarter of the
// alternative blocks in X~^T R (accumulators in registers for the whole kernel). The two groups'
// partials are added in a fixed order at the end, then over the CTAs by k_eval_finalize.
// The kernel is instantiated on the number of 8-alternative blocks NBN = ceil(K / 8) itself (c4:
// 13, not the 16 of K padded to 128 columns: run-time guards around the padding blocks cost more
// than they save) and on the depth CM of a warp's X~^T R accumulators.
#include <algorithm>
#include <cstdlib>

#include "eval_common.h"

namespace mnl {
namespace {

constexpr int XG = 2;        // warp groups per CTA
constexpr int XW = 4;        // warps per group
constexpr int XT = 8 * XW;   // individuals per group tile

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}
__device__ __forceinline__ void group_sync(int grp) {
  asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(32 * XW) : "memory");
}

// row stride of the beta table and the residual rows: >= 8 nbn, = 4 or 12 (mod 16) doubles
// (conflict-free 4 x 8 fragment gathers)
__host__ __device__ constexpr int x_kps(int nbn) {
  int s = 8 * nbn;
  while (s % 16 != 4 && s % 16 != 12) ++s;
  return s;
}

template <int NBN, int CM, bool HV>
__global__ void __launch_bounds__(XG * XW * 32, 1) k_eval_x(const EvalArgs A) {
  extern __shared__ __align__(16) double sm[];
  constexpr int KPS = x_kps(NBN);
  constexpr int WN = NBN >= 4 ? 4 : (NBN >= 2 ? 2 : 1);  // phase-C warp grid of a group: WN x WM warps
  constexpr int WM = XW / WN;
  // alternative blocks per warp in phase C. With four warps across the blocks (NBN >= 4) a warp takes
  // blocks wg, wg + 4, ... of the whole rounds, and the REM = NBN % 4 blocks left over are cut into
  // their (m-block, block) cells, dealt evenly to the four warps (c4: 13 blocks = 3 rounds + 1 block
  // of 7 cells, 2 + 2 + 2 + 1 — instead of one warp with a fourth whole block and three waiting at
  // the group barrier). NBN < 4: blocks cwn, cwn + WN (the last may not exist).
  constexpr bool SPLIT = WN == 4 && (NBN % 4) != 0;
  constexpr int REM = SPLIT ? NBN % 4 : 0;
  constexpr int CN = SPLIT ? NBN / 4 : (NBN + WN - 1) / WN;
  constexpr int RC = SPLIT ? (REM * 8 + 3) / 4 : 1;  // cells per warp at most (MB <= 8)
  const int K = A.K, q = A.q, p = A.p, QP = A.QP, XS = A.XS;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int grp = w / XW, wg = w % XW, gtid = tid - grp * (32 * XW);
  const int r4 = lane & 3, c8 = lane >> 2;
  double* Bs = sm;                                         // [QP][KPS]  Bs[a][k] = beta_k[a]
  double* Gb = Bs + QP * KPS + (size_t)grp * A.SCR;        // this group's buffers
  double* Xs = Gb;                                         // [2][XT][XS] x~ tiles (col 0 = 1)
  double* Rs = Xs + 2 * XT * XS;                           // [XT][KPS]  residuals
  int* chs = reinterpret_cast<int*>(Rs + XT * KPS);        // [2][XT] choices
  for (int idx = tid; idx < QP * KPS; idx += blockDim.x) {
    const int a = idx / KPS, k = idx - a * KPS;
    Bs[idx] = (a < q && k >= 1 && k < K) ? A.coef[(k - 1) * q + a] : 0.0;
  }
  for (int idx = gtid; idx < 2 * XT * XS; idx += 32 * XW) Xs[idx] = ((idx % XS) == 0) ? 1.0 : 0.0;

  const int MB = (QP + 7) / 8;
  const int cwm = wg / WN, cwn = wg % WN;
  double G[CM][CN][2];  // beta gradient: x~ columns 8 (cwm + WM mi) + c8, alternatives of blocks cwn + WN j
#pragma unroll
  for (int i = 0; i < CM; ++i)
#pragma unroll
    for (int j = 0; j < CN; ++j) G[i][j][0] = G[i][j][1] = 0.0;
  double Gr[RC][2];    // ... and this warp's cells of the left-over blocks
  int cellA[RC], cellB[RC];  // their x~ column / alternative offsets (-1: no such cell)
#pragma unroll
  for (int t = 0; t < RC; ++t) {
    Gr[t][0] = Gr[t][1] = 0.0;
    const int cells = REM * MB, per = (cells + 3) / 4, e = wg * per + t;
    const bool have = SPLIT && t < per && e < cells;
    cellA[t] = have ? (e % MB) * 8 + c8 : -1;                    // m-block e % MB
    cellB[t] = have ? (NBN - REM + e / MB) * 8 + c8 : -1;       // block NBN - REM + e / MB
  }
  double l_s = 0.0, l_c = 0.0;  // Neumaier loglik of this lane's rows (lanes with r4 == 0)

  const int64_t ntiles = (A.N + XT - 1) / XT;
  const int64_t t0 = (int64_t)blockIdx.x * XG + grp, tstride = (int64_t)gridDim.x * XG;
  const unsigned xs_s = static_cast<unsigned>(__cvta_generic_to_shared(Xs));
  const int x_i0 = p ? gtid / p : 0, x_a0 = p ? gtid - x_i0 * p : 0;          // gtid = x_i0 p + x_a0
  const int x_di = p ? (32 * XW) / p : 0, x_da = p ? (32 * XW) - x_di * p : 0;  // the group size likewise
  auto prefetch = [&](int64_t tile, int buf) {
    const int64_t i0 = tile * XT;
    const int nt = (int)(A.N - i0 < XT ? A.N - i0 : XT);
    const unsigned dst = xs_s + 8u * (unsigned)(buf * XT * XS);
    const double* src = A.X + i0 * p;
    int i = x_i0, a = x_a0;  // element e = gtid + j 128 = i p + a, advanced without divisions
    for (int e = gtid; e < nt * p; e += 32 * XW) {
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
    for (int ii = gtid; ii < nt; ii += 32 * XW)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                       static_cast<unsigned>(__cvta_generic_to_shared(chs + buf * XT + ii))),
                   "l"(A.choice + i0 + ii)
                   : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  int buf = 0;
  __syncthreads();  // the tables and the ones / zeros of the x~ tiles are in place
  if (t0 < ntiles) prefetch(t0, 0);
  for (int64_t tile = t0; tile < ntiles; tile += tstride, buf ^= 1) {
    const int64_t i0 = tile * XT;
    const int nt = (int)(A.N - i0 < XT ? A.N - i0 : XT);
    // this tile's copies (issued one tile ago) have landed, and — the same barrier — the group is
    // done with the previous tile: its buffer can take the next tile, Rs the next residuals
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    group_sync(grp);
    if (tile + tstride < ntiles) prefetch(tile + tstride, buf ^ 1);
    const double* X_t = Xs + buf * XT * XS;
    const int* ch_t = chs + buf * XT;

    // ---------------- u = X~ B on DMMA (warp wg: rows 8 wg .. 8 wg + 7, all alternative blocks) --------
    const int il = 8 * wg + c8;  // this lane's individual (C-fragment row)
    const bool valid = il < nt;
    const int64_t i = i0 + il;
    double u[NBN][2];
#pragma unroll
    for (int nb = 0; nb < NBN; ++nb) u[nb][0] = u[nb][1] = 0.0;
    for (int a0 = 0; a0 < QP; a0 += 4) {
      const double av = X_t[il * XS + a0 + r4];
#pragma unroll
      for (int nb = 0; nb < NBN; ++nb) dmma884(u[nb][0], u[nb][1], av, Bs[(a0 + r4) * KPS + nb * 8 + c8]);
    }
    double* Rrow = Rs + il * KPS;
    if constexpr (HV) {
      // Hessian-vector product: u holds s_ik = (J_i v)_k; with P_i from the last evaluation (Pr),
      // r_ik = -P_ik (s_ik - sum_l P_il s_il) (P:462-476 applied to v)
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
#pragma unroll
      for (int nb = 0; nb < NBN; ++nb)
        *reinterpret_cast<double2*>(Rrow + nb * 8 + 2 * r4) =
            make_double2(-pk[nb][0] * (u[nb][0] - ps), -pk[nb][1] * (u[nb][1] - ps));
    } else {
      int y = valid ? ch_t[il] : -1;  // -1 (a row beyond N): no alternative matches, residuals 0
      if (valid && (y < 0 || y >= K)) {
        atomicOr(A.err, 1);
        y = 0;
      }
      // shift by the (fp32-rounded) maximum: any shift is exact for the softmax, it only has to
      // keep e^{u - m} <= ~1 (R12)
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
#pragma unroll
      for (int nb = 0; nb < NBN; ++nb) {
        const int k = nb * 8 + 2 * r4;
        double2 P2, R2;
        P2.x = __dmul_rn(u[nb][0], inv_s);  // (rounded products: the same r with and without the P rows)
        P2.y = __dmul_rn(u[nb][1], inv_s);
        R2.x = (k == y ? 1.0 : 0.0) - P2.x;
        R2.y = (k + 1 == y ? 1.0 : 0.0) - P2.y;
        *reinterpret_cast<double2*>(Rrow + k) = R2;
        if (A.writeP && valid) {
          double* pr = A.Pr + i * A.ldP + k;
          if (k + 1 < K) *reinterpret_cast<double2*>(pr) = P2;
          else if (k < K) pr[0] = P2.x;
        }
      }
    }
    group_sync(grp);  // Rs complete

    // ---------------- beta gradient G[a][k] += sum_i x~_ia r_ik on DMMA ----------------
    if (A.want_grad) {
      for (int ks = 0; ks < XT / 4; ++ks) {
        double bf[CN];
#pragma unroll
        for (int j = 0; j < CN; ++j)
          bf[j] = (j < CN - 1 || cwn + WN * j < NBN) ? Rs[(4 * ks + r4) * KPS + (cwn + WN * j) * 8 + c8] : 0.0;
#pragma unroll
        for (int mi = 0; mi < CM; ++mi) {
          const int mb = cwm + WM * mi;
          if (mb < MB) {
            const double af = X_t[(4 * ks + r4) * XS + mb * 8 + c8];
#pragma unroll
            for (int j = 0; j < CN; ++j)
              if (j < CN - 1 || cwn + WN * j < NBN) dmma884(G[mi][j][0], G[mi][j][1], af, bf[j]);
          }
        }
        if constexpr (SPLIT) {
#pragma unroll
          for (int t = 0; t < RC; ++t)
            if (cellA[t] >= 0)
              dmma884(Gr[t][0], Gr[t][1], X_t[(4 * ks + r4) * XS + cellA[t]], Rs[(4 * ks + r4) * KPS + cellB[t]]);
        }
      }
    }
  }

  // ---------------- CTA partials (fixed order): group 0 + group 1 ----------------
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();  // both groups are done: the buffers are free
  double* out = A.part + (size_t)blockIdx.x * A.n_part;
  double* LL = sm;                 // [XG XW 32][2] loglik partials
  double* V = sm + 2 * XG * XW * 32;  // [XG][n_beta]
  LL[2 * tid] = l_s;
  LL[2 * tid + 1] = l_c;
  if (A.want_grad) {
    double* Vg = V + (size_t)grp * A.n_p;
#pragma unroll
    for (int mi = 0; mi < CM; ++mi) {
      const int mb = cwm + WM * mi;
      if (mb < MB) {
        const int a = mb * 8 + c8;
#pragma unroll
        for (int j = 0; j < CN; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int k = (cwn + WN * j) * 8 + 2 * r4 + h;
            if (a < q && k >= 1 && k < K && cwn + WN * j < NBN) Vg[(k - 1) * q + a] = G[mi][j][h];
          }
      }
    }
  }
  if (A.want_grad && SPLIT) {
    double* Vg = V + (size_t)grp * A.n_p;
#pragma unroll
    for (int t = 0; t < RC; ++t)
      if (cellA[t] >= 0) {
        const int a = cellA[t];                      // = 8 m + c8
        const int k0 = cellB[t] - c8 + 2 * r4;      // = 8 block + 2 r4
#pragma unroll
        for (int h = 0; h < 2; ++h)
          if (a < q && k0 + h >= 1 && k0 + h < K) Vg[(k0 + h - 1) * q + a] = Gr[t][h];
      }
  }
  __syncthreads();
  if (tid == 0) {
    double s = 0.0, c = 0.0;
    for (int t = 0; t < XG * XW * 32; t += 4) {  // lanes with r4 == 0 hold rows; (group, warp, lane) order
      neu_add(s, c, LL[2 * t]);
      neu_add(s, c, LL[2 * t + 1]);
    }
    out[0] = s;
    out[1] = c;
  }
  if (!A.want_grad) return;
  for (int idx = tid; idx < A.n_p; idx += blockDim.x) out[2 + idx] = V[idx] + V[A.n_p + idx];
}

template <int NBN, int CM, bool HV>
cudaError_t launch_x(const EvalPlan& plan, const EvalArgs& a, cudaStream_t st) {
  static uint64_t attr_mask = 0;
  cudaError_t e = set_once_per_device(attr_mask, [] {
    return cudaFuncSetAttribute(k_eval_x<NBN, CM, HV>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  });
  if (e != cudaSuccess) return e;
  k_eval_x<NBN, CM, HV><<<plan.x_grid, XG * XW * 32, plan.x_smem, st>>>(a);
  count_launch();
  return cudaGetLastError();
}

int x_qp(const Dims& D) { return (D.q + 3) / 4 * 4; }

}  // namespace

// The two-group X-only plan; plan->x_grid = 0 when the shape does not qualify.
void eval_plan_x(const Dims& D, EvalPlan* plan, int sms) {
  plan->x_grid = 0;
  plan->x_smem = 0;
  plan->x_cm = 0;
  plan->x_hv = 0;
  if (D.d + D.f != 0 || D.K > 128 || D.K < 2 || getenv("MNL_NO_XG")) return;
  const int nbn = (D.K + 7) / 8, KPS = x_kps(nbn), QP = x_qp(D), XS = pad4mod16(QP);
  const int wn = nbn >= 4 ? 4 : (nbn >= 2 ? 2 : 1), wm = XW / wn, cn = (nbn + wn - 1) / wn;
  const int mb = (QP + 7) / 8;
  int cm = 4;  // instantiated depths: 4 and 8
  while (cm * wm < mb) cm *= 2;
  // register budget: the phase-C accumulators (cm x cn blocks) + the phase-B row (nbn blocks)
  if (cm > 8 || 2 * cm * cn + 2 * nbn > 100) return;
  const size_t grp_doubles = (size_t)2 * XT * XS + (size_t)XT * KPS + XT;  // x~ tiles, residuals, choices
  const size_t total = ((size_t)QP * KPS + XG * grp_doubles) * sizeof(double);
  if (total > 227 * 1024) return;
  // the final partials reuse the buffers
  if ((size_t)(2 * XG * XW * 32 + XG * D.n_p) * sizeof(double) > total) return;
  const int64_t ntiles = (D.N + XT - 1) / XT;
  // small problems: the 64-row kernel's latency is lower (MNL_FORCE_XG: tests)
  if (D.N < 8192 && !getenv("MNL_FORCE_XG")) return;
  int64_t grid = sms;
  if (grid * XG > ntiles) grid = (ntiles + XG - 1) / XG;
  plan->x_grid = (int)grid;
  plan->x_smem = total;
  plan->x_cm = cm;
  plan->x_scr = (int)grp_doubles;
  plan->x_hv = 1;
}

cudaError_t launch_eval_x(const Dims& D, const EvalPlan& plan, const double* X, const int32_t* choice,
                          const double* coef, const Packed* pk, bool want_grad, bool writeP, bool hv, double* part,
                          int* err, cudaStream_t st) {
  EvalArgs a{};
  a.N = D.N; a.K = D.K; a.p = D.p; a.f = 0; a.d = 0; a.q = D.q; a.n_p = D.n_p;
  a.off_alpha = D.off_alpha; a.off_gamma = D.off_gamma;
  a.QP = x_qp(D); a.XS = pad4mod16(a.QP); a.SCR = plan.x_scr;
  a.X = X; a.choice = choice; a.coef = coef;
  a.Pr = (writeP || hv) ? pk->Pr : nullptr;
  a.ldP = (writeP || hv) ? pk->ldP : 0;
  a.want_grad = want_grad; a.writeP = writeP && !hv;
  a.part = part; a.n_part = plan.n_part; a.err = err;
#define MNL_X_NBN(NBN_)                                                                                       \
  case NBN_:                                                                                                  \
    if (hv) return plan.x_cm == 4 ? launch_x<NBN_, 4, true>(plan, a, st) : launch_x<NBN_, 8, true>(plan, a, st); \
    return plan.x_cm == 4 ? launch_x<NBN_, 4, false>(plan, a, st) : launch_x<NBN_, 8, false>(plan, a, st);
  switch ((D.K + 7) / 8) {
    MNL_X_NBN(1) MNL_X_NBN(2) MNL_X_NBN(3) MNL_X_NBN(4) MNL_X_NBN(5) MNL_X_NBN(6) MNL_X_NBN(7) MNL_X_NBN(8)
    MNL_X_NBN(9) MNL_X_NBN(10) MNL_X_NBN(11) MNL_X_NBN(12) MNL_X_NBN(13) MNL_X_NBN(14) MNL_X_NBN(15) MNL_X_NBN(16)
  }
#undef MNL_X_NBN
  return cudaErrorInvalidValue;
}

}  // namespace mnl
