// Newton step: -H = L L^T by a tiled Cholesky factorisation, then
// L y = g and L^T delta = y (Eq. "NR update": delta = -H^{-1} g; -H is positive definite
// by global concavity).
//
// k_chol_dag: ONE persistent cooperative kernel, no grid barriers. The lower triangle is cut into
// 64 x 64 tiles and every tile (i, j), i >= j, is one task, left-looking:
//     C = A_ij - sum_{k<j} L_ik L_jk^T                       (DMMA, accumulators in registers)
//     i == j:  L_jj = chol(C) and Linv_j = L_jj^{-1} in shared memory; y_j = Linv_j (b_j - sum_k L_jk y_k)
//     i >  j:  L_ij = C Linv_j^T                             (DMMA)
// Tasks are dealt to the CTAs round-robin in column-major order (a topological order of the
// tile DAG), each CTA runs its tasks in order, and a task waits only for the tiles it reads: one
// flag per tile (release / acquire, tagged with a per-call epoch). The operands (L_ik, L_jk, and
// y_k for the diagonal tasks) come from a tile-major copy of L written by the tasks themselves
// (padded rows of 68 doubles: conflict-free fragment loads), by cp.async.bulk into a two-stage
// mbarrier ring, so the tile of step k + 1 is in flight while step k multiplies. Every A_ij is read
// once (row-major, by its own task) and every L_ij written once: the HBM traffic is that of the
// matrix, not one rewrite of the trailing matrix per panel. The critical path is one chain per
// tile column (last update, potrf, trsm), not three grid-wide barriers per panel.
// With a single tile (n <= 64) the backward solve runs in the same task; otherwise it is one
// cooperative wavefront kernel (k_trsv_wave: CTA b owns block b and folds in the solved blocks as
// their flags are published).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "internal.h"

namespace mnl {
namespace {

constexpr int NB = 64;
constexpr int LDS = NB + 4;  // 68 = 4 (mod 16) doubles: conflict-free 8x4 fragment gathers
constexpr int LDR = NB + 1;  // row-per-thread access patterns
constexpr int TS = NB * LDS; // doubles per stored tile (tile-major L, padded Linv)

// offset of tile (i, j), i >= j, in the tile-major packed lower triangle
__host__ __device__ __forceinline__ int64_t tile_off(int i, int j) { return ((int64_t)i * (i + 1) / 2 + j) * TS; }

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// out[M][N] = alpha * Am[M][K] Bm[K][N] from shared memory on DMMA (row-major operands; M, N
// multiples of 8, K of 4); 8x8 output tiles dealt to warps wid, wid + nw, ...
__device__ __forceinline__ void smem_gemm(double* out, int lo, const double* Am, int la, const double* Bm, int lb, int M,
                                          int N, int K, double alpha, int wid, int nw) {
  const int lane = threadIdx.x & 31, r = lane >> 2, kq = lane & 3;
  const int tn_n = N / 8, tiles = (M / 8) * tn_n;
  for (int t = wid; t < tiles; t += nw) {
    const int tm = t / tn_n, tn = t - tm * tn_n;
    double c0 = 0.0, c1 = 0.0;
    for (int k0 = 0; k0 < K; k0 += 4)
      dmma(c0, c1, Am[(tm * 8 + r) * la + k0 + kq], Bm[(k0 + kq) * lb + tn * 8 + r]);
    out[(tm * 8 + r) * lo + tn * 8 + 2 * kq] = alpha * c0;
    out[(tm * 8 + r) * lo + tn * 8 + 2 * kq + 1] = alpha * c1;
  }
}

// potrf_core: Cholesky of the jb x jb block in S (shared, LDR rows: the lower triangle, identity
// beyond jb, strict upper triangle zero) fused with X = L^{-1}, by 16-column blocks b, pipelined
// across warp roles: warp 0 runs only the critical chain — factor and invert the 16 x 16 diagonal
// block b (lane r owns row r of the block in registers; one shared-memory broadcast per column;
// unscaled right-looking updates a_rk -= a_rc a_kc / a_cc, the scaling by 1 / sqrt(a_cc) applied
// once at the end; then lane r solves for column r of L^{-1}) — while the seven other warps, on
// DMMA, form L_{>b,b} = A_{>b,b} X_bb^T, update the next diagonal block first (which releases warp
// 0 for block b + 1), then the rest of the trailing triangle and row block b of X
// (X_{b,<b} = -X_bb L_{b,<b} X_{<b,<b}). Measured (clock64, one 64 x 64 block): 27.0k cycles, was
// 35.6k with all warps stepping through the sub-panels together; warp 0's chain is the bound (its
// 16 columns take 4.4k cycles alone, 6.6-7.1k beside the workers' shared-memory traffic). S <- L, X <- L^{-1}; returns (in thread 0) whether a pivot
// was not positive (it is replaced by 1 to keep the values finite). Rows / columns >= jb of S and X
// are left undefined when jb < 64 (callers mask them). All 256 threads call it.
constexpr int SB = 16;

// warp 0: the 16 x 16 diagonal block at (c0, c0): S <- L, X <- L^{-1}. Lanes 16..31 mirror 0..15.
// colb: shared [SB] (the broadcast column).
__device__ __forceinline__ bool potrf16_warp(double (*S)[LDR], double (*X)[LDR], int c0, double* colb) {
  const int lane = threadIdx.x & 31, r = lane & 15;
  double a[SB], rsv[SB];
#pragma unroll
  for (int c = 0; c < SB; ++c) a[c] = (c <= r) ? S[c0 + r][c0 + c] : 0.0;
  bool bad = false;
#pragma unroll
  for (int c = 0; c < SB; ++c) {
    if (lane < SB) colb[lane] = a[c];  // column c (rows >= c are current)
    __syncwarp();
    double d = colb[c];
    const bool ok = d > 0.0 && d < INFINITY;
    bad |= !ok;
    d = ok ? d : 1.0;
    const double rs = rsqrt(d);
    rsv[c] = rs;
    const double f = a[c] * (rs * rs);  // a_rc / a_cc
    // unpredicated: lane r also updates its strict upper part (k > r), which is masked below —
    // per-lane predicates cost more issue slots than the extra FMAs
#pragma unroll
    for (int k = c + 1; k < SB; ++k) a[k] = fma(-f, colb[k], a[k]);
    __syncwarp();
  }
#pragma unroll
  for (int c = 0; c < SB; ++c) a[c] = (c <= r) ? a[c] * rsv[c] : 0.0;  // L_rc = a_rc / sqrt(a_cc)
  if (lane < SB) {
#pragma unroll
    for (int c = 0; c < SB; ++c) S[c0 + r][c0 + c] = a[c];
  }
  __syncwarp();
  double x[SB];  // column r of L^{-1}: x_t = (delta_tr - sum_{s<t} L_ts x_s) / L_tt, right-looking
#pragma unroll
  for (int t = 0; t < SB; ++t) x[t] = (t == r) ? 1.0 : 0.0;
#pragma unroll
  for (int t = 0; t < SB; ++t) {
    x[t] *= rsv[t];
#pragma unroll
    for (int u = t + 1; u < SB; ++u) x[u] = fma(-S[c0 + u][c0 + t], x[t], x[u]);
  }
  if (lane < SB) {
#pragma unroll
    for (int t = 0; t < SB; ++t) X[c0 + t][c0 + r] = x[t];
  }
  return bad;
}

// Named barriers of potrf_core (id 0 is __syncthreads): kPanel = block b factored (warp 0 arrives,
// the workers wait), kDiag = the next diagonal block updated (the workers arrive, warp 0 waits),
// kWork = the seven worker warps only.
constexpr int kPanel = 1, kDiag = 2, kWork = 3;
#ifndef POTRF_TRACE
#define POTRF_TRACE(i)
#endif
__device__ __forceinline__ void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void bar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__device__ __noinline__ bool potrf_core(int jb, double* dsm) {
  double(*S)[LDR] = reinterpret_cast<double(*)[LDR]>(dsm);
  double(*X)[LDR] = reinterpret_cast<double(*)[LDR]>(dsm + NB * LDR);
  __shared__ double T[NB][SB + 1];  // L_{r,b} for the row blocks r > b
  __shared__ double M[SB][NB + 1];  // M_b = L_{b,<b} X_{<b,<b}
  __shared__ double colb[SB];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int lr = lane >> 2, lk = lane & 3;
  for (int e = tid; e < NB * NB; e += 256) X[e >> 6][e & 63] = 0.0;
  __syncthreads();
  const int nbk = (jb + SB - 1) / SB;
  bool bad = false;
  if (w == 0) {
    // the critical chain: factor block b as soon as its last update (from panel b - 1) is in
#pragma unroll 1
    for (int b = 0; b < nbk; ++b) {
      POTRF_TRACE(2 * b);
      if (b > 0) bar_sync(kDiag, 256);
      POTRF_TRACE(2 * b + 1);
      bad |= potrf16_warp(S, X, b * SB, colb);
      __syncwarp();
      bar_arrive(kPanel, 256);
    }
  } else {
    // warp 4 shares warp 0's SM sub-partition: it only takes part in the barriers (-2 % measured)
    const int wi = w == 4 ? 1000 : (w < 4 ? w - 1 : w - 2), nw = 6;
#pragma unroll 1
    for (int b = 0; b < nbk; ++b) {
      bar_sync(kPanel, 256);  // L_bb, X_bb in; also: every worker is done with iteration b - 1
      const int c0 = b * SB, r0 = c0 + SB, R = (nbk - 1 - b) * SB;
      if (R > 0) {
        // (2) T = A_{>b,b} X_bb^T
        for (int tt = wi; tt < (R / 8) * 2; tt += nw) {
          const int tm = tt >> 1, tn = tt & 1;
          double c0v = 0.0, c1v = 0.0;
#pragma unroll
          for (int k0 = 0; k0 < SB; k0 += 4)
            dmma(c0v, c1v, S[r0 + tm * 8 + lr][c0 + k0 + lk], X[c0 + tn * 8 + lr][c0 + k0 + lk]);
          T[tm * 8 + lr][tn * 8 + 2 * lk] = c0v;
          T[tm * 8 + lr][tn * 8 + 2 * lk + 1] = c1v;
        }
        bar_sync(kWork, 224);
        for (int e = tid - 32; e < R * SB; e += 224) S[r0 + e / SB][c0 + e % SB] = T[e / SB][e % SB];
        // (3a) the next diagonal block first (8 x 8 tiles (0,0), (1,0), (1,1)), then release warp 0
        if (wi < 3) {
          const int mb = wi > 0, nb_ = wi > 1;
          double c0v = 0.0, c1v = 0.0;
#pragma unroll
          for (int k0 = 0; k0 < SB; k0 += 4) dmma(c0v, c1v, T[mb * 8 + lr][k0 + lk], T[nb_ * 8 + lr][k0 + lk]);
          const int rr = r0 + mb * 8 + lr, cc = r0 + nb_ * 8 + 2 * lk;
          if (cc <= rr) S[rr][cc] -= c0v;
          if (cc + 1 <= rr) S[rr][cc + 1] -= c1v;
        }
        bar_sync(kWork, 224);
        bar_arrive(kDiag, 256);
        // (3b) the rest of the trailing lower triangle, while warp 0 factors block b + 1
        const int MBk = R / 8;
        for (int blk = 3 + wi; blk < MBk * (MBk + 1) / 2; blk += nw) {
          int mb = 0;
          while ((mb + 1) * (mb + 2) / 2 <= blk) ++mb;
          const int nb_ = blk - mb * (mb + 1) / 2;
          double c0v = 0.0, c1v = 0.0;
#pragma unroll
          for (int k0 = 0; k0 < SB; k0 += 4) dmma(c0v, c1v, T[mb * 8 + lr][k0 + lk], T[nb_ * 8 + lr][k0 + lk]);
          const int rr = r0 + mb * 8 + lr, cc = r0 + nb_ * 8 + 2 * lk;
          if (cc <= rr) S[rr][cc] -= c0v;
          if (cc + 1 <= rr) S[rr][cc + 1] -= c1v;
        }
      }
      // (4) row block b of X = L^{-1}: X_{b,<b} = -X_bb M_b, M_b = L_{b,<b} X_{<b,<b} (formed in the
      // previous iteration); then M_{b+1} = L_{b+1,<=b} X_{<=b,<=b}, so that after the last
      // diagonal block only one 16-deep product is left
      if (b > 0) smem_gemm(&X[c0][0], LDR, &X[c0][c0], LDR, &M[0][0], NB + 1, SB, c0, SB, -1.0, wi, nw);
      if (R > 0) {
        bar_sync(kWork, 224);
        smem_gemm(&M[0][0], NB + 1, &S[r0][0], LDR, &X[0][0], LDR, SB, r0, r0, 1.0, wi, nw);
      }
    }
  }
  POTRF_TRACE(8);
  __syncthreads();
  POTRF_TRACE(9);
  return bad;
}

__global__ void __launch_bounds__(256) k_trtri_blocks(int n, const double* A, int lda, double* Linv) {
  extern __shared__ __align__(16) double dsm[];
  double(*S)[LDR] = reinterpret_cast<double(*)[LDR]>(dsm);
  double(*X)[LDR] = reinterpret_cast<double(*)[LDR]>(dsm + NB * LDR);
  const int j0 = blockIdx.x * NB, jb = min(NB, n - j0);
  // inverse of an existing factor: reuse potrf_trtri on L L^T? No — invert L directly, row by row.
  for (int e = threadIdx.x; e < NB * NB; e += 256) {
    const int r = e >> 6, c = e & 63;
    S[r][c] = (r < jb && c <= r) ? A[(int64_t)(j0 + r) * lda + j0 + c] : (r == c ? 1.0 : 0.0);
    X[r][c] = (r == c) ? 1.0 : 0.0;
  }
  __syncthreads();
  const int tid = threadIdx.x, tr = tid >> 4, tc = tid & 15;
  for (int t = 0; t < jb; ++t) {
    const double inv = 1.0 / S[t][t];
    if (tid <= t) X[t][tid] *= inv;
    __syncthreads();
    for (int r = t + 1 + tr; r < jb; r += 16) {
      const double lrt = S[r][t];
      for (int j = tc; j <= t; j += 16) X[r][j] -= lrt * X[t][j];
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < NB * NB; e += 256) {
    const int r = e >> 6, c = e & 63;
    Linv[(int64_t)blockIdx.x * NB * NB + e] = (r < jb && c <= r) ? X[r][c] : 0.0;
  }
}


// 64 x 64 tile A[row0 + r][col0 + c] -> T[r][c] (zero for r >= nr or c >= nc), all 16 loads of a
// thread in flight at once (clamped addresses, masked values; L2 loads: k_inv_diag stores blocks of
// L^{-1} into the upper triangle, on cache lines it may already hold from reading L)
__device__ __forceinline__ void load_tile(double (*T)[LDS], const double* A, int lda, int row0, int col0, int nr,
                                          int nc) {
  const int tid = threadIdx.x;
  double v[16];
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    const int e = tid + 256 * m, r = e >> 6, c = e & 63;
    const int rr = r < nr ? r : (nr > 0 ? nr - 1 : 0), cc = c < nc ? c : (nc > 0 ? nc - 1 : 0);
    v[m] = (nr > 0 && nc > 0) ? __ldcg(A + (int64_t)(row0 + rr) * lda + col0 + cc) : 0.0;
  }
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    const int e = tid + 256 * m, r = e >> 6, c = e & 63;
    T[r][c] = (r < nr && c < nc) ? v[m] : 0.0;
  }
}


// ---- flags, mbarriers, bulk copies -----------------------------------------------------------
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// acc[64x64] += X[64x64] * Y[64x64]^T from two smem tiles (row-major, LDS); 8 warps of 16x32: thread
// (warp w, lane) holds entries (wr + 8a + lane/4, wc + 8b + 2 (lane%4) + h), wr = 16 (w/2), wc = 32 (w%2)
__device__ __forceinline__ void tile_acc_xyT(const double (*Xs)[LDS], const double (*Ys)[LDS], double acc[2][4][2]) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int wr = (w >> 1) * 16, wc = (w & 1) * 32;
  const int lr = lane >> 2, lk = lane & 3;
#pragma unroll 4
  for (int k0 = 0; k0 < NB; k0 += 4) {
    double af[2], bf[4];
#pragma unroll
    for (int a = 0; a < 2; ++a) af[a] = Xs[wr + a * 8 + lr][k0 + lk];
#pragma unroll
    for (int b = 0; b < 4; ++b) bf[b] = Ys[wc + b * 8 + lr][k0 + lk];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
  }
}

__device__ __forceinline__ int tri(int i, int j) { return i * (i + 1) / 2 + j; }

// ---- the tile-DAG factorisation -------------------------------------------------------------
// A: the SPD matrix, row-major (lda), lower triangle read (once; never written by this kernel).
// Lt: tile-major packed L (tile_off), LinvP: Linv_j padded [nt][NB][LDS], Linv: the same unpadded
// [nt][NB][NB] (k_trsv_wave, k_inv_diag). b (optional): right-hand side; ybuf [nt NB] <- L^{-1} b
// (zero padded); with nt == 1 and x != null, x <- (L L^T)^{-1} b directly. flags [nt (nt+1)/2].
//
// Tasks, column-major: column j holds D_j, then (i, j) for i >= j + 2. D_j computes the
// sub-diagonal tile (j, j-1) AND the diagonal tile (j, j): it accumulates both over k < j - 1
// while column j - 1 is still being factored, then, as soon as Linv_{j-1} is published, forms
// L_{j,j-1}, publishes it, applies its last update L_{j,j-1} L_{j,j-1}^T from shared memory and
// factors. The column-to-column critical path is thus potrf, one bulk load of Linv, two 64^3 DMMA
// products, potrf, ... with no flag round trip for the sub-diagonal tile.
constexpr int kDagSmemDoubles = 5 * TS + 3 * NB;  // 2 stages x 2 tiles, Linv_{j-1}, 2 stages x y_k, y_{j-1}

// Task order (topological, with a lookahead of one column for the diagonal tasks): group 0 =
// [D_0, D_1]; group g >= 1 = [(i, g-1) for i = g+1 .. nt-1, then D_{g+1}]. D_j is taken as soon as
// column j-2 is, so its long accumulation runs alongside column j-1 instead of after it.
__device__ __forceinline__ int dag_off_tasks(int nt, int g) { return g == 0 ? 0 : max(0, nt - g - 1); }
__device__ __forceinline__ int dag_group_tasks(int nt, int g) {
  return g == 0 ? min(nt, 2) : dag_off_tasks(nt, g) + (g + 1 < nt ? 1 : 0);
}

// fragment loads of A (row-major) for tile rows i0.., columns j0..: identity beyond n on the
// diagonal, zero in the strict upper triangle
__device__ __forceinline__ void load_a_frag(const double* __restrict__ A, int lda, int n, int i0, int j0,
                                            double (&cv)[2][4][2]) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int wr = (w >> 1) * 16, wc = (w & 1) * 32, lr = lane >> 2, lk = lane & 3;
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int bb = 0; bb < 4; ++bb)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = i0 + wr + a * 8 + lr, c = j0 + wc + bb * 8 + 2 * lk + h;
        cv[a][bb][h] = (r < n && c <= r) ? __ldg(A + (int64_t)r * lda + c) : (r == c ? 1.0 : 0.0);
      }
}

// fragments -> smem tile (LDS rows)
__device__ __forceinline__ void frag_to_smem(double* T, const double (&v)[2][4][2]) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int wr = (w >> 1) * 16, wc = (w & 1) * 32, lr = lane >> 2, lk = lane & 3;
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int bb = 0; bb < 4; ++bb)
      *reinterpret_cast<double2*>(T + (wr + a * 8 + lr) * LDS + wc + bb * 8 + 2 * lk) = make_double2(v[a][bb][0], v[a][bb][1]);
}

__device__ __forceinline__ void frag_zero(double (&v)[2][4][2]) {
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int bb = 0; bb < 4; ++bb) v[a][bb][0] = v[a][bb][1] = 0.0;
}

__global__ void __launch_bounds__(256, 1) k_chol_dag(int n, int nt, const double* __restrict__ A, int lda, double* Lt,
                                                     double* LinvP, double* Linv, const double* __restrict__ b,
                                                     double* ybuf, double* x, int* info, int* flags, int epoch,
                                                     int* next_task) {
  extern __shared__ __align__(16) double dsm[];
  __shared__ __align__(8) uint64_t bars[3];
  __shared__ double bv[NB], yv[NB], part[4][NB];
  __shared__ int task_s;
  double* const TA[2] = {dsm, dsm + 2 * TS};
  double* const TB[2] = {dsm + TS, dsm + 3 * TS};
  double* const LI = dsm + 4 * TS;
  double* const YB[2] = {dsm + 5 * TS, dsm + 5 * TS + NB};
  double* const YL = dsm + 5 * TS + 2 * NB;
  const int tid = threadIdx.x;
  const int rq = tid >> 2, q4 = tid & 3;  // row-per-4-threads mapping (forward solve pieces)
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_init(&bars[2], 1);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  unsigned ph[2] = {0u, 0u}, phl = 0u;  // mbarrier parities (identical in every thread)
  int ntask = 0;
  for (int g = 0; g < nt; ++g) ntask += dag_group_tasks(nt, g);
  auto publish = [&](int fi) {  // every thread's global writes of the task (ordered by the CTA
    __syncthreads();             // barrier, then made gpu-visible by thread 0's fence), then its flag
    if (tid == 0) {
      __threadfence();
      asm volatile("fence.proxy.async;" ::: "memory");
      st_release(flags + fi, epoch);
    }
  };
  auto wait_flag = [&](int fi) {
    while (ld_acquire(flags + fi) != epoch) __nanosleep(64);
  };
  // next_task == nullptr: a single tile (n <= 64) in a single CTA, launched plainly: no task
  // counter, and info is cleared here instead of by a memset before the launch
  if (!next_task && tid == 0) *info = 0;
  int g = 0, grp0 = 0;
  for (int it = 0;; ++it) {
    // dynamic dealing in the topological order: a CTA takes the next task when it is free (the
    // tasks it waits on were all taken before it, by running CTAs, so this cannot deadlock)
    if (tid == 0) task_s = next_task ? atomicAdd(next_task, 1) : it;
    __syncthreads();
    const int t = task_s;
    __syncthreads();
    if (t >= ntask) break;
    while (t >= grp0 + dag_group_tasks(nt, g)) {
      grp0 += dag_group_tasks(nt, g);
      ++g;
    }
    const int u = t - grp0;
    const bool diag = g == 0 || u >= dag_off_tasks(nt, g);
    // diagonal task D_j: rows i = j, partner tile row m = j - 1 (the sub-diagonal tile (j, m));
    // off-diagonal task: tile (i, j), partner tile row m = j
    const int j = diag ? (g == 0 ? u : g + 1) : g - 1;
    const int i = diag ? j : g + 1 + u;
    const int m = diag ? j - 1 : j;
    const int kend = diag ? j - 1 : j;  // k-steps of the accumulation (k < kend)
    const bool want_y = diag && b != nullptr;
    double acc[2][4][2], acc2[2][4][2];  // (i, m) tile; diagonal task: also the (j, j) tile
    frag_zero(acc);
    frag_zero(acc2);
    double xs = 0.0;  // diagonal task: row rq of sum_k L_jk y_k over columns q4 + 4 s
    const unsigned bytes = 2u * TS * 8u + (want_y ? NB * 8u : 0u);
    auto ready = [&](int k) {
      return ld_acquire(flags + tri(i, k)) == epoch && ld_acquire(flags + tri(m, k)) == epoch &&
             (!want_y || ld_acquire(flags + tri(k, k)) == epoch);
    };
    auto issue = [&](int k) {
      const int s = k & 1;
      asm volatile("fence.proxy.async;" ::: "memory");  // generic accesses before the async copy
      mbar_expect(&bars[s], bytes);
      bulk_g2s(TA[s], Lt + tile_off(i, k), TS * 8u, &bars[s]);
      bulk_g2s(TB[s], Lt + tile_off(m, k), TS * 8u, &bars[s]);
      if (want_y) bulk_g2s(YB[s], ybuf + (int64_t)k * NB, NB * 8u, &bars[s]);
    };
    int issued = 0;  // thread 0: steps issued so far
    for (int k = 0; k < kend; ++k) {
      const int s = k & 1;
      if (tid == 0) {
        if (issued == k) {
          while (!ready(k)) __nanosleep(64);
          issue(k);
          ++issued;
        }
        if (issued == k + 1 && k + 1 < kend && ready(k + 1)) {  // lookahead: only if already published
          issue(k + 1);
          ++issued;
        }
      }
      mbar_wait(&bars[s], ph[s]);
      ph[s] ^= 1u;
      const double(*ta)[LDS] = reinterpret_cast<const double(*)[LDS]>(TA[s]);
      const double(*tb)[LDS] = reinterpret_cast<const double(*)[LDS]>(TB[s]);
      tile_acc_xyT(ta, tb, acc);
      if (diag) {
        tile_acc_xyT(ta, ta, acc2);
        if (want_y) {
#pragma unroll
          for (int s4 = 0; s4 < 16; ++s4) xs = fma(ta[rq][q4 + 4 * s4], YB[s][q4 + 4 * s4], xs);
        }
      }
      __syncthreads();  // stage s is free for step k + 2
    }
    if (m >= 0) {
      // L_im = (A_im - acc) Linv_m^T once the diagonal task of column m has published Linv_m (and y_m)
      if (tid == 0) {
        wait_flag(tri(m, m));
        asm volatile("fence.proxy.async;" ::: "memory");
        mbar_expect(&bars[2], TS * 8u + (want_y ? NB * 8u : 0u));
        bulk_g2s(LI, LinvP + (int64_t)m * TS, TS * 8u, &bars[2]);
        if (want_y) bulk_g2s(YL, ybuf + (int64_t)m * NB, NB * 8u, &bars[2]);
      }
      double cv[2][4][2];
      load_a_frag(A, lda, n, i * NB, m * NB, cv);
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int bb = 0; bb < 4; ++bb)
#pragma unroll
          for (int h = 0; h < 2; ++h) cv[a][bb][h] -= acc[a][bb][h];
      frag_to_smem(TA[0], cv);  // the stages are free: the loop ended with a CTA barrier (or did not run)
      __syncthreads();
      mbar_wait(&bars[2], phl);
      phl ^= 1u;
      frag_zero(acc);
      tile_acc_xyT(reinterpret_cast<const double(*)[LDS]>(TA[0]), reinterpret_cast<const double(*)[LDS]>(LI), acc);
      frag_to_smem(Lt + tile_off(i, m), acc);
      if (diag) frag_to_smem(TB[0], acc);  // L_{j,j-1} for the diagonal tile's last update
      publish(tri(i, m));
      if (diag) {  // the last update of the diagonal tile: acc2 += L_jm L_jm^T, xs += L_jm y_m
        const double(*tl)[LDS] = reinterpret_cast<const double(*)[LDS]>(TB[0]);
        tile_acc_xyT(tl, tl, acc2);
        if (want_y) {
#pragma unroll
          for (int s4 = 0; s4 < 16; ++s4) xs = fma(tl[rq][q4 + 4 * s4], YL[q4 + 4 * s4], xs);
        }
        __syncthreads();  // TB[0] is overwritten by the factorisation's workspace
      }
    }
    if (!diag) continue;
    // the diagonal tile: C = A_jj - acc2, L_jj = chol(C), Linv_j, y_j
    double(*S)[LDR] = reinterpret_cast<double(*)[LDR]>(dsm);
    double(*X)[LDR] = reinterpret_cast<double(*)[LDR]>(dsm + NB * LDR);
    const int j0 = j * NB, jb = min(NB, n - j0);
    {
      double cv[2][4][2];
      load_a_frag(A, lda, n, j0, j0, cv);
      const int lane = tid & 31, w = tid >> 5;
      const int wr = (w >> 1) * 16, wc = (w & 1) * 32, lr = lane >> 2, lk = lane & 3;
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int bb = 0; bb < 4; ++bb)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int r = wr + a * 8 + lr, c = wc + bb * 8 + 2 * lk + h;
            S[r][c] = c <= r ? cv[a][bb][h] - acc2[a][bb][h] : 0.0;
          }
    }
    if (want_y) {
      xs += __shfl_xor_sync(0xffffffffu, xs, 1);
      xs += __shfl_xor_sync(0xffffffffu, xs, 2);
      if (q4 == 0) bv[rq] = rq < jb ? __ldg(b + j0 + rq) - xs : 0.0;
    }
    __syncthreads();
    const bool bad = potrf_core(jb, dsm);  // ends with a CTA barrier
    if (tid == 0 && bad) atomicCAS(info, 0, j0 + 1);
    // what the next column's tasks wait for first: Linv_j (padded, for their trsm) and y_j
    for (int e = tid; e < NB * NB / 2; e += 256) {
      const int r = e >> 5, c = 2 * (e & 31);
      const double x0 = (r < jb && c <= r) ? X[r][c] : 0.0, x1 = (r < jb && c + 1 <= r) ? X[r][c + 1] : 0.0;
      *reinterpret_cast<double2*>(LinvP + (int64_t)j * TS + r * LDS + c) = make_double2(x0, x1);
    }
    if (want_y) {  // y_j = Linv_j (b_j - sum_k L_jk y_k)
      double sacc = 0.0;
      for (int tt = q4; tt <= rq && tt < jb; tt += 4) sacc = fma(X[rq][tt], bv[tt], sacc);
      sacc += __shfl_xor_sync(0xffffffffu, sacc, 1);
      sacc += __shfl_xor_sync(0xffffffffu, sacc, 2);
      if (q4 == 0) {
        const double yj = rq < jb ? sacc : 0.0;
        ybuf[j0 + rq] = yj;
        yv[rq] = yj;
      }
      if (nt == 1 && x) {  // single tile: the backward solve x = Linv^T y here as well
        __syncthreads();
        const int c = tid & 63, g = tid >> 6;
        double o = 0.0;
        for (int tt = c + (g - c % 4 + 4) % 4; tt < jb; tt += 4) o = fma(X[tt][c], yv[tt], o);  // rows tt >= c
        part[g][c] = o;
        __syncthreads();
        if (tid < jb) x[tid] = (part[0][tid] + part[1][tid]) + (part[2][tid] + part[3][tid]);
      }
    }
    publish(tri(j, j));
    // then what only the kernels after this one read: L_jj (tile-major) and the unpadded Linv_j
    double* out = Lt + tile_off(j, j);
    for (int e = tid; e < NB * NB / 2; e += 256) {
      const int r = e >> 5, c = 2 * (e & 31);
      const bool in0 = r < jb && c <= r, in1 = r < jb && c + 1 <= r;
      *reinterpret_cast<double2*>(out + r * LDS + c) = make_double2(in0 ? S[r][c] : 0.0, in1 ? S[r][c + 1] : 0.0);
      *reinterpret_cast<double2*>(Linv + (int64_t)j * NB * NB + r * NB + c) =
          make_double2(in0 ? X[r][c] : 0.0, in1 ? X[r][c + 1] : 0.0);
    }
    __syncthreads();  // S / X (the stage buffers) are reused by the next task
  }
}

// tile-major L -> the lower triangle of the row-major A (lda); row r per CTA
__global__ void __launch_bounds__(256) k_untile(int n, const double* __restrict__ Lt, double* A, int lda) {
  const int r = blockIdx.x, ti = r / NB, rr = r % NB;
  for (int c = threadIdx.x; c <= r; c += 256) A[(int64_t)r * lda + c] = Lt[tile_off(ti, c / NB) + rr * LDS + c % NB];
}

// Backward solve L^T z = y on the tile-major factor of k_chol_dag (one CTA per 64-block b, blocks
// solved in descending order): z_b = Linv_b^T (y_b - L_{b+1,b}^T z_{b+1} - sum_{j>=b+2} L_jb^T z_j).
// Off the critical chain, each CTA first forms W_b = Linv_b^T L_{b+1,b}^T (DMMA) and folds in the
// blocks j >= b + 2 as their flags are published, giving w_b = Linv_b^T (y_b - sum_{j>=b+2} ...);
// the chain from block b + 1 to block b is then one 64 x 64 product: z_b = w_b - W_b z_{b+1}.
// Contraction orders are fixed (deterministic). ybuf [nt NB] (zero padded), x [n] out.
__global__ void __launch_bounds__(256, 1) k_trsv_bwd_tiles(int n, const double* __restrict__ Lt,
                                                           const double* __restrict__ LinvP,
                                                           const double* __restrict__ ybuf, double* x, int* flags,
                                                           int epoch) {
  extern __shared__ __align__(16) double dsm[];
  double(*Xs)[LDS] = reinterpret_cast<double(*)[LDS]>(dsm);            // Linv_b^T
  double(*Ys)[LDS] = reinterpret_cast<double(*)[LDS]>(dsm + TS);       // L_{b+1,b}
  double(*Ws)[LDR] = reinterpret_cast<double(*)[LDR]>(dsm + 2 * TS);   // W_b
  __shared__ double part[4][NB], wv[NB], zn[NB];
  const int nblk = (n + NB - 1) / NB;
  const int b = nblk - 1 - blockIdx.x;
  const int b0 = b * NB, bb = min(NB, n - b0);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const bool has_next = b + 1 < nblk;
  for (int e = tid; e < NB * NB; e += 256) {
    const int r = e >> 6, c = e & 63;
    Xs[c][r] = LinvP[(int64_t)b * TS + r * LDS + c];  // transposed
    if (has_next) Ys[r][c] = Lt[tile_off(b + 1, b) + r * LDS + c];
  }
  __syncthreads();
  if (has_next) {  // W_b[r][c] = sum_t Linv_b[t][r] L_{b+1,b}[c][t]
    double acc[2][4][2];
    frag_zero(acc);
    tile_acc_xyT(Xs, Ys, acc);
    const int wr = (w >> 1) * 16, wc = (w & 1) * 32, lr = lane >> 2, lk = lane & 3;
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b2 = 0; b2 < 4; ++b2)
#pragma unroll
        for (int h = 0; h < 2; ++h) Ws[wr + a * 8 + lr][wc + b2 * 8 + 2 * lk + h] = acc[a][b2][h];
  }
  // fold the blocks j >= b + 2 (descending, as they are published): thread -> column c of block b,
  // rows g + 4k of block j
  const int c = tid & 63, g = tid >> 6;
  double s = 0.0;
  for (int j = nblk - 1; j >= b + 2; --j) {
    const int j0 = j * NB, jbb = min(NB, n - j0);
    double Lr[16];
    const double* Lj = Lt + tile_off(j, b);
#pragma unroll
    for (int k = 0; k < 16; ++k) Lr[k] = Lj[(g + 4 * k) * LDS + c];  // zero beyond n (padded tiles)
    if (tid == 0)
      while (ld_acquire(flags + j) != epoch) __nanosleep(32);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int t = g + 4 * k;
      if (t < jbb) s = fma(Lr[k], __ldcg(x + j0 + t), s);
    }
  }
  part[g][c] = s;
  __syncthreads();
  if (tid < NB) wv[tid] = ybuf[b0 + tid] - ((part[0][tid] + part[1][tid]) + (part[2][tid] + part[3][tid]));
  __syncthreads();
  {  // w_b = Linv_b^T v: thread (c, g) sums rows t = g + 4k of Linv_b (Xs[c][t] = Linv_b[t][c])
    double o = 0.0;
#pragma unroll
    for (int k = 0; k < 16; ++k) o = fma(Xs[c][g + 4 * k], wv[g + 4 * k], o);
    part[g][c] = o;
  }
  __syncthreads();
  if (tid < NB) wv[tid] = (part[0][tid] + part[1][tid]) + (part[2][tid] + part[3][tid]);
  // the chain: z_b = w_b - W_b z_{b+1}
  if (has_next) {
    const int bn0 = b0 + NB, bnb = min(NB, n - bn0);
    if (tid == 0)
      while (ld_acquire(flags + b + 1) != epoch) __nanosleep(32);
    __syncthreads();
    if (tid < NB) zn[tid] = tid < bnb ? __ldcg(x + bn0 + tid) : 0.0;
    __syncthreads();
    const int r = tid >> 2, q4 = tid & 3;
    double o = 0.0;
#pragma unroll
    for (int k = 0; k < 16; ++k) o = fma(Ws[r][q4 + 4 * k], zn[q4 + 4 * k], o);
    o += __shfl_xor_sync(0xffffffffu, o, 1);
    o += __shfl_xor_sync(0xffffffffu, o, 2);
    if (q4 == 0 && r < bb) x[b0 + r] = wv[r] - o;
  } else {
    __syncthreads();
    if (tid < bb) x[b0 + tid] = wv[tid];
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    st_release(flags + b, epoch);
  }
}
// ---- triangular solve wavefront ------------------------------------------------------------
// forward (upper = 0): y_b = Linv_b (x_b - sum_{j<b} L[b, j] y_j), block b = blockIdx.x.
// backward (upper = 1): z_b = Linv_b^T (y_b - sum_{j>b} L[j, b]^T z_j), blocks in reverse order.
// The right-hand side is read from xin (which may be x) and the result written to x (row-major L,
// lda). The L block of the next step is loaded into registers before the flag wait; the
// contraction order over blocks and within a block is fixed (deterministic).
__global__ void __launch_bounds__(256) k_trsv_wave(int n, const double* L, int lda, const double* Linv,
                                                   const double* xin, double* x, int* flags, int epoch, int upper) {
  __shared__ double Li[NB][LDR];
  __shared__ double part[4][NB];
  __shared__ double v[NB];
  const int nblk = (n + NB - 1) / NB;
  const int b = upper ? nblk - 1 - blockIdx.x : blockIdx.x;
  const int b0 = b * NB, bb = min(NB, n - b0);
  const int tid = threadIdx.x;
  for (int e = tid; e < NB * NB; e += 256) Li[e >> 6][e & 63] = Linv[(int64_t)b * NB * NB + e];
  // forward: thread -> row r = tid >> 2 of block b, columns q4 + 4k;
  // backward: thread -> column c = tid & 63 of block b, rows g + 4k of block j
  const int r = tid >> 2, q4 = tid & 3, c = tid & 63, g = tid >> 6;
  double acc = 0.0;
  double Lr[16];
  auto load_block = [&](int j) {
    const int j0 = j * NB, jbb = min(NB, n - j0);
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      if (!upper) {
        const int cc = q4 + 4 * k;
        Lr[k] = (r < bb && cc < jbb) ? L[(int64_t)(b0 + r) * lda + j0 + cc] : 0.0;
      } else {
        const int rr = g + 4 * k;
        Lr[k] = (c < bb && rr < jbb) ? L[(int64_t)(j0 + rr) * lda + b0 + c] : 0.0;
      }
    }
  };
  const int steps = (int)blockIdx.x;
  if (steps > 0) load_block(upper ? nblk - 1 : 0);
  for (int step = 0; step < steps; ++step) {
    const int j = upper ? nblk - 1 - step : step;
    const int j0 = j * NB, jbb = min(NB, n - j0);
    if (tid == 0)
      while (ld_acquire(flags + j) != epoch) __nanosleep(32);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int t = upper ? g + 4 * k : q4 + 4 * k;
      if (t < jbb) acc = fma(Lr[k], __ldcg(x + j0 + t), acc);
    }
    if (step + 1 < steps) load_block(upper ? j - 1 : j + 1);
  }
  if (!upper) {
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    acc += __shfl_xor_sync(0xffffffffu, acc, 2);
    if (q4 == 0) part[0][r] = acc;
    __syncthreads();
    if (tid < NB) v[tid] = tid < bb ? xin[b0 + tid] - part[0][tid] : 0.0;
  } else {
    part[g][c] = acc;
    __syncthreads();
    if (tid < NB) {
      const double s = (part[0][tid] + part[1][tid]) + (part[2][tid] + part[3][tid]);
      v[tid] = tid < bb ? xin[b0 + tid] - s : 0.0;
    }
  }
  __syncthreads();
  // apply Linv_b (forward) or Linv_b^T (backward): 4 threads per output
  double o = 0.0;
  if (!upper) {
    for (int t = q4; t <= r; t += 4) o = fma(Li[r][t], v[t], o);
    o += __shfl_xor_sync(0xffffffffu, o, 1);
    o += __shfl_xor_sync(0xffffffffu, o, 2);
    if (q4 == 0 && r < bb) x[b0 + r] = o;
  } else {
    for (int t = c + (g - c % 4 + 4) % 4; t < NB; t += 4) o = fma(Li[t][c], v[t], o);  // rows t >= c, t%4 == g
    part[g][c] = o;
    __syncthreads();
    if (tid < bb) x[b0 + tid] = (part[0][tid] + part[1][tid]) + (part[2][tid] + part[3][tid]);
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) st_release(flags + b, epoch);
}

// ---- diag((L L^T)^{-1}) for standard errors ---------------------
// CTA J owns block column J of W = L^{-1}: W_JJ = Linv[J]; for I = J+1 .. : W_IJ = -Linv[I]
// sum_{K=J}^{I-1} L_IK W_KJ (DMMA 64x64 tiles). The finished blocks W_KJ are kept, transposed, in
// the (unused) strict upper triangle of A at block (J, K); columns of A^{-1} = W^T W have
// diag_c = sum_r W_rc^2, summed in a fixed order (rows of a tile by shuffles, warps via smem, I
// ascending). Block columns are independent; the first one carries the longest chain.
__global__ void __launch_bounds__(256) k_inv_diag(int n, double* A, int lda, const double* Linv, double* se) {
  extern __shared__ __align__(16) double dsm[];
  double(*Xs)[LDS] = reinterpret_cast<double(*)[LDS]>(dsm);
  double(*Ys)[LDS] = reinterpret_cast<double(*)[LDS]>(dsm + NB * LDS);
  __shared__ double colw[4][NB];
  const int nblk = (n + NB - 1) / NB;
  const int J = blockIdx.x, j0 = J * NB, jb = min(NB, n - j0);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int wr = (w >> 1) * 16, wc = (w & 1) * 32, lr = lane >> 2, lk = lane & 3;
  double csum[4][2];  // this thread's 8 columns: sum of squares over rows (its lr == 0 lanes after shuffles)
#pragma unroll
  for (int b = 0; b < 4; ++b) csum[b][0] = csum[b][1] = 0.0;
  auto add_squares = [&](const double (&v)[2][4][2]) {
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        double t = v[0][b][h] * v[0][b][h] + v[1][b][h] * v[1][b][h];
        t += __shfl_xor_sync(0xffffffffu, t, 4);
        t += __shfl_xor_sync(0xffffffffu, t, 8);
        t += __shfl_xor_sync(0xffffffffu, t, 16);
        csum[b][h] += t;
      }
  };
  // W_JJ = Linv[J] (zero beyond jb)
  {
    double v[2][4][2];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b)
#pragma unroll
        for (int h = 0; h < 2; ++h)
          v[a][b][h] = (wr + a * 8 + lr < jb && wc + b * 8 + 2 * lk + h < jb)
                           ? __ldg(Linv + (size_t)J * NB * NB + (wr + a * 8 + lr) * NB + wc + b * 8 + 2 * lk + h)
                           : 0.0;
    add_squares(v);
  }
  for (int I = J + 1; I < nblk; ++I) {
    const int i0 = I * NB, ib = min(NB, n - i0);
    double acc[2][4][2];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    for (int Kb = J; Kb < I; ++Kb) {
      const int k0 = Kb * NB, kb = min(NB, n - k0);
      __syncthreads();
      load_tile(Xs, A, lda, i0, k0, ib, kb);  // L_IK
      if (Kb == J) {                          // W_JJ^T from Linv[J]
        for (int e = tid; e < NB * NB; e += 256) {
          const int r = e >> 6, c = e & 63;
          Ys[c][r] = (r < jb && c < jb) ? __ldg(Linv + (size_t)J * NB * NB + e) : 0.0;
        }
      } else {
        load_tile(Ys, A, lda, j0, k0, jb, kb);  // W_KJ^T, stored transposed at block (J, K)
      }
      __syncthreads();
      tile_acc_xyT(Xs, Ys, acc);
    }
    // W_IJ = -Linv[I] T, T = acc: Xs = Linv[I], Ys = T^T
    __syncthreads();
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b)
#pragma unroll
        for (int h = 0; h < 2; ++h) Ys[wc + b * 8 + 2 * lk + h][wr + a * 8 + lr] = acc[a][b][h];
    for (int e = tid; e < NB * NB; e += 256)
      Xs[e >> 6][e & 63] = ((e >> 6) < ib && (e & 63) < ib) ? __ldg(Linv + (size_t)I * NB * NB + e) : 0.0;
    __syncthreads();
    double wv[2][4][2];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) wv[a][b][0] = wv[a][b][1] = 0.0;
    tile_acc_xyT(Xs, Ys, wv);
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = wr + a * 8 + lr, c = wc + b * 8 + 2 * lk + h;
          wv[a][b][h] = (r < ib && c < jb) ? -wv[a][b][h] : 0.0;
          if (r < ib && c < jb) A[(int64_t)(j0 + c) * lda + i0 + r] = wv[a][b][h];  // W_IJ^T at block (J, I)
        }
    add_squares(wv);
  }
  // combine the four row-warps of each column in a fixed order
  if (lr == 0) {
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) colw[w >> 1][wc + b * 8 + 2 * lk + h] = csum[b][h];
  }
  __syncthreads();
  if (tid < jb) se[j0 + tid] = sqrt(((colw[0][tid] + colw[1][tid]) + colw[2][tid]) + colw[3][tid]);
}

}  // namespace

// Per-workspace factorisation state (one per library workspace, i.e. per device and stream).
struct CholCtx {
  int sms = 0, occ = 0;
  double* Lt = nullptr;  // tile-major L [nt (nt+1)/2][NB][LDS]
  size_t cap_lt = 0;     // tiles
  double* LinvP = nullptr;  // [nt][NB][LDS]
  double* Linv = nullptr;   // [nt][NB][NB]
  double* ybuf = nullptr;   // [nt][NB]
  int cap_nt = 0;
  int* dflags = nullptr;  // k_chol_dag tile flags [nt (nt+1)/2], then its task counter
  int depoch = 0;
  int* flags = nullptr;  // k_trsv_wave block flags [nt]
  int epoch = 0;
  const double* factor = nullptr;  // row-major matrix holding the factor whose Linv blocks are current
  int factor_n = 0;
};

namespace {

constexpr size_t kDyn = 2 * NB * LDS * sizeof(double);
constexpr size_t kDynR = 2 * NB * LDR * sizeof(double);
constexpr size_t kDagSmem = kDagSmemDoubles * sizeof(double);
constexpr size_t kBwdSmem = (2 * TS + NB * LDR) * sizeof(double);

void set_attrs() {
  static uint64_t attr_mask = 0;
  set_once_per_device(attr_mask, [] {
    cudaFuncSetAttribute(k_trtri_blocks, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDynR);
    cudaFuncSetAttribute(k_inv_diag, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDyn);
    cudaFuncSetAttribute(k_trsv_bwd_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBwdSmem);
    return cudaFuncSetAttribute(k_chol_dag, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDagSmem);
  });
}

bool ensure_work(CholCtx& c, int n) {
  set_attrs();
  const int nt = (n + NB - 1) / NB;
  const size_t ntri = (size_t)nt * (nt + 1) / 2;
  if (!c.sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&c.sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c.occ, k_chol_dag, 256, kDagSmem) != cudaSuccess || c.occ < 1)
      return false;
  }
  if (ntri > c.cap_lt) {
    cudaFree(c.Lt);
    cudaFree(c.dflags);
    c.cap_lt = 0;
    if (cudaMalloc(&c.Lt, ntri * TS * sizeof(double)) != cudaSuccess) return false;
    if (cudaMalloc(&c.dflags, (ntri + 1) * sizeof(int)) != cudaSuccess) return false;
    cudaMemset(c.dflags, 0, (ntri + 1) * sizeof(int));
    c.depoch = 0;
    c.cap_lt = ntri;
  }
  if (nt > c.cap_nt) {
    cudaFree(c.LinvP);
    cudaFree(c.Linv);
    cudaFree(c.ybuf);
    cudaFree(c.flags);
    c.cap_nt = 0;
    if (cudaMalloc(&c.LinvP, (size_t)nt * TS * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&c.Linv, (size_t)nt * NB * NB * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&c.ybuf, (size_t)nt * NB * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&c.flags, (size_t)nt * sizeof(int)) != cudaSuccess)
      return false;
    cudaMemset(c.flags, 0, nt * sizeof(int));
    c.epoch = 0;
    c.cap_nt = nt;
  }
  return true;
}

// the wavefront triangular solve on a row-major factor L (lda)
cudaError_t launch_wave(CholCtx& c, int n, const double* L, int lda, const double* xin, double* x, int upper,
                        cudaStream_t st) {
  const int nblk = (n + NB - 1) / NB;
  int epoch = ++c.epoch;
  const double* Linv = c.Linv;
  int* flags = c.flags;
  void* args[] = {(void*)&n,   (void*)&L, (void*)&lda,   (void*)&Linv,  (void*)&xin,
                  (void*)&x, (void*)&flags, (void*)&epoch, (void*)&upper};
  cudaError_t e = cudaLaunchCooperativeKernel((const void*)k_trsv_wave, dim3(nblk), dim3(256), args, 0, st);
  count_launch();
  return e;
}

// the tile-DAG factorisation of the row-major A (read only); with b, also ybuf = L^{-1} b (and, for
// one tile, x = A^{-1} b)
cudaError_t factor_dag(CholCtx& c, int n, const double* A, int lda, int* info, const double* b, double* x,
                       cudaStream_t st) {
  const int nt = (n + NB - 1) / NB;
  const int ntask = nt * (nt + 1) / 2 - (nt - 1);  // the sub-diagonal tiles ride with the diagonal tasks
  const int grid = std::min(ntask, c.sms * c.occ);
  int epoch = ++c.depoch;
  if (nt == 1) {
    // one tile: one CTA, nothing to wait for -- a plain launch, no memsets (c1's Newton step: the
    // whole solve in this one launch)
    k_chol_dag<<<1, 256, kDagSmem, st>>>(n, nt, A, lda, c.Lt, c.LinvP, c.Linv, b, c.ybuf, x, info, c.dflags, epoch,
                                         nullptr);
    count_launch();
    return cudaGetLastError();
  }
  int* next_task = c.dflags + c.cap_lt;  // past every flag slot (never read as a flag)
  cudaMemsetAsync(info, 0, sizeof(int), st);
  cudaMemsetAsync(next_task, 0, sizeof(int), st);
  void* args[] = {(void*)&n,  (void*)&nt,   (void*)&A,    (void*)&lda,  (void*)&c.Lt,    (void*)&c.LinvP,
                  (void*)&c.Linv, (void*)&b, (void*)&c.ybuf, (void*)&x, (void*)&info, (void*)&c.dflags,
                  (void*)&epoch, (void*)&next_task};
  cudaError_t e = cudaLaunchCooperativeKernel((const void*)k_chol_dag, dim3(grid), dim3(256), args, kDagSmem, st);
  count_launch();
  return e;
}

}  // namespace

// Kernels that wait on other CTAs of their grid (k_chol_dag's tile flags, k_trsv_wave's block
// flags) are launched cooperatively; two such grids running at once from different workspaces
// could each hold part of the SMs and wait forever. Every factor / solve section therefore runs
// under one process-wide lock and drains its stream before releasing it.
struct CoopSection {
  static std::mutex& mu() {
    static std::mutex m;
    return m;
  }
  std::lock_guard<std::mutex> lk;
  cudaStream_t st;
  explicit CoopSection(cudaStream_t s) : lk(mu()), st(s) {}
  ~CoopSection() { cudaStreamSynchronize(st); }
};

CholCtx* chol_ctx_create() { return new CholCtx(); }

void chol_ctx_destroy(CholCtx* c) {
  if (!c) return;
  cudaFree(c->Lt);
  cudaFree(c->dflags);
  cudaFree(c->LinvP);
  cudaFree(c->Linv);
  cudaFree(c->ybuf);
  cudaFree(c->flags);
  delete c;
}

cudaError_t launch_cholesky(CholCtx* cc, int n, double* A, int lda, int* info, cudaStream_t st) {
  CoopSection cs(st);
  if (!ensure_work(*cc, n)) return cudaErrorMemoryAllocation;
  cudaError_t e = factor_dag(*cc, n, A, lda, info, nullptr, nullptr, st);
  if (e != cudaSuccess) return e;
  k_untile<<<n, 256, 0, st>>>(n, cc->Lt, A, lda);
  count_launch();
  cc->factor = A;
  cc->factor_n = n;
  return cudaGetLastError();
}

cudaError_t launch_cholesky_solve_fused(CholCtx* cc, int n, double* A, int lda, int* info, const double* b,
                                        double* x, cudaStream_t st) {
  CoopSection cs(st);
  if (!ensure_work(*cc, n)) return cudaErrorMemoryAllocation;
  cc->factor = nullptr;  // A keeps -H: the factor lives in the tile-major copy only
  cc->factor_n = 0;
  cudaError_t e = factor_dag(*cc, n, A, lda, info, b, x, st);
  if (e != cudaSuccess || n <= NB) return e;
  const int nblk = (n + NB - 1) / NB;
  int epoch = ++cc->epoch;
  void* args[] = {(void*)&n, (void*)&cc->Lt, (void*)&cc->LinvP, (void*)&cc->ybuf, (void*)&x, (void*)&cc->flags,
                  (void*)&epoch};
  e = cudaLaunchCooperativeKernel((const void*)k_trsv_bwd_tiles, dim3(nblk), dim3(256), args, kBwdSmem, st);
  count_launch();
  return e;
}

cudaError_t launch_inv_diag_sqrt(CholCtx* cc, int n, double* L, int lda, double* se, cudaStream_t st) {
  CholCtx& c = *cc;
  if (!ensure_work(c, n)) return cudaErrorMemoryAllocation;
  if (c.factor != L || c.factor_n != n) {  // factor from elsewhere: build its Linv blocks
    k_trtri_blocks<<<(n + NB - 1) / NB, 256, kDynR, st>>>(n, L, lda, c.Linv);
    count_launch();
    c.factor = L;
    c.factor_n = n;
  }
  k_inv_diag<<<(n + NB - 1) / NB, 256, kDyn, st>>>(n, L, lda, c.Linv, se);
  count_launch();
  return cudaGetLastError();
}

void chol_forget_factor(CholCtx* cc) {
  cc->factor = nullptr;
  cc->factor_n = 0;
}

cudaError_t launch_chol_solve(CholCtx* cc, int n, const double* L, int lda, const double* b, double* x,
                              cudaStream_t st) {
  CoopSection cs(st);
  CholCtx& c = *cc;
  if (!ensure_work(c, n)) return cudaErrorMemoryAllocation;
  if (c.factor != L || c.factor_n != n) {  // factor from elsewhere: build its Linv blocks
    k_trtri_blocks<<<(n + NB - 1) / NB, 256, kDynR, st>>>(n, L, lda, c.Linv);
    count_launch();
    c.factor = L;
    c.factor_n = n;
  }
  cudaError_t e = launch_wave(c, n, L, lda, b, x, 0, st);
  if (e != cudaSuccess) return e;
  return launch_wave(c, n, L, lda, x, x, 1, st);
}

}  // namespace mnl
