// Newton step: -H = L L^T by a blocked right-looking Cholesky
// factorisation, then L y = g and L^T delta = y (Eq. "NR update": delta = -H^{-1} g;
// -H is positive definite by global concavity).
//
// Per panel j of NB = 64 columns:
//   k_potrf_inv   one CTA: Cholesky of the diagonal block in shared memory, fused with the
//                 inverse of its triangular factor (kept in a workspace, Linv[j]) and, in the
//                 fused factor+solve, the forward-solve piece y_j = Linv[j] b_j;
//   k_trsm_gemm   L21 = A21 Linv[j]^T as a DMMA product (one CTA per 64 rows), fused with the
//                 forward-solve update b_r -= L21_r y_j of its rows;
//   k_syrk_tiles  A22 -= L21 L21^T, one CTA per 64x64 lower tile (DMMA, mma.sync m8n8k4 f64).
// The backward solve L^T x = y is one cooperative wavefront kernel: CTA b owns block b, folds in
// the already-solved blocks as their flags are published, and applies Linv[b]^T (no per-block
// launches).  The standalone solve (mnl_cholesky_solve) runs the same wavefront forward too.
// The matrix is row-major with leading dimension lda; only the lower triangle is referenced.
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

// k_potrf_inv: Cholesky of the jb x jb diagonal block fused with X = L^{-1}, blocked by 16:
// for each 16-column sub-panel: (1) the 16 x 16 diagonal block and its inverse by the whole CTA
// (one thread per entry), (2) L21 = A21 X11^T, (3) A22 -= L21 L21^T on DMMA by all warps;
// finally the off-diagonal blocks of X = L^{-1} on DMMA. With x != null it also applies the
// forward-solve piece y_j = Linv b_j (b_j already holds every earlier panel's update).
constexpr int SB = 16;
__device__ __noinline__ void potrf_block(int n, double* A, int lda, int j0, double* Linv, int* info, double* x,
                                         double* dsm) {
  __syncthreads();  // the CTA may have used dsm for another step just before
  double(*S)[LDR] = reinterpret_cast<double(*)[LDR]>(dsm);
  double(*X)[LDR] = reinterpret_cast<double(*)[LDR]>(dsm + NB * LDR);
  __shared__ double T[NB][SB + 1];
  __shared__ double bv[NB];
  __shared__ double colb[2][SB], xrow[2][SB], pv16[SB];
  const int jb = min(NB, n - j0);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  {  // all 16 loads of a thread in flight at once (clamped addresses, masked values)
    double v[16];
#pragma unroll
    for (int m = 0; m < 16; ++m) {
      const int e = tid + 256 * m, r = e >> 6, c = e & 63;
      const int rr = r < jb ? r : jb - 1, ccl = c < jb ? c : jb - 1;
      v[m] = __ldcg(A + (int64_t)(j0 + rr) * lda + j0 + ccl);  // L2: other CTAs updated it
    }
#pragma unroll
    for (int m = 0; m < 16; ++m) {
      const int e = tid + 256 * m, r = e >> 6, c = e & 63;
      // rows / columns beyond jb: identity (keeps the blocked steps well defined; never written back)
      S[r][c] = (r < jb && c <= r) ? v[m] : (r == c ? 1.0 : 0.0);
      X[r][c] = 0.0;
    }
  }
  if (x && tid < NB) bv[tid] = tid < jb ? __ldcg(x + j0 + tid) : 0.0;
  __syncthreads();
  bool bad_any = false;
  for (int c0 = 0; c0 < NB; c0 += SB) {
    // (1) the 16 x 16 diagonal block and its inverse with all 256 threads, thread (r, c) holding
    // entry (r, c) in a register and one barrier per column: factor with the unscaled update
    // a_rc -= a_rC a_cC / a_CC (column C published to colb at the end of step C - 1), scale once;
    // then X = L^{-1} row by row (row C scaled by 1 / L_CC and published, rows r > C updated).
    {
      const int r = tid >> 4, c = tid & 15;
      double a = (c <= r) ? S[c0 + r][c0 + c] : 0.0;
      if (c == 0) colb[0][r] = a;
      __syncthreads();
      for (int C = 0; C < SB; ++C) {
        const double* cb = colb[C & 1];
        double piv = cb[C];
        const bool bad = !(piv > 0.0) || !isfinite(piv);
        if (bad) piv = 1.0;  // keep the values finite; info reports the failure
        if (tid == 0) {
          pv16[C] = piv;
          bad_any |= bad;
        }
        const double inv = 1.0 / piv;
        if (c > C && r >= c) a = fma(-cb[r] * inv, cb[c], a);
        if (c == C + 1) colb[(C + 1) & 1][r] = a;
        __syncthreads();
      }
      if (c <= r) {
        const double rs = rsqrt(pv16[c]);
        S[c0 + r][c0 + c] = (r == c) ? pv16[c] * rs : a * rs;
      }
      __syncthreads();
      double xv = (r == c) ? 1.0 : 0.0;
      for (int C = 0; C < SB; ++C) {
        if (r == C && c <= C) {
          xv *= 1.0 / S[c0 + C][c0 + C];
          xrow[C & 1][c] = xv;
        }
        __syncthreads();
        if (r > C && c <= C) xv = fma(-S[c0 + r][c0 + C], xrow[C & 1][c], xv);
      }
      X[c0 + r][c0 + c] = (c <= r) ? xv : 0.0;
    }
    __syncthreads();
    const int r0 = c0 + SB, R = NB - r0;
    if (R > 0) {
      // (2) L21 = A21 X11^T  (rows r0.., 16 columns), via registers then in place
      double l21[3];
#pragma unroll
      for (int m = 0; m < 3; ++m) {
        const int e = tid + 256 * m;
        l21[m] = 0.0;
        if (e < R * SB) {
          const int i = r0 + e / SB, j = e % SB;
          double acc = 0.0;
          for (int t = 0; t <= j; ++t) acc = fma(S[i][c0 + t], X[c0 + j][c0 + t], acc);
          l21[m] = acc;
        }
      }
      __syncthreads();
#pragma unroll
      for (int m = 0; m < 3; ++m) {
        const int e = tid + 256 * m;
        if (e < R * SB) S[r0 + e / SB][c0 + e % SB] = l21[m];
      }
      __syncthreads();
      // (3) A22 -= L21 L21^T on DMMA: 8x8 blocks (mb >= nb) of the R x R trailing matrix
      const int MBk = R / 8;
      const int lr = lane >> 2, lk = lane & 3;
      for (int blk = w; blk < MBk * (MBk + 1) / 2; blk += 8) {
        int mb = (int)((sqrt(8.0 * blk + 1.0) - 1.0) * 0.5);
        while ((mb + 1) * (mb + 2) / 2 <= blk) ++mb;
        while (mb * (mb + 1) / 2 > blk) --mb;
        const int nb = blk - mb * (mb + 1) / 2;
        double c0v = 0.0, c1v = 0.0;
#pragma unroll
        for (int k0 = 0; k0 < SB; k0 += 4) {
          const double a = S[r0 + mb * 8 + lr][c0 + k0 + lk];
          const double b = S[r0 + nb * 8 + lr][c0 + k0 + lk];
          dmma(c0v, c1v, a, b);
        }
        const int rr = r0 + mb * 8 + lr, cc = r0 + nb * 8 + 2 * lk;
        if (cc <= rr) S[rr][cc] -= c0v;
        if (cc + 1 <= rr) S[rr][cc + 1] -= c1v;
      }
      __syncthreads();
    }
  }
  if (tid == 0 && bad_any) atomicCAS(info, 0, j0 + 1);
  // (4) off-diagonal blocks of X = L^{-1} (the 16 x 16 diagonal blocks came from step 1) on DMMA:
  // X_ba = -X_bb (L_ba X_aa) for the 16-blocks of each 32-block, then for the two 32-blocks.
  // The strict upper triangle of S is zeroed first (the blocks are read whole).
  for (int e = tid; e < NB * NB; e += 256) {
    const int r = e >> 6, c = e & 63;
    if (c > r) S[r][c] = 0.0;
  }
  __syncthreads();
  {
    double(*T2)[33] = reinterpret_cast<double(*)[33]>(&T[0][0]);  // 32 x 33 view of T (64 x 17)
    const int h = w >> 2, o = 32 * h;
    smem_gemm(&T2[16 * h][0], 33, &S[o + 16][o], LDR, &X[o][o], LDR, 16, 16, 16, 1.0, w & 3, 4);
    __syncthreads();
    smem_gemm(&X[o + 16][o], LDR, &X[o + 16][o + 16], LDR, &T2[16 * h][0], 33, 16, 16, 16, -1.0, w & 3, 4);
    __syncthreads();
    smem_gemm(&T2[0][0], 33, &S[32][0], LDR, &X[0][0], LDR, 32, 32, 32, 1.0, w, 8);
    __syncthreads();
    smem_gemm(&X[32][0], LDR, &X[32][32], LDR, &T2[0][0], 33, 32, 32, 32, -1.0, w, 8);
    __syncthreads();
  }
  for (int e = tid; e < NB * NB; e += 256) {
    const int r = e >> 6, c = e & 63;
    if (r < jb && c <= r) A[(int64_t)(j0 + r) * lda + j0 + c] = S[r][c];
    Linv[e] = (r < jb && c <= r) ? X[r][c] : 0.0;  // [NB][NB], zero outside the triangle
  }
  if (x) {
    const int r = tid >> 2, q = tid & 3;
    double sacc = 0.0;
    for (int t = q; t <= r; t += 4) sacc = fma(X[r][t], bv[t], sacc);
    sacc += __shfl_xor_sync(0xffffffffu, sacc, 1);
    sacc += __shfl_xor_sync(0xffffffffu, sacc, 2);
    if (q == 0 && r < jb) x[j0 + r] = sacc;
  }
}

__global__ void __launch_bounds__(256) k_potrf_inv(int n, double* A, int lda, int j0, double* Linv, int* info,
                                                   double* x) {
  extern __shared__ __align__(16) double dsm[];
  potrf_block(n, A, lda, j0, Linv, info, x, dsm);
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
// thread in flight at once (clamped addresses, masked values; L2 loads: other CTAs of the
// persistent factorisation wrote the tile, and trsm rewrites it)
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

// out[64x64] = X[64x64] * Y[64x64]^T from two smem tiles (row-major, LDS); 8 warps of 16x32
__device__ __forceinline__ void tile_xyT(const double (*Xs)[LDS], const double (*Ys)[LDS], double acc[2][4][2]) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int wr = (w >> 1) * 16, wc = (w & 1) * 32;
  const int lr = lane >> 2, lk = lane & 3;
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
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

// rows [j0+jb + 64*tile, +64): L21 = A21 Linv^T; with x: x_r -= L21_r . y_j
// L1 caching of the operand tiles (cp.async.ca) is safe only across kernel launches: inside the
// persistent factorisation (k_chol_persist) a line fetched for panel j may hold columns that panel
// j's trailing update rewrites, so there (PERSIST) the tiles are staged through registers with
// L2-only loads, all in flight together.
template <bool PERSIST>
__device__ __noinline__ void trsm_tile(int n, double* A, int lda, int j0, const double* Linv, double* x, int tile,
                                       double* dsm) {
  __syncthreads();  // smem reuse across consecutive tiles
  double(*Xs)[LDS] = reinterpret_cast<double(*)[LDS]>(dsm);
  double(*Ys)[LDS] = reinterpret_cast<double(*)[LDS]>(dsm + NB * LDS);
  __shared__ double yv[NB];
  const int jb = min(NB, n - j0);
  const int r0 = j0 + jb + tile * NB;
  const int tid = threadIdx.x;
  if constexpr (PERSIST) {  // one round trip through registers (L2 loads)
    const int nr = n - r0;
    double va[16], vl[16];
#pragma unroll
    for (int m = 0; m < 16; ++m) {
      const int e = tid + 256 * m, r = e >> 6, c = e & 63;
      const bool ok = r < nr && c < jb;
      va[m] = ok ? __ldcg(A + (int64_t)(r0 + r) * lda + j0 + c) : 0.0;
      vl[m] = __ldcg(Linv + e);
    }
#pragma unroll
    for (int m = 0; m < 16; ++m) {
      const int e = tid + 256 * m, r = e >> 6, c = e & 63;
      Xs[r][c] = va[m];
      Ys[r][c] = vl[m];
    }
  } else {  // one round trip: the A21 tile (zero beyond n / jb) and Linv[j] straight into shared memory
    const int nr = n - r0;
#pragma unroll 4
    for (int m = 0; m < 16; ++m) {
      const int e = tid + 256 * m, r = e >> 6, c = e & 63;
      const bool ok = r < nr && c < jb;
      const double* g = A + (int64_t)(r0 + (ok ? r : 0)) * lda + j0 + (ok ? c : 0);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(
                       static_cast<unsigned>(__cvta_generic_to_shared(&Xs[r][c]))),
                   "l"(g), "r"(ok ? 8 : 0)
                   : "memory");
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                       static_cast<unsigned>(__cvta_generic_to_shared(&Ys[r][c]))),
                   "l"(Linv + e)
                   : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  if (x && tid < NB) yv[tid] = tid < jb ? __ldcg(x + j0 + tid) : 0.0;
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  double acc[2][4][2];
  tile_xyT(Xs, Ys, acc);
  __syncthreads();  // done reading Xs: reuse it for the result
  const int lane = tid & 31, w = tid >> 5;
  const int wr = (w >> 1) * 16, wc = (w & 1) * 32, lr = lane >> 2, lk = lane & 3;
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int rl = wr + a * 8 + lr, c = wc + b * 8 + 2 * lk + h;
        Xs[rl][c] = (c < jb) ? acc[a][b][h] : 0.0;
        if (r0 + rl < n && c < jb) A[(int64_t)(r0 + rl) * lda + j0 + c] = acc[a][b][h];
      }
  if (x) {
    __syncthreads();
    const int r = tid >> 2, q4 = tid & 3;
    double s = 0.0;
    for (int t = q4; t < jb; t += 4) s = fma(Xs[r][t], yv[t], s);
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    if (q4 == 0 && r0 + r < n) x[r0 + r] = __ldcg(x + r0 + r) - s;
  }
}

__global__ void __launch_bounds__(256) k_trsm_gemm(int n, double* A, int lda, int j0, const double* Linv, double* x) {
  extern __shared__ __align__(16) double dsm[];
  trsm_tile<false>(n, A, lda, j0, Linv, x, blockIdx.x, dsm);
}

// trailing update tile (ti, tj), ti >= tj, of A22 -= L21 L21^T (tile coordinates relative to the
// first row/column after panel j0)
template <bool PERSIST>
__device__ __noinline__ void syrk_tile(int n, double* A, int lda, int j0, int ti, int tj, double* dsm) {
  __syncthreads();  // smem reuse across consecutive tiles
  double(*Li)[LDS] = reinterpret_cast<double(*)[LDS]>(dsm);
  double(*Lj)[LDS] = reinterpret_cast<double(*)[LDS]>(dsm + NB * LDS);
  const int jb = min(NB, n - j0);
  const int s0 = j0 + jb;
  const int ri = s0 + ti * NB, rj = s0 + tj * NB;
  const int tid = threadIdx.x;
  const int lane = tid & 31, w = tid >> 5;
  const int wr = (w >> 1) * 16, wc = (w & 1) * 32, lr = lane >> 2, lk = lane & 3;
  // one round trip: the two L21 tiles go to shared memory (cp.async, or through registers in the
  // persistent kernel) while this thread's 16 entries of the C tile are loaded into registers
  double cv[2][4][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = ri + wr + a * 8 + lr, c = rj + wc + b * 8 + 2 * lk + h;
        cv[a][b][h] = (r < n && c < n && c <= r) ? __ldcg(A + (int64_t)r * lda + c) : 0.0;
      }
  if constexpr (PERSIST) {
    const int nri = n - ri, nrj = n - rj;
    double vi[16], vj[16];
#pragma unroll
    for (int m = 0; m < 16; ++m) {
      const int e = tid + 256 * m, r = e >> 6, c = e & 63;
      vi[m] = (r < nri && c < jb) ? __ldcg(A + (int64_t)(ri + r) * lda + j0 + c) : 0.0;
      vj[m] = (r < nrj && c < jb) ? __ldcg(A + (int64_t)(rj + r) * lda + j0 + c) : 0.0;
    }
#pragma unroll
    for (int m = 0; m < 16; ++m) {
      const int e = tid + 256 * m, r = e >> 6, c = e & 63;
      Li[r][c] = vi[m];
      Lj[r][c] = vj[m];
    }
  } else {
    const int nri = n - ri, nrj = n - rj;
#pragma unroll 4
    for (int m = 0; m < 16; ++m) {
      const int e = tid + 256 * m, r = e >> 6, c = e & 63;
      const bool oki = r < nri && c < jb, okj = r < nrj && c < jb;
      const double* gi = A + (int64_t)(ri + (oki ? r : 0)) * lda + j0 + (oki ? c : 0);
      const double* gj = A + (int64_t)(rj + (okj ? r : 0)) * lda + j0 + (okj ? c : 0);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(
                       static_cast<unsigned>(__cvta_generic_to_shared(&Li[r][c]))),
                   "l"(gi), "r"(oki ? 8 : 0)
                   : "memory");
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(
                       static_cast<unsigned>(__cvta_generic_to_shared(&Lj[r][c]))),
                   "l"(gj), "r"(okj ? 8 : 0)
                   : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  double acc[2][4][2];
  tile_xyT(Li, Lj, acc);
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = ri + wr + a * 8 + lr, c = rj + wc + b * 8 + 2 * lk + h;
        if (r < n && c < n && c <= r) A[(int64_t)r * lda + c] = cv[a][b][h] - acc[a][b][h];
      }
}

// linear index over the lower triangle of tiles (row-major) -> (ti, tj), ti >= tj
__device__ __forceinline__ void tri_tile(int t, int& ti, int& tj) {
  ti = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
  while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
  while (ti * (ti + 1) / 2 > t) --ti;
  tj = t - ti * (ti + 1) / 2;
}

// col_only = 1: only block-column 0 of the trailing matrix (the next panel, lookahead path);
// col_only = 0: the lower triangle starting at tile (first, first).
__global__ void __launch_bounds__(256) k_syrk_tiles(int n, double* A, int lda, int j0, int col_only, int first) {
  extern __shared__ __align__(16) double dsm[];
  int ti, tj;
  if (col_only) {
    ti = blockIdx.x;
    tj = 0;
  } else {
    tri_tile(blockIdx.x, ti, tj);
    ti += first;
    tj += first;
  }
  syrk_tile<false>(n, A, lda, j0, ti, tj, dsm);
}

// ---- triangular solve wavefront ------------------------------------------------------------
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// forward (upper = 0): y_b = Linv_b (x_b - sum_{j<b} L[b, j] y_j), block b = blockIdx.x.
// backward (upper = 1): z_b = Linv_b^T (y_b - sum_{j>b} L[j, b]^T z_j), blocks in reverse order.
// x is overwritten in place. The L block of the next step is loaded into registers before the
// flag wait; the contraction order over blocks and within a block is fixed (deterministic).
__global__ void __launch_bounds__(256) k_trsv_wave(int n, const double* L, int lda, const double* Linv,
                                                   double* x, int* flags, int epoch, int upper) {
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
    if (tid < NB) v[tid] = tid < bb ? x[b0 + tid] - part[0][tid] : 0.0;
  } else {
    part[g][c] = acc;
    __syncthreads();
    if (tid < NB) {
      const double s = (part[0][tid] + part[1][tid]) + (part[2][tid] + part[3][tid]);
      v[tid] = tid < bb ? x[b0 + tid] - s : 0.0;
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

// ---- persistent factorisation (one cooperative launch) -------------------------------------
// Grid barrier over all CTAs of a cooperative launch: count + generation (sense) in global memory.
// Writes before the barrier are published with a gpu-scope fence; the phases read A / Linv / x
// through L2 (__ldcg), never through a possibly stale L1.
__device__ __forceinline__ void grid_barrier(unsigned* count, unsigned* gen, unsigned& my_gen, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned g = my_gen;
    if (atomicAdd(count, 1u) == nblocks - 1) {
      atomicExch(count, 0u);
      __threadfence();
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(gen), "r"(g + 1) : "memory");
    } else {
      unsigned v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(gen) : "memory");
        if (v == g) __nanosleep(32);
      } while (v == g);
    }
  }
  my_gen += 1;
  __syncthreads();
}

// The blocked right-looking factorisation of factor() in one kernel (n <= 2816), with the same one-panel
// lookahead: per panel j, (B) all CTAs compute the trsm tiles of panel j, (C) all CTAs update
// block column j+1, (A) CTA 0 factors panel j+1 while the other CTAs apply the rest of panel j's
// trailing update. Every tile runs exactly the arithmetic of the multi-kernel path (same device
// functions, same order per entry), so the factor is bitwise identical; only launch and
// cross-stream synchronisation costs go away. bar = {count, generation}.
__global__ void __launch_bounds__(256, 1) k_chol_persist(int n, double* A, int lda, double* Linv, int* info, double* x,
                                                         unsigned* bar) {
  extern __shared__ __align__(16) double dsm[];
  const unsigned G = gridDim.x, b = blockIdx.x;
  unsigned my_gen = 0;
  if (threadIdx.x == 0) my_gen = *reinterpret_cast<volatile unsigned*>(bar + 1);
  const int np = (n + NB - 1) / NB;
  if (b == 0) potrf_block(n, A, lda, 0, Linv, info, x, dsm);
  grid_barrier(bar, bar + 1, my_gen, G);
  for (int j = 0; j + 1 < np; ++j) {
    const int j0 = j * NB, rem = n - j0 - NB, mt = (rem + NB - 1) / NB;
    const double* Lj = Linv + (size_t)j * NB * NB;
    for (int t = b; t < mt; t += G) trsm_tile<true>(n, A, lda, j0, Lj, x, t, dsm);    // (B)
    grid_barrier(bar, bar + 1, my_gen, G);
    for (int t = b; t < mt; t += G) syrk_tile<true>(n, A, lda, j0, t, 0, dsm);       // (C)
    grid_barrier(bar, bar + 1, my_gen, G);
    if (b == 0) {                                                                    // (A)
      potrf_block(n, A, lda, j0 + NB, Linv + (size_t)(j + 1) * NB * NB, info, x, dsm);
    } else {
      const int nrest = (mt - 1) * mt / 2;
      for (int t = b - 1; t < nrest; t += G - 1) {
        int ti, tj;
        tri_tile(t, ti, tj);
        syrk_tile<true>(n, A, lda, j0, ti + 1, tj + 1, dsm);
      }
    }
    grid_barrier(bar, bar + 1, my_gen, G);
  }
}

}  // namespace

// Per-workspace factorisation state (one per library workspace, i.e. per device and stream).
struct CholCtx {
  unsigned* bar = nullptr;  // k_chol_persist's grid barrier {count, generation}
  int persist_grid = -1;    // CTAs of the cooperative launch (0: not available)
  double* Linv = nullptr;
  size_t cap = 0;
  const double* factor = nullptr;  // matrix whose Linv blocks are current
  int factor_n = 0;
  int* flags = nullptr;
  int nflags = 0;
  int epoch = 0;
  // two-stream lookahead path
  cudaStream_t side = nullptr;
  std::vector<cudaEvent_t> ev;
  cudaEvent_t start = nullptr, done = nullptr;
};

namespace {

bool ensure_work(CholCtx& g_cw, int n) {
  const int nblk = (n + NB - 1) / NB;
  const size_t need = (size_t)nblk * NB * NB;
  if (need > g_cw.cap) {
    cudaFree(g_cw.Linv);
    if (cudaMalloc(&g_cw.Linv, need * sizeof(double)) != cudaSuccess) { g_cw.cap = 0; return false; }
    g_cw.cap = need;
  }
  if (nblk > g_cw.nflags) {
    cudaFree(g_cw.flags);
    if (cudaMalloc(&g_cw.flags, nblk * sizeof(int)) != cudaSuccess) { g_cw.nflags = 0; return false; }
    cudaMemset(g_cw.flags, 0, nblk * sizeof(int));
    g_cw.nflags = nblk;
    g_cw.epoch = 0;
  }
  return true;
}

constexpr size_t kDyn = 2 * NB * LDS * sizeof(double);
constexpr size_t kDynR = 2 * NB * LDR * sizeof(double);
void set_attrs() {
  static uint64_t attr_mask = 0;
  set_once_per_device(attr_mask, [] {
    cudaFuncSetAttribute(k_trsm_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDyn);
    cudaFuncSetAttribute(k_syrk_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDyn);
    cudaFuncSetAttribute(k_trtri_blocks, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDynR);
    cudaFuncSetAttribute(k_chol_persist, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDyn);
    return cudaFuncSetAttribute(k_potrf_inv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDynR);
  });
}

cudaError_t launch_wave(CholCtx& g_cw, int n, const double* L, int lda, double* x, int upper, cudaStream_t st) {
  const int nblk = (n + NB - 1) / NB;
  int epoch = ++g_cw.epoch;
  const double* Linv = g_cw.Linv;
  int* flags = g_cw.flags;
  void* args[] = {(void*)&n, (void*)&L, (void*)&lda, (void*)&Linv, (void*)&x, (void*)&flags, (void*)&epoch,
                  (void*)&upper};
  cudaError_t e = cudaLaunchCooperativeKernel((const void*)k_trsv_wave, dim3(nblk), dim3(256), args, 0, st);
  count_launch();
  return e;
}

cudaEvent_t la_event(CholCtx& g_la, size_t i) {
  while (g_la.ev.size() <= i) {
    cudaEvent_t e;
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    g_la.ev.push_back(e);
  }
  return g_la.ev[i];
}

// Factorisation with a one-panel lookahead; with x != null also the forward solve x <- L^{-1} x.
// side stream: [A22 update of the next panel's block column] -> potrf(j+1) -> trsm(j+1)
// main stream: the rest of panel j's trailing update, concurrently.
cudaError_t factor_persist(CholCtx& g_cw, int n, double* A, int lda, int* info, double* x, cudaStream_t st) {
  cudaMemsetAsync(info, 0, sizeof(int), st);
  void* args[] = {(void*)&n, (void*)&A, (void*)&lda, (void*)&g_cw.Linv, (void*)&info, (void*)&x, (void*)&g_cw.bar};
  cudaError_t e = cudaLaunchCooperativeKernel((const void*)k_chol_persist, dim3(g_cw.persist_grid), dim3(256), args,
                                              kDyn, st);
  count_launch();
  g_cw.factor = A;
  g_cw.factor_n = n;
  return e;
}

// CTAs for k_chol_persist: one per SM when the kernel fits there (0 disables the persistent path)
int persist_grid(CholCtx& g_cw) {
  if (g_cw.persist_grid >= 0) return g_cw.persist_grid;
  g_cw.persist_grid = 0;
  if (getenv("MNL_CHOL_STREAMS")) return 0;
  int dev = 0, sms = 0, coop = 0, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
  if (!coop) return 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_chol_persist, 256, kDyn) != cudaSuccess || occ < 1) return 0;
  if (cudaMalloc(&g_cw.bar, 2 * sizeof(unsigned)) != cudaSuccess) return 0;
  cudaMemset(g_cw.bar, 0, 2 * sizeof(unsigned));
  g_cw.persist_grid = sms;  // one CTA per SM: the panel CTA has its SM to itself
  return g_cw.persist_grid;
}

cudaError_t factor(CholCtx& g_cw, int n, double* A, int lda, int* info, double* x, cudaStream_t st) {
  CholCtx& g_la = g_cw;
  set_attrs();
  if (!ensure_work(g_cw, n)) return cudaErrorMemoryAllocation;
  // persistent single launch: since the tiles fetch their operands in one round trip it is faster
  // than the two-stream multi-kernel path at every measured n (2816: 1.92 vs 2.36 ms; 5049: 5.35 vs
  // 5.58 ms); MNL_CHOL_STREAMS=1 forces the multi-kernel path, MNL_CHOL_PERSIST_MAX caps n
  static const int persist_max = getenv("MNL_CHOL_PERSIST_MAX") ? atoi(getenv("MNL_CHOL_PERSIST_MAX")) : 16384;
  if (n <= persist_max && persist_grid(g_cw) > 1) return factor_persist(g_cw, n, A, lda, info, x, st);
  if (!g_la.side) {
    int lo = 0, hi = 0;  // the panel chain is the critical path: give it the highest priority
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    cudaStreamCreateWithPriority(&g_la.side, cudaStreamNonBlocking, hi);
    cudaEventCreateWithFlags(&g_la.start, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&g_la.done, cudaEventDisableTiming);
  }
  cudaStream_t sp = g_la.side;
  const int np = (n + NB - 1) / NB;
  cudaMemsetAsync(info, 0, sizeof(int), st);
  cudaEventRecord(g_la.start, st);
  cudaStreamWaitEvent(sp, g_la.start, 0);
  auto panel = [&](int j) {  // potrf + trsm of panel j on the side stream
    const int j0 = j * NB, jb = std::min(NB, n - j0);
    double* Lj = g_cw.Linv + (size_t)j * NB * NB;
    k_potrf_inv<<<1, 256, kDynR, sp>>>(n, A, lda, j0, Lj, info, x);
    count_launch();
    const int rem = n - j0 - jb;
    if (rem > 0) {
      k_trsm_gemm<<<(rem + NB - 1) / NB, 256, kDyn, sp>>>(n, A, lda, j0, Lj, x);
      count_launch();
    }
  };
  panel(0);
  cudaEventRecord(la_event(g_la, 2 * 0), sp);  // ev_p(0)
  for (int j = 0; j + 1 < np; ++j) {
    const int j0 = j * NB;
    const int rem = n - j0 - NB;
    const int mt = (rem + NB - 1) / NB;
    // main: rest of panel j's trailing update (tiles with tj >= 1)
    cudaStreamWaitEvent(st, la_event(g_la, 2 * j), 0);
    if (mt > 1) {
      k_syrk_tiles<<<(mt - 1) * mt / 2, 256, kDyn, st>>>(n, A, lda, j0, 0, 1);
      count_launch();
    }
    cudaEventRecord(la_event(g_la, 2 * j + 1), st);  // ev_r(j)
    // side: next panel's block column, then its factorisation
    k_syrk_tiles<<<mt, 256, kDyn, sp>>>(n, A, lda, j0, 1, 0);
    count_launch();
    panel(j + 1);
    cudaEventRecord(la_event(g_la, 2 * (j + 1)), sp);  // ev_p(j+1)
    // the next column update (side, iteration j+1) must follow this rest update (main)
    cudaStreamWaitEvent(sp, la_event(g_la, 2 * j + 1), 0);
  }
  cudaEventRecord(g_la.done, sp);
  cudaStreamWaitEvent(st, g_la.done, 0);
  g_cw.factor = A;
  g_cw.factor_n = n;
  return cudaGetLastError();
}

// ---- diag((L L^T)^{-1}) for standard errors ---------------------
// CTA J owns block column J of W = L^{-1}: W_JJ = Linv[J]; for I = J+1 .. : W_IJ = -Linv[I]
// sum_{K=J}^{I-1} L_IK W_KJ (DMMA 64x64 tiles). The finished blocks W_KJ are kept, transposed, in
// the (unused) strict upper triangle of A at block (J, K); columns of A^{-1} = W^T W have
// diag_c = sum_r W_rc^2, summed in a fixed order (rows of a tile by shuffles, warps via smem, I
// ascending). Block columns are independent; the first one carries the longest chain.
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

// Kernels that wait on other CTAs of their grid (k_chol_persist's grid barriers, k_trsv_wave's
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
  cudaFree(c->bar);
  cudaFree(c->Linv);
  cudaFree(c->flags);
  for (cudaEvent_t e : c->ev) cudaEventDestroy(e);
  if (c->start) cudaEventDestroy(c->start);
  if (c->done) cudaEventDestroy(c->done);
  if (c->side) cudaStreamDestroy(c->side);
  delete c;
}

cudaError_t launch_cholesky(CholCtx* cc, int n, double* A, int lda, int* info, cudaStream_t st) {
  CoopSection cs(st);
  return factor(*cc, n, A, lda, info, nullptr, st);
}

cudaError_t launch_cholesky_solve_fused(CholCtx* cc, int n, double* A, int lda, int* info, const double* b,
                                        double* x, cudaStream_t st) {
  CoopSection cs(st);
  if (x != b) cudaMemcpyAsync(x, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, st);
  cudaError_t e = factor(*cc, n, A, lda, info, x, st);
  if (e != cudaSuccess) return e;
  return launch_wave(*cc, n, A, lda, x, 1, st);
}

cudaError_t launch_inv_diag_sqrt(CholCtx* cc, int n, double* L, int lda, double* se, cudaStream_t st) {
  CholCtx& g_cw = *cc;
  set_attrs();
  if (!ensure_work(g_cw, n)) return cudaErrorMemoryAllocation;
  if (g_cw.factor != L || g_cw.factor_n != n) {  // factor from elsewhere: build its Linv blocks
    k_trtri_blocks<<<(n + NB - 1) / NB, 256, kDynR, st>>>(n, L, lda, g_cw.Linv);
    count_launch();
    g_cw.factor = L;
    g_cw.factor_n = n;
  }
  static uint64_t attr_mask = 0;
  set_once_per_device(attr_mask, [] {
    return cudaFuncSetAttribute(k_inv_diag, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDyn);
  });
  k_inv_diag<<<(n + NB - 1) / NB, 256, kDyn, st>>>(n, L, lda, g_cw.Linv, se);
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
  CholCtx& g_cw = *cc;
  set_attrs();
  if (!ensure_work(g_cw, n)) return cudaErrorMemoryAllocation;
  if (g_cw.factor != L || g_cw.factor_n != n) {  // factor from elsewhere: build its Linv blocks
    k_trtri_blocks<<<(n + NB - 1) / NB, 256, kDynR, st>>>(n, L, lda, g_cw.Linv);
    count_launch();
    g_cw.factor = L;
    g_cw.factor_n = n;
  }
  if (x != b) cudaMemcpyAsync(x, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, st);
  cudaError_t e = launch_wave(g_cw, n, L, lda, x, 0, st);
  if (e != cudaSuccess) return e;
  return launch_wave(g_cw, n, L, lda, x, 1, st);
}

}  // namespace mnl
