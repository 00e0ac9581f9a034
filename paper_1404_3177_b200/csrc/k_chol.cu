// Newton step: -H = L L^T by a blocked right-looking Cholesky
// factorisation, then L y = g and L^T delta = y (Eq. "NR update": delta = -H^{-1} g;
// -H is positive definite by global concavity).
//
// Per panel of NB = 64 columns:  potrf of the diagonal block in one CTA (shared memory),
// trsm of the panel below it (one CTA per 64 rows), and the trailing lower-triangular update
// A22 -= L21 L21^T as 64 x 64 DMMA tiles (mma.sync m8n8k4 f64), one CTA per lower tile.
// The matrix is row-major with leading dimension lda; only the lower triangle is referenced.
#include <algorithm>
#include <cmath>

#include "internal.h"

namespace mnl {
namespace {

constexpr int NB = 64;
constexpr int LDS = NB + 4;  // smem leading dimension (== 4 mod 16 doubles: conflict-free frags)

__global__ void __launch_bounds__(256) k_potrf_diag(int n, double* A, int lda, int j0, int* info) {
  __shared__ double S[NB][LDS];
  const int jb = min(NB, n - j0);
  const int tid = threadIdx.x;
  for (int e = tid; e < NB * NB; e += 256) {
    const int r = e / NB, c = e % NB;
    S[r][c] = (r < jb && c <= r) ? A[(int64_t)(j0 + r) * lda + j0 + c] : 0.0;
  }
  __syncthreads();
  for (int c = 0; c < jb; ++c) {
    const double piv = S[c][c];
    const bool bad = !(piv > 0.0) || !isfinite(piv);
    const double dc = bad ? 1.0 : sqrt(piv);
    __syncthreads();
    if (tid == 0) {
      if (bad && *info == 0) *info = j0 + c + 1;
      S[c][c] = dc;
    }
    for (int r = c + 1 + tid; r < jb; r += 256) S[r][c] /= dc;
    __syncthreads();
    // rank-1 update of the trailing lower part of the block
    const int m = jb - c - 1;
    for (int e = tid; e < m * m; e += 256) {
      const int r = c + 1 + e / m, cc = c + 1 + e % m;
      if (cc <= r) S[r][cc] -= S[r][c] * S[cc][c];
    }
    __syncthreads();
  }
  for (int e = tid; e < jb * jb; e += 256) {
    const int r = e / jb, c = e % jb;
    if (c <= r) A[(int64_t)(j0 + r) * lda + j0 + c] = S[r][c];
  }
}

// rows [j0+jb + 64*blockIdx.x, +64): L21 = A21 L11^{-T}
__global__ void __launch_bounds__(256) k_trsm_panel(int n, double* A, int lda, int j0) {
  extern __shared__ __align__(16) double dsm[];
  double(*Lk)[LDS] = reinterpret_cast<double(*)[LDS]>(dsm);
  double(*X)[LDS] = reinterpret_cast<double(*)[LDS]>(dsm + NB * LDS);
  const int jb = min(NB, n - j0);
  const int r0 = j0 + jb + blockIdx.x * NB;
  const int rows = min(NB, n - r0);
  const int tid = threadIdx.x;
  for (int e = tid; e < NB * NB; e += 256) {
    const int r = e / NB, c = e % NB;
    Lk[r][c] = (r < jb && c <= r) ? A[(int64_t)(j0 + r) * lda + j0 + c] : 0.0;
    X[r][c] = (r < rows && c < jb) ? A[(int64_t)(r0 + r) * lda + j0 + c] : 0.0;
  }
  __syncthreads();
  // x L^T = a  column by column: x_c = (a_c - sum_{t<c} x_t L_ct) / L_cc
  for (int c = 0; c < jb; ++c) {
    const double inv = 1.0 / Lk[c][c];
    for (int r = tid; r < rows; r += 256) X[r][c] *= inv;
    __syncthreads();
    const int m = jb - c - 1;
    for (int e = tid; e < rows * m; e += 256) {
      const int r = e / m, cc = c + 1 + e % m;
      X[r][cc] -= X[r][c] * Lk[cc][c];
    }
    __syncthreads();
  }
  for (int e = tid; e < rows * jb; e += 256) {
    const int r = e / jb, c = e % jb;
    A[(int64_t)(r0 + r) * lda + j0 + c] = X[r][c];
  }
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// trailing update: lower tiles (ti >= tj) of A22 -= L21 L21^T, A22 starting at row/col s0
__global__ void __launch_bounds__(256) k_syrk_tiles(int n, double* A, int lda, int j0) {
  extern __shared__ __align__(16) double dsm[];
  double(*Li)[LDS] = reinterpret_cast<double(*)[LDS]>(dsm);
  double(*Lj)[LDS] = reinterpret_cast<double(*)[LDS]>(dsm + NB * LDS);
  const int jb = min(NB, n - j0);
  const int s0 = j0 + jb;
  // blockIdx.x -> (ti, tj), ti >= tj, row-major over the lower triangle
  int t = blockIdx.x, ti = 0;
  while (t > ti) { t -= ti + 1; ++ti; }
  const int tj = t;
  const int ri = s0 + ti * NB, rj = s0 + tj * NB;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  for (int e = tid; e < NB * NB; e += 256) {
    const int r = e / NB, c = e % NB;
    Li[r][c] = (ri + r < n && c < jb) ? A[(int64_t)(ri + r) * lda + j0 + c] : 0.0;
    Lj[r][c] = (rj + r < n && c < jb) ? A[(int64_t)(rj + r) * lda + j0 + c] : 0.0;
  }
  __syncthreads();
  // warp tile 16 (rows) x 32 (cols): warps 4 x 2
  const int wr = (w >> 1) * 16, wc = (w & 1) * 32;
  double acc[2][4][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  const int lr = lane >> 2, lk = lane & 3;
  for (int k0 = 0; k0 < NB; k0 += 4) {
    double af[2], bf[4];
#pragma unroll
    for (int a = 0; a < 2; ++a) af[a] = Li[wr + a * 8 + lr][k0 + lk];
#pragma unroll
    for (int b = 0; b < 4; ++b) bf[b] = Lj[wc + b * 8 + lr][k0 + lk];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
  }
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = ri + wr + a * 8 + lr, c = rj + wc + b * 8 + 2 * lk + h;
        if (r < n && c < n && c <= r) A[(int64_t)r * lda + c] -= acc[a][b][h];
      }
}

// ---- triangular solves -------------------------------------------------------------------
// forward: y_j = L_jj^{-1} b_j  (one CTA), then b[r] -= L[r, j-block] y_j for r below
__global__ void __launch_bounds__(64) k_trsv_lower_diag(int n, const double* L, int lda, int j0, double* x) {
  __shared__ double Ls[NB][NB + 1];
  __shared__ double v[NB];
  const int jb = min(NB, n - j0);
  const int tid = threadIdx.x;
  for (int e = tid; e < NB * NB; e += 64) {
    const int r = e / NB, c = e % NB;
    Ls[r][c] = (r < jb && c <= r) ? L[(int64_t)(j0 + r) * lda + j0 + c] : 0.0;
  }
  if (tid < jb) v[tid] = x[j0 + tid];
  __syncthreads();
  for (int c = 0; c < jb; ++c) {
    if (tid == c) v[c] /= Ls[c][c];
    __syncthreads();
    if (tid > c && tid < jb) v[tid] -= Ls[tid][c] * v[c];
    __syncthreads();
  }
  if (tid < jb) x[j0 + tid] = v[tid];
}
__global__ void __launch_bounds__(256) k_gemv_lower_update(int n, const double* L, int lda, int j0, double* x) {
  // rows r >= j0 + jb: x[r] -= sum_t L[r][j0+t] x[j0+t]; one warp per row
  const int jb = min(NB, n - j0);
  const int lane = threadIdx.x & 31;
  const int r = j0 + jb + blockIdx.x * 8 + (threadIdx.x >> 5);
  if (r >= n) return;
  double s = 0.0;
  for (int t = lane; t < jb; t += 32) s = fma(L[(int64_t)r * lda + j0 + t], x[j0 + t], s);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) x[r] -= s;
}
// backward: x_j = L_jj^{-T} y_j (one CTA), then y[r] -= sum_t L[j0+t][r] x_j[t] for r < j0
__global__ void __launch_bounds__(64) k_trsv_upper_diag(int n, const double* L, int lda, int j0, double* x) {
  __shared__ double Ls[NB][NB + 1];
  __shared__ double v[NB];
  const int jb = min(NB, n - j0);
  const int tid = threadIdx.x;
  for (int e = tid; e < NB * NB; e += 64) {
    const int r = e / NB, c = e % NB;
    Ls[r][c] = (r < jb && c <= r) ? L[(int64_t)(j0 + r) * lda + j0 + c] : 0.0;
  }
  if (tid < jb) v[tid] = x[j0 + tid];
  __syncthreads();
  for (int c = jb - 1; c >= 0; --c) {
    if (tid == c) v[c] /= Ls[c][c];
    __syncthreads();
    if (tid < c) v[tid] -= Ls[c][tid] * v[c];
    __syncthreads();
  }
  if (tid < jb) x[j0 + tid] = v[tid];
}
__global__ void __launch_bounds__(256) k_gemv_upper_update(int n, const double* L, int lda, int j0, double* x) {
  // r < j0: x[r] -= sum_t L[j0+t][r] x[j0+t]   (rows of L are contiguous in r: coalesced)
  const int jb = min(NB, n - j0);
  const int r = blockIdx.x * 256 + threadIdx.x;
  if (r >= j0) return;
  double s = 0.0;
  for (int t = 0; t < jb; ++t) s = fma(L[(int64_t)(j0 + t) * lda + r], x[j0 + t], s);
  x[r] -= s;
}

}  // namespace

cudaError_t launch_cholesky(int n, double* A, int lda, int* info, cudaStream_t st) {
  constexpr size_t kDyn = 2 * NB * LDS * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_trsm_panel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDyn);
    cudaFuncSetAttribute(k_syrk_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDyn);
    attr = true;
  }
  cudaMemsetAsync(info, 0, sizeof(int), st);
  for (int j0 = 0; j0 < n; j0 += NB) {
    const int jb = std::min(NB, n - j0);
    k_potrf_diag<<<1, 256, 0, st>>>(n, A, lda, j0, info);
    count_launch();
    const int rem = n - j0 - jb;
    if (rem > 0) {
      const int mt = (rem + NB - 1) / NB;
      k_trsm_panel<<<mt, 256, kDyn, st>>>(n, A, lda, j0);
      k_syrk_tiles<<<mt * (mt + 1) / 2, 256, kDyn, st>>>(n, A, lda, j0);
      count_launch(2);
    }
  }
  return cudaGetLastError();
}

cudaError_t launch_chol_solve(int n, const double* L, int lda, const double* b, double* x, cudaStream_t st) {
  if (x != b) cudaMemcpyAsync(x, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, st);
  for (int j0 = 0; j0 < n; j0 += NB) {
    k_trsv_lower_diag<<<1, 64, 0, st>>>(n, L, lda, j0, x);
    const int jb = std::min(NB, n - j0);
    const int rem = n - j0 - jb;
    count_launch();
    if (rem > 0) {
      k_gemv_lower_update<<<(rem + 7) / 8, 256, 0, st>>>(n, L, lda, j0, x);
      count_launch();
    }
  }
  const int last = ((n - 1) / NB) * NB;
  for (int j0 = last; j0 >= 0; j0 -= NB) {
    k_trsv_upper_diag<<<1, 64, 0, st>>>(n, L, lda, j0, x);
    count_launch();
    if (j0 > 0) {
      k_gemv_upper_update<<<(j0 + 255) / 256, 256, 0, st>>>(n, L, lda, j0, x);
      count_launch();
    }
  }
  return cudaGetLastError();
}

}  // namespace mnl
