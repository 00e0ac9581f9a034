
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>
constexpr int NB = 64, LDR = NB + 1;
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
constexpr int SB = 16;
template <int C>
__device__ __forceinline__ void chol16_step(double (&d)[16], bool isS, int r, bool& bad_any) {
  const double piv = __shfl_sync(0xffffffffu, d[C], C);
  const bool bad = !(piv > 0.0) || !isfinite(piv);
  bad_any |= bad;
  const double rd = bad ? 1.0 : rsqrt(piv);
  if (isS) {
    if (r == C) d[C] = bad ? 1.0 : piv * rd;
    else if (r > C) d[C] *= rd;
  } else if (r == C) {
#pragma unroll
    for (int j = 0; j <= C; ++j) d[j] *= rd;
  }
#pragma unroll
  for (int cc = C + 1; cc < 16; ++cc) {
    const double lcc = __shfl_sync(0xffffffffu, d[C], cc);
    if (isS && r >= cc) d[cc] = fma(-d[C], lcc, d[cc]);
  }
  const double lrc = __shfl_sync(0xffffffffu, d[C], r);  // L[r][C] from S-lane r
#pragma unroll
  for (int j = 0; j <= C; ++j) {
    const double xcj = __shfl_sync(0xffffffffu, d[j], 16 + C);
    if (!isS && r > C) d[j] = fma(-lrc, xcj, d[j]);
  }
  if constexpr (C + 1 < 16) chol16_step<C + 1>(d, isS, r, bad_any);
}

__global__ void __launch_bounds__(256) k_potrf_inv(int n, double* A, int lda, int j0, double* Linv, int* info,
                                                   double* x, long long* st) {
  long long t0 = clock64();
  extern __shared__ __align__(16) double dsm[];
  double(*S)[LDR] = reinterpret_cast<double(*)[LDR]>(dsm);
  double(*X)[LDR] = reinterpret_cast<double(*)[LDR]>(dsm + NB * LDR);
  __shared__ double T[NB][SB + 1];
  __shared__ double bv[NB];
  const int jb = min(NB, n - j0);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  for (int e = tid; e < NB * NB; e += 256) {
    const int r = e >> 6, c = e & 63;
    // rows / columns beyond jb: identity (keeps the blocked steps well defined; never written back)
    S[r][c] = (r < jb && c <= r) ? A[(int64_t)(j0 + r) * lda + j0 + c] : (r == c ? 1.0 : 0.0);
    X[r][c] = 0.0;
  }
  if (x && tid < NB) bv[tid] = tid < jb ? x[j0 + tid] : 0.0;
  __syncthreads();
  bool bad_any = false;
  if (tid == 0) st[0] = clock64() - t0;
  for (int c0 = 0; c0 < NB; c0 += SB) {
    // (1) warp 0: 16 x 16 diagonal block and its inverse, in registers
    if (w == 0) {
      const bool isS = lane < SB;
      const int r = lane & (SB - 1);
      double d[SB];
#pragma unroll
      for (int j = 0; j < SB; ++j) d[j] = isS ? (j <= r ? S[c0 + r][c0 + j] : 0.0) : (j == r ? 1.0 : 0.0);
      chol16_step<0>(d, isS, r, bad_any);
#pragma unroll
      for (int j = 0; j < SB; ++j) {
        if (isS) {
          if (j <= r) S[c0 + r][c0 + j] = d[j];
        } else {
          X[c0 + r][c0 + j] = (j <= r) ? d[j] : 0.0;
        }
      }
    }
    __syncthreads();
    if (tid == 0) st[1 + c0 / SB * 3] = clock64() - t0;
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
      if (tid == 0) st[2 + c0 / SB * 3] = clock64() - t0;
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
  if (tid == 0) st[13] = clock64() - t0;
  if (tid == 0 && bad_any) atomicCAS(info, 0, j0 + 1);
  // (4) off-diagonal blocks of X = L^{-1}: X_ij = -X_ii sum_{k=j}^{i-1} L_ik X_kj, block rows in order
  for (int bi = 1; bi < NB / SB; ++bi) {
    const int i0 = bi * SB;
    // T[j-cols] = sum_k L_ik X_kj for all j < i0 (16 x i0), then X_i,<i0 = -X_ii T
    for (int e = tid; e < SB * i0; e += 256) {
      const int ii = e / i0, jj = e % i0;
      double acc = 0.0;
      for (int t = (jj / SB) * SB; t < i0; ++t) acc = fma(S[i0 + ii][t], X[t][jj], acc);
      T[jj][ii] = acc;
    }
    __syncthreads();
    for (int e = tid; e < SB * i0; e += 256) {
      const int ii = e / i0, jj = e % i0;
      double acc = 0.0;
      for (int t = 0; t <= ii; ++t) acc = fma(X[i0 + ii][i0 + t], T[jj][t], acc);
      X[i0 + ii][jj] = -acc;
    }
    __syncthreads();
  }
  if (tid == 0) st[14] = clock64() - t0;
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


int main() {
  int n = 64, lda = 64;
  double* hA = new double[n * n];
  for (int i = 0; i < n; ++i) for (int j = 0; j < n; ++j) hA[i * n + j] = (i == j ? n : 0) + 1.0 / (1 + i + j);
  double *A, *Linv; int* info; long long* st;
  cudaMalloc(&A, 8 * n * n); cudaMalloc(&Linv, 8 * 64 * 64); cudaMalloc(&info, 4); cudaMalloc(&st, 8 * 32);
  cudaFuncSetAttribute(k_potrf_inv, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 64 * 65 * 8);
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemcpy(A, hA, 8 * n * n, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_potrf_inv<<<1, 256, 2 * 64 * 65 * 8>>>(n, A, lda, 0, Linv, info, nullptr, st);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long h[32]; cudaMemcpy(h, st, sizeof(h), cudaMemcpyDeviceToHost);
    printf("rep %d %.1f us: load %lld | ", rep, ms * 1e3, h[0]);
    long long prev = h[0];
    for (int s = 0; s < 4; ++s) { printf("sp%d: diag %lld trsm %lld syrk %lld | ", s, h[1+3*s]-prev, h[2+3*s]-h[1+3*s], (s<3? h[3+3*s+1-1]:h[13]) - h[2+3*s]); prev = (s<3? h[1+3*(s+1)] - 0 : h[13]); }
    printf("inv %lld total %lld\n", h[14]-h[13], h[14]);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
