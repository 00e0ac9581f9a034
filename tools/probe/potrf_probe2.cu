
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>
constexpr int NB = 64;
__global__ void __launch_bounds__(256) k_potrf_inv(int n, double* A, int lda, int j0, double* Linv, int* info,
                                                   double* x, long long* stamps) {
  long long t0 = clock64();
  __shared__ double colbuf[2][NB], rowbuf[2][NB], bv[NB];
  __shared__ double piv_s;
  const int jb = min(NB, n - j0);
  const int tid = threadIdx.x, r = tid >> 2, q = tid & 3;
  double Sr[16], Xr[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const int cc = q + 4 * k;
    Sr[k] = (r < jb && cc <= r) ? A[(int64_t)(j0 + r) * lda + j0 + cc] : 0.0;
    Xr[k] = (cc == r) ? 1.0 : 0.0;
  }
  if (x && tid < NB) bv[tid] = tid < jb ? x[j0 + tid] : 0.0;
  bool bad_any = false;
  for (int c = 0; c < jb; ++c) {
    if (tid == 0) stamps[c * 4 + 0] = clock64() - t0;
    const int par = c & 1, kc = c >> 2;
    const bool col_owner = (q == (c & 3));
    if (col_owner && r == c) {
      double v = 0.0;
#pragma unroll
      for (int k = 0; k < 16; ++k)
        if (k == kc) v = Sr[k];
      piv_s = v;
    }
    __syncthreads();
    if (tid == 0) stamps[c * 4 + 1] = clock64() - t0;
    const double piv = piv_s;
    const bool bad = !(piv > 0.0) || !isfinite(piv);
    bad_any |= bad;
    const double rd = bad ? 1.0 : rsqrt(piv);
    if (tid == 0) stamps[c * 4 + 2] = clock64() - t0 + (rd > 1e300 ? 1 : 0);
    if (col_owner && r >= c && r < jb) {
#pragma unroll
      for (int k = 0; k < 16; ++k)
        if (k == kc) {
          Sr[k] = (r == c) ? (bad ? 1.0 : piv * rd) : Sr[k] * rd;
          colbuf[par][r] = Sr[k];
        }
    }
    if (r == c) {
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const int j = q + 4 * k;
        if (j <= c) {
          Xr[k] *= rd;
          rowbuf[par][j] = Xr[k];
        }
      }
    }
    __syncthreads();
    if (tid == 0) stamps[c * 4 + 3] = clock64() - t0;
    if (r > c && r < jb) {
      const double lrc = colbuf[par][r];
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const int cc = q + 4 * k;
        if (cc > c && cc <= r) Sr[k] = fma(-lrc, colbuf[par][cc], Sr[k]);
        if (cc <= c) Xr[k] = fma(-lrc, rowbuf[par][cc], Xr[k]);
      }
    }
  }
  if (tid == 0 && bad_any) atomicCAS(info, 0, j0 + 1);
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const int cc = q + 4 * k;
    if (r < jb && cc <= r) A[(int64_t)(j0 + r) * lda + j0 + cc] = Sr[k];
    Linv[r * NB + cc] = (r < jb && cc <= r) ? Xr[k] : 0.0;  // [NB][NB], zero outside the triangle
  }
  if (x) {
    __syncthreads();
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 16; ++k)
      if (q + 4 * k <= r) s = fma(Xr[k], bv[q + 4 * k], s);
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    if (q == 0 && r < jb) x[j0 + r] = s;
  }
}


int main() {
  int n = 64, lda = 64;
  double* hA = new double[n * n];
  for (int i = 0; i < n; ++i) for (int j = 0; j < n; ++j) hA[i * n + j] = (i == j ? n : 0) + 1.0 / (1 + i + j);
  double *A, *Linv; int* info; long long* st;
  cudaMalloc(&A, 8 * n * n); cudaMalloc(&Linv, 8 * 64 * 64); cudaMalloc(&info, 4); cudaMalloc(&st, 8 * 300);
  cudaMemset(info, 0, 4);
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemcpy(A, hA, 8 * n * n, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_potrf_inv<<<1, 256>>>(n, A, lda, 0, Linv, info, nullptr, st);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long hs[300]; cudaMemcpy(hs, st, sizeof(hs), cudaMemcpyDeviceToHost);
    printf("rep %d: %.1f us\n", rep, ms * 1e3);
    for (int c : {1, 2, 32, 62}) printf("  step %d: sync1=%lld rsqrt=%lld scale+sync2=%lld update=%lld\n", c, hs[c*4+1]-hs[c*4], hs[c*4+2]-hs[c*4+1], hs[c*4+3]-hs[c*4+2], hs[c*4+4]-hs[c*4+3]);
  }
}
