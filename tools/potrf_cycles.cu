// potrf_core cycle probe (the 64 x 64 diagonal-tile factorisation of k_chol_dag): includes k_chol.cu
// and times potrf_core with clock64 on a random SPD block, plus warp 0's per-block timeline.
// Build + run (GPU): nvcc -gencode arch=compute_100a,code=sm_100a -O3 \
//   -Ipaper_1404_3177_b200/csrc -o /tmp/potrf_cycles tools/potrf_cycles.cu && /tmp/potrf_cycles
#ifndef SRC
#define SRC "../paper_1404_3177_b200/csrc/k_chol.cu"
#endif
#include <mutex>
__device__ long long g_tr[10];
#define POTRF_TRACE(i) if ((threadIdx.x & 31) == 0 && threadIdx.x == 0) g_tr[i] = clock64();
#include SRC
#include <cstdio>
#include <vector>
#include <cmath>
namespace mnl { namespace {
__global__ void __launch_bounds__(256, 1) k_probe(const double* A, int jb, double* outL, double* outX, long long* cyc) {
  extern __shared__ __align__(16) double dsm[];
  double(*S)[LDR] = reinterpret_cast<double(*)[LDR]>(dsm);
  double(*X)[LDR] = reinterpret_cast<double(*)[LDR]>(dsm + NB * LDR);
  long long best = 1LL << 60;
  for (int rep = 0; rep < 20; ++rep) {
    for (int e = threadIdx.x; e < NB * NB; e += 256) {
      const int r = e >> 6, c = e & 63;
      S[r][c] = (r < jb && c <= r) ? A[e] : (r == c && r >= jb ? 1.0 : 0.0);
    }
    __syncthreads();
    long long t0 = clock64();
    potrf_core(jb, dsm);
    long long t1 = clock64();
    if (t1 - t0 < best) best = t1 - t0;
    __syncthreads();
  }
  for (int e = threadIdx.x; e < NB * NB; e += 256) { outL[e] = S[e >> 6][e & 63]; outX[e] = X[e >> 6][e & 63]; }
  if (threadIdx.x == 0) *cyc = best;
}
}}
int main() {
  using namespace mnl;
  const int n = 64;
  std::vector<double> A(n * n), G(n * n);
  srand(3);
  for (auto& g : G) g = rand() / (double)RAND_MAX - 0.5;
  for (int i = 0; i < n; ++i) for (int j = 0; j < n; ++j) { double s = 0; for (int k = 0; k < n; ++k) s += G[i*n+k]*G[j*n+k]; A[i*n+j] = s + (i==j ? n : 0); }
  double *dA, *dL, *dX; long long* dc;
  cudaMalloc(&dA, 8*n*n); cudaMalloc(&dL, 8*n*n); cudaMalloc(&dX, 8*n*n); cudaMalloc(&dc, 8);
  cudaMemcpy(dA, A.data(), 8*n*n, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * NB * LDR * 8);
  for (int jb : {16, 18, 40, 64}) {
    k_probe<<<1, 256, 2 * NB * LDR * 8>>>(dA, jb, dL, dX, dc);
    std::vector<double> L(n*n), X(n*n); long long cyc;
    cudaMemcpy(L.data(), dL, 8*n*n, cudaMemcpyDeviceToHost); cudaMemcpy(X.data(), dX, 8*n*n, cudaMemcpyDeviceToHost);
    cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
    double e1 = 0, e2 = 0;
    for (int i = 0; i < jb; ++i) for (int j = 0; j <= i; ++j) {
      double s = 0; for (int k = 0; k <= j; ++k) s += L[i*n+k]*L[j*n+k]; e1 = fmax(e1, fabs(s - A[i*n+j]));
      double t = 0; for (int k = j; k <= i; ++k) t += X[i*n+k]*L[k*n+j]; e2 = fmax(e2, fabs(t - (i==j)));
    }
    long long tr[10]; cudaMemcpyFromSymbol(tr, g_tr, sizeof(tr));
    for (int i = 1; i < 10; ++i) printf(" %lld", tr[i] - tr[0]); printf("\n");
    printf("jb=%d cycles=%lld |LL^T-A|=%.2e |XL-I|=%.2e err=%s\n", jb, cyc, e1, e2, cudaGetErrorString(cudaGetLastError()));
  }
}
std::mutex& mnl::attr_mutex() { static std::mutex m; return m; }
void mnl::count_launch(int) {}
