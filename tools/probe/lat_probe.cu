// Latency probe: dependent DFMA chain, rsqrt(double), __syncthreads (8 warps), shared round trip.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double seed) {
  __shared__ double sh[256];
  double a = seed + threadIdx.x * 1e-9, b = 1.0000001;
  sh[threadIdx.x] = a;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < 1000; ++i) a = fma(a, b, 1e-12);
  long long t1 = clock64();
  for (int i = 0; i < 100; ++i) a = rsqrt(a + 1.0);
  long long t2 = clock64();
  for (int i = 0; i < 100; ++i) __syncthreads();
  long long t3 = clock64();
  int idx = threadIdx.x;
  for (int i = 0; i < 100; ++i) { idx = (int)sh[(idx + 1) & 255] & 255; }
  long long t4 = clock64();
  for (int i = 0; i < 100; ++i) a = 1.0 / (a + 2.0);
  long long t5 = clock64();
  for (int i = 0; i < 100; ++i) a = a + __shfl_xor_sync(0xffffffffu, a, 1);
  long long t6 = clock64();
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5;
  }
  out[threadIdx.x] = a + idx;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8 * 256); cudaMalloc(&c, 8 * 8);
  for (int r = 0; r < 2; ++r) {
    k<<<1, 256>>>(o, c, 1.5);
    long long h[8]; cudaMemcpy(h, c, 64, cudaMemcpyDeviceToHost);
    printf("dfma chain %.1f cyc/op, rsqrt %.1f, syncthreads(8 warps) %.1f, smem roundtrip %.1f, ddiv %.1f, shfl+dadd %.1f\n",
           h[0] / 1000.0, h[1] / 100.0, h[2] / 100.0, h[3] / 100.0, h[4] / 100.0, h[5] / 100.0);
  }
}
