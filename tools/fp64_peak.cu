// FP64 throughput microbenchmark for the roofline denominator.
// Measures, on all SMs, register-resident:
//   (1) DMMA  : mma.sync.aligned.m8n8k4.row.col.f64 (SASS DMMA.8x8x4), 256 FMA / instr / warp
//   (2) DFMA  : fma.rn.f64, 32 FMA / instr / warp
// for several warps-per-SM counts. Prints one JSON object.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

template <int NACC>
__global__ void k_dmma(double* out, int iters) {
  double a = 1.0 + 1e-9 * threadIdx.x, b = 1.0 - 1e-9 * threadIdx.x;
  double c[NACC][2];
#pragma unroll
  for (int j = 0; j < NACC; ++j) { c[j][0] = 0.0; c[j][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < NACC; ++j) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < NACC; ++j) s += c[j][0] + c[j][1];
  if (s == 12345.678) out[0] = s;  // keep live
}

template <int NACC>
__global__ void k_dfma(double* out, int iters) {
  double a = 1.0 + 1e-9 * threadIdx.x, b = 1.0 - 1e-9 * threadIdx.x;
  double c[NACC];
#pragma unroll
  for (int j = 0; j < NACC; ++j) c[j] = j;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < NACC; ++j) c[j] = fma(a, c[j], b);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < NACC; ++j) s += c[j];
  if (s == 12345.678) out[0] = s;
}

int main() {
  int dev = 0; cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, dev));
  int sms = prop.multiProcessorCount;
  double* out; CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"smem_optin\": %zu, \"results\": [\n", prop.name, sms, prop.l2CacheSize, prop.sharedMemPerBlockOptin);
  bool first = true;
  for (int kind = 0; kind < 2; ++kind) {
    for (int warps : {4, 8, 16, 32}) {
      int threads = 32 * warps;
      int iters = kind == 0 ? 20000 : 40000;
      const int NACC = 8;
      auto launch = [&]() {
        if (kind == 0) k_dmma<NACC><<<sms, threads>>>(out, iters);
        else k_dfma<NACC><<<sms, threads>>>(out, iters);
      };
      launch(); CK(cudaDeviceSynchronize());
      // sustained: repeat until ~2 s
      float best = 1e30f, total = 0; int reps = 0;
      while (total < 2000.f && reps < 200) {
        cudaEventRecord(e0); launch(); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1); total += ms; ++reps; if (ms < best) best = ms;
      }
      double fma_per_launch = (double)sms * warps * iters * NACC * (kind == 0 ? 256.0 : 32.0);
      double tf_best = 2.0 * fma_per_launch / (best * 1e-3) / 1e12;
      double tf_avg = 2.0 * fma_per_launch * reps / (total * 1e-3) / 1e12;
      printf("%s {\"kind\": \"%s\", \"warps_per_sm\": %d, \"tflops_best\": %.3f, \"tflops_avg\": %.3f, \"reps\": %d}\n",
             first ? "" : ",", kind == 0 ? "dmma_m8n8k4" : "dfma", warps, tf_best, tf_avg, reps);
      first = false;
    }
  }
  printf("]}\n");
  return 0;
}
