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
#include <vector>

#include "internal.h"

namespace mnl {
namespace {

constexpr int NB = 64;
constexpr int LDS = NB + 4;  // 68 = 4 (mod 16) doubles: conflict-free 8x4 fragment gathers
constexpr int LDR = NB + 1;  // row-per-thread access patterns

// k_potrf_inv: right-looking Cholesky of the jb x jb diagonal block fused with X = L^{-1}, held in
// REGISTERS: thread t owns row r = t / 4 and the columns q + 4k (q = t % 4, k < 16) of both S and X.
// Step c: the owner of S[c][c] publishes the pivot; column c of L and row c of X are scaled by
// 1/sqrt(pivot) by their owners and broadcast through shared memory (double-buffered by step
// parity); every thread then updates its own elements:
//   S[r][cc] -= L[r][c] L[cc][c]  (c < cc <= r),   X[r][j] -= L[r][c] X[c][j]  (r > c, j <= c).
// Two barriers per step and no shared-memory read-modify-write.  With x != null it also applies
// the forward-solve piece y_j = Linv b_j (b_j already holds every earlier panel's update).
__global__ void __launch_bounds__(256) k_potrf_inv(int n, double* A, int lda, int j0, double* Linv, int* info,
                                                   double* x) {
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
    const double piv = piv_s;
    const bool bad = !(piv > 0.0) || !isfinite(piv);
    bad_any |= bad;
    const double rd = bad ? 1.0 : rsqrt(piv);
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

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
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

// rows [j0+jb + 64*blockIdx.x, +64): L21 = A21 Linv^T; with x: x_r -= L21_r . y_j
__global__ void __launch_bounds__(256) k_trsm_gemm(int n, double* A, int lda, int j0, const double* Linv, double* x) {
  extern __shared__ __align__(16) double dsm[];
  double(*Xs)[LDS] = reinterpret_cast<double(*)[LDS]>(dsm);
  double(*Ys)[LDS] = reinterpret_cast<double(*)[LDS]>(dsm + NB * LDS);
  __shared__ double yv[NB];
  const int jb = min(NB, n - j0);
  const int r0 = j0 + jb + blockIdx.x * NB;
  const int tid = threadIdx.x;
  for (int e = tid; e < NB * NB; e += 256) {
    const int r = e >> 6, c = e & 63;
    Xs[r][c] = (r0 + r < n && c < jb) ? A[(int64_t)(r0 + r) * lda + j0 + c] : 0.0;
    Ys[r][c] = Linv[e];
  }
  if (x && tid < NB) yv[tid] = tid < jb ? x[j0 + tid] : 0.0;
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
    if (q4 == 0 && r0 + r < n) x[r0 + r] -= s;
  }
}

// trailing update: lower tiles (ti >= tj) of A22 -= L21 L21^T.
// col_only = 1: only block-column 0 of the trailing matrix (the next panel, lookahead path);
// col_only = 0: the lower triangle starting at tile (first, first).
__global__ void __launch_bounds__(256) k_syrk_tiles(int n, double* A, int lda, int j0, int col_only, int first) {
  extern __shared__ __align__(16) double dsm[];
  double(*Li)[LDS] = reinterpret_cast<double(*)[LDS]>(dsm);
  double(*Lj)[LDS] = reinterpret_cast<double(*)[LDS]>(dsm + NB * LDS);
  const int jb = min(NB, n - j0);
  const int s0 = j0 + jb;
  int ti, tj;
  if (col_only) {
    ti = blockIdx.x;
    tj = 0;
  } else {
    const int t = blockIdx.x;  // -> (ti, tj), ti >= tj, row-major over the lower triangle
    ti = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
    while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
    while (ti * (ti + 1) / 2 > t) --ti;
    tj = t - ti * (ti + 1) / 2;
    ti += first;
    tj += first;
  }
  const int ri = s0 + ti * NB, rj = s0 + tj * NB;
  const int tid = threadIdx.x;
  for (int e = tid; e < NB * NB; e += 256) {
    const int r = e >> 6, c = e & 63;
    Li[r][c] = (ri + r < n && c < jb) ? A[(int64_t)(ri + r) * lda + j0 + c] : 0.0;
    Lj[r][c] = (rj + r < n && c < jb) ? A[(int64_t)(rj + r) * lda + j0 + c] : 0.0;
  }
  __syncthreads();
  double acc[2][4][2];
  tile_xyT(Li, Lj, acc);
  const int lane = tid & 31, w = tid >> 5;
  const int wr = (w >> 1) * 16, wc = (w & 1) * 32, lr = lane >> 2, lk = lane & 3;
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

struct CholWork {
  double* Linv = nullptr;
  size_t cap = 0;
  const double* factor = nullptr;  // matrix whose Linv blocks are current
  int factor_n = 0;
  int* flags = nullptr;
  int nflags = 0;
  int epoch = 0;
};
CholWork g_cw;

bool ensure_work(int n) {
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
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_trsm_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDyn);
    cudaFuncSetAttribute(k_syrk_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDyn);
    cudaFuncSetAttribute(k_trtri_blocks, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDynR);
    attr = true;
  }
}

cudaError_t launch_wave(int n, const double* L, int lda, double* x, int upper, cudaStream_t st) {
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

struct Lookahead {
  cudaStream_t side = nullptr;
  std::vector<cudaEvent_t> ev;
  cudaEvent_t start = nullptr, done = nullptr;
};
Lookahead g_la;

cudaEvent_t la_event(size_t i) {
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
cudaError_t factor(int n, double* A, int lda, int* info, double* x, cudaStream_t st) {
  set_attrs();
  if (!ensure_work(n)) return cudaErrorMemoryAllocation;
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
    k_potrf_inv<<<1, 256, 0, sp>>>(n, A, lda, j0, Lj, info, x);
    count_launch();
    const int rem = n - j0 - jb;
    if (rem > 0) {
      k_trsm_gemm<<<(rem + NB - 1) / NB, 256, kDyn, sp>>>(n, A, lda, j0, Lj, x);
      count_launch();
    }
  };
  panel(0);
  cudaEventRecord(la_event(2 * 0), sp);  // ev_p(0)
  for (int j = 0; j + 1 < np; ++j) {
    const int j0 = j * NB;
    const int rem = n - j0 - NB;
    const int mt = (rem + NB - 1) / NB;
    // main: rest of panel j's trailing update (tiles with tj >= 1)
    cudaStreamWaitEvent(st, la_event(2 * j), 0);
    if (mt > 1) {
      k_syrk_tiles<<<(mt - 1) * mt / 2, 256, kDyn, st>>>(n, A, lda, j0, 0, 1);
      count_launch();
    }
    cudaEventRecord(la_event(2 * j + 1), st);  // ev_r(j)
    // side: next panel's block column, then its factorisation
    k_syrk_tiles<<<mt, 256, kDyn, sp>>>(n, A, lda, j0, 1, 0);
    count_launch();
    panel(j + 1);
    cudaEventRecord(la_event(2 * (j + 1)), sp);  // ev_p(j+1)
    // the next column update (side, iteration j+1) must follow this rest update (main)
    cudaStreamWaitEvent(sp, la_event(2 * j + 1), 0);
  }
  cudaEventRecord(g_la.done, sp);
  cudaStreamWaitEvent(st, g_la.done, 0);
  g_cw.factor = A;
  g_cw.factor_n = n;
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_cholesky(int n, double* A, int lda, int* info, cudaStream_t st) {
  return factor(n, A, lda, info, nullptr, st);
}

cudaError_t launch_cholesky_solve_fused(int n, double* A, int lda, int* info, const double* b, double* x,
                                        cudaStream_t st) {
  if (x != b) cudaMemcpyAsync(x, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, st);
  cudaError_t e = factor(n, A, lda, info, x, st);
  if (e != cudaSuccess) return e;
  return launch_wave(n, A, lda, x, 1, st);
}

cudaError_t launch_chol_solve(int n, const double* L, int lda, const double* b, double* x, cudaStream_t st) {
  set_attrs();
  if (!ensure_work(n)) return cudaErrorMemoryAllocation;
  if (g_cw.factor != L || g_cw.factor_n != n) {  // factor from elsewhere: build its Linv blocks
    k_trtri_blocks<<<(n + NB - 1) / NB, 256, kDynR, st>>>(n, L, lda, g_cw.Linv);
    count_launch();
    g_cw.factor = L;
    g_cw.factor_n = n;
  }
  if (x != b) cudaMemcpyAsync(x, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, st);
  cudaError_t e = launch_wave(n, L, lda, x, 0, st);
  if (e != cudaSuccess) return e;
  return launch_wave(n, L, lda, x, 1, st);
}

}  // namespace mnl
