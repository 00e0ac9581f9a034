// Shared by the pass-1 translation units (k_eval.cu, k_eval_w.cu): the kernel argument block and
// the small device helpers of rows a1-a4. Everything is in an anonymous
// namespace: each unit gets its own copy, nothing is exported.
#pragma once
#include <cmath>
#include <cstdint>

#include "internal.h"

namespace mnl {
namespace {

struct EvalArgs {
  int64_t N;
  int K, p, f, d, q, n_p, off_alpha, off_gamma, QP, XS, TI, SCR;
  int NS, SLOT;  // YZS path: ring slots per warp, doubles per slot (K (f + d))
  double* Rg;    // non-null (stream mode): residual rows r_i [N][K] for k_yz_grad, which then forms
                 // the alpha / gamma gradients by streaming Z and Y (many alternative-varying vars)
  const double* X;
  const double* Y;  // [N][K][f]
  const double* Z;  // [N][K][d]
  const int32_t* choice;
  const double* coef;
  double* Pr;
  int ldP;
  int want_grad;
  int writeP;
  double* part;
  int n_part;
  int* err;
};

__device__ __forceinline__ void neu_add(double& s, double& c, double x) {
  // Neumaier compensated summation (a3: R7 requires compensated loglik sums).
  double t = s + x;
  if (fabs(s) >= fabs(x)) c += (s - t) + x;
  else c += (x - t) + s;
  s = t;
}

// Coefficients of the exponentials below, in constant memory: they enter the DFMAs as constant-bank
// operands (no registers, no move instructions).
__constant__ double c_exp[15] = {1.4426950408889634,            // log2 e
                                 -6.93147180369123816490e-01,   // -ln2 (fdlibm's high part)
                                 -1.90821492927058770002e-10,   // -ln2 (low part)
                                 1.0 / 6.0,        0.5,
                                 1.0 / 120.0,      1.0 / 24.0,
                                 1.0 / 5040.0,     1.0 / 720.0,
                                 1.0 / 362880.0,   1.0 / 40320.0,
                                 1.0 / 39916800.0, 1.0 / 3628800.0,
                                 1.0 / 479001600.0, 1.0};

// 2^j for an integer j <= ~1000 (0 below the normal range)
__device__ __forceinline__ double pow2_int(int j) { return __hiloint2double((max(j, -1023) + 1023) << 20, 0); }

// e^r for |r| <= ~ln2/2: the Taylor polynomial to degree 12 (truncation < 2e-16 relative) in Estrin
// form (short dependency chain).
__device__ __forceinline__ double exp_poly(double r) {
  const double r2 = r * r, r4 = r2 * r2, r8 = r4 * r4;
  const double p01 = c_exp[14] + r;
  const double p23 = fma(r, c_exp[3], c_exp[4]);
  const double p45 = fma(r, c_exp[5], c_exp[6]);
  const double p67 = fma(r, c_exp[7], c_exp[8]);
  const double p89 = fma(r, c_exp[9], c_exp[10]);
  const double pab = fma(r, c_exp[11], c_exp[12]);
  const double q0 = fma(r2, p23, p01), q1 = fma(r2, p67, p45);
  const double q2 = fma(r2, pab, p89);
  const double s0 = fma(r4, q1, q0), s1 = fma(r4, c_exp[13], q2);
  return fma(r8, s1, s0);
}

// e^x for the shifted utilities x = u - m <= ~0 (a2). x = n ln2 + r (|r| <= ln2/2, Cody-Waite with
// fdlibm's split ln2, exact n ln2_hi), e^r by exp_poly, times 2^n built in the exponent field.
// Branch-free (a branch per call would serialise the calls of a lane's alternatives): x below
// -1000 (e^x = 0 in double; -inf for the alternatives >= K) is clamped, 2^n is 0 below the normal
// range (e^x < 2.2e-308), and a NaN propagates.
__device__ __forceinline__ double exp_shifted(double x) {
  const double xc = x < -1000.0 ? -1000.0 : x;
  const double t = rint(xc * c_exp[0]);
  double r = fma(t, c_exp[1], xc);
  r = fma(t, c_exp[2], r);
  return exp_poly(r) * pow2_int(__double2int_rn(t));
}

// 1 / s for the softmax row sums s >= ~1 (the shifted maximum contributes ~1): the hardware
// approximate reciprocal refined by two Newton steps (relative error <= ~1 ulp), instead of the
// ~15-instruction IEEE division.
__device__ __forceinline__ double recip_ge1(double s) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(s));
  double e = fma(-s, r, 1.0);
  r = fma(r, e, r);
  e = fma(-s, r, 1.0);
  return fma(r, e, r);
}

// Sums of 8 per-lane values over the warp (reduce-scatter by butterfly): returns, in every lane, the
// warp sum of component (lane >> 2) & 7.
__device__ __forceinline__ double warp_sum8(const double (&v)[8], int lane) {
  const bool h4 = lane & 16, h3 = lane & 8, h2 = lane & 4;
  double a[4], b[2], c;
#pragma unroll
  for (int t = 0; t < 4; ++t) {  // xor 16: keep components 4 h4 .. 4 h4 + 3
    const double keep = h4 ? v[4 + t] : v[t], send = h4 ? v[t] : v[4 + t];
    a[t] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int t = 0; t < 2; ++t) {  // xor 8: keep 2 of them
    const double keep = h3 ? a[2 + t] : a[t], send = h3 ? a[t] : a[2 + t];
    b[t] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  {  // xor 4: keep 1
    const double keep = h2 ? b[1] : b[0], send = h2 ? b[0] : b[1];
    c = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  }
  c += __shfl_xor_sync(0xffffffffu, c, 2);
  c += __shfl_xor_sync(0xffffffffu, c, 1);
  return c;  // component 4 h4 + 2 h3 + h2
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(bar))),
               "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned a, unsigned parity) {  // a: shared address
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}

}  // namespace
}  // namespace mnl
