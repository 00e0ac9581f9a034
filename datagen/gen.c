/* Seeded synthetic input generator shared by the oracle tests, the GPU parity
 * tests and bench.py.
 *
 * This module holds NONE of the estimator's arithmetic (no softmax, log-
 * likelihood, gradient, Hessian or Newton step).  It draws the data arrays and
 * the true coefficients, and samples each individual's choice from the random-
 * utility model the paper states: the observed utility U_ik (PAPER.md:104-107,
 * Eq. "unormalized utility"; ABI letters) plus i.i.d. Gumbel
 * unobserved utility, the choice being the alternative of
 * maximum total utility (utility maximisation principle).
 *
 * RNG: counter-based.  value(stream, j) = mix64(key(seed, stream) + (j+1)*phi),
 * mix64 = the SplitMix64 finaliser.  Every array is its own stream, drawn in
 * row-major order, so the arrays are identical for any thread count.
 * Uniform(0,1): (u64 >> 11) * 2^-53, shifted by 2^-54 so it never hits 0 or 1.
 * Normal: Box-Muller on draws (2j, 2j+1) of the stream, cosine branch only.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#define PHI 0x9E3779B97F4A7C15ULL

static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
static inline uint64_t stream_key(uint64_t seed, uint64_t stream) {
  return mix64(seed * 0xD1B54A32D192ED03ULL + mix64(stream + 0x632BE59BD9B4E019ULL));
}
static inline double u01(uint64_t key, uint64_t j) {
  uint64_t z = mix64(key + (j + 1) * PHI);
  return ((double)(z >> 11) + 0.5) * 0x1.0p-53;
}
static inline double nrm(uint64_t key, uint64_t j) {
  double a = u01(key, 2 * j), b = u01(key, 2 * j + 1);
  return sqrt(-2.0 * log(a)) * cos(6.283185307179586476925 * b);
}

/* dist: 0 = Normal(0, scale), 1 = Uniform(-scale, scale), 2 = Bernoulli(scale) in {0,1} */
void gen_fill(double* out, int64_t n, uint64_t seed, uint64_t stream, int dist, double scale) {
  uint64_t key = stream_key(seed, stream);
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < n; ++j) {
    if (dist == 0) out[j] = scale * nrm(key, (uint64_t)j);
    else if (dist == 1) out[j] = scale * (2.0 * u01(key, (uint64_t)j) - 1.0);
    else out[j] = u01(key, (uint64_t)j) < scale ? 1.0 : 0.0;
  }
}

/* Same as gen_fill(dist=0/1/2) but writes only column `col` of a row-major
 * [rows][ncols] matrix (used for c3's Bernoulli columns). */
void gen_fill_col(double* out, int64_t rows, int64_t ncols, int64_t col, uint64_t seed,
                  uint64_t stream, int dist, double scale) {
  uint64_t key = stream_key(seed, stream);
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < rows; ++j) {
    double v;
    if (dist == 0) v = scale * nrm(key, (uint64_t)j);
    else if (dist == 1) v = scale * (2.0 * u01(key, (uint64_t)j) - 1.0);
    else v = u01(key, (uint64_t)j) < scale ? 1.0 : 0.0;
    out[j * ncols + col] = v;
  }
}

/* Sample choice[i] = argmax_k (U_ik + G_ik), G_ik ~ Gumbel(0,1) i.i.d.
 * U_ik = xi_k + x_i.beta_k + z_ik.alpha_k + y_ik.gamma  (xi_0 = 0, beta_0 = 0),
 * with coef in the ABI layout of SURVEY.md §0.3:
 *   [beta_1 | ... | beta_{K-1} | alpha_0 | ... | alpha_{K-1} | gamma],
 *   beta_k = [xi_k, beta_k1..beta_kp]. */
void gen_choices(int64_t N, int32_t K, int32_t p, int32_t f, int32_t d,
                 const double* X, const double* Y, const double* Z, const double* coef,
                 uint64_t seed, uint64_t stream, int32_t* choice) {
  uint64_t key = stream_key(seed, stream);
  const int64_t q = (int64_t)p + 1;
  const int64_t off_a = (int64_t)(K - 1) * q, off_g = off_a + (int64_t)K * d;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < N; ++i) {
    double best = -INFINITY; int arg = 0;
    for (int k = 0; k < K; ++k) {
      double u = 0.0;
      if (k >= 1) {
        const double* b = coef + (int64_t)(k - 1) * q;
        u = b[0];
        for (int a = 0; a < p; ++a) u += X[i * p + a] * b[1 + a];
      }
      for (int c = 0; c < d; ++c) u += Z[(i * K + k) * d + c] * coef[off_a + (int64_t)k * d + c];
      for (int e = 0; e < f; ++e) u += Y[(i * K + k) * f + e] * coef[off_g + e];
      double g = -log(-log(u01(key, (uint64_t)(i * K + k))));
      if (u + g > best) { best = u + g; arg = k; }
    }
    choice[i] = arg;
  }
}
