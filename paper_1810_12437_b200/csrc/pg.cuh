// Polya-Gamma PG(1, z) draws (device), shared by the single-chain and the
// fused batched Gibbs kernels.
#pragma once
#include <cmath>

#include "device.cuh"

namespace pcgs {

// =====================================================================
// Polya-Gamma PG(1, z) (restates polya_gamma.py:39-147 per thread)
// =====================================================================
static __device__ __forceinline__ double log_ndtr(double x) {
  if (x < -1.0) return log(0.5 * erfcx(-x * M_SQRT1_2)) - 0.5 * x * x;
  return log1p(-0.5 * erfc(x * M_SQRT1_2));
}
static __device__ __forceinline__ double logaddexp(double a, double b) {
  const double m = fmax(a, b);
  return m + log1p(exp(-fabs(a - b)));
}

static __device__ bool pg_series_accept(double x, Philox& R) {
  const double T = 0.64;
  const double u = R.uniform();
  const bool inside = x <= T;
  double partial = 1.0;
  for (int k = 1; k < 1000; ++k) {
    const double coef = 2.0 * k + 1.0;
    const double term = inside ? coef * exp(-2.0 * k * (k + 1.0) / x)
                               : coef * exp(-0.5 * k * (k + 1.0) * M_PI * M_PI * x);
    if (k & 1) {
      partial -= term;
      if (u <= partial) return true;
    } else {
      partial += term;
      if (!(u < partial)) return false;
    }
  }
  return false;
}

static __device__ double pg_trunc_ig(double h, Philox& R) {
  const double T = 0.64;
  if (h < 1.0 / T) {
    for (;;) {
      const double e1 = R.exponential(), e2 = R.exponential();
      if (e1 * e1 <= 2.0 * e2 / T) {
        const double q = 1.0 + T * e1;
        const double x = T / (q * q);
        if (R.uniform() <= exp(-0.5 * h * h * x)) return x;
      }
    }
  }
  const double mu = 1.0 / h;
  for (;;) {
    const double nrm = R.normal();
    const double y = nrm * nrm;
    double x = mu + 0.5 * mu * mu * y - 0.5 * mu * sqrt(4.0 * mu * y + (mu * y) * (mu * y));
    x = fmax(x, 1e-300);
    if (R.uniform() > mu / (mu + x)) x = mu * mu / x;
    if (x <= T) return x;
  }
}

static __device__ double pg_draw1(double z, Philox& R) {
  const double T = 0.64, SQT = 0.8;
  const double h = 0.5 * fabs(z);
  const double K = M_PI * M_PI / 8.0 + 0.5 * h * h;
  const double log_right = log(M_PI / (2.0 * K)) - K * T;
  const double log_left = M_LN2 + logaddexp(-h + log_ndtr((T * h - 1.0) / SQT), h + log_ndtr(-(T * h + 1.0) / SQT));
  const double prob_right = 1.0 / (1.0 + exp(-(log_right - log_left)));
  for (;;) {
    double x;
    if (R.uniform() < prob_right) x = T + R.exponential() / K;
    else x = pg_trunc_ig(h, R);
    if (pg_series_accept(x, R)) return 0.25 * x;
  }
}


}  // namespace pcgs
