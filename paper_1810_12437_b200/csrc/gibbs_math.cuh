// Conditional draws of the scan's scale updates (device), shared by the
// single-chain scan kernels, the validation entry point pcgs_scale_draws and
// the fused batched Gibbs kernel.
#pragma once
#include <cmath>

#include "device.cuh"

namespace pcgs {

// ---------------------------------------------------------------- scale updates
// Wald(mu, 1) (inverse Gaussian) by Michael-Schucany-Haas, in the
// cancellation-free form x = mu / (1 + a + sqrt(a (a + 2))), a = mu y / 2.
static __device__ double wald1(double mu, Philox& R) {
  const double nrm = R.normal();
  const double a = 0.5 * mu * nrm * nrm;
  const double x = mu / (1.0 + a + sqrt(a * (a + 2.0)));
  return R.uniform() <= mu / (mu + x) ? x : mu * mu / x;
}

// The conditional draws of the scale updates, shared by the scan kernels and
// the validation entry point pcgs_scale_draws.
//
// Global scale.  Bridge (gibbs.py:179-190): phi = tau^-alpha ~
// Gamma(a0 + p/alpha, b0 + sum|beta|^alpha), acc = that sum.  Horseshoe (new,
// DESIGN.md §5): xi | tau ~ IG(1, 1 + 1/tau^2), then tau^2 | beta, lam, xi ~
// IG((p+1)/2, 1/xi + acc/2), acc = sum beta^2 / lam^2; *xi receives xi.
static __device__ double global_draw(int prior, double a0, double b0, double alpha, long long p, double acc,
                              double tau_old, Philox& R, double* xi) {
  if (prior == 0) {
    const double phi = R.gamma(a0 + (double)p / alpha) / (b0 + acc);
    return alpha == 1.0 ? 1.0 / phi : pow(phi, -1.0 / alpha);
  }
  *xi = (1.0 + 1.0 / (tau_old * tau_old)) / R.exponential();
  const double tau2 = fmin(fmax((1.0 / *xi + 0.5 * acc) / R.gamma(0.5 * (double)(p + 1)), 1e-300), 1e300);
  return sqrt(tau2);
}

// Local scale of one coefficient b.  Bridge alpha = 1 (gibbs.py:193-214):
// 1/lam^2 ~ Wald(tau/|b|, 1), the |b|/tau < 1e-10 limit lam = |N(0,1)|
// floored at 1e-150, 1/lam^2 floored at 1e-300.  Horseshoe: nu ~
// IG(1, 1 + 1/lam_old^2), lam^2 ~ IG(1, 1/nu + b^2/(2 tau^2)) clamped to
// [1e-300, 1e300]; *nu receives nu.
static __device__ double local_draw(int prior, double b, double tau, double lam_old, Philox& R, double* nu) {
  if (prior == 0) {
    const double ratio = fabs(b) / tau;
    if (ratio < 1e-10) return fmax(fabs(R.normal()), 1e-150);
    const double inv_sq = wald1(1.0 / ratio, R);
    return pow(fmax(inv_sq, 1e-300), -0.5);
  }
  *nu = (1.0 + 1.0 / (lam_old * lam_old)) / R.exponential();
  const double lam2 = fmin(fmax((1.0 / *nu + 0.5 * b * b / (tau * tau)) / R.exponential(), 1e-300), 1e300);
  return sqrt(lam2);
}


}  // namespace pcgs
