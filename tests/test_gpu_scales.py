"""The scale updates of the device scan against their analytic conditionals,
in the style of the reference's own checks (pkg/tests/test_gibbs.py:100-140):
KS tests of 1e4-1e5 draws against closed-form CDFs and against quadrature
CDFs of the exact conditional.  The draws come from `pcgs_scale_draws`, which
runs the very device functions (`global_draw`, `local_draw`) that k_global and
k_local call inside every scan.

The horseshoe conditionals are new (not in the reference), so besides each
auxiliary inverse-gamma step (closed-form CDFs, or probability-integral
transforms when the rate depends on the auxiliary drawn in the same call) the
auxiliary-variable CHAIN is checked against a quadrature of the exact target
p(tau | sum) ∝ tau^-p exp(-sum / (2 tau^2)) / (1 + tau^2) (half-Cauchy prior)
and p(lam | b, tau) ∝ lam^-1 exp(-b^2 / (2 tau^2 lam^2)) / (1 + lam^2): an
independent derivation, so a shared error in the port and the kernels would
show up here."""
import math

import numpy as np
import pytest
import scipy.integrate
from scipy import stats

from paper_1810_12437_b200.gibbs import scale_draws

pytestmark = pytest.mark.gpu


def quadrature_cdf(logpdf, lo, hi, n=200_001):
    grid = np.geomspace(lo, hi, n)
    lp = logpdf(grid)
    pdf = np.exp(lp - lp.max())
    cdf = scipy.integrate.cumulative_trapezoid(pdf, grid, initial=0.0)
    cdf /= cdf[-1]
    return lambda x: np.interp(x, grid, cdf)


# ------------------------------------------------------------------ bridge (reference conditionals)
def test_bridge_global_two_unit_coefficients():
    """alpha = 1, beta = (1, 1), a0 = b0 = 1: phi = 1/tau ~ Gamma(3, 3), mean 1
    (test_gibbs.py:100-107)."""
    tau, _ = scale_draws("bridge", 0, 100_000, 2.0, p=2, seed=26)
    phis = 1.0 / tau
    se = phis.std(ddof=1) / math.sqrt(phis.size)
    assert abs(phis.mean() - 1.0) <= 4.0 * se


@pytest.mark.parametrize("beta", [np.array([0.5, 1.2, 2.0]), np.array([0.05, 0.1])])
def test_bridge_global_matches_quadrature_posterior(beta):
    """test_gibbs.py:109-128: tau^-p exp(-sum|beta|/tau) pi(tau) on a grid."""
    a0, b0 = 1.5, 0.8
    draws, _ = scale_draws("bridge", 0, 10_000, float(np.abs(beta).sum()), p=beta.size, a0=a0, b0=b0, seed=27)
    cdf = quadrature_cdf(lambda g: -(beta.size + a0 + 1.0) * np.log(g) - (b0 + np.abs(beta).sum()) / g,
                         1e-5, 200.0)
    assert stats.ks_1samp(draws, cdf).pvalue > 0.01


def test_bridge_local_is_inverse_gaussian():
    """test_gibbs.py:131-140: 1/lam^2 ~ InvGauss(tau/|beta|)."""
    beta, tau = 0.8, 1.7
    lam, _ = scale_draws("bridge", 1, 100_000, beta, tau=tau, seed=28)
    res = stats.ks_1samp(lam ** -2.0, stats.invgauss(tau / beta).cdf)
    assert res.pvalue > 0.01


def test_bridge_local_zero_coefficient_limit():
    """|beta|/tau < 1e-10: lam = |N(0,1)| (gibbs.py:205-209)."""
    lam, _ = scale_draws("bridge", 1, 50_000, 0.0, tau=0.3, seed=30)
    assert np.all(lam >= 1e-150)
    assert stats.ks_1samp(lam, stats.halfnorm.cdf).pvalue > 0.01


# ------------------------------------------------------------------ horseshoe (new conditionals)
@pytest.mark.parametrize("lam_old,b,tau", [(1.0, 0.4, 0.7), (0.05, 2.0, 0.1), (30.0, 1e-3, 2.0)])
def test_horseshoe_local_conditionals(lam_old, b, tau):
    """nu ~ IG(1, 1 + 1/lam_old^2); lam^2 | nu ~ IG(1, 1/nu + b^2 / (2 tau^2))."""
    lam, nu = scale_draws("horseshoe", 1, 100_000, b, tau=tau, lam_old=lam_old, seed=31)
    assert stats.ks_1samp(nu, stats.invgamma(1.0, scale=1.0 + 1.0 / lam_old ** 2).cdf).pvalue > 0.01
    rate = 1.0 / nu + 0.5 * b * b / (tau * tau)
    u = stats.invgamma.cdf(lam ** 2, 1.0, scale=rate)          # probability integral transform
    assert stats.kstest(u, "uniform").pvalue > 0.01


@pytest.mark.parametrize("p,acc,tau_old", [(1, 0.3, 1.0), (40, 25.0, 0.2), (2000, 1.5e4, 3.0)])
def test_horseshoe_global_conditionals(p, acc, tau_old):
    """xi ~ IG(1, 1 + 1/tau_old^2); tau^2 | xi ~ IG((p+1)/2, 1/xi + acc/2)."""
    tau, xi = scale_draws("horseshoe", 0, 100_000, acc, tau=tau_old, p=p, seed=32)
    assert stats.ks_1samp(xi, stats.invgamma(1.0, scale=1.0 + 1.0 / tau_old ** 2).cdf).pvalue > 0.01
    u = stats.invgamma.cdf(tau ** 2, 0.5 * (p + 1), scale=1.0 / xi + 0.5 * acc)
    assert stats.kstest(u, "uniform").pvalue > 0.01


def _thinned(chain, burn=1000, thin=20):
    return chain[burn::thin]


@pytest.mark.parametrize("p,acc", [(1, 0.5), (10, 4.0), (200, 150.0)])
def test_horseshoe_global_chain_targets_half_cauchy_conditional(p, acc):
    """The (xi, tau) Gibbs chain with beta, lambda pinned has stationary law
    p(tau | .) ∝ tau^-p exp(-acc / (2 tau^2)) / (1 + tau^2)."""
    chain, _ = scale_draws("horseshoe", 2, 201_000, acc, tau=1.0, p=p, seed=33)
    draws = _thinned(chain)
    cdf = quadrature_cdf(lambda t: -p * np.log(t) - acc / (2 * t * t) - np.log1p(t * t), 1e-4, 1e5)
    assert stats.ks_1samp(draws, cdf).pvalue > 0.01


@pytest.mark.parametrize("b,tau", [(0.5, 1.0), (0.02, 0.1), (3.0, 0.5)])
def test_horseshoe_local_chain_targets_half_cauchy_conditional(b, tau):
    """The (nu, lam) Gibbs chain with beta, tau pinned has stationary law
    p(lam | b, tau) ∝ lam^-1 exp(-b^2 / (2 tau^2 lam^2)) / (1 + lam^2)."""
    chain, _ = scale_draws("horseshoe", 3, 201_000, b, tau=tau, lam_old=1.0, seed=34)
    draws = _thinned(chain)
    cdf = quadrature_cdf(lambda l: -np.log(l) - b * b / (2 * tau * tau * l * l) - np.log1p(l * l), 1e-6, 1e6)
    assert stats.ks_1samp(draws, cdf).pvalue > 0.01


def test_scale_draws_are_reproducible():
    a, _ = scale_draws("horseshoe", 1, 1000, 0.3, tau=0.5, seed=9)
    b, _ = scale_draws("horseshoe", 1, 1000, 0.3, tau=0.5, seed=9)
    c, _ = scale_draws("horseshoe", 1, 1000, 0.3, tau=0.5, seed=10)
    np.testing.assert_array_equal(a, b)
    assert not np.array_equal(a, c)
