"""The CPU restatement's horseshoe conditionals (oracle/port.py:horseshoe_scales,
new, no reference counterpart) against closed-form CDFs and a quadrature of
the exact joint target, so that the oracle the device chains are compared
with is itself pinned (CPU only; the device functions get the same checks in
tests/test_gpu_scales.py)."""
import numpy as np
import scipy.integrate
from scipy import stats

from oracle import port


def test_port_local_conditionals():
    rng = np.random.default_rng(40)
    p = 100_000
    b, tau2, lam2_old = 0.4, 0.49, 1.3
    beta = np.full(p, b)
    lam2, nu, tau2_new, xi = port.horseshoe_scales(beta, np.full(p, lam2_old), np.ones(p), tau2, 1.0, rng)
    assert stats.ks_1samp(nu, stats.invgamma(1.0, scale=1.0 + 1.0 / lam2_old).cdf).pvalue > 0.01
    u = stats.invgamma.cdf(lam2, 1.0, scale=1.0 / nu + 0.5 * b * b / tau2_new)
    assert stats.kstest(u, "uniform").pvalue > 0.01


def test_port_global_conditionals():
    rng = np.random.default_rng(41)
    beta = np.array([0.3, -1.2, 0.05])
    lam2 = np.array([0.5, 2.0, 0.1])
    tau2_old = 0.8
    acc = float(np.sum(beta ** 2 / lam2))
    xis, taus2 = [], []
    for _ in range(20_000):
        _, _, t2, xi = port.horseshoe_scales(beta, lam2, np.ones(3), tau2_old, 1.0, rng)
        xis.append(xi)
        taus2.append(t2)
    xis, taus2 = np.array(xis), np.array(taus2)
    assert stats.ks_1samp(xis, stats.invgamma(1.0, scale=1.0 + 1.0 / tau2_old).cdf).pvalue > 0.01
    u = stats.invgamma.cdf(taus2, 0.5 * (beta.size + 1), scale=1.0 / xis + 0.5 * acc)
    assert stats.kstest(u, "uniform").pvalue > 0.01


def test_port_joint_chain_targets_horseshoe_posterior_of_tau():
    """One coefficient b pinned: the (xi, tau, nu, lam) chain's tau marginal is
    ∫ N(b; 0, tau^2 lam^2) C+(lam) dlam · C+(tau) (2-D quadrature)."""
    rng = np.random.default_rng(42)
    b = np.array([0.7])
    lam2, nu, tau2, xi = np.ones(1), np.ones(1), 1.0, 1.0
    taus = []
    for _ in range(60_000):
        lam2, nu, tau2, xi = port.horseshoe_scales(b, lam2, nu, tau2, xi, rng)
        taus.append(np.sqrt(tau2))
    draws = np.array(taus[1000::10])
    tg = np.geomspace(1e-4, 1e4, 3001)
    lg = np.geomspace(1e-6, 1e6, 4001)
    T, Lm = np.meshgrid(tg, lg, indexing="ij")
    sd = T * Lm
    dens = np.exp(-0.5 * (b[0] / sd) ** 2) / sd / (1.0 + Lm ** 2)
    marg = scipy.integrate.trapezoid(dens, lg, axis=1) / (1.0 + tg ** 2)
    cdf = scipy.integrate.cumulative_trapezoid(marg, tg, initial=0.0)
    cdf /= cdf[-1]
    assert stats.ks_1samp(draws, lambda x: np.interp(x, tg, cdf)).pvalue > 0.01
