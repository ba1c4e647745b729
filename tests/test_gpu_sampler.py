"""Randomised RHS and Polya-Gamma draws on device (reference tests:
test_sampler.py:87-133, test_polya_gamma.py:21-82)."""
import numpy as np
import pytest
from scipy import stats

import paper_1810_12437_b200 as pk
from paper_1810_12437_b200 import synth
from oracle import port

pytestmark = pytest.mark.gpu


def golden_target(g):
    X = pk.SparseDesignMatrix.from_pattern(int(g["n"]), int(g["p"]), g["rp"], g["ci"])
    phi = pk.PrecisionOperator(X, g["om"], g["prior"])
    return X, phi


class ZeroNoise:
    def standard_normal(self, size):
        return np.zeros(size)


def test_linear_term_matches_reference(golden):
    g = golden("pcg")
    _, phi = golden_target(g)
    t = pk.GaussianTarget.from_pseudo_outcome(phi, (g["y"] - 0.5) / g["om"])
    np.testing.assert_allclose(t.linear_term, g["lin"], rtol=1e-12, atol=1e-12)


def test_rhs_host_noise_matches_reference_stream_order(golden):
    g = golden("pcg")
    _, phi = golden_target(g)
    t = pk.GaussianTarget(phi, g["lin"])
    b = pk.generate_rhs(t, np.random.default_rng(99))
    np.testing.assert_allclose(b, g["rhs_b"], rtol=1e-12, atol=1e-12)


def test_zero_noise_gives_linear_term(golden):
    g = golden("pcg")
    _, phi = golden_target(g)
    t = pk.GaussianTarget(phi, g["lin"])
    np.testing.assert_allclose(pk.generate_rhs(t, ZeroNoise()), g["lin"], rtol=0, atol=0)


def test_device_noise_covariance_is_phi():
    """Cov(b) = Phi with device Philox noise (test_sampler.py:116-133)."""
    rng = np.random.default_rng(0)
    dense = (rng.random((30, 6)) < 0.4).astype(float)
    X = pk.SparseDesignMatrix.from_dense(dense)
    om = rng.uniform(0.2, 1.5, 30)
    d = rng.uniform(0.5, 2.0, 6)
    phi = pk.PrecisionOperator(X, om, d)
    t = pk.GaussianTarget(phi, np.zeros(6))
    gen = pk.PhiloxGenerator(1234)
    N = 20000
    B = np.stack([pk.generate_rhs(t, gen) for _ in range(N)])
    full = dense.T @ (om[:, None] * dense) + np.diag(d)
    cov = B.T @ B / N
    se = np.sqrt((full ** 2 + np.outer(np.diag(full), np.diag(full))) / N)
    assert np.all(np.abs(cov - full) < 5 * se)
    assert np.all(np.abs(B.mean(0)) < 5 * np.sqrt(np.diag(full) / N))


def test_cg_sample_equals_direct_solve_with_shared_noise(golden):
    """Shared (eta, delta) -> CG draw equals the Cholesky draw (test_sampler.py:146-159)."""
    g = golden("pcg")
    X, phi = golden_target(g)
    t = pk.GaussianTarget(phi, g["lin"])
    M = pk.Preconditioner(pk.PreconditionerKind.AUGMENTED_PRIOR, g["minv"])
    beta, rep = pk.cg_sample(t, M, np.random.default_rng(8), config=pk.CGConfig(rtol=1e-12),
                             residual_scale=g["scale"])
    Xo = port.design_from_pattern(int(g["n"]), int(g["p"]), g["rp"], g["ci"])
    dense = np.zeros((int(g["n"]), int(g["p"]) + 1))
    rows = np.repeat(np.arange(int(g["n"])), np.diff(Xo.row_ptr))
    dense[rows, Xo.col_idx] = 1.0
    full = dense.T @ (g["om"][:, None] * dense) + np.diag(g["prior"])
    b = port.rhs(Xo, g["lin"], g["om"], g["prior"], np.random.default_rng(8))
    direct = np.linalg.solve(full, b)
    assert np.max(np.abs(beta - direct)) <= 1e-8 * max(1.0, np.max(np.abs(direct)))


class TestPolyaGamma:
    @pytest.mark.parametrize("z", [0.0, 0.5, 1.7, 4.0, 12.0, -3.0])
    def test_moments(self, z):
        n = 200_000
        draws = pk.pg_draw_batch(np.full(n, z), np.random.default_rng(int(abs(z) * 10)))
        assert np.all(draws > 0)
        mean = pk.pg_mean(z)
        # Var PG(1, z) = (sinh z - z) / (4 z^3 cosh^2(z/2)), limit 1/24
        var = 1.0 / 24.0 if z == 0 else (np.sinh(z) - z) / (4 * z ** 3 * np.cosh(z / 2) ** 2)
        assert abs(draws.mean() - mean) < 4 * np.sqrt(var / n)
        assert abs(draws.var() - var) < 6 * var * np.sqrt(2.0 / n) * 3

    def test_laplace_transform(self):
        # E exp(-t w) = cosh(z/2) / cosh(sqrt((z^2 / 2 + t)/2))
        z, t = 1.3, 0.7
        draws = pk.pg_draw_batch(np.full(300_000, z), np.random.default_rng(5))
        lt = np.cosh(z / 2) / np.cosh(np.sqrt((z * z / 2 + t) / 2))
        est = np.exp(-t * draws)
        assert abs(est.mean() - lt) < 4 * est.std() / np.sqrt(len(draws))

    def test_ks_against_oracle_sampler(self):
        for z in (0.0, 2.0, 25.0):
            dev = pk.pg_draw_batch(np.full(20000, z), np.random.default_rng(1))
            cpu = port.pg_batch(np.full(20000, z), np.random.default_rng(2))
            assert stats.ks_2samp(dev, cpu).pvalue > 0.001

    def test_symmetry_and_determinism(self):
        z = np.linspace(-6, 6, 5001)
        a = pk.pg_draw_batch(z, pk.PhiloxGenerator(3))
        g1, g2 = pk.PhiloxGenerator(9), pk.PhiloxGenerator(9)
        assert np.array_equal(pk.pg_draw_batch(z, g1), pk.pg_draw_batch(z, g2))
        assert stats.ks_2samp(a[:2500], a[2501:][::-1]).pvalue > 0.001

    def test_rejects_nonfinite(self):
        with pytest.raises(ValueError):
            pk.pg_draw_batch(np.array([np.inf]), np.random.default_rng(0))
