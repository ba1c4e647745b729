"""Host-side logic of the drop-in package (no GPU): validation, layouts,
configuration objects, and the loud failure of device entry points."""
import math

import numpy as np
import pytest

import paper_1810_12437_b200 as pk
from paper_1810_12437_b200 import gibbs, synth
from paper_1810_12437_b200.cg import _metric_scale
from oracle import port


class TestDesignValidation:
    # the reference's invariants (sparse.py:94-117)
    def test_row_ptr_length(self):
        with pytest.raises(ValueError):
            pk.SparseDesignMatrix(2, 2, [0, 1], [0], [1.0])

    def test_endpoints(self):
        with pytest.raises(ValueError):
            pk.SparseDesignMatrix(1, 2, [0, 2], [0], [1.0])

    def test_nondecreasing(self):
        with pytest.raises(ValueError):
            pk.SparseDesignMatrix(2, 2, [0, 2, 1], [0, 1], [1.0, 1.0])

    def test_column_range(self):
        with pytest.raises(ValueError):
            pk.SparseDesignMatrix(1, 2, [0, 1], [2], [1.0])

    def test_strictly_increasing_within_row(self):
        with pytest.raises(ValueError):
            pk.SparseDesignMatrix(1, 3, [0, 2], [1, 1], [1.0, 1.0])
        pk.SparseDesignMatrix(2, 3, [0, 2, 4], [1, 2, 0, 1], np.ones(4))  # boundary decrease ok

    def test_nonfinite_values(self):
        with pytest.raises(ValueError):
            pk.SparseDesignMatrix(1, 1, [0, 1], [0], [np.nan])

    def test_scales_positive(self):
        with pytest.raises(ValueError):
            pk.SparseDesignMatrix(1, 1, [0, 1], [0], [1.0], col_scales=[0.0])


class TestPatternLayout:
    def test_from_pattern_matches_reference_layout(self):
        d = synth.config_design(1, seed=0)
        X = d.matrix()
        Xo = port.design_from_pattern(d.n, d.p, d.row_ptr, d.col_idx)
        np.testing.assert_array_equal(X.row_ptr, Xo.row_ptr)
        np.testing.assert_array_equal(X.col_idx, Xo.col_idx)
        assert X.nnz == Xo.row_ptr[-1] == d.nnz + d.n
        assert X.n_cols == d.p + 1

    def test_pattern_strips_leading_dense_column(self):
        d = synth.config_design(1, seed=0)
        Xo = port.design_from_pattern(d.n, d.p, d.row_ptr, d.col_idx)
        X = pk.SparseDesignMatrix(d.n, d.p + 1, Xo.row_ptr, Xo.col_idx, Xo.values)
        rp, ci, icpt = X.pattern()
        assert icpt
        np.testing.assert_array_equal(rp, d.row_ptr)
        np.testing.assert_array_equal(ci, d.col_idx)

    def test_hstack_ones_sets_intercept_flag(self):
        d = synth.config_design(1, seed=0)
        X0 = pk.SparseDesignMatrix.from_pattern(d.n, d.p, d.row_ptr, d.col_idx, intercept=False)
        X1 = pk.hstack_dense_columns(np.ones((d.n, 1)), X0)
        assert X1.pattern()[2] and X1.n_cols == d.p + 1

    def test_hstack_general_block_matches_reference(self):
        rng = np.random.default_rng(0)
        dense = (rng.random((6, 4)) < 0.5).astype(float)
        X = pk.SparseDesignMatrix.from_dense(dense)
        cols = rng.standard_normal((6, 2))
        Y = pk.hstack_dense_columns(cols, X)
        np.testing.assert_array_equal(Y.to_dense(), np.hstack([cols, dense]))

    def test_non_binary_design_is_refused_by_the_store(self):
        X = pk.SparseDesignMatrix.from_dense(np.array([[2.0, 0.0], [0.0, 1.0]]))
        with pytest.raises(NotImplementedError):
            X.pattern()

    def test_standardize_matches_column_moments(self):
        d = synth.binary_design(300, 40, 0.01, 0.5, seed=2)
        X = d.matrix()
        dense = X.to_dense_raw()
        X.standardize(exclude=[0])
        col = dense[:, 1:]
        keep = col.std(axis=0, ddof=1) > 0
        np.testing.assert_allclose(X.col_means[1:][keep], col.mean(axis=0)[keep], rtol=1e-13)
        np.testing.assert_allclose(X.col_scales[1:][keep], col.std(axis=0, ddof=1)[keep], rtol=1e-12)
        assert X.col_means[0] == 0.0 and X.col_scales[0] == 1.0
        assert X.standardized and X.pattern()[2]   # the store keeps the raw pattern


class TestSolverConfig:
    def test_cgconfig_validation(self):
        with pytest.raises(ValueError):
            pk.CGConfig(max_iter=0)
        with pytest.raises(ValueError):
            pk.CGConfig(rtol=0.0)
        with pytest.raises(ValueError):
            pk.CGConfig(trace_level="all")

    def test_metric_scale_precedence(self):
        M = pk.prior_preconditioner(2.0, np.array([1.0, 3.0]))

        class Phi:
            prior_precision_diag = np.array([4.0, 16.0])

        np.testing.assert_array_equal(_metric_scale(Phi, M, np.array([1.0, 2.0]), 2), [1.0, 2.0])
        np.testing.assert_allclose(_metric_scale(Phi, M, None, 2), [0.5, 0.25])
        Phi.prior_precision_diag = np.array([0.0, 1.0])   # flat coordinate: fall back to M
        np.testing.assert_allclose(_metric_scale(Phi, M, None, 2), [2.0, 6.0])
        with pytest.raises(ValueError):
            _metric_scale(Phi, pk.identity_preconditioner(2), None, 2)
        with pytest.raises(ValueError):
            _metric_scale(Phi, M, np.array([1.0, -1.0]), 2)

    def test_preconditioners(self):
        M = pk.augmented_prior(0.5, np.array([1.0, 2.0]), np.array([3.0]))
        np.testing.assert_allclose(M.inv_diagonal, [9.0, 0.25, 1.0])
        assert pk.augmented_prior(0.5, np.array([1.0]), np.zeros(0)).kind is pk.PreconditionerKind.PRIOR
        with pytest.raises(pk.DegeneratePreconditionerError):
            pk.Preconditioner(pk.PreconditionerKind.PRIOR, np.array([0.0]))
        with pytest.raises(ValueError):
            pk.prior_preconditioner(-1.0, np.ones(2))

    def test_gamma_policy_and_initial_vector(self):
        assert pk.gamma_policy(None, prior_sd=(np.inf,))[0] == 10.0
        assert pk.gamma_policy(None, c=2.0, prior_sd=(0.5,))[0] == 1.0

        class Chain:
            def unshrunk_sd(self):
                return np.array([0.0])

            def scaled_beta_mean(self):
                return np.array([1.0, 2.0, 3.0])

        assert pk.gamma_policy(Chain())[0] == 1e-3
        np.testing.assert_allclose(pk.initial_vector(Chain(), 2.0, np.array([1.0, 0.5]), 1), [1.0, 4.0, 3.0])
        np.testing.assert_array_equal(pk.initial_vector(None, 1.0, np.ones(2)), np.zeros(2))

    def test_lanczos_tridiagonal(self):
        rep = pk.CGReport(2, "converged", np.zeros(3), np.zeros(2), 3, alphas=np.array([0.5, 0.25]),
                          betas=np.array([0.04]))
        diag, off = rep.lanczos_tridiagonal()
        np.testing.assert_allclose(diag, [2.0, 4.0 + 0.08])
        np.testing.assert_allclose(off, [0.4])


class TestGibbsHost:
    def test_configs(self):
        with pytest.raises(ValueError):
            gibbs.BridgeConfig(alpha=1.5)
        with pytest.raises(ValueError):
            gibbs.BridgeConfig(global_rate=0.0)
        with pytest.raises(ValueError):
            gibbs.HorseshoeConfig(unshrunk_prior_sd=(-1.0,))
        c = gibbs.BridgeConfig(unshrunk_prior_sd=(np.inf, 2.0))
        np.testing.assert_allclose(c.unshrunk_precision(), [0.0, 0.25])
        assert gibbs.HorseshoeConfig(unshrunk_prior_sd=(1.0,)).n_unshrunk == 1

    def test_state_validation(self):
        with pytest.raises(ValueError):
            gibbs.ShrinkageState(np.zeros(2), np.ones(3), np.ones(2), 0.0)
        with pytest.raises(ValueError):
            gibbs.ShrinkageState(np.zeros(2), np.zeros(3), np.ones(2), 1.0)

    def test_run_argument_validation_precedes_device_work(self):
        d = synth.config_design(1, seed=0)
        X = d.matrix()
        y = np.zeros(d.n)
        cfg = gibbs.BridgeConfig(unshrunk_prior_sd=(np.inf,))
        with pytest.raises(ValueError):
            gibbs.gibbs_run(X, y[:-1], cfg, 3)
        with pytest.raises(ValueError):
            gibbs.gibbs_run(X, y + 0.5, cfg, 3)
        with pytest.raises(ValueError):
            gibbs.gibbs_run(X, y, cfg, 3, burn_in=4)
        with pytest.raises(ValueError):
            gibbs.gibbs_run(X, y, cfg, 3, thin=0)
        with pytest.raises(ValueError):
            gibbs.gibbs_run(X, y, cfg, 3, sampler="gibbs")
        with pytest.raises(NotImplementedError):
            gibbs.gibbs_run(X, y, cfg, 3, sampler="direct")
        with pytest.raises(gibbs.UnsupportedUpdateError):
            gibbs.gibbs_run(X, y, gibbs.BridgeConfig(alpha=0.5, unshrunk_prior_sd=(np.inf,)), 3)


class TestSynthetic:
    def test_config_designs_are_seeded(self):
        d = synth.config_design(1, seed=0)
        assert d.nnz == 41978           # SURVEY.md §6, same recipe and seed
        d2 = synth.config_design(1, seed=0)
        np.testing.assert_array_equal(d.col_idx, d2.col_idx)
        assert np.all(np.diff(d.row_ptr) >= 0)

    def test_rare_outcome_offset(self):
        d = synth.binary_design(4000, 200, 1e-3, 0.2, seed=1)
        y, beta = synth.simulate_outcomes(d, seed=0, rate=0.02)
        assert abs(y.mean() - 0.02) < 0.01 and beta.shape == (201,)
        assert np.count_nonzero(beta[1:]) == 10


def test_device_calls_fail_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    X = synth.config_design(1, seed=0).matrix()
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        X.matvec(np.zeros(X.n_cols))


def test_hstack_binary_block_stays_pattern_only():
    """hstack_dense_columns (sparse.py:314-341) of a 0/1 block (an intercept
    and dummy covariates): same dense matrix as the reference layout, stored
    pattern-only so the device path keeps it (unshrunk block with q > 1)."""
    d = synth.binary_design(80, 15, 0.05, 0.4, seed=2)
    X = d.matrix(intercept=False)
    rng = np.random.default_rng(4)
    block = np.column_stack([np.ones(80), rng.random(80) < 0.3, rng.random(80) < 0.7]).astype(float)
    F = pk.hstack_dense_columns(block, X)
    np.testing.assert_array_equal(F.to_dense_raw(), np.column_stack([block, X.to_dense_raw()]))
    rp, ci, icpt = F.pattern()
    assert icpt and F.n_cols == 18 and F.nnz == int(block.sum()) + X.nnz
    v = rng.standard_normal(18)
    np.testing.assert_allclose(port.matvec(port.Csr(80, 18, F.row_ptr, F.col_idx, F.values), v),
                               np.column_stack([block, X.to_dense_raw()]) @ v, rtol=1e-12)
    # a real-valued block keeps the reference layout (explicit entries); the
    # store splits it into a leading dense block and the pattern
    G = pk.hstack_dense_columns(np.column_stack([np.ones(80), rng.standard_normal(80)]), X)
    rp, ci, icpt = G.pattern()
    assert not icpt and G.dense_block.shape == (80, 2)


class TestDenseBlock:
    """Real-valued dense blocks (hstack_dense_columns of a real block,
    sparse.py:314-341): the design splits into a leading dense block, handled
    by the store's affine terms, and a binary pattern."""

    def test_hstack_real_block_splits_into_dense_and_pattern(self):
        d = synth.binary_design(50, 12, 0.05, 0.4, seed=3)
        X0 = pk.SparseDesignMatrix.from_pattern(d.n, d.p, d.row_ptr, d.col_idx, intercept=True)
        rng = np.random.default_rng(1)
        cols = rng.standard_normal((d.n, 2))
        X = pk.hstack_dense_columns(cols, X0)
        rp, ci, icpt = X.pattern()
        dense = X.dense_block
        # the leading block is the real columns plus X0's intercept column
        assert dense.shape == (d.n, 3) and not icpt and X.affine
        np.testing.assert_array_equal(dense[:, :2], cols)
        np.testing.assert_array_equal(dense[:, 2], np.ones(d.n))
        np.testing.assert_array_equal(rp, d.row_ptr)
        np.testing.assert_array_equal(ci, d.col_idx)
        assert X.n_cols == d.p + 3 and X.nnz == d.nnz + 3 * d.n
        full = X.to_dense()
        np.testing.assert_array_equal(full[:, :2], cols)

    def test_values_outside_a_leading_block_are_refused(self):
        X = pk.SparseDesignMatrix.from_dense(np.array([[1.5, 1.0, 0.0], [0.5, 0.0, 2.0]]))
        with pytest.raises(NotImplementedError):
            X.pattern()
