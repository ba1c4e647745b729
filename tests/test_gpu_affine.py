"""Affine designs on the device: real-valued dense blocks
(hstack_dense_columns of a real block, sparse.py:314-341) and column
standardisation (sparse.py:250-297) applied in-kernel around the pattern
passes -- products, the fused PCG, the RHS and Gibbs chains against the CPU
oracle (oracle/port.py restates the reference's value-carrying CSR) and dense
linear algebra."""
import numpy as np
import pytest

import paper_1810_12437_b200 as pk
from paper_1810_12437_b200 import gibbs, synth
from oracle import port

from test_gpu_gibbs import chains_agree

pytestmark = pytest.mark.gpu


def dense_design(seed=3, n=700, p=90, standardize=False, raw_scale=True):
    """[1 | age | bmi | binary pattern], optionally standardised (not the
    ones column); `raw_scale` False draws the two covariates on a unit scale
    (weakly correlated with the ones column, for chains that must mix)."""
    d = synth.binary_design(n, p, 5e-3, 0.3, seed=seed)
    rng = np.random.default_rng(seed)
    B = pk.SparseDesignMatrix.from_pattern(d.n, d.p, d.row_ptr, d.col_idx, intercept=False)
    if raw_scale:
        cov = [rng.normal(50, 10, n), rng.lognormal(3.0, 0.2, n)]
    else:
        cov = [rng.normal(0.3, 1.0, n), rng.uniform(-1.0, 2.0, n)]
    cols = np.column_stack([np.ones(n), *cov])
    X = pk.hstack_dense_columns(cols, B)
    if standardize:
        X.standardize(exclude=[0])
    Xo = port.Csr(X.n_rows, X.n_cols, X.row_ptr, X.col_idx, X.values, X.col_means.copy(),
                  X.col_scales.copy())
    return d, X, Xo


@pytest.mark.parametrize("standardize", [False, True])
@pytest.mark.parametrize("slab_max", [0, 40])
def test_products_match_oracle(standardize, slab_max):
    d, X, Xo = dense_design(standardize=standardize)
    X.slab_max = slab_max             # 40: many slabs each way (multi-slab combine)
    assert X.dense_block.shape == (d.n, 3) and X.affine
    full = X.to_dense()
    rng = np.random.default_rng(1)
    v, w = rng.standard_normal(X.n_cols), rng.standard_normal(d.n)
    om = rng.uniform(0.05, 0.3, d.n)
    diag = np.concatenate([np.zeros(3), rng.uniform(0.5, 4.0, d.p)])
    for got, ref in ((X.matvec(v), port.matvec(Xo, v)), (X.matvec_t(w), port.matvec_t(Xo, w)),
                     (X.gram_diagonal(om), port.gram_diagonal(Xo, om)),
                     (pk.PrecisionOperator(X, om, diag).apply(v), port.phi_apply(Xo, om, diag, v))):
        assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)
    np.testing.assert_allclose(X.matvec(v), full @ v, rtol=1e-10, atol=1e-10)


@pytest.mark.parametrize("standardize,slab_max", [(False, 0), (True, 0), (True, 40)])
def test_fused_pcg_and_rhs_on_affine_design(standardize, slab_max):
    """The persistent PCG kernel with the affine terms (k_pcg<true>): relative
    L2 < 1e-8 vs the oracle at RMS 1e-10 and the iteration count inside the
    oracle's band of summation orders; the RHS equals the reference formula
    with shared noise."""
    d, X, Xo = dense_design(seed=5, standardize=standardize)
    X.slab_max = slab_max            # 40: multi-slab CSR (the row combine of k_pcg<true>)
    rng = np.random.default_rng(2)
    om = rng.uniform(0.05, 0.3, d.n)
    lam = np.abs(rng.standard_cauchy(d.p)) + 0.05
    diag = np.concatenate([np.zeros(3), (0.05 * lam) ** -2.0])
    minv = np.concatenate([np.full(3, 25.0), (0.05 * lam) ** 2])
    phi = pk.PrecisionOperator(X, om, diag)
    t = pk.GaussianTarget(phi, np.zeros(X.n_cols))
    b = pk.generate_rhs(t, np.random.default_rng(4))
    r2 = np.random.default_rng(4)
    eta, delta = r2.standard_normal(d.n), r2.standard_normal(X.n_cols)
    ref_b = port.rhs_given_noise(Xo, np.zeros(X.n_cols), om, diag, eta, delta)
    assert np.linalg.norm(b - ref_b) <= 1e-12 * np.linalg.norm(ref_b)
    M = pk.Preconditioner(pk.PreconditionerKind.AUGMENTED_PRIOR, minv)
    rep = pk.pcg_solve(phi, b, M, config=pk.CGConfig(rtol=1e-10), residual_scale=np.sqrt(minv))
    oref = port.pcg(lambda x: port.phi_apply(Xo, om, diag, x), b, minv, np.sqrt(minv), rtol=1e-10)
    assert np.linalg.norm(rep.solution - oref.x) / np.linalg.norm(oref.x) < 1e-8
    lo, hi, counts = port.iteration_band(Xo, om, diag, b, minv, np.sqrt(minv), rtol=1e-10)
    assert lo <= rep.iterations <= hi, (rep.iterations, counts)
    again = pk.pcg_solve(phi, b, M, config=pk.CGConfig(rtol=1e-10), residual_scale=np.sqrt(minv))
    np.testing.assert_array_equal(rep.solution, again.solution)


def test_pinned_scales_exact_gaussian_with_dense_block():
    """omega, tau, lambda pinned: the chain on a dense-block design samples
    exactly N(Phi^-1 X'kappa, Phi^-1) (test_gibbs.py:249-270)."""
    d, X, Xo = dense_design(seed=7, n=500, p=40)
    rng = np.random.default_rng(0)
    y, _ = synth.simulate_outcomes(d, seed=1, n_signal=4, intercept=False)
    om = rng.uniform(0.1, 0.3, d.n)
    lam = rng.uniform(0.5, 2.0, d.p)
    tau = 0.3
    q = 3
    cfg = gibbs.BridgeConfig(unshrunk_prior_sd=(np.inf, 1.0, 1.0))
    out = gibbs.gibbs_run(X, y, cfg, 3000, seed=2, fixed_omega=om, fixed_tau=tau, fixed_lam=lam,
                          cg_config=gibbs.CGConfig(rtol=1e-10))
    full = X.to_dense()
    prior = np.concatenate([[0.0, 1.0, 1.0], (tau * lam) ** -2.0])
    P = full.T @ (om[:, None] * full) + np.diag(prior)
    cov = np.linalg.inv(P)
    mean = cov @ (full.T @ (y - 0.5))
    z = (out.draws.mean(0) - mean) / np.sqrt(np.diag(cov) / len(out.draws))
    assert np.mean(np.abs(z) > 4) < 0.02
    assert np.median(np.var(out.draws, axis=0) / np.diag(cov)) == pytest.approx(1.0, abs=0.1)
    assert out.draws.shape == (3000, q + d.p)


@pytest.mark.parametrize("standardize", [False, True])
def test_free_chain_with_dense_block_matches_oracle(standardize):
    """Free horseshoe chain on [1 | age | bmi | pattern] (the covariates
    unshrunk, N(0, 1) on the standardised scale): device vs oracle chain by the
    reference's paired-chain rule.  Unstandardised, the covariates are drawn
    on a unit scale: raw age/bmi columns are nearly collinear with the ones
    column and no two finite chains of either sampler mix well enough for a
    second-moment test."""
    d, X, Xo = dense_design(seed=9, n=600, p=60, standardize=standardize, raw_scale=standardize)
    y, _ = synth.simulate_outcomes(d, seed=3, n_signal=5, intercept=False)
    sd = (np.inf, 1.0, 1.0)
    cfg = gibbs.HorseshoeConfig(unshrunk_prior_sd=sd)
    n_iter, burn = 6000, 500
    out = gibbs.gibbs_run(X, y, cfg, n_iter, burn_in=burn, seed=8)
    ref = port.gibbs_horseshoe(Xo, y, n_iter, seed=7, burn_in=burn, unshrunk_sd=sd)
    chains_agree(out.draws, ref.draws, f"dense block (standardised={standardize})")


def test_affine_designs_refused_on_sharded_and_batched_paths():
    from paper_1810_12437_b200 import batched, parallel
    d, X, _ = dense_design(seed=2, n=200, p=20)
    with pytest.raises(NotImplementedError):
        parallel.local_rows(X, 0, 100)
    with pytest.raises(NotImplementedError):
        batched.BatchedPrecisionOperator(X, np.ones((2, d.n)), np.ones((2, X.n_cols)))


def test_standardised_design_without_intercept():
    """A standardised pattern-only design with no intercept column (no
    reparametrisation possible): products, the fused PCG and a Gibbs chain
    run on the affine store; pinned scales give the exact Gaussian."""
    d = synth.binary_design(500, 50, 5e-3, 0.3, seed=12)
    X = d.matrix(intercept=False).standardize()
    Xo = port.Csr(X.n_rows, X.n_cols, X.row_ptr, X.col_idx, X.values, X.col_means.copy(), X.col_scales.copy())
    rng = np.random.default_rng(3)
    om = rng.uniform(0.1, 0.3, d.n)
    lam = rng.uniform(0.5, 2.0, d.p)
    tau = 0.4
    diag = (tau * lam) ** -2.0
    v = rng.standard_normal(d.p)
    ref = port.phi_apply(Xo, om, diag, v)
    assert np.linalg.norm(pk.PrecisionOperator(X, om, diag).apply(v) - ref) <= 1e-12 * np.linalg.norm(ref)
    y, _ = synth.simulate_outcomes(d, seed=2, n_signal=4, intercept=False)
    cfg = gibbs.BridgeConfig()
    out = gibbs.gibbs_run(X, y, cfg, 3000, seed=2, fixed_omega=om, fixed_tau=tau, fixed_lam=lam,
                          cg_config=gibbs.CGConfig(rtol=1e-10))
    full = X.to_dense()
    P = full.T @ (om[:, None] * full) + np.diag(diag)
    cov = np.linalg.inv(P)
    mean = cov @ (full.T @ (y - 0.5))
    z = (out.draws.mean(0) - mean) / np.sqrt(np.diag(cov) / len(out.draws))
    assert np.mean(np.abs(z) > 4) < 0.02
    assert np.median(np.var(out.draws, axis=0) / np.diag(cov)) == pytest.approx(1.0, abs=0.1)
