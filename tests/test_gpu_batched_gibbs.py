"""Batched Gibbs scans (BASELINE config 4; pcgs_batch_gibbs_scan): R chains
whose beta solves share one batched PCG per scan.  Every chain must be the
chain gibbs_run draws for its seed -- exactly (up to the solve tolerance)
when omega, tau and lambda are pinned, and in distribution when they are
free (the reference's paired-chain rule against the CPU oracle)."""
import numpy as np
import pytest

from paper_1810_12437_b200 import gibbs, synth
from oracle import port

from test_gpu_gibbs import chains_agree

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def small():
    d = synth.binary_design(600, 80, 5e-3, 0.3, seed=5)
    y, truth = synth.simulate_outcomes(d, seed=1, n_signal=6)
    return d, y, truth


@pytest.mark.parametrize("R", [2, 4, 8])
def test_pinned_batched_chains_equal_single_chains(small, R):
    """omega, tau, lambda pinned: each batched chain's draws are the draws of
    gibbs_run with its seed, to the tolerance of the solve (rtol 1e-12)."""
    d, y, _ = small
    X = d.matrix()
    rng = np.random.default_rng(3)
    om = rng.uniform(0.1, 0.3, d.n)
    lam = np.abs(rng.standard_cauchy(d.p)) + 0.1
    cfg = gibbs.HorseshoeConfig(unshrunk_prior_sd=(np.inf,))
    kw = dict(fixed_omega=om, fixed_tau=0.3, fixed_lam=lam, cg_config=gibbs.CGConfig(rtol=1e-12))
    seeds = [11 + 7 * c for c in range(R)]
    outs = gibbs.gibbs_run_batched(X, y, cfg, 12, seeds, **kw)
    for c, sd in enumerate(seeds):
        ref = gibbs.gibbs_run(X, y, cfg, 12, seed=sd, **kw)
        err = np.abs(outs[c].draws - ref.draws).max() / np.abs(ref.draws).max()
        assert err < 1e-8, (c, err)
        np.testing.assert_allclose(outs[c].logdensity_trace, ref.logdensity_trace, rtol=1e-9)
        assert outs[c].draws.shape == (12, d.p + 1)


def test_batched_chains_are_deterministic_and_independent_of_batch_mates(small):
    """A chain's trajectory depends on its seed and R only: the same seed in
    another batch (other mates, another position) gives the same draws."""
    d, y, _ = small
    X = d.matrix()
    cfg = gibbs.HorseshoeConfig(unshrunk_prior_sd=(np.inf,))
    a = gibbs.gibbs_run_batched(X, y, cfg, 30, [5, 6, 7, 8])
    b = gibbs.gibbs_run_batched(X, y, cfg, 30, [9, 5, 10, 11])
    np.testing.assert_array_equal(a[0].draws, b[1].draws)
    np.testing.assert_array_equal(a[0].logdensity_trace, b[1].logdensity_trace)
    assert not np.array_equal(a[0].draws, a[1].draws)


@pytest.mark.parametrize("prior,n_iter", [("bridge", 4000), ("horseshoe", 8000)])
def test_batched_posterior_moments_match_oracle(small, prior, n_iter):
    """Free chains: a batched chain against the CPU oracle's chain by the
    reference's paired-chain rule (test_acceptance.py:417-436)."""
    d, y, _ = small
    X = d.matrix()
    Xo = port.design_from_pattern(d.n, d.p, d.row_ptr, d.col_idx)
    burn = 500
    if prior == "bridge":
        cfg = gibbs.BridgeConfig(unshrunk_prior_sd=(np.inf,))
        ref = port.gibbs_bridge(Xo, y, n_iter, seed=7, burn_in=burn, unshrunk_sd=(np.inf,))
    else:
        cfg = gibbs.HorseshoeConfig(unshrunk_prior_sd=(np.inf,))
        ref = port.gibbs_horseshoe(Xo, y, n_iter, seed=7, burn_in=burn, unshrunk_sd=(np.inf,))
    outs = gibbs.gibbs_run_batched(X, y, cfg, n_iter, [21, 22], burn_in=burn)
    chains_agree(outs[1].draws, ref.draws, f"batched {prior}")


def test_batched_scan_reports_aborts_per_chain(small):
    d, y, _ = small
    X = d.matrix()
    cfg = gibbs.BridgeConfig(unshrunk_prior_sd=(np.inf,))
    with pytest.raises(gibbs.GibbsAbortError):
        gibbs.gibbs_run_batched(X, y, cfg, 3, [1, 2], cg_config=gibbs.CGConfig(rtol=1e-14, max_iter=2))
    outs = gibbs.gibbs_run_batched(X, y, cfg, 3, [1, 2], cg_config=gibbs.CGConfig(rtol=1e-14, max_iter=2),
                                   allow_max_iter=True)
    assert all(np.all(o.cg_iteration_counts == 2) for o in outs)
    with pytest.raises(ValueError):
        gibbs.gibbs_run_batched(X, y, cfg, 3, [1, 2, 3])
