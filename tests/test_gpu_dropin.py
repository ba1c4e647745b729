"""Reference features on the device path beyond the binary-raw core:
trace_level="full" iterates (cg.py:143-169), implicitly standardised designs
(sparse.py:178-203, 250-297), and gibbs_run's local_scale_sampler hook
(gibbs.py:262, 311, 328-329; reference test test_gibbs.py:347-363)."""
import numpy as np
import pytest

import paper_1810_12437_b200 as pk
from paper_1810_12437_b200 import gibbs, synth
from oracle import port

pytestmark = pytest.mark.gpu


def test_trace_level_full_records_every_iterate(golden):
    g = golden("pcg")
    X = pk.SparseDesignMatrix.from_pattern(int(g["n"]), int(g["p"]), g["rp"], g["ci"])
    phi = pk.PrecisionOperator(X, g["om"], g["prior"])
    M = pk.Preconditioner(pk.PreconditionerKind.AUGMENTED_PRIOR, g["minv"])
    x0 = 0.5 * g["r6_x"]
    rep = pk.pcg_solve(phi, g["b"], M, x0=x0, config=pk.CGConfig(trace_level="full"),
                       residual_scale=g["scale"])
    assert len(rep.iterates) == rep.iterations + 1
    np.testing.assert_array_equal(rep.iterates[0], x0)
    np.testing.assert_array_equal(rep.iterates[-1], rep.solution)
    # generic operator path too
    dense = X.to_dense_raw()
    mat = dense.T @ (g["om"][:, None] * dense) + np.diag(g["prior"])
    rep2 = pk.pcg_solve(lambda v: mat @ v, g["b"], M, config=pk.CGConfig(trace_level="full", rtol=1e-8),
                        residual_scale=g["scale"])
    assert len(rep2.iterates) == rep2.iterations + 1
    np.testing.assert_array_equal(rep2.iterates[-1], rep2.solution)


def test_standardised_design_products_and_solve():
    d = synth.binary_design(400, 60, 0.01, 0.4, seed=6)
    X = d.matrix().standardize(exclude=[0])
    dense = X.to_dense()
    rng = np.random.default_rng(2)
    v, w = rng.standard_normal(X.n_cols), rng.standard_normal(d.n)
    np.testing.assert_allclose(X.matvec(v), dense @ v, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(X.matvec_t(w), dense.T @ w, rtol=1e-12, atol=1e-11)
    om = rng.uniform(0.1, 1.0, d.n)
    diag = np.concatenate([[0.0], rng.uniform(0.5, 2.0, d.p)])
    np.testing.assert_allclose(X.gram_diagonal(om), (dense ** 2 * om[:, None]).sum(0), rtol=1e-12, atol=1e-12)
    phi = pk.PrecisionOperator(X, om, diag)
    full = dense.T @ (om[:, None] * dense) + np.diag(diag)
    np.testing.assert_allclose(phi.apply(v), full @ v, rtol=1e-12, atol=1e-11)
    b = rng.standard_normal(X.n_cols)
    minv = np.concatenate([[100.0], 1.0 / diag[1:]])
    phi.apply_count = 0
    rep = pk.pcg_solve(phi, b, pk.Preconditioner(pk.PreconditionerKind.AUGMENTED_PRIOR, minv),
                       config=pk.CGConfig(rtol=1e-12), residual_scale=np.sqrt(minv))
    x = np.linalg.solve(full, b)
    assert np.linalg.norm(rep.solution - x) / np.linalg.norm(x) < 1e-8
    assert rep.matvec_count == rep.iterations + 1 == phi.apply_count
    t = pk.GaussianTarget(phi, np.zeros(X.n_cols))
    bb = pk.generate_rhs(t, np.random.default_rng(4))
    r2 = np.random.default_rng(4)
    eta, delta = r2.standard_normal(d.n), r2.standard_normal(X.n_cols)
    np.testing.assert_allclose(bb, dense.T @ (np.sqrt(om) * eta) + np.sqrt(diag) * delta, rtol=1e-11,
                               atol=1e-11)


def test_local_scale_sampler_hook():
    d = synth.binary_design(500, 50, 5e-3, 0.3, seed=9)
    y, _ = synth.simulate_outcomes(d, seed=2, n_signal=4)
    calls = []

    def sampler(beta_shrunk, tau, cfg, rng):
        calls.append((beta_shrunk.shape, tau))
        return np.full(beta_shrunk.shape, 0.7)

    cfg = gibbs.BridgeConfig(unshrunk_prior_sd=(np.inf,))
    out = gibbs.gibbs_run(d.matrix(), y, cfg, 6, seed=3, local_scale_sampler=sampler)
    assert len(calls) == 6 and all(s == (d.p,) for s, _ in calls)
    np.testing.assert_array_equal(out.final_state.lam, np.full(d.p, 0.7))
    assert all(tau > 0 for _, tau in calls)
