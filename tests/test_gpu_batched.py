"""Batched independent chains (csrc/sliced.cu): R right-hand sides share one
walk over the sliced index stream; every chain must equal its own
single-chain oracle solve."""
import numpy as np
import pytest

import paper_1810_12437_b200 as pk
from paper_1810_12437_b200 import batched, synth
from oracle import port

pytestmark = pytest.mark.gpu


def chains(d, R, seed, easy=None):
    rng = np.random.default_rng(seed)
    om = rng.uniform(0.05, 0.4, (R, d.n))
    lam = np.abs(rng.standard_cauchy((R, d.p))) + 0.05
    tau = rng.uniform(0.02, 0.2, R)
    if easy is not None:
        tau[easy] = 1e-3          # prior-dominated chain: converges in a few iterations
    diag = np.concatenate([np.zeros((R, 1)), (tau[:, None] * lam) ** -2.0], axis=1)
    minv = np.concatenate([np.full((R, 1), 100.0), (tau[:, None] * lam) ** 2], axis=1)
    return om, diag, minv


@pytest.mark.parametrize("R", [2, 4, 8])
@pytest.mark.parametrize("slab_max", [0, 64])
def test_batched_phi_matches_oracle_per_chain(R, slab_max):
    d = synth.binary_design(1500, 300, 1e-3, 0.3, seed=2)
    X = d.matrix()
    X.slab_max = slab_max          # 64: many slabs each way, pieces from every slab
    Xo = port.design_from_pattern(d.n, d.p, d.row_ptr, d.col_idx)
    om, diag, _ = chains(d, R, 1)
    V = np.random.default_rng(3).standard_normal((R, d.p + 1))
    op = batched.BatchedPrecisionOperator(X, om, diag)
    out = op.apply(V)
    for c in range(R):
        ref = port.phi_apply(Xo, om[c], diag[c], V[c])
        assert np.linalg.norm(out[c] - ref) <= 1e-12 * np.linalg.norm(ref)


@pytest.mark.parametrize("R", [2, 4, 8])
def test_batched_pcg_matches_single_chain(R):
    d = synth.binary_design(2000, 400, 1e-3, 0.25, seed=5)
    X = d.matrix()
    Xo = port.design_from_pattern(d.n, d.p, d.row_ptr, d.col_idx)
    om, diag, minv = chains(d, R, 7, easy=0)
    rng = np.random.default_rng(9)
    B = np.stack([port.rhs(Xo, np.zeros(d.p + 1), om[c], diag[c], rng) for c in range(R)])
    op = batched.BatchedPrecisionOperator(X, om, diag)
    reps = batched.batched_pcg_solve(op, B, minv, np.sqrt(minv), config=pk.CGConfig(rtol=1e-10))
    its = []
    for c in range(R):
        ref = port.pcg(lambda v: port.phi_apply(Xo, om[c], diag[c], v), B[c], minv[c], np.sqrt(minv[c]),
                       rtol=1e-10)
        assert np.linalg.norm(reps[c].solution - ref.x) / np.linalg.norm(ref.x) < 1e-8
        lo, hi, counts = port.iteration_band(Xo, om[c], diag[c], B[c], minv[c], np.sqrt(minv[c]), rtol=1e-10)
        assert lo <= reps[c].iterations <= hi, (c, reps[c].iterations, counts)
        assert reps[c].termination == "converged"
        assert len(reps[c].rms_precond_residual_trace) == reps[c].iterations + 1
        its.append(reps[c].iterations)
    assert its[0] < max(its)     # the easy chain stopped early while the others kept going


def test_batched_config2_phi_vs_single():
    d = synth.config_design(2, seed=0)
    X = d.matrix()
    om, diag, _ = chains(d, 8, 11)
    V = np.random.default_rng(1).standard_normal((8, d.p + 1))
    out = batched.BatchedPrecisionOperator(X, om, diag).apply(V)
    for c in range(8):
        ref = pk.PrecisionOperator(X, om[c], diag[c]).apply(V[c])
        assert np.linalg.norm(out[c] - ref) <= 1e-12 * np.linalg.norm(ref)


def test_batched_config2_pcg_eight_chains():
    """Config-2 size, 8 chains (config 4's batch) on the systems of the
    reference fixture (tests/golden/config2_parity.npz; chain c = fixture seed
    c mod 5): every chain held to the single-chain parity gates of
    test_gpu_parity_config2 -- relative L2 < 1e-8 vs the reference's RMS-1e-10
    solution, at RMS 1e-6 a genuine stop (true scaled residual <= 1e-6,
    agreeing with the recursive one) and an iteration count inside the
    reference's float64 / long-double band -- and deterministic."""
    from test_gpu_parity_config2 import FIX, floor_band, inputs
    fx = np.load(FIX)
    d = synth.config_design(2, seed=0)
    X = d.matrix()
    Xo = port.design_from_pattern(d.n, d.p, d.row_ptr, d.col_idx)
    ks = [c % len(fx["seeds"]) for c in range(8)]
    sys_ = {k: inputs(d, Xo, int(fx["seeds"][k])) for k in set(ks)}
    om = np.stack([sys_[k][0]["omega"] for k in ks])
    diag = np.stack([sys_[k][0]["prior_diag"] for k in ks])
    minv = np.stack([sys_[k][0]["minv"] for k in ks])
    sc = np.stack([sys_[k][0]["scale"] for k in ks])
    B = np.stack([sys_[k][1] for k in ks])
    op = batched.BatchedPrecisionOperator(X, om, diag)
    reps = batched.batched_pcg_solve(op, B, minv, sc, config=pk.CGConfig(rtol=1e-10))
    again = batched.batched_pcg_solve(op, B, minv, sc, config=pk.CGConfig(rtol=1e-10))
    r6 = batched.batched_pcg_solve(op, B, minv, sc, config=pk.CGConfig(rtol=1e-6))
    for c, k in enumerate(ks):
        assert np.array_equal(reps[c].solution, again[c].solution)
        x_star = fx["x_1e10"][k]
        rel = np.linalg.norm(reps[c].solution - x_star) / np.linalg.norm(x_star)
        cond = sys_[k][0]
        true = port.true_rms(Xo, cond["omega"], cond["prior_diag"], B[c], r6[c].solution, cond["scale"])
        rec = float(r6[c].rms_precond_residual_trace[-1])
        lo, hi, F, counts = floor_band(fx, k)
        print(f"chain {c} (fixture seed {int(fx['seeds'][k])}): rel L2 vs reference {rel:.2e}; RMS-1e-6 "
              f"iterations {r6[c].iterations} (band [{lo}, {hi}], reference {int(fx['iters_ref'][k])}); "
              f"true RMS {true:.3e} (recursive {rec:.3e})")
        assert rel < 1e-8, (c, rel)
        assert true <= 1e-6 and abs(true - rec) <= 1e-3 * rec, (c, true, rec)
        assert lo <= r6[c].iterations <= hi, (c, r6[c].iterations, lo, hi)
    # chains holding the same system get bitwise the same solve (no cross-chain coupling)
    np.testing.assert_array_equal(reps[0].solution, reps[5].solution)


def test_batch_size_validation():
    d = synth.binary_design(100, 20, 0.01, 0.3, seed=1)
    with pytest.raises(ValueError):
        batched.BatchedPrecisionOperator(d.matrix(), np.ones((3, 100)), np.ones((3, 21)))


@pytest.mark.parametrize("R", [2, 8])
def test_batched_edge_cases_empty_rows_columns_no_intercept(R):
    """Empty rows and columns, no intercept, tiny slabs (many slabs, pieces
    split across slabs): every chain's Phi v equals the oracle's."""
    rng = np.random.default_rng(40 + R)
    n, p = 300, 70
    mask = rng.random((n, p)) < 0.08
    mask[::7] = False            # empty rows
    mask[:, ::5] = False         # empty columns
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(mask.sum(1), out=rp[1:])
    ci = np.nonzero(mask)[1].astype(np.int32)
    X = pk.SparseDesignMatrix.from_pattern(n, p, rp, ci, intercept=False)
    X.slab_max = 16
    Xo = port.design_from_pattern(n, p, rp, ci, intercept=False)
    om = rng.uniform(0.05, 0.4, (R, n))
    diag = rng.uniform(0.5, 2.0, (R, p))
    V = rng.standard_normal((R, p))
    out = batched.BatchedPrecisionOperator(X, om, diag).apply(V)
    for c in range(R):
        ref = port.phi_apply(Xo, om[c], diag[c], V[c])
        assert np.linalg.norm(out[c] - ref) <= 1e-12 * np.linalg.norm(ref)
