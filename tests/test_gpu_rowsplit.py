"""Fused row-split PCG (csrc/rowsplit.cu): G row shards hosted by one grid on
one GPU (the single-GPU form of the one-kernel-per-GPU exchange), checked
against the CPU oracle and the unsharded device solve."""
import numpy as np
import pytest
import torch

import paper_1810_12437_b200 as pk
from paper_1810_12437_b200 import parallel, synth
from oracle import port

pytestmark = pytest.mark.gpu


def sharded(d, G, om, diag, slab_max=0):
    X = d.matrix()
    parts = parallel.row_partition(d.row_ptr, G)
    shards = [parallel.local_rows(X, lo, hi) for lo, hi in parts]
    for s in shards:
        s.slab_max = slab_max
    return parallel.ShardedPrecisionOperator(shards, [om[lo:hi] for lo, hi in parts], diag,
                                             group=parallel.EmulatedGroup())


def small_system(seed=8):
    d = synth.binary_design(2500, 400, 1e-3, 0.3, seed=seed)
    rng = np.random.default_rng(1)
    om = rng.uniform(0.05, 0.3, d.n)
    lam = np.abs(rng.standard_cauchy(d.p)) + 0.05
    diag = np.concatenate([[0.0], (0.05 * lam) ** -2.0])
    minv = np.concatenate([[100.0], (0.05 * lam) ** 2])
    Xo = port.design_from_pattern(d.n, d.p, d.row_ptr, d.col_idx)
    b = port.rhs(Xo, np.zeros(d.p + 1), om, diag, rng)
    return d, om, diag, minv, Xo, b


@pytest.mark.parametrize("G,slab_max", [(1, 0), (2, 0), (3, 0), (4, 0), (8, 0), (2, 96), (4, 200)])
def test_fused_rowsplit_matches_oracle(G, slab_max):
    d, om, diag, minv, Xo, b = small_system()
    op = sharded(d, G, om, diag, slab_max)
    M = pk.Preconditioner(pk.PreconditionerKind.AUGMENTED_PRIOR, minv)
    rep = parallel.fused_pcg_solve(op, b, M, config=pk.CGConfig(rtol=1e-10), residual_scale=np.sqrt(minv))
    oref = port.pcg(lambda x: port.phi_apply(Xo, om, diag, x), b, minv, np.sqrt(minv), rtol=1e-10)
    assert np.linalg.norm(rep.solution - oref.x) / np.linalg.norm(oref.x) < 1e-8
    # the iteration band of summation order on this system (float64 orderings, long double)
    lo, hi, counts = port.iteration_band(Xo, om, diag, b, minv, np.sqrt(minv), rtol=1e-10)
    assert lo <= rep.iterations <= hi, (rep.iterations, counts)
    assert rep.termination == "converged"
    assert rep.matvec_count == rep.iterations + 1 == len(rep.rms_precond_residual_trace)
    assert len(rep.alphas) == rep.iterations
    # the trace is the reference metric: RMS of s * r at every iteration
    assert rep.rms_precond_residual_trace[-1] <= 1e-10 < rep.rms_precond_residual_trace[-2]


def test_fused_rowsplit_max_iter_and_warm_start():
    d, om, diag, minv, Xo, b = small_system(seed=3)
    op = sharded(d, 4, om, diag)
    M = pk.Preconditioner(pk.PreconditionerKind.AUGMENTED_PRIOR, minv)
    rep = parallel.fused_pcg_solve(op, b, M, config=pk.CGConfig(rtol=1e-30, max_iter=7),
                                   residual_scale=np.sqrt(minv))
    assert rep.termination == "max_iter" and rep.iterations == 7 and rep.matvec_count == 8
    full = parallel.fused_pcg_solve(op, b, M, config=pk.CGConfig(rtol=1e-10), residual_scale=np.sqrt(minv))
    # warm start at the solution: converged before the first step (cg.py:139-149)
    warm = parallel.fused_pcg_solve(op, b, M, x0=full.solution, config=pk.CGConfig(rtol=1e-6),
                                    residual_scale=np.sqrt(minv))
    assert warm.iterations == 0 and warm.matvec_count == 1


def test_fused_rowsplit_config2_against_reference():
    """Config 2, fixture seed 0 (the reference's own solves,
    tests/golden/config2_parity.npz): G = 2 and 8 row shards, relative L2 vs
    the reference's RMS-1e-10 solution < 1e-8, and at RMS 1e-6 the count in
    the reference's float64 / long-double band (test_gpu_parity_config2); with
    G = 2 also through the flag-exchange protocol (bitwise equal)."""
    from test_gpu_parity_config2 import FIX, floor_band, inputs
    fx = np.load(FIX)
    d = synth.config_design(2, seed=0)
    Xo = port.design_from_pattern(d.n, d.p, d.row_ptr, d.col_idx)
    cond, b = inputs(d, Xo, int(fx["seeds"][0]))
    M = pk.Preconditioner(pk.PreconditionerKind.AUGMENTED_PRIOR, cond["minv"])
    lo, hi, F, counts = floor_band(fx, 0)
    x_star = fx["x_1e10"][0]
    for G in (2, 8):
        op = sharded(d, G, cond["omega"], cond["prior_diag"])
        a = parallel.fused_pcg_solve(op, b, M, config=pk.CGConfig(rtol=1e-10), residual_scale=cond["scale"])
        again = parallel.fused_pcg_solve(op, b, M, config=pk.CGConfig(rtol=1e-10), residual_scale=cond["scale"])
        assert np.array_equal(a.solution, again.solution)          # deterministic
        rel = np.linalg.norm(a.solution - x_star) / np.linalg.norm(x_star)
        assert rel < 1e-8, (G, rel)
        r6 = parallel.fused_pcg_solve(op, b, M, config=pk.CGConfig(rtol=1e-6), residual_scale=cond["scale"])
        print(f"config 2 seed 0, {G} shards: rel L2 {rel:.2e}; {r6.iterations} iterations at RMS 1e-6 "
              f"(band [{lo}, {hi}], reference {int(fx['iters_ref'][0])})")
        assert lo <= r6.iterations <= hi, (G, r6.iterations, lo, hi)
        if G == 2:
            # the cross-GPU flag protocol (per-rank barriers, inbox epochs) at
            # config-2 size: bitwise the grid-barrier exchange
            f = parallel.fused_pcg_solve(op, b, M, config=pk.CGConfig(rtol=1e-10), residual_scale=cond["scale"],
                                         exchange="flags")
            np.testing.assert_array_equal(f.solution, a.solution)
    torch.cuda.synchronize()


@pytest.mark.parametrize("G", [2, 3, 4, 8])
def test_flag_exchange_protocol_is_bitwise_the_grid_exchange(G):
    """The cross-GPU exchange protocol (per-rank barriers, release/acquire
    inbox epochs, volatile peer loads: what a rank per GPU runs) executed
    between G rank groups of one cooperative grid gives bitwise the solve of
    the grid-barrier exchange, call after call (the epochs advance across
    calls), and matches the oracle."""
    d, om, diag, minv, Xo, b = small_system(seed=5)
    M = pk.Preconditioner(pk.PreconditionerKind.AUGMENTED_PRIOR, minv)
    cfg = pk.CGConfig(rtol=1e-10)
    grid_op = sharded(d, G, om, diag)
    flag_op = sharded(d, G, om, diag)
    for _ in range(3):
        a = parallel.fused_pcg_solve(grid_op, b, M, config=cfg, residual_scale=np.sqrt(minv))
        f = parallel.fused_pcg_solve(flag_op, b, M, config=cfg, residual_scale=np.sqrt(minv), exchange="flags")
        np.testing.assert_array_equal(f.solution, a.solution)
        np.testing.assert_array_equal(f.rms_precond_residual_trace, a.rms_precond_residual_trace)
        assert f.iterations == a.iterations
    oref = port.pcg(lambda x: port.phi_apply(Xo, om, diag, x), b, minv, np.sqrt(minv), rtol=1e-10)
    assert np.linalg.norm(f.solution - oref.x) / np.linalg.norm(oref.x) < 1e-8
