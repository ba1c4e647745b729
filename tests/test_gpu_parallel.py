"""Row-sharded Phi on one GPU: G shards in one process, the allreduce emulated
by a fixed-order local sum (the decomposition the multi-GPU path uses)."""
import numpy as np
import pytest
import torch

import paper_1810_12437_b200 as pk
from paper_1810_12437_b200 import parallel, synth
from oracle import port

pytestmark = pytest.mark.gpu


def build(d, G, om, diag):
    X = d.matrix()
    parts = parallel.row_partition(d.row_ptr, G)
    shards = [parallel.local_rows(X, lo, hi) for lo, hi in parts]
    return parallel.ShardedPrecisionOperator(shards, [om[lo:hi] for lo, hi in parts], diag,
                                             group=parallel.EmulatedGroup())


@pytest.mark.parametrize("fused", [False, True])
@pytest.mark.parametrize("G", [1, 2, 5])
def test_sharded_phi_and_pcg_match_full(G, fused):
    d = synth.binary_design(2500, 400, 1e-3, 0.3, seed=8)
    rng = np.random.default_rng(1)
    om = rng.uniform(0.05, 0.3, d.n)
    lam = np.abs(rng.standard_cauchy(d.p)) + 0.05
    diag = np.concatenate([[0.0], (0.05 * lam) ** -2.0])
    minv = np.concatenate([[100.0], (0.05 * lam) ** 2])
    op = build(d, G, om, diag)
    Xo = port.design_from_pattern(d.n, d.p, d.row_ptr, d.col_idx)
    v = rng.standard_normal(d.p + 1)
    ref = port.phi_apply(Xo, om, diag, v)
    np.testing.assert_allclose(op.apply(v), ref, rtol=1e-12, atol=1e-9 * np.abs(ref).max())
    b = port.rhs(Xo, np.zeros(d.p + 1), om, diag, rng)
    M = pk.Preconditioner(pk.PreconditionerKind.AUGMENTED_PRIOR, minv)
    op.apply_count = 0
    rep = parallel.sharded_pcg_solve(op, b, M, config=pk.CGConfig(rtol=1e-10), residual_scale=np.sqrt(minv),
                                     fused=fused)
    oref = port.pcg(lambda x: port.phi_apply(Xo, om, diag, x), b, minv, np.sqrt(minv), rtol=1e-10)
    assert np.linalg.norm(rep.solution - oref.x) / np.linalg.norm(oref.x) < 1e-8
    assert rep.matvec_count == rep.iterations + 1 == op.apply_count


def test_config2_eight_shards_solution():
    d = synth.config_design(2, seed=0)
    cond = synth.config2_conditioning(d, seed=0)
    op = build(d, 8, cond["omega"], cond["prior_diag"])
    rng = np.random.default_rng(4)
    v = rng.standard_normal(d.p + 1)
    full = pk.PrecisionOperator(d.matrix(), cond["omega"], cond["prior_diag"])
    a, b_ = op.apply(v), full.apply(v)
    assert np.linalg.norm(a - b_) / np.linalg.norm(b_) < 1e-12
