"""Device sparse passes vs the oracle and the reference's golden vectors
(reference tests: test_sparse.py:23-111, test_sampler.py:41-83)."""
import numpy as np
import pytest

import paper_1810_12437_b200 as pk
from paper_1810_12437_b200 import synth
from oracle import port

pytestmark = pytest.mark.gpu
RTOL = 1e-12  # the reference's own tolerance for matvec vs dense (test_sparse.py:37)


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - b) / max(np.linalg.norm(b), 1e-300))


def random_pattern(rng, n, p, density):
    mask = rng.random((n, p)) < density
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(mask.sum(1), out=rp[1:])
    return rp, np.nonzero(mask)[1].astype(np.int32)


def test_golden_vectors(golden):
    g = golden("sparse")
    for k in range(int(g["ncases"])):
        n, p, icpt = int(g[f"c{k}_n"]), int(g[f"c{k}_p"]), bool(g[f"c{k}_icpt"])
        X = pk.SparseDesignMatrix.from_pattern(n, p, g[f"c{k}_rp"], g[f"c{k}_ci"], intercept=icpt)
        np.testing.assert_allclose(X.matvec(g[f"c{k}_v"]), g[f"c{k}_Xv"], rtol=RTOL, atol=1e-13)
        np.testing.assert_allclose(X.matvec_t(g[f"c{k}_w"]), g[f"c{k}_Xtw"], rtol=RTOL, atol=1e-13)
        phi = pk.PrecisionOperator(X, g[f"c{k}_om"], g[f"c{k}_d"])
        np.testing.assert_allclose(phi.apply(g[f"c{k}_v"]), g[f"c{k}_phiv"], rtol=RTOL, atol=1e-12)
        np.testing.assert_allclose(X.gram_diagonal(g[f"c{k}_om"]), g[f"c{k}_gdiag"], rtol=RTOL, atol=1e-13)


@pytest.mark.parametrize("slab_max", [0, 16, 48])
def test_random_designs_vs_oracle(slab_max):
    rng = np.random.default_rng(slab_max)
    for _ in range(15):
        n, p = (int(x) for x in rng.integers(1, 300, size=2))
        rp, ci = random_pattern(rng, n, p, float(rng.uniform(0.0, 0.9)))
        for icpt in (True, False):
            X = pk.SparseDesignMatrix.from_pattern(n, p, rp, ci, intercept=icpt)
            X.slab_max = slab_max
            Xo = port.design_from_pattern(n, p, rp, ci, intercept=icpt)
            v, w = rng.standard_normal(X.n_cols), rng.standard_normal(n)
            om, d = rng.uniform(0.05, 2.0, n), rng.uniform(0.0, 3.0, X.n_cols)
            assert rel(X.matvec(v), port.matvec(Xo, v)) < RTOL
            assert rel(X.matvec_t(w), port.matvec_t(Xo, w)) < RTOL
            assert rel(pk.PrecisionOperator(X, om, d).apply(v), port.phi_apply(Xo, om, d, v)) < RTOL


def test_empty_rows_columns_and_identity():
    dense = np.zeros((5, 4))
    dense[1, 2] = 1.0
    dense[4, 0] = 1.0
    X = pk.SparseDesignMatrix.from_dense(dense)
    np.testing.assert_array_equal(X.matvec(np.arange(4.0)), dense @ np.arange(4.0))
    np.testing.assert_array_equal(X.matvec_t(np.arange(5.0)), dense.T @ np.arange(5.0))
    I = pk.SparseDesignMatrix.from_dense(np.eye(2))
    np.testing.assert_array_equal(I.matvec(np.array([3.0, 4.0])), [3.0, 4.0])


def test_dimension_mismatch():
    X = pk.SparseDesignMatrix.from_dense(np.eye(3))
    with pytest.raises(ValueError):
        X.matvec(np.ones(4))
    with pytest.raises(ValueError):
        X.matvec_t(np.ones(4))


def test_adjoint_and_determinism():
    d = synth.config_design(1, seed=0)
    X = d.matrix()
    rng = np.random.default_rng(3)
    v, w = rng.standard_normal(X.n_cols), rng.standard_normal(d.n)
    np.testing.assert_allclose(X.matvec(v) @ w, v @ X.matvec_t(w), rtol=1e-12)
    first = X.matvec_t(w)
    for _ in range(3):
        assert np.array_equal(X.matvec_t(w), first)   # fixed-order reductions: bitwise repeatable
    om = rng.uniform(0.1, 1.0, d.n)
    phi = pk.PrecisionOperator(X, om, np.ones(X.n_cols))
    a = phi.apply(v)
    assert np.array_equal(phi.apply(v), a) and phi.apply_count == 2


def test_tensor_in_tensor_out():
    import torch
    d = synth.config_design(1, seed=0)
    X = d.matrix()
    v = torch.randn(X.n_cols, dtype=torch.float64, device="cuda")
    out = X.matvec(v)
    assert isinstance(out, torch.Tensor) and out.is_cuda
    np.testing.assert_allclose(out.cpu().numpy(), X.matvec(v.cpu().numpy()), rtol=0, atol=0)


def test_precision_operator_validation():
    X = pk.SparseDesignMatrix.from_dense(np.zeros((3, 2)))
    with pytest.raises(ValueError):
        pk.PrecisionOperator(X, np.ones(4), np.ones(2))
    with pytest.raises(ValueError):
        pk.PrecisionOperator(X, -np.ones(3), np.ones(2))
    with pytest.raises(ValueError):
        pk.PrecisionOperator(X, np.ones(3), np.array([1.0, np.nan]))


def test_config2_full_size_phi_vs_oracle():
    d = synth.config_design(2, seed=0)
    X = d.matrix()
    Xo = port.design_from_pattern(d.n, d.p, d.row_ptr, d.col_idx)
    rng = np.random.default_rng(0)
    om = rng.uniform(0.05, 0.5, d.n)
    diag = np.concatenate([[0.0], rng.uniform(0.1, 1e6, d.p)])
    v = rng.standard_normal(d.p + 1)
    phi = pk.PrecisionOperator(X, om, diag)
    assert rel(phi.apply(v), port.phi_apply(Xo, om, diag, v)) < RTOL
    w = rng.standard_normal(d.n)
    assert rel(X.matvec_t(w), port.matvec_t(Xo, w)) < RTOL
    assert rel(X.matvec(v), port.matvec(Xo, v)) < RTOL
