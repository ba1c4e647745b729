"""Seeded synthetic binary designs for the BASELINE.json configurations.

The paper's clinical cohort is proprietary and absent, so
these stand in for it.  Recipe: column j gets a
rate r_j = exp(U(ln a, ln b)); k_j ~ Binomial(n, r_j) distinct rows are chosen
without replacement; the dense intercept is kept separate (pattern flag).
With seed 0, config 2 realises 59,928,655 nonzeros, the figure the survey
measured with the same recipe.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

CONFIGS = {
    1: dict(n=2_000, p=500, rate_lo=1e-3, rate_hi=0.2),
    2: dict(n=72_489, p=22_175, rate_lo=1e-4, rate_hi=0.3),
    3: dict(n=72_489, p=22_175, rate_lo=1e-4, rate_hi=0.3),
    4: dict(n=72_489, p=22_175, rate_lo=1e-4, rate_hi=0.3),
    5: dict(n=1_000_000, p=100_000, rate_lo=1e-5, rate_hi=0.1),
}


@dataclass
class BinaryDesign:
    n: int
    p: int
    row_ptr: np.ndarray   # int64[n+1], shrunk block
    col_idx: np.ndarray   # int32[nnz], shrunk block, sorted within rows
    rates: np.ndarray     # float64[p]

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def matrix(self, intercept=True):
        from .sparse import SparseDesignMatrix
        return SparseDesignMatrix.from_pattern(self.n, self.p, self.row_ptr, self.col_idx,
                                               intercept=intercept, check=False)

    def scipy_csr(self, intercept=True):
        """scipy CSR with the intercept as column 0 (tests / oracle)."""
        import scipy.sparse as sp
        X = sp.csr_matrix((np.ones(self.nnz), self.col_idx.astype(np.int64), self.row_ptr),
                          shape=(self.n, self.p))
        if intercept:
            X = sp.hstack([sp.csr_matrix(np.ones((self.n, 1))), X], format="csr")
            X.sort_indices()
        return X


def binary_design(n, p, rate_lo, rate_hi, seed=0) -> BinaryDesign:
    rng = np.random.default_rng(seed)
    rates = np.exp(rng.uniform(np.log(rate_lo), np.log(rate_hi), size=p))
    counts = rng.binomial(n, rates)
    nnz = int(counts.sum())
    rows = np.empty(nnz, dtype=np.int32)
    cols = np.empty(nnz, dtype=np.int32)
    pos = 0
    for j in range(p):
        k = int(counts[j])
        if k:
            rows[pos:pos + k] = rng.choice(n, size=k, replace=False)
            cols[pos:pos + k] = j
            pos += k
    # CSC (column-major, rows random within a column) -> CSR sorted by (row, col)
    order = np.argsort(rows, kind="stable")  # stable keeps columns ascending within a row
    col_idx = cols[order]
    row_counts = np.bincount(rows, minlength=n)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(row_counts, out=row_ptr[1:])
    return BinaryDesign(n=n, p=p, row_ptr=row_ptr, col_idx=col_idx, rates=rates)


def config_design(config: int, seed=0) -> BinaryDesign:
    c = CONFIGS[config]
    if config == 5:   # 1.09e9 nonzeros: native generator (same recipe, different RNG)
        return native_binary_design(c["n"], c["p"], c["rate_lo"], c["rate_hi"], seed=seed)
    return binary_design(c["n"], c["p"], c["rate_lo"], c["rate_hi"], seed=seed)


def native_binary_design(n, p, rate_lo, rate_hi, seed=0) -> BinaryDesign:
    """The binary_design recipe generated in C++ (libpcgs `pcgs_synth_design`,
    xoshiro256** stream): O(nnz) time and memory, for config 5's ~1.09e9 entries."""
    import ctypes
    from . import _lib
    L = _lib.lib()
    row_ptr = np.empty(n + 1, dtype=np.int64)
    nnz = ctypes.c_int64()
    _lib.check(L.pcgs_synth_design(n, p, float(rate_lo), float(rate_hi), seed, row_ptr.ctypes.data,
                                   None, 0, ctypes.byref(nnz)))
    col_idx = np.empty(nnz.value, dtype=np.int32)
    _lib.check(L.pcgs_synth_design(n, p, float(rate_lo), float(rate_hi), seed, row_ptr.ctypes.data,
                                   col_idx.ctypes.data, col_idx.size, ctypes.byref(nnz)))
    return BinaryDesign(n=n, p=p, row_ptr=row_ptr, col_idx=col_idx, rates=np.full(p, np.nan))


def config2_conditioning(design: BinaryDesign, seed=0, pg_sampler=None):
    """Fixed conditioning values of config 2 (BASELINE.json configs[1]).

    omega_i ~ PG(1, 0) (drawn by `pg_sampler(z, rng)`, default: the device
    sampler), lambda_j = |Cauchy(0,1)|, tau = 1e-3, y ~ Bernoulli(0.02),
    kappa = y - 1/2.  Intercept: flat prior (d_0 = 0) with gamma_0 = 10, the
    reference's cold start (precond.py:148-153).
    Returns dict with omega, lam, tau, y, kappa, prior_diag, minv, scale (all
    in the reference layout: intercept first).
    """
    rng = np.random.default_rng(seed + 1)
    if pg_sampler is None:
        from .polya_gamma import pg_draw_batch as pg_sampler
    omega = np.asarray(pg_sampler(np.zeros(design.n), rng), dtype=np.float64)
    lam = np.abs(rng.standard_cauchy(design.p))
    tau = 1e-3
    y = (rng.random(design.n) < 0.02).astype(np.float64)
    kappa = y - 0.5
    gamma0 = 10.0
    prior_diag = np.concatenate([[0.0], (tau * lam) ** -2.0])
    minv = np.concatenate([[gamma0 ** 2], (tau * lam) ** 2])
    scale = np.concatenate([[gamma0], tau * lam])
    return dict(omega=omega, lam=lam, tau=tau, y=y, kappa=kappa, prior_diag=prior_diag,
                minv=minv, scale=scale, rng=rng)


def simulate_outcomes(design: BinaryDesign, seed=0, n_signal=10, rate=None, intercept=True):
    """Truth beta with `n_signal` N(0,1) nonzeros at random shrunk positions;
    y ~ Bernoulli(logistic(X beta + c)).  With `rate`, the intercept offset c is
    set by bisection so that mean P(y=1) equals `rate` (the rare-outcome
    configurations); otherwise c = 0.  Returns (y, beta_true) with beta_true in
    the reference layout (intercept first when `intercept`)."""
    import scipy.sparse as sp
    rng = np.random.default_rng(seed + 17)
    beta = np.zeros(design.p)
    pos = rng.choice(design.p, size=min(n_signal, design.p), replace=False)
    beta[pos] = rng.standard_normal(len(pos))
    X = sp.csr_matrix((np.ones(design.nnz), design.col_idx.astype(np.int64), design.row_ptr),
                      shape=(design.n, design.p))
    eta = X @ beta
    c = 0.0
    if rate is not None:
        lo, hi = -40.0, 40.0
        for _ in range(200):
            c = 0.5 * (lo + hi)
            m = float(np.mean(1.0 / (1.0 + np.exp(-(eta + c)))))
            if m > rate:
                hi = c
            else:
                lo = c
    prob = 1.0 / (1.0 + np.exp(-(eta + c)))
    y = (rng.random(design.n) < prob).astype(np.float64)
    full = np.concatenate([[c], beta]) if intercept else beta
    return y, full
