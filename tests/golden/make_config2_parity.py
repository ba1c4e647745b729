"""Config-2 parity fixture from the REFERENCE implementation (priorcg), the
paper-scale gate of SURVEY §8(c): for 5 draw seeds of the config-2 recipe
(n=72,489, p=22,175, omega ~ PG(1,0), lambda ~ |Cauchy|, tau=1e-3, b from
generate_rhs) the reference pcg_solve's iteration count at RMS 1e-6, the same
solve with Phi applied in a different summation order (two row halves: the
CPU-vs-CPU floor of the iteration count), the same algorithm in extended
precision (x87 long double: Phi, dot products, single-rounding vector updates,
d'Phi d as z'Omega z + d'Dd -- the roundings the device makes more accurate
than numpy does), and for seed 0 the solution at RMS 1e-10 (the relative-L2
gate).  Inputs are regenerated from the seeds on the
GPU box (synth + oracle/port.py, pinned bit-exact against the reference);
checksums of omega and b are stored to prove it.

Run in the build container (the reference is not on the GPU box):
    python tests/golden/make_config2_parity.py      (~10 min, 5 processes)
"""
import sys
from multiprocessing import Pool
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent / "config2_parity.npz"
SEEDS = [0, 1, 2, 3, 4]
sys.path.insert(0, str(REF))
sys.path.insert(0, str(ROOT))


def inputs(seed):
    """Config-2 inputs of draw seed `seed` (reference PG sampler, reference RHS)."""
    from priorcg import polya_gamma as rpg
    from priorcg.sampler import GaussianTarget, PrecisionOperator, generate_rhs
    from priorcg.sparse import SparseDesignMatrix, hstack_dense_columns
    from paper_1810_12437_b200 import synth
    d = synth.config_design(2, seed=0)
    cond = synth.config2_conditioning(d, seed=seed, pg_sampler=rpg.pg_draw_batch)
    X = hstack_dense_columns(np.ones((d.n, 1)),
                             SparseDesignMatrix(d.n, d.p, d.row_ptr, d.col_idx.astype(np.int64),
                                                np.ones(len(d.col_idx))))
    phi = PrecisionOperator(X, cond["omega"], cond["prior_diag"])
    target = GaussianTarget.from_pseudo_outcome(phi, cond["kappa"] / cond["omega"])
    b = generate_rhs(target, cond["rng"])
    return d, X, cond, phi, b


class SplitPhi:
    """Phi v with the rows in two halves, summed afterwards: the same operator
    in another summation order (the CPU-vs-CPU iteration floor)."""

    def __init__(self, X, omega, diag):
        from priorcg.sampler import PrecisionOperator
        from priorcg.sparse import SparseDesignMatrix
        n = X.n_rows
        h = n // 2
        parts = []
        for lo, hi in ((0, h), (h, n)):
            rp = X.row_ptr[lo:hi + 1] - X.row_ptr[lo]
            sl = slice(X.row_ptr[lo], X.row_ptr[hi])
            Xs = SparseDesignMatrix(hi - lo, X.n_cols, rp, X.col_idx[sl], X.values[sl])
            parts.append(PrecisionOperator(Xs, omega[lo:hi], np.zeros(X.n_cols)))
        self.parts, self.diag = parts, diag
        self.prior_precision_diag = diag

    def apply(self, v):
        return (self.parts[0].apply(v) + self.parts[1].apply(v)) + self.diag * v


def accurate_iterations(Xo_rp, Xo_ci, n, p, cond, b, rtol=1e-6):
    """PCG (cg.py:105-192) with every reduction in long double and one rounding
    per vector update; Xo_* is the reference CSR (intercept first)."""
    import math
    L = np.longdouble
    om = cond["omega"].astype(L)
    diag, minv, scale = cond["prior_diag"], cond["minv"], cond["scale"]
    rp, ci = Xo_rp, Xo_ci
    perm = np.argsort(ci, kind="stable")
    row_of = np.repeat(np.arange(n), np.diff(rp))[perm]
    cstart = np.searchsorted(ci[perm], np.arange(p))
    ner = np.diff(rp) > 0
    empty_c = np.bincount(ci, minlength=p) == 0

    def xz(v):
        z = np.zeros(n, dtype=L)
        z[ner] = np.add.reduceat(v.astype(L)[ci], rp[:-1][ner])
        return z

    def xt(w):
        g = np.add.reduceat(w[row_of], cstart)
        g[empty_c] = 0
        return g

    def dot(u, v):
        return float(np.dot(u.astype(L), v.astype(L)))

    x = np.zeros(p)
    r = b.copy()
    k = 0
    t = scale * r
    rms = math.sqrt(dot(t, t) / p)
    z = minv * r
    rz = dot(r, z)
    dd = z.copy()
    while rms > rtol:
        k += 1
        zz = xz(dd)
        Ad = (xt(om * zz) + diag.astype(L) * dd.astype(L)).astype(np.float64)
        dAd = float(np.dot(zz, om * zz) + np.dot(dd.astype(L), diag.astype(L) * dd.astype(L)))
        alpha = rz / dAd
        x = (x.astype(L) + L(alpha) * dd.astype(L)).astype(np.float64)
        r = (r.astype(L) - L(alpha) * Ad.astype(L)).astype(np.float64)
        t = scale * r
        rms = math.sqrt(dot(t, t) / p)
        if rms <= rtol:
            break
        z = minv * r
        rzn = dot(r, z)
        beta = rzn / rz
        rz = rzn
        dd = (z.astype(L) + L(beta) * dd.astype(L)).astype(np.float64)
    return k


def run(seed):
    from priorcg.cg import CGConfig, pcg_solve
    from priorcg.precond import Preconditioner, PreconditionerKind
    d, X, cond, phi, b = inputs(seed)
    M = Preconditioner(PreconditionerKind.AUGMENTED_PRIOR, cond["minv"])
    out = {"seed": seed, "omega_sum": float(cond["omega"].sum()), "b_sum": float(b.sum()),
           "b_norm": float(np.linalg.norm(b))}
    rep = pcg_solve(phi, b, M, config=CGConfig(rtol=1e-6), residual_scale=cond["scale"])
    out["iters_ref"] = rep.iterations
    split = SplitPhi(X, cond["omega"], cond["prior_diag"])
    rep2 = pcg_solve(split, b, M, config=CGConfig(rtol=1e-6), residual_scale=cond["scale"])
    out["iters_split"] = rep2.iterations
    out["iters_accurate"] = accurate_iterations(X.row_ptr, X.col_idx, X.n_rows, X.n_cols, cond, b)
    if seed == 0:
        rep3 = pcg_solve(phi, b, M, config=CGConfig(rtol=1e-10), residual_scale=cond["scale"])
        out["x_1e10"] = rep3.solution
        out["iters_1e10"] = rep3.iterations
    print(seed, out["iters_ref"], out["iters_split"], out["iters_accurate"], flush=True)
    return out


if __name__ == "__main__":
    with Pool(len(SEEDS)) as pool:
        res = pool.map(run, SEEDS)
    np.savez_compressed(
        OUT, seeds=np.array(SEEDS), iters_ref=np.array([r["iters_ref"] for r in res]),
        iters_split=np.array([r["iters_split"] for r in res]),
        iters_accurate=np.array([r["iters_accurate"] for r in res]),
        omega_sum=np.array([r["omega_sum"] for r in res]), b_sum=np.array([r["b_sum"] for r in res]),
        b_norm=np.array([r["b_norm"] for r in res]), x_1e10=res[0]["x_1e10"],
        iters_1e10=res[0]["iters_1e10"])
    print("wrote", OUT)
