"""Config-2 parity fixture from the REFERENCE implementation (priorcg), the
paper-scale gate of SURVEY §8(c).  For 5 draw seeds of the config-2 recipe
(n=72,489, p=22,175, omega ~ PG(1,0), lambda ~ |Cauchy|, tau=1e-3, b from
the reference's generate_rhs) it records:

* ``iters_<variant>``: iterations to RMS 1e-6 of the SAME float64 PCG
  (cg.py:105-192) in several summation orders / rounding placements, all of
  them float64 programs:
    - ``ref``     the reference pcg_solve + PrecisionOperator, unmodified;
    - ``split``   Phi summed over two row halves, then added;
    - ``perm``    Phi with the rows in a seeded random order and the columns
                  of every row reversed (another reduceat / bincount order);
    - ``cr``      Phi correctly rounded (every sum accumulated in long double,
                  rounded once to float64; the rest of the loop is the
                  reference's float64 numpy code);
    - ``dad``     the reference loop with d'Phi d formed as z'Omega z + d'Dd
                  (z = X d), the formula the device uses;
    - ``fma``     the reference loop with single-rounding x / r / d updates
                  (what fused multiply-adds do);
    - ``fmaAd``   the reference Phi with (Phi d)_j = colsum_j + D_j d_j
                  rounded once (what an FMA does with the huge prior term);
  The spread max - min over these is the float64 ordering floor of the
  iteration count that the device gate uses.
* ``iters_ld``: the same algorithm with every reduction AND update in long
  double (informational, not a gate comparator).
* ``x_1e10``: the reference solution at RMS 1e-10, per seed (the relative-L2
  gate, and the exact solution the rtol-1e-6 errors are measured against).
* ``ref_true_rms`` / ``ref_err``: the reference's rtol-1e-6 solution's TRUE
  scaled residual (oracle.port.true_rms: Phi x accumulated in long double)
  and its relative error vs x_1e10.  The device solution is held to the same
  two quantities in tests/test_gpu_parity_config2.py.

Inputs are regenerated from the seeds on the GPU box (synth + oracle/port.py,
pinned bit-exact against the reference); checksums of omega and b are stored
to prove it.  Run in the build container (the reference is not on the GPU box):
    python tests/golden/make_config2_parity.py      (~45 min on 8 cores)
"""
import math
import sys
from multiprocessing import Pool
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent / "config2_parity.npz"
SEEDS = [0, 1, 2, 3, 4]
VARIANTS = ["ref", "split", "perm", "cr", "dad", "fma", "fmaAd", "ld", "tight"]
GATE_VARIANTS = ["ref", "split", "perm", "cr", "dad", "fma", "fmaAd"]
sys.path.insert(0, str(REF))
sys.path.insert(0, str(ROOT))

_CACHE = {}


def inputs(seed):
    """Config-2 inputs of draw seed `seed` (reference PG sampler, reference RHS)."""
    if seed in _CACHE:
        return _CACHE[seed]
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
    _CACHE.clear()
    _CACHE[seed] = (d, X, cond, phi, b)
    return _CACHE[seed]


class SplitPhi:
    """Phi v with the rows in two halves, summed afterwards."""

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

    def apply(self, v):
        return (self.parts[0].apply(v) + self.parts[1].apply(v)) + self.diag * v


class PermPhi:
    """Phi v with the rows in a seeded random order and every row's columns
    reversed: reduceat row sums and bincount column sums in another order."""

    def __init__(self, X, omega, diag, seed):
        n = X.n_rows
        order = np.random.default_rng(1000 + seed).permutation(n)
        cnt = np.diff(X.row_ptr)[order]
        rp = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(cnt, out=rp[1:])
        ci = np.concatenate([X.col_idx[X.row_ptr[i]:X.row_ptr[i + 1]][::-1] for i in order])
        self.rp, self.ci, self.p = rp, ci, X.n_cols
        self.row_of = np.repeat(np.arange(n), cnt)
        self.ne = np.flatnonzero(cnt > 0)
        self.om = omega[order]
        self.diag = diag

    def apply(self, v):
        z = np.zeros(len(self.om))
        z[self.ne] = np.add.reduceat(v[self.ci], self.rp[self.ne])
        w = self.om * z
        out = np.bincount(self.ci, weights=w[self.row_of], minlength=self.p)
        out += self.diag * v
        return out


class CrPhi:
    """Correctly rounded Phi v (oracle.port.phi_apply_exact)."""

    def __init__(self, X, omega, diag):
        from oracle import port
        self.port = port
        self.Xo = port.Csr(X.n_rows, X.n_cols, X.row_ptr, X.col_idx, X.values)
        self.om, self.diag = omega, diag

    def apply(self, v):
        return self.port.phi_apply_exact(self.Xo, self.om, self.diag, v)


def cg_variant(apply, b, minv, scale, rtol=1e-6, dad=None, fma=False, ld=False):
    """cg.py:105-192 (x0 = 0, prior-kind M) with optional knobs: `dad(d, Ad)`
    replaces float(np.dot(d, Ad)); `fma` rounds x, r, d updates once; `ld`
    makes every dot product and update long double (rounded to float64)."""
    L = np.longdouble
    p = len(b)

    def dot(u, v):
        return float(np.dot(u.astype(L), v.astype(L))) if ld else float(np.dot(u, v))

    def axpy(a, u, y):  # y + a u
        if fma or ld:
            return (y.astype(L) + L(a) * u.astype(L)).astype(np.float64)
        return y + a * u

    x = np.zeros(p)
    r = b - apply(x)
    t = scale * r
    rms = math.sqrt(dot(t, t) / p)
    k = 0
    if rms <= rtol:
        return k, x
    z = minv * r
    rz = dot(r, z)
    d = z.copy()
    while True:
        k += 1
        Ad = apply(d)
        dAd = dad(d, Ad) if dad else dot(d, Ad)
        alpha = rz / dAd
        x = axpy(alpha, d, x)
        r = axpy(-alpha, Ad, r)
        t = scale * r
        rms = math.sqrt(dot(t, t) / p)
        if rms <= rtol:
            return k, x
        z = minv * r
        rzn = dot(r, z)
        beta = rzn / rz
        rz = rzn
        if fma or ld:
            d = (z.astype(L) + L(beta) * d.astype(L)).astype(np.float64)
        else:
            d *= beta
            d += z


def run(task):
    seed, variant = task
    from priorcg.cg import CGConfig, pcg_solve
    from priorcg.precond import Preconditioner, PreconditionerKind
    from oracle import port
    d, X, cond, phi, b = inputs(seed)
    om, diag, minv, scale = cond["omega"], cond["prior_diag"], cond["minv"], cond["scale"]
    M = Preconditioner(PreconditionerKind.AUGMENTED_PRIOR, minv)
    out = {"seed": seed, "variant": variant}
    if variant == "ref":
        rep = pcg_solve(phi, b, M, config=CGConfig(rtol=1e-6), residual_scale=scale)
        out["iters"] = rep.iterations
        out["x"] = rep.solution
        out["omega_sum"] = float(om.sum())
        out["b_sum"] = float(b.sum())
        out["b_norm"] = float(np.linalg.norm(b))
        # sanity: the knob-free restatement reproduces the reference count
        k, _ = cg_variant(phi.apply, b, minv, scale)
        assert k == rep.iterations, (k, rep.iterations)
    elif variant == "tight":
        rep = pcg_solve(phi, b, M, config=CGConfig(rtol=1e-10), residual_scale=scale)
        out["iters"] = rep.iterations
        out["x"] = rep.solution
    elif variant == "split":
        out["iters"], _ = cg_variant(SplitPhi(X, om, diag).apply, b, minv, scale)
    elif variant == "perm":
        out["iters"], _ = cg_variant(PermPhi(X, om, diag, seed).apply, b, minv, scale)
    elif variant == "cr":
        out["iters"], _ = cg_variant(CrPhi(X, om, diag).apply, b, minv, scale)
    elif variant == "dad":
        Xo = port.Csr(X.n_rows, X.n_cols, X.row_ptr, X.col_idx, X.values)

        def dad(dv, Ad):
            z = port.matvec(Xo, dv)
            return float(np.dot(z, om * z) + np.dot(dv, diag * dv))
        out["iters"], _ = cg_variant(phi.apply, b, minv, scale, dad=dad)
    elif variant == "fma":
        out["iters"], _ = cg_variant(phi.apply, b, minv, scale, fma=True)
    elif variant == "fmaAd":
        Xo = port.Csr(X.n_rows, X.n_cols, X.row_ptr, X.col_idx, X.values)
        L = np.longdouble

        def apply_fma_ad(v):
            cs = port.matvec_t(Xo, om * port.matvec(Xo, v))
            return (cs.astype(L) + diag.astype(L) * v.astype(L)).astype(np.float64)
        out["iters"], _ = cg_variant(apply_fma_ad, b, minv, scale)
    elif variant == "ld":
        cr = CrPhi(X, om, diag)
        Xo = cr.Xo

        def dad_ld(dv, Ad):
            L = np.longdouble
            return float(np.dot(dv.astype(L), port.phi_apply_exact_ld(Xo, om, diag, dv)))
        out["iters"], _ = cg_variant(cr.apply, b, minv, scale, dad=dad_ld, ld=True)
    print(seed, variant, out["iters"], flush=True)
    return out


def merge(variants):
    """Add `variants` (iteration counts only) to the existing fixture."""
    with Pool(min(6, len(SEEDS) * len(variants)), maxtasksperchild=1) as pool:
        res = pool.map(run, [(s, v) for s in SEEDS for v in variants], chunksize=1)
    fx = dict(np.load(OUT))
    for v in variants:
        fx[f"iters_{v}"] = np.array([[r for r in res if r["seed"] == s and r["variant"] == v][0]["iters"]
                                     for s in SEEDS])
    fx["gate_variants"] = np.array(GATE_VARIANTS)
    np.savez_compressed(OUT, **fx)
    print("merged", variants, "into", OUT)


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--merge":
        merge(sys.argv[2].split(","))
        sys.exit(0)
    tasks = [(s, v) for s in SEEDS for v in VARIANTS]
    with Pool(6, maxtasksperchild=1) as pool:
        res = pool.map(run, tasks, chunksize=1)
    by = {(r["seed"], r["variant"]): r for r in res}
    from oracle import port
    fields = {f"iters_{v}": np.array([by[(s, v)]["iters"] for s in SEEDS]) for v in VARIANTS}
    x_tight = np.stack([by[(s, "tight")]["x"] for s in SEEDS])
    ref_true, ref_err = [], []
    for i, s in enumerate(SEEDS):
        d, X, cond, phi, b = inputs(s)
        Xo = port.Csr(X.n_rows, X.n_cols, X.row_ptr, X.col_idx, X.values)
        x6 = by[(s, "ref")]["x"]
        ref_true.append(port.true_rms(Xo, cond["omega"], cond["prior_diag"], b, x6, cond["scale"]))
        ref_err.append(np.linalg.norm(x6 - x_tight[i]) / np.linalg.norm(x_tight[i]))
        print(s, "ref true rms", ref_true[-1], "err", ref_err[-1], flush=True)
    np.savez_compressed(
        OUT, seeds=np.array(SEEDS), gate_variants=np.array(GATE_VARIANTS),
        omega_sum=np.array([by[(s, "ref")]["omega_sum"] for s in SEEDS]),
        b_sum=np.array([by[(s, "ref")]["b_sum"] for s in SEEDS]),
        b_norm=np.array([by[(s, "ref")]["b_norm"] for s in SEEDS]),
        x_1e10=x_tight, iters_1e10=fields.pop("iters_tight"),
        ref_true_rms=np.array(ref_true), ref_err=np.array(ref_err), **fields)
    print("wrote", OUT)
