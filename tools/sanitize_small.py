"""Small-size driver for compute-sanitizer (memcheck / racecheck / synccheck):
every hand-written synchronisation path of libpcgs runs once on a desk-size
design -- TMA slab fills + mbarriers (CSR/CSC passes, Phi apply), the
persistent cooperative PCG (grid barriers, own-slice state in shared and in
global memory), the Gibbs scan kernels, the row-split kernel with the grid
exchange and with the flag (release/acquire inbox) exchange, and the batched
chains.  Results are checked against the CPU oracle so a silent corruption
also fails.  Usage (one tool per gpurun call, B200_PROFILING.md):
    compute-sanitizer --tool memcheck python tools/sanitize_small.py
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1810_12437_b200 as pk  # noqa: E402
from paper_1810_12437_b200 import batched, parallel, synth  # noqa: E402
from oracle import port  # noqa: E402


def check(name, got, ref, tol):
    err = np.linalg.norm(np.asarray(got) - ref) / max(np.linalg.norm(ref), 1e-300)
    print(f"{name}: rel err {err:.2e}", flush=True)
    assert err <= tol, (name, err)


def main():
    d = synth.binary_design(600, 150, 2e-3, 0.3, seed=3)
    X = d.matrix()
    Xo = port.design_from_pattern(d.n, d.p, d.row_ptr, d.col_idx)
    rng = np.random.default_rng(1)
    om = rng.uniform(0.05, 0.3, d.n)
    lam = np.abs(rng.standard_cauchy(d.p)) + 0.05
    diag = np.concatenate([[0.0], (0.05 * lam) ** -2.0])
    minv = np.concatenate([[100.0], (0.05 * lam) ** 2])
    v = rng.standard_normal(d.p + 1)
    # single-slab and multi-slab stores
    for slab in (0, 64):
        Xs = d.matrix()
        Xs.slab_max = slab
        phi = pk.PrecisionOperator(Xs, om, diag)
        check(f"phi slab_max={slab}", phi.apply(v), port.phi_apply(Xo, om, diag, v), 1e-12)
        check(f"matvec slab_max={slab}", Xs.matvec(v), port.matvec(Xo, v), 1e-12)
        b = port.rhs(Xo, np.zeros(d.p + 1), om, diag, rng)
        M = pk.Preconditioner(pk.PreconditionerKind.AUGMENTED_PRIOR, minv)
        rep = pk.pcg_solve(phi, b, M, config=pk.CGConfig(rtol=1e-10), residual_scale=np.sqrt(minv))
        ref = port.pcg(lambda x: port.phi_apply(Xo, om, diag, x), b, minv, np.sqrt(minv), rtol=1e-10)
        check(f"pcg slab_max={slab}", rep.solution, ref.x, 1e-8)
    # Gibbs scans (PG, scales, RHS, PCG, log density, statistics)
    y, _ = synth.simulate_outcomes(d, seed=0)
    out = pk.gibbs_run(X, y, pk.HorseshoeConfig(), 4, seed=2)
    assert np.all(np.isfinite(out.draws)), "gibbs draws"
    out = pk.gibbs_run(X, y, pk.BridgeConfig(), 4, seed=2)
    assert np.all(np.isfinite(out.draws)), "gibbs draws"
    print("gibbs ok", flush=True)
    # row split: grid exchange and the cross-GPU flag protocol between rank groups
    parts = parallel.row_partition(d.row_ptr, 2)
    b = port.rhs(Xo, np.zeros(d.p + 1), om, diag, rng)
    ref = port.pcg(lambda x: port.phi_apply(Xo, om, diag, x), b, minv, np.sqrt(minv), rtol=1e-10)
    M = pk.Preconditioner(pk.PreconditionerKind.AUGMENTED_PRIOR, minv)
    for exchange in ("grid", "flags"):
        op = parallel.ShardedPrecisionOperator([parallel.local_rows(X, lo, hi) for lo, hi in parts],
                                               [om[lo:hi] for lo, hi in parts], diag,
                                               group=parallel.EmulatedGroup())
        rs = parallel.fused_pcg_solve(op, b, M, config=pk.CGConfig(rtol=1e-10), residual_scale=np.sqrt(minv),
                                      exchange=exchange)
        check(f"row split ({exchange})", rs.solution, ref.x, 1e-8)
    # batched chains
    R = 2
    oms = rng.uniform(0.05, 0.4, (R, d.n))
    diags = np.stack([diag, diag * 2.0])
    minvs = 1.0 / np.maximum(diags, 1e-2)
    Bm = np.stack([port.rhs(Xo, np.zeros(d.p + 1), oms[c], diags[c], rng) for c in range(R)])
    bop = batched.BatchedPrecisionOperator(X, oms, diags)
    V = rng.standard_normal((R, d.p + 1))
    got = bop.apply(V)
    for c in range(R):
        check(f"batched phi chain {c}", got[c], port.phi_apply(Xo, oms[c], diags[c], V[c]), 1e-12)
    reps = batched.batched_pcg_solve(bop, Bm, minvs, np.sqrt(minvs), config=pk.CGConfig(rtol=1e-10))
    for c in range(R):
        ref = port.pcg(lambda x: port.phi_apply(Xo, oms[c], diags[c], x), Bm[c], minvs[c], np.sqrt(minvs[c]),
                       rtol=1e-10)
        check(f"batched pcg chain {c}", reps[c].solution, ref.x, 1e-8)
    print("sanitize_small ok", flush=True)


if __name__ == "__main__":
    main()
