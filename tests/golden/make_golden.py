"""Writes tests/golden/*.npz from the REFERENCE implementation (priorcg).

Run in the build container (the reference is not on the GPU box):
    python tests/golden/make_golden.py
It imports priorcg read-only from /root/reference/pkg/src.  The fixtures pin
oracle/port.py (tests/test_oracle.py) and the device path (tests/test_gpu_*.py).
"""
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))
import priorcg  # noqa: E402
from priorcg import gibbs as rg  # noqa: E402
from priorcg import polya_gamma as rpg  # noqa: E402
from priorcg.cg import CGConfig, pcg_solve  # noqa: E402
from priorcg.precond import augmented_prior  # noqa: E402
from priorcg.sampler import GaussianTarget, PrecisionOperator, generate_rhs  # noqa: E402
from priorcg.sparse import SparseDesignMatrix, hstack_dense_columns  # noqa: E402

OUT = Path(__file__).resolve().parent


def binary_pattern(rng, n, p, lo, hi):
    rates = np.exp(rng.uniform(np.log(lo), np.log(hi), size=p))
    mask = rng.random((n, p)) < rates[None, :]
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(mask.sum(1), out=rp[1:])
    ci = np.nonzero(mask)[1].astype(np.int32)
    return rp, ci


def ref_design(n, p, rp, ci, intercept=True):
    X = SparseDesignMatrix(n, p, rp, ci.astype(np.int64), np.ones(len(ci)))
    if intercept:
        X = hstack_dense_columns(np.ones((n, 1)), X)
    return X


def sparse_cases():
    rng = np.random.default_rng(2024)
    out = {}
    for k, (n, p, lo, hi, icpt) in enumerate([(1, 5, 0.5, 0.9, True), (7, 3, 0.2, 0.9, False),
                                               (40, 30, 0.01, 0.5, True), (200, 60, 0.001, 0.3, True),
                                               (150, 120, 0.0, 0.0, False), (300, 500, 0.001, 0.2, True)]):
        if hi > 0:
            rp, ci = binary_pattern(rng, n, p, lo, hi)
        else:  # empty design
            rp, ci = np.zeros(n + 1, dtype=np.int64), np.zeros(0, dtype=np.int32)
        X = ref_design(n, p, rp, ci, icpt)
        v = rng.standard_normal(X.n_cols)
        w = rng.standard_normal(n)
        om = rng.uniform(0.05, 2.0, size=n)
        d = rng.uniform(0.0, 3.0, size=X.n_cols)
        phi = PrecisionOperator(X, om, d)
        out.update({f"c{k}_n": n, f"c{k}_p": p, f"c{k}_icpt": int(icpt), f"c{k}_rp": rp, f"c{k}_ci": ci,
                    f"c{k}_v": v, f"c{k}_w": w, f"c{k}_om": om, f"c{k}_d": d,
                    f"c{k}_Xv": X.matvec(v), f"c{k}_Xtw": X.matvec_t(w), f"c{k}_phiv": phi.apply(v),
                    f"c{k}_gdiag": X.gram_diagonal(om)})
    out["ncases"] = 6
    np.savez_compressed(OUT / "sparse.npz", **out)


def pcg_cases():
    rng = np.random.default_rng(77)
    n, p = 600, 150
    rp, ci = binary_pattern(rng, n, p, 1e-3, 0.2)
    X = ref_design(n, p, rp, ci)
    om = rpg.pg_draw_batch(np.zeros(n), rng)
    lam = np.abs(rng.standard_cauchy(p))
    tau = 0.05
    y = (rng.random(n) < 0.1).astype(float)
    prior = np.concatenate([[0.0], (tau * lam) ** -2.0])
    phi = PrecisionOperator(X, om, prior)
    target = GaussianTarget.from_pseudo_outcome(phi, (y - 0.5) / om)
    eta_rng = np.random.default_rng(5)
    b = generate_rhs(target, eta_rng)
    M = augmented_prior(tau, lam, np.array([10.0]))
    scale = np.concatenate([[10.0], tau * lam])
    out = dict(n=n, p=p, rp=rp, ci=ci, om=om, lam=lam, tau=tau, y=y, b=b, minv=M.inv_diagonal,
               scale=scale, prior=prior, lin=target.linear_term)
    for tag, rtol in (("r6", 1e-6), ("r10", 1e-10)):
        rep = pcg_solve(phi, b, M, config=CGConfig(rtol=rtol), residual_scale=scale)
        out.update({f"{tag}_x": rep.solution, f"{tag}_iters": rep.iterations,
                    f"{tag}_trace": rep.rms_precond_residual_trace, f"{tag}_alphas": rep.alphas,
                    f"{tag}_betas": rep.betas, f"{tag}_mv": rep.matvec_count})
    x0 = 0.5 * out["r6_x"]
    rep = pcg_solve(phi, b, M, x0=x0, config=CGConfig(rtol=1e-8, max_iter=7), residual_scale=scale)
    out.update(mi_x0=x0, mi_x=rep.solution, mi_iters=rep.iterations, mi_term=rep.termination,
               mi_trace=rep.rms_precond_residual_trace, mi_betas=rep.betas)
    # generate_rhs stream order: eta (n) then delta (p)
    rhs_rng = np.random.default_rng(99)
    out["rhs_b"] = generate_rhs(target, rhs_rng)
    chk = np.random.default_rng(99)
    out["rhs_eta"] = chk.standard_normal(n)
    out["rhs_delta"] = chk.standard_normal(p + 1)
    np.savez_compressed(OUT / "pcg.npz", **out)


def pg_cases():
    z = np.array([0.0, 0.0, 1e-6, 0.3, -0.3, 1.0, 1.5625, 2.0, 4.0, 10.0, -25.0, 60.0] * 50)
    out = {"z": z}
    for s in (0, 1, 2):
        out[f"draw_{s}"] = rpg.pg_draw_batch(z, np.random.default_rng(s))
    zz = np.linspace(-8, 8, 4001)
    out["zz"] = zz
    out["mean_zz"] = rpg.pg_mean(zz)
    np.savez_compressed(OUT / "pg.npz", **out)


def gibbs_cases():
    rng = np.random.default_rng(11)
    n, p = 250, 40
    rp, ci = binary_pattern(rng, n, p, 0.02, 0.4)
    X = ref_design(n, p, rp, ci)
    beta = np.zeros(p)
    beta[[3, 17, 29]] = [1.5, -2.0, 1.0]
    Xs = ref_design(n, p, rp, ci, intercept=False)
    y = (rng.random(n) < 1 / (1 + np.exp(-(Xs.matvec(beta) - 0.5)))).astype(float)
    cfg = rg.BridgeConfig(unshrunk_prior_sd=(np.inf,))
    ch = rg.gibbs_run(X, y, cfg, 30, burn_in=10, seed=3, thin=2)
    out = dict(n=n, p=p, rp=rp, ci=ci, y=y, draws=ch.draws, tau_draws=ch.tau_draws,
               logdens=ch.logdensity_trace, iters=ch.cg_iteration_counts,
               mean=ch.running_mean_scaled_beta, var=ch.running_var_unshrunk)
    # scale conditionals with fixed seeds
    bs = np.linspace(-2, 2, 41)
    bs[20] = 0.0
    out["bs"] = bs
    out["tau_draws_cond"] = np.array([rg.update_global_scale(bs, cfg, np.random.default_rng(s)) for s in range(20)])
    out["lam_draws_cond"] = np.stack([rg.update_local_scales(bs, 0.7, cfg, np.random.default_rng(s)) for s in range(5)])
    np.savez_compressed(OUT / "gibbs.npz", **out)


def io_cases():
    """Files written by the reference's own writers (matrixio.py, stateio.py)."""
    from priorcg import matrixio, stateio
    d = OUT / "io"
    d.mkdir(exist_ok=True)
    rng = np.random.default_rng(5)
    n, p = 23, 9
    rp, ci = binary_pattern(rng, n, p, 0.05, 0.6)
    X = ref_design(n, p, rp, ci, intercept=True)
    matrixio.write_design(d / "design_sparse.mtx", X)
    dense = np.zeros((n, p))
    dense[np.repeat(np.arange(n), np.diff(rp)), ci] = 1.0
    matrixio.write_design(d / "design_dense.mtx", dense)
    matrixio.write_design_csv(d / "design.csv", dense)
    draws = rng.standard_normal((4, 3))
    matrixio.write_chain_csv(d / "chain.csv", draws, np.exp(rng.standard_normal(4)), rng.standard_normal(4))
    matrixio.write_vector_csv(d / "vector.csv", rng.standard_normal(5) * 1e-7, "beta")
    matrixio.write_spectrum_csv(d / "spectrum.csv", np.array([3.5, 1.0, 1e-3, 0.0]))

    class _T:
        pass
    tr = _T()
    k = 6
    tr.rms_precond_residual = np.exp(-np.arange(k, dtype=float))
    tr.phi_norm_error = rng.random(k)
    tr.l2_error = rng.random(k)
    tr.rel_coord_error = np.where(np.arange(k) == 2, np.nan, rng.random(k))
    matrixio.write_trace_csv(d / "trace.csv", tr)
    state = rg.ShrinkageState(rng.standard_normal(p + 1), rng.uniform(0.1, 2.0, n),
                              rng.uniform(0.5, 3.0, p), 0.37)
    stateio.save_state(d / "state.brgs", state)
    np.savez(d / "expected.npz", rp=rp, ci=ci, dense=dense, draws=draws, beta=state.beta,
             omega=state.omega, lam=state.lam, tau=state.tau)


def error_trace_cases():
    """diagnostics.error_trace on a full-trace reference solve."""
    from priorcg.diagnostics import error_trace
    rng = np.random.default_rng(31)
    n, p = 400, 120
    rp, ci = binary_pattern(rng, n, p, 0.01, 0.3)
    X = ref_design(n, p, rp, ci)
    omega = rpg.pg_draw_batch(np.zeros(n), rng)
    tau = 0.05
    lam = np.abs(rng.standard_cauchy(p))
    diag = np.concatenate([[0.0], (tau * lam) ** -2.0])
    gamma = np.array([10.0])
    M = augmented_prior(tau, lam, gamma)
    phi = PrecisionOperator(X, omega, diag)
    b = X.matvec_t(rng.standard_normal(n)) + np.sqrt(diag) * rng.standard_normal(p + 1)
    scale = np.concatenate([gamma, tau * lam])
    rep = pcg_solve(phi, b, M, config=CGConfig(rtol=1e-12, trace_level="full"), residual_scale=scale)
    dense = np.zeros((n, p + 1))
    dense[:, 0] = 1.0
    dense[np.repeat(np.arange(n), np.diff(rp)), ci + 1] = 1.0
    A = dense.T @ (omega[:, None] * dense) + np.diag(diag)
    x_star = np.linalg.solve(A, b)
    x_star[5] = 0.0  # exercise the |beta*| < 1e-300 guard
    et = error_trace(rep, x_star, phi)
    np.savez(OUT / "errtrace.npz", n=n, p=p, rp=rp, ci=ci, omega=omega, diag=diag, minv=M.inv_diagonal,
             scale=scale, b=b, x_star=x_star, iterates=np.array(rep.iterates),
             rms=np.array(rep.rms_precond_residual_trace), iterations=rep.iterations,
             rel=et.rel_coord_error, l2=et.l2_error, phin=et.phi_norm_error, guarded=et.n_guarded_coords,
             alphas=np.array(rep.alphas), betas=np.array(rep.betas))


def chain_diag_cases():
    """effective_sample_size / standardized_difference_test (diagnostics.py:236-303)."""
    from priorcg.diagnostics import effective_sample_size, standardized_difference_test
    rng = np.random.default_rng(17)
    series = []
    for phi_ar, n in ((0.0, 200), (0.5, 300), (0.9, 500), (-0.4, 150), (0.99, 64)):
        x = np.zeros(n)
        e = rng.standard_normal(n)
        for t in range(1, n):
            x[t] = phi_ar * x[t - 1] + e[t]
        series.append(x)
    series.append(np.full(10, 3.0))
    series.append(np.array([1.0]))
    ess = np.array([effective_sample_size(x) for x in series])
    a = rng.standard_normal((120, 6)).cumsum(0) * 0.1 + rng.standard_normal((120, 6))
    b = rng.standard_normal((90, 6)) + 0.05
    b[:, 2] = a[:90, 2]
    a[:, 5] = 1.0
    b[:, 5] = 1.0
    t = standardized_difference_test(a, b)
    np.savez(OUT / "chaindiag.npz", lengths=[len(x) for x in series], series=np.concatenate(series), ess=ess,
             a=a, b=b, z=t.z_scores, excluded=t.excluded, ess_a=t.ess_a, ess_b=t.ess_b)


if __name__ == "__main__":
    print("priorcg", priorcg.__version__)
    sparse_cases()
    pcg_cases()
    pg_cases()
    gibbs_cases()
    io_cases()
    error_trace_cases()
    chain_diag_cases()
    for f in sorted(OUT.glob("*.npz")):
        print(f.name, f.stat().st_size)
