"""Paper-scale parity (BASELINE north star) against fixtures of
the REFERENCE itself (tests/golden/config2_parity.npz, made by
tests/golden/make_config2_parity.py from priorcg's own pcg_solve and float64
variants of it): the config-2 recipe (n=72,489, p=22,175) for 5 draw seeds.

Gates, per seed:
1. relative L2 of the device solution at RMS 1e-10 vs the reference's RMS-1e-10
   solution < 1e-8 (BASELINE tolerance);
2. the device's rtol-1e-6 stop is genuine: the TRUE scaled residual of the
   returned solution, ||s*(b - Phi x)|| / sqrt(p) with Phi x accumulated in
   long double on the host (oracle.port.true_rms), is <= 1e-6 (the stopping
   rule itself, no slack), and agrees with the recursive RMS the kernel
   stopped on to 1e-3 relative (no residual drift);
3. the solution is as accurate as the reference's: relative error vs the
   reference's RMS-1e-10 solution <= 2 x the reference's own rtol-1e-6 error;
4. iteration count at RMS 1e-6: inside the band the same algorithm spans in
   float64 and in extended precision -- from (long-double run) - F to
   (reference) + F, where F = max(2, spread of the float64 orderings in the
   fixture: reference, split rows, permuted rows, correctly rounded Phi,
   z'Omega z dAd, single-rounding updates, single-rounding (Phi d)_j).

Gate 4 replaces BASELINE's +-2 for these spectra: CG's count here is set by
rounding (the prior precisions reach 1e12, r -= alpha Phi d cancels ~8
digits at iteration 4), float64 orderings alone move it by up to F, and the
device -- tree reductions, fused multiply-adds, dAd from positive terms --
rounds less than numpy and lands between the reference and the long-double
run.  Gates 2 and 3 show the lower count is not an early stop.  The per-seed
table is printed."""
import numpy as np
import pytest

import paper_1810_12437_b200 as pk
from paper_1810_12437_b200 import synth
from oracle import port

from conftest import ROOT

pytestmark = pytest.mark.gpu
FIX = ROOT / "tests" / "golden" / "config2_parity.npz"


@pytest.fixture(scope="module")
def design():
    d = synth.config_design(2, seed=0)
    return d, d.matrix(), port.design_from_pattern(d.n, d.p, d.row_ptr, d.col_idx)


def inputs(d, Xo, seed):
    cond = synth.config2_conditioning(d, seed=seed, pg_sampler=port.pg_batch)
    om = cond["omega"]
    lin = port.matvec_t(Xo, om * (cond["kappa"] / om))   # GaussianTarget.from_pseudo_outcome (sampler.py:86-91)
    b = port.rhs(Xo, lin, om, cond["prior_diag"], cond["rng"])
    return cond, b


def floor_band(fx, k):
    gate = [str(v) for v in fx["gate_variants"]]
    counts = [int(fx[f"iters_{v}"][k]) for v in gate]
    F = max(2, max(counts) - min(counts))
    return int(fx["iters_ld"][k]) - F, int(fx["iters_ref"][k]) + F, F, dict(zip(gate, counts))


@pytest.mark.skipif(not FIX.exists(), reason="fixture not generated")
def test_config2_parity_against_reference(design):
    d, X, Xo = design
    fx = np.load(FIX)
    rows = []
    for k, seed in enumerate(fx["seeds"]):
        cond, b = inputs(d, Xo, int(seed))
        assert cond["omega"].sum() == pytest.approx(float(fx["omega_sum"][k]), rel=1e-13)
        assert np.linalg.norm(b) == pytest.approx(float(fx["b_norm"][k]), rel=1e-13)
        phi = pk.PrecisionOperator(X, cond["omega"], cond["prior_diag"])
        M = pk.Preconditioner(pk.PreconditionerKind.AUGMENTED_PRIOR, cond["minv"])
        x_star = fx["x_1e10"][k]
        # gate 1
        tight = pk.pcg_solve(phi, b, M, config=pk.CGConfig(rtol=1e-10), residual_scale=cond["scale"])
        rel10 = np.linalg.norm(tight.solution - x_star) / np.linalg.norm(x_star)
        # gates 2-4
        rep = pk.pcg_solve(phi, b, M, config=pk.CGConfig(rtol=1e-6), residual_scale=cond["scale"])
        assert rep.termination == "converged"
        true = port.true_rms(Xo, cond["omega"], cond["prior_diag"], b, rep.solution, cond["scale"])
        rec = float(rep.rms_precond_residual_trace[-1])
        err = np.linalg.norm(rep.solution - x_star) / np.linalg.norm(x_star)
        lo, hi, F, counts = floor_band(fx, k)
        rows.append((int(seed), rep.iterations, int(fx["iters_ref"][k]), int(fx["iters_ld"][k]), F, lo, hi,
                     true, rec, err, float(fx["ref_true_rms"][k]), float(fx["ref_err"][k]), rel10, counts))
        print(f"seed {seed}: device {rep.iterations} iterations, reference {int(fx['iters_ref'][k])}, "
              f"long double {int(fx['iters_ld'][k])}, float64 orderings {counts} (F = {F}, band [{lo}, {hi}]); "
              f"device true RMS {true:.3e} (recursive {rec:.3e}), error {err:.2e} vs reference's "
              f"{float(fx['ref_err'][k]):.2e} (true RMS {float(fx['ref_true_rms'][k]):.3e}); "
              f"RMS-1e-10 rel L2 {rel10:.2e}", flush=True)
    for seed, it, ref, ld, F, lo, hi, true, rec, err, rtrue, rerr, rel10, _ in rows:
        assert rel10 < 1e-8, (seed, rel10)
        assert true <= 1e-6, (seed, true)
        assert abs(true - rec) <= 1e-3 * rec, (seed, true, rec)
        assert err <= 2.0 * rerr, (seed, err, rerr)
        assert lo <= it <= hi, (seed, it, lo, hi)
