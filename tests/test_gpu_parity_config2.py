"""Paper-scale parity (BASELINE north star) against fixtures of
the REFERENCE itself (tests/golden/config2_parity.npz, made by
tests/golden/make_config2_parity.py from priorcg's own pcg_solve): the
config-2 recipe (n=72,489, p=22,175) for 5 draw seeds.

* relative L2 of the device solution vs the reference's at RMS 1e-10 < 1e-8;
* iteration count at RMS 1e-6.  On these spectra (prior precisions up to
  1e6/lambda^2) CG's count is set by rounding: the sequences of the device and
  the reference agree to 1e-12 for three iterations and part at the fourth,
  where r = r - alpha Phi d cancels ~8 digits.  The fixture holds three CPU
  runs of the same algorithm: the reference (numpy rounding), the reference
  with Phi summed in another order, and an extended-precision run (long
  double reductions and single-rounding updates, the roundings the device
  makes more accurate).  Measured on 5 seeds the reference sits 3-11 % above
  the accurate run and the device next to the accurate run, at a distance
  that changes with the device's own summation order (the plan).  The gate:
  the device count is within max(2, 5 % of the reference count) of the
  nearest of the three CPU runs, and the per-seed numbers are printed next to
  it (report the floor, do not loosen silently).
Inputs are regenerated here from the seeds (synth + the pinned oracle port)
and checked against the fixture's checksums."""
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


@pytest.mark.skipif(not FIX.exists(), reason="fixture not generated")
def test_config2_parity_against_reference(design):
    d, X, Xo = design
    fx = np.load(FIX)
    rows = []
    for k, seed in enumerate(fx["seeds"]):
        cond, b = inputs(d, Xo, int(seed))
        assert cond["omega"].sum() == pytest.approx(float(fx["omega_sum"][k]), rel=1e-13)
        assert b.sum() == pytest.approx(float(fx["b_sum"][k]), rel=1e-9, abs=1e-9 * float(fx["b_norm"][k]))
        assert np.linalg.norm(b) == pytest.approx(float(fx["b_norm"][k]), rel=1e-13)
        phi = pk.PrecisionOperator(X, cond["omega"], cond["prior_diag"])
        M = pk.Preconditioner(pk.PreconditionerKind.AUGMENTED_PRIOR, cond["minv"])
        rep = pk.pcg_solve(phi, b, M, config=pk.CGConfig(rtol=1e-6), residual_scale=cond["scale"])
        ref, split, acc = int(fx["iters_ref"][k]), int(fx["iters_split"][k]), int(fx["iters_accurate"][k])
        nearest = min(abs(rep.iterations - c) for c in (ref, split, acc))
        rows.append((int(seed), rep.iterations, ref, split, acc))
        assert rep.termination == "converged"
        assert nearest <= max(2, int(np.ceil(0.05 * ref))), rows[-1]
        if k == 0:
            tight = pk.pcg_solve(phi, b, M, config=pk.CGConfig(rtol=1e-10), residual_scale=cond["scale"])
            x = fx["x_1e10"]
            rel = np.linalg.norm(tight.solution - x) / np.linalg.norm(x)
            print(f"config 2 seed {seed}: relative L2 vs the reference at RMS 1e-10 = {rel:.2e} "
                  f"(iterations {tight.iterations} vs {int(fx['iters_1e10'])})")
            assert rel < 1e-8
    for seed, dev, ref, split, acc in rows:
        print(f"config 2 seed {seed}: iterations at RMS 1e-6 device {dev}, reference {ref} "
              f"(|diff| {abs(dev - ref)}), reference with split summation {split}, extended precision {acc}")
