"""Device error traces vs the reference's
diagnostics.error_trace on the same iterates (tests/golden/errtrace.npz)."""
from pathlib import Path

import numpy as np
import pytest

import paper_1810_12437_b200 as pk
from paper_1810_12437_b200 import diagnostics as dg
from paper_1810_12437_b200.cg import CGReport

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"


def golden():
    g = np.load(GOLD / "errtrace.npz")
    X = pk.SparseDesignMatrix.from_pattern(int(g["n"]), int(g["p"]), g["rp"], g["ci"], intercept=True)
    phi = pk.PrecisionOperator(X, g["omega"], g["diag"])
    return g, phi


def test_device_error_trace_on_reference_iterates():
    g, phi = golden()
    its = list(g["iterates"])
    rep = CGReport(iterations=len(its) - 1, termination="converged", rms_precond_residual_trace=g["rms"],
                   solution=its[-1], matvec_count=len(its), alphas=g["alphas"], betas=g["betas"], iterates=its)
    et = dg.error_trace(rep, g["x_star"], phi)
    np.testing.assert_allclose(et.l2_error, g["l2"], rtol=1e-12)
    np.testing.assert_allclose(et.rel_coord_error, g["rel"], rtol=1e-12)
    # the Phi-norm of tiny errors is a difference of O(1) terms: compare relative to the first
    np.testing.assert_allclose(et.phi_norm_error, g["phin"], rtol=1e-9, atol=1e-9 * g["phin"][0])
    assert et.n_guarded_coords == int(g["guarded"])
    np.testing.assert_array_equal(et.rms_precond_residual, g["rms"])


def test_device_solve_then_error_trace():
    g, phi = golden()
    M = pk.Preconditioner(pk.PreconditionerKind.AUGMENTED_PRIOR, g["minv"])
    rep = pk.pcg_solve(phi, g["b"], M, config=pk.CGConfig(rtol=1e-12, trace_level="full"),
                       residual_scale=g["scale"])
    assert rep.iterates_device is not None and abs(rep.iterations - int(g["iterations"])) <= 2
    et = dg.error_trace(rep, g["x_star"], phi)
    # This instance (tiny tau, Cauchy lambda, flat intercept) has a near-breakdown
    # at iteration 6 (the RMS jumps 30x), where summation order alone moves
    # alpha_6 by O(1) -- measured: alphas agree to 1e-15 through k = 4, 5e-9 at
    # k = 5.  Compare the well-determined prefix and the converged end.
    np.testing.assert_allclose(et.l2_error[:5], g["l2"][:5], rtol=1e-9)
    np.testing.assert_allclose(et.rel_coord_error[:5], g["rel"][:5], rtol=1e-7)  # |dx/x*| amplifies tiny x*
    np.testing.assert_allclose(et.phi_norm_error[:5], g["phin"][:5], rtol=1e-8)
    np.testing.assert_allclose(et.l2_error[-1], g["l2"][-1], rtol=1e-6)
    assert et.rel_coord_error[-1] < 1e-10 and g["rel"][-1] < 1e-10  # both at round-off
    ritz = dg.ritz_values(rep)
    ref = dg.ritz_values(CGReport(0, "converged", g["rms"], None, 0, alphas=g["alphas"], betas=g["betas"]))
    np.testing.assert_allclose(ritz[[0, -1]], ref[[0, -1]], rtol=1e-4)
