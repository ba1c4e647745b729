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
    k = min(len(et.l2_error), len(g["l2"])) - 3
    # same trajectory while the errors are far above round-off
    np.testing.assert_allclose(et.l2_error[:k], g["l2"][:k], rtol=1e-6)
    np.testing.assert_allclose(et.rel_coord_error[:k], g["rel"][:k], rtol=1e-6)
    assert et.l2_error[-1] < 1e-8 * et.l2_error[0]
    ritz = dg.ritz_values(rep)
    ref = dg.ritz_values(CGReport(0, "converged", g["rms"], None, 0, alphas=g["alphas"], betas=g["betas"]))
    np.testing.assert_allclose(ritz[[0, -1]], ref[[0, -1]], rtol=1e-6)
