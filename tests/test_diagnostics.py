"""Chain statistics and error-trace host logic vs the reference (CPU).

Golden values: tests/golden/chaindiag.npz and errtrace.npz, written by the
reference's diagnostics.py (tests/golden/make_golden.py)."""
from pathlib import Path

import numpy as np
import pytest

from paper_1810_12437_b200 import diagnostics as dg
from paper_1810_12437_b200.cg import CGReport

GOLD = Path(__file__).resolve().parent / "golden"


def test_effective_sample_size_matches_reference():
    g = np.load(GOLD / "chaindiag.npz")
    series = np.split(g["series"], np.cumsum(g["lengths"])[:-1])
    got = np.array([dg.effective_sample_size(x) for x in series])
    np.testing.assert_allclose(got, g["ess"], rtol=1e-12)


def test_standardized_difference_matches_reference():
    g = np.load(GOLD / "chaindiag.npz")
    t = dg.standardized_difference_test(g["a"], g["b"])
    np.testing.assert_allclose(t.z_scores, g["z"], rtol=1e-11, atol=1e-14)
    np.testing.assert_array_equal(t.excluded, g["excluded"])
    np.testing.assert_allclose(t.ess_a, g["ess_a"], rtol=1e-12)
    with pytest.raises(ValueError):
        dg.standardized_difference_test(g["a"], g["b"][:, :3])
    with pytest.raises(ValueError):
        dg.standardized_difference_test(g["a"][:1], g["b"])


def _dense_phi(g):
    n, p = int(g["n"]), int(g["p"])
    rp, ci = g["rp"], g["ci"]
    X = np.zeros((n, p + 1))
    X[:, 0] = 1.0
    X[np.repeat(np.arange(n), np.diff(rp)), ci + 1] = 1.0
    return X.T @ (g["omega"][:, None] * X) + np.diag(g["diag"])


def _golden_report(g):
    its = list(g["iterates"])
    return CGReport(iterations=int(g["iterations"]), termination="converged",
                    rms_precond_residual_trace=g["rms"], solution=its[-1], matvec_count=len(its),
                    alphas=g["alphas"], betas=g["betas"], iterates=its)


def test_error_trace_host_operator_matches_reference():
    g = np.load(GOLD / "errtrace.npz")
    A = _dense_phi(g)
    et = dg.error_trace(_golden_report(g), g["x_star"], lambda v: A @ v)
    np.testing.assert_allclose(et.l2_error, g["l2"], rtol=1e-12)
    np.testing.assert_allclose(et.rel_coord_error, g["rel"], rtol=1e-12)
    np.testing.assert_allclose(et.phi_norm_error, g["phin"], rtol=1e-7, atol=1e-12)
    assert et.n_guarded_coords == int(g["guarded"])
    with pytest.raises(ValueError):
        rep = _golden_report(g)
        rep.iterates = None
        dg.error_trace(rep, g["x_star"], lambda v: A @ v)


def test_ritz_values_bracket_preconditioned_spectrum():
    g = np.load(GOLD / "errtrace.npz")
    A = _dense_phi(g)
    minv = g["minv"]
    S = np.sqrt(minv)
    ev = np.linalg.eigvalsh(S[:, None] * A * S[None, :])
    ritz = dg.ritz_values(_golden_report(g))
    assert ritz[0] >= ev[0] * (1 - 1e-8) and ritz[-1] <= ev[-1] * (1 + 1e-8)
    np.testing.assert_allclose(ritz[-1], ev[-1], rtol=1e-6)   # extremes converge first
    assert dg.condition_estimate(_golden_report(g)) <= ev[-1] / ev[0] * (1 + 1e-8)
