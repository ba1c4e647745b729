"""Iterate-error traces, the Lanczos view of a solve, and chain checks.

Drop-in for the parts of priorcg.diagnostics on the β-draw path
(pkg/src/priorcg/diagnostics.py):

* `error_trace(report, beta_star, phi)` (diagnostics.py:183-212): the four
  per-iteration error metrics of a `trace_level="full"` solve.  The iterates
  stay in device memory (the device PCG writes them there), the differences,
  norms and relative coordinate errors are evaluated on the GPU, and the
  Φ-norm applies the pattern-only Φ kernel to every iterate's error vector.
* `ritz_values(report)`: eigenvalues of the Lanczos tridiagonal that the CG
  coefficients define (`CGReport.lanczos_tridiagonal`, cg.py:75-86) --
  estimates of the extreme eigenvalues of M⁻¹Φ, available for any solve
  without forming Φ.
* `effective_sample_size`, `standardized_difference_test`
  (diagnostics.py:236-303): the chain-agreement statistics the parity
  procedure prescribes; host numpy over stored draws.

The dense spectrum reports of the reference (desk scale, Φ formed densely)
are out of scope.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _lib


@dataclass
class ErrorTrace:
    """Per-iterate error metrics (diagnostics.py:166-180)."""

    rel_coord_error: np.ndarray
    l2_error: np.ndarray
    phi_norm_error: np.ndarray
    rms_precond_residual: np.ndarray
    n_guarded_coords: int

    def __post_init__(self):
        if len({len(self.rel_coord_error), len(self.l2_error), len(self.phi_norm_error),
                len(self.rms_precond_residual)}) != 1:
            raise ValueError("error trace arrays must share one length")


def _device_phi(phi):
    return getattr(phi, "_pcgs_device_operator", None) is not None and hasattr(phi, "apply_into")


def error_trace(report, beta_star, phi) -> ErrorTrace:
    """rel-coordinate, l2 and Φ-norm error of every stored iterate against
    `beta_star`, plus the RMS residual trace (diagnostics.py:183-212).

    Coordinates with |beta*_j| < 1e-300 are left out of the relative error and
    counted in `n_guarded_coords`.  With a device `PrecisionOperator` the
    whole evaluation runs on the GPU (one Φ-apply per iterate); any other
    `phi` (a callable or an object with `.apply`) is applied as given."""
    if report.iterates is None:
        raise ValueError("error_trace needs a report with stored iterates (trace_level='full')")
    rms = np.asarray(report.rms_precond_residual_trace, dtype=np.float64)
    if not _device_phi(phi):
        return _error_trace_host(report, beta_star, phi, rms)
    t = _lib.torch()
    dev = phi.store.device
    its = getattr(report, "iterates_device", None)
    if its is None:
        its = t.as_tensor(np.stack([np.asarray(v, dtype=np.float64) for v in report.iterates]), device=dev)
    bs = _lib.to_device(beta_star, dev)
    if tuple(bs.shape) != (its.shape[1],):
        raise ValueError("beta_star must have one entry per coefficient")
    D = its - bs[None, :]
    l2 = t.sqrt((D * D).sum(dim=1))
    usable = bs.abs() >= 1e-300
    n_guarded = int(bs.numel() - int(usable.sum()))
    if bool(usable.any()):
        rel = (D[:, usable] / bs[usable]).abs().mean(dim=1)
    else:
        rel = t.zeros(D.shape[0], dtype=D.dtype, device=dev)
    q = t.empty(D.shape[0], dtype=D.dtype, device=dev)
    tmp = t.empty_like(bs)
    for k in range(D.shape[0]):
        phi.apply_into(D[k], tmp)
        q[k] = t.dot(D[k], tmp)
    phin = t.sqrt(t.clamp(q, min=0.0))
    return ErrorTrace(rel_coord_error=rel.cpu().numpy(), l2_error=l2.cpu().numpy(),
                      phi_norm_error=phin.cpu().numpy(), rms_precond_residual=rms,
                      n_guarded_coords=n_guarded)


def _error_trace_host(report, beta_star, phi, rms):
    """User-supplied operator: evaluated as the caller's `phi` dictates."""
    beta_star = np.asarray(beta_star, dtype=np.float64)
    apply_phi = phi.apply if hasattr(phi, "apply") else phi
    usable = np.abs(beta_star) >= 1e-300
    K = len(report.iterates)
    rel, l2, phin = np.zeros(K), np.empty(K), np.empty(K)
    for k, it in enumerate(report.iterates):
        d = np.asarray(it, dtype=np.float64) - beta_star
        l2[k] = math.sqrt(float(d @ d))
        phin[k] = math.sqrt(max(float(d @ np.asarray(apply_phi(d))), 0.0))
        if usable.any():
            rel[k] = float(np.mean(np.abs(d[usable] / beta_star[usable])))
    return ErrorTrace(rel, l2, phin, rms, int(beta_star.size - usable.sum()))


def ritz_values(report) -> np.ndarray:
    """Ascending eigenvalues of the Lanczos tridiagonal of a PCG solve: Ritz
    estimates of the spectrum of the preconditioned operator M⁻¹Φ (the
    extremes converge first), from the α/β the device loop records."""
    diag, off = report.lanczos_tridiagonal()
    if diag.size == 0:
        return np.zeros(0)
    import scipy.linalg
    return scipy.linalg.eigvalsh_tridiagonal(diag, off) if diag.size > 1 else diag.copy()


def condition_estimate(report) -> float:
    """λ_max / λ_min of the Ritz values (a lower bound on κ(M⁻¹Φ))."""
    ev = ritz_values(report)
    return float(ev[-1] / ev[0]) if ev.size and ev[0] > 0 else float("nan")


# ----------------------------------------------------------------- chain checks
def _ess_columns(draws: np.ndarray) -> np.ndarray:
    """ESS of every column at once: autocorrelations by one FFT over the
    draw axis, summed over initial positive pairs (Geyer's initial positive
    sequence), capped at the chain length -- diagnostics.py:236-262."""
    n, m = draws.shape
    if n < 2:
        return np.full(m, float(n))
    x = draws - draws.mean(axis=0)
    var = np.einsum("ij,ij->j", x, x)
    nfft = 1 << (2 * n - 1).bit_length()
    f = np.fft.rfft(x, nfft, axis=0)
    acov = np.fft.irfft(f * np.conj(f), nfft, axis=0)[:n]
    out = np.full(m, float(n))
    ok = (var > 0) & np.isfinite(var)
    npair = n // 2
    for j in np.flatnonzero(ok):
        rho = acov[:, j] / acov[0, j]
        pairs = rho[0:2 * npair:2] + rho[1:2 * npair:2]
        stop = np.flatnonzero(pairs <= 0.0)
        used = pairs[: stop[0]] if stop.size else pairs
        tau = -1.0 + 2.0 * float(used.sum())
        if tau > 0.0:
            out[j] = min(n / tau, float(n))
    return out


def effective_sample_size(x) -> float:
    """ESS of one series (initial-positive-sequence estimator, ≤ len(x))."""
    x = np.asarray(x, dtype=np.float64)
    return float(_ess_columns(x.reshape(-1, 1))[0])


@dataclass
class DifferenceTest:
    """Per-coefficient standardized mean differences of two chains (diagnostics.py:265-271)."""

    z_scores: np.ndarray
    excluded: np.ndarray
    ess_a: np.ndarray
    ess_b: np.ndarray


def standardized_difference_test(chain_a, chain_b, ess_floor=10.0) -> DifferenceTest:
    """z_j = (mean_a - mean_b) / sqrt(var_a/ESS_a + var_b/ESS_b); ≈ N(0,1)
    when both chains target the same posterior.  Coefficients whose ESS is
    below `ess_floor` in either chain are flagged `excluded`."""
    A = np.asarray(getattr(chain_a, "draws", chain_a), dtype=np.float64)
    B = np.asarray(getattr(chain_b, "draws", chain_b), dtype=np.float64)
    if A.ndim != 2 or B.ndim != 2 or A.shape[1] != B.shape[1]:
        raise ValueError("chains must store draws for the same model")
    if min(A.shape[0], B.shape[0]) < 2:
        raise ValueError("need at least two draws per chain")
    ess_a, ess_b = _ess_columns(A), _ess_columns(B)
    diff = A.mean(axis=0) - B.mean(axis=0)
    se = np.sqrt(A.var(axis=0, ddof=1) / ess_a + B.var(axis=0, ddof=1) / ess_b)
    z = np.zeros_like(diff)
    nz = diff != 0.0
    with np.errstate(divide="ignore"):
        z[nz] = diff[nz] / se[nz]
    return DifferenceTest(z_scores=z, excluded=(ess_a < ess_floor) | (ess_b < ess_floor), ess_a=ess_a, ess_b=ess_b)
