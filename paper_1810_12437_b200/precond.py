"""Diagonal preconditioners for the device PCG (drop-in for priorcg.precond).

On the B200 path M⁻¹ is a p-vector (`inv_diagonal`) that the persistent PCG
kernel applies inside its own vector update -- there is no separate
preconditioner kernel.  The factories keep the reference's names, meaning
and errors (pkg/src/priorcg/precond.py:22-153):

=====================  =========================  ==========================
factory                M⁻¹ (inv_diagonal)          reference
=====================  =========================  ==========================
identity_preconditioner  1                         precond.py:82-84
prior_preconditioner     (τλ)²                     precond.py:87-102
jacobi_preconditioner    1 / diag(Φ)               precond.py:105-117
augmented_prior          [γ², (τλ)²]               precond.py:120-134
=====================  =========================  ==========================

diag(XᵀΩX) for Jacobi is one pattern-only CSC pass on the device
(`SparseDesignMatrix.gram_diagonal`).  The block-threshold kind
(precond.py:156-181) is a dense desk-scale comparison and is not on the
B200 path: constructing it raises NotImplementedError.
"""
from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np


class PreconditionerKind(enum.Enum):
    IDENTITY = "identity"
    PRIOR = "prior"
    AUGMENTED_PRIOR = "augmented"
    JACOBI = "jacobi"
    BLOCK_THRESHOLD = "block"


class DegeneratePreconditionerError(ValueError):
    """M⁻¹ would have a zero, negative or non-finite entry (precond.py:30)."""


def _as_f64(x):
    return np.asarray(x, dtype=np.float64)


def _all_positive_finite(x) -> bool:
    x = _as_f64(x)
    return bool(np.all(np.isfinite(x)) and np.all(x > 0))


@dataclass
class Preconditioner:
    """M⁻¹ = diag(inv_diagonal), validated on construction (precond.py:34-79)."""

    kind: PreconditionerKind
    inv_diagonal: np.ndarray

    def __post_init__(self):
        self.inv_diagonal = _as_f64(self.inv_diagonal)
        if not _all_positive_finite(self.inv_diagonal):
            raise DegeneratePreconditionerError(
                "inverse-diagonal entries must be finite and strictly positive")

    @property
    def dim(self) -> int:
        return int(self.inv_diagonal.size)

    def apply_inverse(self, v):
        return self.inv_diagonal * v

    def to_dense_inverse(self):
        return np.diag(self.inv_diagonal)


def identity_preconditioner(p):
    return Preconditioner(PreconditionerKind.IDENTITY, np.ones(p))


def _prior_variances(tau, lam):
    if not (np.isfinite(tau) and tau > 0):
        raise ValueError("tau must be positive and finite")
    if not _all_positive_finite(lam):
        raise ValueError("lambda entries must be positive and finite")
    return (tau * _as_f64(lam)) ** 2


def prior_preconditioner(tau, lam):
    """M⁻¹ = τ²Λ², the prior covariance of the shrunk block."""
    return Preconditioner(PreconditionerKind.PRIOR, _prior_variances(tau, lam))


def augmented_prior(tau, lam, gamma):
    """Prior preconditioner extended over the unshrunk block by γ²."""
    gamma = _as_f64(gamma)
    if gamma.size == 0:
        return prior_preconditioner(tau, lam)
    if not _all_positive_finite(gamma):
        raise ValueError("gamma entries must be positive and finite")
    return Preconditioner(PreconditionerKind.AUGMENTED_PRIOR,
                          np.concatenate([gamma ** 2, _prior_variances(tau, lam)]))


def jacobi_preconditioner(X, omega, tau, lam, prior_precision=None):
    """M⁻¹ = 1/diag(Φ), diag(Φ) = diag(XᵀΩX) + prior precision."""
    if prior_precision is None:
        prior_precision = 1.0 / _prior_variances(tau, lam)
    diag_phi = _as_f64(X.gram_diagonal(omega)) + prior_precision
    if not _all_positive_finite(diag_phi):
        raise DegeneratePreconditionerError("Phi has a nonpositive diagonal entry")
    return Preconditioner(PreconditionerKind.JACOBI, 1.0 / diag_phi)


def gamma_policy(chain, c=1.0, prior_sd=None, sd_cap=10.0, sd_floor=1e-3):
    """γ for the unshrunk block: c × max(running sd of its draws, sd_floor);
    before two draws exist, min(prior sd, sd_cap) (precond.py:137-153)."""
    running = None if chain is None else chain.unshrunk_sd()
    if running is not None:
        base = _as_f64(running)
    elif prior_sd is not None:
        base = np.minimum(_as_f64(prior_sd), sd_cap)
    else:
        raise ValueError("cold-start gamma_policy needs the prior sds")
    return c * np.maximum(base, sd_floor)


def block_threshold(*args, **kwargs):
    raise NotImplementedError(
        "the block-threshold preconditioner is a dense desk-scale comparison "
        "(precond.py:156-181) and is not part of the B200 path")
