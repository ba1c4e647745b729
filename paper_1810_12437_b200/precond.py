"""Preconditioners (drop-in for priorcg.precond, pkg/src/priorcg/precond.py).

Only diagonal kinds reach the device PCG kernel: there M^-1 is the vector
`inv_diagonal` fused into the CG vector update.  The block-threshold kind
(precond.py:156-181) is a dense desk-scale comparison preconditioner and is
out of scope: constructing it raises NotImplementedError.
"""
from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np


class PreconditionerKind(enum.Enum):
    PRIOR = "prior"
    JACOBI = "jacobi"
    AUGMENTED_PRIOR = "augmented"
    BLOCK_THRESHOLD = "block"
    IDENTITY = "identity"


class DegeneratePreconditionerError(ValueError):
    """The requested preconditioner has a non-invertible diagonal (precond.py:30)."""


@dataclass
class Preconditioner:
    """Diagonal M^-1 (precond.py:34-79)."""

    kind: PreconditionerKind
    inv_diagonal: np.ndarray

    def __post_init__(self):
        self.inv_diagonal = np.asarray(self.inv_diagonal, dtype=np.float64)
        if np.any(~np.isfinite(self.inv_diagonal)) or np.any(self.inv_diagonal <= 0):
            raise DegeneratePreconditionerError(
                "inverse-diagonal entries must be finite and strictly positive")

    @property
    def dim(self):
        return len(self.inv_diagonal)

    def apply_inverse(self, v):
        return self.inv_diagonal * v

    def to_dense_inverse(self):
        return np.diag(self.inv_diagonal)


def identity_preconditioner(p):
    return Preconditioner(PreconditionerKind.IDENTITY, np.ones(p))


def prior_preconditioner(tau, lam):
    """M = tau^-2 Lambda^-2 (precond.py:87-102)."""
    lam = np.asarray(lam, dtype=np.float64)
    if not (np.isfinite(tau) and tau > 0):
        raise ValueError("tau must be positive and finite")
    if np.any(~np.isfinite(lam)) or np.any(lam <= 0):
        raise ValueError("lambda entries must be positive and finite")
    return Preconditioner(PreconditionerKind.PRIOR, (tau * lam) ** 2)


def jacobi_preconditioner(X, omega, tau, lam, prior_precision=None):
    """M = diag(Phi) (precond.py:105-117); diag(X'ΩX) is one CSC pass on device."""
    if prior_precision is None:
        lam = np.asarray(lam, dtype=np.float64)
        prior_precision = (tau * lam) ** -2.0
    diag = np.asarray(X.gram_diagonal(omega)) + prior_precision
    if np.any(diag <= 0) or np.any(~np.isfinite(diag)):
        raise DegeneratePreconditionerError("Phi has a nonpositive diagonal entry")
    return Preconditioner(PreconditionerKind.JACOBI, 1.0 / diag)


def augmented_prior(tau, lam, gamma):
    """[gamma^2, (tau lam)^2] over the unshrunk + shrunk blocks (precond.py:120-134)."""
    gamma = np.asarray(gamma, dtype=np.float64)
    if gamma.size == 0:
        return prior_preconditioner(tau, lam)
    if np.any(~np.isfinite(gamma)) or np.any(gamma <= 0):
        raise ValueError("gamma entries must be positive and finite")
    lam = np.asarray(lam, dtype=np.float64)
    return Preconditioner(PreconditionerKind.AUGMENTED_PRIOR,
                          np.concatenate([gamma ** 2, (tau * lam) ** 2]))


def gamma_policy(chain, c=1.0, prior_sd=None, sd_cap=10.0, sd_floor=1e-3):
    """c * running sd of the unshrunk draws, cold start min(prior sd, cap) (precond.py:137-153)."""
    sds = chain.unshrunk_sd() if chain is not None else None
    if sds is None:
        if prior_sd is None:
            raise ValueError("cold-start gamma_policy needs the prior sds")
        sds = np.minimum(np.asarray(prior_sd, dtype=np.float64), sd_cap)
    return c * np.maximum(np.asarray(sds, dtype=np.float64), sd_floor)


def block_threshold(*args, **kwargs):
    raise NotImplementedError(
        "the block-threshold preconditioner is a dense desk-scale comparison "
        "(precond.py:156-181) and is not part of the B200 path")
