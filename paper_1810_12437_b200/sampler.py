"""Gaussian conditional sampler on the B200 (drop-in for priorcg.sampler).

Phi = X' diag(omega) X + diag(prior_precision_diag) is never formed: `apply`
is two pattern-only sparse passes (pcgs_phi_apply), `generate_rhs` one fused
X' pass over kappa + sqrt(omega) eta (pcgs_rhs), and `cg_sample` feeds the
right-hand side to the device PCG kernel.  Semantics follow
pkg/src/priorcg/sampler.py:24-120.

Noise: with a numpy Generator the RHS draws eta (n) then delta (p) from it on
the host, in the reference's stream order (sampler.py:103-104), so identically
seeded samplers consume identical noise.  With a `PhiloxGenerator` the noise is
drawn on device (Philox4x32-10, keyed by seed and a per-call counter).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .cg import CGConfig, pcg_solve
from .precond import Preconditioner
from .sparse import SparseDesignMatrix


class PhiloxGenerator:
    """Counter-based device RNG handle: (seed, stream counter).

    Each device draw consumes one stream id, so successive calls give
    independent noise and a fixed seed reproduces a run bit for bit.
    """

    def __init__(self, seed=0):
        self.seed = int(seed) & ((1 << 64) - 1)
        self.counter = 0

    @classmethod
    def from_numpy(cls, rng):
        return cls(int(rng.integers(0, 2 ** 63)))

    def next_stream(self):
        self.counter += 1
        return self.counter


class PrecisionOperator:
    """Matrix-free Phi on the GPU (sampler.py:24-67).

    Raw binary designs use the fused kernels (`pcgs_phi_apply`, and the
    persistent PCG kernel in `pcg_solve`); standardised designs compose the raw
    passes with the rank-one correction on device (`apply_into`)."""

    def __init__(self, X: SparseDesignMatrix, omega, prior_precision_diag):
        as_tensor = _lib.is_tensor(omega)
        om_h = omega.detach().cpu().numpy() if as_tensor else omega
        diag_h = (prior_precision_diag.detach().cpu().numpy() if _lib.is_tensor(prior_precision_diag)
                  else prior_precision_diag)
        om_h = np.ascontiguousarray(om_h, dtype=np.float64)
        diag_h = np.ascontiguousarray(diag_h, dtype=np.float64)
        if om_h.shape != (X.n_rows,):
            raise ValueError("omega must have one weight per observation")
        if diag_h.shape != (X.n_cols,):
            raise ValueError("prior precision must have one entry per column")
        if not np.all(np.isfinite(om_h)) or np.any(om_h < 0.0):
            raise ValueError("omega must be finite and nonnegative")
        if not np.all(np.isfinite(diag_h)) or np.any(diag_h < 0.0):
            raise ValueError("prior precision must be finite and nonnegative")
        self.X = X
        self.omega = om_h
        self.prior_precision_diag = diag_h
        self.apply_count = 0
        self._dev = {}
        if as_tensor and omega.is_cuda:
            self._dev["omega"] = omega.to(dtype=_lib.torch().float64).contiguous()

    @classmethod
    def from_device(cls, X, omega_t, diag_t, omega_h=None, diag_h=None):
        """Wrap device tensors without host validation copies (hot path)."""
        self = cls.__new__(cls)
        self.X = X
        self.omega = omega_h
        self.prior_precision_diag = diag_h
        self.apply_count = 0
        self._dev = {"omega": omega_t, "diag": diag_t}
        return self

    @property
    def dim(self) -> int:
        return self.X.n_cols

    @property
    def _pcgs_device_operator(self):
        return True

    def apply_into(self, v, out):
        """out = Phi v on CUDA tensors (any design: affine terms in-kernel)."""
        return self.store.phi_apply(self.device_omega(), self.device_diag(), v, out)

    @property
    def store(self):
        dev = self._dev.get("omega")
        return self.X.device_store(dev.device if dev is not None else None)

    def device_omega(self):
        t = self._dev.get("omega")
        if t is None:
            t = _lib.to_device(self.omega, self.store.device)
            self._dev["omega"] = t
        return t

    def device_diag(self):
        t = self._dev.get("diag")
        if t is None:
            t = _lib.to_device(self.prior_precision_diag, self.store.device)
            self._dev["diag"] = t
        return t

    def apply(self, v):
        """Phi v = X'(omega ⊙ X v) + d ⊙ v (sampler.py:53-58)."""
        as_tensor = _lib.is_tensor(v)
        if tuple(v.shape) != (self.dim,):
            raise ValueError("vector length must equal the operator dimension")
        self.apply_count += 1
        st = self.store
        t = _lib.torch()
        vd = _lib.to_device(v, st.device)
        out = t.empty_like(vd)
        self.apply_into(vd, out)
        return out if as_tensor else out.cpu().numpy()

    def dense_matrix(self, dense_cap=None):
        raise NotImplementedError("dense Phi is the CPU oracle's job (sampler.py:60-67); "
                                  "the B200 path is matrix-free")


@dataclass
class GaussianTarget:
    """N(Phi^-1 linear_term, Phi^-1) by its natural parameters (sampler.py:70-91)."""

    precision: PrecisionOperator
    linear_term: object
    kappa: object = None  # n-vector with X' kappa == linear_term, when known (fused RHS)

    def __post_init__(self):
        lt = self.linear_term
        shape = tuple(lt.shape)
        if shape != (self.precision.dim,):
            raise ValueError("linear term length must match the precision")
        if _lib.is_tensor(lt):
            if not bool(_lib.torch().isfinite(lt).all()):
                raise ValueError("linear term must be finite")
        else:
            self.linear_term = np.ascontiguousarray(lt, dtype=np.float64)
            if not np.all(np.isfinite(self.linear_term)):
                raise ValueError("linear term must be finite")

    @classmethod
    def from_pseudo_outcome(cls, precision: PrecisionOperator, y_prime):
        """Linear term X' Omega y' (sampler.py:86-91), on device."""
        if _lib.is_tensor(y_prime):
            w = precision.device_omega() * y_prime.to(precision.device_omega().device)
        else:
            w = np.asarray(precision.omega) * np.asarray(y_prime, dtype=np.float64)
        lt = precision.X.matvec_t(w)
        return cls(precision, lt, kappa=w)


def generate_rhs(target: GaussianTarget, rng) -> np.ndarray:
    """b = linear_term + X' Omega^{1/2} eta + D^{1/2} delta (sampler.py:94-107)."""
    phi = target.precision
    st = phi.store
    dev = st.device
    t = _lib.torch()
    n, p = phi.X.n_rows, phi.dim
    if isinstance(rng, PhiloxGenerator):
        eta_d = delta_d = None
        seed, sid = rng.seed, rng.next_stream()
    else:
        eta = rng.standard_normal(n)
        delta = rng.standard_normal(p)
        eta_d, delta_d = _lib.to_device(eta, dev), _lib.to_device(delta, dev)
        seed, sid = 0, 0
    lin = _lib.to_device(target.linear_term, dev)
    b = t.empty(p, dtype=t.float64, device=dev)
    _lib.check(_lib.lib().pcgs_rhs(st.handle, 0, _lib.ptr(phi.device_omega()),
                                   _lib.ptr(phi.device_diag()), _lib.ptr(lin), _lib.ptr(eta_d),
                                   _lib.ptr(delta_d), seed, sid, _lib.ptr(b),
                                   _lib.stream_ptr(dev)))
    return b if _lib.is_tensor(target.linear_term) else b.cpu().numpy()


def cg_sample(target: GaussianTarget, M: Preconditioner, rng, x0=None,
              config: CGConfig | None = None, residual_scale=None):
    """Draw beta by solving Phi beta = b on the GPU (sampler.py:110-120)."""
    b = generate_rhs(target, rng)
    report = pcg_solve(target.precision, b, M, x0=x0, config=config,
                       residual_scale=residual_scale)
    return report.solution, report


def direct_sample(target: GaussianTarget, rng, dense_cap=None) -> np.ndarray:
    """The reference's dense Cholesky draw (sampler.py:123-135) is not rebuilt
    on the device (a desk-scale oracle only); use
    `cg_sample`, which draws from the same distribution matrix-free."""
    raise NotImplementedError(
        "direct_sample (dense Cholesky) is not on the device path; use cg_sample, which draws "
        "beta ~ N(Phi^-1 b_lin, Phi^-1) matrix-free on the GPU")
