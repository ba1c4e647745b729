"""Prior-preconditioned CG on the B200 (drop-in for priorcg.cg).

`pcg_solve` keeps the reference's signature, stopping rule, counters and
exceptions (pkg/src/priorcg/cg.py:105-192):

* `phi` a device `PrecisionOperator` with a diagonal preconditioner -> the
  whole loop runs in one persistent cooperative kernel (`pcgs_pcg`): both
  sparse passes, the dot products, the axpys, M^-1 and the RMS test, with the
  convergence decision taken on device and no host synchronisation inside.
* any other operator (an object with `.apply`, or a callable, cg.py:110) ->
  the same loop with the vector algebra on device (`pcgs_pcg_op`) and the
  operator called back on the host once per application.

Rounding note: the device computes d'Phi d as z'Ωz + d'Dd with z = X d
(algebraically equal to the reference's d'(Phi d)); every reduction has a
fixed order, so repeated solves are bitwise identical.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .precond import Preconditioner, PreconditionerKind
from .sparse import NotPositiveDefiniteError


class NumericBreakdownError(RuntimeError):
    """Non-finite quantity inside the CG recurrence (cg.py:29-34)."""

    def __init__(self, iteration, message=None):
        super().__init__(message or f"non-finite value at CG iteration {iteration}")
        self.iteration = iteration


@dataclass
class CGConfig:
    """Solver knobs (cg.py:37-51).  ``max_iter`` defaults to 2p at solve time."""

    max_iter: int | None = None
    rtol: float = 1e-6
    trace_level: str = "norms"

    def __post_init__(self):
        if self.max_iter is not None and self.max_iter < 1:
            raise ValueError("max_iter must be at least 1")
        if not self.rtol > 0:
            raise ValueError("rtol must be positive")
        if self.trace_level not in ("none", "norms", "full"):
            raise ValueError("trace_level must be one of none|norms|full")


@dataclass
class CGReport:
    """Outcome of one PCG solve (cg.py:54-86)."""

    iterations: int
    termination: str
    rms_precond_residual_trace: np.ndarray
    solution: np.ndarray
    matvec_count: int
    alphas: np.ndarray = field(default_factory=lambda: np.zeros(0))
    betas: np.ndarray = field(default_factory=lambda: np.zeros(0))
    iterates: list | None = None
    # device copy of the iterates ((iterations+1) x p CUDA tensor) when the
    # solve ran on the GPU at trace_level "full"; diagnostics.error_trace
    # evaluates on it without a round trip
    iterates_device: object = field(default=None, repr=False, compare=False)

    def lanczos_tridiagonal(self):
        """(diagonal, offdiagonal) of the Lanczos matrix from the CG coefficients."""
        k = len(self.alphas)
        diag = np.empty(k)
        off = np.empty(max(k - 1, 0))
        for i in range(k):
            diag[i] = 1.0 / self.alphas[i]
            if i > 0:
                diag[i] += self.betas[i - 1] / self.alphas[i - 1]
            if i < k - 1:
                off[i] = math.sqrt(self.betas[i]) / self.alphas[i]
        return diag, off


def _metric_scale(phi, M, residual_scale, p):
    """Termination scale s, same precedence as cg.py:89-102."""
    if residual_scale is not None:
        scale = np.asarray(residual_scale, dtype=np.float64)
        if scale.shape != (p,) or np.any(scale <= 0) or np.any(~np.isfinite(scale)):
            raise ValueError("residual_scale must be positive, finite, length p")
        return scale
    prior_diag = getattr(phi, "prior_precision_diag", None)
    if prior_diag is not None:
        prior_diag = np.asarray(prior_diag, dtype=np.float64)
        if np.all(prior_diag > 0):
            return prior_diag ** -0.5
    if M.kind in (PreconditionerKind.PRIOR, PreconditionerKind.AUGMENTED_PRIOR):
        return np.sqrt(M.inv_diagonal)
    raise ValueError(
        "cannot derive the residual metric (flat-prior coordinates present); "
        "pass residual_scale explicitly")


def _n_betas(iterations, status):
    if status == _lib.PCGS_MAX_ITER:
        return iterations
    return max(iterations - 1, 0)


def _raise_status(status, fail_iter, dAd_hint=None):
    if status == _lib.PCGS_NOT_PD:
        raise NotPositiveDefiniteError(
            f"direction with d'Phi d <= 0 at CG iteration {fail_iter}")
    if status == _lib.PCGS_NONFINITE:
        raise NumericBreakdownError(fail_iter)


def _is_device_operator(phi):
    return getattr(phi, "_pcgs_device_operator", False)


def pcg_solve_device(phi, b, minv, scale, x0=None, max_iter=None, rtol=1e-6, full=False):
    """Fused device solve on tensors.  Returns (x, trace, alphas, betas, result) tensors.

    `phi` must be a device PrecisionOperator; b, minv, scale, x0 are CUDA
    float64 tensors of length p_total (reference layout).  Nothing is
    synchronised; result = [iterations, status, fail_iter, applies] (int32).
    """
    t = _lib.torch()
    st = phi.store
    dev = st.device
    p = st.p_total
    max_iter = 2 * p if max_iter is None else int(max_iter)
    x = (t.zeros(p, dtype=t.float64, device=dev) if x0 is None
         else x0.to(device=dev, dtype=t.float64).clone())
    trace = t.empty(max_iter + 1, dtype=t.float64, device=dev)
    alphas = t.empty(max_iter, dtype=t.float64, device=dev)
    betas = t.empty(max_iter, dtype=t.float64, device=dev)
    result = t.zeros(4, dtype=t.int32, device=dev)
    iterates = t.empty((max_iter + 1, p), dtype=t.float64, device=dev) if full else None
    omega, diag = phi.device_omega(), phi.device_diag()
    _lib.check(_lib.lib().pcgs_pcg_full(st.handle, _lib.ptr(omega), _lib.ptr(diag), _lib.ptr(minv),
                                        _lib.ptr(scale), _lib.ptr(b), _lib.ptr(x), max_iter, float(rtol),
                                        _lib.ptr(trace), _lib.ptr(alphas), _lib.ptr(betas),
                                        _lib.ptr(iterates), _lib.ptr(result), _lib.stream_ptr(dev)))
    if full:
        return x, trace, alphas, betas, result, iterates
    return x, trace, alphas, betas, result


def _report_from_device(x, trace, alphas, betas, result, iterates=None, as_tensor=False):
    res = result.cpu().numpy()
    iterations, status, fail_iter, applies = (int(v) for v in res)
    _raise_status(status, fail_iter)
    nb = _n_betas(iterations, status)
    its = its_dev = None
    if iterates is not None:
        its_dev = iterates[: iterations + 1]
        h = its_dev.cpu().numpy()
        its = [h[k].copy() for k in range(iterations + 1)]
    return CGReport(
        iterations=iterations,
        termination="converged" if status == _lib.PCGS_CONVERGED else "max_iter",
        rms_precond_residual_trace=trace[: iterations + 1].cpu().numpy(),
        solution=x if as_tensor else x.cpu().numpy(),
        matvec_count=applies,
        alphas=alphas[:iterations].cpu().numpy(),
        betas=betas[:nb].cpu().numpy(),
        iterates=its,
        iterates_device=its_dev,
    )


def pcg_solve(phi, b, M, x0=None, config=None, residual_scale=None):
    """Solve Phi x = b by preconditioned CG on the GPU (cg.py:105-192).

    Same arguments, return value and exceptions as the reference.  `b` / `x0`
    may be numpy arrays (the report then holds numpy arrays) or CUDA tensors.
    """
    cfg = config if config is not None else CGConfig()
    if not isinstance(M, Preconditioner) and getattr(M, "kind", None) is PreconditionerKind.BLOCK_THRESHOLD:
        raise NotImplementedError("block-threshold preconditioning is not on the device path")
    full = cfg.trace_level == "full"
    as_tensor = _lib.is_tensor(b)
    p = int(b.shape[0])
    max_iter = cfg.max_iter if cfg.max_iter is not None else 2 * p
    scale = _metric_scale(phi, M, residual_scale, p)
    minv = np.asarray(M.inv_diagonal, dtype=np.float64)
    if minv.shape != (p,):
        raise ValueError("preconditioner dimension must match b")
    if _is_device_operator(phi):
        dev = phi.store.device
        bd = _lib.to_device(b, dev)
        x0d = None if x0 is None else _lib.to_device(x0, dev)
        out = pcg_solve_device(phi, bd, _lib.to_device(minv, dev), _lib.to_device(scale, dev),
                               x0=x0d, max_iter=max_iter, rtol=cfg.rtol, full=full)
        phi.apply_count += int(out[4][3].item())
        return _report_from_device(*out, as_tensor=as_tensor)
    return _pcg_solve_operator(phi, b, minv, scale, x0, max_iter, cfg.rtol, as_tensor, full)


def _pcg_solve_operator(phi, b, minv, scale, x0, max_iter, rtol, as_tensor, full=False):
    """Generic operator: device vector algebra + host callback per application."""
    t = _lib.torch()
    L = _lib.lib()
    dev = _lib.cuda_device(b.device if as_tensor and b.is_cuda else
                           (phi.store.device if hasattr(phi, "store") else None))
    apply_phi = phi.apply if hasattr(phi, "apply") else phi
    p = int(b.shape[0])
    bd = _lib.to_device(b, dev)
    x = t.zeros(p, dtype=t.float64, device=dev) if x0 is None else _lib.to_device(x0, dev).clone()
    md, sd = _lib.to_device(minv, dev), _lib.to_device(scale, dev)
    host_v = np.empty(p)
    errors = []

    def cb(ctx, vptr, outptr):
        try:
            _lib.check(L.pcgs_copy(host_v.ctypes.data, vptr, 8 * p, 1))
            out = np.ascontiguousarray(apply_phi(host_v.copy()), dtype=np.float64)
            if out.shape != (p,):
                raise ValueError("operator returned a vector of the wrong length")
            _lib.check(L.pcgs_copy(outptr, out.ctypes.data, 8 * p, 0))
            return 0
        except BaseException as exc:  # re-raised after the C loop returns
            errors.append(exc)
            return 1

    dbuf = adbuf = None
    if hasattr(phi, "apply_into"):
        # device-side operator: apply on the engine's own buffers, no host copies
        dbuf = t.empty(p, dtype=t.float64, device=dev)
        adbuf = t.empty(p, dtype=t.float64, device=dev)
        xptr = _lib.ptr(x)

        def cb(ctx, vptr, outptr):  # noqa: F811
            try:
                phi.apply_count = getattr(phi, "apply_count", 0) + 1
                phi.apply_into(x if vptr == xptr else dbuf, adbuf)
                return 0
            except BaseException as exc:
                errors.append(exc)
                return 1

    fn = _lib.APPLY_FN(cb)
    trace = np.zeros(max_iter + 1)
    alphas = np.zeros(max_iter)
    betas = np.zeros(max_iter)
    result = np.zeros(4, dtype=np.int32)
    iterates = t.empty((max_iter + 1, p), dtype=t.float64, device=dev) if full else None
    t.cuda.synchronize(dev)
    rc = L.pcgs_pcg_op_full(fn, None, p, _lib.ptr(md), _lib.ptr(sd), _lib.ptr(bd), _lib.ptr(x),
                            _lib.ptr(dbuf), _lib.ptr(adbuf),
                            max_iter, float(rtol), trace.ctypes.data, alphas.ctypes.data, betas.ctypes.data,
                            _lib.ptr(iterates), result.ctypes.data, _lib.stream_ptr(dev))
    if errors:
        raise errors[0]
    _lib.check(rc)
    iterations, status, fail_iter, applies = (int(v) for v in result)
    _raise_status(status, fail_iter)
    nb = _n_betas(iterations, status)
    return CGReport(
        iterations=iterations,
        termination="converged" if status == _lib.PCGS_CONVERGED else "max_iter",
        rms_precond_residual_trace=trace[: iterations + 1].copy(),
        solution=x if as_tensor else x.cpu().numpy(),
        matvec_count=applies,
        alphas=alphas[:iterations].copy(),
        betas=betas[:nb].copy(),
        iterates=(None if iterates is None else
                  [r.copy() for r in iterates[: iterations + 1].cpu().numpy()]),
        iterates_device=None if iterates is None else iterates[: iterations + 1],
    )


def initial_vector(chain, tau, lam, n_unshrunk=0):
    """Warm start: current scales times the running scaled-draw mean (cg.py:195-211)."""
    lam = np.asarray(lam, dtype=np.float64)
    p_total = n_unshrunk + len(lam)
    mean = chain.scaled_beta_mean() if chain is not None else None
    if mean is None:
        return np.zeros(p_total)
    mean = np.asarray(mean)
    if mean.shape != (p_total,):
        raise ValueError("chain coefficient count does not match tau/lambda")
    return np.concatenate([np.ones(n_unshrunk), tau * lam]) * mean
