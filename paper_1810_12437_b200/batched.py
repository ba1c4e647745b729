"""Batched independent chains on one GPU (BASELINE config 4).

R chains with their own omega, prior diagonal and right-hand side share every
walk over the pattern through the sliced store (csrc/sliced.h): Phi_c v_c
for all c in one SpMM-like pass (`pcgs_batch_phi_apply`) and R PCG solves in
one persistent kernel (`pcgs_batch_pcg`), each chain following the reference
loop (cg.py:105-192) and masked once it terminates.  Host arrays are
chain-major (R, m); the device layout is chain-minor (m, R).
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .cg import CGConfig, CGReport, _n_betas, _raise_status

SUPPORTED = (1, 2, 4, 8)


class BatchStore:
    """Owner of one libpcgs sliced-store handle (R chains, one CUDA device)."""

    KEYS = ["n", "p", "p_total", "nnz", "csr_slabs", "csc_slabs", "csr_vectors", "csc_vectors",
            "csr_pieces", "csc_pieces", "nchains", "grid", "device", "index_bytes", "slab_max",
            "bank_conflict_ppm"]

    def __init__(self, n, p, row_ptr, col_idx, intercept, nchains, device=None, slab_max=0, grid=0):
        if nchains not in SUPPORTED:
            raise ValueError(f"batch size must be one of {SUPPORTED}")
        L = _lib.lib()
        self.device = _lib.cuda_device(device)
        rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
        ci = np.ascontiguousarray(col_idx, dtype=np.int32)
        h = ctypes.c_void_p()
        _lib.check(L.pcgs_batch_create(int(n), int(p), rp.ctypes.data, ci.ctypes.data, int(bool(intercept)),
                                       int(nchains), int(slab_max), int(self.device.index), int(grid),
                                       ctypes.byref(h)))
        self._h = h
        info = np.zeros(16, dtype=np.int64)
        _lib.check(L.pcgs_batch_info(h, info.ctypes.data))
        self.info = info
        self.R = int(nchains)

    @property
    def handle(self):
        return self._h

    def describe(self) -> dict:
        return {k: int(v) for k, v in zip(self.KEYS, self.info)}

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _lib.lib().pcgs_batch_destroy(h)
            except Exception:  # pragma: no cover - interpreter shutdown
                pass
            self._h = None


def _to_dev_cm(a, dev):
    """(R, m) host/torch array -> contiguous chain-minor (m, R) CUDA tensor."""
    t = _lib.torch()
    x = a if _lib.is_tensor(a) else t.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
    return x.to(device=dev, dtype=t.float64).t().contiguous()


class BatchedPrecisionOperator:
    """Phi_c = X' diag(omega_c) X + diag(d_c) for R chains on one design."""

    def __init__(self, X, omegas, prior_diags, device=None):
        R = int(np.shape(omegas)[0])
        if R not in SUPPORTED:
            raise ValueError(f"batch size must be one of {SUPPORTED}")
        if tuple(np.shape(omegas)) != (R, X.n_rows) or tuple(np.shape(prior_diags)) != (R, X.n_cols):
            raise ValueError("omegas must be (R, n) and prior_diags (R, p)")
        om = np.asarray(omegas.cpu() if _lib.is_tensor(omegas) else omegas, dtype=np.float64)
        dg = np.asarray(prior_diags.cpu() if _lib.is_tensor(prior_diags) else prior_diags, dtype=np.float64)
        if not np.all(np.isfinite(om)) or np.any(om < 0):
            raise ValueError("omega must be finite and nonnegative")
        if not np.all(np.isfinite(dg)) or np.any(dg < 0):
            raise ValueError("prior precision must be finite and nonnegative")
        self.X, self.R = X, R
        self.store = X.batch_store(R, device)
        self.dev = self.store.device
        self.omega = _to_dev_cm(om, self.dev)
        self.diag = _to_dev_cm(dg, self.dev)
        self.prior_precision_diag = dg
        self.apply_count = 0

    @property
    def dim(self):
        return self.X.n_cols

    def apply(self, V):
        """(R, p) -> (R, p): Phi_c v_c for every chain."""
        t = _lib.torch()
        as_tensor = _lib.is_tensor(V)
        vd = _to_dev_cm(V, self.dev)
        out = t.empty_like(vd)
        self.apply_count += 1
        _lib.check(_lib.lib().pcgs_batch_phi_apply(self.store.handle, _lib.ptr(self.omega),
                                                   _lib.ptr(self.diag), _lib.ptr(vd), _lib.ptr(out),
                                                   _lib.stream_ptr(self.dev)))
        res = out.t().contiguous()
        return res if as_tensor else res.cpu().numpy()


def batched_pcg_device(op, B_cm, minv_cm, scale_cm, X0_cm=None, max_iter=None, rtol=1e-6):
    """Device solve on chain-minor tensors; returns (X, trace, alphas, betas, result)."""
    t = _lib.torch()
    R, p, dev = op.R, op.dim, op.dev
    max_iter = 2 * p if max_iter is None else int(max_iter)
    x = t.zeros((p, R), dtype=t.float64, device=dev) if X0_cm is None else X0_cm.clone()
    trace = t.empty((R, max_iter + 1), dtype=t.float64, device=dev)
    alphas = t.empty((R, max_iter), dtype=t.float64, device=dev)
    betas = t.empty((R, max_iter), dtype=t.float64, device=dev)
    result = t.zeros((R, 4), dtype=t.int32, device=dev)
    _lib.check(_lib.lib().pcgs_batch_pcg(op.store.handle, _lib.ptr(op.omega), _lib.ptr(op.diag),
                                         _lib.ptr(minv_cm), _lib.ptr(scale_cm), _lib.ptr(B_cm),
                                         _lib.ptr(x), max_iter, float(rtol), _lib.ptr(trace),
                                         _lib.ptr(alphas), _lib.ptr(betas), _lib.ptr(result),
                                         _lib.stream_ptr(dev)))
    return x, trace, alphas, betas, result


def batched_pcg_solve(op, B, minv, scale, X0=None, config=None):
    """R independent PCG solves (cg.py:105-192) sharing the index stream.

    B, minv, scale, X0: (R, p).  Returns a list of R CGReport; a chain that
    hits NotPositiveDefinite / NumericBreakdown raises for that chain.
    """
    cfg = config if config is not None else CGConfig()
    dev = op.dev
    x, trace, alphas, betas, result = batched_pcg_device(
        op, _to_dev_cm(B, dev), _to_dev_cm(minv, dev), _to_dev_cm(scale, dev),
        None if X0 is None else _to_dev_cm(X0, dev), cfg.max_iter, cfg.rtol)
    res = result.cpu().numpy()
    X = x.t().contiguous().cpu().numpy()
    tr, al, be = trace.cpu().numpy(), alphas.cpu().numpy(), betas.cpu().numpy()
    reports = []
    for c in range(op.R):
        it, status, fail_iter, applies = (int(v) for v in res[c])
        _raise_status(status, fail_iter)
        reports.append(CGReport(
            iterations=it, termination="converged" if status == _lib.PCGS_CONVERGED else "max_iter",
            rms_precond_residual_trace=tr[c, :it + 1].copy(), solution=X[c], matvec_count=it + 1,
            alphas=al[c, :it].copy(), betas=be[c, :_n_betas(it, status)].copy()))
    return reports
