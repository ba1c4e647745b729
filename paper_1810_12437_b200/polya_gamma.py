"""Exact Polya-Gamma PG(1, z) draws on the B200 (drop-in for priorcg.polya_gamma).

The device kernel `k_pg` restates the reference's alternating-series
accept/reject sampler (pkg/src/priorcg/polya_gamma.py:39-147: truncation
0.64, exponential right piece, truncated inverse-Gaussian left piece, series
test in ratio form) with one thread per draw and a Philox4x32-10 substream per
index instead of numpy's shared PCG64 stream.
"""
from __future__ import annotations

import numpy as np

from . import _lib


def pg_mean(z):
    """E[PG(1, z)] = tanh(z/2) / (2z), limit 1/4 (polya_gamma.py:22-31)."""
    arr = np.asarray(z, dtype=np.float64)
    small = np.abs(arr) < 1e-4
    safe = np.where(small, 1.0, arr)
    out = np.where(small, 0.25 - arr ** 2 / 48.0, np.tanh(safe / 2.0) / (2.0 * safe))
    if np.isscalar(z) or arr.ndim == 0:
        return float(out)
    return out


def pg_draw_device(z_t, seed, stream_id, out=None):
    """omega ~ PG(1, z) for a CUDA float64 tensor z (no synchronisation)."""
    t = _lib.torch()
    out = t.empty_like(z_t) if out is None else out
    _lib.check(_lib.lib().pcgs_pg_draw(_lib.ptr(z_t), int(z_t.numel()), int(seed) & (2 ** 64 - 1),
                                       int(stream_id), _lib.ptr(out),
                                       _lib.stream_ptr(z_t.device)))
    return out


def pg_draw_batch(z, rng):
    """Independent PG(1, z_i) draws (polya_gamma.py:39-84), on the GPU.

    `rng` is a numpy Generator (one 63-bit key is drawn from it) or a
    sampler.PhiloxGenerator.
    """
    from .sampler import PhiloxGenerator
    as_tensor = _lib.is_tensor(z)
    if not as_tensor:
        z = np.asarray(z, dtype=np.float64)
        if not np.all(np.isfinite(z)):
            raise ValueError("Polya-Gamma tilt must be finite")
    if isinstance(rng, PhiloxGenerator):
        seed, sid = rng.seed, rng.next_stream()
    else:
        seed, sid = int(rng.integers(0, 2 ** 63)), 0
    dev = _lib.cuda_device(z.device if as_tensor and z.is_cuda else None)
    zt = _lib.to_device(z, dev).reshape(-1)
    out = pg_draw_device(zt, seed, sid)
    if as_tensor:
        return out.reshape(z.shape)
    return out.cpu().numpy().reshape(z.shape)


def pg_draw(z, rng):
    return float(pg_draw_batch(np.array([z], dtype=np.float64), rng)[0])
