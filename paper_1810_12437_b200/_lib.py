"""ctypes binding of libpcgs.so (the C ABI declared in include/pcgs.h).

The product path has no CPU fallback: importing a device entry point without
the built library raises immediately, and every call checks the status code
and re-raises the reference's exception classes.
"""
from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import numpy as np

# PCGS_LIBRARY points at an alternative build (A/B timing of two builds)
_LIB_PATH = Path(os.environ.get("PCGS_LIBRARY") or Path(__file__).resolve().with_name("libpcgs.so"))
_lock = threading.Lock()
_lib = None

PCGS_OK = 0
PCGS_EINVAL = -1
PCGS_ECUDA = -2
PCGS_ENOMEM = -3
PCGS_EUNSUP = -4
PCGS_EFORMAT = -5
PCGS_EIO = -6

PCGS_CONVERGED = 0
PCGS_MAX_ITER = 1
PCGS_NOT_PD = -1
PCGS_NONFINITE = -2

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
_U64 = ctypes.c_uint64
_D = ctypes.c_double

APPLY_FN = ctypes.CFUNCTYPE(ctypes.c_int, _P, _P, _P)

# name -> (restype, argtypes); must match include/pcgs.h
SIGNATURES = {
    "pcgs_version": (ctypes.c_int, []),
    "pcgs_last_error": (ctypes.c_char_p, []),
    "pcgs_design_create": (ctypes.c_int, [_I64, _I64, _P, _P, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_int, ctypes.POINTER(_P)]),
    "pcgs_design_create_ex": (ctypes.c_int, [_I64, _I64, _P, _P, ctypes.c_int, ctypes.c_int,
                                             ctypes.c_int, ctypes.c_int, ctypes.POINTER(_P)]),
    "pcgs_design_create_affine": (ctypes.c_int, [_I64, _I64, _P, _P, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                                 ctypes.c_int, ctypes.c_int, ctypes.POINTER(_P)]),
    "pcgs_design_set_affine": (ctypes.c_int, [_P, _P, _P, _P]),
    "pcgs_design_destroy": (ctypes.c_int, [_P]),
    "pcgs_synth_design": (ctypes.c_int, [_I64, _I64, _D, _D, _U64, _P, _P, _I64, _P]),
    "pcgs_mtx_load": (ctypes.c_int, [ctypes.c_char_p, _P, _P]),
    "pcgs_mtx_export": (ctypes.c_int, [_P, _P, _P]),
    "pcgs_mtx_free": (ctypes.c_int, [_P]),
    "pcgs_mtx_write": (ctypes.c_int, [ctypes.c_char_p, _I64, _I64, _P, _P, ctypes.c_int, ctypes.c_int]),
    "pcgs_store_selftest": (ctypes.c_int, [_I64, _I64, _P, _P, ctypes.c_int, ctypes.c_int,
                                           ctypes.c_int, _P]),
    "pcgs_design_info": (ctypes.c_int, [_P, _P]),
    "pcgs_matvec": (ctypes.c_int, [_P, _P, _P, _P]),
    "pcgs_matvec_t": (ctypes.c_int, [_P, _P, _P, _P]),
    "pcgs_phi_apply": (ctypes.c_int, [_P, _P, _P, _P, _P, _P]),
    "pcgs_phi_diagonal": (ctypes.c_int, [_P, _P, _P, _P, _P]),
    "pcgs_rhs": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, _P, _U64, _U64, _P, _P]),
    "pcgs_pcg": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, _P, _I32, _D, _P, _P, _P, _P, _P]),
    "pcgs_pcg_op": (ctypes.c_int, [APPLY_FN, _P, _I64, _P, _P, _P, _P, _P, _P, _I32, _D, _P, _P,
                                   _P, _P, _P]),
    "pcgs_pcg_full": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, _P, _I32, _D, _P, _P, _P, _P, _P, _P]),
    "pcgs_pcg_op_full": (ctypes.c_int, [APPLY_FN, _P, _I64, _P, _P, _P, _P, _P, _P, _I32, _D, _P, _P,
                                        _P, _P, _P, _P]),
    "pcgs_copy": (ctypes.c_int, [_P, _P, _I64, ctypes.c_int]),
    "pcgs_debug_profile": (ctypes.c_int, [_P]),
    "pcgs_debug_option": (ctypes.c_int, [ctypes.c_int, ctypes.c_int]),
    "pcgs_debug_cta_times": (ctypes.c_int, [_P]),
    "pcgs_debug_sync_times": (ctypes.c_int, [_P]),
    "pcgs_pg_draw": (ctypes.c_int, [_P, _I64, _U64, _U64, _P, _P]),
    "pcgs_pg_draw_rows": (ctypes.c_int, [_P, _I64, _I64, _U64, _U64, _P, _P]),
    "pcgs_gibbs_init": (ctypes.c_int, [_P, _P, _P]),
    "pcgs_scale_draws": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _I64, _D, _D, _D, _I64, _D, _D, _D,
                                        _U64, _P, _P, _P]),
    "pcgs_rs_create": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_P)]),
    "pcgs_rs_exchange_handle": (ctypes.c_int, [_P, ctypes.c_int, _P]),
    "pcgs_rs_open_peer": (ctypes.c_int, [_P, ctypes.c_int, _P]),
    "pcgs_rs_pcg": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, _P, _I32, _D, _P, _P, _P, _P, _P]),
    "pcgs_rs_destroy": (ctypes.c_int, [_P]),
    "pcgs_rs_set_exchange": (ctypes.c_int, [_P, ctypes.c_int]),
    "pcgs_rs_gibbs_init": (ctypes.c_int, [_P, _P, _P, _P]),
    "pcgs_rs_gibbs_scan": (ctypes.c_int, [_P, _P, _P, _I32, _I32, _I32, _P]),
    "pcgs_batch_create": (ctypes.c_int, [_I64, _I64, _P, _P, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_int, ctypes.c_int, ctypes.POINTER(_P)]),
    "pcgs_batch_destroy": (ctypes.c_int, [_P]),
    "pcgs_batch_info": (ctypes.c_int, [_P, _P]),
    "pcgs_batch_selftest": (ctypes.c_int, [_I64, _I64, _P, _P, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                           ctypes.c_int, _P]),
    "pcgs_batch_debug_profile": (ctypes.c_int, [_P]),
    "pcgs_batch_gibbs_scan": (ctypes.c_int, [_P, _P, _P, _I32, _I32, _P, _P, _P]),
    "pcgs_batch_gibbs_run": (ctypes.c_int, [_P, _P, _I32, _I32, _I32, _I32, _I32, _P, _P, _P, _P]),
    "pcgs_batch_phi_apply": (ctypes.c_int, [_P, _P, _P, _P, _P, _P]),
    "pcgs_batch_pcg": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, _P, _I32, _D, _P, _P, _P, _P, _P]),
    "pcgs_gibbs_scan": (ctypes.c_int, [_P, _P, _I32, _I32, _I32, _P]),
    "pcgs_gibbs_scan_begin": (ctypes.c_int, [_P, _P, _I32, _P]),
    "pcgs_gibbs_scan_end": (ctypes.c_int, [_P, _P, _I32, _I32, _I32, _P]),
}


class PcgsError(RuntimeError):
    """A CUDA-side failure inside libpcgs."""


def library_path() -> Path:
    return _LIB_PATH


def lib():
    """The loaded library; raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not _LIB_PATH.exists():
            raise ImportError(
                f"{_LIB_PATH} is missing: build it with `python -c \"import __graft_entry__ as g; "
                "g.build()\"` (there is no CPU fallback for the device path)")
        L = ctypes.CDLL(str(_LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc == PCGS_OK:
        return
    msg = lib().pcgs_last_error().decode(errors="replace")
    if rc == PCGS_EINVAL:
        raise ValueError(msg)
    if rc == PCGS_EUNSUP:
        raise NotImplementedError(msg)
    if rc == PCGS_EFORMAT:
        from .io import FileFormatError
        raise FileFormatError(msg)
    if rc == PCGS_EIO:
        raise OSError(msg)
    raise PcgsError(f"pcgs error {rc}: {msg}")


# ----------------------------------------------------------------- torch glue
def torch():
    import torch as _t
    return _t


def cuda_device(device=None):
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError("the pcgs device path needs a CUDA GPU (no CPU fallback)")
    if device is None:
        return t.device("cuda", t.cuda.current_device())
    d = t.device(device)
    if d.type != "cuda":
        raise ValueError(f"pcgs runs on CUDA devices only, got {d}")
    if d.index is None:
        d = t.device("cuda", t.cuda.current_device())
    return d


def stream_ptr(device) -> int:
    return torch().cuda.current_stream(device).cuda_stream


def is_tensor(x) -> bool:
    try:
        import torch as _t
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, _t.Tensor)


def to_device(x, device, dtype="float64"):
    """numpy/torch -> contiguous CUDA tensor (float64 by default)."""
    t = torch()
    dt = getattr(t, dtype)
    if is_tensor(x):
        return x.to(device=device, dtype=dt).contiguous()
    arr = np.ascontiguousarray(x, dtype=np.dtype(dtype))
    host = t.from_numpy(arr)
    return host.to(device=device, non_blocking=False)


def ptr(t) -> int:
    return int(t.data_ptr()) if t is not None else 0
