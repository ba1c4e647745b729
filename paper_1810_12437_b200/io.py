"""Design ingestion, state snapshots and the delimited artifact formats.

Drop-in for priorcg.matrixio (pkg/src/priorcg/matrixio.py) and
priorcg.stateio (pkg/src/priorcg/stateio.py), SURVEY §8(f) row 1.

The reference reads a Matrix Market design with scipy.io.mmread and
densifies it (matrixio.py:48-58), then builds the CSR from the dense array;
at paper scale (config 5: 1e6 x 1e5) that is impossible.  Here
`read_design_pattern` streams the file (plain or gzip) through the native
parser in libpcgs (`pcgs_mtx_load`, one pass, no dense intermediate) straight
into the pattern-only CSR that `SparseDesignMatrix.from_pattern` and the
device store take.  The file contract is unchanged: files written by the
reference's `write_design` read back here and vice versa.

State files (BRGS v1) and the CSV formats are byte-compatible with the
reference (same header strings, `%.17g` floats); `tests/golden/` pins them
with files the reference itself wrote.
"""
from __future__ import annotations

import csv
import ctypes
import io as _io
import os
import struct

import numpy as np

from . import _lib
from .sparse import SparseDesignMatrix

FLOAT_FMT = "%.17g"

CHAIN_FIXED_COLUMNS = ("tau", "logdensity")
TRACE_COLUMNS = ("iter", "rms_precond_residual", "phi_norm_error",
                 "l2_error", "rel_coord_error")
SPECTRUM_COLUMNS = ("index", "eigenvalue", "log10_eigenvalue")
ZSCORE_COLUMNS = ("index", "z_score", "ess_a", "ess_b", "excluded")

FIELDS = ("pattern", "real", "integer")


class FileFormatError(ValueError):
    """A file exists but does not parse as the expected format (matrixio.py:31-32)."""


# ----------------------------------------------------------------- Matrix Market
def read_pattern(path):
    """Parse a 0/1 Matrix Market file into CSR without densifying.

    Returns (n, p, row_ptr int64[n+1], col_idx int32[nnz], info dict).
    Explicit zero entries are dropped; any other non-binary value raises
    NotImplementedError (the device store is pattern-only)."""
    L = _lib.lib()
    h = ctypes.c_void_p()
    info = np.zeros(8, dtype=np.int64)
    _lib.check(L.pcgs_mtx_load(os.fsencode(str(path)), ctypes.byref(h), info.ctypes.data))
    try:
        n, p, nnz = int(info[0]), int(info[1]), int(info[2])
        row_ptr = np.empty(n + 1, dtype=np.int64)
        col_idx = np.empty(nnz, dtype=np.int32)
        _lib.check(L.pcgs_mtx_export(h, row_ptr.ctypes.data, col_idx.ctypes.data if nnz else None))
    finally:
        L.pcgs_mtx_free(h)
    meta = dict(entries=int(info[3]), field=FIELDS[int(info[4])],
                symmetry=("general", "symmetric")[int(info[5])],
                format=("coordinate", "array")[int(info[6])], zeros_dropped=int(info[7]))
    return n, p, row_ptr, col_idx, meta


def read_design_pattern(path, intercept="detect") -> SparseDesignMatrix:
    """Stream a binary design file into a `SparseDesignMatrix` (pattern store).

    intercept: "detect" strips a leading all-ones column into the store's
    dense intercept (what `SparseDesignMatrix.pattern` does for in-memory
    designs); True prepends an intercept column (hstack_dense_columns,
    sparse.py:314-341); False keeps the file's columns as they are."""
    n, p, rp, ci, _ = read_pattern(path)
    if intercept == "detect":
        counts = np.diff(rp)
        has = p >= 1 and n > 0 and bool(np.all(counts >= 1)) and bool(np.all(ci[rp[:-1]] == 0))
        if has:
            keep = np.ones(len(ci), dtype=bool)
            keep[rp[:-1]] = False
            ci = (ci[keep] - 1).astype(np.int32)
            rp = rp - np.arange(n + 1, dtype=np.int64)
            p -= 1
        return SparseDesignMatrix.from_pattern(n, p, rp, ci, intercept=has, check=False)
    return SparseDesignMatrix.from_pattern(n, p, rp, ci, intercept=bool(intercept), check=False)


def _full_pattern(X: SparseDesignMatrix):
    """CSR of every column (intercept included as column 0) from the store's pattern."""
    rp, ci, icpt = X.pattern()
    if not icpt:
        return np.asarray(rp, dtype=np.int64), np.asarray(ci, dtype=np.int32)
    n = X.n_rows
    full_rp = np.asarray(rp, dtype=np.int64) + np.arange(n + 1, dtype=np.int64)
    full_ci = np.insert(np.asarray(ci, dtype=np.int32) + 1, np.asarray(rp[:-1], dtype=np.int64), 0)
    return full_rp, full_ci.astype(np.int32)


def write_design(path, X, field="real") -> None:
    """Write a design to Matrix Market (matrixio.py:35-45).

    `SparseDesignMatrix` and scipy sparse inputs go out in coordinate format
    through the native writer (gzip when the name ends in .gz); `field`
    "real" writes value 1 per entry like scipy.io.mmwrite, "pattern" omits
    it.  Dense arrays go out in array format."""
    path = str(path)
    gz = path.lower().endswith(".gz")
    if isinstance(X, SparseDesignMatrix):
        rp, ci = _full_pattern(X)
        n, p = X.n_rows, X.n_cols
    elif hasattr(X, "tocsr"):
        A = X.tocsr()
        A.sort_indices()
        if A.nnz and not np.all(A.data == 1.0):
            raise NotImplementedError("the pattern store writes 0/1 designs only")
        n, p = A.shape
        rp, ci = A.indptr.astype(np.int64), A.indices.astype(np.int32)
    else:
        _write_array(path, np.asarray(X, dtype=np.float64), gz)
        return
    _lib.check(_lib.lib().pcgs_mtx_write(os.fsencode(path), int(n), int(p), rp.ctypes.data,
                                         ci.ctypes.data if len(ci) else None,
                                         1 if field == "real" else 0, 1 if gz else 0))


def _write_array(path, A, gz):
    A = np.atleast_2d(A)
    buf = _io.StringIO()
    buf.write("%%MatrixMarket matrix array real general\n")
    buf.write(f"{A.shape[0]} {A.shape[1]}\n")
    np.savetxt(buf, A.reshape(-1, order="F"), fmt=FLOAT_FMT)
    data = buf.getvalue().encode()
    if gz:
        import gzip
        with gzip.open(path, "wb") as fh:
            fh.write(data)
    else:
        with open(path, "wb") as fh:
            fh.write(data)


def read_design(path) -> np.ndarray:
    """Matrix Market design as a dense float array (matrixio.py:48-58);
    desk-scale only -- use `read_design_pattern` for real designs."""
    n, p, rp, ci, _ = read_pattern(path)
    dense = np.zeros((n, p))
    rows = np.repeat(np.arange(n), np.diff(rp))
    dense[rows, ci] = 1.0
    return dense


def write_design_csv(path, X) -> None:
    """Dense CSV alternative to Matrix Market, one column per feature (matrixio.py:61-66)."""
    X = np.atleast_2d(np.asarray(X, dtype=np.float64))
    header = ",".join(f"x_{j}" for j in range(X.shape[1]))
    np.savetxt(path, X, fmt=FLOAT_FMT, delimiter=",", header=header, comments="")


def load_design(path) -> np.ndarray:
    """Design from .mtx / .mtx.gz / .csv by extension (matrixio.py:69-79)."""
    suffix = str(path).lower()
    if suffix.endswith(".mtx") or suffix.endswith(".mtx.gz"):
        return read_design(path)
    if suffix.endswith(".csv"):
        header, body = _read_csv(path)
        if not all(name == f"x_{j}" for j, name in enumerate(header)):
            raise FileFormatError(f"{path}: not a design CSV (expected columns x_0, x_1, ...)")
        return body
    raise FileFormatError(f"{path}: design must be .mtx or .csv")


def load_design_pattern(path, intercept="detect") -> SparseDesignMatrix:
    """Like `load_design` but into the pattern store (0/1 designs)."""
    suffix = str(path).lower()
    if suffix.endswith(".mtx") or suffix.endswith(".mtx.gz"):
        return read_design_pattern(path, intercept=intercept)
    dense = load_design(path)
    X = SparseDesignMatrix.from_dense(dense)
    if intercept is True:
        from .sparse import hstack_dense_columns
        return hstack_dense_columns(np.ones((X.n_rows, 1)), X)
    return X


# ----------------------------------------------------------------- CSV formats
# Headed CSV, one record per line, every field printed "%.17g" so values
# round-trip to the bit; the header strings are the public contract
# (matrixio.py:1-28).  Byte-identical to the reference's np.savetxt output.
def _write_csv(path, header, columns) -> None:
    table = np.column_stack([np.asarray(c, dtype=np.float64) for c in columns])
    np.savetxt(path, table, fmt=FLOAT_FMT, delimiter=",", header=",".join(header), comments="")


def _read_csv(path, expected_header=None):
    """(header, float table with one row per record); FileFormatError on a
    missing header, unparsable body or a width/header mismatch."""
    with open(path, newline="") as fh:
        head = fh.readline()
        body_text = fh.read()
    if not head:
        raise FileFormatError(f"{path}: empty file")
    header = tuple(next(csv.reader([head.rstrip("\r\n")])))
    if expected_header is not None and header != tuple(expected_header):
        raise FileFormatError(f"{path}: header {header} does not match the expected "
                              f"{tuple(expected_header)}")
    if not body_text.strip():
        return header, np.empty((0, len(header)))
    try:
        table = np.loadtxt(_io.StringIO(body_text), delimiter=",", ndmin=2)
    except ValueError as exc:
        raise FileFormatError(f"{path}: bad CSV body ({exc})") from exc
    if table.shape[1] != len(header):
        raise FileFormatError(f"{path}: {table.shape[1]} columns under a {len(header)}-column header")
    return header, table


def write_vector_csv(path, values, name) -> None:
    _write_csv(path, (name,), (values,))


def read_vector_csv(path, name=None) -> np.ndarray:
    return _read_csv(path, None if name is None else (name,))[1][:, 0]


def chain_columns(p: int) -> tuple:
    return tuple(f"beta_{j}" for j in range(p)) + CHAIN_FIXED_COLUMNS


def write_chain_csv(path, draws, tau_draws, logdensity) -> None:
    """Stored draws, one row each: beta_0..beta_{p-1}, tau, logdensity (matrixio.py:128-136)."""
    draws = np.atleast_2d(np.asarray(draws, dtype=np.float64))
    if not len(tau_draws) == len(logdensity) == draws.shape[0]:
        raise ValueError("draws, tau and logdensity must align")
    _write_csv(path, chain_columns(draws.shape[1]), [*draws.T, tau_draws, logdensity])


def read_chain_csv(path):
    """(beta draws, tau draws, logdensity) from a chain file (matrixio.py:139-147)."""
    header, table = _read_csv(path)
    p = len(header) - len(CHAIN_FIXED_COLUMNS)
    if p < 1 or header[p:] != CHAIN_FIXED_COLUMNS:
        raise FileFormatError(f"{path}: not a chain file")
    if header[:p] != chain_columns(p)[:p]:
        raise FileFormatError(f"{path}: beta columns out of order")
    return table[:, :p], table[:, p], table[:, p + 1]


def write_trace_csv(path, trace) -> None:
    """Per-iteration CG error metrics (matrixio.py:150-155) of an `ErrorTrace`."""
    k = len(trace.rms_precond_residual)
    _write_csv(path, TRACE_COLUMNS, (np.arange(k), trace.rms_precond_residual, trace.phi_norm_error,
                                     trace.l2_error, trace.rel_coord_error))


def read_trace_csv(path):
    return _read_csv(path, TRACE_COLUMNS)[1]


def write_spectrum_csv(path, eigenvalues) -> None:
    vals = np.asarray(eigenvalues, dtype=np.float64)
    with np.errstate(divide="ignore"):
        _write_csv(path, SPECTRUM_COLUMNS, (np.arange(vals.size), vals, np.log10(vals)))


def read_spectrum_csv(path) -> np.ndarray:
    return _read_csv(path, SPECTRUM_COLUMNS)[1][:, 1]


# ----------------------------------------------------------------- BRGS state files
MAGIC = b"BRGS"
VERSION = 1
_HEADER = struct.Struct("<4sBQQQd")


class StateFormatError(ValueError):
    """State file is truncated, malformed, or not a state file (stateio.py:26-27)."""


class StateVersionError(StateFormatError):
    """State file uses a schema version this build does not read (stateio.py:30-31)."""


def save_state(path, state) -> None:
    """Layout (stateio.py:1-10): magic "BRGS" | version u8 | n u64 | p_total
    u64 | p_shrunk u64 | tau f64 | beta f64[p_total] | omega f64[n] | lam
    f64[p_shrunk], little-endian; `load_state` restores it bit for bit."""
    arrays = [np.ascontiguousarray(a, dtype="<f8") for a in (state.beta, state.omega, state.lam)]
    beta, omega, lam = arrays
    head = _HEADER.pack(MAGIC, VERSION, omega.size, beta.size, lam.size, float(state.tau))
    with open(path, "wb") as fh:
        fh.write(head + b"".join(a.tobytes() for a in arrays))


def load_state(path):
    """Inverse of `save_state`, with the reference's checks (stateio.py:47-69)."""
    from .gibbs import ShrinkageState
    with open(path, "rb") as fh:
        blob = fh.read()
    if len(blob) < _HEADER.size:
        raise StateFormatError(f"{path}: truncated header ({len(blob)} of {_HEADER.size} bytes)")
    magic, version, n, p_total, p_shrunk, tau = _HEADER.unpack_from(blob)
    if magic != MAGIC:
        raise StateFormatError(f"{path}: bad magic {magic!r}")
    if version != VERSION:
        raise StateVersionError(f"{path}: state schema version {version}, this build reads version {VERSION}")
    want = _HEADER.size + 8 * (p_total + n + p_shrunk)
    if len(blob) != want:
        raise StateFormatError(f"{path}: expected {want} bytes for the declared shapes, found {len(blob)}")
    body = np.frombuffer(blob, dtype="<f8", offset=_HEADER.size)
    beta, omega, lam = np.split(body.copy(), [p_total, p_total + n])
    return ShrinkageState(beta, omega, lam, tau)
