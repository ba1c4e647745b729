"""Binary sparse designs on the B200: the drop-in for priorcg.sparse.

`SparseDesignMatrix` keeps the reference constructor and attribute contract
(pkg/src/priorcg/sparse.py:46-117): host CSR arrays, standardisation vectors,
call counters, `matvec` / `matvec_t`.  The kernels run on the GPU through the
pattern-only store of libpcgs (include/pcgs.h: pcgs_design_create): values
are implicit ones, a leading dense all-ones column (the intercept that
`hstack_dense_columns` prepends, sparse.py:314-341) is stripped into a dense
term, and the remaining pattern is re-encoded as uint16 slab-local indices.

`SparseDesignMatrix.from_pattern` builds the same object straight from a
shrunk-block pattern plus an intercept flag without materialising the
reference's float64 `values` (8 B/nnz), which is what paper-scale designs use.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib

DEFAULT_DENSE_CAP = 5000


class DimensionCapError(RuntimeError):
    """Dense operation requested above the dimension cap; use the CG path."""


class NotPositiveDefiniteError(RuntimeError):
    """A matrix that must be positive definite is not (sparse.py:31)."""


class ZeroVarianceColumnError(ValueError):
    """Standardization hit a constant column that was not excluded."""


def _finite_f64(x, name):
    arr = np.ascontiguousarray(x, dtype=np.float64)
    if not np.all(np.isfinite(arr)):
        raise ValueError(f"{name} contains non-finite entries")
    return arr


def _check_csr(n, p, row_ptr, col_idx, nvals):
    """The reference's CSR invariants (sparse.py:94-117)."""
    if row_ptr.shape != (n + 1,):
        raise ValueError("row_ptr must have length n_rows + 1")
    if row_ptr[0] != 0 or row_ptr[-1] != nvals:
        raise ValueError("row_ptr endpoints must be 0 and nnz")
    if np.any(np.diff(row_ptr) < 0):
        raise ValueError("row_ptr must be nondecreasing")
    if len(col_idx) != nvals:
        raise ValueError("col_idx and values must have equal length")
    if col_idx.size:
        if col_idx.min() < 0 or col_idx.max() >= p:
            raise ValueError("col_idx entry out of range")
        d = np.diff(col_idx)
        if d.size:
            bad = d <= 0
            inner = row_ptr[1:-1]
            inner = inner[(inner > 0) & (inner < len(col_idx))] - 1
            bad[inner] = False
            if np.any(bad):
                raise ValueError("col_idx must be strictly increasing within each row")


class DesignStore:
    """Owner of one libpcgs design handle on one CUDA device."""

    def __init__(self, n, p, row_ptr, col_idx, intercept, device=None, slab_max=0, grid=0, q_dense=0):
        L = _lib.lib()
        self.device = _lib.cuda_device(device)
        rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
        ci = np.ascontiguousarray(col_idx, dtype=np.int32)
        h = ctypes.c_void_p()
        _lib.check(L.pcgs_design_create_affine(int(n), int(p), rp.ctypes.data, ci.ctypes.data,
                                               int(bool(intercept)), int(q_dense), int(slab_max),
                                               int(self.device.index), int(grid), ctypes.byref(h)))
        self.q_dense = int(q_dense)
        self._affine = None   # (dense, mu, sc) device tensors kept alive while attached
        self._h = h
        info = np.zeros(16, dtype=np.int64)
        _lib.check(L.pcgs_design_info(h, info.ctypes.data))
        self.info = info
        self.n, self.p, self.p_total, self.nnz = (int(v) for v in info[:4])
        self.intercept = bool(intercept)

    @property
    def handle(self):
        return self._h

    def set_affine(self, dense=None, mu=None, sc=None):
        """Attach the affine terms (dense block values, column means / scales,
        reference layout) to the device handle; None detaches one."""
        self._affine = (dense, mu, sc)
        _lib.check(_lib.lib().pcgs_design_set_affine(
            self._h, _lib.ptr(dense) if dense is not None else None, _lib.ptr(mu) if mu is not None else None,
            _lib.ptr(sc) if sc is not None else None))

    def describe(self) -> dict:
        keys = ["n", "p", "p_total", "nnz", "csr_slabs", "csc_slabs", "csr_vectors",
                "csc_vectors", "csr_slices", "csc_slices", "csc_pieces", "grid", "device",
                "index_bytes", "slab_max"]
        return {k: int(v) for k, v in zip(keys, self.info)}

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _lib.lib().pcgs_design_destroy(h)
            except Exception:  # pragma: no cover - interpreter shutdown
                pass
            self._h = None

    # ---- device primitives (tensors in, tensors out) ----
    def _stream(self):
        return _lib.stream_ptr(self.device)

    def matvec(self, v, out=None):
        t = _lib.torch()
        out = t.empty(self.n, dtype=t.float64, device=self.device) if out is None else out
        _lib.check(_lib.lib().pcgs_matvec(self._h, _lib.ptr(v), _lib.ptr(out), self._stream()))
        return out

    def matvec_t(self, w, out=None):
        t = _lib.torch()
        out = t.empty(self.p_total, dtype=t.float64, device=self.device) if out is None else out
        _lib.check(_lib.lib().pcgs_matvec_t(self._h, _lib.ptr(w), _lib.ptr(out), self._stream()))
        return out

    def phi_apply(self, omega, diag, v, out=None):
        t = _lib.torch()
        out = t.empty(self.p_total, dtype=t.float64, device=self.device) if out is None else out
        _lib.check(_lib.lib().pcgs_phi_apply(self._h, _lib.ptr(omega), _lib.ptr(diag), _lib.ptr(v),
                                             _lib.ptr(out), self._stream()))
        return out

    def phi_diagonal(self, omega, diag, out=None):
        t = _lib.torch()
        out = t.empty(self.p_total, dtype=t.float64, device=self.device) if out is None else out
        _lib.check(_lib.lib().pcgs_phi_diagonal(self._h, _lib.ptr(omega), _lib.ptr(diag),
                                                _lib.ptr(out), self._stream()))
        return out


class SparseDesignMatrix:
    """CSR design whose products run on the GPU (drop-in for sparse.py:46).

    Parameters are the reference's.  Device products require a binary design
    (every stored value 1.0) and identity standardisation; anything else raises
    NotImplementedError at the first device call rather than silently falling
    back to the CPU.
    """

    def __init__(self, n_rows, n_cols, row_ptr, col_idx, values,
                 col_means=None, col_scales=None):
        self.n_rows = int(n_rows)
        self.n_cols = int(n_cols)
        self._row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
        self._col_idx = np.ascontiguousarray(col_idx, dtype=np.int64)
        self._values = _finite_f64(values, "values")
        self._pattern = None  # (shrunk row_ptr, shrunk col_idx int32, intercept)
        self.col_means = _finite_f64(np.zeros(self.n_cols) if col_means is None else col_means,
                                     "col_means")
        self.col_scales = _finite_f64(np.ones(self.n_cols) if col_scales is None else col_scales,
                                      "col_scales")
        self.constant_columns = np.zeros(0, dtype=np.int64)
        self.matvec_calls = 0
        self.matvec_t_calls = 0
        self.weighted_gram_calls = 0
        self._stores = {}
        self.slab_max = 0
        _check_csr(self.n_rows, self.n_cols, self._row_ptr, self._col_idx, len(self._values))
        if self.col_means.shape != (self.n_cols,) or self.col_scales.shape != (self.n_cols,):
            raise ValueError("col_means/col_scales must have length n_cols")
        if np.any(self.col_scales <= 0):
            raise ValueError("col_scales must be strictly positive")

    # ------------------------------------------------------------ constructors
    @classmethod
    def from_dense(cls, dense):
        dense = np.asarray(dense, dtype=np.float64)
        if dense.ndim != 2:
            raise ValueError("expected a 2-d array")
        n, p = dense.shape
        mask = dense != 0.0
        row_ptr = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(mask.sum(axis=1), out=row_ptr[1:])
        rows, cols = np.nonzero(mask)
        return cls(n, p, row_ptr, cols.astype(np.int64), dense[rows, cols])

    @classmethod
    def from_coo(cls, n_rows, n_cols, rows, cols, vals):
        import scipy.sparse
        coo = scipy.sparse.coo_matrix(
            (np.asarray(vals, dtype=np.float64),
             (np.asarray(rows, dtype=np.int64), np.asarray(cols, dtype=np.int64))),
            shape=(n_rows, n_cols))
        csr = coo.tocsr()
        csr.sum_duplicates()
        csr.sort_indices()
        return cls(n_rows, n_cols, csr.indptr, csr.indices, csr.data)

    @classmethod
    def from_pattern(cls, n_rows, n_shrunk, row_ptr, col_idx, intercept=True, check=True):
        """Binary design from the shrunk-block pattern (+ optional dense intercept).

        The reference-layout arrays (`row_ptr`, `col_idx`, `values`, with the
        intercept as column 0) are materialised lazily on first access.
        """
        self = cls.__new__(cls)
        self.n_rows = int(n_rows)
        self.n_cols = int(n_shrunk) + (1 if intercept else 0)
        rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
        ci = np.ascontiguousarray(col_idx, dtype=np.int32)
        if check:
            _check_csr(self.n_rows, int(n_shrunk), rp, ci, int(rp[-1]) if rp.size else 0)
        self._row_ptr = self._col_idx = self._values = None
        self._pattern = (rp, ci, bool(intercept))
        self.col_means = np.zeros(self.n_cols)
        self.col_scales = np.ones(self.n_cols)
        self.constant_columns = np.zeros(0, dtype=np.int64)
        self.matvec_calls = self.matvec_t_calls = self.weighted_gram_calls = 0
        self._stores = {}
        self.slab_max = 0
        return self

    # ------------------------------------------------------------ reference-layout arrays
    def _materialise(self):
        rp, ci, icpt = self._pattern
        n = self.n_rows
        if not icpt:
            self._row_ptr = rp.copy()
            self._col_idx = ci.astype(np.int64)
        else:
            self._row_ptr = rp + np.arange(n + 1, dtype=np.int64)
            counts = np.diff(rp)
            col = np.empty(len(ci) + n, dtype=np.int64)
            first = self._row_ptr[:-1]
            col[first] = 0
            mask = np.ones(len(col), dtype=bool)
            mask[first] = False
            col[mask] = ci.astype(np.int64) + 1
            self._col_idx = col
            del counts
        self._values = np.ones(len(self._col_idx))

    @property
    def row_ptr(self):
        if self._row_ptr is None:
            self._materialise()
        return self._row_ptr

    @property
    def col_idx(self):
        if self._col_idx is None:
            self._materialise()
        return self._col_idx

    @property
    def values(self):
        if self._values is None:
            self._materialise()
        return self._values

    @property
    def nnz(self):
        if self._values is not None:
            return len(self._values)
        if self._pattern is not None:
            rp, _, icpt = self._pattern
            return int(rp[-1]) + (self.n_rows if icpt else 0)
        return len(self._values)

    # ------------------------------------------------------------ pattern + device store
    def pattern(self):
        """(shrunk row_ptr int64, shrunk col_idx int32, intercept flag)."""
        if self._pattern is not None:
            return self._pattern
        if not np.all(self._values == 1.0):
            return self._dense_pattern()
        rp, ci, n = self._row_ptr, self._col_idx, self.n_rows
        counts = np.diff(rp)
        icpt = False
        if self.n_cols >= 1 and n > 0 and np.all(counts >= 1):
            icpt = bool(np.all(ci[rp[:-1]] == 0))
        if icpt:
            keep = np.ones(len(ci), dtype=bool)
            keep[rp[:-1]] = False
            sci = (ci[keep] - 1).astype(np.int32)
            srp = rp - np.arange(n + 1, dtype=np.int64)
        else:
            sci = ci.astype(np.int32)
            srp = rp.copy()
        self._pattern = (srp, sci, icpt)
        return self._pattern

    def _dense_pattern(self):
        """A design [Dn | B] with a leading block of q fully stored real
        columns (hstack_dense_columns of a real block, sparse.py:314-341) and a
        binary remainder: the pattern of B plus the dense values (n, q).  The
        device applies Dn through the affine terms of the store."""
        rp, ci, vals, n = self._row_ptr, self._col_idx, self._values, self.n_rows
        counts = np.diff(rp)
        q = 0
        while q < self.n_cols and n > 0 and np.all(counts > q) and np.all(ci[rp[:-1] + q] == q):
            q += 1
        rest = np.ones(len(ci), dtype=bool)
        if q:
            rest[(rp[:-1, None] + np.arange(q)).ravel()] = False
        if q == 0 or not np.all(vals[rest] == 1.0):
            raise NotImplementedError(
                "the B200 store is pattern-only apart from a leading dense block: every value outside "
                "the leading fully stored columns must be 1.0 (binary design)")
        if q > 32:
            raise NotImplementedError("a leading dense block of more than 32 columns is not on the device path")
        self._dense = np.ascontiguousarray(vals[~rest].reshape(n, q))
        srp = rp - q * np.arange(n + 1, dtype=np.int64)
        sci = (ci[rest] - q).astype(np.int32)
        self._pattern = (srp, sci, False)
        return self._pattern

    @property
    def dense_block(self):
        """Leading dense real columns (n, q) handled by the affine terms, or None."""
        self.pattern()
        return getattr(self, "_dense", None)

    @property
    def affine(self):
        """True when the device applies affine terms (dense block or standardisation)."""
        return self.dense_block is not None or self.standardized

    @property
    def has_intercept(self):
        return self.pattern()[2]

    def device_store(self, device=None, grid=0, raw=False, ranges=0) -> DesignStore:
        """The store on `device`; `grid` > 0 plans it for that many CTAs
        (row-split shards or chains side by side sharing a GPU); `ranges` > 0
        sets the warp ranges per CTA task (the row-split kernel runs 32 warps
        and builds its shards with 32; the default, 16, is the persistent PCG
        kernel's warp count).  The affine
        terms (dense block, standardisation) are attached to it and follow
        later standardize() calls; `raw` = the pattern-only view of a
        pattern-only design (the Gibbs reparametrisation of standardised
        designs samples on the raw pattern)."""
        dev = _lib.cuda_device(device)
        rp, ci, icpt = self.pattern()
        dense = self.dense_block
        key = (dev.index, 1, int(grid), bool(raw), int(ranges))
        st = self._stores.get(key)
        if st is None:
            q = 0 if dense is None else dense.shape[1]
            if ranges:
                _lib.lib().pcgs_debug_option(3, int(ranges))
            try:
                st = DesignStore(self.n_rows, self.n_cols - (1 if icpt else 0) - q, rp, ci, icpt,
                                 device=dev, slab_max=self.slab_max, grid=grid, q_dense=q)
            finally:
                if ranges:
                    _lib.lib().pcgs_debug_option(3, 0)
            self._stores[key] = st
        if raw:
            if dense is not None:
                raise ValueError("a design with a dense block has no raw pattern view")
            return st
        std = self.standardized
        src = (self.col_means if std else None, self.col_scales if std else None)
        cur = getattr(st, "_affine_src", None)
        if dense is None and not std:
            if st._affine is not None:
                st.set_affine(None, None, None)
                st._affine, st._affine_src = None, None
        elif cur is None or cur[0] is not src[0] or cur[1] is not src[1]:
            dd = _lib.to_device(dense, dev) if dense is not None else None
            mu = _lib.to_device(src[0], dev) if std else None
            sc = _lib.to_device(src[1], dev) if std else None
            st.set_affine(dd, mu, sc)
            st._affine_src = src
        return st

    def batch_store(self, nchains, device=None, grid=0):
        """The sliced store of R = `nchains` batched chains on `device`
        (batched.BatchStore; built once per (device, R, grid))."""
        from .batched import BatchStore
        if self.affine:
            raise NotImplementedError("batched chains: designs with a dense block or standardisation are "
                                      "not on the batched path")
        dev = _lib.cuda_device(device)
        key = (dev.index, "batch", int(nchains), int(grid))
        st = self._stores.get(key)
        if st is None:
            rp, ci, icpt = self.pattern()
            st = BatchStore(self.n_rows, self.n_cols - (1 if icpt else 0), rp, ci, icpt, int(nchains),
                            device=dev, slab_max=self.slab_max, grid=grid)
            self._stores[key] = st
        return st

    # ------------------------------------------------------------ kernels
    def matvec(self, v):
        """X v (sparse.py:178-193), on the GPU; numpy in -> numpy out, tensor in -> tensor out."""
        as_tensor = _lib.is_tensor(v)
        if not as_tensor:
            v = np.asarray(v, dtype=np.float64)
        if tuple(v.shape) != (self.n_cols,):
            raise ValueError("matvec: vector length must equal n_cols")
        self.matvec_calls += 1
        st = self.device_store(v.device if as_tensor and v.is_cuda else None)
        out = self.device_matvec(_lib.to_device(v, st.device))
        return out if as_tensor else out.cpu().numpy()

    def matvec_t(self, w):
        """X' w (sparse.py:195-203), on the GPU."""
        as_tensor = _lib.is_tensor(w)
        if not as_tensor:
            w = np.asarray(w, dtype=np.float64)
        if tuple(w.shape) != (self.n_rows,):
            raise ValueError("matvec_t: vector length must equal n_rows")
        self.matvec_t_calls += 1
        st = self.device_store(w.device if as_tensor and w.is_cuda else None)
        out = self.device_matvec_t(_lib.to_device(w, st.device))
        return out if as_tensor else out.cpu().numpy()

    # ------------------------------------------------------------ standardisation
    @property
    def standardized(self):
        return bool(np.any(self.col_means != 0.0) or np.any(self.col_scales != 1.0))

    def device_matvec(self, v):
        """X v on a CUDA tensor: one pattern pass, the affine terms (dense
        block, the shift/scale of sparse.py:188-193) applied in the same kernel."""
        return self.device_store(v.device).matvec(v)

    def device_matvec_t(self, w):
        """X' w on a CUDA tensor (+ the correction of sparse.py:203, in-kernel)."""
        return self.device_store(w.device).matvec_t(w)

    def standardize(self, exclude=None):
        """Centre and scale columns in place (sparse.py:250-297); returns self.

        Column means and sample sds (ddof 1) over all n rows, implicit zeros
        included; `exclude` (bool mask or indices) and constant columns (sd
        below 1e-7 relative to the column's RMS, recorded in
        `constant_columns`) keep mean 0 and scale 1.  The device applies the
        result as a rank-one correction around the pattern-only passes.
        """
        n, m = self.n_rows, self.n_cols
        if n < 2:
            raise ValueError("standardize needs at least 2 rows")
        active = np.ones(m, dtype=bool)
        if exclude is not None:
            ex = np.asarray(exclude)
            if ex.dtype == bool and ex.shape != (m,):
                raise ValueError("boolean exclude mask must have length n_cols")
            active[ex] = False
        col, val = self.col_idx, self.values
        per_col = lambda w: np.bincount(col, weights=w, minlength=m)  # noqa: E731
        mean = per_col(val) / n
        stored = np.bincount(col, minlength=m)
        # centred sum of squares in two passes (stored entries, then the
        # n - stored implicit zeros): no cancellation on near-constant columns
        centred_ss = per_col((val - mean[col]) ** 2) + (n - stored) * mean ** 2
        rms_sq = per_col(val * val) / n
        flat = centred_ss <= (n - 1) * 1e-14 * np.maximum(rms_sq, 1e-300)
        self.constant_columns = np.flatnonzero(flat & active)
        use = active & ~flat
        self.col_means = np.where(use, mean, 0.0)
        self.col_scales = np.where(use, np.sqrt(centred_ss / (n - 1)), 1.0)
        return self

    def gram_diagonal(self, omega):
        """diag(X' diag(omega) X) (sparse.py:235-246): for a binary design, X' omega."""
        as_tensor = _lib.is_tensor(omega)
        if not as_tensor:
            omega = np.asarray(omega, dtype=np.float64)
        if tuple(omega.shape) != (self.n_rows,):
            raise ValueError("gram_diagonal: omega length must equal n_rows")
        st = self.device_store(omega.device if as_tensor and omega.is_cuda else None)
        t = _lib.torch()
        zero = t.zeros(st.p_total, dtype=t.float64, device=st.device)
        om = _lib.to_device(omega, st.device)
        out = st.phi_diagonal(om, zero)   # sum_i omega_i x_ij^2, affine terms in-kernel
        return out if as_tensor else out.cpu().numpy()

    # ------------------------------------------------------------ host views (tests)
    def to_dense_raw(self, dense_cap=DEFAULT_DENSE_CAP):
        _check_cap(self.n_cols, dense_cap, "to_dense_raw")
        out = np.zeros((self.n_rows, self.n_cols))
        rows = np.repeat(np.arange(self.n_rows), np.diff(self.row_ptr))
        out[rows, self.col_idx] = self.values
        return out

    def to_dense(self, dense_cap=DEFAULT_DENSE_CAP):
        raw = self.to_dense_raw(dense_cap=dense_cap)
        return (raw - self.col_means) / self.col_scales


def hstack_dense_columns(cols, X):
    """Prepend dense columns (sparse.py:314-341).

    A single all-ones column in front of a pattern-only design without an
    intercept becomes the store's dense intercept (no CSR copy); any other
    block is materialised in the reference layout.
    """
    cols = np.atleast_2d(np.asarray(cols, dtype=np.float64))
    if cols.shape[0] == 1 and X.n_rows != 1:
        cols = cols.T
    if cols.shape[0] != X.n_rows:
        raise ValueError("column block row count must match the design")
    q = cols.shape[1]
    if q == 0:
        return X
    if (q == 1 and np.all(cols == 1.0) and X._pattern is not None and not X._pattern[2]):
        rp, ci, _ = X._pattern
        return SparseDesignMatrix.from_pattern(X.n_rows, X.n_cols, rp, ci, intercept=True,
                                               check=False)
    n = X.n_rows
    if np.all((cols == 0.0) | (cols == 1.0)) and np.all(X.values == 1.0):
        return _hstack_binary_block(cols == 1.0, X)
    row_ptr = X.row_ptr + q * np.arange(n + 1, dtype=np.int64)
    counts = np.diff(X.row_ptr)
    total = X.nnz + n * q
    col_idx = np.empty(total, dtype=np.int64)
    values = np.empty(total)
    dense_pos = (row_ptr[:-1][:, None] + np.arange(q, dtype=np.int64)).ravel()
    col_idx[dense_pos] = np.tile(np.arange(q, dtype=np.int64), n)
    values[dense_pos] = cols.ravel()
    rows = np.repeat(np.arange(n, dtype=np.int64), counts)
    orig = np.arange(X.nnz, dtype=np.int64) + q * (rows + 1)
    col_idx[orig] = X.col_idx + q
    values[orig] = X.values
    means = np.concatenate([np.zeros(q), X.col_means])
    scales = np.concatenate([np.ones(q), X.col_scales])
    return SparseDesignMatrix(n, X.n_cols + q, row_ptr, col_idx, values,
                              col_means=means, col_scales=scales)


def _hstack_binary_block(mask, X):
    """hstack_dense_columns of a 0/1 block in front of a binary design, stored
    pattern-only (its ones; the reference stores the block's zeros as explicit
    entries, which changes no product): the result stays on the device path, the
    block's leading all-ones column becoming the store's dense intercept and
    the other block columns (dummy covariates, e.g. an unshrunk block with
    q > 1 prior sds) ordinary pattern columns."""
    n, q = mask.shape
    bc = mask.sum(1).astype(np.int64)
    xc = np.diff(X.row_ptr)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(bc + xc, out=row_ptr[1:])
    col_idx = np.empty(int(row_ptr[-1]), dtype=np.int64)
    bi, bj = np.nonzero(mask)                           # row-major: sorted by row, then column
    first = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(bc, out=first[1:])
    col_idx[row_ptr[bi] + (np.arange(len(bi)) - first[bi])] = bj
    rows = np.repeat(np.arange(n, dtype=np.int64), xc)
    col_idx[np.arange(X.nnz, dtype=np.int64) - X.row_ptr[rows] + row_ptr[rows] + bc[rows]] = X.col_idx + q
    means = np.concatenate([np.zeros(q), X.col_means])
    scales = np.concatenate([np.ones(q), X.col_scales])
    return SparseDesignMatrix(n, X.n_cols + q, row_ptr, col_idx, np.ones(len(col_idx)),
                              col_means=means, col_scales=scales)


def _check_cap(dim, dense_cap, what):
    if dense_cap is not None and dim > dense_cap:
        raise DimensionCapError(
            f"{what}: dimension {dim} exceeds the dense cap {dense_cap}; "
            "use the matrix-free CG path or raise the cap explicitly")


class DenseSymmetric:
    """Square symmetric matrix under the dense dimension cap (sparse.py:344-359).

    Kept for the drop-in namespace: the dense Cholesky path it feeds
    (`direct_sample`) is the CPU oracle's and is not on the device path."""

    def __init__(self, entries, dense_cap=DEFAULT_DENSE_CAP):
        a = np.ascontiguousarray(entries, dtype=np.float64)
        if a.ndim != 2 or a.shape[0] != a.shape[1]:
            raise ValueError("expected a square matrix")
        _check_cap(a.shape[0], dense_cap, "DenseSymmetric")
        top = float(np.abs(a).max()) if a.size else 0.0
        if a.size and float(np.abs(a - a.T).max()) > 1e-12 * max(top, 1.0):
            raise ValueError("matrix is not symmetric to 1e-12 relative")
        self.entries = a

    @property
    def dim(self):
        return self.entries.shape[0]
