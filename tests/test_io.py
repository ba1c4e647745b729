"""Design ingestion, BRGS state files and CSV artifacts (CPU).

Golden files in tests/golden/io/ were written by the reference's own writers
(priorcg.matrixio / priorcg.stateio, tests/golden/make_golden.py:io_cases);
scipy.io.mmread / mmwrite (the reference's Matrix Market engine,
matrixio.py:35-58) is the cross-check for files written here.
"""
import gzip
import warnings
from pathlib import Path

import numpy as np
import pytest
import scipy.io
import scipy.sparse as sp

from paper_1810_12437_b200 import io as pio
from paper_1810_12437_b200.gibbs import ShrinkageState
from paper_1810_12437_b200.sparse import SparseDesignMatrix

GOLD = Path(__file__).resolve().parent / "golden" / "io"
EXP = np.load(GOLD / "expected.npz")


def dense_of(n, p, rp, ci):
    d = np.zeros((n, p))
    d[np.repeat(np.arange(n), np.diff(rp)), ci] = 1.0
    return d


def mmread_dense(path):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        m = scipy.io.mmread(str(path))
    return m.toarray() if sp.issparse(m) else np.asarray(m)


# ----------------------------------------------------------------- golden files
def test_reads_reference_sparse_design_with_intercept():
    X = pio.read_design_pattern(GOLD / "design_sparse.mtx")
    rp, ci, icpt = X.pattern()
    assert icpt and X.n_rows == 23 and X.n_cols == 10
    np.testing.assert_array_equal(rp, EXP["rp"])
    np.testing.assert_array_equal(ci, EXP["ci"])


def test_reads_reference_dense_and_csv_designs():
    np.testing.assert_array_equal(pio.load_design(GOLD / "design_dense.mtx"), EXP["dense"])
    np.testing.assert_array_equal(pio.load_design(GOLD / "design.csv"), EXP["dense"])
    full = np.hstack([np.ones((23, 1)), EXP["dense"]])
    np.testing.assert_array_equal(pio.load_design(GOLD / "design_sparse.mtx"), full)
    X = pio.load_design_pattern(GOLD / "design.csv", intercept=True)
    np.testing.assert_array_equal(X.to_dense(), full)


def test_state_file_bit_exact(tmp_path):
    st = pio.load_state(GOLD / "state.brgs")
    np.testing.assert_array_equal(st.beta, EXP["beta"])
    np.testing.assert_array_equal(st.omega, EXP["omega"])
    np.testing.assert_array_equal(st.lam, EXP["lam"])
    assert st.tau == float(EXP["tau"])
    pio.save_state(tmp_path / "s.brgs", st)
    assert (tmp_path / "s.brgs").read_bytes() == (GOLD / "state.brgs").read_bytes()


@pytest.mark.parametrize("mutate,exc", [
    (lambda b: b[:20], pio.StateFormatError),
    (lambda b: b"XRGS" + b[4:], pio.StateFormatError),
    (lambda b: b[:4] + bytes([2]) + b[5:], pio.StateVersionError),
    (lambda b: b[:-8], pio.StateFormatError),
    (lambda b: b + b"\0" * 8, pio.StateFormatError),
])
def test_state_file_errors(tmp_path, mutate, exc):
    f = tmp_path / "bad.brgs"
    f.write_bytes(mutate((GOLD / "state.brgs").read_bytes()))
    with pytest.raises(exc):
        pio.load_state(f)


def test_csv_artifacts_byte_identical(tmp_path):
    draws, tau, ld = pio.read_chain_csv(GOLD / "chain.csv")
    np.testing.assert_array_equal(draws, EXP["draws"])
    pio.write_chain_csv(tmp_path / "c.csv", draws, tau, ld)
    assert (tmp_path / "c.csv").read_bytes() == (GOLD / "chain.csv").read_bytes()

    v = pio.read_vector_csv(GOLD / "vector.csv", "beta")
    pio.write_vector_csv(tmp_path / "v.csv", v, "beta")
    assert (tmp_path / "v.csv").read_bytes() == (GOLD / "vector.csv").read_bytes()

    ev = pio.read_spectrum_csv(GOLD / "spectrum.csv")
    pio.write_spectrum_csv(tmp_path / "s.csv", ev)
    assert (tmp_path / "s.csv").read_bytes() == (GOLD / "spectrum.csv").read_bytes()

    body = pio.read_trace_csv(GOLD / "trace.csv")

    class T:
        rms_precond_residual, phi_norm_error, l2_error, rel_coord_error = body[:, 1], body[:, 2], body[:, 3], body[:, 4]
    pio.write_trace_csv(tmp_path / "t.csv", T)
    assert (tmp_path / "t.csv").read_bytes() == (GOLD / "trace.csv").read_bytes()


def test_csv_errors(tmp_path):
    f = tmp_path / "x.csv"
    f.write_text("")
    with pytest.raises(pio.FileFormatError):
        pio.read_vector_csv(f)
    f.write_text("a,b\n1,2,3\n")
    with pytest.raises(pio.FileFormatError):
        pio.read_vector_csv(f)
    f.write_text("beta\nnope\n")
    with pytest.raises(pio.FileFormatError):
        pio.read_vector_csv(f, "beta")
    f.write_text("x,tau,logdensity\n1,2,3\n")
    with pytest.raises(pio.FileFormatError):
        pio.read_chain_csv(f)
    with pytest.raises(pio.FileFormatError):
        pio.read_trace_csv(GOLD / "chain.csv")
    with pytest.raises(pio.FileFormatError):
        pio.load_design(tmp_path / "d.txt")


# ----------------------------------------------------------------- Matrix Market round trips
def random_pattern(rng, n, p, density):
    mask = rng.random((n, p)) < density
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(mask.sum(1), out=rp[1:])
    return rp, np.nonzero(mask)[1].astype(np.int32)


@pytest.mark.parametrize("field", ["real", "pattern"])
@pytest.mark.parametrize("suffix", [".mtx", ".mtx.gz"])
def test_write_read_roundtrip_matches_scipy(tmp_path, field, suffix):
    rng = np.random.default_rng(len(field) + len(suffix))
    for trial in range(6):
        n, p = (int(v) for v in rng.integers(1, 120, size=2))
        rp, ci = random_pattern(rng, n, p, float(rng.uniform(0, 0.4)))
        X = SparseDesignMatrix.from_pattern(n, p, rp, ci, intercept=bool(trial % 2))
        f = tmp_path / f"d{trial}{suffix}"
        pio.write_design(f, X, field=field)
        np.testing.assert_array_equal(mmread_dense(f), X.to_dense())
        Y = pio.read_design_pattern(f, intercept="detect" if trial % 2 else False)
        np.testing.assert_array_equal(Y.to_dense(), X.to_dense())
        np.testing.assert_array_equal(pio.read_design(f), X.to_dense())


def test_reads_scipy_written_files(tmp_path):
    rng = np.random.default_rng(3)
    rp, ci = random_pattern(rng, 40, 17, 0.25)
    A = dense_of(40, 17, rp, ci)
    scipy.io.mmwrite(str(tmp_path / "s.mtx"), sp.coo_matrix(A))
    scipy.io.mmwrite(str(tmp_path / "a.mtx"), A)
    scipy.io.mmwrite(str(tmp_path / "i.mtx"), sp.coo_matrix(A.astype(np.int64)))
    for name in ("s.mtx", "a.mtx", "i.mtx"):
        np.testing.assert_array_equal(pio.read_design(tmp_path / name), A)
    n, p, rp2, ci2, meta = pio.read_pattern(tmp_path / "i.mtx")
    assert meta["field"] == "integer"
    np.testing.assert_array_equal(rp2, rp)
    np.testing.assert_array_equal(ci2, ci)


def test_parser_tolerates_comments_blank_lines_crlf_and_unsorted(tmp_path):
    text = ("%%MatrixMarket matrix coordinate integer general\r\n% a comment\r\n\r\n"
            "3 4 5\r\n3 1 1\r\n1 4 1\r\n\r\n% mid comment\r\n1 2 1\r\n2 3 0\r\n3 4 1")
    f = tmp_path / "c.mtx"
    f.write_bytes(text.encode())
    n, p, rp, ci, meta = pio.read_pattern(f)
    assert (n, p) == (3, 4) and meta["zeros_dropped"] == 1 and meta["entries"] == 5
    np.testing.assert_array_equal(rp, [0, 2, 2, 4])
    np.testing.assert_array_equal(ci, [1, 3, 0, 3])


def test_symmetric_is_mirrored(tmp_path):
    f = tmp_path / "sym.mtx"
    f.write_text("%%MatrixMarket matrix coordinate pattern symmetric\n3 3 3\n1 1\n3 1\n3 2\n")
    want = np.array([[1, 0, 1], [0, 0, 1], [1, 1, 0]], dtype=float)
    np.testing.assert_array_equal(pio.read_design(f), want)


def test_empty_designs(tmp_path):
    f = tmp_path / "e.mtx"
    f.write_text("%%MatrixMarket matrix coordinate real general\n5 3 0\n")
    n, p, rp, ci, _ = pio.read_pattern(f)
    assert (n, p, len(ci)) == (5, 3, 0)
    np.testing.assert_array_equal(rp, np.zeros(6))
    X = SparseDesignMatrix.from_pattern(4, 0, np.zeros(5, dtype=np.int64), np.zeros(0, np.int32), intercept=True)
    pio.write_design(tmp_path / "i.mtx", X)
    Y = pio.read_design_pattern(tmp_path / "i.mtx")
    assert Y.has_intercept and Y.n_cols == 1


@pytest.mark.parametrize("body,exc", [
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 2.5\n", NotImplementedError),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 -1\n", NotImplementedError),
    ("%%MatrixMarket matrix coordinate complex general\n2 2 1\n1 1 1 0\n", NotImplementedError),
    ("%%MatrixMarket matrix coordinate real skew-symmetric\n2 2 1\n2 1 1\n", NotImplementedError),
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n1 1 1\n", pio.FileFormatError),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1\n", pio.FileFormatError),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n0 1 1\n", pio.FileFormatError),
    ("%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1\n", pio.FileFormatError),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1\n2 2 1\n", pio.FileFormatError),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1\n", pio.FileFormatError),
    ("%%MatrixMarket matrix coordinate pattern general\n2 2 1\n1 1 x\n", pio.FileFormatError),
    ("%%MatrixMarket matrix coordinate real general\n2 2\n", pio.FileFormatError),
    ("%%MatrixMarket vector coordinate real general\n2 2 1\n1 1 1\n", pio.FileFormatError),
    ("just text\n", pio.FileFormatError),
    ("", pio.FileFormatError),
    ("%%MatrixMarket matrix coordinate pattern symmetric\n2 3 1\n1 1\n", pio.FileFormatError),
])
def test_parser_errors(tmp_path, body, exc):
    f = tmp_path / "bad.mtx"
    f.write_text(body)
    with pytest.raises(exc):
        pio.read_pattern(f)


def test_missing_and_corrupt_files(tmp_path):
    with pytest.raises(OSError):
        pio.read_pattern(tmp_path / "nope.mtx")
    good = gzip.compress(b"%%MatrixMarket matrix coordinate pattern general\n2 2 2\n1 1\n2 2\n" * 1)
    f = tmp_path / "t.mtx.gz"
    f.write_bytes(good[: len(good) // 2])
    with pytest.raises((OSError, pio.FileFormatError)):
        pio.read_pattern(f)


def test_streaming_medium_design(tmp_path):
    """~2 M entries through write -> parse -> pattern store, no dense copy."""
    rng = np.random.default_rng(9)
    n, p = 100_000, 2_000
    counts = rng.binomial(p, 0.01, size=n)
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=rp[1:])
    ci = np.concatenate([np.sort(rng.choice(p, size=c, replace=False)) for c in counts]).astype(np.int32)
    X = SparseDesignMatrix.from_pattern(n, p, rp, ci, intercept=True)
    f = tmp_path / "m.mtx.gz"
    pio.write_design(f, X, field="pattern")
    Y = pio.read_design_pattern(f)
    rp2, ci2, icpt = Y.pattern()
    assert icpt
    np.testing.assert_array_equal(rp2, rp)
    np.testing.assert_array_equal(ci2, ci)
