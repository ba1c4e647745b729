"""The C-ABI library: loads, exports every symbol include/pcgs.h declares, and
its host-only builder reproduces designs exactly (no GPU needed)."""
import ctypes
import re

import numpy as np
import pytest

from conftest import ROOT
from paper_1810_12437_b200 import _lib, synth

HEADER = ROOT / "include" / "pcgs.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pcgs_[a-z0-9_]+)\s*\(", text)) - {"pcgs_apply_fn"})


def test_library_loads_and_exports_every_declared_symbol():
    L = _lib.lib()
    names = declared_functions()
    assert len(names) >= 14
    for name in names:
        assert hasattr(L, name), name
        assert name in _lib.SIGNATURES, f"{name} has no ctypes signature"
    assert L.pcgs_version() >= 1


def test_ctypes_signatures_match_header_arity():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    for name in declared_functions():
        m = re.search(rf"\b{name}\s*\(([^)]*)\)", text)
        params = [x for x in m.group(1).split(",") if x.strip() and x.strip() != "void"]
        assert len(params) == len(_lib.SIGNATURES[name][1]), name


def test_no_cpu_fallback_symbols():
    # the product library is device code plus host plumbing only
    assert "pcgs_matvec_cpu" not in _lib.SIGNATURES


def _selftest(n, p, rp, ci, intercept, slab_max, grid=148):
    L = _lib.lib()
    st = np.zeros(8, dtype=np.int64)
    rp = np.ascontiguousarray(rp, dtype=np.int64)
    ci = np.ascontiguousarray(ci, dtype=np.int32)
    rc = L.pcgs_store_selftest(n, p, rp.ctypes.data, ci.ctypes.data, int(intercept), slab_max, grid,
                               st.ctypes.data)
    return rc, L.pcgs_last_error().decode(), st


def random_pattern(rng, n, p, density):
    mask = rng.random((n, p)) < density
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(mask.sum(1), out=rp[1:])
    return rp, np.nonzero(mask)[1].astype(np.int32)


@pytest.mark.parametrize("slab_max", [0, 16, 40, 300])
@pytest.mark.parametrize("intercept", [True, False])
def test_store_roundtrip_random(slab_max, intercept):
    rng = np.random.default_rng(slab_max + intercept)
    for _ in range(12):
        n, p = (int(v) for v in rng.integers(1, 400, size=2))
        rp, ci = random_pattern(rng, n, p, float(rng.uniform(0, 0.6)))
        for grid in (1, 3, 148):
            rc, msg, _ = _selftest(n, p, rp, ci, intercept, slab_max, grid)
            assert rc == 0, msg


def test_store_edge_cases():
    # empty design, single row, single column, a dense row, empty rows
    cases = [
        (5, 4, np.zeros(6, dtype=np.int64), np.zeros(0, dtype=np.int32)),
        (1, 3, np.array([0, 2]), np.array([0, 2], dtype=np.int32)),
        (4, 1, np.array([0, 1, 1, 2, 2]), np.array([0, 0], dtype=np.int32)),
        (3, 2000, np.array([0, 2000, 2000, 2001]),
         np.concatenate([np.arange(2000), [1999]]).astype(np.int32)),
    ]
    for n, p, rp, ci in cases:
        for icpt in (True, False):
            for sm in (0, 16):
                rc, msg, _ = _selftest(n, p, rp, ci, icpt, sm)
                assert rc == 0, msg


def test_store_rejects_malformed_csr():
    for rp, ci, p in [(np.array([0, 2]), np.array([1, 1], dtype=np.int32), 3),   # not increasing
                      (np.array([0, 1]), np.array([3], dtype=np.int32), 3),       # out of range
                      (np.array([1, 1]), np.array([0], dtype=np.int32), 3)]:      # bad start
        rc, _, _ = _selftest(1, p, rp, ci, True, 0)
        assert rc == _lib.PCGS_EINVAL


def _midsize_pattern():
    rng = np.random.default_rng(3)
    n, p = 30000, 6000
    rates = np.exp(rng.uniform(np.log(1e-3), np.log(0.3), p))
    cols = [np.flatnonzero(rng.random(n) < r) for r in rates]
    ci_by_row = [[] for _ in range(n)]
    for j, rows in enumerate(cols):
        for i in rows:
            ci_by_row[i].append(j)
    rp = np.zeros(n + 1, dtype=np.int64)
    rp[1:] = np.cumsum([len(r) for r in ci_by_row])
    ci = np.fromiter((j for r in ci_by_row for j in r), dtype=np.int32, count=int(rp[-1]))
    return n, p, rp, ci


def test_store_config1_layout_and_bank_balance(monkeypatch):
    d = synth.config_design(1, seed=0)
    rc, msg, st = _selftest(d.n, d.p, d.row_ptr, d.col_idx, True, 0)
    assert rc == 0, msg
    assert st[0] == 1 and st[1] == 1       # one slab each way
    assert st[6] / (16 * st[5]) < 0.1      # < 10 % of shared-memory picks conflict
    # index bytes: 2 B per index, padded to 8 per segment; the grouped layout
    # also pads its slices, which at this size (3 columns per CTA) is most of
    # the stream -- at a size that fills the grid the padding is a few percent
    assert st[7] < 2 * 2 * (d.nnz + d.n) * 4.0
    n, p, rp, ci = _midsize_pattern()
    rc, msg, st = _selftest(n, p, rp, ci, True, 0)
    assert rc == 0, msg
    assert st[7] < 2 * 2 * (rp[-1] + n) * 1.12
    assert st[6] / st[5] < 0.35            # predicted extra wavefronts per half-warp gather
    # replicas (PCGS_REPLICAS=1): the same pattern round-trips through the
    # replica indices and the predicted conflicts drop under 8 %
    monkeypatch.setenv("PCGS_REPLICAS", "1")
    rc, msg, st = _selftest(n, p, rp, ci, True, 0)
    assert rc == 0, msg
    assert st[6] / st[5] < 0.08
    rng = np.random.default_rng(12)
    for _ in range(6):
        n, p = (int(v) for v in rng.integers(20, 600, size=2))
        rp, ci = random_pattern(rng, n, p, float(rng.uniform(0.05, 0.7)))
        for grid, sm in ((3, 0), (148, 0), (148, 64)):
            rc, msg, _ = _selftest(n, p, rp, ci, True, sm, grid)
            assert rc == 0, msg


def test_store_roundtrip_with_32_ranges_per_task():
    """Debug option 3 sets the warp ranges per CTA task of the stores built
    from then on (the row-split shards use 32, the default is 16)."""
    L = _lib.lib()
    rng = np.random.default_rng(21)
    try:
        for ranges in (32, 8, 1):
            L.pcgs_debug_option(3, ranges)
            for _ in range(4):
                n, p = (int(v) for v in rng.integers(1, 500, size=2))
                rp, ci = random_pattern(rng, n, p, float(rng.uniform(0, 0.6)))
                for grid, sm in ((2, 0), (148, 0), (148, 32)):
                    rc, msg, _ = _selftest(n, p, rp, ci, True, sm, grid)
                    assert rc == 0, msg
        L.pcgs_debug_option(3, 33)
        rc, msg, _ = _selftest(3, 3, np.array([0, 1, 2, 3]), np.array([0, 1, 2], dtype=np.int32), True, 0)
        assert rc == _lib.PCGS_EINVAL
    finally:
        L.pcgs_debug_option(3, 0)


def test_store_roundtrip_more_grids():
    rng = np.random.default_rng(11)
    for _ in range(10):
        n, p = (int(v) for v in rng.integers(1, 600, size=2))
        rp, ci = random_pattern(rng, n, p, float(rng.uniform(0, 0.7)))
        for grid, sm in ((1, 0), (5, 40), (148, 0), (148, 24)):
            rc, msg, _ = _selftest(n, p, rp, ci, True, sm, grid)
            assert rc == 0, msg


# ------------------------------------------------------------ sliced (batched) store
def _bselftest(n, p, rp, ci, intercept, R, slab_max=0, grid=148):
    L = _lib.lib()
    st = np.zeros(9, dtype=np.int64)
    rp = np.ascontiguousarray(rp, dtype=np.int64)
    ci = np.ascontiguousarray(ci, dtype=np.int32)
    rc = L.pcgs_batch_selftest(n, p, rp.ctypes.data, ci.ctypes.data, int(intercept), R, slab_max, grid,
                               st.ctypes.data)
    return rc, L.pcgs_last_error().decode(), st


@pytest.mark.parametrize("R", [2, 4, 8])
@pytest.mark.parametrize("slab_max", [0, 16, 48])
def test_sliced_store_roundtrip_random(R, slab_max):
    """The sliced store (csrc/sliced.h) walks every CSR entry exactly once in
    both passes, for random patterns, multi-slab cuts and grids of 1..148."""
    rng = np.random.default_rng(10 * R + slab_max)
    for _ in range(8):
        n, p = (int(v) for v in rng.integers(1, 300, size=2))
        rp, ci = random_pattern(rng, n, p, float(rng.uniform(0, 0.6)))
        for icpt in (True, False):
            for grid in (1, 5, 148):
                rc, msg, _ = _bselftest(n, p, rp, ci, icpt, R, slab_max, grid)
                assert rc == 0, msg


def test_sliced_store_edge_cases_and_validation():
    cases = [
        (5, 4, np.zeros(6, dtype=np.int64), np.zeros(0, dtype=np.int32)),
        (1, 3, np.array([0, 2]), np.array([0, 2], dtype=np.int32)),
        (3, 2000, np.array([0, 2000, 2000, 2001]),
         np.concatenate([np.arange(2000), [1999]]).astype(np.int32)),
    ]
    for n, p, rp, ci in cases:
        for R in (2, 8):
            for icpt in (True, False):
                rc, msg, _ = _bselftest(n, p, rp, ci, icpt, R)
                assert rc == 0, msg
    rc, _, _ = _bselftest(1, 3, np.array([0, 2]), np.array([1, 1], dtype=np.int32), True, 8)
    assert rc == _lib.PCGS_EINVAL
    rc, _, _ = _bselftest(1, 3, np.array([0, 1]), np.array([0], dtype=np.int32), True, 3)
    assert rc == _lib.PCGS_EINVAL          # batch size must be 2, 4 or 8


def test_sliced_store_config1_bank_balance_and_padding():
    # short pieces (config 1: ~10 entries per row) leave the builder few
    # choices when many slots share a half-warp (R = 2: 8 slots per half)
    d = synth.config_design(1, seed=0)
    for R, cap in ((2, 0.5), (4, 0.25), (8, 0.12)):
        rc, msg, st = _bselftest(d.n, d.p, d.row_ptr, d.col_idx, True, R)
        assert rc == 0, msg
        vectors = st[2] + st[3]
        assert st[7] / st[6] < cap          # extra shared-memory wavefronts per half-warp load
        assert st[8] / vectors < 0.15       # slot padding (sentinel vectors) < 15 % of the stream
