"""Row-sharded Phi on CPU with world_size 2 over gloo: the partition, the
per-rank local operator, the allreduce composition and a PCG solve through it
(the device local passes are replaced by the oracle in this CPU test)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import port
from paper_1810_12437_b200 import parallel, synth


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_local_apply(shard, omega, diag, v):
    rp, ci, icpt = shard.pattern()
    Xo = port.design_from_pattern(shard.n_rows, shard.n_cols - int(icpt), rp, ci, intercept=icpt)
    return port.phi_apply(Xo, omega, diag, v)


def _worker(rank, world, port_, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        d = synth.binary_design(900, 120, 2e-3, 0.3, seed=3)
        X = d.matrix()
        rng = np.random.default_rng(0)
        om = rng.uniform(0.05, 0.4, d.n)
        lam = np.abs(rng.standard_cauchy(d.p)) + 0.1
        diag = np.concatenate([[0.0], (0.2 * lam) ** -2.0])
        minv = np.concatenate([[100.0], (0.2 * lam) ** 2])
        v = rng.standard_normal(d.p + 1)
        b = rng.standard_normal(d.p + 1)
        parts = parallel.row_partition(d.row_ptr, world)
        lo, hi = parts[rank]
        shard = parallel.local_rows(X, lo, hi)
        op = parallel.ShardedPrecisionOperator([shard], [om[lo:hi]], diag, rank=rank,
                                               group=dist.group.WORLD, local_apply=_oracle_local_apply)
        phiv = op.apply(v)
        res = port.pcg(op.apply, b, minv, np.sqrt(minv), rtol=1e-10)
        q.put((rank, parts, phiv, res.x, res.iterations))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_row_sharded_phi_and_pcg_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_ = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port_, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort(key=lambda t: t[0])
    d = synth.binary_design(900, 120, 2e-3, 0.3, seed=3)
    Xo = port.design_from_pattern(d.n, d.p, d.row_ptr, d.col_idx)
    rng = np.random.default_rng(0)
    om = rng.uniform(0.05, 0.4, d.n)
    lam = np.abs(rng.standard_cauchy(d.p)) + 0.1
    diag = np.concatenate([[0.0], (0.2 * lam) ** -2.0])
    minv = np.concatenate([[100.0], (0.2 * lam) ** 2])
    v = rng.standard_normal(d.p + 1)
    b = rng.standard_normal(d.p + 1)
    full = port.phi_apply(Xo, om, diag, v)
    parts = out[0][1]
    assert parts[0][0] == 0 and parts[-1][1] == d.n
    assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))
    for _, _, phiv, _, _ in out:
        np.testing.assert_allclose(phiv, full, rtol=1e-12, atol=1e-12)
    # replicated vector algebra: every rank holds the same solution
    np.testing.assert_array_equal(out[0][3], out[1][3])
    ref = port.pcg(lambda x: port.phi_apply(Xo, om, diag, x), b, minv, np.sqrt(minv), rtol=1e-10)
    assert np.linalg.norm(out[0][3] - ref.x) / np.linalg.norm(ref.x) < 1e-8
    assert abs(out[0][4] - ref.iterations) <= 2


def test_row_partition_balance():
    d = synth.config_design(1, seed=0)
    for world in (1, 2, 3, 8):
        parts = parallel.row_partition(d.row_ptr, world)
        assert parts[0][0] == 0 and parts[-1][1] == d.n
        loads = [d.row_ptr[h] - d.row_ptr[l] + (h - l) for l, h in parts]
        assert max(loads) - min(loads) <= 2 * (np.diff(d.row_ptr).max() + 1)


def test_local_rows_reassemble():
    d = synth.config_design(1, seed=0)
    X = d.matrix()
    rows = []
    for lo, hi in parallel.row_partition(d.row_ptr, 3):
        sh = parallel.local_rows(X, lo, hi)
        rp, ci, icpt = sh.pattern()
        assert icpt and sh.n_rows == hi - lo
        rows.extend(np.split(ci, rp[1:-1]))
    ref = np.split(d.col_idx, d.row_ptr[1:-1])
    assert len(rows) == len(ref) and all(np.array_equal(a, b) for a, b in zip(rows, ref))


class _FakeRsLib:
    """Stands in for libpcgs in the IPC handle exchange: rank r's handle is 64
    bytes of r; records which peer handles a rank maps."""

    def __init__(self, rank):
        self.rank, self.opened = rank, {}

    def pcgs_rs_exchange_handle(self, h, local, buf):
        import ctypes
        ctypes.memmove(buf, bytes([self.rank]) * 64, 64)
        return 0

    def pcgs_rs_open_peer(self, h, q, buf):
        self.opened[q] = bytes(buf.raw[:64])
        return 0


def _ipc_worker(rank, world, port_, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        L = _FakeRsLib(rank)
        allh = parallel.exchange_ipc_handles(L, None, dist.group.WORLD)
        q.put((rank, [h[0] for h in allh], {k: v[0] for k, v in L.opened.items()}))
    finally:
        dist.destroy_process_group()


def test_row_split_ipc_handle_exchange_gloo():
    """The multi-process plumbing of the fused row split (one rank per GPU):
    every rank maps exactly the other ranks' exchange regions, by rank."""
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.start_processes(_ipc_worker, args=(world, _free_port(), q), nprocs=world, join=True, start_method="spawn")
    got = sorted(q.get() for _ in range(world))
    for rank, handles, opened in got:
        assert handles == list(range(world))
        assert opened == {p: p for p in range(world) if p != rank}
