"""Chain sharding for BASELINE config 4 on CPU (gloo, world size 2): every
chain runs exactly once on exactly one rank with a rank-independent seed, and
the end-of-run gather returns identical, index-ordered outputs everywhere."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1810_12437_b200 import parallel


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _fake_runner(X, y, cfg, n_iter, seed=0, **kw):
    rng = np.random.default_rng(seed)
    return {"seed": seed, "draw": rng.standard_normal(3), "rank": dist.get_rank(), "kw": sorted(kw)}


def _fake_batched(X, y, cfg, n_iter, seeds, **kw):
    """Stands in for gibbs.gibbs_run_batched (device path) in the gloo test:
    records each batch's seeds, a chain's output depends on its seed only."""
    assert len(seeds) in (2, 4, 8)
    return [{"seed": s, "draw": np.random.default_rng(s).standard_normal(3), "rank": dist.get_rank(),
             "batch": list(seeds), "kw": sorted(kw)} for s in seeds]


def _batched_worker(rank, world, port_, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1810_12437_b200 import gibbs
        gibbs.gibbs_run_batched = _fake_batched
        outs = parallel.run_chains(None, None, None, 5, n_chains=11, seed=3, burn_in=1)
        q.put((rank, [(o["seed"], o["rank"], o["draw"].tolist(), o["batch"], o["kw"]) for o in outs]))
    finally:
        dist.destroy_process_group()


def _worker(rank, world, port_, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        outs = parallel.run_chains(None, None, None, 5, n_chains=7, seed=11, runner=_fake_runner, thin=2)
        own = parallel.run_chains(None, None, None, 5, n_chains=7, seed=11, runner=_fake_runner, gather=False)
        q.put((rank, [(o["seed"], o["rank"], o["draw"].tolist(), o["kw"]) for o in outs], sorted(own)))
    finally:
        dist.destroy_process_group()


def test_chain_assignment_partitions():
    for n in range(0, 20):
        for w in range(1, 6):
            got = [c for r in range(w) for c in parallel.chain_assignment(n, w, r)]
            assert got == list(range(n))
            sizes = [len(parallel.chain_assignment(n, w, r)) for r in range(w)]
            assert max(sizes) - min(sizes) <= (1 if n else 0)
    with pytest.raises(ValueError):
        parallel.chain_assignment(4, 2, 2)


def test_chain_seeds_distinct_and_stable():
    seeds = [parallel.chain_seed(3, c) for c in range(64)]
    assert len(set(seeds)) == 64 and all(0 <= s < 2 ** 64 for s in seeds)
    assert seeds == [parallel.chain_seed(3, c) for c in range(64)]
    assert parallel.chain_seed(4, 0) != seeds[0]


def test_two_ranks_gather_all_chains():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_ = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port_, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict((r, (o, own)) for r, o, own in (q.get(timeout=120) for _ in range(world)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    a, b = res[0][0], res[1][0]
    assert a == b and len(a) == 7
    assert [s for s, *_ in a] == [parallel.chain_seed(11, c) for c in range(7)]
    assert [r for _, r, *_ in a] == [0, 0, 0, 0, 1, 1, 1]
    assert all(kw == ["thin"] for *_, kw in a)
    assert res[0][1] == [0, 1, 2, 3] and res[1][1] == [4, 5, 6]


def test_two_ranks_batched_chains_padded_to_full_batches():
    """run_chains' default batched path over gloo world size 2: 11 chains ->
    6 + 5 per rank, each rank's block in batches of 8 padded with extra seeds
    (chain_seed(seed, n_chains + k)), outputs of the padding dropped; every
    rank returns all 11 chains in order, identical on both ranks."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_ = _free_port()
    procs = [ctx.Process(target=_batched_worker, args=(r, world, port_, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict((r, o) for r, o in (q.get(timeout=120) for _ in range(world)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    a, b = res[0], res[1]
    assert a == b and len(a) == 11
    assert [s for s, *_ in a] == [parallel.chain_seed(3, c) for c in range(11)]
    assert [r for _, r, *_ in a] == [0] * 6 + [1] * 5
    pad0 = [parallel.chain_seed(3, 11 + k) for k in range(2)]
    pad1 = [parallel.chain_seed(3, 11 + k) for k in range(3)]
    assert a[0][3] == [parallel.chain_seed(3, c) for c in range(6)] + pad0
    assert a[6][3] == [parallel.chain_seed(3, c) for c in range(6, 11)] + pad1
    assert all(kw == ["burn_in"] for *_, kw in a)
