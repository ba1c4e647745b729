"""Row-sharded Phi across GPUs (BASELINE config 5).

The rows of X are split into contiguous, nnz-balanced shards, one per rank
(one process per GPU, `torch.distributed` with NCCL over NVLink).  p-length
vectors are replicated; per Phi-apply every rank runs its local pattern-only
passes (X_g' Omega_g X_g v, libpcgs) and one allreduce(sum) of the p-length
partial combines them; the prior term D v is contributed by rank 0 only, so
the allreduce result is Phi v on every rank, bitwise identical (one NCCL
algorithm, the same inputs everywhere).  The PCG vector algebra then runs
replicated on every rank in the device PCG engine (`pcgs_pcg_op`), with the
operator supplied as a device-side callback - no host copies of vectors.

A single process can also hold several shards of one device
(`EmulatedGroup`): the allreduce becomes a fixed-order local sum, which is how
the decomposition is validated on one GPU.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .cg import CGReport, _metric_scale, _n_betas, _raise_status
from .sparse import SparseDesignMatrix


def row_partition(row_ptr, world, intercept=True):
    """Contiguous row ranges [lo, hi) balanced by stored entries per rank."""
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    n = len(row_ptr) - 1
    weight = row_ptr + (np.arange(n + 1, dtype=np.int64) if intercept else 0)
    total = int(weight[-1])
    cuts = [0]
    for r in range(1, world):
        target = total * r / world
        c = int(np.searchsorted(weight, target))
        cuts.append(min(max(c, cuts[-1]), n))
    cuts.append(n)
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def local_rows(X: SparseDesignMatrix, lo, hi) -> SparseDesignMatrix:
    """The row block [lo, hi) of a design as its own pattern-only design."""
    if X.affine:
        raise NotImplementedError("row split: designs with a dense block or standardisation are not sharded")
    rp, ci, icpt = X.pattern()
    sub_rp = rp[lo:hi + 1] - rp[lo]
    sub_ci = ci[rp[lo]:rp[hi]]
    p = X.n_cols - (1 if icpt else 0)
    return SparseDesignMatrix.from_pattern(hi - lo, p, sub_rp, sub_ci, intercept=icpt, check=False)


class EmulatedGroup:
    """Stand-in for a process group when all shards live in one process."""

    size = 1


class ShardedPrecisionOperator:
    """Phi = sum_g X_g' Omega_g X_g + D over row shards (this rank's shards
    plus an allreduce over `group`)."""

    def __init__(self, shards, omegas, prior_precision_diag, rank=0, group=None, device=None,
                 local_apply=None):
        t = _lib.torch()
        self.shards = list(shards)
        self.rank = rank
        self.group = group
        self.local_apply = local_apply
        if local_apply is None:
            self.device = _lib.cuda_device(device)
            self.stores = [s.device_store(self.device) for s in self.shards]
            self.omegas = [_lib.to_device(o, self.device) for o in omegas]
            self.diag = _lib.to_device(prior_precision_diag, self.device)
            self.zero = t.zeros_like(self.diag)
            self.tmp = t.empty_like(self.diag)
        else:
            self.device = None
            self.omegas = list(omegas)
            self.diag = prior_precision_diag
        self.prior_precision_diag = np.asarray(
            prior_precision_diag.cpu().numpy() if _lib.is_tensor(prior_precision_diag)
            else prior_precision_diag, dtype=np.float64)
        self.dim = len(self.prior_precision_diag)
        self.apply_count = 0

    def apply_into(self, v, out):
        """out = Phi v on device tensors (all ranks receive the same result)."""
        self.apply_count += 1
        for g, (st, om) in enumerate(zip(self.stores, self.omegas)):
            d = self.diag if (self.rank == 0 and g == 0) else self.zero
            if g == 0:
                st.phi_apply(om, d, v, out)
            else:
                st.phi_apply(om, d, v, self.tmp)
                out.add_(self.tmp)          # emulated allreduce: fixed shard order
        self._allreduce(out)
        return out

    def _allreduce(self, out):
        if self.group is not None and not isinstance(self.group, EmulatedGroup):
            import torch.distributed as dist
            dist.all_reduce(out, op=dist.ReduceOp.SUM, group=self.group)

    def apply(self, v):
        """numpy / tensor apply (for `pcg_solve`'s generic path and the tests)."""
        if self.local_apply is not None:
            self.apply_count += 1
            out = None
            for g, (sh, om) in enumerate(zip(self.shards, self.omegas)):
                d = self.diag if (self.rank == 0 and g == 0) else np.zeros_like(self.diag)
                y = self.local_apply(sh, om, d, v)
                out = y if out is None else out + y
            if self.group is not None:
                import torch
                import torch.distributed as dist
                tt = torch.from_numpy(np.ascontiguousarray(out))
                dist.all_reduce(tt, op=dist.ReduceOp.SUM, group=self.group)
                out = tt.numpy()
            return out
        t = _lib.torch()
        as_tensor = _lib.is_tensor(v)
        vd = _lib.to_device(v, self.device)
        out = t.empty_like(vd)
        self.apply_into(vd, out)
        return out if as_tensor else out.cpu().numpy()


def sharded_pcg_solve(op: ShardedPrecisionOperator, b, M, x0=None, config=None, residual_scale=None,
                      fused=None):
    """pcg_solve (cg.py:105-192) over a row-sharded operator.

    Device shards default to the fused row-split kernel (`fused_pcg_solve`:
    one persistent kernel per GPU, exchange over peer memory).  `fused=False`
    (and host shards, `local_apply`) runs the engine loop instead: device
    vector algebra replicated on every rank, Phi applied through the device
    callback with one allreduce per application."""
    if fused is None:
        fused = op.local_apply is None and (config is None or config.trace_level != "full")
    if fused:
        return fused_pcg_solve(op, b, M, x0=x0, config=config, residual_scale=residual_scale)
    from .cg import CGConfig
    t = _lib.torch()
    L = _lib.lib()
    cfg = config if config is not None else CGConfig()
    p = int(b.shape[0])
    max_iter = cfg.max_iter if cfg.max_iter is not None else 2 * p
    scale = _metric_scale(op, M, residual_scale, p)
    dev = op.device
    bd = _lib.to_device(b, dev)
    x = t.zeros(p, dtype=t.float64, device=dev) if x0 is None else _lib.to_device(x0, dev).clone()
    md = _lib.to_device(np.asarray(M.inv_diagonal, dtype=np.float64), dev)
    sd = _lib.to_device(scale, dev)
    dbuf = t.empty(p, dtype=t.float64, device=dev)
    adbuf = t.empty(p, dtype=t.float64, device=dev)
    errors = []
    xptr = _lib.ptr(x)

    def cb(ctx, vptr, outptr):
        try:
            src = x if vptr == xptr else dbuf   # the first application is on x0 (cg.py:137)
            op.apply_into(src, adbuf)
            return 0
        except BaseException as exc:
            errors.append(exc)
            return 1

    fn = _lib.APPLY_FN(cb)
    trace = np.zeros(max_iter + 1)
    alphas = np.zeros(max_iter)
    betas = np.zeros(max_iter)
    result = np.zeros(4, dtype=np.int32)
    t.cuda.synchronize(dev)
    rc = L.pcgs_pcg_op(fn, None, p, _lib.ptr(md), _lib.ptr(sd), _lib.ptr(bd), _lib.ptr(x),
                       _lib.ptr(dbuf), _lib.ptr(adbuf), max_iter, float(cfg.rtol), trace.ctypes.data,
                       alphas.ctypes.data, betas.ctypes.data, result.ctypes.data,
                       _lib.stream_ptr(dev))
    if errors:
        raise errors[0]
    _lib.check(rc)
    iterations, status, fail_iter, applies = (int(v) for v in result)
    _raise_status(status, fail_iter)
    return CGReport(
        iterations=iterations,
        termination="converged" if status == _lib.PCGS_CONVERGED else "max_iter",
        rms_precond_residual_trace=trace[: iterations + 1].copy(),
        solution=x if _lib.is_tensor(b) else x.cpu().numpy(),
        matvec_count=applies,
        alphas=alphas[:iterations].copy(),
        betas=betas[:_n_betas(iterations, status)].copy(),
        iterates=None,
    )


# ---------------------------------------------------------------------------
# Fused row-split PCG: one persistent kernel per GPU, the X'w exchange over
# peer memory inside it (libpcgs pcgs_rs_*, csrc/rowsplit.cu)
# ---------------------------------------------------------------------------
def exchange_ipc_handles(L, h, group):
    """Share every rank's exchange region: all-gather the 64-byte CUDA IPC
    handles (one object collective at setup) and map every other rank's
    region (pcgs_rs_open_peer); a barrier makes sure every rank has mapped its
    peers before any kernel can signal them.  `L` is the library binding."""
    import torch.distributed as dist
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    mine = ctypes.create_string_buffer(64)
    _lib.check(L.pcgs_rs_exchange_handle(h, 0, mine))
    allh = [None] * world
    dist.all_gather_object(allh, bytes(mine.raw), group=group)
    for q, hb in enumerate(allh):
        if q != rank:
            _lib.check(L.pcgs_rs_open_peer(h, q, ctypes.create_string_buffer(hb, 64)))
    dist.barrier(group=group)
    return allh


class RowSplitPCG:
    """The whole row-split solve in one kernel per GPU.

    * Single process, several shards (`group` None or EmulatedGroup): every
      shard is a rank group of SMs/G CTAs in one cooperative grid; the
      exchange barrier is the grid barrier (the single-GPU form).
    * One shard per process over a torch.distributed `group` (one GPU per
      rank): each rank's exchange region is shared with CUDA IPC (handles
      all-gathered once) and the kernel's exchange barrier is a flag
      handshake over peer memory.
    Bitwise identical results on every rank; no collective per iteration.

    `exchange="flags"` (single process only) runs the cross-GPU protocol
    between the hosted groups inside the one cooperative grid: each group
    synchronises only its own CTAs and meets the others through inbox flags
    and peer loads (pcgs_rs_set_exchange), so the multi-GPU code path runs and
    is checked on one GPU.
    """

    def __init__(self, shards, device=None, group=None, exchange="grid"):
        t = _lib.torch()
        L = _lib.lib()
        self.device = _lib.cuda_device(device)
        self.shards = list(shards)
        real = group is not None and not isinstance(group, EmulatedGroup)
        if real:
            import torch.distributed as dist
            world, rank = dist.get_world_size(group), dist.get_rank(group)
        else:
            world, rank = 1, 0
        if real and world > 1 and len(self.shards) != 1:
            raise ValueError("row split over processes: one shard per rank")
        n_local = len(self.shards)
        nranks = world * n_local if real else n_local
        sms = t.cuda.get_device_properties(self.device).multi_processor_count
        grid = 0 if n_local == 1 else sms // n_local
        self.stores = [s.device_store(self.device, grid=grid, ranges=32) for s in self.shards]
        p_total = {st.p_total for st in self.stores}
        if len(p_total) != 1:
            raise ValueError("row shards must share the column set")
        self.p_total = p_total.pop()
        handles = (ctypes.c_void_p * n_local)(*[st.handle.value for st in self.stores])
        h = ctypes.c_void_p()
        _lib.check(L.pcgs_rs_create(handles, n_local, rank * n_local if real else 0, nranks, ctypes.byref(h)))
        self._h = h
        if exchange not in ("grid", "flags"):
            raise ValueError("exchange must be 'grid' or 'flags'")
        if exchange == "flags":
            if real:
                raise ValueError("exchange='flags' is the single-process validation mode")
            _lib.check(L.pcgs_rs_set_exchange(h, 1))
        if real and world > 1:
            exchange_ipc_handles(L, h, group)
        self.n_local, self.nranks = n_local, nranks

    def solve(self, omegas, prior_diag, minv, scale, b, x0=None, max_iter=None, rtol=1e-6):
        """Device tensors in (omegas: one per local shard); returns (x, trace,
        alphas, betas, result) tensors, nothing synchronised (pcg_solve_device)."""
        t = _lib.torch()
        dev = self.device
        p = self.p_total
        max_iter = 2 * p if max_iter is None else int(max_iter)
        x = (t.zeros(p, dtype=t.float64, device=dev) if x0 is None
             else x0.to(device=dev, dtype=t.float64).clone())
        trace = t.empty(max_iter + 1, dtype=t.float64, device=dev)
        alphas = t.empty(max_iter, dtype=t.float64, device=dev)
        betas = t.empty(max_iter, dtype=t.float64, device=dev)
        result = t.zeros(4, dtype=t.int32, device=dev)
        om = [_lib.to_device(o, dev) for o in omegas]
        optrs = (ctypes.c_void_p * len(om))(*[_lib.ptr(o) for o in om])
        args = [_lib.to_device(v, dev) for v in (prior_diag, minv, scale, b)]
        _lib.check(_lib.lib().pcgs_rs_pcg(self._h, optrs, *[_lib.ptr(a) for a in args], _lib.ptr(x),
                                          max_iter, float(rtol), _lib.ptr(trace), _lib.ptr(alphas),
                                          _lib.ptr(betas), _lib.ptr(result), _lib.stream_ptr(dev)))
        self._keep = (om, args)  # alive until the next call (the launch is asynchronous)
        return x, trace, alphas, betas, result

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _lib.lib().pcgs_rs_destroy(h)
            except Exception:  # pragma: no cover - interpreter shutdown
                pass
            self._h = None


def fused_pcg_solve(op: "ShardedPrecisionOperator", b, M, x0=None, config=None, residual_scale=None,
                    exchange="grid"):
    """pcg_solve (cg.py:105-192) over a row-sharded operator with the fused
    row-split kernel; same report and exceptions as `sharded_pcg_solve`."""
    from .cg import CGConfig, _report_from_device
    cfg = config if config is not None else CGConfig()
    if op.local_apply is not None:
        raise ValueError("the fused row split needs device shards")
    solver = getattr(op, "_rowsplit", None)
    if solver is None or getattr(op, "_rowsplit_exchange", "grid") != exchange:
        solver = op._rowsplit = RowSplitPCG(op.shards, device=op.device, group=op.group, exchange=exchange)
        op._rowsplit_exchange = exchange
    p = int(np.asarray(b).shape[0]) if not _lib.is_tensor(b) else int(b.shape[0])
    scale = _metric_scale(op, M, residual_scale, p)
    # the prior term is added once by every rank in the column step (replicated)
    out = solver.solve(op.omegas, op.diag, np.asarray(M.inv_diagonal, dtype=np.float64), scale, b,
                       x0=None if x0 is None else _lib.to_device(x0, op.device),
                       max_iter=cfg.max_iter, rtol=cfg.rtol)
    rep = _report_from_device(*out, as_tensor=_lib.is_tensor(b))
    op.apply_count += rep.matvec_count
    return rep


# ---------------------------------------------------------------------------
# Row-split Gibbs scan (BASELINE config 5): gibbs_run with X's rows over ranks
# ---------------------------------------------------------------------------
class _RsRows(ctypes.Structure):
    """Mirror of pcgs_rs_rows_t (include/pcgs.h)."""
    _fields_ = [("y", ctypes.c_void_p), ("kappa", ctypes.c_void_p), ("z", ctypes.c_void_p),
                ("omega", ctypes.c_void_p), ("part", ctypes.c_void_p)]


def _row_split_chain_class():
    from .gibbs import DeviceChain, _GibbsArgs, _PART_STRIDE

    class RowSplitChain(DeviceChain):
        """DeviceChain whose scans run over row shards (`RowSplitPCG` context):
        replicated p-state, full-length row vectors of which each hosted rank
        owns its contiguous range."""

        def __init__(self, X, y, cfg, n_iter, parts, hosted, group=None, device=None, exchange="grid", **kw):
            self._parts, self._hosted, self._group = parts, hosted, group
            self._exchange = exchange
            super().__init__(X, y, cfg, n_iter, device=device, **kw)

        def _open_device(self, X, device):
            if X.affine:
                raise NotImplementedError("row split: designs with a dense block or standardisation are "
                                          "not sharded")
            shards = [local_rows(X, *self._parts[r]) for r in self._hosted]
            self.rs = RowSplitPCG(shards, device=device, group=self._group, exchange=self._exchange)
            self.store = None
            self.dev = self.rs.device
            self.grid = self.rs.stores[0].describe()["grid"]

        def _init_device(self):
            t = _lib.torch()
            L = _lib.lib()
            P = _lib.ptr
            self._parts_buf = [t.zeros(_PART_STRIDE * (self.grid + 1), dtype=t.float64, device=self.dev)
                               for _ in self._hosted]
            rows = (_RsRows * len(self._hosted))()
            for k, r in enumerate(self._hosted):
                lo, _ = self._parts[r]
                off = 8 * lo
                rows[k] = _RsRows(P(self.y) + off, P(self.kappa) + off, P(self.z) + off, P(self.omega) + off,
                                  P(self._parts_buf[k]))
            self._rows = rows
            L.pcgs_rs_gibbs_init.argtypes = [ctypes.c_void_p, ctypes.POINTER(_GibbsArgs), ctypes.c_void_p,
                                             ctypes.c_void_p]
            L.pcgs_rs_gibbs_scan.argtypes = [ctypes.c_void_p, ctypes.POINTER(_GibbsArgs), ctypes.c_void_p,
                                             ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p]
            _lib.check(L.pcgs_rs_gibbs_init(self.rs._h, ctypes.byref(self.args), ctypes.addressof(rows),
                                            _lib.stream_ptr(self.dev)))

        def scan(self, t, local_scale_sampler=None, rng=None):
            if local_scale_sampler is not None:
                raise NotImplementedError("row split: local_scale_sampler is not sharded")
            slot = -1
            if t > self.burn_in and (t - self.burn_in - 1) % self.thin == 0:
                slot = self.stored
                self.stored += 1
            _lib.check(_lib.lib().pcgs_rs_gibbs_scan(self.rs._h, ctypes.byref(self.args),
                                                     ctypes.addressof(self._rows), int(t), int(self.count),
                                                     int(slot), _lib.stream_ptr(self.dev)))
            self.count += 1

        def output(self):
            out = super().output()
            real = self._group is not None and not isinstance(self._group, EmulatedGroup)
            if real:
                # every rank holds only its own rows of omega: gather them
                import torch.distributed as dist
                lo, hi = self._parts[self._hosted[0]]
                mine = self.omega[lo:hi].cpu().numpy()
                allp = [None] * dist.get_world_size(self._group)
                dist.all_gather_object(allp, mine, group=self._group)
                out.final_state.omega[:] = np.concatenate(allp)
            return out

    return RowSplitChain


def row_split_gibbs_run(X, y, cfg, n_iter, shards=None, group=None, burn_in=0, seed=0, thin=1,
                        preconditioner="prior", cg_config=None, init_state=None, gamma_scale=1.0,
                        allow_max_iter=False, fixed_omega=None, fixed_tau=None, fixed_lam=None,
                        device=None, sync_every=64, exchange="grid"):
    """gibbs_run (gibbs.py:260-379) with the rows of X split over ranks.

    With a torch.distributed `group` of W processes (one GPU each) rank r
    holds row shard r of an nnz-balanced partition; without one, `shards`
    row shards (default 2) are hosted by one process on one GPU.  Same
    output as gibbs_run on every rank: replicated state, the draws of omega
    and of the RHS noise keyed by global row (the unsharded chain's keys; only
    summation order differs).  Prior or identity preconditioning; no
    local_scale_sampler and no standardised designs on this path.
    `exchange="flags"`: single-process validation of the cross-GPU exchange
    protocol (RowSplitPCG)."""
    from .gibbs import GibbsAbortError, _PRECOND  # noqa: F401
    y = np.asarray(y, dtype=np.float64)
    if y.shape != (X.n_rows,) or not np.all((y == 0.0) | (y == 1.0)):
        raise ValueError("outcomes must be 0/1, one per design row")
    if n_iter < 0 or burn_in < 0 or burn_in > n_iter or thin < 1:
        raise ValueError("need 0 <= burn_in <= n_iter and thin >= 1")
    if preconditioner not in ("prior", "identity"):
        raise NotImplementedError("row split: prior or identity preconditioning")
    real = group is not None and not isinstance(group, EmulatedGroup)
    rp, _, icpt = X.pattern()
    if real:
        import torch.distributed as dist
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        parts = row_partition(rp, world, intercept=icpt)
        hosted = [rank]
    else:
        nsh = int(shards or 2)
        parts = row_partition(rp, nsh, intercept=icpt)
        hosted = list(range(nsh))
    Chain = _row_split_chain_class()
    ch = Chain(X, y, cfg, n_iter, parts, hosted, group=group, device=device, exchange=exchange,
               burn_in=burn_in, thin=thin,
               seed=seed, preconditioner=preconditioner, cg_config=cg_config, init_state=init_state,
               gamma_scale=gamma_scale, fixed_omega=fixed_omega, fixed_tau=fixed_tau, fixed_lam=fixed_lam)
    checked = 0
    for t in range(1, n_iter + 1):
        ch.scan(t)
        if sync_every and t - checked >= sync_every:
            ch.check(checked + 1, t, allow_max_iter)
            checked = t
    if checked < n_iter:
        ch.check(checked + 1, n_iter, allow_max_iter)
    return ch.output()


# ---------------------------------------------------------------------------
# Independent chains across ranks (BASELINE config 4)
# ---------------------------------------------------------------------------
def chain_seed(seed, chain) -> int:
    """Per-chain seed derived from (seed, chain index): distinct, reproducible
    and independent of how chains are spread over ranks."""
    state = np.random.SeedSequence([int(seed) & (2 ** 63 - 1), int(chain)]).generate_state(2, dtype=np.uint32)
    return int(state[0]) | (int(state[1]) << 32)


def chain_assignment(n_chains, world, rank):
    """Contiguous block of chain indices run by `rank` (sizes differ by ≤ 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("need 0 <= rank < world")
    base, extra = divmod(int(n_chains), int(world))
    lo = rank * base + min(rank, extra)
    return list(range(lo, lo + base + (1 if rank < extra else 0)))


def run_chains(X, y, cfg, n_iter, n_chains, seed=0, group=None, gather=True, runner=None, concurrent=None,
               batch=None, **kwargs):
    """Run `n_chains` independent Gibbs chains, sharded over the ranks of
    `group` (default: the initialised torch.distributed world, else one
    process).  Chain c uses `chain_seed(seed, c)`.  How a rank runs its
    block of chains:

    * default: in batches of `batch` = 8 chains whose beta solves share one
      batched PCG per scan (`gibbs.gibbs_run_batched`; BASELINE config 4's
      8 chains per GPU); a short last batch is padded with extra chains
      (seeds beyond n_chains, outputs dropped) so every chain runs in a batch
      of the same size and its trajectory depends on its seed only, never on
      the world size;
    * `concurrent` = k > 1: k slots side by side (one CUDA stream each, the
      store planned for SMs // k CTAs; `gibbs.gibbs_run_concurrent`);
    * `concurrent=1`, a custom `runner`, or host hooks (local_scale_sampler,
      on_progress): one after another through gibbs_run.

    There is no collective while sampling; with `gather` the outputs are
    all-gathered at the end (object collective) and every rank returns all
    chains in index order, otherwise only its own (as {chain: ChainOutput})."""
    import torch.distributed as dist
    if group is None and dist.is_available() and dist.is_initialized():
        group = dist.group.WORLD
    world = dist.get_world_size(group) if group is not None else 1
    rank = dist.get_rank(group) if group is not None else 0
    block = chain_assignment(n_chains, world, rank)
    host_hooks = kwargs.get("local_scale_sampler") is not None or kwargs.get("on_progress") is not None
    if batch is None and concurrent is None and runner is None and not host_hooks:
        batch = 8
    if batch:
        from .gibbs import gibbs_run_batched
        if batch not in (2, 4, 8):
            raise ValueError("batch must be 2, 4 or 8")
        seeds = [chain_seed(seed, c) for c in block]
        outs = []
        for i in range(0, len(seeds), batch):
            grp = seeds[i:i + batch]
            pad = [chain_seed(seed, n_chains + k) for k in range(batch - len(grp))]
            outs += gibbs_run_batched(X, y, cfg, n_iter, grp + pad, **kwargs)[:len(grp)]
        mine = dict(zip(block, outs))
    elif concurrent is not None and concurrent > 1 and runner is None and not host_hooks:
        from .gibbs import gibbs_run_concurrent
        kw = {k: v for k, v in kwargs.items() if k != "sync_every"}
        outs = gibbs_run_concurrent(X, y, cfg, n_iter, [chain_seed(seed, c) for c in block],
                                    concurrent=concurrent, **kw)
        mine = dict(zip(block, outs))
    else:
        if runner is None:
            from .gibbs import gibbs_run as runner
        mine = {c: runner(X, y, cfg, n_iter, seed=chain_seed(seed, c), **kwargs) for c in block}
    if not gather:
        return mine
    if world > 1:
        parts = [None] * world
        dist.all_gather_object(parts, mine, group=group)
        merged = {}
        for part in parts:
            merged.update(part)
        mine = merged
    return [mine[c] for c in range(n_chains)]
