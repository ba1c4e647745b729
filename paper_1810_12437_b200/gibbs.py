"""Shrinkage-prior logistic Gibbs sampler on the B200 (drop-in for priorcg.gibbs).

`gibbs_run` keeps the reference's signature, scan order, warm start, gamma
policy, pinning, thinning and abort semantics (pkg/src/priorcg/gibbs.py:260-379)
but every scan runs on the GPU as one stream of kernels issued by
`pcgs_gibbs_scan` (include/pcgs.h): Polya-Gamma omega, the global and local
scales, the fused randomised right-hand side, the persistent PCG solve, X beta
with the log-likelihood, the log density and the running statistics.  The
host synchronises only every `sync_every` scans to check for aborts.

Priors: `BridgeConfig` (alpha = 1, the reference's exact path) and
`HorseshoeConfig` (half-Cauchy local and global scales through the auxiliary
inverse-gamma scheme; new, not in the reference — DESIGN.md §5).

RNG: the chain is keyed by Philox4x32-10 with `seed`; draws are independent of
numpy's PCG64 stream, so chains are compared with the reference statistically
(posterior moments within Monte Carlo error), not bit for bit.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .cg import CGConfig

_PART_STRIDE = 16


class UnsupportedUpdateError(NotImplementedError):
    """Conditional update outside the exact device path (gibbs.py:36-37)."""


class GibbsAbortError(RuntimeError):
    """A scan failed; carries the 1-based iteration index (gibbs.py:40-45)."""

    def __init__(self, iteration, message):
        super().__init__(f"iteration {iteration}: {message}")
        self.iteration = iteration


@dataclass(frozen=True)
class BridgeConfig:
    """Bridge prior settings (gibbs.py:48-82)."""

    alpha: float = 1.0
    global_shape: float = 1.0
    global_rate: float = 1.0
    unshrunk_prior_sd: tuple = ()

    def __post_init__(self):
        if not 0.0 < self.alpha <= 1.0:
            raise ValueError("bridge exponent alpha must lie in (0, 1]")
        if self.global_shape <= 0.0 or self.global_rate <= 0.0:
            raise ValueError("Gamma prior on tau^-alpha needs positive shape and rate")
        sds = tuple(float(s) for s in self.unshrunk_prior_sd)
        if any(s <= 0.0 or math.isnan(s) for s in sds):
            raise ValueError("unshrunk prior sds must be positive (inf = flat)")
        object.__setattr__(self, "unshrunk_prior_sd", sds)

    @property
    def n_unshrunk(self) -> int:
        return len(self.unshrunk_prior_sd)

    def unshrunk_precision(self) -> np.ndarray:
        sd = np.asarray(self.unshrunk_prior_sd, dtype=np.float64)
        out = np.zeros(sd.shape)
        fin = np.isfinite(sd)
        out[fin] = sd[fin] ** -2.0
        return out


@dataclass(frozen=True)
class HorseshoeConfig:
    """Horseshoe prior: beta_j ~ N(0, tau^2 lam_j^2), lam_j, tau ~ C+(0, 1).

    New (the reference implements only the bridge); `unshrunk_prior_sd` has
    the BridgeConfig meaning for the leading unshrunk block.
    """

    unshrunk_prior_sd: tuple = ()

    def __post_init__(self):
        sds = tuple(float(s) for s in self.unshrunk_prior_sd)
        if any(s <= 0.0 or math.isnan(s) for s in sds):
            raise ValueError("unshrunk prior sds must be positive (inf = flat)")
        object.__setattr__(self, "unshrunk_prior_sd", sds)

    @property
    def n_unshrunk(self) -> int:
        return len(self.unshrunk_prior_sd)

    def unshrunk_precision(self) -> np.ndarray:
        return BridgeConfig(unshrunk_prior_sd=self.unshrunk_prior_sd).unshrunk_precision()


@dataclass
class ShrinkageState:
    """Sampler snapshot (gibbs.py:85-109); `nu`/`xi` are the horseshoe auxiliaries."""

    beta: np.ndarray
    omega: np.ndarray
    lam: np.ndarray
    tau: float
    nu: np.ndarray | None = None
    xi: float | None = None

    def __post_init__(self):
        self.beta = np.ascontiguousarray(self.beta, dtype=np.float64)
        self.omega = np.ascontiguousarray(self.omega, dtype=np.float64)
        self.lam = np.ascontiguousarray(self.lam, dtype=np.float64)
        self.tau = float(self.tau)
        if self.beta.size < self.lam.size:
            raise ValueError("beta must contain the shrunk block")
        if not np.all(np.isfinite(self.beta)):
            raise ValueError("beta must be finite")
        if np.any(self.omega <= 0.0) or not np.all(np.isfinite(self.omega)):
            raise ValueError("omega must be positive and finite")
        if np.any(self.lam <= 0.0) or not np.all(np.isfinite(self.lam)):
            raise ValueError("lambda must be positive and finite")
        if self.tau <= 0.0 or not math.isfinite(self.tau):
            raise ValueError("tau must be positive and finite")


@dataclass
class ChainOutput:
    """Stored draws plus running statistics (gibbs.py:112-136)."""

    draws: np.ndarray
    tau_draws: np.ndarray
    logdensity_trace: np.ndarray
    cg_iteration_counts: np.ndarray
    running_mean_scaled_beta: np.ndarray | None
    running_var_unshrunk: np.ndarray
    final_state: ShrinkageState
    seed: int
    n_unshrunk: int
    stat_count: int = field(default=0)

    def scaled_beta_mean(self):
        if self.stat_count == 0:
            return None
        return self.running_mean_scaled_beta

    def unshrunk_sd(self):
        if self.stat_count < 2 or self.n_unshrunk == 0:
            return None
        return np.sqrt(self.running_var_unshrunk)


class _GibbsArgs(ctypes.Structure):
    """Mirror of pcgs_gibbs_t (include/pcgs.h)."""

    _fields_ = [
        ("prior", ctypes.c_int), ("q", ctypes.c_int), ("precond", ctypes.c_int),
        ("fixed_omega", ctypes.c_int), ("fixed_tau", ctypes.c_int), ("fixed_lam", ctypes.c_int),
        ("max_iter", ctypes.c_int), ("rtol", ctypes.c_double),
        ("a0", ctypes.c_double), ("b0", ctypes.c_double), ("alpha", ctypes.c_double),
        ("gamma_scale", ctypes.c_double),
        ("seed", ctypes.c_uint64),
        ("y", ctypes.c_void_p), ("kappa", ctypes.c_void_p), ("usd_prec", ctypes.c_void_p),
        ("usd_sd", ctypes.c_void_p),
        ("beta", ctypes.c_void_p), ("z", ctypes.c_void_p), ("omega", ctypes.c_void_p),
        ("lam", ctypes.c_void_p), ("nu", ctypes.c_void_p), ("scal", ctypes.c_void_p),
        ("mean", ctypes.c_void_p), ("m2", ctypes.c_void_p),
        ("prior_diag", ctypes.c_void_p), ("minv", ctypes.c_void_p), ("scale", ctypes.c_void_p),
        ("b", ctypes.c_void_p), ("part", ctypes.c_void_p), ("logdens", ctypes.c_void_p),
        ("results", ctypes.c_void_p), ("draws", ctypes.c_void_p), ("tau_draws", ctypes.c_void_p),
        ("trace", ctypes.c_void_p), ("alphas", ctypes.c_void_p), ("betas", ctypes.c_void_p),
        ("cscale", ctypes.c_void_p),
    ]


class _Reparam:
    """Standardised design X_s = (X - 1 mu') S^-1 with an unstandardised
    intercept: X_s b = X b~ for b~_j = b_j / s_j (j >= 1) and
    b~_0 = b_0 - sum_j mu_j b~_j, so the device samples b~ on the raw pattern
    (exactly the same posterior; include/pcgs.h, pcgs_gibbs_t.cscale)."""

    @staticmethod
    def applies(X, cfg):
        if not X.standardized or X.dense_block is not None:
            return False
        flat0 = cfg.n_unshrunk >= 1 and not np.isfinite(cfg.unshrunk_prior_sd[0])
        return bool(X.has_intercept and X.col_means[0] == 0.0 and X.col_scales[0] == 1.0 and flat0)

    def __init__(self, X, cfg):
        self.mu = np.asarray(X.col_means, dtype=np.float64)
        self.s = np.asarray(X.col_scales, dtype=np.float64)

    def to_sampled(self, beta):
        bt = np.asarray(beta, dtype=np.float64) / self.s
        bt[..., 0] -= bt[..., 1:] @ self.mu[1:]
        return bt

    def to_model(self, bt):
        bt = np.asarray(bt, dtype=np.float64)
        beta = bt * self.s
        beta[..., 0] = bt[..., 0] + bt[..., 1:] @ self.mu[1:]
        return beta


_PRECOND = {"prior": 0, "identity": 1, "jacobi": 2}


class DeviceChain:
    """Device-resident state of one chain; `scan(t)` issues one Gibbs scan."""

    def __init__(self, X, y, cfg, n_iter, burn_in=0, thin=1, seed=0, preconditioner="prior",
                 cg_config=None, init_state=None, gamma_scale=1.0, fixed_omega=None,
                 fixed_tau=None, fixed_lam=None, device=None, grid=0):
        t = _lib.torch()
        self.X = X
        self._grid_req = int(grid)
        # standardised pattern-only designs with an unstandardised flat-prior
        # intercept sample on the raw pattern (_Reparam); every other design
        # with affine terms (dense block, standardisation) runs on the affine
        # store directly (model coefficients)
        self.reparam = _Reparam(X, cfg) if _Reparam.applies(X, cfg) else None
        self._open_device(X, device)
        dev = self.dev
        f64 = t.float64
        self.n, self.pt = X.n_rows, X.n_cols
        self.q = cfg.n_unshrunk
        self.p = self.pt - self.q
        self.cfg = cfg
        self.horseshoe = isinstance(cfg, HorseshoeConfig)
        self.n_iter, self.burn_in, self.thin = n_iter, burn_in, thin
        self.seed = int(seed)
        cgc = cg_config if cg_config is not None else CGConfig()
        if cgc.trace_level == "full":
            raise NotImplementedError("trace_level='full' is not on the device path")
        max_iter = cgc.max_iter if cgc.max_iter is not None else 2 * self.pt
        self.max_iter = max_iter
        self.n_store = max(0, (n_iter - burn_in + thin - 1) // thin) if n_iter else 0

        def dt(x):
            return _lib.to_device(x, dev)

        yh = np.asarray(y, dtype=np.float64)
        self.y = dt(yh)
        self.kappa = dt(yh - 0.5)
        sd = np.asarray(cfg.unshrunk_prior_sd, dtype=np.float64)
        self.usd_sd = dt(sd if sd.size else np.zeros(1))
        self.usd_prec = dt(cfg.unshrunk_precision() if sd.size else np.zeros(1))
        if init_state is None:
            beta = np.zeros(self.pt)
            omega = np.full(self.n, 0.25)
            lam = np.ones(self.p)
            tau = 1.0
            nu, xi = np.ones(self.p), 1.0
        else:
            beta, omega, lam, tau = init_state.beta, init_state.omega, init_state.lam, init_state.tau
            nu = init_state.nu if init_state.nu is not None else np.ones(self.p)
            xi = init_state.xi if init_state.xi is not None else 1.0
            if beta.shape != (self.pt,) or lam.shape != (self.p,):
                raise ValueError("initial state does not match the model shape")
        if self.reparam is not None:
            beta = self.reparam.to_sampled(beta)
            self.cscale = dt(self.reparam.s)
        self.beta = dt(beta).clone()
        self.omega = dt(fixed_omega if fixed_omega is not None else omega).clone()
        self.lam = dt(fixed_lam if fixed_lam is not None else lam).clone()
        self.nu = dt(nu).clone()
        self.scal = dt(np.array([fixed_tau if fixed_tau is not None else tau, xi, 0.0, 0.0]))
        self.z = t.empty(self.n + 2, dtype=f64, device=dev)
        self.mean = t.zeros(self.pt, dtype=f64, device=dev)
        self.m2 = t.zeros(max(self.q, 1), dtype=f64, device=dev)
        self.prior_diag = t.empty(self.pt, dtype=f64, device=dev)
        self.minv = t.empty(self.pt, dtype=f64, device=dev)
        self.scale = t.empty(self.pt, dtype=f64, device=dev)
        self.b = t.empty(self.pt, dtype=f64, device=dev)
        self.part = t.zeros(_PART_STRIDE * (self.grid + 1), dtype=f64, device=dev)
        self.logdens = t.zeros(max(n_iter, 1), dtype=f64, device=dev)
        self.results = t.zeros(8 * max(n_iter, 1), dtype=t.int32, device=dev)
        self.draws = t.empty((max(self.n_store, 1), self.pt), dtype=f64, device=dev)
        self.tau_draws = t.empty(max(self.n_store, 1), dtype=f64, device=dev)
        self.trace = t.empty(max_iter + 1, dtype=f64, device=dev)
        self.alphas = t.empty(max_iter + 1, dtype=f64, device=dev)
        self.betas = t.empty(max_iter + 1, dtype=f64, device=dev)
        P = _lib.ptr
        self.args = _GibbsArgs(
            prior=1 if self.horseshoe else 0, q=self.q, precond=_PRECOND[preconditioner],
            fixed_omega=int(fixed_omega is not None), fixed_tau=int(fixed_tau is not None),
            fixed_lam=int(fixed_lam is not None), max_iter=int(max_iter), rtol=float(cgc.rtol),
            a0=float(getattr(cfg, "global_shape", 1.0)), b0=float(getattr(cfg, "global_rate", 1.0)),
            alpha=float(getattr(cfg, "alpha", 1.0)),
            gamma_scale=float(gamma_scale), seed=self.seed & (2 ** 64 - 1),
            y=P(self.y), kappa=P(self.kappa), usd_prec=P(self.usd_prec), usd_sd=P(self.usd_sd),
            beta=P(self.beta), z=P(self.z), omega=P(self.omega), lam=P(self.lam), nu=P(self.nu),
            scal=P(self.scal), mean=P(self.mean), m2=P(self.m2), prior_diag=P(self.prior_diag),
            minv=P(self.minv), scale=P(self.scale), b=P(self.b), part=P(self.part),
            logdens=P(self.logdens), results=P(self.results), draws=P(self.draws),
            tau_draws=P(self.tau_draws), trace=P(self.trace), alphas=P(self.alphas),
            betas=P(self.betas), cscale=P(self.cscale) if self.reparam is not None else None)
        self.count = 0
        self.stored = 0
        L = _lib.lib()
        L.pcgs_gibbs_init.argtypes = [ctypes.c_void_p, ctypes.POINTER(_GibbsArgs), ctypes.c_void_p]
        L.pcgs_gibbs_scan.argtypes = [ctypes.c_void_p, ctypes.POINTER(_GibbsArgs), ctypes.c_int32,
                                      ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p]
        L.pcgs_gibbs_scan_begin.argtypes = [ctypes.c_void_p, ctypes.POINTER(_GibbsArgs), ctypes.c_int32,
                                            ctypes.c_void_p]
        L.pcgs_gibbs_scan_end.argtypes = [ctypes.c_void_p, ctypes.POINTER(_GibbsArgs), ctypes.c_int32,
                                          ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p]
        self._init_device()

    def _open_device(self, X, device):
        self.store = X.device_store(device, grid=self._grid_req, raw=self.reparam is not None)
        self.dev = self.store.device
        self.grid = self.store.describe()["grid"]

    def _init_device(self):
        _lib.check(_lib.lib().pcgs_gibbs_init(self.store.handle, ctypes.byref(self.args),
                                              _lib.stream_ptr(self.dev)))

    def next_slot(self, t):
        """Row of `draws` that scan t stores into (advancing the count), or -1."""
        if t > self.burn_in and (t - self.burn_in - 1) % self.thin == 0:
            self.stored += 1
            return self.stored - 1
        return -1

    def scan(self, t, local_scale_sampler=None, rng=None):
        """Issue scan t (1-based) on the current stream; no synchronisation
        unless a host `local_scale_sampler` has to see beta and tau."""
        slot = self.next_slot(t)
        L = _lib.lib()
        s = _lib.stream_ptr(self.dev)
        if local_scale_sampler is None:
            _lib.check(L.pcgs_gibbs_scan(self.store.handle, ctypes.byref(self.args), int(t),
                                         int(self.count), int(slot), s))
        else:
            _lib.check(L.pcgs_gibbs_scan_begin(self.store.handle, ctypes.byref(self.args), int(t), s))
            torch = _lib.torch()
            torch.cuda.current_stream(self.dev).synchronize()
            beta = self.beta.cpu().numpy()
            if self.reparam is not None:
                beta = self.reparam.to_model(beta)
            tau = float(self.scal[0].item())
            lam = np.asarray(local_scale_sampler(beta[self.q:], tau, self.cfg, rng), dtype=np.float64)
            if lam.shape != (self.p,):
                raise ValueError("local_scale_sampler must return one scale per shrunk coefficient")
            self.lam.copy_(torch.from_numpy(lam))
            self.args.fixed_lam = 1
            try:
                _lib.check(L.pcgs_gibbs_scan_end(self.store.handle, ctypes.byref(self.args), int(t),
                                                 int(self.count), int(slot), s))
            finally:
                self.args.fixed_lam = 0
        self.count += 1

    def check(self, t_lo, t_hi, allow_max_iter=False):
        """Raise GibbsAbortError for the first failed scan in [t_lo, t_hi]."""
        res = self.results[8 * (t_lo - 1): 8 * t_hi].view(-1, 8).cpu().numpy()
        for k, r in enumerate(res):
            t = t_lo + k
            if r[4]:
                raise GibbsAbortError(t, "scale positivity violated")
            if r[1] == _lib.PCGS_NOT_PD:
                raise GibbsAbortError(t, f"beta update failed: d'Phi d <= 0 at CG iteration {r[2]}")
            if r[1] == _lib.PCGS_NONFINITE:
                raise GibbsAbortError(t, f"beta update failed: non-finite value at CG iteration {r[2]}")
            if r[1] == _lib.PCGS_MAX_ITER and not allow_max_iter:
                raise GibbsAbortError(t, f"CG used all {r[0]} iterations without converging")

    def state_snapshot(self) -> ShrinkageState:
        """The current state on the host, in model coordinates (a valid
        `init_state` for a continuing gibbs_run)."""
        scal = self.scal.cpu().numpy()
        beta = self.beta.cpu().numpy()
        if self.reparam is not None:
            beta = self.reparam.to_model(beta)
        return ShrinkageState(beta, self.omega.cpu().numpy(), self.lam.cpu().numpy(), float(scal[0]),
                              nu=self.nu.cpu().numpy() if self.horseshoe else None,
                              xi=float(scal[1]) if self.horseshoe else None)

    def output(self) -> ChainOutput:
        t = self.n_iter
        res = self.results[: 8 * max(t, 1)].view(-1, 8).cpu().numpy()[:t]
        draws = self.draws[: self.stored].cpu().numpy()
        if self.reparam is not None:
            draws = self.reparam.to_model(draws)
        state = self.state_snapshot()
        m2 = self.m2.cpu().numpy()[: self.q]
        var = m2 / (self.count - 1) if self.count >= 2 else np.full(self.q, np.nan)
        return ChainOutput(
            draws=draws,
            tau_draws=self.tau_draws[: self.stored].cpu().numpy(),
            logdensity_trace=self.logdens[:t].cpu().numpy(),
            cg_iteration_counts=res[:, 0].astype(np.int64),
            running_mean_scaled_beta=self.mean.cpu().numpy() if self.count else None,
            running_var_unshrunk=var, final_state=state, seed=self.seed, n_unshrunk=self.q,
            stat_count=self.count)


def _check_run_args(X, y, cfg, n_iter, burn_in, thin, sampler, burn_in_sampler, preconditioner,
                    fixed_lam, local_scale_sampler):
    """gibbs_run's argument checks (gibbs.py:260-300); returns y as float64."""
    y = np.asarray(y, dtype=np.float64)
    if y.shape != (X.n_rows,):
        raise ValueError("outcome length must match the design")
    if not np.all((y == 0.0) | (y == 1.0)):
        raise ValueError("outcomes must be 0/1")
    if n_iter < 0 or burn_in < 0 or burn_in > n_iter:
        raise ValueError("need 0 <= burn_in <= n_iter")
    if thin < 1:
        raise ValueError("thin must be >= 1")
    for name in (sampler, burn_in_sampler):
        if name not in (None, "cg", "direct"):
            raise ValueError(f"unknown sampler {name!r}")
    if "direct" in (sampler, burn_in_sampler):
        raise NotImplementedError("the dense Cholesky sampler is the CPU oracle's; use sampler='cg'")
    if preconditioner not in _PRECOND:
        if str(preconditioner).startswith("block:"):
            raise NotImplementedError("block-threshold preconditioning is not on the device path")
        raise ValueError(f"unknown preconditioner {preconditioner!r}")
    q = cfg.n_unshrunk
    if X.n_cols - q < 0:
        raise ValueError("more unshrunk prior sds than design columns")
    if (isinstance(cfg, BridgeConfig) and cfg.alpha != 1.0 and fixed_lam is None
            and local_scale_sampler is None):
        raise UnsupportedUpdateError(
            "exact local-scale draws exist for alpha = 1 only; pin fixed_lam for other exponents")
    return y


def gibbs_run(X, y, cfg, n_iter, burn_in=0, sampler="cg", seed=0, thin=1, preconditioner="prior",
              cg_config=None, burn_in_sampler=None, init_state=None, local_scale_sampler=None,
              gamma_scale=1.0, allow_max_iter=False, fixed_omega=None, fixed_tau=None,
              fixed_lam=None, on_progress=None, device=None, sync_every=64, grid=0) -> ChainOutput:
    """Run `n_iter` scans on the GPU (gibbs.py:260-379); same arguments and output.

    `sampler`/`burn_in_sampler` must be "cg" (the dense Cholesky sampler is the
    CPU oracle's).  A `local_scale_sampler(beta_shrunk, tau, cfg, rng)` runs on
    the host between the two halves of each scan (one synchronisation per
    scan), with a numpy Generator seeded from `seed`.

    `grid` > 0 plans the store for that many CTAs (chains sharing a GPU
    concurrently, `parallel.run_chains`); 0 = one CTA per SM.

    Standardised designs (`X.standardize(...)`) run through an exact
    reparametrisation on the raw pattern (`_Reparam`; needs an unstandardised
    intercept with a flat prior); draws and the final state come back in the
    model's coordinates, the running statistics of the unshrunk block stay in
    the sampled ones.
    """
    y = _check_run_args(X, y, cfg, n_iter, burn_in, thin, sampler, burn_in_sampler, preconditioner,
                        fixed_lam, local_scale_sampler)
    ch = DeviceChain(X, y, cfg, n_iter, burn_in=burn_in, thin=thin, seed=seed,
                     preconditioner=preconditioner, cg_config=cg_config, init_state=init_state,
                     gamma_scale=gamma_scale, fixed_omega=fixed_omega, fixed_tau=fixed_tau,
                     fixed_lam=fixed_lam, device=device, grid=grid)
    torch = _lib.torch()
    checked = 0
    host_rng = np.random.default_rng(seed) if local_scale_sampler is not None else None
    for t in range(1, n_iter + 1):
        ch.scan(t, local_scale_sampler, host_rng)
        if on_progress is not None:
            torch.cuda.current_stream(ch.dev).synchronize()
            ch.check(t, t, allow_max_iter)
            checked = t
            on_progress(t, n_iter)
        elif sync_every and t - checked >= sync_every:
            ch.check(checked + 1, t, allow_max_iter)
            checked = t
    if checked < n_iter:
        ch.check(checked + 1, n_iter, allow_max_iter)
    return ch.output()


def gibbs_run_concurrent(X, y, cfg, n_iter, seeds, concurrent=4, burn_in=0, thin=1, sampler="cg",
                         preconditioner="prior", cg_config=None, burn_in_sampler=None, init_state=None,
                         gamma_scale=1.0, allow_max_iter=False, fixed_omega=None, fixed_tau=None,
                         fixed_lam=None, device=None, poll_s=2e-4) -> list:
    """Independent chains (one per seed) sharing one GPU: `concurrent` slots,
    each a CUDA stream, with the store planned for SMs // concurrent CTAs so
    the slots' persistent PCG kernels run side by side.  Chain c's output
    equals gibbs_run(..., seed=seeds[c], grid=SMs // concurrent) bit for bit
    (deterministic kernels; the slot only changes what runs beside it).

    Every chain is issued whole (all its scans) onto a free slot; the host then
    waits for whichever slot finishes first (stream polling, no blocking call
    on a busy stream), reads that chain's output, checks it for aborts and
    frees it before issuing the next chain there.  Device memory is bounded by
    `concurrent` chains.  Aborts are reported when the failed chain finishes
    (GibbsAbortError for its first failed scan, as gibbs_run raises it)."""
    import time
    torch = _lib.torch()
    y = _check_run_args(X, y, cfg, n_iter, burn_in, thin, sampler, burn_in_sampler, preconditioner,
                        fixed_lam, None)
    dev = _lib.cuda_device(device)
    concurrent = max(1, int(concurrent))
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    grid = 0 if concurrent == 1 else sms // concurrent
    seeds = list(seeds)
    slots = [torch.cuda.Stream(dev) for _ in range(concurrent)]
    busy = {}          # slot -> (chain index, DeviceChain)
    outs = [None] * len(seeds)

    def finish(k):
        c, ch = busy.pop(k)
        with torch.cuda.stream(slots[k]):
            slots[k].synchronize()
            ch.check(1, n_iter, allow_max_iter) if n_iter else None
            outs[c] = ch.output()

    def free_slot():
        while True:
            for k in range(concurrent):
                if k not in busy:
                    return k
            for k in list(busy):
                if slots[k].query():
                    finish(k)
                    return k
            time.sleep(poll_s)

    for c, sd in enumerate(seeds):
        k = free_slot()
        with torch.cuda.stream(slots[k]):
            ch = DeviceChain(X, y, cfg, n_iter, burn_in=burn_in, thin=thin, seed=sd,
                             preconditioner=preconditioner, cg_config=cg_config,
                             init_state=init_state, gamma_scale=gamma_scale,
                             fixed_omega=fixed_omega, fixed_tau=fixed_tau, fixed_lam=fixed_lam,
                             device=dev, grid=grid)
            for t in range(1, n_iter + 1):
                ch.scan(t)
        busy[k] = (c, ch)
    for k in sorted(busy):
        finish(k)
    return outs


class BatchedChains:
    """R = len(seeds) chains (R in {2, 4, 8}) whose beta solves run as ONE
    batched PCG per scan (`pcgs_batch_gibbs_scan`, the sliced store of
    csrc/sliced.h): every chain keeps its own state, RNG keys and outputs
    (DeviceChain); `scan(t)` issues scan t of every chain.  A chain's
    trajectory depends on its seed and R only (each chain's sums run in the
    same order whatever the other chains hold)."""

    def __init__(self, X, y, cfg, n_iter, seeds, device=None, **kw):
        seeds = list(seeds)
        R = len(seeds)
        if R not in (2, 4, 8):
            raise ValueError("batched chains come in batches of 2, 4 or 8")
        self.chains = [DeviceChain(X, y, cfg, n_iter, seed=sd, device=device, **kw) for sd in seeds]
        mi = {ch.max_iter for ch in self.chains}
        if len(mi) != 1:
            raise ValueError("batched chains must share max_iter")
        self.R = R
        self.dev = self.chains[0].dev
        self.store = self.chains[0].store
        self.bstore = X.batch_store(R, self.dev)
        self._ptrs = (ctypes.c_void_p * R)(*[ctypes.addressof(ch.args) for ch in self.chains])
        self._counts = np.zeros(R, dtype=np.int32)
        self._slots = np.zeros(R, dtype=np.int32)

    def scan(self, t):
        for c, ch in enumerate(self.chains):
            self._counts[c] = ch.count
            self._slots[c] = ch.next_slot(t)
        _lib.check(_lib.lib().pcgs_batch_gibbs_scan(
            self.store.handle, self.bstore.handle, ctypes.cast(self._ptrs, ctypes.c_void_p), self.R, int(t),
            self._counts.ctypes.data, self._slots.ctypes.data, _lib.stream_ptr(self.dev)))
        for ch in self.chains:
            ch.count += 1

    @property
    def fusable(self):
        """True when the scans can run whole inside one persistent kernel
        (`run`): prior preconditioner, no pinned updates, no reparametrisation."""
        a = self.chains[0].args
        return (a.precond == 0 and not (a.fixed_omega or a.fixed_tau or a.fixed_lam)
                and all(ch.reparam is None for ch in self.chains))

    def run(self, t_first, t_last):
        """Scans t_first..t_last of every chain inside ONE persistent kernel
        (`pcgs_batch_gibbs_run`): a chain whose solve ends starts its next scan
        while the others keep iterating.  Same RNG keys, statistics, stored
        draws and log density as `scan(t)` per scan."""
        if not self.fusable:
            raise NotImplementedError("fused batched scans need the prior preconditioner and no pinned updates")
        if t_last < t_first:
            return
        ch0 = self.chains[0]
        for c, ch in enumerate(self.chains):
            self._counts[c] = ch.count
            self._slots[c] = ch.stored
        t = _lib.torch()
        out = t.zeros(2 * self.R, dtype=t.int32, device=self.dev)
        _lib.check(_lib.lib().pcgs_batch_gibbs_run(
            self.bstore.handle, ctypes.cast(self._ptrs, ctypes.c_void_p), self.R, int(t_first), int(t_last),
            int(ch0.burn_in), int(ch0.thin), self._counts.ctypes.data, self._slots.ctypes.data, _lib.ptr(out),
            _lib.stream_ptr(self.dev)))
        for ch in self.chains:          # the same bookkeeping the kernel does (deterministic)
            for tt in range(t_first, t_last + 1):
                ch.next_slot(tt)
            ch.count += t_last - t_first + 1
        self._out_state = out

    def check(self, t_lo, t_hi, allow_max_iter=False):
        for ch in self.chains:
            ch.check(t_lo, t_hi, allow_max_iter)

    def outputs(self):
        return [ch.output() for ch in self.chains]


def gibbs_run_batched(X, y, cfg, n_iter, seeds, burn_in=0, sampler="cg", thin=1, preconditioner="prior",
                      cg_config=None, burn_in_sampler=None, init_state=None, gamma_scale=1.0,
                      allow_max_iter=False, fixed_omega=None, fixed_tau=None, fixed_lam=None, device=None,
                      sync_every=256, fused=False) -> list:
    """gibbs_run (gibbs.py:260-379) for R = len(seeds) independent chains
    (R in {2, 4, 8}) sharing every walk over the pattern; chain c is the
    chain of seed seeds[c].  Every scan runs each chain's updates and then
    one batched PCG for all beta draws (`BatchedChains.scan`); with `fused`
    (prior preconditioner, no pinned updates) the chains instead run whole
    scans inside one persistent kernel at their own pace (`BatchedChains.run`,
    the same chains: same RNG keys, draws equal to the solves' tolerance).
    Returns one ChainOutput per seed."""
    y = _check_run_args(X, y, cfg, n_iter, burn_in, thin, sampler, burn_in_sampler, preconditioner,
                        fixed_lam, None)
    B = BatchedChains(X, y, cfg, n_iter, seeds, device=device, burn_in=burn_in, thin=thin,
                      preconditioner=preconditioner, cg_config=cg_config, init_state=init_state,
                      gamma_scale=gamma_scale, fixed_omega=fixed_omega, fixed_tau=fixed_tau,
                      fixed_lam=fixed_lam)
    checked = 0
    if fused and B.fusable:
        # whole scans inside one persistent kernel, checked every sync_every scans
        step = sync_every if sync_every else n_iter
        for t0 in range(1, n_iter + 1, max(step, 1)):
            t1 = min(n_iter, t0 + max(step, 1) - 1)
            B.run(t0, t1)
            B.check(t0, t1, allow_max_iter)
        return B.outputs()
    for t in range(1, n_iter + 1):
        B.scan(t)
        if sync_every and t - checked >= sync_every:
            B.check(checked + 1, t, allow_max_iter)
            checked = t
    if checked < n_iter:
        B.check(checked + 1, n_iter, allow_max_iter)
    return B.outputs()


def scale_draws(prior, mode, count, b_or_acc, tau=1.0, lam_old=1.0, p=1, a0=1.0, b0=1.0, alpha=1.0,
                seed=0, device=None):
    """Draws of the scan's scale updates on the device (pcgs_scale_draws):
    the same device functions the scan kernels use, exposed for validation
    against their analytic conditionals (test_gibbs.py:114-140 style).
    `prior` is "bridge" or "horseshoe"; `mode` 0 = independent global draws
    (returns tau, xi), 1 = independent local draws (lam, nu), 2 / 3 = the
    single-thread auxiliary chain of the global / local update (tau or lam
    per step, and the auxiliary)."""
    torch = _lib.torch()
    dev = _lib.cuda_device(device)
    out = torch.empty(max(int(count), 1), dtype=torch.float64, device=dev)
    aux = torch.empty_like(out)
    _lib.check(_lib.lib().pcgs_scale_draws(
        0 if prior == "bridge" else 1, int(mode), int(count), float(b_or_acc), float(tau),
        float(lam_old), int(p), float(a0), float(b0), float(alpha), int(seed) & (2 ** 64 - 1),
        _lib.ptr(out), _lib.ptr(aux), _lib.stream_ptr(dev)))
    return out[:count].cpu().numpy(), aux[:count].cpu().numpy()
