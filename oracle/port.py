"""numpy restatement of the reference hot path (TEST INFRASTRUCTURE ONLY).

Every function names the reference lines it follows (paths relative to
/root/reference/pkg/src/priorcg/).  Arithmetic is replayed with the same numpy
primitives in the same order (reduceat row sums, bincount column sums, the
same Generator calls in the same sequence), so where the reference is
deterministic the port reproduces it bit for bit; tests/test_oracle.py checks
that against tests/golden/*.npz written by the reference itself.

The horseshoe conditionals at the bottom have no reference counterpart
(SURVEY.md §0 gap 1); they are new code, validated statistically.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
from scipy.special import expit, gammaln, log_ndtr

# ============================================================== sparse design
@dataclass
class Csr:
    """CSR with standardisation vectors (sparse.py:46-92)."""

    n: int
    p: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray
    col_means: np.ndarray | None = None
    col_scales: np.ndarray | None = None

    def __post_init__(self):
        self.row_ptr = np.asarray(self.row_ptr, dtype=np.int64)
        self.col_idx = np.asarray(self.col_idx, dtype=np.int64)
        self.values = np.asarray(self.values, dtype=np.float64)
        if self.col_means is None:
            self.col_means = np.zeros(self.p)
        if self.col_scales is None:
            self.col_scales = np.ones(self.p)
        counts = np.diff(self.row_ptr)
        self.row_of = np.repeat(np.arange(self.n, dtype=np.int64), counts)   # sparse.py:153-157
        self.nonempty = np.flatnonzero(counts > 0)                             # sparse.py:159-162


def design_from_pattern(n, p, row_ptr, col_idx, intercept=True) -> Csr:
    """Reference layout of a binary design: the intercept is column 0 of the
    CSR, first in every row, as hstack_dense_columns builds it (sparse.py:314-341)."""
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    col_idx = np.asarray(col_idx, dtype=np.int64)
    if not intercept:
        return Csr(n, p, row_ptr.copy(), col_idx.copy(), np.ones(len(col_idx)))
    rp = row_ptr + np.arange(n + 1, dtype=np.int64)
    ci = np.empty(len(col_idx) + n, dtype=np.int64)
    head = rp[:-1]
    mask = np.ones(len(ci), dtype=bool)
    mask[head] = False
    ci[head] = 0
    ci[mask] = col_idx + 1
    return Csr(n, p + 1, rp, ci, np.ones(len(ci)))


def matvec(X: Csr, v):
    """X v with the rank-one standardisation shift (sparse.py:178-193, 164-169)."""
    u = np.asarray(v, dtype=np.float64) / X.col_scales
    prod = X.values * u[X.col_idx]
    out = np.zeros(X.n)
    if X.nonempty.size:
        out[X.nonempty] = np.add.reduceat(prod, X.row_ptr[X.nonempty])
    shift = X.col_means @ u
    if shift != 0.0:
        out -= shift
    return out


def matvec_t(X: Csr, w):
    """X' w (sparse.py:195-203): bincount scatter in storage order."""
    w = np.asarray(w, dtype=np.float64)
    raw = np.bincount(X.col_idx, weights=X.values * w[X.row_of], minlength=X.p)
    return (raw - w.sum() * X.col_means) / X.col_scales


def phi_apply(X: Csr, omega, prior_diag, v):
    """Phi v = X'(omega X v) + d v (sampler.py:53-58)."""
    out = matvec_t(X, omega * matvec(X, v))
    out += prior_diag * v
    return out


def _csc_cache(X: Csr):
    if not hasattr(X, "_csc_perm"):
        X._csc_perm = np.argsort(X.col_idx, kind="stable")
        X._csc_rows = X.row_of[X._csc_perm]
        X._csc_vals = X.values[X._csc_perm]
        cnt = np.bincount(X.col_idx, minlength=X.p)
        X._csc_start = np.concatenate([[0], np.cumsum(cnt)[:-1]])
        X._csc_nonempty = cnt > 0


def _phi_ld_core(X: Csr, omega, prior_diag, vL):
    """Phi v (sampler.py:53-58) of the standardised value-carrying CSR
    (sparse.py:178-203) with every sum accumulated in long double."""
    L = np.longdouble
    _csc_cache(X)
    sc, mu = np.asarray(X.col_scales).astype(L), np.asarray(X.col_means).astype(L)
    u = vL / sc
    z = np.zeros(X.n, dtype=L)
    if X.nonempty.size:
        z[X.nonempty] = np.add.reduceat(np.asarray(X.values).astype(L) * u[X.col_idx], X.row_ptr[X.nonempty])
    z -= np.dot(mu, u)
    w = np.asarray(omega, dtype=np.float64).astype(L) * z
    g = np.zeros(X.p, dtype=L)
    ne = X._csc_nonempty
    g[ne] = np.add.reduceat(X._csc_vals.astype(L) * w[X._csc_rows], X._csc_start[ne])
    g = (g - mu * w.sum()) / sc
    return g + np.asarray(prior_diag).astype(L) * vL


def phi_apply_exact_ld(X: Csr, omega, prior_diag, v):
    """Phi v with every sum accumulated in x87 long double (64-bit mantissa),
    returned in long double; rounded once to float64 (phi_apply_exact) it is
    to within an ulp the correctly rounded Phi v of sampler.py:53-58 (for
    binary unstandardised designs every value / shift / scale is exact).  Used
    to measure the TRUE residual b - Phi x of a solution, independent of any
    fp64 summation order (tests/test_gpu_parity_config2.py)."""
    return _phi_ld_core(X, omega, prior_diag, np.asarray(v, dtype=np.float64).astype(np.longdouble))


def phi_apply_exact(X: Csr, omega, prior_diag, v):
    """phi_apply_exact_ld rounded once to float64."""
    return phi_apply_exact_ld(X, omega, prior_diag, v).astype(np.float64)


def true_rms(X: Csr, omega, prior_diag, b, x, scale):
    """RMS of the scaled TRUE residual s*(b - Phi x) (the cg.py:150-151 metric),
    Phi x from phi_apply_exact and the difference taken in long double."""
    L = np.longdouble
    L_ax = phi_apply_exact_ld(X, omega, prior_diag, x)
    t = np.asarray(scale).astype(L) * (np.asarray(b).astype(L) - L_ax)
    return float(np.sqrt(np.dot(t, t) / len(b)))


def gram_diagonal(X: Csr, omega):
    """diag(X' Omega X) (sparse.py:235-246)."""
    w = np.asarray(omega)[X.row_of]
    sq = np.bincount(X.col_idx, weights=X.values ** 2 * w, minlength=X.p)
    g = np.bincount(X.col_idx, weights=X.values * w, minlength=X.p)
    mu = X.col_means
    return (sq - 2.0 * mu * g + np.sum(omega) * mu ** 2) / X.col_scales ** 2


# ============================================================== PCG
class NotPD(RuntimeError):
    pass


class Breakdown(RuntimeError):
    def __init__(self, k):
        super().__init__(f"non-finite value at CG iteration {k}")
        self.iteration = k


@dataclass
class PcgResult:
    x: np.ndarray
    iterations: int
    termination: str
    trace: np.ndarray
    alphas: np.ndarray
    betas: np.ndarray
    applies: int


def pcg(apply, b, minv, scale, x0=None, max_iter=None, rtol=1e-6, callback=None) -> PcgResult:
    """Hestenes-Stiefel PCG with the RMS scaled-residual stop (cg.py:105-192).
    `callback(x)` sees every iterate (x0 first), as trace_level="full" records
    them (cg.py:160-170)."""
    b = np.asarray(b, dtype=np.float64)
    p = b.shape[0]
    max_iter = 2 * p if max_iter is None else max_iter
    x = np.zeros(p) if x0 is None else np.array(x0, dtype=np.float64)
    r = b - apply(x)
    applies = 1
    t = scale * r
    rms = math.sqrt(float(np.dot(t, t)) / p)
    if not np.isfinite(rms):
        raise Breakdown(0)
    trace, alphas, betas = [rms], [], []
    if callback is not None:
        callback(x.copy())
    k = 0
    if rms > rtol:
        z = minv * r
        rz = float(np.dot(r, z))
        d = z.copy()
        while k < max_iter:
            k += 1
            Ad = apply(d)
            applies += 1
            dAd = float(np.dot(d, Ad))
            if not dAd > 0:
                raise NotPD(f"d'Phi d = {dAd} at CG iteration {k}")
            alpha = rz / dAd
            alphas.append(alpha)
            x += alpha * d
            r -= alpha * Ad
            if callback is not None:
                callback(x.copy())
            t = scale * r
            rms = math.sqrt(float(np.dot(t, t)) / p)
            trace.append(rms)
            if rms <= rtol:
                break
            if not np.isfinite(rms):
                raise Breakdown(k)
            z = minv * r
            rz_new = float(np.dot(r, z))
            beta = rz_new / rz
            betas.append(beta)
            rz = rz_new
            d *= beta
            d += z
    return PcgResult(x, k, "converged" if rms <= rtol else "max_iter", np.array(trace),
                     np.array(alphas), np.array(betas), applies)


def _reordered(X: Csr) -> Csr:
    """The same matrix with the rows in reverse order and every row's columns
    reversed (cached): another reduceat / bincount summation order."""
    if not hasattr(X, "_rev"):
        n = X.n
        cnt = np.diff(X.row_ptr)[::-1]
        rp = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(cnt, out=rp[1:])
        ci = X.col_idx[::-1].copy()            # rows reversed AND columns reversed within rows
        X._rev = Csr(n, X.p, rp, ci, X.values[::-1].copy(), X.col_means, X.col_scales)
    return X._rev


def phi_apply_ordered(X: Csr, omega, prior_diag, v, order="ref"):
    """Phi v in float64 with a chosen summation order: "ref" (the reference's,
    sampler.py:53-58), "rev" (rows and row entries reversed), "split" (two row
    halves summed afterwards), "cr" (correctly rounded: phi_apply_exact)."""
    if order == "ref":
        return phi_apply(X, omega, prior_diag, v)
    if order == "cr":
        return phi_apply_exact(X, omega, prior_diag, v)
    if order == "rev":
        Xr = _reordered(X)
        return phi_apply(Xr, np.asarray(omega)[::-1], prior_diag, v)
    if order == "split":
        h = X.n // 2
        out = np.zeros(X.p)
        for lo, hi in ((0, h), (h, X.n)):
            rp = X.row_ptr[lo:hi + 1] - X.row_ptr[lo]
            sl = slice(X.row_ptr[lo], X.row_ptr[hi])
            Xs = Csr(hi - lo, X.p, rp, X.col_idx[sl], X.values[sl], X.col_means, X.col_scales)
            out = out + matvec_t(Xs, np.asarray(omega)[lo:hi] * matvec(Xs, v))
        return out + prior_diag * v
    raise ValueError(order)


def pcg_long_double(X: Csr, omega, prior_diag, b, minv, scale, x0=None, rtol=1e-6, max_iter=None):
    """The PCG recurrence of cg.py:105-192 with every operation in long
    double (Phi from phi_apply_exact_ld): the extended-precision reference
    point of the iteration-count band.  Returns the iteration count."""
    L = np.longdouble
    p = len(b)
    max_iter = 2 * p if max_iter is None else max_iter
    bL, mL, sL = (np.asarray(a, dtype=np.float64).astype(L) for a in (b, minv, scale))
    x = np.zeros(p, dtype=L) if x0 is None else np.asarray(x0, dtype=np.float64).astype(L)
    r = bL - phi_apply_exact_ld(X, omega, prior_diag, x.astype(np.float64))
    t = sL * r
    rms = math.sqrt(float(np.dot(t, t)) / p)
    k = 0
    if rms <= rtol:
        return 0
    z = mL * r
    rz = np.dot(r, z)
    d = z.copy()
    while k < max_iter:
        k += 1
        Ad = _phi_ld_vec(X, omega, prior_diag, d)
        alpha = rz / np.dot(d, Ad)
        x = x + alpha * d
        r = r - alpha * Ad
        t = sL * r
        rms = math.sqrt(float(np.dot(t, t)) / p)
        if rms <= rtol:
            break
        z = mL * r
        rzn = np.dot(r, z)
        d = z + (rzn / rz) * d
        rz = rzn
    return k


def _phi_ld_vec(X: Csr, omega, prior_diag, v):
    """phi_apply_exact_ld for a long-double input vector (no rounding to float64)."""
    return _phi_ld_core(X, omega, prior_diag, v)


def iteration_band(X: Csr, omega, prior_diag, b, minv, scale, rtol=1e-6, max_iter=None):
    """The iteration-count band of a PCG solve (tests' parity gate for the
    count): the counts of the float64 recurrence under the summation orders of
    phi_apply_ordered and of the long-double recurrence; F = max(2, spread of
    the float64 counts); band = [min(all) - F, reference + F].  Returns
    (lo, hi, counts dict)."""
    counts = {o: pcg(lambda v, o=o: phi_apply_ordered(X, omega, prior_diag, v, o), b, minv, scale,
                     rtol=rtol, max_iter=max_iter).iterations for o in ("ref", "rev", "split", "cr")}
    counts["ld"] = pcg_long_double(X, omega, prior_diag, b, minv, scale, rtol=rtol, max_iter=max_iter)
    f64 = [counts[o] for o in ("ref", "rev", "split", "cr")]
    F = max(2, max(f64) - min(f64))
    return min(min(f64), counts["ld"]) - F, counts["ref"] + F, counts


def metric_scale(prior_diag, minv, residual_scale=None, prior_kind=True):
    """Termination scale precedence (cg.py:89-102)."""
    if residual_scale is not None:
        return np.asarray(residual_scale, dtype=np.float64)
    if prior_diag is not None and np.all(prior_diag > 0):
        return np.asarray(prior_diag) ** -0.5
    if prior_kind:
        return np.sqrt(minv)
    raise ValueError("cannot derive the residual metric")


def rhs(X: Csr, linear, omega, prior_diag, rng):
    """b = lin + X' Omega^{1/2} eta + D^{1/2} delta; eta (n) drawn before delta (p)
    (sampler.py:94-107)."""
    eta = rng.standard_normal(X.n)
    delta = rng.standard_normal(X.p)
    b = linear + matvec_t(X, np.sqrt(omega) * eta)
    b += np.sqrt(prior_diag) * delta
    return b


def rhs_given_noise(X: Csr, linear, omega, prior_diag, eta, delta):
    b = linear + matvec_t(X, np.sqrt(omega) * eta)
    b += np.sqrt(prior_diag) * delta
    return b


# ============================================================== Polya-Gamma
_T = 0.64
_SQT = math.sqrt(_T)


def pg_batch(z, rng):
    """PG(1, z) by the alternating-series method (polya_gamma.py:39-84); the
    Generator is consumed in the same order as the reference."""
    z = np.asarray(z, dtype=np.float64)
    h = np.atleast_1d(0.5 * np.abs(z)).ravel()
    out = np.empty(h.shape)
    K = np.pi ** 2 / 8.0 + 0.5 * h ** 2
    lr = np.log(np.pi / (2.0 * K)) - K * _T
    ll = math.log(2.0) + np.logaddexp(-h + log_ndtr((_T * h - 1.0) / _SQT),
                                      h + log_ndtr(-(_T * h + 1.0) / _SQT))
    pr = expit(lr - ll)
    todo = np.arange(h.size)
    while todo.size:
        m = todo.size
        go_right = rng.random(m) < pr[todo]
        x = np.empty(m)
        nr = int(go_right.sum())
        if nr:
            x[go_right] = _T + rng.standard_exponential(nr) / K[todo][go_right]
        if nr < m:
            x[~go_right] = _tig(h[todo][~go_right], rng)
        acc = _series(x, rng)
        out[todo[acc]] = x[acc]
        todo = todo[~acc]
    return (out / 4.0).reshape(z.shape)


def _series(x, rng):
    """Series acceptance in ratio form (polya_gamma.py:87-110)."""
    u = rng.random(x.size)
    left = x <= _T
    s = np.ones_like(x)
    yes = np.zeros(x.size, dtype=bool)
    open_ = np.ones(x.size, dtype=bool)
    k = 0
    while open_.any():
        k += 1
        a = np.where(left, (2.0 * k + 1.0) * np.exp(-2.0 * k * (k + 1.0) / x),
                     (2.0 * k + 1.0) * np.exp(-0.5 * k * (k + 1.0) * np.pi ** 2 * x))
        if k % 2:
            s -= a
            hit = open_ & (u <= s)
            yes |= hit
            open_ &= ~hit
        else:
            s += a
            open_ &= u < s
    return yes


def _tig(h, rng):
    """IG(1/h, 1) truncated to (0, 0.64] (polya_gamma.py:113-147)."""
    out = np.empty(h.shape)
    far = h < 1.0 / _T
    todo = np.flatnonzero(far)
    while todo.size:
        m = todo.size
        e1 = rng.standard_exponential(m)
        e2 = rng.standard_exponential(m)
        ok = e1 * e1 <= 2.0 * e2 / _T
        x = _T / (1.0 + _T * e1) ** 2
        ok &= rng.random(m) <= np.exp(-0.5 * h[todo] ** 2 * x)
        out[todo[ok]] = x[ok]
        todo = todo[~ok]
    todo = np.flatnonzero(~far)
    while todo.size:
        m = todo.size
        mu = 1.0 / h[todo]
        y = rng.standard_normal(m) ** 2
        x = mu + 0.5 * mu * mu * y - 0.5 * mu * np.sqrt(4.0 * mu * y + (mu * y) ** 2)
        x = np.maximum(x, 1e-300)
        flip = rng.random(m) > mu / (mu + x)
        x = np.where(flip, mu * mu / x, x)
        ok = x <= _T
        out[todo[ok]] = x[ok]
        todo = todo[~ok]
    return out


def pg_mean(z):
    z = np.asarray(z, dtype=np.float64)
    small = np.abs(z) < 1e-4
    safe = np.where(small, 1.0, z)
    return np.where(small, 0.25 - z ** 2 / 48.0, np.tanh(safe / 2.0) / (2.0 * safe))


# ============================================================== Gibbs (bridge, reference)
def bridge_tau(beta_shrunk, alpha, a0, b0, rng):
    """phi = tau^-alpha ~ Gamma(a0 + p/alpha, b0 + sum|beta|^alpha) (gibbs.py:179-190)."""
    rate = b0 + float(np.sum(np.abs(beta_shrunk) ** alpha))
    shape = a0 + beta_shrunk.size / alpha
    return float((rng.gamma(shape) / rate) ** (-1.0 / alpha))


def bridge_lambda(beta_shrunk, tau, rng):
    """alpha = 1: 1/lam^2 ~ IG(tau/|beta|, 1); |beta|/tau < 1e-10 -> lam^2 ~ chi2_1
    (gibbs.py:193-214)."""
    ratio = np.abs(beta_shrunk) / tau
    lam = np.empty(ratio.shape)
    lim = ratio < 1e-10
    if lim.any():
        lam[lim] = np.maximum(np.abs(rng.standard_normal(int(lim.sum()))), 1e-150)
    rest = ~lim
    if rest.any():
        lam[rest] = np.maximum(rng.wald(1.0 / ratio[rest], 1.0), 1e-300) ** -0.5
    return lam


def bridge_log_density(beta, tau, z, y, q, alpha, a0, b0, unshrunk_sd):
    """log pi(beta, tau | y) up to a constant (gibbs.py:217-241); z = X beta."""
    loglik = float(y @ z - np.sum(np.logaddexp(0.0, z)))
    s = beta[q:]
    p = s.size
    out = loglik + p * (math.log(alpha) - math.log(2.0) - float(gammaln(1.0 / alpha)))
    out -= p * math.log(tau) + float(np.sum(np.abs(s / tau) ** alpha))
    if q:
        sd = np.asarray(unshrunk_sd, dtype=np.float64)
        fin = np.isfinite(sd)
        u = beta[:q][fin] / sd[fin]
        out -= 0.5 * float(u @ u)
        out -= float(np.sum(np.log(sd[fin]))) + 0.5 * fin.sum() * math.log(2.0 * math.pi)
    out += a0 * math.log(b0) - float(gammaln(a0)) + math.log(alpha) \
        - (alpha * a0 + 1.0) * math.log(tau) - b0 * tau ** -alpha
    return out


class Welford:
    """Running mean of scaled draws, variance of the unshrunk block (gibbs.py:139-167)."""

    def __init__(self, p_total, q):
        self.count = 0
        self.mean = np.zeros(p_total)
        self.m2 = np.zeros(q)
        self.q = q

    def update(self, scaled):
        self.count += 1
        delta = scaled - self.mean
        self.mean += delta / self.count
        if self.q:
            self.m2 += delta[:self.q] * (scaled[:self.q] - self.mean[:self.q])

    def sd(self):
        if self.count < 2 or self.q == 0:
            return None
        return np.sqrt(self.m2 / (self.count - 1))


@dataclass
class ChainResult:
    draws: np.ndarray
    tau_draws: np.ndarray
    logdens: np.ndarray
    cg_iters: np.ndarray
    beta: np.ndarray
    omega: np.ndarray
    lam: np.ndarray
    tau: float
    extra: dict


def gibbs_bridge(X: Csr, y, n_iter, seed=0, burn_in=0, thin=1, alpha=1.0, a0=1.0, b0=1.0,
                 unshrunk_sd=(), rtol=1e-6, max_iter=None, gamma_scale=1.0) -> ChainResult:
    """The reference scan (gibbs.py:260-379) for the CG sampler with the prior
    preconditioner: omega -> tau -> lambda -> beta, then the log density."""
    y = np.asarray(y, dtype=np.float64)
    q = len(unshrunk_sd)
    p_total = X.p
    p = p_total - q
    rng = np.random.default_rng(seed)
    beta = np.zeros(p_total)
    omega = np.full(X.n, 0.25)
    lam = np.ones(p)
    tau = 1.0
    sd = np.asarray(unshrunk_sd, dtype=np.float64)
    uprec = np.zeros(q)
    uprec[np.isfinite(sd)] = sd[np.isfinite(sd)] ** -2.0
    stats = Welford(p_total, q)
    n_store = max(0, (n_iter - burn_in + thin - 1) // thin) if n_iter else 0
    draws = np.empty((n_store, p_total))
    taus = np.empty(n_store)
    logd = np.empty(n_iter)
    iters = []
    stored = 0
    for t in range(1, n_iter + 1):
        omega = pg_batch(matvec(X, beta), rng)                          # gibbs.py:170-176
        y_prime = (y - 0.5) / omega
        tau = bridge_tau(beta[q:], alpha, a0, b0, rng)                   # gibbs.py:179-190
        lam = bridge_lambda(beta[q:], tau, rng)                          # gibbs.py:193-214
        prior = np.concatenate([uprec, (tau * lam) ** -2.0])             # gibbs.py:334
        lin = matvec_t(X, omega * y_prime)                               # sampler.py:86-91
        if q:
            s = stats.sd()
            g = gamma_scale * np.maximum(np.minimum(sd, 10.0) if s is None else s, 1e-3)
        else:
            g = np.zeros(0)                                              # precond.py:137-153
        minv = np.concatenate([g ** 2, (tau * lam) ** 2])                # precond.py:120-134
        scale = np.concatenate([g, tau * lam])
        x0 = np.zeros(p_total) if stats.count == 0 else \
            np.concatenate([np.ones(q), tau * lam]) * stats.mean         # cg.py:195-211
        b = rhs(X, lin, omega, prior, rng)
        res = pcg(lambda v: phi_apply(X, omega, prior, v), b, minv, scale, x0,
                  max_iter=max_iter, rtol=rtol)
        iters.append(res.iterations)
        beta = res.x
        logd[t - 1] = bridge_log_density(beta, tau, matvec(X, beta), y, q, alpha, a0, b0, sd)
        stats.update(np.concatenate([beta[:q], beta[q:] / (tau * lam)]))
        if t > burn_in and (t - burn_in - 1) % thin == 0:
            draws[stored] = beta
            taus[stored] = tau
            stored += 1
    return ChainResult(draws[:stored], taus[:stored], logd, np.array(iters), beta, omega, lam, tau,
                       {"stats_mean": stats.mean.copy()})


# ============================================================== horseshoe (NEW, no reference)
def ig_draw(shape, rate, rng):
    """Inverse-gamma(shape, rate) = rate / Gamma(shape, 1), one independent
    Gamma variate per element of `rate`."""
    if np.ndim(rate) == 0:
        return rate / rng.gamma(shape)
    return rate / rng.gamma(shape, size=np.shape(rate))


def horseshoe_scales(beta_shrunk, lam2, nu, tau2, xi, rng):
    """Half-Cauchy local and global scales through the auxiliary inverse-gamma
    representation (Makalic & Schmidt 2016):
        lam_j^2 | nu_j ~ IG(1/2, 1/nu_j),  nu_j ~ IG(1/2, 1)
        tau^2   | xi   ~ IG(1/2, 1/xi),    xi   ~ IG(1/2, 1)
    Scan order: xi | tau, tau^2 | beta, lam, xi, nu | lam,
    lam^2 | beta, tau, nu.  Returns (lam2, nu, tau2, xi)."""
    p = beta_shrunk.size
    b2 = beta_shrunk ** 2
    xi = ig_draw(1.0, 1.0 + 1.0 / tau2, rng)
    tau2 = ig_draw(0.5 * (p + 1), 1.0 / xi + 0.5 * float(np.sum(b2 / lam2)), rng)
    tau2 = min(max(tau2, 1e-300), 1e300)
    nu = ig_draw(1.0, 1.0 + 1.0 / lam2, rng)
    lam2 = ig_draw(1.0, 1.0 / nu + 0.5 * b2 / tau2, rng)
    lam2 = np.clip(lam2, 1e-300, 1e300)
    return lam2, nu, tau2, xi


def horseshoe_log_density(beta, tau, lam, z, y, q, unshrunk_sd):
    """log p(y | beta) + log N(beta_s; 0, tau^2 lam^2) + log C+(lam) + log C+(tau),
    with the unshrunk block's Gaussian/flat prior (the horseshoe analogue of
    gibbs.py:217-241, conditional on lambda because the horseshoe marginal
    has no closed form)."""
    loglik = float(y @ z - np.sum(np.logaddexp(0.0, z)))
    s = beta[q:]
    sc = tau * lam
    out = loglik - float(np.sum(np.log(sc))) - 0.5 * float(np.sum((s / sc) ** 2)) \
        - 0.5 * s.size * math.log(2.0 * math.pi)
    out += float(np.sum(math.log(2.0 / math.pi) - np.log1p(lam ** 2)))
    out += math.log(2.0 / math.pi) - math.log1p(tau ** 2)
    if q:
        sd = np.asarray(unshrunk_sd, dtype=np.float64)
        fin = np.isfinite(sd)
        u = beta[:q][fin] / sd[fin]
        out -= 0.5 * float(u @ u) + float(np.sum(np.log(sd[fin]))) \
            + 0.5 * fin.sum() * math.log(2.0 * math.pi)
    return out


def gibbs_horseshoe(X: Csr, y, n_iter, seed=0, burn_in=0, thin=1, unshrunk_sd=(),
                    rtol=1e-6, max_iter=None, gamma_scale=1.0) -> ChainResult:
    """Horseshoe logistic Gibbs sampler with the reference's beta update
    (prior-preconditioned CG, warm start, gamma policy)."""
    y = np.asarray(y, dtype=np.float64)
    q = len(unshrunk_sd)
    p_total = X.p
    p = p_total - q
    rng = np.random.default_rng(seed)
    beta = np.zeros(p_total)
    omega = np.full(X.n, 0.25)
    lam2, nu, tau2, xi = np.ones(p), np.ones(p), 1.0, 1.0
    sd = np.asarray(unshrunk_sd, dtype=np.float64)
    uprec = np.zeros(q)
    uprec[np.isfinite(sd)] = sd[np.isfinite(sd)] ** -2.0
    stats = Welford(p_total, q)
    n_store = max(0, (n_iter - burn_in + thin - 1) // thin) if n_iter else 0
    draws = np.empty((n_store, p_total))
    taus = np.empty(n_store)
    logd = np.empty(n_iter)
    iters = []
    stored = 0
    z = matvec(X, beta)
    kappa = y - 0.5
    for t in range(1, n_iter + 1):
        omega = pg_batch(z, rng)
        lam2, nu, tau2, xi = horseshoe_scales(beta[q:], lam2, nu, tau2, xi, rng)
        tau = math.sqrt(tau2)
        lam = np.sqrt(lam2)
        prior = np.concatenate([uprec, (tau * lam) ** -2.0])
        lin = matvec_t(X, kappa)
        if q:
            s = stats.sd()
            g = gamma_scale * np.maximum(np.minimum(sd, 10.0) if s is None else s, 1e-3)
        else:
            g = np.zeros(0)
        minv = np.concatenate([g ** 2, (tau * lam) ** 2])
        scale = np.concatenate([g, tau * lam])
        x0 = np.zeros(p_total) if stats.count == 0 else \
            np.concatenate([np.ones(q), tau * lam]) * stats.mean
        b = rhs(X, lin, omega, prior, rng)
        res = pcg(lambda v: phi_apply(X, omega, prior, v), b, minv, scale, x0,
                  max_iter=max_iter, rtol=rtol)
        iters.append(res.iterations)
        beta = res.x
        z = matvec(X, beta)
        logd[t - 1] = horseshoe_log_density(beta, tau, lam, z, y, q, sd)
        stats.update(np.concatenate([beta[:q], beta[q:] / (tau * lam)]))
        if t > burn_in and (t - burn_in - 1) % thin == 0:
            draws[stored] = beta
            taus[stored] = tau
            stored += 1
    return ChainResult(draws[:stored], taus[:stored], logd, np.array(iters), beta, omega,
                       np.sqrt(lam2), math.sqrt(tau2), {"nu": nu, "xi": xi})
