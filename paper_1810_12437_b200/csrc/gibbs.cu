// Device Gibbs scan for sparse Bayesian logistic regression (reference:
// pkg/src/priorcg/gibbs.py:260-379).  One call = one scan, no host sync:
//   omega | beta        Polya-Gamma            (gibbs.py:170-176)
//   tau   | beta (...)  global scale           (gibbs.py:179-190; horseshoe: new)
//   lam   | beta, tau   local scales           (gibbs.py:193-214; horseshoe: new)
//   beta  | omega, lam, tau  randomised RHS + persistent PCG (gibbs.py:334-351)
//   log density, Welford warm-start statistics, stored draw (gibbs.py:362-369)
#include <cuda_runtime.h>

#include <cmath>
#include <string>

#include "gibbs_math.cuh"
#include "internal.cuh"
#include "rowsplit.h"

namespace {

// ---------------------------------------------------------------- CSR with log-likelihood
struct EpiLogit {  // z_i = v0 + s (+ dense row term); acc += y_i z_i - log(1 + e^{z_i})
  double* z;
  const double* y;
  double v0;
  double acc;
  bool multi;
  AffRow ar;
  __device__ void emit(long long seg, double s) {
    if (multi) {
      z[seg] = s;
      return;
    }
    const double zi = v0 + s + (ar.q ? ar(seg) : 0.0);
    z[seg] = zi;
    const double yi = __ldg(y + seg);
    acc += yi * zi - (fmax(zi, 0.0) + log1p(exp(-fabs(zi))));
  }
};

template <int kT, int kRingB>
__global__ void __launch_bounds__(kT, 1) k_csr_logit(DesignDev D, const double* beta, const double* y,
                                                           double* z_or_part, double* part, const double* cbuf) {
  extern __shared__ __align__(128) double sv[];
  __shared__ double red[64];
  FillVecRef f{beta, D.lead(), 0, D.aff.sc};
  const double v0 = row_const(D, beta, cbuf);
  EpiLogit e{z_or_part, y, v0, 0.0, D.csr.nslab > 1, aff_row(D, cbuf)};
  run_pass<kRingB>(D.csr, sv, f, e);
  const double t = block_sum(e.acc, red);
  if (threadIdx.x == 0) part[blockIdx.x * kPartStride] = t;
}

// multi column slab: z_i = v0 + sum_s zpart, log-likelihood partials per CTA
__global__ void __launch_bounds__(kThreads) k_rows_logit(DesignDev D, const double* zpart, const double* beta,
                                                         const double* y, double* z, double* part,
                                                         const double* cbuf) {
  __shared__ double red[64];
  const double v0 = row_const(D, beta, cbuf);
  const AffRow ar = aff_row(D, cbuf);
  double acc = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < D.n; i += (long long)gridDim.x * blockDim.x) {
    double zi = 0.0;
    for (int s = 0; s < D.csr.nslab; ++s) zi += zpart[(long long)s * D.n + i];
    zi += v0;
    if (ar.q) zi += ar(i);
    z[i] = zi;
    const double yi = __ldg(y + i);
    acc += yi * zi - (fmax(zi, 0.0) + log1p(exp(-fabs(zi))));
  }
  const double t = block_sum(acc, red);
  if (threadIdx.x == 0) part[blockIdx.x * kPartStride] = t;
}

// Validation kernel (pcgs_scale_draws): mode 0 = count independent global
// draws from (acc, tau_old) with the scan keys t = 1..count; mode 1 = count
// independent local draws of coefficient b from lam_old (element keys);
// mode 2 / 3 = ONE thread iterating the global / local update count times
// from tau_old / lam_old (the auxiliary-variable Gibbs chain, whose
// stationary law is the exact conditional of tau given acc / of lam given b).
__global__ void k_scale_draws(int prior, int mode, long long count, double b_or_acc, double tau, double lam_old,
                              long long p, double a0, double b0, double alpha, unsigned long long seed,
                              double* out, double* aux) {
  if (mode >= 2) {
    if (blockIdx.x != 0 || threadIdx.x != 0) return;
    double cur = mode == 2 ? tau : lam_old;
    for (long long i = 0; i < count; ++i) {
      double a = 0.0;
      if (mode == 2) {
        Philox R(seed, kStreamGlobal ^ (unsigned long long)(i + 1), 0u);
        cur = global_draw(prior, a0, b0, alpha, p, b_or_acc, cur, R, &a);
      } else {
        Philox R(seed, kStreamLocal ^ (unsigned long long)(i + 1), 0u);
        cur = local_draw(prior, b_or_acc, tau, cur, R, &a);
      }
      out[i] = cur;
      if (aux) aux[i] = a;
    }
    return;
  }
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count; i += (long long)gridDim.x * blockDim.x) {
    double a = 0.0, v;
    if (mode == 0) {
      Philox R(seed, kStreamGlobal ^ (unsigned long long)(i + 1), 0u);
      v = global_draw(prior, a0, b0, alpha, p, b_or_acc, tau, R, &a);
    } else {
      Philox R(seed, kStreamLocal ^ 1ull, (unsigned)i);
      v = local_draw(prior, b_or_acc, tau, lam_old, R, &a);
    }
    out[i] = v;
    if (aux) aux[i] = a;
  }
}

// Partial-sum lines (one 128-byte line per CTA, kPartStride doubles):
//   [c*16 + 0]  log-likelihood of X beta (CSR pass)
//   [c*16 + 1]  log-prior terms of the current draw (k_stats)
//   [c*16 + 2]  sum feeding the next tau update (k_stats / k_tau_sums)
__device__ __forceinline__ double tau_term(const pcgs_gibbs_t& G, double b, long long k) {
  if (G.prior == 0) return G.alpha == 1.0 ? fabs(b) : pow(fabs(b), G.alpha);
  const double l = G.lam[k];
  return b * b / (l * l);
}

// column scale of the reparametrised coefficient j (standardised designs)
__device__ __forceinline__ double col_scale(const pcgs_gibbs_t& G, long long j) {
  return G.cscale ? G.cscale[j] : 1.0;
}

// partial sums for the tau update from the current beta / lambda (chain start)
__global__ void __launch_bounds__(256) k_tau_sums(pcgs_gibbs_t G, long long pt) {
  __shared__ double red[64];
  const int q = G.q;
  double acc = 0.0;
  for (long long j = q + blockIdx.x * (long long)blockDim.x + threadIdx.x; j < pt; j += (long long)gridDim.x * blockDim.x)
    acc += tau_term(G, col_scale(G, j) * G.beta[j], j - q);
  acc = block_sum(acc, red);
  if (threadIdx.x == 0) G.part[(long long)blockIdx.x * kPartStride + 2] = acc;
}

// k_global: one warp.  Bridge: phi = tau^-alpha ~ Gamma(a0 + p/alpha, b0 + sum|beta|^alpha)
// (gibbs.py:179-190).  Horseshoe: xi | tau ~ IG(1, 1 + 1/tau^2), then
// tau^2 | beta, lam, xi ~ IG((p+1)/2, 1/xi + sum beta^2 / (2 lam^2)).
__global__ void __launch_bounds__(32) k_global(pcgs_gibbs_t G, long long pt, int t, int ncta) {
  const int lane = threadIdx.x;
  double acc = 0.0;
  for (int c = lane; c < ncta; c += 32) acc += G.part[(long long)c * kPartStride + 2];
  acc = warp_sum(acc);
  if (lane == 0) {
    Philox R(G.seed, kStreamGlobal ^ (unsigned long long)t, 0u);
    double xi = G.scal[1];
    const double tau = global_draw(G.prior, G.a0, G.b0, G.alpha, pt - G.q, acc, G.scal[0], R, &xi);
    if (G.prior != 0) G.scal[1] = xi;
    G.scal[0] = tau;
    if (!(tau > 0.0) || !isfinite(tau)) G.results[8 * (t - 1) + 4] = 1;
  }
}

// k_local: elementwise over p_total.  Local scales (bridge: gibbs.py:193-214;
// horseshoe: nu_j ~ IG(1, 1 + 1/lam_j^2), lam_j^2 ~ IG(1, 1/nu_j + beta_j^2/(2 tau^2))),
// then the prior diagonal (gibbs.py:334), the preconditioner (precond.py:120-153),
// the metric scale [gamma, tau lam] (gibbs.py:348) and the warm start (cg.py:195-211)
// written into beta.
__global__ void k_local(pcgs_gibbs_t G, long long pt, int t, int count) {
  const int q = G.q;
  const double tau = G.scal[0];
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < pt; j += (long long)gridDim.x * blockDim.x) {
    const double cs = col_scale(G, j);
    if (j < q) {
      // unshrunk coefficient: prior precision, gamma policy (precond.py:137-153)
      double sd;
      if (count >= 2) sd = sqrt(G.m2[j] / (double)(count - 1));
      else sd = fmin(G.usd_sd[j] / cs, 10.0);
      const double gam = G.gamma_scale * fmax(sd, 1e-3);
      G.prior_diag[j] = G.usd_prec[j] * cs * cs;
      G.minv[j] = gam * gam;
      G.scale[j] = gam;
      G.beta[j] = count > 0 ? G.mean[j] : 0.0;
      continue;
    }
    const long long k = j - q;
    double lam = G.lam[k];
    if (!G.fixed_lam) {
      Philox R(G.seed, kStreamLocal ^ (unsigned long long)t, (unsigned)k);
      double nu = 0.0;
      lam = local_draw(G.prior, cs * G.beta[j], tau, lam, R, &nu);
      if (G.prior != 0) G.nu[k] = nu;
      G.lam[k] = lam;
    }
    if (!(lam > 0.0) || !isfinite(lam)) G.results[8 * (t - 1) + 4] = 1;
    const double tl = tau * lam / cs;  // prior sd of the (reparametrised) coefficient
    G.prior_diag[j] = 1.0 / (tl * tl);
    G.minv[j] = tl * tl;
    G.scale[j] = tl;
    G.beta[j] = count > 0 ? tl * G.mean[j] : 0.0;
  }
}

// identity / Jacobi preconditioners (gibbs.py:244-257) overwrite minv
__global__ void k_precond(pcgs_gibbs_t G, long long pt, const double* diag_phi) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < pt; j += (long long)gridDim.x * blockDim.x)
    G.minv[j] = G.precond == 1 ? 1.0 : 1.0 / diag_phi[j];
}

// k_post: one warp.  log density (bridge: gibbs.py:217-241; horseshoe: joint
// density given lambda) from the partial lines.
__global__ void __launch_bounds__(32) k_post(pcgs_gibbs_t G, long long pt, int t, int ncta_ll, int ncta_st) {
  const int lane = threadIdx.x;
  double ll = 0.0, pr = 0.0;
  for (int c = lane; c < ncta_ll; c += 32) ll += G.part[(long long)c * kPartStride];
  for (int c = lane; c < ncta_st; c += 32) pr += G.part[(long long)c * kPartStride + 1];
  ll = warp_sum(ll);
  pr = warp_sum(pr);
  if (lane == 0) {
    const long long p = pt - G.q;
    const double tau = G.scal[0];
    double out = ll + pr;
    if (G.prior == 0) {
      const double a = G.alpha;
      out += (double)p * (log(a) - log(2.0) - lgamma(1.0 / a)) - (double)p * log(tau);
      out += G.a0 * log(G.b0) - lgamma(G.a0) + log(a) - (a * G.a0 + 1.0) * log(tau) - G.b0 * pow(tau, -a);
    } else {
      out += log(2.0 / M_PI) - log1p(tau * tau);
    }
    G.logdens[t - 1] = out;
  }
}

// Welford update of the scaled draws [beta_q, beta/(tau lam)] (gibbs.py:139-167),
// the stored draw (gibbs.py:366-369), and per-CTA partials of the log-prior
// terms of this draw and of the sum the next tau update needs.
__global__ void __launch_bounds__(256) k_stats(pcgs_gibbs_t G, long long pt, int count_new, int slot) {
  __shared__ double red[64];
  const int q = G.q;
  const double tau = G.scal[0];
  double lp = 0.0, ts = 0.0;
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < pt; j += (long long)gridDim.x * blockDim.x) {
    const double bt = G.beta[j];             // sampled coordinate
    const double b = col_scale(G, j) * bt;   // model coefficient (shrinkage, prior)
    const double scaled = j < q ? bt : b / (tau * G.lam[j - q]);
    const double delta = scaled - G.mean[j];
    const double m = G.mean[j] + delta / (double)count_new;
    G.mean[j] = m;
    if (j < q) G.m2[j] += delta * (scaled - m);
    if (slot >= 0) G.draws[(long long)slot * pt + j] = bt;
    if (slot >= 0 && j == 0) G.tau_draws[slot] = tau;
    if (j < q) {
      const double sd = G.usd_sd[j];
      if (isfinite(sd)) {
        const double u = b / sd;
        lp -= 0.5 * u * u + log(sd) + 0.5 * log(2.0 * M_PI);
      }
    } else {
      const long long k = j - q;
      if (G.prior == 0) {
        lp -= G.alpha == 1.0 ? fabs(b / tau) : pow(fabs(b / tau), G.alpha);
      } else {
        const double l = G.lam[k];
        const double sc = tau * l;
        const double u = b / sc;
        lp += -log(sc) - 0.5 * u * u - 0.5 * log(2.0 * M_PI) + log(2.0 / M_PI) - log1p(l * l);
      }
      ts += tau_term(G, b, k);
    }
  }
  block_sum2(lp, ts, red);
  if (threadIdx.x == 0) {
    G.part[(long long)blockIdx.x * kPartStride + 1] = lp;
    G.part[(long long)blockIdx.x * kPartStride + 2] = ts;
  }
}

int launch_logit(pcgs_design* d, pcgs_gibbs_t* g, cudaStream_t s) {
  const DesignDev& D = d->dev;
  Scratch S(s);
  double* cbuf;
  int rc;
  if ((rc = aff_pre(d, g->beta, S, s, &cbuf))) return rc;
  if (D.csr.nslab == 1) {
    PASS_LAUNCH(k_csr_logit, D, smem_bytes(D), s, D, g->beta, g->y, g->z, g->part, cbuf);
  } else {
    double* zp = S.get<double>((size_t)D.csr.nslab * D.n);
    if (!zp) return fail(PCGS_ENOMEM, "scratch allocation failed");
    PASS_LAUNCH(k_csr_logit, D, smem_bytes(D), s, D, g->beta, g->y, zp, g->part, cbuf);
    k_rows_logit<<<D.G, kThreads, 0, s>>>(D, zp, g->beta, g->y, g->z, g->part, cbuf);
  }
  CUDA_TRY(cudaGetLastError());
  return PCGS_OK;
}

}  // namespace

extern "C" {

int pcgs_scale_draws(int prior, int mode, int64_t count, double b_or_acc, double tau, double lam_old, int64_t p,
                     double a0, double b0, double alpha, uint64_t seed, double* out, double* aux,
                     pcgs_stream_t stream) {
  if ((prior != 0 && prior != 1) || mode < 0 || mode > 3 || count < 0 || (count > 0 && !out))
    return fail(PCGS_EINVAL, "bad argument");
  if (prior == 0 && mode % 2 == 1 && alpha != 1.0) return fail(PCGS_EUNSUP, "bridge local draws need alpha = 1");
  if (count == 0) return PCGS_OK;
  const int blocks = mode >= 2 ? 1 : (int)std::min<int64_t>((count + 255) / 256, 148 * 8);
  k_scale_draws<<<blocks, mode >= 2 ? 32 : 256, 0, (cudaStream_t)stream>>>(
      prior, mode, count, b_or_acc, tau, lam_old, p, a0, b0, alpha, seed, out, aux);
  CUDA_TRY(cudaGetLastError());
  return PCGS_OK;
}

int pcgs_gibbs_init(pcgs_design_t d, pcgs_gibbs_t* g, pcgs_stream_t stream) {
  if (!d || !g || !g->beta || !g->z || !g->y || !g->part) return fail(PCGS_EINVAL, "null argument");
  int rc0;
  if ((rc0 = raise_smem_limit(k_csr_logit<512, 2>)) || (rc0 = raise_smem_limit(k_csr_logit<1024, 1>))) return rc0;
  k_tau_sums<<<d->dev.G, 256, 0, (cudaStream_t)stream>>>(*g, d->dev.pt);
  CUDA_TRY(cudaGetLastError());
  return launch_logit(d, g, (cudaStream_t)stream);
}

int pcgs_gibbs_scan_begin(pcgs_design_t d, pcgs_gibbs_t* g, int32_t t, pcgs_stream_t stream) {
  if (!d || !g || t < 1) return fail(PCGS_EINVAL, "bad argument");
  const DesignDev& D = d->dev;
  cudaStream_t s = (cudaStream_t)stream;
  int rc;
  // omega | beta (z = X beta of the previous scan), then tau | beta
  if (!g->fixed_omega) {
    if ((rc = pcgs_pg_draw(g->z, D.n, g->seed, (uint64_t)t, g->omega, stream))) return rc;
  }
  if (!g->fixed_tau) k_global<<<1, 32, 0, s>>>(*g, D.pt, t, D.G);
  CUDA_TRY(cudaGetLastError());
  return PCGS_OK;
}

}  // extern "C"

// The halves of scan_end around the beta solve (shared by the single-chain
// and the batched scans).
static int scan_prep(pcgs_design* d, pcgs_gibbs_t* g, int32_t t, int32_t count, cudaStream_t s) {
  const DesignDev& D = d->dev;
  const long long pt = D.pt;
  const int eblocks = (int)std::min<long long>((pt + 255) / 256, 4 * D.G);
  int rc;
  // lambda | beta, tau; prior diagonal, M^-1, metric scale, x0
  k_local<<<eblocks, 256, 0, s>>>(*g, pt, t, count);
  if (g->precond == 2) {
    if ((rc = pcgs_phi_diagonal(d, g->omega, g->prior_diag, g->b, s))) return rc;
    k_precond<<<eblocks, 256, 0, s>>>(*g, pt, g->b);
  } else if (g->precond == 1) {
    k_precond<<<eblocks, 256, 0, s>>>(*g, pt, nullptr);
  }
  CUDA_TRY(cudaGetLastError());
  // randomised right-hand side (one fused X' pass)
  return pcgs_rhs(d, g->kappa, g->omega, g->prior_diag, nullptr, nullptr, nullptr, g->seed, (uint64_t)t, g->b, s);
}

static int scan_post(pcgs_design* d, pcgs_gibbs_t* g, int32_t t, int32_t count, int32_t slot, cudaStream_t s) {
  const DesignDev& D = d->dev;
  int rc;
  // z = X beta with the log-likelihood, statistics, stored draw, log density
  if ((rc = launch_logit(d, g, s))) return rc;
  k_stats<<<D.G, 256, 0, s>>>(*g, D.pt, count + 1, slot);
  k_post<<<1, 32, 0, s>>>(*g, D.pt, t, D.G, D.G);
  CUDA_TRY(cudaGetLastError());
  return PCGS_OK;
}

// Chain-minor packing of the R chains' solve inputs / unpacking of the
// solutions and reports (batched scan).
struct PackArgs {
  const double* src[8];
  double* dst;
};
__global__ void k_pack(PackArgs A, int R, long long m) {
  const long long nr = m * R;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nr; e += (long long)gridDim.x * blockDim.x)
    A.dst[e] = A.src[e % R][e / R];
}
struct UnpackArgs {
  double* dst[8];
  const double* src;
};
__global__ void k_unpack(UnpackArgs A, int R, long long m) {
  const long long nr = m * R;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nr; e += (long long)gridDim.x * blockDim.x)
    A.dst[e % R][e / R] = A.src[e];
}
struct ResultArgs {
  int* dst[8];
};
__global__ void k_results(ResultArgs A, const int* res, int R) {
  const int i = threadIdx.x;
  if (i < 4 * R) A.dst[i / 4][i % 4] = res[i];
}

extern "C" {

int pcgs_gibbs_scan_end(pcgs_design_t d, pcgs_gibbs_t* g, int32_t t, int32_t count, int32_t slot,
                        pcgs_stream_t stream) {
  if (!d || !g || t < 1) return fail(PCGS_EINVAL, "bad argument");
  cudaStream_t s = (cudaStream_t)stream;
  int rc;
  if ((rc = scan_prep(d, g, t, count, s))) return rc;
  if ((rc = pcgs_pcg(d, g->omega, g->prior_diag, g->minv, g->scale, g->b, g->beta, g->max_iter, g->rtol, g->trace,
                     g->alphas, g->betas, g->results + 8 * (t - 1), stream)))
    return rc;
  return scan_post(d, g, t, count, slot, s);
}

int pcgs_batch_gibbs_scan(pcgs_design_t d, pcgs_batch_t bt, pcgs_gibbs_t* const* gs, int32_t nchains, int32_t t,
                          const int32_t* counts, const int32_t* slots, pcgs_stream_t stream) {
  if (!d || !bt || !gs || !counts || !slots || t < 1) return fail(PCGS_EINVAL, "bad argument");
  int64_t info[16];
  int rc;
  if ((rc = pcgs_batch_info(bt, info))) return rc;
  const int R = (int)info[10];
  if (nchains != R) return fail(PCGS_EINVAL, "nchains must equal the batch store's chain count");
  const DesignDev& D = d->dev;
  if (info[0] != D.n || info[2] != D.pt) return fail(PCGS_EINVAL, "batch store and design differ in shape");
  for (int c = 0; c < R; ++c) {
    if (!gs[c]) return fail(PCGS_EINVAL, "null chain");
    if (gs[c]->max_iter != gs[0]->max_iter || gs[c]->rtol != gs[0]->rtol)
      return fail(PCGS_EINVAL, "batched chains must share max_iter and rtol");
  }
  cudaStream_t s = (cudaStream_t)stream;
  // each chain's own omega, tau, lambda, prior diagonal, M^-1, scale, x0, RHS
  for (int c = 0; c < R; ++c) {
    if ((rc = pcgs_gibbs_scan_begin(d, gs[c], t, stream))) return rc;
    if ((rc = scan_prep(d, gs[c], t, counts[c], s))) return rc;
  }
  // R solves in one batched kernel on chain-minor copies
  const long long n = D.n, pt = D.pt;
  const int mi = gs[0]->max_iter;
  Scratch S(s);
  double* om = S.get<double>((size_t)n * R);
  double* vec = S.get<double>((size_t)pt * R * 5);
  double* tr = S.get<double>((size_t)R * (mi + 1) * 3);
  int* res = S.get<int>((size_t)R * 4);
  if (!om || !vec || !tr || !res) return fail(PCGS_ENOMEM, "scratch allocation failed");
  double *dg = vec, *mv = vec + pt * R, *sc = vec + 2 * pt * R, *bb = vec + 3 * pt * R, *xx = vec + 4 * pt * R;
  const int blocks = 4 * D.G;
  {
    PackArgs P;
    for (int c = 0; c < R; ++c) P.src[c] = gs[c]->omega;
    P.dst = om;
    k_pack<<<blocks, 256, 0, s>>>(P, R, n);
    for (int f = 0; f < 5; ++f) {
      for (int c = 0; c < R; ++c) {
        pcgs_gibbs_t* g = gs[c];
        P.src[c] = f == 0 ? g->prior_diag : f == 1 ? g->minv : f == 2 ? g->scale : f == 3 ? g->b : g->beta;
      }
      P.dst = vec + (long long)f * pt * R;
      k_pack<<<blocks, 256, 0, s>>>(P, R, pt);
    }
    CUDA_TRY(cudaGetLastError());
  }
  double *trace = tr, *alphas = tr + (size_t)R * (mi + 1), *betas = alphas + (size_t)R * (mi + 1);
  if ((rc = pcgs_batch_pcg(bt, om, dg, mv, sc, bb, xx, mi, gs[0]->rtol, trace, alphas, betas, res, stream)))
    return rc;
  {
    UnpackArgs U;
    for (int c = 0; c < R; ++c) U.dst[c] = gs[c]->beta;
    U.src = xx;
    k_unpack<<<blocks, 256, 0, s>>>(U, R, pt);
    ResultArgs RA;
    for (int c = 0; c < R; ++c) RA.dst[c] = gs[c]->results + 8 * (t - 1);
    k_results<<<1, 32, 0, s>>>(RA, res, R);
    CUDA_TRY(cudaGetLastError());
    for (int c = 0; c < R; ++c) {
      CUDA_TRY(cudaMemcpyAsync(gs[c]->trace, trace + (size_t)c * (mi + 1), sizeof(double) * (mi + 1),
                               cudaMemcpyDeviceToDevice, s));
      CUDA_TRY(cudaMemcpyAsync(gs[c]->alphas, alphas + (size_t)c * mi, sizeof(double) * mi,
                               cudaMemcpyDeviceToDevice, s));
      CUDA_TRY(cudaMemcpyAsync(gs[c]->betas, betas + (size_t)c * mi, sizeof(double) * mi,
                               cudaMemcpyDeviceToDevice, s));
    }
  }
  for (int c = 0; c < R; ++c)
    if ((rc = scan_post(d, gs[c], t, counts[c], slots[c], s))) return rc;
  return PCGS_OK;
}

int pcgs_gibbs_scan(pcgs_design_t d, pcgs_gibbs_t* g, int32_t t, int32_t count, int32_t slot,
                    pcgs_stream_t stream) {
  int rc = pcgs_gibbs_scan_begin(d, g, t, stream);
  if (rc) return rc;
  return pcgs_gibbs_scan_end(d, g, t, count, slot, stream);
}

// ---------------------------------------------------------------------------
// Row-split scan (BASELINE config 5): rows of X over the
// ranks of a pcgs_rs context, p-vectors replicated.  Per scan: PG draws on
// each rank's rows (Philox keyed by global row, so the draws are those of the
// unsharded chain), tau / lambda replicated (same keys everywhere), RHS and
// PCG in the fused row-split kernel (one exchange for b, one per iteration),
// X beta and the log-likelihood per rank, one scalar exchange for the log
// density, replicated statistics.
// ---------------------------------------------------------------------------
static int rs_logit(pcgs_rs_t rs, pcgs_gibbs_t* g, const pcgs_rs_rows_t* rows, cudaStream_t s) {
  for (int l = 0; l < rs_n_local(rs); ++l) {
    pcgs_design_t d;
    int64_t row0;
    int rc;
    if ((rc = rs_local(rs, l, &d, &row0))) return rc;
    if ((rc = raise_smem_limit(k_csr_logit<512, 2>)) || (rc = raise_smem_limit(k_csr_logit<1024, 1>))) return rc;
    pcgs_gibbs_t gl = *g;
    gl.y = rows[l].y;
    gl.z = rows[l].z;
    gl.part = rows[l].part;
    if ((rc = launch_logit(d, &gl, s))) return rc;
  }
  return PCGS_OK;
}

int pcgs_rs_gibbs_init(pcgs_rs_t rs, pcgs_gibbs_t* g, const pcgs_rs_rows_t* rows, pcgs_stream_t stream) {
  if (!rs || !g || !rows || !g->beta || !g->part) return fail(PCGS_EINVAL, "null argument");
  if (g->precond == 2) return fail(PCGS_EUNSUP, "row split: the Jacobi preconditioner is not sharded");
  if (g->cscale) return fail(PCGS_EUNSUP, "row split: standardised designs are not sharded");
  pcgs_design_t d;
  int64_t row0;
  int rc;
  if ((rc = rs_local(rs, 0, &d, &row0))) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  k_tau_sums<<<rs_grid(rs), 256, 0, s>>>(*g, d->dev.pt);
  CUDA_TRY(cudaGetLastError());
  return rs_logit(rs, g, rows, s);
}

int pcgs_rs_gibbs_scan(pcgs_rs_t rs, pcgs_gibbs_t* g, const pcgs_rs_rows_t* rows, int32_t t, int32_t count,
                       int32_t slot, pcgs_stream_t stream) {
  if (!rs || !g || !rows || t < 1) return fail(PCGS_EINVAL, "bad argument");
  const int nl = rs_n_local(rs), Gr = rs_grid(rs);
  cudaStream_t s = (cudaStream_t)stream;
  const double* omegas[8];
  const double* kappas[8];
  long long pt = 0;
  int rc;
  for (int l = 0; l < nl; ++l) {
    pcgs_design_t d;
    int64_t row0;
    if ((rc = rs_local(rs, l, &d, &row0))) return rc;
    pt = d->dev.pt;
    if (!g->fixed_omega &&
        (rc = pcgs_pg_draw_rows(rows[l].z, d->dev.n, row0, g->seed, (uint64_t)t, rows[l].omega, stream)))
      return rc;
    omegas[l] = rows[l].omega;
    kappas[l] = rows[l].kappa;
  }
  if (!g->fixed_tau) k_global<<<1, 32, 0, s>>>(*g, pt, t, Gr);
  const int eblocks = (int)std::min<long long>((pt + 255) / 256, 4 * Gr);
  k_local<<<eblocks, 256, 0, s>>>(*g, pt, t, count);
  if (g->precond == 1) k_precond<<<eblocks, 256, 0, s>>>(*g, pt, nullptr);
  CUDA_TRY(cudaGetLastError());
  RsSolve S{omegas, kappas, g->seed, (uint64_t)t, g->b, g->prior_diag, g->minv, g->scale, nullptr, g->beta,
            g->max_iter, g->rtol, g->trace, g->alphas, g->betas, g->results + 8 * (t - 1)};
  if ((rc = rs_solve(rs, S, s))) return rc;
  if ((rc = rs_logit(rs, g, rows, s))) return rc;
  const double* parts[8];
  for (int l = 0; l < nl; ++l) parts[l] = rows[l].part;
  if ((rc = rs_sum(rs, parts, g->part, s))) return rc;  // line 0, slot 0: total log-likelihood
  k_stats<<<Gr, 256, 0, s>>>(*g, pt, count + 1, slot);
  k_post<<<1, 32, 0, s>>>(*g, pt, t, 1, Gr);
  CUDA_TRY(cudaGetLastError());
  return PCGS_OK;
}

}  // extern "C"
