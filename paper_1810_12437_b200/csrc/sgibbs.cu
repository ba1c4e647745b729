// Fused batched Gibbs chains (BASELINE config 4): R chains run whole Gibbs
// scans inside ONE persistent cooperative kernel on the sliced store, each
// at its own pace.  Every batched iteration walks the pattern once for all R
// chains (CSR pass | row combine | CSC pass | column step | direction), and
// what a chain's lanes compute in it depends on the chain's state:
//
//   SOLVE  one PCG iteration of the chain's beta solve (cg.py:105-192);
//   GIBBS  the updates between two solves (gibbs.py:300-351): the CSR pass
//          gives z = X beta_t, the combine draws omega_{t+1} ~ PG(1, z)
//          (polya_gamma.py:39-147) and u = kappa + sqrt(omega) eta, the CSC
//          pass gives X'u, the step draws tau_{t+1} | beta_t, lambda_t
//          (gibbs.py:179-190; horseshoe: DESIGN.md §5) and lambda_{t+1}
//          (gibbs.py:193-214), forms the prior diagonal, M^-1, the metric
//          scale, x0 (cg.py:195-211) and b = X'u + sqrt(d) delta
//          (sampler.py:94-107), and writes the log density of scan t
//          (gibbs.py:217-241);
//   INIT   the solve's first application r = b - Phi x0;
//   DONE   idle.
//
// A chain whose solve converges records its result, updates its Welford
// statistics and stored draw (gibbs.py:139-167, 362-369) in the direction
// phase and starts its next scan in the next iteration, while the other
// chains keep iterating: the batch no longer waits for its slowest solve.
// The RNG keys are those of the single-chain scan (Philox (seed, purpose ^
// scan, element)), so a chain is the chain gibbs_run draws for its seed, up
// to the summation order of the solves.
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <string>

#include "gibbs_math.cuh"
#include "pg.cuh"
#include "sliced.cuh"

namespace cg = cooperative_groups;

namespace {

constexpr int kModeGibbs = 0, kModeInit = 1, kModeSolve = 2, kModeDone = 3;

struct ChainDev {
  const double* y;      // n
  const double* kappa;  // n
  double* beta;         // p_total, reference layout: in = state at launch, out = final draw
  double* omega;        // n: out = final omega
  double* lam;          // p
  double* nu;           // p
  double* scal;         // [tau, xi]
  double* mean;         // p_total
  double* m2;           // q
  double* draws;        // [store][p_total]
  double* tau_draws;    // [store]
  double* logdens;      // [n_iter]
  int* results;         // [n_iter][8]
  double *trace, *alphas, *betas;  // the last solve's trace (max_iter + 1)
  unsigned long long seed;
  int t_first, t_last;  // scans of this launch (1-based, inclusive)
  int count, stored;    // statistics updates / stored draws at launch start
};

struct GibbsCfgS {
  int prior, q, burn_in, thin, max_iter;
  double rtol, a0, b0, alpha, gamma_scale;
  const double* usd_prec;  // q
  const double* usd_sd;    // q
};

struct FusedArgs {
  BatchDev D;
  GibbsCfgS G;
  ChainDev ch[8];
  double *om, *w, *zpiece, *pieces, *dg;  // chain-minor: n R, n R, pieces R, pieces R, p_total R
  double *x, *r, *d, *z;                  // own state, chain-minor p_total R (internal column order)
  double *minv, *scale, *diag, *b;        // idem
  double* part;                           // per CTA: 6 R partials
  int* out_state;                         // [R][2]: count, stored after the launch
  unsigned long long* prof;               // debug: [8 a + k] phase stamps of iterations a < 64
};

template <int R>
__host__ __device__ constexpr int fused_ps() {
  return 16 * ((6 * R + 15) / 16);
}

__device__ __forceinline__ double loglik_term(double y, double z) {
  return y * z - (fmax(z, 0.0) + log1p(exp(-fabs(z))));
}

// bridge (gibbs.py:188-190) or horseshoe term of the tau
// update for a shrunk coefficient b with local scale l
__device__ __forceinline__ double tau_term_s(const GibbsCfgS& G, double b, double l) {
  if (G.prior == 0) return G.alpha == 1.0 ? fabs(b) : pow(fabs(b), G.alpha);
  return b * b / (l * l);
}

template <int R>
__global__ void __launch_bounds__(kSThreads, 1) k_sgibbs(FusedArgs A) {
  extern __shared__ __align__(128) double sv[];
  __shared__ double red[32 * R];
  __shared__ double sred[6 * R];
  __shared__ double st_rz[R], st_beta[R], st_alpha[R], st_tau[R], st_xi[R];
  __shared__ int st_mode[R], st_t[R], st_a[R], st_count[R], st_stored[R], st_prev[R], st_stop[R], st_status[R],
      st_fail[R];
  __shared__ int st_any;
  __shared__ unsigned long long mbar;
  BulkFill bf;
  bulk_init(bf, &mbar);
  const int tid = threadIdx.x;
  const int c_t = tid & (R - 1);
  constexpr int PS = fused_ps<R>();
  const BatchDev& D = A.D;
  const GibbsCfgS& G = A.G;
  const long long n = D.n, p = D.p, pt = D.pt, lead = D.icpt;
  const long long chunk = (pt + gridDim.x - 1) / gridDim.x;
  const long long j0 = (long long)blockIdx.x * chunk;
  const long long e0 = j0 * R, e1 = min(j0 + chunk, pt) * R;  // own elements
  const int q = G.q;
  const long long pshr = pt - q;  // shrunk coefficients
  double* mypart = A.part + (long long)blockIdx.x * PS;

  // ---- launch start: every chain enters GIBBS for its first scan with the
  // state it was given; the tau sums of that state -> slot D
  if (tid < R) {
    const ChainDev& C = A.ch[tid];
    st_mode[tid] = C.t_first <= C.t_last ? kModeGibbs : kModeDone;
    st_t[tid] = C.t_first;   // scan being prepared / solved
    st_prev[tid] = 0;        // no completed scan of this launch yet
    st_a[tid] = 0;
    st_count[tid] = C.count;
    st_stored[tid] = C.stored;
    st_tau[tid] = C.scal[0];
    st_xi[tid] = C.scal[1];
    st_rz[tid] = 0.0;
    st_stop[tid] = 0;
    st_status[tid] = PCGS_MAX_ITER;
    st_fail[tid] = -1;
  }
  __syncthreads();
  {
    double ts = 0.0;
    for (long long e = e0 + tid; e < e1; e += kSThreads) {
      const long long j = e / R;
      const long long r = ref_index(j, p, lead);
      const ChainDev& C = A.ch[c_t];
      const double bv = C.beta[r];
      A.x[e] = bv;
      A.dg[e] = bv;
      if (r >= q) ts += tau_term_s(G, bv, C.lam[r - q]);
    }
    const double t = block_sum_chain<R>(ts, red);
    if (tid < R) {
      mypart[3 * R + tid] = t;  // D: tau sums
      mypart[4 * R + tid] = 0.0;
      mypart[5 * R + tid] = 0.0;
      mypart[tid] = 0.0;
    }
  }
  cg::this_grid().sync();

  const bool prof_cta = A.prof && blockIdx.x == 0 && tid == 0;
  int it = 0;
  auto stamp = [&](int k) {
    if (prof_cta && it < 64) A.prof[8 * it + k] = stimer();
  };
  for (;; ++it) {
    stamp(0);
    // ---------------- CSR pass over dg (d, x0 or beta per chain) ----------------
    __shared__ double v0s[R];
    if (tid < R) v0s[tid] = D.icpt ? __ldcg(A.dg + p * R + tid) : 0.0;
    {
      FillRows<R> f{A.dg, &bf};
      EpiPiece e{A.zpiece, R};
      run_spass<R>(D.csr, sv, f, e);
    }
    cg::this_grid().sync();
    stamp(1);
    // ---------------- row combine per chain mode ----------------
    {
      const int mode = st_mode[c_t];
      const ChainDev& C = A.ch[c_t];
      const unsigned long long t_next = (unsigned long long)st_t[c_t];
      const bool draw = mode == kModeGibbs && st_t[c_t] <= C.t_last;
      double wz = 0.0, ll = 0.0;
      const long long nr = n * R;
      for (long long e = (long long)blockIdx.x * kSThreads + tid; e < nr; e += (long long)gridDim.x * kSThreads) {
        const long long i = e / R;
        double wi = 0.0;
        if (mode != kModeDone) {
          double z = 0.0;
          const long long q1 = D.csr.out_ptr[i + 1];
          for (long long qq = D.csr.out_ptr[i]; qq < q1; ++qq) z += __ldcg(A.zpiece + qq * R + c_t);
          z += v0s[c_t];
          if (mode == kModeGibbs) {
            ll += loglik_term(__ldg(C.y + i), z);
            if (draw) {
              Philox Rp(C.seed, kStreamPG ^ t_next, (unsigned)i);
              const double om = pg_draw1(z, Rp);
              A.om[e] = om;
              Philox Re(C.seed, kStreamEta ^ t_next, (unsigned)i);
              wi = __ldg(C.kappa + i) + sqrt(om) * Re.normal();
            }
          } else {
            wi = __ldcg(A.om + e) * z;
            wz += wi * z;
          }
        }
        A.w[e] = wi;
      }
      const double s1 = block_sum_chain<R>(wz, red);
      const double s2 = block_sum_chain<R>(ll, red);
      if (tid < R) {
        mypart[tid] += s1;            // A: dAd (+ the D d^2 part written with d)
        mypart[5 * R + tid] = s2;     // F: log-likelihood of z = X beta (GIBBS)
      }
    }
    cg::this_grid().sync();
    stamp(2);
    // ---------------- CSC pass over w ----------------
    {
      FillRows<R> f{A.w, &bf};
      EpiPiece e{A.pieces, R};
      run_spass<R>(D.csc, sv, f, e);
    }
    cg::this_grid().sync();
    stamp(3);

    // ---------------- column step ----------------
    reduce_parts(A.part, PS, 0, R, sred);          // A
    reduce_parts(A.part, PS, 3 * R, 3 * R, sred);  // D tau sums, E log prior, F log-likelihood
    if (tid < R) {
      const int c = tid;
      const ChainDev& C = A.ch[c];
      st_alpha[c] = 0.0;
      if (st_mode[c] == kModeSolve) {
        const double dAd = sred[c];
        if (!(dAd > 0.0)) {
          st_stop[c] = 1;
          st_status[c] = PCGS_NOT_PD;
          st_fail[c] = st_a[c];
        } else {
          st_alpha[c] = st_rz[c] / dAd;
          if (blockIdx.x == 0) C.alphas[st_a[c] - 1] = st_alpha[c];
        }
      } else if (st_mode[c] == kModeGibbs) {
        const int t_done = st_t[c] - 1;  // the completed scan whose beta was just multiplied
        const double tau_t = st_tau[c];
        if (st_prev[c] && blockIdx.x == 0) {  // log density of scan t_done (k_post)
          double out = sred[5 * R + c] + sred[4 * R + c];
          if (G.prior == 0) {
            const double a = G.alpha;
            out += (double)pshr * (log(a) - log(2.0) - lgamma(1.0 / a)) - (double)pshr * log(tau_t);
            out += G.a0 * log(G.b0) - lgamma(G.a0) + log(a) - (G.a0 * a + 1.0) * log(tau_t) - G.b0 * pow(tau_t, -a);
          } else {
            out += log(2.0 / M_PI) - log1p(tau_t * tau_t);
          }
          C.logdens[t_done - 1] = out;
        }
        if (st_t[c] <= C.t_last) {  // tau | beta, lambda (k_global)
          Philox Rg(C.seed, kStreamGlobal ^ (unsigned long long)st_t[c], 0u);
          double xi = st_xi[c];
          const double tau = global_draw(G.prior, G.a0, G.b0, G.alpha, pshr, sred[3 * R + c], tau_t, Rg, &xi);
          if (G.prior != 0) st_xi[c] = xi;
          st_tau[c] = tau;
          if (blockIdx.x == 0) {
            C.scal[0] = tau;
            C.scal[1] = st_xi[c];
            if (!(tau > 0.0) || !isfinite(tau)) C.results[8 * (st_t[c] - 1) + 4] = 1;
          }
        }
      }
    }
    __syncthreads();
    double trms = 0.0, trz = 0.0;
    {
      const int mode = st_mode[c_t];
      const ChainDev& C = A.ch[c_t];
      const double alpha = st_alpha[c_t];
      const int count = st_count[c_t];
      const double tau = st_tau[c_t];
      const unsigned long long t_next = (unsigned long long)st_t[c_t];
      const bool prep = mode == kModeGibbs && st_t[c_t] <= C.t_last;
      const long long Q0 = stage_own_pieces<R>(A.pieces, D.csc.out_ptr, e0 / R, e1 / R, sv, D.smem_doubles);
      auto colsum = [&](long long j) {
        double g = 0.0;
        const long long q1 = D.csc.out_ptr[j + 1];
        if (Q0 >= 0) {
          for (long long qq = D.csc.out_ptr[j]; qq < q1; ++qq) g += sv[(qq - Q0) * R + c_t];
        } else {
          for (long long qq = D.csc.out_ptr[j]; qq < q1; ++qq) g += __ldcg(A.pieces + qq * R + c_t);
        }
        return g;
      };
      for (long long e = e0 + tid; e < e1; e += kSThreads) {
        const long long j = e / R;
        const long long r = ref_index(j, p, lead);
        if (mode == kModeSolve || mode == kModeInit) {
          double Ad = colsum(j);
          const double dv = A.d[e];
          Ad += A.diag[e] * (mode == kModeInit ? A.x[e] : dv);
          double rv;
          if (mode == kModeInit) {
            rv = A.b[e] - Ad;
          } else {
            rv = A.r[e];
            if (alpha != 0.0) {
              A.x[e] = fma(alpha, dv, A.x[e]);
              rv = fma(-alpha, Ad, rv);
            }
          }
          A.r[e] = rv;
          const double zn = A.minv[e] * rv;
          A.z[e] = zn;
          const double tj = A.scale[e] * rv;
          trms += tj * tj;
          trz += rv * zn;
        } else if (prep) {
          // lambda | beta, tau; prior diagonal, M^-1, metric scale, x0 (k_local), b
          double dg_, mv, sc, x0;
          if (r < q) {
            double sd;
            if (count >= 2) sd = sqrt(C.m2[r] / (double)(count - 1));
            else sd = fmin(G.usd_sd[r], 10.0);
            const double gam = G.gamma_scale * fmax(sd, 1e-3);
            dg_ = G.usd_prec[r];
            mv = gam * gam;
            sc = gam;
            x0 = count > 0 ? C.mean[r] : 0.0;
          } else {
            const long long k = r - q;
            Philox Rl(C.seed, kStreamLocal ^ t_next, (unsigned)k);
            double nu = 0.0;
            const double lam = local_draw(G.prior, A.x[e], tau, C.lam[k], Rl, &nu);
            if (G.prior != 0) C.nu[k] = nu;
            C.lam[k] = lam;
            if (!(lam > 0.0) || !isfinite(lam)) C.results[8 * (t_next - 1) + 4] = 1;
            const double tl = tau * lam;
            dg_ = 1.0 / (tl * tl);
            mv = tl * tl;
            sc = tl;
            x0 = count > 0 ? tl * C.mean[r] : 0.0;
          }
          const double g = colsum(j);
          Philox Rd(C.seed, kStreamDelta ^ t_next, (unsigned)r);
          A.b[e] = g + sqrt(dg_) * Rd.normal();
          A.diag[e] = dg_;
          A.minv[e] = mv;
          A.scale[e] = sc;
          A.x[e] = x0;
        }
      }
    }
    {
      const double s1 = block_sum_chain<R>(trms, red);
      const double s2 = block_sum_chain<R>(trz, red);
      if (tid < R) {
        mypart[R + tid] = s1;
        mypart[2 * R + tid] = s2;
      }
    }
    cg::this_grid().sync();
    stamp(4);

    // ---------------- per chain: convergence, statistics, next state ----------------
    reduce_parts(A.part, PS, R, 2 * R, sred);  // B rms, C rz
    if (tid < R) {
      const int c = tid;
      const ChainDev& C = A.ch[c];
      const int mode = st_mode[c];
      st_beta[c] = 0.0;
      int stop = st_mode[c] == kModeSolve && st_stop[c] == 1 ? 1 : 0;  // NOT_PD found in the step
      if (mode == kModeSolve || mode == kModeInit) {
        const int k = st_a[c];  // iterations completed
        const double rms = sqrt(sred[R + c] / (double)pt), rzn = sred[2 * R + c];
        if (!stop) {
          if (blockIdx.x == 0) C.trace[k] = rms;
          if (rms <= G.rtol) {
            stop = 1;
            st_status[c] = PCGS_CONVERGED;
            st_fail[c] = -1;
          } else if (!isfinite(rms)) {
            stop = 1;
            st_status[c] = PCGS_NONFINITE;
            st_fail[c] = k;
          } else {
            if (k >= 1) {
              st_beta[c] = rzn / st_rz[c];
              if (blockIdx.x == 0) C.betas[k - 1] = st_beta[c];
            }
            st_rz[c] = rzn;
            if (k >= G.max_iter) {
              stop = 1;
              st_status[c] = PCGS_MAX_ITER;
              st_fail[c] = -1;
            }
          }
        }
        if (stop && blockIdx.x == 0) {
          int* res = C.results + 8 * (st_t[c] - 1);
          res[0] = k;
          res[1] = st_status[c];
          res[2] = st_status[c] == PCGS_NOT_PD || st_status[c] == PCGS_NONFINITE ? st_fail[c] : -1;
          res[3] = k + 1;
        }
      }
      st_stop[c] = stop;
    }
    __syncthreads();
    // element work of the transition (statistics of a finished solve; new directions)
    double dd = 0.0, lp = 0.0, ts = 0.0;
    {
      const int mode = st_mode[c_t];
      const ChainDev& C = A.ch[c_t];
      const bool fin = (mode == kModeSolve || mode == kModeInit) && st_stop[c_t];
      const double beta = st_beta[c_t];
      const double tau = st_tau[c_t];
      const int t = st_t[c_t];
      const int count_new = st_count[c_t] + 1;
      int slot = -1;
      if (fin && t > G.burn_in && (t - G.burn_in - 1) % G.thin == 0) slot = st_stored[c_t];
      for (long long e = e0 + tid; e < e1; e += kSThreads) {
        const long long j = e / R;
        const long long r = ref_index(j, p, lead);
        double dn = 0.0;
        if (fin) {  // k_stats: Welford, stored draw, log prior, the next tau sums
          const double bv = A.x[e];
          double scaled = bv;
          if (r >= q) scaled = bv / (tau * C.lam[r - q]);
          const double delta = scaled - C.mean[r];
          const double m = C.mean[r] + delta / (double)count_new;
          C.mean[r] = m;
          if (r < q) C.m2[r] += delta * (scaled - m);
          if (slot >= 0) C.draws[(long long)slot * pt + r] = bv;
          if (slot >= 0 && r == 0) C.tau_draws[slot] = tau;
          if (r < q) {
            const double sd = G.usd_sd[r];
            if (isfinite(sd)) {
              const double u = bv / sd;
              lp -= 0.5 * u * u + log(sd) + 0.5 * log(2.0 * M_PI);
            }
          } else {
            const double l = C.lam[r - q];
            if (G.prior == 0) {
              lp -= G.alpha == 1.0 ? fabs(bv / tau) : pow(fabs(bv / tau), G.alpha);
            } else {
              const double sc = tau * l;
              const double u = bv / sc;
              lp += -log(sc) - 0.5 * u * u - 0.5 * log(2.0 * M_PI) + log(2.0 / M_PI) - log1p(l * l);
            }
            ts += tau_term_s(G, bv, l);
          }
          dn = bv;  // the next CSR pass multiplies beta (GIBBS)
        } else if (mode == kModeSolve || mode == kModeInit) {
          dn = mode == kModeInit ? A.z[e] : fma(beta, A.d[e], A.z[e]);
          A.d[e] = dn;
          dd += A.diag[e] * dn * dn;
        } else if (mode == kModeGibbs && t <= C.t_last) {
          dn = A.x[e];  // x0: the next iteration applies Phi to it (INIT)
          A.d[e] = 0.0;
        }
        A.dg[e] = dn;
      }
    }
    {
      const double s1 = block_sum_chain<R>(dd, red);
      const double s2 = block_sum_chain<R>(lp, red);
      const double s3 = block_sum_chain<R>(ts, red);
      if (tid < R) {
        const int c = tid;
        const int mode = st_mode[c];
        const bool fin = (mode == kModeSolve || mode == kModeInit) && st_stop[c];
        mypart[c] = s1;                       // A: the D d^2 part of the next dAd
        if (fin) {
          mypart[3 * R + c] = s3;             // D
          mypart[4 * R + c] = s2;             // E
        }
      }
    }
    __syncthreads();
    if (tid < R) {  // next state (identical in every CTA)
      const int c = tid;
      const ChainDev& C = A.ch[c];
      const int mode = st_mode[c];
      if (mode == kModeSolve || mode == kModeInit) {
        if (st_stop[c]) {
          const int t = st_t[c];
          if (t > G.burn_in && (t - G.burn_in - 1) % G.thin == 0) ++st_stored[c];
          ++st_count[c];
          st_prev[c] = 1;
          st_t[c] = t + 1;
          st_mode[c] = kModeGibbs;  // its log density, then the next scan (or DONE after the last)
        } else {
          st_mode[c] = kModeSolve;
          st_a[c] = st_a[c] + 1;
        }
      } else if (mode == kModeGibbs) {
        if (st_t[c] <= C.t_last) {
          st_mode[c] = kModeInit;
          st_a[c] = 0;
          st_stop[c] = 0;
        } else {
          st_mode[c] = kModeDone;
        }
      }
    }
    __syncthreads();
    if (tid == 0) {
      int any = 0;
      for (int c = 0; c < R; ++c) any |= st_mode[c] != kModeDone;
      st_any = any;
    }
    cg::this_grid().sync();
    stamp(5);
    if (!st_any) break;
  }

  // ---- write back the final state: beta (last draw), omega, counters
  __syncthreads();
  for (long long e = e0 + tid; e < e1; e += kSThreads) {
    const long long j = e / R;
    A.ch[c_t].beta[ref_index(j, p, lead)] = A.x[e];
  }
  {
    const long long nr = n * R;
    for (long long e = (long long)blockIdx.x * kSThreads + tid; e < nr; e += (long long)gridDim.x * kSThreads)
      A.ch[c_t].omega[e / R] = A.om[e];
  }
  if (blockIdx.x == 0 && tid < R) {
    A.out_state[2 * tid + 0] = st_count[tid];
    A.out_state[2 * tid + 1] = st_stored[tid];
  }
}

template <int R>
int run_fused(const BatchDev& D, FusedArgs& A, cudaStream_t s) {
  int rc;
  if ((rc = raise_smem_limit(k_sgibbs<R>))) return rc;
  Scratch S(s);
  A.D = D;
  const size_t nR = (size_t)D.n * R, pR = (size_t)D.pt * R;
  A.om = S.get<double>(nR);
  A.w = S.get<double>(nR);
  A.zpiece = S.get<double>((size_t)D.csr.npiece * R);
  A.pieces = S.get<double>((size_t)D.csc.npiece * R);
  A.dg = S.get<double>(pR + 16);
  double* own = S.get<double>(8 * pR);
  A.part = S.get<double>((size_t)fused_ps<R>() * D.G);
  if (!A.om || !A.w || !A.zpiece || !A.pieces || !A.dg || !own || !A.part)
    return fail(PCGS_ENOMEM, "scratch allocation failed");
  A.x = own;
  A.r = own + pR;
  A.d = own + 2 * pR;
  A.z = own + 3 * pR;
  A.minv = own + 4 * pR;
  A.scale = own + 5 * pR;
  A.diag = own + 6 * pR;
  A.b = own + 7 * pR;
  CUDA_TRY(cudaMemsetAsync(own, 0, 8 * pR * sizeof(double), s));
  CUDA_TRY(cudaMemsetAsync(A.om, 0, nR * sizeof(double), s));
  void* args[] = {&A};
  CUDA_TRY(cudaLaunchCooperativeKernel((const void*)k_sgibbs<R>, D.G, kSThreads, args, (size_t)D.smem_doubles * 8, s));
  return PCGS_OK;
}

}  // namespace

extern "C" {

int pcgs_batch_gibbs_run(pcgs_batch_t bt, pcgs_gibbs_t* const* gs, int32_t nchains, int32_t t_first,
                         int32_t t_last, int32_t burn_in, int32_t thin, const int32_t* counts,
                         const int32_t* stored, int32_t* out_state, pcgs_stream_t stream) {
  if (!bt || !gs || !counts || !stored || !out_state || t_first < 1 || thin < 1 || burn_in < 0)
    return fail(PCGS_EINVAL, "bad argument");
  const BatchDev& D = bt->dev;
  if (nchains != D.R) return fail(PCGS_EINVAL, "nchains must equal the batch store's chain count");
  const pcgs_gibbs_t& g0 = *gs[0];
  FusedArgs A;
  memset(&A, 0, sizeof(A));
  A.G = GibbsCfgS{g0.prior, g0.q, burn_in, thin, g0.max_iter, g0.rtol, g0.a0, g0.b0, g0.alpha, g0.gamma_scale,
                  g0.usd_prec, g0.usd_sd};
  if (g0.prior == 0 && g0.alpha != 1.0) return fail(PCGS_EUNSUP, "bridge local draws need alpha = 1");
  for (int c = 0; c < nchains; ++c) {
    const pcgs_gibbs_t& g = *gs[c];
    if (g.prior != g0.prior || g.q != g0.q || g.max_iter != g0.max_iter || g.rtol != g0.rtol ||
        g.a0 != g0.a0 || g.b0 != g0.b0 || g.alpha != g0.alpha || g.gamma_scale != g0.gamma_scale)
      return fail(PCGS_EINVAL, "fused chains must share the model and solver settings");
    if (g.fixed_omega || g.fixed_tau || g.fixed_lam || g.precond != 0 || g.cscale)
      return fail(PCGS_EUNSUP, "fused chains: pinned updates, other preconditioners and reparametrised designs "
                               "run through pcgs_batch_gibbs_scan");
    ChainDev& C = A.ch[c];
    C.y = g.y;
    C.kappa = g.kappa;
    C.beta = g.beta;
    C.omega = g.omega;
    C.lam = g.lam;
    C.nu = g.nu;
    C.scal = g.scal;
    C.mean = g.mean;
    C.m2 = g.m2;
    C.draws = g.draws;
    C.tau_draws = g.tau_draws;
    C.logdens = g.logdens;
    C.results = g.results;
    C.trace = g.trace;
    C.alphas = g.alphas;
    C.betas = g.betas;
    C.seed = g.seed;
    C.t_first = t_first;
    C.t_last = t_last;
    C.count = counts[c];
    C.stored = stored[c];
  }
  A.out_state = out_state;
  A.prof = batch_profile_buffer();
  cudaStream_t s = (cudaStream_t)stream;
  switch (D.R) {
    case 2: return run_fused<2>(D, A, s);
    case 4: return run_fused<4>(D, A, s);
    case 8: return run_fused<8>(D, A, s);
    default: return fail(PCGS_EINVAL, "fused chains come in batches of 2, 4 or 8");
  }
}

}  // extern "C"
