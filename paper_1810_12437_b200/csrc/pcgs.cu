// pcgs: B200-native kernels and C ABI for the prior-preconditioned CG sampler
// hot path (reference: pkg/src/priorcg/{sparse,sampler,cg,polya_gamma}.py).
//
// Kernel inventory:
//   k_csr_*      X v over column slabs         (sparse.py:178-193)
//   k_csc_*      X' w over row slabs           (sparse.py:195-203)
//   k_assemble   per-column piece sums + diagonal terms
//   k_rhs_u      u = kappa + sqrt(omega) eta per row (RHS input of one CSC pass)
//   k_pcg        the whole PCG solve, one persistent cooperative kernel
//                (cg.py:105-192, operator sampler.py:53-58)
//   k_pg         Polya-Gamma PG(1, z) draws    (polya_gamma.py:39-147)
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "internal.cuh"
#include "mtx.h"

namespace cg = cooperative_groups;

// =====================================================================
// error plumbing
// =====================================================================
static unsigned long long* g_prof = nullptr;  // debug: phase timestamps of the next pcgs_pcg
static int g_dbg = 0;
static int g_l2_persist_mb = 0;
static int g_nranges = 0;  // debug option 3: warp ranges per task of stores created from now on (0: default)
static thread_local std::string g_err;
void set_last_error(const std::string& msg) { g_err = msg; }

// =====================================================================
// standalone kernels (one pass each; launched with the plan's G CTAs)
// =====================================================================
template <int kT, int kRingB>
__global__ void __launch_bounds__(kT, 1) k_csr_matvec(DesignDev D, const double* v, double* out,
                                                            const double* cbuf) {
  extern __shared__ __align__(128) double sv[];
  FillVecRef f{v, D.lead(), 0, D.aff.sc};
  const double v0 = row_const(D, v, cbuf);
  if (D.csr.nslab == 1) {
    EpiZ e{out, v0, aff_row(D, cbuf)};
    run_pass<kRingB>(D.csr, sv, f, e, D.dbg);
  } else {
    EpiStore e{out, (long long)D.csr.nslab * D.n};  // out is the (nslab x n) partial buffer
    run_pass<kRingB>(D.csr, sv, f, e, D.dbg);
  }
}

template <int kT, int kRingB>
__global__ void __launch_bounds__(kT, 1) k_csr_phi(DesignDev D, const double* v, const double* omega, double* w,
                                                         const double* cbuf) {
  extern __shared__ __align__(128) double sv[];
  FillVecRef f{v, D.lead(), 0, D.aff.sc};
  const double v0 = row_const(D, v, cbuf);
  if (D.csr.nslab == 1) {
    EpiW e{w, omega, v0, 0.0, aff_row(D, cbuf)};
    run_pass<kRingB>(D.csr, sv, f, e);
  } else {
    EpiStore e{w, (long long)D.csr.nslab * D.n};
    run_pass<kRingB>(D.csr, sv, f, e);
  }
}

// multi column slab: z_i = v0 + sum_s part[s*n+i] (+ row term); out = scale ? scale*z : z
__global__ void k_rows_combine(DesignDev D, const double* part, const double* v, const double* scale, double* out,
                               const double* cbuf) {
  const double v0 = row_const(D, v, cbuf);
  const AffRow ar = aff_row(D, cbuf);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < D.n; i += (long long)gridDim.x * blockDim.x) {
    double z = 0.0;
    for (int s = 0; s < D.csr.nslab; ++s) z += part[(long long)s * D.n + i];
    z += v0;
    if (ar.q) z += ar(i);
    out[i] = scale ? __ldg(scale + i) * z : z;
  }
}

// Affine designs, CSR side: cbuf[0] = u_icpt - mu'u, cbuf[1 + k] = u of dense
// column k (u = v / s); one CTA, fixed-order sum.
__global__ void __launch_bounds__(kThreads) k_aff_pre(DesignDev D, const double* v, double* cbuf) {
  __shared__ double red[64];
  const AffineDev& F = D.aff;
  double acc = 0.0;
  for (long long r = threadIdx.x; r < D.pt; r += kThreads) {
    const double u = F.sc ? v[r] / F.sc[r] : v[r];
    if (F.mu) acc += F.mu[r] * u;
  }
  acc = block_sum(acc, red);
  if (threadIdx.x == 0) cbuf[0] = (D.icpt ? (F.sc ? v[0] / F.sc[0] : v[0]) : 0.0) - acc;
  for (int k = threadIdx.x; k < F.q; k += kThreads) {
    const long long r = D.icpt + k;
    cbuf[1 + k] = F.sc ? v[r] / F.sc[r] : v[r];
  }
}

// Affine designs, transpose side: per-CTA partials of W = sum_i w_i,
// G_k = sum_i Dn[i,k] w_i and (squares) G2_k = sum_i Dn[i,k]^2 w_i, in line
// c * (1 + 2q); then k_aff_tw_fin sums the lines in CTA order into gbuf.
constexpr int kAffMaxQ = 32;
__global__ void __launch_bounds__(256) k_aff_tw_part(DesignDev D, const double* w, int squares, double* part) {
  __shared__ double red[64];
  const int q = D.aff.q, S = 1 + 2 * q;
  double accW = 0.0, accG[kAffMaxQ], accG2[kAffMaxQ];
  for (int k = 0; k < q; ++k) accG[k] = accG2[k] = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < D.n; i += (long long)gridDim.x * blockDim.x) {
    const double wi = __ldcg(w + i);
    accW += wi;
    for (int k = 0; k < q; ++k) {
      const double x = __ldg(D.aff.dense + i * q + k);
      accG[k] += x * wi;
      if (squares) accG2[k] += x * x * wi;
    }
  }
  const double tW = block_sum(accW, red);
  if (threadIdx.x == 0) part[(long long)blockIdx.x * S] = tW;
  for (int k = 0; k < q; ++k) {
    const double t = block_sum(accG[k], red);
    if (threadIdx.x == 0) part[(long long)blockIdx.x * S + 1 + k] = t;
    if (squares) {
      const double t2 = block_sum(accG2[k], red);
      if (threadIdx.x == 0) part[(long long)blockIdx.x * S + 1 + q + k] = t2;
    }
  }
}
__global__ void k_aff_tw_fin(const double* part, int ncta, int S, double* gbuf) {
  for (int k = threadIdx.x; k < S; k += blockDim.x) {
    double s = 0.0;
    for (int c = 0; c < ncta; ++c) s += part[(long long)c * S + k];
    gbuf[k] = s;
  }
}

// raw column sum of internal column j -> X_eff' w entry: (g - mu W) / s, with
// g the pattern sum (pieces) or the dense partial G_k; mode 3 (diag(X'Omega X)
// with w = omega) uses the squared form (g (1 - 2 mu) + mu^2 W) / s^2 for
// binary columns and (G2 - 2 mu G + mu^2 W) / s^2 for dense ones.
__device__ __forceinline__ double aff_col(const DesignDev& D, long long j, long long r, double raw,
                                          const double* gbuf, int mode) {
  const AffineDev& F = D.aff;
  const double W = gbuf[0];
  const double mu = F.mu ? __ldg(F.mu + r) : 0.0, s = F.sc ? __ldg(F.sc + r) : 1.0;
  const long long k = j - D.p - D.icpt;  // dense column index (k >= 0)
  if (mode == 3) {
    if (k >= 0) return (gbuf[1 + F.q + k] - 2.0 * mu * raw + mu * mu * W) / (s * s);
    return (raw * (1.0 - 2.0 * mu) + mu * mu * W) / (s * s);
  }
  return (raw - mu * W) / s;
}

// u_i = kappa_i + sqrt(omega_i) eta_i for every row (the RHS pass's input)
__global__ void k_rhs_u(FillRhs f, long long n, double* u) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    u[i] = f((int)i);
}

template <int kT, int kRingB>
__global__ void __launch_bounds__(kT, 1) k_csc_vec(DesignDev D, const double* w, double* pieces) {
  extern __shared__ __align__(128) double sv[];
  __shared__ unsigned long long mbar;
  BulkFill bf;
  bulk_init(bf, &mbar);
  FillVecN f{w, &bf};
  EpiStore e{pieces, D.csc.nseg};
  run_pass<kRingB>(D.csc, sv, f, e, D.dbg);
}

// out[ref(j)] = column_sum(j) + diag_j * v[ref(j)]  (diag/v may be null)
//               + sqrt(diag_j) * delta_j           (mode 2: RHS noise)
__global__ void k_assemble(DesignDev D, const double* pieces, const double* diag, const double* v,
                           const double* delta, unsigned long long seed, unsigned long long stream, int mode,
                           double* out, const double* linear = nullptr, const double* gbuf = nullptr) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < D.pt; j += (long long)gridDim.x * blockDim.x) {
    const long long r = ref_index(j, D.p, D.lead());
    double s;
    if (gbuf) {
      const long long k = j - D.p - D.icpt;
      const double raw = k >= 0 ? gbuf[1 + k] : column_sum(D.csc, pieces, D.pt, j);
      s = aff_col(D, j, r, raw, gbuf, mode);
    } else {
      s = column_sum(D.csc, pieces, D.pt, j);
    }
    if (mode == 1) {
      s += __ldg(diag + r) * __ldg(v + r);
    } else if (mode == 2) {
      if (linear) s = __ldg(linear + r) + s;
      double e;
      if (delta) {
        e = __ldg(delta + r);
      } else {
        Philox R(seed, stream, (unsigned)r);
        e = R.normal();
      }
      s += sqrt(__ldg(diag + r)) * e;
    } else if (mode == 3) {
      s += __ldg(diag + r);
    }
    out[r] = s;
  }
}

// =====================================================================
// persistent PCG kernel
// =====================================================================
struct PcgArgs {
  DesignDev D;
  const double* omega;  // n
  const double* diag;   // prior precision, reference layout
  const double* minv;   // reference layout
  const double* scale;  // reference layout
  const double* b;      // reference layout
  double* x;            // in x0 / out solution, reference layout
  int max_iter;
  double rtol;
  double* trace;
  double* alphas;
  double* betas;
  int* result;
  // scratch
  double* w;       // n (+pad)
  double* zpart;   // nslab_csr * n (multi column slab only)
  double* pieces;  // csc nseg
  double* zv;      // p_total internal layout: minv * r
  double* dvg;     // 2 * p_total internal layout: search directions
  double* part;    // 4 * G partial sums: dAd, rms, rz, spare
  unsigned long long* prof;  // optional: CTA-0 phase timestamps (ns), 4 per apply
  double* iterates;  // optional (trace_level "full"): [max_iter+1][p_total], reference layout
  double* apart;     // affine designs: per-CTA lines of W and the dense sums G_k (1 + q each)
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// debug: per-CTA arrival/departure stamps at the four grid barriers of one
// PCG iteration (debug option key 1 bit 128), [16 * cta + 2 * barrier + {0,1}],
// and stamps inside phase C at [16 * cta + 8 + k]
__device__ unsigned long long* g_sync_times = nullptr;
constexpr int kSyncTraceIter = 10;
// The persistent PCG kernel runs 16 warps of 128 registers, each walking two of
// a task's 32 warp ranges with two-block register batches: they keep the LSU
// pipe as busy as 32 warps of 64 registers (70.5 vs 69.8 us per iteration at
// config 2), and the register room pays for the step phase on column-major
// piece slots and the hooks in the slab fills' TMA wait, which spilled at 64
// registers (67.7 us).  The standalone passes and the row-split
// kernel stay at 32 warps (their streams ran 9 % slower on 16).
#ifndef PCGS_PCG_WARPS
#define PCGS_PCG_WARPS 16
#endif
constexpr int kPcgWarps = PCGS_PCG_WARPS;
constexpr int kPcgThreads = kPcgWarps * 32;
constexpr int kPcgRing = kPcgWarps <= 16 ? 2 : 1;  // blocks per register batch of the grouped walk
constexpr int kMaxGrid = 256;  // persistent-kernel grid bound (one CTA per SM; B200: 148)

struct FillDir {  // search direction: first ? a : a + beta * b   (internal layout)
  const double* a;
  const double* b;
  double beta;
  int first;
  long long lo;
  __device__ double operator()(int j) const {
    const double aj = __ldcg(a + lo + j);
    return first ? aj : fma(beta, __ldcg(b + lo + j), aj);
  }
  __device__ void operator()(double* sv, long long l, int len) {
    lo = l;
    fill_smem(sv, len, *this);
  }
};

// Shared-memory layout of k_pcg: [slab vector | own-slice state | piece slots]
// The CSC pass of k_pcg stores piece q at its column-major slot (store.h:
// piece_perm), so the pieces of a CTA's owned columns are one contiguous run
// [cp[j0], cp[j0 + chunk]) of the pieces array; their slot offsets relative to
// the run's start are staged in shared memory when they fit (cp), otherwise
// read from the design's global col_piece_ptr.
struct OwnState {
  double *x, *r, *d, *m, *s, *D, *b, *z;
  const int* cp;   // shared copy [chunk + 1] of relative slot offsets, or null
};

// The owned run of piece slots, set up where it is used (the step phase).
struct PieceRun {
  const int* cp;   // OwnState::cp
  const int* gcp;  // global col_piece_ptr
  long long j0, pt;
  int q_lo;        // first slot of the owned run
  __device__ __forceinline__ int rel(int t) const {
    if (cp) return cp[t];
    const long long j = j0 + t < pt ? j0 + t : pt;
    return __ldg(gcp + j) - q_lo;
  }
};
__device__ __forceinline__ PieceRun piece_run(const OwnState& o, const DesignDev& D, long long j0) {
  PieceRun r{o.cp, D.csc.col_piece_ptr, j0, D.pt, 0};
  r.q_lo = __ldg(r.gcp + (j0 < D.pt ? j0 : D.pt));
  return r;
}

__host__ __device__ inline bool pp_in_smem(const DesignDev& D) {
  const long long chunk = (D.pt + D.G - 1) / D.G;
  const long long own = D.own_in_global ? 0 : chunk * 8 * 8;
  const long long bytes = (long long)D.smem_doubles * 8 + own + (chunk + 1) * 4;
  return bytes + 1024 <= 227 * 1024;
}

__device__ __forceinline__ OwnState own_state(double* sv, const DesignDev& D, int chunk, long long j0) {
  OwnState o;
  double* base = D.own_in_global ? D.own_global + (size_t)blockIdx.x * 8 * chunk : sv + D.smem_doubles;
  double* after = D.own_in_global ? sv + D.smem_doubles : base + 8 * chunk;
  o.x = base;
  o.r = base + chunk;
  o.d = base + 2 * chunk;
  o.m = base + 3 * chunk;
  o.s = base + 4 * chunk;
  o.D = base + 5 * chunk;
  o.b = base + 6 * chunk;
  o.z = base + 7 * chunk;
  o.cp = pp_in_smem(D) ? (const int*)after : nullptr;
  return o;
}

size_t pcg_smem_bytes(const DesignDev& D) {
  const long long chunk = (D.pt + D.G - 1) / D.G;
  size_t b = (size_t)D.smem_doubles * 8 + (D.own_in_global ? 0 : (size_t)chunk * 8 * 8) + 16;
  if (pp_in_smem(D)) b += (size_t)(chunk + 1) * 4;
  return b;
}

// Stages the pieces of the CTA's owned columns (one contiguous run of the
// column-major slots) into the idle slab area in one coalesced round; returns
// false when they do not fit (then the column sums read global memory).
__device__ __forceinline__ bool stage_pieces(const PieceRun& o, const double* pieces, int chunk, double* stage,
                                             int cap) {
  const int total = o.rel(chunk);
  if (total > cap) return false;
  for (int q = threadIdx.x; q < total; q += (int)blockDim.x) stage[q] = __ldcg(pieces + o.q_lo + q);
  __syncthreads();
  return true;
}

// Sum of the pieces of owned column t: slab-major, then piece order (fixed).
__device__ __forceinline__ double owned_column_sum(const PieceRun& o, const double* pieces, int t,
                                                   const double* stage, bool staged) {
  const int q0 = o.rel(t), q1 = o.rel(t + 1);
  double sum = 0.0;
  if (staged)
    for (int q = q0; q < q1; ++q) sum += stage[q];
  else
    for (int q = q0; q < q1; ++q) sum += __ldcg(pieces + o.q_lo + q);
  return sum;
}

// CSC slab fill whose TMA wait carries the grid sum of the CSR pass's dAd
// partials (complete since the CSR barrier): warp 1 reduces them while the
// first slab is in flight, so the step phase finds d'Ad in *out (`done`
// records it; a CTA with no CSC work leaves the sum to the step phase).
#ifndef PCGS_DAD_IN_FILL
#define PCGS_DAD_IN_FILL 1
#endif
struct FillVecNDad {
  const double* w;
  BulkFill* bf;
  const double* part;
  int G;
  double* out;
  bool pending, done;
  static constexpr bool kHooked = true;
  template <class Hook>
  __device__ void operator()(double* sv, long long l, int len, Hook hook) {
    const bool go = pending;
    done = done || go;
    bulk_fill(*bf, sv, w + l, len, [&] {
      hook();
      if (go && threadIdx.x >= 32 && threadIdx.x < 64) {
        const double s = warp_sum(lane_partials(part, G, threadIdx.x & 31));
        if (threadIdx.x == 32) *out = s;
      }
    });
    pending = false;
  }
};

// CSR slab fill of the published direction whose TMA wait also fetches the
// intercept's entry (one thread, into shared memory): every thread's epilogue
// constant is set from it after the fill's closing barrier.
struct FillBulkV0 {
  const double* src;
  BulkFill* bf;
  const double* icpt_src;  // null: no intercept
  double* slot;            // shared memory
  double* v0;              // the calling thread's epilogue constant
  static constexpr bool kHooked = true;
  template <class Hook>
  __device__ void operator()(double* sv, long long l, int len, Hook hook) {
    bulk_fill(*bf, sv, src + l, len, [&] {
      hook();
      if (threadIdx.x == 64) *slot = icpt_src ? __ldcg(icpt_src) : 0.0;
    });
    *v0 = *slot;
  }
};

__device__ __forceinline__ void traced_sync(const PcgArgs& A, int a, int k) {
  const bool tr = (A.D.dbg & 128) && a == kSyncTraceIter && threadIdx.x == 0 && g_sync_times;
  if (tr) g_sync_times[16 * blockIdx.x + 2 * k] = gtimer();
  cg::this_grid().sync();
  if (tr) g_sync_times[16 * blockIdx.x + 2 * k + 1] = gtimer();
}

__device__ __forceinline__ void trace_stamp(const PcgArgs& A, int a, int k) {
  if ((A.D.dbg & 128) && a == kSyncTraceIter && threadIdx.x == 0 && g_sync_times)
    g_sync_times[16 * blockIdx.x + 8 + k] = gtimer();
}

// Affine designs: u = v / s of reference column r (the gathered quantity).
__device__ __forceinline__ double aff_u(const DesignDev& D, long long r, double v) {
  return D.aff.sc ? v / __ldg(D.aff.sc + r) : v;
}
// CTA partial of mu' u over the CTA's own columns -> part slot 3 (call with the whole CTA)
__device__ __forceinline__ void aff_mu_partial(const PcgArgs& A, double acc, double* red) {
  const double t = block_sum(acc, red);
  if (threadIdx.x == 0) A.part[blockIdx.x * kPartStride + 3] = t;
}

template <bool AFF>
__global__ void __launch_bounds__(kPcgThreads, 1) k_pcg(PcgArgs A) {
  // Loop state lives in shared memory so that the inlined streaming passes
  // get the whole register budget (1024 threads -> 64 registers).
  extern __shared__ __align__(128) double sv[];
  __shared__ double red[64];
  __shared__ double bc[4];
  __shared__ double st_rz;
  __shared__ int st_status, st_iter, st_fail, st_applies;
  __shared__ unsigned long long mbar;
  __shared__ double affg[AFF ? 1 + kAffMaxQ : 1];  // affine designs: W, G_k
  BulkFill bf;
  bulk_init(bf, &mbar);
  const int tid = threadIdx.x;

  // ---- own slice of the p_total coordinates, kept in shared memory ----
  {
    const long long pt = A.D.pt;
    const int chunk = (int)((pt + gridDim.x - 1) / gridDim.x);
    const long long j0 = (long long)blockIdx.x * chunk;
    const long long dvs = (pt + 15) / 16 * 16;
    const OwnState o = own_state(sv, A.D, chunk, j0);
    for (int t = tid; t < chunk; t += kPcgThreads) {
      const long long j = j0 + t;
      double xv = 0, m = 0, sc = 0, dg = 0, bv = 0;
      if (j < pt) {
        const long long rj = ref_index(j, A.D.p, A.D.lead());
        xv = A.x[rj];
        m = __ldg(A.minv + rj);
        sc = __ldg(A.scale + rj);
        dg = __ldg(A.diag + rj);
        bv = __ldg(A.b + rj);
        A.dvg[dvs + j] = AFF ? aff_u(A.D, rj, xv) : xv;  // v = x0 for the first application
        if (A.iterates) A.iterates[rj] = xv;
      }
      o.x[t] = xv;
      o.r[t] = 0.0;
      o.d[t] = xv;
      o.m[t] = m;
      o.s[t] = sc;
      o.D[t] = dg;
      o.b[t] = bv;
      o.z[t] = 0.0;
    }
    if (o.cp) {
      int* cpw = const_cast<int*>(o.cp);
      const int* gcp = A.D.csc.col_piece_ptr;
      const int q_lo = __ldg(gcp + min(j0, pt));
      for (int t = tid; t <= chunk; t += kPcgThreads) cpw[t] = __ldg(gcp + min(j0 + t, pt)) - q_lo;
    }
    if (tid == 0) {
      st_rz = 0.0;
      st_status = PCGS_MAX_ITER;
      st_iter = 0;
      st_fail = -1;
      st_applies = 0;
    }
    if (AFF) {
      double mu_u = 0.0;
      if (A.D.aff.mu)
        for (int t = tid; t < chunk; t += kPcgThreads) {
          const long long j = j0 + t;
          if (j < pt) {
            const long long rj = ref_index(j, A.D.p, A.D.lead());
            mu_u += __ldg(A.D.aff.mu + rj) * aff_u(A.D, rj, o.x[t]);
          }
        }
      aff_mu_partial(A, mu_u, red);
    }
  }
  cg::this_grid().sync();

  for (int a = 0;; ++a) {
    const long long pt = A.D.pt;
    const int chunk = (int)((pt + gridDim.x - 1) / gridDim.x);
    const long long j0 = (long long)blockIdx.x * chunk;
    const long long dvs = (pt + 15) / 16 * 16;
    const OwnState o = own_state(sv, A.D, chunk, j0);
    const bool prof = A.prof && blockIdx.x == 0 && tid == 0 && a < 64;
    // ---------------- convergence test of iteration a-1 ----------------
    if (a > 0) {
      double s_rms, s_rz;
      reduce_partials2(A.part + 1, gridDim.x, bc, s_rms, s_rz);
      const double rms = sqrt(s_rms / (double)pt);
      if (blockIdx.x == 0 && tid == 0) A.trace[a - 1] = rms;
      const int k = a - 1;  // iterations completed
      int stop = 0;
      if (rms <= A.rtol) stop = 1;
      else if (!isfinite(rms)) stop = 2;
      double beta = 0.0;
      if (!stop) {
        if (a >= 2) {
          beta = s_rz / st_rz;
          if (blockIdx.x == 0 && tid == 0) A.betas[a - 2] = beta;
        }
        if (k >= A.max_iter) stop = 3;
      }
      __syncthreads();
      if (tid == 0) {
        st_rz = s_rz;
        if (stop) {
          st_status = stop == 1 ? PCGS_CONVERGED : stop == 2 ? PCGS_NONFINITE : PCGS_MAX_ITER;
          st_iter = k;
          if (stop == 2) st_fail = k;
        }
      }
      if (stop) break;
      // new direction d = z + beta d on the owned slice, published for the fill
      // (affine designs publish u = d / s and the CTA partial of mu'u)
      double mu_u = 0.0;
      for (int t = tid; t < chunk; t += kPcgThreads) {
        const double dn = a == 1 ? o.z[t] : fma(beta, o.d[t], o.z[t]);
        o.d[t] = dn;
        if (j0 + t < pt) {
          if (AFF) {
            const long long rj = ref_index(j0 + t, A.D.p, A.D.lead());
            const double u = aff_u(A.D, rj, dn);
            A.dvg[(a & 1) * dvs + j0 + t] = u;
            if (A.D.aff.mu) mu_u += __ldg(A.D.aff.mu + rj) * u;
          } else {
            A.dvg[(a & 1) * dvs + j0 + t] = dn;
          }
        }
      }
      if (AFF) aff_mu_partial(A, mu_u, red);
      traced_sync(A, a, 0);
    }
    if (prof) A.prof[4 * a + 0] = gtimer();

    // ---------------- phase A: CSR pass, w = omega (X v) ----------------
    double acc_dAd = 0.0;
    for (int t = tid; t < chunk; t += kPcgThreads) acc_dAd += o.D[t] * o.d[t] * o.d[t];
    const double* vcur = A.dvg + (a == 0 ? dvs : (a & 1) * dvs);
    if (!AFF) {
      const bool multi = A.D.csr.nslab > 1;
      EpiCsr e{multi ? A.zpart : A.w, A.omega, 0.0, 0.0, multi};
      const double* icpt_src = A.D.icpt ? vcur + A.D.p : nullptr;
      if (A.D.csr.cta_task_ptr[blockIdx.x] == A.D.csr.cta_task_ptr[blockIdx.x + 1]) {
        // a CTA without CSR work still needs the row constant (combine loop)
        if (tid == 0) bc[2] = icpt_src ? __ldcg(icpt_src) : 0.0;
        __syncthreads();
      }
      FillBulkV0 f{vcur, &bf, icpt_src, bc + 2, &e.v0};
      run_pass<kPcgRing>(A.D.csr, sv, f, e, A.D.dbg);
      acc_dAd += e.acc;
    } else {
      // row constant u_icpt - mu'u (grid sum of the CTA partials, fixed order);
      // the dense block's u values are read from the published vector
      const double mu_u = reduce_partials(A.part + 3, gridDim.x, bc + 3);
      if (tid == 0) bc[2] = (A.D.icpt ? __ldcg(vcur + A.D.p) : 0.0) - mu_u;
      __syncthreads();
      const bool multi = A.D.csr.nslab > 1;
      EpiCsrA e{multi ? A.zpart : A.w, A.omega, bc[2], 0.0, multi,
                AffRow{A.D.aff.dense, vcur + A.D.p + A.D.icpt, A.D.aff.q}};
      FillBulkH f{vcur, &bf};
      run_pass<kPcgRing>(A.D.csr, sv, f, e, A.D.dbg);
      acc_dAd += e.acc;
    }
    if (A.D.csr.nslab > 1) {
      cg::this_grid().sync();
      const long long n = A.D.n;
      const double v0 = bc[2];
      const AffRow ar{A.D.aff.dense, vcur + A.D.p + A.D.icpt, AFF ? A.D.aff.q : 0};
      for (long long i = (long long)blockIdx.x * kPcgThreads + tid; i < n; i += (long long)gridDim.x * kPcgThreads) {
        double z = 0.0;
        for (int s = 0; s < A.D.csr.nslab; ++s) z += __ldcg(A.zpart + (long long)s * n + i);
        z += v0;
        if (AFF && ar.q) z += ar(i);
        const double wi = __ldg(A.omega + i) * z;
        A.w[i] = wi;
        acc_dAd += wi * z;
      }
    }
    {
      const double t = block_sum(acc_dAd, red);
      if (tid == 0) A.part[blockIdx.x * kPartStride] = t;
    }
    if (prof) A.prof[4 * a + 1] = gtimer();
    traced_sync(A, a, 1);
    if (AFF) {  // W = sum w and G_k = sum Dn[i,k] w_i: CTA partials over a row range
      const int q = A.D.aff.q, L = 1 + q;
      const long long n = A.D.n, r0 = n * blockIdx.x / gridDim.x, r1 = n * (blockIdx.x + 1) / gridDim.x;
      for (int k = 0; k < L; ++k) {
        double acc = 0.0;
        for (long long i = r0 + tid; i < r1; i += kPcgThreads) {
          const double wi = __ldcg(A.w + i);
          acc += k == 0 ? wi : __ldg(A.D.aff.dense + i * q + (k - 1)) * wi;
        }
        const double t = block_sum(acc, red);
        if (tid == 0) A.apart[(long long)blockIdx.x * L + k] = t;
      }
    }

    // ---------------- phase B: CSC pass, pieces of X' w ----------------
    bool dad_pending;
    {
      FillVecNDad f{A.w, &bf, A.part, (int)gridDim.x, bc, PCGS_DAD_IN_FILL && a > 0, false};
      EpiStore e{A.pieces, A.D.csc.nseg};  // A.D.csc.ids are the column-major piece slots (host: pcgs_pcg_full)
      run_pass<kPcgRing>(A.D.csc, sv, f, e, A.D.dbg);
      dad_pending = a > 0 && !f.done;
    }
    if (prof) A.prof[4 * a + 2] = gtimer();
    traced_sync(A, a, 2);
    if (tid == 0) ++st_applies;
    if (prof) A.prof[4 * a + 3] = gtimer();

    // ---------------- phase C: assemble, step, residual ----------------
    double alpha = 0.0;
    trace_stamp(A, a, 0);
    // (CTAs without CSC work: warp 0's loads of the dAd partials overlap the
    // piece staging round trip)
    double dpart = 0.0;
    if (dad_pending && tid < 32) dpart = lane_partials(A.part, gridDim.x, tid);
    const PieceRun pr = piece_run(o, A.D, j0);
    const bool staged = stage_pieces(pr, A.pieces, chunk, sv, A.D.smem_doubles);
    trace_stamp(A, a, 1);
    if (a > 0) {
      if (dad_pending) {
        if (tid < 32) {
          dpart = warp_sum(dpart);
          if (tid == 0) bc[0] = dpart;
        }
        __syncthreads();
      }
      const double dAd = bc[0];
      if (!(dAd > 0.0)) {
        if (tid == 0) {
          st_status = PCGS_NOT_PD;
          st_iter = a;
          st_fail = a;
        }
        break;
      }
      alpha = st_rz / dAd;
      if (blockIdx.x == 0 && tid == 0) A.alphas[a - 1] = alpha;
    }
    trace_stamp(A, a, 2);
    if (AFF) {  // grid totals of W and G_k (warp k sums line slot k over the CTAs, fixed order)
      const int L = 1 + A.D.aff.q, warp = tid >> 5, lane = tid & 31;
      if (warp < L) {
        double acc = 0.0;
        for (int c = lane; c < (int)gridDim.x; c += 32) acc += __ldcg(A.apart + (long long)c * L + warp);
        acc = warp_sum(acc);
        if (lane == 0) affg[warp] = acc;
      }
      __syncthreads();
    }
    // affine designs: raw column sum -> (g - mu W) / s, dense columns from G_k
    auto aff_ad = [&](int t, double cs) -> double {
      if (!AFF) return cs;
      const long long j = j0 + t, r = ref_index(j, A.D.p, A.D.lead()), k = j - A.D.p - A.D.icpt;
      const double raw = k >= 0 ? affg[1 + k] : cs;
      const double mu = A.D.aff.mu ? __ldg(A.D.aff.mu + r) : 0.0, sc = A.D.aff.sc ? __ldg(A.D.aff.sc + r) : 1.0;
      return (raw - mu * affg[0]) / sc;
    };
    double t_rms = 0.0, t_rz = 0.0;
    for (int t = tid; t < chunk; t += kPcgThreads) {
      if (j0 + t >= pt) continue;
      const double Ad = aff_ad(t, owned_column_sum(pr, A.pieces, t, sv, staged)) + o.D[t] * o.d[t];
      double rv;
      if (a == 0) {
        rv = o.b[t] - Ad;
      } else {
        o.x[t] = fma(alpha, o.d[t], o.x[t]);
        rv = fma(-alpha, Ad, o.r[t]);
        if (A.iterates) A.iterates[(long long)a * pt + ref_index(j0 + t, A.D.p, A.D.lead())] = o.x[t];
      }
      o.r[t] = rv;
      const double zn = o.m[t] * rv;
      o.z[t] = zn;
      const double tj = o.s[t] * rv;
      t_rms += tj * tj;
      t_rz += rv * zn;
    }
    trace_stamp(A, a, 3);
    block_sum2(t_rms, t_rz, red);
    if (tid == 0) {
      A.part[blockIdx.x * kPartStride + 1] = t_rms;
      A.part[blockIdx.x * kPartStride + 2] = t_rz;
    }
    trace_stamp(A, a, 4);
    traced_sync(A, a, 3);
  }

  __syncthreads();
  {
    const long long pt = A.D.pt;
    const int chunk = (int)((pt + gridDim.x - 1) / gridDim.x);
    const long long j0 = (long long)blockIdx.x * chunk;
    const OwnState o = own_state(sv, A.D, chunk, j0);
    for (int t = tid; t < chunk; t += kPcgThreads)
      if (j0 + t < pt) A.x[ref_index(j0 + t, A.D.p, A.D.lead())] = o.x[t];
  }
  if (blockIdx.x == 0 && tid == 0) {
    A.result[0] = st_iter;
    A.result[1] = st_status;
    A.result[2] = st_fail;
    A.result[3] = st_applies;
  }
}

#include "pg.cuh"

__global__ void k_pg(const double* z, long long n, unsigned long long seed, unsigned long long stream, double* omega,
                     long long row0) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    Philox R(seed, stream, (unsigned)(row0 + i));
    omega[i] = pg_draw1(z[i], R);
  }
}

// =====================================================================
// C ABI
// =====================================================================
extern "C" {

int pcgs_version(void) { return 1; }
const char* pcgs_last_error(void) { return g_err.c_str(); }


static int set_smem_attrs() {
  int rc;
  if ((rc = raise_smem_limit(k_csr_matvec<512, 2>)) || (rc = raise_smem_limit(k_csr_matvec<1024, 1>)) ||
      (rc = raise_smem_limit(k_csr_phi<512, 2>)) || (rc = raise_smem_limit(k_csr_phi<1024, 1>)) ||
      (rc = raise_smem_limit(k_csc_vec<512, 2>)) || (rc = raise_smem_limit(k_csc_vec<1024, 1>)) ||
      (rc = raise_smem_limit(k_pcg<false>)) || (rc = raise_smem_limit(k_pcg<true>)))
    return rc;
  return PCGS_OK;
}

int pcgs_design_create(int64_t n, int64_t p, const int64_t* row_ptr_h, const int32_t* col_idx_h, int intercept,
                       int slab_max, int device, pcgs_design_t* out) {
  return pcgs_design_create_ex(n, p, row_ptr_h, col_idx_h, intercept, slab_max, device, 0, out);
}

int pcgs_design_create_ex(int64_t n, int64_t p, const int64_t* row_ptr_h, const int32_t* col_idx_h, int intercept,
                          int slab_max, int device, int grid, pcgs_design_t* out) {
  return pcgs_design_create_affine(n, p, row_ptr_h, col_idx_h, intercept, 0, slab_max, device, grid, out);
}

int pcgs_design_set_affine(pcgs_design_t d, const double* dense, const double* mu, const double* sc) {
  if (!d) return fail(PCGS_EINVAL, "null design");
  AffineDev& F = d->dev.aff;
  if (F.q > 0 && !dense) return fail(PCGS_EINVAL, "the design has dense columns: dense values required");
  F.dense = F.q > 0 ? dense : nullptr;
  F.mu = mu;
  F.sc = sc;
  F.on = F.q > 0 || mu || sc;
  return PCGS_OK;
}

int pcgs_design_create_affine(int64_t n, int64_t p, const int64_t* row_ptr_h, const int32_t* col_idx_h,
                              int intercept, int q_dense, int slab_max, int device, int grid, pcgs_design_t* out) {
  if (!out || !row_ptr_h || (!col_idx_h && row_ptr_h[n] > 0)) return fail(PCGS_EINVAL, "null argument");
  *out = nullptr;
  CUDA_TRY(cudaSetDevice(device));
  cudaDeviceProp prop;
  CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  const int sms = std::min(prop.multiProcessorCount, kMaxGrid);
  if (grid < 0 || grid > sms) return fail(PCGS_EINVAL, "grid must be in [0, SM count]");
  const int G = grid > 0 ? grid : sms;
  if (q_dense < 0 || q_dense > kAffMaxQ) return fail(PCGS_EINVAL, "dense block: at most 32 columns");
  DesignHost H;
  std::string err = build_design(n, p, row_ptr_h, col_idx_h, intercept, slab_max, G, H, q_dense,
                                 g_nranges > 0 ? g_nranges : kDefaultRanges);
  if (!err.empty()) return fail(PCGS_EINVAL, err);
  pcgs_design* D = new pcgs_design();
  D->dev.aff = AffineDev{0, q_dense, nullptr, nullptr, nullptr};
  D->device = device;
  DesignDev& dd = D->dev;
  dd.n = n;
  dd.p = p;
  dd.pt = H.p_total;
  dd.icpt = H.intercept;
  dd.G = G;
  int64_t maxlen = 0;
  for (const PassHost* P : {&H.csr, &H.csc})
    for (int q = 0; q < P->nslab; ++q) maxlen = std::max<int64_t>(maxlen, P->slab_lo[q + 1] - P->slab_lo[q]);
  dd.smem_doubles = std::max((int)((maxlen + 1 + 15) / 16 * 16), H.slab_area);  // slab + sentinel + replicas
  dd.own_global = nullptr;
  int rc;
  {
    // own-slice PCG state next to the slab when it fits, else in global
    // memory allocated by each solve (pcgs_pcg_full)
    const long long chunk = (H.p_total + G - 1) / G;
    dd.own_in_global = (long long)dd.smem_doubles * 8 + chunk * 64 + 16 + 1024 > 227 * 1024;
  }
  if ((rc = upload_pass(D, H.csr, dd.csr)) || (rc = upload_pass(D, H.csc, dd.csc))) {
    pcgs_design_destroy(D);
    return rc;
  }
  if ((rc = set_smem_attrs())) {
    pcgs_design_destroy(D);
    return rc;
  }
  // make freed stream-ordered scratch stay cached in the pool
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    // scratch freed on one chain's stream must not be handed to another
    // stream behind an inserted dependency: that would serialise chains that
    // run side by side (gibbs_run_concurrent)
    int no = 0;
    cudaMemPoolSetAttribute(pool, cudaMemPoolReuseAllowInternalDependencies, &no);
  }
  int64_t* I = D->info;
  memset(I, 0, sizeof(D->info));
  I[0] = n;
  I[1] = p;
  I[2] = H.p_total;
  I[3] = H.nnz;
  I[4] = H.csr.nslab;
  I[5] = H.csc.nslab;
  I[6] = (int64_t)(H.csr.idx.size() / kVecIdx);
  I[7] = (int64_t)(H.csc.idx.size() / kVecIdx);
  I[8] = (int64_t)H.csr.blocks.size();
  I[9] = (int64_t)H.csc.blocks.size();
  I[10] = H.csc.nseg;
  I[11] = G;
  I[12] = device;
  I[13] = (int64_t)(H.csr.idx.size() + H.csc.idx.size()) * 2;
  I[14] = H.slab_max;
  I[15] = (H.csr.lds_conflict_excess + H.csc.lds_conflict_excess) * 1000000 /
          std::max<int64_t>(1, H.csr.lds_groups + H.csc.lds_groups);
  *out = D;
  return PCGS_OK;
}

int pcgs_store_selftest(int64_t n, int64_t p, const int64_t* row_ptr_h, const int32_t* col_idx_h, int intercept,
                        int slab_max, int grid, int64_t* stats_h) {
  if (!row_ptr_h || grid < 1) return fail(PCGS_EINVAL, "null argument");
  DesignHost H;
  std::string err = build_design(n, p, row_ptr_h, col_idx_h, intercept, slab_max, grid, H, 0,
                                 g_nranges > 0 ? g_nranges : kDefaultRanges);
  if (!err.empty()) return fail(PCGS_EINVAL, err);
  err = verify_design(H, row_ptr_h, col_idx_h);
  if (stats_h) {
    stats_h[0] = H.csr.nslab;
    stats_h[1] = H.csc.nslab;
    stats_h[2] = (int64_t)(H.csr.idx.size() / kVecIdx);
    stats_h[3] = (int64_t)(H.csc.idx.size() / kVecIdx);
    stats_h[4] = H.csc.nseg;
    stats_h[5] = H.csr.lds_groups + H.csc.lds_groups;
    stats_h[6] = H.csr.lds_conflict_excess + H.csc.lds_conflict_excess;
    stats_h[7] = (int64_t)(H.csr.idx.size() + H.csc.idx.size()) * 2;
  }
  if (!err.empty()) return fail(PCGS_EUNSUP - 100, "store self-test failed: " + err);
  return PCGS_OK;
}

int pcgs_synth_design(int64_t n, int64_t p, double rate_lo, double rate_hi, uint64_t seed, int64_t* row_ptr_h,
                      int32_t* col_idx_h, int64_t cap, int64_t* nnz_h) {
  if (n < 1 || p < 0 || !(rate_lo > 0) || !(rate_hi >= rate_lo) || !row_ptr_h || !nnz_h)
    return fail(PCGS_EINVAL, "bad argument");
  static thread_local std::vector<int64_t> rp;
  static thread_local std::vector<int32_t> ci;
  if (!col_idx_h) {  // first call: generate and report nnz
    *nnz_h = synth_binary_design(n, p, rate_lo, rate_hi, seed, rp, ci);
    memcpy(row_ptr_h, rp.data(), (n + 1) * sizeof(int64_t));
    return PCGS_OK;
  }
  if (cap < (int64_t)ci.size()) return fail(PCGS_EINVAL, "col_idx buffer too small");
  memcpy(col_idx_h, ci.data(), ci.size() * sizeof(int32_t));
  *nnz_h = (int64_t)ci.size();
  std::vector<int64_t>().swap(rp);
  std::vector<int32_t>().swap(ci);
  return PCGS_OK;
}

struct pcgs_mtx {
  pcgs::MtxPattern m;
};

static int mtx_status(int kind) {
  return kind == pcgs::kMtxIo ? PCGS_EIO : kind == pcgs::kMtxFormat ? PCGS_EFORMAT : PCGS_EUNSUP;
}

int pcgs_mtx_load(const char* path, pcgs_mtx_t* out, int64_t* info_h) {
  if (!path || !out || !info_h) return fail(PCGS_EINVAL, "null argument");
  *out = nullptr;
  auto* h = new (std::nothrow) pcgs_mtx;
  if (!h) return fail(PCGS_ENOMEM, "host allocation failed");
  std::string msg;
  int rc;
  try {
    rc = pcgs::mtx_load(path, h->m, msg);
  } catch (const std::bad_alloc&) {
    delete h;
    return fail(PCGS_ENOMEM, std::string(path) + ": host memory exhausted while parsing");
  }
  if (rc != pcgs::kMtxOk) {
    delete h;
    return fail(mtx_status(rc), msg);
  }
  const auto& m = h->m;
  const int64_t info[8] = {m.n, m.p, (int64_t)m.col_idx.size(), m.entries, m.field, m.symmetry, m.format,
                           m.zeros_dropped};
  memcpy(info_h, info, sizeof info);
  *out = h;
  return PCGS_OK;
}

int pcgs_mtx_export(pcgs_mtx_t h, int64_t* row_ptr_h, int32_t* col_idx_h) {
  if (!h || !row_ptr_h || (!col_idx_h && !h->m.col_idx.empty())) return fail(PCGS_EINVAL, "null argument");
  memcpy(row_ptr_h, h->m.row_ptr.data(), h->m.row_ptr.size() * sizeof(int64_t));
  if (!h->m.col_idx.empty()) memcpy(col_idx_h, h->m.col_idx.data(), h->m.col_idx.size() * sizeof(int32_t));
  return PCGS_OK;
}

int pcgs_mtx_free(pcgs_mtx_t h) {
  delete h;
  return PCGS_OK;
}

int pcgs_mtx_write(const char* path, int64_t n, int64_t p, const int64_t* row_ptr_h, const int32_t* col_idx_h,
                   int field, int gz) {
  if (!path || n < 0 || p < 0 || !row_ptr_h || (field != 0 && field != 1)) return fail(PCGS_EINVAL, "bad argument");
  if (row_ptr_h[0] != 0) return fail(PCGS_EINVAL, "row_ptr must start at 0");
  for (int64_t r = 0; r < n; ++r)
    if (row_ptr_h[r + 1] < row_ptr_h[r]) return fail(PCGS_EINVAL, "row_ptr must be non-decreasing");
  if (row_ptr_h[n] > 0 && !col_idx_h) return fail(PCGS_EINVAL, "null col_idx");
  for (int64_t t = 0; t < row_ptr_h[n]; ++t)
    if (col_idx_h[t] < 0 || col_idx_h[t] >= p) return fail(PCGS_EINVAL, "column index out of range");
  std::string msg;
  const int rc = pcgs::mtx_write(path, n, p, row_ptr_h, col_idx_h, field, gz, msg);
  return rc == pcgs::kMtxOk ? PCGS_OK : fail(mtx_status(rc), msg);
}

int pcgs_design_destroy(pcgs_design_t d) {
  if (!d) return PCGS_OK;
  cudaSetDevice(d->device);
  for (void* p : d->allocs) cudaFree(p);
  delete d;
  return PCGS_OK;
}

int pcgs_design_info(pcgs_design_t d, int64_t* info_h) {
  if (!d || !info_h) return fail(PCGS_EINVAL, "null argument");
  memcpy(info_h, d->info, sizeof(d->info));
  return PCGS_OK;
}

}  // extern "C"

// Affine designs: the CSR row constants (cbuf) of a reference-layout vector v.
int aff_pre(pcgs_design* d, const double* v, Scratch& S, cudaStream_t s, double** cbuf) {
  *cbuf = nullptr;
  const DesignDev& D = d->dev;
  if (!D.aff.on) return PCGS_OK;
  *cbuf = S.get<double>(1 + D.aff.q);
  if (!*cbuf) return fail(PCGS_ENOMEM, "scratch allocation failed");
  k_aff_pre<<<1, kThreads, 0, s>>>(D, v, *cbuf);
  CUDA_TRY(cudaGetLastError());
  return PCGS_OK;
}

extern "C" {

// Affine designs: W and the dense-column sums of w (gbuf, see k_aff_tw_part).
static int aff_tw(pcgs_design_t d, const double* w, int squares, Scratch& S, cudaStream_t s, double** gbuf) {
  *gbuf = nullptr;
  const DesignDev& D = d->dev;
  if (!D.aff.on) return PCGS_OK;
  const int Sw = 1 + 2 * D.aff.q;
  double* part = S.get<double>((size_t)D.G * Sw);
  *gbuf = S.get<double>(Sw);
  if (!part || !*gbuf) return fail(PCGS_ENOMEM, "scratch allocation failed");
  k_aff_tw_part<<<D.G, 256, 0, s>>>(D, w, squares, part);
  k_aff_tw_fin<<<1, 64, 0, s>>>(part, D.G, Sw, *gbuf);
  CUDA_TRY(cudaGetLastError());
  return PCGS_OK;
}

static int launch_csr(pcgs_design_t d, bool phi, const double* v, const double* omega, double* out, cudaStream_t s,
                      Scratch& S) {
  const DesignDev& D = d->dev;
  const size_t sm = smem_bytes(D);
  double* cbuf;
  int rc;
  if ((rc = aff_pre(d, v, S, s, &cbuf))) return rc;
  if (D.csr.nslab == 1) {
    if (phi) PASS_LAUNCH(k_csr_phi, D, sm, s, D, v, omega, out, cbuf);
    else PASS_LAUNCH(k_csr_matvec, D, sm, s, D, v, out, cbuf);
  } else {
    double* part = S.get<double>((size_t)D.csr.nslab * D.n);
    if (!part) return fail(PCGS_ENOMEM, "scratch allocation failed");
    if (phi) PASS_LAUNCH(k_csr_phi, D, sm, s, D, v, omega, part, cbuf);
    else PASS_LAUNCH(k_csr_matvec, D, sm, s, D, v, part, cbuf);
    k_rows_combine<<<D.G * 4, 256, 0, s>>>(D, part, v, phi ? omega : nullptr, out, cbuf);
  }
  CUDA_TRY(cudaGetLastError());
  return PCGS_OK;
}

int pcgs_matvec(pcgs_design_t d, const double* v, double* out, pcgs_stream_t stream) {
  if (!d || !v || !out) return fail(PCGS_EINVAL, "null argument");
  d->dev.dbg = g_dbg;
  cudaStream_t s = (cudaStream_t)stream;
  Scratch S(s);
  return launch_csr(d, false, v, nullptr, out, s, S);
}

int pcgs_matvec_t(pcgs_design_t d, const double* w, double* out, pcgs_stream_t stream) {
  if (!d || !w || !out) return fail(PCGS_EINVAL, "null argument");
  d->dev.dbg = g_dbg;
  const DesignDev& D = d->dev;
  cudaStream_t s = (cudaStream_t)stream;
  Scratch S(s);
  double* pieces = S.get<double>(D.csc.nseg);
  if (!pieces) return fail(PCGS_ENOMEM, "scratch allocation failed");
  double* gbuf;
  int rc;
  if ((rc = aff_tw(d, w, 0, S, s, &gbuf))) return rc;
  PASS_LAUNCH(k_csc_vec, D, smem_bytes(D), s, D, w, pieces);
  k_assemble<<<(int)((D.pt + 255) / 256), 256, 0, s>>>(D, pieces, nullptr, nullptr, nullptr, 0, 0, 0, out, nullptr,
                                                       gbuf);
  CUDA_TRY(cudaGetLastError());
  return PCGS_OK;
}

int pcgs_phi_apply(pcgs_design_t d, const double* omega, const double* prior_diag, const double* v, double* out,
                   pcgs_stream_t stream) {
  if (!d || !omega || !prior_diag || !v || !out) return fail(PCGS_EINVAL, "null argument");
  const DesignDev& D = d->dev;
  cudaStream_t s = (cudaStream_t)stream;
  Scratch S(s);
  double* w = S.get<double>(D.n + 2);
  double* pieces = S.get<double>(D.csc.nseg);
  if (!w || !pieces) return fail(PCGS_ENOMEM, "scratch allocation failed");
  int rc = launch_csr(d, true, v, omega, w, s, S);
  if (rc) return rc;
  double* gbuf;
  if ((rc = aff_tw(d, w, 0, S, s, &gbuf))) return rc;
  PASS_LAUNCH(k_csc_vec, D, smem_bytes(D), s, D, w, pieces);
  k_assemble<<<(int)((D.pt + 255) / 256), 256, 0, s>>>(D, pieces, prior_diag, v, nullptr, 0, 0, 1, out, nullptr,
                                                       gbuf);
  CUDA_TRY(cudaGetLastError());
  return PCGS_OK;
}

int pcgs_phi_diagonal(pcgs_design_t d, const double* omega, const double* prior_diag, double* out,
                      pcgs_stream_t stream) {
  if (!d || !omega || !prior_diag || !out) return fail(PCGS_EINVAL, "null argument");
  const DesignDev& D = d->dev;
  cudaStream_t s = (cudaStream_t)stream;
  Scratch S(s);
  double* pieces = S.get<double>(D.csc.nseg);
  if (!pieces) return fail(PCGS_ENOMEM, "scratch allocation failed");
  double* gbuf;
  int rc;
  if ((rc = aff_tw(d, omega, 1, S, s, &gbuf))) return rc;
  PASS_LAUNCH(k_csc_vec, D, smem_bytes(D), s, D, omega, pieces);
  k_assemble<<<(int)((D.pt + 255) / 256), 256, 0, s>>>(D, pieces, prior_diag, nullptr, nullptr, 0, 0, 3, out, nullptr,
                                                       gbuf);
  CUDA_TRY(cudaGetLastError());
  return PCGS_OK;
}

int pcgs_rhs(pcgs_design_t d, const double* kappa, const double* omega, const double* prior_diag,
             const double* linear, const double* eta, const double* delta, uint64_t seed, uint64_t stream_id,
             double* b, pcgs_stream_t stream) {
  if (!d || !omega || !prior_diag || !b) return fail(PCGS_EINVAL, "null argument");
  const DesignDev& D = d->dev;
  cudaStream_t s = (cudaStream_t)stream;
  Scratch S(s);
  double* pieces = S.get<double>(D.csc.nseg);
  double* u = S.get<double>(D.n + 2);
  if (!pieces || !u) return fail(PCGS_ENOMEM, "scratch allocation failed");
  // u = kappa + sqrt(omega) eta once per row (Philox once per row), then the
  // CSC pass TMA-fills its row slabs from u like any X' w
  FillRhs f{kappa, omega, eta, seed, kStreamEta ^ stream_id, 0};
  k_rhs_u<<<(int)std::min<long long>((D.n + 255) / 256, 148 * 8), 256, 0, s>>>(f, D.n, u);
  double* gbuf;
  int rc;
  if ((rc = aff_tw(d, u, 0, S, s, &gbuf))) return rc;
  PASS_LAUNCH(k_csc_vec, D, smem_bytes(D), s, D, u, pieces);
  k_assemble<<<(int)((D.pt + 255) / 256), 256, 0, s>>>(D, pieces, prior_diag, nullptr, delta, seed,
                                                       kStreamDelta ^ stream_id, 2, b, linear, gbuf);
  CUDA_TRY(cudaGetLastError());
  return PCGS_OK;
}

int pcgs_pcg(pcgs_design_t d, const double* omega, const double* prior_diag, const double* minv, const double* scale,
             const double* b, double* x, int32_t max_iter, double rtol, double* trace, double* alphas, double* betas,
             int32_t* result, pcgs_stream_t stream) {
  return pcgs_pcg_full(d, omega, prior_diag, minv, scale, b, x, max_iter, rtol, trace, alphas, betas, nullptr, result,
                       stream);
}

int pcgs_pcg_full(pcgs_design_t d, const double* omega, const double* prior_diag, const double* minv,
                  const double* scale, const double* b, double* x, int32_t max_iter, double rtol, double* trace,
                  double* alphas, double* betas, double* iterates, int32_t* result, pcgs_stream_t stream) {
  if (!d || !omega || !prior_diag || !minv || !scale || !b || !x || !trace || !alphas || !betas || !result)
    return fail(PCGS_EINVAL, "null argument");
  if (max_iter < 1) return fail(PCGS_EINVAL, "max_iter must be at least 1");
  const DesignDev& D = d->dev;
  cudaStream_t s = (cudaStream_t)stream;
  Scratch S(s);
  PcgArgs A;
  A.D = D;
  A.omega = omega;
  A.diag = prior_diag;
  A.minv = minv;
  A.scale = scale;
  A.b = b;
  A.x = x;
  A.max_iter = max_iter;
  A.rtol = rtol;
  A.trace = trace;
  A.alphas = alphas;
  A.betas = betas;
  A.result = result;
  A.w = S.get<double>(D.n + 2);
  A.zpart = D.csr.nslab > 1 ? S.get<double>((size_t)D.csr.nslab * D.n) : nullptr;
  A.pieces = S.get<double>(D.csc.nseg);
  A.zv = S.get<double>(D.pt + 2);
  A.dvg = S.get<double>(2 * ((D.pt + 15) / 16 * 16) + 16);
  A.part = S.get<double>((size_t)kPartStride * D.G);
  A.prof = g_prof;
  A.D.dbg = g_dbg;
  A.D.csc.ids = D.csc.ids_perm;  // k_pcg's CSC pass emits to the column-major piece slots (store.h)
  A.iterates = iterates;
  if (D.own_in_global) {  // per-solve state: concurrent solves on one design must not share it
    const long long chunk = (D.pt + D.G - 1) / D.G;
    A.D.own_global = S.get<double>((size_t)D.G * 8 * chunk);
    if (!A.D.own_global) return fail(PCGS_ENOMEM, "scratch allocation failed (PCG state)");
  }
  if (!A.w || !A.pieces || !A.zv || !A.dvg || !A.part || (D.csr.nslab > 1 && !A.zpart))
    return fail(PCGS_ENOMEM, "scratch allocation failed");
  A.apart = nullptr;
  if (D.aff.on) {
    A.apart = S.get<double>((size_t)D.G * (1 + D.aff.q));
    if (!A.apart) return fail(PCGS_ENOMEM, "scratch allocation failed");
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(D.G);
  cfg.blockDim = dim3(kPcgThreads);
  cfg.dynamicSmemBytes = pcg_smem_bytes(D);
  cfg.stream = s;
  cudaLaunchAttribute attrs[2];
  int na = 0;
  attrs[na].id = cudaLaunchAttributeCooperative;
  attrs[na].val.cooperative = 1;
  ++na;
  if (g_l2_persist_mb > 0) {
    // keep the leading part of the CSC index stream resident in L2 across
    // iterations (persisting carve-out); the rest streams
    static bool limit_set = false;
    const size_t want = (size_t)g_l2_persist_mb << 20;
    if (!limit_set) {
      cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want);
      limit_set = true;
    }
    attrs[na].id = cudaLaunchAttributeAccessPolicyWindow;
    attrs[na].val.accessPolicyWindow.base_ptr = (void*)D.csc.vec;
    attrs[na].val.accessPolicyWindow.num_bytes = want;
    attrs[na].val.accessPolicyWindow.hitRatio = 1.0f;
    attrs[na].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attrs[na].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    ++na;
  }
  cfg.attrs = attrs;
  cfg.numAttrs = na;
  if (D.aff.on) CUDA_TRY(cudaLaunchKernelEx(&cfg, k_pcg<true>, A));
  else CUDA_TRY(cudaLaunchKernelEx(&cfg, k_pcg<false>, A));
  return PCGS_OK;
}

// ---------------------------------------------------------------------------
// Generic-operator PCG: the reference loop (cg.py:105-192) with the vector
// algebra on device and the operator supplied as a callback (any duck-typed
// `phi`, cg.py:110-113).  Desk-scale: one CTA per vector kernel, host reads
// the three scalars of every iteration exactly as the reference does.
// ---------------------------------------------------------------------------
__device__ double block_sum_1024(double v, double* red) { return block_sum(v, red); }

// mode 0: r = b - Ad, x kept; sums (s r)^2
// mode 1: z = minv r, d = z;   sums r.z
// mode 2: sums d.Ad
// mode 3: x += a d, r -= a Ad, z = minv r; sums (s r)^2, r.z
// mode 4: d = z + beta d
__global__ void __launch_bounds__(kThreads) k_opvec(int mode, long long p, double a, const double* b,
                                                    const double* minv, const double* scale, double* x,
                                                    double* r, double* z, double* d, const double* Ad,
                                                    double* out2) {
  __shared__ double red[64];
  double s0 = 0.0, s1 = 0.0;
  for (long long i = threadIdx.x; i < p; i += blockDim.x) {
    if (mode == 0) {
      const double ri = b[i] - Ad[i];
      r[i] = ri;
      const double t = scale[i] * ri;
      s0 += t * t;
    } else if (mode == 1) {
      const double zi = minv[i] * r[i];
      z[i] = zi;
      d[i] = zi;
      s1 += r[i] * zi;
    } else if (mode == 2) {
      s0 += d[i] * Ad[i];
    } else if (mode == 3) {
      x[i] = fma(a, d[i], x[i]);
      const double ri = fma(-a, Ad[i], r[i]);
      r[i] = ri;
      const double zi = minv[i] * ri;
      z[i] = zi;
      const double t = scale[i] * ri;
      s0 += t * t;
      s1 += ri * zi;
    } else {
      d[i] = fma(a, d[i], z[i]);
    }
  }
  block_sum2(s0, s1, red);
  if (threadIdx.x == 0 && out2) {
    out2[0] = s0;
    out2[1] = s1;
  }
}

int pcgs_pcg_op(pcgs_apply_fn fn, void* ctx, int64_t p, const double* minv, const double* scale, const double* b,
                double* x, double* dbuf, double* adbuf, int32_t max_iter, double rtol, double* trace_h,
                double* alphas_h, double* betas_h, int32_t* result_h, pcgs_stream_t stream) {
  return pcgs_pcg_op_full(fn, ctx, p, minv, scale, b, x, dbuf, adbuf, max_iter, rtol, trace_h, alphas_h, betas_h,
                          nullptr, result_h, stream);
}

int pcgs_pcg_op_full(pcgs_apply_fn fn, void* ctx, int64_t p, const double* minv, const double* scale,
                     const double* b, double* x, double* dbuf, double* adbuf, int32_t max_iter, double rtol,
                     double* trace_h, double* alphas_h, double* betas_h, double* iterates, int32_t* result_h,
                     pcgs_stream_t stream) {
  if (!fn || p < 1 || !minv || !scale || !b || !x || !trace_h || !alphas_h || !betas_h || !result_h)
    return fail(PCGS_EINVAL, "null argument");
  if (max_iter < 1) return fail(PCGS_EINVAL, "max_iter must be at least 1");
  cudaStream_t s = (cudaStream_t)stream;
  Scratch S(s);
  double* r = S.get<double>(p);
  double* z = S.get<double>(p);
  double* dv = dbuf ? dbuf : S.get<double>(p);
  double* Ad = adbuf ? adbuf : S.get<double>(p);
  double* sc = S.get<double>(2);
  if (!r || !z || !dv || !Ad || !sc) return fail(PCGS_ENOMEM, "scratch allocation failed");
  double h2[2];
  auto run = [&](int mode, double a, double* outp) -> int {
    k_opvec<<<1, kThreads, 0, s>>>(mode, p, a, b, minv, scale, x, r, z, dv, Ad, outp);
    CUDA_TRY(cudaGetLastError());
    if (outp) {
      CUDA_TRY(cudaMemcpyAsync(h2, outp, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
      CUDA_TRY(cudaStreamSynchronize(s));
    }
    return PCGS_OK;
  };
  auto apply = [&](const double* v) -> int {
    CUDA_TRY(cudaStreamSynchronize(s));
    int rc = fn(ctx, v, Ad);
    if (rc) return fail(PCGS_ECUDA, "operator callback failed");
    return PCGS_OK;
  };
  int rc;
  int applies = 0, k = 0;
  result_h[2] = -1;
  if (iterates) CUDA_TRY(cudaMemcpyAsync(iterates, x, p * sizeof(double), cudaMemcpyDeviceToDevice, s));
  if ((rc = apply(x))) return rc;
  ++applies;
  if ((rc = run(0, 0.0, sc))) return rc;
  double rms = std::sqrt(h2[0] / (double)p);
  trace_h[0] = rms;
  auto finish = [&](int status, int fail_iter) {
    result_h[0] = k;
    result_h[1] = status;
    result_h[2] = fail_iter;
    result_h[3] = applies;
    return PCGS_OK;
  };
  if (!std::isfinite(rms)) return finish(PCGS_NONFINITE, 0);
  if (!(rms > rtol)) return finish(PCGS_CONVERGED, -1);
  if ((rc = run(1, 0.0, sc))) return rc;
  double rz = h2[1];
  while (k < max_iter) {
    ++k;
    if ((rc = apply(dv))) return rc;
    ++applies;
    if ((rc = run(2, 0.0, sc))) return rc;
    const double dAd = h2[0];
    if (!(dAd > 0)) return finish(PCGS_NOT_PD, k);
    const double alpha = rz / dAd;
    alphas_h[k - 1] = alpha;
    if ((rc = run(3, alpha, sc))) return rc;
    if (iterates)
      CUDA_TRY(cudaMemcpyAsync(iterates + (size_t)k * p, x, p * sizeof(double), cudaMemcpyDeviceToDevice, s));
    rms = std::sqrt(h2[0] / (double)p);
    trace_h[k] = rms;
    if (rms <= rtol) return finish(PCGS_CONVERGED, -1);
    if (!std::isfinite(rms)) return finish(PCGS_NONFINITE, k);
    const double beta = h2[1] / rz;
    betas_h[k - 1] = beta;
    rz = h2[1];
    if ((rc = run(4, beta, nullptr))) return rc;
  }
  return finish(PCGS_MAX_ITER, -1);
}

int pcgs_debug_profile(void* buf) {
  g_prof = (unsigned long long*)buf;
  return PCGS_OK;
}

int pcgs_debug_sync_times(void* buf) {
  unsigned long long* p = (unsigned long long*)buf;
  CUDA_TRY(cudaMemcpyToSymbol(g_sync_times, &p, sizeof(p)));
  return PCGS_OK;
}

int pcgs_debug_cta_times(void* buf) {
  unsigned long long* p = (unsigned long long*)buf;
  CUDA_TRY(cudaMemcpyToSymbol(g_cta_times, &p, sizeof(p)));
  return PCGS_OK;
}

int pcgs_debug_option(int key, int value) {
  if (key == 1) g_dbg = value;
  if (key == 2) g_l2_persist_mb = value;
  if (key == 3) g_nranges = value;
  return PCGS_OK;
}

int pcgs_copy(void* dst, const void* src, int64_t bytes, int kind) {
  if (bytes < 0 || (bytes > 0 && (!dst || !src))) return fail(PCGS_EINVAL, "null argument");
  if (bytes == 0) return PCGS_OK;
  const cudaMemcpyKind k = kind == 0 ? cudaMemcpyHostToDevice : kind == 1 ? cudaMemcpyDeviceToHost
                                                                          : cudaMemcpyDeviceToDevice;
  CUDA_TRY(cudaMemcpy(dst, src, (size_t)bytes, k));
  return PCGS_OK;
}

int pcgs_pg_draw(const double* z, int64_t n, uint64_t seed, uint64_t stream_id, double* omega,
                 pcgs_stream_t stream) {
  return pcgs_pg_draw_rows(z, n, 0, seed, stream_id, omega, stream);
}

int pcgs_pg_draw_rows(const double* z, int64_t n, int64_t row0, uint64_t seed, uint64_t stream_id, double* omega,
                      pcgs_stream_t stream) {
  if (n < 0 || (n > 0 && (!z || !omega))) return fail(PCGS_EINVAL, "null argument");
  if (n == 0) return PCGS_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int blocks = (int)std::min<int64_t>((n + 127) / 128, 148 * 16);
  k_pg<<<blocks, 128, 0, s>>>(z, n, seed, kStreamPG ^ stream_id, omega, row0);
  CUDA_TRY(cudaGetLastError());
  return PCGS_OK;
}

}  // extern "C"
