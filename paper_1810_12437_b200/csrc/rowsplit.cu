// Row-split PCG: the whole solve over R row shards in one persistent kernel
// per GPU, with the per-iteration exchange of the X'w partials fused into the
// kernel over peer memory (BASELINE config 5).
//
// Reference semantics: pcg_solve (pkg/src/priorcg/cg.py:105-192) on
// Phi = sum_r X_r' Omega_r X_r + D (sampler.py:53-58), rows of X split into
// contiguous shards (parallel.row_partition).  p-length vectors are
// replicated on every rank.  Per iteration each rank
//   A. runs its CSR pass over its rows (z_r = X_r d, w_r = omega_r z_r, and
//      the partial z_r' Omega_r z_r),
//   B. runs its CSC pass (pieces of X_r' w_r), then, after a local grid
//      barrier, sums the pieces of every column into its partial vector
//      g_r = X_r' w_r in a parity-double-buffered exchange region,
//   X. meets every other rank at one exchange barrier,
//   C. forms Phi d = sum_q g_q + D d for its owned columns (coalesced peer
//      loads over NVLink, rank order) and takes the CG step on its replicated
//      vectors.
// Every rank sums the same numbers in the same order, so all ranks hold
// bitwise identical iterates and take identical convergence decisions; there
// is no other collective.  dAd = sum_r z_r' Omega_r z_r + d'Dd (the rank
// partials in rank order, the prior term from the replicated owned slices).
//
// One grid can also host several ranks (`n_local` > 1): rank groups of Gr
// CTAs each, the exchange barrier then being the grid barrier.  That is how
// the decomposition runs and is validated on a single GPU; with one rank per
// GPU (`n_local` = 1) the barrier adds a flag exchange over peer memory
// (system-scope release/acquire) between two grid barriers.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "internal.cuh"
#include "rowsplit.h"

namespace cg = cooperative_groups;

namespace {

constexpr int kRsMaxRanks = 64;
constexpr int kRsMaxLocal = 8;    // ranks hosted by one grid
constexpr int kMaxGridRs = 256;

// Exchange region of one rank (one allocation, IPC-shareable):
//   header (64 B) | inbox flags [kRsMaxRanks] u64 | scalar slot (64 B) |
//   part [2][16 * G] f64 | gsum [2][p_total (padded)] f64
struct RsHeader {
  long long pt, G, bytes, n;
  long long pad[4];
};

struct RsLayout {
  size_t flags, scal, part, gsum, gstride, bytes;
  static RsLayout of(long long pt, long long G) {
    RsLayout L;
    L.flags = sizeof(RsHeader);
    L.scal = L.flags + kRsMaxRanks * sizeof(unsigned long long);
    L.part = L.scal + 64;
    L.gsum = L.part + 2 * (size_t)kPartStride * G * sizeof(double);
    L.gstride = (size_t)(pt + 31) / 32 * 32;  // doubles per parity
    L.bytes = L.gsum + 2 * L.gstride * sizeof(double);
    L.bytes = (L.bytes + 255) / 256 * 256;
    return L;
  }
};

struct RsPeer {                  // every rank, as this GPU sees it
  const double* part;            // [2][16 G] (local or peer-mapped)
  const double* gsum;            // [2][gstride]: X_q' w_q, internal column layout
  unsigned long long* inbox;     // the rank's flag array (peer-mapped for remote ranks)
  double* scal;                  // the rank's scalar exchange slot
  long long gstride, n, row0;    // doubles per gsum parity; shard rows; first global row
  int remote;
};

struct RsGroup {                 // a rank hosted by this grid
  DesignDev D;                   // the rank's shard, planned for Gr CTAs
  double* w;                     // n_r (+pad)
  double* zpart;                 // nslab_csr * n_r (multi column slab)
  double* dvg;                   // 2 * p_total (internal layout): published directions
  double* pieces;                // local CSC pieces (nseg)
  double* part;                  // exchange part [2][16 Gr]
  double* gsum;                  // exchange gsum [2][gstride]
  long long gstride;
  double* own;                   // own-slice state in global memory (Gr * 8 * chunk), or null
  int rank;
};

struct RsArgs {
  const RsGroup* groups;
  const double* omega[kRsMaxLocal];  // shard rows of each hosted rank (per call)
  int n_local, Gr, nranks, smem_doubles;
  const RsPeer* peers;
  unsigned long long* epoch;     // device counter: exchanges completed by earlier calls
  const double *diag, *minv, *scale, *b;  // reference layout, replicated
  double* x;                     // in x0 / out solution
  int max_iter;
  double rtol;
  double *trace, *alphas, *betas;
  int* result;
  // generate_rhs before the solve (sampler.py:94-107): b = X'(kappa + sqrt(omega) eta) + sqrt(d) delta
  int rhs;
  const double* kappa[kRsMaxLocal];
  unsigned long long seed, stream_id;
  double* b_out;                 // replicated b (reference layout), written by the lead group
  // Flag-exchange validation mode (pcgs_rs_set_exchange): every hosted group
  // is an independent rank -- group barriers instead of grid barriers, and the
  // cross-GPU flag protocol (release/acquire inbox epochs, volatile peer
  // loads) at every exchange.  One cooperative grid keeps all groups
  // co-resident, so the protocol runs on one GPU without ranks that wait on
  // separate launches.
  int flags;
  unsigned long long* gbar;      // per hosted group: monotonic arrival counter (one 128 B line each)
};

struct RsSumArgs {               // sum of a per-CTA partial over every rank's CTAs
  const double* part[kRsMaxLocal];
  int ncta, n_local, nranks, my_rank, flags;
  const RsPeer* peers;
  unsigned long long* epoch;
  double* out;
};

__device__ __forceinline__ double ld_peer(const double* p, bool remote) { return remote ? __ldcv(p) : __ldcg(p); }

// Watchdog of the cross-rank waits: a peer that never arrives (a rank that
// died or never launched) traps after kRsWaitNs instead of hanging the GPU;
// the host sees a launch failure.
constexpr unsigned long long kRsWaitNs = 30ull * 1000ull * 1000ull * 1000ull;
__device__ __forceinline__ unsigned long long rs_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void rs_wait_sys(const unsigned long long* flag, unsigned long long e) {
  const unsigned long long t0 = rs_now();
  unsigned long long v;
  for (;;) {
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory");
    if (v >= e) return;
    if (rs_now() - t0 > kRsWaitNs) {
      printf("pcgs row split: a peer rank did not arrive within %llu s (epoch %llu)\n", kRsWaitNs / 1000000000ull, e);
      __trap();
    }
  }
}

// Barrier over the CTAs of one rank: the grid barrier, or in the flag
// validation mode a barrier over the rank's own group of Gr CTAs (thread 0 of
// every CTA arrives on a monotonic counter with a release fence and spins
// with acquire loads until the group's arrivals reach the next multiple of
// Gr; counters persist across launches, every launch adding whole rounds).
__device__ __forceinline__ void group_barrier(unsigned long long* ctr, int n) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned long long old = atomicAdd(ctr, 1ull);
    const unsigned long long target = (old / (unsigned long long)n + 1ull) * (unsigned long long)n;
    unsigned long long v;
    do {
      asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

__device__ __forceinline__ void rank_sync(const RsArgs& A, int gi) {
  if (A.flags) group_barrier(A.gbar + 16 * gi, A.Gr);
  else cg::this_grid().sync();
}

// Exchange barrier: every local CTA has published its pieces and partials;
// then (ranks on other GPUs, or every group in the flag validation mode) one
// thread per peer signals the peer's inbox and waits for the peer's signal.
__device__ void rs_exchange(const RsArgs& A, int gi, int cta, int my_rank, unsigned long long e) {
  if (A.n_local == A.nranks && !A.flags) {
    cg::this_grid().sync();
    return;
  }
  __threadfence_system();
  rank_sync(A, gi);
  if (cta == 0 && threadIdx.x < A.nranks && (int)threadIdx.x != my_rank) {
    const RsPeer& q = A.peers[threadIdx.x];
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(q.inbox + my_rank), "l"(e) : "memory");
    const RsPeer& me = A.peers[my_rank];
    rs_wait_sys(me.inbox + threadIdx.x, e);
  }
  rank_sync(A, gi);
}

// Local column sums: g[j] = sum of this shard's CSC pieces of column j
// (slab-major, piece order), for the CTA's owned columns; the piece pointers
// of up to 8 slabs are loaded before the pieces, so a column costs two L2
// round trips per 8 slabs.
__device__ __forceinline__ void rs_assemble(const RsGroup& G, long long j0, int chunk, double* g) {
  const long long pt = G.D.pt;
  const int S = G.D.csc.nslab;
  for (int t = threadIdx.x; t < chunk; t += kThreads) {
    const long long j = j0 + t;
    if (j >= pt) break;
    double s = 0.0;
    for (int s0 = 0; s0 < S; s0 += 8) {
      int q0[8], q1[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int* pp = G.D.csc.piece_ptr + (long long)(s0 + u) * (pt + 1) + j;
        q0[u] = s0 + u < S ? __ldg(pp) : 0;
        q1[u] = s0 + u < S ? __ldg(pp + 1) : 0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        for (int q = q0[u]; q < q1[u]; ++q) s += __ldcg(G.pieces + q);
    }
    g[j] = s;
  }
}

// The same column sums through shared memory when the shard has <= 8 CSC
// slabs and the owned pieces fit the idle slab area: one round of coalesced
// piece loads into `stage`, then 4-lane groups per column (lane g takes slabs
// g, g+4), xor-tree totals.  Returns false (nothing written) otherwise.
__device__ __forceinline__ bool rs_assemble_flat(const RsGroup& G, long long j0, int chunk, double* g, double* stage,
                                                 int cap) {
  constexpr int K = 8, GS = 4;
  const long long pt = G.D.pt;
  const int S = G.D.csc.nslab;
  if (S > K) return false;
  const long long jend = min(j0 + chunk, pt);
  if (jend <= j0) return true;
  const int* ppb = G.D.csc.piece_ptr;
  int p0[K], off[K + 1];
  off[0] = 0;
#pragma unroll
  for (int s = 0; s < K; ++s) {
    p0[s] = s < S ? __ldg(ppb + (long long)s * (pt + 1) + j0) : 0;
    off[s + 1] = off[s] + (s < S ? __ldg(ppb + (long long)s * (pt + 1) + jend) - p0[s] : 0);
  }
  if (off[K] > cap) return false;
  for (int i = threadIdx.x; i < off[K]; i += kThreads) {
    int sl = 0;
#pragma unroll
    for (int u = 1; u < K; ++u) sl += i >= off[u] ? 1 : 0;
    int ps = p0[0], os = off[0];
#pragma unroll
    for (int u = 1; u < K; ++u)
      if (sl == u) {
        ps = p0[u];
        os = off[u];
      }
    stage[i] = __ldcg(G.pieces + ps + (i - os));
  }
  __syncthreads();
  const int gl = threadIdx.x & (GS - 1);
  for (int t0 = 0; t0 < chunk; t0 += kThreads / GS) {
    const int t = t0 + (int)threadIdx.x / GS;
    const long long j = j0 + t;
    double sum = 0.0;
    if (j < jend) {
      for (int sl = gl; sl < S; sl += GS) {
        int base = 0, pz = 0;
#pragma unroll
        for (int u = 0; u < K; ++u)
          if (sl == u) {
            base = off[u];
            pz = p0[u];
          }
        const int* pp = ppb + (long long)sl * (pt + 1);
        const int q0 = __ldg(pp + j) - pz, q1 = __ldg(pp + j + 1) - pz;
        for (int q = q0; q < q1; ++q) sum += stage[base + q];
      }
    }
#pragma unroll
    for (int m = 1; m < GS; m <<= 1) sum += __shfl_xor_sync(0xffffffffu, sum, m);
    if (gl == 0 && j < jend) g[j] = sum;
  }
  __syncthreads();  // the stage area is the next pass's slab
  return true;
}

// sum over ranks (rank order) of g_q[j], parity `par`
__device__ __forceinline__ double rs_gather(const RsArgs& A, long long j, int par) {
  double v[kRsMaxRanks > 8 ? 8 : kRsMaxRanks];
  double s = 0.0;
  for (int q0 = 0; q0 < A.nranks; q0 += 8) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int q = q0 + u;
      v[u] = 0.0;
      if (q < A.nranks) {
        const RsPeer& P = A.peers[q];
        v[u] = ld_peer(P.gsum + par * P.gstride + j, P.remote);
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) s += v[u];
  }
  return s;
}

__global__ void __launch_bounds__(kThreads, 1) k_pcg_rs(RsArgs A) {
  extern __shared__ __align__(128) double sv[];
  __shared__ double red[64];
  __shared__ double bc[4];
  __shared__ double st_rz;
  __shared__ int st_status, st_iter, st_fail, st_applies;
  __shared__ unsigned long long mbar, st_epoch;
  __shared__ RsGroup G;
  const int tid = threadIdx.x, lane = tid & 31;
  const int gi = blockIdx.x / A.Gr, cta = blockIdx.x % A.Gr;
  if (tid == 0) {
    G = A.groups[gi];
    st_epoch = *A.epoch;
  }
  const double* omega = A.omega[gi];
  BulkFill bf;
  bulk_init(bf, &mbar);  // ends with a CTA barrier
  const bool lead = gi == 0;  // the first hosted group writes the outputs
  const long long pt = G.D.pt;
  const int Gr = A.Gr;
  const int chunk = (int)((pt + Gr - 1) / Gr);
  const long long j0 = (long long)cta * chunk;
  const long long dvs = (pt + 15) / 16 * 16;
  double* ob = G.own ? G.own + (size_t)cta * 8 * chunk : sv + A.smem_doubles;
  double *ox = ob, *orr = ob + chunk, *od = ob + 2 * chunk, *om = ob + 3 * chunk, *os = ob + 4 * chunk,
         *oD = ob + 5 * chunk, *obv = ob + 6 * chunk, *oz = ob + 7 * chunk;
  for (int t = tid; t < chunk; t += kThreads) {
    const long long j = j0 + t;
    double xv = 0, m = 0, sc = 0, dg = 0, bv = 0;
    if (j < pt) {
      const long long rj = ref_index(j, G.D.p, G.D.icpt);
      xv = A.x[rj];
      m = __ldg(A.minv + rj);
      sc = __ldg(A.scale + rj);
      dg = __ldg(A.diag + rj);
      bv = __ldg(A.b + rj);
      G.dvg[dvs + j] = xv;  // the first application is on x0 (cg.py:137)
    }
    ox[t] = xv;
    orr[t] = 0.0;
    od[t] = xv;
    om[t] = m;
    os[t] = sc;
    oD[t] = dg;
    obv[t] = bv;
    oz[t] = 0.0;
  }
  if (tid == 0) {
    st_rz = 0.0;
    st_status = PCGS_MAX_ITER;
    st_iter = 0;
    st_fail = -1;
    st_applies = 0;
  }
  rank_sync(A, gi);

  // ---------------- R: the randomised right-hand side (one exchange) ----------------
  int e_off = 0;
  if (A.rhs) {
    {
      FillRhs f{A.kappa[gi], omega, nullptr, A.seed, kStreamEta ^ A.stream_id, 0, A.peers[G.rank].row0};
      EpiStore e{G.pieces, G.D.csc.nseg};
      run_pass(G.D.csc, sv, f, e, 0, cta);
    }
    rank_sync(A, gi);
    if (!rs_assemble_flat(G, j0, chunk, G.gsum + G.gstride, sv, A.smem_doubles))
      rs_assemble(G, j0, chunk, G.gsum + G.gstride);  // parity 1: iteration 0 writes parity 0
    if (A.nranks == 1) __syncthreads();
    else rs_exchange(A, gi, cta, G.rank, st_epoch + 1ull);
    for (int t = tid; t < chunk; t += kThreads) {
      const long long j = j0 + t;
      if (j >= pt) break;
      const long long rj = ref_index(j, G.D.p, G.D.icpt);
      Philox R(A.seed, kStreamDelta ^ A.stream_id, (unsigned)rj);
      const double bj = rs_gather(A, j, 1) + sqrt(oD[t]) * R.normal();
      obv[t] = bj;
      if (lead && A.b_out) A.b_out[rj] = bj;
    }
    e_off = 1;
    __syncthreads();
  }

  for (int a = 0;; ++a) {
    const int par = a & 1;
    // ---------------- convergence test of iteration a-1 (replicated) ----------------
    if (a > 0) {
      double s_rms, s_rz;
      reduce_partials2(G.part + (par ^ 1) * kPartStride * Gr + 1, Gr, bc, s_rms, s_rz);
      const double rms = sqrt(s_rms / (double)pt);
      if (lead && cta == 0 && tid == 0) A.trace[a - 1] = rms;
      const int k = a - 1;
      int stop = 0;
      if (rms <= A.rtol) stop = 1;
      else if (!isfinite(rms)) stop = 2;
      double beta = 0.0;
      if (!stop) {
        if (a >= 2) {
          beta = s_rz / st_rz;
          if (lead && cta == 0 && tid == 0) A.betas[a - 2] = beta;
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
      for (int t = tid; t < chunk; t += kThreads) {
        const double dn = a == 1 ? oz[t] : fma(beta, od[t], oz[t]);
        od[t] = dn;
        if (j0 + t < pt) G.dvg[par * dvs + j0 + t] = dn;
      }
      rank_sync(A, gi);
    }

    // ---------------- A: CSR pass over this rank's rows ----------------
    double acc = 0.0;
    {
      const double* vcur = G.dvg + (a == 0 ? dvs : par * dvs);
      if (tid == 0) bc[2] = G.D.icpt ? __ldcg(vcur + G.D.p) : 0.0;
      __syncthreads();
      const bool multi = G.D.csr.nslab > 1;
      EpiCsr e{multi ? G.zpart : G.w, omega, bc[2], 0.0, multi};
      FillBulk f{vcur, &bf};
      run_pass(G.D.csr, sv, f, e, 0, cta);
      acc = e.acc;
    }
    if (G.D.csr.nslab > 1) {
      rank_sync(A, gi);
      const long long n = G.D.n;
      const double v0 = bc[2];
      for (long long i = (long long)cta * kThreads + tid; i < n; i += (long long)Gr * kThreads) {
        double z = 0.0;
        for (int s = 0; s < G.D.csr.nslab; ++s) z += __ldcg(G.zpart + (long long)s * n + i);
        z += v0;
        const double wi = __ldg(omega + i) * z;
        G.w[i] = wi;
        acc += wi * z;
      }
    }
    {
      double dterm = 0.0;
      for (int t = tid; t < chunk; t += kThreads) dterm += oD[t] * od[t] * od[t];
      block_sum2(acc, dterm, red);
      if (tid == 0) {
        G.part[par * kPartStride * Gr + cta * kPartStride + 0] = acc;    // exchanged
        G.part[par * kPartStride * Gr + cta * kPartStride + 3] = dterm;  // local
      }
    }
    rank_sync(A, gi);

    // ---------------- B: CSC pass, local column sums g_r = X_r' w_r ----------------
    {
      FillVecN f{G.w, &bf};
      EpiStore e{G.pieces, G.D.csc.nseg};
      run_pass(G.D.csc, sv, f, e, 0, cta);
    }
    rank_sync(A, gi);
    const bool solo = A.nranks == 1;  // one rank: each CTA reads only its own columns' sums
    if (!solo && cta == 0 && tid < 32) {  // this rank's z'Omega z total (slot 4 of line 0), exchanged
      const double t = warp_sum(lane_partials(G.part + par * kPartStride * Gr, Gr, lane));
      if (tid == 0) G.part[par * kPartStride * Gr + 4] = t;
    }
    if (!rs_assemble_flat(G, j0, chunk, G.gsum + par * G.gstride, sv, A.smem_doubles))
      rs_assemble(G, j0, chunk, G.gsum + par * G.gstride);
    if (tid == 0) ++st_applies;
    if (solo) __syncthreads();
    else rs_exchange(A, gi, cta, G.rank, st_epoch + (unsigned long long)(e_off + a) + 1ull);

    // ---------------- C: assemble owned columns over all ranks, step ----------------
    double alpha = 0.0;
    if (a > 0) {
      // dAd: the ranks' z'Omega z totals in rank order, then the replicated prior term
      if (tid < 32 && solo) {
        const double s = warp_sum(lane_partials(G.part + par * kPartStride * Gr, Gr, lane)) +
                         warp_sum(lane_partials(G.part + par * kPartStride * Gr + 3, Gr, lane));
        if (tid == 0) bc[0] = s;
      } else if (tid < 32) {
        double v = 0.0;
        for (int q = lane; q < A.nranks; q += 32) {
          const RsPeer& P = A.peers[q];
          v = ld_peer(P.part + par * kPartStride * Gr + 4, P.remote);
        }
        // rank order: lane q holds rank q (nranks <= 64: two rounds at most)
        double s = 0.0;
        for (int q = 0; q < A.nranks && q < 32; ++q) s += __shfl_sync(0xffffffffu, v, q);
        if (A.nranks > 32) {
          double v2 = 0.0;
          if (lane + 32 < A.nranks) {
            const RsPeer& P = A.peers[lane + 32];
            v2 = ld_peer(P.part + par * kPartStride * Gr + 4, P.remote);
          }
          for (int q = 32; q < A.nranks; ++q) s += __shfl_sync(0xffffffffu, v2, q - 32);
        }
        s += warp_sum(lane_partials(G.part + par * kPartStride * Gr + 3, Gr, lane));
        if (tid == 0) bc[0] = s;
      }
      __syncthreads();
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
      if (lead && cta == 0 && tid == 0) A.alphas[a - 1] = alpha;
    }
    double t_rms = 0.0, t_rz = 0.0;
    for (int t = tid; t < chunk; t += kThreads) {
      const long long j = j0 + t;
      if (j >= pt) break;
      const double Ad = rs_gather(A, j, par) + oD[t] * od[t];
      double rv;
      if (a == 0) {
        rv = obv[t] - Ad;
      } else {
        ox[t] = fma(alpha, od[t], ox[t]);
        rv = fma(-alpha, Ad, orr[t]);
      }
      orr[t] = rv;
      const double zn = om[t] * rv;
      oz[t] = zn;
      const double tj = os[t] * rv;
      t_rms += tj * tj;
      t_rz += rv * zn;
    }
    block_sum2(t_rms, t_rz, red);
    if (tid == 0) {
      G.part[par * kPartStride * Gr + cta * kPartStride + 1] = t_rms;
      G.part[par * kPartStride * Gr + cta * kPartStride + 2] = t_rz;
    }
    rank_sync(A, gi);
  }

  __syncthreads();
  if (lead) {
    for (int t = tid; t < chunk; t += kThreads)
      if (j0 + t < pt) A.x[ref_index(j0 + t, G.D.p, G.D.icpt)] = ox[t];
  }
  if (lead && cta == 0 && tid == 0) {
    A.result[0] = st_iter;
    A.result[1] = st_status;
    A.result[2] = st_fail;
    A.result[3] = st_applies;
  }
  // exchanges used by this call: every rank ran the same number of iterations
  cg::this_grid().sync();
  if (blockIdx.x == 0 && tid == 0) *A.epoch = st_epoch + (unsigned long long)(e_off + st_applies);
}

// Sum over ranks (rank order) of per-CTA partials (line slot 0): one warp.
// Ranks on other GPUs publish their local sums in their scalar slots and meet
// at a flag exchange (one epoch).
__global__ void __launch_bounds__(32) k_rs_sum(RsSumArgs A) {
  const int lane = threadIdx.x;
  if (A.flags) {  // validation mode: block r acts as rank r (cooperative launch, one block per rank)
    const int r = blockIdx.x;
    const unsigned long long e = *A.epoch + 1ull;  // read before this rank signals anyone
    double x = 0.0;
    for (int c = lane; c < A.ncta; c += 32) x += __ldcg(A.part[r] + (long long)c * kPartStride);
    const double v = warp_sum(x);
    const RsPeer& me = A.peers[r];
    if (lane == 0) *me.scal = v;
    __threadfence_system();
    __syncwarp();
    for (int q = lane; q < A.nranks; q += 32) {
      if (q == r) continue;
      asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(A.peers[q].inbox + r), "l"(e) : "memory");
      rs_wait_sys(me.inbox + q, e);
    }
    __syncwarp();
    if (lane == 0 && r == 0) {  // every peer has signalled, so every block has read the epoch
      double t = 0.0;
      for (int q = 0; q < A.nranks; ++q) t += q == r ? v : ld_peer(A.peers[q].scal, true);
      *A.out = t;
      *A.epoch = e;
    }
    return;
  }
  double v[kRsMaxLocal];
  for (int l = 0; l < A.n_local; ++l) {
    double x = 0.0;
    for (int c = lane; c < A.ncta; c += 32) x += __ldcg(A.part[l] + (long long)c * kPartStride);
    v[l] = warp_sum(x);
  }
  if (A.n_local == A.nranks) {
    if (lane == 0) {
      double t = 0.0;
      for (int l = 0; l < A.n_local; ++l) t += v[l];
      *A.out = t;
    }
    return;
  }
  const unsigned long long e = *A.epoch + 1ull;
  const RsPeer& me = A.peers[A.my_rank];
  if (lane == 0) *me.scal = v[0];
  __threadfence_system();
  __syncwarp();
  for (int q = lane; q < A.nranks; q += 32) {
    if (q == A.my_rank) continue;
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(A.peers[q].inbox + A.my_rank), "l"(e) : "memory");
    rs_wait_sys(me.inbox + q, e);
  }
  __syncwarp();
  if (lane == 0) {
    double t = 0.0;
    for (int q = 0; q < A.nranks; ++q) t += q == A.my_rank ? v[0] : ld_peer(A.peers[q].scal, true);
    *A.out = t;
    *A.epoch = e;
  }
}

}  // namespace

// =====================================================================
// context
// =====================================================================
struct pcgs_rs {
  int device = 0, n_local = 0, rank0 = 0, nranks = 0, Gr = 0, smem_doubles = 0;
  long long pt = 0, p = 0;
  std::vector<pcgs_design_t> designs;      // local ranks
  std::vector<void*> exch;                 // per rank: exchange base (local alloc or IPC-mapped)
  std::vector<int> opened;                 // per rank: 1 when IPC-mapped (to close)
  std::vector<void*> allocs;               // owned device allocations
  std::vector<RsPeer> peers;
  std::vector<RsHeader> hdr;
  unsigned long long* epoch = nullptr;
  std::vector<double*> w, zpart, dvg, own;
  RsGroup* groups_dev = nullptr;
  RsPeer* peers_dev = nullptr;
  std::vector<double*> pieces;
  bool ready = false;
  bool own_in_smem = true;
  int flags = 0;                           // flag-exchange validation mode (one grid)
  unsigned long long* gbar = nullptr;      // group barrier counters (flag mode)
};

namespace {

int rs_alloc(pcgs_rs* R, size_t bytes, void** out) {
  void* p = nullptr;
  CUDA_TRY(cudaMalloc(&p, bytes));
  R->allocs.push_back(p);
  *out = p;
  return PCGS_OK;
}

size_t rs_smem_bytes(const pcgs_rs* R) {
  const long long chunk = (R->pt + R->Gr - 1) / R->Gr;
  return (size_t)R->smem_doubles * 8 + (R->own_in_smem ? (size_t)chunk * 64 : 0) + 16;
}

}  // namespace

extern "C" {

int pcgs_rs_create(const pcgs_design_t* designs, int n_local, int rank0, int nranks, pcgs_rs_t* out) {
  if (!designs || !out || n_local < 1 || n_local > kRsMaxLocal || nranks < n_local || (n_local > 1 && n_local != nranks) || nranks > kRsMaxRanks || rank0 < 0 ||
      rank0 + n_local > nranks)
    return fail(PCGS_EINVAL, "row split: bad rank layout");
  *out = nullptr;
  pcgs_rs* R = new pcgs_rs();
  R->n_local = n_local;
  R->rank0 = rank0;
  R->nranks = nranks;
  R->device = designs[0]->device;
  R->Gr = designs[0]->dev.G;
  R->pt = designs[0]->dev.pt;
  R->p = designs[0]->dev.p;
  auto bail = [&](int rc) {
    pcgs_rs_destroy(R);
    return rc;
  };
  for (int l = 0; l < n_local; ++l) {
    const DesignDev& D = designs[l]->dev;
    if (designs[l]->device != R->device || D.G != R->Gr || D.pt != R->pt || D.p != R->p || D.icpt != designs[0]->dev.icpt)
      return bail(fail(PCGS_EINVAL, "row split: local shards must share device, grid and columns"));
    R->smem_doubles = std::max(R->smem_doubles, D.smem_doubles);
    R->designs.push_back(designs[l]);
  }
  if ((long long)R->Gr * n_local > kMaxGridRs) return bail(fail(PCGS_EINVAL, "row split: grid too large"));
  if (cudaSetDevice(R->device) != cudaSuccess) return bail(fail(PCGS_ECUDA, "cudaSetDevice failed"));
  const long long chunk = (R->pt + R->Gr - 1) / R->Gr;
  R->own_in_smem = (long long)R->smem_doubles * 8 + chunk * 64 + 16 + 1024 + 2048 <= 227 * 1024;
  R->exch.assign(nranks, nullptr);
  R->opened.assign(nranks, 0);
  R->hdr.assign(nranks, RsHeader{});
  R->peers.assign(nranks, RsPeer{});
  int rc;
  void* p;
  if ((rc = rs_alloc(R, sizeof(unsigned long long), &p))) return bail(rc);
  R->epoch = (unsigned long long*)p;
  if (cudaMemset(R->epoch, 0, sizeof(unsigned long long)) != cudaSuccess) return bail(fail(PCGS_ECUDA, "memset"));
  for (int l = 0; l < n_local; ++l) {
    const DesignDev& D = designs[l]->dev;
    const RsLayout L = RsLayout::of(D.pt, D.G);
    if ((rc = rs_alloc(R, L.bytes, &p))) return bail(rc);
    if (cudaMemset(p, 0, L.bytes) != cudaSuccess) return bail(fail(PCGS_ECUDA, "memset"));
    RsHeader h{D.pt, D.G, (long long)L.bytes, D.n, {0, 0, 0, 0}};
    if (cudaMemcpy(p, &h, sizeof(h), cudaMemcpyHostToDevice) != cudaSuccess)
      return bail(fail(PCGS_ECUDA, "exchange setup copy failed"));
    R->exch[rank0 + l] = p;
    R->hdr[rank0 + l] = h;
    if ((rc = rs_alloc(R, (size_t)std::max<long long>(D.csc.nseg, 1) * 8, &p))) return bail(rc);
    R->pieces.push_back((double*)p);
    const long long n = D.n;
    double* b;
    if ((rc = rs_alloc(R, (size_t)(n + 2) * 8, &p))) return bail(rc);
    R->w.push_back((double*)p);
    b = nullptr;
    if (D.csr.nslab > 1) {
      if ((rc = rs_alloc(R, (size_t)D.csr.nslab * n * 8, &p))) return bail(rc);
      b = (double*)p;
    }
    R->zpart.push_back(b);
    if ((rc = rs_alloc(R, (size_t)(2 * ((D.pt + 15) / 16 * 16) + 16) * 8, &p))) return bail(rc);
    R->dvg.push_back((double*)p);
    b = nullptr;
    if (!R->own_in_smem) {
      if ((rc = rs_alloc(R, (size_t)R->Gr * 8 * chunk * 8, &p))) return bail(rc);
      b = (double*)p;
    }
    R->own.push_back(b);
  }
  if ((rc = rs_alloc(R, sizeof(unsigned long long) * 16 * n_local, &p))) return bail(rc);
  R->gbar = (unsigned long long*)p;
  if (cudaMemset(R->gbar, 0, sizeof(unsigned long long) * 16 * n_local) != cudaSuccess)
    return bail(fail(PCGS_ECUDA, "memset"));
  if ((rc = rs_alloc(R, sizeof(RsGroup) * n_local, &p))) return bail(rc);
  R->groups_dev = (RsGroup*)p;
  if ((rc = rs_alloc(R, sizeof(RsPeer) * nranks, &p))) return bail(rc);
  R->peers_dev = (RsPeer*)p;
  if ((rc = raise_smem_limit(k_pcg_rs))) return bail(rc);
  *out = R;
  return PCGS_OK;
}

int pcgs_rs_exchange_handle(pcgs_rs_t R, int local, void* handle_h) {
  if (!R || !handle_h || local < 0 || local >= R->n_local) return fail(PCGS_EINVAL, "bad argument");
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaSetDevice(R->device));
  CUDA_TRY(cudaIpcGetMemHandle(&h, R->exch[R->rank0 + local]));
  memcpy(handle_h, &h, sizeof(h));
  return PCGS_OK;
}

int pcgs_rs_open_peer(pcgs_rs_t R, int rank, const void* handle_h) {
  if (!R || !handle_h || rank < 0 || rank >= R->nranks || (rank >= R->rank0 && rank < R->rank0 + R->n_local))
    return fail(PCGS_EINVAL, "row split: peer rank out of range or local");
  CUDA_TRY(cudaSetDevice(R->device));
  cudaIpcMemHandle_t h;
  memcpy(&h, handle_h, sizeof(h));
  void* p = nullptr;
  CUDA_TRY(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  R->exch[rank] = p;
  R->opened[rank] = 1;
  RsHeader hd;
  CUDA_TRY(cudaMemcpy(&hd, p, sizeof(hd), cudaMemcpyDeviceToHost));
  if (hd.pt != R->pt || hd.G != R->Gr) return fail(PCGS_EINVAL, "row split: peer shard has other columns or grid");
  R->hdr[rank] = hd;
  return PCGS_OK;
}

// Builds the peer table once every rank's exchange region is known: local
// piece_ptr copies of remote ranks, the (rank, slab) summation order.
static int rs_finalize(pcgs_rs* R) {
  for (int q = 0; q < R->nranks; ++q) {
    if (!R->exch[q]) return fail(PCGS_EINVAL, "row split: rank " + std::to_string(q) + " has no exchange region");
    const RsHeader& h = R->hdr[q];
    const RsLayout L = RsLayout::of(h.pt, h.G);
    RsPeer P{};
    char* base = (char*)R->exch[q];
    P.part = (const double*)(base + L.part);
    P.gsum = (const double*)(base + L.gsum);
    P.inbox = (unsigned long long*)(base + L.flags);
    P.scal = (double*)(base + L.scal);
    P.gstride = (long long)L.gstride;
    P.n = h.n;
    P.row0 = q == 0 ? 0 : R->peers[q - 1].row0 + R->peers[q - 1].n;
    P.remote = R->opened[q] || R->flags;
    R->peers[q] = P;
  }
  CUDA_TRY(cudaMemcpy(R->peers_dev, R->peers.data(), sizeof(RsPeer) * R->nranks, cudaMemcpyHostToDevice));
  std::vector<RsGroup> groups(R->n_local);
  for (int l = 0; l < R->n_local; ++l) {
    const int q = R->rank0 + l;
    RsGroup& g = groups[l];
    g.D = R->designs[l]->dev;
    g.D.dbg = 0;
    g.w = R->w[l];
    g.zpart = R->zpart[l];
    g.dvg = R->dvg[l];
    g.part = const_cast<double*>(R->peers[q].part);
    g.gsum = const_cast<double*>(R->peers[q].gsum);
    g.gstride = R->peers[q].gstride;
    g.pieces = R->pieces[l];
    g.own = R->own[l];
    g.rank = q;
  }
  CUDA_TRY(cudaMemcpy(R->groups_dev, groups.data(), sizeof(RsGroup) * R->n_local, cudaMemcpyHostToDevice));
  R->ready = true;
  return PCGS_OK;
}

int pcgs_rs_pcg(pcgs_rs_t R, const double* const* omegas_h, const double* prior_diag, const double* minv,
                const double* scale, const double* b, double* x, int32_t max_iter, double rtol, double* trace,
                double* alphas, double* betas, int32_t* result, pcgs_stream_t stream) {
  if (!R || !omegas_h || !b) return fail(PCGS_EINVAL, "null argument");
  RsSolve S{omegas_h, nullptr, 0, 0, nullptr, prior_diag, minv, scale, b, x, max_iter, rtol, trace, alphas, betas,
            result};
  return rs_solve(R, S, (cudaStream_t)stream);
}

int pcgs_rs_set_exchange(pcgs_rs_t R, int mode) {
  if (!R || (mode != 0 && mode != 1)) return fail(PCGS_EINVAL, "bad argument");
  if (R->ready) return fail(PCGS_EINVAL, "row split: set the exchange mode before the first solve");
  if (mode == 1 && R->n_local != R->nranks)
    return fail(PCGS_EINVAL, "row split: the flag validation mode hosts every rank in one grid");
  R->flags = mode;
  return PCGS_OK;
}

int pcgs_rs_destroy(pcgs_rs_t R) {
  if (!R) return PCGS_OK;
  cudaSetDevice(R->device);
  cudaDeviceSynchronize();
  for (int q = 0; q < R->nranks; ++q)
    if (R->opened[q] && R->exch[q]) cudaIpcCloseMemHandle(R->exch[q]);
  for (void* p : R->allocs) cudaFree(p);
  delete R;
  return PCGS_OK;
}

}  // extern "C"

int rs_solve(pcgs_rs_t R, const RsSolve& S, cudaStream_t s) {
  if (!R || !S.omegas || !S.diag || !S.minv || !S.scale || (!S.b && !S.kappas) || !S.x || !S.trace || !S.alphas ||
      !S.betas || !S.result)
    return fail(PCGS_EINVAL, "null argument");
  if (S.max_iter < 1) return fail(PCGS_EINVAL, "max_iter must be at least 1");
  CUDA_TRY(cudaSetDevice(R->device));
  int rc;
  if (!R->ready && (rc = rs_finalize(R))) return rc;
  RsArgs A{};
  A.groups = R->groups_dev;
  for (int l = 0; l < R->n_local; ++l) {
    A.omega[l] = S.omegas[l];
    A.kappa[l] = S.kappas ? S.kappas[l] : nullptr;
  }
  A.n_local = R->n_local;
  A.Gr = R->Gr;
  A.nranks = R->nranks;
  A.smem_doubles = R->smem_doubles;
  A.peers = R->peers_dev;
  A.epoch = R->epoch;
  A.diag = S.diag;
  A.minv = S.minv;
  A.scale = S.scale;
  A.b = S.kappas ? S.diag : S.b;  // unread when the RHS is generated
  A.x = S.x;
  A.max_iter = S.max_iter;
  A.rtol = S.rtol;
  A.trace = S.trace;
  A.alphas = S.alphas;
  A.betas = S.betas;
  A.result = S.result;
  A.rhs = S.kappas ? 1 : 0;
  A.seed = S.seed;
  A.stream_id = S.stream_id;
  A.b_out = S.b_out;
  A.flags = R->flags;
  A.gbar = R->gbar;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(R->Gr * R->n_local);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = rs_smem_bytes(R);
  cfg.stream = s;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeCooperative;
  attr.val.cooperative = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  CUDA_TRY(cudaLaunchKernelEx(&cfg, k_pcg_rs, A));
  return PCGS_OK;
}

int rs_sum(pcgs_rs_t R, const double* const* parts, double* out, cudaStream_t s) {
  int rc;
  if (!R->ready && (rc = rs_finalize(R))) return rc;
  RsSumArgs A{};
  for (int l = 0; l < R->n_local; ++l) A.part[l] = parts[l];
  A.ncta = R->Gr;
  A.n_local = R->n_local;
  A.nranks = R->nranks;
  A.my_rank = R->rank0;
  A.peers = R->peers_dev;
  A.epoch = R->epoch;
  A.out = out;
  A.flags = R->flags;
  if (R->flags) {  // one block per emulated rank, co-resident (they wait on one another)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(R->nranks);
    cfg.blockDim = dim3(32);
    cfg.stream = s;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeCooperative;
    attr.val.cooperative = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    CUDA_TRY(cudaLaunchKernelEx(&cfg, k_rs_sum, A));
    return PCGS_OK;
  }
  k_rs_sum<<<1, 32, 0, s>>>(A);
  CUDA_TRY(cudaGetLastError());
  return PCGS_OK;
}

int rs_local(pcgs_rs_t R, int l, pcgs_design_t* d, int64_t* row0) {
  if (!R || l < 0 || l >= R->n_local) return fail(PCGS_EINVAL, "bad local rank");
  int rc;
  if (!R->ready && (rc = rs_finalize(R))) return rc;
  *d = R->designs[l];
  *row0 = R->peers[R->rank0 + l].row0;
  return PCGS_OK;
}

int rs_n_local(pcgs_rs_t R) { return R->n_local; }
int rs_grid(pcgs_rs_t R) { return R->Gr; }
