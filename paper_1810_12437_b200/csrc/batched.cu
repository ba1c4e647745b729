// Batched independent chains (BASELINE config 4; SURVEY §8e "chain batching"):
// R chains share every walk over the pattern-only index stream.  All vectors
// are chain-minor: element (j, c) at [j * R + c].  The design handle passed
// here must have been created with slab_max <= pcgs_batch_slab_max(R) so that
// R slab vectors fit one CTA's shared memory.
#include <cuda_runtime.h>

#include <cmath>
#include <string>

#include "batched.cuh"
#include "internal.cuh"

namespace cg = cooperative_groups;

namespace {

template <int R>
struct EpiCsrB {  // multi column slab: partial store; else w = omega (v0 + s)
  double* out;
  const double* omega;
  const double* v0;  // R intercept values (shared memory)
  double* acc;       // R per-thread partials of w z (dAd), may be null
  bool multi;
  __device__ void emit(long long seg, const double (&s)[R]) {
#pragma unroll
    for (int c = 0; c < R; ++c) {
      if (multi) {
        out[seg * R + c] = s[c];
      } else {
        const double z = v0[c] + s[c];
        const double w = __ldg(omega + seg * R + c) * z;
        out[seg * R + c] = w;
        if (acc) acc[c] += w * z;
      }
    }
  }
};

template <int R>
struct EpiStoreB {
  double* out;
  __device__ void emit(long long seg, const double (&s)[R]) {
#pragma unroll
    for (int c = 0; c < R; ++c) out[seg * R + c] = s[c];
  }
};

template <int R>
__global__ void __launch_bounds__(kThreads, 1) k_csr_b(DesignDev D, const double* v, const double* omega,
                                                       double* out) {
  extern __shared__ __align__(128) double sv[];
  __shared__ unsigned long long mbar;
  __shared__ double v0[R];
  BulkFill bf;
  bulk_init(bf, &mbar);
  if (threadIdx.x < R) v0[threadIdx.x] = D.icpt ? v[threadIdx.x] : 0.0;
  __syncthreads();
  FillBulkB<R> f{v + (long long)D.icpt * R, &bf};
  EpiCsrB<R> e{out, omega, v0, nullptr, D.csr.nslab > 1};
  run_pass_b<R>(D.csr, sv, f, e);
}

template <int R>
__global__ void k_rows_combine_b(DesignDev D, const double* zpart, const double* v, const double* omega,
                                 double* w) {
  const long long nr = D.n * R;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nr; e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / R;
    const int c = (int)(e - i * R);
    double z = 0.0;
    for (int s = 0; s < D.csr.nslab; ++s) z += zpart[((long long)s * D.n + i) * R + c];
    z += D.icpt ? v[c] : 0.0;
    w[e] = omega ? __ldg(omega + e) * z : z;
  }
}

template <int R>
__global__ void __launch_bounds__(kThreads, 1) k_csc_b(DesignDev D, const double* w, double* pieces) {
  extern __shared__ __align__(128) double sv[];
  __shared__ unsigned long long mbar;
  BulkFill bf;
  bulk_init(bf, &mbar);
  FillBulkB<R> f{w, &bf};
  EpiStoreB<R> e{pieces};
  run_pass_b<R>(D.csc, sv, f, e);
}

// out[(ref j) R + c] = sum of pieces + diag * v
template <int R>
__global__ void k_assemble_b(DesignDev D, const double* pieces, const double* diag, const double* v, double* out) {
  const long long nr = D.pt * R;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nr; e += (long long)gridDim.x * blockDim.x) {
    const long long j = e / R;
    const int c = (int)(e - j * R);
    double s = 0.0;
    for (int sl = 0; sl < D.csc.nslab; ++sl) {
      const int* pp = D.csc.piece_ptr + (long long)sl * (D.pt + 1);
      for (int q = pp[j]; q < pp[j + 1]; ++q) s += pieces[(long long)q * R + c];
    }
    const long long r = ref_index(j, D.p, D.icpt) * R + c;
    out[r] = diag ? s + diag[r] * v[r] : s;
  }
}

// ---------------------------------------------------------------------------
// batched persistent PCG: the reference loop (cg.py:105-192) per chain, chains
// that finish are masked (zero direction) until every chain is done
// ---------------------------------------------------------------------------
struct PcgArgsB {
  DesignDev D;
  const double *omega, *diag, *minv, *scale, *b;  // chain-minor, reference layout
  double* x;
  int max_iter;
  double rtol;
  double *trace, *alphas, *betas;  // [c][max_iter+1], [c][max_iter]
  int* result;                     // [c][4]
  double *w, *zpart, *pieces, *dvg, *part;
};

template <int R>
__host__ __device__ constexpr int part_stride_b() {
  return 16 * ((3 * R + 15) / 16);
}

template <int R>
size_t pcg_b_smem(const DesignDev& D) {
  const long long chunk = (D.pt + D.G - 1) / D.G;
  return (size_t)D.smem_doubles * R * 8 + (size_t)chunk * R * 8 * 8 + (size_t)D.csc.nslab * (chunk + 1) * 4 + 64;
}

template <int R>
__global__ void __launch_bounds__(kThreads, 1) k_pcg_b(PcgArgsB A) {
  extern __shared__ __align__(128) double sv[];
  __shared__ double red[64];
  __shared__ double sred[3 * R];
  __shared__ double st_rz[R], st_beta[R], st_alpha[R], v0s[R];
  __shared__ int st_active[R], st_status[R], st_iter[R], st_fail[R];
  __shared__ int st_applies, st_any;
  __shared__ unsigned long long mbar;
  BulkFill bf;
  bulk_init(bf, &mbar);
  const int tid = threadIdx.x;
  const int PS = part_stride_b<R>();
  const long long pt = A.D.pt;
  const int chunk = (int)((pt + gridDim.x - 1) / gridDim.x);
  const long long j0 = (long long)blockIdx.x * chunk;
  const long long dvs = ((pt * R) + 15) / 16 * 16;
  const int S = A.D.csc.nslab;
  double* base = sv + (long long)A.D.smem_doubles * R;
  double *ox = base, *orr = base + chunk * R, *od = base + 2 * chunk * R, *om = base + 3 * chunk * R;
  double *os = base + 4 * chunk * R, *oD = base + 5 * chunk * R, *ob = base + 6 * chunk * R;
  double* oz = base + 7 * chunk * R;
  int* pp = (int*)(base + 8 * chunk * R);

  for (int e = tid; e < chunk * R; e += kThreads) {
    const int t = e / R, c = e - t * R;
    const long long j = j0 + t;
    double xv = 0, m = 0, sc = 0, dg = 0, bv = 0;
    if (j < pt) {
      const long long r = ref_index(j, A.D.p, A.D.icpt) * R + c;
      xv = A.x[r];
      m = __ldg(A.minv + r);
      sc = __ldg(A.scale + r);
      dg = __ldg(A.diag + r);
      bv = __ldg(A.b + r);
      A.dvg[dvs + j * R + c] = xv;
    }
    ox[e] = xv;
    orr[e] = 0.0;
    od[e] = xv;
    om[e] = m;
    os[e] = sc;
    oD[e] = dg;
    ob[e] = bv;
    oz[e] = 0.0;
  }
  for (int t = tid; t < S * (chunk + 1); t += kThreads) {
    const int s = t / (chunk + 1), q = t % (chunk + 1);
    pp[t] = A.D.csc.piece_ptr[(long long)s * (pt + 1) + min(j0 + q, pt)];
  }
  if (tid < R) {
    st_rz[tid] = 0.0;
    st_beta[tid] = 0.0;
    st_active[tid] = 1;
    st_status[tid] = PCGS_MAX_ITER;
    st_iter[tid] = 0;
    st_fail[tid] = -1;
  }
  if (tid == 0) st_applies = 0;
  cg::this_grid().sync();

  for (int a = 0;; ++a) {
    // ---------------- per-chain convergence test of iteration a-1 ----------------
    if (a > 0) {
      __syncthreads();
      if (tid < 32) {  // reduce rms / rz partials of every chain (fixed order)
        double s[2 * R];
#pragma unroll
        for (int k = 0; k < 2 * R; ++k) s[k] = 0.0;
        for (int q = tid; q < (int)gridDim.x; q += 32) {
#pragma unroll
          for (int k = 0; k < 2 * R; ++k) s[k] += __ldcg(A.part + (long long)q * PS + R + k);
        }
#pragma unroll
        for (int k = 0; k < 2 * R; ++k) {
          const double v = warp_sum(s[k]);
          if (tid == 0) sred[R + k] = v;
        }
      }
      __syncthreads();
      if (tid < R) {
        const int c = tid;
        if (st_active[c]) {
          const double rms = sqrt(sred[R + c] / (double)pt), rzn = sred[2 * R + c];
          const int k = a - 1;
          if (blockIdx.x == 0) A.trace[(long long)c * (A.max_iter + 1) + k] = rms;
          double beta = 0.0;
          if (rms <= A.rtol) {
            st_active[c] = 0;
            st_status[c] = PCGS_CONVERGED;
            st_iter[c] = k;
          } else if (!isfinite(rms)) {
            st_active[c] = 0;
            st_status[c] = PCGS_NONFINITE;
            st_iter[c] = k;
            st_fail[c] = k;
          } else {
            if (a >= 2) {
              beta = rzn / st_rz[c];
              if (blockIdx.x == 0) A.betas[(long long)c * A.max_iter + a - 2] = beta;
            }
            st_rz[c] = rzn;
            if (k >= A.max_iter) {
              st_active[c] = 0;
              st_status[c] = PCGS_MAX_ITER;
              st_iter[c] = k;
            }
          }
          st_beta[c] = beta;
        } else {
          st_beta[c] = 0.0;
        }
      }
      __syncthreads();
      if (tid == 0) {
        int any = 0;
        for (int c = 0; c < R; ++c) any |= st_active[c];
        st_any = any;
      }
      __syncthreads();
      if (!st_any) break;
      for (int e = tid; e < chunk * R; e += kThreads) {
        const int t = e / R, c = e - t * R;
        const double dn = st_active[c] ? (a == 1 ? oz[e] : fma(st_beta[c], od[e], oz[e])) : 0.0;
        od[e] = dn;
        if (j0 + t < pt) A.dvg[(long long)(a & 1) * dvs + (j0 + t) * R + c] = dn;
      }
      cg::this_grid().sync();
    }

    // ---------------- phase A: CSR pass, w = omega (X v) per chain ----------------
    double accd[R];
#pragma unroll
    for (int c = 0; c < R; ++c) accd[c] = 0.0;
    for (int e = tid; e < chunk * R; e += kThreads) {
      const int c = e % R;
#pragma unroll
      for (int k = 0; k < R; ++k)
        if (k == c) accd[k] += oD[e] * od[e] * od[e];
    }
    const double* vcur = A.dvg + (a == 0 ? dvs : (long long)(a & 1) * dvs);
    if (tid < R) v0s[tid] = A.D.icpt ? __ldcg(vcur + A.D.p * R + tid) : 0.0;
    __syncthreads();
    const bool multi = A.D.csr.nslab > 1;
    {
      EpiCsrB<R> e{multi ? A.zpart : A.w, A.omega, v0s, accd, multi};
      FillBulkB<R> f{vcur, &bf};
      run_pass_b<R>(A.D.csr, sv, f, e);
    }
    if (multi) {
      cg::this_grid().sync();
      const long long nr = A.D.n * R;
      for (long long e = (long long)blockIdx.x * kThreads + tid; e < nr; e += (long long)gridDim.x * kThreads) {
        const long long i = e / R;
        const int c = (int)(e - i * R);
        double z = 0.0;
        for (int s = 0; s < A.D.csr.nslab; ++s) z += __ldcg(A.zpart + ((long long)s * A.D.n + i) * R + c);
        z += v0s[c];
        const double wi = __ldg(A.omega + e) * z;
        A.w[e] = wi;
#pragma unroll
        for (int k = 0; k < R; ++k)
          if (k == c) accd[k] += wi * z;
      }
    }
#pragma unroll
    for (int c = 0; c < R; ++c) {
      const double t = block_sum(accd[c], red);
      if (tid == 0) A.part[(long long)blockIdx.x * PS + c] = t;
    }
    cg::this_grid().sync();

    // ---------------- phase B: CSC pass, pieces of X' w ----------------
    {
      FillBulkB<R> f{A.w, &bf};
      EpiStoreB<R> e{A.pieces};
      run_pass_b<R>(A.D.csc, sv, f, e);
    }
    cg::this_grid().sync();
    if (tid == 0) ++st_applies;

    // ---------------- phase C: per-chain step ----------------
    if (a > 0) {
      __syncthreads();
      if (tid < 32) {
        double s[R];
#pragma unroll
        for (int k = 0; k < R; ++k) s[k] = 0.0;
        for (int q = tid; q < (int)gridDim.x; q += 32) {
#pragma unroll
          for (int k = 0; k < R; ++k) s[k] += __ldcg(A.part + (long long)q * PS + k);
        }
#pragma unroll
        for (int k = 0; k < R; ++k) {
          const double v = warp_sum(s[k]);
          if (tid == 0) sred[k] = v;
        }
      }
      __syncthreads();
      if (tid < R) {
        const int c = tid;
        st_alpha[c] = 0.0;
        if (st_active[c]) {
          const double dAd = sred[c];
          if (!(dAd > 0.0)) {
            st_active[c] = 0;
            st_status[c] = PCGS_NOT_PD;
            st_iter[c] = a;
            st_fail[c] = a;
          } else {
            st_alpha[c] = st_rz[c] / dAd;
            if (blockIdx.x == 0) A.alphas[(long long)c * A.max_iter + a - 1] = st_alpha[c];
          }
        }
      }
      __syncthreads();
    }
    double trms[R], trz[R];
#pragma unroll
    for (int c = 0; c < R; ++c) trms[c] = trz[c] = 0.0;
    for (int e = tid; e < chunk * R; e += kThreads) {
      const int t = e / R, c = e - t * R;
      if (j0 + t >= pt) continue;
      double Ad = 0.0;
      for (int s = 0; s < S; ++s)
        for (int q = pp[s * (chunk + 1) + t]; q < pp[s * (chunk + 1) + t + 1]; ++q)
          Ad += __ldcg(A.pieces + (long long)q * R + c);
      Ad += oD[e] * od[e];
      double rv = orr[e];
      if (a == 0) {
        rv = ob[e] - Ad;
      } else if (st_active[c] && st_alpha[c] != 0.0) {
        ox[e] = fma(st_alpha[c], od[e], ox[e]);
        rv = fma(-st_alpha[c], Ad, rv);
      }
      orr[e] = rv;
      const double zn = om[e] * rv;
      oz[e] = zn;
      const double tj = os[e] * rv;
#pragma unroll
      for (int k = 0; k < R; ++k)
        if (k == c) {
          trms[k] += tj * tj;
          trz[k] += rv * zn;
        }
    }
#pragma unroll
    for (int c = 0; c < R; ++c) {
      double x1 = trms[c], x2 = trz[c];
      block_sum2(x1, x2, red);
      if (tid == 0) {
        A.part[(long long)blockIdx.x * PS + R + c] = x1;
        A.part[(long long)blockIdx.x * PS + 2 * R + c] = x2;
      }
    }
    cg::this_grid().sync();
  }

  __syncthreads();
  for (int e = tid; e < chunk * R; e += kThreads) {
    const int t = e / R, c = e - t * R;
    if (j0 + t < pt) A.x[ref_index(j0 + t, A.D.p, A.D.icpt) * R + c] = ox[e];
  }
  if (blockIdx.x == 0 && tid < R) {
    A.result[tid * 4 + 0] = st_iter[tid];
    A.result[tid * 4 + 1] = st_status[tid];
    A.result[tid * 4 + 2] = st_fail[tid];
    A.result[tid * 4 + 3] = st_applies;
  }
}

template <int R>
int set_attrs_b(const DesignDev& D) {
  const int bytes = (int)smem_bytes(D) * R;
  CUDA_TRY(cudaFuncSetAttribute(k_csr_b<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  CUDA_TRY(cudaFuncSetAttribute(k_csc_b<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  CUDA_TRY(cudaFuncSetAttribute(k_pcg_b<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pcg_b_smem<R>(D)));
  return PCGS_OK;
}

template <int R>
int phi_apply_b(const DesignDev& D, const double* omega, const double* diag, const double* v, double* out,
                cudaStream_t s) {
  int rc;
  if ((rc = set_attrs_b<R>(D))) return rc;
  Scratch S(s);
  double* w = S.get<double>((size_t)D.n * R + 16);
  double* pieces = S.get<double>((size_t)D.csc.nseg * R);
  double* zpart = D.csr.nslab > 1 ? S.get<double>((size_t)D.csr.nslab * D.n * R) : nullptr;
  if (!w || !pieces || (D.csr.nslab > 1 && !zpart)) return fail(PCGS_ENOMEM, "scratch allocation failed");
  if (D.csr.nslab > 1) {
    k_csr_b<R><<<D.G, kThreads, smem_bytes(D) * R, s>>>(D, v, omega, zpart);
    k_rows_combine_b<R><<<D.G * 4, 256, 0, s>>>(D, zpart, v, omega, w);
  } else {
    k_csr_b<R><<<D.G, kThreads, smem_bytes(D) * R, s>>>(D, v, omega, w);
  }
  k_csc_b<R><<<D.G, kThreads, smem_bytes(D) * R, s>>>(D, w, pieces);
  k_assemble_b<R><<<(int)((D.pt * R + 255) / 256), 256, 0, s>>>(D, pieces, diag, v, out);
  CUDA_TRY(cudaGetLastError());
  return PCGS_OK;
}

template <int R>
int pcg_b(const DesignDev& D, PcgArgsB& A, cudaStream_t s) {
  if (pcg_b_smem<R>(D) > 227 * 1024 - 2048)
    return fail(PCGS_EUNSUP, "batched PCG state does not fit shared memory for this batch size and design");
  int rc;
  if ((rc = set_attrs_b<R>(D))) return rc;
  if ((D.pt + D.G - 1) / D.G * R > kThreads * 8) return fail(PCGS_EUNSUP, "p_total too large for batched PCG");
  Scratch S(s);
  A.D = D;
  A.w = S.get<double>((size_t)D.n * R + 16);
  A.pieces = S.get<double>((size_t)D.csc.nseg * R);
  A.zpart = D.csr.nslab > 1 ? S.get<double>((size_t)D.csr.nslab * D.n * R) : nullptr;
  A.dvg = S.get<double>(2 * (((size_t)D.pt * R + 15) / 16 * 16) + 16);
  A.part = S.get<double>((size_t)part_stride_b<R>() * D.G);
  if (!A.w || !A.pieces || !A.dvg || !A.part || (D.csr.nslab > 1 && !A.zpart))
    return fail(PCGS_ENOMEM, "scratch allocation failed");
  void* args[] = {&A};
  CUDA_TRY(cudaLaunchCooperativeKernel((const void*)k_pcg_b<R>, D.G, kThreads, args, pcg_b_smem<R>(D), s));
  return PCGS_OK;
}

}  // namespace

extern "C" {

int pcgs_batch_slab_max(int nchains) {
  if (nchains != 2 && nchains != 4 && nchains != 8) return fail(PCGS_EINVAL, "nchains must be 2, 4 or 8");
  return (22528 - 16) / nchains - 16;
}

int pcgs_batch_phi_apply(pcgs_design_t d, int nchains, const double* omega, const double* prior_diag, const double* v,
                         double* out, pcgs_stream_t stream) {
  if (!d || !omega || !v || !out) return fail(PCGS_EINVAL, "null argument");
  const DesignDev& D = d->dev;
  cudaStream_t s = (cudaStream_t)stream;
  if ((long long)D.smem_doubles * nchains > 22528 + 16 * nchains)
    return fail(PCGS_EINVAL, "design slabs too large for this batch: create it with pcgs_batch_slab_max");
  switch (nchains) {
    case 2: return phi_apply_b<2>(D, omega, prior_diag, v, out, s);
    case 4: return phi_apply_b<4>(D, omega, prior_diag, v, out, s);
    case 8: return phi_apply_b<8>(D, omega, prior_diag, v, out, s);
    default: return fail(PCGS_EINVAL, "nchains must be 2, 4 or 8");
  }
}

int pcgs_batch_pcg(pcgs_design_t d, int nchains, const double* omega, const double* prior_diag, const double* minv,
                   const double* scale, const double* b, double* x, int32_t max_iter, double rtol, double* trace,
                   double* alphas, double* betas, int32_t* result, pcgs_stream_t stream) {
  if (!d || !omega || !prior_diag || !minv || !scale || !b || !x || !trace || !alphas || !betas || !result)
    return fail(PCGS_EINVAL, "null argument");
  if (max_iter < 1) return fail(PCGS_EINVAL, "max_iter must be at least 1");
  if ((long long)d->dev.smem_doubles * nchains > 22528 + 16 * nchains)
    return fail(PCGS_EINVAL, "design slabs too large for this batch: create it with pcgs_batch_slab_max");
  PcgArgsB A;
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
  cudaStream_t s = (cudaStream_t)stream;
  switch (nchains) {
    case 2: return pcg_b<2>(d->dev, A, s);
    case 4: return pcg_b<4>(d->dev, A, s);
    case 8: return pcg_b<8>(d->dev, A, s);
    default: return fail(PCGS_EINVAL, "nchains must be 2, 4 or 8");
  }
}

}  // extern "C"
