// Batched independent chains (BASELINE config 4; SURVEY §8e "chain batching"):
// R chains share every walk over the pattern through the sliced store
// (sliced.h).  All device vectors are chain-minor, element (j, c) at
// [j * R + c]; a warp is 32/R slots of R lanes, lane (slot, c) sums chain c
// of its slot's piece, so there is no cross-lane reduction in the streaming
// loop and one index costs R lane-LDS.64 that fill a wavefront.
//
// Reference: PrecisionOperator.apply (pkg/src/priorcg/sampler.py:53-58) per
// chain, pcg_solve (cg.py:105-192) per chain with chains masked once they
// terminate.
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <string>

#include "internal.cuh"
#include "sliced.cuh"

namespace cg = cooperative_groups;

namespace {

template <class T>
int upload_b(pcgs_batch* B, const std::vector<T>& h, const T** out) {
  if (h.empty()) {
    *out = nullptr;
    return PCGS_OK;
  }
  void* p = nullptr;
  CUDA_TRY(cudaMalloc(&p, h.size() * sizeof(T)));
  B->allocs.push_back(p);
  CUDA_TRY(cudaMemcpy(p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
  *out = (const T*)p;
  return PCGS_OK;
}

int upload_spass(pcgs_batch* B, const SPassHost& H, SPassDev& P) {
  int rc;
  const uint16_t* idx;
  if ((rc = upload_b(B, H.idx, &idx))) return rc;
  P.vec = (const uint4*)idx;
  const SliceDesc* sl;
  if ((rc = upload_b(B, H.slices, &sl))) return rc;
  P.slices = (const uint2*)sl;
  if ((rc = upload_b(B, H.piece, &P.piece))) return rc;
  const uint32_t* ws;
  if ((rc = upload_b(B, H.warp_slices, &ws))) return rc;
  P.warp_slices = (const uint2*)ws;
  const Task* t;
  if ((rc = upload_b(B, H.tasks, &t))) return rc;
  P.task = (const int2*)t;
  if ((rc = upload_b(B, H.cta_task_ptr, &P.cta_task_ptr))) return rc;
  std::vector<long long> lo(H.slab_lo.begin(), H.slab_lo.end());
  if ((rc = upload_b(B, lo, &P.slab_lo))) return rc;
  std::vector<long long> op(H.out_ptr.begin(), H.out_ptr.end());
  if ((rc = upload_b(B, op, &P.out_ptr))) return rc;
  P.nslab = H.nslab;
  P.npiece = H.npiece;
  return PCGS_OK;
}

// ------------------------------------------------------------------ kernels (single apply)
template <int R>
__global__ void __launch_bounds__(kSThreads, 1) k_scsr(BatchDev D, const double* v_ref, double* zpiece) {
  extern __shared__ __align__(128) double sv[];
  __shared__ unsigned long long mbar;
  BulkFill bf;
  bulk_init(bf, &mbar);
  FillRows<R> f{v_ref + (long long)D.icpt * R, &bf};
  EpiPiece e{zpiece, R};
  run_spass<R>(D.csr, sv, f, e);
}

template <int R>
__global__ void __launch_bounds__(kSThreads, 1) k_scsc(BatchDev D, const double* w, double* pieces) {
  extern __shared__ __align__(128) double sv[];
  __shared__ unsigned long long mbar;
  BulkFill bf;
  bulk_init(bf, &mbar);
  FillRows<R> f{w, &bf};
  EpiPiece e{pieces, R};
  run_spass<R>(D.csc, sv, f, e);
}

// w = omega (sum of the row's pieces + v0)
template <int R>
__global__ void k_scombine(BatchDev D, const double* zpiece, const double* v_ref, const double* omega, double* w) {
  const long long nr = D.n * R;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nr; e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / R;
    const int c = (int)(e & (R - 1));
    double z = 0.0;
    for (long long q = D.csr.out_ptr[i]; q < D.csr.out_ptr[i + 1]; ++q) z += zpiece[q * R + c];
    z += D.icpt ? v_ref[c] : 0.0;
    w[e] = omega ? __ldg(omega + e) * z : z;
  }
}

// out (reference layout) = sum of the column's pieces + diag * v
template <int R>
__global__ void k_sassemble(BatchDev D, const double* pieces, const double* diag, const double* v_ref, double* out) {
  const long long nr = D.pt * R;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nr; e += (long long)gridDim.x * blockDim.x) {
    const long long j = e / R;
    const int c = (int)(e & (R - 1));
    double s = 0.0;
    for (long long q = D.csc.out_ptr[j]; q < D.csc.out_ptr[j + 1]; ++q) s += pieces[q * R + c];
    const long long r = ref_index(j, D.p, D.icpt) * R + c;
    out[r] = diag ? s + diag[r] * v_ref[r] : s;
  }
}

// ---------------------------------------------------------------------------
// batched persistent PCG: the reference loop (cg.py:105-192) per chain; a
// chain that terminates keeps a zero direction until every chain is done.
// Per iteration: CSR pass (pieces of X d) | row combine (w = omega z, z'Omega z)
// | CSC pass (pieces of X'w) | column step (x, r, z, partials) | direction.
// ---------------------------------------------------------------------------
struct PcgArgsS {
  BatchDev D;
  const double *omega, *diag, *minv, *scale, *b;  // chain-minor, reference layout
  double* x;
  int max_iter;
  double rtol;
  double *trace, *alphas, *betas;  // [c][max_iter+1], [c][max_iter]
  int* result;                     // [c][4]
  double *zpiece, *w, *pieces, *dg, *own, *part;
  unsigned long long* prof;  // debug: [8 a + k] phase stamps of iterations a < 64 (pcgs_batch_debug_profile)
};

template <int R>
__host__ __device__ constexpr int part_stride_s() {
  return 16 * ((3 * R + 15) / 16);
}

template <int R>
__global__ void __launch_bounds__(kSThreads, 1) k_spcg(PcgArgsS A) {
  extern __shared__ __align__(128) double sv[];
  __shared__ double red[32 * R];
  __shared__ double sred[3 * R];
  __shared__ double st_rz[R], st_beta[R], st_alpha[R], v0s[R];
  __shared__ int st_active[R], st_status[R], st_iter[R], st_fail[R];
  __shared__ int st_applies, st_any;
  __shared__ unsigned long long mbar;
  BulkFill bf;
  bulk_init(bf, &mbar);
  const int tid = threadIdx.x;
  const int c_t = tid & (R - 1);  // the chain of this thread in element loops (strides are multiples of R)
  constexpr int PS = part_stride_s<R>();
  const BatchDev& D = A.D;
  const long long pt = D.pt;
  const long long chunk = (pt + gridDim.x - 1) / gridDim.x;
  const long long j0 = (long long)blockIdx.x * chunk;
  const long long jend = min(j0 + chunk, pt);
  const long long e0 = j0 * R, e1 = jend * R;  // own elements
  const long long ptR = pt * R;
  double *ox = A.own, *orr = A.own + ptR, *od = A.own + 2 * ptR, *oz = A.own + 3 * ptR;

  // own slice: x0, the first direction (v = x0), r, z
  for (long long e = e0 + tid; e < e1; e += kSThreads) {
    const long long j = e / R;
    const long long r = ref_index(j, D.p, D.icpt) * R + c_t;
    const double xv = A.x[r];
    ox[e] = xv;
    od[e] = xv;
    orr[e] = 0.0;
    oz[e] = 0.0;
    A.dg[e] = xv;
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
  // dAd prior part of the first application is not used (a = 0 has no alpha)
  cg::this_grid().sync();

  const bool prof_cta = A.prof && blockIdx.x == 0 && tid == 0;
  auto stamp = [&](int a, int k) {
    if (prof_cta && a < 64) A.prof[8 * a + k] = stimer();
  };
  for (int a = 0;; ++a) {
    stamp(a, 0);
    // ---------------- phase A: CSR pass, pieces of X d ----------------
    if (tid < R) v0s[tid] = D.icpt ? __ldcg(A.dg + D.p * R + tid) : 0.0;
    {
      FillRows<R> f{A.dg, &bf};
      EpiPiece e{A.zpiece, R};
      run_spass<R>(D.csr, sv, f, e);
    }
    cg::this_grid().sync();
    stamp(a, 1);
    // ---------------- row combine: w = omega z, z' Omega z per chain ----------------
    double wz = 0.0;
    {
      const long long nr = D.n * R;
      for (long long e = (long long)blockIdx.x * kSThreads + tid; e < nr; e += (long long)gridDim.x * kSThreads) {
        const long long i = e / R;
        double z = 0.0;
        const long long q1 = D.csr.out_ptr[i + 1];
        for (long long q = D.csr.out_ptr[i]; q < q1; ++q) z += __ldcg(A.zpiece + q * R + c_t);
        z += v0s[c_t];
        const double wi = __ldg(A.omega + e) * z;
        A.w[e] = wi;
        wz += wi * z;
      }
    }
    {
      const double t = block_sum_chain<R>(wz, red);
      if (tid < R) A.part[(long long)blockIdx.x * PS + tid] += t;  // + the D d^2 part written with d
    }
    cg::this_grid().sync();
    stamp(a, 2);
    // ---------------- phase B: CSC pass, pieces of X' w ----------------
    {
      FillRows<R> f{A.w, &bf};
      EpiPiece e{A.pieces, R};
      run_spass<R>(D.csc, sv, f, e);
    }
    cg::this_grid().sync();
    stamp(a, 3);
    if (tid == 0) ++st_applies;

    // ---------------- phase C: per-chain step on the own columns ----------------
    if (a > 0) {
      reduce_parts(A.part, PS, 0, R, sred);
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
    double trms = 0.0, trz = 0.0;
    {
      const bool live = st_active[c_t] && st_alpha[c_t] != 0.0;
      const double alpha = st_alpha[c_t];
      // own columns in NH rounds whose pieces fit the idle slab (staged; else global loads)
      const long long jb0 = e0 / R, jb1 = e1 / R;
      const int NH = stage_rounds<R>(D.csc.out_ptr, jb0, jb1, D.smem_doubles);
      for (int h = 0; h < NH; ++h) {
      const long long ja = jb0 + (jb1 - jb0) * h / NH, jz = jb0 + (jb1 - jb0) * (h + 1) / NH;
      if (h > 0) __syncthreads();
      const long long Q0 = stage_own_pieces<R>(A.pieces, D.csc.out_ptr, ja, jz, sv, D.smem_doubles);
      for (long long e = ja * R + tid; e < jz * R; e += kSThreads) {
        const long long j = e / R;
        double Ad = 0.0;
        const long long q1 = D.csc.out_ptr[j + 1];
        if (Q0 >= 0) {
          for (long long q = D.csc.out_ptr[j]; q < q1; ++q) Ad += sv[(q - Q0) * R + c_t];
        } else {
          for (long long q = D.csc.out_ptr[j]; q < q1; ++q) Ad += __ldcg(A.pieces + q * R + c_t);
        }
        const long long r = ref_index(j, D.p, D.icpt) * R + c_t;
        const double dv = od[e];
        Ad += __ldg(A.diag + r) * dv;
        double rv = orr[e];
        if (a == 0) {
          rv = __ldg(A.b + r) - Ad;
        } else if (live) {
          ox[e] = fma(alpha, dv, ox[e]);
          rv = fma(-alpha, Ad, rv);
        }
        orr[e] = rv;
        const double zn = __ldg(A.minv + r) * rv;
        oz[e] = zn;
        const double tj = __ldg(A.scale + r) * rv;
        trms += tj * tj;
        trz += rv * zn;
      }
      }
    }
    {
      const double s1 = block_sum_chain<R>(trms, red);
      const double s2 = block_sum_chain<R>(trz, red);
      if (tid < R) {
        A.part[(long long)blockIdx.x * PS + R + tid] = s1;
        A.part[(long long)blockIdx.x * PS + 2 * R + tid] = s2;
      }
    }
    cg::this_grid().sync();
    stamp(a, 4);

    // ---------------- convergence test, beta, new direction ----------------
    reduce_parts(A.part, PS, R, 2 * R, sred);
    if (tid < R) {
      const int c = tid;
      double beta = 0.0;
      if (st_active[c]) {
        const double rms = sqrt(sred[R + c] / (double)pt), rzn = sred[2 * R + c];
        const int k = a;  // iterations completed
        if (blockIdx.x == 0) A.trace[(long long)c * (A.max_iter + 1) + k] = rms;
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
          if (a >= 1) {
            beta = rzn / st_rz[c];
            if (blockIdx.x == 0) A.betas[(long long)c * A.max_iter + a - 1] = beta;
          }
          st_rz[c] = rzn;
          if (k >= A.max_iter) {
            st_active[c] = 0;
            st_status[c] = PCGS_MAX_ITER;
            st_iter[c] = k;
          }
        }
      }
      st_beta[c] = beta;
    }
    __syncthreads();
    if (tid == 0) {
      int any = 0;
      for (int c = 0; c < R; ++c) any |= st_active[c];
      st_any = any;
    }
    __syncthreads();
    if (!st_any) break;
    double dd = 0.0;
    {
      const bool act = st_active[c_t];
      const double beta = st_beta[c_t];
      for (long long e = e0 + tid; e < e1; e += kSThreads) {
        const double dn = act ? (a == 0 ? oz[e] : fma(beta, od[e], oz[e])) : 0.0;
        od[e] = dn;
        A.dg[e] = dn;
        const long long r = ref_index(e / R, D.p, D.icpt) * R + c_t;
        dd += __ldg(A.diag + r) * dn * dn;
      }
    }
    {
      const double t = block_sum_chain<R>(dd, red);
      if (tid < R) A.part[(long long)blockIdx.x * PS + tid] = t;
    }
    cg::this_grid().sync();
    stamp(a, 5);
  }

  __syncthreads();
  for (long long e = e0 + tid; e < e1; e += kSThreads) {
    const long long j = e / R;
    A.x[ref_index(j, D.p, D.icpt) * R + c_t] = ox[e];
  }
  if (blockIdx.x == 0 && tid < R) {
    A.result[tid * 4 + 0] = st_iter[tid];
    A.result[tid * 4 + 1] = st_status[tid];
    A.result[tid * 4 + 2] = st_fail[tid];
    A.result[tid * 4 + 3] = st_applies;
  }
}

size_t slab_bytes(const BatchDev& D) { return (size_t)D.smem_doubles * 8; }

unsigned long long* g_bprof = nullptr;  // pcgs_batch_debug_profile

template <int R>
int raise_all_s() {
  int rc;
  if ((rc = raise_smem_limit(k_scsr<R>)) || (rc = raise_smem_limit(k_scsc<R>)) ||
      (rc = raise_smem_limit(k_spcg<R>)))
    return rc;
  return PCGS_OK;
}

template <int R>
int phi_apply_s(const BatchDev& D, const double* omega, const double* diag, const double* v, double* out,
                cudaStream_t s) {
  int rc;
  if ((rc = raise_all_s<R>())) return rc;
  Scratch S(s);
  double* zp = S.get<double>((size_t)D.csr.npiece * R);
  double* w = S.get<double>((size_t)D.n * R);
  double* pieces = S.get<double>((size_t)D.csc.npiece * R);
  if (!zp || !w || !pieces) return fail(PCGS_ENOMEM, "scratch allocation failed");
  k_scsr<R><<<D.G, kSThreads, slab_bytes(D), s>>>(D, v, zp);
  k_scombine<R><<<D.G * 4, 256, 0, s>>>(D, zp, v, omega, w);
  k_scsc<R><<<D.G, kSThreads, slab_bytes(D), s>>>(D, w, pieces);
  k_sassemble<R><<<(int)std::min<long long>((D.pt * R + 255) / 256, 4 * D.G), 256, 0, s>>>(D, pieces, diag, v, out);
  CUDA_TRY(cudaGetLastError());
  return PCGS_OK;
}

template <int R>
int pcg_s(const BatchDev& D, PcgArgsS& A, cudaStream_t s) {
  int rc;
  if ((rc = raise_all_s<R>())) return rc;
  Scratch S(s);
  A.D = D;
  A.prof = g_bprof;
  A.zpiece = S.get<double>((size_t)D.csr.npiece * R);
  A.w = S.get<double>((size_t)D.n * R);
  A.pieces = S.get<double>((size_t)D.csc.npiece * R);
  A.dg = S.get<double>((size_t)D.pt * R + 16);
  A.own = S.get<double>((size_t)4 * D.pt * R);
  A.part = S.get<double>((size_t)part_stride_s<R>() * D.G);
  if (!A.zpiece || !A.w || !A.pieces || !A.dg || !A.own || !A.part)
    return fail(PCGS_ENOMEM, "scratch allocation failed");
  CUDA_TRY(cudaMemsetAsync(A.part, 0, sizeof(double) * part_stride_s<R>() * D.G, s));
  void* args[] = {&A};
  CUDA_TRY(cudaLaunchCooperativeKernel((const void*)k_spcg<R>, D.G, kSThreads, args, slab_bytes(D), s));
  return PCGS_OK;
}

}  // namespace

extern "C" {

int pcgs_batch_create(int64_t n, int64_t p, const int64_t* row_ptr_h, const int32_t* col_idx_h, int intercept,
                      int nchains, int slab_max, int device, int grid, pcgs_batch_t* out) {
  if (!out || !row_ptr_h || (!col_idx_h && row_ptr_h[n] > 0)) return fail(PCGS_EINVAL, "null argument");
  *out = nullptr;
  if (nchains != 1 && nchains != 2 && nchains != 4 && nchains != 8)
    return fail(PCGS_EINVAL, "nchains must be 1, 2, 4 or 8");
  CUDA_TRY(cudaSetDevice(device));
  cudaDeviceProp prop;
  CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  const int sms = std::min(prop.multiProcessorCount, 256);
  if (grid < 0 || grid > sms) return fail(PCGS_EINVAL, "grid must be in [0, SM count]");
  const int G = grid > 0 ? grid : sms;
  SlicedHost H;
  std::string err = build_sliced(n, p, row_ptr_h, col_idx_h, intercept, nchains, slab_max, G, H);
  if (!err.empty()) return fail(PCGS_EINVAL, err);
  pcgs_batch* B = new pcgs_batch();
  B->device = device;
  BatchDev& d = B->dev;
  d.n = n;
  d.p = p;
  d.pt = H.p_total;
  d.icpt = H.intercept;
  d.G = G;
  d.R = nchains;
  int64_t maxlen = 0;
  for (const SPassHost* P : {&H.csr, &H.csc})
    for (int q = 0; q < P->nslab; ++q) maxlen = std::max<int64_t>(maxlen, P->slab_lo[q + 1] - P->slab_lo[q]);
  d.smem_doubles = (int)((maxlen + 1) * nchains);
  int rc;
  if ((rc = upload_spass(B, H.csr, d.csr)) || (rc = upload_spass(B, H.csc, d.csc))) {
    pcgs_batch_destroy(B);
    return rc;
  }
  int64_t* I = B->info;
  memset(I, 0, sizeof(B->info));
  I[0] = n;
  I[1] = p;
  I[2] = H.p_total;
  I[3] = H.nnz;
  I[4] = H.csr.nslab;
  I[5] = H.csc.nslab;
  I[6] = (int64_t)(H.csr.idx.size() / kVecIdx);
  I[7] = (int64_t)(H.csc.idx.size() / kVecIdx);
  I[8] = H.csr.npiece;
  I[9] = H.csc.npiece;
  I[10] = nchains;
  I[11] = G;
  I[12] = device;
  I[13] = (int64_t)(H.csr.idx.size() + H.csc.idx.size()) * 2;
  I[14] = H.slab_max;
  I[15] = (H.csr.lds_excess + H.csc.lds_excess) * 1000000 / std::max<int64_t>(1, H.csr.lds_groups + H.csc.lds_groups);
  *out = B;
  return PCGS_OK;
}

int pcgs_batch_destroy(pcgs_batch_t b) {
  if (!b) return PCGS_OK;
  for (void* p : b->allocs) cudaFree(p);
  delete b;
  return PCGS_OK;
}

int pcgs_batch_info(pcgs_batch_t b, int64_t* info_h) {
  if (!b || !info_h) return fail(PCGS_EINVAL, "null argument");
  memcpy(info_h, b->info, sizeof(b->info));
  return PCGS_OK;
}

int pcgs_batch_selftest(int64_t n, int64_t p, const int64_t* row_ptr_h, const int32_t* col_idx_h, int intercept,
                        int nchains, int slab_max, int grid, int64_t* stats_h) {
  if (!row_ptr_h || grid < 1) return fail(PCGS_EINVAL, "null argument");
  SlicedHost H;
  std::string err = build_sliced(n, p, row_ptr_h, col_idx_h, intercept, nchains, slab_max, grid, H);
  if (!err.empty()) return fail(PCGS_EINVAL, err);
  err = verify_sliced(H, row_ptr_h, col_idx_h);
  if (stats_h) {
    stats_h[0] = H.csr.nslab;
    stats_h[1] = H.csc.nslab;
    stats_h[2] = (int64_t)(H.csr.idx.size() / kVecIdx);
    stats_h[3] = (int64_t)(H.csc.idx.size() / kVecIdx);
    stats_h[4] = H.csr.npiece;
    stats_h[5] = H.csc.npiece;
    stats_h[6] = H.csr.lds_groups + H.csc.lds_groups;
    stats_h[7] = H.csr.lds_excess + H.csc.lds_excess;
    stats_h[8] = H.csr.pad_vectors + H.csc.pad_vectors;
  }
  if (!err.empty()) return fail(PCGS_EUNSUP - 100, "sliced store self-test failed: " + err);
  return PCGS_OK;
}

}  // extern "C"
unsigned long long* batch_profile_buffer() { return g_bprof; }
extern "C" {

int pcgs_batch_debug_profile(void* buf) {
  g_bprof = (unsigned long long*)buf;
  return PCGS_OK;
}

int pcgs_batch_phi_apply(pcgs_batch_t bt, const double* omega, const double* prior_diag, const double* v,
                         double* out, pcgs_stream_t stream) {
  if (!bt || !omega || !v || !out) return fail(PCGS_EINVAL, "null argument");
  const BatchDev& D = bt->dev;
  cudaStream_t s = (cudaStream_t)stream;
  switch (D.R) {
    case 1: return phi_apply_s<1>(D, omega, prior_diag, v, out, s);
    case 2: return phi_apply_s<2>(D, omega, prior_diag, v, out, s);
    case 4: return phi_apply_s<4>(D, omega, prior_diag, v, out, s);
    case 8: return phi_apply_s<8>(D, omega, prior_diag, v, out, s);
    default: return fail(PCGS_EINVAL, "bad batch handle");
  }
}

int pcgs_batch_pcg(pcgs_batch_t bt, const double* omega, const double* prior_diag, const double* minv,
                   const double* scale, const double* b, double* x, int32_t max_iter, double rtol, double* trace,
                   double* alphas, double* betas, int32_t* result, pcgs_stream_t stream) {
  if (!bt || !omega || !prior_diag || !minv || !scale || !b || !x || !trace || !alphas || !betas || !result)
    return fail(PCGS_EINVAL, "null argument");
  if (max_iter < 1) return fail(PCGS_EINVAL, "max_iter must be at least 1");
  PcgArgsS A;
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
  switch (bt->dev.R) {
    case 1: return pcg_s<1>(bt->dev, A, s);
    case 2: return pcg_s<2>(bt->dev, A, s);
    case 4: return pcg_s<4>(bt->dev, A, s);
    case 8: return pcg_s<8>(bt->dev, A, s);
    default: return fail(PCGS_EINVAL, "bad batch handle");
  }
}

}  // extern "C"
