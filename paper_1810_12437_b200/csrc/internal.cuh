// Host-side internals shared by the pcgs translation units (not part of the ABI).
#pragma once
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "device.cuh"
#include "pcgs.h"

using namespace pcgs;

void set_last_error(const std::string& msg);

inline int fail(int code, const std::string& msg) {
  set_last_error(msg);
  return code;
}
#define CUDA_TRY(x)                                                                  \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess)                                                           \
      return fail(PCGS_ECUDA, std::string(#x " failed: ") + cudaGetErrorString(e_)); \
  } while (0)

// =====================================================================
// design handle
// =====================================================================
struct pcgs_design {
  DesignDev dev;
  int device;
  int64_t info[16];
  std::vector<void*> allocs;
};

template <class T>
inline int upload(pcgs_design* D, const std::vector<T>& h, const T** out) {
  if (h.empty()) {
    *out = nullptr;
    return PCGS_OK;
  }
  void* p = nullptr;
  CUDA_TRY(cudaMalloc(&p, h.size() * sizeof(T)));
  D->allocs.push_back(p);
  CUDA_TRY(cudaMemcpy(p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
  *out = (const T*)p;
  return PCGS_OK;
}

inline int upload_pass(pcgs_design* D, const PassHost& H, PassDev& P) {
  int rc;
  const uint16_t* idx;
  if ((rc = upload(D, H.idx, &idx))) return rc;
  P.vec = (const uint4*)idx;
  const BlockDesc* b;
  if ((rc = upload(D, H.blocks, &b))) return rc;
  P.blocks = (const uint2*)b;
  if ((rc = upload(D, H.ids, &P.ids))) return rc;
  P.grouped = H.grouped;
  P.nranges = H.nranges;
  P.rep_ptr = nullptr;
  P.rep_src = nullptr;
  if (!H.rep_src.empty()) {
    if ((rc = upload(D, H.rep_ptr, &P.rep_ptr))) return rc;
    const uint16_t* rs;
    if ((rc = upload(D, H.rep_src, &rs))) return rc;
    P.rep_src = (const unsigned short*)rs;
  }
  const WarpRange* w;
  if ((rc = upload(D, H.warps, &w))) return rc;
  P.warps = (const uint4*)w;
  const Task* t;
  if ((rc = upload(D, H.tasks, &t))) return rc;
  P.task = (const int2*)t;
  if ((rc = upload(D, H.cta_task_ptr, &P.cta_task_ptr))) return rc;
  std::vector<long long> lo(H.slab_lo.begin(), H.slab_lo.end());
  if ((rc = upload(D, lo, &P.slab_lo))) return rc;
  if ((rc = upload(D, H.piece_ptr, &P.piece_ptr))) return rc;
  if ((rc = upload(D, H.col_piece_ptr, &P.col_piece_ptr))) return rc;
  P.ids_perm = nullptr;
  if (!H.piece_perm.empty() && H.grouped) {
    std::vector<uint32_t> ip(H.ids);
    for (uint32_t& v : ip)
      if (v != 0xffffffffu) v = (uint32_t)H.piece_perm[v];
    if ((rc = upload(D, ip, &P.ids_perm))) return rc;
  }
  P.nslab = H.nslab;
  P.nseg = H.nseg;
  return PCGS_OK;
}

// scratch buffers for one call, stream-ordered
struct Scratch {
  cudaStream_t s;
  std::vector<void*> bufs;
  explicit Scratch(cudaStream_t st) : s(st) {}
  ~Scratch() {
    for (void* b : bufs) cudaFreeAsync(b, s);
  }
  template <class T>
  T* get(size_t count) {
    void* p = nullptr;
    if (count == 0) count = 1;
    if (cudaMallocAsync(&p, count * sizeof(T), s) != cudaSuccess) return nullptr;
    bufs.push_back(p);
    return (T*)p;
  }
};

// =====================================================================
// fills and epilogues
// =====================================================================
struct FillVecRef {  // CSR slab of a reference-layout p_total vector (u = v / s when scaled)
  const double* v;
  int lead;           // reference offset of pattern column 0
  long long lo;
  const double* sc;   // affine column scales (reference layout) or null
  __device__ double operator()(int j) const {
    const long long r = lead + lo + j;
    const double x = __ldcg(v + r);
    return sc ? x / __ldg(sc + r) : x;
  }
  __device__ void operator()(double* sv, long long l, int len) {
    lo = l;
    fill_smem(sv, len, *this);
  }
};

struct FillVecN {  // CSC slab of an n-vector: TMA bulk copy
  const double* w;
  BulkFill* bf;
  __device__ void operator()(double* sv, long long l, int len) { bulk_fill(*bf, sv, w + l, len); }
};

struct FillBulk {  // TMA copy of an internal-layout vector slab
  const double* src;
  BulkFill* bf;
  __device__ void operator()(double* sv, long long l, int len) { bulk_fill(*bf, sv, src + l, len); }
};

struct FillBulkH {  // FillBulk taking run_pass's hook (k_pcg: the warps' prefetch runs in the TMA wait)
  const double* src;
  BulkFill* bf;
  static constexpr bool kHooked = true;
  template <class Hook>
  __device__ void operator()(double* sv, long long l, int len, Hook hook) { bulk_fill(*bf, sv, src + l, len, hook); }
};

struct FillRhs {  // u_i = kappa_i + sqrt(omega_i) * eta_i
  const double* kappa;
  const double* omega;
  const double* eta;  // null: Philox
  unsigned long long seed, stream;
  long long lo;
  long long row0 = 0;  // global index of local row 0 (row shards): Philox keys are global rows
  __device__ double operator()(int j) const {
    const long long i = lo + j;
    double e;
    if (eta) {
      e = __ldg(eta + i);
    } else {
      Philox R(seed, stream, (unsigned)(row0 + i));
      e = R.normal();
    }
    return (kappa ? __ldg(kappa + i) : 0.0) + sqrt(__ldg(omega + i)) * e;
  }
  __device__ void operator()(double* sv, long long l, int len) {
    lo = l;
    fill_smem(sv, len, *this);
  }
};

struct EpiStore {  // out[seg] = s
  double* out;
  long long cap = -1;  // checked builds: number of output slots (-1: unchecked)
  __device__ void emit(long long seg, double s) {
    PCGS_CHECK(seg >= 0 && (cap < 0 || seg < cap));
    out[seg] = s;
  }
};

// Row term of the dense block: (Dn u_D)_i = sum_k Dn[i, k] u_k (q = 0: none).
struct AffRow {
  const double* dense;  // n x q
  const double* u;      // q values of u_D
  int q;
  __device__ __forceinline__ double operator()(long long i) const {
    double t = 0.0;
    for (int k = 0; k < q; ++k) t += __ldg(dense + i * q + k) * __ldcg(u + k);
    return t;
  }
};

// The CSR row constant: u_icpt - mu'u for affine designs (cbuf[0], k_aff_pre),
// else the intercept value v[0] (or 0).
__device__ __forceinline__ double row_const(const DesignDev& D, const double* v, const double* cbuf) {
  return cbuf ? __ldcg(cbuf) : (D.icpt ? __ldg(v) : 0.0);
}
__device__ __forceinline__ AffRow aff_row(const DesignDev& D, const double* cbuf) {
  return AffRow{D.aff.dense, cbuf ? cbuf + 1 : nullptr, cbuf ? D.aff.q : 0};
}

struct EpiZ {  // matvec, single column slab: out[i] = v0 + s (+ dense row term)
  double* out;
  double v0;
  AffRow ar;
  __device__ void emit(long long seg, double s) { out[seg] = v0 + s + (ar.q ? ar(seg) : 0.0); }
};

struct EpiW {  // Phi apply, single column slab: w_i = omega_i z_i, z_i = v0 + s (+ row term); acc += w_i z_i
  double* w;
  const double* omega;
  double v0;
  double acc;
  AffRow ar;
  __device__ void emit(long long seg, double s) {
    const double z = v0 + s + (ar.q ? ar(seg) : 0.0);
    const double wi = __ldg(omega + seg) * z;
    w[seg] = wi;
    acc += wi * z;
  }
};

struct EpiCsr {  // runtime choice: multi column slab -> partial store, else EpiW
  double* out;
  const double* omega;
  double v0;
  double acc;
  bool multi;
  __device__ void emit(long long seg, double s) {
    if (multi) {
      out[seg] = s;
    } else {
      const double z = v0 + s;
      const double wi = __ldg(omega + seg) * z;
      out[seg] = wi;
      acc += wi * z;
    }
  }
};


struct EpiCsrA {  // EpiCsr with the affine row term (dense block) for the affine PCG kernel
  double* out;
  const double* omega;
  double v0;
  double acc;
  bool multi;
  AffRow ar;
  __device__ void emit(long long seg, double s) {
    if (multi) {
      out[seg] = s;
    } else {
      const double z = v0 + s + (ar.q ? ar(seg) : 0.0);
      const double wi = __ldg(omega + seg) * z;
      out[seg] = wi;
      acc += wi * z;
    }
  }
};

// Affine designs: launches k_aff_pre for the CSR row constants of v (cbuf is
// null for pattern-only designs).
int aff_pre(pcgs_design* d, const double* v, Scratch& S, cudaStream_t s, double** cbuf);

inline size_t smem_bytes(const DesignDev& D) { return (size_t)D.smem_doubles * sizeof(double); }
// threads per CTA of the standalone pass kernels: one warp per range of the store's tasks
inline int pass_threads(const DesignDev& D) { return D.csr.nranges * 32; }
// The standalone pass kernels come in two builds: 16 warps of 128 registers
// with two-block register batches (stores with <= 16 ranges per task) and 32
// warps of 64 registers with one-block batches.
#define PASS_LAUNCH(kern, D, smem, s, ...)                                            \
  do {                                                                                \
    if (pass_threads(D) <= 512) kern<512, 2><<<(D).G, pass_threads(D), smem, s>>>(__VA_ARGS__); \
    else kern<1024, 1><<<(D).G, pass_threads(D), smem, s>>>(__VA_ARGS__);             \
  } while (0)

// Raises a kernel's dynamic shared-memory limit to the device's opt-in maximum
// (minus its static shared memory).  The limit is a per-kernel, per-process
// attribute: setting it to a design's own need would lower it for designs
// created earlier, so every kernel is always set to the maximum (idempotent;
// the launch's dynamicSmemBytes decides what is actually used).
template <class K>
inline int raise_smem_limit(K kernel) {
  int dev = 0, optin = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  CUDA_TRY(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  cudaFuncAttributes fa;
  CUDA_TRY(cudaFuncGetAttributes(&fa, kernel));
  CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                optin - (int)fa.sharedSizeBytes));
  return PCGS_OK;
}
