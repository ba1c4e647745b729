// Microbenchmark: index stream staged through a per-warp TMA ring in shared
// memory (cp.async.bulk + mbarrier) vs per-warp register batches, both with a
// 177 KB fp64 slab in shared memory and bank-balanced uint16 gathers.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ long lmin(long a, long b) { return a < b ? a : b; }
__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* m, int c) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" :: "r"(su32(m)), "r"(c));
}
__device__ __forceinline__ void mbar_wait(unsigned long long* m, unsigned ph) {
  asm volatile("{\n.reg .pred P;\nW%=:\n"
               "mbarrier.try_wait.parity.shared.b64 P, [%0], %1;\n"
               "@!P bra W%=;\n}" :: "r"(su32(m)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* m) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" :: "r"(su32(m)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(su32(dst)), "l"(src), "r"(bytes), "r"(su32(m)) : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(p), "r"(bytes) : "memory");
}

__device__ void fill_slab(double* sv, const double* v, int p, unsigned long long* mb) {
  unsigned bytes = ((p * 8 + 15) / 16) * 16;
  if (threadIdx.x == 0) {
    mbar_init(mb, 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" :: "r"(su32(mb)), "r"(bytes));
    for (unsigned off = 0; off < bytes; off += 32768) {
      unsigned sz = bytes - off < 32768 ? bytes - off : 32768;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   :: "r"(su32((char*)sv + off)), "l"((const char*)v + off), "r"(sz), "r"(su32(mb)) : "memory");
    }
  }
  __syncthreads();
  mbar_wait(mb, 0);
}

__device__ __forceinline__ double gather8(uint4 q, const double* sv) {
  const unsigned w[4] = {q.x, q.y, q.z, q.w};
  double a = 0, b = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) { a += sv[w[k] & 0xffff]; b += sv[w[k] >> 16]; }
  return a + b;
}

// register batches of B blocks (32 vectors each) per warp range, optional L2 prefetch window
template <int B, bool PF>
__global__ void __launch_bounds__(1024, 1) k_reg(const uint4* __restrict__ idx, long nvec,
                                                  const double* __restrict__ v, int p, double* out) {
  extern __shared__ __align__(128) double sv[];
  __shared__ unsigned long long mb;
  fill_slab(sv, v, p, &mb);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long nw = (long)gridDim.x * 32, w = (long)blockIdx.x * 32 + warp;
  const long per = (nvec / 32 + nw - 1) / nw * 32;
  const long v0 = w * per, v1 = lmin(nvec, v0 + per);
  double acc = 0;
  if (PF && lane == 0 && v0 < v1) prefetch_l2(idx + v0, (unsigned)lmin(16 * 512, (v1 - v0) * 16));
  for (long b = v0; b < v1; b += 32 * B) {
    if (PF && lane == 0 && b + 16 * 32 < v1) prefetch_l2(idx + b + 16 * 32, (unsigned)lmin(B * 512, (v1 - b - 16 * 32) * 16));
    uint4 q[B];
#pragma unroll
    for (int u = 0; u < B; ++u) { long i = b + u * 32 + lane; q[u] = i < v1 ? ldg_stream(idx + i) : make_uint4(0, 0, 0, 0); }
#pragma unroll
    for (int u = 0; u < B; ++u) acc += gather8(q[u], sv);
  }
  out[blockIdx.x * 1024 + threadIdx.x] = acc;
}

// software-pipelined register batches: loads for batch i+1 issued before batch i is consumed
template <int B, int THREADS>
__global__ void __launch_bounds__(THREADS, 1) k_pipe(const uint4* __restrict__ idx, long nvec,
                                                      const double* __restrict__ v, int p, double* out) {
  extern __shared__ __align__(128) double sv[];
  __shared__ unsigned long long mb;
  fill_slab(sv, v, p, &mb);
  constexpr int W = THREADS / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long nw = (long)gridDim.x * W, w = (long)blockIdx.x * W + warp;
  const long per = (nvec / 32 + nw - 1) / nw * 32;
  const long v0 = w * per, v1 = lmin(nvec, v0 + per);
  double acc = 0;
  uint4 q[B], r[B];
#pragma unroll
  for (int u = 0; u < B; ++u) { long i = v0 + u * 32 + lane; q[u] = i < v1 ? ldg_stream(idx + i) : make_uint4(0, 0, 0, 0); }
  for (long b = v0; b < v1; b += 32 * B) {
#pragma unroll
    for (int u = 0; u < B; ++u) { long i = b + 32 * B + u * 32 + lane; r[u] = i < v1 ? ldg_stream(idx + i) : make_uint4(0, 0, 0, 0); }
#pragma unroll
    for (int u = 0; u < B; ++u) acc += gather8(q[u], sv);
#pragma unroll
    for (int u = 0; u < B; ++u) q[u] = r[u];
  }
  out[blockIdx.x * THREADS + threadIdx.x] = acc;
}

// per-warp TMA ring: S stages of C blocks (C*512 bytes) each
template <int S, int C, bool PF>
__global__ void __launch_bounds__(1024, 1) k_ring(const uint4* __restrict__ idx, long nvec,
                                                   const double* __restrict__ v, int p, int ring_off, double* out) {
  extern __shared__ __align__(128) double sv[];
  __shared__ unsigned long long mb;
  __shared__ unsigned long long rb[32][S];
  uint4* ring = reinterpret_cast<uint4*>(reinterpret_cast<char*>(sv) + ring_off);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint4* my = ring + warp * S * C * 32;
  const long nw = (long)gridDim.x * 32, w = (long)blockIdx.x * 32 + warp;
  const long per = (nvec / 32 + nw - 1) / nw * 32;
  const long v0 = w * per, v1 = lmin(nvec, v0 + per);
  const long nchunk = v1 > v0 ? (v1 - v0 + C * 32 - 1) / (C * 32) : 0;
  if (lane == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&rb[warp][s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
    if (PF && v0 < v1) prefetch_l2(idx + v0, (unsigned)lmin(16 * 512, (v1 - v0) * 16));
  }
  fill_slab(sv, v, p, &mb);  // contains __syncthreads
  if (lane == 0)
    for (int s = 0; s < S && s < nchunk; ++s) {
      long a = v0 + (long)s * C * 32;
      bulk_g2s(my + s * C * 32, idx + a, (unsigned)(lmin(C * 32, v1 - a) * 16), &rb[warp][s]);
    }
  __syncwarp();
  double acc = 0;
  for (long c = 0; c < nchunk; ++c) {
    const int s = (int)(c % S);
    const unsigned ph = (unsigned)((c / S) & 1);
    if (PF && lane == 0) { long a = v0 + (c + 16 / C) * C * 32; if (a < v1) prefetch_l2(idx + a, (unsigned)(lmin(C * 32, v1 - a) * 16)); }
    mbar_wait(&rb[warp][s], ph);
    const long a = v0 + c * C * 32;
    const int nv = (int)lmin(C * 32, v1 - a);
    uint4 q[C];
#pragma unroll
    for (int u = 0; u < C; ++u) q[u] = u * 32 + lane < nv ? my[s * C * 32 + u * 32 + lane] : make_uint4(0, 0, 0, 0);
    __syncwarp();
    if (lane == 0 && c + S < nchunk) {
      long a2 = v0 + (c + S) * C * 32;
      bulk_g2s(my + s * C * 32, idx + a2, (unsigned)(lmin(C * 32, v1 - a2) * 16), &rb[warp][s]);
    }
#pragma unroll
    for (int u = 0; u < C; ++u) acc += gather8(q[u], sv);
  }
  out[blockIdx.x * 1024 + threadIdx.x] = acc;
}

int main() {
  const long nnz = 60000000;
  const int p = 22176;
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  int nsm = prop.multiProcessorCount;
  std::mt19937_64 g(1);
  std::vector<uint16_t> iu(nnz), ihw(nnz), ipf(nnz);
  for (long i = 0; i < nnz; ++i) iu[i] = (uint16_t)(g() % p);
  // conflict-free: each half-warp group of 16 takes one index per bank pair
  for (long b = 0; b + 256 <= nnz; b += 256)
    for (int t = 0; t < 256; ++t) {
      int gi = t / 16, pos = t % 16, slot = gi / 2, lane = (gi % 2) * 16 + pos;
      int pair = (pos + gi * 5) % 16;
      ipf[b + lane * 8 + slot] = (uint16_t)(((g() % (p / 16 - 1)) * 16) + pair);
    }
  for (long b = (nnz / 256) * 256; b < nnz; ++b) ipf[b] = iu[b];
  uint16_t *d_iu, *d_pf;
  CK(cudaMalloc(&d_iu, nnz * 2)); CK(cudaMalloc(&d_pf, nnz * 2));
  CK(cudaMemcpy(d_iu, iu.data(), nnz * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_pf, ipf.data(), nnz * 2, cudaMemcpyHostToDevice));
  std::vector<double> hv(p);
  for (int i = 0; i < p; ++i) hv[i] = (double)(i % 97) * 0.5;
  double *d_v, *d_out;
  CK(cudaMalloc(&d_v, p * 8)); CK(cudaMalloc(&d_out, 64L << 20));
  CK(cudaMemcpy(d_v, hv.data(), p * 8, cudaMemcpyHostToDevice));
  char* d_flush; size_t flushsz = 256L << 20;
  CK(cudaMalloc(&d_flush, flushsz));
  const int slab = ((p * 8 + 16 + 127) / 128) * 128;
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  auto timeit = [&](const char* name, auto launch) {
    float best = 1e30f, tot = 0; const int reps = 10;
    for (int r = 0; r < reps + 2; ++r) {
      CK(cudaMemsetAsync(d_flush, r, flushsz));
      CK(cudaEventRecord(e0)); launch(); CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1)); CK(cudaGetLastError());
      float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
      if (r >= 2) { best = std::min(best, ms); tot += ms; }
    }
    printf("%-34s best %8.2f us avg %8.2f us  idx %7.1f GB/s\n", name, best * 1e3, tot / reps * 1e3,
           nnz * 2.0 / (best * 1e-3) / 1e9);
  };
  long nv = nnz / 8;
#define REG(B, PF, data, name) { auto kf = k_reg<B, PF>; CK(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, slab)); \
    timeit(name, [&] { kf<<<nsm, 1024, slab>>>((const uint4*)data, nv, d_v, p, d_out); }); }
#define RING(S, C, PF, data, name) { auto kf = k_ring<S, C, PF>; int sm = slab + 32 * S * C * 512; \
    CK(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, sm)); \
    timeit(name, [&] { kf<<<nsm, 1024, sm>>>((const uint4*)data, nv, d_v, p, slab, d_out); }); }
  REG(4, false, d_pf, "reg B=4 conflict-free");
  REG(2, false, d_pf, "reg B=2 conflict-free");
  REG(6, false, d_pf, "reg B=6 conflict-free");
#define PIPE(B, T, name) { auto kf = k_pipe<B, T>; CK(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, slab)); \
    timeit(name, [&] { kf<<<nsm, T, slab>>>((const uint4*)d_pf, nv, d_v, p, d_out); }); }
  PIPE(2, 1024, "pipe B=2 T=1024");
  PIPE(3, 1024, "pipe B=3 T=1024");
  PIPE(4, 1024, "pipe B=4 T=1024");
  PIPE(4, 512, "pipe B=4 T=512");
  PIPE(6, 512, "pipe B=6 T=512");
  PIPE(8, 512, "pipe B=8 T=512");
  PIPE(8, 256, "pipe B=8 T=256");
  PIPE(12, 256, "pipe B=12 T=256");
  printf("done\n");
  return 0;
}
