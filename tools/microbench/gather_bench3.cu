// Microbenchmark: random fp64 gathers for the pattern-only SpMV on B200.
// Compares: index stream alone (HBM), smem-staged gathers (random / bank-balanced),
// L1 gathers through ld.global.nc, int32 vs uint16 index streams.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_bench gather_bench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
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

__global__ void k_stream(const uint4* __restrict__ idx, long nvec, double* out) {
  long tid = blockIdx.x * (long)blockDim.x + threadIdx.x;
  long stride = (long)gridDim.x * blockDim.x;
  unsigned acc = 0;
  for (long i = tid; i < nvec; i += stride) {
    uint4 q = ldg_stream(idx + i);
    acc += q.x ^ q.y ^ q.z ^ q.w;
  }
  if (acc == 0x12345678u) out[tid] = acc;
}

template <int UNROLL>
__global__ void __launch_bounds__(1024, 1) k_smem_u16(const uint4* __restrict__ idx, long nvec,
                                                      const double* __restrict__ v, int p, double* out) {
  extern __shared__ double sv[];
  for (int i = threadIdx.x; i < p; i += blockDim.x) sv[i] = v[i];
  __syncthreads();
  long tid = blockIdx.x * (long)blockDim.x + threadIdx.x;
  long stride = (long)gridDim.x * blockDim.x;
  double acc = 0.0;
  long i = tid;
  for (; i + (UNROLL - 1) * stride < nvec; i += UNROLL * stride) {
    uint4 q[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) q[u] = ldg_stream(idx + i + u * stride);
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const unsigned w[4] = {q[u].x, q[u].y, q[u].z, q[u].w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        acc += sv[w[k] & 0xffff];
        acc += sv[w[k] >> 16];
      }
    }
  }
  for (; i < nvec; i += stride) {
    uint4 q = ldg_stream(idx + i);
    const unsigned w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) { acc += sv[w[k] & 0xffff]; acc += sv[w[k] >> 16]; }
  }
  out[tid] = acc;
}

// hi/lo word split: two 32-bit smem arrays
template <int UNROLL>
__global__ void __launch_bounds__(1024, 1) k_smem_split(const uint4* __restrict__ idx, long nvec,
                                                        const double* __restrict__ v, int p, double* out) {
  extern __shared__ unsigned sw[];
  unsigned* lo = sw;
  unsigned* hi = sw + p;
  for (int i = threadIdx.x; i < p; i += blockDim.x) {
    unsigned long long b = __double_as_longlong(v[i]);
    lo[i] = (unsigned)b; hi[i] = (unsigned)(b >> 32);
  }
  __syncthreads();
  long tid = blockIdx.x * (long)blockDim.x + threadIdx.x;
  long stride = (long)gridDim.x * blockDim.x;
  double acc = 0.0;
  long i = tid;
  for (; i + (UNROLL - 1) * stride < nvec; i += UNROLL * stride) {
    uint4 q[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) q[u] = ldg_stream(idx + i + u * stride);
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const unsigned w[4] = {q[u].x, q[u].y, q[u].z, q[u].w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        unsigned a = w[k] & 0xffff, b = w[k] >> 16;
        acc += __hiloint2double(hi[a], lo[a]);
        acc += __hiloint2double(hi[b], lo[b]);
      }
    }
  }
  out[tid] = acc;
}

template <int UNROLL>
__global__ void k_l1_u16(const uint4* __restrict__ idx, long nvec, const double* __restrict__ v, double* out) {
  long tid = blockIdx.x * (long)blockDim.x + threadIdx.x;
  long stride = (long)gridDim.x * blockDim.x;
  double acc = 0.0;
  long i = tid;
  for (; i + (UNROLL - 1) * stride < nvec; i += UNROLL * stride) {
    uint4 q[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) q[u] = ldg_stream(idx + i + u * stride);
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const unsigned w[4] = {q[u].x, q[u].y, q[u].z, q[u].w};
#pragma unroll
      for (int k = 0; k < 4; ++k) { acc += __ldg(v + (w[k] & 0xffff)); acc += __ldg(v + (w[k] >> 16)); }
    }
  }
  out[tid] = acc;
}

template <int UNROLL>
__global__ void k_l1_i32(const uint4* __restrict__ idx, long nvec, const double* __restrict__ v, double* out) {
  long tid = blockIdx.x * (long)blockDim.x + threadIdx.x;
  long stride = (long)gridDim.x * blockDim.x;
  double acc = 0.0;
  long i = tid;
  for (; i + (UNROLL - 1) * stride < nvec; i += UNROLL * stride) {
    uint4 q[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) q[u] = ldg_stream(idx + i + u * stride);
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      acc += __ldg(v + q[u].x); acc += __ldg(v + q[u].y); acc += __ldg(v + q[u].z); acc += __ldg(v + q[u].w);
    }
  }
  out[tid] = acc;
}

// gathers from an n-length (580 KB, L2-resident) vector with int32 indices: the naive CSC pass
template <int UNROLL>
__global__ void k_l2_i32(const uint4* __restrict__ idx, long nvec, const double* __restrict__ v, double* out) {
  long tid = blockIdx.x * (long)blockDim.x + threadIdx.x;
  long stride = (long)gridDim.x * blockDim.x;
  double acc = 0.0;
  long i = tid;
  for (; i + (UNROLL - 1) * stride < nvec; i += UNROLL * stride) {
    uint4 q[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) q[u] = ldg_stream(idx + i + u * stride);
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      acc += __ldg(v + q[u].x); acc += __ldg(v + q[u].y); acc += __ldg(v + q[u].z); acc += __ldg(v + q[u].w);
    }
  }
  out[tid] = acc;
}


template <int UNROLL>
__global__ void __launch_bounds__(1024, 1) k_smem_u16_macc(const uint4* __restrict__ idx, long nvec,
                                                      const double* __restrict__ v, int p, double* out) {
  extern __shared__ double sv[];
  for (int i = threadIdx.x; i < p; i += blockDim.x) sv[i] = v[i];
  __syncthreads();
  long tid = blockIdx.x * (long)blockDim.x + threadIdx.x;
  long stride = (long)gridDim.x * blockDim.x;
  double acc[8] = {0,0,0,0,0,0,0,0};
  long i = tid;
  for (; i + (UNROLL - 1) * stride < nvec; i += UNROLL * stride) {
    uint4 q[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) q[u] = ldg_stream(idx + i + u * stride);
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const unsigned w[4] = {q[u].x, q[u].y, q[u].z, q[u].w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        acc[2*k] += sv[w[k] & 0xffff];
        acc[2*k+1] += sv[w[k] >> 16];
      }
    }
  }
  out[tid] = acc[0]+acc[1]+acc[2]+acc[3]+acc[4]+acc[5]+acc[6]+acc[7];
}
template <int UNROLL>
__global__ void __launch_bounds__(512) k_stream_u(const uint4* __restrict__ idx, long nvec, double* out) {
  long tid = blockIdx.x * (long)blockDim.x + threadIdx.x;
  long stride = (long)gridDim.x * blockDim.x;
  unsigned acc = 0;
  long i = tid;
  for (; i + (UNROLL - 1) * stride < nvec; i += UNROLL * stride) {
    uint4 q[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) q[u] = ldg_stream(idx + i + u * stride);
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) acc += q[u].x ^ q[u].y ^ q[u].z ^ q[u].w;
  }
  for (; i < nvec; i += stride) { uint4 q = ldg_stream(idx + i); acc += q.x ^ q.y ^ q.z ^ q.w; }
  if (acc == 0x12345678u) out[tid] = acc;
}

template <int MODE>
__global__ void __launch_bounds__(1024, 1) k_iso(const uint4* __restrict__ idx, long nvec,
                                                 const double* __restrict__ v, int p, double* out) {
  extern __shared__ double sv[];
  for (int i = threadIdx.x; i < p; i += blockDim.x) sv[i] = v[i];
  __syncthreads();
  const unsigned long long* su = reinterpret_cast<const unsigned long long*>(sv);
  const unsigned* s32 = reinterpret_cast<const unsigned*>(sv);
  long tid = blockIdx.x * (long)blockDim.x + threadIdx.x;
  long stride = (long)gridDim.x * blockDim.x;
  double acc = 0.0; unsigned long long x = 0; unsigned x32 = 0;
  long i = tid;
  for (; i + 3 * stride < nvec; i += 4 * stride) {
    uint4 q[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) q[u] = ldg_stream(idx + i + u * stride);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const unsigned w[4] = {q[u].x, q[u].y, q[u].z, q[u].w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        unsigned a = w[k] & 0xffff, b = w[k] >> 16;
        if (MODE == 0) { x ^= su[a]; x ^= su[b]; }
        else if (MODE == 1) { x32 ^= s32[2*a]; x32 ^= s32[2*b]; }
        else if (MODE == 2) { acc += __longlong_as_double((long long)a << 40); acc += __longlong_as_double((long long)b << 40); }
        else if (MODE == 3) { x += a * 2654435761ull; x += b * 2654435761ull; }
      }
    }
  }
  out[tid] = acc + (double)x + (double)x32;
}
int main(int argc, char** argv) {
  const long nnz = 60000000;       // ~config-2 nnz
  const int p = 22176;             // smem vector length (config 2 + intercept)
  const int nrow = 72489;
  int dev = 0;
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, dev));
  printf("device %s SMs %d L2 %d MB smemOptin %zu KB\n", prop.name, prop.multiProcessorCount,
         prop.l2CacheSize >> 20, prop.sharedMemPerBlockOptin >> 10);
  int nsm = prop.multiProcessorCount;

  std::mt19937_64 g(1);
  std::vector<uint16_t> iu(nnz), ib(nnz);
  std::vector<uint32_t> i32(nnz), i32n(nnz);
  for (long i = 0; i < nnz; ++i) { iu[i] = (uint16_t)(g() % p); i32[i] = iu[i]; i32n[i] = (uint32_t)(g() % nrow); }
  // bank-balanced permutation of each 256-index warp block: the smem kernel's warp reads
  // uint4 i = tid (+stride...) so lane l of warp w reads vec (blockstart + l); instruction k
  // gathers element k of each lane's 8-vector. Sort each block of 256 by bank pair (idx%16)
  // and deal round-robin so element t goes to (lane t/8, slot t%8).
  // NOTE: the grid-stride loop maps consecutive lanes to consecutive uint4s, so a warp block is
  // 32 consecutive uint4 = 256 consecutive indices.
  for (long b = 0; b + 256 <= nnz; b += 256) {
    uint16_t tmp[256];
    std::copy(iu.begin() + b, iu.begin() + b + 256, tmp);
    std::stable_sort(tmp, tmp + 256, [](uint16_t x, uint16_t y) { return (x & 15) < (y & 15); });
    // element t of sorted -> slot (t % 8) of lane (t / 8)?  instruction k takes t = lane*8+k ...
    // we want instruction k (slot k) to take t = k, k+8, ..., i.e. every 8th sorted element.
    for (int t = 0; t < 256; ++t) {
      int slot = t % 8, lane = t / 8;
      // within-uint4 element order: word k holds elements 2k (lo) and 2k+1 (hi)
      ib[b + lane * 8 + slot] = tmp[t];
    }
  }
  for (long b = (nnz / 256) * 256; b < nnz; ++b) ib[b] = iu[b];

  uint16_t *d_iu, *d_ib; uint32_t *d_i32, *d_i32n; double *d_v, *d_vn, *d_out;
  CK(cudaMalloc(&d_iu, nnz * 2)); CK(cudaMalloc(&d_ib, nnz * 2));
  CK(cudaMalloc(&d_i32, nnz * 4)); CK(cudaMalloc(&d_i32n, nnz * 4));
  CK(cudaMalloc(&d_v, p * 8)); CK(cudaMalloc(&d_vn, nrow * 8));
  CK(cudaMalloc(&d_out, 64L * 1024 * 1024));
  CK(cudaMemcpy(d_iu, iu.data(), nnz * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_ib, ib.data(), nnz * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_i32, i32.data(), nnz * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_i32n, i32n.data(), nnz * 4, cudaMemcpyHostToDevice));
  std::vector<double> hv(nrow);
  for (int i = 0; i < nrow; ++i) hv[i] = (double)(i % 97) * 0.5;
  CK(cudaMemcpy(d_v, hv.data(), p * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_vn, hv.data(), nrow * 8, cudaMemcpyHostToDevice));
  // L2 flush buffer
  char* d_flush; size_t flushsz = 256L << 20;
  CK(cudaMalloc(&d_flush, flushsz));


  std::vector<uint16_t> iideal(nnz), ibc(nnz), ihw(nnz);
  for (long b = 0; b + 256 <= nnz; b += 256) {
    // ideal: slot k of lane l reads (base + l + 32*k) mod p  -> consecutive doubles per instruction
    int base = (int)(g() % (p - 300));
    for (int l = 0; l < 32; ++l) for (int k = 0; k < 8; ++k) { iideal[b + l*8 + k] = (uint16_t)(base + l + 32*k); ibc[b + l*8 + k] = (uint16_t)(base + k); }
    // half-warp balanced: bucket the 256 random indices by bank pair (idx%16), then for each slot k
    // and half h, pick one index from each bucket in turn (round-robin over buckets)
    std::vector<uint16_t> bucket[16];
    for (int t = 0; t < 256; ++t) bucket[iu[b+t] & 15].push_back(iu[b+t]);
    int bi = 0;
    std::vector<uint16_t> order; order.reserve(256);
    // interleave buckets: repeatedly take one from each non-empty bucket starting at rotating bi
    while ((int)order.size() < 256) {
      for (int c = 0; c < 16 && (int)order.size() < 256; ++c) {
        int bb = (bi + c) & 15;
        if (!bucket[bb].empty()) { order.push_back(bucket[bb].back()); bucket[bb].pop_back(); }
      }
      bi++;
    }
    // order[t]: consecutive 16 entries mostly distinct banks -> assign group of 16 to one half-warp slot
    for (int t = 0; t < 256; ++t) {
      int grp = t / 16, pos = t % 16;        // 16 groups = 8 slots x 2 halves
      int slot = grp / 2, half = grp % 2;
      int lane = half * 16 + pos;
      ihw[b + lane*8 + slot] = order[t];
    }
  }
  for (long b = (nnz / 256) * 256; b < nnz; ++b) { iideal[b] = ibc[b] = ihw[b] = iu[b]; }
  uint16_t *d_ideal, *d_bc, *d_hw;
  CK(cudaMalloc(&d_ideal, nnz * 2)); CK(cudaMalloc(&d_bc, nnz * 2)); CK(cudaMalloc(&d_hw, nnz * 2));
  CK(cudaMemcpy(d_ideal, iideal.data(), nnz * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_bc, ibc.data(), nnz * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_hw, ihw.data(), nnz * 2, cudaMemcpyHostToDevice));
  size_t smem = (size_t)p * 8;
  CK(cudaFuncSetAttribute(k_smem_u16<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(k_smem_u16<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(k_smem_split<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));

  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  auto timeit = [&](const char* name, double bytes, double gathers, auto launch) {
    float best = 1e30f, tot = 0;
    const int reps = 10;
    for (int r = 0; r < reps + 2; ++r) {
      CK(cudaMemsetAsync(d_flush, r, flushsz));
      CK(cudaEventRecord(e0));
      launch();
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      CK(cudaGetLastError());
      float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
      if (r >= 2) { best = std::min(best, ms); tot += ms; }
    }
    printf("%-28s best %8.2f us  avg %8.2f us  %7.1f GB/s  %6.2f Ggather/s  %5.2f gathers/clk/SM@1.9GHz\n",
           name, best * 1e3, tot / reps * 1e3, bytes / (best * 1e-3) / 1e9, gathers / (best * 1e-3) / 1e9,
           gathers / (best * 1e-3) / 1.9e9 / nsm);
  };
  long nv16 = nnz / 8, nv32 = nnz / 4;
  for (int bpsm : {4, 8, 16}) {
    char nm[64]; snprintf(nm, 64, "stream u16 (%d blk/SM)", bpsm);
    timeit(nm, nnz * 2.0, 0, [&] { k_stream<<<nsm * bpsm, 256>>>((const uint4*)d_iu, nv16, d_out); });
  }
  timeit("stream i32", nnz * 4.0, 0, [&] { k_stream<<<nsm * 8, 256>>>((const uint4*)d_i32, nv32, d_out); });
  timeit("smem u16 random U4", nnz * 2.0, nnz, [&] { k_smem_u16<4><<<nsm, 1024, smem>>>((const uint4*)d_iu, nv16, d_v, p, d_out); });
  timeit("smem u16 random U8", nnz * 2.0, nnz, [&] { k_smem_u16<8><<<nsm, 1024, smem>>>((const uint4*)d_iu, nv16, d_v, p, d_out); });
  timeit("smem u16 balanced U4", nnz * 2.0, nnz, [&] { k_smem_u16<4><<<nsm, 1024, smem>>>((const uint4*)d_ib, nv16, d_v, p, d_out); });
  timeit("smem u16 balanced U8", nnz * 2.0, nnz, [&] { k_smem_u16<8><<<nsm, 1024, smem>>>((const uint4*)d_ib, nv16, d_v, p, d_out); });
  timeit("smem split random U4", nnz * 2.0, nnz, [&] { k_smem_split<4><<<nsm, 1024, smem>>>((const uint4*)d_iu, nv16, d_v, p, d_out); });
  timeit("smem split balanced U4", nnz * 2.0, nnz, [&] { k_smem_split<4><<<nsm, 1024, smem>>>((const uint4*)d_ib, nv16, d_v, p, d_out); });
  for (int bpsm : {2, 4, 8}) {
    char nm[64]; snprintf(nm, 64, "L1 u16 random (%d blk/SM)", bpsm);
    timeit(nm, nnz * 2.0, nnz, [&] { k_l1_u16<4><<<nsm * bpsm, 256>>>((const uint4*)d_iu, nv16, d_v, d_out); });
  }
  timeit("L1 u16 balanced", nnz * 2.0, nnz, [&] { k_l1_u16<4><<<nsm * 4, 256>>>((const uint4*)d_ib, nv16, d_v, d_out); });
  timeit("L1 i32 random (p vec)", nnz * 4.0, nnz, [&] { k_l1_i32<4><<<nsm * 4, 256>>>((const uint4*)d_i32, nv32, d_v, d_out); });
  timeit("L2 i32 random (n vec)", nnz * 4.0, nnz, [&] { k_l2_i32<4><<<nsm * 4, 256>>>((const uint4*)d_i32n, nv32, d_vn, d_out); });

  CK(cudaFuncSetAttribute(k_smem_u16_macc<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  timeit("stream_u U8 x512 (4blk)", nnz * 2.0, 0, [&] { k_stream_u<8><<<nsm * 4, 512>>>((const uint4*)d_iu, nv16, d_out); });
  timeit("stream_u U4 x512 (4blk)", nnz * 2.0, 0, [&] { k_stream_u<4><<<nsm * 4, 512>>>((const uint4*)d_iu, nv16, d_out); });
  timeit("stream_u U8 x512 (2blk)", nnz * 2.0, 0, [&] { k_stream_u<8><<<nsm * 2, 512>>>((const uint4*)d_iu, nv16, d_out); });
  timeit("stream_u U8 i32 x512 (4blk)", nnz * 4.0, 0, [&] { k_stream_u<8><<<nsm * 4, 512>>>((const uint4*)d_i32, nv32, d_out); });
  timeit("smem ideal U4", nnz * 2.0, nnz, [&] { k_smem_u16<4><<<nsm, 1024, smem>>>((const uint4*)d_ideal, nv16, d_v, p, d_out); });
  timeit("smem bcast U4", nnz * 2.0, nnz, [&] { k_smem_u16<4><<<nsm, 1024, smem>>>((const uint4*)d_bc, nv16, d_v, p, d_out); });
  timeit("smem halfwarp-bal U4", nnz * 2.0, nnz, [&] { k_smem_u16<4><<<nsm, 1024, smem>>>((const uint4*)d_hw, nv16, d_v, p, d_out); });
  timeit("smem macc random U4", nnz * 2.0, nnz, [&] { k_smem_u16_macc<4><<<nsm, 1024, smem>>>((const uint4*)d_iu, nv16, d_v, p, d_out); });
  timeit("smem macc ideal U4", nnz * 2.0, nnz, [&] { k_smem_u16_macc<4><<<nsm, 1024, smem>>>((const uint4*)d_ideal, nv16, d_v, p, d_out); });
  timeit("smem macc hw-bal U4", nnz * 2.0, nnz, [&] { k_smem_u16_macc<4><<<nsm, 1024, smem>>>((const uint4*)d_hw, nv16, d_v, p, d_out); });
  timeit("smem split ideal U4", nnz * 2.0, nnz, [&] { k_smem_split<4><<<nsm, 1024, smem>>>((const uint4*)d_ideal, nv16, d_v, p, d_out); });
  timeit("smem split hw-bal U4", nnz * 2.0, nnz, [&] { k_smem_split<4><<<nsm, 1024, smem>>>((const uint4*)d_hw, nv16, d_v, p, d_out); });

  CK(cudaFuncSetAttribute(k_iso<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(k_iso<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(k_iso<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  CK(cudaFuncSetAttribute(k_iso<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  timeit("iso lds64-xor ideal", nnz * 2.0, nnz, [&] { k_iso<0><<<nsm, 1024, smem>>>((const uint4*)d_ideal, nv16, d_v, p, d_out); });
  timeit("iso lds64-xor random", nnz * 2.0, nnz, [&] { k_iso<0><<<nsm, 1024, smem>>>((const uint4*)d_iu, nv16, d_v, p, d_out); });
  timeit("iso lds32-xor ideal", nnz * 2.0, nnz, [&] { k_iso<1><<<nsm, 1024, smem>>>((const uint4*)d_ideal, nv16, d_v, p, d_out); });
  timeit("iso lds32-xor random", nnz * 2.0, nnz, [&] { k_iso<1><<<nsm, 1024, smem>>>((const uint4*)d_iu, nv16, d_v, p, d_out); });
  timeit("iso dadd only", nnz * 2.0, nnz, [&] { k_iso<2><<<nsm, 1024, smem>>>((const uint4*)d_iu, nv16, d_v, p, d_out); });
  timeit("iso int only", nnz * 2.0, nnz, [&] { k_iso<3><<<nsm, 1024, smem>>>((const uint4*)d_iu, nv16, d_v, p, d_out); });
  printf("done\n");


  return 0;
}
