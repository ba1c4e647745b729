// What read bandwidth can a streaming kernel reach on B200, by access pattern?
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <algorithm>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ long lmin(long a, long b) { return a < b ? a : b; }

// grid-stride, B loads in flight per thread
template <int B>
__global__ void __launch_bounds__(1024, 1) k_gs(const uint4* __restrict__ a, long nv, unsigned* out) {
  const long stride = (long)gridDim.x * blockDim.x;
  unsigned acc = 0;
  long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  for (; i + (B - 1) * stride < nv; i += B * stride) {
    uint4 q[B];
#pragma unroll
    for (int u = 0; u < B; ++u) q[u] = ldg_stream(a + i + u * stride);
#pragma unroll
    for (int u = 0; u < B; ++u) acc ^= q[u].x + q[u].w;
  }
  for (; i < nv; i += stride) acc ^= ldg_stream(a + i).y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// per-warp contiguous range, B blocks of 32 vectors per batch
template <int B, int T>
__global__ void __launch_bounds__(T, 1) k_warp(const uint4* __restrict__ a, long nv, unsigned* out) {
  constexpr int W = T / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long nw = (long)gridDim.x * W, w = (long)blockIdx.x * W + warp;
  const long per = (nv / 32 + nw - 1) / nw * 32;
  const long v0 = w * per, v1 = lmin(nv, v0 + per);
  unsigned acc = 0;
  for (long b = v0; b < v1; b += 32 * B) {
    uint4 q[B];
#pragma unroll
    for (int u = 0; u < B; ++u) { long i = b + u * 32 + lane; q[u] = i < v1 ? ldg_stream(a + i) : make_uint4(0, 0, 0, 0); }
#pragma unroll
    for (int u = 0; u < B; ++u) acc ^= q[u].x + q[u].w;
  }
  out[blockIdx.x * T + threadIdx.x] = acc;
}

// per-CTA contiguous range, warps interleaved within the CTA's range
template <int B>
__global__ void __launch_bounds__(1024, 1) k_cta(const uint4* __restrict__ a, long nv, unsigned* out) {
  const long per = (nv / 1024 + gridDim.x - 1) / gridDim.x * 1024;
  const long v0 = blockIdx.x * per, v1 = lmin(nv, v0 + per);
  unsigned acc = 0;
  for (long b = v0 + threadIdx.x; b < v1; b += 1024 * B) {
    uint4 q[B];
#pragma unroll
    for (int u = 0; u < B; ++u) { long i = b + u * 1024; q[u] = i < v1 ? ldg_stream(a + i) : make_uint4(0, 0, 0, 0); }
#pragma unroll
    for (int u = 0; u < B; ++u) acc ^= q[u].x + q[u].w;
  }
  out[blockIdx.x * 1024 + threadIdx.x] = acc;
}

int main() {
  const long bytes = 120L << 20;
  const long nv = bytes / 16;
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  const int nsm = prop.multiProcessorCount;
  uint4* a; unsigned* out; char* fl;
  CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&out, 64 << 20)); CK(cudaMalloc(&fl, 256L << 20));
  CK(cudaMemset(a, 1, bytes));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  auto timeit = [&](const char* name, auto launch) {
    float best = 1e30f, tot = 0; const int reps = 10;
    for (int r = 0; r < reps + 2; ++r) {
      CK(cudaMemsetAsync(fl, r, 256L << 20));
      CK(cudaEventRecord(e0)); launch(); CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1)); CK(cudaGetLastError());
      float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
      if (r >= 2) { best = std::min(best, ms); tot += ms; }
    }
    printf("%-30s best %7.2f us avg %7.2f us  %7.1f GB/s (best)\n", name, best * 1e3, tot / reps * 1e3, bytes / (best * 1e-3) / 1e9);
  };
  timeit("empty launch", [&] { k_gs<1><<<nsm, 1024>>>(a, 0, out); });
  timeit("grid-stride B=1", [&] { k_gs<1><<<nsm, 1024>>>(a, nv, out); });
  timeit("grid-stride B=4", [&] { k_gs<4><<<nsm, 1024>>>(a, nv, out); });
  timeit("grid-stride B=8", [&] { k_gs<8><<<nsm, 1024>>>(a, nv, out); });
  timeit("grid-stride B=4 x2 CTAs/SM", [&] { k_gs<4><<<2 * nsm, 1024>>>(a, nv, out); });
  timeit("warp-range B=4", [&] { k_warp<4, 1024><<<nsm, 1024>>>(a, nv, out); });
  timeit("warp-range B=8", [&] { k_warp<8, 1024><<<nsm, 1024>>>(a, nv, out); });
  timeit("warp-range B=16 T=512", [&] { k_warp<16, 512><<<nsm, 512>>>(a, nv, out); });
  timeit("cta-range B=4", [&] { k_cta<4><<<nsm, 1024>>>(a, nv, out); });
  timeit("cta-range B=8", [&] { k_cta<8><<<nsm, 1024>>>(a, nv, out); });
  printf("done\n");
  return 0;
}
