// How long do 148 CTAs take to TMA-copy the same 177 KB vector into their
// shared memory (the PCG slab fill), plain vs cluster multicast?
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <algorithm>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int CL>
__global__ void __launch_bounds__(1024, 1) k_fill(const double* __restrict__ v, int p, int reps, double* out) {
  extern __shared__ __align__(128) double sv[];
  __shared__ unsigned long long mb;
  const unsigned bytes = (unsigned)(p * 8);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" :: "r"(su32(&mb)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (CL > 1) cg::this_cluster().sync(); else __syncthreads();
  unsigned rank = 0;
  if (CL > 1) rank = cg::this_cluster().block_rank();
  double acc = 0;
  for (int r = 0; r < reps; ++r) {
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" :: "r"(su32(&mb)), "r"(bytes));
      // this CTA's share of the slab, multicast to every CTA of the cluster
      const unsigned share = (bytes / CL + 15) / 16 * 16;
      const unsigned lo = rank * share, hi = min(bytes, lo + share);
      for (unsigned off = lo; off < hi; off += 32768) {
        const unsigned sz = min(32768u, hi - off);
        if (CL > 1) {
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;"
                       :: "r"(su32((char*)sv + off)), "l"((const char*)v + off), "r"(sz), "r"(su32(&mb)), "h"((unsigned short)((1 << CL) - 1)) : "memory");
        } else {
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       :: "r"(su32((char*)sv + off)), "l"((const char*)v + off), "r"(sz), "r"(su32(&mb)) : "memory");
        }
      }
    }
    asm volatile("{\n.reg .pred P;\nW%=:\nmbarrier.try_wait.parity.shared.b64 P, [%0], %1;\n@!P bra W%=;\n}"
                 :: "r"(su32(&mb)), "r"((unsigned)(r & 1)) : "memory");
    acc += sv[(threadIdx.x * 37 + r) % p];
    // every CTA of the cluster must be done reading before the next multicast overwrites
    if (CL > 1) cg::this_cluster().sync(); else __syncthreads();
  }
  out[blockIdx.x * 1024 + threadIdx.x] = acc;
}

int main() {
  const int p = 22176;
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  const int nsm = prop.multiProcessorCount;
  double *v, *out; CK(cudaMalloc(&v, p * 8)); CK(cudaMalloc(&out, 8L << 20));
  CK(cudaMemset(v, 0, p * 8));
  const int smem = p * 8 + 256;
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  auto run = [&](auto kern, int cl, int grid, const char* name) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    if (cl > 1) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid); cfg.blockDim = dim3(1024); cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = cl; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = cl > 1 ? 1 : 0;
    if (cl > 1) { int nc = 0; CK(cudaOccupancyMaxActiveClusters(&nc, kern, &cfg)); printf("  %s: max active clusters %d (grid needs %d)\n", name, nc, grid / cl); }
    for (int reps : {1, 101}) {
      float best = 1e9;
      for (int t = 0; t < 5; ++t) {
        CK(cudaEventRecord(e0));
        CK(cudaLaunchKernelEx(&cfg, kern, (const double*)v, p, reps, out));
        CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaGetLastError());
        float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); best = std::min(best, ms);
      }
      if (reps == 1) printf("%-22s 1 fill: %.2f us", name, best * 1e3);
      else printf("   per extra fill: %.2f us\n", 0.0);
      static float one; if (reps == 1) one = best; else printf("\r%-22s 1 fill %.2f us, per fill (101 reps) %.2f us\n", name, one * 1e3, (best - one) / 100 * 1e3);
    }
  };
  run(k_fill<1>, 1, nsm, "plain 148 CTAs");
  run(k_fill<2>, 2, nsm, "multicast cluster 2");
  run(k_fill<4>, 4, 144, "multicast cluster 4");
  run(k_fill<1>, 1, 144, "plain 144 CTAs");
  printf("done\n");
  return 0;
}
