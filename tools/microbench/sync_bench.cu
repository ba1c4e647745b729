// grid-wide barrier cost on B200: cooperative-groups grid.sync vs a hand barrier
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void k_cg(int iters, double* out) {
  cg::grid_group g = cg::this_grid();
  double acc = 0;
  for (int i = 0; i < iters; ++i) { acc += i; g.sync(); }
  if (threadIdx.x == 0) out[blockIdx.x] = acc;
}

__device__ unsigned int g_count = 0;
__device__ volatile unsigned int g_gen = 0;
__device__ __forceinline__ void hand_sync(unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned gen = g_gen;
    __threadfence();
    if (atomicAdd(&g_count, 1) == nblocks - 1) { g_count = 0; __threadfence(); g_gen = gen + 1; }
    else { while (g_gen == gen) { } }
    __threadfence();
  }
  __syncthreads();
}
__global__ void k_hand(int iters, double* out) {
  double acc = 0;
  for (int i = 0; i < iters; ++i) { acc += i; hand_sync(gridDim.x); }
  if (threadIdx.x == 0) out[blockIdx.x] = acc;
}

int main() {
  double* d; CK(cudaMalloc(&d, 4096 * 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int threads : {256, 512, 1024}) {
    int iters = 2000;
    void* args[] = {&iters, &d};
    CK(cudaLaunchCooperativeKernel((void*)k_cg, 148, threads, args, 0, 0));
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    CK(cudaLaunchCooperativeKernel((void*)k_cg, 148, threads, args, 0, 0));
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("cg grid.sync  threads %4d: %.3f us/sync\n", threads, ms * 1e3 / iters);
    cudaEventRecord(e0);
    CK(cudaLaunchCooperativeKernel((void*)k_hand, 148, threads, args, 0, 0));
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("hand barrier  threads %4d: %.3f us/sync\n", threads, ms * 1e3 / iters);
  }
  return 0;
}
