// Which lane groups must hit distinct bank pairs for a conflict-free LDS.64?
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <algorithm>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void k(const int* __restrict__ idx, int iters, double* out) {
  __shared__ double sv[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sv[i] = i * 0.5;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  int a = idx[lane];
  double acc = 0;
  for (int it = 0; it < iters; ++it) {
    acc += sv[a];
    a = (a + 1024) & 4095;   // keep the bank pattern, defeat CSE
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  std::mt19937 g(3);
  auto layout = [&](int kind) {
    std::vector<int> v(32);
    std::vector<int> perm(16);
    for (int i = 0; i < 16; ++i) perm[i] = i;
    for (int l = 0; l < 32; ++l) {
      int pair;
      switch (kind) {
        case 0: pair = l % 16; break;                         // consecutive doubles
        case 1: { if (l % 16 == 0) std::shuffle(perm.begin(), perm.end(), g); pair = perm[l % 16]; break; }  // distinct per half
        case 2: pair = (l / 2) % 16; break;                   // lanes 2i, 2i+1 same pair (different rows)
        case 3: pair = g() % 16; break;                       // random
        case 4: { if (l % 8 == 0) std::shuffle(perm.begin(), perm.end(), g); pair = perm[l % 8]; break; } // distinct per quarter only
        case 5: pair = (l < 16) ? l : (l - 16 + 8) % 16; break;  // distinct per half, halves overlap shifted
        case 6: { pair = (l & 1) ? 8 + (l / 2) % 8 : (l / 2) % 8; break; }  // even lanes pairs 0-7, odd lanes 8-15
        case 7: pair = (l == 1) ? 0 : l % 16; break;           // one duplicate, half 0 only
        case 8: pair = (l % 16) / 2; break;                    // 8 pairs x 2 lanes in each half
        case 9: pair = (l % 16 == 1) ? 0 : l % 16; break;      // one duplicate in each half
        case 10: pair = (l == 1 || l == 2) ? 0 : l % 16; break; // one 3-way, half 0 only
        default: pair = 0;
      }
      int row = 1 + (g() % 200);            // different address in the same pair -> conflict candidate
      v[l] = row * 16 + pair;
    }
    return v;
  };
  int* d_idx; double* d_out;
  CK(cudaMalloc(&d_idx, 32 * sizeof(int)));
  CK(cudaMalloc(&d_out, 1 << 20));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[] = {"consecutive", "distinct-per-half", "lane-pairs-share", "random", "distinct-per-quarter",
                         "halves-shifted", "even/odd-split", "one-dup-half0", "doubled-8x2", "one-dup-each-half", "3way-half0"};
  for (int kind = 0; kind < 11; ++kind) {
    std::vector<int> v = layout(kind);
    CK(cudaMemcpy(d_idx, v.data(), 32 * sizeof(int), cudaMemcpyHostToDevice));
    const int iters = 20000;
    k<<<148, 32>>>(d_idx, iters, d_out);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    k<<<148, 32>>>(d_idx, iters, d_out);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-22s %.3f ns/LDS.64 (single warp per SM, dependent chain)\n", names[kind], ms * 1e6 / iters);
  }
  return 0;
}
