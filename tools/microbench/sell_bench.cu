// Microbenchmark: lane-owned pieces ("sliced" layout) for the CSR pass.
// Each warp streams slices of 32 pieces (one per lane, K consecutive lanes per
// row), accumulates per lane with no segmented reduction, and combines the K
// lanes of a row with K-1 shuffles at the end of the slice.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <numeric>
#include <random>
#include <array>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ void fill_slab(double* sv, const double* v, int p, unsigned long long* mb) {
  unsigned bytes = ((p * 8 + 15) / 16) * 16;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" :: "r"(su32(mb)));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" :: "r"(su32(mb)), "r"(bytes));
    for (unsigned off = 0; off < bytes; off += 32768) {
      unsigned sz = bytes - off < 32768 ? bytes - off : 32768;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   :: "r"(su32((char*)sv + off)), "l"((const char*)v + off), "r"(sz), "r"(su32(mb)) : "memory");
    }
  }
  if (threadIdx.x == 32) sv[p] = 0.0;
  __syncthreads();
  asm volatile("{\n.reg .pred P;\nW%=:\n"
               "mbarrier.try_wait.parity.shared.b64 P, [%0], 0;\n"
               "@!P bra W%=;\n}" :: "r"(su32(mb)) : "memory");
}

__device__ __forceinline__ double gather8(uint4 q, const double* sv) {
  const unsigned w[4] = {q.x, q.y, q.z, q.w};
  double a = 0, b = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) { a += sv[w[k] & 0xffff]; b += sv[w[k] >> 16]; }
  return a + b;
}

// slices: {vec offset, steps}; out id per (slice, lane) = row for lanes with lane % K == 0
template <int K, int B, bool GATHER>
__global__ void __launch_bounds__(1024, 1) k_sell(const uint4* __restrict__ vec, const uint2* __restrict__ slices,
                                                   const int* __restrict__ rows, const int* __restrict__ warp_ptr,
                                                   const double* __restrict__ v, int p, double* __restrict__ out) {
  extern __shared__ __align__(128) double sv[];
  __shared__ unsigned long long mb;
  fill_slab(sv, v, p, &mb);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int w = blockIdx.x * 32 + warp;
  for (int s = warp_ptr[w]; s < warp_ptr[w + 1]; ++s) {
    const uint2 S = __ldg(slices + s);
    const uint4* base = vec + S.x + lane;
    const int T = (int)S.y;
    double acc = 0;
    int t = 0;
    for (; t + B <= T; t += B) {
      uint4 q[B];
#pragma unroll
      for (int u = 0; u < B; ++u) q[u] = ldg_stream(base + (t + u) * 32);
#pragma unroll
      for (int u = 0; u < B; ++u) acc += GATHER ? gather8(q[u], sv) : (double)(q[u].x ^ q[u].w);
    }
    for (; t < T; ++t) { uint4 q = ldg_stream(base + t * 32); acc += GATHER ? gather8(q, sv) : (double)(q.x ^ q.w); }
#pragma unroll
    for (int o = 1; o < K; o <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane % K == 0) { const int r = __ldg(rows + s * 32 + lane); if (r >= 0) out[r] = acc; }
  }
}

int main(int argc, char** argv) {
  const int n = 72489, p = 22176;
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  const int nsm = prop.multiProcessorCount, nw = nsm * 32;
  std::mt19937_64 g(7);
  std::vector<std::vector<uint16_t>> rowidx(n);
  long nnz = 0;
  for (int r = 0; r < n; ++r) {
    int len = 780 + (int)(g() % 95);
    rowidx[r].resize(len);
    for (auto& x : rowidx[r]) x = (uint16_t)(g() % p);
    nnz += len;
  }
  std::vector<double> hv(p);
  for (int i = 0; i < p; ++i) hv[i] = (double)(i % 97) * 0.5;
  std::vector<double> ref(n);
  for (int r = 0; r < n; ++r) { double s = 0; for (auto x : rowidx[r]) s += hv[x]; ref[r] = s; }
  double *d_v, *d_out; CK(cudaMalloc(&d_v, p * 8)); CK(cudaMalloc(&d_out, n * 8));
  CK(cudaMemcpy(d_v, hv.data(), p * 8, cudaMemcpyHostToDevice));
  char* d_flush; size_t flushsz = 256L << 20; CK(cudaMalloc(&d_flush, flushsz));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  const int slab = ((p * 8 + 16 + 127) / 128) * 128;

  auto run = [&](int K, bool balance, auto kern, const char* name) {
    // pieces: row r split into K near-equal parts; slices of 32/K rows sorted by length
    std::vector<int> order(n);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return rowidx[a].size() > rowidx[b].size(); });
    const int rps = 32 / K;
    const int nsl = (n + rps - 1) / rps;
    std::vector<uint2> slices(nsl);
    std::vector<int> rows((size_t)nsl * 32, -1);
    std::vector<uint16_t> idx;
    long extra = 0, groups = 0;
    for (int s = 0; s < nsl; ++s) {
      int maxlen = 0;
      for (int q = 0; q < rps && s * rps + q < n; ++q) maxlen = std::max<int>(maxlen, rowidx[order[s * rps + q]].size());
      const int T = ((maxlen + K - 1) / K + 7) / 8;  // steps
      slices[s] = make_uint2((unsigned)(idx.size() / 8), (unsigned)T);
      size_t base = idx.size();
      idx.resize(base + (size_t)T * 32 * 8, (uint16_t)p);
      // per-lane pools
      std::vector<std::array<std::vector<uint16_t>, 16>> pool(32);
      for (int l = 0; l < 32; ++l) {
        const int q = l / K, part = l % K;
        if (s * rps + q >= n) continue;
        const int r = order[s * rps + q];
        if (part == 0) rows[(size_t)s * 32 + l] = r;
        const auto& ri = rowidx[r];
        const size_t a = ri.size() * part / K, b = ri.size() * (part + 1) / K;
        for (size_t i = a; i < b; ++i) pool[l][ri[i] & 15].push_back(ri[i]);
      }
      for (int t = 0; t < T; ++t)
        for (int slot = 0; slot < 8; ++slot)
          for (int h = 0; h < 2; ++h) {
            int mult[16] = {};
            int worst = 0;
            bool pad = false;
            for (int l = h * 16; l < h * 16 + 16; ++l) {
              auto& P = pool[l];
              int best = -1;
              for (int k = 0; k < 16; ++k) {
                if (P[k].empty()) continue;
                if (!balance) { best = k; break; }
                if (best < 0 || mult[k] < mult[best] || (mult[k] == mult[best] && P[k].size() > P[best].size())) best = k;
              }
              if (best < 0) { if (!pad) { pad = true; worst = std::max(worst, ++mult[p & 15]); } continue; }
              const uint16_t x = P[best].back(); P[best].pop_back();
              worst = std::max(worst, ++mult[x & 15]);
              idx[base + ((size_t)t * 32 + l) * 8 + slot] = x;
            }
            extra += worst - 1; groups++;
          }
    }
    // warps: contiguous slice ranges balanced by steps
    std::vector<long> pre(nsl + 1, 0);
    for (int s = 0; s < nsl; ++s) pre[s + 1] = pre[s] + slices[s].y;
    std::vector<int> wp(nw + 1, 0);
    for (int w = 0; w <= nw; ++w) {
      long target = pre[nsl] * w / nw;
      wp[w] = (int)(std::lower_bound(pre.begin(), pre.end(), target) - pre.begin());
    }
    wp[nw] = nsl;
    uint4* d_vec; uint2* d_sl; int *d_rows, *d_wp;
    CK(cudaMalloc(&d_vec, idx.size() * 2)); CK(cudaMalloc(&d_sl, nsl * 8));
    CK(cudaMalloc(&d_rows, rows.size() * 4)); CK(cudaMalloc(&d_wp, (nw + 1) * 4));
    CK(cudaMemcpy(d_vec, idx.data(), idx.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_sl, slices.data(), nsl * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_rows, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_wp, wp.data(), (nw + 1) * 4, cudaMemcpyHostToDevice));
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, slab));
    float best = 1e30f, tot = 0; const int reps = 10;
    for (int r = 0; r < reps + 2; ++r) {
      CK(cudaMemsetAsync(d_flush, r, flushsz));
      CK(cudaEventRecord(e0));
      kern<<<nsm, 1024, slab>>>(d_vec, d_sl, d_rows, d_wp, d_v, p, d_out);
      CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaGetLastError());
      float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
      if (r >= 2) { best = std::min(best, ms); tot += ms; }
    }
    std::vector<double> ho(n);
    CK(cudaMemcpy(ho.data(), d_out, n * 8, cudaMemcpyDeviceToHost));
    double err = 0;
    for (int r = 0; r < n; ++r) err = std::max(err, std::abs(ho[r] - ref[r]));
    printf("%-30s K=%d best %7.2f us avg %7.2f us  bytes %.1f MB  pad %.2f%%  extra-wavefront %.3f  maxerr %.2e\n", name, K,
           best * 1e3, tot / reps * 1e3, idx.size() * 2 / 1e6, 100.0 * (idx.size() - nnz) / nnz, (double)extra / groups, err);
    cudaFree(d_vec); cudaFree(d_sl); cudaFree(d_rows); cudaFree(d_wp);
  };
  run(1, true, k_sell<1, 4, true>, "sell B=4 balanced");
  run(2, true, k_sell<2, 4, true>, "sell B=4 balanced");
  run(4, true, k_sell<4, 4, true>, "sell B=4 balanced");
  run(2, false, k_sell<2, 4, true>, "sell B=4 unbalanced");
  run(2, true, k_sell<2, 2, true>, "sell B=2 balanced");
  run(2, true, k_sell<2, 6, true>, "sell B=6 balanced");
  run(2, true, k_sell<2, 4, false>, "sell B=4 stream only");
  run(4, true, k_sell<4, 4, false>, "sell B=4 stream only");
  printf("done\n");
  return 0;
}
