// Batched (multi-chain) pattern-only passes: R independent chains share one
// walk over the index stream (SpMM with R right-hand sides, BASELINE config 4).
// Vectors are chain-minor (v[j * R + c]), so a slab of R vectors is one
// contiguous block that the TMA engine copies into shared memory, and one
// index gathers R doubles with R/2 LDS.128.
#pragma once
#include "device.cuh"

namespace pcgs {

constexpr int kRingB = 2;  // blocks per load batch (R doubles of state per block)

template <int R>
__device__ __forceinline__ void gather8_b(uint4 q, const double* sv, double (&s)[R]) {
  const unsigned w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
  for (int c = 0; c < R; ++c) s[c] = 0.0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const double* pa = sv + (size_t)(w[k] & 0xffffu) * R;
    const double* pb = sv + (size_t)(w[k] >> 16) * R;
#pragma unroll
    for (int c = 0; c < R; c += 2) {
      const double2 xa = *reinterpret_cast<const double2*>(pa + c);
      const double2 xb = *reinterpret_cast<const double2*>(pb + c);
      s[c] += xa.x + xb.x;
      s[c + 1] += xa.y + xb.y;
    }
  }
}

template <int R, class Epi>
__device__ __forceinline__ void block_reduce_b(uint2 dsc, const double (&s)[R], int lane, double (&acc)[R],
                                               unsigned& open_id, bool& have_open, Epi& epi) {
  const unsigned M = dsc.y;
  if (M == 0u) {
#pragma unroll
    for (int c = 0; c < R; ++c) acc[c] += s[c];
    return;
  }
  const int f = __ffs(M) - 1;
  const int Lh = 31 - __clz(M);
  {
    double t[R];
#pragma unroll
    for (int c = 0; c < R; ++c) t[c] = warp_sum(acc[c] + (lane < f ? s[c] : 0.0));
    if (have_open && lane == 0) epi.emit((long long)open_id, t);
  }
  if (f != Lh) {
    double x[R];
#pragma unroll
    for (int c = 0; c < R; ++c) x[c] = (lane >= f && lane < Lh) ? s[c] : 0.0;
    const unsigned le = lane == 31 ? 0xffffffffu : ((2u << lane) - 1u);
    const unsigned after = M & ~le;
    const int end = after ? (__ffs(after) - 2) : 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
      for (int c = 0; c < R; ++c) {
        const double t = __shfl_down_sync(0xffffffffu, x[c], o);
        if (lane + o <= end) x[c] += t;
      }
    }
    if (((M >> lane) & 1u) && lane < Lh) epi.emit((long long)(dsc.x + __popc(M & (le >> 1))), x);
  }
#pragma unroll
  for (int c = 0; c < R; ++c) acc[c] = lane >= Lh ? s[c] : 0.0;
  open_id = dsc.x + __popc(M) - 1;
  have_open = true;
}

template <int R, class Epi>
__device__ __forceinline__ void process_warp_b(const PassDev& P, int warp0, const double* sv, Epi& epi) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint4 Rg = __ldg(P.warps + warp0 + warp);
  const int nvec = (int)Rg.y;
  if (nvec == 0) return;
  const int nb = (nvec + 31) >> 5;
  const uint4* base = P.vec + Rg.x;
  const uint2* bd = P.blocks + Rg.z;
  double acc[R];
#pragma unroll
  for (int c = 0; c < R; ++c) acc[c] = 0.0;
  unsigned open_id = 0;
  bool have_open = false;
  for (int k0 = 0; k0 < nb; k0 += kRingB) {
    uint4 q[kRingB];
    const uint2 dl = lane < kRingB && k0 + lane < nb ? __ldg(bd + k0 + lane) : make_uint2(0u, 0u);
#pragma unroll
    for (int u = 0; u < kRingB; ++u) {
      const int v = (k0 + u) * 32 + lane;
      if (v < nvec) q[u] = ldg_stream(base + v);
    }
#pragma unroll
    for (int u = 0; u < kRingB; ++u) {
      const int k = k0 + u;
      if (k < nb) {
        uint2 dsc;
        dsc.x = __shfl_sync(0xffffffffu, dl.x, u);
        dsc.y = __shfl_sync(0xffffffffu, dl.y, u);
        double s[R];
        if (k * 32 + lane < nvec) {
          gather8_b<R>(q[u], sv, s);
        } else {
#pragma unroll
          for (int c = 0; c < R; ++c) s[c] = 0.0;
        }
        block_reduce_b<R>(dsc, s, lane, acc, open_id, have_open, epi);
      }
    }
  }
  double t[R];
#pragma unroll
  for (int c = 0; c < R; ++c) t[c] = warp_sum(acc[c]);
  if (have_open && lane == 0) epi.emit((long long)open_id, t);
}

template <int R, class Fill, class Epi>
__device__ __forceinline__ void run_pass_b(const PassDev& P, double* sv, Fill& fill, Epi& epi) {
  const int c = blockIdx.x;
  const int t0 = P.cta_task_ptr[c], t1 = P.cta_task_ptr[c + 1];
  for (int t = t0; t < t1; ++t) {
    const int2 T = __ldg(P.task + t);
    const long long lo = P.slab_lo[T.x], hi = P.slab_lo[T.x + 1];
    prefetch_warp(P, T.y, 0);
    __syncthreads();
    fill(sv, lo, (int)(hi - lo));
    process_warp_b<R>(P, T.y, sv, epi);
  }
}

// TMA copy of rows [lo, lo+len) of a chain-minor R-column buffer; zero sentinel row
template <int R>
struct FillBulkB {
  const double* src;
  BulkFill* bf;
  __device__ void operator()(double* sv, long long lo, int len) {
    bulk_fill(*bf, sv, src + lo * R, len * R);  // also zeroes sv[len * R]
    if (threadIdx.x > 0 && threadIdx.x < R) sv[(long long)len * R + threadIdx.x] = 0.0;
    __syncthreads();
  }
};

}  // namespace pcgs
