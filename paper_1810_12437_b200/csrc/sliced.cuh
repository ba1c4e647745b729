// Device side of the sliced store (batched chains): the handle, the
// streaming walk over slices, fills and reductions shared by the batched PCG
// (sliced.cu) and the fused batched Gibbs kernel (sgibbs.cu).  See sliced.h.
#pragma once
#include <cuda_runtime.h>

#include <vector>

#include "internal.cuh"
#include "sliced.h"

struct SPassDev {
  const uint4* vec;
  const uint2* slices;       // {v0, len}
  const unsigned* piece;     // 32/R per slice
  const uint2* warp_slices;  // [s0, s1) per warp range
  const int2* task;          // {slab, first warp range}
  const int* cta_task_ptr;
  const long long* slab_lo;
  const long long* out_ptr;  // pieces of output j: [out_ptr[j], out_ptr[j+1])
  int nslab;
  long long npiece;
};

struct BatchDev {
  long long n, p, pt;
  int icpt;
  int G;
  int R;
  int smem_doubles;  // slab + sentinel row, in doubles
  SPassDev csr, csc;
};

struct pcgs_batch {
  BatchDev dev;
  int device;
  int64_t info[16];
  std::vector<void*> allocs;
};

// ------------------------------------------------------------------ streaming
// sliding L2 prefetch distance ahead of the loads, bytes of the warp's stream
static constexpr unsigned kSPrefetch = 4096;

static __device__ __forceinline__ unsigned long long stimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <int R>
__device__ __forceinline__ unsigned row_addr(unsigned sb, unsigned idx) {
  return sb + idx * (unsigned)(8 * R);
}

// Sum over the 8 indices of one vector, chain c (sb already includes c * 8).
template <int R>
__device__ __forceinline__ double gather8_lane(uint4 q, unsigned sb) {
  const double a = lds64(row_addr<R>(sb, lo16(q.x))) + lds64(row_addr<R>(sb, hi16(q.x)));
  const double b = lds64(row_addr<R>(sb, lo16(q.y))) + lds64(row_addr<R>(sb, hi16(q.y)));
  const double c = lds64(row_addr<R>(sb, lo16(q.z))) + lds64(row_addr<R>(sb, hi16(q.z)));
  const double d = lds64(row_addr<R>(sb, lo16(q.w))) + lds64(row_addr<R>(sb, hi16(q.w)));
  return (a + b) + (c + d);
}

// One warp walks its slice range: lane (slot, c) sums chain c of its slot's
// piece over the slice's steps and emits it.  The warp's slices are
// contiguous in the stream, so the walk is one flat run of steps (slot s of
// step g at vector first + g * NS + s) with slice boundaries every L steps:
// the index loads of the next batch are issued before the current batch is
// consumed (software pipelining across slice boundaries), and the next
// slice's descriptor is loaded one slice ahead.
#ifndef PCGS_SLICED_BATCH
#define PCGS_SLICED_BATCH 4
#endif
#ifndef PCGS_SLICED_PIPE
#define PCGS_SLICED_PIPE 0
#endif
#if !PCGS_SLICED_PIPE
// per-slice batches of U steps, loads of a batch issued together
template <int R, class Epi>
__device__ __forceinline__ void walk_slices(const SPassDev& P, int wr, const double* sv, Epi& epi,
                                            int slab_len = 0) {
  constexpr int NS = 32 / R;
  constexpr int U = PCGS_SLICED_BATCH;
  const int lane = threadIdx.x & 31, slot = lane / R, c = lane & (R - 1);
  const uint2 ws = __ldg(P.warp_slices + wr);
  if (ws.x >= ws.y) return;
  const unsigned sb = smem_addr(sv) + (unsigned)c * 8u;
  const uint2 first = __ldg(P.slices + ws.x), last = __ldg(P.slices + ws.y - 1);
  const char* stream0 = (const char*)(P.vec + first.x);
  const unsigned total = (unsigned)(((size_t)last.x + (size_t)last.y * NS - first.x) * 16u);
  unsigned next_pf = kSPrefetch;
  for (unsigned q = ws.x; q < ws.y; ++q) {
    const uint2 D = __ldg(P.slices + q);
    const unsigned pid = __ldg(P.piece + (size_t)q * NS + slot);
    const uint4* vp = P.vec + D.x + slot;
    {
      const unsigned end = min(total, (unsigned)((const char*)(P.vec + D.x + (size_t)D.y * NS) - stream0) + kSPrefetch);
      for (; next_pf < end; next_pf += 32u * 128u) {
        const unsigned off = next_pf + (unsigned)lane * 128u;
        if (off < end) asm volatile("prefetch.global.L2 [%0];" ::"l"(stream0 + off));
      }
    }
    double acc = 0.0;
    unsigned t = 0;
    for (; t + U <= D.y; t += U) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = ldg_stream(vp + (size_t)(t + u) * NS);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (PCGS_CHECKED) check_vec(v[u], slab_len);
        acc += gather8_lane<R>(v[u], sb);
      }
    }
    for (; t < D.y; ++t) {
      const uint4 v = ldg_stream(vp + (size_t)t * NS);
      if (PCGS_CHECKED) check_vec(v, slab_len);
      acc += gather8_lane<R>(v, sb);
    }
    PCGS_CHECK(pid == 0xffffffffu || (long long)pid < P.npiece);
    if (pid != 0xffffffffu) epi.emit(pid, c, acc);
  }
}
#else
template <int R, class Epi>
__device__ __noinline__ void walk_slices(const SPassDev& P, int wr, const double* sv, Epi& epi, int slab_len = 0) {
  constexpr int NS = 32 / R;
  constexpr int U = PCGS_SLICED_BATCH;
  const int lane = threadIdx.x & 31, slot = lane / R, c = lane & (R - 1);
  const uint2 ws = __ldg(P.warp_slices + wr);
  if (ws.x >= ws.y) return;
  const unsigned sb = smem_addr(sv) + (unsigned)c * 8u;
  const uint2 first = __ldg(P.slices + ws.x), last = __ldg(P.slices + ws.y - 1);
  const char* stream0 = (const char*)(P.vec + first.x);
  const unsigned T = (unsigned)(((size_t)last.x - first.x) / NS + last.y);  // steps of the warp
  const unsigned total = T * NS * 16u;                                      // bytes of the warp stream
  const uint4* base = P.vec + first.x + slot;
  unsigned q = ws.x;
  unsigned bnd = first.y;  // step at which slice q ends
  unsigned pid = __ldg(P.piece + (size_t)q * NS + slot);
  uint2 nD = q + 1 < ws.y ? __ldg(P.slices + q + 1) : make_uint2(0u, 0u);
  unsigned npid = q + 1 < ws.y ? __ldg(P.piece + (size_t)(q + 1) * NS + slot) : 0xffffffffu;
  unsigned next_pf = kSPrefetch;  // bytes of the warp stream prefetched so far
  double acc = 0.0;
  uint4 cur[U];
#pragma unroll
  for (int u = 0; u < U; ++u)
    if ((unsigned)u < T) cur[u] = ldg_stream(base + (size_t)u * NS);
  for (unsigned g0 = 0; g0 < T; g0 += U) {
    // sliding L2 prefetch kSPrefetch bytes ahead of the loads
    {
      const unsigned end = min(total, (g0 + 2 * U) * NS * 16u + kSPrefetch);
      if (next_pf < end) {
        const unsigned off = next_pf + (unsigned)lane * 128u;
        if (off < end) asm volatile("prefetch.global.L2 [%0];" ::"l"(stream0 + off));
        next_pf += 32u * 128u;
      }
    }
    uint4 nxt[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (g0 + U + u < T) nxt[u] = ldg_stream(base + (size_t)(g0 + U + u) * NS);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const unsigned g = g0 + u;
      if (g < T) {
        if (g == bnd) {  // slice q done: emit, advance to q + 1 (pieces are never empty)
          if (pid != 0xffffffffu) epi.emit(pid, c, acc);
          acc = 0.0;
          ++q;
          bnd += nD.y;
          pid = npid;
          if (q + 1 < ws.y) {
            nD = __ldg(P.slices + q + 1);
            npid = __ldg(P.piece + (size_t)(q + 1) * NS + slot);
          }
        }
        acc += gather8_lane<R>(cur[u], sb);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) cur[u] = nxt[u];
  }
  if (pid != 0xffffffffu) epi.emit(pid, c, acc);
}
#endif

// TMA copy of elements [lo, lo+len) of a chain-minor R-column vector into the
// slab; the sentinel row (R doubles at element len) is zeroed.
template <int R>
struct FillRows {
  const double* src;
  BulkFill* bf;
  __device__ void operator()(double* sv, long long lo, int len) {
    if (threadIdx.x > 0 && threadIdx.x < R) sv[(long long)len * R + threadIdx.x] = 0.0;
    bulk_fill(*bf, sv, src + lo * R, len * R);  // zeroes sv[len * R] and ends with a barrier
  }
};

struct EpiPiece {  // out[piece * R + c] = s
  double* out;
  int R;
  __device__ __forceinline__ void emit(unsigned pid, int c, double s) { out[(size_t)pid * R + c] = s; }
};

template <int R, class Fill, class Epi>
__device__ __forceinline__ void run_spass(const SPassDev& P, double* sv, Fill& fill, Epi& epi) {
  const int c = blockIdx.x;
  const int t0 = P.cta_task_ptr[c], t1 = P.cta_task_ptr[c + 1];
  const int warp = threadIdx.x >> 5;
  for (int t = t0; t < t1; ++t) {
    const int2 T = __ldg(P.task + t);
    const long long lo = P.slab_lo[T.x], hi = P.slab_lo[T.x + 1];
    // first stretch of the warp's stream into L2 while the slab is filled
    {
      const uint2 ws = __ldg(P.warp_slices + T.y + warp);
      if (ws.x < ws.y) {
        const uint2 f = __ldg(P.slices + ws.x), l = __ldg(P.slices + ws.y - 1);
        const unsigned total = (unsigned)(((size_t)l.x + (size_t)l.y * (32 / R) - f.x) * 16u);
        const unsigned off = (threadIdx.x & 31) * 128u;
        if (off < total) asm volatile("prefetch.global.L2 [%0];" ::"l"((const char*)(P.vec + f.x) + off));
      }
    }
    __syncthreads();
    fill(sv, lo, (int)(hi - lo));
    walk_slices<R>(P, T.y + warp, sv, epi, (int)(hi - lo));
  }
}

// debug: the stamp buffer set by pcgs_batch_debug_profile (batched kernels)
unsigned long long* batch_profile_buffer();

// run_spass with the walk out of line: inside a persistent kernel with much
// live state (the fused Gibbs kernel) the caller's registers are saved once per
// pass and the streaming loop keeps the whole register budget.
template <int R, class Epi>
__device__ __noinline__ void walk_slices_ni(const SPassDev& P, int wr, const double* sv, Epi& epi, int slab_len) {
  walk_slices<R>(P, wr, sv, epi, slab_len);
}
template <int R, class Fill, class Epi>
__device__ __forceinline__ void run_spass_ni(const SPassDev& P, double* sv, Fill& fill, Epi& epi) {
  const int c = blockIdx.x;
  const int t0 = P.cta_task_ptr[c], t1 = P.cta_task_ptr[c + 1];
  const int warp = threadIdx.x >> 5;
  for (int t = t0; t < t1; ++t) {
    const int2 T = __ldg(P.task + t);
    const long long lo = P.slab_lo[T.x], hi = P.slab_lo[T.x + 1];
    {
      const uint2 ws = __ldg(P.warp_slices + T.y + warp);
      if (ws.x < ws.y) {
        const uint2 f = __ldg(P.slices + ws.x), l = __ldg(P.slices + ws.y - 1);
        const unsigned total = (unsigned)(((size_t)l.x + (size_t)l.y * (32 / R) - f.x) * 16u);
        const unsigned off = (threadIdx.x & 31) * 128u;
        if (off < total) asm volatile("prefetch.global.L2 [%0];" ::"l"((const char*)(P.vec + f.x) + off));
      }
    }
    __syncthreads();
    fill(sv, lo, (int)(hi - lo));
    walk_slices_ni<R>(P, T.y + warp, sv, epi, (int)(hi - lo));
  }
}

// Per-chain block sums: thread holds a value of chain (tid & (R-1)); returns,
// in threads c < R, the CTA total of chain c (fixed order).
template <int R>
__device__ __forceinline__ double block_sum_chain(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o >= R; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane < R) red[warp * R + lane] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x < R)
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w * R + threadIdx.x];
  return s;
}

// Grid totals of partial slots [k0, k0 + m) (m <= 32): warp k sums slot k0 + k
// over the CTAs (lane-strided, then a fixed tree), the result lands in
// out[k0 + k]; every CTA computes the same numbers in the same order.
static __device__ __forceinline__ void reduce_parts(const double* part, int PS, int k0, int m, double* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (warp < m) {
    double s = 0.0;
    for (int q = lane; q < (int)gridDim.x; q += 32) s += __ldcg(part + (long long)q * PS + k0 + warp);
    s = warp_sum(s);
    if (lane == 0) out[k0 + warp] = s;
  }
  __syncthreads();
}

