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

// Pair mapping: chains 2k, 2k+1 of the 8 indices of one vector (sb includes k * 16).
__device__ __forceinline__ double2 lds128(unsigned a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
  return v;
}
template <int R>
__device__ __forceinline__ double2 gather8_pair(uint4 q, unsigned sb) {
  const double2 a0 = lds128(row_addr<R>(sb, lo16(q.x))), a1 = lds128(row_addr<R>(sb, hi16(q.x)));
  const double2 b0 = lds128(row_addr<R>(sb, lo16(q.y))), b1 = lds128(row_addr<R>(sb, hi16(q.y)));
  const double2 c0 = lds128(row_addr<R>(sb, lo16(q.z))), c1 = lds128(row_addr<R>(sb, hi16(q.z)));
  const double2 d0 = lds128(row_addr<R>(sb, lo16(q.w))), d1 = lds128(row_addr<R>(sb, hi16(q.w)));
  double2 r;
  r.x = ((a0.x + a1.x) + (b0.x + b1.x)) + ((c0.x + c1.x) + (d0.x + d1.x));
  r.y = ((a0.y + a1.y) + (b0.y + b1.y)) + ((c0.y + c1.y) + (d0.y + d1.y));
  return r;
}

// One warp walks its slice range: each slot walks one piece per slice, lane
// (slot, k) summing its chains (pair mapping: chains 2k, 2k+1; single
// mapping: chain k) over the slice's steps and emitting the sums, batches of
// U steps with all loads of a batch issued together.
#ifndef PCGS_SLICED_BATCH
#define PCGS_SLICED_BATCH 4
#endif
// Quad mapping: 4 chains of the 8 indices of one vector; the lane reads its
// two 16-byte chunks in slot-rotated order (sb0 / sb1 hold the rotation),
// sums per instruction are un-rotated by the caller.
template <int R>
__device__ __forceinline__ void gather8_quad(uint4 q, unsigned sb0, unsigned sb1, double2& s0, double2& s1) {
  s0 = gather8_pair<R>(q, sb0);
  s1 = gather8_pair<R>(q, sb1);
}

template <int R, class Epi>
__device__ __forceinline__ void walk_slices(const SPassDev& P, int wr, const double* sv, Epi& epi,
                                            int slab_len = 0) {
  constexpr int NS = sliced_slots(R), LS = sliced_lanes_per_slot(R), C = sliced_cpl(R);
  constexpr int U = PCGS_SLICED_BATCH;
  const int lane = threadIdx.x & 31, slot = lane / LS, k = lane & (LS - 1);
  const uint2 ws = __ldg(P.warp_slices + wr);
  if (ws.x >= ws.y) return;
  // chunk c of a row = chains 2c, 2c+1; lane k owns chunks [k C/2, (k+1) C/2)
  const int rot = C == 4 ? (slot & 1) : 0;
  const unsigned sb = smem_addr(sv) + (unsigned)k * (unsigned)(8 * C);
  const unsigned sb0 = sb + 16u * (unsigned)rot, sb1 = sb + 16u * (unsigned)(1 - rot);
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
    double acc = 0.0, acc2 = 0.0, acc3 = 0.0, acc4 = 0.0;
    auto step = [&](uint4 v) {
      if (PCGS_CHECKED) check_vec(v, slab_len);
      if (C == 4) {
        double2 g0, g1;
        gather8_quad<R>(v, sb0, sb1, g0, g1);
        acc += g0.x;
        acc2 += g0.y;
        acc3 += g1.x;
        acc4 += g1.y;
      } else if (C == 2) {
        const double2 g = gather8_pair<R>(v, sb);
        acc += g.x;
        acc2 += g.y;
      } else {
        acc += gather8_lane<R>(v, sb);
      }
    };
    unsigned t = 0;
    for (; t + U <= D.y; t += U) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = ldg_stream(vp + (size_t)(t + u) * NS);
#pragma unroll
      for (int u = 0; u < U; ++u) step(v[u]);
    }
    for (; t < D.y; ++t) step(ldg_stream(vp + (size_t)t * NS));
    PCGS_CHECK(pid == 0xffffffffu || (long long)pid < P.npiece);
    if (pid != 0xffffffffu) {
      if (C == 4) {  // un-rotate: instruction 0 read chunk 2k + rot
        if (rot) {
          epi.emit2(pid, 4 * k, acc3, acc4);
          epi.emit2(pid, 4 * k + 2, acc, acc2);
        } else {
          epi.emit2(pid, 4 * k, acc, acc2);
          epi.emit2(pid, 4 * k + 2, acc3, acc4);
        }
      } else if (C == 2) {
        epi.emit2(pid, 2 * k, acc, acc2);
      } else {
        epi.emit(pid, k, acc);
      }
    }
  }
}

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
  __device__ __forceinline__ void emit2(unsigned pid, int c, double s0, double s1) {
    *reinterpret_cast<double2*>(out + (size_t)pid * R + c) = make_double2(s0, s1);
  }
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
        const unsigned total = (unsigned)(((size_t)l.x + (size_t)l.y * sliced_slots(R) - f.x) * 16u);
        const unsigned off = (threadIdx.x & 31) * 128u;
        if (off < total) asm volatile("prefetch.global.L2 [%0];" ::"l"((const char*)(P.vec + f.x) + off));
      }
    }
    __syncthreads();
    fill(sv, lo, (int)(hi - lo));
    walk_slices<R>(P, T.y + warp, sv, epi, (int)(hi - lo));
  }
}

// Step phase: the pieces of the CTA's own columns [j0, jend) are contiguous
// (output-major numbering); stage them into the idle slab with coalesced
// 16-byte loads so every column sum reads shared memory.  Returns the first
// staged piece, or -1 (same in every thread) when they do not fit.
template <int R>
__device__ __forceinline__ long long stage_own_pieces(const double* pieces, const long long* out_ptr, long long j0,
                                                      long long jend, double* sv, long long cap) {
  if (j0 >= jend) return -1;
  const long long Q0 = __ldg(out_ptr + j0), Q1 = __ldg(out_ptr + jend);
  const long long len = (Q1 - Q0) * R;
  if (len > cap) return -1;
  const double2* src = reinterpret_cast<const double2*>(pieces + Q0 * R);
  double2* dst = reinterpret_cast<double2*>(sv);
  for (long long i = threadIdx.x; i < len / 2; i += kSThreads) dst[i] = __ldcg(src + i);
  __syncthreads();
  return Q0;
}

// Rounds (1 or 2; 1 if neither fits) in which the own columns' pieces are staged.
template <int R>
__device__ __forceinline__ int stage_rounds(const long long* out_ptr, long long j0, long long jend, long long cap) {
  if (j0 >= jend) return 1;
  const long long Q0 = __ldg(out_ptr + j0), Q1 = __ldg(out_ptr + jend);
  if ((Q1 - Q0) * R <= cap) return 1;
  const long long jm = j0 + (jend - j0) / 2;
  const long long Qm = __ldg(out_ptr + jm);
  return ((Qm - Q0) * R <= cap && (Q1 - Qm) * R <= cap) ? 2 : 1;
}

// debug: the stamp buffer set by pcgs_batch_debug_profile (batched kernels)
unsigned long long* batch_profile_buffer();

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

