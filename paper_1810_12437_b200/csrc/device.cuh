// Device building blocks shared by every pcgs kernel.
#pragma once
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "store.h"

namespace pcgs {

struct PassDev {
  const uint4* vec;          // uint16 index vectors (8 per uint4)
  const int4* bundle;        // Bundle {vec_off, seg0, mask, nvec|long}
  const int4* task;          // Task {slab, b0, b1, split}
  const int* cta_task_ptr;   // G+1
  const int* warp_split;     // kWarps+1 per task
  const long long* slab_lo;  // nslab+1
  const int* piece_ptr;      // CSC: nslab*(p_total+1)
  int nslab;
  long long nseg;
};

struct DesignDev {
  long long n, p, pt;  // rows, shrunk columns, p + intercept
  int icpt;
  int G;               // CTAs the static plan was built for
  int smem_doubles;    // dynamic shared memory per CTA, in doubles
  PassDev csr, csc;
};

// ------------------------------------------------------------------ utilities
__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic CTA sum; the result is valid in every thread.
__device__ __forceinline__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double r = (lane < (int)(blockDim.x >> 5)) ? red[lane] : 0.0;
  r = warp_sum(r);
  return r;
}

// Two sums at once (one barrier pair).
__device__ __forceinline__ void block_sum2(double& a, double& b, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  a = warp_sum(a);
  b = warp_sum(b);
  __syncthreads();
  if (lane == 0) { red[warp] = a; red[32 + warp] = b; }
  __syncthreads();
  const int nw = blockDim.x >> 5;
  double ra = lane < nw ? red[lane] : 0.0, rb = lane < nw ? red[32 + lane] : 0.0;
  a = warp_sum(ra);
  b = warp_sum(rb);
}

// Every CTA reduces the same G partials in the same order (bitwise identical).
__device__ __forceinline__ double reduce_partials(const double* part, int G) {
  const int lane = threadIdx.x & 31;
  double s = 0.0;
  for (int q = lane; q < G; q += 32) s += __ldcg(part + q);
  return warp_sum(s);
}

__device__ __forceinline__ double gather8(uint4 q, const double* sv) {
  double a = sv[q.x & 0xffffu] + sv[q.x >> 16];
  double b = sv[q.y & 0xffffu] + sv[q.y >> 16];
  double c = sv[q.z & 0xffffu] + sv[q.z >> 16];
  double d = sv[q.w & 0xffffu] + sv[q.w >> 16];
  return (a + b) + (c + d);
}

// ------------------------------------------------------------------ fills
// sv[j] = f(j) for j in [0, len); sv[len] = 0 (the segment sentinel).  Loads are
// batched 16 per thread so the fill is one or two L2 round trips.
template <class F>
__device__ __forceinline__ void fill_smem(double* sv, int len, F& f) {
  constexpr int U = 8;
  for (int j0 = threadIdx.x; j0 < len; j0 += kThreads * U) {
    double vals[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      int j = j0 + u * kThreads;
      vals[u] = j < len ? f(j) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      int j = j0 + u * kThreads;
      if (j < len) sv[j] = vals[u];
    }
  }
  if (threadIdx.x == 0) sv[len] = 0.0;
  __syncthreads();
}

// ------------------------------------------------------------------ passes
template <class Epi>
__device__ __forceinline__ void seg_emit(int4 D, double s, int lane, Epi& epi) {
  const unsigned mask = (unsigned)D.z;
  const int nv = D.w;
  const unsigned le = lane == 31 ? 0xffffffffu : ((2u << lane) - 1u);
  const int rank = __popc(mask & le) - 1;
  const unsigned after = mask & ~le;
  int end = after ? (__ffs(after) - 2) : (nv - 1);
  if (lane >= nv) end = lane;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    double t = __shfl_down_sync(0xffffffffu, s, o);
    if (lane + o <= end) s += t;
  }
  if (lane < nv && ((mask >> lane) & 1u)) epi.emit((long long)(unsigned)D.y + rank, s);
}

template <class Epi>
__device__ __forceinline__ void process_long(const PassDev& P, int4 D, const double* sv, int lane, Epi& epi) {
  const int nv = D.w & 0x7fffffff;
  const uint4* base = P.vec + (unsigned)D.x;
  double s = 0.0;
  for (int b0 = 0; b0 < nv; b0 += 128) {
    uint4 q[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      int v = b0 + u * 32 + lane;
      if (v < nv) q[u] = ldg_stream(base + v);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      int v = b0 + u * 32 + lane;
      if (v < nv) s += gather8(q[u], sv);
    }
  }
  s = warp_sum(s);
  if (lane == 0) epi.emit((long long)(unsigned)D.y, s);
}

template <class Epi>
__device__ __forceinline__ void process_bundles(const PassDev& P, int4 T, const double* sv, Epi& epi) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int b = P.warp_split[T.w + warp];
  const int b1 = P.warp_split[T.w + warp + 1];
  while (b < b1) {
    const int nb = min(4, b1 - b);
    int4 d = make_int4(0, 0, 0, 0);
    if (lane < nb) d = __ldg(P.bundle + b + lane);
    int4 D[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      D[u].x = __shfl_sync(0xffffffffu, d.x, u);
      D[u].y = __shfl_sync(0xffffffffu, d.y, u);
      D[u].z = __shfl_sync(0xffffffffu, d.z, u);
      D[u].w = __shfl_sync(0xffffffffu, d.w, u);
    }
    if (D[0].w < 0) {  // long bundle (flag in the sign bit)
      process_long(P, D[0], sv, lane, epi);
      b += 1;
      continue;
    }
    int m = 1;
    while (m < nb && D[m].w >= 0) ++m;
    uint4 q[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (u < m && lane < D[u].w) q[u] = ldg_stream(P.vec + (unsigned)D[u].x + lane);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (u < m) {
        double s = lane < D[u].w ? gather8(q[u], sv) : 0.0;
        seg_emit(D[u], s, lane, epi);
      }
    }
    b += m;
  }
}

// Runs every task of this CTA: fill the slab vector into shared memory, then
// walk the warp's bundle range.  `fill(sv, lo, len)` must end with a barrier.
template <class Fill, class Epi>
__device__ __forceinline__ void run_pass(const PassDev& P, double* sv, Fill& fill, Epi& epi) {
  const int c = blockIdx.x;
  const int t0 = P.cta_task_ptr[c], t1 = P.cta_task_ptr[c + 1];
  for (int t = t0; t < t1; ++t) {
    const int4 T = __ldg(P.task + t);
    const long long lo = P.slab_lo[T.x], hi = P.slab_lo[T.x + 1];
    __syncthreads();
    fill(sv, lo, (int)(hi - lo));
    process_bundles(P, T, sv, epi);
  }
}

// Sum of the CSC pieces of internal column j (slab-major, fixed order).
__device__ __forceinline__ double column_sum(const PassDev& csc, const double* pieces, long long pt, long long j) {
  double s = 0.0;
  for (int sl = 0; sl < csc.nslab; ++sl) {
    const int* pp = csc.piece_ptr + (long long)sl * (pt + 1);
    const int q0 = pp[j], q1 = pp[j + 1];
    for (int q = q0; q < q1; ++q) s += __ldcg(pieces + q);
  }
  return s;
}

// internal column j (shrunk 0..p-1, intercept p) -> reference coordinate
__device__ __forceinline__ long long ref_index(long long j, long long p, int icpt) {
  return j < p ? j + icpt : 0;
}

// ------------------------------------------------------------------ Philox4x32-10
struct Philox {
  uint2 key;
  uint4 ctr;
  uint4 buf;
  int avail;  // 32-bit words left in buf

  __device__ __forceinline__ Philox(unsigned long long seed, unsigned long long stream, unsigned elem) {
    key = make_uint2((unsigned)seed, (unsigned)(seed >> 32));
    ctr = make_uint4(0u, elem, (unsigned)stream, (unsigned)(stream >> 32));
    avail = 0;
  }
  __device__ __forceinline__ static uint4 round10(uint4 c, uint2 k) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
      const unsigned hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
      const unsigned hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
      c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
      k.x += 0x9E3779B9u;
      k.y += 0xBB67AE85u;
    }
    return c;
  }
  __device__ __forceinline__ unsigned next32() {
    if (avail == 0) {
      buf = round10(ctr, key);
      ctr.x++;
      avail = 4;
    }
    const unsigned r = avail == 4 ? buf.x : avail == 3 ? buf.y : avail == 2 ? buf.z : buf.w;
    --avail;
    return r;
  }
  // uniform in (0, 1], 53 random bits
  __device__ __forceinline__ double uniform_pos() {
    const unsigned a = next32() >> 5, b = next32() >> 6;
    return ((double)a * 67108864.0 + (double)b + 1.0) * (1.0 / 9007199254740992.0);
  }
  // uniform in [0, 1)
  __device__ __forceinline__ double uniform() {
    const unsigned a = next32() >> 5, b = next32() >> 6;
    return ((double)a * 67108864.0 + (double)b) * (1.0 / 9007199254740992.0);
  }
  __device__ __forceinline__ double exponential() { return -log(uniform_pos()); }
  __device__ __forceinline__ double normal() {
    const double u1 = uniform_pos(), u2 = uniform();
    return sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
  }
  // Marsaglia-Tsang Gamma(shape, 1), shape > 0
  __device__ double gamma(double shape) {
    double boost = 1.0;
    if (shape < 1.0) {
      boost = pow(uniform_pos(), 1.0 / shape);
      shape += 1.0;
    }
    const double d = shape - 1.0 / 3.0, c = 1.0 / sqrt(9.0 * d);
    for (;;) {
      double x, v;
      do {
        x = normal();
        v = 1.0 + c * x;
      } while (v <= 0.0);
      v = v * v * v;
      const double u = uniform_pos();
      if (u < 1.0 - 0.0331 * (x * x) * (x * x)) return d * v * boost;
      if (log(u) < 0.5 * x * x + d * (1.0 - v + log(v))) return d * v * boost;
    }
  }
};

// stream identifiers (high bits select the purpose, low bits the scan)
constexpr unsigned long long kStreamEta = 1ull << 56;
constexpr unsigned long long kStreamDelta = 2ull << 56;
constexpr unsigned long long kStreamPG = 3ull << 56;
constexpr unsigned long long kStreamLocal = 4ull << 56;
constexpr unsigned long long kStreamGlobal = 5ull << 56;
constexpr unsigned long long kStreamAux = 6ull << 56;

}  // namespace pcgs
