// Device building blocks shared by every pcgs kernel.
#pragma once
#include <type_traits>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "store.h"

namespace pcgs {

struct PassDev {
  const uint4* vec;          // uint16 index vectors (8 per uint4)
  const uint2* blocks;       // BlockDesc {first_id, mask} per 32-vector block;
                             // grouped layout: per slice {ids offset, steps | log2 W << 24}
  const unsigned* ids;       // grouped layout: segment ids of the slices' lane groups
  int grouped;
  int nranges;               // warp ranges per task (store.h)
  const int* rep_ptr;             // nslab+1 offsets into rep_src (null: no replicas)
  const unsigned short* rep_src;  // replica k of slab s copies slab entry rep_src[rep_ptr[s] + k]
  const uint4* warps;        // WarpRange {v0, nvec, blk0, pad}
  const int2* task;          // Task {slab, warp0}
  const int* cta_task_ptr;   // G+1
  const long long* slab_lo;  // nslab+1
  const int* piece_ptr;      // CSC: nslab*(p_total+1)
  const int* col_piece_ptr;  // CSC: p_total+1 column-major slot ranges (store.h)
  const unsigned* ids_perm;  // CSC: `ids` mapped through piece_perm (k_pcg's CSC pass walks with these)
  int nslab;
  long long nseg;
};

// Affine terms of a design beyond its binary pattern:
// X_eff = ([P | 1? | Dn] - 1 mu') diag(1/s), i.e. a dense real block Dn of q
// columns next to the pattern P (and the intercept), and column centring /
// scaling.  The reference layout is [intercept? | dense q | pattern p]
// (hstack_dense_columns prepends, sparse.py:314-341); the internal layout is
// [pattern p | intercept? | dense q].  Every pass gathers u = v / s and adds
// the scalar c0 = u_icpt - mu'u plus the row term (Dn u_D)_i to each row sum;
// the transposes map raw column sums g to (g_j - mu_j W) / s_j, W = sum w.
struct AffineDev {
  int on;              // any affine term present
  int q;               // dense columns
  const double* dense; // n x q row-major (reference columns icpt .. icpt+q-1)
  const double* mu;    // reference layout, length pt (null: no centring)
  const double* sc;    // reference layout, length pt (null: no scaling)
};

struct DesignDev {
  long long n, p, pt;  // rows, shrunk columns, p + intercept + dense columns
  int icpt;
  int G;               // CTAs the static plan was built for
  int smem_doubles;    // dynamic shared memory per CTA, in doubles
  int dbg;             // tuning experiments: bit 0 skip gathers, bit 1 skip segmented reduce
  PassDev csr, csc;
  int own_in_global;   // PCG own-slice state does not fit next to the slab in shared memory
                       // (very wide designs): it lives in global memory instead
  double* own_global;  // that buffer (8 x chunk per CTA); allocated per solve, never per
                       // design, so solves on one design from several streams stay apart
  AffineDev aff;
  __host__ __device__ int lead() const { return icpt + aff.q; }  // reference offset of pattern column 0
};

// ------------------------------------------------------------------ checked builds
// PCGS_CHECKED=1 (tools/build_variant.py checked -DPCGS_CHECKED=1) compiles
// bounds checks into the streaming loops and epilogues -- every gathered
// index within its slab (sentinel included), every emitted segment / piece
// id within its output -- trapping on a violation.  compute-sanitizer is
// closed on this GPU pool; the GPU suite run against the checked library is
// the substitute (profiles/sanitizer_r02.txt).
#ifndef PCGS_CHECKED
#define PCGS_CHECKED 0
#endif
#if PCGS_CHECKED
#define PCGS_CHECK(cond)                                                                        \
  do {                                                                                          \
    if (!(cond)) {                                                                              \
      printf("pcgs check failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__,  \
             (int)blockIdx.x, (int)threadIdx.x);                                                \
      __trap();                                                                                 \
    }                                                                                           \
  } while (0)
#else
#define PCGS_CHECK(cond) \
  do {                   \
  } while (0)
#endif
__device__ __forceinline__ void check_vec(uint4 q, int len) {
  PCGS_CHECK((q.x & 0xffffu) <= (unsigned)len && (q.x >> 16) <= (unsigned)len);
  PCGS_CHECK((q.y & 0xffffu) <= (unsigned)len && (q.y >> 16) <= (unsigned)len);
  PCGS_CHECK((q.z & 0xffffu) <= (unsigned)len && (q.z >> 16) <= (unsigned)len);
  PCGS_CHECK((q.w & 0xffffu) <= (unsigned)len && (q.w >> 16) <= (unsigned)len);
}

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

// Cross-CTA partial sums: CTA c's value lives alone in a 128-byte line
// (part[c * kPartStride]) so that the G readers of the G lines spread over L2
// slices.  Every CTA reduces the same G partials in the same order (bitwise
// identical everywhere); only warp 0 loads them, the result is broadcast
// through shared memory.  Must be called by the whole CTA.
constexpr int kPartStride = 16;
constexpr int kPartLoads = 8;  // partial loads per lane: grids up to 256 CTAs

// Lane-strided sum of partials q = lane, lane+32, ... (< G) in that order; all
// loads are issued before the first add, so the L2 round trips overlap.
__device__ __forceinline__ double lane_partials(const double* part, int G, int lane) {
  double v[kPartLoads];
#pragma unroll
  for (int u = 0; u < kPartLoads; ++u) {
    const int q = lane + 32 * u;
    v[u] = q < G ? __ldcg(part + (long long)q * kPartStride) : 0.0;
  }
  double s = 0.0;
#pragma unroll
  for (int u = 0; u < kPartLoads; ++u) s += v[u];
  return s;
}

__device__ __forceinline__ double reduce_partials(const double* part, int G, double* bcast) {
  const int lane = threadIdx.x & 31;
  __syncthreads();
  if (threadIdx.x < 32) {
    const double s = warp_sum(lane_partials(part, G, lane));
    if (lane == 0) *bcast = s;
  }
  __syncthreads();
  return *bcast;
}

__device__ __forceinline__ void reduce_partials2(const double* part, int G, double* bcast, double& a, double& b) {
  const int lane = threadIdx.x & 31;
  __syncthreads();
  if (threadIdx.x < 32) {
    double s0 = lane_partials(part, G, lane), s1 = lane_partials(part + 1, G, lane);
    s0 = warp_sum(s0);
    s1 = warp_sum(s1);
    if (lane == 0) {
      bcast[0] = s0;
      bcast[1] = s1;
    }
  }
  __syncthreads();
  a = bcast[0];
  b = bcast[1];
}

__device__ __forceinline__ double gather8(uint4 q, const double* sv) {
  double a = sv[q.x & 0xffffu] + sv[q.x >> 16];
  double b = sv[q.y & 0xffffu] + sv[q.y >> 16];
  double c = sv[q.z & 0xffffu] + sv[q.z >> 16];
  double d = sv[q.w & 0xffffu] + sv[q.w >> 16];
  return (a + b) + (c + d);
}

// The same sum from a 32-bit shared-window address `sb` of the slab: each
// address is one extract plus one LEA (sb + index * 8), where the generic
// form costs a shift, a mask and an add per index.
__device__ __forceinline__ double lds64(unsigned a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
// halves of a packed index pair, zero-extended by a byte permute (opaque to
// the optimiser, so the address stays extract + LEA)
__device__ __forceinline__ unsigned lo16(unsigned x) {
  unsigned r;
  asm("prmt.b32 %0, %1, 0, 0x4410;" : "=r"(r) : "r"(x));
  return r;
}
__device__ __forceinline__ unsigned hi16(unsigned x) {
  unsigned r;
  asm("prmt.b32 %0, %1, 0, 0x4432;" : "=r"(r) : "r"(x));
  return r;
}
__device__ __forceinline__ unsigned slab_addr(unsigned sb, unsigned idx) { return sb + (idx << 3); }
__device__ __forceinline__ double gather8s(uint4 q, unsigned sb) {
  const double a = lds64(slab_addr(sb, lo16(q.x))) + lds64(slab_addr(sb, hi16(q.x)));
  const double b = lds64(slab_addr(sb, lo16(q.y))) + lds64(slab_addr(sb, hi16(q.y)));
  const double c = lds64(slab_addr(sb, lo16(q.z))) + lds64(slab_addr(sb, hi16(q.z)));
  const double d = lds64(slab_addr(sb, lo16(q.w))) + lds64(slab_addr(sb, hi16(q.w)));
  return (a + b) + (c + d);
}
#ifndef PCGS_LDS_ASM
#define PCGS_LDS_ASM 1
#endif

// ------------------------------------------------------------------ fills
// sv[j] = f(j) for j in [0, len); sv[len] = 0 (the segment sentinel).  Loads are
// batched 16 per thread so the fill is one or two L2 round trips.
template <class F>
__device__ __forceinline__ void fill_smem(double* sv, int len, F& f) {
  constexpr int U = 8;
  const int nthr = (int)blockDim.x;
  for (int j0 = threadIdx.x; j0 < len; j0 += nthr * U) {
    double vals[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      int j = j0 + u * nthr;
      vals[u] = j < len ? f(j) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      int j = j0 + u * nthr;
      if (j < len) sv[j] = vals[u];
    }
  }
  if (threadIdx.x == 0) sv[len] = 0.0;
  __syncthreads();
}

// Bulk (TMA engine) copy of a 16-byte aligned global slab into shared memory,
// completion tracked by an mbarrier; an odd tail element is copied by a thread.
__device__ __forceinline__ unsigned smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

struct BulkFill {
  unsigned long long* mbar;  // in shared memory, initialised by bulk_init
  unsigned phase;
};

__device__ __forceinline__ void bulk_init(BulkFill& B, unsigned long long* mbar) {
  B.mbar = mbar;
  B.phase = 0;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_addr(mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
}

struct NoHook {
  __device__ void operator()() const {}
};

// `hook` runs on every thread between the copy's issue and the wait, so
// independent latency-bound work (e.g. a grid-partial reduction) overlaps it.
template <class Hook = NoHook>
__device__ __forceinline__ void bulk_fill(BulkFill& B, double* sv, const double* src, int len, Hook hook = Hook{}) {
  const int n2 = len & ~1;
  if (threadIdx.x == 0) {
    const unsigned bytes = (unsigned)n2 * 8u;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("fence.proxy.async.global;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_addr(B.mbar)), "r"(bytes)
                 : "memory");
#ifndef PCGS_FILL_CHUNK
#define PCGS_FILL_CHUNK 32768
#endif
    const unsigned CH = PCGS_FILL_CHUNK;
    for (unsigned off = 0; off < bytes; off += CH) {
      const unsigned sz = bytes - off < CH ? bytes - off : CH;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_addr((char*)sv + off)),
          "l"((const char*)src + off), "r"(sz), "r"(smem_addr(B.mbar))
          : "memory");
    }
  }
  if ((len & 1) && threadIdx.x == 32) sv[len - 1] = __ldcg(src + len - 1);
  hook();
  asm volatile(
      "{\n.reg .pred P;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared.b64 P, [%0], %1;\n"
      "@!P bra WAIT_%=;\n}" ::"r"(smem_addr(B.mbar)),
      "r"(B.phase)
      : "memory");
  B.phase ^= 1u;
  if (threadIdx.x == 0) sv[len] = 0.0;
  __syncthreads();
}

// ------------------------------------------------------------------ passes
// ---------------------------------------------------------------------------
// Flat per-warp stream: block k of a warp range is vectors [32k, 32k+32), one
// per lane.  Index loads run kRing blocks ahead in a register ring; the block
// descriptors (start mask + first segment id) drive a segmented reduction whose
// open segment is carried across blocks in a per-lane accumulator.
// ---------------------------------------------------------------------------
// Blocks per load batch.  Tuned on the config-2 PCG iteration with the
// prefetch windows below (tools/ab_variants.sh): 1 -> 103, 2 -> 93.4, 3 -> 94.2,
// 4 -> 96.1, 5 -> 112 us (4+ spill at the 64-register cap); issuing the next
// batch before consuming the current one (software pipelining) was slower
// at every depth (2: 105.8 us).
#ifndef PCGS_RING
#define PCGS_RING 2
#endif
// Debug modes of the streaming loop (skip gathers / reductions / prefetch,
// debug-option key 1 bits 1, 2, 4, 16) exist only in builds with
// -DPCGS_DEBUG_MODES=1 (tools/pass_modes.py); the production loop has none.
#ifndef PCGS_DEBUG_MODES
#define PCGS_DEBUG_MODES 0
#endif
constexpr bool kDebugModes = PCGS_DEBUG_MODES != 0;
constexpr int kRing = PCGS_RING;
static_assert((kRing & (kRing - 1)) == 0, "kRing must be a power of two");
#ifndef PCGS_LANE_PREFETCH
#define PCGS_LANE_PREFETCH 1
#endif
#ifndef PCGS_L1_NEXT
#define PCGS_L1_NEXT 0
#endif
#ifndef PCGS_DESC_PRED
#define PCGS_DESC_PRED 1
#endif

// `M` is the block's segment-start mask; `first_id` (the id of the segment
// starting at the lowest set bit) is fetched lazily by shuffling `dl_x` from
// lane `u` -- only blocks that contain a segment start need it.
template <class Epi>
__device__ __forceinline__ void block_reduce(unsigned M, unsigned dl_x, int u, double s, int lane, double& acc,
                                             unsigned& open_id, bool& have_open, Epi& epi) {
  if (M == 0u) {
    acc += s;
    return;
  }
  uint2 dsc;
  dsc.x = __shfl_sync(0xffffffffu, dl_x, u);
  dsc.y = M;
  const int f = __ffs(M) - 1;
  const int Lh = 31 - __clz(M);
  // close the open segment: its lanes < f plus every lane's carried partial
  {
    const double c = warp_sum(acc + (lane < f ? s : 0.0));
    if (have_open && lane == 0) epi.emit((long long)open_id, c);
  }
  // segments that start and end inside this block: starts in [f, Lh)
  if (f != Lh) {
    double x = (lane >= f && lane < Lh) ? s : 0.0;
    const unsigned le = lane == 31 ? 0xffffffffu : ((2u << lane) - 1u);
    const unsigned after = M & ~le;
    const int end = after ? (__ffs(after) - 2) : 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double t = __shfl_down_sync(0xffffffffu, x, o);
      if (lane + o <= end) x += t;
    }
    if (((M >> lane) & 1u) && lane < Lh) epi.emit((long long)(dsc.x + __popc(M & (le >> 1))), x);
  }
  acc = lane >= Lh ? s : 0.0;
  open_id = dsc.x + __popc(M) - 1;
  have_open = true;
}

// L2 prefetch (TMA engine; no registers or scoreboards) of the first
// kPrefetchBlocks blocks of a warp's range, issued before the slab fill; the
// batch loop then keeps a sliding window of kPrefetchBlocks ahead of its loads,
// so DRAM requests arrive in consumption order.
// Prefetch windows (blocks of 512 B per warp), tuned on the config-2 PCG
// iteration (tools/ab_prefetch.sh, ab_variants.sh): with 4-block batches
// 16/16 -> 100.0 us, 8/8 -> 96.6, 6/6 -> 96.0; with 2-block batches 4/4 ->
// 93.4 us.  A large first window floods HBM just when the slab fill needs the
// memory system; a short sliding distance keeps prefetches in consumption order.
#ifndef PCGS_PREFETCH_DIST
#define PCGS_PREFETCH_DIST 4
#endif
constexpr int kPrefetchBlocks = PCGS_PREFETCH_DIST;  // sliding L2 prefetch distance, blocks
#ifndef PCGS_PREFETCH0
#define PCGS_PREFETCH0 4
#endif
constexpr int kPrefetchFirst = PCGS_PREFETCH0;  // blocks prefetched before the slab fill
__device__ __forceinline__ void prefetch_range(const PassDev& P, int range, int dbg) {
  const int lane = threadIdx.x & 31;
  if (lane != 0 || (kDebugModes && (dbg & 4))) return;
  const uint4 R = __ldg(P.warps + range);
  const int nvec = (int)R.y;
  if (nvec == 0) return;
  const int nb = (nvec + 31) >> 5;
  const char* p0 = (const char*)(P.vec + R.x);
  const unsigned total = (unsigned)nvec * 16u;
  const unsigned bytes = (kDebugModes && (dbg & 16)) ? total : min(total, (unsigned)kPrefetchFirst * 512u);
  for (unsigned off = 0; off < bytes; off += 16384u) {
    const unsigned sz = bytes - off < 16384u ? bytes - off : 16384u;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p0 + off), "r"(sz) : "memory");
  }
  const uint2* bd = P.blocks + R.z;
  const unsigned long long d0 = (unsigned long long)bd & ~15ull;
  const unsigned long long d1 = ((unsigned long long)(bd + (P.grouped ? (int)R.w : nb)) + 15ull) & ~15ull;
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(d0), "r"((unsigned)(d1 - d0)) : "memory");
}

// A CTA of blockDim.x / 32 warps walks the P.nranges ranges of a task: warp w takes
// ranges w, w + nwarps, ...
__device__ __forceinline__ void prefetch_warp(const PassDev& P, int warp0, int dbg) {
  const int nw = (int)(blockDim.x >> 5);
  for (int r = (int)(threadIdx.x >> 5); r < P.nranges; r += nw) prefetch_range(P, warp0 + r, dbg);
}

template <class Epi>
__device__ __forceinline__ void process_warp(const PassDev& P, int warp0, const double* sv, Epi& epi, int dbg = 0,
                                             int slab_len = 0) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint4 R = __ldg(P.warps + warp0 + warp);
  const int nvec = (int)R.y;
  if (nvec == 0) return;
  const int nb = (nvec + 31) >> 5;
  const uint4* base = P.vec + R.x;
  const uint2* bd = P.blocks + R.z;
  const unsigned sb = smem_addr(sv);
  double acc = 0.0;
  unsigned open_id = 0;
  bool have_open = false;
  // batches of kRing blocks: all loads of a batch issued together, then
  // consumed.  Batches of full blocks run without bound checks; the last,
  // partial batch takes the checked path.
  const int nfull = (nvec >> 5) / kRing * kRing;  // blocks in full batches
  auto batch = [&](int k0, auto checked) {
    constexpr bool kChecked = decltype(checked)::value;
    uint4 q[kRing];
    if (!(kDebugModes && (dbg & 20))) {
#if PCGS_LANE_PREFETCH
      // sliding L2 prefetch, one 128-byte line per lane (4 lines per block):
      // a per-lane prefetch needs no uniform address (the bulk form costs a
      // waterfall loop of R2UR conversions per batch)
      const unsigned off = (unsigned)(k0 + kPrefetchBlocks) * 512u + (unsigned)lane * 128u;
      if (lane < 4 * kRing && off < (unsigned)nvec * 16u)
        asm volatile("prefetch.global.L2 [%0];" ::"l"((const char*)base + off));
#if PCGS_L1_NEXT
      // experiment: the next batch's lines into L1 (lanes 16..16+4 kRing)
      {
        const unsigned off1 = (unsigned)(k0 + kRing) * 512u + (unsigned)(lane - 16) * 128u;
        if (lane >= 16 && lane < 16 + 4 * kRing && off1 < (unsigned)nvec * 16u)
          asm volatile("prefetch.global.L1 [%0];" ::"l"((const char*)base + off1));
      }
#endif
#else
      if (lane == 0 && k0 + kPrefetchBlocks < nb) {
        const int kb = k0 + kPrefetchBlocks;
        const int ke = min(nb, kb + kRing);
        const unsigned v_end = (unsigned)min(nvec, ke * 32);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"((const char*)(base + kb * 32)),
                     "r"((v_end - (unsigned)kb * 32u) * 16u)
                     : "memory");
      }
#endif
    }
    // block descriptors of the batch: lane u's copy feeds block u (full
    // batches load unconditionally: no divergent branch around the load)
#if PCGS_DESC_PRED
    // only lanes < kRing load (predicated, no branch): 16 B of register
    // writeback per batch instead of 32 lanes x 8 B through the L1 data pipe
    uint2 dl = make_uint2(0u, 0u);
    if (lane < kRing && (!kChecked || k0 + lane < nb)) dl = __ldg(bd + k0 + lane);
#else
    const uint2 dl = !kChecked ? __ldg(bd + k0 + (lane & (kRing - 1)))
                               : (lane < kRing && k0 + lane < nb ? __ldg(bd + k0 + lane) : make_uint2(0u, 0u));
#endif
#pragma unroll
    for (int u = 0; u < kRing; ++u) {
      const int v = (k0 + u) * 32 + lane;
      if (!kChecked || v < nvec) q[u] = ldg_stream(base + v);
    }
#pragma unroll
    for (int u = 0; u < kRing; ++u) {
      const int k = k0 + u;
      if (!kChecked || k < nb) {
        const unsigned M = __shfl_sync(0xffffffffu, dl.y, u);
        const bool live = !kChecked || k * 32 + lane < nvec;
        double s;
        if (kDebugModes && (dbg & 1)) s = live ? (double)(q[u].x ^ q[u].y ^ q[u].z ^ q[u].w) : 0.0;
        else s = live ? (PCGS_LDS_ASM ? gather8s(q[u], sb) : gather8(q[u], sv)) : 0.0;
        if (PCGS_CHECKED && live) check_vec(q[u], slab_len);
        if (kDebugModes && (dbg & 2)) acc += s + (double)M;
        else block_reduce(M, dl.x, u, s, lane, acc, open_id, have_open, epi);
      }
    }
  };
  for (int k0 = 0; k0 < nfull; k0 += kRing) batch(k0, std::false_type());
  if (nfull < nb) batch(nfull, std::true_type());
  const double c = warp_sum(acc);
  if (have_open && lane == 0) epi.emit((long long)open_id, c);
}


// ---------------------------------------------------------------------------
// Grouped layout (store.h): every lane sums its own vectors into a private
// accumulator; when a slice ends (a warp-uniform block count) the W lanes of
// each group add their accumulators by log2 W butterfly steps and the group's
// first lane emits the segment.  No per-block masks, no segmented scan: the
// cross-lane traffic is 2 log2 W shuffles per slice.
// ---------------------------------------------------------------------------
// Blocks per register batch and software pipelining of the grouped walk,
// measured on the config-2 PCG iteration (tools/gpu_ab_grouped.sh): batches of 2
// without pipelining 73.3 us; two batches of 1 block, one in flight while the
// other is consumed, 70.6 (two batches of 2 spill: 75.4; of 3: 98.5); with the
// shared window base pinned in a register 70.2; L2 prefetch distance 4 blocks
// 69.5 (8: 70.0, 12: 71.7, 16: 73.1); prefetching the lines of 8 blocks every
// 4th iteration instead of 2 blocks every iteration: 75.0.  With 16 warps of
// 128 registers (k_pcg) the batches hold 2 blocks each (1: 79.0, 2: 70.5,
// 3: 71.7 us).
#ifndef PCGS_GRING
#define PCGS_GRING 1
#endif
constexpr int kGRing = PCGS_GRING;  // 32-warp kernels (64 registers); k_pcg (16 warps) passes 2
#ifndef PCGS_GPIPE
#define PCGS_GPIPE 1
#endif
// sliding L2 prefetch distance of the pipelined walk, blocks: 0 = two blocks
// past the register batches (4 with one-block batches, 6 with two-block ones:
// at 16 warps 2 -> 71.9 us, 4 -> 67.2, 6 -> 66.6, 8 -> 66.8, 12 -> 67.8)
#ifndef PCGS_GPREFETCH
#define PCGS_GPREFETCH 0
#endif
#ifndef PCGS_SB_OPAQUE
#define PCGS_SB_OPAQUE 1
#endif

template <int kGRing, class Epi>
__device__ __forceinline__ void process_warp_grouped(const PassDev& P, int range, const double* sv, Epi& epi,
                                                     int slab_len = 0) {
  const int lane = threadIdx.x & 31;
  const uint4 R = __ldg(P.warps + range);
  const int nvec = (int)R.y;
  if (nvec == 0) return;
  const int nb = nvec >> 5;
  const uint4* base = P.vec + R.x;
  const uint2* sd = P.blocks + R.z;
  const int nsl = (int)R.w;
  unsigned sb = smem_addr(sv);
#if PCGS_SB_OPAQUE
  asm volatile("" : "+r"(sb));  // keep the shared window base in a register (else the
                                // generic->shared conversion is redone in every block)
#endif
  // slice state: `end` = block count at which the current slice closes
  uint2 dn = __ldg(sd);
  int s = 0, end = 0;
  unsigned lw = 0, id = 0xffffffffu;
  auto advance = [&]() {
    if (s < nsl) {
      end += (int)(dn.y & 0xffffffu);
      lw = dn.y >> 24;
      id = __ldg(P.ids + dn.x + ((unsigned)lane >> lw));
      ++s;
      if (s < nsl) dn = __ldg(sd + s);
    } else {
      end = -1;
    }
  };
  advance();
  double acc = 0.0;
  // closes the current slice when block `k` was its last
  auto close_if_end = [&](int k) {
    if (k + 1 == end) {
      double t = acc;
      if (lw > 0) t += __shfl_xor_sync(0xffffffffu, t, 1);
      if (lw > 1) t += __shfl_xor_sync(0xffffffffu, t, 2);
      if (lw > 2) t += __shfl_xor_sync(0xffffffffu, t, 4);
      if (lw > 3) t += __shfl_xor_sync(0xffffffffu, t, 8);
      if (lw > 4) t += __shfl_xor_sync(0xffffffffu, t, 16);
      if ((lane & ((1 << lw) - 1)) == 0 && id != 0xffffffffu) epi.emit((long long)id, t);
      acc = 0.0;
      advance();
    }
  };
#if PCGS_GPIPE
  // two register batches of kGRing blocks: the loads of one batch are in
  // flight while the other is consumed (the index loads' latency is what the
  // 8 warps per scheduler cannot hide on their own)
  auto load = [&](uint4(&q)[kGRing], int k0) {
#pragma unroll
    for (int u = 0; u < kGRing; ++u)
      if (k0 + u < nb) q[u] = ldg_stream(base + (k0 + u) * 32 + lane);
  };
  auto consume = [&](uint4(&q)[kGRing], int k0) {
#pragma unroll
    for (int u = 0; u < kGRing; ++u)
      if (k0 + u < nb) {
        if (PCGS_CHECKED) check_vec(q[u], slab_len);
        acc += gather8s(q[u], sb);
        close_if_end(k0 + u);
      }
  };
  uint4 qa[kGRing], qb[kGRing];
  load(qa, 0);
  for (int k0 = 0; k0 < nb; k0 += 2 * kGRing) {
    load(qb, k0 + kGRing);
    {
      constexpr int kGPrefetch = PCGS_GPREFETCH > 0 ? PCGS_GPREFETCH : 2 * kGRing + 2;
      const unsigned off = (unsigned)(k0 + kGPrefetch) * 512u + (unsigned)lane * 128u;
      if (lane < 8 * kGRing && off < (unsigned)nvec * 16u)
        asm volatile("prefetch.global.L2 [%0];" ::"l"((const char*)base + off));
    }
    consume(qa, k0);
    load(qa, k0 + 2 * kGRing);
    consume(qb, k0 + kGRing);
  }
#else
  const int nfull = nb / kGRing * kGRing;
  auto batch = [&](int k0, auto checked) {
    constexpr bool kChecked = decltype(checked)::value;
    uint4 q[kGRing];
    {
      const unsigned off = (unsigned)(k0 + kPrefetchBlocks) * 512u + (unsigned)lane * 128u;
      if (lane < 4 * kGRing && off < (unsigned)nvec * 16u)
        asm volatile("prefetch.global.L2 [%0];" ::"l"((const char*)base + off));
    }
#pragma unroll
    for (int u = 0; u < kGRing; ++u)
      if (!kChecked || k0 + u < nb) q[u] = ldg_stream(base + (k0 + u) * 32 + lane);
#pragma unroll
    for (int u = 0; u < kGRing; ++u) {
      if (!kChecked || k0 + u < nb) {
        if (PCGS_CHECKED) check_vec(q[u], slab_len);
        acc += gather8s(q[u], sb);
        close_if_end(k0 + u);
      }
    }
  };
  for (int k0 = 0; k0 < nfull; k0 += kGRing) batch(k0, std::false_type());
  if (nfull < nb) batch(nfull, std::true_type());
#endif
}

// Runs every task of this CTA: fill the slab vector into shared memory, then
// walk the warp's bundle range.  `fill(sv, lo, len)` must end with a barrier.
// Not inlined: inside the persistent PCG kernel the caller's live state is
// saved once per pass and the streaming loop gets the whole register budget.
__device__ unsigned long long* g_cta_times = nullptr;  // debug: per-CTA [start, filled, end]

// Fill functors that declare `static constexpr bool kHooked = true` take a
// fourth argument, a callable run by every thread between the issue of the
// bulk copy and the wait for it.
template <class F, class = void>
struct fill_takes_hook : std::false_type {};
template <class F>
struct fill_takes_hook<F, std::void_t<decltype(F::kHooked)>> : std::true_type {};

template <int kRingBlocks = kGRing, class Fill, class Epi>
__device__ __forceinline__ void run_pass(const PassDev& P, double* sv, Fill& fill, Epi& epi, int dbg = 0,
                                         int cta = -1) {
  const int c = cta < 0 ? (int)blockIdx.x : cta;  // CTA index within the plan (row-split groups)
  unsigned long long t_start = 0;
  if ((dbg & 64) && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
  const int t0 = P.cta_task_ptr[c], t1 = P.cta_task_ptr[c + 1];
  for (int t = t0; t < t1; ++t) {
    const int2 T = __ldg(P.task + t);
    const long long lo = P.slab_lo[T.x], hi = P.slab_lo[T.x + 1];
    if constexpr (fill_takes_hook<Fill>::value) {
      // bulk fills: the copy is issued first; the warps' L2 prefetch (a
      // dependent load of the warp range, then the prefetch instructions)
      // runs while it is in flight
      __syncthreads();
      fill(sv, lo, (int)(hi - lo), [&] { prefetch_warp(P, T.y, dbg); });
    } else {
      prefetch_warp(P, T.y, dbg);
      __syncthreads();
      if (dbg & 8) {
        if (threadIdx.x == 0) sv[hi - lo] = 0.0;
        __syncthreads();
      } else {
        fill(sv, lo, (int)(hi - lo));
      }
    }
    // replicas (store.h): second copies of the slab's most gathered entries
    // behind the sentinel, at other bank pairs (the fill ended with a barrier)
    int nrep = 0;
    if (P.rep_ptr) {
      const int r0 = P.rep_ptr[T.x];
      nrep = P.rep_ptr[T.x + 1] - r0;
      if (nrep > 0) {
        double* rp = sv + (hi - lo) + 1;
        for (int k = threadIdx.x; k < nrep; k += (int)blockDim.x) rp[k] = sv[__ldg(P.rep_src + r0 + k)];
        __syncthreads();
      }
    }
    if ((dbg & 64) && threadIdx.x == 0 && g_cta_times) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      g_cta_times[3 * c + 0] = t_start;
      g_cta_times[3 * c + 1] = t;
    }
#if PCGS_FLAT_WALK
    if (!P.grouped) process_warp(P, T.y, sv, epi, dbg, (int)(hi - lo));
    else
#endif
    {
        const int nw = (int)(blockDim.x >> 5);
        for (int r = (int)(threadIdx.x >> 5); r < P.nranges; r += nw)
          process_warp_grouped<kRingBlocks>(P, T.y + r, sv, epi, (int)(hi - lo) + nrep);
      }
  }
  if (dbg & 64) {
    __syncthreads();
    if (threadIdx.x == 0 && g_cta_times) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      g_cta_times[3 * c + 2] = t;
    }
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

// internal column j (pattern 0..p-1, then the `lead` intercept / dense
// columns) -> reference coordinate; lead = intercept + dense columns
__host__ __device__ __forceinline__ long long ref_index(long long j, long long p, int lead) {
  return j < p ? j + lead : j - p;
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
