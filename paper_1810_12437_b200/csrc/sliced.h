// Sliced store for batched chains (host side; DESIGN.md §7 "batched chains").
//
// R chains (R in {2, 4, 8}) share one walk over the pattern.  A warp's 32
// lanes are S = 32/R SLOTS of R lanes: lane (slot s, chain c) = s * R + c.
// Each slot walks one output PIECE (a run of indices of one row / column
// within one slab) and lane c of the slot accumulates chain c, so a piece
// is summed inside its lanes with no cross-lane reduction.  The S pieces a
// warp walks in lockstep form a SLICE; slice vectors are interleaved
// (vector t of slot s at v0 + t * S + s), so one warp load of the S slots'
// next vectors is S * 16 contiguous bytes.  A slot whose piece is shorter
// than the slice walks the slab's SENTINEL index (a zero row).
//
// Gathered vectors are chain-minor, element (j, c) at [j * R + c], so one
// index fetches R consecutive doubles: a warp LDS.64 touches S rows of 8R
// bytes.  For 64-bit loads a 16-lane half-warp is one shared-memory
// wavefront when its H = 16/R slots read distinct bank groups, i.e. have
// distinct index mod H; inside a piece the index order is free, so the
// builder places indices to make the H slots of each half-warp differ mod H.
//
// Pieces are capped at kSlicedPieceMax vectors (fine-grained balance) and
// numbered output-major (all pieces of row / column j are contiguous:
// out_ptr[j] .. out_ptr[j+1]), so the per-output sums read one contiguous
// range in a fixed order.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "store.h"

namespace pcgs {
// warps per CTA of the batched (sliced-store) kernels; the single-chain tiled
// store has its own count (store.h: kWarps)
constexpr int kSWarps = 32;
constexpr int kSThreads = kSWarps * 32;
}  // namespace pcgs

namespace pcgs {

constexpr int kSlicedPieceMax = 32;  // vectors per piece

// Lane mapping: a slot (one piece per slice) is R/C lanes, each lane summing
// C consecutive chains of the slot's piece with C/2 LDS.128 per index
// (C = 1: one LDS.64).  The slot's 16-byte index vector reaches every lane of
// the slot, so more chains per lane means less register writeback of the
// index stream (1/(2C) of the gather wavefronts).  Bank groups: a 128-bit
// shared load is one wavefront per quarter-warp (64-bit: half-warp); the
// quarter's slots fall into C/2 classes (slot mod C/2) whose lanes read
// different 16-byte chunks of a row at every instruction (the quad mapping
// reads a lane's two chunks in slot-rotated order), so within a class H =
// 16/R slots share the bank groups and must have indices distinct mod H.
//   pair   (C = 2, R >= 2; default)  R/2 lanes per slot
//   quad   (C = 4, R >= 4)            R/4 lanes per slot
//   single (C = 1)                    R lanes per slot
// PCGS_SLICED_CPL caps C (1, 2 or 4).  Measured at config 2 (per 8-chain
// iteration): single 372 us, pair 340, quad 341 (R = 4: pair 186, quad 197):
// past the pair mapping the index writeback no longer limits and the quad's
// extra instructions cost.
#ifndef PCGS_SLICED_CPL
#define PCGS_SLICED_CPL 2
#endif
#ifdef __CUDACC__
#define PCGS_HD __host__ __device__
#else
#define PCGS_HD
#endif
PCGS_HD constexpr int sliced_cpl(int R) {  // chains per lane
  return (PCGS_SLICED_CPL >= 4 && R >= 4) ? 4 : (PCGS_SLICED_CPL >= 2 && R >= 2) ? 2 : 1;
}
PCGS_HD constexpr int sliced_lanes_per_slot(int R) { return R / sliced_cpl(R); }
PCGS_HD constexpr int sliced_slots(int R) { return 32 / sliced_lanes_per_slot(R); }

struct SliceDesc {  // 8 bytes, device-readable as uint2
  uint32_t v0;      // first vector of the slice
  uint32_t len;     // steps (vectors per slot)
};

struct SPassHost {
  int nslab = 0;
  std::vector<int64_t> slab_lo;      // nslab+1, in gathered-vector elements
  std::vector<uint16_t> idx;         // vectors * 8
  std::vector<SliceDesc> slices;
  std::vector<uint32_t> piece;       // S per slice: output piece id per slot (0xffffffff: idle slot)
  std::vector<uint32_t> warp_slices; // per warp range: [first slice, end slice) pairs
  std::vector<Task> tasks;           // {slab, first warp range}, kSWarps ranges per task
  std::vector<int32_t> cta_task_ptr; // G+1
  std::vector<int64_t> out_ptr;      // n_out+1: pieces of output j are [out_ptr[j], out_ptr[j+1])
  int64_t npiece = 0;
  int64_t lds_groups = 0, lds_excess = 0, pad_vectors = 0;
};

struct SlicedHost {
  int64_t n = 0, p = 0, p_total = 0, nnz = 0;
  int intercept = 0;
  int R = 0;
  int slab_max = 0;
  SPassHost csr, csc;
};

// largest slab (in elements, excluding the sentinel) for R chain-minor doubles
int sliced_slab_max(int R);

// Validates the CSR (sparse.py:94-117 invariants) and builds both sliced
// passes for G CTAs.  Returns an empty string on success.
std::string build_sliced(int64_t n, int64_t p, const int64_t* row_ptr, const int32_t* col_idx, int intercept,
                         int R, int slab_max, int G, SlicedHost& out);

// Host-only check: reconstructs both passes and compares with the CSR.
std::string verify_sliced(const SlicedHost& H, const int64_t* row_ptr, const int32_t* col_idx);

}  // namespace pcgs
