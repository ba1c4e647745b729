// Pattern-only tiled store for a binary design (host side of the pcgs library).
//
// Layout (both directions share it):
//   * the gathered vector is cut into SLABS that fit one CTA's shared memory
//     (CSR: column slabs of v; CSC: row slabs of w = ω⊙Xv);
//   * every output SEGMENT (CSR: a row within a column slab; CSC: a piece of
//     a column within a row slab) is a run of uint16 slab-local indices padded
//     to a multiple of 8 with the slab's SENTINEL index (which points at a
//     zero in shared memory), so a 16-byte vector never straddles segments;
//   * the segments of a slab are cut into WARP RANGES (contiguous, balanced by
//     vector count, cut only at segment boundaries).  A warp streams its range
//     32 vectors (one per lane) at a time; every 32-vector BLOCK carries a
//     descriptor {id of the first segment starting in it, 32-bit start mask},
//     so the kernel's loads never depend on segment structure and can be
//     prefetched many blocks ahead;
//   * inside a segment the index order is free (the sum is order-independent
//     in exact arithmetic), so the builder places indices so that each 16-lane
//     half-warp LDS.64 of a block touches distinct shared-memory bank pairs.
//
// GROUPED layout (PassHost::grouped, the default; PCGS_LAYOUT=flat selects
// the flat stream above in builds with -DPCGS_FLAT_WALK=1): a segment is summed inside a fixed GROUP of
// W = 1, 2, 4, ... 32 adjacent lanes (W grows with the segment's length), so a
// block needs no segmented warp reduction -- the cross-lane work is log2 W
// butterfly steps when a SLICE ends.  A slice is 32/W segments of one width
// class and similar length walked in lockstep for T = ceil(max nv / W) steps;
// step t is one 32-vector block (lane g*W + k holds vector t*W + k of the
// slice's g-th segment, sentinel-padded).  A CTA's segments are sorted by
// length before slicing (padding stays small), its slices are dealt to the
// task's warp ranges (PassHost::nranges, below) longest first, each to the
// least loaded range, and a range's slices are contiguous in the stream.  `blocks` then holds one descriptor per slice
// {offset into `ids`, T | log2 W << 24} and `ids` the 32/W segment ids of
// each slice (0xffffffff: empty group); WarpRange.pad counts the slices.
//
// REPLICAS (grouped layout): shared memory left behind the longest slab holds
// second copies of a slab's most gathered entries, each at a bank pair other
// than its original's (replica k of slab s sits at index len + 1 + k and
// copies entry rep_src[rep_ptr[s] + k]; the kernels copy them after every
// slab fill).  An occurrence of a replicated entry may use either address, so
// the placement can balance the bank pairs of a half-warp gather beyond what
// one segment's own index set allows.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

// The flat-stream layout and its walk (PCGS_LAYOUT=flat) are compiled in only
// on request (tools/build_variant.py flat -DPCGS_FLAT_WALK=1): next to the
// grouped walk the flat one costs the persistent kernels registers.
#ifndef PCGS_FLAT_WALK
#define PCGS_FLAT_WALK 0
#endif

namespace pcgs {

// Warps per CTA of the kernels that walk one warp range per warp, and the most
// warp ranges a CTA task can hold.  A store is built with `nranges` ranges per
// task (PassHost::nranges): 16 by default -- the persistent PCG kernel runs 16
// warps of 128 registers (pcgs.cu) -- and 32 for the row-split shards, whose
// kernel runs 32 warps of 64 registers.  A CTA of nw warps walks any store:
// warp w takes ranges w, w + nw, ... (warps beyond nranges idle).
constexpr int kWarps = 32;
constexpr int kDefaultRanges = 16;
constexpr int kThreads = kWarps * 32;  // 1024
constexpr int kVecIdx = 8;             // uint16 indices per 16-byte vector

struct WarpRange {    // 16 bytes, device-readable as uint4
  uint32_t v0;        // first vector of the range in the pass stream
  uint32_t nvec;      // vectors in the range
  uint32_t blk0;      // first block descriptor
  uint32_t pad;       // grouped layout: slices in the range
};

struct BlockDesc {    // 8 bytes, device-readable as uint2
  uint32_t first_id;  // id of the segment starting at the lowest set mask bit
  uint32_t mask;      // bit l: vector (32k + l) starts a segment
};

struct Task {         // one (slab, 16 warp ranges) assignment of a CTA
  int32_t slab;
  int32_t warp0;      // first of nranges consecutive WarpRange entries
};

struct PassHost {
  int nslab = 0;
  std::vector<int64_t> slab_lo;        // nslab+1 boundaries in gathered-vector coords
  std::vector<uint16_t> idx;           // nvec * 8 indices
  std::vector<BlockDesc> blocks;
  std::vector<uint32_t> ids;           // grouped layout: segment ids per slice group
  int grouped = 0;
  int nranges = kDefaultRanges;        // warp ranges per task
  std::vector<int32_t> rep_ptr;        // grouped layout: nslab+1 offsets into rep_src
  std::vector<uint16_t> rep_src;       // replica k of slab s copies slab entry rep_src[rep_ptr[s] + k]
  int64_t pad_vectors = 0;             // grouped layout: all-sentinel vector slots
  std::vector<WarpRange> warps;
  std::vector<Task> tasks;
  std::vector<int32_t> cta_task_ptr;   // G+1
  int64_t nseg = 0;                    // number of output segments
  std::vector<int32_t> piece_ptr;      // CSC: slab-major piece_ptr[s*(ncols+1) + j]
  // CSC, column-major view of the same pieces (the persistent PCG kernel's step
  // phase): piece id q is stored at slot piece_perm[q]; the slots of column j
  // are [col_piece_ptr[j], col_piece_ptr[j+1]), slab-major inside the column
  std::vector<int32_t> piece_perm, col_piece_ptr;
  // statistics
  int64_t lds_groups = 0, lds_conflict_excess = 0;
};

struct DesignHost {
  int64_t n = 0, p = 0, p_total = 0, nnz = 0;
  int intercept = 0;
  int q_dense = 0;    // dense real columns after the pattern (and intercept) in the internal layout
  int slab_max = 0;
  int slab_area = 0;  // doubles of shared memory for a slab, its sentinel and its replicas
  PassHost csr, csc;
};

// The CSR invariants of SparseDesignMatrix._validate (sparse.py:94-117);
// empty string when they hold.
std::string validate_csr(int64_t n, int64_t p, const int64_t* row_ptr, const int32_t* col_idx);

// Validates the CSR (sparse.py:94-117 invariants) and builds both passes for a
// grid of G CTAs.  Returns an empty string on success, else an error message.
std::string build_design(int64_t n, int64_t p, const int64_t* row_ptr, const int32_t* col_idx,
                         int intercept, int slab_max, int G, DesignHost& out, int q_dense = 0,
                         int nranges = kDefaultRanges);

// Native synthetic binary design (bench/test infrastructure): returns nnz.
int64_t synth_binary_design(int64_t n, int64_t p, double rate_lo, double rate_hi, uint64_t seed,
                            std::vector<int64_t>& row_ptr, std::vector<int32_t>& col_idx);

// Host-only check: reconstructs both passes and compares with the CSR.
std::string verify_design(const DesignHost& D, const int64_t* row_ptr, const int32_t* col_idx);

}  // namespace pcgs
