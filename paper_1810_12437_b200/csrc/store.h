// Pattern-only tiled store for a binary design (host side of the pcgs library).
//
// Layout (both directions share it):
//   * the gathered vector is cut into SLABS that fit one CTA's shared memory
//     (CSR: column slabs of v; CSC: row slabs of w = ω⊙Xv);
//   * every output SEGMENT (CSR: a row within a column slab; CSC: a piece of
//     a column within a row slab) is a run of uint16 slab-local indices padded
//     to a multiple of 8 with the slab's SENTINEL index (which points at a
//     zero in shared memory), so one 16-byte vector never straddles segments;
//   * segments are packed into BUNDLES of one warp's work: either up to 32
//     short segments (one 16-byte vector per lane) or one long segment that
//     the warp walks 32 vectors at a time;
//   * inside a segment the index order is free (the sum is order-independent
//     in exact arithmetic), so the builder permutes indices so that each
//     16-lane half-warp LDS.64 touches 16 distinct shared-memory bank pairs.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace pcgs {

constexpr int kWarps = 16;            // warps per CTA of the pass kernels
constexpr int kThreads = kWarps * 32; // 512
constexpr int kVecIdx = 8;            // uint16 indices per 16-byte vector
constexpr uint32_t kLongFlag = 0x80000000u;

struct Bundle {      // 16 bytes, device-readable as int4
  uint32_t vec_off;  // first vector (units of 8 indices) in the pass stream
  uint32_t seg0;     // first output segment id
  uint32_t mask;     // multi: bit l set when lane l starts a new segment
  uint32_t nvec;     // number of vectors; kLongFlag set for a long bundle
};

struct Task {        // one (slab, bundle range) assignment of a CTA
  int32_t slab;
  int32_t b0, b1;    // bundle range [b0, b1)
  int32_t split;     // offset into warp_split (kWarps + 1 entries)
};

struct PassHost {
  int nslab = 0;
  std::vector<int64_t> slab_lo;      // nslab+1 boundaries in gathered-vector coords
  std::vector<uint16_t> idx;         // nvec * 8 indices
  std::vector<Bundle> bundles;
  int64_t nseg = 0;                  // number of output segments
  // CTA plan
  std::vector<int32_t> cta_task_ptr; // G+1
  std::vector<Task> tasks;
  std::vector<int32_t> warp_split;   // per task: kWarps+1 bundle boundaries
  // CSC only: piece pointer, slab-major: piece_ptr[s*(ncols+1) + j]
  std::vector<int32_t> piece_ptr;
};

struct DesignHost {
  int64_t n = 0, p = 0, p_total = 0, nnz = 0;
  int intercept = 0;
  int slab_max = 0;
  PassHost csr, csc;
};

// Validates the CSR (sparse.py:94-117 invariants) and builds both passes for a
// grid of G CTAs.  Returns an empty string on success, else an error message.
std::string build_design(int64_t n, int64_t p, const int64_t* row_ptr, const int32_t* col_idx,
                         int intercept, int slab_max, int G, DesignHost& out);

}  // namespace pcgs
