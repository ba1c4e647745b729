// Streaming Matrix Market ingestion straight into the pattern store's CSR
// (host side of the pcgs library).
//
// The reference reads a design with scipy.io.mmread and densifies it
// (pkg/src/priorcg/matrixio.py:48-58), which is infeasible at paper scale.
// Here the file is parsed once, in a single streaming pass through zlib
// (plain and gzip files alike), into (row, col) pairs, then counting-sorted
// into CSR with strictly increasing columns per row -- the invariants
// SparseDesignMatrix._validate checks (sparse.py:94-117).  Values must be
// 0 or 1: explicit zeros are dropped (as densify-then-from_dense drops them),
// anything else is rejected because the store is pattern-only.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace pcgs {

enum MtxField { kMtxPattern = 0, kMtxReal = 1, kMtxInteger = 2 };
enum MtxSymmetry { kMtxGeneral = 0, kMtxSymmetric = 1 };
enum MtxFormat { kMtxCoordinate = 0, kMtxArray = 1 };

enum MtxError { kMtxOk = 0, kMtxIo = 1, kMtxFormat = 2, kMtxUnsupported = 3 };

struct MtxPattern {
  int64_t n = 0, p = 0, entries = 0;  // declared size and entry count
  int field = kMtxPattern, symmetry = kMtxGeneral, format = kMtxCoordinate;
  int64_t zeros_dropped = 0;
  std::vector<int64_t> row_ptr;       // n + 1
  std::vector<int32_t> col_idx;       // nnz, sorted within rows
};

// Parses `path`; on failure returns the MtxError kind and sets `msg`.
int mtx_load(const char* path, MtxPattern& out, std::string& msg);

// Writes a CSR pattern as "coordinate pattern general" (field 0) or
// "coordinate real general" with value 1 (field 1); gzip-compressed if `gz`.
int mtx_write(const char* path, int64_t n, int64_t p, const int64_t* row_ptr, const int32_t* col_idx,
              int field, int gz, std::string& msg);

}  // namespace pcgs
