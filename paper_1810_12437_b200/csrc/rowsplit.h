// Internal interface of the row-split context (csrc/rowsplit.cu) for the
// row-split Gibbs scan (csrc/gibbs.cu); not part of the C ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "pcgs.h"

struct RsSolve {                 // one row-split PCG call
  const double* const* omegas;   // per local rank (shard rows)
  const double* const* kappas;   // per local rank, or null: b is given
  uint64_t seed, stream_id;      // RHS noise keys (kappas != null)
  double* b_out;                 // RHS written here (kappas != null), may be null
  const double *diag, *minv, *scale, *b;
  double* x;
  int32_t max_iter;
  double rtol;
  double *trace, *alphas, *betas;
  int32_t* result;
};

int rs_solve(pcgs_rs_t R, const RsSolve& S, cudaStream_t s);
// *out = sum over every rank's CTAs of parts[l][c * 16] (c < the shard grid)
int rs_sum(pcgs_rs_t R, const double* const* parts, double* out, cudaStream_t s);
int rs_local(pcgs_rs_t R, int l, pcgs_design_t* d, int64_t* row0);
int rs_n_local(pcgs_rs_t R);
int rs_grid(pcgs_rs_t R);
