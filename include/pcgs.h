/*
 * pcgs.h — C ABI of the B200-native prior-preconditioned CG sampler path.
 *
 * This is the drop-in boundary for the β-draw hot path of the reference
 * package `priorcg` (arXiv 1810.12437).  The reference is pure Python; its
 * plug-in seam is duck typing (`pcg_solve(phi, ...)` accepts any operator with
 * `.apply`, reference pkg/src/priorcg/cg.py:105-113), so every entry point below
 * replaces one numpy routine of the reference and is bound from Python with
 * ctypes.  All vectors use the reference's column layout:
 * the dense intercept (when present) is coordinate 0, the shrunk block follows
 * (pkg/src/priorcg/sparse.py:314-341, `hstack_dense_columns`).
 *
 * Conventions
 *  - Every function returns PCGS_OK (0) or a negative PCGS_E* code;
 *    pcgs_last_error() returns a thread-local message for the last failure.
 *  - Pointers are DEVICE pointers unless the parameter name ends in `_h`.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  No entry
 *    point synchronises the stream except pcgs_design_create.
 *  - A design handle is immutable after create: it may be used concurrently
 *    from several host threads on distinct streams (the reference's concurrency
 *    model: pure kernels over immutable data).
 */
#ifndef PCGS_H
#define PCGS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PCGS_OK 0
#define PCGS_EINVAL (-1)   /* bad argument (maps to ValueError)            */
#define PCGS_ECUDA (-2)    /* CUDA runtime error                            */
#define PCGS_ENOMEM (-3)   /* device or host allocation failed              */
#define PCGS_EUNSUP (-4)   /* configuration not supported by this build     */
#define PCGS_EFORMAT (-5)  /* malformed input file (maps to FileFormatError) */
#define PCGS_EIO (-6)      /* file cannot be opened/read/written (OSError)  */

/* PCG termination codes written to result[1] by pcgs_pcg (device int32). */
#define PCGS_CONVERGED 0   /* CGReport.termination == "converged"           */
#define PCGS_MAX_ITER 1    /* CGReport.termination == "max_iter"            */
#define PCGS_NOT_PD (-1)   /* NotPositiveDefiniteError, cg.py:157-160       */
#define PCGS_NONFINITE (-2)/* NumericBreakdownError(k), cg.py:141-142,172   */

typedef struct pcgs_design* pcgs_design_t;
typedef struct pcgs_mtx* pcgs_mtx_t;
typedef void* pcgs_stream_t; /* cudaStream_t */

int pcgs_version(void);
const char* pcgs_last_error(void);

/* Build the pattern-only store of a binary design and upload it to `device`.
 * Replaces the CSR container SparseDesignMatrix (sparse.py:46-117) for 0/1
 * designs: values are implicit ones, indices are re-encoded as uint16
 * slab-local offsets (CSR over column slabs, CSC over row slabs).
 *   n, p          rows and SHRUNK columns (the intercept is not counted in p)
 *   row_ptr_h     int64[n+1], host; col_idx_h int32[nnz], host, columns of the
 *                 shrunk block only, strictly increasing within a row
 *   intercept     1 if the design carries the dense all-ones column in front
 *                 (hstack_dense_columns, sparse.py:314-341), else 0
 *   slab_max      0 = automatic (largest slab that fits shared memory); a small
 *                 value forces many slabs (used by the tests)
 * Synchronous.  Returns PCGS_EINVAL for malformed CSR (sparse.py:94-117). */
int pcgs_design_create(int64_t n, int64_t p, const int64_t* row_ptr_h,
                       const int32_t* col_idx_h, int intercept, int slab_max,
                       int device, pcgs_design_t* out);
/* pcgs_design_create with an explicit CTA count for the static plan
 * (0 = one CTA per SM); row-split shards hosted by one grid use SMs / n. */
int pcgs_design_create_ex(int64_t n, int64_t p, const int64_t* row_ptr_h,
                          const int32_t* col_idx_h, int intercept, int slab_max,
                          int device, int grid, pcgs_design_t* out);

/* A design with affine terms: `q_dense` dense real columns
 * (hstack_dense_columns of a real block, sparse.py:314-341) in reference
 * columns intercept .. intercept + q_dense - 1, ahead of the pattern columns
 * (q_dense > 0 needs intercept = 0: a leading ones column is one of the
 * dense columns).  Their values and any standardisation (sparse.py:250-297)
 * are attached with pcgs_design_set_affine. */
int pcgs_design_create_affine(int64_t n, int64_t p, const int64_t* row_ptr_h,
                              const int32_t* col_idx_h, int intercept, int q_dense,
                              int slab_max, int device, int grid, pcgs_design_t* out);
/* Device arrays of the affine terms (owned by the caller, kept alive while the
 * design is used): dense n x q_dense row-major, column means `mu` and scales
 * `sc` in the reference layout (NULL: none).  Every product then applies
 * X_eff = ([P | Dn] - 1 mu') diag(1/sc). */
int pcgs_design_set_affine(pcgs_design_t d, const double* dense, const double* mu,
                           const double* sc);
int pcgs_design_destroy(pcgs_design_t d);
/* Bench/test utility: native synthetic binary design (log-uniform column
 * rates, Binomial row counts; BASELINE config 5 scale).  Call once with
 * col_idx_h = NULL to generate and receive row_ptr_h[n+1] and *nnz_h, then
 * again with a col_idx_h buffer of capacity `cap` to receive the columns. */
int pcgs_synth_design(int64_t n, int64_t p, double rate_lo, double rate_hi, uint64_t seed,
                      int64_t* row_ptr_h, int32_t* col_idx_h, int64_t cap, int64_t* nnz_h);
/* Streaming Matrix Market ingestion (host-only, no GPU), replacing the
 * densifying reader of the reference (matrixio.py:48-79: scipy.io.mmread +
 * toarray, then SparseDesignMatrix.from_dense).  `path` may be plain or gzip.
 * pcgs_mtx_load parses the whole file in one pass into CSR and returns
 * info_h[8] = {n, p, nnz, declared entries, field (0 pattern, 1 real,
 * 2 integer), symmetry (0 general, 1 symmetric), format (0 coordinate,
 * 1 array), explicit zeros dropped}; pcgs_mtx_export copies row_ptr_h[n+1]
 * and col_idx_h[nnz] out (columns strictly increasing per row); pcgs_mtx_free
 * releases the parse.  Values must be 0/1 (PCGS_EUNSUP otherwise: the store
 * is pattern-only); duplicates, out-of-range or missing entries give
 * PCGS_EFORMAT; unreadable files PCGS_EIO. */
int pcgs_mtx_load(const char* path, pcgs_mtx_t* out, int64_t* info_h);
int pcgs_mtx_export(pcgs_mtx_t m, int64_t* row_ptr_h, int32_t* col_idx_h);
int pcgs_mtx_free(pcgs_mtx_t m);
/* Writes a CSR pattern as Matrix Market "coordinate pattern general"
 * (field 0) or "coordinate real general" with value 1 (field 1, what
 * scipy.io.mmwrite writes for the reference's write_design,
 * matrixio.py:35-45); gzip-compressed when gz != 0. */
int pcgs_mtx_write(const char* path, int64_t n, int64_t p, const int64_t* row_ptr_h,
                   const int32_t* col_idx_h, int field, int gz);
/* Host-only: builds the store for a grid of `grid` CTAs and verifies that both
 * tiled passes reproduce the input pattern exactly (no GPU needed).
 * stats_h[8]: csr slabs, csc slabs, csr vectors, csc vectors, csc pieces,
 * shared-memory load groups (slot x half-warp), extra shared-memory
 * wavefronts those groups cost (bank-pair conflicts), index bytes. */
int pcgs_store_selftest(int64_t n, int64_t p, const int64_t* row_ptr_h,
                        const int32_t* col_idx_h, int intercept, int slab_max,
                        int grid, int64_t* stats_h);
/* info_h[16]: n, p, p_total, nnz, csr_slabs, csc_slabs, csr_vectors,
 * csc_vectors, csr_slices, csc_slices, csc_pieces, grid, device,
 * index_bytes (both directions), reserved, reserved */
int pcgs_design_info(pcgs_design_t d, int64_t* info_h);

/* out[n] = X v, v[p_total].  Replaces SparseDesignMatrix.matvec
 * (sparse.py:178-193) for the unstandardised binary design. */
int pcgs_matvec(pcgs_design_t d, const double* v, double* out, pcgs_stream_t stream);

/* out[p_total] = X' w, w[n].  Replaces SparseDesignMatrix.matvec_t
 * (sparse.py:195-203). */
int pcgs_matvec_t(pcgs_design_t d, const double* w, double* out, pcgs_stream_t stream);

/* out = X' (omega ⊙ X v) + prior_diag ⊙ v.  Replaces PrecisionOperator.apply
 * (sampler.py:53-58). */
int pcgs_phi_apply(pcgs_design_t d, const double* omega, const double* prior_diag,
                   const double* v, double* out, pcgs_stream_t stream);

/* out[p_total] = X' (omega) + prior_diag: the diagonal of Phi for a binary
 * design (gram_diagonal, sparse.py:235-246, plus the prior; the Jacobi
 * preconditioner's M of precond.py:105-117). */
int pcgs_phi_diagonal(pcgs_design_t d, const double* omega, const double* prior_diag,
                      double* out, pcgs_stream_t stream);

/* Randomised right-hand side (generate_rhs, sampler.py:94-107, with the linear
 * term of GaussianTarget.from_pseudo_outcome, sampler.py:86-91):
 *   b = X'(kappa + sqrt(omega) ⊙ eta) + sqrt(prior_diag) ⊙ delta
 * kappa may be NULL (zero); `linear` (p_total, may be NULL) is added as the
 * target's precomputed linear term.
 * eta[n] / delta[p_total] are taken from the given device arrays when non-NULL
 * (host-noise injection: the reference's stream order, eta then delta), else
 * drawn on device from Philox4x32-10 keyed by (seed, stream_id). */
int pcgs_rhs(pcgs_design_t d, const double* kappa, const double* omega,
             const double* prior_diag, const double* linear, const double* eta,
             const double* delta, uint64_t seed, uint64_t stream_id, double* b,
             pcgs_stream_t stream);

/* Prior-preconditioned CG on Phi = X'ΩX + diag(prior_diag), the whole loop on
 * device in one persistent cooperative kernel (pcg_solve, cg.py:105-192).
 *   minv[p_total]   diagonal of M^-1 (Preconditioner.inv_diagonal)
 *   scale[p_total]  termination metric scale s (cg.py:89-102)
 *   x               in: x0, out: solution
 *   trace[max_iter+1], alphas[max_iter], betas[max_iter]: device outputs
 *   result[4] (device int32): iterations, termination code, failing
 *   iteration, operator applications.  Nothing is synchronised. */
int pcgs_pcg(pcgs_design_t d, const double* omega, const double* prior_diag,
             const double* minv, const double* scale, const double* b, double* x,
             int32_t max_iter, double rtol, double* trace, double* alphas,
             double* betas, int32_t* result, pcgs_stream_t stream);

/* pcgs_pcg with trace_level "full" (cg.py:143-146, 167-169): iterates
 * [max_iter+1][p_total] (device, reference layout) receives x0 and every
 * iterate; NULL = off. */
int pcgs_pcg_full(pcgs_design_t d, const double* omega, const double* prior_diag,
                  const double* minv, const double* scale, const double* b, double* x,
                  int32_t max_iter, double rtol, double* trace, double* alphas,
                  double* betas, double* iterates, int32_t* result, pcgs_stream_t stream);

/* Generic-operator PCG (pcg_solve with a duck-typed operator, cg.py:105-113):
 * the same loop, vector algebra on device, Phi supplied by a callback
 * fn(ctx, v, out) on device buffers of length p (returns 0 on success).
 * dbuf/adbuf (may be NULL): caller-owned device buffers used as the search
 * direction and its product, so a device-side callback (e.g. the row-sharded
 * operator with its allreduce) can address them without copies.
 * trace_h/alphas_h/betas_h/result_h are HOST arrays; synchronises every
 * iteration (desk-scale path, used by the reference's operator tests). */
typedef int (*pcgs_apply_fn)(void* ctx, const double* v, double* out);
int pcgs_pcg_op(pcgs_apply_fn fn, void* ctx, int64_t p, const double* minv,
                const double* scale, const double* b, double* x, double* dbuf,
                double* adbuf, int32_t max_iter, double rtol, double* trace_h,
                double* alphas_h, double* betas_h, int32_t* result_h,
                pcgs_stream_t stream);

/* pcgs_pcg_op with trace_level "full": iterates [max_iter+1][p] (device). */
int pcgs_pcg_op_full(pcgs_apply_fn fn, void* ctx, int64_t p, const double* minv,
                     const double* scale, const double* b, double* x, double* dbuf,
                     double* adbuf, int32_t max_iter, double rtol, double* trace_h,
                     double* alphas_h, double* betas_h, double* iterates,
                     int32_t* result_h, pcgs_stream_t stream);

/* Synchronous copy helper for operator callbacks: kind 0 host->device,
 * 1 device->host, 2 device->device. */
int pcgs_copy(void* dst, const void* src, int64_t bytes, int kind);

/* Debug: device buffer (>= 256 uint64) receiving CTA-0 phase timestamps
 * (globaltimer ns; 4 per operator application) of subsequent pcgs_pcg calls;
 * NULL disables. */
int pcgs_debug_profile(void* buf);
/* Debug/tuning switches: key 1 = debug bits of the pass kernels (64: per-CTA
 * pass timestamps, 128: barrier trace of PCG iteration 10), key 2 = L2
 * persisting window over the CSC index stream in MB (0 = off), key 3 = warp
 * ranges per CTA task of the stores created from now on (0 = the default 16,
 * the persistent PCG kernel's warp count; the row-split shards use 32). */
int pcgs_debug_option(int key, int value);
/* Debug: device buffer (3 uint64 per CTA) for per-CTA pass timestamps when
 * the debug-option key 1 bit 64 is set. */
int pcgs_debug_cta_times(void* buf);
/* Debug: device buffer (16 uint64 per CTA) receiving, for PCG iteration 10,
 * each CTA's arrival / departure times at the four grid barriers of an
 * iteration ([0..7]) and stamps inside the step phase ([8..12]) when the
 * debug-option key 1 bit 128 is set. */
int pcgs_debug_sync_times(void* buf);

/* ------------------------------------------------------------------------
 * Row-split PCG (replaces the per-application
 * allreduce of parallel.ShardedPrecisionOperator around cg.py:105-192).
 * Rows of X are split into contiguous shards, one per rank; p-vectors are
 * replicated.  One persistent kernel per GPU runs the whole solve; the X'w
 * pieces of every rank are exchanged inside the kernel over peer memory
 * (one exchange barrier per iteration, no NCCL call).  A context hosts
 * n_local consecutive ranks [rank0, rank0 + n_local) of nranks on one GPU:
 * n_local == nranks runs every shard in one grid (single-GPU emulation),
 * n_local == 1 is one rank per GPU, the other ranks' exchange regions mapped
 * with CUDA IPC (pcgs_rs_exchange_handle on the owner, pcgs_rs_open_peer on
 * every other rank).  Local shard designs must be created with the same grid
 * (pcgs_design_create_ex) and columns.
 * ------------------------------------------------------------------------ */
typedef struct pcgs_rs* pcgs_rs_t;
int pcgs_rs_create(const pcgs_design_t* designs, int n_local, int rank0, int nranks,
                   pcgs_rs_t* out);
/* 64-byte cudaIpcMemHandle_t of local rank `local`'s exchange region. */
int pcgs_rs_exchange_handle(pcgs_rs_t rs, int local, void* handle_h);
int pcgs_rs_open_peer(pcgs_rs_t rs, int rank, const void* handle_h);
/* pcgs_pcg over the row shards: omegas_h[l] = device omega of local rank l
 * (shard rows); prior_diag, minv, scale, b, x (x0 in, solution out), trace,
 * alphas, betas, result as pcgs_pcg (device), replicated on every rank.
 * Asynchronous; every rank of the solve must launch it. */
int pcgs_rs_pcg(pcgs_rs_t rs, const double* const* omegas_h, const double* prior_diag,
                const double* minv, const double* scale, const double* b, double* x,
                int32_t max_iter, double rtol, double* trace, double* alphas,
                double* betas, int32_t* result, pcgs_stream_t stream);
/* Exchange protocol of a context whose ranks are all hosted by one grid
 * (n_local == nranks), set before the first solve: 0 = the grid barrier
 * (default); 1 = flag validation mode, in which every hosted group behaves
 * as an independent rank -- barriers over its own CTAs only, and at every
 * exchange the cross-GPU protocol of n_local = 1 contexts (st.release.sys of
 * the epoch into every peer's inbox, ld.acquire.sys spins, volatile peer
 * loads, the scalar exchange by flags).  The grid is one cooperative launch,
 * so the groups are co-resident and the protocol runs on one GPU; results
 * are bitwise those of mode 0. */
int pcgs_rs_set_exchange(pcgs_rs_t rs, int mode);
int pcgs_rs_destroy(pcgs_rs_t rs);

/* omega[i] ~ PG(1, z[i]) (pg_draw_batch, polya_gamma.py:39-84), Philox keyed
 * by (seed, stream_id), one thread per draw. */
int pcgs_pg_draw(const double* z, int64_t n, uint64_t seed, uint64_t stream_id,
                 double* omega, pcgs_stream_t stream);
/* pcgs_pg_draw over a row shard whose first row is global row `row0`: the
 * draws are those of the unsharded call (Philox element = global row). */
int pcgs_pg_draw_rows(const double* z, int64_t n, int64_t row0, uint64_t seed,
                      uint64_t stream_id, double* omega, pcgs_stream_t stream);

/* ------------------------------------------------------------------------
 * Device Gibbs scan (gibbs_run, gibbs.py:260-379).  All pointers are device
 * arrays owned by the caller; vectors of length p_total use the reference
 * layout (unshrunk block first).  One pcgs_gibbs_scan call issues one scan on
 * `stream` without synchronising: omega -> tau -> lambda -> beta (RHS + PCG)
 * -> X beta + log density -> Welford statistics and the stored draw.
 * ------------------------------------------------------------------------ */
typedef struct {
  int prior;          /* 0: bridge alpha = 1 (reference), 1: horseshoe        */
  int q;              /* leading unshrunk coefficients                       */
  int precond;        /* 0 prior (augmented), 1 identity, 2 Jacobi          */
  int fixed_omega, fixed_tau, fixed_lam; /* pinned updates (gibbs.py:321-329) */
  int max_iter;       /* CG iteration cap                                    */
  double rtol;        /* CG RMS stopping threshold                           */
  double a0, b0;      /* bridge: Gamma(a0, b0) prior on tau^-alpha          */
  double alpha;       /* bridge exponent (local updates need alpha = 1)     */
  double gamma_scale; /* gamma policy constant c (precond.py:137)           */
  uint64_t seed;      /* Philox key of the chain                             */
  const double* y;        /* n outcomes (0/1)                                */
  const double* kappa;    /* n: y - 1/2                                      */
  const double* usd_prec; /* q prior precisions of the unshrunk block (0 flat) */
  const double* usd_sd;   /* q prior sds (inf = flat), gamma cold start       */
  double* beta;       /* p_total: current draw (in: previous draw)           */
  double* z;          /* n: X beta                                           */
  double* omega;      /* n                                                   */
  double* lam;        /* p: local scales                                     */
  double* nu;         /* p: horseshoe auxiliaries                            */
  double* scal;       /* [0] tau, [1] xi (horseshoe auxiliary)               */
  double* mean;       /* p_total: running mean of scaled draws               */
  double* m2;         /* q: running sum of squares of the unshrunk draws     */
  double* prior_diag; double* minv; double* scale; double* b; /* p_total work */
  double* part;       /* 16 * grid: per-CTA partial sums                     */
  double* logdens;    /* n_iter                                              */
  int32_t* results;   /* 8 per scan: PCG result[4], [4] positivity violation */
  double* draws;      /* n_store x p_total                                   */
  double* tau_draws;  /* n_store                                             */
  double* trace; double* alphas; double* betas; /* PCG scratch (max_iter+1) */
  /* Standardised designs (SparseDesignMatrix.standardize, sparse.py:250-297):
   * NULL for a raw design.  Otherwise p_total column scales s_j (1 for the
   * intercept and unstandardised columns) and the scan samples the exact
   * reparametrisation b~_j = b_j / s_j, b~_0 = b_0 - sum_j mu_j b_j / s_j,
   * for which X_s b = X b~ on the raw pattern: beta, mean, m2 and draws hold
   * b~ (the host maps draws back); the scale updates, log prior and tau sums
   * use b_j = s_j b~_j, and the prior / preconditioner / metric are those of
   * b~ (precision s_j^2 / (tau lam_j)^2).  Needs an unstandardised intercept
   * with a flat prior as coefficient 0. */
  const double* cscale;
} pcgs_gibbs_t;

/* Validation entry point for the scale updates of the scan (the same device
 * functions k_global / k_local call; replaces the reference's
 * update_global_scale gibbs.py:179-190 and update_local_scales gibbs.py:193-214
 * as a unit under test, mirroring test_gibbs.py:114-140).  prior 0 bridge,
 * 1 horseshoe.  mode 0: `count` independent global draws from the sum
 * `b_or_acc` (bridge: sum |beta|^alpha; horseshoe: sum beta^2/lam^2) over p
 * coefficients and tau_old = `tau`, out = tau, aux = xi (horseshoe);
 * mode 1: `count` independent local draws of one coefficient b = `b_or_acc`
 * given tau and lam_old, out = lam, aux = nu (horseshoe);
 * mode 2 / 3: one thread iterating the global / local update `count` times
 * (the auxiliary-variable Gibbs chain), out = the chain of tau / lam. */
int pcgs_scale_draws(int prior, int mode, int64_t count, double b_or_acc, double tau,
                     double lam_old, int64_t p, double a0, double b0, double alpha,
                     uint64_t seed, double* out, double* aux, pcgs_stream_t stream);

/* z = X beta and its log-likelihood partials (start of a chain / resume). */
int pcgs_gibbs_init(pcgs_design_t d, pcgs_gibbs_t* g, pcgs_stream_t stream);
/* Scan t (1-based).  `count` = number of statistics updates so far; `slot` =
 * row of `draws` to store this scan in, or -1. */
int pcgs_gibbs_scan(pcgs_design_t d, pcgs_gibbs_t* g, int32_t t, int32_t count,
                    int32_t slot, pcgs_stream_t stream);
/* The same scan in two halves, for a host-side local-scale update between
 * them (gibbs_run's local_scale_sampler hook, gibbs.py:262, 311, 328-329):
 * begin = omega and tau; end = lambda (unless fixed_lam), RHS, PCG, X beta,
 * statistics, log density. */
int pcgs_gibbs_scan_begin(pcgs_design_t d, pcgs_gibbs_t* g, int32_t t,
                          pcgs_stream_t stream);
int pcgs_gibbs_scan_end(pcgs_design_t d, pcgs_gibbs_t* g, int32_t t, int32_t count,
                        int32_t slot, pcgs_stream_t stream);

/* Row-split Gibbs scan (gibbs_run over row shards):
 * `g` holds the replicated state (p-vectors, scalars, outputs; its part
 * buffer has 16 * (grid + 1) doubles) and rows[l] the rows of local rank l.
 * Bitwise identical replicated state on every rank; the draws of omega and
 * of the RHS noise are keyed by global row, as in the unsharded scan.
 * Prior / identity preconditioners, unstandardised designs. */
typedef struct {
  const double* y;      /* shard outcomes (0/1)                               */
  const double* kappa;  /* shard y - 1/2                                      */
  double* z;            /* shard X beta                                       */
  double* omega;        /* shard Polya-Gamma draws                            */
  double* part;         /* 16 * grid: the shard's per-CTA partial lines       */
} pcgs_rs_rows_t;
int pcgs_rs_gibbs_init(pcgs_rs_t rs, pcgs_gibbs_t* g, const pcgs_rs_rows_t* rows,
                       pcgs_stream_t stream);
int pcgs_rs_gibbs_scan(pcgs_rs_t rs, pcgs_gibbs_t* g, const pcgs_rs_rows_t* rows,
                       int32_t t, int32_t count, int32_t slot, pcgs_stream_t stream);

/* ------------------------------------------------------------------------
 * Batched independent chains (BASELINE config 4): R chains share
 * one walk over the pattern (pattern-only SpMM with R right-hand sides)
 * through a SLICED store: a warp is 32/R slots of R lanes, lane (slot, c)
 * sums chain c of one output piece.  Device vectors are chain-minor:
 * element (j, c) at [j * R + c], reference coordinates (intercept first);
 * R in {2, 4, 8}.  Replaces, per chain, PrecisionOperator.apply
 * (sampler.py:53-58) and pcg_solve (cg.py:105-192).
 * ------------------------------------------------------------------------ */
typedef struct pcgs_batch* pcgs_batch_t;
/* Validates the CSR (sparse.py:94-117) and builds the sliced store for
 * `nchains` chains on `device`, planned for `grid` CTAs (0: one per SM);
 * slab_max 0 = the largest slab the chains fit in shared memory. */
int pcgs_batch_create(int64_t n, int64_t p, const int64_t* row_ptr_h,
                      const int32_t* col_idx_h, int intercept, int nchains,
                      int slab_max, int device, int grid, pcgs_batch_t* out);
int pcgs_batch_destroy(pcgs_batch_t b);
/* info[16]: n, p, p_total, nnz, csr/csc slabs, csr/csc vectors, csr/csc
 * pieces, nchains, grid, device, index bytes, slab_max, bank-conflict ppm. */
int pcgs_batch_info(pcgs_batch_t b, int64_t* info);
/* Host-only: builds the sliced store and rebuilds the pattern from it
 * (stats[9]: slabs, vectors, pieces, LDS groups, conflict excess, padding). */
int pcgs_batch_selftest(int64_t n, int64_t p, const int64_t* row_ptr_h,
                        const int32_t* col_idx_h, int intercept, int nchains,
                        int slab_max, int grid, int64_t* stats);
/* Debug: device buffer of 8 * 64 uint64 that pcgs_batch_pcg fills with
 * %globaltimer stamps of the phases of its first 64 iterations (NULL: off). */
int pcgs_batch_debug_profile(void* buf);
/* out_c = X'(Omega_c X v_c) + D_c v_c for every chain c. */
int pcgs_batch_phi_apply(pcgs_batch_t b, const double* omega, const double* prior_diag,
                         const double* v, double* out, pcgs_stream_t stream);
/* Per-chain PCG in one persistent kernel; chains that finish are masked.
 * trace[c*(max_iter+1)+k], alphas/betas[c*max_iter+k],
 * result[c*4 + {iterations, status, fail_iter, applies}]. */
int pcgs_batch_pcg(pcgs_batch_t b, const double* omega, const double* prior_diag,
                   const double* minv, const double* scale, const double* rhs, double* x,
                   int32_t max_iter, double rtol, double* trace, double* alphas,
                   double* betas, int32_t* result, pcgs_stream_t stream);

/* One Gibbs scan t of R = nchains batched chains (BASELINE config 4): every
 * chain's own omega, tau, lambda and RHS (as pcgs_gibbs_scan), the R beta
 * solves in one batched PCG on `b` (pcgs_batch_pcg), then every chain's
 * X beta, statistics and log density.  gs[c] are the chains' states on design
 * `d` (same pattern as `b`), sharing max_iter and rtol; counts[c] / slots[c]
 * as in pcgs_gibbs_scan.  Replaces R calls of the reference's scan
 * (gibbs.py:300-369). */
int pcgs_batch_gibbs_scan(pcgs_design_t d, pcgs_batch_t b, pcgs_gibbs_t* const* gs,
                          int32_t nchains, int32_t t, const int32_t* counts,
                          const int32_t* slots, pcgs_stream_t stream);

/* Scans t_first .. t_last of R = nchains batched chains in ONE persistent
 * kernel (BASELINE config 4): each chain runs whole Gibbs scans at its own
 * pace -- its omega / tau / lambda / RHS updates, its PCG solve, its
 * statistics and log density -- while the batch walks the pattern once per
 * iteration for all chains, so a chain whose solve finishes starts its next
 * scan instead of waiting for the slowest (gibbs.py:300-369 per chain, the
 * RNG keys of pcgs_gibbs_scan).  gs[c] as for pcgs_batch_gibbs_scan (prior
 * preconditioner, no pinned updates, no reparametrisation); counts[c] /
 * stored[c] = statistics updates / stored draws before t_first; out_state
 * (device, 2 per chain) receives them after t_last. */
int pcgs_batch_gibbs_run(pcgs_batch_t b, pcgs_gibbs_t* const* gs, int32_t nchains,
                         int32_t t_first, int32_t t_last, int32_t burn_in, int32_t thin,
                         const int32_t* counts, const int32_t* stored, int32_t* out_state,
                         pcgs_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* PCGS_H */
