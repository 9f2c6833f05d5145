/*
 * kde.h — C ABI of the B200-native all-pairs kernel-sum engine for the bandwidth selectors of
 * Andrzejewski, Gramacki & Gramacki, "Density Estimations for Approximate Query Processing on
 * SIMD Architectures" (arxiv 1505.01998).  P:NNN = PAPER.md line NNN.
 *
 * Conventions (apply to every call below):
 *  - Ownership: the caller owns every buffer.  Sample matrices (X; Y of kde_evaluate) are fp64,
 *    d x n, row-major: dimension a of sample i at X[a*n + i], the paper's layout (P:263-273,
 *    Eq. 19).  They may be DEVICE pointers on the context's GPU or HOST pointers (pageable or
 *    pinned, told apart with cudaPointerGetAttributes): a host array is copied once per call
 *    into a context-owned device buffer on the context stream, and all compute runs on the GPU.
 *    A device pointer of another GPU is KDE_E_INVALID.  Candidate arrays and outputs are HOST
 *    pointers.  (Parameter names keep the _dev suffix of the common, device-resident case.)
 *  - Errors: a call returns KDE_OK or an error code; on error the outputs are untouched and
 *    kde_last_error(ctx) holds a one-line message.  No C++ exception crosses the boundary.
 *    A CUDA or NCCL failure poisons the context (every later call returns the same code).
 *  - Synchronisation: work is enqueued on the context's stream; each call returns after the
 *    host results are available (it synchronises that stream).
 *  - Multi-GPU (SPMD): with world > 1 every rank calls the same function with identical
 *    arguments (each on its own copy of X).  The upper-triangular tile set is split into
 *    round-robin chunks of tile ids across ranks (kde_shard_tiles) and one NCCL all-reduce of exact fixed-point partial sums
 *    combines them, so every rank returns bit-identical results, equal to the 1-GPU result.
 *  - Determinism: results are bit-for-bit reproducible for a given (X, n, d, candidates),
 *    independent of the number of GPUs, the grid size and of which candidates share a batch.
 *  - Limits: 2 <= n <= 2^31-1 (1 <= n for kde_raw_sums), 1 <= d <= 16.
 *  - Threading: a context must not be used from two threads at once.
 */
#ifndef KDE_B200_H
#define KDE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  KDE_OK = 0,
  KDE_E_INVALID = 1,              /* null pointer, bad size, r not in {4,6,8}, non-finite X     */
  KDE_E_NOT_UNIVARIATE = 2,       /* PLUGIN / Psi_r with d != 1                          */
  KDE_E_INSUFFICIENT_SAMPLES = 3, /* n < 2                                                       */
  KDE_E_DEGENERATE = 4,           /* variance estimate <= 0 (all samples equal)       */
  KDE_E_SINGULAR_COV = 5,         /* covariance not positive definite (det Sigma <= 0)    */
  KDE_E_NONPOSITIVE_BW = 6,       /* a candidate h or g <= 0 or non-finite                      */
  KDE_E_DIM_MISMATCH = 7,         /* d out of range for this call                               */
  KDE_E_NUMERIC = 8,              /* Psi6-hat >= 0 or Psi4-hat <= 0 (impossible in exact arith.) */
  KDE_E_NO_FEASIBLE = 9,          /* LSCV_H: no positive-definite vertex to start from          */
  KDE_E_CUDA = 10,
  KDE_E_NCCL = 11,
  KDE_E_OOM = 12
} kde_status;

typedef struct kde_ctx kde_ctx;

/* Intermediate values of the PLUGIN chain, steps 1-8 of P:203-256 (Eq. 11-18). */
typedef struct {
  double V_hat, sigma_hat, psi8_ns, g1, psi6, g2, psi4, h;
} kde_plugin_trace;

typedef enum { KDE_PLUGIN = 0, KDE_LSCV_h = 1, KDE_LSCV_H = 2 } kde_method;

typedef struct {
  int32_t n_grid;        /* LSCV_h: number of h on Z(h0) = [h0/f, f*h0]; 150 */
  double range_factor;   /* LSCV_h: f = 4 (Eq. 27)                                             */
  int32_t max_iter;      /* LSCV_H Nelder-Mead iterations; 500                                   */
  double tol_rel;        /* LSCV_H stop when f_worst - f_best <= tol_rel*|f_best|; 1e-7          */
  double penalty;        /* LSCV_H objective assigned to a non-positive-definite H; 1e300        */
  int32_t speculative;   /* LSCV_H: 1 = evaluate {reflect, expand, contract_out, contract_in} as
                            one GPU batch per iteration; 0 (default) = serial NM, 1-2 GPU rounds of
                            1 candidate per iteration.  Same decisions either way; serial does ~2x
                            fewer evaluations and is ~1.5x faster end to end */
  int32_t refine_steps;  /* LSCV_h: after the grid argmin, up to this many bracket sections (16 new
                            h per step, one GPU pass each) around it ("Golden ratio"); 0 = off */
  double refine_tol;     /* LSCV_h: stop refining when the bracket is narrower than tol * h; 1e-9 */
  int32_t nm_starts;     /* LSCV_H: independent Nelder-Mead runs from vech(H_start) * 4^-k,
                            k < nm_starts, evaluated together in one GPU batch per round; 1 */
  int32_t nm_loop;       /* LSCV_H: 0 = the serial single-start loop runs device-resident on one
                            GPU (one CUDA graph with a conditional WHILE node: decide, whiten,
                            pair kernel per round, no host round trip; same decisions as the host
                            loop); 1 = host loop (one synchronisation per round).  Multi-start,
                            speculative and multi-rank selections always use the host loop; 0 */
  int32_t nm_param;      /* LSCV_H search variables (row f4): 0 = vech(H) with the penalty for
                            non-positive-definite vertices (reading Z8); 1 = vech(L) of a
                            lower-triangular factor, H = L L^T (every vertex is positive semi-definite,
                            only a zero diagonal is penalised), start L = chol(H_start), the initial
                            simplex and the 4^-k start scaling applied to L; host loop; 0 */
} kde_select_opts;

typedef struct {
  kde_method method;
  int32_t d;
  double h;                /* PLUGIN / LSCV_h bandwidth (scalar)                               */
  double vechH[136];       /* LSCV_H: vech of the selected H, d(d+1)/2 entries      */
  double objective;        /* LSCV: g at the selected bandwidth; PLUGIN: 0                      */
  int32_t iterations;      /* LSCV_H Nelder-Mead iterations; LSCV_h: selected grid index        */
  int32_t evaluations;     /* number of objective values computed on the GPU                    */
  int32_t stop_reason;     /* LSCV_H: 1 = tolerance, 2 = max_iter; LSCV_h: refinement steps done */
  kde_plugin_trace trace;  /* PLUGIN only                                                       */
} kde_bandwidth;

/* Exact fixed-point value: value = (hi*2^80 + mid*2^40 + lo) * 2^-scale_exp (see kde_fixed_value).
 * Partial sums from different tiles / ranks add limb-wise without rounding. */
typedef struct {
  int64_t hi, mid, lo;
  int32_t scale_exp;
  int32_t pad_;
} kde_fixed;

/* ---------------------------------------------------------------- context & memory */

/* Create a context on CUDA `device`, enqueuing on `cuda_stream` (a cudaStream_t; NULL = the
 * legacy default stream).  For world > 1, `nccl_unique_id` points to the 128-byte ncclUniqueId
 * rank 0 obtained from kde_nccl_unique_id() and broadcast to all ranks; the library creates its
 * own NCCL communicator (NCCL is loaded at run time, libnccl.so.2).  world == 1 with a non-NULL
 * id creates a single-rank communicator, so the collective path runs (used by the tests); world > 1
 * without an id needs kde_set_host_allreduce before any call that sums pairs. */
kde_status kde_create(kde_ctx **out, int device, void *cuda_stream, const void *nccl_unique_id,
                      int rank, int world);
/* Test transport for world > 1 without NCCL (e.g. several ranks sharing one GPU, where NCCL refuses
 * to run): the library copies each pass's int64 partial sums to pinned host memory and calls
 * fn(data, count, user), which must replace data[] by its element-wise sum over all ranks (e.g. a
 * gloo all-reduce) and return 0; the sums are then copied back.  Only for a context created with
 * world > 1 and no NCCL id.  Production multi-GPU runs use NCCL. */
typedef int (*kde_host_allreduce_fn)(int64_t *data, size_t count, void *user);
kde_status kde_set_host_allreduce(kde_ctx *ctx, kde_host_allreduce_fn fn, void *user);
void kde_destroy(kde_ctx *ctx);
const char *kde_last_error(const kde_ctx *ctx);
/* Fill a 128-byte buffer with a fresh ncclUniqueId (rank 0 only). */
kde_status kde_nccl_unique_id(void *out128);

/* Device workspace the pair-sum calls need for (n, d, n_cand); the caller may provide it with
 * kde_set_workspace (memory stays owned by the caller and must outlive its use); otherwise the
 * context allocates what it needs with cudaMalloc on first use.  The sorted-sample copy (Psi),
 * the per-candidate whitened data sets (LSCV_H, d x n fp32 per candidate, up to 256 candidates or
 * 1 GiB per launch), KDE-evaluation scratch, staged host inputs and the materialised S(v) buffer
 * are always context-owned (freed by kde_destroy). */
size_t kde_workspace_bytes(int64_t n, int32_t d, int32_t n_cand);
kde_status kde_set_workspace(kde_ctx *ctx, void *dev_ptr, size_t bytes);

void kde_default_opts(kde_select_opts *opts);

/* ---------------------------------------------------------------- the five entry points */

/* Psi_r-hat(g_c) for c < n_g, r in {4,6,8}:
 *   Psi_r-hat(g) = [2 sum_{i<j} K^(r)((x_i-x_j)/g) + n K^(r)(0)] / (n^2 g^(r+1)),
 *   K^(r)(u) = He_r(u) exp(-u^2/2)/sqrt(2 pi)   (Eq. 15, Eq. 17; the
 *   diagonal term read inside the bracket, reading Z1).  x_dev: n fp64 (d = 1).
 *   Errors: KDE_E_INVALID (r, n<1, NULL), KDE_E_NONPOSITIVE_BW (g <= 0). */
kde_status kde_psi_r(kde_ctx *ctx, const double *x_dev, int64_t n, int32_t r, const double *g_host,
                     int32_t n_g, double *psi_host);

/* PLUGIN bandwidth (Sec. 4.4.1): V-hat, sigma-hat, Psi8^NS, g1, Psi6-hat(g1), g2,
 * Psi4-hat(g2), h.  Errors: KDE_E_INSUFFICIENT_SAMPLES, KDE_E_DEGENERATE, KDE_E_NUMERIC. */
kde_status kde_plugin_h(kde_ctx *ctx, const double *x_dev, int64_t n, double *h_host,
                        kde_plugin_trace *trace_or_null);

/* LSCV_h objective g(h_c) for c < n_h (Eq. 24-27 / modified Eq. 36-41):
 *   g(h) = h^-d [2 n^-2 sum_{i<j} T((X_i-X_j)/h) + n^-1 R(K)],  T = K*K - 2K with the
 *   Sigma-shaped Gaussian K, R(K) = (4 pi)^{-d/2}|Sigma|^{-1/2} (reading Z2),
 *   Sigma the unbiased sample covariance (Eq. 20-23).
 * Errors: KDE_E_SINGULAR_COV, KDE_E_NONPOSITIVE_BW, KDE_E_INSUFFICIENT_SAMPLES. */
kde_status kde_lscv_h_scores(kde_ctx *ctx, const double *X_dev, int64_t n, int32_t d,
                             const double *h_host, int32_t n_h, double *g_host);

/* LSCV_H objective g(H_c) for c < n_H (Eq. 30-34):
 *   g(H) = 2 n^-2 sum_{i<j} [(K*K)_H - 2 K_H](X_i - X_j) + n^-1 (4 pi)^{-d/2} |H|^{-1/2}.
 * vechH_host: n_H rows of d(d+1)/2 doubles, vech order of P:351-363 (lower triangle, column by
 * column).  A candidate that fails the Cholesky positive-definiteness test gets `penalty`
 * (1e300 when penalty_or_nan is NaN) instead of an error. */
kde_status kde_lscv_H_scores(kde_ctx *ctx, const double *X_dev, int64_t n, int32_t d,
                             const double *vechH_host, int32_t n_H, double penalty_or_nan,
                             double *g_host);

/* Full selector (Sec. 4.4), samples X_dev as for the score calls (device or host fp64,
 * d x n row-major; owned by the caller, read only):
 *   KDE_PLUGIN (d = 1): the chain of Sec. 4.4.1, P:199-256 (out->h, out->trace);
 *   KDE_LSCV_h: h0 of Eq. 25 (reading Z3), grid of opts->n_grid points on
 *     Z(h0) = [h0/f, f h0] (Eq. 27, f = opts->range_factor, readings Z4), argmin of g(h)
 *     (Eq. 28; ties -> smaller h), optional bracket refinement (opts->refine_steps);
 *   KDE_LSCV_H: Nelder-Mead over vech(H) (readings Z8) from H_start of Eq. 35,
 *     non-PD vertices get opts->penalty; opts->nm_starts starts, opts->nm_loop 0 = device-resident
 *     loop when eligible (one GPU, one start).
 * opts_or_null: NULL = kde_default_opts.  out: host struct written on KDE_OK only.
 * Errors: KDE_E_NOT_UNIVARIATE (PLUGIN with d > 1), KDE_E_SINGULAR_COV, KDE_E_NO_FEASIBLE (no PD H
 * found), KDE_E_INVALID (bad options), and those of the score calls. */
kde_status kde_select_bandwidth(kde_ctx *ctx, kde_method method, const double *X_dev, int64_t n,
                                int32_t d, const kde_select_opts *opts_or_null, kde_bandwidth *out);

/* ---------------------------------------------------------------- the paper's own design (f3) */

/* LSCV_h scores by the paper's two-phase algorithm (Sec. 6.2): phase 1 materialises
 * S(v) = v^T Sigma^-1 v for all pairs of this rank's tiles in device memory (the fun2 tile writer
 * of Sec. 5.5, Eq. 44-56; 4 bytes per pair, allocated by the context), phase 2 streams it once per
 * batch of h_per_pass in {1,2,4,8,16} candidates (1 = one pass per h, the paper's grid rows) and
 * reduces Eq. 38-41.  Same values as kde_lscv_h_scores up to rounding; an HBM-bound ablation.
 * kde_last_aux_ms() returns phase 1's device time, kde_last_profile() phase 2's. */
kde_status kde_lscv_h_scores_materialized(kde_ctx *ctx, const double *X_dev, int64_t n, int32_t d,
                                          const double *h_host, int32_t n_h, int32_t h_per_pass,
                                          double *g_host);
double kde_last_aux_ms(const kde_ctx *ctx);

/* ---------------------------------------------------------------- using the bandwidth (f2) */

/* KDE evaluation (Eq. kde-def-H / K_H / gaussian): for each query y_q (column q of
 * the d x m row-major DEVICE array Y_dev),
 *   f_host[q] = n^-1 sum_i |H|^{-1/2} (2 pi)^{-d/2} exp(-1/2 (y_q - X_i)^T H^-1 (y_q - X_i)).
 * vechH_host: d(d+1)/2 doubles; the scalar-h estimator of Eq. kde-def is H = h^2 I.
 * Non-positive-definite H -> KDE_E_NONPOSITIVE_BW.  With world > 1 every rank computes all m
 * values (no collective).  Accuracy: relative 1e-5 (fp32 terms) or, in the far tails, absolute
 * 1e-12 of max fhat: from m n >= 2^32 on, samples and queries are sorted by coordinate 0 and sample
 * tiles farther than sqrt(log2 n + 42) whitened units from a block of queries are skipped, which moves
 * any f_host[q] by at most 2.3e-13 of max fhat. */
kde_status kde_evaluate(kde_ctx *ctx, const double *X_dev, int64_t n, int32_t d, const double *Y_dev,
                        int64_t m, const double *vechH_host, double *f_host);

/* Approximate aggregates over a range, univariate (Eq. count, Eq. sum): for interval
 * q = [lo_host[q], hi_host[q]],  COUNT = n int fhat,  SUM = n int x fhat,  AVG = SUM/COUNT, with
 * fhat the Gaussian KDE of bandwidth h (closed forms of the integrals, fp64).  Any of the three
 * output arrays may be NULL. */
kde_status kde_aqp_1d(kde_ctx *ctx, const double *x_dev, int64_t n, double h, const double *lo_host,
                      const double *hi_host, int32_t n_q, double *count_host, double *sum_host,
                      double *avg_host);

/* ---------------------------------------------------------------- lower level (tests, tools) */

typedef enum {
  KDE_SUM_PSI4 = 4, KDE_SUM_PSI6 = 6, KDE_SUM_PSI8 = 8,  /* 1 sum per candidate g              */
  KDE_SUM_LSCV_h = 1,   /* 2 sums per candidate h: sum e, sum e^2, e = exp(-S(v)/(4h^2))       */
  KDE_SUM_LSCV_H = 2    /* 2 sums per candidate H: sum e, sum e^2, e = exp(-v^T H^-1 v / 4)     */
} kde_sum_kind;

/* The raw pairwise sums RR_fun over the tiles of shard `shard_rank` of `shard_world`
 * (shard_world = 0: this context's own rank/world, all-reduced), as exact fixed-point values:
 *   PSI_r : out[c]       = sum_{i<j} He_r(u) exp(-u^2/2),  u = (x_i - x_j)/g_c
 *   LSCV_h: out[2c+{0,1}] = sum_{i<j} e, e^2 with e = exp(-(X_i-X_j)^T Sigma^-1 (X_i-X_j)/(4h_c^2))
 *   LSCV_H: out[2c+{0,1}] = sum_{i<j} e, e^2 with e = exp(-(X_i-X_j)^T H_c^-1 (X_i-X_j)/4)
 * cand_host: g_c, h_c, or vech(H_c) rows.  Non-PD H_c gives KDE_E_INVALID here. */
kde_status kde_raw_sums(kde_ctx *ctx, kde_sum_kind kind, const double *X_dev, int64_t n, int32_t d,
                        const double *cand_host, int32_t n_cand, int32_t shard_rank,
                        int32_t shard_world, kde_fixed *out);
double kde_fixed_value(const kde_fixed *v);
/* Exact limb-wise sum of two fixed-point values with the same scale_exp. */
kde_fixed kde_fixed_add(kde_fixed a, kde_fixed b);

/* Bounded far-tile skips of the fp32-term passes.  Pure host functions (no GPU).
 * kde_psi_skip_gap: the closed-form (data-independent) threshold tau on the sorted gap min|x_i - x_j|/g
 *   above which a tile of the Psi_r(g) sum (Eq. 15/17) may be skipped, given r in {4,6,8},
 *   g > 0 and the unbiased sample variance var >= 0 (Eq. 11): even if all n^2/2 pairs sat at u = tau, the
 *   skipped terms would sum to at most 1e-9 |Psi-hat_r(g)| (a lower bound on |Psi-hat_r(g)| = R(f^(r/2))
 *   over densities of f's variance, Terrell's maximal smoothing); 13 (only tiles whose fp32 terms are all
 *   exactly 0) when no smaller tau guarantees that, and for bad arguments.  The passes themselves use the
 *   data-aware threshold <= this one (same 1e-9 guarantee from the actual tile gaps; kde_last_psi_gaps).
 * kde_lscv_skip_theta: theta_cf = min(130, log2 n + 30); LSCV tiles are skipped within the budget of
 *   n(n-1)/2 terms e = exp(-S/(4h^2)) <= 2^-theta_cf (Eq. 24/30) — every skipped term
 *   below 2^-theta_cf (Nelder-Mead searches), or a data-aware threshold whose skipped tiles provably stay
 *   within the same total (scores, grid selection, raw sums) — which moves g(h) / g(H) by at most
 *   9.4e-10 (1 + kappa') |g|, kappa' = (A + B)/|g| its cancellation (<= 32 on fp32 terms). */
double kde_psi_skip_gap(int32_t r, double g, double var);
double kde_lscv_skip_theta(int64_t n);

/* Tile traversal (Eq. 42-43, with an exact integer fix-up): linear tile id bx ->
 * column l and row q (q <= l) of the upper-triangular tile grid, column l holding l+1 tiles. */
void kde_tile_coords(int64_t bx, int64_t *l, int64_t *q);

/* The work partition the library uses for a sum of `kind` over n samples in d dimensions
 * (SURVEY §8(e)): tile edge T and the total tiles of the upper-triangular grid (tile ids of Eq.
 * 42-43, column by column).  Rank `rank` of `world` evaluates the tile ids
 *   (c * world + rank) * chunk + w,   c = 0, 1, ...,  0 <= w < chunk,  id < tiles_total
 * (round-robin chunks of *chunk = 16 consecutive ids for world > 1, so that every rank gets the same
 * mix of diagonal, near and exactly-zero tiles on sorted data), *rank_tiles of them; its local index
 * i in [0, *rank_tiles) is tile id kde_shard_tile(i, rank, world).  world = 1: every id, in order.
 * Pure host functions (no GPU needed).  KDE_E_INVALID / -1 for bad arguments. */
kde_status kde_shard_tiles(kde_sum_kind kind, int64_t n, int32_t d, int32_t rank, int32_t world,
                           int32_t *tile_edge, int64_t *tiles_total, int64_t *rank_tiles, int32_t *chunk);
int64_t kde_shard_tile(int64_t i, int32_t rank, int32_t world);

/* Kernel timing of the last call on this context: number of pair-kernel launches, their
 * summed device time (ms, CUDA events on the context stream) and the algorithmic pair-kernel
 * evaluations they performed (pairs i<j on this rank x candidates). */
kde_status kde_last_profile(const kde_ctx *ctx, int32_t *launches, double *pair_ms,
                            double *evals, int32_t *all_launches);
/* Term precision of the Psi_r sums (kde_psi_r, kde_plugin_h, KDE_SUM_PSI* raw sums; Eq. 15/17,
 * P:227-247):
 *   0 (default) automatic: every pass runs with fp32 terms (fp64/exact accumulation, tile-local
 *     centring) and also yields a cancellation estimate kappa = 2A/|2S + n He_r(0)| (A ~ sum|t|);
 *     a pass with kappa > 1e4 is re-run with fp64 terms (for kde_plugin_h the decision is taken on
 *     the device, inside the chain), so Psi-hat stays within 1e-5 for any g > 0.
 *     Shard-only raw sums (shard_world > 0) are never re-run (the decision needs the full sum).
 *   1 = fp64 terms for every pass (libdevice exp, fp64 Horner in u^2), the exact-parity mode.
 *  -1 = fp32 terms only (diagnostics).
 * The same modes govern the LSCV objectives of kde_lscv_h_scores, kde_lscv_H_scores and the LSCV_h
 * grid selection (Eq. 24/30): in mode 0 a candidate whose objective
 * g = A - B + C cancels beyond kLscvKappaMax = 32 ((A + B)/|g|, so the fp32 terms' ~1.5e-7 on the raw
 * sums could exceed 1e-5 on g) is re-run with fp64 terms; mode 1 re-runs every candidate.  Nelder-Mead
 * searches use fp32 terms in modes 0 and -1 (host and device loops decide identically); in mode 1 the
 * search runs on the host loop with fp64 terms for every g(H) (the exact-parity search).  kde_raw_sums
 * always returns fp32-term sums.  The fp32-term passes skip far tiles whose terms are provably
 * negligible (kde_psi_skip_gap, kde_lscv_skip_theta: at most 1e-9 |Psi-hat| resp. 9.4e-10 (1 + kappa') |g|);
 * the fp64-term passes skip only tiles whose terms are exactly 0.
 * Results stay deterministic and partition-invariant in every mode. */
kde_status kde_set_precision(kde_ctx *ctx, int32_t fp64_terms);
/* Number of Psi passes and LSCV candidates of the last call that were (re-)run with fp64 terms, and
 * the largest cancellation estimate kappa of its fp32-term Psi passes (diagnostics). */
int32_t kde_last_fp64_passes(const kde_ctx *ctx);
double kde_last_psi_kappa(const kde_ctx *ctx);
/* Far-tile skip thresholds (in units of g, on the sorted gap) of the last call's fp32-term Psi passes, in
 * pass order: the data-aware bounded threshold (the smallest tau of the grid
 * 6, 6.25, ..., 12.75 whose skipped tiles provably move Psi-hat by at most 1e-9 relative, never above
 * kde_psi_skip_gap), 13 under KDE_DEBUG_SKIP_EXACT=1, inf under KDE_DEBUG_PSI_NOSKIP=1.  Writes at most
 * `max` values to out (host) and returns the number of passes (diagnostics). */
int32_t kde_last_psi_gaps(const kde_ctx *ctx, double *out, int32_t max);
/* Turn per-launch event timing on/off (default off; adds an event pair per launch). */
kde_status kde_set_profiling(kde_ctx *ctx, int32_t on);

#ifdef __cplusplus
}
#endif
#endif /* KDE_B200_H */
