// kde_internal.h — declarations shared by the host library (kde_*.cpp) and the CUDA
// launchers (kde_psi.cu, kde_lscv_*.cu, kde_eval.cu, kde_materialized.cu, kde_nm_dev.cu).  Product code
// only; nothing here is shared with oracle/.
#pragma once
#include <cmath>
#include <cstdint>
#include <cuda_runtime.h>

namespace kde {

constexpr int kThreads = 256;          // threads per CTA of every pair kernel
constexpr int kMaxCand = 32;           // candidates per pair-kernel launch (upper bound)
constexpr int kMaxDim = 16;

// Fixed-point limbs of one output value on the device: value*2^S = hi*2^80 + mid*2^40 +
// (unsigned) lo + carry*2^64.  Every tile commit adds |hi|, |mid|, |lo| < 2^40 (sign-magnitude
// split); hi and mid stay far from overflow because the a-priori bound caps the sum of |commits|
// at 2^100, and lo's unsigned wrap-arounds are counted in the carry limb (add_limbs), so the
// value is exact for any number of commits (n up to 2^31).  Readers fold the carry; before a
// cross-rank sum each rank's limbs are normalised (normalize_limbs) so the int64 sums cannot wrap.
constexpr int kLimbs = 4;
constexpr int kMaxDevices = 64;   // per-device caches of one-time kernel setup
constexpr int kWorkCounters = 1024;   // dynamic-scheduling counters the workspace holds after the limbs

// Current CUDA device (per-device caches: the dynamic shared-memory opt-in is a device attribute).
inline int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d < 0 || d >= kMaxDevices ? 0 : d;
}

// Which functor a launch runs.
enum class Kind : int { Psi4 = 4, Psi6 = 6, Psi8 = 8, LscvScalar = 1, LscvMatrix = 2 };

// Per-launch parameters (copied into the kernel parameter space = constant bank).
struct PsiParams {
  // He_r coefficients are compile-time; see FPsi (kde_pair.cuh) for the exponent scheme.
  double fac[16];    // 2^((r-1) c0 - o_k), exact in fp64 (applied at the fp64 flush)
  float o[16];       // class k = 8 * (tile parity) + row slot: o_k = fp32((r-1) c0 - 16 - k/16); aligned pairs
  float c0;          // fp32(-log2(e)/2): exp(-s/2) = 2^(s c0)
};
struct LscvScalarParams {
  float kappa[kMaxCand];   // -1/h_c^2 (data pre-scaled by sqrt(log2 e / 4) L^-1)
  float smax[kMaxCand];    // 125 / |kappa_c|: software-exp clamp on s (exp2_sw2_fma)
  // Per-candidate far-tile bound on s (lscv_skip_s of this candidate alone): a tile whose coordinate-0
  // gap g has fp32(g^2) > skip_c[c] adds nothing to candidate c, whether or not the whole tile is
  // skipped for its batch, so a candidate's sums do not depend on the batch it travels in.
  float skip_c[kMaxCand];
};
// Tiles whose sorted gap min|y_i - y_j| exceeds these contribute exactly 0 and are skipped:
// fp32 path: MUFU input <= -0.72 s - 16 < -126 (flushed to 0) for s > 152.5; fp64: exp(-s/2)
// underflows to 0 for s > 1490.4.
constexpr double kPsiSkipGap32 = 13.0, kPsiSkipGap64 = 40.0;
// (KDE_DEBUG_PSI_NOSKIP=1 in the environment disables the skip: results are bit-identical.)
double psi_skip_gap(bool fp64);

// Bounded far-tile skip.  The fp32-term passes also skip tiles whose terms are not
// exactly 0 but provably negligible: at most kSkipEps relative to the result.
//   Psi: (-1)^{r/2} Psi-hat_r(g) = R(f^(r/2)) exactly, f = the KDE of the sample with bandwidth g/sqrt(2)
//   (Eq. 15/17 with the diagonal, reading Z1), a density of variance V_b + g^2/2 <= V + g^2/2.  Among
//   densities of variance v, R(f^(s)) >= R*_s v^{-(2s+1)/2}, attained by f ~ (1 - x^2/((2s+5)v))^{s+1}
//   (Terrell 1990, maximal smoothing; R*_2 = 35/243).  Every dropped pair has u >= tau and
//   |He_r(u)| e^{-u^2/2} <= tau^r e^{-tau^2/2} (tau >= 6), there are at most n^2/2 of them, so
//   |dropped| / |Psi-hat| <= tau^r e^{-tau^2/2} / (sqrt(2 pi) R*_s q^{(r+1)/2}), q = g^2 / (V + g^2/2);
//   psi_bounded_gap returns a tau <= kPsiSkipGap32 that makes this <= kSkipEps (the smallest, from
//   above, to Newton's accuracy).
//   LSCV (Eq. 24/30, g = A - B + C, C = c4/n the diagonal term): every dropped term e <= 2^-theta, at
//   most n^2/2 of them, so |dA| <= c4 2^-theta = C n 2^-theta; theta = log2 n + 30 (lscv_skip_theta)
//   gives |dA| <= 2^-30 C <= 9.4e-10 (1 + kappa') |g|, kappa' = (A + B)/|g|: at most 0.6% of the
//   fp32 terms' own ~1.5e-7 kappa'.
// KDE_DEBUG_SKIP_EXACT=1 keeps only the exact-zero skips (bit-identical to no skip at all).
constexpr double kSkipEps = 1e-9;
#ifdef __CUDACC__
#define KDE_HDI __host__ __device__ inline
#else
#define KDE_HDI inline
#endif
// log of the per-pair target kSkipEps sqrt(2 pi) R*_{r/2} q^{(r+1)/2}, q = g^2/(var + g^2/2): n^2 times the
// target is kSkipEps times Terrell's lower bound on |2S + n He_r(0)| = n^2 g^{r+1} sqrt(2 pi) |Psi-hat_r(g)|.
KDE_HDI double psi_skip_log_target(int r, double g, double var) {
  const double Rs = r == 4 ? 35.0 / 243.0
                           : (r == 6 ? 14175.0 * sqrt(11.0) / 161051.0 : 1091475.0 * sqrt(13.0) / 4826809.0);
  const double q = g * g / (var + 0.5 * g * g);
  return log(kSkipEps * 2.5066282746310002 * Rs) + 0.5 * (r + 1) * log(q);
}
KDE_HDI bool psi_skip_args_ok(double g, double var) {
  return g > 0.0 && var >= 0.0 && var < 1e300 && g < 1e150;
}
// Closed form (data-independent): every one of the n^2/2 pairs could sit at u = tau.
KDE_HDI double psi_bounded_gap(int r, double g, double var) {
  if (!psi_skip_args_ok(g, var)) return kPsiSkipGap32;
  const double lt = psi_skip_log_target(r, g, var);
  // f(tau) = r log tau - tau^2/2 - lt is concave and decreasing for tau > sqrt(r): Newton from the right
  // of the root stays right of it (tangents lie above a concave f), so every iterate satisfies f <= 0.
  double t = kPsiSkipGap32;
  if (r * log(t) - 0.5 * t * t - lt > 0.0) return kPsiSkipGap32;
  for (int it = 0; it < 8; ++it) {
    const double f = r * log(t) - 0.5 * t * t - lt, fp = r / t - t;
    const double tn = t - f / fp;
    if (!(tn < t) || tn < 6.0) break;
    const bool done = t - tn < 1e-9;   // quadratic convergence: 4-5 steps from 13
    t = tn;
    if (done) break;
  }
  return t;
}
// Data-aware threshold: up to 296 CTAs (fixed shares of the tile ids) and one
// finalising warp, in a fixed order, bound, for each tau of the grid 6, 6.25, ..., 12.75, the
// terms of the tiles a pass would skip, sum over tiles (l, q < l) with sorted gap > tau of
// 2 T cols(l) gap^r e^{-gap^2/2} (each pair of such a tile has u >= gap >= 6), and writes to *out the
// smallest tau whose bound is at most n^2 e^{psi_skip_log_target} (kSkipEps of Terrell's lower bound), or
// the closed form psi_bounded_gap if that is smaller.  y = the pass's sorted scaled samples (launch_psi_prep),
// g and var from device memory (g_dev, var_dev) or the values.  Deterministic (fixed order).
cudaError_t launch_psi_gap_select(int r, const double* y, int64_t n, int T, const double* g_dev, double g_val,
                                  const double* var_dev, double var_val, double* out, double* scratch,
                                  cudaStream_t s);   // scratch: 296 x 28 doubles (two launches)
// LSCV_H sets, data-aware bounded skip: one CTA per prepared set (whitened coordinate
// 0 at X + s * set_stride, sorted) bounds what a pass drops for each theta of the grid theta_cf,
// theta_cf - 1, ..., 8 — sum over tiles (l, q < l) with fp32(g^2) > theta of T cols(l) 2^-fp32(g^2), the
// pair kernel's own skip test — and writes to out[s] the smallest theta whose bound is at most
// n(n-1)/2 2^-theta_cf (the closed form's worst case, so the objective bound is unchanged).
cudaError_t launch_lscv_sets_skip_select(const float* X, int64_t set_stride, int n_sets, int64_t n, int T,
                                         float theta_cf, float* out, cudaStream_t s);
// LSCV_h, data-aware bounded skip: one CTA per candidate c (kappa[c] < 0, device) on the prepared data's
// coordinate 0 (sorted); bounds on s are fp32(theta/|kappa_c|) for theta = theta_cf, theta_cf - 1, ..., 8
// and the bound on what candidate c drops is the sum over tiles with fp32(g^2) > that of
// T cols(l) 2^(kappa_c g^2) (x 1.0001: the kernel's fp32 exponent); out[c] = the smallest admissible bound
// within n(n-1)/2 2^-theta_cf.
cudaError_t launch_lscv_h_skip_select(const float* X0, int64_t n, int T, const float* kappa, int n_cand,
                                      float theta_cf, float* out, cudaStream_t s);
// Below this many tiles per side the selection is not run (a few tiles hardly skip; small-n latency) and
// the pass keeps the exact-zero threshold.
constexpr int64_t kGapSelectMinTiles = 16;
// Psi skip threshold of one pass: bounded (default), exact-zero (KDE_DEBUG_SKIP_EXACT=1) or none
// (KDE_DEBUG_PSI_NOSKIP=1).  Host only (reads the environment at every call).
double psi_skip_gap_for(int r, double g, double var);
bool skip_bounded();   // false under KDE_DEBUG_SKIP_EXACT=1

struct LaunchCfg {
  const float* X;          // D rows of ld floats (fp32, prepared), device
  int64_t n, ld;           // samples, padded row length (multiple of the tile)
  // this launch's tiles: local indices [tile_begin, tile_end) of rank part_rank of part_world
  // (kde_tiles.cuh shard_tile: round-robin chunks; world 1 = the tile ids themselves)
  int64_t tile_begin, tile_end;
  int part_rank = 0, part_world = 1;
  int tile;                // tile edge T (rows = columns)
  int scale_exp;           // fixed-point exponent S
  unsigned long long* limbs;   // [n_out][3] accumulators, device
  int n_out;               // outputs written per data set by this launch
  cudaStream_t stream;
  int sm_count;
  const unsigned long long* clamp = nullptr;   // Psi: device flag "some |x'| > 3e4"
  // Several prepared data sets (LSCV_H: one per candidate) in one launch: set s lives at
  // X + s * set_stride and writes outputs [s * n_out, (s + 1) * n_out); work unit = (set, tile).
  int n_sets = 1;
  int64_t set_stride = 0;  // floats
  // Psi (tile-local centring): X holds fp32(y_j - c_l) per column tile l, Y64 the
  // fp64 scaled sorted samples y (rows are formed as fp32(y_i - c_l) per tile), centres[l] = c_l.
  const double* Y64 = nullptr;
  const float* centres = nullptr;
  unsigned long long* skipped = nullptr;   // Psi: pairs of skipped (exactly zero) tiles, or null
  double skip_gap = kPsiSkipGap32;         // Psi: skip tiles whose sorted gap exceeds this (inf: never)
  const double* skip_gap_dev = nullptr;    // Psi: the threshold in device memory (PLUGIN chain), or null
  // Dynamic tile scheduling: a unit counter that is 0 when the launch starts (the caller zeroes it
  // with the limbs), or null for the static stride.
  unsigned long long* work = nullptr;
  // Sets whose count is decided on the device (the device-resident Nelder–Mead): the kernel reads
  // *n_sets_dev (<= n_sets, which sizes the grid).
  const int* n_sets_dev = nullptr;
  // LSCV (any d), data sorted by coordinate 0 (launch_sort_rows): skip a tile (l, q), q < l, when
  // fp32(x_{lT} - x_{qT+T-1})^2 > skip_s, a lower bound on every s of its pairs under which every
  // term is exactly 0 (lscv_skip_s; +inf = never).  `skipped` then counts the skipped pairs.
  float skip_s = __builtin_inff();
  const float* skip_s_sets = nullptr;   // LSCV_H sets: per-set bounds (launch_lscv_sets_skip_select), or null
  const float* skip_c_dev = nullptr;    // LSCV_h batch: per-candidate bounds (launch_lscv_h_skip_select), or null
  // Programmatic dependent launch (the device-resident Nelder–Mead graph): the kernel may start while
  // the previous one finishes and waits for it (griddepcontrol.wait) before reading its outputs.
  bool pdl = false;
  int reserve_ctas = 0;   // resident CTA slots the persistent grid leaves free (for a programmatic successor)
};

// Launchers (kde_psi.cu, kde_lscv_scalar.cu, kde_lscv_matrix.cu).  Return cudaSuccess or the launch error.
cudaError_t launch_psi(int r, const LaunchCfg& c, const PsiParams& p);
cudaError_t prepare_psi(int r, const LaunchCfg& c);   // one-time setup of launch_psi's kernel
// Psi data prep: sorted x -> y = (x - mean[0]) * w[0] (fp64, ld entries, zero padded), the
// per-column-tile centres c_l = fp32(y[min(l T + T/2, n-1)]) and Yc = fp32(y - c_l) (tile T).
cudaError_t launch_psi_prep(const double* x, int64_t n, const double* mean_dev, const double* w_dev, int T,
                            double* Y64, float* Yc, float* centres, int64_t ld, cudaStream_t s,
                            unsigned long long* flag, double clamp_thresh);
// fp64-term Psi pass over 256-tiles of y (Y64 of launch_psi_prep): kde_set_precision(ctx, 1), or the
// automatic re-run of a pass whose cancellation estimate exceeds what fp32 terms carry.  With a
// non-null `gate` the kernel returns at once unless *gate != 0 (device-side decision).
constexpr int kPsi64Tile = 256;
cudaError_t launch_psi64(int r, const double* y, int64_t n, int64_t tile_begin, int64_t tile_end, int S,
                         unsigned long long* limbs, int sm_count, cudaStream_t s,
                         const unsigned long long* gate = nullptr, double skip_gap = kPsiSkipGap64,
                         int part_rank = 0, int part_world = 1);

cudaError_t launch_lscv_scalar(int d, int nb, const LaunchCfg& c, const LscvScalarParams& p);
// LSCV_H with per-candidate whitened data (one candidate per set, c.n_sets sets).
cudaError_t launch_lscv_white(int d, const LaunchCfg& c);
cudaError_t prepare_lscv_white(int d, const LaunchCfg& c);   // one-time setup (before a graph capture)
int tile_for(Kind k, int d, int64_t n);       // tile edge the launcher uses
int cand_per_launch(Kind k, int d);           // B

// O(n) kernels.
cudaError_t launch_moments1(const double* X, int64_t n, int d, double* part, int nblk,
                            cudaStream_t s);
cudaError_t launch_moments2(const double* X, int64_t n, int d, const double* mean_dev,
                            double* part, int nblk, cudaStream_t s);
cudaError_t launch_reduce_parts(const double* part, int nblk, int width, double* out,
                                cudaStream_t s);
struct PrepParams {
  double W[kMaxDim * kMaxDim];   // row-major d x d
  double mean[kMaxDim];
};
// One prepared data set per PrepParams entry, set s into Y + s * set_stride, for the first
// *n_sets_dev of max_sets entries (count decided on the device).
cudaError_t launch_prep_sets(const double* X, int64_t n, int d, const PrepParams* pp_dev, const int* n_sets_dev,
                             int max_sets, float* Y, int64_t set_stride, int64_t ld, cudaStream_t s,
                             unsigned long long* flag, unsigned long long* trace = nullptr,
                             const int* calls = nullptr, bool pdl = false);
cudaError_t launch_prep_params(const double* X, int64_t n, int d, const PrepParams& pp, float* Y, int64_t ld,
                               cudaStream_t s, float pad = 0.f, unsigned long long* overflow_flag = nullptr,
                               double clamp_thresh = 0.0);
cudaError_t launch_prep(const double* X, int64_t n, int d, const double* W_dev,
                        const double* mean_dev, float* Y, int64_t ld, cudaStream_t s,
                        float pad = 0.f, unsigned long long* overflow_flag = nullptr,
                        double clamp_thresh = 0.0);
// fp64-term LSCV sums of one candidate (kde_lscv64.cu): Y = fp64 whitened data (d rows of ld, sorted by
// coordinate 0, ld a multiple of lscv64_tile()), e = exp2(kappa |y_i - y_j|^2), outputs (sum e, sum e^2).
int lscv64_tile();
cudaError_t launch_prep64(const double* X, int64_t n, int d, const PrepParams& pp, double* Y, int64_t ld,
                          cudaStream_t s);
cudaError_t launch_lscv64(int d, const double* Y, int64_t n, int64_t ld, int64_t tb, int64_t te, double kappa,
                          double skip_s, int S, unsigned long long* limbs, int sm_count, cudaStream_t s,
                          int part_rank = 0, int part_world = 1);

// Device-resident PLUGIN chain (kde_psi.cu).  Layout of the workspace's `small` block (doubles):
// mean[16] | W[256] | sums[136] | flags (2 x u64) | trace[8] | status.
// mean[16] | W[256] | sums[136] | flags (2 x u64) | trace[8] | status | gate (2 x u64: the Psi6 /
// Psi4 pass needs its fp64-term re-run) | kappa (2: the passes' cancellation estimates) | skipped
// (u64: pairs in tiles the fp32 kernel skipped as exactly zero, kPluginSkipped).  Limbs of the chain: [Psi6 S, Psi6 A, Psi4 S, Psi4 A,
// Psi6 S fp64, Psi4 S fp64] (kPluginOuts outputs).
struct PluginDev {
  double *mean, *W, *sums, *trace, *status;
  unsigned long long* gate;
  __host__ __device__ explicit PluginDev(double* small)
      : mean(small), W(small + 16), sums(small + 272), trace(small + 410), status(small + 418),
        gate(reinterpret_cast<unsigned long long*>(small + 419)) {}
};
constexpr int kPluginOuts = 6;
constexpr int kSkippedSlot = 423;   // small + 423: skipped-pair counter (PLUGIN chain and psi_raw)
constexpr int kGapSlot = 424;       // small + 424, 425: the PLUGIN passes' bounded skip thresholds (chain)
constexpr int kSmallDoubles = 426;
cudaError_t launch_plugin_chain(int stage, int64_t n, double* small, const unsigned long long* limbs, int S,
                                cudaStream_t s, int psi_mode = 0);
// Automatic Psi precision: an fp32-term pass (S = sum t, A ~ sum |t| at 16-column-group level) is
// re-run with fp64 terms when kappa = 2A / |2S + n He_r(0)| exceeds kPsiKappaMax.
// Calibrated (profiles/r02_psi_kappa.jsonl): fp32-term error <= ~3e-10 kappa for kappa > 10^3, so
// 1e4 keeps the fp32 path within ~3e-6; the C4 passes have kappa <= 5.8e3 and stay on fp32 terms.
constexpr double kPsiKappaMax = 1.0e4;

// KDE evaluation on an m x n rectangle (kde_eval.cu).
struct EvalLaunch {
  const float* Y;        // D x ldm whitened queries (sorted by coordinate 0 when skip_s is finite)
  const float* X;        // D x ldn whitened samples, padded with +inf (sorted likewise)
  int64_t m, ldm, ldn;   // ldm multiple of eval_rows_per_block(), ldn of eval_cols_per_tile()
  int64_t n = 0;         // samples
  float skip_s = __builtin_inff();   // bounded far-tile skip on the coordinate-0 gap^2
  const int* perm = nullptr;         // out[perm[q]] = fhat(sorted query q), or null (identity)
  int* range = nullptr;              // scratch: 2 ints per block of eval_rows_per_block() queries
  double* part;          // scratch [splits][ldm]
  size_t part_capacity;  // doubles available in part
  double scale;          // n^-1 (2 pi)^{-d/2} |H|^{-1/2}
  double* out;           // m results (device)
  cudaStream_t stream;
  int sm_count;
};
cudaError_t launch_eval(int d, const EvalLaunch& c);
int eval_rows_per_block();
int eval_cols_per_tile();
// Column splits eval_kernel<d> uses for an m x n problem (the launch and the host's scratch
// sizing share this): scratch = splits * ldm doubles.
cudaError_t eval_splits(int d, int sm_count, int64_t ldm, int64_t ldn, int* splits);
// The paper's two-phase LSCV_h (kde_materialized.cu).
int mat_tile();
int64_t mat_chunk();
cudaError_t launch_mat_write(int d, const float* X, int64_t n, int64_t ld, int64_t tb, int64_t te, float* buf,
                             int sm_count, cudaStream_t s, int part_rank = 0, int part_world = 1);
cudaError_t launch_mat_reduce(int B, const float* buf, int64_t nvalues, const LscvScalarParams& p, int S,
                              unsigned long long* limbs, int sm_count, cudaStream_t s);
// Univariate AQP closed forms (kde_eval.cu): out[2q] = COUNT, out[2q+1] = SUM.
int aqp_blocks(int64_t n);
cudaError_t launch_aqp(const double* x, int64_t n, double h, const double* lo, const double* hi, int nq,
                       double* part, int nblk, double* out, cudaStream_t s);
int moments_blocks(int64_t n);
size_t sort_temp_bytes(int64_t n);
// Canonical form of `count` outputs' limbs (hi, mid in [0,2^40), lo in [0,2^40), carry 0) so
// that a sum over ranks of int64 limbs cannot wrap.
cudaError_t launch_normalize_limbs(unsigned long long* limbs, int count, cudaStream_t s);
cudaError_t launch_sort(const double* in, double* out, int64_t n, void* temp, size_t temp_bytes,
                        cudaStream_t s);
// d x n samples reordered by ascending coordinate 0 (stable, ties by index): Xs = X[:, perm].
// Scratch: keys (n doubles), idx (2 n ints), CUB temp (sort_rows_temp_bytes).
size_t sort_rows_temp_bytes(int64_t n);
cudaError_t launch_sort_rows(const double* X, int64_t n, int d, double* Xs, double* keys, int* idx, void* temp,
                             size_t temp_bytes, cudaStream_t s);

// Host/device tile map (Eq. 42-43 + integer fix-up).
void tile_coords_host(int64_t bx, int64_t* l, int64_t* q);

}  // namespace kde
