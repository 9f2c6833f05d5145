// kde_host.h — declarations shared by the host translation units of the C ABI in include/kde.h:
//   kde_runtime.cpp   context, workspace, NCCL glue, input staging, the pair-pass driver
//   kde_linalg.cpp    small dense fp64 linear algebra (Cholesky, inverses, SPD square root)
//   kde_nm.cpp        Nelder–Mead (host state machine; reading Z8)
//   kde_selectors.cpp the three selectors and their ABI calls (Sec. 4.4)
//   kde_extras.cpp    KDE evaluation / AQP (f2) and the paper's two-phase LSCV_h (f3)
// P:NNN = PAPER.md line NNN.  Product code: shares nothing with oracle/.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <vector>

#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: ranges cost nothing without a profiler

#include "../../include/kde.h"
#include "kde_internal.h"

typedef struct ncclComm* ncclComm_t;

// ------------------------------------------------------------------ context
struct kde_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int rank = 0, world = 1;
  ncclComm_t comm = nullptr;
  int sm_count = 148;
  kde_status sticky = KDE_OK;
  char err[512] = {0};
  // workspace
  void* ext_ws = nullptr;
  size_t ext_bytes = 0;
  void* own_ws = nullptr;
  size_t own_bytes = 0;
  // materialised S(v) buffer (f3 ablation), context-owned
  void* mat_ws = nullptr;
  void* skip_ws = nullptr;   // LSCV_h data-aware skip: candidates' kappa and bounds
  size_t skip_bytes = 0;
  size_t mat_bytes = 0;
  double prof_aux_ms = 0.0;
  // KDE evaluation / AQP scratch, context-owned
  void* ev_ws = nullptr;
  size_t ev_bytes = 0;
  // per-candidate whitened LSCV_H data sets, context-owned
  void* white_ws = nullptr;
  size_t white_bytes = 0;
  // sorted copy of univariate samples (+ CUB temp), context-owned
  void* sort_ws = nullptr;
  size_t sort_bytes = 0;
  // LSCV samples sorted by coordinate 0 (d x n fp64 | keys | perm | CUB temp), context-owned
  void* rows_ws = nullptr;
  size_t rows_bytes = 0;
  // fp64 whitened samples of the LSCV fp64-term re-run (d x ld doubles), context-owned
  void* f64_ws = nullptr;
  size_t f64_bytes = 0;
  // device copies of host-resident inputs (slot 0: samples X, slot 1: queries Y), context-owned
  void* in_ws[2] = {nullptr, nullptr};
  size_t in_bytes[2] = {0, 0};
  // pinned host staging for limbs
  long long* h_limbs = nullptr;
  size_t h_limbs_cap = 0;
  // Psi term precision: 0 = automatic (fp32 terms, fp64 re-run when the pass's cancellation
  // estimate says fp32 terms cannot carry 1e-5), 1 = always fp64 terms (kde_set_precision),
  // -1 = always fp32 terms (diagnostics).  The fp64 scaled-sample buffer is context-owned.
  int psi_mode = 0;
  // PLUGIN chain: event-pair index and evals of each gated fp64 re-run (profiling), pairs to leave
  // out of the pair time (a gated pass that did not run)
  int gate_pair[2] = {-1, -1};
  double gate_evals[2] = {0.0, 0.0};
  std::vector<char> ev_excl;
  // host-staged collective (test transport for world > 1 without NCCL, kde_set_host_allreduce)
  kde_host_allreduce_fn har_fn = nullptr;
  void* har_user = nullptr;
  long long* har_buf = nullptr;
  size_t har_cap = 0;
  // CUDA graph of the PLUGIN chain, replayed while its key (pointers, n, mode) is unchanged
  bool graphs = true;
  cudaStream_t cap_stream = nullptr;          // capture stream (the caller's may be the legacy one)
  // second stream of a multi-launch pass (run_sums): launch k+1 fills launch k's tail
  cudaStream_t side_stream = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaGraphExec_t plug_exec = nullptr;
  std::vector<uintptr_t> plug_key, plug_seen;   // captured key; key of the last direct run
  int32_t plug_prof_launches = 0, plug_prof_all = 0;
  double plug_prof_evals = 0.0;
  size_t plug_ev_used = 0;
  // device-resident Nelder–Mead (kde_nm_dev.cu): state block, its graph, pinned staging
  void* nm_ws = nullptr;
  size_t nm_bytes = 0;
  cudaGraphExec_t nm_exec = nullptr;
  std::vector<uintptr_t> nm_key;
  void* nm_host = nullptr;
  size_t nm_host_cap = 0;
  // profiling
  bool profiling = false;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  int32_t prof_launches = 0, prof_all = 0;
  double prof_ms = 0.0, prof_evals = 0.0;
  // Psi passes re-run with fp64 terms by the automatic precision during the last call
  int32_t psi_escalations = 0;
  double psi_kappa_max = 0.0;   // largest cancellation estimate of the last call's fp32 Psi passes
  std::vector<double> psi_gaps;  // far-tile skip thresholds of the last call's fp32 Psi passes
};

namespace kde {
namespace host {

// Scoped NVTX range (tracing): moments, prep, sort, psi pass, lscv batch, allreduce...
struct Range {
  explicit Range(const char* name) { nvtxRangePushA(name); }
  ~Range() { nvtxRangePop(); }
};

kde_status fail(kde_ctx* c, kde_status s, const char* fmt, ...);

// A failed call leaves the runtime's last-error slot set (cudaMalloc, a launch): clear it so the
// next call on this thread does not see a stale error (allocation failures are not sticky).
#define CUDA_TRY(ctx, expr)                                                                 \
  do {                                                                                      \
    cudaError_t e_ = (expr);                                                                \
    if (e_ != cudaSuccess) {                                                                \
      if (e_ == cudaErrorMemoryAllocation) cudaGetLastError();                              \
      return ::kde::host::fail(ctx, e_ == cudaErrorMemoryAllocation ? KDE_E_OOM : KDE_E_CUDA, \
                               "CUDA error %s at %s:%d", cudaGetErrorString(e_), __FILE__, __LINE__); \
    }                                                                                       \
  } while (0)

#define TRY(expr)                       \
  do {                                  \
    kde_status s_ = (expr);             \
    if (s_ != KDE_OK) return s_;        \
  } while (0)

constexpr double kPi = 3.14159265358979323846;
constexpr double kLog2e = 1.44269504088896340736;
inline float int_as_float_host(uint32_t b) { float f; std::memcpy(&f, &b, 4); return f; }

// Workspace layout (all offsets 256-byte aligned): Y | part | small | limbs.  Everything but the
// limbs sits at offsets that depend only on (d, ld), so a call that prepares Y once and then
// launches batches with different output counts (Nelder-Mead) sees the same prep flags.
struct Ws {
  float* Y;                 // prepared fp32 data, d x ld
  unsigned long long* limbs;
  double* part;             // moments partials
  double* small;            // mean[16], W[256], sums[136], flags (2 x 8 bytes) at small + 408, ... (kSmallDoubles)
  unsigned long long* flag() const { return reinterpret_cast<unsigned long long*>(small + 408); }
};
size_t align256(size_t b);
size_t ws_bytes(int64_t ld, int32_t d, int32_t n_out);
kde_status get_ws(kde_ctx* c, int64_t ld, int32_t d, int32_t n_out, Ws* w);
kde_status check_ctx(kde_ctx* c);
kde_status grow(kde_ctx* c, void** buf, size_t* cap, size_t need);

// ------------------------------------------------------------------ small dense linear algebra
// Row-major d x d matrices in std::vector<double> (kde_linalg.cpp).
bool cholesky(const std::vector<double>& A, int d, std::vector<double>& L);
std::vector<double> tri_lower_inverse(const std::vector<double>& L, int d);
bool gen_inverse(const std::vector<double>& A, int d, std::vector<double>& R);
bool spd_sqrt(const std::vector<double>& A, int d, std::vector<double>& S);
std::vector<double> unvech(const double* v, int d);
void vech(const std::vector<double>& A, int d, double* v);

// ------------------------------------------------------------------ fixed point
int scale_exp_for(double bound_per_term, int64_t n);
kde_fixed limbs_to_fixed(const long long* l, int S);
double fixed_value(const kde_fixed& f);

// ------------------------------------------------------------------ GPU building blocks
struct Moments {
  std::vector<double> mean, cov;   // cov row-major d x d (unbiased)
};
kde_status gpu_moments(kde_ctx* c, const double* X, int64_t n, int d, Ws& w, Moments& m);
kde_status ensure_sort_ws(kde_ctx* c, int64_t n);
kde_status gpu_sorted(kde_ctx* c, const double* x, int64_t n, const double** out);
// LSCV: X (d x n) reordered by ascending coordinate 0 (context-owned copy; X itself if it already is
// that copy), so that tiles whose pairs are all exactly zero can be skipped (lscv_skip_s).
kde_status gpu_sorted_rows(kde_ctx* c, const double* X, int64_t n, int d, const double** out);
// Skip bound on s for LSCV sums: every term exp2(s * kappa) with s * |kappa| > 130 is exactly 0
// (ex2.approx.ftz flushes results below 2^-126); +inf when KDE_DEBUG_LSCV_NOSKIP=1.
// Far-tile bound on s for terms 2^(kappa s), |kappa| >= min_abs_kappa, at n samples: 130/|kappa| (every
// term exactly 0) or, bounded skip (default), min(130, log2 n + 30)/|kappa| (kde_internal.h);
// +inf under KDE_DEBUG_LSCV_NOSKIP=1.
float lscv_skip_s(double min_abs_kappa, int64_t n);
kde_status gpu_prep_into(kde_ctx* c, const double* X, int64_t n, int d, const std::vector<double>& W,
                         const std::vector<double>& mean, int64_t ld, Ws& w, float* Y, double clamp_thresh = 0.0);
kde_status gpu_prep(kde_ctx* c, const double* X, int64_t n, int d, const std::vector<double>& W,
                    const std::vector<double>& mean, int64_t ld, Ws& w, double clamp_thresh = 0.0);
int64_t n_tiles(int64_t n, int T);
void shard_range(int64_t tiles, int rank, int world, int64_t* b, int64_t* e);
double pairs_in_range(int64_t n, int T, int64_t b, int64_t e);
double pairs_in_shard(int64_t n, int T, int64_t count, int rank, int world);
cudaEvent_t next_event(kde_ctx* c);
void prof_reset(kde_ctx* c);
kde_status prof_collect(kde_ctx* c);

// A "sum job": a sequence of pair-kernel launches over the same prepared data, writing
// n_out fixed-point outputs.
struct SumLaunch {
  Kind kind;
  int r = 0;                  // psi order
  int nb = 1;                 // candidates in this launch
  int out_offset = 0;         // first output index
  int n_out = 0;
  kde::PsiParams psi;
  kde::LscvScalarParams ls;
  const float* X = nullptr;         // prepared data if not the workspace's Y (LSCV_H sets)
  const double* Y64 = nullptr;      // Psi: fp64 scaled rows (tile-local centring)
  const float* centres = nullptr;   // Psi: per-column-tile centres
  unsigned long long* skipped = nullptr;   // Psi: skipped-pair counter
  double skip_gap = kPsiSkipGap32;         // Psi: exact-zero tile skip threshold
  const double* skip_gap_dev = nullptr;    // Psi: the threshold in device memory (data-aware selection)
  float skip_s = __builtin_inff();         // LSCV on sorted data: exact-zero tile skip bound on s
  const float* skip_s_sets = nullptr;      // LSCV_H sets: per-set data-aware bounds (device), or null
  const float* skip_c_dev = nullptr;       // LSCV_h: the batch's per-candidate data-aware bounds (device), or null
  int n_sets = 1;                   // LSCV_H: candidates (one data set each), n_out per set
  int64_t set_stride = 0;
};
kde_status allreduce_limbs(kde_ctx* c, unsigned long long* limbs, size_t count);
kde_status run_sums(kde_ctx* c, int d, int64_t n, int64_t ld, int T, int scale, Ws& w,
                    const std::vector<SumLaunch>& launches, int n_out, int shard_rank, int shard_world,
                    bool allreduce, std::vector<kde_fixed>& out, bool limbs_zeroed = false);
kde_status stage_input(kde_ctx* c, const double*& X, size_t count, int slot);
kde_status validate_X(kde_ctx* c, const double*& X, int64_t n, int32_t d, int64_t nmin);

// ------------------------------------------------------------------ LSCV_H candidates
struct HCand {
  bool pd = false;
  double det = 0.0;
  std::vector<double> W;      // whitening sqrt(log2 e / 4) L^-1 (row-major), H = L L^T, fp64
};
HCand h_candidate(const double* vh, int d);
double lscv_H_finalize(int64_t n, int d, double det, double S1, double S2);
kde_status lscv_H_eval(kde_ctx* c, const double* X, int64_t n, int d, const Moments& m,
                       const std::vector<std::vector<double>>& vs, double penalty, std::vector<double>& g,
                       int* evals, bool auto_precision = false);
struct LscvhPrep {
  std::vector<double> Lc;   // Cholesky of Sigma
  double det = 0.0;
};
kde_status lscv_h_prepare(kde_ctx* c, const Moments& m, int d, LscvhPrep& p);
// LSCV automatic precision: the factor (A + B) / |A - B + C| by which
// g = A - B + C, A = 2 c4 S1 / n^2, B = 4 c2 S2 / n^2, C = c4 / n (times h^-d for LSCV_h) amplifies the
// relative error of the raw sums; a candidate above kLscvKappaMax is re-run with fp64 terms.
constexpr double kLscvKappaMax = 32.0;
double lscv_cancellation(int64_t n, int d, double det, double S1, double S2);
// fp64-term (sum e, sum e^2) of one candidate over all pairs (all ranks, all-reduced): Xs sorted by
// coordinate 0, W the whitening (with sqrt(log2 e / 4)), e = exp2(kappa |W (x_i - x_j)|^2).
kde_status lscv_sums64(kde_ctx* c, const double* Xs, int64_t n, int d, const std::vector<double>& W,
                       const std::vector<double>& mean, double kappa, kde_fixed out[2]);
double lscv_h_finalize(int64_t n, int d, double det, double h, double S1, double S2);

// ------------------------------------------------------------------ Nelder–Mead (kde_nm.cpp)
struct NMResult {
  std::vector<double> x;
  double f = 0.0;
  int iterations = 0, stop = 2, evals = 0;
};
kde_status nelder_mead_multi(kde_ctx* c, const double* X, int64_t n, int d, const Moments& m,
                             const std::vector<std::vector<std::vector<double>>>& sims, int max_iter,
                             double tol, double penalty, bool speculative, NMResult& best, int* total_evals,
                             bool chol_param = false);
// vech(L L^T) for x = vech(L), L lower triangular (the Cholesky-factor search variables, row f4).
void vech_llt(const double* x, int d, double* out);
// The same serial NM as one CUDA graph with a device-side loop (kde_nm_dev.cu): single GPU, one start.
kde_status nelder_mead_device(kde_ctx* c, const double* X, int64_t n, int d, const Moments& m,
                              const std::vector<std::vector<double>>& sim, int max_iter, double tol,
                              double penalty, NMResult& best);

}  // namespace host
}  // namespace kde
