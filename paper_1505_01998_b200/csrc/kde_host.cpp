// kde_host.cpp — host side of the C ABI in include/kde.h: context, workspace, NCCL glue,
// the fp64 scalar chains of the three selectors, small linear algebra and Nelder–Mead.
// P:NNN = PAPER.md line NNN.  Product code: shares nothing with oracle/.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: ranges cost nothing without a profiler

#include "../../include/kde.h"
#include "kde_internal.h"

using kde::Kind;

// ------------------------------------------------------------------ NCCL (loaded at run time)
namespace {
typedef struct ncclComm* ncclComm_t;
struct ncclUniqueId { char internal[128]; };
typedef int ncclResult_t;
constexpr int kNcclInt64 = 4, kNcclSum = 0;
struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
      api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
      api.AllReduce = (decltype(api.AllReduce))dlsym(h, "ncclAllReduce");
      api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
      api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
      api.ok = api.GetUniqueId && api.CommInitRank && api.AllReduce && api.CommDestroy;
    }
  }
  return api;
}
}  // namespace

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
  // device copies of host-resident inputs (slot 0: samples X, slot 1: queries Y), context-owned
  void* in_ws[2] = {nullptr, nullptr};
  size_t in_bytes[2] = {0, 0};
  // pinned host staging for limbs
  long long* h_limbs = nullptr;
  size_t h_limbs_cap = 0;
  // fp64-term Psi mode (kde_set_precision) and its fp64 scaled-sample buffer, context-owned
  bool fp64 = false;
  void* y64 = nullptr;
  size_t y64_bytes = 0;
  // host-staged collective (test transport for world > 1 without NCCL, kde_set_host_allreduce)
  kde_host_allreduce_fn har_fn = nullptr;
  void* har_user = nullptr;
  long long* har_buf = nullptr;
  size_t har_cap = 0;
  // CUDA graph of the PLUGIN chain, replayed while its key (pointers, n, mode) is unchanged
  bool graphs = true;
  cudaStream_t cap_stream = nullptr;          // capture stream (the caller's may be the legacy one)
  cudaGraphExec_t plug_exec = nullptr;
  std::vector<uintptr_t> plug_key, plug_seen;   // captured key; key of the last direct run
  int32_t plug_prof_launches = 0, plug_prof_all = 0;
  double plug_prof_evals = 0.0;
  size_t plug_ev_used = 0;
  // profiling
  bool profiling = false;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  int32_t prof_launches = 0, prof_all = 0;
  double prof_ms = 0.0, prof_evals = 0.0;
};

namespace {

// Scoped NVTX range (tracing): moments, prep, sort, psi pass, lscv batch, allreduce...
struct Range {
  explicit Range(const char* name) { nvtxRangePushA(name); }
  ~Range() { nvtxRangePop(); }
};

kde_status fail(kde_ctx* c, kde_status s, const char* fmt, ...) {
  if (c) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(c->err, sizeof(c->err), fmt, ap);
    va_end(ap);
    if (s == KDE_E_CUDA || s == KDE_E_NCCL) c->sticky = s;
  }
  return s;
}

#define CUDA_TRY(ctx, expr)                                                                 \
  do {                                                                                      \
    cudaError_t e_ = (expr);                                                                \
    if (e_ != cudaSuccess)                                                                  \
      return fail(ctx, e_ == cudaErrorMemoryAllocation ? KDE_E_OOM : KDE_E_CUDA,            \
                  "CUDA error %s at %s:%d", cudaGetErrorString(e_), __FILE__, __LINE__);    \
  } while (0)

#define TRY(expr)                       \
  do {                                  \
    kde_status s_ = (expr);             \
    if (s_ != KDE_OK) return s_;        \
  } while (0)

constexpr double kPi = 3.14159265358979323846;
inline float __int_as_float_host(uint32_t b) { float f; std::memcpy(&f, &b, 4); return f; }
constexpr double kLog2e = 1.44269504088896340736;

// Workspace layout (all offsets 256-byte aligned): Y | part | small | limbs.  Everything but the
// limbs sits at offsets that depend only on (d, ld), so a call that prepares Y once and then
// launches batches with different output counts (Nelder-Mead) sees the same prep flags.
struct Ws {
  float* Y;                 // prepared fp32 data, d x ld
  unsigned long long* limbs;
  double* part;             // moments partials
  double* small;            // mean[16], W[256], sums[136], flags (2 x 8 bytes) at small + 408
  unsigned long long* flag() const { return reinterpret_cast<unsigned long long*>(small + 408); }
};

size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

size_t ws_bytes(int64_t ld, int32_t d, int32_t n_out) {
  return align256((size_t)d * ld * sizeof(float)) +
         align256((size_t)std::max(n_out, 1) * kde::kLimbs * sizeof(long long)) +
         align256((size_t)1024 * 136 * sizeof(double)) + align256((16 + 256 + 136 + 16) * sizeof(double));
}

kde_status get_ws(kde_ctx* c, int64_t ld, int32_t d, int32_t n_out, Ws* w) {
  size_t need = ws_bytes(ld, d, n_out);
  char* base;
  if (c->ext_ws && c->ext_bytes >= need) {
    base = (char*)c->ext_ws;
  } else {
    if (c->own_bytes < need) {
      if (c->own_ws) {
        CUDA_TRY(c, cudaStreamSynchronize(c->stream));
        cudaFree(c->own_ws);
        c->own_ws = nullptr;
        c->own_bytes = 0;
      }
      size_t cap = need + need / 4;
      CUDA_TRY(c, cudaMalloc(&c->own_ws, cap));
      c->own_bytes = cap;
      // defined contents once: run_sums copies [prep flags .. limbs) in one transfer, gap included
      CUDA_TRY(c, cudaMemsetAsync(c->own_ws, 0, cap, c->stream));
    }
    base = (char*)c->own_ws;
  }
  w->Y = (float*)base;
  base += align256((size_t)d * ld * sizeof(float));
  w->part = (double*)base;
  base += align256((size_t)1024 * 136 * sizeof(double));
  w->small = (double*)base;
  base += align256((16 + 256 + 136 + 16) * sizeof(double));
  w->limbs = (unsigned long long*)base;
  return KDE_OK;
}

kde_status check_ctx(kde_ctx* c) {
  if (!c) return KDE_E_INVALID;
  if (c->sticky != KDE_OK) return c->sticky;
  CUDA_TRY(c, cudaSetDevice(c->device));
  return KDE_OK;
}

// ------------------------------------------------------------------ small dense linear algebra
// Row-major d x d matrices in std::vector<double>.

// Cholesky A = L L^T with a relative pivot test (positive-definiteness, reading Z8).
bool cholesky(const std::vector<double>& A, int d, std::vector<double>& L) {
  L.assign((size_t)d * d, 0.0);
  double mx = 0.0;
  for (int i = 0; i < d; ++i) {
    if (!std::isfinite(A[i * d + i])) return false;
    mx = std::max(mx, std::fabs(A[i * d + i]));
  }
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j)
      if (!std::isfinite(A[i * d + j]) || A[i * d + j] != A[j * d + i]) return false;
  for (int j = 0; j < d; ++j) {
    double s = A[j * d + j];
    for (int k = 0; k < j; ++k) s -= L[j * d + k] * L[j * d + k];
    if (!(s > 1e-12 * mx)) return false;
    L[j * d + j] = std::sqrt(s);
    for (int i = j + 1; i < d; ++i) {
      double t = A[i * d + j];
      for (int k = 0; k < j; ++k) t -= L[i * d + k] * L[j * d + k];
      L[i * d + j] = t / L[j * d + j];
    }
  }
  return true;
}

// Inverse of a lower-triangular matrix by forward substitution.
std::vector<double> tri_lower_inverse(const std::vector<double>& L, int d) {
  std::vector<double> M((size_t)d * d, 0.0);
  for (int col = 0; col < d; ++col) {
    for (int i = 0; i < d; ++i) {
      double s = (i == col) ? 1.0 : 0.0;
      for (int k = 0; k < i; ++k) s -= L[i * d + k] * M[k * d + col];
      M[i * d + col] = s / L[i * d + i];
    }
  }
  return M;
}

// Principal square root of an SPD matrix by the Denman–Beavers iteration (the paper used
// ALGLIB; reading Z9).  Y_{k+1} = (Y_k + Z_k^-1)/2, Z_{k+1} = (Z_k + Y_k^-1)/2.
bool gen_inverse(const std::vector<double>& A, int d, std::vector<double>& R) {
  // Gauss–Jordan with partial pivoting on a general matrix.
  std::vector<double> M = A;
  R.assign((size_t)d * d, 0.0);
  for (int i = 0; i < d; ++i) R[i * d + i] = 1.0;
  for (int c = 0; c < d; ++c) {
    int p = c;
    for (int r = c + 1; r < d; ++r)
      if (std::fabs(M[r * d + c]) > std::fabs(M[p * d + c])) p = r;
    if (M[p * d + c] == 0.0) return false;
    if (p != c)
      for (int k = 0; k < d; ++k) { std::swap(M[p * d + k], M[c * d + k]); std::swap(R[p * d + k], R[c * d + k]); }
    double piv = M[c * d + c];
    for (int k = 0; k < d; ++k) { M[c * d + k] /= piv; R[c * d + k] /= piv; }
    for (int r = 0; r < d; ++r) {
      if (r == c) continue;
      double f = M[r * d + c];
      if (f == 0.0) continue;
      for (int k = 0; k < d; ++k) { M[r * d + k] -= f * M[c * d + k]; R[r * d + k] -= f * R[c * d + k]; }
    }
  }
  return true;
}

bool spd_sqrt(const std::vector<double>& A, int d, std::vector<double>& S) {
  std::vector<double> Y = A, Z((size_t)d * d, 0.0), Yi, Zi;
  for (int i = 0; i < d; ++i) Z[i * d + i] = 1.0;
  for (int it = 0; it < 100; ++it) {
    if (!gen_inverse(Y, d, Yi) || !gen_inverse(Z, d, Zi)) return false;
    double diff = 0.0, nrm = 0.0;
    for (size_t k = 0; k < Y.size(); ++k) {
      double yn = 0.5 * (Y[k] + Zi[k]);
      double zn = 0.5 * (Z[k] + Yi[k]);
      diff = std::max(diff, std::fabs(yn - Y[k]));
      nrm = std::max(nrm, std::fabs(yn));
      Y[k] = yn;
      Z[k] = zn;
    }
    if (diff <= 1e-15 * nrm) break;
  }
  S = Y;
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < i; ++j) S[i * d + j] = S[j * d + i] = 0.5 * (S[i * d + j] + S[j * d + i]);
  return true;
}

std::vector<double> unvech(const double* v, int d) {
  std::vector<double> A((size_t)d * d);
  int t = 0;
  for (int j = 0; j < d; ++j)
    for (int i = j; i < d; ++i) { A[i * d + j] = A[j * d + i] = v[t]; ++t; }
  return A;
}

void vech(const std::vector<double>& A, int d, double* v) {
  int t = 0;
  for (int j = 0; j < d; ++j)
    for (int i = j; i < d; ++i) v[t++] = A[i * d + j];
}

// ------------------------------------------------------------------ fixed point
int scale_exp_for(double bound_per_term, int64_t n) {
  double pairs = (double)n * (double)(n - 1) * 0.5;
  double G = std::max(1.0, bound_per_term * std::max(pairs, 1.0));
  return 100 - (int)std::ceil(std::log2(G));
}

kde_fixed limbs_to_fixed(const long long* l, int S) {
  kde_fixed f;
  f.hi = l[0]; f.mid = l[1]; f.lo = l[2]; f.scale_exp = S; f.pad_ = 0;
  return f;
}

double fixed_value(const kde_fixed& f) {
  __int128 T = (__int128)f.hi * ((__int128)1 << 80) + (__int128)f.mid * ((__int128)1 << 40) + (__int128)f.lo;
  return std::ldexp((double)T, -f.scale_exp);
}

// ------------------------------------------------------------------ GPU building blocks
struct Moments {
  std::vector<double> mean, cov;   // cov row-major d x d (unbiased)
};

// Two-pass fp64 moments on the GPU (Eq. 11, Eq. 20-23 read as the unbiased sample covariance,
// reading Z10).  Returns KDE_E_INVALID for non-finite data.
kde_status gpu_moments(kde_ctx* c, const double* X, int64_t n, int d, Ws& w, Moments& m) {
  Range r("kde.moments");
  const int nblk = kde::moments_blocks(n);
  double* sums = w.small + 16 + 256;
  double* mean_dev = w.small;
  double hs[136];
  CUDA_TRY(c, kde::launch_moments1(X, n, d, w.part, nblk, c->stream));
  CUDA_TRY(c, kde::launch_reduce_parts(w.part, nblk, d, sums, c->stream));
  c->prof_all += 2;
  CUDA_TRY(c, cudaMemcpyAsync(hs, sums, d * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  m.mean.assign(d, 0.0);
  for (int a = 0; a < d; ++a) {
    if (!std::isfinite(hs[a])) return fail(c, KDE_E_INVALID, "non-finite sample values");
    m.mean[a] = hs[a] / (double)n;
  }
  CUDA_TRY(c, cudaMemcpyAsync(mean_dev, m.mean.data(), d * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  const int width = d * (d + 1) / 2;
  CUDA_TRY(c, kde::launch_moments2(X, n, d, mean_dev, w.part, nblk, c->stream));
  CUDA_TRY(c, kde::launch_reduce_parts(w.part, nblk, width, sums, c->stream));
  c->prof_all += 2;
  CUDA_TRY(c, cudaMemcpyAsync(hs, sums, width * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  m.cov.assign((size_t)d * d, 0.0);
  int t = 0;
  for (int a = 0; a < d; ++a)
    for (int b = a; b < d; ++b) {
      double v = hs[t++] / (double)(n - 1);
      if (!std::isfinite(v)) return fail(c, KDE_E_INVALID, "non-finite sample values");
      m.cov[a * d + b] = m.cov[b * d + a] = v;
    }
  return KDE_OK;
}

kde_status grow(kde_ctx* c, void** buf, size_t* cap, size_t need) {
  if (*cap >= need) return KDE_OK;
  if (*buf) {
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    cudaFree(*buf);
    *buf = nullptr;
    *cap = 0;
  }
  CUDA_TRY(c, cudaMalloc(buf, need));
  *cap = need;
  return KDE_OK;
}

// Sorted copy of n univariate samples (context-owned scratch); returns the device pointer.
kde_status ensure_sort_ws(kde_ctx* c, int64_t n) {
  const size_t need = align256((size_t)n * sizeof(double)) + align256(kde::sort_temp_bytes(n));
  if (c->sort_bytes < need) {
    if (c->sort_ws) {
      CUDA_TRY(c, cudaStreamSynchronize(c->stream));
      cudaFree(c->sort_ws);
      c->sort_ws = nullptr;
      c->sort_bytes = 0;
    }
    CUDA_TRY(c, cudaMalloc(&c->sort_ws, need));
    c->sort_bytes = need;
  }
  return KDE_OK;
}

kde_status gpu_sorted(kde_ctx* c, const double* x, int64_t n, const double** out) {
  Range r("kde.sort");
  const size_t tmp = kde::sort_temp_bytes(n);
  TRY(ensure_sort_ws(c, n));
  double* xs = (double*)c->sort_ws;
  void* temp = (char*)c->sort_ws + align256((size_t)n * sizeof(double));
  CUDA_TRY(c, kde::launch_sort(x, xs, n, temp, tmp, c->stream));
  c->prof_all += 10;   // CUB onesweep for 64-bit keys: histogram, exclusive sum, 8 passes
  *out = xs;
  return KDE_OK;
}

// y = fp32(W (x - mean)), padded with zeros to ld, written to Y (default: the workspace's Y).
// gpu_prep_into does not clear the prep flags (several sets prepared for one launch share them).
kde_status gpu_prep_into(kde_ctx* c, const double* X, int64_t n, int d, const std::vector<double>& W,
                         const std::vector<double>& mean, int64_t ld, Ws& w, float* Y,
                         double clamp_thresh = 0.0) {
  Range r("kde.prep");
  kde::PrepParams pp;                      // W and mean travel in the kernel parameters
  std::copy(W.begin(), W.begin() + (size_t)d * d, pp.W);
  std::copy(mean.begin(), mean.begin() + d, pp.mean);
  CUDA_TRY(c, kde::launch_prep_params(X, n, d, pp, Y, ld, c->stream, 0.f, w.flag(), clamp_thresh));
  c->prof_all += 1;
  return KDE_OK;
}

kde_status gpu_prep(kde_ctx* c, const double* X, int64_t n, int d, const std::vector<double>& W,
                    const std::vector<double>& mean, int64_t ld, Ws& w, double clamp_thresh = 0.0) {
  CUDA_TRY(c, cudaMemsetAsync(w.flag(), 0, 2 * sizeof(unsigned long long), c->stream));
  return gpu_prep_into(c, X, n, d, W, mean, ld, w, w.Y, clamp_thresh);
}

int64_t n_tiles(int64_t n, int T) {
  int64_t nb = (n + T - 1) / T;
  return nb * (nb + 1) / 2;
}

void shard_range(int64_t tiles, int rank, int world, int64_t* b, int64_t* e) {
  *b = (int64_t)((__int128)tiles * rank / world);
  *e = (int64_t)((__int128)tiles * (rank + 1) / world);
}

// Algorithmic pairs i<j inside tiles [b, e), one column of tiles at a time (the tile numbering
// is column-major, Eq. 42-43): O(#columns) instead of O(#tiles) host work per pass.
double pairs_in_range(int64_t n, int T, int64_t b, int64_t e) {
  if (e <= b) return 0.0;
  int64_t lb, qb, le, qe;
  kde::tile_coords_host(b, &lb, &qb);
  kde::tile_coords_host(e - 1, &le, &qe);
  double s = 0.0;
  for (int64_t l = lb; l <= le; ++l) {
    const int64_t q0 = (l == lb) ? qb : 0, q1 = (l == le) ? qe : l;   // tiles q0..q1 of column l
    const double cols = (double)std::min<int64_t>(T, n - l * (int64_t)T);
    const int64_t off = std::min<int64_t>(q1, l - 1) - q0 + 1;          // q < l: T x cols pairs
    if (off > 0) s += (double)off * (double)T * cols;
    if (q1 == l) s += cols * (cols - 1.0) * 0.5;                        // diagonal tile
  }
  return s;
}

cudaEvent_t next_event(kde_ctx* c) {
  if (c->ev_used == c->ev_pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    c->ev_pool.push_back(e);
  }
  return c->ev_pool[c->ev_used++];
}

void prof_reset(kde_ctx* c) {
  c->ev_used = 0;
  c->prof_launches = 0;
  c->prof_all = 0;
  c->prof_ms = 0.0;
  c->prof_evals = 0.0;
  c->prof_aux_ms = 0.0;
}

kde_status prof_collect(kde_ctx* c) {
  if (!c->profiling) return KDE_OK;
  double ms = 0.0;
  for (size_t k = 0; k + 1 < c->ev_used; k += 2) {
    float x = 0.f;
    CUDA_TRY(c, cudaEventElapsedTime(&x, c->ev_pool[k], c->ev_pool[k + 1]));
    ms += x;
  }
  c->prof_ms = ms;
  return KDE_OK;
}

// A "sum job": a sequence of pair-kernel launches over the same prepared data, writing
// n_out fixed-point outputs.  Launch closures receive (LaunchCfg with limbs offset).
struct SumLaunch {
  Kind kind;
  int r = 0;                  // psi order
  int nb = 1;                 // candidates in this launch
  int out_offset = 0;         // first output index
  int n_out = 0;
  kde::PsiParams psi;
  kde::LscvScalarParams ls;
  const float* X = nullptr;         // prepared data if not the workspace's Y (LSCV_H sets)
  int n_sets = 1;                   // LSCV_H: candidates (one data set each), n_out per set
  int64_t set_stride = 0;
};

// Sum `count` int64 limbs in device memory across the ranks: NCCL on the context stream, or (test
// transport, no NCCL) staged through pinned host memory and the caller's all-reduce callback.
kde_status allreduce_limbs(kde_ctx* c, unsigned long long* limbs, size_t count) {
  if (c->comm) {
    Range ra("kde.allreduce");
    NcclApi& api = nccl();
    ncclResult_t r = api.AllReduce(limbs, limbs, count, kNcclInt64, kNcclSum, c->comm, c->stream);
    if (r != 0) return fail(c, KDE_E_NCCL, "ncclAllReduce: %s", api.GetErrorString ? api.GetErrorString(r) : "?");
    return KDE_OK;
  }
  if (c->world <= 1) return KDE_OK;
  if (!c->har_fn) return fail(c, KDE_E_NCCL, "world > 1 without a collective (NCCL id or host all-reduce)");
  Range ra("kde.allreduce_host");
  if (c->har_cap < count) {
    if (c->har_buf) cudaFreeHost(c->har_buf);
    c->har_buf = nullptr;
    CUDA_TRY(c, cudaMallocHost(&c->har_buf, count * sizeof(long long)));
    c->har_cap = count;
  }
  CUDA_TRY(c, cudaMemcpyAsync(c->har_buf, limbs, count * sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  if (c->har_fn(reinterpret_cast<int64_t*>(c->har_buf), count, c->har_user) != 0)
    return fail(c, KDE_E_NCCL, "host all-reduce callback failed");
  CUDA_TRY(c, cudaMemcpyAsync(limbs, c->har_buf, count * sizeof(long long), cudaMemcpyHostToDevice, c->stream));
  return KDE_OK;
}

// Launch the given pair kernels over shard tiles, all-reduce (if requested), fetch fixed-point
// outputs.  Data must already be prepared in w.Y with leading dimension ld.
kde_status run_sums(kde_ctx* c, int d, int64_t n, int64_t ld, int T, int scale, Ws& w,
                    const std::vector<SumLaunch>& launches, int n_out, int shard_rank,
                    int shard_world, bool allreduce, std::vector<kde_fixed>& out, bool limbs_zeroed = false) {
  Range rr("kde.pair_pass");
  if (!limbs_zeroed)
    CUDA_TRY(c, cudaMemsetAsync(w.limbs, 0, (size_t)n_out * kde::kLimbs * sizeof(long long), c->stream));
  int64_t tiles = n_tiles(n, T), tb, te;
  shard_range(tiles, shard_rank, shard_world, &tb, &te);
  const double pairs = c->profiling ? pairs_in_range(n, T, tb, te) : 0.0;
  for (const SumLaunch& L : launches) {
    kde::LaunchCfg cfg;
    cfg.X = w.Y; cfg.n = n; cfg.ld = ld; cfg.tile_begin = tb; cfg.tile_end = te; cfg.tile = T;
    cfg.scale_exp = scale; cfg.limbs = w.limbs + (size_t)L.out_offset * kde::kLimbs;
    cfg.n_out = L.n_out; cfg.stream = c->stream; cfg.sm_count = c->sm_count;
    cfg.clamp = w.flag() + 1;
    if (L.X) cfg.X = L.X;
    cfg.n_sets = L.n_sets;
    cfg.set_stride = L.set_stride;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (c->profiling) { e0 = next_event(c); e1 = next_event(c); cudaEventRecord(e0, c->stream); }
    cudaError_t err = cudaSuccess;
    switch (L.kind) {
      case Kind::Psi4: case Kind::Psi6: case Kind::Psi8: err = kde::launch_psi(L.r, cfg, L.psi); break;
      case Kind::LscvScalar: err = kde::launch_lscv_scalar(d, L.nb, cfg, L.ls); break;
      case Kind::LscvMatrix: err = kde::launch_lscv_white(d, cfg); break;
    }
    if (err != cudaSuccess) return fail(c, KDE_E_CUDA, "pair kernel launch: %s", cudaGetErrorString(err));
    if (tb < te) c->prof_all += 1;
    if (c->profiling) {
      cudaEventRecord(e1, c->stream);
      c->prof_launches++;
      c->prof_evals += pairs * (double)L.nb * (double)L.n_sets;
    }
  }
  if (allreduce) TRY(allreduce_limbs(c, w.limbs, (size_t)n_out * kde::kLimbs));
  // one device-to-host copy of [prep flags .. limbs): the workspace places the limbs right after
  // the fixed-size block that holds the flags (get_ws)
  const size_t gap = (size_t)(reinterpret_cast<const char*>(w.limbs) - reinterpret_cast<const char*>(w.flag())) /
                     sizeof(long long);
  const size_t need = gap + (size_t)n_out * kde::kLimbs;
  if (c->h_limbs_cap < need) {
    if (c->h_limbs) cudaFreeHost(c->h_limbs);
    c->h_limbs = nullptr;
    CUDA_TRY(c, cudaMallocHost(&c->h_limbs, need * sizeof(long long)));
    c->h_limbs_cap = need;
  }
  CUDA_TRY(c, cudaMemcpyAsync(c->h_limbs, w.flag(), need * sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  if (c->h_limbs[0]) return fail(c, KDE_E_INVALID, "scaled sample differences exceed 1e18 (outliers vs. bandwidth)");
  out.resize(n_out);
  for (int k = 0; k < n_out; ++k) out[k] = limbs_to_fixed(c->h_limbs + gap + (size_t)k * kde::kLimbs, scale);
  return KDE_OK;
}

// ------------------------------------------------------------------ Psi_r
// The kernel evaluates He_r in t = u^2 - (r-1) with exact integer coefficients; the parameters
// are the exponent scale c0 and, per accumulator class k, the MUFU offset o_k and the exact
// fp64 factor that undoes it: 2^(u^2 c0) = 2^(t c0 + o_k) * 2^((r-1) c0 - o_k).
void psi_coeffs(int r, kde::PsiParams& p) {
  std::memset(&p, 0, sizeof(p));
  p.c0 = (float)(-kLog2e / 2.0);
  const double Kc0 = (double)(r == 8 ? 0 : r - 1) * (double)p.c0;   // K of FPsi; exact in fp64
  for (int k = 0; k < 16; ++k) {   // k = 8 * (tile parity) + row slot; shift (row slot)/8 + parity/16
    p.o[k] = (float)(Kc0 - (16.0 + (k % 8) / 8.0 + (k / 8) / 16.0));
    p.fac[k] = std::exp2(Kc0 - (double)p.o[k]);                    // exponent exact in fp64
  }
}

double he_at_zero(int r) { return r == 4 ? 3.0 : (r == 6 ? -15.0 : 105.0); }

Kind psi_kind(int r) { return r == 4 ? Kind::Psi4 : (r == 6 ? Kind::Psi6 : Kind::Psi8); }

// fp64-term mode: one Psi_r pass over this rank's 256-tiles of the fp64 scaled samples y, into
// `limbs` (3 int64), then the all-reduce.
kde_status psi64_pass(kde_ctx* c, int r, const double* y, int64_t n, int S, unsigned long long* limbs) {
  Range rr("kde.pair_pass_fp64");
  int64_t tb, te;
  shard_range(n_tiles(n, kde::kPsi64Tile), c->rank, c->world, &tb, &te);
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  const unsigned rec = (c->cap_stream && c->stream == c->cap_stream) ? cudaEventRecordExternal : cudaEventRecordDefault;
  if (c->profiling) { e0 = next_event(c); e1 = next_event(c); CUDA_TRY(c, cudaEventRecordWithFlags(e0, c->stream, rec)); }
  CUDA_TRY(c, kde::launch_psi64(r, y, n, tb, te, S, limbs, c->sm_count, c->stream));
  if (tb < te) c->prof_all += 1;
  if (c->profiling) {
    CUDA_TRY(c, cudaEventRecordWithFlags(e1, c->stream, rec));
    c->prof_launches++;
    c->prof_evals += pairs_in_range(n, kde::kPsi64Tile, tb, te);
  }
  TRY(allreduce_limbs(c, limbs, kde::kLimbs));
  return KDE_OK;
}

// Raw Psi sums S_r(g) = sum_{i<j} He_r(u) e^{-u^2/2} for each g (one prep + one launch per g).
kde_status psi_raw(kde_ctx* c, const double* x, int64_t n, int r, const double* g, int ng,
                   const Moments& m, int shard_rank, int shard_world, bool allreduce,
                   std::vector<kde_fixed>& out, bool presorted = false) {
  const int T = kde::tile_for(psi_kind(r), 1, n);
  const int64_t ld = (n + T - 1) / T * T;
  Ws w;
  TRY(get_ws(c, ld, 1, 1, &w));
  const int S = scale_exp_for(2.0 * std::fabs(he_at_zero(r)), n);
  if (!presorted) {
    const double* xs = nullptr;
    TRY(gpu_sorted(c, x, n, &xs));
    x = xs;
  }
  out.clear();
  if (c->fp64) {                       // fp64-term mode (kde_set_precision)
    TRY(grow(c, &c->y64, &c->y64_bytes, (size_t)std::max<int64_t>(n, 1) * sizeof(double)));
    double* y = static_cast<double*>(c->y64);
    for (int k = 0; k < ng; ++k) {
      const double hv[2] = {m.mean[0], 1.0 / g[k]};
      CUDA_TRY(c, cudaMemcpyAsync(w.small, hv, sizeof(hv), cudaMemcpyHostToDevice, c->stream));
      CUDA_TRY(c, kde::launch_scale64(x, n, w.small, w.small + 1, y, c->stream));
      CUDA_TRY(c, cudaMemsetAsync(w.limbs, 0, kde::kLimbs * sizeof(long long), c->stream));
      if (allreduce) {
        TRY(psi64_pass(c, r, y, n, S, w.limbs));
      } else {                         // one shard, no collective
        int64_t tb, te;
        shard_range(n_tiles(n, kde::kPsi64Tile), shard_rank, shard_world, &tb, &te);
        CUDA_TRY(c, kde::launch_psi64(r, y, n, tb, te, S, w.limbs, c->sm_count, c->stream));
      }
      long long hl[kde::kLimbs];
      CUDA_TRY(c, cudaMemcpyAsync(hl, w.limbs, sizeof(hl), cudaMemcpyDeviceToHost, c->stream));
      CUDA_TRY(c, cudaStreamSynchronize(c->stream));
      out.push_back(limbs_to_fixed(hl, S));
    }
    return KDE_OK;
  }
  for (int k = 0; k < ng; ++k) {
    std::vector<double> W = {1.0 / g[k]};
    TRY(gpu_prep(c, x, n, 1, W, m.mean, ld, w, 3.0e4));
    SumLaunch L;
    L.kind = psi_kind(r); L.r = r; L.nb = 1; L.out_offset = 0; L.n_out = 1;
    psi_coeffs(r, L.psi);
    std::vector<kde_fixed> o;
    TRY(run_sums(c, 1, n, ld, T, S, w, {L}, 1, shard_rank, shard_world, allreduce, o));
    out.push_back(o[0]);
  }
  return KDE_OK;
}

double psi_finalize(int r, int64_t n, double g, double S) {
  const double s2p = std::sqrt(2.0 * kPi);
  const double nn = (double)n;
  return (2.0 * S / s2p + nn * he_at_zero(r) / s2p) / (nn * nn * std::pow(g, r + 1));
}

// ------------------------------------------------------------------ LSCV_h
struct LscvhPrep {
  std::vector<double> Lc;   // Cholesky of Sigma
  double det = 0.0;
};

kde_status lscv_h_prepare(kde_ctx* c, const Moments& m, int d, LscvhPrep& p) {
  if (!cholesky(m.cov, d, p.Lc)) return fail(c, KDE_E_SINGULAR_COV, "covariance matrix is not positive definite");
  p.det = 1.0;
  for (int i = 0; i < d; ++i) p.det *= p.Lc[i * d + i] * p.Lc[i * d + i];
  if (!(p.det > 0.0) || !std::isfinite(p.det)) return fail(c, KDE_E_SINGULAR_COV, "det(Sigma) <= 0");
  return KDE_OK;
}

kde_status lscv_h_raw(kde_ctx* c, const double* X, int64_t n, int d, const double* h, int nh,
                      const Moments& m, const LscvhPrep& pp, int shard_rank, int shard_world,
                      bool allreduce, std::vector<kde_fixed>& out) {
  const int T = kde::tile_for(Kind::LscvScalar, d, n);
  const int nb = kde::cand_per_launch(Kind::LscvScalar, d);
  const int64_t ld = (n + T - 1) / T * T;
  const int nbatch = (nh + nb - 1) / nb;
  const int n_out = 2 * nbatch * nb;
  Ws w;
  TRY(get_ws(c, ld, d, n_out, &w));
  // W = sqrt(log2 e / 4) L^-1  =>  |W v|^2 = (log2 e / 4) v^T Sigma^-1 v
  std::vector<double> W = tri_lower_inverse(pp.Lc, d);
  for (double& v : W) v *= std::sqrt(kLog2e / 4.0);
  TRY(gpu_prep(c, X, n, d, W, m.mean, ld, w));
  std::vector<SumLaunch> Ls;
  for (int b = 0; b < nbatch; ++b) {
    SumLaunch L;
    L.kind = Kind::LscvScalar; L.nb = nb; L.out_offset = 2 * b * nb; L.n_out = 2 * nb;
    for (int j = 0; j < kde::kMaxCand; ++j) {
      int idx = std::min(b * nb + j, nh - 1);   // pad with a valid candidate
      L.ls.kappa[j] = (float)(-1.0 / (h[idx] * h[idx]));
    }
    Ls.push_back(L);
  }
  std::vector<kde_fixed> o;
  TRY(run_sums(c, d, n, ld, T, scale_exp_for(1.0, n), w, Ls, n_out, shard_rank, shard_world, allreduce, o));
  out.assign(o.begin(), o.begin() + 2 * nh);
  return KDE_OK;
}

double lscv_h_finalize(int64_t n, int d, double det, double h, double S1, double S2) {
  const double nn = (double)n;
  const double c4 = std::pow(4.0 * kPi, -0.5 * d) / std::sqrt(det);
  const double c2 = std::pow(2.0 * kPi, -0.5 * d) / std::sqrt(det);
  return std::pow(h, -d) * (2.0 * (c4 * S1 - 2.0 * c2 * S2) / (nn * nn) + c4 / nn);
}

// ------------------------------------------------------------------ LSCV_H
struct HCand {
  bool pd = false;
  double det = 0.0;
  std::vector<double> L;      // Cholesky factor of H (row-major lower), fp64
};

HCand h_candidate(const double* vh, int d) {
  HCand hc;
  std::vector<double> H = unvech(vh, d), L;
  if (!cholesky(H, d, L)) return hc;
  hc.pd = true;
  hc.det = 1.0;
  for (int i = 0; i < d; ++i) hc.det *= L[i * d + i] * L[i * d + i];
  hc.L = std::move(L);
  return hc;
}

// Raw LSCV_H sums for PD candidates `cands` (all must be PD).  Each candidate gets its own
// whitened fp32 copy of the data, x'_c = sqrt(log2 e / 4) L_c^-1 (x - mean) with H_c = L_c L_c^T,
// so that v^T H_c^-1 v = (4 / log2 e) |x'_ci - x'_cj|^2: the pair kernel then needs no quadratic
// form (2d + 2 FP32 ops per eval instead of d(d+1)/2 + 2 per candidate plus the monomials), and
// the sum of squares does not lose accuracy with cond(H).  Candidates are
// independent work units, so a candidate's sums are bit-identical alone or inside any batch.
kde_status lscv_H_raw(kde_ctx* c, const double* X, int64_t n, int d, const std::vector<HCand>& cands,
                      const Moments& m, int shard_rank, int shard_world, bool allreduce,
                      std::vector<kde_fixed>& out) {
  const int T = kde::tile_for(Kind::LscvMatrix, d, n);
  const int64_t ld = (n + T - 1) / T * T;
  const int64_t set_floats = (int64_t)d * ld;
  const int nc = (int)cands.size();
  // sets per launch: up to 256 candidates within ~1 GiB of prepared data
  const int per_launch = (int)std::max<int64_t>(1, std::min<int64_t>(256, (1LL << 28) / set_floats));
  Ws w;
  TRY(get_ws(c, ld, d, 2 * std::min(nc, per_launch), &w));
  out.clear();
  for (int b0 = 0; b0 < nc; b0 += per_launch) {
    const int cnt = std::min(per_launch, nc - b0);
    TRY(grow(c, &c->white_ws, &c->white_bytes, (size_t)cnt * set_floats * sizeof(float)));
    float* Yw = static_cast<float*>(c->white_ws);
    // prep flags and this launch's limbs are one contiguous span of the workspace (get_ws): one memset
    const size_t span = (size_t)(reinterpret_cast<char*>(w.limbs + (size_t)2 * cnt * kde::kLimbs) -
                                 reinterpret_cast<char*>(w.flag()));
    CUDA_TRY(c, cudaMemsetAsync(w.flag(), 0, span, c->stream));
    for (int j = 0; j < cnt; ++j) {
      std::vector<double> W = tri_lower_inverse(cands[b0 + j].L, d);
      for (double& v : W) v *= std::sqrt(kLog2e / 4.0);
      TRY(gpu_prep_into(c, X, n, d, W, m.mean, ld, w, Yw + (size_t)j * set_floats));
    }
    SumLaunch L;
    L.kind = Kind::LscvMatrix; L.nb = 1; L.out_offset = 0; L.n_out = 2 * cnt;
    L.X = Yw; L.n_sets = cnt; L.set_stride = set_floats;
    std::vector<kde_fixed> o;
    TRY(run_sums(c, d, n, ld, T, scale_exp_for(1.0, n), w, {L}, 2 * cnt, shard_rank, shard_world, allreduce, o,
                 /*limbs_zeroed=*/true));
    out.insert(out.end(), o.begin(), o.end());
  }
  return KDE_OK;
}

double lscv_H_finalize(int64_t n, int d, double det, double S1, double S2) {
  const double nn = (double)n;
  const double c4 = std::pow(4.0 * kPi, -0.5 * d) / std::sqrt(det);
  const double c2 = std::pow(2.0 * kPi, -0.5 * d) / std::sqrt(det);
  return 2.0 * (c4 * S1 - 2.0 * c2 * S2) / (nn * nn) + c4 / nn;
}

// Evaluate g(H) for a list of vech vectors (non-PD -> penalty); one GPU batch for all PD ones.
kde_status lscv_H_eval(kde_ctx* c, const double* X, int64_t n, int d, const Moments& m,
                       const std::vector<std::vector<double>>& vs, double penalty,
                       std::vector<double>& g, int* evals) {
  std::vector<HCand> pdc;
  std::vector<int> idx;
  g.assign(vs.size(), penalty);
  for (size_t k = 0; k < vs.size(); ++k) {
    HCand hc = h_candidate(vs[k].data(), d);
    if (hc.pd) { pdc.push_back(std::move(hc)); idx.push_back((int)k); }
  }
  if (pdc.empty()) return KDE_OK;
  std::vector<kde_fixed> o;
  TRY(lscv_H_raw(c, X, n, d, pdc, m, c->rank, c->world, true, o));
  for (size_t j = 0; j < pdc.size(); ++j)
    g[idx[j]] = lscv_H_finalize(n, d, pdc[j].det, fixed_value(o[2 * j]), fixed_value(o[2 * j + 1]));
  if (evals) *evals += (int)pdc.size();
  return KDE_OK;
}

// Input arrays may be device or host memory (include/kde.h): a host array (pageable or pinned)
// is copied into a context-owned device buffer on the context stream, so the rest of the call
// always reads device memory.  A device pointer of another GPU is rejected.
kde_status stage_input(kde_ctx* c, const double*& X, size_t count, int slot) {
  cudaPointerAttributes at;
  cudaError_t e = cudaPointerGetAttributes(&at, X);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(c, KDE_E_INVALID, "cannot classify the input pointer: %s", cudaGetErrorString(e));
  }
  if (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) {
    if (at.type == cudaMemoryTypeDevice && at.device != c->device)
      return fail(c, KDE_E_INVALID, "input lives on device %d, context on device %d", at.device, c->device);
    return KDE_OK;
  }
  Range r("kde.h2d");
  TRY(grow(c, &c->in_ws[slot], &c->in_bytes[slot], std::max<size_t>(count, 1) * sizeof(double)));
  CUDA_TRY(c, cudaMemcpyAsync(c->in_ws[slot], X, count * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  X = static_cast<const double*>(c->in_ws[slot]);
  return KDE_OK;
}

kde_status validate_X(kde_ctx* c, const double*& X, int64_t n, int32_t d, int64_t nmin) {
  if (!X) return fail(c, KDE_E_INVALID, "null sample pointer");
  if (d < 1 || d > kde::kMaxDim) return fail(c, KDE_E_DIM_MISMATCH, "d=%d outside [1,16]", d);
  if (n < nmin) return fail(c, n < 1 ? KDE_E_INVALID : KDE_E_INSUFFICIENT_SAMPLES, "n=%lld too small", (long long)n);
  if (n > 2147483647LL) return fail(c, KDE_E_INVALID, "n > 2^31-1");
  return stage_input(c, X, (size_t)n * (size_t)d, 0);
}

// ------------------------------------------------------------------ Nelder–Mead (reading Z8)
struct NMResult {
  std::vector<double> x;
  double f = 0.0;
  int iterations = 0, stop = 2, evals = 0;
};

// One Nelder–Mead run as a state machine: propose() lists the points whose objective values the
// next decision needs, accept() takes those values and applies the serial NM logic (rho = 1,
// chi = 2, gamma = sigma = 1/2; stable order by (f, index); stop on
// f_worst - f_best <= tol |f_best| or max_iter).  Speculative mode proposes reflect, expand,
// outside and inside contraction together; the decisions are those of serial NM on the same
// values.  Several runs can share one GPU batch (multi-start, row f4).
struct NMRun {
  enum Phase { INIT, STEP, SERIAL_R, SERIAL_1, SHRINK, DONE } phase = INIT;
  std::vector<std::vector<double>> sim;
  std::vector<double> fs;
  int M = 0, it = 0, max_iter = 500, stop = 2;
  double tol = 1e-7;
  bool speculative = true;
  std::vector<double> xbar, xr, xe, xc, xcc;
  double fr = 0.0;
  int serial_pick = 0;   // SERIAL_1: 1 = expand, 2 = outside contraction, 3 = inside contraction

  static std::vector<double> comb(const std::vector<double>& a, double s, const std::vector<double>& b,
                                  const std::vector<double>& c) {
    std::vector<double> r(a.size());
    for (size_t k = 0; k < a.size(); ++k) r[k] = a[k] + s * (b[k] - c[k]);
    return r;
  }

  // Sort, test the stopping rule and prepare the trial points of the next iteration.
  void begin_iteration() {
    std::vector<int> ord(M + 1);
    std::iota(ord.begin(), ord.end(), 0);
    std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return fs[a] < fs[b]; });
    std::vector<std::vector<double>> s2;
    std::vector<double> f2;
    for (int k : ord) { s2.push_back(sim[k]); f2.push_back(fs[k]); }
    sim.swap(s2);
    fs.swap(f2);
    if (fs[M] - fs[0] <= tol * std::fabs(fs[0])) { stop = 1; phase = DONE; return; }
    if (it >= max_iter) { stop = 2; phase = DONE; return; }
    ++it;
    xbar.assign(sim[0].size(), 0.0);
    for (int k = 0; k < M; ++k)
      for (size_t u = 0; u < xbar.size(); ++u) xbar[u] += sim[k][u];
    for (double& v : xbar) v /= (double)M;
    xr = comb(xbar, 1.0, xbar, sim[M]);
    xe = comb(xbar, 2.0, xr, xbar);
    xc = comb(xbar, 0.5, xr, xbar);
    xcc = comb(xbar, 0.5, sim[M], xbar);
    phase = speculative ? STEP : SERIAL_R;
  }

  std::vector<std::vector<double>> propose() const {
    switch (phase) {
      case INIT: return sim;
      case STEP: return {xr, xe, xc, xcc};
      case SERIAL_R: return {xr};
      case SERIAL_1: return {serial_pick == 1 ? xe : (serial_pick == 2 ? xc : xcc)};
      case SHRINK: {
        std::vector<std::vector<double>> sh;
        for (int k = 1; k <= M; ++k) sh.push_back(comb(sim[0], 0.5, sim[k], sim[0]));
        return sh;
      }
      default: return {};
    }
  }

  // Decide with f_r known and (speculatively or not) the one follow-up value.
  // Returns true if the follow-up value is still needed (serial mode).
  void decide(double fr_, bool have_follow, double fe, double fc, double fcc) {
    if (fr_ < fs[0]) {
      if (!have_follow) { serial_pick = 1; fr = fr_; phase = SERIAL_1; return; }
      if (fe < fr_) { sim[M] = xe; fs[M] = fe; } else { sim[M] = xr; fs[M] = fr_; }
      begin_iteration();
      return;
    }
    if (fr_ < fs[M - 1]) { sim[M] = xr; fs[M] = fr_; begin_iteration(); return; }
    if (fr_ < fs[M]) {
      if (!have_follow) { serial_pick = 2; fr = fr_; phase = SERIAL_1; return; }
      if (fc <= fr_) { sim[M] = xc; fs[M] = fc; begin_iteration(); return; }
    } else {
      if (!have_follow) { serial_pick = 3; fr = fr_; phase = SERIAL_1; return; }
      if (fcc < fs[M]) { sim[M] = xcc; fs[M] = fcc; begin_iteration(); return; }
    }
    phase = SHRINK;
  }

  void accept(const std::vector<double>& g) {
    switch (phase) {
      case INIT: fs = g; begin_iteration(); break;
      case STEP: decide(g[0], true, g[1], g[2], g[3]); break;
      case SERIAL_R: decide(g[0], false, 0, 0, 0); break;
      case SERIAL_1: {
        const double v = g[0];
        decide(fr, true, serial_pick == 1 ? v : 0, serial_pick == 2 ? v : 0, serial_pick == 3 ? v : 0);
        break;
      }
      case SHRINK: {
        for (int k = 1; k <= M; ++k) { sim[k] = comb(sim[0], 0.5, sim[k], sim[0]); fs[k] = g[k - 1]; }
        begin_iteration();
        break;
      }
      default: break;
    }
  }
};

// Run several NM instances in lockstep; every round evaluates the union of their proposals as
// one GPU batch (lscv_H_eval), so per-run decisions equal those of a lone run.
kde_status nelder_mead_multi(kde_ctx* c, const double* X, int64_t n, int d, const Moments& m,
                             const std::vector<std::vector<std::vector<double>>>& sims, int max_iter,
                             double tol, double penalty, bool speculative, NMResult& best, int* total_evals) {
  std::vector<NMRun> runs(sims.size());
  for (size_t r = 0; r < sims.size(); ++r) {
    runs[r].sim = sims[r];
    runs[r].M = (int)sims[r].size() - 1;
    runs[r].max_iter = max_iter;
    runs[r].tol = tol;
    runs[r].speculative = speculative;
  }
  int evals = 0;
  while (true) {
    std::vector<std::vector<double>> batch;
    std::vector<std::pair<size_t, size_t>> span;   // (run, count)
    for (size_t r = 0; r < runs.size(); ++r) {
      if (runs[r].phase == NMRun::DONE) continue;
      auto p = runs[r].propose();
      span.push_back({r, p.size()});
      for (auto& v : p) batch.push_back(std::move(v));
    }
    if (batch.empty()) break;
    std::vector<double> g;
    TRY(lscv_H_eval(c, X, n, d, m, batch, penalty, g, &evals));
    size_t off = 0;
    for (auto& sp : span) {
      std::vector<double> gv(g.begin() + off, g.begin() + off + sp.second);
      off += sp.second;
      runs[sp.first].accept(gv);
    }
  }
  size_t bi = 0;
  for (size_t r = 1; r < runs.size(); ++r)
    if (runs[r].fs[0] < runs[bi].fs[0]) bi = r;
  best.x = runs[bi].sim[0];
  best.f = runs[bi].fs[0];
  best.iterations = runs[bi].it;
  best.stop = runs[bi].stop;
  best.evals = evals;
  if (total_evals) *total_evals = evals;
  return KDE_OK;
}

}  // namespace

// ================================================================== C ABI
extern "C" {

void kde_default_opts(kde_select_opts* o) {
  if (!o) return;
  o->n_grid = 150;
  o->range_factor = 4.0;    // Eq. 27
  o->max_iter = 500;
  o->tol_rel = 1e-7;
  o->penalty = 1e300;
  o->speculative = 0;       // serial rounds: fewer candidates, faster on B200
  o->refine_steps = 0;
  o->refine_tol = 1e-9;
  o->nm_starts = 1;
}

kde_status kde_nccl_unique_id(void* out128) {
  if (!out128) return KDE_E_INVALID;
  NcclApi& api = nccl();
  if (!api.ok) return KDE_E_NCCL;
  ncclUniqueId id;
  if (api.GetUniqueId(&id) != 0) return KDE_E_NCCL;
  std::memcpy(out128, &id, sizeof(id));
  return KDE_OK;
}

kde_status kde_create(kde_ctx** out, int device, void* stream, const void* nccl_id, int rank, int world) {
  if (!out || world < 1 || rank < 0 || rank >= world) return KDE_E_INVALID;
  *out = nullptr;
  kde_ctx* c = new (std::nothrow) kde_ctx();
  if (!c) return KDE_E_OOM;
  c->device = device;
  c->stream = (cudaStream_t)stream;
  c->rank = rank;
  c->world = world;
  c->graphs = getenv("KDE_NO_GRAPHS") == nullptr;   // diagnostics: enqueue the PLUGIN chain directly
  if (cudaSetDevice(device) != cudaSuccess ||
      cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) {
    delete c;
    return KDE_E_CUDA;
  }
  if (nccl_id) {   // world == 1 with an id: single-rank communicator (tests); world > 1 without an
                   // id: no transport until kde_set_host_allreduce (test transport)
    NcclApi& api = nccl();
    if (!nccl_id || !api.ok) { delete c; return KDE_E_NCCL; }
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof(id));
    if (api.CommInitRank(&c->comm, world, id, rank) != 0) { delete c; return KDE_E_NCCL; }
  }
  *out = c;
  return KDE_OK;
}

void kde_destroy(kde_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream); else cudaDeviceSynchronize();
  if (c->plug_exec) cudaGraphExecDestroy(c->plug_exec);
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  if (c->comm) nccl().CommDestroy(c->comm);
  if (c->own_ws) cudaFree(c->own_ws);
  if (c->sort_ws) cudaFree(c->sort_ws);
  if (c->white_ws) cudaFree(c->white_ws);
  if (c->y64) cudaFree(c->y64);
  if (c->ev_ws) cudaFree(c->ev_ws);
  if (c->mat_ws) cudaFree(c->mat_ws);
  for (void* p : c->in_ws)
    if (p) cudaFree(p);
  if (c->h_limbs) cudaFreeHost(c->h_limbs);
  if (c->har_buf) cudaFreeHost(c->har_buf);
  for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
  delete c;
}

const char* kde_last_error(const kde_ctx* c) { return c ? c->err : "null context"; }

size_t kde_workspace_bytes(int64_t n, int32_t d, int32_t n_cand) {
  if (n < 1 || d < 1 || d > kde::kMaxDim) return 0;
  int64_t ld = (n + 2047) / 2048 * 2048;
  return ws_bytes(ld, d, 2 * (std::max(n_cand, 1) + 2 * kde::kMaxCand));
}

kde_status kde_set_workspace(kde_ctx* c, void* p, size_t bytes) {
  if (!c) return KDE_E_INVALID;
  c->ext_ws = p;
  c->ext_bytes = p ? bytes : 0;
  return KDE_OK;
}

kde_status kde_set_precision(kde_ctx* c, int32_t fp64_terms) {
  if (!c) return KDE_E_INVALID;
  c->fp64 = fp64_terms != 0;
  return KDE_OK;
}

kde_status kde_set_host_allreduce(kde_ctx* c, kde_host_allreduce_fn fn, void* user) {
  if (!c) return KDE_E_INVALID;
  if (c->comm) return fail(c, KDE_E_INVALID, "context already has an NCCL communicator");
  c->har_fn = fn;
  c->har_user = user;
  return KDE_OK;
}

kde_status kde_set_profiling(kde_ctx* c, int32_t on) {
  if (!c) return KDE_E_INVALID;
  c->profiling = on != 0;
  return KDE_OK;
}

kde_status kde_last_profile(const kde_ctx* c, int32_t* launches, double* ms, double* evals, int32_t* all) {
  if (!c) return KDE_E_INVALID;
  if (launches) *launches = c->prof_launches;
  if (ms) *ms = c->prof_ms;
  if (evals) *evals = c->prof_evals;
  if (all) *all = c->prof_all;
  return KDE_OK;
}

void kde_tile_coords(int64_t bx, int64_t* l, int64_t* q) {
  int64_t a = 0, b = 0;
  if (bx >= 0) kde::tile_coords_host(bx, &a, &b);
  if (l) *l = a;
  if (q) *q = b;
}

kde_status kde_shard_tiles(kde_sum_kind kind, int64_t n, int32_t d, int32_t rank, int32_t world,
                           int32_t* tile_edge, int64_t* tiles_total, int64_t* tb, int64_t* te) {
  if (n < 1 || d < 1 || d > kde::kMaxDim || world < 1 || rank < 0 || rank >= world) return KDE_E_INVALID;
  Kind k;
  switch (kind) {
    case KDE_SUM_PSI4: k = Kind::Psi4; break;
    case KDE_SUM_PSI6: k = Kind::Psi6; break;
    case KDE_SUM_PSI8: k = Kind::Psi8; break;
    case KDE_SUM_LSCV_h: k = Kind::LscvScalar; break;
    case KDE_SUM_LSCV_H: k = Kind::LscvMatrix; break;
    default: return KDE_E_INVALID;
  }
  const int T = kde::tile_for(k, d, n);
  const int64_t tiles = n_tiles(n, T);
  int64_t b, e;
  shard_range(tiles, rank, world, &b, &e);
  if (tile_edge) *tile_edge = T;
  if (tiles_total) *tiles_total = tiles;
  if (tb) *tb = b;
  if (te) *te = e;
  return KDE_OK;
}

double kde_fixed_value(const kde_fixed* v) { return v ? fixed_value(*v) : NAN; }

kde_fixed kde_fixed_add(kde_fixed a, kde_fixed b) {
  kde_fixed r = a;
  r.hi = (int64_t)((uint64_t)a.hi + (uint64_t)b.hi);
  r.mid = (int64_t)((uint64_t)a.mid + (uint64_t)b.mid);
  r.lo = (int64_t)((uint64_t)a.lo + (uint64_t)b.lo);
  return r;
}

kde_status kde_psi_r(kde_ctx* c, const double* x, int64_t n, int32_t r, const double* g, int32_t ng, double* psi) {
  TRY(check_ctx(c));
  prof_reset(c);
  TRY(validate_X(c, x, n, 1, 1));
  if (!(r == 4 || r == 6 || r == 8)) return fail(c, KDE_E_INVALID, "r=%d not in {4,6,8}", r);
  if (!g || !psi || ng < 1) return fail(c, KDE_E_INVALID, "null candidate/output array");
  for (int k = 0; k < ng; ++k)
    if (!(g[k] > 0.0) || !std::isfinite(g[k])) return fail(c, KDE_E_NONPOSITIVE_BW, "g[%d] <= 0", k);
  Ws w;
  TRY(get_ws(c, (n + 2047) / 2048 * 2048, 1, 2, &w));
  Moments m;
  if (n >= 2) {
    TRY(gpu_moments(c, x, n, 1, w, m));
  } else {
    m.mean = {0.0};
  }
  std::vector<kde_fixed> o;
  TRY(psi_raw(c, x, n, r, g, ng, m, c->rank, c->world, true, o));
  TRY(prof_collect(c));
  for (int k = 0; k < ng; ++k) psi[k] = psi_finalize(r, n, g[k], fixed_value(o[k]));
  return KDE_OK;
}

// One Psi_r pair pass of the device-resident PLUGIN chain: kernel over this rank's tiles into
// `limbs`, then (world > 1) the all-reduce of the 3 limbs, all enqueued on the context stream.
static kde_status plugin_pass(kde_ctx* c, int r, int64_t n, int64_t ld, int T, int S, Ws& w,
                              unsigned long long* limbs, int64_t tb, int64_t te, double pairs) {
  Range rr("kde.pair_pass");
  kde::LaunchCfg cfg;
  cfg.X = w.Y; cfg.n = n; cfg.ld = ld; cfg.tile_begin = tb; cfg.tile_end = te; cfg.tile = T;
  cfg.scale_exp = S; cfg.limbs = limbs; cfg.n_out = 1; cfg.stream = c->stream; cfg.sm_count = c->sm_count;
  cfg.clamp = w.flag() + 1;
  kde::PsiParams p;
  psi_coeffs(r, p);
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  // external event records: inside a graph capture they become timing event nodes
  const unsigned rec = (c->cap_stream && c->stream == c->cap_stream) ? cudaEventRecordExternal : cudaEventRecordDefault;
  if (c->profiling) { e0 = next_event(c); e1 = next_event(c); CUDA_TRY(c, cudaEventRecordWithFlags(e0, c->stream, rec)); }
  cudaError_t err = kde::launch_psi(r, cfg, p);
  if (err != cudaSuccess) return fail(c, KDE_E_CUDA, "pair kernel launch: %s", cudaGetErrorString(err));
  if (tb < te) c->prof_all += 1;
  if (c->profiling) {
    CUDA_TRY(c, cudaEventRecordWithFlags(e1, c->stream, rec));
    c->prof_launches++;
    c->prof_evals += pairs;
  }
  TRY(allreduce_limbs(c, limbs, kde::kLimbs));
  return KDE_OK;
}

// PLUGIN (Sec. 4.4.1): moments, sort, prep and the two pair passes, with the scalar
// steps 1-8 computed by single-thread kernels on the device between them, so the whole chain is
// enqueued without a host round trip and the call synchronises once.  The steps' formulas are those
// of the host reading (Z1, Z10, Z11); failures are recorded on the device and reported in order.
// Enqueue the whole chain on c->stream (no allocation, no synchronisation: capturable).
static kde_status plugin_enqueue(kde_ctx* c, const double* x, int64_t n, int T, int64_t ld, Ws& w) {
  kde::PluginDev dv(w.small);
  const int nblk = kde::moments_blocks(n);
  cudaStream_t st = c->stream;
  // flags (2 x u64), trace (8) and status (1) start at zero
  CUDA_TRY(c, cudaMemsetAsync(w.flag(), 0, (kde::kSmallDoubles - 408) * sizeof(double), st));
  {
    Range r("kde.moments");
    CUDA_TRY(c, kde::launch_moments1(x, n, 1, w.part, nblk, st));
    CUDA_TRY(c, kde::launch_reduce_parts(w.part, nblk, 1, dv.sums, st));
    CUDA_TRY(c, kde::launch_plugin_chain(0, n, w.small, nullptr, 0, st));             // mean
    CUDA_TRY(c, kde::launch_moments2(x, n, 1, dv.mean, w.part, nblk, st));
    CUDA_TRY(c, kde::launch_reduce_parts(w.part, nblk, 1, dv.sums, st));
    CUDA_TRY(c, kde::launch_plugin_chain(1, n, w.small, nullptr, 0, st));             // steps 1-4
    c->prof_all += 6;
  }
  const double* xs = nullptr;                                                          // sorted once (§3)
  TRY(gpu_sorted(c, x, n, &xs));
  int64_t tb, te;
  shard_range(n_tiles(n, T), c->rank, c->world, &tb, &te);
  const double pairs = c->profiling ? pairs_in_range(n, T, tb, te) : 0.0;
  const int S6 = scale_exp_for(2.0 * 15.0, n), S4 = scale_exp_for(2.0 * 3.0, n);
  CUDA_TRY(c, cudaMemsetAsync(w.limbs, 0, 2 * kde::kLimbs * sizeof(long long), st));
  if (c->fp64) {                                                                       // fp64 terms
    double* y = static_cast<double*>(c->y64);
    CUDA_TRY(c, kde::launch_scale64(xs, n, dv.mean, dv.W, y, st));                     // x/g1
    TRY(psi64_pass(c, 6, y, n, S6, w.limbs));                                          // step 5
    CUDA_TRY(c, kde::launch_plugin_chain(2, n, w.small, w.limbs, S6, st));             // Psi6, g2
    CUDA_TRY(c, kde::launch_scale64(xs, n, dv.mean, dv.W, y, st));                     // x/g2
    TRY(psi64_pass(c, 4, y, n, S4, w.limbs + kde::kLimbs));                            // step 7
  } else {
    CUDA_TRY(c, kde::launch_prep(xs, n, 1, dv.W, dv.mean, w.Y, ld, st, 0.f, w.flag(), 3.0e4));   // x/g1
    TRY(plugin_pass(c, 6, n, ld, T, S6, w, w.limbs, tb, te, pairs));                   // step 5
    CUDA_TRY(c, kde::launch_plugin_chain(2, n, w.small, w.limbs, S6, st));             // Psi6, g2
    CUDA_TRY(c, kde::launch_prep(xs, n, 1, dv.W, dv.mean, w.Y, ld, st, 0.f, w.flag(), 3.0e4));   // x/g2
    TRY(plugin_pass(c, 4, n, ld, T, S4, w, w.limbs + kde::kLimbs, tb, te, pairs));     // step 7
  }
  CUDA_TRY(c, kde::launch_plugin_chain(3, n, w.small, w.limbs + kde::kLimbs, S4, st)); // Psi4, h
  c->prof_all += 4;
  CUDA_TRY(c, cudaMemcpyAsync(c->h_limbs, w.flag(), (kde::kSmallDoubles - 408) * sizeof(double),
                              cudaMemcpyDeviceToHost, st));
  return KDE_OK;
}

// PLUGIN (Sec. 4.4.1): moments, sort, prep and the two pair passes, with the scalar
// steps 1-8 computed by single-thread kernels on the device between them, so the whole chain is
// enqueued without a host round trip and the call synchronises once.  The chain is captured once
// as a CUDA graph and replayed while its inputs (pointers, n, mode) are unchanged.  The steps'
// formulas are those of the host reading (Z1, Z10, Z11); failures are recorded on the device and
// reported in order.
static kde_status plugin_impl(kde_ctx* c, const double* x, int64_t n, kde_plugin_trace* tr) {
  const int T = kde::tile_for(Kind::Psi6, 1, n);
  const int64_t ld = (n + T - 1) / T * T;
  Ws w;
  TRY(get_ws(c, ld, 1, 2, &w));                   // everything the chain touches exists before
  TRY(ensure_sort_ws(c, n));                      // a capture starts
  if (c->fp64) TRY(grow(c, &c->y64, &c->y64_bytes, (size_t)n * sizeof(double)));
  const size_t cnt = kde::kSmallDoubles - 408;    // flags, trace, status
  if (c->h_limbs_cap < cnt) {
    if (c->h_limbs) cudaFreeHost(c->h_limbs);
    c->h_limbs = nullptr;
    CUDA_TRY(c, cudaMallocHost(&c->h_limbs, cnt * sizeof(long long)));
    c->h_limbs_cap = cnt;
  }
  for (int r : {6, 4}) {                          // kernel attributes: not settable while capturing
    kde::LaunchCfg cfg;
    cfg.n = n; cfg.tile = T; cfg.sm_count = c->sm_count;
    CUDA_TRY(c, kde::prepare_psi(r, cfg));
  }
  cudaStream_t st = c->stream;
  const std::vector<uintptr_t> key = {(uintptr_t)x, (uintptr_t)n, (uintptr_t)w.Y, (uintptr_t)c->sort_ws,
                                      (uintptr_t)c->h_limbs, (uintptr_t)c->profiling, (uintptr_t)c->comm,
                                      (uintptr_t)c->fp64, (uintptr_t)c->y64};
  // The first call with a given key runs directly (and does any lazy module loading and library
  // setup outside a capture); a second call with the same key captures, later ones replay.
  // (single-GPU contexts only: with a communicator the all-reduces stay plain stream operations)
  if (!c->graphs || c->comm || c->world > 1 || (key != c->plug_seen && !(c->plug_exec && key == c->plug_key))) {
    TRY(plugin_enqueue(c, x, n, T, ld, w));
    c->plug_seen = key;
  } else {
    if (!(c->plug_exec && key == c->plug_key)) {
      Range r("kde.capture");
      if (!c->cap_stream) CUDA_TRY(c, cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
      if (c->plug_exec) { cudaGraphExecDestroy(c->plug_exec); c->plug_exec = nullptr; }
      CUDA_TRY(c, cudaStreamSynchronize(st));
      cudaGetLastError();
      CUDA_TRY(c, cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeRelaxed));
      c->stream = c->cap_stream;
      const int32_t l0 = c->prof_launches, a0 = c->prof_all;
      const double e0 = c->prof_evals;
      const kde_status es = plugin_enqueue(c, x, n, T, ld, w);
      c->stream = st;
      cudaGraph_t g = nullptr;
      const cudaError_t ce = cudaStreamEndCapture(c->cap_stream, &g);
      if (es != KDE_OK) { if (g) cudaGraphDestroy(g); return es; }
      if (ce != cudaSuccess) return fail(c, KDE_E_CUDA, "graph capture: %s", cudaGetErrorString(ce));
      const cudaError_t ie = cudaGraphInstantiate(&c->plug_exec, g, 0);
      cudaGraphDestroy(g);
      if (ie != cudaSuccess) { c->plug_exec = nullptr; return fail(c, KDE_E_CUDA, "graph instantiate: %s", cudaGetErrorString(ie)); }
      c->plug_key = key;
      c->plug_prof_launches = c->prof_launches - l0;
      c->plug_prof_all = c->prof_all - a0;
      c->plug_prof_evals = c->prof_evals - e0;
      c->plug_ev_used = c->ev_used;
    } else {
      c->prof_launches += c->plug_prof_launches;
      c->prof_all += c->plug_prof_all;
      c->prof_evals += c->plug_prof_evals;
      c->ev_used = c->plug_ev_used;   // the graph records the same pool events
    }
    CUDA_TRY(c, cudaGraphLaunch(c->plug_exec, st));
  }
  CUDA_TRY(c, cudaStreamSynchronize(st));
  const unsigned long long* flags = reinterpret_cast<const unsigned long long*>(c->h_limbs);
  double res[9];
  std::memcpy(res, c->h_limbs + 2, sizeof(res));
  const int status = (int)res[8];
  if (status == KDE_E_INVALID) return fail(c, KDE_E_INVALID, "non-finite sample values");
  if (status == KDE_E_DEGENERATE) return fail(c, KDE_E_DEGENERATE, "variance estimate <= 0");
  if (flags[0]) return fail(c, KDE_E_INVALID, "scaled sample differences exceed 1e18 (outliers vs. bandwidth)");
  if (status == KDE_E_NUMERIC)
    return fail(c, KDE_E_NUMERIC, !(res[4] < 0.0) ? "Psi6-hat >= 0" : "Psi4-hat <= 0");
  kde_plugin_trace t;
  t.V_hat = res[0]; t.sigma_hat = res[1]; t.psi8_ns = res[2]; t.g1 = res[3];
  t.psi6 = res[4]; t.g2 = res[5]; t.psi4 = res[6]; t.h = res[7];
  *tr = t;
  return KDE_OK;
}

kde_status kde_plugin_h(kde_ctx* c, const double* x, int64_t n, double* h, kde_plugin_trace* tr) {
  TRY(check_ctx(c));
  prof_reset(c);
  TRY(validate_X(c, x, n, 1, 2));
  if (!h) return fail(c, KDE_E_INVALID, "null output");
  kde_plugin_trace t;
  TRY(plugin_impl(c, x, n, &t));
  TRY(prof_collect(c));
  *h = t.h;
  if (tr) *tr = t;
  return KDE_OK;
}

static kde_status lscv_h_scores_impl(kde_ctx* c, const double* X, int64_t n, int d, const double* h,
                                     int nh, double* g) {
  Ws w;
  TRY(get_ws(c, (n + 2047) / 2048 * 2048, d, 2, &w));
  Moments m;
  TRY(gpu_moments(c, X, n, d, w, m));
  LscvhPrep pp;
  TRY(lscv_h_prepare(c, m, d, pp));
  std::vector<kde_fixed> o;
  TRY(lscv_h_raw(c, X, n, d, h, nh, m, pp, c->rank, c->world, true, o));
  for (int k = 0; k < nh; ++k)
    g[k] = lscv_h_finalize(n, d, pp.det, h[k], fixed_value(o[2 * k]), fixed_value(o[2 * k + 1]));
  return KDE_OK;
}

kde_status kde_lscv_h_scores(kde_ctx* c, const double* X, int64_t n, int32_t d, const double* h,
                             int32_t nh, double* g) {
  TRY(check_ctx(c));
  prof_reset(c);
  TRY(validate_X(c, X, n, d, 2));
  if (!h || !g || nh < 1) return fail(c, KDE_E_INVALID, "null candidate/output array");
  for (int k = 0; k < nh; ++k)
    if (!(h[k] > 0.0) || !std::isfinite(h[k])) return fail(c, KDE_E_NONPOSITIVE_BW, "h[%d] <= 0", k);
  std::vector<double> tmp(nh);
  TRY(lscv_h_scores_impl(c, X, n, d, h, nh, tmp.data()));
  TRY(prof_collect(c));
  std::copy(tmp.begin(), tmp.end(), g);
  return KDE_OK;
}

kde_status kde_lscv_H_scores(kde_ctx* c, const double* X, int64_t n, int32_t d, const double* vh,
                             int32_t nH, double penalty, double* g) {
  TRY(check_ctx(c));
  prof_reset(c);
  TRY(validate_X(c, X, n, d, 2));
  if (!vh || !g || nH < 1) return fail(c, KDE_E_INVALID, "null candidate/output array");
  if (std::isnan(penalty)) penalty = 1e300;
  const int P = d * (d + 1) / 2;
  Ws w;
  TRY(get_ws(c, (n + 2047) / 2048 * 2048, d, 2, &w));
  Moments m;
  TRY(gpu_moments(c, X, n, d, w, m));
  std::vector<std::vector<double>> vs;
  for (int k = 0; k < nH; ++k) vs.emplace_back(vh + (size_t)k * P, vh + (size_t)(k + 1) * P);
  std::vector<double> out;
  TRY(lscv_H_eval(c, X, n, d, m, vs, penalty, out, nullptr));
  TRY(prof_collect(c));
  std::copy(out.begin(), out.end(), g);
  return KDE_OK;
}

kde_status kde_raw_sums(kde_ctx* c, kde_sum_kind kind, const double* X, int64_t n, int32_t d,
                        const double* cand, int32_t nc, int32_t srank, int32_t sworld, kde_fixed* out) {
  TRY(check_ctx(c));
  prof_reset(c);
  TRY(validate_X(c, X, n, d, 1));
  if (!cand || !out || nc < 1) return fail(c, KDE_E_INVALID, "null candidate/output array");
  bool allreduce = sworld == 0;
  if (sworld == 0) { srank = c->rank; sworld = c->world; }
  if (srank < 0 || srank >= sworld) return fail(c, KDE_E_INVALID, "bad shard");
  Ws w;
  TRY(get_ws(c, (n + 2047) / 2048 * 2048, d, 2, &w));
  Moments m;
  if (n >= 2) {
    TRY(gpu_moments(c, X, n, d, w, m));
  } else {
    m.mean.assign(d, 0.0);
    m.cov.assign((size_t)d * d, 0.0);
  }
  std::vector<kde_fixed> o;
  if (kind == KDE_SUM_PSI4 || kind == KDE_SUM_PSI6 || kind == KDE_SUM_PSI8) {
    if (d != 1) return fail(c, KDE_E_NOT_UNIVARIATE, "Psi sums need d = 1");
    for (int k = 0; k < nc; ++k)
      if (!(cand[k] > 0.0)) return fail(c, KDE_E_NONPOSITIVE_BW, "g <= 0");
    TRY(psi_raw(c, X, n, (int)kind, cand, nc, m, srank, sworld, allreduce, o));
  } else if (kind == KDE_SUM_LSCV_h) {
    if (n < 2) return fail(c, KDE_E_INSUFFICIENT_SAMPLES, "n < 2");
    for (int k = 0; k < nc; ++k)
      if (!(cand[k] > 0.0)) return fail(c, KDE_E_NONPOSITIVE_BW, "h <= 0");
    LscvhPrep pp;
    TRY(lscv_h_prepare(c, m, d, pp));
    TRY(lscv_h_raw(c, X, n, d, cand, nc, m, pp, srank, sworld, allreduce, o));
  } else if (kind == KDE_SUM_LSCV_H) {
    const int P = d * (d + 1) / 2;
    std::vector<HCand> hc;
    for (int k = 0; k < nc; ++k) {
      hc.push_back(h_candidate(cand + (size_t)k * P, d));
      if (!hc.back().pd) return fail(c, KDE_E_INVALID, "candidate %d is not positive definite", k);
    }
    if (n < 2) m.mean.assign(d, 0.0);
    TRY(lscv_H_raw(c, X, n, d, hc, m, srank, sworld, allreduce, o));
  } else {
    return fail(c, KDE_E_INVALID, "unknown sum kind");
  }
  TRY(prof_collect(c));
  std::copy(o.begin(), o.end(), out);
  return KDE_OK;
}

kde_status kde_evaluate(kde_ctx* c, const double* X, int64_t n, int32_t d, const double* Y, int64_t m,
                        const double* vh, double* f) {
  TRY(check_ctx(c));
  prof_reset(c);
  TRY(validate_X(c, X, n, d, 1));
  if (!Y || !vh || !f || m < 0) return fail(c, KDE_E_INVALID, "null query/bandwidth/output pointer");
  if (m == 0) return KDE_OK;
  if (m > 2147483647LL) return fail(c, KDE_E_INVALID, "m > 2^31-1");
  TRY(stage_input(c, Y, (size_t)m * (size_t)d, 1));
  std::vector<double> H = unvech(vh, d), L;
  if (!cholesky(H, d, L)) return fail(c, KDE_E_NONPOSITIVE_BW, "bandwidth matrix is not positive definite");
  double det = 1.0;
  for (int i = 0; i < d; ++i) det *= L[i * d + i] * L[i * d + i];
  // W^T W = (log2 e / 2) H^-1  =>  2^-|W v|^2 = exp(-v^T H^-1 v / 2)
  std::vector<double> W = tri_lower_inverse(L, d);
  for (double& v : W) v *= std::sqrt(kLog2e / 2.0);
  const int64_t R = kde::eval_rows_per_block(), TC = kde::eval_cols_per_tile();
  const int64_t ldm = (m + R - 1) / R * R, ldn = (n + TC - 1) / TC * TC;
  const size_t parts = (size_t)kde::eval_max_splits(c->sm_count) * (size_t)ldm;
  const size_t need = align256((size_t)d * ldm * 4) + align256((size_t)d * ldn * 4) + align256(parts * 8) +
                      align256((size_t)m * 8);
  TRY(grow(c, &c->ev_ws, &c->ev_bytes, need));
  char* p = (char*)c->ev_ws;
  float* Yw = (float*)p; p += align256((size_t)d * ldm * 4);
  float* Xw = (float*)p; p += align256((size_t)d * ldn * 4);
  double* part = (double*)p; p += align256(parts * 8);
  double* out = (double*)p;
  Ws w;
  TRY(get_ws(c, 256, d, 2, &w));
  // centre both sets on the sample mean (fp32 accuracy of the differences)
  const int nblk = kde::moments_blocks(n);
  double* sums = w.small + 16 + 256;
  double hs[16];
  CUDA_TRY(c, kde::launch_moments1(X, n, d, w.part, nblk, c->stream));
  CUDA_TRY(c, kde::launch_reduce_parts(w.part, nblk, d, sums, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(hs, sums, d * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  std::vector<double> mean(d);
  for (int a = 0; a < d; ++a) {
    if (!std::isfinite(hs[a])) return fail(c, KDE_E_INVALID, "non-finite sample values");
    mean[a] = hs[a] / (double)n;
  }
  kde::PrepParams pp;
  std::copy(W.begin(), W.begin() + (size_t)d * d, pp.W);
  std::copy(mean.begin(), mean.begin() + d, pp.mean);
  CUDA_TRY(c, cudaMemsetAsync(w.flag(), 0, sizeof(unsigned long long), c->stream));
  CUDA_TRY(c, kde::launch_prep_params(X, n, d, pp, Xw, ldn, c->stream, __int_as_float_host(0x7f800000), w.flag()));
  CUDA_TRY(c, kde::launch_prep_params(Y, m, d, pp, Yw, ldm, c->stream, 0.f, w.flag()));
  kde::EvalLaunch el;
  el.Y = Yw; el.X = Xw; el.m = m; el.ldm = ldm; el.ldn = ldn; el.part = part; el.part_capacity = parts;
  el.scale = std::pow(2.0 * kPi, -0.5 * d) / std::sqrt(det) / (double)n;
  el.out = out; el.stream = c->stream; el.sm_count = c->sm_count;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (c->profiling) { e0 = next_event(c); e1 = next_event(c); cudaEventRecord(e0, c->stream); }
  c->prof_all += 1 + 2 + 2 + 2;   // moments1 + reduce, 2 x prep, eval + reduce
  cudaError_t err = kde::launch_eval(d, el);
  if (err != cudaSuccess) return fail(c, KDE_E_CUDA, "eval launch: %s", cudaGetErrorString(err));
  if (c->profiling) {
    cudaEventRecord(e1, c->stream);
    c->prof_launches++;
    c->prof_evals += (double)m * (double)n;
  }
  std::vector<double> tmp(m);
  CUDA_TRY(c, cudaMemcpyAsync(tmp.data(), out, (size_t)m * 8, cudaMemcpyDeviceToHost, c->stream));
  unsigned long long overflow = 0;
  CUDA_TRY(c, cudaMemcpyAsync(&overflow, w.flag(), sizeof(overflow), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  if (overflow) return fail(c, KDE_E_INVALID, "whitened sample/query values exceed 1e18");
  TRY(prof_collect(c));
  std::copy(tmp.begin(), tmp.end(), f);
  return KDE_OK;
}

kde_status kde_aqp_1d(kde_ctx* c, const double* x, int64_t n, double h, const double* lo, const double* hi,
                      int32_t nq, double* count, double* sum, double* avg) {
  TRY(check_ctx(c));
  prof_reset(c);
  TRY(validate_X(c, x, n, 1, 1));
  if (!lo || !hi || nq < 1) return fail(c, KDE_E_INVALID, "null interval arrays");
  if (!(h > 0.0) || !std::isfinite(h)) return fail(c, KDE_E_NONPOSITIVE_BW, "h <= 0");
  for (int q = 0; q < nq; ++q)
    if (!(lo[q] <= hi[q])) return fail(c, KDE_E_INVALID, "interval %d has lo > hi or NaN", q);
  const int nblk = kde::aqp_blocks(n);
  const size_t need = align256((size_t)nq * nblk * 2 * 8) + 3 * align256((size_t)nq * 2 * 8);
  TRY(grow(c, &c->ev_ws, &c->ev_bytes, need));
  char* p = (char*)c->ev_ws;
  double* part = (double*)p; p += align256((size_t)nq * nblk * 2 * 8);
  double* dlo = (double*)p; p += align256((size_t)nq * 2 * 8);
  double* dhi = (double*)p; p += align256((size_t)nq * 2 * 8);
  double* out = (double*)p;
  CUDA_TRY(c, cudaMemcpyAsync(dlo, lo, nq * 8, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(dhi, hi, nq * 8, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, kde::launch_aqp(x, n, h, dlo, dhi, nq, part, nblk, out, c->stream));
  c->prof_all += 2;
  std::vector<double> tmp((size_t)nq * 2);
  CUDA_TRY(c, cudaMemcpyAsync(tmp.data(), out, (size_t)nq * 16, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  for (int q = 0; q < nq; ++q) {
    if (count) count[q] = tmp[2 * q];
    if (sum) sum[q] = tmp[2 * q + 1];
    if (avg) avg[q] = tmp[2 * q + 1] / tmp[2 * q];
  }
  return KDE_OK;
}

kde_status kde_lscv_h_scores_materialized(kde_ctx* c, const double* X, int64_t n, int32_t d, const double* h,
                                          int32_t nh, int32_t h_per_pass, double* g) {
  TRY(check_ctx(c));
  prof_reset(c);
  TRY(validate_X(c, X, n, d, 2));
  if (!h || !g || nh < 1) return fail(c, KDE_E_INVALID, "null candidate/output array");
  if (!(h_per_pass == 1 || h_per_pass == 2 || h_per_pass == 4 || h_per_pass == 8 || h_per_pass == 16))
    return fail(c, KDE_E_INVALID, "h_per_pass must be 1, 2, 4, 8 or 16");
  for (int k = 0; k < nh; ++k)
    if (!(h[k] > 0.0) || !std::isfinite(h[k])) return fail(c, KDE_E_NONPOSITIVE_BW, "h[%d] <= 0", k);
  const int T = kde::mat_tile();
  const int64_t ld = (n + T - 1) / T * T;
  const int B = h_per_pass;
  const int nbatch = (nh + B - 1) / B;
  const int n_out = 2 * nbatch * B;
  Ws w;
  TRY(get_ws(c, ld, d, n_out, &w));
  Moments m;
  TRY(gpu_moments(c, X, n, d, w, m));
  LscvhPrep pp;
  TRY(lscv_h_prepare(c, m, d, pp));
  std::vector<double> W = tri_lower_inverse(pp.Lc, d);
  for (double& v : W) v *= std::sqrt(kLog2e / 4.0);
  TRY(gpu_prep(c, X, n, d, W, m.mean, ld, w));
  int64_t tb, te;
  shard_range(n_tiles(n, T), c->rank, c->world, &tb, &te);
  const int64_t nvalues = (te - tb) * (int64_t)T * T;
  TRY(grow(c, &c->mat_ws, &c->mat_bytes, (size_t)std::max<int64_t>(nvalues, 1) * sizeof(float)));
  float* buf = (float*)c->mat_ws;
  cudaEvent_t a0 = nullptr, a1 = nullptr;
  if (c->profiling) { a0 = next_event(c); a1 = next_event(c); cudaEventRecord(a0, c->stream); }
  CUDA_TRY(c, kde::launch_mat_write(d, w.Y, n, ld, tb, te, buf, c->sm_count, c->stream));   // phase 1
  c->prof_all += 1;
  if (c->profiling) cudaEventRecord(a1, c->stream);
  CUDA_TRY(c, cudaMemsetAsync(w.limbs, 0, (size_t)n_out * kde::kLimbs * sizeof(long long), c->stream));
  const int S = scale_exp_for(1.0, n);
  const double pairs = c->profiling ? pairs_in_range(n, T, tb, te) : 0.0;
  for (int b = 0; b < nbatch; ++b) {                                                          // phase 2
    kde::LscvScalarParams p;
    for (int j = 0; j < kde::kMaxCand; ++j) {
      const int idx = std::min(b * B + j, nh - 1);
      p.kappa[j] = (float)(-1.0 / (h[idx] * h[idx]));
    }
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (c->profiling) { e0 = next_event(c); e1 = next_event(c); cudaEventRecord(e0, c->stream); }
    CUDA_TRY(c, kde::launch_mat_reduce(B, buf, nvalues, p, S, w.limbs + (size_t)2 * b * B * kde::kLimbs,
                                       c->sm_count, c->stream));
    c->prof_all += 1;
    if (c->profiling) {
      cudaEventRecord(e1, c->stream);
      c->prof_launches++;
      c->prof_evals += pairs * B;
    }
  }
  TRY(allreduce_limbs(c, w.limbs, (size_t)n_out * kde::kLimbs));
  std::vector<long long> hl((size_t)n_out * kde::kLimbs);
  CUDA_TRY(c, cudaMemcpyAsync(hl.data(), w.limbs, hl.size() * sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
  unsigned long long overflow = 0;
  CUDA_TRY(c, cudaMemcpyAsync(&overflow, w.flag(), sizeof(overflow), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  if (overflow) return fail(c, KDE_E_INVALID, "scaled sample differences exceed 1e18");
  if (c->profiling) {
    float x = 0.f;
    cudaEventElapsedTime(&x, a0, a1);
    c->prof_aux_ms = x;
    double ms = 0.0;
    for (size_t k = 2; k + 1 < c->ev_used; k += 2) {
      CUDA_TRY(c, cudaEventElapsedTime(&x, c->ev_pool[k], c->ev_pool[k + 1]));
      ms += x;
    }
    c->prof_ms = ms;
  }
  for (int k = 0; k < nh; ++k) {
    const double S1 = fixed_value(limbs_to_fixed(&hl[(size_t)2 * k * kde::kLimbs], S));
    const double S2 = fixed_value(limbs_to_fixed(&hl[(size_t)(2 * k + 1) * kde::kLimbs], S));
    g[k] = lscv_h_finalize(n, d, pp.det, h[k], S1, S2);
  }
  return KDE_OK;
}

double kde_last_aux_ms(const kde_ctx* c) { return c ? c->prof_aux_ms : 0.0; }

kde_status kde_select_bandwidth(kde_ctx* c, kde_method method, const double* X, int64_t n, int32_t d,
                                const kde_select_opts* opts_in, kde_bandwidth* out) {
  TRY(check_ctx(c));
  prof_reset(c);
  if (!out) return fail(c, KDE_E_INVALID, "null output");
  kde_select_opts o;
  kde_default_opts(&o);
  if (opts_in) o = *opts_in;
  TRY(validate_X(c, X, n, d, 2));
  kde_bandwidth r;
  std::memset(&r, 0, sizeof(r));
  r.method = method;
  r.d = d;
  if (method == KDE_PLUGIN) {
    if (d != 1) return fail(c, KDE_E_NOT_UNIVARIATE, "PLUGIN is univariate (P:196)");
    TRY(plugin_impl(c, X, n, &r.trace));
    r.h = r.trace.h;
    r.evaluations = 2;
  } else if (method == KDE_LSCV_h) {
    if (o.n_grid < 2 || !(o.range_factor > 1.0)) return fail(c, KDE_E_INVALID, "bad grid options");
    // Eq. 25 as written (reading Z3): R(K)/mu2^2 = 1/(2^d pi^{d/2} d^2), R(f'') = d(d+2)/(2^{d+2} pi^{d/2})
    const double dd = d;
    const double ratio = 1.0 / (std::pow(2.0, dd) * std::pow(kPi, dd / 2) * dd * dd);
    const double Rf2 = dd * (dd + 2) / (std::pow(2.0, dd + 2) * std::pow(kPi, dd / 2));
    const double h0 = std::pow(ratio / (Rf2 * (double)n), 1.0 / (dd + 4));
    const double lo = h0 / o.range_factor, hi = h0 * o.range_factor;       // Eq. 27
    std::vector<double> hs(o.n_grid), gs(o.n_grid);
    for (int k = 0; k < o.n_grid; ++k) hs[k] = lo + k * (hi - lo) / (o.n_grid - 1);
    TRY(lscv_h_scores_impl(c, X, n, d, hs.data(), o.n_grid, gs.data()));
    int best = 0;
    for (int k = 1; k < o.n_grid; ++k)
      if (gs[k] < gs[best]) best = k;                                    // ties -> smaller h
    r.h = hs[best];
    r.objective = gs[best];
    r.iterations = best;
    r.evaluations = o.n_grid;
    // Optional refinement (f4): bracket = the grid neighbours of the argmin; each step scores
    // 16 equally spaced interior points in one pass and re-brackets around the best known point
    // (ties -> smaller h).  A batched form of the section search the paper suggests.
    if (o.refine_steps > 0) {
      std::vector<std::pair<double, double>> pts;   // (h, g) known inside the bracket, sorted by h
      pts.push_back({hs[best > 0 ? best - 1 : 0], gs[best > 0 ? best - 1 : 0]});
      if (best > 0) pts.push_back({hs[best], gs[best]});
      if (best + 1 < o.n_grid) pts.push_back({hs[best + 1], gs[best + 1]});
      int steps = 0;
      while (steps < o.refine_steps) {
        const double a = pts.front().first, b = pts.back().first;
        if (!(b - a > o.refine_tol * r.h)) break;
        std::vector<double> hh(16), gg(16);
        for (int k = 0; k < 16; ++k) hh[k] = a + (k + 1) * (b - a) / 17.0;
        TRY(lscv_h_scores_impl(c, X, n, d, hh.data(), 16, gg.data()));
        r.evaluations += 16;
        for (int k = 0; k < 16; ++k) pts.push_back({hh[k], gg[k]});
        std::sort(pts.begin(), pts.end());
        size_t bi = 0;
        for (size_t k = 1; k < pts.size(); ++k)
          if (pts[k].second < pts[bi].second) bi = k;
        r.h = pts[bi].first;
        r.objective = pts[bi].second;
        const size_t lo_i = bi > 0 ? bi - 1 : 0, hi_i = bi + 1 < pts.size() ? bi + 1 : bi;
        std::vector<std::pair<double, double>> nb(pts.begin() + lo_i, pts.begin() + hi_i + 1);
        pts.swap(nb);
        ++steps;
      }
      r.stop_reason = steps;
    }
  } else if (method == KDE_LSCV_H) {
    Ws w;
    TRY(get_ws(c, (n + 2047) / 2048 * 2048, d, 2, &w));
    Moments m;
    TRY(gpu_moments(c, X, n, d, w, m));
    std::vector<double> Lc, root;
    if (!cholesky(m.cov, d, Lc)) return fail(c, KDE_E_SINGULAR_COV, "covariance not positive definite");
    if (!spd_sqrt(m.cov, d, root)) return fail(c, KDE_E_SINGULAR_COV, "matrix square root failed");
    // Eq. 35 as written: H_start = (4/(d+2))^{1/(d+4)} n^{-1/(d+4)} Sigma^{1/2}
    const double f = std::pow(4.0 / (d + 2), 1.0 / (d + 4)) * std::pow((double)n, -1.0 / (d + 4));
    for (double& v : root) v *= f;
    const int P = d * (d + 1) / 2;
    std::vector<double> x0(P);
    vech(root, d, x0.data());
    std::vector<std::vector<double>> sim = {x0};
    int t = 0;
    for (int b = 0; b < d; ++b)
      for (int a = b; a < d; ++a) {
        const double delta = 0.1 * (a == b ? root[a * d + a] : std::sqrt(root[a * d + a] * root[b * d + b]));
        std::vector<double> v = x0;
        v[t] += delta;
        sim.push_back(v);
        ++t;
      }
    // start k of o.nm_starts: vech(H_start) scaled by 4^-k (the paper's Eq. 35 start first)
    std::vector<std::vector<std::vector<double>>> sims;
    const int K = std::max(1, o.nm_starts);
    for (int k = 0; k < K; ++k) {
      const double sc = std::pow(4.0, -k);
      std::vector<std::vector<double>> sk;
      for (const auto& v : sim) {
        std::vector<double> w(v);
        for (double& e : w) e *= sc;
        sk.push_back(w);
      }
      sims.push_back(sk);
    }
    NMResult nm;
    TRY(nelder_mead_multi(c, X, n, d, m, sims, o.max_iter, o.tol_rel, o.penalty, o.speculative != 0, nm, nullptr));
    if (!(nm.f < o.penalty)) return fail(c, KDE_E_NO_FEASIBLE, "no positive-definite H found");
    for (int k = 0; k < P; ++k) r.vechH[k] = nm.x[k];
    r.objective = nm.f;
    r.iterations = nm.iterations;
    r.evaluations = nm.evals;
    r.stop_reason = nm.stop;
  } else {
    return fail(c, KDE_E_INVALID, "unknown method");
  }
  TRY(prof_collect(c));
  *out = r;
  return KDE_OK;
}

}  // extern "C"
