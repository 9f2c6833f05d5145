// kde_runtime.cpp — context, workspace, NCCL glue (loaded at run time), input staging, fixed point
// and the pair-pass driver (run_sums) of the C ABI in include/kde.h; also the context-level ABI
// calls (create/destroy, modes, profiling, tile map).  P:NNN = PAPER.md line NNN.
#include <dlfcn.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "kde_host.h"
#include "kde_tiles.cuh"

using kde::Kind;
using namespace kde::host;

// ------------------------------------------------------------------ NCCL (loaded at run time)
namespace {
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

namespace kde {
namespace host {

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

size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

size_t ws_bytes(int64_t ld, int32_t d, int32_t n_out) {
  return align256((size_t)d * ld * sizeof(float)) +
         align256((size_t)std::max(n_out, 1) * kde::kLimbs * sizeof(long long) +
                  (size_t)kde::kWorkCounters * sizeof(long long)) +
         align256((size_t)1024 * 136 * sizeof(double)) + align256(kde::kSmallDoubles * sizeof(double));
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
  base += align256(kde::kSmallDoubles * sizeof(double));
  w->limbs = (unsigned long long*)base;
  return KDE_OK;
}

kde_status check_ctx(kde_ctx* c) {
  if (!c) return KDE_E_INVALID;
  if (c->sticky != KDE_OK) return c->sticky;
  CUDA_TRY(c, cudaSetDevice(c->device));
  return KDE_OK;
}

// ------------------------------------------------------------------ fixed point
int scale_exp_for(double bound_per_term, int64_t n) {
  double pairs = (double)n * (double)(n - 1) * 0.5;
  double G = std::max(1.0, bound_per_term * std::max(pairs, 1.0));
  return 100 - (int)std::ceil(std::log2(G));
}

// Device limbs (hi, mid, unsigned lo, carry; kde_internal.h) -> the ABI's canonical 3-limb form
// value * 2^S = hi 2^80 + mid 2^40 + lo with mid, lo in [0, 2^40) (exact: |value 2^S| < 2^101).
kde_fixed limbs_to_fixed(const long long* l, int S) {
  const __int128 T = (__int128)l[0] * ((__int128)1 << 80) + (__int128)l[1] * ((__int128)1 << 40) +
                     (__int128)(unsigned long long)l[2] + (__int128)l[3] * ((__int128)1 << 64);
  const __int128 m40 = ((__int128)1 << 40) - 1;
  kde_fixed f;
  f.hi = (int64_t)(T >> 80); f.mid = (int64_t)((T >> 40) & m40); f.lo = (int64_t)(T & m40);
  f.scale_exp = S; f.pad_ = 0;
  return f;
}

double fixed_value(const kde_fixed& f) {
  __int128 T = (__int128)f.hi * ((__int128)1 << 80) + (__int128)f.mid * ((__int128)1 << 40) + (__int128)f.lo;
  return std::ldexp((double)T, -f.scale_exp);
}

// ------------------------------------------------------------------ GPU building blocks

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

kde_status gpu_sorted_rows(kde_ctx* c, const double* X, int64_t n, int d, const double** out) {
  if (c->rows_ws && X == static_cast<const double*>(c->rows_ws)) {   // already the sorted copy
    *out = X;
    return KDE_OK;
  }
  Range r("kde.sort_rows");
  const size_t tmp = kde::sort_rows_temp_bytes(n);
  const size_t xs_b = align256((size_t)n * d * sizeof(double)), keys_b = align256((size_t)n * sizeof(double)),
               idx_b = align256((size_t)2 * n * sizeof(int));
  TRY(grow(c, &c->rows_ws, &c->rows_bytes, xs_b + keys_b + idx_b + align256(tmp)));
  char* base = static_cast<char*>(c->rows_ws);
  double* xs = reinterpret_cast<double*>(base);
  CUDA_TRY(c, kde::launch_sort_rows(X, n, d, xs, reinterpret_cast<double*>(base + xs_b),
                                    reinterpret_cast<int*>(base + xs_b + keys_b), base + xs_b + keys_b + idx_b, tmp,
                                    c->stream));
  c->prof_all += 12;   // iota, CUB onesweep pairs (histogram, exclusive sum, 8 passes), gather
  *out = xs;
  return KDE_OK;
}

float lscv_skip_s(double min_abs_kappa, int64_t n) {
  const char* e = getenv("KDE_DEBUG_LSCV_NOSKIP");   // tests / diagnostics: read at every call
  if ((e && atoi(e) == 1) || !(min_abs_kappa > 0.0)) return __builtin_inff();
  const double theta = kde::skip_bounded() ? kde_lscv_skip_theta(n) : 130.0;
  const double b = theta / min_abs_kappa;
  return b < 1e30 ? (float)b : __builtin_inff();
}

// y = fp32(W (x - mean)), padded with zeros to ld, written to Y (default: the workspace's Y).
// gpu_prep_into does not clear the prep flags (several sets prepared for one launch share them).
kde_status gpu_prep_into(kde_ctx* c, const double* X, int64_t n, int d, const std::vector<double>& W,
                         const std::vector<double>& mean, int64_t ld, Ws& w, float* Y,
                         double clamp_thresh) {
  Range r("kde.prep");
  kde::PrepParams pp;                      // W and mean travel in the kernel parameters
  std::copy(W.begin(), W.begin() + (size_t)d * d, pp.W);
  std::copy(mean.begin(), mean.begin() + d, pp.mean);
  CUDA_TRY(c, kde::launch_prep_params(X, n, d, pp, Y, ld, c->stream, 0.f, w.flag(), clamp_thresh));
  c->prof_all += 1;
  return KDE_OK;
}

kde_status gpu_prep(kde_ctx* c, const double* X, int64_t n, int d, const std::vector<double>& W,
                    const std::vector<double>& mean, int64_t ld, Ws& w, double clamp_thresh) {
  CUDA_TRY(c, cudaMemsetAsync(w.flag(), 0, 2 * sizeof(unsigned long long), c->stream));
  return gpu_prep_into(c, X, n, d, W, mean, ld, w, w.Y, clamp_thresh);
}

int64_t n_tiles(int64_t n, int T) {
  int64_t nb = (n + T - 1) / T;
  return nb * (nb + 1) / 2;
}

// Local tile-index range [0, shard_count) of rank `rank` of `world` (round-robin chunks, kde_tiles.cuh);
// the kernels map a local index to its tile id with shard_tile.
void shard_range(int64_t tiles, int rank, int world, int64_t* b, int64_t* e) {
  *b = 0;
  *e = kde::shard_count(tiles, rank, world);
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

// Algorithmic pairs in a rank's tiles (local range [0, count) of shard_range): one contiguous run of
// tile ids per round-robin chunk.
double pairs_in_shard(int64_t n, int T, int64_t count, int rank, int world) {
  if (world <= 1) return pairs_in_range(n, T, 0, count);
  double s = 0.0;
  for (int64_t i = 0; i < count; i += kde::kShardChunk) {
    const int64_t t0 = kde::shard_tile(i, rank, world);
    s += pairs_in_range(n, T, t0, t0 + std::min<int64_t>(kde::kShardChunk, count - i));
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
  c->ev_excl.clear();
  c->psi_escalations = 0;
  c->psi_kappa_max = 0.0;
  c->psi_gaps.clear();
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
    if (k / 2 < c->ev_excl.size() && c->ev_excl[k / 2]) continue;
    float x = 0.f;
    CUDA_TRY(c, cudaEventElapsedTime(&x, c->ev_pool[k], c->ev_pool[k + 1]));
    ms += x;
  }
  c->prof_ms = ms;
  return KDE_OK;
}


// Sum `count` int64 limbs in device memory across the ranks: NCCL on the context stream, or (test
// transport, no NCCL) staged through pinned host memory and the caller's all-reduce callback.
kde_status allreduce_limbs(kde_ctx* c, unsigned long long* limbs, size_t count) {
  if (c->world > 1 || c->comm)   // canonical per-rank limbs: the int64 sum over ranks cannot wrap
    CUDA_TRY(c, kde::launch_normalize_limbs(limbs, (int)(count / kde::kLimbs), c->stream));
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
                    int shard_world, bool allreduce, std::vector<kde_fixed>& out, bool limbs_zeroed) {
  Range rr("kde.pair_pass");
  // dynamic-scheduling counters (one per launch) follow this run's limbs; zeroed with them
  unsigned long long* work = w.limbs + (size_t)n_out * kde::kLimbs;
  if (!limbs_zeroed)
    CUDA_TRY(c, cudaMemsetAsync(w.limbs, 0, ((size_t)n_out * kde::kLimbs + launches.size()) * sizeof(long long),
                                c->stream));
  // LSCV exact-zero tile skip (profiling): pairs of skipped tiles, in the small block's skipped slot (zeroed
  // here, read back with the limbs below) and left out of the evaluated pairs
  unsigned long long* lscv_skipped = reinterpret_cast<unsigned long long*>(w.small + kde::kSkippedSlot);
  bool any_skip = false;
  for (const SumLaunch& L : launches) any_skip |= L.skip_s < __builtin_inff();
  if (c->profiling && any_skip) CUDA_TRY(c, cudaMemsetAsync(lscv_skipped, 0, sizeof(unsigned long long), c->stream));
  int64_t tiles = n_tiles(n, T), tb, te;
  shard_range(tiles, shard_rank, shard_world, &tb, &te);
  const double pairs = c->profiling ? pairs_in_shard(n, T, te, shard_rank, shard_world) : 0.0;
  // Several launches (LSCV_h candidate batches): alternate two streams, so that launch k+1's CTAs take the
  // SM slots launch k's CTAs free during its tail (its last units; the outputs and the scheduling
  // counters of the launches are disjoint).  Profiling then times the whole span as one window.
  const char* one_env = getenv("KDE_DEBUG_ONE_STREAM");   // A/B and tests: read at every call
  const bool one_stream = one_env && atoi(one_env) == 1;
  const bool two = launches.size() >= 2 && !one_stream && !(c->cap_stream && c->stream == c->cap_stream);
  cudaEvent_t span0 = nullptr, span1 = nullptr;
  if (two) {
    if (!c->side_stream) CUDA_TRY(c, cudaStreamCreateWithFlags(&c->side_stream, cudaStreamNonBlocking));
    if (!c->ev_fork) CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
    if (!c->ev_join) CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
    if (c->profiling) { span0 = next_event(c); span1 = next_event(c); CUDA_TRY(c, cudaEventRecord(span0, c->stream)); }
    CUDA_TRY(c, cudaEventRecord(c->ev_fork, c->stream));
    CUDA_TRY(c, cudaStreamWaitEvent(c->side_stream, c->ev_fork, 0));
  }
  for (const SumLaunch& L : launches) {
    kde::LaunchCfg cfg;
    cfg.X = w.Y; cfg.n = n; cfg.ld = ld; cfg.tile_begin = tb; cfg.tile_end = te; cfg.tile = T;
    cfg.part_rank = shard_rank; cfg.part_world = shard_world;
    cfg.scale_exp = scale; cfg.limbs = w.limbs + (size_t)L.out_offset * kde::kLimbs;
    cfg.n_out = L.n_out; cfg.stream = c->stream; cfg.sm_count = c->sm_count;
    cfg.clamp = w.flag() + 1;
    if (L.X) cfg.X = L.X;
    cfg.n_sets = L.n_sets;
    cfg.set_stride = L.set_stride;
    cfg.Y64 = L.Y64;
    cfg.centres = L.centres;
    cfg.skipped = L.skipped;
    cfg.skip_gap = L.skip_gap;
    cfg.skip_gap_dev = L.skip_gap_dev;
    cfg.skip_s = L.skip_s;
    cfg.skip_s_sets = L.skip_s_sets;
    cfg.skip_c_dev = L.skip_c_dev;
    if (c->profiling && L.skip_s < __builtin_inff()) cfg.skipped = lscv_skipped;
    cfg.work = work + (&L - launches.data());
    if (two && ((&L - launches.data()) & 1)) cfg.stream = c->side_stream;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (c->profiling && !two) { e0 = next_event(c); e1 = next_event(c); cudaEventRecord(e0, c->stream); }
    cudaError_t err = cudaSuccess;
    switch (L.kind) {
      case Kind::Psi4: case Kind::Psi6: case Kind::Psi8: err = kde::launch_psi(L.r, cfg, L.psi); break;
      case Kind::LscvScalar: err = kde::launch_lscv_scalar(d, L.nb, cfg, L.ls); break;
      case Kind::LscvMatrix: err = kde::launch_lscv_white(d, cfg); break;
    }
    if (err != cudaSuccess) return fail(c, KDE_E_CUDA, "pair kernel launch: %s", cudaGetErrorString(err));
    if (tb < te) c->prof_all += 1;
    if (c->profiling) {
      if (!two) cudaEventRecord(e1, c->stream);
      c->prof_launches++;
      c->prof_evals += pairs * (double)L.nb * (double)L.n_sets;
    }
  }
  if (two) {
    CUDA_TRY(c, cudaEventRecord(c->ev_join, c->side_stream));
    CUDA_TRY(c, cudaStreamWaitEvent(c->stream, c->ev_join, 0));
    if (c->profiling) CUDA_TRY(c, cudaEventRecord(span1, c->stream));
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
  if (c->profiling && any_skip) {   // skipped pairs x candidates per pair (the same for every launch here)
    unsigned long long sk = 0;
    std::memcpy(&sk, c->h_limbs + (kde::kSkippedSlot - 408), sizeof(sk));
    c->prof_evals -= (double)sk * (double)launches.front().nb;
  }
  out.resize(n_out);
  for (int k = 0; k < n_out; ++k) out[k] = limbs_to_fixed(c->h_limbs + gap + (size_t)k * kde::kLimbs, scale);
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

}  // namespace host
}  // namespace kde

// ================================================================== C ABI (context level)
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
  o->nm_loop = 0;           // device-resident Nelder-Mead where it applies
  o->nm_param = 0;          // search over vech(H) (the paper's reading); 1 = over the Cholesky factor
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
  if (c->nm_exec) cudaGraphExecDestroy(c->nm_exec);
  if (c->nm_ws) cudaFree(c->nm_ws);
  if (c->nm_host) cudaFreeHost(c->nm_host);
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  if (c->side_stream) cudaStreamDestroy(c->side_stream);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->comm) nccl().CommDestroy(c->comm);
  if (c->own_ws) cudaFree(c->own_ws);
  if (c->sort_ws) cudaFree(c->sort_ws);
  if (c->rows_ws) cudaFree(c->rows_ws);
  if (c->f64_ws) cudaFree(c->f64_ws);
  if (c->white_ws) cudaFree(c->white_ws);
  if (c->ev_ws) cudaFree(c->ev_ws);
  if (c->mat_ws) cudaFree(c->mat_ws);
  if (c->skip_ws) cudaFree(c->skip_ws);
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
  c->psi_mode = fp64_terms > 0 ? 1 : (fp64_terms < 0 ? -1 : 0);
  return KDE_OK;
}

kde_status kde_set_host_allreduce(kde_ctx* c, kde_host_allreduce_fn fn, void* user) {
  if (!c) return KDE_E_INVALID;
  if (c->comm) return fail(c, KDE_E_INVALID, "context already has an NCCL communicator");
  c->har_fn = fn;
  c->har_user = user;
  return KDE_OK;
}

int32_t kde_last_fp64_passes(const kde_ctx* c) { return c ? c->psi_escalations : 0; }

double kde_last_psi_kappa(const kde_ctx* c) { return c ? c->psi_kappa_max : 0.0; }

int32_t kde_last_psi_gaps(const kde_ctx* c, double* out, int32_t max) {
  if (!c) return 0;
  const int32_t cnt = (int32_t)c->psi_gaps.size();
  for (int32_t k = 0; k < cnt && k < max && out; ++k) out[k] = c->psi_gaps[k];
  return cnt;
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
                           int32_t* tile_edge, int64_t* tiles_total, int64_t* rank_tiles, int32_t* chunk) {
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
  if (tile_edge) *tile_edge = T;
  if (tiles_total) *tiles_total = tiles;
  if (rank_tiles) *rank_tiles = kde::shard_count(tiles, rank, world);
  if (chunk) *chunk = world > 1 ? kde::kShardChunk : (int32_t)std::min<int64_t>(tiles, INT32_MAX);
  return KDE_OK;
}

double kde_psi_skip_gap(int32_t r, double g, double var) {
  return (r == 4 || r == 6 || r == 8) ? kde::psi_bounded_gap(r, g, var) : kde::kPsiSkipGap32;
}

double kde_lscv_skip_theta(int64_t n) { return std::min(130.0, std::log2((double)std::max<int64_t>(n, 2)) + 30.0); }

int64_t kde_shard_tile(int64_t i, int32_t rank, int32_t world) {
  return (world < 1 || rank < 0 || rank >= world || i < 0) ? -1 : kde::shard_tile(i, rank, world);
}

double kde_fixed_value(const kde_fixed* v) { return v ? fixed_value(*v) : NAN; }

kde_fixed kde_fixed_add(kde_fixed a, kde_fixed b) {
  kde_fixed r = a;
  r.hi = (int64_t)((uint64_t)a.hi + (uint64_t)b.hi);
  r.mid = (int64_t)((uint64_t)a.mid + (uint64_t)b.mid);
  r.lo = (int64_t)((uint64_t)a.lo + (uint64_t)b.lo);
  return r;
}

double kde_last_aux_ms(const kde_ctx* c) { return c ? c->prof_aux_ms : 0.0; }

}  // extern "C"
