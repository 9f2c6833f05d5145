// kde_psi.cu — Psi_r pair-kernel instantiations, tile/batch policy, O(n) kernels (see kde_pair.cuh).
#include <cub/device/device_radix_sort.cuh>
#include <algorithm>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "kde_pair.cuh"

namespace kde {

void tile_coords_host(int64_t bx, int64_t* l, int64_t* q) { tile_coords(bx, *l, *q); }

double psi_skip_gap(bool fp64) {
  const char* e = getenv("KDE_DEBUG_PSI_NOSKIP");   // tests / diagnostics: read at every call
  if (e && atoi(e) == 1) return INFINITY;
  return fp64 ? kPsiSkipGap64 : kPsiSkipGap32;
}

bool skip_bounded() {
  const char* e = getenv("KDE_DEBUG_SKIP_EXACT");   // tests / diagnostics: read at every call
  return !(e && atoi(e) == 1);
}

double psi_skip_gap_for(int r, double g, double var) {
  const double exact = psi_skip_gap(false);
  if (!(exact < INFINITY) || !skip_bounded()) return exact;
  return psi_bounded_gap(r, g, var);
}

// ------------------------------------------------------------------ dispatch

int tile_for(Kind k, int d, int64_t n) {
  switch (k) {
    case Kind::Psi4: case Kind::Psi6: case Kind::Psi8: {
      static const char* dbg = getenv("KDE_DEBUG_PSI_TILE");   // tests / diagnostics only
      if (dbg && (atoi(dbg) == 512 || atoi(dbg) == 2048)) return atoi(dbg);
      return n >= (int64_t)128 * 2048 ? 2048 : 512;
    }
    case Kind::LscvScalar: return 512;
    case Kind::LscvMatrix: {
      // the largest of 1024 (d <= 4: 512 threads, 2 CTAs/SM), 512 and 256-row tiles that leaves
      // ~20 tiles per resident CTA (wave tail).  1024 halves the per-unit barrier/epilogue share
      // at the same 32 resident warps: C5 2.81 -> 2.71 s.
      static const char* dbg = getenv("KDE_DEBUG_LSCVH_TILE");   // tests / diagnostics only
      const int force = dbg ? atoi(dbg) : 0;
      if (force == 1024 && d <= 4) return 1024;
      if (force == 256 || force == 512) return force;
      const int64_t nb2 = (n + 1023) / 1024, nb = (n + 511) / 512;
      if (d <= 4 && nb2 * (nb2 + 1) / 2 >= 6000) return 1024;
      return nb * (nb + 1) / 2 >= 6000 ? 512 : 256;
    }
  }
  return 512;
}

int cand_per_launch(Kind k, int d) {
  switch (k) {
    case Kind::Psi4: case Kind::Psi6: case Kind::Psi8: return 1;
    case Kind::LscvScalar: return nb_scalar(d);
    case Kind::LscvMatrix: return 1;   // one candidate per whitened data set
  }
  return 1;
}

// Small n (fewer tiles of 512 than ~2 waves of 64-thread CTAs, 16 per SM): split each tile's
// columns into 8 work units of 64, so the launch fills the GPU.
static bool psi_split(const LaunchCfg& c) {
  static const char* dbg = getenv("KDE_DEBUG_PSI_SPLIT");   // diagnostics only
  if (dbg) return c.tile == 512 && atoi(dbg) == 1;
  const int64_t nb = (c.n + c.tile - 1) / c.tile;
  return c.tile == 512 && nb * (nb + 1) / 2 < 2 * 16 * (int64_t)c.sm_count;
}

template <int R>
static cudaError_t launch_psi_r(const LaunchCfg& c, const PsiParams& p) {
  if (c.tile == 2048) return launch_pair<FPsi<R, 256>>(c, p);
  return psi_split(c) ? launch_pair<FPsi<R, 64, 8>>(c, p) : launch_pair<FPsi<R, 64>>(c, p);
}

template <int R>
static cudaError_t prepare_psi_r(const LaunchCfg& c) {
  int occ;
  if (c.tile == 2048) return pair_occupancy<FPsi<R, 256>>(&occ);
  return psi_split(c) ? pair_occupancy<FPsi<R, 64, 8>>(&occ) : pair_occupancy<FPsi<R, 64>>(&occ);
}

cudaError_t prepare_psi(int r, const LaunchCfg& c) {
  switch (r) {
    case 4: return prepare_psi_r<4>(c);
    case 6: return prepare_psi_r<6>(c);
    case 8: return prepare_psi_r<8>(c);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_psi(int r, const LaunchCfg& c, const PsiParams& p) {
  switch (r) {
    case 4: return launch_psi_r<4>(c, p);
    case 6: return launch_psi_r<6>(c, p);
    case 8: return launch_psi_r<8>(c, p);
  }
  return cudaErrorInvalidValue;
}

// Candidates per launch: chosen so that no instantiation spills at 128 registers (2 CTAs/SM).
// ------------------------------------------------------------------ O(n) kernels (fp64)
// Deterministic moments (R_fun): fixed block count for a given n, fixed per-thread
// order, warp butterfly, fixed cross-warp order, then one block adds the partials in order.

constexpr int kMomThreads = 256;

int moments_blocks(int64_t n) {
  int64_t b = (n + 4 * kMomThreads - 1) / (4 * kMomThreads);
  if (b > 1024) b = 1024;
  if (b < 1) b = 1;
  return (int)b;
}

template <int MODE>   // 1: sum x_a; 2: sum (x_a - m_a)(x_b - m_b), a <= b
__global__ void __launch_bounds__(kMomThreads) moments_kernel(const double* __restrict__ X, int64_t n,
                                                               int d, const double* __restrict__ mean,
                                                               double* __restrict__ part) {
  __shared__ double red[kMomThreads / 32][kMaxDim * (kMaxDim + 1) / 2];
  const int width = MODE == 1 ? d : d * (d + 1) / 2;
  double acc[kMaxDim * (kMaxDim + 1) / 2];
  for (int k = 0; k < width; ++k) acc[k] = 0.0;
  const int64_t stride = (int64_t)gridDim.x * kMomThreads;
  for (int64_t i = (int64_t)blockIdx.x * kMomThreads + threadIdx.x; i < n; i += stride) {
    if (MODE == 1) {
      for (int a = 0; a < d; ++a) acc[a] += X[a * n + i];
    } else {
      double v[kMaxDim];
      for (int a = 0; a < d; ++a) v[a] = X[a * n + i] - mean[a];
      int t = 0;
      for (int a = 0; a < d; ++a)
        for (int b = a; b < d; ++b) acc[t++] += v[a] * v[b];
    }
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int k = 0; k < width; ++k) {
    double s = warp_sum(acc[k]);
    if (lane == 0) red[w][k] = s;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < width; k += kMomThreads) {
    double s = red[0][k];
    for (int ww = 1; ww < kMomThreads / 32; ++ww) s += red[ww][k];
    part[(size_t)blockIdx.x * width + k] = s;
  }
}

// One block per output k; thread t adds partials t, t+256, ... in order, then the fixed warp
// butterfly and fixed cross-warp order: deterministic for a given block count.
__global__ void __launch_bounds__(kMomThreads) reduce_parts_kernel(const double* __restrict__ part,
                                                                   int nblk, int width,
                                                                   double* __restrict__ out) {
  __shared__ double red[kMomThreads / 32];
  const int k = blockIdx.x;
  double s = 0.0;
  for (int b = threadIdx.x; b < nblk; b += kMomThreads) s += part[(size_t)b * width + k];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = red[0];
    for (int w = 1; w < kMomThreads / 32; ++w) t += red[w];
    out[k] = t;
  }
}

cudaError_t launch_moments1(const double* X, int64_t n, int d, double* part, int nblk,
                            cudaStream_t s) {
  moments_kernel<1><<<nblk, kMomThreads, 0, s>>>(X, n, d, nullptr, part);
  return cudaGetLastError();
}

cudaError_t launch_moments2(const double* X, int64_t n, int d, const double* mean_dev,
                            double* part, int nblk, cudaStream_t s) {
  moments_kernel<2><<<nblk, kMomThreads, 0, s>>>(X, n, d, mean_dev, part);
  return cudaGetLastError();
}

cudaError_t launch_reduce_parts(const double* part, int nblk, int width, double* out,
                                cudaStream_t s) {
  reduce_parts_kernel<<<width, kMomThreads, 0, s>>>(part, nblk, width, out);
  return cudaGetLastError();
}

// Data prep (row a1 of SURVEY §8(a)): y_a = fp32( sum_b W_ab (x_b - mean_b) ), padding `pad`.
// flag[0]: some scaled value beyond 1e18 (error); flag[1]: some beyond clamp_thresh (> 0).
__device__ __forceinline__ void prep_body(const double* __restrict__ X, int64_t n, int d,
                                          const double* W, const double* mean,
                                          float* __restrict__ Y, int64_t ld, float pad,
                                          unsigned long long* __restrict__ flag, double clamp_thresh) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  bool bad = false, big = false;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ld; i += stride) {
    if (i < n) {
      double v[kMaxDim];
      for (int b = 0; b < d; ++b) v[b] = X[b * n + i] - mean[b];
      for (int a = 0; a < d; ++a) {
        double s = 0.0;
        for (int b = 0; b < d; ++b) s = fma(W[a * d + b], v[b], s);
        bad |= !(fabs(s) <= 1.0e18);   // squares of differences must stay finite in fp32
        big |= clamp_thresh > 0.0 && fabs(s) > clamp_thresh;
        Y[a * ld + i] = (float)s;
      }
    } else {
      for (int a = 0; a < d; ++a) Y[a * ld + i] = pad;
    }
  }
  if (bad && flag) atomicOr(flag, 1ull);
  if (big && flag) atomicOr(flag + 1, 1ull);
}

// W and mean in device memory (the device-resident PLUGIN chain writes them).
__global__ void prep_kernel(const double* __restrict__ X, int64_t n, int d, const double* __restrict__ W,
                            const double* __restrict__ mean, float* __restrict__ Y, int64_t ld, float pad,
                            unsigned long long* __restrict__ flag, double clamp_thresh) {
  prep_body(X, n, d, W, mean, Y, ld, pad, flag, clamp_thresh);
}

// W and mean passed by value in the kernel parameters (no host-to-device copy per prep).
__global__ void prep_kernel_p(const double* __restrict__ X, int64_t n, int d, const __grid_constant__ PrepParams pp,
                              float* __restrict__ Y, int64_t ld, float pad, unsigned long long* __restrict__ flag,
                              double clamp_thresh) {
  prep_body(X, n, d, pp.W, pp.mean, Y, ld, pad, flag, clamp_thresh);
}

// Several sets, parameters in device memory, the set count decided on the device (blockIdx.y = set).
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// trace (diagnostics, KDE_DEBUG_NM_TRACE): slot 4 (*calls - 1) + 2 = start of block (0, 0), + 3 = the
// latest block end (globaltimer ns).
__global__ void prep_sets_kernel(const double* __restrict__ X, int64_t n, int d, const PrepParams* __restrict__ pp,
                                 const int* __restrict__ n_sets, float* __restrict__ Y, int64_t set_stride,
                                 int64_t ld, unsigned long long* __restrict__ flag, unsigned long long* trace,
                                 const int* calls) {
  pdl_wait();   // programmatic launch after the Nelder–Mead decision: its outputs are visible past here
  pdl_trigger();   // the pair kernel may start launching (it waits for this grid's completion)
  const int set = blockIdx.y;
  if (set >= *n_sets) return;
  if (trace && threadIdx.x == 0 && blockIdx.x == 0 && set == 0) trace[16 * (*calls - 1) + 2] = global_ns();
  prep_body(X, n, d, pp[set].W, pp[set].mean, Y + (int64_t)set * set_stride, ld, 0.f, flag, 0.0);
  if (trace) {
    __syncthreads();
    if (threadIdx.x == 0) atomicMax(trace + 16 * (*calls - 1) + 3, global_ns());
  }
}

static unsigned prep_blocks(int64_t ld) {
  int64_t blocks = (ld + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  return (unsigned)blocks;
}

cudaError_t launch_prep(const double* X, int64_t n, int d, const double* W_dev,
                        const double* mean_dev, float* Y, int64_t ld, cudaStream_t s, float pad,
                        unsigned long long* flag, double clamp_thresh) {
  prep_kernel<<<prep_blocks(ld), 256, 0, s>>>(X, n, d, W_dev, mean_dev, Y, ld, pad, flag, clamp_thresh);
  return cudaGetLastError();
}

cudaError_t launch_prep_sets(const double* X, int64_t n, int d, const PrepParams* pp_dev, const int* n_sets_dev,
                             int max_sets, float* Y, int64_t set_stride, int64_t ld, cudaStream_t s,
                             unsigned long long* flag, unsigned long long* trace, const int* calls, bool pdl) {
  unsigned bx = prep_blocks(ld);
  const unsigned per = (148u * 16u + (unsigned)max_sets - 1) / (unsigned)max_sets;   // ~16 blocks/SM overall
  if (bx > per) bx = per > 0 ? per : 1;
  if (pdl) {
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(bx, (unsigned)max_sets);
    lc.blockDim = dim3(256);
    lc.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    return cudaLaunchKernelEx(&lc, prep_sets_kernel, X, n, d, pp_dev, n_sets_dev, Y, set_stride, ld, flag, trace, calls);
  }
  prep_sets_kernel<<<dim3(bx, (unsigned)max_sets), 256, 0, s>>>(X, n, d, pp_dev, n_sets_dev, Y, set_stride, ld, flag, trace,
                                                                  calls);
  return cudaGetLastError();
}

cudaError_t launch_prep_params(const double* X, int64_t n, int d, const PrepParams& pp, float* Y, int64_t ld,
                               cudaStream_t s, float pad, unsigned long long* flag, double clamp_thresh) {
  prep_kernel_p<<<prep_blocks(ld), 256, 0, s>>>(X, n, d, pp, Y, ld, pad, flag, clamp_thresh);
  return cudaGetLastError();
}

// Psi data prep (rows a1 of SURVEY §8(a) + tile-local centring): sorted x ->
// y = (x - mean) * w in fp64 (Y64, zero padded to ld), per column tile l the centre
// c_l = fp32(y[min(l T + T/2, n - 1)]) and Yc = fp32(y - c_l) (padding 0).  Flags as prep_body:
// flag[0] some |y| > 1e18 (error), flag[1] some |y| > clamp_thresh.
__global__ void psi_prep_kernel(const double* __restrict__ x, int64_t n, const double* __restrict__ mean,
                                const double* __restrict__ w, int T, double* __restrict__ Y64,
                                float* __restrict__ Yc, float* __restrict__ centres, int64_t ld,
                                unsigned long long* __restrict__ flag, double clamp_thresh) {
  const double m = mean[0], s = w[0];
  bool bad = false, big = false;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ld; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = i / T;
    int64_t mid = l * T + T / 2;
    if (mid > n - 1) mid = n - 1;
    const float c = __double2float_rn((x[mid] - m) * s);   // the same expression as y[mid]
    if (i == l * T) centres[l] = c;
    if (i < n) {
      const double y = (x[i] - m) * s;
      bad |= !(fabs(y) <= 1.0e18);
      big |= fabs(y) > clamp_thresh;
      Y64[i] = y;
      Yc[i] = __double2float_rn(y - (double)c);
    } else {
      Y64[i] = 0.0;
      Yc[i] = 0.f;
    }
  }
  if (bad && flag) atomicOr(flag, 1ull);
  if (big && flag) atomicOr(flag + 1, 1ull);
}

cudaError_t launch_psi_prep(const double* x, int64_t n, const double* mean_dev, const double* w_dev, int T,
                            double* Y64, float* Yc, float* centres, int64_t ld, cudaStream_t s,
                            unsigned long long* flag, double clamp_thresh) {
  psi_prep_kernel<<<prep_blocks(ld), 256, 0, s>>>(x, n, mean_dev, w_dev, T, Y64, Yc, centres, ld, flag, clamp_thresh);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ fp64-term Psi mode
// Every term in fp64 (libdevice exp, Horner in s with the integer coefficients of He_r, fp64 tile
// sums) on the fp64 scaled samples of psi_prep_kernel: kde_set_precision(ctx, 1), or the automatic
// re-run of a pass whose cancellation estimate exceeds what fp32 terms carry.
// Same tile map (256-tiles), fixed-point limbs and multi-GPU partition as the fp32 path; sorted
// data: tiles whose smallest pair distance exceeds kPsiSkipGap64 add exactly 0 and are skipped.
template <int R>
__device__ __forceinline__ double he64(double s) {   // He_r(u) in s = u^2
  if (R == 4) return (s - 6.0) * s + 3.0;
  if (R == 6) return ((s - 15.0) * s + 45.0) * s - 15.0;
  return (((s - 28.0) * s + 210.0) * s - 420.0) * s + 105.0;
}

template <int R>
__global__ void __launch_bounds__(kPsi64Tile) psi64_kernel(const double* __restrict__ y, int64_t n, int64_t tb,
                                                           int64_t te, int S, unsigned long long* __restrict__ limbs,
                                                           const unsigned long long* __restrict__ gate,
                                                           double skip_gap, int part_rank, int part_world) {
  __shared__ double cs[kPsi64Tile];
  __shared__ double red[kPsi64Tile / 32];
  const int tid = threadIdx.x;
  if (gate != nullptr && *gate == 0) return;   // device-side decision: the fp32 pass sufficed
  for (int64_t u = tb + blockIdx.x; u < te; u += gridDim.x) {   // this rank's local tile indices
    int64_t l, q;
    tile_coords(shard_tile(u, part_rank, part_world), l, q);
    if (q < l && y[l * kPsi64Tile] - y[q * kPsi64Tile + kPsi64Tile - 1] > skip_gap) continue;   // exact 0
    const int64_t jc = l * kPsi64Tile + tid, i = q * kPsi64Tile + tid;
    __syncthreads();
    cs[tid] = jc < n ? y[jc] : 0.0;
    __syncthreads();
    const int jlim = (int)(n - l * kPsi64Tile < kPsi64Tile ? n - l * kPsi64Tile : kPsi64Tile);
    double acc = 0.0;
    if (i < n) {
      const double xi = y[i];
      for (int j = (q == l ? tid + 1 : 0); j < jlim; ++j) {
        const double u = xi - cs[j];
        const double s = u * u;
        acc += he64<R>(s) * exp(-0.5 * s);
      }
    }
    double v[1] = {acc};
    commit_tile<1, kPsi64Tile>(v, red, limbs, S);
  }
}

cudaError_t launch_psi64(int r, const double* y, int64_t n, int64_t tb, int64_t te, int S,
                         unsigned long long* limbs, int sm_count, cudaStream_t s, const unsigned long long* gate,
                         double skip_gap, int part_rank, int part_world) {
  if (te <= tb) return cudaSuccess;
  int64_t grid = te - tb;
  if (grid > (int64_t)sm_count * 8) grid = (int64_t)sm_count * 8;
  switch (r) {
    case 4: psi64_kernel<4><<<(unsigned)grid, kPsi64Tile, 0, s>>>(y, n, tb, te, S, limbs, gate, skip_gap, part_rank, part_world); break;
    case 6: psi64_kernel<6><<<(unsigned)grid, kPsi64Tile, 0, s>>>(y, n, tb, te, S, limbs, gate, skip_gap, part_rank, part_world); break;
    case 8: psi64_kernel<8><<<(unsigned)grid, kPsi64Tile, 0, s>>>(y, n, tb, te, S, limbs, gate, skip_gap, part_rank, part_world); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------------ device-resident PLUGIN chain
// The scalar steps of Sec. 4.4.1 (Eq. 11-18) run in single-thread kernels between the
// O(n) and O(n^2) kernels, so kde_plugin_h enqueues the whole chain without a host round trip
// (one synchronisation at the end).  State in the workspace's `small` block (PluginDev layout).
__device__ __forceinline__ double limbs_value_dev(const unsigned long long* l, int S) {
  return ldexp((double)limbs_total(l), -S);
}

__device__ __forceinline__ void set_status(double* st, int code) {
  if (st[0] == 0.0) st[0] = (double)code;   // first failure wins
}

// Data-aware bounded-skip threshold (kde_internal.h launch_psi_gap_select).
constexpr int kGapCands = 28;     // tau_c = 6 + c/4 < 13
constexpr int kGapMaxCtas = 296;  // partial sums of at most this many CTAs (scratch: kGapMaxCtas x kGapCands)
static int gap_ctas(int64_t tiles) {
  const int64_t g = (tiles + 1023) / 1024;
  return (int)(g < 1 ? 1 : (g > kGapMaxCtas ? kGapMaxCtas : g));
}

// Stage 1: CTA b bounds the skippable mass of its contiguous share of tile ids for every candidate tau
// (fixed per-thread order and warp/CTA reduction order) and writes kGapCands partials.
__global__ void __launch_bounds__(256) psi_gap_partial_kernel(int r, const double* __restrict__ y, int64_t n, int T,
                                                              double* __restrict__ part) {
  __shared__ double red[8][kGapCands];
  double acc[kGapCands];
#pragma unroll
  for (int c = 0; c < kGapCands; ++c) acc[c] = 0.0;
  const int64_t nt = (n + T - 1) / T, tiles = nt * (nt + 1) / 2;
  const int64_t chunk = (tiles + gridDim.x - 1) / gridDim.x;
  const int64_t b0 = (int64_t)blockIdx.x * chunk, b1 = b0 + chunk < tiles ? b0 + chunk : tiles;
  for (int64_t id = b0 + threadIdx.x; id < b1; id += blockDim.x) {
    int64_t l, q;
    tile_coords(id, l, q);
    if (q >= l) continue;
    const double gap = y[l * T] - y[q * T + T - 1];   // the Psi kernel's skip test (pair_unit)
    if (!(gap > 6.0)) continue;
    const int64_t cols = n - l * T < T ? n - l * T : T;
    const double b = 2.0 * (double)T * (double)cols * exp((double)r * log(gap) - 0.5 * gap * gap);
#pragma unroll
    for (int c = 0; c < kGapCands; ++c)
      if (gap > 6.0 + 0.25 * c) acc[c] += b;
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int c = 0; c < kGapCands; ++c) {
    double v = acc[c];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[wid][c] = v;
  }
  __syncthreads();
  if (threadIdx.x < kGapCands) {
    double v = 0.0;
    for (int w = 0; w < 8; ++w) v += red[w][threadIdx.x];
    part[(int64_t)blockIdx.x * kGapCands + threadIdx.x] = v;
  }
}

// Stage 2 (one warp): the CTAs' partials in CTA order, then the smallest admissible tau (acc is
// non-increasing in c), never above the closed form.
__global__ void psi_gap_finalize_kernel(int r, int64_t n, int nparts, const double* __restrict__ part,
                                        const double* g_dev, double g_val, const double* var_dev, double var_val,
                                        double* out) {
  __shared__ int ok[kGapCands];
  const double g = g_dev != nullptr ? *g_dev : g_val, var = var_dev != nullptr ? *var_dev : var_val;
  if (threadIdx.x < kGapCands) {
    double v = 0.0;
    for (int b = 0; b < nparts; ++b) v += part[(int64_t)b * kGapCands + threadIdx.x];
    const double lim = (double)n * (double)n * exp(psi_skip_log_target(r, g, var));
    ok[threadIdx.x] = psi_skip_args_ok(g, var) && v * (1.0 + 1e-9) <= lim;
  }
  __syncwarp();
  if (threadIdx.x == 0) {
    double tau = psi_bounded_gap(r, g, var);
    for (int c = 0; c < kGapCands; ++c)
      if (ok[c]) {
        tau = fmin(tau, 6.0 + 0.25 * c);
        break;
      }
    *out = tau;
  }
}

cudaError_t launch_psi_gap_select(int r, const double* y, int64_t n, int T, const double* g_dev, double g_val,
                                  const double* var_dev, double var_val, double* out, double* scratch,
                                  cudaStream_t s) {
  const int64_t nt = (n + T - 1) / T;
  const int G = gap_ctas(nt * (nt + 1) / 2);
  psi_gap_partial_kernel<<<G, 256, 0, s>>>(r, y, n, T, scratch);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  psi_gap_finalize_kernel<<<1, 32, 0, s>>>(r, n, G, scratch, g_dev, g_val, var_dev, var_val, out);
  return cudaGetLastError();
}

// stage 0: mean = sum / n.  stage 1: V-hat, sigma-hat, Psi8^NS, g1 (steps 1-4), W = 1/g1.
// stage 4 (5): after the fp32-term Psi6 (Psi4) pass, decide whether it is re-run with fp64 terms
// (gate): psi_mode 1 always, 0 when kappa = 2A / |2S + n He_r(0)| > kPsiKappaMax, -1 never.
// stage 2: Psi6-hat(g1) (step 5) from the fp64 or fp32 sum, g2 (step 6), W = 1/g2.
// stage 3: Psi4-hat(g2) (step 7), h (step 8).  `limbs` = the chain's kPluginOuts outputs.
__global__ void plugin_chain_kernel(int stage, int64_t n, double* small, const unsigned long long* limbs,
                                    int S, int psi_mode) {
  PluginDev dv(small);
  const double nn = (double)n, pi = 3.14159265358979323846, s2p = sqrt(2.0 * pi);
  double* t = dv.trace;   // V_hat, sigma_hat, psi8_ns, g1, psi6, g2, psi4, h
  if (stage == 0) {
    const double sum = dv.sums[0];
    if (!isfinite(sum)) set_status(dv.status, 1);                          // KDE_E_INVALID
    dv.mean[0] = sum / nn;
  } else if (stage == 1) {
    const double V = dv.sums[0] / (nn - 1.0);
    if (!isfinite(V)) set_status(dv.status, 1);
    t[0] = V;                                                              // Eq. 11
    if (!(V > 0.0)) set_status(dv.status, 4);                              // KDE_E_DEGENERATE
    t[1] = sqrt(V);                                                        // Eq. 12
    t[2] = 105.0 / (32.0 * sqrt(pi) * pow(t[1], 9.0));                     // Eq. 13
    const double K6_0 = -15.0 / s2p;
    t[3] = pow(-2.0 * K6_0 / (t[2] * nn), 1.0 / 9.0);                      // Eq. 14
    dv.W[0] = 1.0 / t[3];
    small[kGapSlot] = psi_bounded_gap(6, t[3], V);   // closed-form skip bound (§3.11; refined by the selection)
  } else if (stage == 4 || stage == 5) {
    const int k = stage - 4;                                               // 0: Psi6, 1: Psi4
    const unsigned long long* L = limbs + (size_t)(2 * k) * kLimbs;
    const double Sr = limbs_value_dev(L, S), A = limbs_value_dev(L + kLimbs, S);
    const double kappa = 2.0 * A / fabs(2.0 * Sr + nn * (k == 0 ? -15.0 : 3.0));
    dv.gate[k] = psi_mode > 0 || (psi_mode == 0 && !(kappa <= kPsiKappaMax)) ? 1ull : 0ull;
    small[421 + k] = kappa;                                                // reported (kde_last_psi_kappa)
  } else if (stage == 2) {
    const double Sr = limbs_value_dev(limbs + (size_t)(dv.gate[0] ? 4 : 0) * kLimbs, S);
    t[4] = (2.0 * Sr / s2p + nn * -15.0 / s2p) / (nn * nn * pow(t[3], 7.0));   // Eq. 15, reading Z1
    if (!(t[4] < 0.0)) set_status(dv.status, 8);                           // KDE_E_NUMERIC
    const double K4_0 = 3.0 / s2p;
    t[5] = pow(-2.0 * K4_0 / (t[4] * nn), 1.0 / 7.0);                      // Eq. 16
    dv.W[0] = 1.0 / t[5];
    small[kGapSlot + 1] = psi_bounded_gap(4, t[5], t[0]);
  } else {
    const double Sr = limbs_value_dev(limbs + (size_t)(dv.gate[1] ? 5 : 2) * kLimbs, S);
    t[6] = (2.0 * Sr / s2p + nn * 3.0 / s2p) / (nn * nn * pow(t[5], 5.0));     // Eq. 17
    if (!(t[6] > 0.0)) set_status(dv.status, 8);
    const double RK = 1.0 / (2.0 * sqrt(pi));
    t[7] = pow(RK / (t[6] * nn), 0.2);                                     // Eq. 18
  }
}

cudaError_t launch_plugin_chain(int stage, int64_t n, double* small, const unsigned long long* limbs, int S,
                                cudaStream_t s, int psi_mode) {
  plugin_chain_kernel<<<1, 1, 0, s>>>(stage, n, small, limbs, S, psi_mode);
  return cudaGetLastError();
}

// Canonical limbs before a cross-rank int64 sum (kde_internal.h): total = hi 2^80 + mid 2^40 + lo
// with mid, lo in [0, 2^40), carry 0.
__global__ void normalize_limbs_kernel(unsigned long long* limbs, int count) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < count; k += gridDim.x * blockDim.x) {
    unsigned long long* l = limbs + (size_t)k * kLimbs;
    const __int128 T = limbs_total(l);
    const __int128 m40 = ((__int128)1 << 40) - 1;
    l[0] = (unsigned long long)(long long)(T >> 80);
    l[1] = (unsigned long long)(long long)((T >> 40) & m40);
    l[2] = (unsigned long long)(long long)(T & m40);
    l[3] = 0ull;
  }
}

cudaError_t launch_normalize_limbs(unsigned long long* limbs, int count, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  normalize_limbs_kernel<<<(count + 255) / 256, 256, 0, s>>>(limbs, count);
  return cudaGetLastError();
}

// Ascending sort of n fp64 samples (CUB radix sort, keys only: deterministic).  The pair sums
// are invariant under permutation; sorted input keeps the term magnitudes inside a column
// group homogeneous, which makes the fp32 group sums of FPsi nearly lossless.
size_t sort_temp_bytes(int64_t n) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, bytes, (const double*)nullptr, (double*)nullptr, (int)n);
  return bytes;
}

cudaError_t launch_sort(const double* in, double* out, int64_t n, void* temp, size_t temp_bytes,
                        cudaStream_t s) {
  return cub::DeviceRadixSort::SortKeys(temp, temp_bytes, in, out, (int)n, 0, 64, s);
}

// LSCV data sorted by coordinate 0 (exact far-tile skip): stable radix sort of
// (x_0j, j), then a gather of all d rows.  Whitening keeps the order of coordinate 0 (W is lower
// triangular with W_00 > 0), so every prepared set is sorted by its first coordinate too.
size_t sort_rows_temp_bytes(int64_t n) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const double*)nullptr, (double*)nullptr, (const int*)nullptr,
                                  (int*)nullptr, (int)n);
  return bytes;
}

__global__ void iota_kernel(int* idx, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    idx[i] = (int)i;
}

__global__ void gather_rows_kernel(const double* __restrict__ X, int64_t n, int d, const int* __restrict__ perm,
                                   double* __restrict__ Xs) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = perm[i];
    for (int a = 0; a < d; ++a) Xs[a * n + i] = X[a * n + j];
  }
}

cudaError_t launch_sort_rows(const double* X, int64_t n, int d, double* Xs, double* keys, int* idx, void* temp,
                             size_t temp_bytes, cudaStream_t s) {
  const unsigned blocks = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 8);
  iota_kernel<<<blocks, 256, 0, s>>>(idx, n);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  e = cub::DeviceRadixSort::SortPairs(temp, temp_bytes, X, keys, idx, idx + n, (int)n, 0, 64, s);
  if (e != cudaSuccess) return e;
  gather_rows_kernel<<<blocks, 256, 0, s>>>(X, n, d, idx + n, Xs);
  return cudaGetLastError();
}


}  // namespace kde
