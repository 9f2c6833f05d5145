// kde_eval.cu — KDE evaluation at query points and univariate AQP aggregates.
//
// fhat(y_q) = n^-1 |H|^{-1/2} (2 pi)^{-d/2} sum_i exp(-1/2 (y_q - X_i)^T H^-1 (y_q - X_i))
// (Eq. kde-def-H, K_H, gaussian: P:114-140) over a rectangle of m queries x n samples.  Both sets
// are whitened on the device, y' = W (y - mu), x' = W (x - mu) with W^T W = (log2 e / 2) H^-1,
// so every term is 2^-|y' - x'|^2: D sub + D FMA + one MUFU.EX2 per (query, sample).
//
// Work unit = (block of 512 query rows, contiguous split of the sample columns).  A unit streams
// its column tiles through shared memory with TMA bulk copies (double-buffered on mbarriers),
// keeps two query rows per thread packed in fp32x2 lanes, sums 16-column groups in fp32 and adds
// them with Fast2Sum, then writes one fp64 partial per (split, row).  A second kernel adds the
// splits in a fixed order: results do not depend on the grid size.  Terms are all positive (no
// cancellation), so MUFU.EX2's bias needs no offset scheme here.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "kde_device.cuh"
#include "kde_internal.h"

namespace kde {

constexpr int kEvNT = 256;            // threads per CTA
constexpr int kEvRows = 2 * kEvNT;    // query rows per unit (2 per thread, packed)
constexpr int kEvTC = 1024;           // sample columns per tile
constexpr int kEvG = 16;              // columns per compensated group

struct EvalArgs {
  const float* Y;     // D x ldm whitened queries (padded with 0), sorted by coordinate 0
  const float* X;     // D x ldn whitened samples (padded with +inf -> term 0), sorted by coordinate 0
  int64_t m, n, ldm, ldn;
  int row_blocks, splits, tiles_per_split, n_tiles;
  float skip_s;       // far sample tiles: skipped when fp32(coordinate-0 gap)^2 > skip_s (+inf: never)
  const int* range;   // per row block its sample tiles [ta, tb] (eval_range_kernel), or null: all
  double* part;       // [splits][ldm]
};

// Bounded far-tile skip (row f2): queries and samples are sorted by whitened coordinate
// 0, so the sample tiles a block of sorted queries needs form one contiguous range [ta, tb]; every other
// tile has all its terms 2^-s <= 2^-skip_s (s >= fp32(gap)^2, rounding is monotone).  Thread 0 finds the
// range by binary search (eval_range_kernel, one thread per row block); the column split then divides
// [ta, tb].
__device__ __forceinline__ bool ev_tile_below(const EvalArgs& a, int t, float qmin) {   // skipped, below
  const int64_t j = (int64_t)t * kEvTC + kEvTC - 1;
  const float tmax = a.X[j < a.n ? j : a.n - 1];
  if (!(tmax < qmin)) return false;
  const float g = __fsub_rn(qmin, tmax);
  return __fmul_rn(g, g) > a.skip_s;
}
__device__ __forceinline__ bool ev_tile_above(const EvalArgs& a, int t, float qmax) {   // skipped, above
  const float tmin = a.X[(int64_t)t * kEvTC];
  if (!(tmin > qmax)) return false;
  const float g = __fsub_rn(tmin, qmax);
  return __fmul_rn(g, g) > a.skip_s;
}

template <int D>
__global__ void __launch_bounds__(kEvNT, D <= 4 ? 4 : 2) eval_kernel(const EvalArgs a) {   // d <= 4: <= 64 registers, 4 CTAs/SM
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* cols = reinterpret_cast<float*>(smem_raw);                        // [2][D][TC]
  uint64_t* bar = reinterpret_cast<uint64_t*>(cols + 2 * D * kEvTC);      // [2]
  const int tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  auto issue = [&](int tile, int buf) {
    float* dst = cols + buf * D * kEvTC;
    mbar_expect_tx(&bar[buf], (uint32_t)(D * kEvTC * sizeof(float)));
#pragma unroll
    for (int d = 0; d < D; ++d)
      tma_load_1d(dst + d * kEvTC, a.X + d * a.ldn + (int64_t)tile * kEvTC,
                  (uint32_t)(kEvTC * sizeof(float)), &bar[buf]);
  };

  const int units = a.row_blocks * a.splits;
  __shared__ int s_range[2];
  uint32_t k = 0;   // running tile counter of this CTA (buffer = k & 1, parity = (k >> 1) & 1)
  for (int u = blockIdx.x; u < units; u += gridDim.x) {
    const int rb = u % a.row_blocks, cs = u / a.row_blocks;
    __syncthreads();   // previous unit finished reading both buffers (and s_range)
    if (tid == 0) {    // this split's share of the row block's sample tiles [ta, tb]
      const int ta = a.range != nullptr ? a.range[2 * rb] : 0;
      const int tb = a.range != nullptr ? a.range[2 * rb + 1] : a.n_tiles - 1;
      const int len = tb - ta + 1 > 0 ? tb - ta + 1 : 0;
      s_range[0] = ta + (int)((int64_t)len * cs / a.splits);
      s_range[1] = ta + (int)((int64_t)len * (cs + 1) / a.splits);
    }
    __syncthreads();
    const int t0 = s_range[0], t1 = s_range[1];
    const int64_t r0 = (int64_t)rb * kEvRows + tid;
    if (t0 >= t1) {   // nothing of this split is within reach: an exact zero partial
      a.part[(int64_t)cs * a.ldm + r0] = 0.0;
      a.part[(int64_t)cs * a.ldm + r0 + kEvNT] = 0.0;
      continue;
    }
    if (tid == 0) issue(t0, k & 1);
    f2 y[D];
#pragma unroll
    for (int d = 0; d < D; ++d) y[d] = pk(__ldg(a.Y + d * a.ldm + r0), __ldg(a.Y + d * a.ldm + r0 + kEvNT));
    f2 acc = pk(0.f, 0.f), cmp = pk(0.f, 0.f);
    for (int t = t0; t < t1; ++t, ++k) {
      if (tid == 0 && t + 1 < t1) issue(t + 1, (k + 1) & 1);
      mbar_wait(&bar[k & 1], (k >> 1) & 1);
      const float* sc = cols + (k & 1) * D * kEvTC;
#pragma unroll 2   // two column groups per iteration (f2 d=1: 12.83 -> 12.65 ms)
      for (int j = 0; j < kEvTC; j += kEvG) {
        f2 grp = pk(0.f, 0.f);
#pragma unroll
        for (int j4 = 0; j4 < kEvG; j4 += 4) {
          float cv[D][4];
#pragma unroll
          for (int d = 0; d < D; ++d) {
            const float4 c4 = *reinterpret_cast<const float4*>(sc + d * kEvTC + j + j4);
            cv[d][0] = c4.x; cv[d][1] = c4.y; cv[d][2] = c4.z; cv[d][3] = c4.w;
          }
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            f2 v = sub2(y[0], pk(cv[0][kk], cv[0][kk]));
            f2 s = mul2(v, v);
#pragma unroll
            for (int d = 1; d < D; ++d) {
              v = sub2(y[d], pk(cv[d][kk], cv[d][kk]));
              s = fma2(v, v, s);
            }
            if (kk == 3) {   // a quarter of the exponentials on the FMA pipe (slot kk = 3)
              grp = add2(grp, exp2_sw2(sub2(pk(0.f, 0.f), s)));
            } else {
              float s0, s1;
              upk(s, s0, s1);
              grp = add2(grp, pk(ex2(-s0), ex2(-s1)));
            }
          }
        }
        const f2 s2 = add2(acc, grp);          // Fast2Sum(acc, grp): terms > 0, acc grows
        cmp = add2(cmp, sub2(grp, sub2(s2, acc)));
        acc = s2;
      }
      __syncthreads();   // all threads done with this buffer before it is refilled
    }
    float a0, a1, c0, c1;
    upk(acc, a0, a1);
    upk(cmp, c0, c1);
    a.part[(int64_t)cs * a.ldm + r0] = (double)a0 + (double)c0;
    a.part[(int64_t)cs * a.ldm + r0 + kEvNT] = (double)a1 + (double)c1;
  }
}

__global__ void eval_range_kernel(const EvalArgs a, int* __restrict__ range) {
  const int rb = blockIdx.x * blockDim.x + threadIdx.x;
  if (rb >= a.row_blocks) return;
  const int64_t q0 = (int64_t)rb * kEvRows, q1 = q0 + kEvRows - 1 < a.m - 1 ? q0 + kEvRows - 1 : a.m - 1;
  const float qmin = a.Y[q0], qmax = a.Y[q1];
  int lo = 0, hi = a.n_tiles;   // first tile not skipped below the block
  while (lo < hi) { const int mid = (lo + hi) >> 1; if (ev_tile_below(a, mid, qmin)) lo = mid + 1; else hi = mid; }
  const int ta = lo;
  lo = ta; hi = a.n_tiles;      // first tile skipped above it
  while (lo < hi) { const int mid = (lo + hi) >> 1; if (ev_tile_above(a, mid, qmax)) hi = mid; else lo = mid + 1; }
  range[2 * rb] = ta;
  range[2 * rb + 1] = lo - 1;
}

__global__ void eval_reduce_kernel(const double* __restrict__ part, int splits, int64_t ldm,
                                   int64_t m, double scale, const int* __restrict__ perm, double* __restrict__ out) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < m; q += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int c = 0; c < splits; ++c) s += part[(int64_t)c * ldm + q];
    out[perm != nullptr ? perm[q] : q] = s * scale;   // sorted query q is the caller's query perm[q]
  }
}

int eval_rows_per_block() { return kEvRows; }
int eval_cols_per_tile() { return kEvTC; }

template <int D>
static cudaError_t eval_occupancy(int* occ_out) {
  const size_t smem = 2 * D * kEvTC * sizeof(float) + 16;
  static int occ_dev[kMaxDevices];   // 0 = not yet set up on that device (the opt-in is per device)
  int& occ = occ_dev[current_device()];
  if (occ <= 0) {
    cudaError_t e = cudaFuncSetAttribute(eval_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int o = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, eval_kernel<D>, kEvNT, smem);
    if (e != cudaSuccess) return e;
    occ = o > 0 ? o : 1;
  }
  *occ_out = occ;
  return cudaSuccess;
}

// Columns are split so that there are >= 2 waves of (row block, split) units (deterministic for a
// given m, n and SM count); returns the number of splits actually used.
static int eval_split_count(int sm_count, int occ, int64_t ldm, int64_t ldn, int* tiles_per_split) {
  const int row_blocks = (int)(ldm / kEvRows), n_tiles = (int)(ldn / kEvTC);
  const int target = 2 * sm_count * occ;
  int splits = (target + row_blocks - 1) / row_blocks;
  if (splits > n_tiles) splits = n_tiles;
  if (splits < 1) splits = 1;
  const int tps = (n_tiles + splits - 1) / splits;
  if (tiles_per_split) *tiles_per_split = tps;
  return (n_tiles + tps - 1) / tps;
}

template <int D>
static cudaError_t eval_splits_d(int sm_count, int64_t ldm, int64_t ldn, int* splits) {
  int occ = 1;
  cudaError_t e = eval_occupancy<D>(&occ);
  if (e != cudaSuccess) return e;
  *splits = eval_split_count(sm_count, occ, ldm, ldn, nullptr);
  return cudaSuccess;
}

template <int D>
static cudaError_t launch_eval_d(const EvalLaunch& c) {
  const size_t smem = 2 * D * kEvTC * sizeof(float) + 16;
  int occ = 1;
  cudaError_t e0 = eval_occupancy<D>(&occ);
  if (e0 != cudaSuccess) return e0;
  EvalArgs a;
  a.Y = c.Y; a.X = c.X; a.m = c.m; a.n = c.n; a.ldm = c.ldm; a.ldn = c.ldn; a.skip_s = c.skip_s;
  a.row_blocks = (int)(c.ldm / kEvRows);
  a.n_tiles = (int)(c.ldn / kEvTC);
  a.splits = eval_split_count(c.sm_count, occ, c.ldm, c.ldn, &a.tiles_per_split);
  a.part = c.part;
  a.range = nullptr;
  if ((size_t)a.splits * (size_t)c.ldm > c.part_capacity) return cudaErrorInvalidValue;
  if (c.skip_s < INFINITY && c.range != nullptr) {
    eval_range_kernel<<<(a.row_blocks + 127) / 128, 128, 0, c.stream>>>(a, c.range);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    a.range = c.range;
  }
  const int units = a.row_blocks * a.splits;
  int grid = c.sm_count * occ;
  if (grid > units) grid = units;
  eval_kernel<D><<<grid, kEvNT, smem, c.stream>>>(a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  int blocks = (int)((c.m + 255) / 256);
  if (blocks > 4096) blocks = 4096;
  if (blocks < 1) blocks = 1;
  eval_reduce_kernel<<<blocks, 256, 0, c.stream>>>(c.part, a.splits, c.ldm, c.m, c.scale, c.perm, c.out);
  return cudaGetLastError();
}


cudaError_t eval_splits(int d, int sm_count, int64_t ldm, int64_t ldn, int* splits) {
  switch (d) {
    case 1: return eval_splits_d<1>(sm_count, ldm, ldn, splits);   case 2: return eval_splits_d<2>(sm_count, ldm, ldn, splits);
    case 3: return eval_splits_d<3>(sm_count, ldm, ldn, splits);   case 4: return eval_splits_d<4>(sm_count, ldm, ldn, splits);
    case 5: return eval_splits_d<5>(sm_count, ldm, ldn, splits);   case 6: return eval_splits_d<6>(sm_count, ldm, ldn, splits);
    case 7: return eval_splits_d<7>(sm_count, ldm, ldn, splits);   case 8: return eval_splits_d<8>(sm_count, ldm, ldn, splits);
    case 9: return eval_splits_d<9>(sm_count, ldm, ldn, splits);   case 10: return eval_splits_d<10>(sm_count, ldm, ldn, splits);
    case 11: return eval_splits_d<11>(sm_count, ldm, ldn, splits); case 12: return eval_splits_d<12>(sm_count, ldm, ldn, splits);
    case 13: return eval_splits_d<13>(sm_count, ldm, ldn, splits); case 14: return eval_splits_d<14>(sm_count, ldm, ldn, splits);
    case 15: return eval_splits_d<15>(sm_count, ldm, ldn, splits); case 16: return eval_splits_d<16>(sm_count, ldm, ldn, splits);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_eval(int d, const EvalLaunch& c) {
  switch (d) {
    case 1: return launch_eval_d<1>(c);   case 2: return launch_eval_d<2>(c);
    case 3: return launch_eval_d<3>(c);   case 4: return launch_eval_d<4>(c);
    case 5: return launch_eval_d<5>(c);   case 6: return launch_eval_d<6>(c);
    case 7: return launch_eval_d<7>(c);   case 8: return launch_eval_d<8>(c);
    case 9: return launch_eval_d<9>(c);   case 10: return launch_eval_d<10>(c);
    case 11: return launch_eval_d<11>(c); case 12: return launch_eval_d<12>(c);
    case 13: return launch_eval_d<13>(c); case 14: return launch_eval_d<14>(c);
    case 15: return launch_eval_d<15>(c); case 16: return launch_eval_d<16>(c);
  }
  return cudaErrorInvalidValue;
}

// ------------------------------------------------------------------ univariate AQP
// For the Gaussian kernel the integrals of Eq. count / Eq. sum have closed forms per sample:
//   n int_a^b fhat = sum_i [Phi(beta_i) - Phi(alpha_i)],
//   n int_a^b t fhat = sum_i [x_i (Phi(beta_i) - Phi(alpha_i)) + h (phi(alpha_i) - phi(beta_i))],
// alpha_i = (a - x_i)/h, beta_i = (b - x_i)/h; evaluated in fp64 (erfc tail form, no
// cancellation) with a fixed-order block reduction.
constexpr int kAqpThreads = 256;

__device__ __forceinline__ double phi_diff(double al, double be) {
  const double r = 0.70710678118654752440;   // 1/sqrt(2)
  if (al > 0.0) return 0.5 * (erfc(al * r) - erfc(be * r));
  if (be < 0.0) return 0.5 * (erfc(-be * r) - erfc(-al * r));
  return 1.0 - 0.5 * (erfc(-al * r) + erfc(be * r));
}

__global__ void __launch_bounds__(kAqpThreads) aqp_kernel(const double* __restrict__ x, int64_t n,
                                                          double h, const double* __restrict__ lo,
                                                          const double* __restrict__ hi,
                                                          double* __restrict__ part, int q0) {
  __shared__ double red[kAqpThreads / 32][2];
  const int q = q0 + blockIdx.y;
  const double a = lo[q], b = hi[q], ih = 1.0 / h;
  const double k = 0.39894228040143267794;   // 1/sqrt(2 pi)
  double c = 0.0, s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * kAqpThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kAqpThreads) {
    const double xi = x[i];
    const double al = (a - xi) * ih, be = (b - xi) * ih;
    const double p = phi_diff(al, be);
    c += p;
    s += xi * p + h * k * (exp(-0.5 * al * al) - exp(-0.5 * be * be));
  }
  c = warp_sum(c);
  s = warp_sum(s);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) { red[w][0] = c; red[w][1] = s; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double cc = 0.0, ss = 0.0;
    for (int ww = 0; ww < kAqpThreads / 32; ++ww) { cc += red[ww][0]; ss += red[ww][1]; }
    part[((int64_t)q * gridDim.x + blockIdx.x) * 2 + 0] = cc;
    part[((int64_t)q * gridDim.x + blockIdx.x) * 2 + 1] = ss;
  }
}

__global__ void aqp_reduce_kernel(const double* __restrict__ part, int nblk, int nq, double* __restrict__ out) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += gridDim.x * blockDim.x) {
    double c = 0.0, s = 0.0;
    for (int b = 0; b < nblk; ++b) { c += part[((int64_t)q * nblk + b) * 2]; s += part[((int64_t)q * nblk + b) * 2 + 1]; }
    out[2 * q] = c;
    out[2 * q + 1] = s;
  }
}

int aqp_blocks(int64_t n) {
  int64_t b = (n + 4 * kAqpThreads - 1) / (4 * kAqpThreads);
  if (b > 256) b = 256;
  if (b < 1) b = 1;
  return (int)b;
}

cudaError_t launch_aqp(const double* x, int64_t n, double h, const double* lo, const double* hi, int nq,
                       double* part, int nblk, double* out, cudaStream_t s) {
  for (int q0 = 0; q0 < nq; q0 += 65535) {   // gridDim.y <= 65535: intervals in chunks
    const int cnt = nq - q0 < 65535 ? nq - q0 : 65535;
    aqp_kernel<<<dim3(nblk, cnt), kAqpThreads, 0, s>>>(x, n, h, lo, hi, part, q0);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  aqp_reduce_kernel<<<(nq + 127) / 128, 128, 0, s>>>(part, nblk, nq, out);
  return cudaGetLastError();
}

}  // namespace kde
