// kde_materialized.cu — the paper's two-phase LSCV_h (Sec. 6.2), SURVEY §8(f) f3.
//
// Phase 1 (the "fun2" tile writer of Sec. 5.5, Eq. 44-56): for every pair i<j of the
//   rank's triangular tiles write s_ij = (log2 e / 4) (X_i - X_j)^T Sigma^-1 (X_i - X_j) as fp32
//   to a device buffer (data pre-whitened, so s = |x_i' - x_j'|^2); positions outside i<j or
//   past n hold +inf.  Layout: tile t occupies [t*T*T, (t+1)*T*T), column-major inside the
//   tile (consecutive threads = consecutive rows -> coalesced stores).
// Phase 2 (the per-h map-reduce of Sec. 6.2.1): stream the buffer once per batch of B
//   candidates; for each value e = 2^(s kappa_c), accumulate sum e and sum e^2 per candidate.
//   With B = 1 this is the paper's design (one grid row per h), HBM-bound; B > 1 amortises
//   one buffer read over B candidates.  Each 16384-value chunk's fp64 partial is added as
//   exact fixed-point limbs (deterministic).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "kde_device.cuh"
#include "kde_internal.h"
#include "kde_tiles.cuh"

namespace kde {

constexpr int kMatT = 256;   // tile edge
constexpr int kP2Threads = 256;
constexpr int kP2Vec = 64;   // float4 per thread per chunk (one 256x256 tile: epilogue every 256 KB)
constexpr int64_t kP2Chunk = (int64_t)kP2Threads * kP2Vec * 4;

int mat_tile() { return kMatT; }
int64_t mat_chunk() { return kP2Chunk; }

template <int D>
__global__ void __launch_bounds__(kMatT) mat_write_kernel(const float* __restrict__ X, int64_t n, int64_t ld,
                                                          int64_t tb, int64_t te, float* __restrict__ buf,
                                                          int part_rank, int part_world) {
  __shared__ float cs[D][kMatT];
  const int tid = threadIdx.x;
  for (int64_t t = tb + blockIdx.x; t < te; t += gridDim.x) {   // local tile indices of this rank
    int64_t l, q;
    tile_coords(shard_tile(t, part_rank, part_world), l, q);
    __syncthreads();
#pragma unroll
    for (int d = 0; d < D; ++d) cs[d][tid] = X[d * ld + l * kMatT + tid];
    float xr[D];
#pragma unroll
    for (int d = 0; d < D; ++d) xr[d] = X[d * ld + q * kMatT + tid];
    __syncthreads();
    const int64_t jlim = n - l * kMatT;
    const bool diag = (q == l);
    float* out = buf + (t - tb) * (int64_t)kMatT * kMatT;
#pragma unroll 4
    for (int jj = 0; jj < kMatT; ++jj) {
      float dd = __fsub_rn(xr[0], cs[0][jj]);
      float s = __fmul_rn(dd, dd);
#pragma unroll
      for (int d = 1; d < D; ++d) {
        dd = __fsub_rn(xr[d], cs[d][jj]);
        s = __fmaf_rn(dd, dd, s);
      }
      const bool ok = (jj < jlim) && (!diag || jj > tid) && (q * kMatT + tid < n);
      out[(int64_t)jj * kMatT + tid] = ok ? s : __int_as_float(0x7f800000);
    }
  }
}

template <int B>
__global__ void __launch_bounds__(kP2Threads) mat_reduce_kernel(const float4* __restrict__ buf, int64_t nchunks,
                                                                const LscvScalarParams p, int S,
                                                                unsigned long long* __restrict__ limbs) {
  __shared__ double red[kP2Threads / 32][2 * B];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  for (int64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    float a1[B], a2[B];
#pragma unroll
    for (int c = 0; c < B; ++c) a1[c] = a2[c] = 0.f;
    const float4* src = buf + ch * (kP2Chunk / 4);
#pragma unroll 4
    for (int v = 0; v < kP2Vec; ++v) {
      const float4 f = __ldcs(src + v * kP2Threads + tid);   // streamed once per pass
      const float sv[4] = {f.x, f.y, f.z, f.w};
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int c = 0; c < B; ++c) {
          const float e = ex2(__fmul_rn(sv[k], p.kappa[c]));
          a1[c] = __fadd_rn(a1[c], e);
          a2[c] = __fmaf_rn(e, e, a2[c]);
        }
    }
    double v[2 * B];
#pragma unroll
    for (int c = 0; c < B; ++c) { v[2 * c] = warp_sum((double)a1[c]); v[2 * c + 1] = warp_sum((double)a2[c]); }
    if (lane == 0)
#pragma unroll
      for (int k = 0; k < 2 * B; ++k) red[w][k] = v[k];
    __syncthreads();
    if (tid < 2 * B) {
      double s = red[0][tid];
      for (int ww = 1; ww < kP2Threads / 32; ++ww) s += red[ww][tid];
      add_limbs(s, S, limbs + (size_t)tid * kLimbs);
    }
    __syncthreads();
  }
}

cudaError_t launch_mat_write(int d, const float* X, int64_t n, int64_t ld, int64_t tb, int64_t te, float* buf,
                             int sm_count, cudaStream_t s, int pr, int pw) {
  if (te <= tb) return cudaSuccess;
  int64_t grid = te - tb;
  if (grid > (int64_t)sm_count * 8) grid = (int64_t)sm_count * 8;
  switch (d) {
#define W(DD) case DD: mat_write_kernel<DD><<<(unsigned)grid, kMatT, 0, s>>>(X, n, ld, tb, te, buf, pr, pw); break;
    W(1) W(2) W(3) W(4) W(5) W(6) W(7) W(8) W(9) W(10) W(11) W(12) W(13) W(14) W(15) W(16)
#undef W
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_mat_reduce(int B, const float* buf, int64_t nvalues, const LscvScalarParams& p, int S,
                              unsigned long long* limbs, int sm_count, cudaStream_t s) {
  const int64_t nchunks = nvalues / kP2Chunk;   // nvalues is a multiple of the chunk (tile = 65536)
  if (nchunks <= 0) return cudaSuccess;
  int64_t grid = nchunks;
  if (grid > (int64_t)sm_count * 8) grid = (int64_t)sm_count * 8;
  const float4* b4 = reinterpret_cast<const float4*>(buf);
  switch (B) {
    case 1: mat_reduce_kernel<1><<<(unsigned)grid, kP2Threads, 0, s>>>(b4, nchunks, p, S, limbs); break;
    case 2: mat_reduce_kernel<2><<<(unsigned)grid, kP2Threads, 0, s>>>(b4, nchunks, p, S, limbs); break;
    case 4: mat_reduce_kernel<4><<<(unsigned)grid, kP2Threads, 0, s>>>(b4, nchunks, p, S, limbs); break;
    case 8: mat_reduce_kernel<8><<<(unsigned)grid, kP2Threads, 0, s>>>(b4, nchunks, p, S, limbs); break;
    case 16: mat_reduce_kernel<16><<<(unsigned)grid, kP2Threads, 0, s>>>(b4, nchunks, p, S, limbs); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace kde
