// kde_lscv_matrix.cu — LSCV_H pair-kernel instantiations: FLscvScalar<D, NT, 1, UNIT> over one
// per-candidate whitened data set per candidate (see kde_pair.cuh, kde_selectors.cpp lscv_H_raw).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "kde_pair.cuh"

namespace kde {

template <int D>
static cudaError_t lscv_white_d(const LaunchCfg& c) {
  LscvScalarParams p{};
  if constexpr (D <= 4)   // large n: 1024-row tiles, 512 threads at 2 CTAs/SM (tile_for)
    if (c.tile == 1024) return launch_pair<FLscvScalar<D, 512, 1, true, 0u, 2>>(c, p);
  return c.tile == 256 ? launch_pair<FLscvScalar<D, 128, 1, true>>(c, p)
                       : launch_pair<FLscvScalar<D, 256, 1, true>>(c, p);
}

template <int D>
static cudaError_t prepare_white_d(const LaunchCfg& c) {
  int occ;
  if constexpr (D <= 4)
    if (c.tile == 1024) return pair_occupancy<FLscvScalar<D, 512, 1, true, 0u, 2>>(&occ);
  return c.tile == 256 ? pair_occupancy<FLscvScalar<D, 128, 1, true>>(&occ)
                       : pair_occupancy<FLscvScalar<D, 256, 1, true>>(&occ);
}

cudaError_t prepare_lscv_white(int d, const LaunchCfg& c) {
  switch (d) {
    case 1: return prepare_white_d<1>(c);   case 2: return prepare_white_d<2>(c);
    case 3: return prepare_white_d<3>(c);   case 4: return prepare_white_d<4>(c);
    case 5: return prepare_white_d<5>(c);   case 6: return prepare_white_d<6>(c);
    case 7: return prepare_white_d<7>(c);   case 8: return prepare_white_d<8>(c);
    case 9: return prepare_white_d<9>(c);   case 10: return prepare_white_d<10>(c);
    case 11: return prepare_white_d<11>(c); case 12: return prepare_white_d<12>(c);
    case 13: return prepare_white_d<13>(c); case 14: return prepare_white_d<14>(c);
    case 15: return prepare_white_d<15>(c); case 16: return prepare_white_d<16>(c);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_lscv_white(int d, const LaunchCfg& c) {
  switch (d) {
    case 1: return lscv_white_d<1>(c);   case 2: return lscv_white_d<2>(c);
    case 3: return lscv_white_d<3>(c);   case 4: return lscv_white_d<4>(c);
    case 5: return lscv_white_d<5>(c);   case 6: return lscv_white_d<6>(c);
    case 7: return lscv_white_d<7>(c);   case 8: return lscv_white_d<8>(c);
    case 9: return lscv_white_d<9>(c);   case 10: return lscv_white_d<10>(c);
    case 11: return lscv_white_d<11>(c); case 12: return lscv_white_d<12>(c);
    case 13: return lscv_white_d<13>(c); case 14: return lscv_white_d<14>(c);
    case 15: return lscv_white_d<15>(c); case 16: return lscv_white_d<16>(c);
  }
  return cudaErrorInvalidValue;
}

// Data-aware bounded skip for LSCV_H sets (kde_internal.h launch_lscv_sets_skip_select).
constexpr int kThetaCands = 48;   // theta_c = theta_cf - c, c < 48, not below 8
__global__ void __launch_bounds__(256) lscv_sets_skip_select_kernel(const float* __restrict__ X, int64_t set_stride,
                                                                    int64_t n, int T, float theta_cf,
                                                                    float* __restrict__ out) {
  __shared__ double red[8][kThetaCands];
  __shared__ int ok[kThetaCands];
  const float* Xs = X + (int64_t)blockIdx.x * set_stride;   // the set's whitened coordinate 0 (sorted)
  double acc[kThetaCands];
#pragma unroll
  for (int c = 0; c < kThetaCands; ++c) acc[c] = 0.0;
  const int64_t nt = (n + T - 1) / T, tiles = nt * (nt + 1) / 2;
  for (int64_t id = threadIdx.x; id < tiles; id += blockDim.x) {   // fixed per-thread order
    int64_t l, q;
    tile_coords(id, l, q);
    if (q >= l) continue;
    const float g = __fsub_rn(Xs[l * T], Xs[q * T + T - 1]);   // lscv_tile_skipped's test, exactly
    const float g2 = __fmul_rn(g, g);
    if (!(g2 > 8.0f)) continue;
    const int64_t cols = n - l * T < T ? n - l * T : T;
    const double b = (double)T * (double)cols * exp2(-(double)g2);   // every term e = 2^-s, s >= g2
#pragma unroll
    for (int c = 0; c < kThetaCands; ++c)
      if (g2 > theta_cf - (float)c) acc[c] += b;
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int c = 0; c < kThetaCands; ++c) {
    double v = acc[c];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[wid][c] = v;
  }
  __syncthreads();
  if (threadIdx.x < kThetaCands) {
    double v = 0.0;
    for (int w = 0; w < 8; ++w) v += red[w][threadIdx.x];
    const double budget = (double)n * (double)(n - 1) * 0.5 * exp2(-(double)theta_cf);
    ok[threadIdx.x] = theta_cf - (float)threadIdx.x >= 8.0f && v * (1.0 + 1e-9) <= budget;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float th = theta_cf;
    for (int c = 0; c < kThetaCands; ++c) {   // the bound grows as theta falls: stop at the first failure
      if (!ok[c]) break;
      th = theta_cf - (float)c;
    }
    out[blockIdx.x] = th;
  }
}

cudaError_t launch_lscv_sets_skip_select(const float* X, int64_t set_stride, int n_sets, int64_t n, int T,
                                         float theta_cf, float* out, cudaStream_t s) {
  if (n_sets <= 0) return cudaSuccess;
  lscv_sets_skip_select_kernel<<<(unsigned)n_sets, 256, 0, s>>>(X, set_stride, n, T, theta_cf, out);
  return cudaGetLastError();
}

}  // namespace kde
