// kde_lscv64.cu — fp64-term LSCV sums: the automatic-precision re-run of a candidate
// whose objective g = 2(c4 S1 - 2 c2 S2)/n^2 + c4/n cancels so much that the fp32 terms' error
// (~1.5e-7 relative on S1, S2) could exceed the 1e-5 contract, and the kde_set_precision(ctx, 1) mode.
// Every term in fp64: the data whitened in fp64 (prep64_kernel: the fp32 prep's arithmetic without
// the final rounding), s = |y_i - y_j|^2, e = exp2(kappa s) (libdevice), fp64 sums over 256-tiles, the
// same fixed-point limbs, tile map and rank partition as the fp32 path.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "kde_pair.cuh"

namespace kde {

constexpr int kL64Tile = 256;

// y_a = sum_b W_ab (x_b - mean_b) in fp64 (the same fma order as prep_body), zero padded to ld.
__global__ void prep64_kernel(const double* __restrict__ X, int64_t n, int d, const __grid_constant__ PrepParams pp,
                              double* __restrict__ Y, int64_t ld) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ld; i += stride) {
    if (i < n) {
      double v[kMaxDim];
      for (int b = 0; b < d; ++b) v[b] = X[b * n + i] - pp.mean[b];
      for (int a = 0; a < d; ++a) {
        double s = 0.0;
        for (int b = 0; b < d; ++b) s = fma(pp.W[a * d + b], v[b], s);
        Y[a * ld + i] = s;
      }
    } else {
      for (int a = 0; a < d; ++a) Y[a * ld + i] = 0.0;
    }
  }
}

// Outputs (sum e, sum e^2) over this launch's tiles.  Rows sorted by coordinate 0: a tile whose
// coordinate-0 gap g has g^2 > skip_s (= 1100 / |kappa|: exp2 underflows to 0 in fp64) adds exactly 0.
template <int D>
__global__ void __launch_bounds__(kL64Tile) lscv64_kernel(const double* __restrict__ Y, int64_t n, int64_t ld,
                                                          int64_t tb, int64_t te, double kappa, double skip_s, int S,
                                                          unsigned long long* __restrict__ limbs, int part_rank,
                                                          int part_world) {
  __shared__ double cs[D][kL64Tile];
  __shared__ double red[(kL64Tile / 32) * 2];
  const int tid = threadIdx.x;
  for (int64_t u = tb + blockIdx.x; u < te; u += gridDim.x) {   // this rank's local tile indices
    int64_t l, q;
    tile_coords(shard_tile(u, part_rank, part_world), l, q);
    if (q < l) {
      const double g = Y[l * kL64Tile] - Y[q * kL64Tile + kL64Tile - 1];
      if (g * g > skip_s) continue;   // uniform per CTA
    }
    __syncthreads();
#pragma unroll
    for (int a = 0; a < D; ++a) cs[a][tid] = Y[a * ld + l * kL64Tile + tid];
    __syncthreads();
    const int64_t i = q * kL64Tile + tid;
    const int jlim = (int)(n - l * kL64Tile < kL64Tile ? n - l * kL64Tile : kL64Tile);
    double a1 = 0.0, a2 = 0.0;
    if (i < n) {
      double xi[D];
#pragma unroll
      for (int a = 0; a < D; ++a) xi[a] = Y[a * ld + i];
      for (int j = (q == l ? tid + 1 : 0); j < jlim; ++j) {
        double s = 0.0;
#pragma unroll
        for (int a = 0; a < D; ++a) {
          const double u = xi[a] - cs[a][j];
          s = fma(u, u, s);
        }
        const double e = exp2(kappa * s);
        a1 += e;
        a2 = fma(e, e, a2);
      }
    }
    double v[2] = {a1, a2};
    commit_tile<2, kL64Tile>(v, red, limbs, S);
  }
}

int lscv64_tile() { return kL64Tile; }

cudaError_t launch_prep64(const double* X, int64_t n, int d, const PrepParams& pp, double* Y, int64_t ld,
                          cudaStream_t s) {
  const unsigned blocks = (unsigned)std::min<int64_t>((ld + 255) / 256, 148 * 16);
  prep64_kernel<<<blocks, 256, 0, s>>>(X, n, d, pp, Y, ld);
  return cudaGetLastError();
}

template <int D>
static cudaError_t launch64_d(const double* Y, int64_t n, int64_t ld, int64_t tb, int64_t te, double kappa,
                              double skip_s, int S, unsigned long long* limbs, int sm_count, cudaStream_t s,
                              int pr, int pw) {
  const int64_t grid = std::min<int64_t>(te - tb, (int64_t)sm_count * 8);
  lscv64_kernel<D><<<(unsigned)grid, kL64Tile, 0, s>>>(Y, n, ld, tb, te, kappa, skip_s, S, limbs, pr, pw);
  return cudaGetLastError();
}

cudaError_t launch_lscv64(int d, const double* Y, int64_t n, int64_t ld, int64_t tb, int64_t te, double kappa,
                          double skip_s, int S, unsigned long long* limbs, int sm_count, cudaStream_t s, int pr,
                          int pw) {
  if (te <= tb) return cudaSuccess;
  switch (d) {
    case 1: return launch64_d<1>(Y, n, ld, tb, te, kappa, skip_s, S, limbs, sm_count, s, pr, pw);
    case 2: return launch64_d<2>(Y, n, ld, tb, te, kappa, skip_s, S, limbs, sm_count, s, pr, pw);
    case 3: return launch64_d<3>(Y, n, ld, tb, te, kappa, skip_s, S, limbs, sm_count, s, pr, pw);
    case 4: return launch64_d<4>(Y, n, ld, tb, te, kappa, skip_s, S, limbs, sm_count, s, pr, pw);
    case 5: return launch64_d<5>(Y, n, ld, tb, te, kappa, skip_s, S, limbs, sm_count, s, pr, pw);
    case 6: return launch64_d<6>(Y, n, ld, tb, te, kappa, skip_s, S, limbs, sm_count, s, pr, pw);
    case 7: return launch64_d<7>(Y, n, ld, tb, te, kappa, skip_s, S, limbs, sm_count, s, pr, pw);
    case 8: return launch64_d<8>(Y, n, ld, tb, te, kappa, skip_s, S, limbs, sm_count, s, pr, pw);
    case 9: return launch64_d<9>(Y, n, ld, tb, te, kappa, skip_s, S, limbs, sm_count, s, pr, pw);
    case 10: return launch64_d<10>(Y, n, ld, tb, te, kappa, skip_s, S, limbs, sm_count, s, pr, pw);
    case 11: return launch64_d<11>(Y, n, ld, tb, te, kappa, skip_s, S, limbs, sm_count, s, pr, pw);
    case 12: return launch64_d<12>(Y, n, ld, tb, te, kappa, skip_s, S, limbs, sm_count, s, pr, pw);
    case 13: return launch64_d<13>(Y, n, ld, tb, te, kappa, skip_s, S, limbs, sm_count, s, pr, pw);
    case 14: return launch64_d<14>(Y, n, ld, tb, te, kappa, skip_s, S, limbs, sm_count, s, pr, pw);
    case 15: return launch64_d<15>(Y, n, ld, tb, te, kappa, skip_s, S, limbs, sm_count, s, pr, pw);
    case 16: return launch64_d<16>(Y, n, ld, tb, te, kappa, skip_s, S, limbs, sm_count, s, pr, pw);
  }
  return cudaErrorInvalidValue;
}

}  // namespace kde
