// kde_lscv_scalar.cu — LSCV_h pair-kernel instantiations (see kde_pair.cuh).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "kde_pair.cuh"

namespace kde {

// d <= 4: 8 candidates per pair visit at 4 CTAs/SM (3 until round 2), a quarter of the exponentials in software on
// the FMA pipe (measured on C2: 478 ms vs 490 ms for 16 candidates, all on MUFU); d > 4: the
// per-pair work dominates, 16 candidates on MUFU.
// Software-exp column masks (bit j mod 16): KDE_DEBUG_LSCVh_SW selects an A/B variant for d = 1
// (diagnostics only; results stay deterministic for each setting).
constexpr unsigned kSwDefault = 0x8888u;   // columns 3, 7, 11, 15 of every 16: a quarter

static int sw_variant() {
  static const char* e = getenv("KDE_DEBUG_LSCVh_SW");
  return e ? atoi(e) : 0;
}

template <int D>
static cudaError_t lscv_scalar_d(const LaunchCfg& c, const LscvScalarParams& p) {
  if constexpr (D == 1) {
    switch (sw_variant()) {
      case 1: return launch_pair<FLscvScalar<1, 256, 8, false, 0x8888u, 3, true>>(c, p);   // round-1 kernel
      case 2: return launch_pair<FLscvScalar<1, 256, 8, false, 0x888Au, 3>>(c, p);         // 5/16
      case 3: return launch_pair<FLscvScalar<1, 256, 8, false, 0x0888u, 3>>(c, p);         // 3/16
      case 4: return launch_pair<FLscvScalar<1, 256, 8, false, 0x8A8Au, 3>>(c, p);         // 6/16
      case 5: return launch_pair<FLscvScalar<1, 256, 8, false, 0x0808u, 3>>(c, p);         // 2/16
      case 6: return launch_pair<FLscvScalar<1, 256, 8, false, 0x4210u, 3>>(c, p);         // 3/16 spread
      case 7: return launch_pair<FLscvScalar<1, 256, 8, false, 0x1248u, 3>>(c, p);         // 4/16 spread
      case 8: return launch_pair<FLscvScalar<1, 256, 8, false, 0x0888u, 3, true>>(c, p);   // 3/16, select exp
      case 12: return launch_pair<FLscvScalar<1, 256, 8, false, 0x888Au, 3, false, true, true>>(c, p);  // 5/16
      case 14: return launch_pair<FLscvScalar<1, 256, 8, false, 0x8A8Au, 3, false, true, true>>(c, p);  // 6/16
      case 16: return launch_pair<FLscvScalar<1, 256, 8, false, 0x8888u, 4, false, true, true>>(c, p);  // 4 CTAs/SM
      case 17: return launch_pair<FLscvScalar<1, 256, 8, false, 0x8888u, 3, false, true, true, 2>>(c, p);  // 32 cols/iter
      case 18: return launch_pair<FLscvScalar<1, 256, 8, false, 0x0888u, 3, false, true, true>>(c, p);  // 3/16
      case 19: return launch_pair<FLscvScalar<1, 256, 8, false, 0x4924u, 3, false, true, true>>(c, p);  // 4/16 spread (2,5,8,11,14)
      case 20: return launch_pair<FLscvScalar<1, 256, 8, false, 0x888Au, 4, false, true, true>>(c, p);  // 4 CTAs, 5/16
      case 21: return launch_pair<FLscvScalar<1, 256, 8, false, 0x8A8Au, 4, false, true, true>>(c, p);  // 4 CTAs, 6/16
      case 22: return launch_pair<FLscvScalar<1, 256, 8, false, 0x8888u, 4, false, false, true>>(c, p); // 4 CTAs, col-major
      case 23: return launch_pair<FLscvScalar<1, 256, 8, false, 0x8888u, 4, false, true, false>>(c, p); // 4 CTAs, plain exp
      case 25: return launch_pair<FLscvScalar<1, 256, 8, false, 0x0888u, 4, false, true, true>>(c, p);  // 4 CTAs, 3/16
      default: break;
    }
  }
  if constexpr (D <= 4) {
    switch (sw_variant()) {
      case 9: return launch_pair<FLscvScalar<D, 256, 8, false, kSwDefault, 3, false, true, false>>(c, p);    // cand-major
      case 10: return launch_pair<FLscvScalar<D, 256, 8, false, kSwDefault, 3, false, false, true>>(c, p);   // fma exp
      case 15: return launch_pair<FLscvScalar<D, 256, 8, false, kSwDefault, 3, false, false, false>>(c, p);  // round-2 kernel
      case 24: return launch_pair<FLscvScalar<D, 256, 8, false, kSwDefault, 4, false, true, true>>(c, p);    // 4 CTAs/SM
      case 26: return launch_pair<FLscvScalar<D, 256, 8, false, kSwDefault, 3, false, true, true>>(c, p);    // 3 CTAs/SM
      default: break;
    }
    // default (C2 A/B, profiles/r02_lscv_h_variants2.jsonl): candidate-major order, product folded into
    // the software exp's range reduction, 4 CTAs/SM (64 registers; the spills sit outside the column loop):
    // C2 405.5 (round-2 kernel) -> 400.5 (3 CTAs) -> 385.5 ms
    return launch_pair<FLscvScalar<D, 256, nb_scalar(D), false, kSwDefault, 4, false, true, true>>(c, p);
  } else {
    return launch_pair<FLscvScalar<D, 256, nb_scalar(D)>>(c, p);
  }
}

cudaError_t launch_lscv_scalar(int d, int nb, const LaunchCfg& c, const LscvScalarParams& p) {
  (void)nb;
  switch (d) {
    case 1: return lscv_scalar_d<1>(c, p);   case 2: return lscv_scalar_d<2>(c, p);
    case 3: return lscv_scalar_d<3>(c, p);   case 4: return lscv_scalar_d<4>(c, p);
    case 5: return lscv_scalar_d<5>(c, p);   case 6: return lscv_scalar_d<6>(c, p);
    case 7: return lscv_scalar_d<7>(c, p);   case 8: return lscv_scalar_d<8>(c, p);
    case 9: return lscv_scalar_d<9>(c, p);   case 10: return lscv_scalar_d<10>(c, p);
    case 11: return lscv_scalar_d<11>(c, p); case 12: return lscv_scalar_d<12>(c, p);
    case 13: return lscv_scalar_d<13>(c, p); case 14: return lscv_scalar_d<14>(c, p);
    case 15: return lscv_scalar_d<15>(c, p); case 16: return lscv_scalar_d<16>(c, p);
  }
  return cudaErrorInvalidValue;
}

// Data-aware bounded skip for LSCV_h (kde_internal.h launch_lscv_h_skip_select).
constexpr int kThetaCandsH = 48;   // theta_c = theta_cf - c, c < 48, not below 8
__global__ void __launch_bounds__(256) lscv_h_skip_select_kernel(const float* __restrict__ X0, int64_t n, int T,
                                                                 const float* __restrict__ kappa, float theta_cf,
                                                                 float* __restrict__ out) {
  __shared__ double red[8][kThetaCandsH];
  __shared__ int ok[kThetaCandsH];
  const float k = kappa[blockIdx.x];   // < 0
  const float ak = -k;
  double acc[kThetaCandsH];
#pragma unroll
  for (int c = 0; c < kThetaCandsH; ++c) acc[c] = 0.0;
  const int64_t nt = (n + T - 1) / T, tiles = nt * (nt + 1) / 2;
  for (int64_t id = threadIdx.x; id < tiles; id += blockDim.x) {   // fixed per-thread order
    int64_t l, q;
    tile_coords(id, l, q);
    if (q >= l) continue;
    const float g = __fsub_rn(X0[l * T], X0[q * T + T - 1]);   // the pair kernel's skip test, exactly
    const float g2 = __fmul_rn(g, g);
    if (!(g2 > __fdiv_rn(8.0f, ak))) continue;
    const int64_t cols = n - l * T < T ? n - l * T : T;
    const double b = (double)T * (double)cols * exp2((double)k * (double)g2);   // e <= 2^(kappa g^2)
#pragma unroll
    for (int c = 0; c < kThetaCandsH; ++c)
      if (g2 > __fdiv_rn(theta_cf - (float)c, ak)) acc[c] += b;
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int c = 0; c < kThetaCandsH; ++c) {
    double v = acc[c];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[wid][c] = v;
  }
  __syncthreads();
  if (threadIdx.x < kThetaCandsH) {
    double v = 0.0;
    for (int w = 0; w < 8; ++w) v += red[w][threadIdx.x];
    const double budget = (double)n * (double)(n - 1) * 0.5 * exp2(-(double)theta_cf);
    ok[threadIdx.x] = theta_cf - (float)threadIdx.x >= 8.0f && v * 1.0001 <= budget;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float th = theta_cf;
    for (int c = 0; c < kThetaCandsH; ++c) {   // the bound grows as theta falls: stop at the first failure
      if (!ok[c]) break;
      th = theta_cf - (float)c;
    }
    out[blockIdx.x] = __fdiv_rn(th, ak);
  }
}

cudaError_t launch_lscv_h_skip_select(const float* X0, int64_t n, int T, const float* kappa, int n_cand,
                                      float theta_cf, float* out, cudaStream_t s) {
  if (n_cand <= 0) return cudaSuccess;
  lscv_h_skip_select_kernel<<<(unsigned)n_cand, 256, 0, s>>>(X0, n, T, kappa, theta_cf, out);
  return cudaGetLastError();
}

}  // namespace kde
