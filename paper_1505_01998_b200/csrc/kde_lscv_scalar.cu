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

}  // namespace kde
