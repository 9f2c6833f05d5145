// kde_lscv_matrix.cu — LSCV_H pair-kernel instantiations (see kde_pair.cuh).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "kde_pair.cuh"

namespace kde {

template <int D, int NT>
static cudaError_t lscv_mono_dt(int nb, const LaunchCfg& c, const LscvMatrixParams& p) {
  if (nb <= 1) return launch_pair<FLscvMono<D, NT, 1>>(c, p);   // serial Nelder-Mead steps
  if (nb <= 2) return launch_pair<FLscvMono<D, NT, 2>>(c, p);
  if (nb <= 4) return launch_pair<FLscvMono<D, NT, 4>>(c, p);
  if (nb <= 8) return launch_pair<FLscvMono<D, NT, 8>>(c, p);
  return launch_pair<FLscvMono<D, NT, 16>>(c, p);
}

template <int D>
static cudaError_t lscv_mono_d(int nb, const LaunchCfg& c, const void* params) {
  const auto& p = *static_cast<const LscvMatrixParams*>(params);
  return c.tile == 256 ? lscv_mono_dt<D, 128>(nb, c, p) : lscv_mono_dt<D, 256>(nb, c, p);
}

template <int D>
static cudaError_t lscv_chol_d(const LaunchCfg& c, const void* params) {
  const auto& p = *static_cast<const LscvCholParams*>(params);
  constexpr int NB = nb_chol(D);
  static_assert(NB * D * (D + 1) / 2 <= 4 * 136, "chol params");
  return launch_pair<FLscvChol<D, NB>>(c, p);
}

cudaError_t launch_lscv_matrix(int d, int nb, const LaunchCfg& c, const void* params,
                               size_t bytes) {
  (void)bytes;
  switch (d) {
    case 1: return lscv_mono_d<1>(nb, c, params);
    case 2: return lscv_mono_d<2>(nb, c, params);
    case 3: return lscv_mono_d<3>(nb, c, params);
    case 4: return lscv_mono_d<4>(nb, c, params);
    case 5: return lscv_chol_d<5>(c, params);   case 6: return lscv_chol_d<6>(c, params);
    case 7: return lscv_chol_d<7>(c, params);   case 8: return lscv_chol_d<8>(c, params);
    case 9: return lscv_chol_d<9>(c, params);   case 10: return lscv_chol_d<10>(c, params);
    case 11: return lscv_chol_d<11>(c, params); case 12: return lscv_chol_d<12>(c, params);
    case 13: return lscv_chol_d<13>(c, params); case 14: return lscv_chol_d<14>(c, params);
    case 15: return lscv_chol_d<15>(c, params); case 16: return lscv_chol_d<16>(c, params);
  }
  return cudaErrorInvalidValue;
}

}  // namespace kde
