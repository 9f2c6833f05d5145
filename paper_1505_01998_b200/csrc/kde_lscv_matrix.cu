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

}  // namespace kde
