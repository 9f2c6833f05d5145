// kde_internal.h — declarations shared by the host library (kde_host.cpp) and the CUDA
// launchers (kde_kernels.cu).  Product code only; nothing here is shared with oracle/.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace kde {

constexpr int kThreads = 256;          // threads per CTA of every pair kernel
constexpr int kMaxCand = 32;           // candidates per pair-kernel launch (upper bound)
constexpr int kMaxDim = 16;

// Fixed-point limbs of one output value on the device: value*2^S = hi*2^80 + mid*2^40 +
// (unsigned) lo + carry*2^64.  Every tile commit adds |hi|, |mid|, |lo| < 2^40 (sign-magnitude
// split); hi and mid stay far from overflow because the a-priori bound caps the sum of |commits|
// at 2^100, and lo's unsigned wrap-arounds are counted in the carry limb (add_limbs), so the
// value is exact for any number of commits (n up to 2^31).  Readers fold the carry; before a
// cross-rank sum each rank's limbs are normalised (normalize_limbs) so the int64 sums cannot wrap.
constexpr int kLimbs = 4;
constexpr int kMaxDevices = 64;   // per-device caches of one-time kernel setup

// Current CUDA device (per-device caches: the dynamic shared-memory opt-in is a device attribute).
inline int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d < 0 || d >= kMaxDevices ? 0 : d;
}

// Which functor a launch runs.
enum class Kind : int { Psi4 = 4, Psi6 = 6, Psi8 = 8, LscvScalar = 1, LscvMatrix = 2 };

// Per-launch parameters (copied into the kernel parameter space = constant bank).
struct PsiParams {
  // He_r coefficients are compile-time; see FPsi (kde_pair.cuh) for the exponent scheme.
  double fac[16];    // 2^((r-1) c0 - o_k), exact in fp64 (applied at the fp64 flush)
  float o[16];       // class k = 8 * (tile parity) + row slot: o_k = fp32((r-1) c0 - 16 - k/16); aligned pairs
  float c0;          // fp32(-log2(e)/2): exp(-s/2) = 2^(s c0)
};
struct LscvScalarParams {
  float kappa[kMaxCand];   // -1/h_c^2 (data pre-scaled by sqrt(log2 e / 4) L^-1)
};
struct LaunchCfg {
  const float* X;          // D rows of ld floats (fp32, prepared), device
  int64_t n, ld;           // samples, padded row length (multiple of the tile)
  int64_t tile_begin, tile_end;
  int tile;                // tile edge T (rows = columns)
  int scale_exp;           // fixed-point exponent S
  unsigned long long* limbs;   // [n_out][3] accumulators, device
  int n_out;               // outputs written per data set by this launch
  cudaStream_t stream;
  int sm_count;
  const unsigned long long* clamp = nullptr;   // Psi: device flag "some |x'| > 3e4"
  // Several prepared data sets (LSCV_H: one per candidate) in one launch: set s lives at
  // X + s * set_stride and writes outputs [s * n_out, (s + 1) * n_out); work unit = (set, tile).
  int n_sets = 1;
  int64_t set_stride = 0;  // floats
};

// Launchers (kde_psi.cu, kde_lscv_scalar.cu, kde_lscv_matrix.cu).  Return cudaSuccess or the launch error.
cudaError_t launch_psi(int r, const LaunchCfg& c, const PsiParams& p);
cudaError_t prepare_psi(int r, const LaunchCfg& c);   // one-time setup of launch_psi's kernel
// fp64-term Psi mode (kde_set_precision): y = (x - mean[0]) * w[0] in fp64, then 256-tiles of fp64 terms.
constexpr int kPsi64Tile = 256;
cudaError_t launch_scale64(const double* x, int64_t n, const double* mean_dev, const double* w_dev, double* y,
                           cudaStream_t s);
cudaError_t launch_psi64(int r, const double* y, int64_t n, int64_t tile_begin, int64_t tile_end, int S,
                         unsigned long long* limbs, int sm_count, cudaStream_t s);
cudaError_t launch_lscv_scalar(int d, int nb, const LaunchCfg& c, const LscvScalarParams& p);
// LSCV_H with per-candidate whitened data (one candidate per set, c.n_sets sets).
cudaError_t launch_lscv_white(int d, const LaunchCfg& c);
int tile_for(Kind k, int d, int64_t n);       // tile edge the launcher uses
int cand_per_launch(Kind k, int d);           // B

// O(n) kernels.
cudaError_t launch_moments1(const double* X, int64_t n, int d, double* part, int nblk,
                            cudaStream_t s);
cudaError_t launch_moments2(const double* X, int64_t n, int d, const double* mean_dev,
                            double* part, int nblk, cudaStream_t s);
cudaError_t launch_reduce_parts(const double* part, int nblk, int width, double* out,
                                cudaStream_t s);
struct PrepParams {
  double W[kMaxDim * kMaxDim];   // row-major d x d
  double mean[kMaxDim];
};
cudaError_t launch_prep_params(const double* X, int64_t n, int d, const PrepParams& pp, float* Y, int64_t ld,
                               cudaStream_t s, float pad = 0.f, unsigned long long* overflow_flag = nullptr,
                               double clamp_thresh = 0.0);
cudaError_t launch_prep(const double* X, int64_t n, int d, const double* W_dev,
                        const double* mean_dev, float* Y, int64_t ld, cudaStream_t s,
                        float pad = 0.f, unsigned long long* overflow_flag = nullptr,
                        double clamp_thresh = 0.0);

// Device-resident PLUGIN chain (kde_psi.cu).  Layout of the workspace's `small` block (doubles):
// mean[16] | W[256] | sums[136] | flags (2 x u64) | trace[8] | status.
struct PluginDev {
  double *mean, *W, *sums, *trace, *status;
  __host__ __device__ explicit PluginDev(double* small)
      : mean(small), W(small + 16), sums(small + 272), trace(small + 410), status(small + 418) {}
};
constexpr int kSmallDoubles = 424;
cudaError_t launch_plugin_chain(int stage, int64_t n, double* small, const unsigned long long* limbs, int S,
                                cudaStream_t s);

// KDE evaluation on an m x n rectangle (kde_eval.cu).
struct EvalLaunch {
  const float* Y;        // D x ldm whitened queries
  const float* X;        // D x ldn whitened samples, padded with +inf
  int64_t m, ldm, ldn;   // ldm multiple of eval_rows_per_block(), ldn of eval_cols_per_tile()
  double* part;          // scratch [splits][ldm]
  size_t part_capacity;  // doubles available in part
  double scale;          // n^-1 (2 pi)^{-d/2} |H|^{-1/2}
  double* out;           // m results (device)
  cudaStream_t stream;
  int sm_count;
};
cudaError_t launch_eval(int d, const EvalLaunch& c);
int eval_rows_per_block();
int eval_cols_per_tile();
// Column splits eval_kernel<d> uses for an m x n problem (the launch and the host's scratch
// sizing share this): scratch = splits * ldm doubles.
cudaError_t eval_splits(int d, int sm_count, int64_t ldm, int64_t ldn, int* splits);
// The paper's two-phase LSCV_h (kde_materialized.cu).
int mat_tile();
int64_t mat_chunk();
cudaError_t launch_mat_write(int d, const float* X, int64_t n, int64_t ld, int64_t tb, int64_t te, float* buf,
                             int sm_count, cudaStream_t s);
cudaError_t launch_mat_reduce(int B, const float* buf, int64_t nvalues, const LscvScalarParams& p, int S,
                              unsigned long long* limbs, int sm_count, cudaStream_t s);
// Univariate AQP closed forms (kde_eval.cu): out[2q] = COUNT, out[2q+1] = SUM.
int aqp_blocks(int64_t n);
cudaError_t launch_aqp(const double* x, int64_t n, double h, const double* lo, const double* hi, int nq,
                       double* part, int nblk, double* out, cudaStream_t s);
int moments_blocks(int64_t n);
size_t sort_temp_bytes(int64_t n);
// Canonical form of `count` outputs' limbs (hi, mid in [0,2^40), lo in [0,2^40), carry 0) so
// that a sum over ranks of int64 limbs cannot wrap.
cudaError_t launch_normalize_limbs(unsigned long long* limbs, int count, cudaStream_t s);
cudaError_t launch_sort(const double* in, double* out, int64_t n, void* temp, size_t temp_bytes,
                        cudaStream_t s);

// Host/device tile map (Eq. 42-43 + integer fix-up).
void tile_coords_host(int64_t bx, int64_t* l, int64_t* q);

}  // namespace kde
