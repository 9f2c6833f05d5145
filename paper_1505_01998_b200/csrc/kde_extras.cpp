// kde_extras.cpp — off-selector uses of the pair engine: KDE evaluation f(y; H) and the AQP
// closed forms (row f2), and the paper's two-phase materialised LSCV_h (row f3,
// P:606-696).  P:NNN = PAPER.md line NNN.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "kde_host.h"

using kde::Kind;
using namespace kde::host;

extern "C" {

kde_status kde_evaluate(kde_ctx* c, const double* X, int64_t n, int32_t d, const double* Y, int64_t m,
                        const double* vh, double* f) {
  TRY(check_ctx(c));
  prof_reset(c);
  TRY(validate_X(c, X, n, d, 1));
  if (!Y || !vh || !f || m < 0) return fail(c, KDE_E_INVALID, "null query/bandwidth/output pointer");
  if (m == 0) return KDE_OK;
  if (m > 2147483647LL) return fail(c, KDE_E_INVALID, "m > 2^31-1");
  TRY(stage_input(c, Y, (size_t)m * (size_t)d, 1));
  std::vector<double> H = unvech(vh, d), L;
  if (!cholesky(H, d, L)) return fail(c, KDE_E_NONPOSITIVE_BW, "bandwidth matrix is not positive definite");
  double det = 1.0;
  for (int i = 0; i < d; ++i) det *= L[i * d + i] * L[i * d + i];
  // W^T W = (log2 e / 2) H^-1  =>  2^-|W v|^2 = exp(-v^T H^-1 v / 2)
  std::vector<double> W = tri_lower_inverse(L, d);
  for (double& v : W) v *= std::sqrt(kLog2e / 2.0);
  const int64_t R = kde::eval_rows_per_block(), TC = kde::eval_cols_per_tile();
  const int64_t ldm = (m + R - 1) / R * R, ldn = (n + TC - 1) / TC * TC;
  int splits = 1;
  CUDA_TRY(c, kde::eval_splits(d, c->sm_count, ldm, ldn, &splits));
  const size_t parts = (size_t)splits * (size_t)ldm;
  // bounded far-tile skip: samples and queries sorted by coordinate 0; a sample tile
  // whose coordinate-0 gap to a query block has gap^2 > log2 n + 42 is skipped (every term <= 2^-gap^2):
  // at most n terms of 2^-(log2 n + 42) each move fhat by <= 2^-42 n^-1 sum ... = 2.3e-13 (2 pi)^{-d/2}
  // |H|^{-1/2}, which is <= 2.3e-13 of max fhat (fhat at any sample point is at least that scale).
  const char* e_nos = getenv("KDE_DEBUG_EVAL_NOSKIP");   // A/B and tests: read at every call
  // (worth its two sorts from about 2^32 pairs on: below that the launch is a fraction of a millisecond)
  const bool skip = kde::skip_bounded() && !(e_nos && atoi(e_nos) == 1) && (double)m * (double)n >= 4294967296.0;
  const size_t sort_tmp = skip ? kde::sort_rows_temp_bytes(m) : 0;
  const size_t need = align256((size_t)d * ldm * 4) + align256((size_t)d * ldn * 4) + align256(parts * 8) +
                      align256((size_t)m * 8) +
                      (skip ? align256((size_t)m * d * 8) + align256((size_t)m * 8) + align256((size_t)2 * m * 4) +
                                  align256((size_t)2 * (ldm / R) * 4) + align256(sort_tmp)
                            : 0);
  TRY(grow(c, &c->ev_ws, &c->ev_bytes, need));
  char* p = (char*)c->ev_ws;
  float* Yw = (float*)p; p += align256((size_t)d * ldm * 4);
  float* Xw = (float*)p; p += align256((size_t)d * ldn * 4);
  double* part = (double*)p; p += align256(parts * 8);
  double* out = (double*)p; p += align256((size_t)m * 8);
  const int* perm = nullptr;
  int* range = nullptr;
  if (skip) {
    range = (int*)p; p += align256((size_t)2 * (ldm / R) * 4);
    double* ys = (double*)p; p += align256((size_t)m * d * 8);
    double* keys = (double*)p; p += align256((size_t)m * 8);
    int* idx = (int*)p; p += align256((size_t)2 * m * 4);
    CUDA_TRY(c, kde::launch_sort_rows(Y, m, d, ys, keys, idx, p, sort_tmp, c->stream));
    c->prof_all += 12;
    Y = ys;
    perm = idx + m;                                 // sorted query q = the caller's query perm[q]
    TRY(gpu_sorted_rows(c, X, n, d, &X));           // samples by coordinate 0 (context-owned copy)
  }
  Ws w;
  TRY(get_ws(c, 256, d, 2, &w));
  // centre both sets on the sample mean (fp32 accuracy of the differences)
  const int nblk = kde::moments_blocks(n);
  double* sums = w.small + 16 + 256;
  double hs[16];
  CUDA_TRY(c, kde::launch_moments1(X, n, d, w.part, nblk, c->stream));
  CUDA_TRY(c, kde::launch_reduce_parts(w.part, nblk, d, sums, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(hs, sums, d * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  std::vector<double> mean(d);
  for (int a = 0; a < d; ++a) {
    if (!std::isfinite(hs[a])) return fail(c, KDE_E_INVALID, "non-finite sample values");
    mean[a] = hs[a] / (double)n;
  }
  kde::PrepParams pp;
  std::copy(W.begin(), W.begin() + (size_t)d * d, pp.W);
  std::copy(mean.begin(), mean.begin() + d, pp.mean);
  CUDA_TRY(c, cudaMemsetAsync(w.flag(), 0, sizeof(unsigned long long), c->stream));
  CUDA_TRY(c, kde::launch_prep_params(X, n, d, pp, Xw, ldn, c->stream, int_as_float_host(0x7f800000), w.flag()));
  CUDA_TRY(c, kde::launch_prep_params(Y, m, d, pp, Yw, ldm, c->stream, 0.f, w.flag()));
  kde::EvalLaunch el;
  el.Y = Yw; el.X = Xw; el.m = m; el.ldm = ldm; el.ldn = ldn; el.part = part; el.part_capacity = parts;
  el.scale = std::pow(2.0 * kPi, -0.5 * d) / std::sqrt(det) / (double)n;
  el.out = out; el.stream = c->stream; el.sm_count = c->sm_count;
  el.n = n; el.perm = perm; el.range = range;
  el.skip_s = skip ? (float)(std::log2((double)std::max<int64_t>(n, 2)) + 42.0) : __builtin_inff();
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (c->profiling) { e0 = next_event(c); e1 = next_event(c); cudaEventRecord(e0, c->stream); }
  c->prof_all += 1 + 2 + 2 + 2;   // moments1 + reduce, 2 x prep, eval + reduce
  cudaError_t err = kde::launch_eval(d, el);
  if (err != cudaSuccess) return fail(c, KDE_E_CUDA, "eval launch: %s", cudaGetErrorString(err));
  if (c->profiling) {
    cudaEventRecord(e1, c->stream);
    c->prof_launches++;
    c->prof_evals += (double)m * (double)n;
  }
  std::vector<double> tmp(m);
  CUDA_TRY(c, cudaMemcpyAsync(tmp.data(), out, (size_t)m * 8, cudaMemcpyDeviceToHost, c->stream));
  unsigned long long overflow = 0;
  CUDA_TRY(c, cudaMemcpyAsync(&overflow, w.flag(), sizeof(overflow), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  if (overflow) return fail(c, KDE_E_INVALID, "whitened sample/query values exceed 1e18");
  TRY(prof_collect(c));
  std::copy(tmp.begin(), tmp.end(), f);
  return KDE_OK;
}

kde_status kde_aqp_1d(kde_ctx* c, const double* x, int64_t n, double h, const double* lo, const double* hi,
                      int32_t nq, double* count, double* sum, double* avg) {
  TRY(check_ctx(c));
  prof_reset(c);
  TRY(validate_X(c, x, n, 1, 1));
  if (!lo || !hi || nq < 1) return fail(c, KDE_E_INVALID, "null interval arrays");
  if (!(h > 0.0) || !std::isfinite(h)) return fail(c, KDE_E_NONPOSITIVE_BW, "h <= 0");
  for (int q = 0; q < nq; ++q)
    if (!(lo[q] <= hi[q])) return fail(c, KDE_E_INVALID, "interval %d has lo > hi or NaN", q);
  const int nblk = kde::aqp_blocks(n);
  const size_t need = align256((size_t)nq * nblk * 2 * 8) + 3 * align256((size_t)nq * 2 * 8);
  TRY(grow(c, &c->ev_ws, &c->ev_bytes, need));
  char* p = (char*)c->ev_ws;
  double* part = (double*)p; p += align256((size_t)nq * nblk * 2 * 8);
  double* dlo = (double*)p; p += align256((size_t)nq * 2 * 8);
  double* dhi = (double*)p; p += align256((size_t)nq * 2 * 8);
  double* out = (double*)p;
  CUDA_TRY(c, cudaMemcpyAsync(dlo, lo, nq * 8, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(dhi, hi, nq * 8, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, kde::launch_aqp(x, n, h, dlo, dhi, nq, part, nblk, out, c->stream));
  c->prof_all += 2;
  std::vector<double> tmp((size_t)nq * 2);
  CUDA_TRY(c, cudaMemcpyAsync(tmp.data(), out, (size_t)nq * 16, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  for (int q = 0; q < nq; ++q) {
    if (count) count[q] = tmp[2 * q];
    if (sum) sum[q] = tmp[2 * q + 1];
    if (avg) avg[q] = tmp[2 * q + 1] / tmp[2 * q];
  }
  return KDE_OK;
}

kde_status kde_lscv_h_scores_materialized(kde_ctx* c, const double* X, int64_t n, int32_t d, const double* h,
                                          int32_t nh, int32_t h_per_pass, double* g) {
  TRY(check_ctx(c));
  prof_reset(c);
  TRY(validate_X(c, X, n, d, 2));
  if (!h || !g || nh < 1) return fail(c, KDE_E_INVALID, "null candidate/output array");
  if (!(h_per_pass == 1 || h_per_pass == 2 || h_per_pass == 4 || h_per_pass == 8 || h_per_pass == 16))
    return fail(c, KDE_E_INVALID, "h_per_pass must be 1, 2, 4, 8 or 16");
  for (int k = 0; k < nh; ++k)
    if (!(h[k] > 0.0) || !std::isfinite(h[k])) return fail(c, KDE_E_NONPOSITIVE_BW, "h[%d] <= 0", k);
  const int T = kde::mat_tile();
  const int64_t ld = (n + T - 1) / T * T;
  const int B = h_per_pass;
  const int nbatch = (nh + B - 1) / B;
  const int n_out = 2 * nbatch * B;
  Ws w;
  TRY(get_ws(c, ld, d, n_out, &w));
  Moments m;
  TRY(gpu_moments(c, X, n, d, w, m));
  LscvhPrep pp;
  TRY(lscv_h_prepare(c, m, d, pp));
  std::vector<double> W = tri_lower_inverse(pp.Lc, d);
  for (double& v : W) v *= std::sqrt(kLog2e / 4.0);
  TRY(gpu_prep(c, X, n, d, W, m.mean, ld, w));
  int64_t tb, te;
  shard_range(n_tiles(n, T), c->rank, c->world, &tb, &te);
  const int64_t nvalues = (te - tb) * (int64_t)T * T;
  TRY(grow(c, &c->mat_ws, &c->mat_bytes, (size_t)std::max<int64_t>(nvalues, 1) * sizeof(float)));
  float* buf = (float*)c->mat_ws;
  cudaEvent_t a0 = nullptr, a1 = nullptr;
  if (c->profiling) { a0 = next_event(c); a1 = next_event(c); cudaEventRecord(a0, c->stream); }
  CUDA_TRY(c, kde::launch_mat_write(d, w.Y, n, ld, tb, te, buf, c->sm_count, c->stream, c->rank, c->world));   // phase 1
  c->prof_all += 1;
  if (c->profiling) cudaEventRecord(a1, c->stream);
  CUDA_TRY(c, cudaMemsetAsync(w.limbs, 0, (size_t)n_out * kde::kLimbs * sizeof(long long), c->stream));
  const int S = scale_exp_for(1.0, n);
  const double pairs = c->profiling ? pairs_in_shard(n, T, te, c->rank, c->world) : 0.0;
  for (int b = 0; b < nbatch; ++b) {                                                          // phase 2
    kde::LscvScalarParams p;
    for (int j = 0; j < kde::kMaxCand; ++j) {
      const int idx = std::min(b * B + j, nh - 1);
      p.kappa[j] = (float)(-1.0 / (h[idx] * h[idx]));
      p.smax[j] = (float)(125.0 / -(double)p.kappa[j]);
    }
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (c->profiling) { e0 = next_event(c); e1 = next_event(c); cudaEventRecord(e0, c->stream); }
    CUDA_TRY(c, kde::launch_mat_reduce(B, buf, nvalues, p, S, w.limbs + (size_t)2 * b * B * kde::kLimbs,
                                       c->sm_count, c->stream));
    c->prof_all += 1;
    if (c->profiling) {
      cudaEventRecord(e1, c->stream);
      c->prof_launches++;
      c->prof_evals += pairs * B;
    }
  }
  TRY(allreduce_limbs(c, w.limbs, (size_t)n_out * kde::kLimbs));
  std::vector<long long> hl((size_t)n_out * kde::kLimbs);
  CUDA_TRY(c, cudaMemcpyAsync(hl.data(), w.limbs, hl.size() * sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
  unsigned long long overflow = 0;
  CUDA_TRY(c, cudaMemcpyAsync(&overflow, w.flag(), sizeof(overflow), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  if (overflow) return fail(c, KDE_E_INVALID, "scaled sample differences exceed 1e18");
  if (c->profiling) {
    float x = 0.f;
    cudaEventElapsedTime(&x, a0, a1);
    c->prof_aux_ms = x;
    double ms = 0.0;
    for (size_t k = 2; k + 1 < c->ev_used; k += 2) {
      CUDA_TRY(c, cudaEventElapsedTime(&x, c->ev_pool[k], c->ev_pool[k + 1]));
      ms += x;
    }
    c->prof_ms = ms;
  }
  for (int k = 0; k < nh; ++k) {
    const double S1 = fixed_value(limbs_to_fixed(&hl[(size_t)2 * k * kde::kLimbs], S));
    const double S2 = fixed_value(limbs_to_fixed(&hl[(size_t)(2 * k + 1) * kde::kLimbs], S));
    g[k] = lscv_h_finalize(n, d, pp.det, h[k], S1, S2);
  }
  return KDE_OK;
}

}  // extern "C"
