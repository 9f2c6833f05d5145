// kde_selectors.cpp — the three bandwidth selectors of Sec. 4.4 on top of the pair
// kernels: Psi_r sums and the device-resident PLUGIN chain (Eq. 11-18), LSCV_h (Eq. 19-28) and
// LSCV_H (Eq. 29-35) with Nelder–Mead; ABI calls kde_psi_r, kde_plugin_h, kde_lscv_h_scores,
// kde_lscv_H_scores, kde_raw_sums, kde_select_bandwidth.  P:NNN = PAPER.md line NNN.
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
#include "kde_nm.cuh"

using kde::Kind;
using namespace kde::host;

namespace kde {
namespace host {

// ------------------------------------------------------------------ Psi_r
// The kernel evaluates He_r in t = u^2 - (r-1) with exact integer coefficients; the parameters
// are the exponent scale c0 and, per accumulator class k, the MUFU offset o_k and the exact
// fp64 factor that undoes it: 2^(u^2 c0) = 2^(t c0 + o_k) * 2^((r-1) c0 - o_k).
void psi_coeffs(int r, kde::PsiParams& p) {
  std::memset(&p, 0, sizeof(p));
  p.c0 = (float)(-kLog2e / 2.0);
  const double Kc0 = (double)(r == 8 ? 0 : r - 1) * (double)p.c0;   // K of FPsi; exact in fp64
  for (int k = 0; k < 16; ++k) {   // k = 8 * (tile parity) + row slot; shift (row slot)/8 + parity/16
    p.o[k] = (float)(Kc0 - (16.0 + (k % 8) / 8.0 + (k / 8) / 16.0));
    p.fac[k] = std::exp2(Kc0 - (double)p.o[k]);                    // exponent exact in fp64
  }
}

double he_at_zero(int r) { return r == 4 ? 3.0 : (r == 6 ? -15.0 : 105.0); }

Kind psi_kind(int r) { return r == 4 ? Kind::Psi4 : (r == 6 ? Kind::Psi6 : Kind::Psi8); }

// Psi workspace: Yc (fp32 tile-centred columns, ld) | Y64 (fp64 scaled samples, ld) | centres
// (ld / T): get_ws with d = 4 rows of ld floats.
struct PsiBufs {
  float* Yc;
  double* Y64;
  float* centres;
};
PsiBufs psi_bufs(const Ws& w, int64_t ld) {
  return PsiBufs{w.Y, reinterpret_cast<double*>(w.Y + ld), w.Y + 3 * ld};
}

// Cancellation of an fp32-term Psi pass as seen by Psi-hat: kappa = 2A / |2S + n He_r(0)| with
// S = sum t and A ~ sum |t| (the kernel's group-level estimate); Psi-hat's error is ~kappa times
// the terms' systematic error.
double psi_kappa(int r, int64_t n, double S, double A) {
  return 2.0 * A / std::fabs(2.0 * S + (double)n * he_at_zero(r));
}

// One fp64-term Psi_r pass over this rank's 256-tiles of Y64 into `limbs`, then the all-reduce.
// gate != null (PLUGIN chain): the kernel runs only if the device decided so; its profiling events
// are kept aside (slot) and counted after the chain if it ran.
kde_status psi64_pass(kde_ctx* c, int r, const double* y, int64_t n, int S, unsigned long long* limbs,
                      const unsigned long long* gate = nullptr, int slot = -1) {
  Range rr("kde.pair_pass_fp64");
  int64_t tb, te;
  shard_range(n_tiles(n, kde::kPsi64Tile), c->rank, c->world, &tb, &te);
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  const unsigned rec = (c->cap_stream && c->stream == c->cap_stream) ? cudaEventRecordExternal : cudaEventRecordDefault;
  if (c->profiling) {
    if (gate) c->gate_pair[slot] = (int)(c->ev_used / 2);
    e0 = next_event(c); e1 = next_event(c);
    CUDA_TRY(c, cudaEventRecordWithFlags(e0, c->stream, rec));
  }
  CUDA_TRY(c, kde::launch_psi64(r, y, n, tb, te, S, limbs, c->sm_count, c->stream, gate, kde::psi_skip_gap(true),
                                c->rank, c->world));
  if (tb < te) c->prof_all += 1;
  if (c->profiling) {
    CUDA_TRY(c, cudaEventRecordWithFlags(e1, c->stream, rec));
    const double pairs = pairs_in_shard(n, kde::kPsi64Tile, te, c->rank, c->world);
    if (gate) {
      c->gate_evals[slot] = pairs;
    } else {
      c->prof_launches++;
      c->prof_evals += pairs;
    }
  }
  TRY(allreduce_limbs(c, limbs, kde::kLimbs));
  return KDE_OK;
}

// Raw Psi sums S_r(g) = sum_{i<j} He_r(u) e^{-u^2/2} for each g: sort once, then per g the prep
// (fp64 y, tile centres, centred fp32 columns) and the fp32-term pass, whose cancellation
// estimate decides (psi_mode 0, full sums only) whether the pass is re-run with fp64 terms;
// psi_mode 1 runs fp64 terms only, -1 fp32 terms only.
kde_status psi_raw(kde_ctx* c, const double* x, int64_t n, int r, const double* g, int ng,
                   const Moments& m, int shard_rank, int shard_world, bool allreduce,
                   std::vector<kde_fixed>& out, bool presorted = false) {
  const int T = kde::tile_for(psi_kind(r), 1, n);
  const int64_t ld = (n + T - 1) / T * T;
  Ws w;
  TRY(get_ws(c, ld, 4, 2, &w));
  const PsiBufs b = psi_bufs(w, ld);
  const int S = scale_exp_for(2.0 * std::fabs(he_at_zero(r)), n);
  if (!presorted) {
    const double* xs = nullptr;
    TRY(gpu_sorted(c, x, n, &xs));
    x = xs;
  }
  out.clear();
  for (int k = 0; k < ng; ++k) {
    const double hv[2] = {m.mean[0], 1.0 / g[k]};
    CUDA_TRY(c, cudaMemcpyAsync(w.small, hv, sizeof(hv), cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(c, cudaMemsetAsync(w.flag(), 0, (kde::kSmallDoubles - 408) * sizeof(double), c->stream));
    CUDA_TRY(c, kde::launch_psi_prep(x, n, w.small, w.small + 1, T, b.Y64, b.Yc, b.centres, ld, c->stream,
                                     w.flag(), 3.0e4));
    c->prof_all += 1;
    if (c->psi_mode != 1) {
      SumLaunch L;
      L.kind = psi_kind(r); L.r = r; L.nb = 1; L.out_offset = 0; L.n_out = 2;
      L.X = b.Yc; L.Y64 = b.Y64; L.centres = b.centres;
      L.skipped = reinterpret_cast<unsigned long long*>(w.small + kde::kSkippedSlot);
      const double var = m.cov.empty() ? 0.0 : m.cov[0];
      L.skip_gap = kde::psi_skip_gap_for(r, g[k], var);
      const bool select = L.skip_gap < INFINITY && kde::skip_bounded() && (n + T - 1) / T >= kde::kGapSelectMinTiles;
      if (select) {   // data-aware threshold on the device, read by the pass
        CUDA_TRY(c, kde::launch_psi_gap_select(r, b.Y64, n, T, nullptr, g[k], nullptr, var, w.small + kde::kGapSlot,
                                               w.part, c->stream));
        c->prof_all += 2;
        L.skip_gap_dev = w.small + kde::kGapSlot;
      }
      psi_coeffs(r, L.psi);
      std::vector<kde_fixed> o;
      TRY(run_sums(c, 1, n, ld, T, S, w, {L}, 2, shard_rank, shard_world, allreduce, o));
      {   // run_sums copied the small block's tail (prep flags .. limbs) to the host
        double gap = L.skip_gap;
        if (L.skip_gap_dev) std::memcpy(&gap, c->h_limbs + (kde::kGapSlot - 408), sizeof(gap));
        c->psi_gaps.push_back(gap);
      }
      if (c->profiling) {   // run_sums copied the small block's tail with the limbs
        unsigned long long sk = 0;
        std::memcpy(&sk, c->h_limbs + (kde::kSkippedSlot - 408), sizeof(sk));
        c->prof_evals -= (double)sk;
      }
      const double kappa = psi_kappa(r, n, fixed_value(o[0]), fixed_value(o[1]));
      if (allreduce) c->psi_kappa_max = std::max(c->psi_kappa_max, kappa);
      const bool escalate = allreduce && c->psi_mode == 0 && !(kappa <= kde::kPsiKappaMax);
      if (!escalate) {
        out.push_back(o[0]);
        continue;
      }
      c->psi_escalations++;
    }
    CUDA_TRY(c, cudaMemsetAsync(w.limbs, 0, kde::kLimbs * sizeof(long long), c->stream));
    if (allreduce) {
      TRY(psi64_pass(c, r, b.Y64, n, S, w.limbs));
    } else {                         // one shard, no collective
      int64_t tb, te;
      shard_range(n_tiles(n, kde::kPsi64Tile), shard_rank, shard_world, &tb, &te);
      CUDA_TRY(c, kde::launch_psi64(r, b.Y64, n, tb, te, S, w.limbs, c->sm_count, c->stream, nullptr,
                                    kde::psi_skip_gap(true), shard_rank, shard_world));
      if (tb < te) c->prof_all += 1;
    }
    long long hl[2 + kde::kLimbs];   // prep flags, then the limbs
    CUDA_TRY(c, cudaMemcpyAsync(hl, w.flag(), 2 * sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaMemcpyAsync(hl + 2, w.limbs, kde::kLimbs * sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    if (hl[0]) return fail(c, KDE_E_INVALID, "scaled sample differences exceed 1e18 (outliers vs. bandwidth)");
    out.push_back(limbs_to_fixed(hl + 2, S));
  }
  return KDE_OK;
}

double psi_finalize(int r, int64_t n, double g, double S) {
  const double s2p = std::sqrt(2.0 * kPi);
  const double nn = (double)n;
  return (2.0 * S / s2p + nn * he_at_zero(r) / s2p) / (nn * nn * std::pow(g, r + 1));
}

// ------------------------------------------------------------------ LSCV_h

kde_status lscv_h_prepare(kde_ctx* c, const Moments& m, int d, LscvhPrep& p) {
  if (!cholesky(m.cov, d, p.Lc)) return fail(c, KDE_E_SINGULAR_COV, "covariance matrix is not positive definite");
  p.det = 1.0;
  for (int i = 0; i < d; ++i) p.det *= p.Lc[i * d + i] * p.Lc[i * d + i];
  if (!(p.det > 0.0) || !std::isfinite(p.det)) return fail(c, KDE_E_SINGULAR_COV, "det(Sigma) <= 0");
  return KDE_OK;
}

kde_status lscv_h_raw(kde_ctx* c, const double* X, int64_t n, int d, const double* h, int nh,
                      const Moments& m, const LscvhPrep& pp, int shard_rank, int shard_world,
                      bool allreduce, std::vector<kde_fixed>& out) {
  const int T = kde::tile_for(Kind::LscvScalar, d, n);
  const int nb = kde::cand_per_launch(Kind::LscvScalar, d);
  const int64_t ld = (n + T - 1) / T * T;
  const int nbatch = (nh + nb - 1) / nb;
  const int n_out = 2 * nbatch * nb;
  Ws w;
  TRY(get_ws(c, ld, d, n_out, &w));
  // sorted by coordinate 0 (the whitened coordinate 0 keeps that order): far tiles are skipped
  TRY(gpu_sorted_rows(c, X, n, d, &X));
  // W = sqrt(log2 e / 4) L^-1  =>  |W v|^2 = (log2 e / 4) v^T Sigma^-1 v
  std::vector<double> W = tri_lower_inverse(pp.Lc, d);
  for (double& v : W) v *= std::sqrt(kLog2e / 4.0);
  TRY(gpu_prep(c, X, n, d, W, m.mean, ld, w));
  // batches of ascending h: each batch's widest h sets its far-tile skip bound (a candidate's sums do not
  // depend on its batch, so the order only changes how many tiles are skipped)
  std::vector<int> order(nh);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return h[a] < h[b]; });
  std::vector<SumLaunch> Ls;
  for (int b = 0; b < nbatch; ++b) {
    SumLaunch L;
    L.kind = Kind::LscvScalar; L.nb = nb; L.out_offset = 2 * b * nb; L.n_out = 2 * nb;
    double kmin = 1e300;
    for (int j = 0; j < kde::kMaxCand; ++j) {
      int idx = order[std::min(b * nb + j, nh - 1)];   // pad with a valid candidate
      L.ls.kappa[j] = (float)(-1.0 / (h[idx] * h[idx]));
      L.ls.smax[j] = (float)(125.0 / -(double)L.ls.kappa[j]);
      L.ls.skip_c[j] = lscv_skip_s(-(double)L.ls.kappa[j], n);   // this candidate's own bound
      if (j < nb) kmin = std::min(kmin, -(double)L.ls.kappa[j]);
    }
    L.skip_s = lscv_skip_s(kmin, n);   // the batch's widest h bounds every candidate's terms
    Ls.push_back(L);
  }
  // data-aware bounds: one selection CTA per (padded) candidate, read by the batches
  if (Ls.front().skip_s < __builtin_inff() && kde::skip_bounded() && (n + T - 1) / T >= kde::kGapSelectMinTiles) {
    const size_t cnt = (size_t)nbatch * nb;
    TRY(grow(c, &c->skip_ws, &c->skip_bytes, 2 * cnt * sizeof(float)));
    float* kap_dev = static_cast<float*>(c->skip_ws);
    float* thr_dev = kap_dev + cnt;
    std::vector<float> kap(cnt);
    for (int b = 0; b < nbatch; ++b)
      for (int j = 0; j < nb; ++j) kap[(size_t)b * nb + j] = Ls[b].ls.kappa[j];
    CUDA_TRY(c, cudaMemcpyAsync(kap_dev, kap.data(), cnt * sizeof(float), cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(c, kde::launch_lscv_h_skip_select(w.Y, n, T, kap_dev, (int)cnt, (float)kde_lscv_skip_theta(n), thr_dev,
                                               c->stream));
    c->prof_all += 1;
    for (int b = 0; b < nbatch; ++b) Ls[b].skip_c_dev = thr_dev + (size_t)b * nb;
  }
  std::vector<kde_fixed> o;
  TRY(run_sums(c, d, n, ld, T, scale_exp_for(1.0, n), w, Ls, n_out, shard_rank, shard_world, allreduce, o));
  out.resize(2 * (size_t)nh);
  for (int k = 0; k < nh; ++k) {
    out[2 * (size_t)order[k]] = o[2 * (size_t)k];
    out[2 * (size_t)order[k] + 1] = o[2 * (size_t)k + 1];
  }
  return KDE_OK;
}

double lscv_cancellation(int64_t n, int d, double det, double S1, double S2) {
  const double nn = (double)n;
  const double c4 = std::pow(4.0 * kPi, -0.5 * d) / std::sqrt(det);
  const double c2 = std::pow(2.0 * kPi, -0.5 * d) / std::sqrt(det);
  const double A = 2.0 * c4 * S1 / (nn * nn), B = 4.0 * c2 * S2 / (nn * nn), C = c4 / nn;
  return (A + B) / std::fabs(A - B + C);   // +inf for g = 0
}

kde_status lscv_sums64(kde_ctx* c, const double* Xs, int64_t n, int d, const std::vector<double>& W,
                       const std::vector<double>& mean, double kappa, kde_fixed out[2]) {
  Range r("kde.lscv64");
  const int T = kde::lscv64_tile();
  const int64_t ld = (n + T - 1) / T * T;
  TRY(grow(c, &c->f64_ws, &c->f64_bytes, (size_t)d * ld * sizeof(double)));
  double* Y = static_cast<double*>(c->f64_ws);
  kde::PrepParams pp;
  std::copy(W.begin(), W.begin() + (size_t)d * d, pp.W);
  std::copy(mean.begin(), mean.begin() + d, pp.mean);
  CUDA_TRY(c, kde::launch_prep64(Xs, n, d, pp, Y, ld, c->stream));
  Ws w;
  TRY(get_ws(c, ld, d, 2, &w));
  CUDA_TRY(c, cudaMemsetAsync(w.limbs, 0, 2 * kde::kLimbs * sizeof(long long), c->stream));
  int64_t tb, te;
  shard_range(n_tiles(n, T), c->rank, c->world, &tb, &te);
  const int S = scale_exp_for(1.0, n);
  // exp2(kappa s) is exactly 0 in fp64 for kappa s < -1100 (below the smallest subnormal 2^-1074)
  CUDA_TRY(c, kde::launch_lscv64(d, Y, n, ld, tb, te, kappa, 1100.0 / -kappa, S, w.limbs, c->sm_count, c->stream,
                                 c->rank, c->world));
  c->prof_all += tb < te ? 2 : 1;
  TRY(allreduce_limbs(c, w.limbs, 2 * kde::kLimbs));
  long long hl[2 * kde::kLimbs];
  CUDA_TRY(c, cudaMemcpyAsync(hl, w.limbs, sizeof(hl), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  out[0] = limbs_to_fixed(hl, S);
  out[1] = limbs_to_fixed(hl + kde::kLimbs, S);
  c->psi_escalations++;
  return KDE_OK;
}

double lscv_h_finalize(int64_t n, int d, double det, double h, double S1, double S2) {
  const double nn = (double)n;
  const double c4 = std::pow(4.0 * kPi, -0.5 * d) / std::sqrt(det);
  const double c2 = std::pow(2.0 * kPi, -0.5 * d) / std::sqrt(det);
  return std::pow(h, -d) * (2.0 * (c4 * S1 - 2.0 * c2 * S2) / (nn * nn) + c4 / nn);
}

// ------------------------------------------------------------------ LSCV_H

// PD test, |H| and the whitening W = sqrt(log2 e / 4) L^-1 of one candidate, with the arithmetic the
// device-resident Nelder–Mead uses too (kde_nm.cuh), so both loops prepare identical data sets.
HCand h_candidate(const double* vh, int d) {
  HCand hc;
  double L[kde::kMaxDim * kde::kMaxDim], det = 0.0;
  if (!kde::nm_cholesky_vech(vh, d, L, &det)) return hc;
  hc.pd = true;
  hc.det = det;
  hc.W.assign((size_t)d * d, 0.0);
  kde::nm_whitening(L, d, std::sqrt(kLog2e / 4.0), hc.W.data());
  return hc;
}

// Raw LSCV_H sums for PD candidates `cands` (all must be PD).  Each candidate gets its own
// whitened fp32 copy of the data, x'_c = sqrt(log2 e / 4) L_c^-1 (x - mean) with H_c = L_c L_c^T,
// so that v^T H_c^-1 v = (4 / log2 e) |x'_ci - x'_cj|^2: the pair kernel then needs no quadratic
// form (2d + 2 FP32 ops per eval instead of d(d+1)/2 + 2 per candidate plus the monomials), and
// the sum of squares does not lose accuracy with cond(H).  Candidates are
// independent work units, so a candidate's sums are bit-identical alone or inside any batch.
// data_aware: per-set bounded skip thresholds chosen on the device (launch_lscv_sets_skip_select) —
// scores and raw sums; the Nelder–Mead searches keep the closed form, so host and device loops agree.
kde_status lscv_H_raw(kde_ctx* c, const double* X, int64_t n, int d, const std::vector<HCand>& cands,
                      const Moments& m, int shard_rank, int shard_world, bool allreduce,
                      std::vector<kde_fixed>& out, bool data_aware = false) {
  const int T = kde::tile_for(Kind::LscvMatrix, d, n);
  const int64_t ld = (n + T - 1) / T * T;
  const int64_t set_floats = (int64_t)d * ld;
  const int nc = (int)cands.size();
  // sets per launch: up to 256 candidates within ~1 GiB of prepared data
  const int per_launch = (int)std::max<int64_t>(1, std::min<int64_t>(256, (1LL << 28) / set_floats));
  Ws w;
  TRY(get_ws(c, ld, d, 2 * std::min(nc, per_launch), &w));
  TRY(gpu_sorted_rows(c, X, n, d, &X));   // by coordinate 0 (no-op when X is the sorted copy)
  out.clear();
  for (int b0 = 0; b0 < nc; b0 += per_launch) {
    const int cnt = std::min(per_launch, nc - b0);
    TRY(grow(c, &c->white_ws, &c->white_bytes, (size_t)cnt * set_floats * sizeof(float) + (size_t)cnt * sizeof(float)));
    float* Yw = static_cast<float*>(c->white_ws);
    float* thr = Yw + (size_t)cnt * set_floats;   // per-set skip bounds (data-aware selection)
    // prep flags and this launch's limbs are one contiguous span of the workspace (get_ws): one memset
    const size_t span = (size_t)(reinterpret_cast<char*>(w.limbs + (size_t)2 * cnt * kde::kLimbs + 1) -
                                 reinterpret_cast<char*>(w.flag()));   // + run_sums' one work counter
    CUDA_TRY(c, cudaMemsetAsync(w.flag(), 0, span, c->stream));
    for (int j = 0; j < cnt; ++j)
      TRY(gpu_prep_into(c, X, n, d, cands[b0 + j].W, m.mean, ld, w, Yw + (size_t)j * set_floats));
    SumLaunch L;
    L.kind = Kind::LscvMatrix; L.nb = 1; L.out_offset = 0; L.n_out = 2 * cnt;
    L.X = Yw; L.n_sets = cnt; L.set_stride = set_floats;
    L.skip_s = lscv_skip_s(1.0, n);   // e = 2^-s with s = |x'_i - x'_j|^2
    if (data_aware && L.skip_s < __builtin_inff() && kde::skip_bounded() && (n + T - 1) / T >= kde::kGapSelectMinTiles) {
      CUDA_TRY(c, kde::launch_lscv_sets_skip_select(Yw, set_floats, cnt, n, T, L.skip_s, thr, c->stream));
      c->prof_all += 1;
      L.skip_s_sets = thr;
    }
    std::vector<kde_fixed> o;
    TRY(run_sums(c, d, n, ld, T, scale_exp_for(1.0, n), w, {L}, 2 * cnt, shard_rank, shard_world, allreduce, o,
                 /*limbs_zeroed=*/true));
    out.insert(out.end(), o.begin(), o.end());
  }
  return KDE_OK;
}

double lscv_H_finalize(int64_t n, int d, double det, double S1, double S2) {
  return kde::nm_lscv_H_finalize((double)n, std::pow(4.0 * kPi, -0.5 * d), std::pow(2.0 * kPi, -0.5 * d), det, S1, S2);
}

// Evaluate g(H) for a list of vech vectors (non-PD -> penalty); one GPU batch for all PD ones.
kde_status lscv_H_eval(kde_ctx* c, const double* X, int64_t n, int d, const Moments& m,
                       const std::vector<std::vector<double>>& vs, double penalty,
                       std::vector<double>& g, int* evals, bool auto_precision) {
  std::vector<HCand> pdc;
  std::vector<int> idx;
  g.assign(vs.size(), penalty);
  for (size_t k = 0; k < vs.size(); ++k) {
    HCand hc = h_candidate(vs[k].data(), d);
    if (hc.pd) { pdc.push_back(std::move(hc)); idx.push_back((int)k); }
  }
  if (pdc.empty()) return KDE_OK;
  std::vector<kde_fixed> o;
  TRY(gpu_sorted_rows(c, X, n, d, &X));
  TRY(lscv_H_raw(c, X, n, d, pdc, m, c->rank, c->world, true, o, /*data_aware=*/auto_precision));
  for (size_t j = 0; j < pdc.size(); ++j) {
    double S1 = fixed_value(o[2 * j]), S2 = fixed_value(o[2 * j + 1]);
    // automatic precision (scores calls; Nelder-Mead searches keep fp32 terms, §3.10)
    if (auto_precision && c->psi_mode != -1 &&
        (c->psi_mode == 1 || !(lscv_cancellation(n, d, pdc[j].det, S1, S2) <= kLscvKappaMax))) {
      kde_fixed f[2];
      TRY(lscv_sums64(c, X, n, d, pdc[j].W, m.mean, -1.0, f));
      S1 = fixed_value(f[0]);
      S2 = fixed_value(f[1]);
    }
    g[idx[j]] = lscv_H_finalize(n, d, pdc[j].det, S1, S2);
  }
  if (evals) *evals += (int)pdc.size();
  return KDE_OK;
}

}  // namespace host
}  // namespace kde

extern "C" {

kde_status kde_psi_r(kde_ctx* c, const double* x, int64_t n, int32_t r, const double* g, int32_t ng, double* psi) {
  TRY(check_ctx(c));
  prof_reset(c);
  TRY(validate_X(c, x, n, 1, 1));
  if (!(r == 4 || r == 6 || r == 8)) return fail(c, KDE_E_INVALID, "r=%d not in {4,6,8}", r);
  if (!g || !psi || ng < 1) return fail(c, KDE_E_INVALID, "null candidate/output array");
  for (int k = 0; k < ng; ++k)
    if (!(g[k] > 0.0) || !std::isfinite(g[k])) return fail(c, KDE_E_NONPOSITIVE_BW, "g[%d] <= 0", k);
  Ws w;
  TRY(get_ws(c, (n + 2047) / 2048 * 2048, 1, 2, &w));
  Moments m;
  if (n >= 2) {
    TRY(gpu_moments(c, x, n, 1, w, m));
  } else {
    m.mean = {0.0};
  }
  std::vector<kde_fixed> o;
  TRY(psi_raw(c, x, n, r, g, ng, m, c->rank, c->world, true, o));
  TRY(prof_collect(c));
  for (int k = 0; k < ng; ++k) psi[k] = psi_finalize(r, n, g[k], fixed_value(o[k]));
  return KDE_OK;
}

// PLUGIN passes read their bounded skip threshold from the chain's small block: the closed form written by
// the chain stage that produces g (psi_plugin_bounded), replaced by the data-aware one when enough tiles
// make the selection worth its launch (psi_plugin_select).
static bool psi_plugin_bounded() { return kde::psi_skip_gap(false) < INFINITY && kde::skip_bounded(); }
static bool psi_plugin_select(int64_t n, int T) {
  return psi_plugin_bounded() && (n + T - 1) / T >= kde::kGapSelectMinTiles;
}

// One fp32-term Psi_r pair pass of the device-resident PLUGIN chain: kernel over this rank's
// tiles into `limbs` (S, A), then (world > 1) the all-reduce, all enqueued on the context stream.
static kde_status plugin_pass(kde_ctx* c, int r, int64_t n, int64_t ld, int T, int S, const PsiBufs& b,
                              unsigned long long* clamp, unsigned long long* limbs, int64_t tb, int64_t te,
                              double pairs, unsigned long long* skipped, unsigned long long* work,
                              const double* gap_dev) {
  Range rr("kde.pair_pass");
  kde::LaunchCfg cfg;
  cfg.X = b.Yc; cfg.n = n; cfg.ld = ld; cfg.tile_begin = tb; cfg.tile_end = te; cfg.tile = T;
  cfg.part_rank = c->rank; cfg.part_world = c->world;
  cfg.scale_exp = S; cfg.limbs = limbs; cfg.n_out = 2; cfg.stream = c->stream; cfg.sm_count = c->sm_count;
  cfg.clamp = clamp; cfg.Y64 = b.Y64; cfg.centres = b.centres;
  cfg.skipped = skipped;
  cfg.skip_gap = kde::psi_skip_gap(false);
  // bounded far-tile skip: the pass's data-aware threshold (launch_psi_gap_select, after the prep)
  if (psi_plugin_bounded()) cfg.skip_gap_dev = gap_dev;
  cfg.work = work;
  kde::PsiParams p;
  psi_coeffs(r, p);
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  // external event records: inside a graph capture they become timing event nodes
  const unsigned rec = (c->cap_stream && c->stream == c->cap_stream) ? cudaEventRecordExternal : cudaEventRecordDefault;
  if (c->profiling) { e0 = next_event(c); e1 = next_event(c); CUDA_TRY(c, cudaEventRecordWithFlags(e0, c->stream, rec)); }
  cudaError_t err = kde::launch_psi(r, cfg, p);
  if (err != cudaSuccess) return fail(c, KDE_E_CUDA, "pair kernel launch: %s", cudaGetErrorString(err));
  if (tb < te) c->prof_all += 1;
  if (c->profiling) {
    CUDA_TRY(c, cudaEventRecordWithFlags(e1, c->stream, rec));
    c->prof_launches++;
    c->prof_evals += pairs;
  }
  TRY(allreduce_limbs(c, limbs, 2 * kde::kLimbs));
  return KDE_OK;
}

// PLUGIN (Sec. 4.4.1): moments, sort, prep and the two pair passes, with the scalar
// steps 1-8 computed by single-thread kernels on the device between them, so the whole chain is
// enqueued without a host round trip and the call synchronises once.  Each Psi pass runs with
// fp32 terms; a device-side decision (stage 4 / 5: the pass's cancellation estimate, or the
// precision mode) gates an fp64-term re-run of that pass on the same fp64 samples, and the next
// stage reads whichever sum is valid.  Failures are recorded on the device and reported in order.
// Enqueue the whole chain on c->stream (no allocation, no synchronisation: capturable).
static kde_status plugin_enqueue(kde_ctx* c, const double* x, int64_t n, int T, int64_t ld, Ws& w) {
  kde::PluginDev dv(w.small);
  const PsiBufs b = psi_bufs(w, ld);
  const int nblk = kde::moments_blocks(n);
  cudaStream_t st = c->stream;
  // flags (2 x u64), trace (8), status (1) and gates (2) start at zero
  CUDA_TRY(c, cudaMemsetAsync(w.flag(), 0, (kde::kSmallDoubles - 408) * sizeof(double), st));
  {
    Range r("kde.moments");
    CUDA_TRY(c, kde::launch_moments1(x, n, 1, w.part, nblk, st));
    CUDA_TRY(c, kde::launch_reduce_parts(w.part, nblk, 1, dv.sums, st));
    CUDA_TRY(c, kde::launch_plugin_chain(0, n, w.small, nullptr, 0, st));             // mean
    CUDA_TRY(c, kde::launch_moments2(x, n, 1, dv.mean, w.part, nblk, st));
    CUDA_TRY(c, kde::launch_reduce_parts(w.part, nblk, 1, dv.sums, st));
    CUDA_TRY(c, kde::launch_plugin_chain(1, n, w.small, nullptr, 0, st));             // steps 1-4
    c->prof_all += 6;
  }
  const double* xs = nullptr;                                                          // sorted once (§3)
  TRY(gpu_sorted(c, x, n, &xs));
  int64_t tb, te;
  shard_range(n_tiles(n, T), c->rank, c->world, &tb, &te);
  const double pairs = c->profiling ? pairs_in_shard(n, T, te, c->rank, c->world) : 0.0;
  const int S6 = scale_exp_for(2.0 * 15.0, n), S4 = scale_exp_for(2.0 * 3.0, n);
  const int mode = c->psi_mode;
  unsigned long long* L = w.limbs;                       // [S6, A6, S4, A4, S6 fp64, S4 fp64]
  unsigned long long* work = L + kde::kPluginOuts * kde::kLimbs;   // one scheduling counter per pass
  CUDA_TRY(c, cudaMemsetAsync(L, 0, (kde::kPluginOuts * kde::kLimbs + 2) * sizeof(long long), st));
  const int Ss[2] = {S6, S4};
  for (int k = 0; k < 2; ++k) {                                                        // Psi6(g1), Psi4(g2)
    const int r = k == 0 ? 6 : 4;
    CUDA_TRY(c, kde::launch_psi_prep(xs, n, dv.mean, dv.W, T, b.Y64, b.Yc, b.centres, ld, st, w.flag(), 3.0e4));
    if (mode != 1 && psi_plugin_select(n, T)) {   // data-aware threshold
      CUDA_TRY(c, kde::launch_psi_gap_select(r, b.Y64, n, T, dv.trace + (k == 0 ? 3 : 5), 0.0, dv.trace, 0.0,
                                             w.small + kde::kGapSlot + k, w.part, st));
      c->prof_all += 2;
    }
    if (mode != 1)
      TRY(plugin_pass(c, r, n, ld, T, Ss[k], b, w.flag() + 1, L + (size_t)(2 * k) * kde::kLimbs, tb, te, pairs,
                      reinterpret_cast<unsigned long long*>(w.small + kde::kSkippedSlot), work + k,
                      w.small + kde::kGapSlot + k));
    CUDA_TRY(c, kde::launch_plugin_chain(4 + k, n, w.small, L, Ss[k], st, mode));     // fp64 re-run?
    TRY(psi64_pass(c, r, b.Y64, n, Ss[k], L + (size_t)(4 + k) * kde::kLimbs, dv.gate + k, k));
    CUDA_TRY(c, kde::launch_plugin_chain(k == 0 ? 2 : 3, n, w.small, L, Ss[k], st));  // steps 5-6 / 7-8
    c->prof_all += 3;
  }
  CUDA_TRY(c, cudaMemcpyAsync(c->h_limbs, w.flag(), (kde::kSmallDoubles - 408) * sizeof(double),
                              cudaMemcpyDeviceToHost, st));
  return KDE_OK;
}

// PLUGIN (Sec. 4.4.1): the chain above, captured once as a CUDA graph and replayed while
// its inputs (pointers, n, mode) are unchanged.  The steps' formulas are those of the host reading
// (Z1, Z10, Z11); failures are recorded on the device and reported in order.
static kde_status plugin_impl(kde_ctx* c, const double* x, int64_t n, kde_plugin_trace* tr) {
  const int T = kde::tile_for(Kind::Psi6, 1, n);
  const int64_t ld = (n + T - 1) / T * T;
  Ws w;
  TRY(get_ws(c, ld, 4, kde::kPluginOuts, &w));    // everything the chain touches exists before
  TRY(ensure_sort_ws(c, n));                      // a capture starts
  const size_t cnt = kde::kSmallDoubles - 408;    // flags, trace, status, gates
  if (c->h_limbs_cap < cnt) {
    if (c->h_limbs) cudaFreeHost(c->h_limbs);
    c->h_limbs = nullptr;
    CUDA_TRY(c, cudaMallocHost(&c->h_limbs, cnt * sizeof(long long)));
    c->h_limbs_cap = cnt;
  }
  for (int r : {6, 4}) {                          // kernel attributes: not settable while capturing
    kde::LaunchCfg cfg;
    cfg.n = n; cfg.tile = T; cfg.sm_count = c->sm_count;
    CUDA_TRY(c, kde::prepare_psi(r, cfg));
  }
  cudaStream_t st = c->stream;
  const std::vector<uintptr_t> key = {(uintptr_t)x, (uintptr_t)n, (uintptr_t)w.Y, (uintptr_t)c->sort_ws,
                                      (uintptr_t)c->h_limbs, (uintptr_t)c->profiling, (uintptr_t)c->comm,
                                      (uintptr_t)(c->psi_mode + 1),
                                      (uintptr_t)(kde::psi_skip_gap(false) < INFINITY) + 2 * kde::skip_bounded()};
  // The first call with a given key runs directly (and does any lazy module loading and library
  // setup outside a capture); a second call with the same key captures, later ones replay.
  // (single-GPU contexts only: with a communicator the all-reduces stay plain stream operations)
  if (!c->graphs || c->comm || c->world > 1 || (key != c->plug_seen && !(c->plug_exec && key == c->plug_key))) {
    TRY(plugin_enqueue(c, x, n, T, ld, w));
    c->plug_seen = key;
  } else {
    if (!(c->plug_exec && key == c->plug_key)) {
      Range r("kde.capture");
      if (!c->cap_stream) CUDA_TRY(c, cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
      if (c->plug_exec) { cudaGraphExecDestroy(c->plug_exec); c->plug_exec = nullptr; }
      CUDA_TRY(c, cudaStreamSynchronize(st));
      cudaGetLastError();
      CUDA_TRY(c, cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeRelaxed));
      c->stream = c->cap_stream;
      const int32_t l0 = c->prof_launches, a0 = c->prof_all;
      const double e0 = c->prof_evals;
      const kde_status es = plugin_enqueue(c, x, n, T, ld, w);
      c->stream = st;
      cudaGraph_t g = nullptr;
      const cudaError_t ce = cudaStreamEndCapture(c->cap_stream, &g);
      if (es != KDE_OK) { if (g) cudaGraphDestroy(g); return es; }
      if (ce != cudaSuccess) return fail(c, KDE_E_CUDA, "graph capture: %s", cudaGetErrorString(ce));
      const cudaError_t ie = cudaGraphInstantiate(&c->plug_exec, g, 0);
      cudaGraphDestroy(g);
      if (ie != cudaSuccess) { c->plug_exec = nullptr; return fail(c, KDE_E_CUDA, "graph instantiate: %s", cudaGetErrorString(ie)); }
      c->plug_key = key;
      c->plug_prof_launches = c->prof_launches - l0;
      c->plug_prof_all = c->prof_all - a0;
      c->plug_prof_evals = c->prof_evals - e0;
      c->plug_ev_used = c->ev_used;
    } else {
      c->prof_launches += c->plug_prof_launches;
      c->prof_all += c->plug_prof_all;
      c->prof_evals += c->plug_prof_evals;
      c->ev_used = c->plug_ev_used;   // the graph records the same pool events
    }
    CUDA_TRY(c, cudaGraphLaunch(c->plug_exec, st));
  }
  CUDA_TRY(c, cudaStreamSynchronize(st));
  const unsigned long long* flags = reinterpret_cast<const unsigned long long*>(c->h_limbs);
  double res[9];
  std::memcpy(res, c->h_limbs + 2, sizeof(res));
  const unsigned long long* gates = flags + 11;
  double kap[2];                                  // small[421..422]
  std::memcpy(kap, c->h_limbs + 13, sizeof(kap));
  if (c->psi_mode != 1) {
    c->psi_kappa_max = std::max(kap[0], kap[1]);
    const double exact = kde::psi_skip_gap(false);
    for (int k = 0; k < 2; ++k) {
      double gap = exact;
      if (psi_plugin_bounded()) std::memcpy(&gap, c->h_limbs + (kde::kGapSlot - 408 + k), sizeof(gap));
      c->psi_gaps.push_back(gap);
    }
  }
  if (c->profiling) {                             // pairs of exactly-zero tiles the kernels skipped
    unsigned long long sk = 0;
    std::memcpy(&sk, c->h_limbs + (kde::kSkippedSlot - 408), sizeof(sk));
    c->prof_evals -= (double)sk;
  }
  for (int k = 0; k < 2; ++k) {                   // fp64 re-runs that actually ran
    if (gates[k]) {
      if (c->psi_mode == 0) c->psi_escalations++;
      if (c->profiling) { c->prof_launches++; c->prof_evals += c->gate_evals[k]; }
    } else if (c->profiling && c->gate_pair[k] >= 0) {
      if (c->ev_excl.size() <= (size_t)c->gate_pair[k]) c->ev_excl.resize(c->gate_pair[k] + 1, 0);
      c->ev_excl[c->gate_pair[k]] = 1;            // its (empty) launch is not a pair pass
    }
  }
  const int status = (int)res[8];
  if (status == KDE_E_INVALID) return fail(c, KDE_E_INVALID, "non-finite sample values");
  if (status == KDE_E_DEGENERATE) return fail(c, KDE_E_DEGENERATE, "variance estimate <= 0");
  if (flags[0]) return fail(c, KDE_E_INVALID, "scaled sample differences exceed 1e18 (outliers vs. bandwidth)");
  if (status == KDE_E_NUMERIC)
    return fail(c, KDE_E_NUMERIC, !(res[4] < 0.0) ? "Psi6-hat >= 0" : "Psi4-hat <= 0");
  kde_plugin_trace t;
  t.V_hat = res[0]; t.sigma_hat = res[1]; t.psi8_ns = res[2]; t.g1 = res[3];
  t.psi6 = res[4]; t.g2 = res[5]; t.psi4 = res[6]; t.h = res[7];
  *tr = t;
  return KDE_OK;
}

kde_status kde_plugin_h(kde_ctx* c, const double* x, int64_t n, double* h, kde_plugin_trace* tr) {
  TRY(check_ctx(c));
  prof_reset(c);
  TRY(validate_X(c, x, n, 1, 2));
  if (!h) return fail(c, KDE_E_INVALID, "null output");
  kde_plugin_trace t;
  TRY(plugin_impl(c, x, n, &t));
  TRY(prof_collect(c));
  *h = t.h;
  if (tr) *tr = t;
  return KDE_OK;
}

static kde_status lscv_h_scores_impl(kde_ctx* c, const double* X, int64_t n, int d, const double* h,
                                     int nh, double* g) {
  Ws w;
  TRY(get_ws(c, (n + 2047) / 2048 * 2048, d, 2, &w));
  Moments m;
  TRY(gpu_moments(c, X, n, d, w, m));
  LscvhPrep pp;
  TRY(lscv_h_prepare(c, m, d, pp));
  TRY(gpu_sorted_rows(c, X, n, d, &X));
  std::vector<kde_fixed> o;
  TRY(lscv_h_raw(c, X, n, d, h, nh, m, pp, c->rank, c->world, true, o));
  std::vector<double> W;
  for (int k = 0; k < nh; ++k) {
    double S1 = fixed_value(o[2 * k]), S2 = fixed_value(o[2 * k + 1]);
    // automatic precision: a candidate whose objective cancels beyond what fp32 terms carry (or every
    // candidate in the fp64-term mode) is re-run with fp64 terms (§3.10)
    if (c->psi_mode != -1 && (c->psi_mode == 1 || !(lscv_cancellation(n, d, pp.det, S1, S2) <= kLscvKappaMax))) {
      if (W.empty()) {
        W = tri_lower_inverse(pp.Lc, d);
        for (double& v : W) v *= std::sqrt(kLog2e / 4.0);
      }
      kde_fixed f[2];
      TRY(lscv_sums64(c, X, n, d, W, m.mean, -1.0 / (h[k] * h[k]), f));
      S1 = fixed_value(f[0]);
      S2 = fixed_value(f[1]);
    }
    g[k] = lscv_h_finalize(n, d, pp.det, h[k], S1, S2);
  }
  return KDE_OK;
}

kde_status kde_lscv_h_scores(kde_ctx* c, const double* X, int64_t n, int32_t d, const double* h,
                             int32_t nh, double* g) {
  TRY(check_ctx(c));
  prof_reset(c);
  TRY(validate_X(c, X, n, d, 2));
  if (!h || !g || nh < 1) return fail(c, KDE_E_INVALID, "null candidate/output array");
  for (int k = 0; k < nh; ++k)
    if (!(h[k] > 0.0) || !std::isfinite(h[k])) return fail(c, KDE_E_NONPOSITIVE_BW, "h[%d] <= 0", k);
  std::vector<double> tmp(nh);
  TRY(lscv_h_scores_impl(c, X, n, d, h, nh, tmp.data()));
  TRY(prof_collect(c));
  std::copy(tmp.begin(), tmp.end(), g);
  return KDE_OK;
}

kde_status kde_lscv_H_scores(kde_ctx* c, const double* X, int64_t n, int32_t d, const double* vh,
                             int32_t nH, double penalty, double* g) {
  TRY(check_ctx(c));
  prof_reset(c);
  TRY(validate_X(c, X, n, d, 2));
  if (!vh || !g || nH < 1) return fail(c, KDE_E_INVALID, "null candidate/output array");
  if (std::isnan(penalty)) penalty = 1e300;
  const int P = d * (d + 1) / 2;
  Ws w;
  TRY(get_ws(c, (n + 2047) / 2048 * 2048, d, 2, &w));
  Moments m;
  TRY(gpu_moments(c, X, n, d, w, m));
  std::vector<std::vector<double>> vs;
  for (int k = 0; k < nH; ++k) vs.emplace_back(vh + (size_t)k * P, vh + (size_t)(k + 1) * P);
  std::vector<double> out;
  TRY(lscv_H_eval(c, X, n, d, m, vs, penalty, out, nullptr, /*auto_precision=*/true));
  TRY(prof_collect(c));
  std::copy(out.begin(), out.end(), g);
  return KDE_OK;
}

kde_status kde_raw_sums(kde_ctx* c, kde_sum_kind kind, const double* X, int64_t n, int32_t d,
                        const double* cand, int32_t nc, int32_t srank, int32_t sworld, kde_fixed* out) {
  TRY(check_ctx(c));
  prof_reset(c);
  TRY(validate_X(c, X, n, d, 1));
  if (!cand || !out || nc < 1) return fail(c, KDE_E_INVALID, "null candidate/output array");
  bool allreduce = sworld == 0;
  if (sworld == 0) { srank = c->rank; sworld = c->world; }
  if (srank < 0 || srank >= sworld) return fail(c, KDE_E_INVALID, "bad shard");
  Ws w;
  TRY(get_ws(c, (n + 2047) / 2048 * 2048, d, 2, &w));
  Moments m;
  if (n >= 2) {
    TRY(gpu_moments(c, X, n, d, w, m));
  } else {
    m.mean.assign(d, 0.0);
    m.cov.assign((size_t)d * d, 0.0);
  }
  std::vector<kde_fixed> o;
  if (kind == KDE_SUM_PSI4 || kind == KDE_SUM_PSI6 || kind == KDE_SUM_PSI8) {
    if (d != 1) return fail(c, KDE_E_NOT_UNIVARIATE, "Psi sums need d = 1");
    for (int k = 0; k < nc; ++k)
      if (!(cand[k] > 0.0)) return fail(c, KDE_E_NONPOSITIVE_BW, "g <= 0");
    TRY(psi_raw(c, X, n, (int)kind, cand, nc, m, srank, sworld, allreduce, o));
  } else if (kind == KDE_SUM_LSCV_h) {
    if (n < 2) return fail(c, KDE_E_INSUFFICIENT_SAMPLES, "n < 2");
    for (int k = 0; k < nc; ++k)
      if (!(cand[k] > 0.0)) return fail(c, KDE_E_NONPOSITIVE_BW, "h <= 0");
    LscvhPrep pp;
    TRY(lscv_h_prepare(c, m, d, pp));
    TRY(lscv_h_raw(c, X, n, d, cand, nc, m, pp, srank, sworld, allreduce, o));
  } else if (kind == KDE_SUM_LSCV_H) {
    const int P = d * (d + 1) / 2;
    std::vector<HCand> hc;
    for (int k = 0; k < nc; ++k) {
      hc.push_back(h_candidate(cand + (size_t)k * P, d));
      if (!hc.back().pd) return fail(c, KDE_E_INVALID, "candidate %d is not positive definite", k);
    }
    if (n < 2) m.mean.assign(d, 0.0);
    TRY(lscv_H_raw(c, X, n, d, hc, m, srank, sworld, allreduce, o, /*data_aware=*/true));
  } else {
    return fail(c, KDE_E_INVALID, "unknown sum kind");
  }
  TRY(prof_collect(c));
  std::copy(o.begin(), o.end(), out);
  return KDE_OK;
}

kde_status kde_select_bandwidth(kde_ctx* c, kde_method method, const double* X, int64_t n, int32_t d,
                                const kde_select_opts* opts_in, kde_bandwidth* out) {
  TRY(check_ctx(c));
  prof_reset(c);
  if (!out) return fail(c, KDE_E_INVALID, "null output");
  kde_select_opts o;
  kde_default_opts(&o);
  if (opts_in) o = *opts_in;
  TRY(validate_X(c, X, n, d, 2));
  kde_bandwidth r;
  std::memset(&r, 0, sizeof(r));
  r.method = method;
  r.d = d;
  if (method == KDE_PLUGIN) {
    if (d != 1) return fail(c, KDE_E_NOT_UNIVARIATE, "PLUGIN is univariate (P:196)");
    TRY(plugin_impl(c, X, n, &r.trace));
    r.h = r.trace.h;
    r.evaluations = 2;
  } else if (method == KDE_LSCV_h) {
    if (o.n_grid < 2 || !(o.range_factor > 1.0)) return fail(c, KDE_E_INVALID, "bad grid options");
    // Eq. 25 as written (reading Z3): R(K)/mu2^2 = 1/(2^d pi^{d/2} d^2), R(f'') = d(d+2)/(2^{d+2} pi^{d/2})
    const double dd = d;
    const double ratio = 1.0 / (std::pow(2.0, dd) * std::pow(kPi, dd / 2) * dd * dd);
    const double Rf2 = dd * (dd + 2) / (std::pow(2.0, dd + 2) * std::pow(kPi, dd / 2));
    const double h0 = std::pow(ratio / (Rf2 * (double)n), 1.0 / (dd + 4));
    const double lo = h0 / o.range_factor, hi = h0 * o.range_factor;       // Eq. 27
    std::vector<double> hs(o.n_grid), gs(o.n_grid);
    for (int k = 0; k < o.n_grid; ++k) hs[k] = lo + k * (hi - lo) / (o.n_grid - 1);
    TRY(lscv_h_scores_impl(c, X, n, d, hs.data(), o.n_grid, gs.data()));
    int best = 0;
    for (int k = 1; k < o.n_grid; ++k)
      if (gs[k] < gs[best]) best = k;                                    // ties -> smaller h
    r.h = hs[best];
    r.objective = gs[best];
    r.iterations = best;
    r.evaluations = o.n_grid;
    // Optional refinement (f4): bracket = the grid neighbours of the argmin; each step scores
    // 16 equally spaced interior points in one pass and re-brackets around the best known point
    // (ties -> smaller h).  A batched form of the section search the paper suggests.
    if (o.refine_steps > 0) {
      std::vector<std::pair<double, double>> pts;   // (h, g) known inside the bracket, sorted by h
      pts.push_back({hs[best > 0 ? best - 1 : 0], gs[best > 0 ? best - 1 : 0]});
      if (best > 0) pts.push_back({hs[best], gs[best]});
      if (best + 1 < o.n_grid) pts.push_back({hs[best + 1], gs[best + 1]});
      int steps = 0;
      while (steps < o.refine_steps) {
        const double a = pts.front().first, b = pts.back().first;
        if (!(b - a > o.refine_tol * r.h)) break;
        std::vector<double> hh(16), gg(16);
        for (int k = 0; k < 16; ++k) hh[k] = a + (k + 1) * (b - a) / 17.0;
        TRY(lscv_h_scores_impl(c, X, n, d, hh.data(), 16, gg.data()));
        r.evaluations += 16;
        for (int k = 0; k < 16; ++k) pts.push_back({hh[k], gg[k]});
        std::sort(pts.begin(), pts.end());
        size_t bi = 0;
        for (size_t k = 1; k < pts.size(); ++k)
          if (pts[k].second < pts[bi].second) bi = k;
        r.h = pts[bi].first;
        r.objective = pts[bi].second;
        const size_t lo_i = bi > 0 ? bi - 1 : 0, hi_i = bi + 1 < pts.size() ? bi + 1 : bi;
        std::vector<std::pair<double, double>> nb(pts.begin() + lo_i, pts.begin() + hi_i + 1);
        pts.swap(nb);
        ++steps;
      }
      r.stop_reason = steps;
    }
  } else if (method == KDE_LSCV_H) {
    Ws w;
    TRY(get_ws(c, (n + 2047) / 2048 * 2048, d, 2, &w));
    Moments m;
    TRY(gpu_moments(c, X, n, d, w, m));
    std::vector<double> Lc, root;
    if (!cholesky(m.cov, d, Lc)) return fail(c, KDE_E_SINGULAR_COV, "covariance not positive definite");
    if (!spd_sqrt(m.cov, d, root)) return fail(c, KDE_E_SINGULAR_COV, "matrix square root failed");
    // Eq. 35 as written: H_start = (4/(d+2))^{1/(d+4)} n^{-1/(d+4)} Sigma^{1/2}
    const double f = std::pow(4.0 / (d + 2), 1.0 / (d + 4)) * std::pow((double)n, -1.0 / (d + 4));
    for (double& v : root) v *= f;
    const int P = d * (d + 1) / 2;
    if (o.nm_param != 0 && o.nm_param != 1) return fail(c, KDE_E_INVALID, "nm_param must be 0 or 1");
    const bool chol_param = o.nm_param == 1;
    if (chol_param) {   // search over the Cholesky factor (row f4): start from L = chol(H_start)
      std::vector<double> L;
      if (!cholesky(root, d, L)) return fail(c, KDE_E_SINGULAR_COV, "H_start not positive definite");
      root = L;         // lower triangular; the simplex rule below reads its diagonal
    }
    std::vector<double> x0(P);
    vech(root, d, x0.data());
    std::vector<std::vector<double>> sim = {x0};
    int t = 0;
    for (int b = 0; b < d; ++b)
      for (int a = b; a < d; ++a) {
        const double delta = 0.1 * (a == b ? root[a * d + a] : std::sqrt(root[a * d + a] * root[b * d + b]));
        std::vector<double> v = x0;
        v[t] += delta;
        sim.push_back(v);
        ++t;
      }
    // start k of o.nm_starts: vech(H_start) scaled by 4^-k (the paper's Eq. 35 start first)
    std::vector<std::vector<std::vector<double>>> sims;
    const int K = std::max(1, o.nm_starts);
    for (int k = 0; k < K; ++k) {
      const double sc = std::pow(4.0, -k);
      std::vector<std::vector<double>> sk;
      for (const auto& v : sim) {
        std::vector<double> w(v);
        for (double& e : w) e *= sc;
        sk.push_back(w);
      }
      sims.push_back(sk);
    }
    NMResult nm;
    TRY(gpu_sorted_rows(c, X, n, d, &X));   // once for the whole search (far-tile skip)
    // device-resident loop: one GPU, one start, serial rounds, whitened sets within ~1 GiB
    const int64_t Tm = kde::tile_for(Kind::LscvMatrix, d, n), ldT = (n + Tm - 1) / Tm * Tm;
    const bool dev_loop = o.nm_loop == 0 && K == 1 && o.speculative == 0 && c->world == 1 && !c->comm && c->psi_mode != 1 &&
                          !chol_param &&
                          !c->har_fn && (double)(P + 1) * d * (double)ldT * 4.0 <= (double)(1LL << 30);
    if (dev_loop)
      TRY(nelder_mead_device(c, X, n, d, m, sims[0], o.max_iter, o.tol_rel, o.penalty, nm));
    else
      TRY(nelder_mead_multi(c, X, n, d, m, sims, o.max_iter, o.tol_rel, o.penalty, o.speculative != 0, nm, nullptr,
                            chol_param));
    if (!(nm.f < o.penalty)) return fail(c, KDE_E_NO_FEASIBLE, "no positive-definite H found");
    if (chol_param) {
      std::vector<double> h(P);
      vech_llt(nm.x.data(), d, h.data());
      nm.x = h;
    }
    for (int k = 0; k < P; ++k) r.vechH[k] = nm.x[k];
    r.objective = nm.f;
    r.iterations = nm.iterations;
    r.evaluations = nm.evals;
    r.stop_reason = nm.stop;
  } else {
    return fail(c, KDE_E_INVALID, "unknown method");
  }
  TRY(prof_collect(c));
  *out = r;
  return KDE_OK;
}

}  // extern "C"
