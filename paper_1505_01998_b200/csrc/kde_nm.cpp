// kde_nm.cpp — Nelder–Mead over vech(H) for LSCV_H (reading Z8): the serial /
// speculative state machine and the lockstep multi-start driver whose rounds evaluate one GPU
// batch each.
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

namespace kde {
namespace host {

// One Nelder–Mead run as a state machine: propose() lists the points whose objective values the
// next decision needs, accept() takes those values and applies the serial NM logic (rho = 1,
// chi = 2, gamma = sigma = 1/2; stable order by (f, index); stop on
// f_worst - f_best <= tol |f_best| or max_iter).  Speculative mode proposes reflect, expand,
// outside and inside contraction together; the decisions are those of serial NM on the same
// values.  Several runs can share one GPU batch (multi-start, row f4).
struct NMRun {
  enum Phase { INIT, STEP, SERIAL_R, SERIAL_1, SHRINK, DONE } phase = INIT;
  std::vector<std::vector<double>> sim;
  std::vector<double> fs;
  int M = 0, it = 0, max_iter = 500, stop = 2;
  double tol = 1e-7;
  bool speculative = true;
  std::vector<double> xbar, xr, xe, xc, xcc;
  double fr = 0.0;
  int serial_pick = 0;   // SERIAL_1: 1 = expand, 2 = outside contraction, 3 = inside contraction

  static std::vector<double> comb(const std::vector<double>& a, double s, const std::vector<double>& b,
                                  const std::vector<double>& c) {
    std::vector<double> r(a.size());
    for (size_t k = 0; k < a.size(); ++k) r[k] = a[k] + s * (b[k] - c[k]);
    return r;
  }

  // Sort, test the stopping rule and prepare the trial points of the next iteration.
  void begin_iteration() {
    std::vector<int> ord(M + 1);
    std::iota(ord.begin(), ord.end(), 0);
    std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return fs[a] < fs[b]; });
    std::vector<std::vector<double>> s2;
    std::vector<double> f2;
    for (int k : ord) { s2.push_back(sim[k]); f2.push_back(fs[k]); }
    sim.swap(s2);
    fs.swap(f2);
    if (fs[M] - fs[0] <= tol * std::fabs(fs[0])) { stop = 1; phase = DONE; return; }
    if (it >= max_iter) { stop = 2; phase = DONE; return; }
    ++it;
    xbar.assign(sim[0].size(), 0.0);
    for (int k = 0; k < M; ++k)
      for (size_t u = 0; u < xbar.size(); ++u) xbar[u] += sim[k][u];
    for (double& v : xbar) v /= (double)M;
    xr = comb(xbar, 1.0, xbar, sim[M]);
    xe = comb(xbar, 2.0, xr, xbar);
    xc = comb(xbar, 0.5, xr, xbar);
    xcc = comb(xbar, 0.5, sim[M], xbar);
    phase = speculative ? STEP : SERIAL_R;
  }

  std::vector<std::vector<double>> propose() const {
    switch (phase) {
      case INIT: return sim;
      case STEP: return {xr, xe, xc, xcc};
      case SERIAL_R: return {xr};
      case SERIAL_1: return {serial_pick == 1 ? xe : (serial_pick == 2 ? xc : xcc)};
      case SHRINK: {
        std::vector<std::vector<double>> sh;
        for (int k = 1; k <= M; ++k) sh.push_back(comb(sim[0], 0.5, sim[k], sim[0]));
        return sh;
      }
      default: return {};
    }
  }

  // Decide with f_r known and (speculatively or not) the one follow-up value.
  // Returns true if the follow-up value is still needed (serial mode).
  void decide(double fr_, bool have_follow, double fe, double fc, double fcc) {
    if (fr_ < fs[0]) {
      if (!have_follow) { serial_pick = 1; fr = fr_; phase = SERIAL_1; return; }
      if (fe < fr_) { sim[M] = xe; fs[M] = fe; } else { sim[M] = xr; fs[M] = fr_; }
      begin_iteration();
      return;
    }
    if (fr_ < fs[M - 1]) { sim[M] = xr; fs[M] = fr_; begin_iteration(); return; }
    if (fr_ < fs[M]) {
      if (!have_follow) { serial_pick = 2; fr = fr_; phase = SERIAL_1; return; }
      if (fc <= fr_) { sim[M] = xc; fs[M] = fc; begin_iteration(); return; }
    } else {
      if (!have_follow) { serial_pick = 3; fr = fr_; phase = SERIAL_1; return; }
      if (fcc < fs[M]) { sim[M] = xcc; fs[M] = fcc; begin_iteration(); return; }
    }
    phase = SHRINK;
  }

  void accept(const std::vector<double>& g) {
    switch (phase) {
      case INIT: fs = g; begin_iteration(); break;
      case STEP: decide(g[0], true, g[1], g[2], g[3]); break;
      case SERIAL_R: decide(g[0], false, 0, 0, 0); break;
      case SERIAL_1: {
        const double v = g[0];
        decide(fr, true, serial_pick == 1 ? v : 0, serial_pick == 2 ? v : 0, serial_pick == 3 ? v : 0);
        break;
      }
      case SHRINK: {
        for (int k = 1; k <= M; ++k) { sim[k] = comb(sim[0], 0.5, sim[k], sim[0]); fs[k] = g[k - 1]; }
        begin_iteration();
        break;
      }
      default: break;
    }
  }
};

// Run several NM instances in lockstep; every round evaluates the union of their proposals as
// one GPU batch (lscv_H_eval), so per-run decisions equal those of a lone run.
kde_status nelder_mead_multi(kde_ctx* c, const double* X, int64_t n, int d, const Moments& m,
                             const std::vector<std::vector<std::vector<double>>>& sims, int max_iter,
                             double tol, double penalty, bool speculative, NMResult& best, int* total_evals) {
  std::vector<NMRun> runs(sims.size());
  for (size_t r = 0; r < sims.size(); ++r) {
    runs[r].sim = sims[r];
    runs[r].M = (int)sims[r].size() - 1;
    runs[r].max_iter = max_iter;
    runs[r].tol = tol;
    runs[r].speculative = speculative;
  }
  int evals = 0;
  while (true) {
    std::vector<std::vector<double>> batch;
    std::vector<std::pair<size_t, size_t>> span;   // (run, count)
    for (size_t r = 0; r < runs.size(); ++r) {
      if (runs[r].phase == NMRun::DONE) continue;
      auto p = runs[r].propose();
      span.push_back({r, p.size()});
      for (auto& v : p) batch.push_back(std::move(v));
    }
    if (batch.empty()) break;
    std::vector<double> g;
    TRY(lscv_H_eval(c, X, n, d, m, batch, penalty, g, &evals));
    size_t off = 0;
    for (auto& sp : span) {
      std::vector<double> gv(g.begin() + off, g.begin() + off + sp.second);
      off += sp.second;
      runs[sp.first].accept(gv);
    }
  }
  size_t bi = 0;
  for (size_t r = 1; r < runs.size(); ++r)
    if (runs[r].fs[0] < runs[bi].fs[0]) bi = r;
  best.x = runs[bi].sim[0];
  best.f = runs[bi].fs[0];
  best.iterations = runs[bi].it;
  best.stop = runs[bi].stop;
  best.evals = evals;
  if (total_evals) *total_evals = evals;
  return KDE_OK;
}

}  // namespace host
}  // namespace kde
