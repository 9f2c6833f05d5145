// kde_nm.cpp — the host Nelder–Mead loop for LSCV_H (reading Z8): the state machine of
// kde_nm.cuh driven round by round, several runs in lockstep (multi-start, row f4) with one GPU
// batch per round; used for multi-start, speculative and multi-rank selections (the single-GPU
// serial case runs device-resident, kde_nm_dev.cu).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <memory>
#include <numeric>
#include <string>
#include <vector>

#include "kde_host.h"
#include "kde_nm.cuh"

namespace kde {
namespace host {

// Run several NM instances (kde_nm.cuh) in lockstep; every round evaluates the union of their
// proposals as one GPU batch (lscv_H_eval), so per-run decisions equal those of a lone run.
kde_status nelder_mead_multi(kde_ctx* c, const double* X, int64_t n, int d, const Moments& m,
                             const std::vector<std::vector<std::vector<double>>>& sims, int max_iter,
                             double tol, double penalty, bool speculative, NMResult& best, int* total_evals,
                             bool chol_param) {
  const int P = d * (d + 1) / 2;
  std::vector<std::unique_ptr<kde::NMState>> runs;
  for (const auto& sim : sims) {
    runs.emplace_back(new kde::NMState());
    kde::NMState& s = *runs.back();
    s.P = P; s.max_iter = max_iter; s.tol = tol; s.speculative = speculative ? 1 : 0;
    for (int v = 0; v <= P; ++v)
      for (int k = 0; k < P; ++k) s.sim[v][k] = sim[v][k];
  }
  std::vector<double> prop((size_t)(kde::kNMMaxP + 1) * kde::kNMMaxP);
  auto* rows = reinterpret_cast<double(*)[kde::kNMMaxP]>(prop.data());
  int evals = 0;
  while (true) {
    std::vector<std::vector<double>> batch;
    std::vector<std::pair<size_t, size_t>> span;   // (run, count)
    for (size_t r = 0; r < runs.size(); ++r) {
      if (runs[r]->phase == kde::NMState::DONE) continue;
      const int cnt = kde::nm_propose(*runs[r], rows);
      span.push_back({r, (size_t)cnt});
      for (int v = 0; v < cnt; ++v) {
        batch.emplace_back(rows[v], rows[v] + P);
        if (chol_param) vech_llt(rows[v], d, batch.back().data());   // H = L L^T of the vertex
      }
    }
    if (batch.empty()) break;
    std::vector<double> g;
    // fp64-term mode (kde_set_precision(ctx, 1)): every candidate with fp64 terms, the exact-parity
    // search of SURVEY c5; otherwise fp32 terms, as the device-resident loop
    TRY(lscv_H_eval(c, X, n, d, m, batch, penalty, g, &evals, /*auto_precision=*/c->psi_mode == 1));
    size_t off = 0;
    for (auto& sp : span) {
      kde::nm_accept(*runs[sp.first], g.data() + off);
      off += sp.second;
    }
  }
  size_t bi = 0;
  for (size_t r = 1; r < runs.size(); ++r)
    if (runs[r]->fs[0] < runs[bi]->fs[0]) bi = r;
  best.x.assign(runs[bi]->sim[0], runs[bi]->sim[0] + P);
  best.f = runs[bi]->fs[0];
  best.iterations = runs[bi]->it;
  best.stop = runs[bi]->stop;
  best.evals = evals;
  if (total_evals) *total_evals = evals;
  return KDE_OK;
}

}  // namespace host
}  // namespace kde
