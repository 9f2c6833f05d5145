// kde_nm_dev.cu — the device-resident Nelder–Mead loop of LSCV_H (reading Z8; the
// objective g(H) of Eq. 30-34).  The paper calls the optimizer inherently sequential with one g(H)
// per step; on B200 a host round trip per step (~30 us: D2H, sync, host decision, launches)
// is ~17% of a C3 step, so the whole loop runs as ONE CUDA graph:
//
//     WHILE (cond) {  nm_decide_kernel  ->  prep_sets_kernel  ->  pair_kernel_sets  }
//
// nm_decide_kernel (one thread) takes the previous round's exact limbs, finalises g(H) for each
// proposal (non-PD: the penalty), advances the state machine of kde_nm.cuh, proposes the next
// points, tests them for positive definiteness and writes each PD candidate's whitening
// parameters; prep_sets_kernel whitens the samples once per candidate and the pair kernel reads
// the candidate count from device memory.  When the state machine stops, the decide kernel sets
// the graph's conditional to 0.  The NM arithmetic is the host loop's (kde_nm.cuh), and this file
// is compiled with -fmad=false, so the device loop makes the same decisions on the same values.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "kde_device.cuh"
#include "kde_host.h"
#include "kde_nm.cuh"

namespace kde {

struct NMDevHeader {
  int d, S, max_sets;
  int n_prop, n_sets, pending, evals, rounds;
  double nn, pow4, pow2, penalty, wscale;
  double mean[kMaxDim];
  unsigned long long* limbs;   // 2 outputs (sum e, sum e^2) x kLimbs per set
  unsigned long long* work;    // the pair kernel's dynamic-scheduling counter
  PrepParams* pp;              // max_sets entries
};

struct NMDevBlock {
  NMDevHeader h;
  NMState st;
  double prop[kNMMaxP + 1][kNMMaxP];
  double g[kNMMaxP + 1];
  double det[kNMMaxP + 1];
  int slot[kNMMaxP + 1];       // set index of a PD proposal, -1 if not PD
  double L[kMaxDim * kMaxDim]; // Cholesky scratch (global memory: the decide thread keeps no big stack)
};

__device__ __forceinline__ double limbs_value(const unsigned long long* l, int S) {
  return ldexp((double)limbs_total(l), -S);
}

// One decision step (see the file comment) on a state `s` of any capacity.
template <class St, int OUT>
__device__ void decide_body(NMDevHeader& h, St& s, double (*prop)[OUT], double* g, double* det, int* slot,
                            double* L, cudaGraphConditionalHandle cond) {
  if (h.pending) {                                   // the previous round's values
    for (int i = 0; i < h.n_prop; ++i) {
      const int k = slot[i];
      g[i] = k < 0 ? h.penalty
                   : nm_lscv_H_finalize(h.nn, h.pow4, h.pow2, det[i],
                                        limbs_value(h.limbs + (size_t)(2 * k) * kLimbs, h.S),
                                        limbs_value(h.limbs + (size_t)(2 * k + 1) * kLimbs, h.S));
    }
    h.evals += h.n_sets;
    nm_accept(s, g);
    h.pending = 0;
  }
  while (true) {
    if (s.phase == St::DONE) {
      h.n_sets = 0;
      cudaGraphSetConditional(cond, 0);
      return;
    }
    h.n_prop = nm_propose(s, prop);
    h.n_sets = 0;
    for (int i = 0; i < h.n_prop; ++i) {
      double dt = 0.0;
      if (nm_cholesky_vech(prop[i], h.d, L, &dt)) {
        const int k = h.n_sets++;
        slot[i] = k;
        det[i] = dt;
        nm_whitening(L, h.d, h.wscale, h.pp[k].W);
        for (int a = 0; a < h.d; ++a) h.pp[k].mean[a] = h.mean[a];
      } else {
        slot[i] = -1;
      }
    }
    if (h.n_sets == 0) {                             // every proposal non-PD: no GPU pass needed
      for (int i = 0; i < h.n_prop; ++i) g[i] = h.penalty;
      nm_accept(s, g);
      continue;
    }
    for (size_t k = 0; k < (size_t)2 * h.n_sets * kLimbs; ++k) h.limbs[k] = 0ull;
    *h.work = 0ull;
    h.pending = 1;
    ++h.rounds;
    return;
  }
}

// d <= 4 (P <= 10): the decision runs on a shared-memory copy of the state (one thread; global
// memory latency would otherwise dominate the step); larger d works on the global block.
constexpr int kSmallP = 10;

__global__ void nm_decide_kernel(NMDevBlock* b, cudaGraphConditionalHandle cond) {
  if (b->st.P <= kSmallP) {
    __shared__ alignas(16) unsigned char sbuf[sizeof(NMStateT<kSmallP>)];
    __shared__ double sprop[kSmallP + 1][kSmallP], sg[kSmallP + 1], sdet[kSmallP + 1], sL[kMaxDim * kMaxDim];
    __shared__ int sslot[kSmallP + 1];
    __shared__ NMDevHeader sh;
    NMStateT<kSmallP>& ss = *reinterpret_cast<NMStateT<kSmallP>*>(sbuf);
    sh = b->h;
    nm_state_copy(ss, b->st);
    for (int i = 0; i <= kSmallP; ++i) { sdet[i] = b->det[i]; sslot[i] = b->slot[i]; }
    decide_body(sh, ss, sprop, sg, sdet, sslot, sL, cond);
    nm_state_copy(b->st, ss);
    for (int i = 0; i <= kSmallP; ++i) { b->det[i] = sdet[i]; b->slot[i] = sslot[i]; }
    b->h = sh;
  } else {
    decide_body(b->h, b->st, b->prop, b->g, b->det, b->slot, b->L, cond);
  }
}

namespace host {

// Single-GPU, single-start, serial LSCV_H Nelder–Mead from the simplex `sim` as one graph launch.
// X: the caller's fp64 samples (device), m: their moments.  Results as nelder_mead_multi.
kde_status nelder_mead_device(kde_ctx* c, const double* X, int64_t n, int d, const Moments& m,
                              const std::vector<std::vector<double>>& sim, int max_iter, double tol,
                              double penalty, NMResult& best) {
  const int P = d * (d + 1) / 2;
  const int max_sets = P + 1;                        // INIT evaluates the whole simplex
  const int T = kde::tile_for(Kind::LscvMatrix, d, n);
  const int64_t ld = (n + T - 1) / T * T;
  const int64_t set_floats = (int64_t)d * ld;
  Ws w;
  TRY(get_ws(c, ld, d, 2 * max_sets, &w));
  TRY(grow(c, &c->white_ws, &c->white_bytes, (size_t)max_sets * set_floats * sizeof(float)));
  const size_t blk = (sizeof(NMDevBlock) + 255) & ~size_t(255);
  TRY(grow(c, &c->nm_ws, &c->nm_bytes, blk + (size_t)max_sets * sizeof(PrepParams)));
  NMDevBlock* dblk = static_cast<NMDevBlock*>(c->nm_ws);
  PrepParams* pp = reinterpret_cast<PrepParams*>(static_cast<char*>(c->nm_ws) + blk);
  float* Yw = static_cast<float*>(c->white_ws);
  const size_t up = offsetof(NMDevBlock, prop);      // header + state: what a call uploads / reads back
  if (c->nm_host_cap < up) {
    if (c->nm_host) cudaFreeHost(c->nm_host);
    c->nm_host = nullptr;
    CUDA_TRY(c, cudaMallocHost(&c->nm_host, up));
    c->nm_host_cap = up;
  }
  {
    kde::LaunchCfg cfg;                              // kernel attributes: not settable while capturing
    cfg.n = n; cfg.tile = T; cfg.sm_count = c->sm_count; cfg.n_sets = max_sets; cfg.tile_begin = 0; cfg.tile_end = 0;
    CUDA_TRY(c, kde::prepare_lscv_white(d, cfg));
  }
  // the initial state: constants, the simplex, phase INIT
  NMDevBlock* hb = static_cast<NMDevBlock*>(c->nm_host);
  std::memset(static_cast<void*>(hb), 0, up);
  NMDevHeader& h = hb->h;
  h.d = d; h.S = scale_exp_for(1.0, n); h.max_sets = max_sets;
  h.nn = (double)n; h.pow4 = std::pow(4.0 * kPi, -0.5 * d); h.pow2 = std::pow(2.0 * kPi, -0.5 * d);
  h.penalty = penalty; h.wscale = std::sqrt(kLog2e / 4.0);
  for (int a = 0; a < d; ++a) h.mean[a] = m.mean[a];
  h.limbs = w.limbs; h.pp = pp;
  h.work = w.limbs + (size_t)2 * max_sets * kLimbs;
  NMState& s = hb->st;
  s.P = P; s.max_iter = max_iter; s.tol = tol; s.speculative = 0; s.phase = NMState::INIT; s.it = 0; s.stop = 2;
  for (int v = 0; v <= P; ++v)
    for (int k = 0; k < P; ++k) s.sim[v][k] = sim[v][k];
  cudaStream_t st = c->stream;
  CUDA_TRY(c, cudaMemcpyAsync(dblk, hb, up, cudaMemcpyHostToDevice, st));
  CUDA_TRY(c, cudaMemsetAsync(w.flag(), 0, 2 * sizeof(unsigned long long), st));
  // the graph (built once per key, replayed afterwards)
  const std::vector<uintptr_t> key = {(uintptr_t)X, (uintptr_t)n, (uintptr_t)d, (uintptr_t)w.limbs,
                                      (uintptr_t)Yw, (uintptr_t)dblk, (uintptr_t)T};
  if (!(c->nm_exec && key == c->nm_key)) {
    Range r("kde.nm_capture");
    if (c->nm_exec) { cudaGraphExecDestroy(c->nm_exec); c->nm_exec = nullptr; }
    if (!c->cap_stream) CUDA_TRY(c, cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
    cudaGraph_t g = nullptr;
    CUDA_TRY(c, cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle cond;
    cudaError_t e = cudaGraphConditionalHandleCreate(&cond, g, 1, cudaGraphCondAssignDefault);
    cudaGraphNodeParams cp = {};
    cudaGraphNode_t node;
    if (e == cudaSuccess) {
      cp.type = cudaGraphNodeTypeConditional;
      cp.conditional.handle = cond;
      cp.conditional.type = cudaGraphCondTypeWhile;
      cp.conditional.size = 1;
      e = cudaGraphAddNode(&node, g, nullptr, 0, &cp);
    }
    cudaGraph_t body = e == cudaSuccess ? cp.conditional.phGraph_out[0] : nullptr;
    if (e == cudaSuccess) e = cudaStreamBeginCaptureToGraph(c->cap_stream, body, nullptr, nullptr, 0,
                                                            cudaStreamCaptureModeRelaxed);
    if (e == cudaSuccess) {
      nm_decide_kernel<<<1, 1, 0, c->cap_stream>>>(dblk, cond);
      cudaError_t le = cudaGetLastError();
      if (le == cudaSuccess)
        le = kde::launch_prep_sets(X, n, d, pp, &dblk->h.n_sets, max_sets, Yw, set_floats, ld, c->cap_stream, w.flag());
      if (le == cudaSuccess) {
        kde::LaunchCfg cfg;
        cfg.X = Yw; cfg.n = n; cfg.ld = ld; cfg.tile = T; cfg.scale_exp = h.S; cfg.limbs = w.limbs;
        cfg.n_out = 2; cfg.stream = c->cap_stream; cfg.sm_count = c->sm_count; cfg.clamp = nullptr;
        cfg.n_sets = max_sets; cfg.set_stride = set_floats; cfg.n_sets_dev = &dblk->h.n_sets;
        cfg.work = w.limbs + (size_t)2 * max_sets * kLimbs;
        shard_range(n_tiles(n, T), 0, 1, &cfg.tile_begin, &cfg.tile_end);
        le = kde::launch_lscv_white(d, cfg);
      }
      cudaGraph_t cap = nullptr;
      const cudaError_t ce = cudaStreamEndCapture(c->cap_stream, &cap);
      e = le != cudaSuccess ? le : ce;
    }
    if (e == cudaSuccess) e = cudaGraphInstantiate(&c->nm_exec, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) {
      c->nm_exec = nullptr;
      cudaGetLastError();
      return fail(c, KDE_E_CUDA, "device Nelder-Mead graph: %s", cudaGetErrorString(e));
    }
    c->nm_key = key;
  }
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (c->profiling) { e0 = next_event(c); e1 = next_event(c); CUDA_TRY(c, cudaEventRecord(e0, st)); }
  {
    Range r("kde.nm_loop");
    CUDA_TRY(c, cudaGraphLaunch(c->nm_exec, st));
  }
  if (c->profiling) CUDA_TRY(c, cudaEventRecord(e1, st));
  unsigned long long flag = 0;
  CUDA_TRY(c, cudaMemcpyAsync(hb, dblk, up, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(c, cudaMemcpyAsync(&flag, w.flag(), sizeof(flag), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(c, cudaStreamSynchronize(st));
  if (flag) return fail(c, KDE_E_INVALID, "whitened sample differences exceed 1e18");
  c->prof_all += 3 * hb->h.rounds + 1;
  if (c->profiling) {   // one interval: the whole loop (decide, prep and pair kernels of every round)
    c->prof_launches += hb->h.rounds;
    c->prof_evals += (double)hb->h.evals * pairs_in_range(n, T, 0, n_tiles(n, T));
  }
  best.x.assign(hb->st.sim[0], hb->st.sim[0] + P);
  best.f = hb->st.fs[0];
  best.iterations = hb->st.it;
  best.stop = hb->st.stop;
  best.evals = hb->h.evals;
  return KDE_OK;
}

}  // namespace host
}  // namespace kde
