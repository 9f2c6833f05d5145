// kde_nm_dev.cu — the device-resident Nelder–Mead loop of LSCV_H (reading Z8; the
// objective g(H) of Eq. 30-34).  The paper calls the optimizer inherently sequential with one g(H)
// per step; on B200 a host round trip per step (~30 us: D2H, sync, host decision, launches)
// is ~17% of a C3 step, so the whole loop runs as ONE CUDA graph:
//
//     WHILE (cond) {  nm_decide_kernel  ->  prep_sets_kernel  ->  pair_kernel_sets  }
//
// nm_decide_kernel (one thread decides; the CTA loads and stores its state) takes the previous round's exact limbs, finalises g(H) for each
// proposal (non-PD: the penalty), advances the state machine of kde_nm.cuh, proposes the next
// points, tests them for positive definiteness and writes each PD candidate's whitening
// parameters; prep_sets_kernel whitens the samples once per candidate and the pair kernel reads
// the candidate count from device memory.  When the state machine stops, the decide kernel sets
// the graph's conditional to 0.  The NM arithmetic is the host loop's (kde_nm.cuh), and this file
// is compiled with -fmad=false, so the device loop makes the same decisions on the same values.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
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
  unsigned long long* trace;   // diagnostics (KDE_DEBUG_NM_TRACE): 16 globaltimer slots per decide call, or null
  int calls;                   // decide-kernel calls so far
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

__device__ __forceinline__ unsigned long long nm_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// One decision step (see the file comment) on a state `s` of any capacity.  lsrc: the previous
// round's limbs (h.limbs or a shared-memory copy); tp: trace slots of this call (diagnostics) or null.
// Loops stay rolled: on one thread the kernel's time is instruction latency, and a compact body is
// cheaper to fetch (kde_nm.cuh).
template <class St, int OUT>
__device__ void decide_body(NMDevHeader& h, St& s, double (*prop)[OUT], double* g, double* det, int* slot,
                            double* L, const unsigned long long* lsrc, cudaGraphConditionalHandle cond,
                            unsigned long long* tp = nullptr) {
  if (h.pending) {                                   // the previous round's values
#pragma unroll 1
    for (int i = 0; i < h.n_prop; ++i) {
      const int k = slot[i];
      g[i] = k < 0 ? h.penalty
                   : nm_lscv_H_finalize(h.nn, h.pow4, h.pow2, det[i],
                                        limbs_value(lsrc + (size_t)(2 * k) * kLimbs, h.S),
                                        limbs_value(lsrc + (size_t)(2 * k + 1) * kLimbs, h.S));
    }
    if (tp) tp[4] = nm_ns();
    h.evals += h.n_sets;
    nm_accept(s, g);
    h.pending = 0;
    if (tp) tp[5] = nm_ns();
  }
  while (true) {
    if (s.phase == St::DONE) {
      h.n_sets = 0;
      cudaGraphSetConditional(cond, 0);
      return;
    }
    h.n_prop = nm_propose(s, prop);
    if (tp) tp[6] = nm_ns();
    h.n_sets = 0;
#pragma unroll 1
    for (int i = 0; i < h.n_prop; ++i) {
      double dt = 0.0;
      if (nm_cholesky_vech(prop[i], h.d, L, &dt)) {
        const int k = h.n_sets++;
        slot[i] = k;
        det[i] = dt;
        nm_whitening(L, h.d, h.wscale, h.pp[k].W);
#pragma unroll 1
        for (int a = 0; a < h.d; ++a) h.pp[k].mean[a] = h.mean[a];
      } else {
        slot[i] = -1;
      }
    }
    if (h.n_sets == 0) {                             // every proposal non-PD: no GPU pass needed
#pragma unroll 1
      for (int i = 0; i < h.n_prop; ++i) g[i] = h.penalty;
      nm_accept(s, g);
      continue;
    }
    if (tp) tp[7] = nm_ns();
#pragma unroll 1
    for (size_t k = 0; k < (size_t)2 * h.n_sets * kLimbs; ++k) h.limbs[k] = 0ull;
    *h.work = 0ull;
    h.pending = 1;
    ++h.rounds;
    return;
  }
}

// d <= 4 (P <= 10): the decision runs on a shared-memory copy of the state, the header and the
// previous round's limbs, which the CTA's threads load and store in parallel; one thread decides.
// Larger d: one thread on the global block.  Two kernels, so the small one stays compact.
// EARLY (a decide launched programmatically after a pair kernel, whose grid leaves it one CTA slot):
// the state, which only this kernel writes, is loaded while the pair pass is still running, the limbs
// after griddepcontrol.wait.  Measured per round (KDE_DEBUG_NM_TRACE, C3): 15.2 us with one thread and
// unrolled loops (~1 MB of SASS), 8.2 us rolled, 7.0 us with the early state load; a rehearsal of the
// decision during the pair pass (to warm the instruction cache) took 24 us next to the pair CTAs and
// did not shorten the real one: what is left is the latency of the fp64 code on one thread.
constexpr int kSmallP = 10;
constexpr int kNMTraceCalls = 1024;
constexpr int kDecideThreads = 128;

template <class T>
__device__ __forceinline__ void copy_words(T* dst, const T* src, int tid) {
  static_assert(sizeof(T) % 8 == 0 && alignof(T) >= 8, "word copy");
  auto* d = reinterpret_cast<unsigned long long*>(dst);
  auto* q = reinterpret_cast<const unsigned long long*>(src);
  for (int i = tid; i < (int)(sizeof(T) / 8); i += kDecideThreads) d[i] = q[i];
}

// Parallel copy of the used part of a state (the elements nm_state_copy copies).
template <int A, int B>
__device__ __forceinline__ void state_copy_par(NMStateT<A>& d, const NMStateT<B>& s, int P, int tid) {
  if (tid == 0) {
    d.P = s.P; d.phase = s.phase; d.it = s.it; d.max_iter = s.max_iter; d.stop = s.stop;
    d.serial_pick = s.serial_pick; d.speculative = s.speculative; d.tol = s.tol; d.fr = s.fr;
  }
  for (int i = tid; i < (P + 1) * P; i += kDecideThreads) d.sim[i / P][i % P] = s.sim[i / P][i % P];
  for (int i = tid; i <= P; i += kDecideThreads) d.fs[i] = s.fs[i];
  for (int i = tid; i < P; i += kDecideThreads) {
    d.xbar[i] = s.xbar[i]; d.xr[i] = s.xr[i]; d.xe[i] = s.xe[i]; d.xc[i] = s.xc[i]; d.xcc[i] = s.xcc[i];
  }
}

template <bool SMALL>
__global__ void __launch_bounds__(kDecideThreads) nm_decide_kernel(NMDevBlock* b, cudaGraphConditionalHandle cond,
                                                                   int early) {
  const int tid = threadIdx.x;
  unsigned long long* trace = b->h.trace;
  const int call = b->h.calls;
  if constexpr (SMALL) {
    const int P = b->st.P;
    __shared__ alignas(16) unsigned char sbuf[sizeof(NMStateT<kSmallP>)];
    __shared__ double sprop[kSmallP + 1][kSmallP], sg[kSmallP + 1], sdet[kSmallP + 1], sL[kMaxDim * kMaxDim];
    __shared__ int sslot[kSmallP + 1];
    __shared__ NMDevHeader sh;
    __shared__ unsigned long long slimbs[2 * (kSmallP + 1) * kLimbs];
    NMStateT<kSmallP>& ss = *reinterpret_cast<NMStateT<kSmallP>*>(sbuf);
    copy_words(&sh, &b->h, tid);
    state_copy_par(ss, b->st, P, tid);
    for (int i = tid; i <= kSmallP; i += kDecideThreads) { sdet[i] = b->det[i]; sslot[i] = b->slot[i]; }
    if (early) pdl_wait();   // the pair pass has completed: its limbs are visible
    if (tid == 0 && trace && call < kNMTraceCalls) trace[16 * call] = nm_ns();
    const unsigned long long* gl = b->h.limbs;
    const int nl = 2 * min(b->h.max_sets, kSmallP + 1) * kLimbs;
    for (int i = tid; i < nl; i += kDecideThreads) slimbs[i] = gl[i];
    __syncthreads();
    if (tid == 0)
      decide_body(sh, ss, sprop, sg, sdet, sslot, sL, slimbs, cond,
                  trace && call < kNMTraceCalls ? trace + 16 * call : nullptr);
    __syncthreads();
    state_copy_par(b->st, ss, P, tid);
    for (int i = tid; i <= kSmallP; i += kDecideThreads) { b->det[i] = sdet[i]; b->slot[i] = sslot[i]; }
    if (tid == 0) sh.calls = call + 1 < kNMTraceCalls ? call + 1 : kNMTraceCalls - 1;
    __syncthreads();
    copy_words(&b->h, &sh, tid);
  } else {
    if (early) pdl_wait();
    if (tid == 0) {
      if (trace && call < kNMTraceCalls) trace[16 * call] = nm_ns();
      decide_body(b->h, b->st, b->prop, b->g, b->det, b->slot, b->L, b->h.limbs, cond);
      b->h.calls = call + 1 < kNMTraceCalls ? call + 1 : kNMTraceCalls - 1;
    }
  }
  if (tid == 0 && trace && call < kNMTraceCalls) trace[16 * call + 1] = nm_ns();
}

// Programmatic dependent launches inside the loop body (KDE_DEBUG_NM_PDL=0 turns them off); rounds per
// evaluation of the loop condition (KDE_DEBUG_NM_UNROLL, default 4).
static bool nm_pdl() {
  const char* e = std::getenv("KDE_DEBUG_NM_PDL");
  return !(e && std::atoi(e) == 0);
}
static int nm_unroll() {
  const char* e = std::getenv("KDE_DEBUG_NM_UNROLL");
  const int u = e ? std::atoi(e) : 4;
  return u < 1 ? 1 : (u > 16 ? 16 : u);
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
  TRY(gpu_sorted_rows(c, X, n, d, &X));   // by coordinate 0 (no-op when the caller sorted already)
  TRY(grow(c, &c->white_ws, &c->white_bytes, (size_t)max_sets * set_floats * sizeof(float)));
  const size_t blk = (sizeof(NMDevBlock) + 255) & ~size_t(255);
  const bool tracing = std::getenv("KDE_DEBUG_NM_TRACE") && std::atoi(std::getenv("KDE_DEBUG_NM_TRACE")) == 1;
  const size_t pp_b = ((size_t)max_sets * sizeof(PrepParams) + 255) & ~size_t(255);
  const size_t tr_b = tracing ? 16 * kNMTraceCalls * sizeof(unsigned long long) : 0;
  TRY(grow(c, &c->nm_ws, &c->nm_bytes, blk + pp_b + tr_b));
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
  h.trace = tracing ? reinterpret_cast<unsigned long long*>(static_cast<char*>(c->nm_ws) + blk + pp_b) : nullptr;
  h.calls = 0;
  h.work = w.limbs + (size_t)2 * max_sets * kLimbs;
  NMState& s = hb->st;
  s.P = P; s.max_iter = max_iter; s.tol = tol; s.speculative = 0; s.phase = NMState::INIT; s.it = 0; s.stop = 2;
  for (int v = 0; v <= P; ++v)
    for (int k = 0; k < P; ++k) s.sim[v][k] = sim[v][k];
  cudaStream_t st = c->stream;
  CUDA_TRY(c, cudaMemcpyAsync(dblk, hb, up, cudaMemcpyHostToDevice, st));
  // prep flags .. the skipped-pair counter (kSkippedSlot)
  CUDA_TRY(c, cudaMemsetAsync(w.flag(), 0, (kSkippedSlot - 408 + 1) * sizeof(unsigned long long), st));
  if (tracing) CUDA_TRY(c, cudaMemsetAsync(h.trace, 0, tr_b, st));
  // g, det, slot: the decide kernel copies all kSmallP + 1 entries (only the first n_prop are ever used)
  CUDA_TRY(c, cudaMemsetAsync(&dblk->g, 0, offsetof(NMDevBlock, L) - offsetof(NMDevBlock, g), st));
  // the graph (built once per key, replayed afterwards)
  const std::vector<uintptr_t> key = {(uintptr_t)X, (uintptr_t)n, (uintptr_t)d, (uintptr_t)w.limbs,
                                      (uintptr_t)Yw, (uintptr_t)dblk, (uintptr_t)T, (uintptr_t)tracing,
                                      (uintptr_t)nm_pdl(), (uintptr_t)nm_unroll()};
  if (!(c->nm_exec && key == c->nm_key)) {
    Range r("kde.nm_capture");
    if (c->nm_exec) { cudaGraphExecDestroy(c->nm_exec); c->nm_exec = nullptr; }
    if (!c->cap_stream) CUDA_TRY(c, cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
    // WHILE (cond) { nm_unroll() x [decide -> whiten -> pair pass] }: the conditional is evaluated once
    // per nm_unroll() rounds; after the decision that stops the search the rest of the body finds no
    // sets and returns at once.  Within the body every launch after the first is programmatic (PDL),
    // and a pair grid followed by a decide leaves it one CTA slot (its state loads overlap the pass).
    const bool pdl = nm_pdl();
    cudaGraph_t g = nullptr;
    CUDA_TRY(c, cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle cond;
    cudaError_t e = cudaGraphConditionalHandleCreate(&cond, g, 1, cudaGraphCondAssignDefault);
    auto launch_decide = [&](bool early) -> cudaError_t {
      cudaLaunchConfig_t lc = {};
      lc.gridDim = dim3(1);
      lc.blockDim = dim3(P <= kSmallP ? kDecideThreads : 32);
      lc.stream = c->cap_stream;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      lc.attrs = at;
      lc.numAttrs = early ? 1 : 0;
      return P <= kSmallP ? cudaLaunchKernelEx(&lc, nm_decide_kernel<true>, dblk, cond, (int)early)
                          : cudaLaunchKernelEx(&lc, nm_decide_kernel<false>, dblk, cond, (int)early);
    };
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
      cudaError_t le = cudaSuccess;
      const int U = nm_unroll();
      for (int u = 0; u < U && le == cudaSuccess; ++u) {
        le = launch_decide(pdl && u > 0);
        if (le == cudaSuccess)
          le = kde::launch_prep_sets(X, n, d, pp, &dblk->h.n_sets, max_sets, Yw, set_floats, ld, c->cap_stream,
                                     w.flag(), h.trace, &dblk->h.calls, pdl);
        if (le == cudaSuccess) {
          kde::LaunchCfg cfg;
          cfg.X = Yw; cfg.n = n; cfg.ld = ld; cfg.tile = T; cfg.scale_exp = h.S; cfg.limbs = w.limbs;
          cfg.n_out = 2; cfg.stream = c->cap_stream; cfg.sm_count = c->sm_count; cfg.clamp = nullptr;
          cfg.n_sets = max_sets; cfg.set_stride = set_floats; cfg.n_sets_dev = &dblk->h.n_sets;
          cfg.work = w.limbs + (size_t)2 * max_sets * kLimbs;
          cfg.skip_s = lscv_skip_s(1.0, n);
          cfg.skipped = reinterpret_cast<unsigned long long*>(w.small + kSkippedSlot);
          cfg.pdl = pdl;
          cfg.reserve_ctas = pdl && u + 1 < U ? 1 : 0;   // the next decide's slot
          shard_range(n_tiles(n, T), 0, 1, &cfg.tile_begin, &cfg.tile_end);
          le = kde::launch_lscv_white(d, cfg);
        }
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
  unsigned long long fl[kSkippedSlot - 408 + 1];
  CUDA_TRY(c, cudaMemcpyAsync(hb, dblk, up, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(c, cudaMemcpyAsync(fl, w.flag(), sizeof(fl), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(c, cudaStreamSynchronize(st));
  if (fl[0]) return fail(c, KDE_E_INVALID, "whitened sample differences exceed 1e18");
  if (tracing) {   // diagnostics: the per-round timeline of the loop (globaltimer ns) to stderr
    const int calls = hb->h.calls;
    std::vector<unsigned long long> tr((size_t)16 * kNMTraceCalls);
    CUDA_TRY(c, cudaMemcpy(tr.data(), h.trace, tr.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    double sd = 0, sg = 0, sp = 0, sr = 0, fin = 0, acc = 0, prp = 0, chol = 0;
    int nr = 0;
    for (int i = 0; i + 1 < calls; ++i) {
      const unsigned long long* t = tr.data() + 16 * (size_t)i;
      if (t[2] == 0 || t[16] == 0) continue;   // a decide call that launched no pass
      sd += (double)(t[1] - t[0]);
      sg += (double)(t[2] - t[1]);
      sp += (double)(t[3] - t[2]);
      sr += (double)(t[16] - t[3]);
      if (t[4]) { fin += (double)(t[4] - t[0]); acc += (double)(t[5] - t[4]); }
      if (t[6]) { prp += (double)(t[6] - std::max(t[5], t[0])); chol += (double)(t[7] - t[6]); }
      ++nr;
    }
    if (nr > 0) {
      std::fprintf(stderr, "nm_trace decide parts (us): load+finalize %.3f accept %.3f propose %.3f cholesky+whiten %.3f\n",
                   fin / nr / 1e3, acc / nr / 1e3, prp / nr / 1e3, chol / nr / 1e3);
      std::fprintf(stderr, "nm_trace rounds=%d decide_us=%.3f decide_to_prep_us=%.3f prep_us=%.3f prep_to_next_decide_us=%.3f\n",
                   nr, sd / nr / 1e3, sg / nr / 1e3, sp / nr / 1e3, sr / nr / 1e3);
    }
  }
  c->prof_all += 3 * hb->h.calls;   // decide, whitening and pair kernel per decide call (unrolled body)
  if (c->profiling) {   // one interval: the whole loop (decide, prep and pair kernels of every round)
    c->prof_launches += hb->h.rounds;
    c->prof_evals += (double)hb->h.evals * pairs_in_range(n, T, 0, n_tiles(n, T)) - (double)fl[kSkippedSlot - 408];
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
