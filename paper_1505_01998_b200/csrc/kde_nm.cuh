// kde_nm.cuh — Nelder–Mead over x = vech(H) for LSCV_H ("well known Nelder-Mead";
// parameters, start simplex, ordering and stopping are reading Z8), written once as
// __host__ __device__ code on a fixed-size state so that the host loop (kde_nm.cpp: multi-start,
// speculative batches, multi-rank) and the device-resident loop (kde_nm_dev.cu: one CUDA graph with
// a conditional WHILE node, no host round trip per round) run the same arithmetic: both sides are
// compiled without FMA contraction (x86-64 host code has no FMA; kde_nm_dev.cu is built with
// -fmad=false), so the same objective values give the same decisions bit for bit.
//
// The state machine: propose() lists the points whose objective values the next decision needs,
// accept() takes those values and applies the serial logic (rho = 1, chi = 2, gamma = sigma = 1/2;
// stable order by (f, index); stop on f_worst - f_best <= tol |f_best| or max_iter).  Speculative
// mode proposes reflect, expand, outside and inside contraction together; its decisions equal
// those of serial NM on the same values.  Also here: the Cholesky PD test (pivot > 1e-12 max diag,
// reading Z8) and the LSCV_H finalize of Eq. 30-34, which both loops need.
#pragma once
#include <math.h>
#include <stdint.h>

#include "kde_internal.h"

#ifndef KDE_HD
#define KDE_HD __host__ __device__
#endif
// The device runs this code on one thread per round of the loop (kde_nm_dev.cu), where instruction
// fetch dominates: unrolled copies of these small loops grew the decide kernel to ~1 MB of SASS and
// 12.8 us per round (KDE_DEBUG_NM_TRACE; 8.2 us rolled).  Loops stay rolled on the device (no effect on
// results: the same operations in the same order).
#if defined(__CUDA_ARCH__)
#define KDE_ROLLED _Pragma("unroll 1")
#else
#define KDE_ROLLED
#endif

namespace kde {

constexpr int kNMMaxP = kMaxDim * (kMaxDim + 1) / 2;   // 136 parameters at d = 16

// PMAX = capacity in parameters: kNMMaxP for the host / the global device block, small for the
// device's shared-memory working copy (d <= 4); the arithmetic does not depend on PMAX.
template <int PMAX>
struct NMStateT {
  enum Phase { INIT = 0, STEP = 1, SERIAL_R = 2, SERIAL_1 = 3, SHRINK = 4, DONE = 5 };
  int P = 0;                    // parameters (vertices P + 1)
  int phase = INIT, it = 0, max_iter = 500, stop = 2, serial_pick = 0, speculative = 0;
  double tol = 1e-7, fr = 0.0;
  double sim[PMAX + 1][PMAX];
  double fs[PMAX + 1];
  double xbar[PMAX], xr[PMAX], xe[PMAX], xc[PMAX], xcc[PMAX];
};
using NMState = NMStateT<kNMMaxP>;

// Copy the used part of one state into another of a different capacity.
template <int A, int B>
KDE_HD inline void nm_state_copy(NMStateT<A>& d, const NMStateT<B>& s) {
  d.P = s.P; d.phase = s.phase; d.it = s.it; d.max_iter = s.max_iter; d.stop = s.stop;
  d.serial_pick = s.serial_pick; d.speculative = s.speculative; d.tol = s.tol; d.fr = s.fr;
  KDE_ROLLED
  for (int v = 0; v <= s.P; ++v) {
    d.fs[v] = s.fs[v];
    KDE_ROLLED
    for (int k = 0; k < s.P; ++k) d.sim[v][k] = s.sim[v][k];
  }
  KDE_ROLLED
  for (int k = 0; k < s.P; ++k) {
    d.xbar[k] = s.xbar[k]; d.xr[k] = s.xr[k]; d.xe[k] = s.xe[k]; d.xc[k] = s.xc[k]; d.xcc[k] = s.xcc[k];
  }
}

// r = a + s (b - c), component by component (the one combination formula of the method)
KDE_HD inline void nm_comb(double* r, const double* a, double s, const double* b, const double* c, int P) {
  KDE_ROLLED
  for (int k = 0; k < P; ++k) r[k] = a[k] + s * (b[k] - c[k]);
}

KDE_HD inline void nm_copy(double* d, const double* s, int P) {
  KDE_ROLLED
  for (int k = 0; k < P; ++k) d[k] = s[k];
}

// Sort (stable, by f then vertex index), test the stopping rule, prepare the trial points.
template <class St>
KDE_HD inline void nm_begin_iteration(St& s) {
  const int M = s.P;
  KDE_ROLLED
  for (int i = 1; i <= M; ++i) {               // insertion sort: stable, the order of std::stable_sort
    int j = i;
    while (j > 0 && s.fs[j] < s.fs[j - 1]) {
      const double tf = s.fs[j]; s.fs[j] = s.fs[j - 1]; s.fs[j - 1] = tf;
      KDE_ROLLED
      for (int k = 0; k < s.P; ++k) { const double t = s.sim[j][k]; s.sim[j][k] = s.sim[j - 1][k]; s.sim[j - 1][k] = t; }
      --j;
    }
  }
  if (s.fs[M] - s.fs[0] <= s.tol * fabs(s.fs[0])) { s.stop = 1; s.phase = St::DONE; return; }
  if (s.it >= s.max_iter) { s.stop = 2; s.phase = St::DONE; return; }
  ++s.it;
  KDE_ROLLED
  for (int k = 0; k < s.P; ++k) s.xbar[k] = 0.0;
  KDE_ROLLED
  for (int v = 0; v < M; ++v)
    KDE_ROLLED
    for (int k = 0; k < s.P; ++k) s.xbar[k] += s.sim[v][k];
  KDE_ROLLED
  for (int k = 0; k < s.P; ++k) s.xbar[k] /= (double)M;
  nm_comb(s.xr, s.xbar, 1.0, s.xbar, s.sim[M], s.P);
  nm_comb(s.xe, s.xbar, 2.0, s.xr, s.xbar, s.P);
  nm_comb(s.xc, s.xbar, 0.5, s.xr, s.xbar, s.P);
  nm_comb(s.xcc, s.xbar, 0.5, s.sim[M], s.xbar, s.P);
  s.phase = s.speculative ? St::STEP : St::SERIAL_R;
}

// Points needed next, written row by row (stride OUT) into out; returns how many.
template <class St, int OUT>
KDE_HD inline int nm_propose(const St& s, double (*out)[OUT]) {
  switch (s.phase) {
    case St::INIT:
      KDE_ROLLED
      for (int v = 0; v <= s.P; ++v) nm_copy(out[v], s.sim[v], s.P);
      return s.P + 1;
    case St::STEP:
      nm_copy(out[0], s.xr, s.P); nm_copy(out[1], s.xe, s.P);
      nm_copy(out[2], s.xc, s.P); nm_copy(out[3], s.xcc, s.P);
      return 4;
    case St::SERIAL_R:
      nm_copy(out[0], s.xr, s.P);
      return 1;
    case St::SERIAL_1:
      nm_copy(out[0], s.serial_pick == 1 ? s.xe : (s.serial_pick == 2 ? s.xc : s.xcc), s.P);
      return 1;
    case St::SHRINK:
      KDE_ROLLED
      for (int v = 1; v <= s.P; ++v) nm_comb(out[v - 1], s.sim[0], 0.5, s.sim[v], s.sim[0], s.P);
      return s.P;
    default:
      return 0;
  }
}

// Decide with f_r known and (speculatively or not) the one follow-up value.
template <class St>
KDE_HD inline void nm_decide(St& s, double fr, bool have_follow, double fe, double fc, double fcc) {
  const int M = s.P;
  if (fr < s.fs[0]) {
    if (!have_follow) { s.serial_pick = 1; s.fr = fr; s.phase = St::SERIAL_1; return; }
    if (fe < fr) { nm_copy(s.sim[M], s.xe, s.P); s.fs[M] = fe; } else { nm_copy(s.sim[M], s.xr, s.P); s.fs[M] = fr; }
    nm_begin_iteration(s);
    return;
  }
  if (fr < s.fs[M - 1]) { nm_copy(s.sim[M], s.xr, s.P); s.fs[M] = fr; nm_begin_iteration(s); return; }
  if (fr < s.fs[M]) {
    if (!have_follow) { s.serial_pick = 2; s.fr = fr; s.phase = St::SERIAL_1; return; }
    if (fc <= fr) { nm_copy(s.sim[M], s.xc, s.P); s.fs[M] = fc; nm_begin_iteration(s); return; }
  } else {
    if (!have_follow) { s.serial_pick = 3; s.fr = fr; s.phase = St::SERIAL_1; return; }
    if (fcc < s.fs[M]) { nm_copy(s.sim[M], s.xcc, s.P); s.fs[M] = fcc; nm_begin_iteration(s); return; }
  }
  s.phase = St::SHRINK;
}

// Values g[0 .. count) of the points nm_propose() listed.
template <class St>
KDE_HD inline void nm_accept(St& s, const double* g) {
  switch (s.phase) {
    case St::INIT:
      KDE_ROLLED
      for (int v = 0; v <= s.P; ++v) s.fs[v] = g[v];
      nm_begin_iteration(s);
      break;
    case St::STEP: nm_decide(s, g[0], true, g[1], g[2], g[3]); break;
    case St::SERIAL_R: nm_decide(s, g[0], false, 0.0, 0.0, 0.0); break;
    case St::SERIAL_1: {
      const double v = g[0];
      nm_decide(s, s.fr, true, s.serial_pick == 1 ? v : 0.0, s.serial_pick == 2 ? v : 0.0,
                s.serial_pick == 3 ? v : 0.0);
      break;
    }
    case St::SHRINK:
      KDE_ROLLED
      for (int v = 1; v <= s.P; ++v) {
        nm_comb(s.sim[v], s.sim[0], 0.5, s.sim[v], s.sim[0], s.P);
        s.fs[v] = g[v - 1];
      }
      nm_begin_iteration(s);
      break;
    default: break;
  }
}

// ------------------------------------------------------------------ LSCV_H candidate arithmetic
// Cholesky H = L L^T of vech(H) (row-major lower L) with the relative pivot test (positive
// definiteness, reading Z8): returns false for a non-PD, asymmetric or non-finite H.  det = |H|.
KDE_HD inline int nm_vech_index(int i, int j, int d) {   // entry (i, j), i >= j, of vech
  return j * d - j * (j - 1) / 2 + (i - j);
}

KDE_HD inline bool nm_cholesky_vech(const double* vh, int d, double* L, double* det) {
  double mx = 0.0;
  KDE_ROLLED
  for (int i = 0; i < d; ++i) {
    const double a = vh[nm_vech_index(i, i, d)];
    if (!isfinite(a)) return false;
    mx = fmax(mx, fabs(a));
  }
  KDE_ROLLED
  for (int k = 0; k < d * (d + 1) / 2; ++k)
    if (!isfinite(vh[k])) return false;
  KDE_ROLLED
  for (int i = 0; i < d * d; ++i) L[i] = 0.0;
  KDE_ROLLED
  for (int j = 0; j < d; ++j) {
    double s = vh[nm_vech_index(j, j, d)];
    KDE_ROLLED
    for (int k = 0; k < j; ++k) s -= L[j * d + k] * L[j * d + k];
    if (!(s > 1e-12 * mx)) return false;
    L[j * d + j] = sqrt(s);
    KDE_ROLLED
    for (int i = j + 1; i < d; ++i) {
      double u = vh[nm_vech_index(i, j, d)];
      KDE_ROLLED
      for (int k = 0; k < j; ++k) u -= L[i * d + k] * L[j * d + k];
      L[i * d + j] = u / L[j * d + j];
    }
  }
  double p = 1.0;
  KDE_ROLLED
  for (int i = 0; i < d; ++i) p *= L[i * d + i] * L[i * d + i];
  *det = p;
  return true;
}

// W = sqrt(log2 e / 4) L^-1 (forward substitution), the candidate's whitening.
KDE_HD inline void nm_whitening(const double* L, int d, double scale, double* W) {
  KDE_ROLLED
  for (int col = 0; col < d; ++col)
    KDE_ROLLED
    for (int i = 0; i < d; ++i) {
      double s = (i == col) ? 1.0 : 0.0;
      KDE_ROLLED
      for (int k = 0; k < i; ++k) s -= L[i * d + k] * W[k * d + col];
      W[i * d + col] = s / L[i * d + i];
    }
  KDE_ROLLED
  for (int i = 0; i < d * d; ++i) W[i] *= scale;
}

// g(H) of Eq. 30-34 from the raw sums S1 = sum e^{-q/4}, S2 = sum e^{-q/2}, with
// c4 = (4 pi)^{-d/2} |H|^{-1/2}, c2 = (2 pi)^{-d/2} |H|^{-1/2}; pow4 = (4 pi)^{-d/2} and
// pow2 = (2 pi)^{-d/2} are passed in (computed once on the host).
KDE_HD inline double nm_lscv_H_finalize(double n, double pow4, double pow2, double det, double S1, double S2) {
  const double c4 = pow4 / sqrt(det);
  const double c2 = pow2 / sqrt(det);
  return 2.0 * (c4 * S1 - 2.0 * c2 * S2) / (n * n) + c4 / n;
}

}  // namespace kde
