#pragma once
// kde_pair.cuh — sm_100a kernels of the all-pairs kernel-sum engine (arxiv 1505.01998).
//
// One persistent pair-kernel family evaluates RR_fun(A) = sum_{i<j} fun(A_i - A_j) (P:472,
// Sec. 5.4) and RR^v_fun (Sec. 5.5) for a batch of candidate bandwidths per pair
// visit.  Design:
//  * work unit = one T x T tile (l, q), q <= l, of the upper-triangular pair matrix,
//    numbered column by column and mapped back with Eq. 42-43 + an integer fix-up;
//    variants: a column chunk of a tile (small-n Psi, CS > 1) or a (data set, tile) pair
//    (LSCV_H: one whitened data set per candidate, pair_kernel_sets);
//  * persistent CTAs claim the units of their rank's tiles (round-robin chunks of tile ids,
//    kde_tiles.cuh shard_tile) dynamically, one unit ahead of the one they evaluate;
//  * the T column samples (D rows) of the next tile are staged in shared memory by TMA bulk
//    copies (cp.async.bulk + mbarrier, double-buffered); the T row samples sit in registers
//    (R per thread); columns are read back with broadcast LDS.128;
//  * per eval: FP32 difference and square (sum of squares), one MUFU.EX2 (or, for a quarter of
//    the LSCV_h terms, a software exp2 on the FMA pipe), Horner or accumulate FMAs;
//  * every tile's partial is reduced in a fixed order (fp32 per thread -> fp64 warp butterfly ->
//    fixed cross-warp order) and added as exact fixed-point limbs with integer atomics, so the
//    result is independent of grid size, tile-to-CTA assignment, batch composition and GPU count.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include <type_traits>

#include "kde_device.cuh"
#include "kde_internal.h"
#include "kde_tiles.cuh"

namespace kde {

// LSCV_h candidates per pair visit: d <= 4: 8 at 4 CTAs/SM (64 registers); larger d: 16, then 8,
// so that no instantiation spills.
constexpr int nb_scalar(int d) { return d <= 4 ? 8 : (d <= 12 ? 16 : 8); }


// ------------------------------------------------------------------ small device helpers

// Per-tile epilogue: fixed-order reduction of NOUT per-thread values, then limb atomics.
template <int NOUT, int NT>
__device__ __forceinline__ void commit_tile(double (&v)[NOUT], double* red,
                                            unsigned long long* limbs, int S) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NOUT; ++k) v[k] = warp_sum(v[k]);
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NOUT; ++k) red[w * NOUT + k] = v[k];
  }
  __syncthreads();
  for (int k = threadIdx.x; k < NOUT; k += NT) {
    double s = red[k];
#pragma unroll
    for (int ww = 1; ww < NW; ++ww) s += red[ww * NOUT + k];
    add_limbs(s, S, limbs + (size_t)k * kLimbs);
  }
  __syncthreads();
}

struct Args {
  const float* X;
  int64_t n, ld, tile_begin, tile_end;
  int scale_exp;
  unsigned long long* limbs;
  const unsigned long long* clamp;   // device flag set by the prep kernel (Psi only), or null
  int n_sets;                        // data sets (work unit = (set, tile)), set s at X + s*set_stride
  int64_t set_stride;
  const double* Y64;                 // Psi: fp64 scaled sorted samples (rows), or null
  const float* centres;              // Psi: per-column-tile centres c_l
  unsigned long long* skipped;       // Psi: counter of pairs in skipped tiles, or null
  const int* n_sets_dev;             // sets: the count in device memory (device-resident loops), or null
  double skip_gap;                   // Psi: tiles with a larger sorted gap are exactly zero
  unsigned long long* work;          // dynamic scheduling: unit counter (zero at launch), or null
  float skip_s;                      // LSCV on coordinate-0-sorted data: skip bound on s (+inf: never)
  int part_rank, part_world;         // tile_begin/tile_end index this rank's round-robin tiles (shard_tile)
  const double* skip_gap_dev;        // Psi: skip_gap in device memory (PLUGIN chain), or null
  const float* skip_s_sets;          // LSCV_H sets: per-set skip bound on s (data-aware selection), or null
  const float* skip_c_dev;           // LSCV_h batch: per-candidate skip bounds on s (data-aware), or null
};

// Work distribution.  Static: CTA b takes units b, b + grid, ...  Dynamic (a.work != null): CTA b
// starts with unit b and then takes grid + atomicAdd(work, 1) one unit ahead (so the next unit's TMA
// still overlaps the current one), broadcast through shared memory; units whose cost varies
// (skipped exact-zero tiles, diagonal tiles, ragged tails) then cannot leave a CTA behind.  The
// result is independent of the assignment (exact limbs), so both are deterministic.
__device__ __forceinline__ int64_t next_unit_issue(const Args& a, int64_t u, int64_t* s_next, uint32_t k) {
  if (a.work == nullptr) return u + gridDim.x;
  if (threadIdx.x == 0) s_next[(k + 1) & 1] = (int64_t)gridDim.x + (int64_t)atomicAdd(a.work, 1ull);
  __syncthreads();
  return s_next[(k + 1) & 1];
}

// ------------------------------------------------------------------ functors

// Psi_r: term He_r(u) exp(-u^2/2) with x pre-scaled by 1/g, so s = (x_i'-x_j')^2 = u^2.
// He_r is a polynomial in s with integer coefficients.  Shifting by the mean of
// its roots, t = s - K with K = r - 1, removes the next-to-leading term and keeps the
// coefficients exact integers (depressed form; expand (t+K) to recover P:231/P:247):
//     He_4 = t^2 - 6,   He_6 = t (t^2 - 30) - 40,
// and t comes from the difference in one FFMA, t = fma(d, d, -K): one FP32 op per eval fewer
// than Horner in s (r = 6: 6 instead of 7).  He_8 stays Horner in s (its depressed form
// ((t^2 - 84) t - 224) t + 252 cancels 40x near s = 0).  exp(-s/2) = 2^(s c0), c0 = -log2(e)/2, is taken
// from MUFU.EX2 as
//     2^(s c0) = ex2(t c0 + o_k) * 2^(K c0 - o_k),   o_k = fp32(K c0 - 16 - r/8 - p/16),
// k = (p, r) = accumulator class: r = the row slot (0..7), p = the tile-id parity, 16 classes;
// the factor 2^(K c0 - o_k) is applied exactly in fp64 at the flush.  The MUFU input is then
// s c0 - 16 - k/16 up to one rounding: MUFU.EX2's relative error has a near-constant bias
// (-5.1e-8) only for inputs in [-32,-16), and a different, input-dependent one on (-1, 0] where
// the dominant near pairs live; the sums of Psi_r cancel 1000-5000x at the PLUGIN bandwidths, so
// that bias pattern alone cost 2e-5..5e-5 relative.  Offsetting into one binade and averaging
// over 16 fractional shifts brings Psi-hat to ~1e-6 at C4 at no per-eval cost (measured against
// the oracle: 8 shifts 2.7e-6, 16 shifts 5.4e-7, 32 shifts 8.9e-7).
template <int RORD, int NT_, int CS_ = 1>
struct FPsi {
  static constexpr int NT = NT_, D = 1, R = 8, T = NT_ * 8, NOUT = 2, MINB = 768 / NT_;
  static constexpr int CS = CS_, CW = T / CS_;                     // column chunks per tile, width
  static constexpr int CH = CS_ > 1 ? CW : (T < 1024 ? T : 1024);  // columns per fp64 flush
  static constexpr int NP = R / 2;   // row pairs (r = 2p, 2p+1) packed into fp32x2 lanes
  static constexpr int G = 16;       // columns per compensated group
  // K: the shift of the depressed form (r = 4, 6); r = 8 keeps Horner in s = u^2 (K = 0): its depressed
  // form cancels 40x at s = 0 (2401 - 4116 + 1568 + 252 = 105) and measured 1.3e-5 worst case
  // (tests/diag/fuzz_wide.py, 300 cases) against 1.1e-6 for Horner in s.
  static constexpr float K = RORD == 8 ? 0.f : (float)(RORD - 1);
  static constexpr bool kClampable = true, kSets = false, kCentred = true;
  using Params = PsiParams;
  f2 xr[NP];
  double acc, accA;
  int jbase;   // first column of this work unit's chunk (CS > 1)
  int par;     // tile-id parity: second index of the MUFU offset class (16 classes)

  // Rows are interleaved: thread t owns rows q*T + 8t + r, r = 0..7.  The data are sorted
  // (kde_selectors.cpp), so the 8 row classes r see statistically identical distances; the
  // tile-id parity p doubles the classes across tiles.
  // Tile-local centring: the columns of tile column l arrive as fp32(y_j - c_l)
  // and the rows are formed here as fp32(y_i - c_l) from the fp64 y, so a difference carries the
  // fp32 rounding of |y - c_l| (about |u| plus the tile's span on sorted data) instead of |y|:
  // for small bandwidths |y| = |x - mean|/g reaches 10^2..10^3 and that input rounding alone
  // cost 2.3e-5 relative at n = 40 000, g = 0.02 (emulated; measured 2.4e-5 on the GPU).
  __device__ __forceinline__ void load_rows_c(const double* __restrict__ Y64, int64_t i0, float c) {
    const double2* p = reinterpret_cast<const double2*>(Y64 + i0);
    const double cc = (double)c;
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      const double2 u = __ldg(p + q);
      xr[q] = pk(__double2float_rn(u.x - cc), __double2float_rn(u.y - cc));
    }
    acc = 0.0;
    accA = 0.0;
  }
  static __device__ __forceinline__ int64_t row0(int64_t q) { return q * T + 8 * (int64_t)threadIdx.x; }

  // He_r(t + K): depressed form for r = 4, 6; Horner in s for r = 8 (K = 0); two lanes at once.
  __device__ __forceinline__ f2 poly(f2 t) const {
    if (RORD == 4) return fma2(t, t, pk(-6.f, -6.f));
    if (RORD == 6) return fma2(fma2(t, t, pk(-30.f, -30.f)), t, pk(-40.f, -40.f));
    return fma2(fma2(fma2(add2(t, pk(-28.f, -28.f)), t, pk(210.f, 210.f)), t, pk(-420.f, -420.f)), t,
                pk(105.f, 105.f));   // r = 8: Horner in s (t = s)
  }

  // Accumulation: the G = 16 terms of one column group of a row are summed in
  // fp32 (sorted data: the terms of a group have similar magnitude), then added to the row's
  // running sum with Fast2Sum (rounding error kept in a compensation register); fp64 flush
  // every 1024 columns.  A plain fp32 running sum drops the one-signed far-pair tail terms
  // (~1e-7..1e-6) next to near-pair sums (~10): measured -1.4e-5 relative at T=2048.
  template <bool MASK, bool CLAMP = false>
  __device__ __forceinline__ void compute(const float* __restrict__ sc, const Params& p, bool diag,
                                          int jlim) {
    const int ib = 8 * threadIdx.x;   // local index of row r is ib + r
    const f2 c0 = pk(p.c0, p.c0);
    const f2 mk = pk(-K, -K);
    f2 o[NP];
#pragma unroll
    for (int q = 0; q < NP; ++q) o[q] = reinterpret_cast<const f2*>(p.o + 8 * par)[q];   // 64-bit constant loads
    const int J0 = CS > 1 ? jbase : 0, J1 = CS > 1 ? jbase + CW : T;
    for (int jc = J0; jc < J1; jc += CH) {
      if (MASK && jc >= jlim) break;
      f2 a[NP], cmp[NP];
      float aabs = 0.f;
#pragma unroll
      for (int q = 0; q < NP; ++q) a[q] = cmp[q] = pk(0.f, 0.f);
#pragma unroll 2   // two 16-column groups per iteration (C4 step 250.1 -> 247.1 ms; x4: 258 ms)
      for (int j = jc; j < jc + CH; j += G) {
        f2 grp[NP];
#pragma unroll
        for (int q = 0; q < NP; ++q) grp[q] = pk(0.f, 0.f);
#pragma unroll
        for (int j4 = 0; j4 < G; j4 += 4) {
          const float4 c4 = *reinterpret_cast<const float4*>(sc + j + j4);
          const float cv[4] = {c4.x, c4.y, c4.z, c4.w};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
#pragma unroll
            for (int q = 0; q < NP; ++q) {
              const f2 d = sub2(xr[q], pk(cv[k], cv[k]));
              f2 t = fma2(d, d, mk);                        // t = s - K, one rounding
              if (MASK || CLAMP) {
                // t >= 1e4 gives 2^(-7213) == 0 exactly.  CLAMP (data with |x'| > 3e4, flagged
                // by the prep kernel) keeps He_r finite for far outliers (t^4 overflows fp32
                // beyond t ~ 4e9), so no inf * 0 = NaN; other data never need it.
                float t0, t1;
                upk(t, t0, t1);
                if (CLAMP) {
                  t0 = fminf(t0, 1.0e4f);
                  t1 = fminf(t1, 1.0e4f);
                }
                if (MASK) {
                  const int jj = j + j4 + k;
                  const bool ok0 = (jj < jlim) && (!diag || jj > ib + 2 * q);
                  const bool ok1 = (jj < jlim) && (!diag || jj > ib + 2 * q + 1);
                  t0 = ok0 ? t0 : 1.0e4f;
                  t1 = ok1 ? t1 : 1.0e4f;
                }
                t = pk(t0, t1);
              }
              float a0, a1;
              upk(fma2(t, c0, o[q]), a0, a1);
              const f2 e = pk(ex2(a0), ex2(a1));
              grp[q] = fma2(poly(t), e, grp[q]);
            }
          }
        }
#pragma unroll
        for (int q = 0; q < NP; ++q) {
          const f2 s2 = add2(a[q], grp[q]);                 // Fast2Sum(a, grp), per lane
          const f2 z = sub2(s2, a[q]);
          cmp[q] = add2(cmp[q], sub2(grp[q], z));
          a[q] = s2;
          float g0, g1;                                     // cancellation estimate: sum of
          upk(grp[q], g0, g1);                              // |16-column group sums| (FADD |.|)
          aabs = __fadd_rn(aabs, fabsf(g0));
          aabs = __fadd_rn(aabs, fabsf(g1));
        }
      }
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < NP; ++q) {
        float a0, a1, c0_, c1_;
        upk(a[q], a0, a1);
        upk(cmp[q], c0_, c1_);
        s += ((double)a0 + (double)c0_) * p.fac[8 * par + 2 * q];
        s += ((double)a1 + (double)c1_) * p.fac[8 * par + 2 * q + 1];
      }
      acc += s;
      accA += (double)aabs;
    }
  }

  // v[0] = the tile's sum; v[1] = its cancellation estimate A (sum of |group sums|, scaled by the
  // middle offset class's factor: an estimate within 2^(+-7/16) of the exact scaling).
  __device__ __forceinline__ void outputs(double (&v)[NOUT], const Params& p) const {
    v[0] = acc;
    v[1] = accA * p.fac[8 * par + 4];
  }
};

// LSCV_h (any d): data pre-whitened and scaled, x' = sqrt(log2 e / 4) L^-1 (x - mean) with
// Sigma = L L^T, so s = |x_i' - x_j'|^2 = (log2 e / 4) S(v) (S(v) of Eq. 37) and for candidate
// h_c:  e = 2^(s * kappa_c) = exp(-S(v)/(4 h_c^2)),  e^2 = exp(-S(v)/(2 h_c^2)).
// The thread's two rows are packed in fp32x2 lanes (lane-exact, halves the issue slots).
// UNIT (LSCV_H, one candidate per data set): the data are whitened by the candidate itself,
// x' = sqrt(log2 e / 4) L_c^-1 (x - mean) with H_c = L_c L_c^T, so s = (log2 e / 4) v^T H_c^-1 v
// and e = 2^-s (the negation is a MUFU operand modifier): 2d + 2 FP32 ops per eval.
// SWM (LSCV_h): a 16-bit column mask; column j takes its exponentials from the software exp2 on the
// FMA pipe (exp2_sw2_fast) instead of MUFU.EX2 when bit (j mod 16) is set (chosen by column, so a
// candidate's sum does not depend on its batch).  SWM = 0: MUFU only.  SWSEL: the older exp2_sw2
// (compare + select to exactly 0 below -125) instead of the clamp-only variant.
template <int D_, int NT_, int NB_, bool UNIT = false, unsigned SWM = 0, int MINB_ = 0, bool SWSEL = false,
          bool CMAJ = false, bool SWFMA = false, int UNR_ = 0>
struct FLscvScalar {
  static_assert(!UNIT || NB_ == 1, "UNIT sets carry one candidate");
  static constexpr int NT = NT_, D = D_, R = 2, T = NT_ * 2, NB = NB_, NOUT = 2 * NB_;
  // UNIT (LSCV_H sets): d <= 3 at 4 CTAs of 256 (64 registers); d = 4 at 3 CTAs with the column loop
  // unrolled x4 (C5 2.81 s vs 2.87 s at 4 CTAs; the same change costs C3 (d = 2) 4.5%)
  static constexpr int MINB = MINB_ > 0 ? MINB_ : (UNIT && D <= 3 ? 1024 : (UNIT && D == 4 ? 768 : 512)) / NT_;
  // column-loop unroll: UNIT d <= 2 x8 (C3 pair time 15.64 -> 15.37 ms), d = 3, 4 x4 (no spills);
  // LSCV_h with software-exp columns: 16 columns per iteration (the mask period)
  static constexpr bool SW = SWM != 0;
  static constexpr int STEP = SW ? 16 : 4;
  static constexpr int UNR = UNR_ > 0 ? UNR_ : (UNIT && D <= 2 ? 8 : (UNIT && D <= 4 ? 4 : 1));
  static constexpr bool kClampable = false, kSets = UNIT;
  static constexpr int CS = 1;
  using Params = LscvScalarParams;
  f2 xr[D];
  f2 a1[NB], a2[NB];
  int par;   // unused (interface shared with FPsi)

  __device__ __forceinline__ void load_rows(const float* __restrict__ X, int64_t ld,
                                            int64_t i0) {
#pragma unroll
    for (int a = 0; a < D; ++a) xr[a] = pk(__ldg(X + a * ld + i0), __ldg(X + a * ld + i0 + NT));
#pragma unroll
    for (int c = 0; c < NB; ++c) a1[c] = a2[c] = pk(0.f, 0.f);
  }

  // One candidate's term for one column (s = the pair's whitened squared distance, both lanes).
  template <bool MASK>
  __device__ __forceinline__ void term(f2 s, int c, int col, bool ok0, bool ok1, const Params& p) {
    f2 e;
    if (SW && ((SWM >> (col & 15)) & 1u)) {
      if (SWSEL) {
        e = exp2_sw2(mul2(s, pk(p.kappa[c], p.kappa[c])));
      } else {
        e = SWFMA ? exp2_sw2_fma(s, p.kappa[c], p.smax[c]) : exp2_sw2_fast(mul2(s, pk(p.kappa[c], p.kappa[c])));
        if (MASK) {   // masked lanes: exactly 0 (the clamp would leave 2^-125)
          float e0, e1;
          upk(e, e0, e1);
          e = pk(ok0 ? e0 : 0.f, ok1 ? e1 : 0.f);
        }
      }
    } else {
      float q0, q1;
      upk(mul2(s, pk(p.kappa[c], p.kappa[c])), q0, q1);
      e = pk(ex2(q0), ex2(q1));
    }
    a1[c] = add2(a1[c], e);
    a2[c] = fma2(e, e, a2[c]);
  }

  template <bool MASK, bool CLAMP = false>
  __device__ __forceinline__ void compute(const float* __restrict__ sc, const Params& p, bool diag,
                                          int jlim) {
    const int tid = threadIdx.x;
    const int jend = MASK ? ((jlim + STEP - 1) / STEP) * STEP : T;
#pragma unroll UNR
    for (int j0 = 0; j0 < jend; j0 += STEP) {
#pragma unroll
      for (int g4 = 0; g4 < STEP; g4 += 4) {
        const int j = j0 + g4;
        float cv[D][4];
#pragma unroll
        for (int a = 0; a < D; ++a) {
          const float4 c4 = *reinterpret_cast<const float4*>(sc + a * T + j);
          cv[a][0] = c4.x; cv[a][1] = c4.y; cv[a][2] = c4.z; cv[a][3] = c4.w;
        }
        if (!UNIT && CMAJ) {   // candidate-major: each candidate's software-exp column sits among its MUFU ones
          f2 sk[4];
          bool okk0[4], okk1[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) sk[k] = dist<MASK>(cv, k, j + k, diag, jlim, tid, okk0[k], okk1[k]);
#pragma unroll
          for (int c = 0; c < NB; ++c)
#pragma unroll
            for (int k = 0; k < 4; ++k) term<MASK>(sk[k], c, g4 + k, okk0[k], okk1[k], p);
        } else {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            bool ok0, ok1;
            const f2 s = dist<MASK>(cv, k, j + k, diag, jlim, tid, ok0, ok1);
            if (UNIT) {
              float q0, q1;
              upk(s, q0, q1);
              const f2 e = pk(ex2(-q0), ex2(-q1));
              a1[0] = add2(a1[0], e);
              a2[0] = fma2(e, e, a2[0]);
            } else {
#pragma unroll
              for (int c = 0; c < NB; ++c) term<MASK>(s, c, g4 + k, ok0, ok1, p);
            }
          }
        }
      }
    }
  }

  // Squared whitened distance of the thread's two rows to column k of the staged group (both lanes);
  // masked lanes (ragged tail, diagonal tile) get s = +inf, so e = 2^-inf = 0.
  template <bool MASK>
  __device__ __forceinline__ f2 dist(const float (&cv)[D][4], int k, int jj, bool diag, int jlim, int tid,
                                     bool& ok0, bool& ok1) const {
    f2 dd = sub2(xr[0], pk(cv[0][k], cv[0][k]));
    f2 s = mul2(dd, dd);
#pragma unroll
    for (int a = 1; a < D; ++a) {
      dd = sub2(xr[a], pk(cv[a][k], cv[a][k]));
      s = fma2(dd, dd, s);
    }
    ok0 = ok1 = true;
    if (MASK) {
      float s0, s1;
      upk(s, s0, s1);
      const float inf = __int_as_float(0x7f800000);
      ok0 = (jj < jlim) && (!diag || jj > tid);
      ok1 = (jj < jlim) && (!diag || jj > NT + tid);
      s = pk(ok0 ? s0 : inf, ok1 ? s1 : inf);
    }
    return s;
  }

  __device__ __forceinline__ void outputs(double (&v)[NOUT], const Params&) const {
#pragma unroll
    for (int c = 0; c < NB; ++c) {
      float x0, x1, y0, y1;
      upk(a1[c], x0, x1);
      upk(a2[c], y0, y1);
      v[2 * c] = (double)x0 + (double)x1;
      v[2 * c + 1] = (double)y0 + (double)y1;
    }
  }
};

// ------------------------------------------------------------------ the persistent pair kernel

// First row index a thread loads for row-block q (functors may interleave rows).
template <class F, class = void>
struct HasRow0 : std::false_type {};
template <class F>
struct HasRow0<F, decltype((void)F::row0(0))> : std::true_type {};
template <class F>
__device__ __forceinline__ int64_t row_origin(int64_t q) {
  if constexpr (HasRow0<F>::value) return F::row0(q);
  else return q * F::T + threadIdx.x;
}

// Functors with tile-local centring (FPsi) read their rows from the fp64 samples; the others from X.
template <class F, class = void>
struct IsCentred : std::false_type {};
template <class F>
struct IsCentred<F, std::enable_if_t<F::kCentred>> : std::true_type {};

// LSCV on data sorted by coordinate 0: every pair of tile (l, q), q < l, has |fp32(x_i0 - x_j0)| >= g
// (rounding is monotone) and s >= fp32(g^2) (the other squares only add), so fp32(g^2) > skip_s makes
// every term exactly 0.  X = the (set's) prepared data; false for skip_s = +inf and for Psi functors.
template <class F>
__device__ __forceinline__ bool lscv_tile_skipped(const float* X, int64_t l, int64_t q, float skip_s) {
  if constexpr (IsCentred<F>::value) {
    return false;
  } else {
    if (q >= l) return false;
    const float g = __fsub_rn(X[l * F::T], X[q * F::T + F::T - 1]);
    return __fmul_rn(g, g) > skip_s;
  }
}

// Evaluate one work unit (tile (l, q), column chunk `chunk` when F::CS > 1) whose column samples
// are in shared memory at `sc`, and commit its outputs.  Sorted Psi data: a tile whose smallest
// pair distance exceeds `gap` (kPsiSkipGap32: every MUFU input underflows, the tile adds exactly 0;
// psi_bounded_gap: its terms are provably negligible, kde_internal.h) is skipped, so small
// bandwidths cost only the tiles near the diagonal.
template <class F>
__device__ __forceinline__ void pair_unit(const Args& a, const typename F::Params& p, int64_t tile,
                                          int64_t l, int64_t q, int chunk, const float* sc, double* red,
                                          unsigned long long* limbs, bool clamp, uint64_t* bar, uint32_t parity,
                                          bool skip, double gap) {
  constexpr int T = F::T, NOUT = F::NOUT;
  F f;
  if constexpr (IsCentred<F>::value) {
    if (q < l && a.Y64[l * T] - a.Y64[q * T + T - 1] > gap) {   // uniform per CTA
      if (threadIdx.x == 0 && a.skipped != nullptr) {   // pairs of this unit, for the profile
        int64_t c0 = 0, c1 = a.n - l * (int64_t)T;
        if (F::CS > 1) c0 = (int64_t)chunk * (T / F::CS), c1 = c1 < c0 + T / F::CS ? c1 : c0 + T / F::CS;
        else c1 = c1 < T ? c1 : T;
        if (c1 > c0) atomicAdd(a.skipped, (unsigned long long)(T * (c1 - c0)));
      }
      mbar_wait(bar, parity);   // a skipped unit still consumes its buffer's phase
      return;
    }
    f.load_rows_c(a.Y64, row_origin<F>(q), a.centres[l]);
  } else {
    if (skip) {   // LSCV far tile (lscv_tile_skipped, decided when the unit's TMA was issued)
      if (threadIdx.x == 0 && a.skipped != nullptr) {
        const int64_t c1 = a.n - l * (int64_t)T;
        atomicAdd(a.skipped, (unsigned long long)(T * (c1 < T ? c1 : T)));
      }
      mbar_wait(bar, parity);
      __syncthreads();   // the unit's skip flag slot is rewritten by the next issue
      return;
    }
    f.load_rows(a.X, a.ld, row_origin<F>(q));
  }
  mbar_wait(bar, parity);      // the row loads above overlap the column chunk's TMA
  if constexpr (F::CS > 1) f.jbase = chunk * F::CW;
  f.par = (int)(tile & 1);
  const bool diag = (q == l);
  const int64_t jl = a.n - l * (int64_t)T;
  if (clamp) {
    if (!diag && jl >= T) f.template compute<false, true>(sc, p, false, T);
    else f.template compute<true, true>(sc, p, diag, (int)(jl < T ? jl : T));
  } else {
    if (!diag && jl >= T) f.template compute<false, false>(sc, p, false, T);
    else f.template compute<true, false>(sc, p, diag, (int)(jl < T ? jl : T));
  }
  double v[NOUT];
  f.outputs(v, p);
  if constexpr (std::is_same<typename F::Params, LscvScalarParams>::value && !F::kSets) {
    // LSCV_h batch: the tile was evaluated for the batch's widest h, but a candidate whose own bound
    // skips it takes nothing from it (the same as in any other batch: batch-independent sums)
    if (q < l) {
      const float g = __fsub_rn(a.X[l * T], a.X[q * T + T - 1]);
      const float g2 = __fmul_rn(g, g);
#pragma unroll
      for (int c = 0; c < NOUT / 2; ++c)
        if (g2 > (a.skip_c_dev != nullptr ? a.skip_c_dev[c] : p.skip_c[c])) v[2 * c] = v[2 * c + 1] = 0.0;
    }
  }
  commit_tile<NOUT, F::NT>(v, red, limbs, a.scale_exp);
}

// Work unit u of the rank's share: local tile tile_begin + u / CS (tile id shard_tile(...)), column chunk u % CS (CS = 1: whole
// tiles).  Persistent CTAs stride over the units; the next unit's column chunk is staged by TMA
// into the other buffer while the current one is evaluated.
template <class F>
__global__ void __launch_bounds__(F::NT, F::MINB) pair_kernel(const Args a,
                                                        const __grid_constant__ typename F::Params p) {
  constexpr int T = F::T, D = F::D, NOUT = F::NOUT, NW = F::NT / 32, CS = F::CS;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* cols = reinterpret_cast<float*>(smem_raw);                 // [2][D][T]
  double* red = reinterpret_cast<double*>(cols + 2 * D * T);        // [NW][NOUT]
  uint64_t* bar = reinterpret_cast<uint64_t*>(red + NW * NOUT);      // [2]
  const int tid = threadIdx.x;
  __shared__ int64_t s_next[2];
  __shared__ int s_skip[2];   // per buffer: the staged unit is an exactly-zero LSCV tile

  const int64_t units = (a.tile_end - a.tile_begin) * CS;
  // LSCV_h batch: the tile skip bound is the widest of the candidates' own (data-aware) bounds
  float skip_s = a.skip_s;
  if (a.skip_c_dev != nullptr && tid == 0) {
    skip_s = a.skip_c_dev[0];
    for (int c = 1; c < NOUT / 2; ++c) skip_s = fmaxf(skip_s, a.skip_c_dev[c]);
  }
  // thread 0 stages unit u's column chunk into buffer `buf` (TMA) and decides its skip flag
  auto issue = [&](int64_t u, int buf) {
    int64_t l, q;
    tile_coords(shard_tile(a.tile_begin + u / CS, a.part_rank, a.part_world), l, q);
    s_skip[buf] = lscv_tile_skipped<F>(a.X, l, q, skip_s);
    float* dst = cols + buf * D * T;
    mbar_expect_tx(&bar[buf], (uint32_t)(D * T * sizeof(float)));
#pragma unroll
    for (int d = 0; d < D; ++d)
      tma_load_1d(dst + d * T, a.X + d * a.ld + l * T, (uint32_t)(T * sizeof(float)), &bar[buf]);
  };
  int64_t u = blockIdx.x;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (u < units) issue(u, 0);
  }
  __syncthreads();
  const bool clamp = F::kClampable && a.clamp != nullptr && *a.clamp != 0;   // uniform per launch
  const double gap = a.skip_gap_dev != nullptr ? *a.skip_gap_dev : a.skip_gap;
  uint32_t k = 0;
  while (u < units) {
    const int64_t tile = shard_tile(a.tile_begin + u / CS, a.part_rank, a.part_world);
    int64_t l, q;
    tile_coords(tile, l, q);
    const int64_t un = next_unit_issue(a, u, s_next, k);
    const bool skip = s_skip[k & 1];   // read before the issue below can rewrite the other slot
    if (tid == 0 && un < units) issue(un, (k + 1) & 1);
    pair_unit<F>(a, p, tile, l, q, (int)(u % CS), cols + (k & 1) * D * T, red, a.limbs, clamp, &bar[k & 1],
                 (k >> 1) & 1, skip, gap);
    u = un;
    ++k;
  }
}

// Several data sets per launch (LSCV_H: one whitened copy of the data per candidate).
template <class F>
__global__ void __launch_bounds__(F::NT, F::MINB) pair_kernel_sets(const Args a,
                                                        const __grid_constant__ typename F::Params p) {
  constexpr int T = F::T, D = F::D, NOUT = F::NOUT, NW = F::NT / 32;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* cols = reinterpret_cast<float*>(smem_raw);                 // [2][D][T]
  double* red = reinterpret_cast<double*>(cols + 2 * D * T);        // [NW][NOUT]
  uint64_t* bar = reinterpret_cast<uint64_t*>(red + NW * NOUT);      // [2]
  const int tid = threadIdx.x;
  __shared__ int64_t s_next[2];
  __shared__ int s_skip[2];

  pdl_trigger();   // a programmatic successor (the Nelder–Mead decision) may take its slot right away
  pdl_wait();      // a programmatic launch (device-resident Nelder–Mead) waits for the whitening here
  // Work units u in [0, n_sets * tiles): set = u / tiles, local tile = tile_begin + u % tiles (set-major,
  // so consecutive CTAs share a set's data in L2).
  const int64_t per = a.tile_end - a.tile_begin;
  const int64_t units = per * (a.n_sets_dev != nullptr ? *a.n_sets_dev : a.n_sets);
  auto issue = [&](int64_t u, int buf) {
    const int64_t set = u / per;
    int64_t l, q;
    tile_coords(shard_tile(a.tile_begin + (u - set * per), a.part_rank, a.part_world), l, q);
    const float* Xs = a.X + set * a.set_stride;
    s_skip[buf] = lscv_tile_skipped<F>(Xs, l, q, a.skip_s_sets != nullptr ? a.skip_s_sets[set] : a.skip_s);
    float* dst = cols + buf * D * T;
    mbar_expect_tx(&bar[buf], (uint32_t)(D * T * sizeof(float)));
#pragma unroll
    for (int d = 0; d < D; ++d)
      tma_load_1d(dst + d * T, Xs + d * a.ld + l * T, (uint32_t)(T * sizeof(float)), &bar[buf]);
  };
  int64_t u = blockIdx.x;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (u < units) issue(u, 0);
  }
  __syncthreads();
  const bool clamp = F::kClampable && a.clamp != nullptr && *a.clamp != 0;   // uniform per launch
  uint32_t k = 0;
  while (u < units) {
    const int64_t set = u / per;
    const int64_t tile = shard_tile(a.tile_begin + (u - set * per), a.part_rank, a.part_world);
    int64_t l, q;
    tile_coords(tile, l, q);
    const int64_t un = next_unit_issue(a, u, s_next, k);
    const bool skip = s_skip[k & 1];
    if (tid == 0 && un < units) issue(un, (k + 1) & 1);
    Args as = a;
    as.X = a.X + set * a.set_stride;
    pair_unit<F>(as, p, tile, l, q, 0, cols + (k & 1) * D * T, red, a.limbs + set * NOUT * kLimbs, clamp,
                 &bar[k & 1], (k >> 1) & 1, skip, a.skip_gap);
    u = un;
    ++k;
  }
}

// One-time per-instantiation setup (shared-memory opt-in, resident CTAs per SM).  Not allowed
// inside a stream capture, so graph users call it before capturing (prepare_* below).
template <class F>
inline cudaError_t pair_occupancy(int* occ_out) {
  constexpr size_t smem = 2 * F::D * F::T * sizeof(float) + (F::NT / 32) * F::NOUT * sizeof(double) + 16;
  static int occ_dev[kMaxDevices];   // 0 = not yet set up on that device
  int& occ = occ_dev[current_device()];
  if (occ <= 0) {
    const void* kern;
    if constexpr (F::kSets) kern = (const void*)pair_kernel_sets<F>;
    else kern = (const void*)pair_kernel<F>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int o = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, F::NT, smem);
    if (e != cudaSuccess) return e;
    occ = o > 0 ? o : 1;
  }
  *occ_out = occ;
  return cudaSuccess;
}

template <class F>
inline cudaError_t launch_pair(const LaunchCfg& c, const typename F::Params& p) {
  if (c.tile_end <= c.tile_begin) return cudaSuccess;
  constexpr size_t smem = 2 * F::D * F::T * sizeof(float) + (F::NT / 32) * F::NOUT * sizeof(double) + 16;
  int occ = 1;
  cudaError_t e = pair_occupancy<F>(&occ);
  if (e != cudaSuccess) return e;
  const int64_t units = (c.tile_end - c.tile_begin) * c.n_sets * F::CS;
  int64_t grid = (int64_t)c.sm_count * occ - c.reserve_ctas;
  if (grid > units) grid = units;
  if (grid < 1) grid = 1;
  Args a{c.X, c.n, c.ld, c.tile_begin, c.tile_end, c.scale_exp, c.limbs, c.clamp, c.n_sets, c.set_stride,
         c.Y64, c.centres, c.skipped, c.n_sets_dev, c.skip_gap, c.work, c.skip_s, c.part_rank, c.part_world,
         c.skip_gap_dev, c.skip_s_sets, c.skip_c_dev};
  if constexpr (F::kSets) {
    if (c.pdl) {
      cudaLaunchConfig_t lc = {};
      lc.gridDim = dim3((unsigned)grid);
      lc.blockDim = dim3(F::NT);
      lc.dynamicSmemBytes = smem;
      lc.stream = c.stream;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      lc.attrs = at;
      lc.numAttrs = 1;
      return cudaLaunchKernelEx(&lc, pair_kernel_sets<F>, a, p);
    }
    pair_kernel_sets<F><<<(unsigned)grid, F::NT, smem, c.stream>>>(a, p);
  } else {
    pair_kernel<F><<<(unsigned)grid, F::NT, smem, c.stream>>>(a, p);
  }
  return cudaGetLastError();
}

}  // namespace kde
