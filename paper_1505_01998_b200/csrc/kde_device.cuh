// kde_device.cuh — device helpers shared by the sm_100a kernels (kde_pair.cuh and every kernel unit).
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

namespace kde {

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Packed fp32x2 arithmetic (sm_100a FADD2 / FMUL2 / FFMA2): two lanes per instruction, each
// rounded to nearest exactly like the scalar op, so packing never changes a result bit.
typedef unsigned long long f2;
__device__ __forceinline__ f2 pk(float a, float b) {
  f2 r;
  asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void upk(f2 v, float& a, float& b) {
  asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ f2 add2(f2 a, f2 b) { f2 d; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ f2 sub2(f2 a, f2 b) { f2 d; asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ f2 mul2(f2 a, f2 b) { f2 d; asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) {
  f2 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

// 2^a for two lanes on the FMA pipe (offloads MUFU.EX2): a is clamped to
// >= -125, a = j + f with j = rint(a) (magic-number add), f in [-1/2, 1/2]; 2^f by a degree-5
// minimax polynomial (relative error 7.5e-8, 2.4e-7 after fp32 Horner); 2^j added to the
// exponent bits.  Used only where terms are positive and the objective cancels little (LSCV
// sums, KDE evaluation); never for Psi_r.  Arguments below -125 (or NaN-free -inf) return 0.
__device__ __forceinline__ f2 exp2_sw2(f2 q) {
  float q0, q1;
  upk(q, q0, q1);
  const f2 a = pk(fmaxf(q0, -125.f), fmaxf(q1, -125.f));
  const f2 magic = pk(12582912.f, 12582912.f);   // 1.5 * 2^23
  const f2 t = add2(a, magic);
  const f2 fr = sub2(a, sub2(t, magic));
  f2 p = fma2(pk(1.3276472454890609e-03f, 1.3276472454890609e-03f), fr,
              pk(9.675540961325169e-03f, 9.675540961325169e-03f));
  p = fma2(p, fr, pk(5.550713092088699e-02f, 5.550713092088699e-02f));
  p = fma2(p, fr, pk(2.4022120237350464e-01f, 2.4022120237350464e-01f));
  p = fma2(p, fr, pk(6.931469440460205e-01f, 6.931469440460205e-01f));
  p = fma2(p, fr, pk(1.0000001192092896f, 1.0000001192092896f));
  float t0, t1, p0, p1;
  upk(t, t0, t1);
  upk(p, p0, p1);
  // below -125 return exactly 0 (like MUFU.EX2.FTZ's flush), so padding and far pairs add nothing
  return pk(q0 >= -125.f ? __int_as_float(__float_as_int(p0) + (__float_as_int(t0) << 23)) : 0.f,
            q1 >= -125.f ? __int_as_float(__float_as_int(p1) + (__float_as_int(t1) << 23)) : 0.f);
}

// As exp2_sw2 without the zero select: the argument is clamped to >= -125, so arguments below
// return 2^-125 (~2.4e-38, an absolute error far below any term that matters) instead of 0.  One
// FMNMX per lane plus the magic-number split, the degree-5 polynomial and one LEA per lane: no
// compare, no predication.  Callers mask invalid pairs themselves.
__device__ __forceinline__ f2 exp2_sw2_fast(f2 q) {
  float q0, q1;
  upk(q, q0, q1);
  const f2 a = pk(fmaxf(q0, -125.f), fmaxf(q1, -125.f));
  const f2 magic = pk(12582912.f, 12582912.f);   // 1.5 * 2^23
  const f2 t = add2(a, magic);
  const f2 fr = sub2(a, sub2(t, magic));
  f2 p = fma2(pk(1.3276472454890609e-03f, 1.3276472454890609e-03f), fr,
              pk(9.675540961325169e-03f, 9.675540961325169e-03f));
  p = fma2(p, fr, pk(5.550713092088699e-02f, 5.550713092088699e-02f));
  p = fma2(p, fr, pk(2.4022120237350464e-01f, 2.4022120237350464e-01f));
  p = fma2(p, fr, pk(6.931469440460205e-01f, 6.931469440460205e-01f));
  p = fma2(p, fr, pk(1.0000001192092896f, 1.0000001192092896f));
  float t0, t1, p0, p1;
  upk(t, t0, t1);
  upk(p, p0, p1);
  return pk(__int_as_float(__float_as_int(p0) + (__float_as_int(t0) << 23)),
            __int_as_float(__float_as_int(p1) + (__float_as_int(t1) << 23)));
}

// As exp2_sw2_fast for 2^(s kappa) with the product folded into the range reduction: s is clamped to
// <= smax = 125 / |kappa| (FMNMX), t = fma(s, kappa, magic) rounds s kappa to an integer j in its low
// bits, -j = magic - t, and f = fma(s, kappa, -j) is the exactly rounded fraction (one FP32 op per
// lane fewer than forming q = s kappa first).
__device__ __forceinline__ f2 exp2_sw2_fma(f2 s, float kappa, float smax) {
  float s0, s1;
  upk(s, s0, s1);
  const f2 sc = pk(fminf(s0, smax), fminf(s1, smax));
  const f2 k2 = pk(kappa, kappa);
  const f2 magic = pk(12582912.f, 12582912.f);   // 1.5 * 2^23
  const f2 t = fma2(sc, k2, magic);
  const f2 fr = fma2(sc, k2, sub2(magic, t));
  f2 p = fma2(pk(1.3276472454890609e-03f, 1.3276472454890609e-03f), fr,
              pk(9.675540961325169e-03f, 9.675540961325169e-03f));
  p = fma2(p, fr, pk(5.550713092088699e-02f, 5.550713092088699e-02f));
  p = fma2(p, fr, pk(2.4022120237350464e-01f, 2.4022120237350464e-01f));
  p = fma2(p, fr, pk(6.931469440460205e-01f, 6.931469440460205e-01f));
  p = fma2(p, fr, pk(1.0000001192092896f, 1.0000001192092896f));
  float t0, t1, p0, p1;
  upk(t, t0, t1);
  upk(p, p0, p1);
  return pk(__int_as_float(__float_as_int(p0) + (__float_as_int(t0) << 23)),
            __int_as_float(__float_as_int(p1) + (__float_as_int(t1) << 23)));
}

// Programmatic dependent launch: wait until the preceding grid has completed and its memory is visible
// (a no-op for a kernel launched without the attribute); let the dependent grid start launching.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// TMA bulk copy global -> shared, completion counted on `bar` (UBLKCP in SASS).
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Exact fixed-point split of v * 2^S (|v| 2^S < 2^120): sign-magnitude limbs of 40 bits.  The
// lo limb is an unsigned mod-2^64 accumulator; its carry-outs minus the borrows of negative
// addends go to the carry limb (dst[3], units of 2^64), so (unsigned) lo + 2^64 carry is the exact
// sum whatever the number and order of the commits (the difference true - lo is order-free).
__device__ __forceinline__ void add_limbs(double v, int S, unsigned long long* dst) {
  double a = fabs(ldexp(v, S));
  double h = floor(ldexp(a, -80));
  double r = a - ldexp(h, 80);            // exact: the low bits of a
  double m = floor(ldexp(r, -40));
  double lo = rint(r - ldexp(m, 40));     // integer part; rounding < 2^-S absolute
  long long H = (long long)h, M = (long long)m, L = (long long)lo;
  if (v < 0) { H = -H; M = -M; L = -L; }
  atomicAdd(dst + 0, (unsigned long long)H);
  atomicAdd(dst + 1, (unsigned long long)M);
  const unsigned long long u = (unsigned long long)L;
  const unsigned long long old = atomicAdd(dst + 2, u);
  const long long c = (long long)(old + u < old) - (long long)(L < 0);
  if (c != 0) atomicAdd(dst + 3, (unsigned long long)c);
}

// Value of one output's limbs (device side of the host's limbs_to_fixed / fixed_value).
__device__ __forceinline__ __int128 limbs_total(const unsigned long long* l) {
  return (__int128)(long long)l[0] * ((__int128)1 << 80) + (__int128)(long long)l[1] * ((__int128)1 << 40) +
         (__int128)l[2] + (__int128)(long long)l[3] * ((__int128)1 << 64);
}

}  // namespace kde
