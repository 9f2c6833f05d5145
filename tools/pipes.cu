// Per-SM-per-clock throughput of the instruction mixes the pair kernels are built from
// (DESIGN.md §4): register-form FFMA, FFMA2 (fma.rn.f32x2), F2F.F64.F32 + DADD, DFMA, and
// MUFU.EX2 mixed with FFMA.  All CTAs co-resident; clock from clock64 of one CTA.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pipes tools/pipes.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d;
}

constexpr int IT = 4096;
// mode 0: FFMA reg form (a = a*b + c, all registers), 8 chains
// mode 1: FFMA2 reg form, 8 chains (16 FMAs per iteration)
// mode 2: F2F.F64.F32 + DADD (d += (double)f), 8 chains
// mode 3: DFMA, 8 chains
// mode 4: MUFU.EX2 only, 8 chains
__global__ void kern(int mode, float* out, long long* clk, float b, float c) {
  long long t0 = clock64();
  float f[8]; double d[8]; unsigned long long v[8];
  for (int k = 0; k < 8; ++k) { f[k] = threadIdx.x * 1e-3f + k; d[k] = f[k]; v[k] = ((unsigned long long)__float_as_uint(f[k]) << 32) | __float_as_uint(f[k]); }
  unsigned long long bb = ((unsigned long long)__float_as_uint(b) << 32) | __float_as_uint(b);
  unsigned long long cc = ((unsigned long long)__float_as_uint(c) << 32) | __float_as_uint(c);
  if (mode == 0) {
    for (int i = 0; i < IT; ++i)
#pragma unroll
      for (int k = 0; k < 8; ++k) f[k] = fmaf(f[k], b, c);
  } else if (mode == 1) {
    for (int i = 0; i < IT; ++i)
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = ffma2(v[k], bb, cc);
  } else if (mode == 2) {
    for (int i = 0; i < IT; ++i)
#pragma unroll
      for (int k = 0; k < 8; ++k) { d[k] += (double)f[k]; f[k] = f[k] * b; }
  } else if (mode == 3) {
    double db = b, dc = c;
    for (int i = 0; i < IT; ++i)
#pragma unroll
      for (int k = 0; k < 8; ++k) d[k] = fma(d[k], db, dc);
  } else {
    for (int i = 0; i < IT; ++i)
#pragma unroll
      for (int k = 0; k < 8; ++k) f[k] = ex2(f[k]);
  }
  long long t1 = clock64();
  float s = 0;
  for (int k = 0; k < 8; ++k) s += f[k] + (float)d[k] + __uint_as_float((unsigned)v[k]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int threads = 512, blocks = sms * 2;
  float* out; long long* clk;
  cudaMalloc(&out, 4 * threads * blocks); cudaMalloc(&clk, 8);
  const char* names[5] = {"FFMA reg", "FFMA2 reg (x2 ops)", "F2F.F64.F32+DADD (+FMUL)", "DFMA", "MUFU.EX2"};
  const double ops_per_it[5] = {8, 16, 8, 8, 8};
  for (int mode = 0; mode < 5; ++mode) {
    kern<<<blocks, threads>>>(mode, out, clk, 0.9999f, 1e-6f);
    cudaDeviceSynchronize();
    long long cyc; cudaMemcpy(&cyc, clk, 8, cudaMemcpyDeviceToHost);
    // per SM: blocks/sms CTAs of `threads`, all resident; cycles for one CTA ~ the SM's time
    double ops_sm = (double)threads * (blocks / sms) * IT * ops_per_it[mode];
    printf("%-28s %7.1f ops/clk/SM\n", names[mode], ops_sm / cyc);
  }
  return 0;
}
