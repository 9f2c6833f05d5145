// Does FP64-pipe work overlap the pair kernels' FP32/MUFU mixes?  (a candidate
// "third pipe" for offloading exponentials or squared distances.)  Each mode runs a fixed mix per
// iteration on independent chains at the pair kernels' occupancy (3 CTAs x 256 threads per SM), plus
// `dp` extra DFMA per iteration; the time against dp = 0 says whether the DFMAs come for free.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dp_overlap tools/dp_overlap.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d;
}

constexpr int IT = 2048;

// MIX 0 (Psi-like): 8 MUFU + 24 FFMA2 per iteration; MIX 1 (LSCV_H d = 4-like): 2 MUFU + 10 FFMA2.
template <int MIX, int DP>
__global__ void __launch_bounds__(256, 3) kern(float* out, float b, float c) {
  float f[8];
  unsigned long long v[8];
  double d[4];
  for (int k = 0; k < 8; ++k) {
    f[k] = -(threadIdx.x * 1e-3f + k);
    v[k] = ((unsigned long long)__float_as_uint(f[k]) << 32) | __float_as_uint(f[k]);
  }
  for (int k = 0; k < 4; ++k) d[k] = f[k];
  const unsigned long long bb = ((unsigned long long)__float_as_uint(b) << 32) | __float_as_uint(b);
  const unsigned long long cc = ((unsigned long long)__float_as_uint(c) << 32) | __float_as_uint(c);
  const double db = b, dc = c;
  for (int i = 0; i < IT; ++i) {
    constexpr int NM = MIX == 0 ? 8 : 2, NF = MIX == 0 ? 24 : 10;
#pragma unroll
    for (int k = 0; k < NM; ++k) f[k] = ex2(f[k]) * b;
#pragma unroll
    for (int k = 0; k < NF; ++k) v[k & 7] = ffma2(v[k & 7], bb, cc);
#pragma unroll
    for (int k = 0; k < DP; ++k) d[k & 3] = fma(d[k & 3], db, dc);
  }
  float s = 0;
  for (int k = 0; k < 8; ++k) s += f[k] + __uint_as_float((unsigned)v[k]);
  for (int k = 0; k < 4; ++k) s += (float)d[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MIX, int DP>
static void run(float* out, int blocks) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kern<MIX, DP><<<blocks, 256>>>(out, 0.999f, 1e-3f);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) kern<MIX, DP><<<blocks, 256>>>(out, 0.999f, 1e-3f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("{\"mix\": \"%s\", \"dfma_per_iter\": %d, \"ms\": %.4f}\n", MIX == 0 ? "psi (8 MUFU + 24 FFMA2)" : "lscvH4 (2 MUFU + 10 FFMA2)",
         DP, ms / 5);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 3 * 4;
  float* out;
  cudaMalloc(&out, sizeof(float) * 256 * blocks);
  run<0, 0>(out, blocks); run<0, 4>(out, blocks); run<0, 8>(out, blocks); run<0, 16>(out, blocks); run<0, 24>(out, blocks);
  run<1, 0>(out, blocks); run<1, 2>(out, blocks); run<1, 4>(out, blocks); run<1, 8>(out, blocks);
  return 0;
}
