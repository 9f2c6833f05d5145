// Pipe-throughput microbenchmark for the roofline denominators of the pair-sum kernels
// (SURVEY §8(d) d4/d6): MUFU.EX2 (ex2.approx.ftz.f32) and FFMA issue rates per SM per clock
// on the live B200, with the SM clock sampled from %clock64 vs. CUDA-event time.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/peaks tools/peaks.cu
// Output: one JSON line.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); return 1; } } while (0)

__device__ __forceinline__ float ex2(float x) {
  float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y;
}

// 8 independent chains per thread; each step is one MUFU.EX2 + one FFMA (so the MUFU
// input changes and the compiler cannot hoist). The FFMA share is 1:1, well below the 8:1
// pipe ratio, so MUFU binds.
__global__ void k_ex2(float* out, int iters, long long* clk) {
  float a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = -0.001f * (threadIdx.x + k);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = ex2(a[k]) * -0.5f;
  }
  long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}

// 16 independent FFMA chains per thread.
__global__ void k_ffma(float* out, int iters, long long* clk) {
  float a[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) a[k] = 1.0f + 1e-7f * (threadIdx.x + k);
  const float b = 0.999999f, c = 1e-7f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) a[k] = fmaf(a[k], b, c);
  }
  long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 16; ++k) s += a[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}

int main() {
  int dev = 0, sms = 0;
  CK(cudaSetDevice(dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int threads = 512, blocks = sms * 4;
  float* out; long long* clk;
  CK(cudaMalloc(&out, sizeof(float) * threads * blocks));
  CK(cudaMalloc(&clk, sizeof(long long)));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  const int iters = 20000;
  double res[2][3];
  for (int which = 0; which < 2; ++which) {
    float best = 1e30f; long long cyc = 0;
    for (int rep = 0; rep < 5; ++rep) {
      CK(cudaEventRecord(e0));
      if (which == 0) k_ex2<<<blocks, threads>>>(out, iters, clk);
      else k_ffma<<<blocks, threads>>>(out, iters, clk);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
      if (ms < best) { best = ms; CK(cudaMemcpy(&cyc, clk, sizeof(cyc), cudaMemcpyDeviceToHost)); }
    }
    double ops = (double)blocks * threads * iters * (which == 0 ? 8 : 16);
    double per_s = ops / (best * 1e-3);
    // clock estimate: one CTA's measured cycles over the kernel time (all CTAs co-resident: 4/SM)
    double mhz = cyc / (best * 1e-3) / 1e6;
    res[which][0] = per_s; res[which][1] = mhz; res[which][2] = per_s / (sms * mhz * 1e6);
  }
  printf("{\"sms\": %d, \"ex2_per_s\": %.4e, \"ex2_clk_mhz\": %.0f, \"ex2_per_clk_per_sm\": %.2f, "
         "\"ffma_per_s\": %.4e, \"ffma_clk_mhz\": %.0f, \"ffma_per_clk_per_sm\": %.2f}\n",
         sms, res[0][0], res[0][1], res[0][2], res[1][0], res[1][1], res[1][2]);
  return 0;
}
