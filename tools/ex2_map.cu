// Relative error eps(x) = ex2.approx.ftz(x)/2^x - 1 of MUFU.EX2 over every fp32 x in [-40, 1):
// mean/mean|.| per unit interval, and per 1/32 sub-bin inside [-1, 0).
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2(float x) { float y; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__global__ void k(double* s, double* a, unsigned long long* c, unsigned long long base) {
  unsigned long long idx = base + blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
  float x = __uint_as_float((unsigned int)idx);
  if (!(x >= -40.f && x < 1.f)) return;
  double e = (double)ex2(x) / exp2((double)x) - 1.0;
  int bin = (int)floor((double)x) + 40;
  atomicAdd(&s[bin], e); atomicAdd(&a[bin], fabs(e)); atomicAdd(&c[bin], 1ull);
  if (x >= -1.f && x < 0.f) {
    int sb = 41 + (int)floor(((double)x + 1.0) * 32.0);
    atomicAdd(&s[sb], e); atomicAdd(&a[sb], fabs(e)); atomicAdd(&c[sb], 1ull);
  }
}
int main() {
  const int NB = 41 + 32;
  double *s, *a; unsigned long long* c;
  cudaMalloc(&s, NB * 8); cudaMalloc(&a, NB * 8); cudaMalloc(&c, NB * 8);
  cudaMemset(s, 0, NB * 8); cudaMemset(a, 0, NB * 8); cudaMemset(c, 0, NB * 8);
  for (unsigned long long base = 0; base < (1ull << 32); base += (1ull << 30))
    k<<<(1u << 30) / 256, 256>>>(s, a, c, base);
  double hs[NB], ha[NB]; unsigned long long hc[NB];
  cudaMemcpy(hs, s, NB * 8, cudaMemcpyDeviceToHost); cudaMemcpy(ha, a, NB * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(hc, c, NB * 8, cudaMemcpyDeviceToHost);
  for (int b = 0; b < 41; ++b) if (hc[b]) printf("x in [%3d,%3d): mean eps %+.3e  mean|eps| %.3e\n", b - 40, b - 39, hs[b] / hc[b], ha[b] / hc[b]);
  for (int b = 41; b < NB; ++b) if (hc[b]) printf("x in [%+.4f,%+.4f): mean eps %+.3e  mean|eps| %.3e\n", -1 + (b - 41) / 32.0, -1 + (b - 40) / 32.0, hs[b] / hc[b], ha[b] / hc[b]);
  return 0;
}
