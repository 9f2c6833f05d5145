// Single-thread dependent-chain latency of fp64 ops on this GPU (why the device Nelder-Mead decision
// takes ~7 us: DESIGN.md §4).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lat_probe tools/lat_probe.cu
#include <cstdio>
__global__ void k(double* out, long long* clk, double a, double b, int mode) {
  double x = a, y = b;
  long long t0 = clock64();
  #pragma unroll 1
  for (int i = 0; i < 100; ++i) {
    if (mode == 0) x = fma(x, y, 1e-3);
    else if (mode == 1) x = 1.0 + y / x;
    else if (mode == 2) x = sqrt(x) + 0.5;
    else if (mode == 3) x = x * y + 1e-3;
    else { float f = (float)x; f = __fmaf_rn(f, (float)y, 1e-3f); x = f; }
  }
  long long t1 = clock64();
  out[0] = x; clk[0] = t1 - t0;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8); cudaMalloc(&c, 8);
  const char* names[5] = {"DFMA", "DDIV (1 + y/x)", "DSQRT (+0.5)", "DMUL+DADD", "F2F+FFMA+F2F"};
  for (int m = 0; m < 5; ++m) {
    k<<<1,1>>>(o, c, 1.1, 0.9, m); cudaDeviceSynchronize();
    k<<<1,1>>>(o, c, 1.1, 0.9, m); long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%s: %.1f cycles per iteration\n", names[m], h / 100.0);
  }
}
