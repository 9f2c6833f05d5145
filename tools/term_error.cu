// Error-source experiment for the Psi_r pair terms: for all pairs i<j of a
// sample, accumulate (t_variant - t_exact) in fp64 for several fp32 evaluation variants, where
// t_exact is the fp64 term He_r(u) exp(-u^2/2), u = (x_i - x_j)/g.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/term_error tools/term_error.cu
// Run:   tools/term_error data.bin r g
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2(float x) { float y; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }

template <int R> __device__ __forceinline__ double P64(double s) {
  if (R == 4) return (s - 6) * s + 3;
  if (R == 6) return ((s - 15) * s + 45) * s - 15;
  return (((s - 28) * s + 210) * s - 420) * s + 105;
}
template <int R> __device__ __forceinline__ float P32(float s) {
  if (R == 4) return __fmaf_rn(__fadd_rn(s, -6.f), s, 3.f);
  if (R == 6) return __fmaf_rn(__fmaf_rn(__fadd_rn(s, -15.f), s, 45.f), s, -15.f);
  return __fmaf_rn(__fmaf_rn(__fmaf_rn(__fadd_rn(s, -28.f), s, 210.f), s, -420.f), s, 105.f);
}
// fp32 software exp2 (Cody-Waite + degree-7 Taylor/minimax-ish), for comparison
__device__ __forceinline__ float sw_exp2(float a) {
  float j = rintf(a);
  float f = __fsub_rn(a, j);           // [-0.5, 0.5]
  // 2^f = e^{f ln2}: Taylor degree 7 in f*ln2 (error < 1e-9 on [-.35,.35])
  const float c[8] = {1.f, 0.69314718056f, 0.24022650695f, 0.05550410866f, 0.00961812911f,
                      0.00133335581f, 0.00015403530f, 0.00001525273f};
  float p = c[7];
  for (int k = 6; k >= 0; --k) p = __fmaf_rn(p, f, c[k]);
  return ldexpf(p, (int)j);
}

constexpr int NV = 19;
template <int R>
__global__ void k(const double* x, int n, double g, double* out) {
  // out[v] += sum(t_v - t_exact), out[NV] += sum|t_exact|, out[NV+1] += sum t_exact
  double acc[NV + 2] = {0};
  const double L2E = 1.4426950408889634;
  const float c0 = (float)(-L2E / 2);
  const float c0_hi = c0, c0_lo = (float)(-L2E / 2 - (double)c0);
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < (long long)n * n; p += (long long)gridDim.x * blockDim.x) {
    int i = (int)(p / n), j = (int)(p % n);
    if (j <= i) continue;
    double xi = x[i] / g, xj = x[j] / g;
    double u = xi - xj, s = u * u;
    double te = P64<R>(s) * exp(-0.5 * s);
    acc[NV] += fabs(te); acc[NV + 1] += te;
    float fi = (float)xi, fj = (float)xj;
    float d = __fsub_rn(fi, fj), sf = __fmul_rn(d, d);
    // v0: current kernel: fp32 x', c0 fp32, MUFU
    float t0 = __fmul_rn(P32<R>(sf), ex2(__fmul_rn(sf, c0)));
    acc[0] += (double)t0 - te;
    // v1: exact-ish constant via split: a = s*c_hi + s*c_lo
    float a1 = __fmaf_rn(sf, c0_hi, __fmul_rn(sf, c0_lo));
    acc[1] += (double)__fmul_rn(P32<R>(sf), ex2(a1)) - te;
    // v2: exact s (fp64 difference rounded once), c split, MUFU
    float s2 = (float)s;
    float a2 = (float)(s * (-0.5 * L2E));
    acc[2] += (double)__fmul_rn(P32<R>(s2), ex2(a2)) - te;
    // v3: v2 but exp from fp64 (isolates MUFU error)
    acc[3] += (double)P32<R>(s2) * exp2((double)a2) - te;
    // v4: v2 with software fp32 exp2
    acc[4] += (double)__fmul_rn(P32<R>(s2), sw_exp2(a2)) - te;
    // v5: v2 but poly in fp64 (isolates Horner rounding), MUFU exp
    acc[5] += P64<R>((double)s2) * (double)ex2(a2) - te;
    // v6..v9: current kernel arithmetic + MUFU input shift phi_k = k/K (K = 2,4,8,8'),
    // class k = (i + 3j) mod K, result scaled by 2^-phi_k in fp64
    {
      const int Ks[4] = {2, 4, 8, 8};
      for (int q = 0; q < 4; ++q) {
        int K = Ks[q];
        int kk = (i + 3 * j) % K;
        double phi = (double)kk / K + (q == 3 ? 0.0371 * kk : 0.0);
        float a = __fmaf_rn(sf, c0, (float)phi);
        double e = (double)ex2(a) * exp2(-(double)(float)phi);
        acc[6 + q] += (double)P32<R>(sf) * e - te;
      }
    }
    // v10: MUFU on the reduced fraction f in [-1/2,1/2], exact 2^j
    {
      float a = __fmul_rn(sf, c0);
      float t = __fadd_rn(a, 12582912.f);
      float jj = __fsub_rn(t, 12582912.f);
      float f = __fsub_rn(a, jj);
      float e = ldexpf(ex2(f), (int)jj);
      acc[10] += (double)__fmul_rn(P32<R>(sf), e) - te;
    }
    // v11..v14: MUFU input offset by -B (B = 2, 8, 16, 64): e = ex2(s*c0 - B) * 2^B
    {
      const float Bs[4] = {2.f, 8.f, 16.f, 64.f};
      for (int q = 0; q < 4; ++q) {
        float e = ex2(__fmaf_rn(sf, c0, -Bs[q]));
        acc[11 + q] += (double)__fmul_rn(P32<R>(sf), e) * exp2((double)Bs[q]) - te;
      }
    }
    // v15..v17: offset -16 plus fractional shift phi_k = k/K, K = 4, 8, 32 (class (i+3j) mod K)
    {
      const int Ks[3] = {4, 8, 32};
      for (int q = 0; q < 3; ++q) {
        const int K = Ks[q];
        const int kk = (i + 3 * j) % K;
        const float off = 16.f + (float)kk / K;
        float e = ex2(__fmaf_rn(sf, c0, -off));
        acc[15 + q] += (double)__fmul_rn(P32<R>(sf), e) * exp2((double)off) - te;
      }
    }
    // v18: offset -16 + K=8 with class = i % 8 (row-based, as in the kernel)
    {
      const float off = 16.f + (float)(i % 8) / 8;
      float e = ex2(__fmaf_rn(sf, c0, -off));
      acc[18] += (double)__fmul_rn(P32<R>(sf), e) * exp2((double)off) - te;
    }
  }
  for (int v = 0; v < NV + 2; ++v) atomicAdd(&out[v], acc[v]);
}

int main(int argc, char** argv) {
  FILE* f = fopen(argv[1], "rb");
  int r = atoi(argv[2]);
  double g = atof(argv[3]);
  fseek(f, 0, SEEK_END);
  int n = (int)(ftell(f) / 8);
  fseek(f, 0, SEEK_SET);
  std::vector<double> h(n);
  fread(h.data(), 8, n, f);
  fclose(f);
  double *dx, *dout;
  cudaMalloc(&dx, n * 8);
  cudaMalloc(&dout, 32 * 8);
  cudaMemcpy(dx, h.data(), n * 8, cudaMemcpyHostToDevice);
  cudaMemset(dout, 0, 32 * 8);
  if (r == 4) k<4><<<148 * 8, 256>>>(dx, n, g, dout);
  else if (r == 6) k<6><<<148 * 8, 256>>>(dx, n, g, dout);
  else k<8><<<148 * 8, 256>>>(dx, n, g, dout);
  double o[32];
  cudaMemcpy(o, dout, 32 * 8, cudaMemcpyDeviceToHost);
  const char* names[NV] = {"current", "c0 split", "s from fp64", "exact exp", "sw exp2", "fp64 poly", "shift K=2", "shift K=4", "shift K=8", "shift K=8 irr", "reduced f", "offset -2", "offset -8", "offset -16", "offset -64", "-16 + K=4", "-16 + K=8", "-16 + K=32", "-16 + row K=8"};
  printf("n=%d r=%d g=%g sum=%.10e sum|t|=%.6e cond=%.1f\n", n, r, g, o[NV + 1], o[NV], o[NV] / fabs(o[NV + 1]));
  for (int v = 0; v < NV; ++v) printf("  %-12s rel.err of sum = %+.3e   (per |t|: %+.3e)\n", names[v], o[v] / fabs(o[NV + 1]), o[v] / o[NV]);
  return 0;
}
