// kde_linalg.cpp — small dense fp64 linear algebra of the host chains (row-major d x d):
// Cholesky with the PD test of reading Z8, triangular and general inverses, the SPD square root
// of Eq. 35 (reading Z9), vech/unvech.  Product code: independent of oracle/.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "kde_host.h"

namespace kde {
namespace host {

// Cholesky A = L L^T with a relative pivot test (positive-definiteness, reading Z8).
bool cholesky(const std::vector<double>& A, int d, std::vector<double>& L) {
  L.assign((size_t)d * d, 0.0);
  double mx = 0.0;
  for (int i = 0; i < d; ++i) {
    if (!std::isfinite(A[i * d + i])) return false;
    mx = std::max(mx, std::fabs(A[i * d + i]));
  }
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j)
      if (!std::isfinite(A[i * d + j]) || A[i * d + j] != A[j * d + i]) return false;
  for (int j = 0; j < d; ++j) {
    double s = A[j * d + j];
    for (int k = 0; k < j; ++k) s -= L[j * d + k] * L[j * d + k];
    if (!(s > 1e-12 * mx)) return false;
    L[j * d + j] = std::sqrt(s);
    for (int i = j + 1; i < d; ++i) {
      double t = A[i * d + j];
      for (int k = 0; k < j; ++k) t -= L[i * d + k] * L[j * d + k];
      L[i * d + j] = t / L[j * d + j];
    }
  }
  return true;
}

// Inverse of a lower-triangular matrix by forward substitution.
std::vector<double> tri_lower_inverse(const std::vector<double>& L, int d) {
  std::vector<double> M((size_t)d * d, 0.0);
  for (int col = 0; col < d; ++col) {
    for (int i = 0; i < d; ++i) {
      double s = (i == col) ? 1.0 : 0.0;
      for (int k = 0; k < i; ++k) s -= L[i * d + k] * M[k * d + col];
      M[i * d + col] = s / L[i * d + i];
    }
  }
  return M;
}

// Principal square root of an SPD matrix by the Denman–Beavers iteration (the paper used
// ALGLIB; reading Z9).  Y_{k+1} = (Y_k + Z_k^-1)/2, Z_{k+1} = (Z_k + Y_k^-1)/2.
bool gen_inverse(const std::vector<double>& A, int d, std::vector<double>& R) {
  // Gauss–Jordan with partial pivoting on a general matrix.
  std::vector<double> M = A;
  R.assign((size_t)d * d, 0.0);
  for (int i = 0; i < d; ++i) R[i * d + i] = 1.0;
  for (int c = 0; c < d; ++c) {
    int p = c;
    for (int r = c + 1; r < d; ++r)
      if (std::fabs(M[r * d + c]) > std::fabs(M[p * d + c])) p = r;
    if (M[p * d + c] == 0.0) return false;
    if (p != c)
      for (int k = 0; k < d; ++k) { std::swap(M[p * d + k], M[c * d + k]); std::swap(R[p * d + k], R[c * d + k]); }
    double piv = M[c * d + c];
    for (int k = 0; k < d; ++k) { M[c * d + k] /= piv; R[c * d + k] /= piv; }
    for (int r = 0; r < d; ++r) {
      if (r == c) continue;
      double f = M[r * d + c];
      if (f == 0.0) continue;
      for (int k = 0; k < d; ++k) { M[r * d + k] -= f * M[c * d + k]; R[r * d + k] -= f * R[c * d + k]; }
    }
  }
  return true;
}

bool spd_sqrt(const std::vector<double>& A, int d, std::vector<double>& S) {
  std::vector<double> Y = A, Z((size_t)d * d, 0.0), Yi, Zi;
  for (int i = 0; i < d; ++i) Z[i * d + i] = 1.0;
  for (int it = 0; it < 100; ++it) {
    if (!gen_inverse(Y, d, Yi) || !gen_inverse(Z, d, Zi)) return false;
    double diff = 0.0, nrm = 0.0;
    for (size_t k = 0; k < Y.size(); ++k) {
      double yn = 0.5 * (Y[k] + Zi[k]);
      double zn = 0.5 * (Z[k] + Yi[k]);
      diff = std::max(diff, std::fabs(yn - Y[k]));
      nrm = std::max(nrm, std::fabs(yn));
      Y[k] = yn;
      Z[k] = zn;
    }
    if (diff <= 1e-15 * nrm) break;
  }
  S = Y;
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < i; ++j) S[i * d + j] = S[j * d + i] = 0.5 * (S[i * d + j] + S[j * d + i]);
  return true;
}

std::vector<double> unvech(const double* v, int d) {
  std::vector<double> A((size_t)d * d);
  int t = 0;
  for (int j = 0; j < d; ++j)
    for (int i = j; i < d; ++i) { A[i * d + j] = A[j * d + i] = v[t]; ++t; }
  return A;
}

void vech(const std::vector<double>& A, int d, double* v) {
  int t = 0;
  for (int j = 0; j < d; ++j)
    for (int i = j; i < d; ++i) v[t++] = A[i * d + j];
}

void vech_llt(const double* x, int d, double* out) {
  std::vector<double> L((size_t)d * d, 0.0);
  int t = 0;
  for (int j = 0; j < d; ++j)
    for (int i = j; i < d; ++i) L[(size_t)i * d + j] = x[t++];
  std::vector<double> H((size_t)d * d, 0.0);
  for (int i = 0; i < d; ++i)
    for (int j = 0; j <= i; ++j) {
      double s = 0.0;
      for (int k = 0; k <= j; ++k) s += L[(size_t)i * d + k] * L[(size_t)j * d + k];   // (L L^T)_ij, k <= min(i, j)
      H[(size_t)i * d + j] = H[(size_t)j * d + i] = s;
    }
  vech(H, d, out);
}

}  // namespace host
}  // namespace kde
