// Ridge factorisation of ridge_factor_kernel (one CTA on the plan's side
// stream, concurrent with the mode's MTTKRP).
#pragma once

#include "common.cuh"

namespace ntf {

// ---------------------------------------------------------------------------
// Ridge Cholesky in shared memory (solver.ridge_cholesky, solver.py:167-175):
// H = G_a o G_b (o G_c for order 4) + rho*I (companion Gram, solver.py:196-204), lower factor
// L with L L^T = H.  Right-looking, one barrier per column: the trailing
// update uses the unscaled column (L[i][j] L[k][j] / pivot) and columns are
// scaled at the end.  A non-positive or non-finite pivot raises NOT_PD.
// ---------------------------------------------------------------------------
// col (L in global memory): a shared-memory copy of the pivot column, so the
// trailing update reads one global element per update instead of three.
__device__ inline void build_and_factor(double* L, int ldl, int R, const double* __restrict__ Ga,
                                        const double* __restrict__ Gb, double rho, int* status,
                                        bool* bad, const double* __restrict__ Gc = nullptr,
                                        double* col = nullptr) {
  const int tid = threadIdx.x;
  for (int e = tid; e < R * R; e += blockDim.x) {
    const int i = e / R, k = e - (e / R) * R;
    double h = Ga[e] * Gb[e];
    if (Gc) h *= Gc[e];  // order 4: ((G_a o G_b) o G_c), highest mode first
    if (i == k) h += rho;
    L[i * ldl + k] = h;
  }
  __syncthreads();
  for (int j = 0; j < R; ++j) {
    const double piv = L[j * ldl + j];
    if (!(piv > 0.0) || !isfinite(piv)) {
      if (tid == 0) {
        raise_status(status, kDevNotPD);
        *bad = true;
      }
      __syncthreads();
      return;
    }
    const double inv = 1.0 / piv;
    const int n = R - j - 1;  // trailing order; update the lower triangle i >= k > j
    if (col) {
      for (int i = j + 1 + tid; i < R; i += blockDim.x) col[i] = L[i * ldl + j];
      __syncthreads();
      for (int e = tid; e < n * n; e += blockDim.x) {
        const int ii = e / n, kk = e - (e / n) * n;
        if (kk > ii) continue;
        const int i = j + 1 + ii, k = j + 1 + kk;
        L[i * ldl + k] -= col[i] * col[k] * inv;
      }
    } else {
      for (int e = tid; e < n * n; e += blockDim.x) {
        const int ii = e / n, kk = e - (e / n) * n;
        if (kk > ii) continue;
        const int i = j + 1 + ii, k = j + 1 + kk;
        L[i * ldl + k] -= L[i * ldl + j] * L[k * ldl + j] * inv;
      }
    }
    __syncthreads();
  }
  // scale: L[i][j] = U[i][j] / sqrt(U[j][j]) for i > j, L[j][j] = sqrt(U[j][j])
  for (int e = tid; e < R * R; e += blockDim.x) {
    const int i = e / R, k = e - (e / R) * R;
    if (k < i) L[i * ldl + k] = L[i * ldl + k] / sqrt(L[k * ldl + k]);
  }
  __syncthreads();
  for (int j = tid; j < R; j += blockDim.x) L[j * ldl + j] = sqrt(L[j * ldl + j]);
  __syncthreads();
}

// Ridge buffer (out), written by one block with smem >= ridge_smem_doubles(R):
//   [0, R*R)            L, row-major lower Cholesky factor of H
//   [R*R, R*R+R)        1 / diag(L)
//   [R*R+R, 2R*R+R)     H^-1 = L^-T L^-1  (R <= 64 only)
//   [2R*R+R, 3R*R+R)    H = G_a o G_b + rho I
// Ranks above kRidgeSmemMaxR (R (R+1) doubles no longer fit the 227 KB of
// shared memory) factor in place in `out` (global memory, L2-resident); the
// kernel runs on the side stream, concurrently with the mode's MTTKRP.
constexpr int kRidgeSmemMaxR = 160;
__host__ __device__ inline int ridge_smem_doubles(int R) {
  if (R > kRidgeSmemMaxR) return R;  // the pivot-column copy only
  return (R <= 64 ? 2 : 1) * R * (R + 1) + R;
}
__host__ __device__ inline int ridge_threads(int R) { return R > kRidgeSmemMaxR ? 1024 : 256; }

__device__ inline void ridge_factor_block(const double* Ga, const double* Gb, double rho, int R,
                                          double* out, int* status, double* sm,
                                          const double* Gc = nullptr) {
  const bool in_place = R > kRidgeSmemMaxR;
  const int ldl = in_place ? R : R + 1;
  double* L = in_place ? out : sm;
  double* Li = L + R * ldl;  // L^-1 (lower), R <= 64
  __shared__ bool bad;
  if (threadIdx.x == 0) bad = false;
  __syncthreads();
  double* Hout = out + 2 * R * R + R;
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    const int i = e / R, k = e - (e / R) * R;
    double h = Ga[e] * Gb[e];
    if (Gc) h *= Gc[e];
    Hout[e] = h + (i == k ? rho : 0.0);
  }
  build_and_factor(L, ldl, R, Ga, Gb, rho, status, &bad, Gc, in_place ? sm : nullptr);
  if (bad) return;
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    const int i = e / R, k = e - (e / R) * R;
    out[e] = k <= i ? L[i * ldl + k] : 0.0;
  }
  double* rdiag = Li + R * ldl;  // [R] 1/L[i][i] (R <= 64 path)
  for (int j = threadIdx.x; j < R; j += blockDim.x) {
    const double r = 1.0 / L[j * ldl + j];
    out[R * R + j] = r;
    if (R <= 64) rdiag[j] = r;
  }
  if (R > 64) return;
  __syncthreads();
  // L^-1 by forward substitution on the identity, one column per thread
  for (int j = threadIdx.x; j < R; j += blockDim.x) {
    for (int i = 0; i < R; ++i) {
      double s = i == j ? 1.0 : 0.0;
      if (i < j) {
        Li[i * ldl + j] = 0.0;
        continue;
      }
      for (int k = j; k < i; ++k) s -= L[i * ldl + k] * Li[k * ldl + j];
      Li[i * ldl + j] = s * rdiag[i];
    }
  }
  __syncthreads();
  // H^-1 = L^-T L^-1: (a, b) = sum_{i >= max(a,b)} Li[i][a] Li[i][b]
  double* Hinv = out + R * R + R;
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    const int a = e / R, b = e - (e / R) * R;
    double s = 0.0;
    for (int i = a > b ? a : b; i < R; ++i) s += Li[i * ldl + a] * Li[i * ldl + b];
    Hinv[e] = s;
  }
}

}  // namespace ntf
