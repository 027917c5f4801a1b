// Sparse COO MTTKRP and squared error (reference tensors.py:263-273, 291-301).
// fp64 CUDA-core kernels; every reduction has a fixed order, so results are
// run-to-run deterministic, and the MTTKRP reproduces np.add.at bit for bit.
#include "mttkrp_coo.cuh"

namespace ntf {

namespace {

constexpr int kCooWarps = 8;  // output rows per 256-thread block

// One warp per output row, lanes over the rank columns (up to 4 per lane);
// the row's entries in perm order, each (row, column) summed sequentially.
struct Factors {
  const double* f[4];
};

__global__ void __launch_bounds__(kCooWarps * 32) mttkrp_coo_kernel(CooView t, int mode, Factors F,
                                                                    int R, double* __restrict__ out,
                                                                    const int* stop_flag) {
  pdl_trigger();
  pdl_wait();  // factors come from the preceding row updates
  if (stop_flag && *stop_flag) return;
  const int m = mode - 1;
  const int N = t.order;
  // companions, highest mode first (tensors.py:223-225, 266-270)
  int c[3] = {0, 0, 0};
  for (int q = N - 1, k = 0; q >= 0; --q)
    if (q != m) c[k++] = q;
  const int c0 = c[0], c1 = c[1], c2 = c[2];
  const double* F0 = F.f[c0];
  const double* F1 = F.f[c1];
  const double* F2 = N == 4 ? F.f[c2] : nullptr;
  const int lane = threadIdx.x & 31;
  const int cb = static_cast<int>(blockIdx.y) * 128;  // column chunk (ranks above 128)
  const int64_t row = static_cast<int64_t>(blockIdx.x) * kCooWarps + (threadIdx.x >> 5);
  if (row >= t.dims[m]) return;
  const int64_t* perm = t.perm[m];
  const int64_t e0 = t.rowptr[m][row], e1 = t.rowptr[m][row + 1];
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t e = e0; e < e1; ++e) {
    const int64_t q = perm ? perm[e] : e;
    const int64_t i0 = t.idx[q * N + c0], i1 = t.idx[q * N + c1];
    const int64_t i2 = F2 ? t.idx[q * N + c2] : 0;
    const double v = t.vals[q];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int r = cb + lane + 32 * u;
      if (r < R) {  // explicit rounding: no FMA contraction, as numpy's multiply-then-add
        double p = __dmul_rn(F0[i0 * R + r], F1[i1 * R + r]);
        if (F2) p = __dmul_rn(p, F2[i2 * R + r]);
        acc[u] = __dadd_rn(acc[u], __dmul_rn(p, v));
      }
    }
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int r = cb + lane + 32 * u;
    if (r < R) out[row * R + r] = acc[u];
  }
}

constexpr int kSqBlocks = 256, kSqThreads = 256;

// Per-block partials of (sum vals^2, sum_e vals_e * sum_r A B C); fixed
// strided entry subsets per thread, tree reduction in fixed order.
__global__ void __launch_bounds__(kSqThreads) coo_cross_kernel(CooView t, Factors F, int R,
                                                               double* __restrict__ part) {
  const int N = t.order;
  const double* A = F.f[0];
  __shared__ double s0[kSqThreads], s1[kSqThreads];
  double x2 = 0.0, cross = 0.0;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(kSqThreads) + threadIdx.x; e < t.nnz;
       e += static_cast<int64_t>(gridDim.x) * kSqThreads) {
    const double v = t.vals[e];
    x2 += v * v;
    if (A) {
      double w = 0.0;
      for (int r = 0; r < R; ++r) {
        double p = A[t.idx[e * N] * R + r];  // rows = A[i] * B[j] * C[k] (* D[l]) (tensors.py:292-294)
        for (int m = 1; m < N; ++m) p *= F.f[m][t.idx[e * N + m] * R + r];
        w += p;
      }
      cross += v * w;
    }
  }
  s0[threadIdx.x] = x2;
  s1[threadIdx.x] = cross;
  __syncthreads();
  for (int o = kSqThreads / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      s0[threadIdx.x] += s0[threadIdx.x + o];
      s1[threadIdx.x] += s1[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[blockIdx.x * 2] = s0[0];
    part[blockIdx.x * 2 + 1] = s1[0];
  }
}

// One block: sum the partials in order, then sum over (r, s) of the Hadamard
// of the three factor Grams (each Gram entry a fixed-order dot product), and
// combine as tensors.py:299-300.
__global__ void __launch_bounds__(kSqThreads) coo_finish_kernel(CooView t, Factors F, int R,
                                                                const double* __restrict__ part,
                                                                double* __restrict__ out2) {
  __shared__ double red[kSqThreads];
  const double* A = F.f[0];
  double g = 0.0;
  if (A) {
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
      const int r = e / R, s = e - (e / R) * R;
      double h = 1.0;
      for (int m = 0; m < t.order; ++m) {  // Hadamard of the factor Grams (tensors.py:295-298)
        const double* Fm = F.f[m];
        double gm = 0.0;
        for (int64_t i = 0; i < t.dims[m]; ++i) gm += Fm[i * R + r] * Fm[i * R + s];
        h = m == 0 ? gm : h * gm;
      }
      g += h;
    }
  }
  red[threadIdx.x] = g;
  __syncthreads();
  for (int o = kSqThreads / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double x2 = 0.0, cross = 0.0;
    for (int b = 0; b < kSqBlocks; ++b) {
      x2 += part[b * 2];
      cross += part[b * 2 + 1];
    }
    out2[0] = x2;
    out2[1] = A ? fmax(x2 - 2.0 * cross + red[0], 0.0) : 0.0;
  }
}

}  // namespace

cudaError_t mttkrp_coo_launch(const CooView& t_in, int mode, const double* const F[4], int R,
                              double* out, const int* stop_flag, cudaStream_t stream) {
  CooView t = t_in;
  if (t.order == 0) t.order = 3;
  if (R < 1 || R > NTF_MAX_RANK || mode < 1 || mode > t.order) return cudaErrorInvalidValue;
  Factors f{};
  for (int m = 0; m < t.order; ++m) f.f[m] = F[m];
  const int64_t rows = t.dims[mode - 1];
  const unsigned blocks = static_cast<unsigned>((rows + kCooWarps - 1) / kCooWarps);
  return launch_pdl(mttkrp_coo_kernel, dim3(blocks, (R + 127) / 128), dim3(kCooWarps * 32), 0, stream, t,
                    mode, f, R, out, stop_flag);
}

size_t coo_sq_error_workspace_bytes(int64_t nnz, int R) {
  (void)nnz;
  (void)R;
  return static_cast<size_t>(kSqBlocks) * 2 * sizeof(double);
}

cudaError_t coo_sq_error_launch(const CooView& t_in, const double* const F[4], int R, double* out2,
                                void* ws, cudaStream_t stream) {
  CooView t = t_in;
  if (t.order == 0) t.order = 3;
  Factors f{};
  for (int m = 0; m < t.order; ++m) f.f[m] = F ? F[m] : nullptr;
  double* part = static_cast<double*>(ws);
  coo_cross_kernel<<<kSqBlocks, kSqThreads, 0, stream>>>(t, f, R, part);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  coo_finish_kernel<<<1, kSqThreads, 0, stream>>>(t, f, R, part, out2);
  return cudaGetLastError();
}

}  // namespace ntf
