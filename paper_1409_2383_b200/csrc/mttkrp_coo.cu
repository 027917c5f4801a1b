// Sparse COO MTTKRP and squared error (reference tensors.py:263-273, 291-301).
// fp64 CUDA-core kernels; every reduction has a fixed order, so results are
// run-to-run deterministic, and the MTTKRP reproduces np.add.at bit for bit.
#include "mttkrp_coo.cuh"

namespace ntf {

namespace {

constexpr int kCooWarps = 8;  // output rows per 256-thread block

// One warp per output row, lanes over the rank columns (up to 4 per lane);
// the row's entries in perm order, each (row, column) summed sequentially.
__global__ void __launch_bounds__(kCooWarps * 32) mttkrp_coo_kernel(CooView t, int mode,
                                                                    const double* __restrict__ A,
                                                                    const double* __restrict__ B,
                                                                    const double* __restrict__ C,
                                                                    int R, double* __restrict__ out,
                                                                    const int* stop_flag) {
  pdl_trigger();
  pdl_wait();  // factors come from the preceding row updates
  if (stop_flag && *stop_flag) return;
  const int m = mode - 1;
  // companions, highest mode first (tensors.py:223-225, 266-270)
  const int c0 = m == 2 ? 1 : 2, c1 = m == 0 ? 1 : 0;
  const double* F[3] = {A, B, C};
  const double* F0 = F[c0];
  const double* F1 = F[c1];
  const int lane = threadIdx.x & 31;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * kCooWarps + (threadIdx.x >> 5);
  if (row >= t.dims[m]) return;
  const int64_t* perm = t.perm[m];
  const int64_t e0 = t.rowptr[m][row], e1 = t.rowptr[m][row + 1];
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t e = e0; e < e1; ++e) {
    const int64_t q = perm ? perm[e] : e;
    const int64_t i0 = t.idx[q * 3 + c0], i1 = t.idx[q * 3 + c1];
    const double v = t.vals[q];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int r = lane + 32 * u;
      if (r < R) {  // explicit rounding: no FMA contraction, as numpy's multiply-then-add
        const double c = __dmul_rn(__dmul_rn(F0[i0 * R + r], F1[i1 * R + r]), v);
        acc[u] = __dadd_rn(acc[u], c);
      }
    }
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int r = lane + 32 * u;
    if (r < R) out[row * R + r] = acc[u];
  }
}

constexpr int kSqBlocks = 256, kSqThreads = 256;

// Per-block partials of (sum vals^2, sum_e vals_e * sum_r A B C); fixed
// strided entry subsets per thread, tree reduction in fixed order.
__global__ void __launch_bounds__(kSqThreads) coo_cross_kernel(CooView t, const double* __restrict__ A,
                                                               const double* __restrict__ B,
                                                               const double* __restrict__ C, int R,
                                                               double* __restrict__ part) {
  __shared__ double s0[kSqThreads], s1[kSqThreads];
  double x2 = 0.0, cross = 0.0;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(kSqThreads) + threadIdx.x; e < t.nnz;
       e += static_cast<int64_t>(gridDim.x) * kSqThreads) {
    const double v = t.vals[e];
    x2 += v * v;
    if (A) {
      const int64_t i = t.idx[e * 3], j = t.idx[e * 3 + 1], k = t.idx[e * 3 + 2];
      double w = 0.0;
      for (int r = 0; r < R; ++r) {
        double p = A[i * R + r];  // rows = A[i] * B[j] * C[k] (tensors.py:292-294)
        p *= B[j * R + r];
        p *= C[k * R + r];
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
__global__ void __launch_bounds__(kSqThreads) coo_finish_kernel(CooView t, const double* __restrict__ A,
                                                                const double* __restrict__ B,
                                                                const double* __restrict__ C, int R,
                                                                const double* __restrict__ part,
                                                                double* __restrict__ out2) {
  __shared__ double red[kSqThreads];
  double g = 0.0;
  if (A) {
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
      const int r = e / R, s = e - (e / R) * R;
      double ga = 0.0, gb = 0.0, gc = 0.0;
      for (int64_t i = 0; i < t.dims[0]; ++i) ga += A[i * R + r] * A[i * R + s];
      for (int64_t i = 0; i < t.dims[1]; ++i) gb += B[i * R + r] * B[i * R + s];
      for (int64_t i = 0; i < t.dims[2]; ++i) gc += C[i * R + r] * C[i * R + s];
      g += ga * gb * gc;
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

cudaError_t mttkrp_coo_launch(const CooView& t, int mode, const double* A, const double* B,
                              const double* C, int R, double* out, const int* stop_flag,
                              cudaStream_t stream) {
  if (R < 1 || R > 128 || mode < 1 || mode > 3) return cudaErrorInvalidValue;
  const int64_t rows = t.dims[mode - 1];
  const unsigned blocks = static_cast<unsigned>((rows + kCooWarps - 1) / kCooWarps);
  return launch_pdl(mttkrp_coo_kernel, dim3(blocks), dim3(kCooWarps * 32), 0, stream, t, mode, A, B,
                    C, R, out, stop_flag);
}

size_t coo_sq_error_workspace_bytes(int64_t nnz, int R) {
  (void)nnz;
  (void)R;
  return static_cast<size_t>(kSqBlocks) * 2 * sizeof(double);
}

cudaError_t coo_sq_error_launch(const CooView& t, const double* A, const double* B, const double* C,
                                int R, double* out2, void* ws, cudaStream_t stream) {
  double* part = static_cast<double*>(ws);
  coo_cross_kernel<<<kSqBlocks, kSqThreads, 0, stream>>>(t, A, B, C, R, part);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  coo_finish_kernel<<<1, kSqThreads, 0, stream>>>(t, A, B, C, R, part, out2);
  return cudaGetLastError();
}

}  // namespace ntf
