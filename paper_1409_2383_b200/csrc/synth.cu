// Counter-based synthetic NTF tensors, generated in HBM.
//
// Stands in for the reference's synthetic protocol (bench.py:34-46: U[0,1)
// true factors, X = [[A,B,C]] + i.i.d. Gaussian noise at a given SNR) with a
// generator whose every element is a pure function of its global index, so a
// rank generates only its own slabs (X[I_p,:,:], X[:,J_p,:], X[:,:,K_p]) and
// the bytes do not depend on how the tensor is sharded:
//   x[i,j,k] = clean + sigma * z(e),  e = (i J + j) K + k
//   clean    = sum_{r = 0..R-1} (A[i,r] B[j,r]) C[k,r]   sequential in r
//   z(e)     = sqrt(-2 ln u1) cos(2 pi u2)  (Box-Muller), u1 in (0,1] and
//              u2 in [0,1) from SplitMix64 words 2e+1 and 2e+2 of `key`
// ln and cos are evaluated with fixed polynomials in correctly rounded
// +, -, *, /, sqrt only (explicit __d*_rn intrinsics: no FMA contraction),
// so the host restatements (oracle/synth_oracle.c, oracle/ntf_oracle.py
// synth_box) reproduce every byte.  The true factors and sigma come from the
// host (paper_1409_2383_b200/synth.py).
#include <algorithm>

#include "synth.cuh"

namespace ntf {

namespace {

constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;
constexpr double kSqrt2 = 0x1.6a09e667f3bcdp+0;
constexpr double kPio2 = 0x1.921fb54442d18p+0;
constexpr double kLn2Hi = 0x1.62e42fee00000p-1;
constexpr double kLn2Lo = 0x1.a39ef35793c76p-33;
// 1/(2k+1), k = 0..11: ln m = 2 s sum s^(2k)/(2k+1), s = (m-1)/(m+1)
__constant__ double kLn[12] = {0x1.0000000000000p+0, 0x1.5555555555555p-2, 0x1.999999999999ap-3,
                               0x1.2492492492492p-3, 0x1.c71c71c71c71cp-4, 0x1.745d1745d1746p-4,
                               0x1.3b13b13b13b14p-4, 0x1.1111111111111p-4, 0x1.e1e1e1e1e1e1ep-5,
                               0x1.af286bca1af28p-5, 0x1.8618618618618p-5, 0x1.642c8590b2164p-5};
// (-1)^k / (2k)!  and  (-1)^k / (2k+1)!, k = 0..10
__constant__ double kCos[11] = {0x1.0000000000000p+0,  -0x1.0000000000000p-1, 0x1.5555555555555p-5,
                                -0x1.6c16c16c16c17p-10, 0x1.a01a01a01a01ap-16, -0x1.27e4fb7789f5cp-22,
                                0x1.1eed8eff8d898p-29,  -0x1.93974a8c07c9dp-37, 0x1.ae7f3e733b81fp-45,
                                -0x1.6827863b97d97p-53, 0x1.e542ba4020225p-62};
__constant__ double kSin[11] = {0x1.0000000000000p+0,  -0x1.5555555555555p-3, 0x1.1111111111111p-7,
                                -0x1.a01a01a01a01ap-13, 0x1.71de3a556c734p-19, -0x1.ae64567f544e4p-26,
                                0x1.6124613a86d09p-33,  -0x1.ae7f3e733b81fp-41, 0x1.952c77030ad4ap-49,
                                -0x1.2f49b46814157p-57, 0x1.71b8ef6dcf572p-66};

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// standard normal of element e (Box-Muller, cosine branch)
__device__ double std_normal(uint64_t key, uint64_t e) {
  const uint64_t w1 = mix64(key + (2 * e + 1) * kGamma);
  const uint64_t w2 = mix64(key + (2 * e + 2) * kGamma);
  // ln u1, u1 = m 2^E with m in (sqrt(1/2), sqrt(2)]
  const double u1 = __dmul_rn(static_cast<double>((w1 >> 11) + 1), 0x1p-53);
  int ex = 0;
  const double mant = frexp(u1, &ex);  // exact: u1 = mant 2^ex, mant in [0.5, 1)
  double m = __dmul_rn(mant, 2.0);
  int E = ex - 1;
  if (m > kSqrt2) {
    m = mant;
    E = ex;
  }
  const double s = __ddiv_rn(__dsub_rn(m, 1.0), __dadd_rn(m, 1.0));
  const double s2 = __dmul_rn(s, s);
  double p = kLn[11];
#pragma unroll
  for (int k = 10; k >= 0; --k) p = __dadd_rn(__dmul_rn(p, s2), kLn[k]);
  const double lnm = __dmul_rn(__dmul_rn(2.0, s), p);
  const double Ed = static_cast<double>(E);
  const double ln = __dadd_rn(__dmul_rn(Ed, kLn2Hi), __dadd_rn(__dmul_rn(Ed, kLn2Lo), lnm));
  const double rad = __dsqrt_rn(__dmul_rn(-2.0, ln));
  // cos(2 pi u2): quadrant q, fraction f of the quadrant, folded to g <= 1/2
  const uint64_t n2 = w2 >> 11;
  const int q = static_cast<int>(n2 >> 51);
  const uint64_t fi = n2 & ((1ull << 51) - 1);
  const bool sw = fi > (1ull << 50);
  const double g = __dmul_rn(static_cast<double>(sw ? (1ull << 51) - fi : fi), 0x1p-51);
  const double th = __dmul_rn(g, kPio2);
  const double t2 = __dmul_rn(th, th);
  double c = kCos[10], sn = kSin[10];
#pragma unroll
  for (int k = 9; k >= 0; --k) {
    c = __dadd_rn(__dmul_rn(c, t2), kCos[k]);
    sn = __dadd_rn(__dmul_rn(sn, t2), kSin[k]);
  }
  sn = __dmul_rn(th, sn);
  const double cq = sw ? sn : c;  // cos(pi f / 2)
  const double sq = sw ? c : sn;  // sin(pi f / 2)
  const double v = q == 0 ? cq : (q == 1 ? -sq : (q == 2 ? -cq : sq));
  return __dmul_rn(rad, v);
}

template <typename T>
__device__ __forceinline__ T to_out(double x);
template <>
__device__ __forceinline__ float to_out<float>(double x) {
  return __double2float_rn(x);
}
template <>
__device__ __forceinline__ double to_out<double>(double x) {
  return x;
}

constexpr int kPQ = 8;  // (i, j) rows per pass of the tile kernel

// One k-tile of kt columns per block (thread = k), C^T of the tile staged in
// shared memory, kPQ (i, j) rows per pass with their A*B products broadcast
// from shared memory; the block walks a contiguous range of rows.
template <typename T>
__global__ void __launch_bounds__(128) synth_tile_kernel(T* __restrict__ out, SynthBox b,
                                                         const double* __restrict__ A,
                                                         const double* __restrict__ B,
                                                         const double* __restrict__ C, int R,
                                                         double sigma, uint64_t key, int kt,
                                                         int64_t rows_per_block) {
  extern __shared__ double sm[];
  double* ct = sm;               // [R][kt]
  double* pr = sm + R * kt;      // [kPQ][R]
  const int64_t bi = b.hi[0] - b.lo[0], bj = b.hi[1] - b.lo[1], bk = b.hi[2] - b.lo[2];
  const int64_t kofs = static_cast<int64_t>(blockIdx.x) * kt;
  const int nk = static_cast<int>(bk - kofs < kt ? bk - kofs : kt);
  for (int idx = threadIdx.x; idx < R * kt; idx += blockDim.x) {
    const int r = idx / kt, kk = idx - (idx / kt) * kt;
    ct[idx] = kk < nk ? C[(b.lo[2] + kofs + kk) * R + r] : 0.0;
  }
  const int64_t rows = bi * bj;
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * rows_per_block;
  const int64_t r1 = rows < r0 + rows_per_block ? rows : r0 + rows_per_block;
  const int64_t J = b.dims[1], K = b.dims[2];
  for (int64_t row = r0; row < r1; row += kPQ) {
    const int nq = static_cast<int>(r1 - row < kPQ ? r1 - row : kPQ);
    __syncthreads();  // C^T staged / the previous rows' products consumed
    for (int idx = threadIdx.x; idx < kPQ * R; idx += blockDim.x) {
      const int q = idx / R, r = idx - (idx / R) * R;
      double v = 0.0;
      if (q < nq) {
        const int64_t rr = row + q;
        const int64_t i = b.lo[0] + rr / bj, j = b.lo[1] + rr % bj;
        v = __dmul_rn(A[i * R + r], B[j * R + r]);
      }
      pr[idx] = v;
    }
    __syncthreads();
    for (int kk = threadIdx.x; kk < nk; kk += blockDim.x) {
      double acc[kPQ];
#pragma unroll
      for (int q = 0; q < kPQ; ++q) acc[q] = 0.0;
      for (int r = 0; r < R; ++r) {
        const double c = ct[r * kt + kk];
#pragma unroll
        for (int q = 0; q < kPQ; ++q) acc[q] = __dadd_rn(acc[q], __dmul_rn(pr[q * R + r], c));
      }
      const int64_t k = b.lo[2] + kofs + kk;
#pragma unroll
      for (int q = 0; q < kPQ; ++q) {
        if (q < nq) {
          const int64_t rr = row + q;
          const int64_t i = b.lo[0] + rr / bj, j = b.lo[1] + rr % bj;
          const uint64_t e = static_cast<uint64_t>((i * J + j) * K + k);
          const double x = __dadd_rn(acc[q], __dmul_rn(sigma, std_normal(key, e)));
          out[rr * bk + kofs + kk] = to_out<T>(x);
        }
      }
    }
  }
}

// Any rank: one thread per element, factors read through the cache.
template <typename T>
__global__ void synth_direct_kernel(T* __restrict__ out, SynthBox b, const double* __restrict__ A,
                                    const double* __restrict__ B, const double* __restrict__ C,
                                    int R, double sigma, uint64_t key) {
  const int64_t bi = b.hi[0] - b.lo[0], bj = b.hi[1] - b.lo[1], bk = b.hi[2] - b.lo[2];
  const int64_t n = bi * bj * bk;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t kk = t % bk, rr = t / bk;
    const int64_t i = b.lo[0] + rr / bj, j = b.lo[1] + rr % bj, k = b.lo[2] + kk;
    double acc = 0.0;
    for (int r = 0; r < R; ++r)
      acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(A[i * R + r], B[j * R + r]), C[k * R + r]));
    const uint64_t e = static_cast<uint64_t>((i * b.dims[1] + j) * b.dims[2] + k);
    out[t] = to_out<T>(__dadd_rn(acc, __dmul_rn(sigma, std_normal(key, e))));
  }
}

int sm_count_synth() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

template <typename T>
cudaError_t launch_typed(T* out, const SynthBox& b, const double* A, const double* B, const double* C,
                         int R, double sigma, uint64_t key, cudaStream_t stream) {
  const int64_t bi = b.hi[0] - b.lo[0], bj = b.hi[1] - b.lo[1], bk = b.hi[2] - b.lo[2];
  if (bi <= 0 || bj <= 0 || bk <= 0) return cudaSuccess;
  const int sms = sm_count_synth();
  constexpr size_t kBudget = 160 * 1024;
  int kt = 0;
  for (int cand : {128, 64, 32})
    if (static_cast<size_t>(R) * (cand + kPQ) * sizeof(double) <= kBudget) {
      kt = cand;
      break;
    }
  if (kt == 0) {
    const int64_t n = bi * bj * bk;
    const int blocks = static_cast<int>(std::min<int64_t>((n + 255) / 256, 32 * sms));
    synth_direct_kernel<T><<<blocks, 256, 0, stream>>>(out, b, A, B, C, R, sigma, key);
    return cudaGetLastError();
  }
  while (kt > 32 && kt / 2 >= bk) kt /= 2;  // short k extents: narrower tiles
  const size_t smem = static_cast<size_t>(R) * (kt + kPQ) * sizeof(double);
  cudaError_t e = cudaFuncSetAttribute(synth_tile_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(kBudget));
  if (e != cudaSuccess) return e;
  const int64_t ktiles = (bk + kt - 1) / kt;
  const int64_t rows = bi * bj;
  int64_t gy = std::max<int64_t>(1, (8 * sms + ktiles - 1) / ktiles);
  gy = std::min<int64_t>(gy, std::min<int64_t>(65535, (rows + kPQ - 1) / kPQ));
  int64_t rpb = (rows + gy - 1) / gy;
  rpb = ((rpb + kPQ - 1) / kPQ) * kPQ;
  gy = (rows + rpb - 1) / rpb;
  if (ktiles > 0x7fffffff) return cudaErrorInvalidValue;
  synth_tile_kernel<T><<<dim3(static_cast<unsigned>(ktiles), static_cast<unsigned>(gy)), kt, smem, stream>>>(
      out, b, A, B, C, R, sigma, key, kt, rpb);
  return cudaGetLastError();
}

}  // namespace

cudaError_t synth_dense_launch(int x_dtype, void* out, const SynthBox& box, const double* A,
                               const double* B, const double* C, int R, double sigma, uint64_t key,
                               cudaStream_t stream) {
  if (x_dtype == NTF_F32)
    return launch_typed(static_cast<float*>(out), box, A, B, C, R, sigma, key, stream);
  return launch_typed(static_cast<double*>(out), box, A, B, C, R, sigma, key, stream);
}

}  // namespace ntf
