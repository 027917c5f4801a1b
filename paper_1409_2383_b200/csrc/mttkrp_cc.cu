// Dense MTTKRP on CUDA cores (sm_100a), all three modes, fp32 or fp64 tensor.
//
// Replaces tensors.mttkrp_factors dense branch (reference tensors.py:254-262):
//   M_n = X_(n) @ khatri_rao(companions, highest mode first)
// without the cached unfolding copy (tensors.py:63-71) and without the
// materialised Khatri-Rao matrix (tensors.py:203-220).  Every mode streams the
// native row-major X[i][j][k] exactly once.
//
// GEMM view used for all modes:  out[m, r] = sum_q X(m, q) * W(q, r),
//   W(q, r) = F_hi[q_hi, r] * F_lo[q_lo, r]   (KR row formed on the fly)
//   KIND_Q (modes 1, 2):  q = o*K + k, k the contiguous tensor index,
//       mode 1: m = i, o = j  (X(m,q) = X[i*JK + q]),   W = B[j] * C[k]
//       mode 2: m = j, o = i  (X(m,q) = X[i*JK + j*K + k]), W = A[i] * C[k]
//   KIND_M (mode 3):       q = p = i*J + j, m = k contiguous,  W = A[i] * B[j]
//
// Tiling: a CTA owns BM = 32*TM output rows and all R columns; warp w owns
// columns [w*TR, (w+1)*TR).  Lane l owns rows l + 32*t (t < TM).  The
// reduction range is cut into chunks of BQ q-values; a CTA streams a
// contiguous run of chunks (split-K) through a 3-stage cp.async ring, forms
// the chunk's KR rows W (fp64 product rounded once to the compute type) in
// shared memory, and accumulates with register-tiled FMAs where W is a warp
// broadcast.  Precision recipe for fp32 tensors: fp32 FMA chains
// of BQ terms, folded into a double-float (hi, lo) accumulator each chunk, so
// no structured rounding of the factors and no long fp32 chains.  Each CTA
// writes its fp64 partial; splits are summed in a fixed order by the consumer
// (deterministic, no float atomics).
#include "mttkrp_cc.cuh"

namespace ntf {

namespace {

template <typename XT>
struct ComputeTraits;
template <>
struct ComputeTraits<float> {
  using acc_t = float;
};
template <>
struct ComputeTraits<double> {
  using acc_t = double;
};

template <typename XT, int TM>
struct TileGeom {
  static constexpr int BM = 32 * TM;
  static constexpr int BQ = 32;
  static constexpr int STAGES = 3;
  // KIND_Q tile [BM][BQ+1] (odd pitch -> conflict-free column reads)
  static constexpr int kPitchQ = BQ + 1;
  static constexpr int kTileQ = BM * kPitchQ;
  // KIND_M tile [BQ][BM]
  static constexpr int kTileM = BQ * BM;
  static constexpr int kTile = kTileQ > kTileM ? kTileQ : kTileM;
};

__device__ __forceinline__ void fast_two_sum_acc(float& hi, float& lo, float a) {
  // (hi, lo) += a with Fast2Sum: exact when |hi| >= |a|, which holds after the
  // first chunk because one output's chunk sums are a small share of the total.
  const float s = hi + a;
  const float err = a - (s - hi);
  hi = s;
  lo += err;
}

template <typename XT, int TM, int TR, bool KIND_M, int VEC>
__global__ void __launch_bounds__(256, 1) mttkrp_cc_kernel(MttkrpCCParams p) {
  using G = TileGeom<XT, TM>;
  using acc_t = typename ComputeTraits<XT>::acc_t;
  constexpr int BM = G::BM;
  constexpr int BQ = G::BQ;
  constexpr int STAGES = G::STAGES;
  constexpr bool kTwoLevel = sizeof(XT) == 4;

  if (p.stop_flag && *p.stop_flag) return;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  XT* xs = reinterpret_cast<XT*>(smem_raw);                 // [STAGES][kTile]
  XT* ws = xs + STAGES * G::kTile;                           // [2][BQ][R_pad]

  const int R = p.R;
  const int R_pad = p.R_pad;
  const int tid = threadIdx.x;
  const int nthreads = blockDim.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int r0 = warp * TR;

  const int mtile = blockIdx.x;
  const int split = blockIdx.y;
  const int64_t m0 = static_cast<int64_t>(mtile) * BM;
  const int64_t c_begin = static_cast<int64_t>(split) * p.chunks_per_split;
  int64_t c_end = c_begin + p.chunks_per_split;
  if (c_end > p.n_chunks) c_end = p.n_chunks;

  const XT* __restrict__ X = static_cast<const XT*>(p.X);
  const double* __restrict__ Fhi = p.Fhi;
  const double* __restrict__ Flo = p.Flo;

  // ---------------- stage loaders ----------------
  auto load_x = [&](int64_t c, int stage) {
    XT* dst = xs + stage * G::kTile;
    const int64_t q0 = c * BQ;
    if constexpr (!KIND_M) {
      // tile [BM][BQ]: element (m, kk) at dst[m*pitch + kk]; lanes run along kk
      const int kk = tid % BQ;
      const uint32_t q = static_cast<uint32_t>(q0) + kk;
      const bool qvalid = q < p.Q;
      const uint32_t o = qvalid ? q / static_cast<uint32_t>(p.K) : 0u;
      const uint32_t k = qvalid ? q - o * static_cast<uint32_t>(p.K) : 0u;
      const int64_t base = static_cast<int64_t>(o) * p.s_o + k;
      const int rstep = nthreads / BQ;
      for (int m = tid / BQ; m < BM; m += rstep) {
        const int64_t gm = m0 + m;
        const bool valid = qvalid && gm < p.M;
        const XT* src = valid ? X + gm * p.s_m + base : X;
        cp_async_ca<sizeof(XT)>(dst + m * G::kPitchQ + kk, src, valid);
      }
    } else {
      // tile [BQ][BM]: element (qq, m) at dst[qq*BM + m]; contiguous along m
      constexpr int EPV = VEC / sizeof(XT);  // elements per vector
      constexpr int VPR = BM / EPV;          // vectors per row
      for (int v = tid; v < BQ * VPR; v += nthreads) {
        const int qq = v / VPR;
        const int m = (v % VPR) * EPV;
        const int64_t q = q0 + qq;
        const int64_t gm = m0 + m;
        if constexpr (VEC == 16) {
          const bool valid = q < p.Q && gm < p.M;  // M % EPV == 0 guaranteed by host
          const XT* src = valid ? X + q * p.s_m + gm : X;
          cp_async_cg16(dst + qq * BM + m, src, valid);
        } else {
          const bool valid = q < p.Q && gm < p.M;
          const XT* src = valid ? X + q * p.s_m + gm : X;
          cp_async_ca<sizeof(XT)>(dst + qq * BM + m, src, valid);
        }
      }
    }
  };

  // KR rows of chunk c: W[qq][r] = Fhi[hi(q)][r] * Flo[lo(q)][r] in fp64, rounded
  // once to the compute type.  One warp per q-row (indices advanced
  // incrementally, no per-element division), lanes along r (coalesced).
  auto form_w = [&](int64_t c, int buf) {
    XT* dst = ws + buf * BQ * R_pad;
    const int nwarps = nthreads >> 5;
    uint32_t q = static_cast<uint32_t>(c * BQ) + warp;
    uint32_t hi_i = q / p.lo_extent;
    uint32_t lo_i = q - hi_i * p.lo_extent;
    for (int qq = warp; qq < BQ; qq += nwarps) {
      const bool qv = q < p.Q;
      const double* fh = Fhi + static_cast<int64_t>(hi_i) * R;
      const double* fl = Flo + static_cast<int64_t>(lo_i) * R;
      for (int r = lane; r < R_pad; r += 32) {
        XT w = XT(0);
        if (qv && r < R) w = static_cast<XT>(fh[r] * fl[r]);
        dst[qq * R_pad + r] = w;
      }
      q += nwarps;
      lo_i += nwarps;
      while (lo_i >= p.lo_extent) {
        lo_i -= p.lo_extent;
        ++hi_i;
      }
    }
  };

  // ---------------- accumulators ----------------
  acc_t acc[TM][TR];
  float hi[kTwoLevel ? TM : 1][kTwoLevel ? TR : 1];
  float lo[kTwoLevel ? TM : 1][kTwoLevel ? TR : 1];
#pragma unroll
  for (int t = 0; t < TM; ++t)
#pragma unroll
    for (int j = 0; j < TR; ++j) acc[t][j] = acc_t(0);
  if constexpr (kTwoLevel) {
#pragma unroll
    for (int t = 0; t < TM; ++t)
#pragma unroll
      for (int j = 0; j < TR; ++j) {
        hi[t][j] = 0.f;
        lo[t][j] = 0.f;
      }
  }

  const bool active_r = r0 < R;  // warps entirely in the padding skip the math

  if (c_begin < c_end) {
    load_x(c_begin, 0);
    cp_async_commit();
    if (c_begin + 1 < c_end) load_x(c_begin + 1, 1);
    cp_async_commit();
    form_w(c_begin, 0);

    for (int64_t c = c_begin; c < c_end; ++c) {
      const int it = static_cast<int>(c - c_begin);
      cp_async_wait<1>();
      __syncthreads();
      if (c + 2 < c_end) load_x(c + 2, (it + 2) % STAGES);
      cp_async_commit();

      if (active_r) {
        const XT* xt = xs + (it % STAGES) * G::kTile;
        const XT* wt = ws + (it & 1) * BQ * R_pad + r0;
#pragma unroll 4
        for (int qq = 0; qq < BQ; ++qq) {
          XT xv[TM];
#pragma unroll
          for (int t = 0; t < TM; ++t) {
            const int m = lane + 32 * t;
            xv[t] = KIND_M ? xt[qq * BM + m] : xt[m * G::kPitchQ + qq];
          }
          XT wv[TR];
          if constexpr (sizeof(XT) == 4 && TR % 4 == 0) {
#pragma unroll
            for (int j = 0; j < TR; j += 4) {
              const float4 v = *reinterpret_cast<const float4*>(wt + qq * R_pad + j);
              wv[j] = v.x;
              wv[j + 1] = v.y;
              wv[j + 2] = v.z;
              wv[j + 3] = v.w;
            }
          } else if constexpr (sizeof(XT) == 8 && TR % 2 == 0) {
#pragma unroll
            for (int j = 0; j < TR; j += 2) {
              const double2 v = *reinterpret_cast<const double2*>(wt + qq * R_pad + j);
              wv[j] = v.x;
              wv[j + 1] = v.y;
            }
          } else {
#pragma unroll
            for (int j = 0; j < TR; ++j) wv[j] = wt[qq * R_pad + j];
          }
#pragma unroll
          for (int t = 0; t < TM; ++t)
#pragma unroll
            for (int j = 0; j < TR; ++j) acc[t][j] = fma(xv[t], wv[j], acc[t][j]);
        }
        if constexpr (kTwoLevel) {
#pragma unroll
          for (int t = 0; t < TM; ++t)
#pragma unroll
            for (int j = 0; j < TR; ++j) {
              fast_two_sum_acc(hi[t][j], lo[t][j], acc[t][j]);
              acc[t][j] = 0.f;
            }
        }
      }
      if (c + 1 < c_end) form_w(c + 1, (it + 1) & 1);
    }
    cp_async_wait<0>();
  }

  // ---------------- write this split's fp64 partial ----------------
  if (!active_r) return;
  double* out = p.ws + static_cast<int64_t>(split) * p.M * R;
#pragma unroll
  for (int t = 0; t < TM; ++t) {
    const int64_t gm = m0 + lane + 32 * t;
    if (gm >= p.M) continue;
#pragma unroll
    for (int j = 0; j < TR; ++j) {
      const int r = r0 + j;
      if (r >= R) continue;
      double v;
      if constexpr (kTwoLevel)
        v = static_cast<double>(hi[t][j]) + static_cast<double>(lo[t][j]);
      else
        v = static_cast<double>(acc[t][j]);
      out[gm * R + r] = v;
    }
  }
}

// Sum the split partials in a fixed order: out[m, r] = sum_s ws[s][m][r].
__global__ void mttkrp_reduce_kernel(const double* __restrict__ ws, int64_t splits, int64_t n,
                                     double* __restrict__ out, const int* stop_flag) {
  if (stop_flag && *stop_flag) return;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t k = 0; k < splits; ++k) s += ws[k * n + e];
    out[e] = s;
  }
}

template <typename XT, int TM, int TR, bool KIND_M, int VEC>
cudaError_t launch_variant(const MttkrpCCParams& p, const MttkrpCCLaunch& L, cudaStream_t stream) {
  auto kern = mttkrp_cc_kernel<XT, TM, TR, KIND_M, VEC>;
  cudaError_t err =
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L.smem_bytes);
  if (err != cudaSuccess) return err;
  kern<<<dim3(L.n_mtiles, L.splits), L.threads, L.smem_bytes, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace

// ---------------------------------------------------------------------------
// host side: geometry and dispatch
// ---------------------------------------------------------------------------

static int sm_count_cached() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

MttkrpCCLaunch mttkrp_cc_plan(int mode, int x_dtype, int64_t I, int64_t J, int64_t K, int R) {
  MttkrpCCLaunch L{};
  const bool f32 = x_dtype == NTF_F32;
  L.TM = f32 ? 4 : 2;
  L.TR = f32 ? (R > 64 ? 16 : 8) : (R > 32 ? 8 : 4);
  const int BM = 32 * L.TM;
  const int BQ = 32;
  L.R_pad = ((R + L.TR - 1) / L.TR) * L.TR;
  L.threads = (L.R_pad / L.TR) * 32;
  if (L.threads < 64) L.threads = 64;  // keep loaders busy; extra warps skip math
  const int64_t M = mode == 1 ? I : (mode == 2 ? J : K);
  const int64_t Q = mode == 3 ? I * J : (mode == 1 ? J * K : I * K);
  L.M = M;
  L.Q = Q;
  L.n_mtiles = static_cast<int>((M + BM - 1) / BM);
  L.n_chunks = (Q + BQ - 1) / BQ;
  const int esz = f32 ? 4 : 8;
  const int tile = BM * (BQ + 1) > BQ * BM ? BM * (BQ + 1) : BQ * BM;
  L.smem_bytes = 3 * tile * esz + 2 * BQ * L.R_pad * esz;
  // Occupancy-driven split count: fill every SM ~4 CTAs deep.
  int per_sm = static_cast<int>((227 * 1024) / (L.smem_bytes + 1024));
  if (per_sm < 1) per_sm = 1;
  if (per_sm > 4) per_sm = 4;
  const int64_t target = static_cast<int64_t>(sm_count_cached()) * per_sm * 2;
  int64_t splits = (target + L.n_mtiles - 1) / L.n_mtiles;
  if (splits < 1) splits = 1;
  if (splits > L.n_chunks) splits = L.n_chunks;
  L.chunks_per_split = (L.n_chunks + splits - 1) / splits;
  L.splits = static_cast<int>((L.n_chunks + L.chunks_per_split - 1) / L.chunks_per_split);
  L.vec16 = (mode == 3) && f32 && (K % 4 == 0) && (M % 4 == 0);
  return L;
}

size_t mttkrp_cc_workspace_bytes(const MttkrpCCLaunch& L, int R) {
  return static_cast<size_t>(L.splits) * L.M * R * sizeof(double);
}

cudaError_t mttkrp_cc_launch(int mode, int x_dtype, const void* X, int64_t I, int64_t J, int64_t K,
                             const double* A, const double* B, const double* C, int R,
                             const MttkrpCCLaunch& L, double* ws, const int* stop_flag,
                             cudaStream_t stream) {
  MttkrpCCParams p{};
  p.X = X;
  p.R = R;
  p.R_pad = L.R_pad;
  p.M = L.M;
  p.Q = L.Q;
  p.K = K;
  p.n_chunks = L.n_chunks;
  p.chunks_per_split = L.chunks_per_split;
  p.ws = ws;
  p.stop_flag = stop_flag;
  if (mode == 1) {
    p.s_m = J * K;
    p.s_o = K;
    p.Fhi = B;
    p.Flo = C;
    p.lo_extent = static_cast<uint32_t>(K);
  } else if (mode == 2) {
    p.s_m = K;
    p.s_o = J * K;
    p.Fhi = A;
    p.Flo = C;
    p.lo_extent = static_cast<uint32_t>(K);
  } else {
    p.s_m = K;  // row pitch of the [P][K] view
    p.s_o = 0;
    p.Fhi = A;
    p.Flo = B;
    p.lo_extent = static_cast<uint32_t>(J);
  }
  const bool f32 = x_dtype == NTF_F32;
  if (f32) {
    if (L.TR == 16) {
      if (mode == 3)
        return L.vec16 ? launch_variant<float, 4, 16, true, 16>(p, L, stream)
                       : launch_variant<float, 4, 16, true, 4>(p, L, stream);
      return launch_variant<float, 4, 16, false, 4>(p, L, stream);
    }
    if (mode == 3)
      return L.vec16 ? launch_variant<float, 4, 8, true, 16>(p, L, stream)
                     : launch_variant<float, 4, 8, true, 4>(p, L, stream);
    return launch_variant<float, 4, 8, false, 4>(p, L, stream);
  }
  if (L.TR == 8) {
    if (mode == 3) return launch_variant<double, 2, 8, true, 8>(p, L, stream);
    return launch_variant<double, 2, 8, false, 8>(p, L, stream);
  }
  if (mode == 3) return launch_variant<double, 2, 4, true, 8>(p, L, stream);
  return launch_variant<double, 2, 4, false, 8>(p, L, stream);
}

cudaError_t mttkrp_reduce_launch(const double* ws, int splits, int64_t M, int R, double* out,
                                 const int* stop_flag, cudaStream_t stream) {
  const int64_t n = M * R;
  int blocks = static_cast<int>((n + 255) / 256);
  if (blocks > 4 * sm_count_cached()) blocks = 4 * sm_count_cached();
  if (blocks < 1) blocks = 1;
  mttkrp_reduce_kernel<<<blocks, 256, 0, stream>>>(ws, splits, n, out, stop_flag);
  return cudaGetLastError();
}

}  // namespace ntf
