// Dense MTTKRP in fp64 arithmetic (sm_100a, fp64 tensor pipe), all three modes,
// fp32 or fp64 tensor: the "cuda_core" engine (no tcgen05, no fp16 slicing).
//
// Replaces tensors.mttkrp_factors dense branch (reference tensors.py:254-262):
//   M_n = X_(n) @ khatri_rao(companions, highest mode first)
// without the cached unfolding copy (tensors.py:63-71) and without the
// materialised Khatri-Rao matrix (tensors.py:203-220).  Every mode streams the
// native row-major X[i][j][k] exactly once.
//
// GEMM view used for all modes:  out[m, r] = sum_q X(m, q) * W(q, r),
//   W(q, r) = F_hi[q / L, r] * F_lo[q % L, r]   (KR row formed on the fly)
//   KIND_Q (modes 1, 2):  q = o*K + k, k the contiguous tensor index, L = K
//       mode 1: m = i, o = j  (X(m,q) = X[i*JK + q]),        W = B[j] * C[k]
//       mode 2: m = j, o = i  (X(m,q) = X[i*JK + j*K + k]),  W = A[i] * C[k]
//   KIND_M (mode 3):       q = p = i*J + j, m = k contiguous, L = J, W = A[i] * B[j]
//
// Tiling.  A CTA owns BM = 32*TM output rows and all R columns (ranks above
// 128: one grid z-slice per 128-column chunk).  The reduction range is cut
// into chunks of BQ = 32 q-values; each chunk's stage (the X tile + the fp64
// F_hi / F_lo rows its Khatri-Rao rows need) is streamed by 16-byte cp.async
// through a ring of up to five stages by four producer warps.  The math runs on the fp64
// tensor pipe: DMMA warp w owns rows [16w, 16w + 16) and all columns as
// m8n8k4 fragments (A = X, converted to fp64 when the tensor is fp32; B = the
// KR row, F_lo[l, n] * F_hi[h, n] rounded once as the reference's khatri_rao,
// formed in registers as the fragment is loaded; fp64 accumulators).  Tile
// pitches are chosen so every fragment load is bank-conflict free.
//
// Precision: fp64 arithmetic throughout for fp32 and fp64 tensors alike (the
// fp32 tensor values are exact in fp64), so this engine reproduces the
// reference's arithmetic up to summation order whatever the tensor's type.
//
// Split-K.  CTAs of one m-tile stream contiguous chunk ranges.  The CTAs of a
// thread-block cluster (CS splits) reduce their fp64 partial tiles through
// distributed shared memory in fixed rank order, so only S/CS partials reach
// HBM; the consumer sums those in fixed order.  No float atomics: results are
// bitwise run-to-run deterministic.
#include <cooperative_groups.h>

#include <cstdlib>
#include <type_traits>

#include "mttkrp_cc.cuh"

namespace cg = cooperative_groups;

namespace ntf {

namespace {

constexpr int kBQ = 32;
constexpr int kMaxStages = 5;
constexpr int kClusterSplits = 8;
constexpr int kColChunk = 128;  // output columns per CTA (16 8-column blocks)

template <typename XT, int TM, bool KIND_M, bool VEC>
struct Geom {
  static constexpr int BM = 32 * TM;
  static constexpr int VW = 16 / sizeof(XT);  // elements per 16 B
  // Pitches that make the m8n8k4 A fragments (KIND_Q: 8 rows x 4 consecutive
  // q; KIND_M: 4 q-rows x 8 consecutive m) bank-conflict free: 4 (mod 16)
  // doubles, or 4 resp. 8 (mod 32) floats; all multiples of 16 bytes
  static constexpr int kPitchQ = kBQ + 4;
  static constexpr int kPitchM = BM + (sizeof(XT) == 8 ? 4 : 8);
  static constexpr int kTileElems = KIND_M ? kBQ * kPitchM : BM * kPitchQ;
};

// D (8x8, fp64) += A (8x4, row) * B (4x8, col): lane (g = lane / 4, t = lane % 4)
// holds A[g][t], B[t][g] and D[g][2t], D[g][2t + 1].  Full fp64 rate on sm_100a
// (37 TFLOP/s measured, tools/ubench/f64_rate.cu) with one operand fetch per
// 8 multiply-adds of a lane.
__device__ __forceinline__ void dmma_m8n8k4(double (&d)[2], double a, double b) {
#if defined(NTF_DIAG) && defined(NTF_CC_SKIP_DMMA)  // diagnostic builds only: time the data path alone
  d[0] += a;
  d[1] += b;
  return;
#endif
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// f(integral_constant<N>) for the N in [NMIN, NMAX] equal to nb (NMAX otherwise)
template <int NMAX, int NMIN, typename F>
__device__ __forceinline__ void dispatch_nb(int nb, F&& f) {
  if constexpr (NMAX <= NMIN || NMAX <= 1) {
    f(std::integral_constant<int, NMAX>{});
  } else {
    if (nb >= NMAX) f(std::integral_constant<int, NMAX>{});
    else dispatch_nb<NMAX - 1, NMIN>(nb, f);
  }
}

// a * b rounded to nearest, pinned in program order between the DMMAs
__device__ __forceinline__ double dmul_rn_pinned(double a, double b) {
#if defined(NTF_DIAG) && defined(NTF_CC_SKIP_DMUL)  // diagnostic builds only
  return a;
#endif
  double r;
  asm volatile("mul.rn.f64 %0, %1, %2;\n" : "=d"(r) : "d"(a), "d"(b));
  return r;
}

constexpr int kProdWarps = 4;  // producer warps (stage loads) beside the DMMA warps

__device__ __forceinline__ void named_bar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_bar_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}

template <typename XT, int TM, int TR, bool KIND_M, bool VEC>
__global__ void __launch_bounds__((32 * TM / 16 + kProdWarps) * 32, 1) mttkrp_cc_kernel(MttkrpCCParams p) {
  using G = Geom<XT, TM, KIND_M, VEC>;
  constexpr int BM = G::BM;
  constexpr int VW = G::VW;
  // TR: the 8-column blocks a DMMA warp can hold (4, 8 or 16)

  if (p.stop_flag && *p.stop_flag) return;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  // stage s: [X tile | hi rows (max_hi x R2 doubles) | lo rows (BQ x R2)]
  // Column chunk blockIdx.z: columns [c0, c0 + R) of the R_full-column
  // factors and output (ranks above kColChunk; one chunk otherwise).
  const int R_full = p.R;
  const int c0 = static_cast<int>(blockIdx.z) * kColChunk;
  const int R = R_full - c0 < kColChunk ? R_full - c0 : kColChunk;
  const int R_pad = p.R_pad;
  // pitch of the staged factor rows: 4 or 12 (mod 16) doubles (see the plan)
  const int R2 = R_pad;
  unsigned char* stage_base = smem_raw;
  const int stage_bytes = p.stage_bytes;
  auto x_tile = [&](int s) { return reinterpret_cast<XT*>(stage_base + s * stage_bytes); };
  auto hi_rows = [&](int s) {
    return reinterpret_cast<double*>(stage_base + s * stage_bytes + G::kTileElems * sizeof(XT));
  };
  auto lo_rows = [&](int s) { return hi_rows(s) + p.max_hi * R2; };

  const int tid = threadIdx.x;
  const int nthreads = blockDim.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  // warps [0, BM / 16) issue the DMMAs, the kProdWarps warps after them run
  // the stage loads (ltid / lthreads: the loaders' thread numbering)
  constexpr int kMathWarps = BM / 16;
  const int ltid = tid - 32 * kMathWarps;
  constexpr int lthreads = 32 * kProdWarps;

  const int64_t m0 = static_cast<int64_t>(blockIdx.x) * BM;
  const int split = blockIdx.y;
  const int64_t c_begin = static_cast<int64_t>(split) * p.chunks_per_split;
  int64_t c_end = c_begin + p.chunks_per_split;
  if (c_end > p.n_chunks) c_end = p.n_chunks;

  const XT* __restrict__ X = static_cast<const XT*>(p.X);
  const uint32_t L = p.lo_extent;

  // ---------------- stage loader: X tile + factor rows of chunk c ----------
  auto load_stage = [&](int64_t c, int s) {
    const uint32_t q0 = static_cast<uint32_t>(c * kBQ);
    XT* xt = x_tile(s);
    if constexpr (!KIND_M) {
      if constexpr (VEC) {
        constexpr int VPR = kBQ / VW;  // vectors per row
        const int vq = ltid % VPR;
        const uint32_t q = q0 + vq * VW;
        const bool qv = q < p.Q;
        const uint32_t o = qv ? q / static_cast<uint32_t>(p.K) : 0u;
        const uint32_t k = qv ? q - o * static_cast<uint32_t>(p.K) : 0u;
        const int64_t base = static_cast<int64_t>(o) * p.s_o + k;
        for (int m = ltid / VPR; m < BM; m += lthreads / VPR) {
          const int64_t gm = m0 + m;
          const bool valid = qv && gm < p.M;
          cp_async_cg16(xt + m * G::kPitchQ + vq * VW, valid ? X + gm * p.s_m + base : X, valid);
        }
      } else {
        const int kk = ltid % kBQ;
        const uint32_t q = q0 + kk;
        const bool qv = q < p.Q;
        const uint32_t o = qv ? q / static_cast<uint32_t>(p.K) : 0u;
        const uint32_t k = qv ? q - o * static_cast<uint32_t>(p.K) : 0u;
        const int64_t base = static_cast<int64_t>(o) * p.s_o + k;
        for (int m = ltid / kBQ; m < BM; m += lthreads / kBQ) {
          const int64_t gm = m0 + m;
          const bool valid = qv && gm < p.M;
          cp_async_ca<sizeof(XT)>(xt + m * G::kPitchQ + kk, valid ? X + gm * p.s_m + base : X,
                                  valid);
        }
      }
    } else {
      if constexpr (VEC) {
        constexpr int VPR = BM / VW;
        const int vm = ltid % VPR;
        const int64_t gm = m0 + vm * VW;
        for (int qq = ltid / VPR; qq < kBQ; qq += lthreads / VPR) {
          const uint32_t q = q0 + qq;
          const bool valid = q < p.Q && gm < p.M;  // host guarantees M % VW == 0
          cp_async_cg16(xt + qq * G::kPitchM + vm * VW,
                        valid ? X + static_cast<int64_t>(q) * p.s_m + gm : X, valid);
        }
      } else {
        for (int e = ltid; e < kBQ * BM; e += lthreads) {
          const int qq = e / BM, m = e - (e / BM) * BM;
          const uint32_t q = q0 + qq;
          const int64_t gm = m0 + m;
          const bool valid = q < p.Q && gm < p.M;
          cp_async_ca<sizeof(XT)>(xt + qq * G::kPitchM + m,
                                  valid ? X + static_cast<int64_t>(q) * p.s_m + gm : X, valid);
        }
      }
    }
    // factor rows: hi rows h0 .. h0+max_hi-1, lo rows lo(qq) for qq < BQ
    const uint32_t h0 = q0 / L;
    const uint32_t l0 = q0 - h0 * L;
    double* hs = hi_rows(s);
    double* ls = lo_rows(s);
    const double* Fhi = p.Fhi + c0;
    const double* Flo = p.Flo + c0;
    if (((R | R_full) & 1) == 0) {
      const int vpr = R >> 1;  // 16-byte vectors per row
      const int nh = p.max_hi * vpr;
      // e / vpr as a multiply-high: exact for e * (vpr - 1) < 2^32
      const uint32_t vmagic = 0xFFFFFFFFu / static_cast<uint32_t>(vpr) + 1u;
      for (int e = ltid; e < nh + kBQ * vpr; e += lthreads) {
        if (e < nh) {
          const int row = vpr == 1 ? e : static_cast<int>(__umulhi(static_cast<uint32_t>(e), vmagic)), v = e - row * vpr;
          const uint32_t h = h0 + row;
          const bool valid = h < p.hi_extent;
          cp_async_cg16(hs + row * R2 + 2 * v, valid ? Fhi + static_cast<int64_t>(h) * R_full + 2 * v : Fhi,
                        valid);
        } else {
          const int e2 = e - nh;
          const int qq = vpr == 1 ? e2 : static_cast<int>(__umulhi(static_cast<uint32_t>(e2), vmagic)), v = e2 - qq * vpr;
          uint32_t lo = l0 + qq;
          lo = L >= kBQ ? (lo >= L ? lo - L : lo) : lo % L;
          cp_async_cg16(ls + qq * R2 + 2 * v, Flo + static_cast<int64_t>(lo) * R_full + 2 * v, true);
        }
      }
    } else {
      const int nh = p.max_hi * R;
      for (int e = ltid; e < nh + kBQ * R; e += lthreads) {
        if (e < nh) {
          const int row = e / R, r = e - (e / R) * R;
          const uint32_t h = h0 + row;
          const bool valid = h < p.hi_extent;
          cp_async_ca<8>(hs + row * R2 + r, valid ? Fhi + static_cast<int64_t>(h) * R_full + r : Fhi,
                         valid);
        } else {
          const int e2 = e - nh;
          const int qq = e2 / R, r = e2 - (e2 / R) * R;
          const uint32_t lo = (l0 + qq) % L;
          cp_async_ca<8>(ls + qq * R2 + r, Flo + static_cast<int64_t>(lo) * R_full + r, true);
        }
      }
    }
  };

  // ---------------- accumulators ----------------
  // DMMA warp w owns rows [16w, 16w + 16) and all columns: two 8-row blocks x
  // TR 8-column blocks of m8n8k4 accumulator fragments
  double dacc[2][TR][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < TR; ++j) dacc[i][j][0] = dacc[i][j][1] = 0.0;
  const int nb8 = (R + 7) >> 3;  // 8-column blocks in use

  {
    // Warp-specialised pipeline: the producers keep the loads two chunks
    // ahead (three stages); the DMMA warps read the X fragments and the F_lo
    // rows straight from the stage and form each KR fragment as they load it
    // (one DMUL per two DMMAs: F_lo[l, n] * F_hi[h, n], rounded once, as the
    // reference's khatri_rao), so no warp ever waits on address arithmetic.
    // Named barriers 1..5: stage landed, 8..12: stage consumed, 15: producers.
    constexpr int kAll = (kMathWarps + kProdWarps) * 32;
    const int n_it = static_cast<int>(c_end - c_begin);
    const int ns = p.n_stages;  // 2..5: as many stages as fit (latency of the loads, see the plan)
    if (n_it > 0 && warp >= kMathWarps) {
      load_stage(c_begin, 0);
      cp_async_commit();
      for (int k = 1; k < ns - 1; ++k) {  // prologue: ns - 1 chunks in flight
        if (k < n_it) load_stage(c_begin + k, k);
        cp_async_commit();
      }
      for (int it = 0; it < n_it; ++it) {
        // this thread's copies of chunk it (ns - 2 younger groups may be pending)
        if (ns >= 5) cp_async_wait<3>();
        else if (ns == 4) cp_async_wait<2>();
        else if (ns == 3) cp_async_wait<1>();
        else cp_async_wait<0>();
        named_bar_sync(15, 32 * kProdWarps);     // ... and every producer's
        named_bar_arrive(1 + it % ns, kAll);
        if (it >= 1) named_bar_sync(8 + (it - 1) % ns, kAll);  // chunk it - 1 consumed: its stage is free
#if !(defined(NTF_DIAG) && defined(NTF_CC_SKIP_LOAD))  // diagnostic builds only: time the math alone
        if (it + ns - 1 < n_it) load_stage(c_begin + it + ns - 1, (it + ns - 1) % ns);
#endif
        cp_async_commit();
      }
      named_bar_sync(8 + (n_it - 1) % ns, kAll);
      cp_async_wait<0>();
    } else if (n_it > 0) {
      const int g = lane >> 2, t4 = lane & 3;
      for (int it = 0; it < n_it; ++it) {
        const int st = it % ns;
        const uint32_t q0 = static_cast<uint32_t>((c_begin + it) * kBQ);
        const uint32_t l0 = q0 - (q0 / L) * L;
        named_bar_sync(1 + st, kAll);
        const XT* xt = x_tile(st);
        const XT* xa = KIND_M ? xt + t4 * G::kPitchM + warp * 16 + g
                              : xt + (warp * 16 + g) * G::kPitchQ + t4;
        const double* lb = lo_rows(st) + t4 * R2 + g;  // F_lo[l0 + k + t4][8 j + g]
        const double* hb = hi_rows(st) + g;            // F_hi[h0 + row][8 j + g]
        // fragments of K step k + 1 are fetched before the DMMAs of step k issue
        // NB: 8-column blocks issued (exactly nb8 on the common path: a
        // predicated-off DMMA still occupies the pipe; 33..64 columns all
        // cost the same with a fixed TR = 8)
        auto run_chunk = [&](auto straddle, auto nbtag) {
          constexpr int NB = decltype(nbtag)::value;
          constexpr bool kStraddle = decltype(straddle)::value;  // some q row belongs to a later F_hi row
          auto hrow = [&](int k4) {
            const uint32_t lsum = l0 + k4 + t4;
            const int hoff = L >= kBQ ? (lsum >= L ? 1 : 0) : static_cast<int>(lsum / L);
            return hb + hoff * R2;
          };
          // K step k: [shared loads of step k + 1] [DMMAs of the first row
          // block] [KR products of step k + 1] [DMMAs of the second row block]:
          // every multiply finds its operands loaded and every DMMA its KR
          // value computed half a step earlier (the DMULs share the fp64 pipe
          // with the DMMAs and issue in order)
          double hv[NB];
          if constexpr (!kStraddle) {
#pragma unroll
            for (int j = 0; j < NB; ++j) hv[j] = hb[8 * j];
          } else {
            const double* hr = hrow(0);
#pragma unroll
            for (int j = 0; j < NB; ++j) hv[j] = j < nb8 ? hr[8 * j] : 0.0;
          }
          double a0 = static_cast<double>(xa[0]);
          double a1 = static_cast<double>(KIND_M ? xa[8] : xa[8 * G::kPitchQ]);
          double w[NB];
#pragma unroll
          for (int j = 0; j < NB; ++j) w[j] = dmul_rn_pinned((!kStraddle || j < nb8) ? lb[8 * j] : 0.0, hv[j]);
#pragma unroll
          for (int k4 = 0; k4 < kBQ; k4 += 4) {
            const bool more = k4 + 4 < kBQ;
            double a0n = 0.0, a1n = 0.0, wn[NB];
            if (more) {
              a0n = static_cast<double>(KIND_M ? xa[(k4 + 4) * G::kPitchM] : xa[k4 + 4]);
              a1n = static_cast<double>(KIND_M ? xa[(k4 + 4) * G::kPitchM + 8] : xa[8 * G::kPitchQ + k4 + 4]);
#pragma unroll
              for (int j = 0; j < NB; ++j)
                wn[j] = (!kStraddle || j < nb8) ? lb[(k4 + 4) * R2 + 8 * j] : 0.0;
              if constexpr (kStraddle) {
                const double* hr = hrow(k4 + 4);
#pragma unroll
                for (int j = 0; j < NB; ++j) hv[j] = j < nb8 ? hr[8 * j] : 0.0;
              }
            }
#pragma unroll
            for (int j = 0; j < NB; ++j)
              if (!kStraddle || j < nb8) dmma_m8n8k4(dacc[0][j], a0, w[j]);
            if (more) {
#pragma unroll
              for (int j = 0; j < NB; ++j) wn[j] = dmul_rn_pinned(wn[j], hv[j]);
            }
#pragma unroll
            for (int j = 0; j < NB; ++j)
              if (!kStraddle || j < nb8) dmma_m8n8k4(dacc[1][j], a1, w[j]);
            if (more) {
              a0 = a0n;
              a1 = a1n;
#pragma unroll
              for (int j = 0; j < NB; ++j) w[j] = wn[j];
            }
          }
        };
        if (l0 + kBQ > L) run_chunk(std::true_type{}, std::integral_constant<int, TR>{});
        else dispatch_nb<TR, TR / 2 + 1>(nb8, [&](auto nbtag) { run_chunk(std::false_type{}, nbtag); });
        named_bar_arrive(8 + st, kAll);
      }
    }
  }

  // ------------- cluster (DSMEM) reduction of the split partials -------------
  cg::cluster_group cluster = cg::this_cluster();
  __syncthreads();
  double* part = reinterpret_cast<double*>(smem_raw);  // [BM][R], reuses the stage ring
  {
    const int g = lane >> 2, t4 = lane & 3;
#pragma unroll
    for (int i = 0; i < 2 && warp < kMathWarps; ++i) {
      const int m = warp * 16 + 8 * i + g;
#pragma unroll
      for (int j = 0; j < TR; ++j) {
        const int r = 8 * j + 2 * t4;
        if (r < R) part[m * R + r] = dacc[i][j][0];
        if (r + 1 < R) part[m * R + r + 1] = dacc[i][j][1];
      }
    }
  }
  cluster.sync();
  const int cs = static_cast<int>(cluster.num_blocks());
  const int crank = static_cast<int>(cluster.block_rank());
  const int rows_per = BM / cs;
  const int64_t group = split / cs;
  double* out = p.ws + group * p.M * R_full + c0;
  for (int e = tid; e < rows_per * R; e += nthreads) {
    const int lm = crank * rows_per + e / R;
    const int r = e - (e / R) * R;
    double s = 0.0;
    for (int b = 0; b < cs; ++b) {
      const double* rp = cluster.map_shared_rank(part, b);
      s += rp[lm * R + r];
    }
    const int64_t gm = m0 + lm;
    if (gm < p.M) out[gm * R_full + r] = s;
  }
  cluster.sync();
}

// Sum the split-group partials in a fixed order: out[m, r] = sum_g ws[g][m][r].
__global__ void mttkrp_reduce_kernel(const double* __restrict__ ws, int64_t groups, int64_t n,
                                     double* __restrict__ out, const int* stop_flag,
                                     int64_t tail_e0, int64_t groups_tail) {
  if (stop_flag && *stop_flag) return;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    const int64_t ng = e >= tail_e0 ? groups_tail : groups;
    for (int64_t k = 0; k < ng; ++k) s += ws[k * n + e];
    out[e] = s;
  }
}

enum VariantOp { kLaunch = 0, kPrepare = 1, kQueryClusters = 2 };
thread_local int g_active_clusters = 0;

template <typename XT, int TM, int TR, bool KIND_M, bool VEC>
cudaError_t launch_variant(const MttkrpCCParams& p, const MttkrpCCLaunch& L, cudaStream_t stream,
                           int op) {
  auto kern = mttkrp_cc_kernel<XT, TM, TR, KIND_M, VEC>;
  if (op != kLaunch) {
    cudaError_t e = allow_dyn_smem(reinterpret_cast<const void*>(kern), L.smem_bytes);
    if (e != cudaSuccess || op == kPrepare) return e;
    cudaLaunchConfig_t q{};
    q.gridDim = dim3(1, L.cluster, 1);
    q.blockDim = dim3(L.threads, 1, 1);
    q.dynamicSmemBytes = L.smem_bytes;
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = 1;
    a[0].val.clusterDim.y = L.cluster;
    a[0].val.clusterDim.z = 1;
    q.attrs = a;
    q.numAttrs = 1;
    return cudaOccupancyMaxActiveClusters(&g_active_clusters, kern, &q);
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(L.n_mtiles, L.splits, L.col_chunks);
  cfg.blockDim = dim3(L.threads, 1, 1);
  cfg.dynamicSmemBytes = L.smem_bytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = L.cluster;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, p);
}

template <typename XT, int TM, int TR>
cudaError_t dispatch_kind(int mode, const MttkrpCCParams& p, const MttkrpCCLaunch& L,
                          cudaStream_t stream, int prep) {
  if (mode == 3)
    return L.vec ? launch_variant<XT, TM, TR, true, true>(p, L, stream, prep)
                 : launch_variant<XT, TM, TR, true, false>(p, L, stream, prep);
  return L.vec ? launch_variant<XT, TM, TR, false, true>(p, L, stream, prep)
               : launch_variant<XT, TM, TR, false, false>(p, L, stream, prep);
}

cudaError_t dispatch(int mode, int x_dtype, const MttkrpCCParams& p, const MttkrpCCLaunch& L,
                     cudaStream_t stream, int prep) {
  // TR = 8-column blocks per warp; BM = 32 TM rows on BM / 16 DMMA warps
  if (x_dtype == NTF_F32) {
    if (L.TR == 16) return dispatch_kind<float, 2, 16>(mode, p, L, stream, prep);
    if (L.TR == 8) return dispatch_kind<float, 4, 8>(mode, p, L, stream, prep);
    return dispatch_kind<float, 4, 4>(mode, p, L, stream, prep);
  }
  if (L.TR == 16) return dispatch_kind<double, 2, 16>(mode, p, L, stream, prep);
  if (L.TR == 8) return dispatch_kind<double, 4, 8>(mode, p, L, stream, prep);
  return dispatch_kind<double, 4, 4>(mode, p, L, stream, prep);
}

int sm_count_cached() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

int smem_optin_cached() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&n, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess || n <= 0)
      n = 232448;  // sm_100a (no device: geometry queries on a CPU-only host)
    cudaGetLastError();
  }
  return n;
}

void fill_params(MttkrpCCParams& p, int mode, const void* X, int64_t I, int64_t J, int64_t K,
                 const double* A, const double* B, const double* C, int R, const MttkrpCCLaunch& L,
                 double* ws, const int* stop_flag) {
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
  p.stage_bytes = L.stage_bytes;
  p.n_stages = L.stages;
  p.max_hi = L.max_hi;
  if (mode == 1) {
    p.s_m = J * K;
    p.s_o = K;
    p.Fhi = B;
    p.Flo = C;
    p.lo_extent = static_cast<uint32_t>(K);
    p.hi_extent = static_cast<uint32_t>(J);
  } else if (mode == 2) {
    p.s_m = K;
    p.s_o = J * K;
    p.Fhi = A;
    p.Flo = C;
    p.lo_extent = static_cast<uint32_t>(K);
    p.hi_extent = static_cast<uint32_t>(I);
  } else {
    p.s_m = K;  // row pitch of the [P][K] view
    p.s_o = 0;
    p.Fhi = A;
    p.Flo = B;
    p.lo_extent = static_cast<uint32_t>(J);
    p.hi_extent = static_cast<uint32_t>(I);
  }
}

}  // namespace

// ---------------------------------------------------------------------------
// host side: geometry and dispatch
// ---------------------------------------------------------------------------
MttkrpCCLaunch mttkrp_cc_plan(int mode, int x_dtype, int64_t I, int64_t J, int64_t K, int R_full) {
  MttkrpCCLaunch L{};
  // ranks above kColChunk: one grid z-slice per 128-column chunk (each
  // streams X again); the geometry below is that of one chunk
  L.col_chunks = (R_full + kColChunk - 1) / kColChunk;
  const int R = R_full < kColChunk ? R_full : kColChunk;
  const bool f32 = x_dtype == NTF_F32;
  const int esz = f32 ? 4 : 8;
  const int VW = 16 / esz;
  // Each DMMA warp holds 16 rows x all columns (TR 8-column blocks); the
  // staged factor rows' pitch is 4 or 12 (mod 16) doubles (conflict-free B fragments)
  L.TR = R > 64 ? 16 : (R > 32 ? 8 : 4);
  L.TM = R > 64 ? 2 : 4;  // 64 rows above 64 columns (registers, shared memory)
  L.R_pad = (R + 7) & ~7;
  while (L.R_pad % 16 != 4 && L.R_pad % 16 != 12) ++L.R_pad;
  L.threads = (32 * L.TM / 16 + kProdWarps) * 32;  // DMMA warps + producers
  const int BM = 32 * L.TM;
  const int64_t M = mode == 1 ? I : (mode == 2 ? J : K);
  const int64_t Q = mode == 3 ? I * J : (mode == 1 ? J * K : I * K);
  const int64_t lo_ext = mode == 3 ? J : K;
  L.M = M;
  L.Q = Q;
  L.n_mtiles = static_cast<int>((M + BM - 1) / BM);
  L.n_chunks = (Q + kBQ - 1) / kBQ;
  // 16-byte cp.async needs whole vectors that never straddle a row/o boundary
  L.vec = (K % VW == 0) && (mode != 3 || M % VW == 0);
  const int tile = (mode == 3 ? kBQ * (BM + (f32 ? 8 : 4)) : BM * (kBQ + 4)) * esz;  // Geom::kPitchM / kPitchQ
  L.max_hi = static_cast<int>(std::min<int64_t>(kBQ, (kBQ - 1) / lo_ext + 2));
  int fac = (L.max_hi + kBQ) * L.R_pad * 8;  // staged factor rows
  L.stage_bytes = ((tile + fac) + 15) & ~15;
  // as many stages as fit, up to kMaxStages (the loads of ns - 1 chunks are in flight)
  L.stages = std::min(kMaxStages, std::max(2, smem_optin_cached() / L.stage_bytes));
#if defined(NTF_DIAG)
  if (const char* e = getenv("NTF_CC_STAGES")) L.stages = std::min(L.stages, std::max(2, atoi(e)));
#endif
  L.smem_bytes = L.stages * L.stage_bytes;
  const int part_bytes = BM * R * 8;  // cluster-reduction tile reuses the stage ring
  if (part_bytes > L.smem_bytes) L.smem_bytes = part_bytes;
  // One wave: as many clusters as can be co-resident (whole clusters per GPC),
  // spread over the m-tiles; splits are whole clusters.  The cluster size
  // (8, 4, 2 or 1 splits reduced through DSMEM) is the largest that keeps the
  // most CTAs resident: 8-CTA clusters leave SMs idle when the co-resident
  // cluster count is not a multiple of the tile count (1000 rows in 8 tiles
  // of 128: 15 clusters of 8 give 64 CTAs, 72 pairs give 144).
  const int64_t max_chunks = L.n_chunks;
  int64_t splits = 1;
  int best_cluster = kClusterSplits;
  int64_t best_ctas = 0;
  for (int cl = kClusterSplits; cl >= 1; cl >>= 1) {
    L.cluster = cl;
    int active = 0;
    {
      MttkrpCCParams p{};
      if (dispatch(mode, x_dtype, p, L, nullptr, kQueryClusters) == cudaSuccess)
        active = g_active_clusters;
      cudaGetLastError();
    }
    if (active <= 0) active = sm_count_cached() / cl;
    int64_t per_tile = active / L.n_mtiles;
    if (per_tile < 1) per_tile = 1;
    int64_t sp = per_tile * cl;
    const int64_t max_splits = ((max_chunks + cl - 1) / cl) * cl;
    if (sp > max_splits) sp = max_splits;
    const int64_t ctas = sp * L.n_mtiles;
    // a smaller cluster must win by more than 10% (its extra partials cost HBM traffic)
    if (best_ctas == 0 || ctas * 10 > best_ctas * 11) {
      best_ctas = ctas;
      splits = sp;
      best_cluster = cl;
    }
  }
  L.cluster = best_cluster;
  L.chunks_per_split = (L.n_chunks + splits - 1) / splits;
  L.splits = static_cast<int>(splits);
  L.groups = L.splits / L.cluster;
  return L;
}

size_t mttkrp_cc_workspace_bytes(const MttkrpCCLaunch& L, int R) {
  return static_cast<size_t>(L.groups) * L.M * R * sizeof(double);
}

cudaError_t mttkrp_cc_prepare(int mode, int x_dtype, const MttkrpCCLaunch& L) {
  MttkrpCCParams p{};
  return dispatch(mode, x_dtype, p, L, nullptr, kPrepare);
}

cudaError_t mttkrp_cc_launch(int mode, int x_dtype, const void* X, int64_t I, int64_t J, int64_t K,
                             const double* A, const double* B, const double* C, int R,
                             const MttkrpCCLaunch& L, double* ws, const int* stop_flag,
                             cudaStream_t stream) {
  MttkrpCCParams p{};
  fill_params(p, mode, X, I, J, K, A, B, C, R, L, ws, stop_flag);
  return dispatch(mode, x_dtype, p, L, stream, kLaunch);
}

cudaError_t mttkrp_reduce_launch(const double* ws, int groups, int64_t M, int R, double* out,
                                 const int* stop_flag, cudaStream_t stream, int64_t tail_row0,
                                 int groups_tail) {
  const int64_t n = M * R;
  int blocks = static_cast<int>((n + 255) / 256);
  if (blocks > 4 * sm_count_cached()) blocks = 4 * sm_count_cached();
  if (blocks < 1) blocks = 1;
  const int64_t tail_e0 = tail_row0 >= M ? n : tail_row0 * R;
  mttkrp_reduce_kernel<<<blocks, 256, 0, stream>>>(ws, groups, n, out, stop_flag, tail_e0,
                                                    groups_tail);
  return cudaGetLastError();
}

}  // namespace ntf
