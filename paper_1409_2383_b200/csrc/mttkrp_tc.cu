// Dense MTTKRP on the 5th-generation tensor cores (tcgen05, sm_100a) for fp32
// tensors.  Same contraction as mttkrp_cc.cu (reference tensors.py:254-262):
//   out[m, n] = sum_q X(m, q) W(q, n),  W(q, n) = F_hi[o, n] * F_lo[l, n]
//
// Numerics: exact fixed-point slicing on kind::f16 MMAs.
//   X  = xs * (S0 + S1)          S0 integers |S0| <= 2^11, S1 in 2^-11 units,
//                                xs = 2^(e-11) global (computed once per tensor)
//   W  = ws(n) * (T0 + T1 + T2)  T0 integers |T0| <= 2^7, T1 in 2^-7 and T2 in
//                                2^-14 units, ws(n) = 2^(f(n)-7) per column
// All slices are exact fp16 values.  Per 64-wide q chunk the tensor core forms
//   ACC0 = sum S0*T0                          (integers < 2^24: EXACT in fp32)
//   ACC1 = sum S0*T1 + S1*T0 + S0*T2 + S1*T1  (a 2^-7-scaled correction)
// so the dominant term carries no accumulation rounding at all (whatever the
// tensor core's rounding mode), and the correction's rounding is ~2^-29 of the
// result.  The epilogue folds ACC0 into a double-float accumulator (Fast2Sum)
// and ACC1 into its low word; dropped terms (S1*T2 ~ 2^-25, slice residues
// ~2^-23 of the column/tensor maxima) are i.i.d. per element, never a
// structured rounding of the factors (SURVEY 8(d) precision findings).
//
// Chunking.  All modes view X as 3-D (K, J, I) and walk chunks (o, l0): the
// reduction index q = (o, l) with l in [l0, l0+64) along one tensor axis:
//   mode 1: m = i, o = j, l = k   W = B[j] * C[k]   A tile K-major
//   mode 2: m = j, o = i, l = k   W = A[i] * C[k]   A tile K-major
//   mode 3: m = k, o = i, l = j   W = A[i] * B[j]   A tile MN-major (X^T)
// TMA zero-fills the out-of-range tail of each (o, .) run, so no byte is
// fetched twice.  The chunk's factor rows (F_lo[l0..l0+63], F_hi[o]) ride on
// the same TMA stage as the X tiles.
//
// Pipeline (one CTA per SM, warp-specialised, mbarrier handshakes):
//   warp 0      TMA producer: S0/S1 tiles (128B-swizzled) + factor rows
//   warp 1      TMEM allocator + single-thread MMA issuer (tcgen05.mma)
//   warps 2-5   KR formers: W slices of the chunk from the staged fp64 rows,
//               written in the UMMA K-major SW128 layout
//   warps 6-9   epilogue: tcgen05.ld of the two accumulators (double-buffered
//               in TMEM), double-float accumulation, fp64 partial per split.
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include <cstdlib>

#include "mttkrp_tc.cuh"

namespace ntf {

namespace {

constexpr int kTM = 128;     // MMA M (rows per tile, TMEM lanes)
constexpr int kBK = 64;      // q per chunk (fp16: 128 B rows, one SW128 atom)
constexpr int kUK = 16;      // MMA K for kind::f16
constexpr int kEpiWarps = 4;
// KR-former warps: more for small N (light epilogue, registers to spare)
__host__ __device__ constexpr int wf_warps(int NT) { return NT <= 2 ? 8 : 4; }
// warps: 0 X-tile TMA, 1 MMA, 2 factor-row TMA, KR formers, 4 epilogue
__host__ __device__ constexpr int tc_threads(int NT) { return (3 + wf_warps(NT) + kEpiWarps) * 32; }

// ----------------------------------------------------------------------------
// PTX wrappers
// ----------------------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
        "selp.u32 %0, 1, 0, P1;\n"
        "}\n"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
  } while (!done);
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                            int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%3, %4, %5}], [%2];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                            int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%3, %4}], [%2];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}

__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}

__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
          smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tc_mma_f16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                           uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// 32 lanes x 32 bits, 16 consecutive columns per thread
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

// UMMA shared-memory descriptor, SWIZZLE_128B (layout type 2), version 1.
__device__ __forceinline__ uint64_t smem_desc(const void* p, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  const uint64_t addr = smem_u32(p);
  uint64_t d = 0;
  d |= (addr >> 4) & 0x3FFFull;
  d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= 1ull << 46;
  d |= 2ull << 61;
  return d;
}

// kind::f16 instruction descriptor: F16 x F16 -> F32, M=128
__host__ __device__ constexpr uint32_t make_idesc(int N, bool a_mn_major) {
  return (1u << 4)                                 // D format F32
         | (0u << 7) | (0u << 10)                  // A, B format F16
         | ((a_mn_major ? 1u : 0u) << 15)          // A major
         | (0u << 16)                              // B K-major
         | ((static_cast<uint32_t>(N) >> 3) << 17) // N >> 3
         | ((static_cast<uint32_t>(kTM) >> 4) << 24);  // M >> 4
}

// accumulator sets (5N fp32 columns each) resident in TMEM: double-buffered
// when two fit in the 512 columns, so the MMA never waits for the epilogue
__host__ __device__ constexpr int acc_bufs(int N) { return 10 * N <= 512 ? 2 : 1; }

__host__ __device__ constexpr uint32_t tmem_cols(int N) {
  return acc_bufs(N) * 5 * N <= 32    ? 32
         : acc_bufs(N) * 5 * N <= 64  ? 64
         : acc_bufs(N) * 5 * N <= 128 ? 128
         : acc_bufs(N) * 5 * N <= 256 ? 256
                                      : 512;
}

struct TcParams {
  CUtensorMap tmap0;         // S0 plane, 3-D (K, J, I)
  CUtensorMap tmap1;         // S1 plane
  CUtensorMap tmap_lo;       // F_lo rows, 2-D (R, rows), box (R, 64)
  CUtensorMap tmap_hi;       // F_hi rows, 2-D (R, rows), box (R, 1)
  int mode, R;
  int64_t M;
  int64_t l_extent;          // extent of the chunked axis (K or J)
  int64_t n_chunks, chunks_per_split, chunks_per_o;
  int n_mtiles, splits;
  int x_stages, w_stages, f_stages;
  int stage_bytes;           // X tiles + factor rows
  const double* cm_hi;       // [R] max |F_hi[:, n]| (kept current by the row update)
  const double* cm_lo;       // [R] max |F_lo[:, n]|
  const double* xscale;      // tensor split scale (device scalar)
  double* ws;                // [splits][M][R] partials
  const int* stop_flag;
  int debug;                 // profiling only (NTF_TC_DEBUG): 1 skip KR, 2 skip MMA
};

__device__ __forceinline__ void fast_two_sum(float& hi, float& lo, float a) {
  const float s = hi + a;
  const float err = a - (s - hi);
  hi = s;
  lo += err;
}

// W slices for one (n, 8-q octet): 3 x 16 bytes at the swizzled positions.
// t (|t| <= 128) is converted to fp32 once: its rounding error (<= 2^-17) is
// far below the T2 quantum (2^-14), so slicing in fp32 loses nothing.
__device__ __forceinline__ void emit_w_octet(unsigned char* t0, unsigned char* t1, unsigned char* t2,
                                             int n, int oct, const double (&w)[8]) {
  __align__(16) __half2 h0[4], h1[4], h2[4];
  // round-to-nearest-even via the 1.5*2^23 magic constant (two FADDs, exact
  // for |x| < 2^22) instead of the slower FRND
  constexpr float kMagic = 12582912.0f;
#pragma unroll
  for (int u = 0; u < 8; u += 2) {
    float a0[2], a1[2], a2[2];
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      const float tf = static_cast<float>(w[u + v]);
      a0[v] = __fsub_rn(__fadd_rn(tf, kMagic), kMagic);     // integer, |a0| <= 128
      const float r1 = (tf - a0[v]) * 128.0f;                // exact, |r1| <= 64
      a1[v] = __fsub_rn(__fadd_rn(r1, kMagic), kMagic);
      const float r2 = (r1 - a1[v]) * 128.0f;
      a2[v] = __fsub_rn(__fadd_rn(r2, kMagic), kMagic);
    }
    h0[u / 2] = __floats2half2_rn(a0[0], a0[1]);                          // exact
    h1[u / 2] = __floats2half2_rn(a1[0] * 0.0078125f, a1[1] * 0.0078125f);  // 2^-7 units
    h2[u / 2] = __floats2half2_rn(a2[0] * 6.103515625e-05f, a2[1] * 6.103515625e-05f);  // 2^-14
  }
  const int off = n * 128 + ((oct ^ (n & 7)) << 4);
  *reinterpret_cast<uint4*>(t0 + off) = *reinterpret_cast<const uint4*>(h0);
  *reinterpret_cast<uint4*>(t1 + off) = *reinterpret_cast<const uint4*>(h1);
  *reinterpret_cast<uint4*>(t2 + off) = *reinterpret_cast<const uint4*>(h2);
}

template <int NT>  // N / 16
__global__ void __launch_bounds__(tc_threads(NT), 1) mttkrp_tc_kernel(const __grid_constant__ TcParams p) {
  constexpr int kWfWarps = wf_warps(NT);
  constexpr int N = NT * 16;
  constexpr int kAccBufs = acc_bufs(N);
  if (p.stop_flag && *p.stop_flag) return;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // carve: [X stages: S0 16KB | S1 16KB]  (released by the MMA)
  //        [factor stages: lo rows 64*R*8 | hi row R*8]  (released by KR formers)
  //        [W stages: T0 | T1 | T2 (N*128 each)] [barriers]
  // 1 KB alignment by offset (keeps the pointer in the shared address space,
  // so the compiler emits LDS/STS instead of generic loads/stores)
  unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  constexpr int kXTile = kTM * kBK * 2;  // 16 KB
  constexpr int kWTile = N * kBK * 2;    // N * 128 B
  const int SX = p.x_stages, SW = p.w_stages, SF = p.f_stages;
  const int R = p.R;
  const int SB = p.stage_bytes;          // factor stage bytes (1 KB aligned)
  unsigned char* xbase = base;
  unsigned char* fbase = xbase + SX * 2 * kXTile;
  unsigned char* wbase = fbase + SF * SB;
  uint64_t* bars = reinterpret_cast<uint64_t*>(wbase + SW * 3 * kWTile);
  uint64_t* x_full = bars;
  uint64_t* x_empty = x_full + SX;
  uint64_t* f_full = x_empty + SX;
  uint64_t* f_empty = f_full + SF;
  uint64_t* w_full = f_empty + SF;
  uint64_t* w_empty = w_full + SW;
  uint64_t* acc_full = w_empty + SW;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  // per-column W scales: wsc[n] = 2^(7 - f(n)) with max|F_hi[:,n]| max|F_lo[:,n]|
  // <= 2^f(n), so |t| = |W| 2^(7-f) <= 128; wsc[N + n] = xscale * 2^(f(n) - 7)
  double* wsc = reinterpret_cast<double*>(acc_empty + 4);
  if (threadIdx.x < N) {
    const int n = threadIdx.x;
    const double prod = n < p.R ? p.cm_hi[n] * p.cm_lo[n] : 0.0;
    int f = 0;
    if (prod > 0.0) frexp(prod, &f);  // prod < 2^f
    // a column that decayed to ~1e-300 (large penalties shrink factor columns
    // geometrically) must not overflow the scale: clamp (represented as zero)
    if (f < -1000) f = -1000;
    wsc[n] = ldexp(1.0, 7 - f);
    wsc[N + n] = *p.xscale * ldexp(1.0, f - 7);
  }

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  constexpr int kWfFirst = 3;
  constexpr int kEpiFirst = 3 + kWfWarps;
  constexpr int kWfThreads = kWfWarps * 32;

  const int tile = blockIdx.x % p.n_mtiles;
  const int split = blockIdx.x / p.n_mtiles;
  const int64_t m0 = static_cast<int64_t>(tile) * kTM;
  const int64_t c_begin = static_cast<int64_t>(split) * p.chunks_per_split;
  int64_t c_end = c_begin + p.chunks_per_split;
  if (c_end > p.n_chunks) c_end = p.n_chunks;
  const int n_iter = c_begin < c_end ? static_cast<int>(c_end - c_begin) : 0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < SX; ++s) {
      mbar_init(&x_full[s], 1);
      mbar_init(&x_empty[s], 1);  // MMA commit
    }
    for (int s = 0; s < SF; ++s) {
      mbar_init(&f_full[s], 1);
      mbar_init(&f_empty[s], kWfThreads);  // KR formers consumed the rows
    }
    for (int s = 0; s < SW; ++s) {
      mbar_init(&w_full[s], kWfThreads);
      mbar_init(&w_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&acc_full[s], 1);
      mbar_init(&acc_empty[s], kEpiWarps * 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(tmem_cols(N)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 2) {
    // ---------------------------- factor-row producer -------------------------
    if (lane == 0) {
      // factor rows of each chunk: F_lo[l0 .. l0+63] and F_hi[o]
      const uint32_t fac_bytes = static_cast<uint32_t>((kBK + 1) * R * 8);
      for (int it = 0; it < n_iter; ++it) {
        const int fs = it % SF;
        mbar_wait(&f_empty[fs], ((it / SF) & 1) ^ 1);
        unsigned char* dlo = fbase + fs * SB;
        unsigned char* dhi = dlo + kBK * R * 8;
        mbar_arrive_expect_tx(&f_full[fs], fac_bytes);
        const int64_t c = c_begin + it;
        const int o = static_cast<int>(c / p.chunks_per_o);
        const int l0 = static_cast<int>((c - static_cast<int64_t>(o) * p.chunks_per_o) * kBK);
        tma_load_2d(dlo, &p.tmap_lo, &f_full[fs], 0, l0);
        tma_load_2d(dhi, &p.tmap_hi, &f_full[fs], 0, o);
      }
    }
  } else if (warp == 0) {
    // ------------------------------ X-tile producer ---------------------------
    if (lane == 0) {
      for (int it = 0; it < n_iter; ++it) {
        const int s = it % SX;
        mbar_wait(&x_empty[s], ((it / SX) & 1) ^ 1);
        unsigned char* d0 = xbase + s * 2 * kXTile;
        unsigned char* d1 = d0 + kXTile;
        mbar_arrive_expect_tx(&x_full[s], 2 * kXTile);
        const int64_t c = c_begin + it;
        const int o = static_cast<int>(c / p.chunks_per_o);
        const int l0 = static_cast<int>((c - static_cast<int64_t>(o) * p.chunks_per_o) * kBK);
        const int mm = static_cast<int>(m0);
        if (p.mode == 1) {
          tma_load_3d(d0, &p.tmap0, &x_full[s], l0, o, mm);
          tma_load_3d(d1, &p.tmap1, &x_full[s], l0, o, mm);
        } else if (p.mode == 2) {
          tma_load_3d(d0, &p.tmap0, &x_full[s], l0, mm, o);
          tma_load_3d(d1, &p.tmap1, &x_full[s], l0, mm, o);
        } else {  // two 64-m boxes per plane
          tma_load_3d(d0, &p.tmap0, &x_full[s], mm, l0, o);
          tma_load_3d(d0 + kXTile / 2, &p.tmap0, &x_full[s], mm + 64, l0, o);
          tma_load_3d(d1, &p.tmap1, &x_full[s], mm, l0, o);
          tma_load_3d(d1 + kXTile / 2, &p.tmap1, &x_full[s], mm + 64, l0, o);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------ MMA issuer --------------------------------
    if (lane == 0) {
      // Two wide MMAs per K step, each reading its A tile once: the W slices
      // T0|T1|T2 are consecutive N-row blocks of one K-major B operand.
      //   cols [0, 3N):  S0 * [T0 | T1 | T2]     cols [3N, 5N): S1 * [T0 | T1]
      const bool mn = p.mode == 3;
      const uint32_t idesc3 = make_idesc(3 * N, mn);
      const uint32_t idesc2 = make_idesc(2 * N, mn);
      for (int it = 0; it < n_iter; ++it) {
        const int s = it % SX, sw = it % SW, ab = it % kAccBufs;
        mbar_wait(&x_full[s], (it / SX) & 1);
        mbar_wait(&w_full[sw], (it / SW) & 1);
        mbar_wait(&acc_empty[ab], ((it / kAccBufs) & 1) ^ 1);
        tc_fence_after();
        const unsigned char* a0 = xbase + s * 2 * kXTile;
        const unsigned char* a1 = a0 + kXTile;
        const unsigned char* b0 = wbase + sw * 3 * kWTile;
        const uint32_t d0 = tmem + ab * 5 * N;
        const uint32_t d1 = d0 + 3 * N;
#pragma unroll
        for (int kk = 0; kk < ((p.debug & 2) && it >= 2 ? 0 : kBK / kUK); ++kk) {
          uint64_t da0, da1;
          if (mn) {  // A = X^T: MN-major, atoms of 64 m (8 KB apart), 8 q-rows per 1 KB
            da0 = smem_desc(a0 + kk * 2048, kXTile / 2, 1024);
            da1 = smem_desc(a1 + kk * 2048, kXTile / 2, 1024);
          } else {   // K-major: 128 B rows, 8-row groups 1 KB apart, +32 B per K step
            da0 = smem_desc(a0 + kk * 32, 16, 1024);
            da1 = smem_desc(a1 + kk * 32, 16, 1024);
          }
          const uint64_t db = smem_desc(b0 + kk * 32, 16, 1024);
          const uint32_t acc = kk > 0 ? 1u : 0u;
          tc_mma_f16(d0, da0, db, idesc3, acc);   // S0*T0 (exact), S0*T1, S0*T2
          tc_mma_f16(d1, da1, db, idesc2, acc);   // S1*T0, S1*T1
        }
        tc_commit(&x_empty[s]);
        tc_commit(&w_empty[sw]);
        tc_commit(&acc_full[ab]);
      }
    }
  } else if (warp < kEpiFirst) {
    // ------------------------------ KR formers --------------------------------
    // thread t owns column n = t % N (lanes along n: conflict-free row reads)
    // and octets t / N, t / N + kWfThreads / N, ...
    const int t = threadIdx.x - kWfFirst * 32;
    const int n = t % N;
    const int oct0 = t / N;
    constexpr int kOctStep = kWfThreads / N > 0 ? kWfThreads / N : 1;
    const bool active = t < N * (kBK / 8) && (kWfThreads >= N || true);
    const double sc = n < R ? wsc[n] : 0.0;
    for (int it = 0; it < n_iter; ++it) {
      const int fs = it % SF, sw = it % SW;
      mbar_wait(&f_full[fs], (it / SF) & 1);
      mbar_wait(&w_empty[sw], ((it / SW) & 1) ^ 1);
      const unsigned char* srow = fbase + fs * SB;
      const double* lo_s = reinterpret_cast<const double*>(srow);
      const double* hi_s = lo_s + kBK * R;
      unsigned char* t0 = wbase + sw * 3 * kWTile;
      unsigned char* t1 = t0 + kWTile;
      unsigned char* t2 = t1 + kWTile;
      if (active && !((p.debug & 1) && it >= SW)) {
        const double hs = n < R ? hi_s[n] * sc : 0.0;
        for (int oct = oct0; oct < kBK / 8; oct += kOctStep) {
          double w[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) w[u] = n < R ? hs * lo_s[(oct * 8 + u) * R + n] : 0.0;
          emit_w_octet(t0, t1, t2, n, oct, w);
        }
      }
      fence_proxy_async();
      mbar_arrive(&w_full[sw]);
      mbar_arrive(&f_empty[fs]);  // factor rows consumed
    }
  } else {
    // ------------------------------ epilogue ----------------------------------
    const int q4 = warp & 3;          // TMEM lane quarter of this warp
    const int row = q4 * 32 + lane;   // tile row == TMEM lane
    float hi[N], lo[N];
#pragma unroll
    for (int j = 0; j < N; ++j) {
      hi[j] = 0.f;
      lo[j] = 0.f;
    }
    for (int it = 0; it < n_iter; ++it) {
      const int ab = it % kAccBufs;
      mbar_wait(&acc_full[ab], (it / kAccBufs) & 1);
      tc_fence_after();
      const uint32_t taddr = tmem + (static_cast<uint32_t>(q4 * 32) << 16) + ab * 5 * N;
#pragma unroll
      for (int j = 0; j < ((p.debug & 4) && it >= 2 ? 0 : NT); ++j) {
        float a0[16], a1[16], a2[16];
        tmem_ld16(taddr + j * 16, a0);           // S0*T0 (exact integers)
        tmem_ld16(taddr + N + j * 16, a1);       // S0*T1
        tmem_ld16(taddr + 2 * N + j * 16, a2);   // S0*T2
        tmem_wait_ld();
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          fast_two_sum(hi[j * 16 + u], lo[j * 16 + u], a0[u]);
          a1[u] += a2[u];
        }
        tmem_ld16(taddr + 3 * N + j * 16, a0);   // S1*T0
        tmem_ld16(taddr + 4 * N + j * 16, a2);   // S1*T1
        tmem_wait_ld();
#pragma unroll
        for (int u = 0; u < 16; ++u) lo[j * 16 + u] += (a1[u] + a0[u]) + a2[u];
      }
      tc_fence_before();
      mbar_arrive(&acc_empty[ab]);
    }
    // fp64 partial of this split: out = (hi + lo) * xscale * ws(n)
    const int64_t gm = m0 + row;
    if (gm < p.M) {
      double* out = p.ws + (static_cast<int64_t>(split) * p.M + gm) * R;
#pragma unroll
      for (int j = 0; j < N; ++j)
        if (j < R) out[j] = (static_cast<double>(hi[j]) + static_cast<double>(lo[j])) * wsc[N + j];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem),
                 "r"(tmem_cols(N)));
  }
}

// ----------------------------------------------------------------------------
// tensor split: max|X| then S0 / S1 planes
// ----------------------------------------------------------------------------
__global__ void absmax_kernel(const float* __restrict__ X, int64_t n, unsigned* out) {
  float m = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    m = fmaxf(m, fabsf(X[i]));
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, __float_as_uint(m));  // order-free: max is exact
}

__global__ void split_kernel(const float* __restrict__ X, int64_t n, const unsigned* amax,
                             __half* __restrict__ s0, __half* __restrict__ s1, double* xscale) {
  const float mx = __uint_as_float(*amax);
  int e = 0;
  if (mx > 0.f) frexpf(mx, &e);            // mx < 2^e
  const float up = ldexpf(1.0f, 11 - e);   // X * 2^(11-e) in [-2048, 2048]
  if (blockIdx.x == 0 && threadIdx.x == 0) *xscale = ldexp(1.0, e - 11);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float s = X[i] * up;              // exact (power-of-two scaling)
    const float a0 = rintf(s);
    const float r = (s - a0) * 2048.0f;     // exact
    const float a1 = rintf(r);
    s0[i] = __float2half_rn(a0);
    s1[i] = __float2half_rn(a1 * 4.8828125e-04f);  // 2^-11 units
  }
}

// out[r] = max_i |F[i][r]| (one block per column; max is order-free)
__global__ void colmax_kernel(const double* __restrict__ F, int64_t rows, int R, double* out) {
  const int r = blockIdx.x;
  double m = 0.0;
  for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) m = fmax(m, fabs(F[i * R + r]));
  __shared__ double sh[32];
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) m = fmax(m, sh[w]);
    out[r] = m;
  }
}

PFN_cuTensorMapEncodeTiled_v12000 get_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

int sm_count_tc() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// fp64 factor rows [rows][R] as a 2-D tensor map with box (R, box_rows)
cudaError_t encode_factor_map(CUtensorMap* map, const double* F, int64_t rows, int R,
                              int box_rows) {
  auto enc = get_encoder();
  if (!enc) return cudaErrorNotSupported;
  cuuint64_t gdim[2] = {static_cast<cuuint64_t>(R), static_cast<cuuint64_t>(rows)};
  cuuint64_t gstr[1] = {static_cast<cuuint64_t>(R) * 8};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(R), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(F), gdim, gstr, box,
                   es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <int NT>
cudaError_t launch_nt(const TcParams& p, const MttkrpTCLaunch& L, cudaStream_t stream, bool prep) {
  auto kern = mttkrp_tc_kernel<NT>;
  if (prep) return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L.smem_bytes);
  kern<<<L.n_mtiles * L.splits, L.threads, L.smem_bytes, stream>>>(p);
  return cudaGetLastError();
}

cudaError_t dispatch_tc(const TcParams& p, const MttkrpTCLaunch& L, cudaStream_t stream, bool prep) {
  switch (L.N / 16) {
    case 1: return launch_nt<1>(p, L, stream, prep);
    case 2: return launch_nt<2>(p, L, stream, prep);
    case 3: return launch_nt<3>(p, L, stream, prep);
    case 4: return launch_nt<4>(p, L, stream, prep);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

// ----------------------------------------------------------------------------
// host API
// ----------------------------------------------------------------------------
bool mttkrp_tc_supported(int x_dtype, int R) {
  // even R: the fp64 factor rows are TMA boxes of R*8 bytes (multiple of 16)
  return x_dtype == NTF_F32 && R >= 2 && R <= 64 && R % 2 == 0;
}

bool mttkrp_tc_auto(int x_dtype, int R) {
  static int enabled = -1;
  if (enabled < 0) {
    const char* env = getenv("NTF_B200_TC");
    enabled = env ? (env[0] != '0') : 1;
  }
  return enabled && mttkrp_tc_supported(x_dtype, R);
}

bool mttkrp_tc_shape_ok(int mode, int64_t I, int64_t J, int64_t K) {
  // TMA global strides are multiples of 16 B (K % 8 == 0 for the fp16 planes);
  // coordinates are int32.
  (void)mode;
  if (K % 8 != 0) return false;
  if (I >= (1 << 30) || J >= (1 << 30) || K >= (1 << 30)) return false;
  return true;
}

MttkrpTCLaunch mttkrp_tc_plan(int mode, int x_dtype, int64_t I, int64_t J, int64_t K, int R) {
  (void)x_dtype;
  MttkrpTCLaunch L{};
  L.mode = mode;
  L.R = R;
  L.N = ((R + 15) / 16) * 16;
  L.M = mode == 1 ? I : (mode == 2 ? J : K);
  L.Q = mode == 3 ? I * J : (mode == 1 ? J * K : I * K);
  L.n_mtiles = static_cast<int>((L.M + kTM - 1) / kTM);
  const int64_t l_ext = mode == 3 ? J : K;
  const int64_t o_ext = mode == 1 ? J : I;
  L.chunks_per_o = (l_ext + kBK - 1) / kBK;
  L.n_chunks = o_ext * L.chunks_per_o;
  L.n_wf_warps = wf_warps(L.N / 16);
  L.threads = tc_threads(L.N / 16);
  // X ring as deep as shared memory allows (bytes in flight hide HBM latency);
  // the factor-row and KR rings only need to stay a few chunks ahead.
  const int xs = 2 * kTM * kBK * 2;
  L.stage_bytes = ((kBK + 1) * R * 8 + 1023) & ~1023;  // factor stage
  const int wsz = 3 * L.N * kBK * 2;
  L.x_stages = 4;
  L.f_stages = 3;
  L.w_stages = 3;
  if (const char* e2 = getenv("NTF_TC_WSTAGES")) L.w_stages = atoi(e2);
  auto total = [&]() {
    // + barriers, TMEM slot and the 2N per-column scales
    return 1024 + L.x_stages * xs + L.f_stages * L.stage_bytes + L.w_stages * wsz + 512 + 16 * L.N;
  };
  const char* env = getenv("NTF_TC_XSTAGES");
  if (env) L.x_stages = atoi(env);
  while (total() > 227 * 1024 && L.x_stages > 2) --L.x_stages;
  while (total() > 227 * 1024 && L.f_stages > 2) --L.f_stages;
  L.smem_bytes = total();
  L.tmem_cols = static_cast<int>(tmem_cols(L.N));
  // one CTA per SM; split the chunk range so that the grid is one wave
  const int sms = sm_count_tc();
  // one SM is left free so the mode's ridge Cholesky (side stream) runs
  // concurrently instead of queueing behind the MTTKRP
  int splits = (sms - 1) / L.n_mtiles;
  if (splits < 1) splits = 1;
  if (splits > L.n_chunks) splits = static_cast<int>(L.n_chunks);
  L.chunks_per_split = (L.n_chunks + splits - 1) / splits;
  L.splits = static_cast<int>((L.n_chunks + L.chunks_per_split - 1) / L.chunks_per_split);
  L.wscale = nullptr;
  L.bound = false;
  return L;
}

size_t mttkrp_tc_workspace_bytes(const MttkrpTCLaunch& L, int R) {
  return static_cast<size_t>(L.splits) * L.M * R * sizeof(double);
}

cudaError_t mttkrp_tc_prepare(const MttkrpTCLaunch& L) {
  TcParams p{};
  return dispatch_tc(p, L, nullptr, true);
}

cudaError_t tc_tensor_create(const float* X, const int64_t dims[3], TcTensor* out,
                             cudaStream_t stream) {
  const int64_t n = dims[0] * dims[1] * dims[2];
  TcTensor t;
  for (int i = 0; i < 3; ++i) t.dims[i] = dims[i];
  cudaError_t e;
  if ((e = cudaMalloc(&t.s0, n * sizeof(__half))) != cudaSuccess) return e;
  if ((e = cudaMalloc(&t.s1, n * sizeof(__half))) != cudaSuccess) {
    tc_tensor_destroy(&t);
    return e;
  }
  if ((e = cudaMalloc(&t.xscale, sizeof(double) + sizeof(unsigned) * 2)) != cudaSuccess) {
    tc_tensor_destroy(&t);
    return e;
  }
  unsigned* amax = reinterpret_cast<unsigned*>(t.xscale + 1);
  cudaMemsetAsync(amax, 0, sizeof(unsigned), stream);
  const int blocks = 4 * sm_count_tc();
  absmax_kernel<<<blocks, 256, 0, stream>>>(X, n, amax);
  split_kernel<<<blocks, 256, 0, stream>>>(X, n, amax, t.s0, t.s1, t.xscale);
  if ((e = cudaGetLastError()) != cudaSuccess) {
    tc_tensor_destroy(&t);
    return e;
  }
  *out = t;
  return cudaSuccess;
}

void tc_tensor_destroy(TcTensor* t) {
  if (!t) return;
  cudaFree(t->s0);
  cudaFree(t->s1);
  cudaFree(t->xscale);
  t->s0 = t->s1 = nullptr;
  t->xscale = nullptr;
}

cudaError_t mttkrp_tc_bind(MttkrpTCLaunch& L, const TcTensor& t) {
  auto enc = get_encoder();
  if (!enc) return cudaErrorNotSupported;
  const int64_t I = t.dims[0], J = t.dims[1], K = t.dims[2];
  cuuint64_t gdim[3] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(J),
                        static_cast<cuuint64_t>(I)};
  cuuint64_t gstr[2] = {static_cast<cuuint64_t>(K * 2), static_cast<cuuint64_t>(J * K * 2)};
  cuuint32_t box[3];
  if (L.mode == 1) {
    box[0] = 64; box[1] = 1; box[2] = 128;
  } else if (L.mode == 2) {
    box[0] = 64; box[1] = 128; box[2] = 1;
  } else {
    box[0] = 64; box[1] = 64; box[2] = 1;
  }
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r0 = enc(&L.tmap0, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, t.s0, gdim, gstr, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUresult r1 = enc(&L.tmap1, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, t.s1, gdim, gstr, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r0 != CUDA_SUCCESS || r1 != CUDA_SUCCESS) return cudaErrorInvalidValue;
  if (!L.wscale) {
    cudaError_t e = cudaMalloc(&L.wscale, sizeof(double) * 2 * L.N);
    if (e != cudaSuccess) return e;
  }
  L.fac_lo = nullptr;
  L.fac_hi = nullptr;
  L.bound = true;
  return cudaSuccess;
}

void mttkrp_tc_unbind(MttkrpTCLaunch& L) {
  cudaFree(L.wscale);
  L.wscale = nullptr;
  L.bound = false;
}

cudaError_t colmax_launch(const double* F, int64_t rows, int R, double* out, cudaStream_t stream) {
  colmax_kernel<<<R, 256, 0, stream>>>(F, rows, R, out);
  return cudaGetLastError();
}

cudaError_t mttkrp_tc_launch(MttkrpTCLaunch& L, const TcTensor& t, const double* A,
                             const double* B, const double* C, const double* colmax3, double* ws,
                             const int* stop_flag, cudaStream_t stream) {
  if (!L.bound) return cudaErrorInvalidValue;
  const int64_t I = t.dims[0], J = t.dims[1], K = t.dims[2];
  const double *Fhi, *Flo;
  int64_t hi_rows, lo_rows;
  if (L.mode == 1) {
    Fhi = B; Flo = C; hi_rows = J; lo_rows = K;
  } else if (L.mode == 2) {
    Fhi = A; Flo = C; hi_rows = I; lo_rows = K;
  } else {
    Fhi = A; Flo = B; hi_rows = I; lo_rows = J;
  }
  // factor tensor maps are cached per factor pointer (plan buffers are fixed)
  if (Flo != L.fac_lo) {
    cudaError_t e = encode_factor_map(&L.tmap_lo, Flo, lo_rows, L.R, kBK);
    if (e != cudaSuccess) return e;
    L.fac_lo = Flo;
  }
  if (Fhi != L.fac_hi) {
    cudaError_t e = encode_factor_map(&L.tmap_hi, Fhi, hi_rows, L.R, 1);
    if (e != cudaSuccess) return e;
    L.fac_hi = Fhi;
  }
  TcParams p{};
  p.tmap0 = L.tmap0;
  p.tmap1 = L.tmap1;
  p.tmap_lo = L.tmap_lo;
  p.tmap_hi = L.tmap_hi;
  p.mode = L.mode;
  p.R = L.R;
  p.M = L.M;
  p.l_extent = L.mode == 3 ? J : K;
  p.n_chunks = L.n_chunks;
  p.chunks_per_split = L.chunks_per_split;
  p.chunks_per_o = L.chunks_per_o;
  p.n_mtiles = L.n_mtiles;
  p.splits = L.splits;
  p.x_stages = L.x_stages;
  p.w_stages = L.w_stages;
  p.f_stages = L.f_stages;
  p.stage_bytes = L.stage_bytes;
  p.ws = ws;
  p.stop_flag = stop_flag;
  {
    static int dbg = -1;
    if (dbg < 0) {
      const char* env = getenv("NTF_TC_DEBUG");
      dbg = env ? atoi(env) : 0;
    }
    p.debug = dbg;
  }
  p.xscale = t.xscale;
  if (colmax3) {  // plan: column maxima kept current by the row-update kernels
    const int hm = L.mode == 1 ? 1 : 0, lm = L.mode == 3 ? 1 : 2;
    p.cm_hi = colmax3 + hm * L.R;
    p.cm_lo = colmax3 + lm * L.R;
  } else {        // one-shot call: compute them here
    colmax_kernel<<<L.R, 256, 0, stream>>>(Fhi, hi_rows, L.R, L.wscale);
    colmax_kernel<<<L.R, 256, 0, stream>>>(Flo, lo_rows, L.R, L.wscale + L.R);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    p.cm_hi = L.wscale;
    p.cm_lo = L.wscale + L.R;
  }
  return dispatch_tc(p, L, stream, false);
}

}  // namespace ntf
