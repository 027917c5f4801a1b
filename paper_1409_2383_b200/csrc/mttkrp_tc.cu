// Dense MTTKRP on the 5th-generation tensor cores (tcgen05, sm_100a) for fp32
// tensors.  Same contraction as mttkrp_cc.cu (reference tensors.py:254-262):
//   out[m, n] = sum_o F_hi[o, n] * sum_l X(m, o, l) F_lo[l, n]
// with (o, l) the two non-m tensor axes:
//   mode 1: m = i, o = j, l = k   (F_hi, F_lo) = (B, C)
//   mode 2: m = j, o = i, l = k   (F_hi, F_lo) = (A, C)
//   mode 3: m = k, o = i, l = j   (F_hi, F_lo) = (A, B)
//
// Numerics: fixed-point slicing on kind::f16 MMAs with an exact leading term.
//   X    = xs * (S0 + S1)        S0 integers |S0| <= 2^11, S1 = fp16 of the
//                                exact remainder in [-1/2, 1/2] (11 significant
//                                bits of it), xs = 2^(e-11) global
//   F_lo = ls(n) * (T0 + T1 + T2)  T0 integers |T0| <= 2^t, T1, T2 = fp16 of the
//                                successive exact remainders (T2 possibly
//                                subnormal), ls(n) = 2^(f(n)-t) per column;
//   Fh   = fp16(F_lo / ls(n))    F_lo to 11 significant bits
//   (N <= 85: T2 is stored as 2^11 T2 in its own accumulator, scaled back in
//   the epilogue, so its fp16 subnormal floor sits at 2^-36 instead of 2^-25)
// The tensor core forms, per unit of G consecutive 64-wide l blocks at one o,
//   ACC0 = sum S0*T0                       integers < 2^24: EXACT in fp32
//   ACC1 = sum S0*T1 + S1*Fh,  ACC2 = sum S0*T2        (corrections; for
//   N > 85 ACC2's terms go straight into ACC1: two sets of 2N columns fit)
// i.e. 4N MMA columns per K step (S1 multiplies the 11-bit Fh: its weight is
// 2^-11 below S0's, so Fh's 2^-12 relative rounding sits at ~2^-23 of the
// product and averages out over the contraction).  t = 7, 6, 5, 5 for
// G = 1..4 keeps |ACC0| <= 2^11 * 2^t * 64G <= 2^24.  F_lo is represented to
// 2^-25 of 2^t (2^-30 of its column maximum at t = 5), X to 2^-24 of its
// maximum.  The epilogue multiplies the unit's accumulators by F_hi[o, n]
// held as an fp32 pair (exact product split with FMA) and accumulates in
// double-float (TwoSum, packed f32x2 on two columns at a time), so F_hi
// enters at ~2^-48.
//
// Data layout: the split tensor is stored once per mode as a BLOCK IMAGE
// (image_split_kernel): for each m-tile and unit (g, o) in g-major order, each
// l block is the no-swizzle K-major UMMA image of both planes.  A CTA owns one
// m-tile and a contiguous range of units, so it streams ONE contiguous byte
// range, block after block (long sequential DRAM runs; the natural layout's
// 128-byte row pieces ran at 4.4-4.8 TB/s, the image at 6.7).  The W slices of
// a group do not depend on o: formed once per MTTKRP (w_slice_kernel) and
// copied into shared memory once per group; the epilogue drains TMEM once per
// unit.
//
// CTA pairs (CG = 2, the default): two CTAs on one TPC take two consecutive
// m-tiles with the same unit range; the leader issues tcgen05.mma.cta_group::2
// (M = 256: each CTA's 128 rows of A from its own shared memory, each MMA's
// N' rows of B split between them), so each CTA holds only half of the W
// slices (twice the l blocks per unit for the same shared memory) and one MMA
// instruction serves both SMs.  Both CTAs load their blocks with 2-CTA tensor
// -map loads that complete on the leader's barriers; the leader's commits
// multicast to both CTAs; each CTA drains its own TMEM lanes.
//
// Roles (one CTA per SM, mbarrier handshakes, all ring indices incremental):
//   warp 0        producer: one copy per X block into an SX-stage ring
//   warps 1, 3    MMA issuers on alternate units (a single issuing thread is
//                 bound by per-instruction issue latency for small-N MMAs);
//                 each owns its accumulator sets, both release X slots
//                 (a pair's peer CTA: idle)
//   warp 2        W slices of each group + F_hi pair rows
//   warps 4..     epilogue, 8 or 16 warps (2 or 4 column groups per
//                 TMEM lane quarter, by N): per unit tcgen05.ld, F_hi scaling,
//                 double-float accumulation; finally the fp64 partial of the CTA.
#include <cudaTypedefs.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "mttkrp_tc.cuh"

namespace ntf {

namespace {

constexpr int kTM = 128;     // MMA M (rows per tile, TMEM lanes)
constexpr int kBK = 64;      // l per block (fp16: 128 B rows, one SW128 atom)
constexpr int kUK = 16;      // MMA K for kind::f16
constexpr int kFMin = -990;  // exponent clamp of the column scales (2^(7+22-kFMin) finite)
// epilogue warps: 2 or 4 per TMEM lane quarter (column groups), keeping
// the double-float accumulators (2 x N / groups per thread) in registers
// (the per-thread column count N*4/warps must be a multiple of 8).  N <= 32
// runs 8 warps too: the last unit's drain is on the kernel's critical tail
// (c2: 599 vs 594 it/s with 4 warps)
#ifndef NTF_EPI_SMALL
#define NTF_EPI_SMALL 8
#endif
#ifndef NTF_EPI_N112
#define NTF_EPI_N112 8
#endif
__host__ __device__ constexpr int epi_warps(int NT) {
  return NT <= 2 ? NTF_EPI_SMALL : ((NT == 6 || NT == 8) ? 16 : (NT == 7 ? NTF_EPI_N112 : 8));
}
// warps: 0 X producer, 1 and 3 MMA issuers (alternate units; warp 3 idle
// when only one accumulator set fits), 2 W slices + F_hi rows, 4.. epilogue
// (warp & 3 = its TMEM lane quarter)
__host__ __device__ constexpr int tc_threads(int NT) { return (4 + epi_warps(NT)) * 32; }

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

// try_wait with a suspend-time hint: the thread sleeps until the phase
// completes (or the hint expires) instead of re-polling the barrier
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n"
        "selp.u32 %0, 1, 0, P1;\n"
        "}\n"
        : "=r"(done)
        : "r"(addr), "r"(parity), "r"(1000000u)
        : "memory");
  } while (!done);
}

// NTF_TC_DEBUG & 32: cycles each role spends waiting (printed per CTA)
// wm: bit 0 profile (count the cycles), bit 1 wait with a suspend-time hint
__device__ __forceinline__ void mbar_wait_p(uint64_t* bar, uint32_t parity, int wm, long long& acc) {
  if (!(wm & 1)) {
    if (wm & 2) mbar_wait_sleep(bar, parity);
    else mbar_wait(bar, parity);
    return;
  }
  const long long t0 = clock64();
  mbar_wait(bar, parity);
  acc += clock64() - t0;
}

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// one lane of a converged warp (the warp's loop stays warp-uniform, so
// descriptors and barrier addresses live in uniform registers)
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n"
      ".reg .pred P;\n"
      "elect.sync _|P, 0xffffffff;\n"
      "selp.u32 %0, 1, 0, P;\n"
      "}\n"
      : "=r"(pred));
  return pred != 0;
}

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}

__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}

// Completion of this thread's earlier tcgen05 ops arrives on `bar`; for a CTA
// pair (CG = 2) on the barrier at the same offset in BOTH CTAs.
template <int CG>
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  if constexpr (CG == 1) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
            smem_u32(bar))
        : "memory");
  } else {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
        "[%0], %1;\n" ::"r"(smem_u32(bar)),
        "h"(static_cast<uint16_t>(3))
        : "memory");
  }
}

// D[tmem] (+)= A[smem] * B[smem]; CG = 2: M = 256 over the CTA pair (each
// CTA's A rows and half of B's N rows at the same shared-memory offsets),
// issued by the pair's leader only.
// COLL: 0 plain; 1 keep A in the tensor core's operand collector for the next
// MMA (collector::a::fill); 2 take A from the collector, last use
// (collector::a::lastuse).  Only valid when ONE thread issues every MMA of the
// CTA (pair): another issuer's MMAs would interleave and replace the kept A.
template <int CG, int COLL = 0>
__device__ __forceinline__ void tc_mma_f16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                           uint32_t idesc, uint32_t accumulate) {
  if constexpr (CG == 2 && COLL == 1) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::f16.collector::a::fill [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
  } else if constexpr (CG == 2 && COLL == 2) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::f16.collector::a::lastuse [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
  } else if constexpr (CG == 1) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
  } else {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
  }
}

// 2-D tensor-map load into this CTA's shared memory whose completion (bytes)
// is counted on the mbarrier at `bar_cluster` (a shared::cluster address: for
// a CTA pair the leader's barrier, cta_group::2).
__device__ __forceinline__ void tma_load_2sm(void* dst, const CUtensorMap* map, int32_t c0, int32_t c1,
                                             uint32_t bar_cluster) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3}], [%4];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar_cluster)
      : "memory");
}

__device__ __forceinline__ uint32_t mapa_u32(uint32_t addr, uint32_t cta) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(addr), "r"(cta));
  return r;
}

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// arrive on the barrier at `bar`'s offset in CTA `cta` of the cluster (default
// .release.cta semantics: a cluster-scope release per arrival measured ~2x
// slower epilogues in the pair's peer CTA)
__device__ __forceinline__ void mbar_arrive_remote(uint64_t* bar, uint32_t cta) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(remote) : "r"(smem_u32(bar)), "r"(cta));
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];\n" ::"r"(remote) : "memory");
}

// wait with acquire at cluster scope (arrivals from the peer CTA)
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%1], %2;\n"
        "selp.u32 %0, 1, 0, P1;\n"
        "}\n"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
  } while (!done);
}

// store a word into the same shared-memory offset of CTA `cta` of the cluster
__device__ __forceinline__ void st_cluster_u32(uint32_t* p, uint32_t cta, uint32_t v) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(remote) : "r"(smem_u32(p)), "r"(cta));
  asm volatile("st.shared::cluster.u32 [%0], %1;\n" ::"r"(remote), "r"(v) : "memory");
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

// 32 lanes x 32 bits, 8 consecutive columns per thread
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

// 32 lanes x 32 bits, 4 consecutive columns per thread
__device__ __forceinline__ void tmem_ld4(uint32_t taddr, float (&v)[4]) {
  uint32_t r[4];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 4; ++i) v[i] = __uint_as_float(r[i]);
}

template <int W>
__device__ __forceinline__ void tmem_ld(uint32_t taddr, float (&v)[W]) {
  if constexpr (W == 16) tmem_ld16(taddr, v);
  else if constexpr (W == 8) tmem_ld8(taddr, v);
  else tmem_ld4(taddr, v);
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

// UMMA shared-memory descriptor, no swizzle (layout type 0): K-major core
// matrices of 8 rows x 16 B; lbo = stride between K-adjacent core matrices,
// sbo = stride between M-adjacent (8-row) core matrices.
__device__ __forceinline__ uint64_t smem_desc_noswz(const void* p, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  const uint64_t addr = smem_u32(p);
  uint64_t d = 0;
  d |= (addr >> 4) & 0x3FFFull;
  d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= 1ull << 46;
  return d;
}

// kind::f16 instruction descriptor: F16 x F16 -> F32, M = 128 per CTA of the group
__host__ __device__ constexpr uint32_t make_idesc(int N, bool a_mn_major, int cg = 1) {
  return (1u << 4)                                 // D format F32
         | (0u << 7) | (0u << 10)                  // A, B format F16
         | ((a_mn_major ? 1u : 0u) << 15)          // A major
         | (0u << 16)                              // B K-major
         | ((static_cast<uint32_t>(N) >> 3) << 17) // N >> 3
         | ((static_cast<uint32_t>(kTM * cg) >> 4) << 24);  // M >> 4
}

// Accumulator set per unit: [ACC0 | ACC1 | ACC2] (3N fp32 columns), or for
// N > 85 (3N > 256, the MMA N limit) the merged [ACC0 | ACC12] (2N columns):
// ACC2's terms (2^-11 below ACC1's) are accumulated into ACC1 directly, which
// loses nothing (ACC1's own fp32 rounding dominates) and lets two sets fit.
// As many sets as fit (up to 4) so the MMA runs ahead of the epilogue.
__host__ __device__ constexpr bool merged_acc(int N) { return 3 * N > 256; }
// Packed T0 / T1 ranges (merged sets only; NP = N - 8 when R <= N - 8, else
// NP = N): the MMA N' must be a multiple of 16, but S0 x [T0|T1] only needs
// 2 NP columns to be one: R = 100 runs it at N' = 208 instead of 224 (ACC0 in
// columns [0, NP), ACC12 in [NP, NP + N)), and the epilogue drains NP instead
// of N columns per accumulator.
__host__ __device__ constexpr int set_cols(int N, int NP) { return merged_acc(N) ? NP + N : 3 * N; }
__host__ __device__ constexpr int set_cols(int N) { return set_cols(N, N); }
__host__ __device__ constexpr int acc_bufs_fit(int N) {
  return 512 / set_cols(N) >= 4 ? 4 : 512 / set_cols(N);
}
// MMA issuer warps: two (alternate units, each with its own X ring and its
// own accumulator sets) whenever two or more sets fit; an even set count then.
__host__ __device__ constexpr int mma_issuers(int N) { return acc_bufs_fit(N) >= 2 ? 2 : 1; }
__host__ __device__ constexpr int acc_bufs(int N) {
  return mma_issuers(N) == 2 ? (acc_bufs_fit(N) & ~1) : 1;
}

// Bits of F_lo's integer slice T0 (|T0| <= 2^t) that keep ACC0 = sum S0*T0
// over a unit's 64 G products exact in fp32: 2^11 * 2^t * 64 G <= 2^24.
__host__ __device__ constexpr int t_bits(int G) {
  return G <= 1 ? 7 : (G <= 2 ? 6 : (G <= 4 ? 5 : 4));
}

// The B operand (W slices) of one 64-wide l block, virtual rows
// [T0 | T1 | T2 | Fh] (Fh = F_lo rounded to fp16, the operand of S1).  Per K
// step the MMAs read contiguous row ranges of it:
//   N <= 85: S0 x [T0|T1|T2] (rows [0, 3N)), S1 x Fh ([3N, 4N))
//   N >  85: S0 x [T0|T1] ([0, 2NP): NP rows each), S0 x T2 (N rows), S1 x Fh (N rows)
// For a CTA pair each MMA's N' rows are split in halves between the CTAs
// (the leader's descriptor addresses both CTAs' shared memory at the same
// offset), so CTA c stores the c-th half of every range, ranges in order:
// w_rows / CG rows per CTA and l block.  Returns CTA and row of virtual row v.
__host__ __device__ constexpr int w_ranges(int N) { return merged_acc(N) ? 3 : 2; }
__host__ __device__ constexpr int w_range_begin(int N, int NP, int k) {
  return merged_acc(N) ? (k == 0 ? 0 : (k == 1 ? 2 * NP : 2 * NP + N)) : (k == 0 ? 0 : 3 * N);
}
__host__ __device__ constexpr int w_range_end(int N, int NP, int k) {
  return merged_acc(N) ? (k == 0 ? 2 * NP : (k == 1 ? 2 * NP + N : 2 * NP + 2 * N)) : (k == 0 ? 3 * N : 4 * N);
}
__host__ __device__ constexpr int w_rows(int N, int NP) { return merged_acc(N) ? 2 * NP + 2 * N : 4 * N; }
// virtual row of column n of slice sl (0..3 = T0, T1, T2, Fh); -1: not stored
// (a padding column of a packed range)
__host__ __device__ constexpr int w_virtual_row(int N, int NP, int sl, int n) {
  return !merged_acc(N) ? sl * N + n
                        : (sl < 2 ? (n < NP ? sl * NP + n : -1) : (sl == 2 ? 2 * NP + n : 2 * NP + N + n));
}
__host__ __device__ inline void w_row_slot(int N, int NP, int CG, int v, int& cta, int& row) {
  int off = 0;
  for (int k = 0; k < w_ranges(N); ++k) {
    const int b = w_range_begin(N, NP, k), e = w_range_end(N, NP, k), h = (e - b) / CG;
    if (v < e) {
      cta = (v - b) / h;
      row = off + (v - b) - cta * h;
      return;
    }
    off += h;
  }
  cta = 0;
  row = 0;
}

__host__ __device__ constexpr uint32_t tmem_cols(int N) {
  return acc_bufs(N) * set_cols(N) <= 32    ? 32
         : acc_bufs(N) * set_cols(N) <= 64  ? 64
         : acc_bufs(N) * set_cols(N) <= 128 ? 128
         : acc_bufs(N) * set_cols(N) <= 256 ? 256
                                      : 512;
}

struct TcParams {
  // CTA pairs: tensor maps over the image (rows of 128 B; box = one full /
  // one last l block of an m-tile) and over the W slices (box = one l block
  // of one CTA), so each CTA's loads complete on the pair leader's barriers
  CUtensorMap map_full, map_tail, map_w;
  const unsigned char* img;  // this mode's block image of the split tensor (see tc_tensor_create)
  int64_t tile_bytes;        // bytes of one full m-tile in the image
  int r8_full, r8_tail;      // stored rows (multiple of 8) of a full / the ragged last m-tile
  int ct;                    // 8-element chunks of the last l block (8 when l_ext % 64 == 0)
  int mode, R;
  int64_t M;
  int l_ext, n_o, n_lb, G;   // l extent, o extent, 64-wide l blocks, blocks per unit
  int n_full, splits, splits_tail;
  int tm;                    // rows per m-tile (<= 128; MMA M is 128, rows >= tm ignored)
  int x_stages, h_stages;
  int slot_ks;               // K steps (16 l values) per X ring slot
  int stage_bytes;           // X ring slot stride (slot_ks * 64 * r8_full bytes, 128 B aligned)
  const float2* hpair;       // [n_o][N/2] float4 {hi(n), hi(n+1), lo(n), lo(n+1)}, n even: F_hi[o, n] * 2^-e(n)
                             // as fp32 (hi, lo) pairs, packed by column pair for the f32x2 epilogue
  const unsigned char* wsl;  // [CG][n_lb][w_rows / CG][128 B] W slices of F_lo (w_slice_kernel)
  const double* cm_hi;       // [R] max |F_hi[:, n]| (kept current by the row update)
  const double* cm_lo;       // [R] max |F_lo[:, n]|
  const double* xscale;      // tensor split scale (device scalar)
  double* cm_self;           // [R] this mode's column maxima: zeroed here, re-accumulated
                             // by the row update that follows (NULL: untouched)
  double* ws;                // [splits][M][R] partials
  const int* stop_flag;
  int debug;                 // NTF_DIAG builds only (NTF_TC_DEBUG): 2 skip MMA, 4 skip TMEM
                             // drain, 16 skip X loads, 32 per-role wait cycles,
                             // 64 plain arrives for commits, 128 skip W slicing,
                             // 256 per-CTA globaltimer stamps, 2048 sleeping waits
  unsigned long long* times;  // NTF_TC_DEBUG & 256: per-CTA globaltimer stamps [8]
  int n_tiles;                // m-tiles (CG = 2: even, every tile stored with r8_full rows)
  uint32_t ub_full[kTcMaxSplits + 1];  // unit range of each CTA of a full tile
  uint32_t ub_tail[kTcMaxSplits + 1];  // ... of the ragged last tile
};

// ring slot + phase, advanced without divisions
struct Ring {
  int idx = 0;
  uint32_t phase = 0;
  __device__ __forceinline__ void next(int n) {
    if (++idx == n) {
      idx = 0;
      phase ^= 1u;
    }
  }
};

// unit (g, o) walk in g-major order
struct UnitIt {
  int g, o;
  __device__ __forceinline__ void next(int n_o) {
    if (++o == n_o) {
      o = 0;
      ++g;
    }
  }
};

// Packed fp32 pairs (f32x2: FFMA2 / FADD2 / FMUL2 on sm_100a): the epilogue
// treats two adjacent accumulator columns per instruction.  Every operation is
// an explicitly rounded PTX instruction, so the error-free transformations
// below stay exact (no contraction across them).
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 f2pack(float lo_col, float hi_col) {
  f32x2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo_col), "f"(hi_col));
  return r;
}
__device__ __forceinline__ void f2unpack(f32x2 v, float& lo_col, float& hi_col) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo_col), "=f"(hi_col) : "l"(v));
}
__device__ __forceinline__ f32x2 f2mul(f32x2 a, f32x2 b) {
  f32x2 r;
  asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f32x2 f2fma(f32x2 a, f32x2 b, f32x2 c) {
  f32x2 r;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ f32x2 f2add(f32x2 a, f32x2 b) {
  f32x2 r;
  asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f32x2 f2sub(f32x2 a, f32x2 b) {
  f32x2 r;
  asm volatile("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f32x2 f2neg(f32x2 a) { return a ^ 0x8000000080000000ull; }

// (hi, lo) += p exactly (Knuth TwoSum), on both lanes
__device__ __forceinline__ void two_sum2(f32x2& hi, f32x2& lo, f32x2 p) {
  const f32x2 s = f2add(hi, p);
  const f32x2 bp = f2sub(s, hi);
  lo = f2add(lo, f2add(f2sub(hi, f2sub(s, bp)), f2sub(p, bp)));
  hi = s;
}

// N / 16; CTAs per MMA group (1, or 2: a CTA pair with M = 256); packed T0 / T1 ranges (R <= N - 8)
template <int NT, int CG, int PK = 0>
__global__ void __launch_bounds__(tc_threads(NT), 1) mttkrp_tc_kernel(const __grid_constant__ TcParams p) {
  constexpr int N = NT * 16;
  constexpr int NP = N - 8 * PK;           // columns of ACC0 and of the T0 / T1 ranges (see set_cols)
  static_assert(PK == 0 || merged_acc(N), "packed ranges exist for merged accumulator sets only");
  constexpr int kEpi = epi_warps(NT);
  constexpr int NC = NP * 4 / kEpi;        // columns per epilogue thread
  // TMEM load width: 16 columns where it divides NC and registers allow
// 8-column TMEM loads up to 64 columns per thread (c5, N = 112 over 8 warps:
// drain alone 3.03 vs 3.25 ms per mode with 4-column loads)
#ifndef NTF_LW_WIDE
#define NTF_LW_WIDE 64
#endif
  constexpr int LW = (NC % 16 == 0 && NC <= 32 && kEpi < 16) ? 16 : ((NC > NTF_LW_WIDE || NC % 4) ? 4 : 8);
  constexpr int LT = NC % LW;              // a last, narrower load (packed ranges: 52 = 6 x 8 + 4)
  static_assert(LT == 0 || LT == 4, "epilogue columns must be a multiple of 4");
#ifndef NTF_PK_COLLECT
#define NTF_PK_COLLECT 1
#endif
  // Packed pair kernel: ONE issuer (its MMAs are long enough, 104 + 56 + 56
  // cycles per K step, for a single thread to keep the pipe fed) on both
  // accumulator sets, so the S0 operand of a K step's first MMA can stay in
  // the collector for the second (tc_mma_f16 COLL) instead of being read from
  // shared memory again.
  constexpr bool kCollect = PK != 0 && CG == 2 && NTF_PK_COLLECT != 0;
  constexpr int kAccBufs = kCollect ? 2 : acc_bufs(N);
  constexpr int kIssuers = kCollect ? 1 : mma_issuers(N);
  const int kXStage = p.stage_bytes;       // one X slot (slot_ks K steps of both planes), 128 B aligned
  constexpr int kWrows = w_rows(N, NP) / CG;  // W rows of one l block held by this CTA
  constexpr int kWlb = kWrows * kBK * 2;   // their bytes
  constexpr int kFirstEpi = 4;
  const uint64_t g_entry = gtimer();
  pdl_trigger();
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1 KB alignment by offset (keeps the pointer in the shared address space)
  unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int SX = p.x_stages, SH = p.h_stages, G = p.G;
  const int R = p.R;
  // [W slices of a group (SW128, 1 KB aligned)][F_hi pair ring][X ring][barriers]
  unsigned char* wbase = base;
  float2* hbase = reinterpret_cast<float2*>(wbase + G * kWlb);  // [SH][N]
  unsigned char* xbase = reinterpret_cast<unsigned char*>(hbase + SH * N);  // 128 B aligned (N % 16 == 0)
  uint64_t* x_full = reinterpret_cast<uint64_t*>(xbase + SX * kXStage);
  uint64_t* x_empty = x_full + SX;
  uint64_t* h_full = x_empty + SX;
  uint64_t* h_empty = h_full + SH;
  uint64_t* w_full = h_empty + SH;
  uint64_t* w_empty = w_full + 1;
  uint64_t* acc_full = w_empty + 1;
  uint64_t* acc_empty = acc_full + 4;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 4);
  uint32_t* stop_slot = tmem_slot + 1;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t crank = CG == 2 ? cluster_ctarank() : 0;  // 0: the pair's leader (issues the MMAs)
  const bool leader = crank == 0;
  // this CTA's tile and unit range (a pair: consecutive tiles, one unit range)
  int tile, split;
  const uint32_t* ub;
  if constexpr (CG == 2) {
    const int pair = blockIdx.x / 2, n_tp = p.n_tiles / 2;
    tile = (pair % n_tp) * 2 + static_cast<int>(crank);
    split = pair / n_tp;
    ub = p.ub_full;
  } else if (static_cast<int>(blockIdx.x) < p.n_full * p.splits) {
    tile = blockIdx.x % p.n_full;
    split = blockIdx.x / p.n_full;
    ub = p.ub_full;
  } else {
    tile = p.n_full;
    split = blockIdx.x - p.n_full * p.splits;
    ub = p.ub_tail;
  }
  const int64_t m0 = static_cast<int64_t>(tile) * p.tm;
  const int u_begin = static_cast<int>(ub[split]);
  const int u_end = static_cast<int>(ub[split + 1]);
  const int n_o = p.n_o;
  const UnitIt u0{u_begin / n_o, u_begin - (u_begin / n_o) * n_o};
  auto lbs_of = [&](int g) { return min(G, p.n_lb - g * G); };

  if (threadIdx.x == 0) {
    // A pair's loads (both CTAs' X blocks and W halves) complete on the
    // leader's x_full / w_full; the leader's commits reach x_empty / w_empty
    // / acc_full in both CTAs (multicast); the peer's x_empty has no second
    // issuer, so it counts the owner's commit only.
    for (int s = 0; s < SX; ++s) {
      mbar_init(&x_full[s], 1);
      mbar_init(&x_empty[s], leader ? kIssuers : 1);  // owner's MMA commit (+ the other issuer's arrive)
    }
    for (int s = 0; s < SH; ++s) {
      mbar_init(&h_full[s], 1);
      mbar_init(&h_empty[s], kEpi);
    }
    mbar_init(w_full, 1);
    mbar_init(w_empty, kIssuers);  // one commit per MMA issuer
    for (int s = 0; s < kAccBufs; ++s) {
      mbar_init(&acc_full[s], 1);
      mbar_init(&acc_empty[s], kEpi * CG);  // both CTAs' epilogue warps (the peer's remotely)
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    // stop decision: the leader's read of the flag, so both CTAs of a pair agree
    if (leader) {
      const uint32_t stop = (p.stop_flag && *reinterpret_cast<const volatile int*>(p.stop_flag)) ? 1u : 0u;
      *stop_slot = stop;
      if constexpr (CG == 2) st_cluster_u32(stop_slot, 1, stop);
    }
  }
  if (warp == 1) {
    if constexpr (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                       smem_u32(tmem_slot)),
                   "r"(tmem_cols(N)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                       smem_u32(tmem_slot)),
                   "r"(tmem_cols(N)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
    }
  }
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync_all();  // barriers initialised and the stop word delivered pair-wide
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const bool stopped = *reinterpret_cast<volatile uint32_t*>(stop_slot) != 0;
  // Diagnostic flags.  The host fills p.debug only in NTF_DIAG builds
  // (diag_env), so in a release library it is always 0 and no environment
  // setting changes what this kernel does.  For CTA pairs the flags are a
  // compile-time 0 and every branch folds away.  Single CTAs keep the runtime
  // (always-false) tests: that codegen (130 vs 116 registers) measured 12%
  // faster per outer iteration at c2 under PDL (1.755 vs 2.003 ms/step,
  // identical kernel durations with PDL off, tools/step_time.py); presumably the larger
  // register footprint keeps other kernels' early blocks off the MTTKRP's
  // SMs (not verified).
  const int dbg = (kDiagBuild || CG == 1) ? p.debug : 0;
  const bool prof = (dbg & 32) != 0;
  const int wm = (prof ? 1 : 0) | ((dbg & 2048) ? 2 : 0);
  const uint64_t g_ready = (prof || (dbg & 256)) ? gtimer() : 0;
  long long wt[3] = {0, 0, 0};
  const long long t_start = prof ? clock64() : 0;
  uint64_t t_role = 0;  // NTF_TC_DEBUG & 256: end of this role's loop
  uint32_t x_kb = 0;     // ... and the bytes this CTA streamed (KiB)

  // Roles 0-2: warp-uniform loops (descriptors and barrier addresses stay in
  // uniform registers); one elected lane issues.
  // This CTA's m-tile in the image: stored rows, block sizes and the byte
  // offset of its first unit.  A CTA's units are consecutive (g-major) and
  // the image stores them consecutively, so the CTA streams ONE contiguous
  // byte range, block after block.
  const int r8 = tile < p.n_full ? p.r8_full : p.r8_tail;
  const uint32_t blk_full = 256u * static_cast<uint32_t>(r8);  // 2 planes x 8 chunks x r8 x 16 B
  const uint32_t blk_tail = 32u * static_cast<uint32_t>(p.ct * r8);
  // A block is 4 (the last l block: ct / 2) K steps of 64 * r8 bytes each
  // ([plane][2 chunks][r8 rows][16 B]); the X ring moves slot_ks of them per slot.
  const uint32_t ks_bytes = 64u * static_cast<uint32_t>(r8);
  const int slot_ks = p.slot_ks;
  if (stopped) {
    // converged earlier: nothing to compute (the row update skips as well)
  } else if (warp == 0) {
    // ------------------------------ X-block producer --------------------------
    const bool no_x = (dbg & 16) != 0;
    const int n_lb = p.n_lb;
    int64_t off = static_cast<int64_t>(tile) * p.tile_bytes +
                  static_cast<int64_t>(u0.g) * n_o * G * blk_full;
    {  // units (u0.g, 0 .. u0.o - 1) of the first group precede this CTA's range
      const int nl = lbs_of(u0.g);
      const bool has_tail = u0.g * G + nl == n_lb;
      const int64_t unit_bytes = has_tail ? (nl - 1) * int64_t(blk_full) + blk_tail : nl * int64_t(blk_full);
      off += static_cast<int64_t>(u0.o) * unit_bytes;
    }
    // One X ring in stream order.  With two issuers a slot is released
    // when BOTH have passed it (x_empty counts 2: the owner's commit after its
    // MMAs, the other issuer's arrive after observing the load), so neither
    // can fall a full ring behind and every parity wait stays unambiguous.
    // A pair's peer CTA fills its own ring the same way; the leader's
    // commits and arrivals reach its x_empty too.
    Ring xr;
    UnitIt ui = u0;
    const int64_t off0 = off;
    for (int u = u_begin; u < u_end; ++u) {
      const int nl = lbs_of(ui.g);
      for (int j = 0; j < nl; ++j) {
        const bool last_lb = ui.g * G + j == n_lb - 1;
        const int nks = last_lb ? p.ct / 2 : kBK / kUK;
        for (int k0 = 0; k0 < nks; k0 += slot_ks) {
          mbar_wait_p(&x_empty[xr.idx], xr.phase ^ 1u, wm, wt[0]);
          uint64_t* bar = &x_full[xr.idx];
          const uint32_t bytes = static_cast<uint32_t>(min(slot_ks, nks - k0)) * ks_bytes;
          if (elect_one()) {
            if constexpr (CG == 2) {
              // both CTAs' blocks count on the leader's barrier (slot_ks = 4: one
              // block per slot, one tensor-map load of 2 r8 rows of 128 B)
              if (no_x) {
                if (leader) mbar_arrive(bar);
              } else {
                if (leader) mbar_arrive_expect_tx(bar, 2 * bytes);
                tma_load_2sm(xbase + xr.idx * kXStage, last_lb ? &p.map_tail : &p.map_full, 0,
                             static_cast<int32_t>(off >> 7), mapa_u32(smem_u32(bar), 0));
              }
            } else if (no_x) {
              mbar_arrive(bar);
            } else {
              mbar_arrive_expect_tx(bar, bytes);
              bulk_load(xbase + xr.idx * kXStage, p.img + off, bytes, bar);
            }
          }
          __syncwarp();
          off += bytes;
          xr.next(SX);
        }
      }
      ui.next(n_o);
    }
    t_role = gtimer();
    x_kb = static_cast<uint32_t>((off - off0) >> 10);
  } else if ((warp == 1 || warp == 3) && !leader) {
    // CTA pair, peer: the leader issues every MMA of the pair
  } else if (warp == 1 || warp == 3) {
    // ------------------------------ MMA issuers --------------------------------
   if (warp == 1 || kIssuers == 2) {  // warp 3 idles when one accumulator set fits
    // Per K step (W rows: see w_row_slot):
    //   N <= 85: [ACC0|ACC1|ACC2] (=|+=) S0 x [T0|T1|T2];  ACC1 += S1 x Fh
    //   N >  85: [ACC0|ACC12] (=|+=) S0 x [T0|T1];  ACC12 += S0 x T2;  ACC12 += S1 x Fh
    // A (one K step of the X block) is a no-swizzle K-major image: 8-row x
    // 16 B core matrices, row groups 128 B apart (SBO), the step's two
    // 8-element chunks r8*16 B apart (LBO); plane S1 follows plane S0.
    const bool no_mma = (dbg & 2) != 0, plain_arrive = (dbg & 64) != 0;
    constexpr bool kMerged = merged_acc(N);
    const uint32_t idesc_a = make_idesc(kMerged ? 2 * NP : 3 * N, false, CG);
    const uint32_t idesc_n = make_idesc(N, false, CG);
    // B operand offsets (rows of this CTA's W block, descriptor units of 16 B)
    constexpr uint64_t kB1 = ((w_range_end(N, NP, 0) - w_range_begin(N, NP, 0)) / CG) * 128 / 16;
    constexpr uint64_t kB2 = kMerged ? kB1 + (N / CG) * 128 / 16 : kB1;
    const uint32_t lbo = static_cast<uint32_t>(r8) * 16u;
    const uint64_t da_base = smem_desc_noswz(xbase, lbo, 128);
    const uint64_t db_base = smem_desc(wbase, 16, 1024);
    const uint32_t a_plane = (2 * lbo) >> 4;  // descriptor units (16 B): plane S1 of a K step
    const uint32_t a_kstep = ks_bytes >> 4;   // next K step within a slot
    const int n_lb = p.n_lb, ct = p.ct;
    // Issuer warps take alternate units, each with its own accumulator sets
    // (set b serves units u with u % kAccBufs == b, an even count), and both
    // walk the shared X ring in order (see the producer).  A single issuing
    // thread is bound by the per-instruction issue latency of small-N MMAs.
    const int mine = warp == 1 ? 0 : 1;
    Ring xr, ar;
    UnitIt ui = u0;
    int cur_g = -1;
    uint32_t wphase = 0;
    auto wait_slot = [&](int slot, uint32_t phase) { mbar_wait_p(&x_full[slot], phase, wm, wt[0]); };
    for (int u = u_begin; u < u_end; ++u) {
      if (ui.g != cur_g) {  // new group: its W slices must be resident (both halves)
        if (cur_g >= 0) {
          if (elect_one()) tc_commit<CG>(w_empty);
          __syncwarp();
        }
        mbar_wait_p(w_full, wphase, wm, wt[2]);
        wphase ^= 1u;
        cur_g = ui.g;
      }
      const int nl = lbs_of(ui.g);
      const int owner = kIssuers == 2 ? ((u - u_begin) & 1) : 0;
      if (owner != mine) {  // the other issuer's unit: observe and release its X slots
        for (int j = 0; j < nl; ++j) {
          const int nks = (ui.g * G + j == n_lb - 1) ? ct / 2 : kBK / kUK;
          for (int k0 = 0; k0 < nks; k0 += slot_ks) {
            wait_slot(xr.idx, xr.phase);
            if (elect_one()) mbar_arrive(&x_empty[xr.idx]);
            __syncwarp();
            xr.next(SX);
          }
        }
        ar.next(kAccBufs);
        ui.next(n_o);
        continue;
      }
      mbar_wait_p(&acc_empty[ar.idx], ar.phase ^ 1u, wm, wt[1]);  // (a pair: both CTAs drained)
      tc_fence_after();
      const uint32_t d0 = tmem + ar.idx * set_cols(N, NP);
      const uint32_t d1 = d0 + NP;
      for (int j = 0; j < nl; ++j) {
        const int nks = (ui.g * G + j == n_lb - 1) ? ct / 2 : kBK / kUK;
        const uint64_t db = db_base + static_cast<uint64_t>((j * kWlb) >> 4);
        for (int k0 = 0; k0 < nks; k0 += slot_ks) {
          const int slot = xr.idx;
          const int nk = min(slot_ks, nks - k0);
          wait_slot(slot, xr.phase);
          tc_fence_after();
          const uint64_t da = da_base + static_cast<uint64_t>((slot * kXStage) >> 4);
          if (elect_one()) {
            if (!no_mma) {
              for (int kk = 0; kk < nk; ++kk) {
                const int ks = k0 + kk;  // K step within the l block
                const uint32_t first = (j | ks) ? 1u : 0u;
                const uint64_t a0 = da + kk * a_kstep, a1 = a0 + a_plane;
                const uint64_t b = db + ks * (32 >> 4);
                if constexpr (kCollect) {
                  tc_mma_f16<CG, 1>(d0, a0, b, idesc_a, first);
                  tc_mma_f16<CG, 2>(d1, a0, b + kB1, idesc_n, 1u);
                } else {
                  tc_mma_f16<CG>(d0, a0, b, idesc_a, first);
                  if constexpr (kMerged) tc_mma_f16<CG>(d1, a0, b + kB1, idesc_n, 1u);
                }
                tc_mma_f16<CG>(d1, a1, b + kB2, idesc_n, 1u);
              }
            }
            if (plain_arrive) mbar_arrive(&x_empty[slot]);  // profiling: no tensor-pipe commit
            else tc_commit<CG>(&x_empty[slot]);
          }
          __syncwarp();
          xr.next(SX);
        }
      }
      if (elect_one()) {
        if (plain_arrive) mbar_arrive(&acc_full[ar.idx]);
        else tc_commit<CG>(&acc_full[ar.idx]);
      }
      __syncwarp();
      ar.next(kAccBufs);
      ui.next(n_o);
    }
    t_role = gtimer();
   }
  } else if (warp == 2) {
    // ------- W slices of each group + F_hi pair rows (bulk copies, many in flight) -------
    // Everything from here on reads what the preceding kernels produced
    // (w_slice_kernel formed both the W slices and the F_hi pair table).
    pdl_wait();
    // this mode's column maxima are re-accumulated by the row update that follows
    if (blockIdx.x == 0 && p.cm_self)
      for (int n = lane; n < R; n += 32) p.cm_self[n] = 0.0;
    __syncwarp();
    const unsigned char* wsl = p.wsl + static_cast<int64_t>(crank) * p.n_lb * kWlb;  // this CTA's W half
    Ring hr;
    UnitIt ui = u0;
    int seg = 0;
    for (int u = u_begin; u < u_end; ++u) {
      if (u == u_begin || ui.o == 0) {  // group start: the previous group's MMAs are done
        if (seg > 0) mbar_wait_p(w_empty, (seg - 1) & 1, wm, wt[2]);
        if (elect_one()) {
          const int nl = lbs_of(ui.g);
          const uint32_t bytes = static_cast<uint32_t>(nl * kWlb);
          if constexpr (CG == 2) {  // one tensor-map load per l block; both halves count on the leader
            if (leader) mbar_arrive_expect_tx(w_full, 2 * bytes);
            const uint32_t wbar = mapa_u32(smem_u32(w_full), 0);
            for (int j = 0; j < nl; ++j)
              tma_load_2sm(wbase + j * kWlb, &p.map_w, 0,
                           static_cast<int32_t>((crank * p.n_lb + ui.g * G + j) * kWrows), wbar);
          } else {
            mbar_arrive_expect_tx(w_full, bytes);
            bulk_load(wbase, wsl + static_cast<int64_t>(ui.g) * G * kWlb, bytes, w_full);
          }
        }
        __syncwarp();
        ++seg;
      }
      mbar_wait_p(&h_empty[hr.idx], hr.phase ^ 1u, wm, wt[0]);
      if (elect_one()) {
        mbar_arrive_expect_tx(&h_full[hr.idx], N * 8);
        bulk_load(hbase + hr.idx * N, p.hpair + static_cast<int64_t>(ui.o) * N, N * 8, &h_full[hr.idx]);
      }
      __syncwarp();
      hr.next(SH);
      ui.next(n_o);
    }
    t_role = gtimer();
  } else if (warp >= kFirstEpi) {
    // ------------------------------ epilogue ----------------------------------
    const int e = warp - kFirstEpi;
    const int q4 = warp & 3;            // TMEM lane quarter of this warp
    const int c0 = (e >> 2) * NC;       // this warp's column range
    const int row = q4 * 32 + lane;     // tile row == TMEM lane
    f32x2 hi[NC / 2], lo[NC / 2];       // double-float accumulators, column pairs
    const f32x2 kT2Unscale = f2pack(0x1p-11f, 0x1p-11f);
#pragma unroll
    for (int j = 0; j < NC / 2; ++j) {
      hi[j] = 0ull;
      lo[j] = 0ull;
    }
    // Per-column output scale xs * 2^(f-t) * 2^e, with max|F_lo[:,n]| < 2^f,
    // max|F_hi[:,n]| < 2^e (the clamps of w_slice_kernel).  Formed here, one
    // column per thread, while the first unit's loads are in flight (off the
    // kernel's tail), after this thread's own wait on the preceding kernel (a
    // CTA with no unit never synchronises with the W-loading warp).
    double* sc = reinterpret_cast<double*>(tmem_slot + 2);  // [N], 8-byte aligned after the two slot words
    pdl_wait();
    {
      const int n = static_cast<int>(threadIdx.x) - kFirstEpi * 32;
      if (n < N) {
        double s = 0.0;
        if (n < R) {
          int f = 0, e2 = 0;
          const double cl = p.cm_lo[n], ch = p.cm_hi[n];
          if (cl > 0.0) frexp(cl, &f);
          if (ch > 0.0) frexp(ch, &e2);
          // columns decayed to ~1e-300 (large penalties shrink factor columns
          // geometrically) must not overflow the scales: clamp as the slicer (kFMin)
          s = *p.xscale * ldexp(1.0, max(f, kFMin) - t_bits(G) + max(e2, kFMin));
        }
        sc[n] = s;
      }
    }
    asm volatile("bar.sync 1, %0;\n" ::"r"(kEpi * 32) : "memory");
    Ring ar, hr;
    for (int u = u_begin; u < u_end; ++u) {
      mbar_wait_p(&acc_full[ar.idx], ar.phase, wm, wt[0]);
      mbar_wait_p(&h_full[hr.idx], hr.phase, wm, wt[1]);
      tc_fence_after();
      const uint32_t taddr = tmem + (static_cast<uint32_t>(q4 * 32) << 16) + ar.idx * set_cols(N, NP) + c0;
      const float4* hs = reinterpret_cast<const float4*>(hbase + hr.idx * N + c0);
      // W columns [off, off + W) of this thread's range: ACC0 (S0*T0, exact
      // integers), ACC1 (S0*T1 + S1*Fh, + ACC2's terms when merged), ACC2 (S0*T2)
      auto drain = [&](auto wtag, const int off) {
        constexpr int W = decltype(wtag)::value;
        float a0[W], a1[W], a2[W];
        tmem_ld<W>(taddr + off, a0);
        tmem_ld<W>(taddr + NP + off, a1);
        if constexpr (!merged_acc(N)) tmem_ld<W>(taddr + 2 * N + off, a2);
        tmem_wait_ld();
#pragma unroll
        for (int v = 0; v < W; v += 2) {
          const float4 h = hs[(off + v) >> 1];  // {hi, hi', lo, lo'} of columns v, v+1
          const f32x2 hx = f2pack(h.x, h.y), hy = f2pack(h.z, h.w);
          const f32x2 a = f2pack(a0[v], a0[v + 1]);
          f32x2 a12 = f2pack(a1[v], a1[v + 1]);
          // ACC2 = S0 x (T2 2^11): scaled back here (exact power of two)
          if constexpr (!merged_acc(N)) a12 = f2fma(f2pack(a2[v], a2[v + 1]), kT2Unscale, a12);
          const f32x2 pr = f2mul(a, hx);
          const f32x2 er = f2fma(a, hx, f2neg(pr));  // a*hx = pr + er exactly
          const f32x2 cr = f2fma(a12, hx, f2fma(a, hy, er));
          const int q = (off + v) >> 1;
          two_sum2(hi[q], lo[q], pr);
          lo[q] = f2add(lo[q], cr);
        }
      };
      if (!(dbg & 4)) {
#pragma unroll
        for (int j = 0; j < NC / LW; ++j) drain(std::integral_constant<int, LW>{}, j * LW);
        if constexpr (LT != 0) drain(std::integral_constant<int, LT>{}, (NC / LW) * LW);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (leader) mbar_arrive(&acc_empty[ar.idx]);
        else mbar_arrive_remote(&acc_empty[ar.idx], 0);  // the peer's TMEM reads are done
        mbar_arrive(&h_empty[hr.idx]);
      }
      ar.next(kAccBufs);
      hr.next(SH);
    }
    t_role = gtimer();
    // fp64 partial of this CTA: out = (hi + lo) * xs * 2^(f-t) * 2^e.  The
    // tile's rows are one contiguous range of the partial buffer: staged
    // row-major in the (now idle) X ring, then written with coalesced stores
    // (a thread's own row is R doubles apart from its neighbours').
    const int rows_valid = static_cast<int>(p.M - m0 < p.tm ? p.M - m0 : p.tm);
    double* out0 = p.ws + (static_cast<int64_t>(split) * p.M + m0) * R;
    float hf[NC], lf[NC];
#pragma unroll
    for (int j = 0; j < NC / 2; ++j) {
      f2unpack(hi[j], hf[2 * j], hf[2 * j + 1]);
      f2unpack(lo[j], lf[2 * j], lf[2 * j + 1]);
    }
    if (p.tm * R * 8 <= SX * kXStage) {
      double* stage = reinterpret_cast<double*>(xbase);
      if (row < rows_valid) {
#pragma unroll
        for (int j = 0; j < NC; ++j) {
          const int n = c0 + j;
          if (n < R)
            stage[row * R + n] = (static_cast<double>(hf[j]) + static_cast<double>(lf[j])) * sc[n];
        }
      }
      asm volatile("bar.sync 1, %0;\n" ::"r"(kEpi * 32) : "memory");
      const int total = rows_valid * R;
      for (int i = threadIdx.x - kFirstEpi * 32; i < total; i += kEpi * 32) out0[i] = stage[i];
    } else if (row < rows_valid) {
      double* out = out0 + static_cast<int64_t>(row) * R;
#pragma unroll
      for (int j = 0; j < NC; ++j) {
        const int n = c0 + j;
        if (n < R)
          out[n] = (static_cast<double>(hf[j]) + static_cast<double>(lf[j])) * sc[n];
      }
    }
  }
  if (prof && lane == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1) && warp <= 4)
    printf("tc cta %d warp %d units %d loop %lld wait %lld %lld %lld gt %llu %llu %llu\n", blockIdx.x,
           warp, u_end - u_begin, clock64() - t_start, wt[0], wt[1], wt[2],
           (unsigned long long)g_entry, (unsigned long long)(g_ready - g_entry),
           (unsigned long long)(gtimer() - g_entry));
  if ((dbg & 256) && lane == 0 && warp <= 3) {
    unsigned long long* ts = p.times + static_cast<int64_t>(blockIdx.x) * 8;
    ts[2 + warp] = t_role;
    if (warp == 0) {
      ts[0] = g_entry;
      ts[1] = g_ready;
      uint32_t smid;
      asm volatile("mov.u32 %0, %%smid;\n" : "=r"(smid));
      ts[7] = static_cast<unsigned long long>(u_end - u_begin) | (static_cast<unsigned long long>(smid) << 16) |
              (static_cast<unsigned long long>(x_kb) << 32);
    }
  }
  // every MMA into this CTA's TMEM has completed (the epilogue saw its last
  // commit); a pair also waits for the peer before releasing the columns
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync_all();
  else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if constexpr (CG == 1)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(tmem_cols(N)));
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(tmem_cols(N)));
    if ((dbg & 256) && lane == 0) p.times[static_cast<int64_t>(blockIdx.x) * 8 + 6] = gtimer();
  }
}

// ----------------------------------------------------------------------------
// W slices of F_lo for every 64-row l block, in the UMMA K-major SW128 layout
// the MTTKRP CTAs bulk-copy into shared memory:
//   wsl[cta][lb][row][128 B],  element l of a row at ((l/8) ^ (row&7))*16 + (l%8)*2
// with the virtual rows [T0 | T1 | T2 | Fh] (N each) placed by w_row_slot:
//   v = F_lo[l, n] * 2^(t - f(n)) = T0 + T1 + T2 (+ <= 2^-23 rounding),
//   T0 integer (|T0| <= 2^t), T1 in 2^-11 units, T2 in 2^-22 units (fp16
//   exact, T2 possibly subnormal); Fh = fp16(v), the 11-bit operand of the
//   low tensor plane S1.  One thread per (l block, n, octet).
// ----------------------------------------------------------------------------
__global__ void w_slice_kernel(const double* __restrict__ F, int l_ext, int R, int N, int NP, int CG, int n_lb,
                               bool t2_scaled,
                               const double* __restrict__ cm, int t, unsigned char* __restrict__ wsl,
                               const double* __restrict__ Fhi, int n_o,
                               const double* __restrict__ cm_hi, float2* __restrict__ hpair,
                               const int* stop_flag) {
  pdl_trigger();
  pdl_wait();  // F_lo, F_hi and their column maxima come from the preceding row updates
  // (no stop-flag read here: it would add a dependent round trip to every
  // mode update, and slicing after a stop is harmless — the MTTKRP checks it)
  (void)stop_flag;
  // Work item e: the F_hi pair entry e (hpair[o][n] = F_hi[o, n] * 2^-e(n) as
  // an fp32 (hi, lo) pair, max|F_hi[:, n]| < 2^e(n)) and the 8-value W slice
  // chunk e of F_lo.  Every global load of a thread is issued before any
  // result is used, so the kernel costs one L2 round trip after the wait.
  const int64_t total_h = static_cast<int64_t>(n_o) * N;
  const int total_w = n_lb * N * (kBK / 8);
  const int64_t total = total_h > total_w ? total_h : total_w;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const bool do_h = e < total_h, do_w = e < total_w;
    const int n = static_cast<int>(e % N);  // column of both items
    const int64_t o = e / N;
    const int oc = static_cast<int>(o);
    const int lb = oc / (kBK / 8), oct = oc % (kBK / 8);
    const bool vh = do_h && n < R, vw = do_w && n < R;
    const double cmh = vh ? cm_hi[n] : 0.0;
    const double fh = vh ? Fhi[o * R + n] : 0.0;
    const double cml = vw ? cm[n] : 0.0;
    double x[8];
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      const int l = lb * kBK + oct * 8 + v;
      x[v] = (vw && l < l_ext) ? F[static_cast<int64_t>(l) * R + n] : 0.0;
    }
    if (do_h) {
      double h = 0.0;
      if (vh) {
        int ex = 0;
        if (cmh > 0.0) frexp(cmh, &ex);
        h = fh * ldexp(1.0, -max(ex, kFMin));
      }
      const float hx = static_cast<float>(h);
      float* hp = reinterpret_cast<float*>(hpair) + o * (2 * N) + (n >> 1) * 4 + (n & 1);
      hp[0] = hx;                                                   // packed by column pair:
      hp[2] = static_cast<float>(h - static_cast<double>(hx));      // {hi, hi', lo, lo'}
    }
    if (do_w) {
      double sc = 0.0;
      if (vw) {
        int f = 0;
        if (cml > 0.0) frexp(cml, &f);
        sc = ldexp(1.0, t + 22 - max(f, kFMin));  // v in 2^-22 units of the T0 scale
      }
      __align__(16) __half hs[4][8];
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        // v = F_lo * 2^(t-f), exact (a power-of-two scale); T0 = rint(v) is an
        // integer, |T0| <= 2^t (ACC0's exactness rests on it); the remainders
        // r1 = v - T0 and r2 = r1 - T1 are exact in fp64 and each rounded once
        // to fp16 (11 significant bits of the remainder itself, not of a fixed
        // 2^-11 grid): |v - (T0+T1+T2)| <= max(2^-12 |r2|, 2^-25) <= 2^-25.
        const double vv = x[v] * (sc * 0x1p-22);
        const double t0 = rint(vv);
        const double r1 = vv - t0;
        const __half h1 = __double2half(r1);
        const double r2 = r1 - static_cast<double>(__half2float(h1));
        hs[0][v] = __double2half(t0);
        hs[1][v] = h1;
        // N <= 85 (T2 in its own accumulator ACC2): T2 carries 2^11 r2, which
        // moves its fp16 subnormal floor from 2^-25 to 2^-36 (factor columns
        // with a few large entries and many small ones keep ~22 relative
        // bits in the small ones); the epilogue scales ACC2 back
        hs[2][v] = __double2half(t2_scaled ? r2 * 2048.0 : r2);
        hs[3][v] = __double2half(vv);  // Fh = fp16(v), the operand of the low plane S1
      }
      const int rows_cta = w_rows(N, NP) / CG;
#pragma unroll
      for (int sl = 0; sl < 4; ++sl) {
        int cta = 0, row = 0;
        const int vr = w_virtual_row(N, NP, sl, n);
        if (vr < 0) continue;  // a padding column (n >= R) of a packed range: not stored
        w_row_slot(N, NP, CG, vr, cta, row);
        unsigned char* wb = wsl + (static_cast<int64_t>(cta) * n_lb + lb) * rows_cta * 128;
        *reinterpret_cast<uint4*>(wb + row * 128 + ((oct ^ (row & 7)) << 4)) =
            *reinterpret_cast<const uint4*>(hs[sl]);
      }
    }
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

// One mode's block image of the split tensor.  For each m-tile t (r8
// stored rows, a multiple of 8; rows >= M are zero), each unit (g, o) in
// g-major order and each l block j of the unit, K step by K step:
//   [K step s < chunks(lb)/2][plane][chunk c < 2][row < r8][8 fp16]   (chunk = 8 l values)
// i.e. each K step is the no-swizzle K-major UMMA image of both planes, so
// one bulk copy moves any run of K steps into shared memory and a CTA's
// units are one contiguous byte range.
// The last l block stores only ct chunks (l_ext rounded up to 16).
// Values: X * 2^(11-e) = S0 + S1, S0 = rint (|S0| <= 2^11, exact in fp16),
// S1 = fp16 of the exact remainder (|S1| <= 1/2), xscale = 2^(e-11).
struct ImgGeom {
  int mode;
  int64_t I, J, K, M;
  int n_o, l_ext, n_lb, G, tm, n_full, n_tiles, r8_full, r8_tail, ct;
  int64_t tile_bytes;
};

__global__ void image_split_kernel(const float* __restrict__ X, ImgGeom g, const unsigned* amax,
                                   unsigned char* __restrict__ img, double* xscale) {
  const float mx = __uint_as_float(*amax);
  int ex = 0;
  if (mx > 0.f) frexpf(mx, &ex);            // mx < 2^ex
  const float up = ldexpf(1.0f, 11 - ex);   // X * 2^(11-ex) in [-2048, 2048]
  if (blockIdx.x == 0 && threadIdx.x == 0) *xscale = ldexp(1.0, ex - 11);
  const int64_t total = static_cast<int64_t>(g.n_tiles) * g.n_o * g.n_lb * 1024;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int row = static_cast<int>(e & 127);
    const int c = static_cast<int>((e >> 7) & 7);
    int64_t rest = e >> 10;
    const int lb = static_cast<int>(rest % g.n_lb);
    rest /= g.n_lb;
    const int o = static_cast<int>(rest % g.n_o);
    const int t = static_cast<int>(rest / g.n_o);
    const int r8 = t < g.n_full ? g.r8_full : g.r8_tail;
    const int chunks = lb == g.n_lb - 1 ? g.ct : 8;
    if (row >= r8 || c >= chunks) continue;
    const int64_t bf = 256 * static_cast<int64_t>(r8), bt = 32 * static_cast<int64_t>(g.ct) * r8;
    const int gi = lb / g.G, j = lb - gi * g.G;
    const int nl = min(g.G, g.n_lb - gi * g.G);
    const int64_t unit_bytes = (nl - 1) * bf + (gi * g.G + nl == g.n_lb ? bt : bf);
    const int64_t off = t * g.tile_bytes + static_cast<int64_t>(gi) * g.n_o * g.G * bf +
                        o * unit_bytes + j * bf + static_cast<int64_t>(c >> 1) * 64 * r8 +
                        static_cast<int64_t>(c & 1) * r8 * 16 + row * 16;
    const int64_t m = static_cast<int64_t>(t) * g.tm + row;
    const int l0 = lb * 64 + c * 8;
    __align__(16) __half h0[8], h1[8];
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      const int l = l0 + v;
      float x = 0.f;
      if (m < g.M && l < g.l_ext) {
        const int64_t idx = g.mode == 1 ? (m * g.J + o) * g.K + l
                            : g.mode == 2 ? (static_cast<int64_t>(o) * g.J + m) * g.K + l
                                          : (static_cast<int64_t>(o) * g.J + l) * g.K + m;
        x = X[idx];
      }
      const float sv = x * up;                // exact (power-of-two scaling)
      const float a0 = rintf(sv);             // S0: integer, |S0| <= 2^11
      h0[v] = __float2half_rn(a0);
      h1[v] = __float2half_rn(sv - a0);       // S1: the exact remainder in [-1/2, 1/2], rounded once to fp16
    }
    *reinterpret_cast<uint4*>(img + off) = *reinterpret_cast<const uint4*>(h0);
    *reinterpret_cast<uint4*>(img + off + 32 * static_cast<int64_t>(r8)) = *reinterpret_cast<const uint4*>(h1);
  }
}

// The same image for modes 1 and 2, where l = k is the tensor's contiguous
// index: a block stages 32 rows x one 64-wide l block of one (tile, o) through
// shared memory, so the tensor is read in 256-byte row pieces (the direct
// kernel above reads 32-byte pieces megabytes apart: 2.3 TB/s read + write)
// and the image is written as before, 16 bytes per (plane, chunk, row) with
// consecutive rows adjacent.
__global__ void __launch_bounds__(256) image_split_rows_kernel(const float* __restrict__ X, ImgGeom g,
                                                               const unsigned* amax,
                                                               unsigned char* __restrict__ img, double* xscale) {
  __shared__ float tile[32][65];
  const float mx = __uint_as_float(*amax);
  int ex = 0;
  if (mx > 0.f) frexpf(mx, &ex);
  const float up = ldexpf(1.0f, 11 - ex);
  if (blockIdx.x == 0 && threadIdx.x == 0) *xscale = ldexp(1.0, ex - 11);
  const int rg_per_tile = (g.r8_full + 31) / 32;  // 32-row groups per tile (the ragged tile may use fewer)
  const int64_t total = static_cast<int64_t>(g.n_tiles) * g.n_o * g.n_lb * rg_per_tile;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t b = blockIdx.x; b < total; b += gridDim.x) {
    const int rg = static_cast<int>(b % rg_per_tile);
    int64_t rest = b / rg_per_tile;
    const int lb = static_cast<int>(rest % g.n_lb);
    rest /= g.n_lb;
    const int o = static_cast<int>(rest % g.n_o);
    const int t = static_cast<int>(rest / g.n_o);
    const int r8 = t < g.n_full ? g.r8_full : g.r8_tail;
    const int chunks = lb == g.n_lb - 1 ? g.ct : 8;
    const int row0 = rg * 32;
    if (row0 < r8) {  // block-uniform
      // stage: warp w loads rows w, w + 8, ...; lanes along l (two floats each)
      const int l0 = lb * 64;
      for (int rr = warp; rr < 32; rr += 8) {
        const int64_t m = static_cast<int64_t>(t) * g.tm + row0 + rr;
        const float* src = g.mode == 1 ? X + (m * g.J + o) * g.K : X + (static_cast<int64_t>(o) * g.J + m) * g.K;
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int l = l0 + lane + 32 * u;
          tile[rr][lane + 32 * u] = (m < g.M && row0 + rr < r8 && l < g.l_ext) ? src[l] : 0.f;
        }
      }
    }
    __syncthreads();
    if (row0 < r8) {
      const int row = row0 + lane, c = warp;  // thread: one row, one chunk of 8 l values
      if (row < r8 && c < chunks) {
        const int64_t bf = 256 * static_cast<int64_t>(r8), bt = 32 * static_cast<int64_t>(g.ct) * r8;
        const int gi = lb / g.G, j = lb - gi * g.G;
        const int nl = min(g.G, g.n_lb - gi * g.G);
        const int64_t unit_bytes = (nl - 1) * bf + (gi * g.G + nl == g.n_lb ? bt : bf);
        const int64_t off = t * g.tile_bytes + static_cast<int64_t>(gi) * g.n_o * g.G * bf +
                            o * unit_bytes + j * bf + static_cast<int64_t>(c >> 1) * 64 * r8 +
                            static_cast<int64_t>(c & 1) * r8 * 16 + row * 16;
        __align__(16) __half h0[8], h1[8];
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          const float sv = tile[lane][c * 8 + v] * up;  // exact (power-of-two scaling)
          const float a0 = rintf(sv);
          h0[v] = __float2half_rn(a0);
          h1[v] = __float2half_rn(sv - a0);
        }
        *reinterpret_cast<uint4*>(img + off) = *reinterpret_cast<const uint4*>(h0);
        *reinterpret_cast<uint4*>(img + off + 32 * static_cast<int64_t>(r8)) = *reinterpret_cast<const uint4*>(h1);
      }
    }
    __syncthreads();
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

// NTF_TC_DEBUG & 256: per-CTA stamps of the last launch (diagnostics only)
constexpr int kTcTimesCtas = 1024;
__device__ unsigned long long g_tc_times[kTcTimesCtas * 8];

unsigned long long* tc_debug_times() {
  void* ptr = nullptr;
  cudaGetSymbolAddress(&ptr, g_tc_times);
  return static_cast<unsigned long long*>(ptr);
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

template <int NT, int CG, int PK = 0>
cudaError_t launch_nt(const TcParams& p, const MttkrpTCLaunch& L, cudaStream_t stream, bool prep) {
  auto kern = mttkrp_tc_kernel<NT, CG, PK>;
  if (prep) return allow_dyn_smem(reinterpret_cast<const void*>(kern), L.smem_bytes);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(L.n_full * L.splits + L.splits_tail);
  cfg.blockDim = dim3(L.threads);
  cfg.dynamicSmemBytes = L.smem_bytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (pdl_switch()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (CG == 2) {  // CTA pairs on one TPC (tcgen05 cta_group::2)
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = 2;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kern, p);
}

template <int CG>
cudaError_t dispatch_cg(const TcParams& p, const MttkrpTCLaunch& L, cudaStream_t stream, bool prep) {
  switch (L.N / 16) {
    case 1: return launch_nt<1, CG>(p, L, stream, prep);
    case 2: return launch_nt<2, CG>(p, L, stream, prep);
    case 3: return launch_nt<3, CG>(p, L, stream, prep);
    case 4: return launch_nt<4, CG>(p, L, stream, prep);
    case 5: return launch_nt<5, CG>(p, L, stream, prep);
    case 6: return launch_nt<6, CG>(p, L, stream, prep);
    case 7:
      if constexpr (CG == 2) {  // R <= 104 (c5: R = 100): packed T0 / T1 ranges
        if (L.np != L.N) return launch_nt<7, CG, 1>(p, L, stream, prep);
      }
      return launch_nt<7, CG>(p, L, stream, prep);
    case 8: return launch_nt<8, CG>(p, L, stream, prep);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t dispatch_tc(const TcParams& p, const MttkrpTCLaunch& L, cudaStream_t stream, bool prep) {
  return L.cg == 2 ? dispatch_cg<2>(p, L, stream, prep) : dispatch_cg<1>(p, L, stream, prep);
}

// Split units [0, n_g * n_o) (g-major) into `parts` contiguous ranges of
// about equal cost.  A unit costs its streamed bytes (in full-block units:
// the last l block stores only ct of 8 chunks) plus a fixed per-unit share
// for its accumulator drain and handshakes, which grows with N.
void partition_units(const MttkrpTCLaunch& L, int parts, uint32_t* ub) {
  const int64_t units = static_cast<int64_t>(L.n_g) * L.n_o;
  // measured, single CTAs: c2 best near 3, R = 64..100 near 4..6; CTA pairs (the
  // unit's drain is spread over two SMs): c5 7.35 / 7.43 / 7.69 ms per mode at
  // 2.5 / 4 / 5.5, c2 and c3 flat
  // Merged sets (N > 85) are tensor-/epilogue-bound, not HBM-bound: a unit takes
  // about the same time whatever its bytes (c5 timeline, tools/tc_timeline.py: the
  // last group's 3.25-block units cost 3.71 us against 3.76 us for 4-block units,
  // so the CTAs of the last split ran 1980 units against 1752 and finished 12%
  // after the rest); per outer iteration 110.1 / 109.2 / 108.0 / 107.0 / 107.9 ms
  // at 2.5 / 5 / 10 / 20 / 40.
  double unit_fixed = L.cg == 2 ? (merged_acc(L.N) ? 20.0 : 2.5) : 2.0 + L.N / 32.0;
  if (const char* e = diag_env("NTF_TC_UNITCOST")) unit_fixed = atof(e);
  auto cost = [&](int g) {
    const int nl = std::min(L.G, L.n_lb - g * L.G);
    const bool tail = g * L.G + nl == L.n_lb;
    return (tail ? (nl - 1) + L.ct / 8.0 : nl) + unit_fixed;
  };
  double total = 0.0;
  for (int g = 0; g < L.n_g; ++g) total += cost(g) * L.n_o;
  ub[0] = 0;
  int k = 1;
  double acc = 0.0;
  for (int64_t u = 0; u < units && k < parts; ++u) {
    acc += cost(static_cast<int>(u / L.n_o));
    while (k < parts && acc >= total * k / parts) ub[k++] = static_cast<uint32_t>(u + 1);
  }
  while (k <= parts) ub[k++] = static_cast<uint32_t>(units);
}

}  // namespace

// diagnostics: copy the per-CTA stamps of the last NTF_TC_DEBUG&256 launch
int tc_debug_read_times(unsigned long long* host, int ctas) {
  ctas = std::min(ctas, kTcTimesCtas);
  return cudaMemcpy(host, tc_debug_times(), sizeof(unsigned long long) * 8 * ctas,
                    cudaMemcpyDeviceToHost) == cudaSuccess ? ctas : -1;
}

// ----------------------------------------------------------------------------
// host API
// ----------------------------------------------------------------------------
bool mttkrp_tc_supported(int x_dtype, int R) {
  return x_dtype == NTF_F32 && R >= 1 && R <= 128;
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
  // The block image is written element-wise (no stride constraints); l/o
  // coordinates and unit ranges are 32-bit.
  if (I < 1 || J < 1 || K < 1) return false;
  if (I >= (1 << 30) || J >= (1 << 30) || K >= (1 << 30)) return false;
  const int64_t l_ext = mode == 3 ? J : K, o_ext = mode == 1 ? J : I;
  if (((l_ext + kBK - 1) / kBK) * o_ext >= (int64_t(1) << 31)) return false;
  return true;
}

MttkrpTCLaunch mttkrp_tc_plan(int mode, int x_dtype, int64_t I, int64_t J, int64_t K, int R) {
  (void)x_dtype;
  MttkrpTCLaunch L{};
  L.mode = mode;
  L.R = R;
  L.N = ((R + 15) / 16) * 16;
  L.np = L.N;
  L.M = mode == 1 ? I : (mode == 2 ? J : K);
  L.Q = mode == 3 ? I * J : (mode == 1 ? J * K : I * K);
  L.l_ext = static_cast<int>(mode == 3 ? J : K);
  L.n_o = static_cast<int>(mode == 1 ? J : I);
  L.n_lb = (L.l_ext + kBK - 1) / kBK;
  L.threads = tc_threads(L.N / 16);
  // CTA pairs (tcgen05 cta_group::2, M = 256 over two SMs of a TPC): each
  // CTA keeps only half of the W slices resident, so a unit (one TMEM
  // drain) spans more l blocks, and one MMA instruction serves both SMs.
  // Below ~1 GB of tensor per mode the pair kernel's longer prologue (cluster
  // barrier, 2-CTA tensor maps) is not hidden behind the previous kernel
  // (outer iteration, graph replay: c2 1.65 ms single vs 1.90 ms pairs; c4
  // 10.50 vs 10.25, c3 12.2 vs 10.5, c5 137.8 vs 114.2).
  L.cg = L.M * L.Q >= (int64_t(1) << 28) ? 2 : 1;
  if (const char* e = diag_env("NTF_TC_CG")) L.cg = atoi(e) == 1 ? 1 : 2;
  // Packed T0 / T1 ranges (set_cols): instantiated where it pays, the pair
  // kernel at N = 112 with R <= 104 (BASELINE c5, R = 100: 432 instead of 448
  // MMA columns per K step, 104 instead of 112 columns drained per accumulator).
  if (L.cg == 2 && L.N == 112 && R <= 104) L.np = 104;
  if (const char* e = diag_env("NTF_TC_PACK")) { if (atoi(e) == 0) L.np = L.N; }
  // Equal m-tiles of tm <= 128 rows (a multiple of 8, the core-matrix
  // height), so every CTA of a full tile streams the same bytes.  Pairs
  // take two consecutive tiles: an even tile count, and every tile stored
  // with tm rows (the last one zero-padded) so both CTAs of a pair share the
  // leader's A descriptor.  Single CTAs: the last tile may be shorter.
  {
    const int64_t nt = L.cg == 2 ? 2 * ((L.M + 2 * kTM - 1) / (2 * kTM)) : (L.M + kTM - 1) / kTM;
    L.tm = static_cast<int>(8 * ((L.M + 8 * nt - 1) / (8 * nt)));
    L.n_mtiles = static_cast<int>(nt);
  }
  // Shared memory: resident W slices of a group (G blocks x 4N/cg x 128 B) +
  // F_hi pair ring + the X ring, whose slots hold slot_ks K steps (64 tm
  // bytes each).  Measured (per mode, c2/c3/c4/c5): one K step per slot
  // (8 KB, a deep ring) 104/1069/645/11200 us, two 69/752/428/9866, a whole
  // 64-wide l block (4 K steps) 56/693/336/9318: every X slot costs the MMA
  // issuer a barrier wait and a tcgen05.commit, so slots are whole blocks.
  // G is the largest (<= 4: T0 keeps t = 5 bits, F_lo 27 bits) that leaves
  // a ring of at least min_ring bytes.
  L.slot_ks = 4;
  if (const char* e = diag_env("NTF_TC_SLOTKS")) L.slot_ks = std::max(1, std::min(4, atoi(e)));
  const int xs = ((L.slot_ks * 64 * L.tm + 127) / 128) * 128;
  L.stage_bytes = xs;
  L.h_stages = 8;
  const int wlb = w_rows(L.N, L.np) / L.cg * kBK * 2;  // W bytes of one l block in one CTA
  const int limit = 226 * 1024;  // the opt-in 227 KB less the kernel's 1 KB of static shared memory
  auto fixed_bytes = [&](int G) {
    return 1024 + G * wlb + L.h_stages * L.N * 8 + (2 * L.h_stages + 14) * 8 + 16 + 3 * L.N * 8;
  };
  auto total = [&](int G, int SX) { return fixed_bytes(G) + SX * (xs + 24); };
  int min_ring = 64 * 1024;
  if (const char* e = diag_env("NTF_TC_MINRING")) min_ring = atoi(e) * 1024;
  L.G = 1;
  for (int G : {4, 3, 2, 1})
    if (limit - fixed_bytes(G) >= min_ring) {
      L.G = G;
      break;
    }
  if (const char* e = diag_env("NTF_TC_G")) L.G = atoi(e);
  L.G = std::max(1, std::min(L.G, L.n_lb));
  L.x_stages = kTcMaxXStages;
  if (const char* e = diag_env("NTF_TC_XSTAGES")) L.x_stages = std::max(2, std::min(kTcMaxXStages, atoi(e)));
  while (total(L.G, L.x_stages) > limit && L.x_stages > 2) --L.x_stages;
  L.smem_bytes = total(L.G, L.x_stages);
  L.tmem_cols = static_cast<int>(tmem_cols(L.N));
  L.n_g = (L.n_lb + L.G - 1) / L.G;
  const int64_t units = static_cast<int64_t>(L.n_g) * L.n_o;
  // One CTA per SM, one wave.  Two SMs are left free so the mode's ridge
  // Cholesky (side stream) and the early row-update blocks run concurrently.
  const int cap = std::min(sm_count_tc() - 2, kTcMaxSplits);
  {
    const int rem = L.l_ext % kBK;
    L.ct = rem == 0 ? 8 : 2 * ((rem + 15) / 16);
  }
  L.tile_bytes = static_cast<int64_t>(L.n_o) * 32 * L.tm * (8 * (L.n_lb - 1) + L.ct);
  auto clampu = [&](int64_t s) { return static_cast<int>(std::max<int64_t>(1, std::min(s, units))); };
  if (L.cg == 2) {
    // every tile padded to tm rows: one partition shared by all pairs
    L.n_full = L.n_mtiles;
    L.r8_full = L.tm;
    L.r8_tail = 0;
    L.img_bytes = static_cast<size_t>(L.n_full) * L.tile_bytes;
    L.splits = clampu(static_cast<int64_t>(cap / 2 / (L.n_full / 2)));
    L.splits_tail = 0;
    if (const char* e = diag_env("NTF_TC_SPLITS")) L.splits = clampu(std::min(atoi(e), cap / L.n_full));
    partition_units(L, L.splits, L.ub_full);
  } else {
    // CTAs go to tiles in proportion to their cost (a 400-row mode is 3 full
    // tiles + 16 rows: equal splits would leave a fifth of the SMs streaming
    // almost nothing); a block of a ragged tile costs about a full one.
    L.n_full = static_cast<int>(L.M / L.tm);
    const int tail = static_cast<int>(L.M % L.tm);
    L.r8_full = L.tm;
    L.r8_tail = tail ? 8 * ((tail + 7) / 8) : 0;
    L.img_bytes = static_cast<size_t>(L.n_full) * L.tile_bytes +
                  (tail ? static_cast<size_t>(L.n_o) * 32 * L.r8_tail * (8 * (L.n_lb - 1) + L.ct) : 0);
    const double wt = tail ? 1.0 : 0.0;
    if (L.n_full == 0) {
      L.splits = 0;
      L.splits_tail = clampu(cap);
    } else {
      L.splits = clampu(static_cast<int64_t>(cap / (L.n_full + wt)));
      L.splits_tail = 0;
      if (tail)
        L.splits_tail = clampu(std::min<int64_t>(static_cast<int64_t>(L.splits * wt + 0.5),
                                                 cap - static_cast<int64_t>(L.n_full) * L.splits));
    }
    if (L.splits) partition_units(L, L.splits, L.ub_full);
    if (L.splits_tail) partition_units(L, L.splits_tail, L.ub_tail);
  }
  L.wscale = nullptr;
  L.wsl = nullptr;
  L.hpair = nullptr;
  L.bound = false;
  return L;
}

size_t mttkrp_tc_workspace_bytes(const MttkrpTCLaunch& L, int R) {
  return static_cast<size_t>(std::max(L.splits, L.splits_tail)) * L.M * R * sizeof(double);
}

cudaError_t mttkrp_tc_prepare(const MttkrpTCLaunch& L) {
  TcParams p{};
  return dispatch_tc(p, L, nullptr, true);
}

cudaError_t tc_tensor_fill(const MttkrpTCLaunch& L, const TcTensor& t, cudaStream_t stream,
                           const TcTensor* same_values) {
  const int64_t n = t.dims[0] * t.dims[1] * t.dims[2];
  unsigned* amax = reinterpret_cast<unsigned*>(t.xscale + 1);
  if (same_values && same_values->src == t.src && same_values->xscale &&
      same_values->dims[0] * same_values->dims[1] * same_values->dims[2] == n) {
    amax = reinterpret_cast<unsigned*>(same_values->xscale + 1);  // max|X| of the same values
  } else {
    cudaError_t e = cudaMemsetAsync(amax, 0, sizeof(unsigned), stream);
    if (e != cudaSuccess) return e;
    absmax_kernel<<<4 * sm_count_tc(), 256, 0, stream>>>(t.src, n, amax);
  }
  ImgGeom g;
  g.mode = L.mode;
  g.I = t.dims[0];
  g.J = t.dims[1];
  g.K = t.dims[2];
  g.M = L.M;
  g.n_o = L.n_o;
  g.l_ext = L.l_ext;
  g.n_lb = L.n_lb;
  g.G = L.G;
  g.tm = L.tm;
  g.n_full = L.n_full;
  g.n_tiles = L.n_full + (L.r8_tail ? 1 : 0);
  g.r8_full = L.r8_full;
  g.r8_tail = L.r8_tail;
  g.ct = L.ct;
  g.tile_bytes = L.tile_bytes;
  if (L.mode == 3)  // m = k contiguous: the direct kernel's reads coalesce along the rows
    image_split_kernel<<<8 * sm_count_tc(), 256, 0, stream>>>(t.src, g, amax, t.img, t.xscale);
  else
    image_split_rows_kernel<<<16 * sm_count_tc(), 256, 0, stream>>>(t.src, g, amax, t.img, t.xscale);
  return cudaGetLastError();
}

cudaError_t tc_tensor_create(const MttkrpTCLaunch& L, const float* X, const int64_t dims[3],
                             TcTensor* out, cudaStream_t stream, const TcTensor* same_values) {
  TcTensor t;
  for (int i = 0; i < 3; ++i) t.dims[i] = dims[i];
  t.mode = L.mode;
  t.img_bytes = L.img_bytes;
  t.src = X;
  cudaError_t e;
  if ((e = ntf::dev_alloc(&t.img, L.img_bytes)) != cudaSuccess) return e;
  if ((e = ntf::dev_alloc(&t.xscale, sizeof(double) + sizeof(unsigned) * 2)) != cudaSuccess) {
    tc_tensor_destroy(&t);
    return e;
  }
  if ((e = tc_tensor_fill(L, t, stream, same_values)) != cudaSuccess) {
    tc_tensor_destroy(&t);
    return e;
  }
  *out = t;
  return cudaSuccess;
}

void tc_tensor_destroy(TcTensor* t) {
  if (!t) return;
  ntf::dev_free(t->img);
  ntf::dev_free(t->xscale);
  t->img = nullptr;
  t->xscale = nullptr;
}

namespace {
// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
PFN_cuTensorMapEncodeTiled_v12000 tmap_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// rows x 128 B of bytes at `base`, loaded box_rows rows at a time, no swizzle
cudaError_t rows128_map(CUtensorMap* m, const void* base, uint64_t rows, uint32_t box_rows) {
  auto enc = tmap_encode();
  if (!enc || box_rows < 1 || box_rows > 256) return cudaErrorInvalidValue;
  const cuuint64_t dims[2] = {128, rows};
  const cuuint64_t strides[1] = {128};
  const cuuint32_t box[2] = {128, box_rows};
  const cuuint32_t es[2] = {1, 1};
  const CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}
}  // namespace

cudaError_t mttkrp_tc_bind(MttkrpTCLaunch& L, const TcTensor& t) {
  if (t.mode != L.mode || t.img_bytes != L.img_bytes) return cudaErrorInvalidValue;
  if (!L.wscale) {
    cudaError_t e = ntf::dev_alloc(&L.wscale, sizeof(double) * 2 * L.N);
    if (e != cudaSuccess) return e;
  }
  if (!L.wsl) {
    cudaError_t e = ntf::dev_alloc(&L.wsl, static_cast<size_t>(L.n_lb) * 4 * L.N * kBK * 2);
    if (e != cudaSuccess) return e;
  }
  if (!L.hpair) {
    cudaError_t e = ntf::dev_alloc(&L.hpair, static_cast<size_t>(L.n_o) * L.N * sizeof(float2));
    if (e != cudaSuccess) return e;
  }
  if (L.cg == 2) {  // tensor maps of this image and of the W slices (CTA-pair loads)
    const int wrows = w_rows(L.N, L.np) / 2;
    cudaError_t e = rows128_map(&L.map_full, t.img, L.img_bytes / 128, static_cast<uint32_t>(2 * L.r8_full));
    if (e == cudaSuccess)
      e = rows128_map(&L.map_tail, t.img, L.img_bytes / 128, static_cast<uint32_t>(L.ct * L.r8_full / 4));
    if (e == cudaSuccess)
      e = rows128_map(&L.map_w, L.wsl, static_cast<uint64_t>(2) * L.n_lb * wrows, static_cast<uint32_t>(wrows));
    if (e != cudaSuccess) return e;
  }
  L.bound = true;
  return cudaSuccess;
}

void mttkrp_tc_unbind(MttkrpTCLaunch& L) {
  ntf::dev_free(L.wscale);
  ntf::dev_free(L.wsl);
  ntf::dev_free(L.hpair);
  L.wscale = nullptr;
  L.wsl = nullptr;
  L.hpair = nullptr;
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
  TcParams p{};
  p.img = t.img;
  p.tile_bytes = L.tile_bytes;
  p.r8_full = L.r8_full;
  p.r8_tail = L.r8_tail;
  p.ct = L.ct;
  p.mode = L.mode;
  p.R = L.R;
  p.M = L.M;
  p.l_ext = L.l_ext;
  p.n_o = L.n_o;
  p.n_lb = L.n_lb;
  p.G = L.G;
  p.n_full = L.n_full;
  p.splits = L.splits;
  p.splits_tail = L.splits_tail;
  p.tm = L.tm;
  p.x_stages = L.x_stages;
  p.slot_ks = L.slot_ks;
  p.stage_bytes = L.stage_bytes;
  p.h_stages = L.h_stages;
  p.hpair = L.hpair;
  p.wsl = L.wsl;
  p.n_tiles = L.n_mtiles;
  if (L.cg == 2) {
    p.map_full = L.map_full;
    p.map_tail = L.map_tail;
    p.map_w = L.map_w;
  }
  p.ws = ws;
  p.stop_flag = stop_flag;
  for (int i = 0; i <= kTcMaxSplits; ++i) {
    p.ub_full[i] = L.ub_full[i];
    p.ub_tail[i] = L.ub_tail[i];
  }
  {
    static int dbg = -1;
    if (dbg < 0) {
      const char* env = diag_env("NTF_TC_DEBUG");
      dbg = env ? atoi(env) : 0;
    }
    p.debug = dbg;
    if (dbg & 256) p.times = tc_debug_times();
  }
  p.xscale = t.xscale;
  if (colmax3) {  // plan: column maxima kept current by the row-update kernels
    const int hm = L.mode == 1 ? 1 : 0, lm = L.mode == 3 ? 1 : 2;
    p.cm_hi = colmax3 + hm * L.R;
    p.cm_lo = colmax3 + lm * L.R;
    p.cm_self = const_cast<double*>(colmax3) + (L.mode - 1) * L.R;
  } else {        // one-shot call: compute them here
    colmax_kernel<<<L.R, 256, 0, stream>>>(Fhi, hi_rows, L.R, L.wscale);
    colmax_kernel<<<L.R, 256, 0, stream>>>(Flo, lo_rows, L.R, L.wscale + L.R);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    p.cm_hi = L.wscale;
    p.cm_lo = L.wscale + L.R;
  }
  {
    const int t = t_bits(L.G);
    const int total = std::max(L.n_lb * L.N * (kBK / 8), L.n_o * L.N);
    const int blocks = std::min((total + 63) / 64, 8 * sm_count_tc());
    if (!(p.debug & 128)) {
      cudaError_t e = launch_pdl(w_slice_kernel, dim3(blocks), dim3(64), 0, stream, Flo, L.l_ext,
                                 L.R, L.N, L.np, L.cg, L.n_lb, !merged_acc(L.N), p.cm_lo, t, L.wsl, Fhi, L.n_o, p.cm_hi,
                                 L.hpair, stop_flag);
      if (e != cudaSuccess) return e;
    }
  }
  return dispatch_tc(p, L, stream, false);
}

}  // namespace ntf
