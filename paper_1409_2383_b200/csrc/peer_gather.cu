// Row all-gather of a factor over NVLink peer memory: one kernel per mode
// update of the sharded engine, replacing pack -> ncclAllGather -> unpack.
//
// Reference semantics: after the block-row updates of mode n every node holds
// the whole updated factor (blocks.py:171-196, mesh.py:149-237: the wave's
// broadcast of the updated row blocks).  Here each rank pushes its owned rows
// straight into every peer's staging buffer with P2P stores, signals one
// arrival per CTA on every peer's counter (release at system scope), waits
// for all ranks' arrivals on its own counter (acquire), and copies the other
// ranks' rows from its staging buffer into its factor.
//
// Staging is double-buffered by the parity of the per-buffer gather sequence
// number: a rank can only start gather t+1 after its gather t saw every
// peer's arrival for t, which each peer signalled after finishing gather t-1,
// so nobody overwrites a parity a peer is still reading.  The staging buffer
// (not the peer's factor) is the target because a peer may still be reading
// its factor (as an MTTKRP companion) when the pushes of the next update land.
#include <cstdint>

#include "peer_gather.cuh"

namespace ntf {
namespace {

__device__ __forceinline__ unsigned int ld_acquire_sys(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void red_release_sys_add(unsigned int* p, unsigned int v) {
  asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint64_t now_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Copy doubles [lo, hi) of src to dst with CTA c of `ctas` taking one
// contiguous, 16-byte-aligned share (double2 body, scalar tail).
__device__ __forceinline__ void copy_share(double* __restrict__ dst, const double* __restrict__ src,
                                           int64_t lo, int64_t hi, int c, int ctas) {
  const int64_t n = hi - lo;
  if (n <= 0) return;
  const int64_t per = ((n + ctas - 1) / ctas + 1) & ~int64_t(1);  // even share
  const int64_t a = lo + per * c;
  const int64_t b = min(hi, a + per);
  if (a >= b) return;
  int64_t i = a + threadIdx.x * 2;
  const bool aligned = ((reinterpret_cast<uintptr_t>(dst + a) | reinterpret_cast<uintptr_t>(src + a)) & 15) == 0;
  if (aligned) {
    for (; i + 1 < b; i += 2 * blockDim.x)
      *reinterpret_cast<double2*>(dst + i) = *reinterpret_cast<const double2*>(src + i);
    if (i < b) dst[i] = src[i];  // odd tail: only the thread that reaches it
  } else {
    for (int64_t j = a + threadIdx.x; j < b; j += blockDim.x) dst[j] = src[j];
  }
}

// One rank's gather, CTA c of `ctas`.  A status word already set (an
// earlier wait timed out somewhere in this fit) makes the gather a no-op: no
// pushes, no arrivals, no sequence change, so a rank that fell out of step
// never writes into a parity its peers read; the host checks the word after
// every outer iteration and all ranks abort together.
__device__ __forceinline__ void peer_gather_body(const PeerGatherArgs& a, int c, int ctas) {
  __shared__ unsigned int s_seq;
  __shared__ int s_ok;
  const int R = a.R;
  const int64_t rows = a.row_offset[a.nranks];
  const int64_t plane = rows * R;  // doubles per staging parity
  if (threadIdx.x == 0) {
    s_seq = *reinterpret_cast<volatile unsigned int*>(peer_seq(a.base[a.me]));
    s_ok = (a.status && *reinterpret_cast<volatile int*>(a.status) != 0) ? 0 : 1;
  }
  __syncthreads();
  if (!s_ok) return;
  const unsigned int seq = s_seq;
  const int64_t par = seq & 1u;

  // 1. push the owned rows into every peer's staging (same row positions)
  const int64_t lo = a.row_offset[a.me] * R, hi = a.row_offset[a.me + 1] * R;
  for (int q = 0; q < a.nranks; ++q) {
    if (q == a.me) continue;
    copy_share(peer_staging(a.base[q]) + par * plane, a.full, lo, hi, c, ctas);
  }
  __syncthreads();
  // 2. one arrival per CTA on every rank's counter (own included), then wait
  //    until all ranks' CTAs have arrived for this sequence number
  if (threadIdx.x == 0) {
    __threadfence_system();  // the CTA's P2P stores (ordered by bar.sync) before the arrivals
    for (int q = 0; q < a.nranks; ++q) red_release_sys_add(peer_arrivals(a.base[q]), 1u);
    const unsigned int target = (seq + 1u) * static_cast<unsigned int>(a.nranks) * ctas;
    const unsigned int* mine = peer_arrivals(a.base[a.me]);
    const uint64_t t0 = now_ns();
    while (static_cast<int>(ld_acquire_sys(mine) - target) < 0) {
      if (now_ns() - t0 > static_cast<uint64_t>(a.timeout_ns)) {
        s_ok = 0;
        if (a.status) atomicExch(a.status, kPeerGatherTimeout);
        break;
      }
      __nanosleep(64);
    }
  }
  __syncthreads();
  if (!s_ok) return;
  // 3. the other ranks' rows: own staging -> factor
  const double* st = peer_staging(a.base[a.me]) + par * plane;
  for (int q = 0; q < a.nranks; ++q) {
    if (q == a.me) continue;
    copy_share(a.full, st, a.row_offset[q] * R, a.row_offset[q + 1] * R, c, ctas);
  }
  // every CTA of this launch read seq before arriving, and CTA 0 is past the
  // wait, so all of them have read it: advance for the next launch
  if (c == 0 && threadIdx.x == 0) *peer_seq(a.base[a.me]) = seq + 1u;
}

__global__ void __launch_bounds__(kPeerGatherThreads) peer_gather_kernel(PeerGatherArgs a) {
  peer_gather_body(a, blockIdx.x, gridDim.x);
}

// Every rank's gather in ONE cooperative launch on one device (block b plays
// CTA b % ctas of rank b / ctas): the ranks' spin-waits on one another are
// only safe when all their CTAs are co-resident, which separate launches on
// one GPU do not guarantee.  Runs the real protocol concurrently for tests.
__global__ void __launch_bounds__(kPeerGatherThreads) peer_gather_group_kernel(PeerGatherGroup g) {
  const int ctas = g.args[0].ctas;
  peer_gather_body(g.args[blockIdx.x / ctas], blockIdx.x % ctas, ctas);
}

}  // namespace

// Largest CTA count whose CTAs are co-resident on this device (the kernel's
// CTAs spin-wait on arrivals from all CTAs of every rank).
int peer_gather_max_ctas(int ranks_in_launch) {
  int dev = 0, sms = 0, per_sm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
  const void* k = ranks_in_launch > 1 ? reinterpret_cast<const void*>(peer_gather_group_kernel)
                                      : reinterpret_cast<const void*>(peer_gather_kernel);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kPeerGatherThreads, 0) != cudaSuccess)
    return 0;
  return per_sm * sms / (ranks_in_launch > 1 ? ranks_in_launch : 1);
}

cudaError_t peer_gather_launch(const PeerGatherArgs& a, cudaStream_t stream) {
  peer_gather_kernel<<<a.ctas, kPeerGatherThreads, 0, stream>>>(a);
  return cudaGetLastError();
}

cudaError_t peer_gather_group_launch(const PeerGatherGroup& g, int nranks, cudaStream_t stream) {
  PeerGatherGroup arg = g;
  void* params[] = {&arg};
  return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(peer_gather_group_kernel),
                                     dim3(nranks * g.args[0].ctas), dim3(kPeerGatherThreads), params, 0,
                                     stream);
}

}  // namespace ntf
