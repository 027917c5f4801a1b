// Microbenchmark: mbarrier handshake costs on sm_100a (diagnostics only).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void init(uint64_t* b, int c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  uint32_t d = 0;
  do {
    asm volatile("{\n.reg .pred P;\nmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\nselp.u32 %0,1,0,P;\n}" : "=r"(d) : "r"(su32(b)), "r"(ph) : "memory");
  } while (!d);
}
__device__ __forceinline__ void commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(b)) : "memory");
}

// mode 0: ping-pong ring, producer warp 0 / consumer warp 1, whole warps (elect lane 0 arrives)
// mode 1: same, single threads
// mode 2: consumer uses tcgen05.commit instead of arrive
// mode 3: single thread: wait on an already-complete barrier, n times (latency)
__global__ void k(int mode, int depth, int n, long long* out) {
  __shared__ uint64_t full[16], empty[16];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < depth; ++i) { init(&full[i], 1); init(&empty[i], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (mode == 3) {
    if (threadIdx.x == 0) {
      arrive(&full[0]);  // phase 0 complete
      long long t0 = clock64();
      for (int i = 0; i < n; ++i) wait(&full[0], 0);
      out[0] = clock64() - t0;
    }
    return;
  }
  if (mode >= 4) {
    __shared__ alignas(128) unsigned char buf[4096];
    if (threadIdx.x == 0 || (mode == 7 && warp == 0)) {
      if (mode != 7 && threadIdx.x == 0) { init(&full[1], n + 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
      if (mode == 7 && lane == 0) arrive(&full[0]);
      __syncwarp(mode == 7 ? 0xffffffffu : 1u);
      long long t0 = clock64();
      for (int i = 0; i < n; ++i) {
        if (mode == 4) arrive(&full[1]);
        else if (mode == 5) commit(&full[1]);
        else if (mode == 6) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[1])), "r"(0) : "memory");
        else if (mode == 7) wait(&full[0], 0);
        else if (mode == 9) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        else if (mode == 10) asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        else if (mode == 11) { long long c = clock64(); asm volatile("" :: "l"(c)); }
        else if (mode == 12) { arrive(&full[1]); asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
        else if (mode == 8) {
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[1])), "r"(512) : "memory");
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(buf + (i & 7) * 512)), "l"(out + 64), "r"(512), "r"(su32(&full[1])) : "memory");
        }
      }
      if (lane == 0) out[0] = clock64() - t0;
    }
    return;
  }
  const bool single = mode != 0;
  if (single && lane != 0) return;
  long long t0 = clock64();
  int idx = 0; uint32_t ph = 0;
  if (warp == 0) {
    for (int i = 0; i < n; ++i) {
      wait(&empty[idx], ph ^ 1u);
      if (lane == 0) arrive(&full[idx]);
      if (!single) __syncwarp();
      if (++idx == depth) { idx = 0; ph ^= 1u; }
    }
  } else if (warp == 1) {
    for (int i = 0; i < n; ++i) {
      wait(&full[idx], ph);
      if (lane == 0) { if (mode == 2) commit(&empty[idx]); else arrive(&empty[idx]); }
      if (!single) __syncwarp();
      if (++idx == depth) { idx = 0; ph ^= 1u; }
    }
    if (lane == 0) out[0] = clock64() - t0;
  }
}

int main() {
  long long* d; cudaMalloc(&d, 8192); cudaMemset(d, 0, 8192);
  const int n = 20000;
  for (int mode = 3; mode < 13; ++mode)
    for (int depth : {1, 2, 4, 8}) {
      if (mode >= 3 && depth > 1) continue;
      k<<<1, 64>>>(mode, depth, n, d);
      long long h = 0;
      cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      cudaError_t e = cudaGetLastError();
      printf("mode %d depth %d: %.1f cycles/iter %s\n", mode, depth, double(h) / n, e ? cudaGetErrorString(e) : "");
    }
  return 0;
}
