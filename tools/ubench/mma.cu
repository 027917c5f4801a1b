// Microbenchmark (diagnostics): tcgen05.mma (kind::f16, M=128) issue/exec cost
// from one thread, SS operands in shared memory (zeros), commit + wait at end.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc_noswz(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (addr >> 4) & 0x3FFFull;
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= 1ull << 46;
  return d;
}
__host__ __device__ constexpr uint32_t idesc(int N) { return (1u << 4) | ((uint32_t(N) >> 3) << 17) | ((128u >> 4) << 24); }
template <int N, int PER_COMMIT, int ISSUERS = 1>
__global__ void k(int n, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar))); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  if ((threadIdx.x & 31) == 0 && warp < ISSUERS) {
    const uint64_t da = desc_noswz(su32(sm), 128 * 16, 128);
    const uint64_t db = desc_noswz(su32(sm + 32768), N * 16, 128);
    uint32_t ph = 0;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                   ::"r"(tmem + warp * 128), "l"(da + (i & 3) * 4), "l"(db + (i & 3) * 4), "r"(idesc(N)), "r"(i & 7) : "memory");
      if ((i + 1) % PER_COMMIT == 0) {
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
      }
    }
    long long t1 = clock64();
    // drain: wait for the last commit
    if (ISSUERS > 1) { out[0] = t1 - t0; }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
    uint32_t done = 0;
    const int ncommit = n / PER_COMMIT + 1;
    // the barrier completes a phase per commit; wait for the final phase parity
    ph = (ncommit - 1) & 1;
    if (ISSUERS == 1) do { asm volatile("{\n.reg .pred P;\nmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\nselp.u32 %0,1,0,P;\n}" : "=r"(done) : "r"(su32(&bar)), "r"(ph) : "memory"); } while (!done);
    long long t2 = clock64();
    if (warp == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}
template <int N, int PC, int IS = 1> void run(long long* d) {
  const int n = 4000;
  cudaFuncSetAttribute(k<N, PC, IS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<N, PC, IS><<<1, 128, 65536 + 1024>>>(n, d);
  cudaEventRecord(e1); cudaEventSynchronize(e1); float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
  printf("issuers %d: kernel %.1f us for %d MMAs per issuer\n", IS, ms * 1e3, n);
  long long h[2] = {0, 0};
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("N=%3d commit/%d: issue %.1f cyc/mma, total %.1f cyc/mma (floor %d) %s\n", N, PC, double(h[0]) / n,
         double(h[1]) / n, 128 * N / 256, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  long long* d; cudaMalloc(&d, 64);
  run<64, 1000000>(d); run<96, 1000000>(d); run<128, 1000000>(d); run<192, 1000000>(d); run<256, 1000000>(d);
  run<96, 8>(d); run<64, 8>(d); run<96, 1000000, 2>(d); run<96, 1000000, 4>(d); run<64, 1000000, 2>(d); run<256, 1000000, 2>(d);
  return 0;
}
