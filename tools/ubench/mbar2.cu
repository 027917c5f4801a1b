// Microbenchmark (diagnostics): per-op cost of mbarrier / tcgen05 sync ops in a
// clean single-thread loop (op selected at compile time).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void init(uint64_t* b, int c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void arrive(uint32_t b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b) : "memory"); }
__device__ __forceinline__ void wait(uint32_t b, uint32_t ph) {
  uint32_t d = 0;
  do { asm volatile("{\n.reg .pred P;\nmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\nselp.u32 %0,1,0,P;\n}" : "=r"(d) : "r"(b), "r"(ph) : "memory"); } while (!d);
}
template <int OP>
__global__ void k(int n, long long* out) {
  __shared__ uint64_t bar[4];
  __shared__ alignas(128) unsigned char buf[4096];
  if (threadIdx.x != 0) return;
  init(&bar[0], 1); init(&bar[1], (1 << 20) - 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const uint32_t b0 = su32(&bar[0]), b1 = su32(&bar[1]);
  arrive(b0);
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if constexpr (OP == 0) { asm volatile("" ::: "memory"); }
    if constexpr (OP == 1) wait(b0, 0);
    if constexpr (OP == 2) arrive(b1);
    if constexpr (OP == 3) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(b1) : "memory");
    if constexpr (OP == 4) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b1), "r"(0) : "memory");
    if constexpr (OP == 5) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if constexpr (OP == 6) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b1), "r"(512) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(buf + (i & 7) * 512)), "l"(out + 64), "r"(512), "r"(b1) : "memory"); }
    if constexpr (OP == 7) { wait(b0, 0); arrive(b1); }
    if constexpr (OP == 8) { wait(b0, 0); asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(b1) : "memory"); }
  }
  out[0] = clock64() - t0;
}
template <int OP> void run(const char* name, long long* d) {
  const int n = 20000;
  k<OP><<<1, 32>>>(n, d);
  long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("%-28s %.1f cycles/op %s\n", name, double(h) / n, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  long long* d; cudaMalloc(&d, 8192); cudaMemset(d, 0, 8192);
  run<0>("empty", d); run<1>("try_wait(complete)", d); run<2>("arrive", d); run<3>("tcgen05.commit", d);
  run<4>("arrive.expect_tx", d); run<5>("tcgen05.fence::after", d); run<6>("expect_tx+bulk 512B", d);
  run<7>("wait+arrive", d); run<8>("wait+commit", d);
  return 0;
}
