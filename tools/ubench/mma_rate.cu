// tcgen05.mma issue-rate probe on one B200: kind::f16 (K = 16) against
// kind::i8 (K = 32), M = 128, N = 256, one CTA per SM, operands resident in
// shared memory (no loads in the loop), accumulators in TMEM.  Reports the
// tensor rate a streaming kernel could draw on at most, at whatever clock the
// board holds under that load (DESIGN 4: the int8 variant of the slicing).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_rate mma_rate.cu && ./mma_rate
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint64_t desc_sw128(const void* p) {  // K-major, SWIZZLE_128B, 8-row groups 1 KB apart
  uint64_t d = (smem_u32(p) >> 4) & 0x3FFFull;
  d |= static_cast<uint64_t>(16 >> 4) << 16;
  d |= static_cast<uint64_t>(1024 >> 4) << 32;
  d |= 1ull << 46;
  d |= 2ull << 61;
  return d;
}

template <bool I8>
__global__ void __launch_bounds__(128, 1) rate_kernel(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_slot;
  // A: 128 rows x 128 B, B: 256 rows x 128 B (one swizzle atom of K: 64 halves / 128 bytes)
  for (int i = threadIdx.x; i < (128 + 256) * 128 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(base)[i] = I8 ? 0x01ff0102u * (i % 7) : 0x3c003800u;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tmem_slot;
  // instruction descriptor: M = 128, N = 256, K-major A and B
  //   f16: D = F32 (1 << 4), A = B = F16 (0);  i8: D = S32 (2 << 4), A = B = S8 (1)
  const uint32_t idesc = (I8 ? (2u << 4) | (1u << 7) | (1u << 10) : (1u << 4)) | ((256u >> 3) << 17) | ((128u >> 4) << 24);
  const uint64_t da = desc_sw128(base), db = desc_sw128(base + 128 * 128);
  long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0) {
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      // the 4 K steps of one 128-byte swizzle atom (32 B each), two accumulator halves of TMEM
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const uint32_t d = tmem + ((it & 1) ? 256u : 0u);
        const uint32_t acc = (it > 1 || ks > 0) ? 1u : 0u;
        if (I8)
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                       "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                       "l"(da + ks * 2), "l"(db + ks * 2), "r"(idesc), "r"(acc)
                       : "memory");
        else
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                       "l"(da + ks * 2), "l"(db + ks * 2), "r"(idesc), "r"(acc)
                       : "memory");
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar))
                 : "memory");
    uint32_t done = 0;
    do {
      asm volatile("{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], 0;\nselp.u32 %0, 1, 0, P1;\n}\n"
                   : "=r"(done)
                   : "r"(smem_u32(&bar))
                   : "memory");
    } while (!done);
    t1 = clock64();
    cycles[blockIdx.x] = static_cast<unsigned long long>(t1 - t0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
  }
}

template <bool I8>
void run(const char* name, int sms, int iters) {
  unsigned long long* cyc;
  cudaMalloc(&cyc, sizeof(unsigned long long) * sms);
  const int smem = (128 + 256) * 128 + 1024;
  cudaFuncSetAttribute(rate_kernel<I8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  rate_kernel<I8><<<sms, 128, smem>>>(iters / 8, cyc);  // warm-up
  cudaDeviceSynchronize();
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    rate_kernel<I8><<<sms, 128, smem>>>(iters, cyc);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    if (err != cudaSuccess) {
      printf("%s: %s\n", name, cudaGetErrorString(err));
      return;
    }
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long c0 = 0;
    cudaMemcpy(&c0, cyc, sizeof(c0), cudaMemcpyDeviceToHost);
    const double k = I8 ? 32.0 : 16.0;
    const double ops = 2.0 * 128 * 256 * k * 4.0 * iters * sms;
    printf("%s: %d SMs x %d x 4 MMAs (M128 N256 K%d): %.2f ms, %.0f T%s/s, %.1f cycles per MMA, ~%.0f MHz\n", name, sms,
           iters, static_cast<int>(k), ms, ops / (ms * 1e-3) / 1e12, I8 ? "OP" : "FLOP",
           static_cast<double>(c0) / (4.0 * iters), c0 / (ms * 1e-3) / 1e6);
  }
  cudaFree(cyc);
}

int main() {
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  const int sms = prop.multiProcessorCount;
  printf("%s, %d SMs\n", prop.name, sms);
  run<false>("kind::f16", sms, 400000);
  run<true>("kind::i8 ", sms, 400000);
  run<false>("kind::f16", sms, 400000);
  return 0;
}
