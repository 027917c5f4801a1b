// fp64 throughput probes on one B200: DFMA (register operands) and the
// m8n8k4 fp64 mma.sync, each with enough independent accumulators.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o f64_rate f64_rate.cu && ./f64_rate
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dmma_kernel(double* out, int iters, double a, double b) {
  double c[16][2];
#pragma unroll
  for (int i = 0; i < 16; ++i) c[i][0] = c[i][1] = threadIdx.x + i;
  double av[4] = {a, a + 1, a + 2, a + 3}, bv[4] = {b, b + 1, b + 2, b + 3};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i * 4 + j][0]), "+d"(c[i * 4 + j][1])
                     : "d"(av[i]), "d"(bv[j]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NACC>
__global__ void dmma_chain_kernel(double* out, int iters, double a, double b) {
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i][0] = c[i][1] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NACC>
void chain(double* out, int threads) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  float ms;
  dmma_chain_kernel<NACC><<<148, threads>>>(out, 100, 1.0000001, 1e-9);
  cudaEventRecord(e0);
  dmma_chain_kernel<NACC><<<148, threads>>>(out, iters, 1.0000001, 1e-9);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("DMMA  %d independent accumulators, %d warps/SM: %.2f TFLOP/s, %.1f ns per round of %d\n", NACC,
         threads / 32, 512.0 * NACC * iters * 148 * (threads / 32) / (ms * 1e-3) / 1e12, ms * 1e6 / iters, NACC);
}

int main() {
  double* out;
  cudaMalloc(&out, 148 * 8 * 1024 * sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int threads : {128, 256, 512, 1024}) {
    const int blocks = 148 * (1024 / threads), iters = 20000;
    float ms;
    dfma_kernel<<<blocks, threads>>>(out, 100, 1.0000001, 1e-9);
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("DFMA  %4d thr/blk x %4d blk: %.2f TFLOP/s\n", threads, blocks,
           2.0 * 16 * iters * blocks * threads / (ms * 1e-3) / 1e12);
    dmma_kernel<<<blocks, threads>>>(out, 100, 1.0000001, 1e-9);
    cudaEventRecord(e0);
    dmma_kernel<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("DMMA  %4d thr/blk x %4d blk: %.2f TFLOP/s\n", threads, blocks,
           512.0 * 16 * iters * blocks * (threads / 32) / (ms * 1e-3) / 1e12);
  }
  // occupancy sweep at one block per SM: how many warps the DMMA pipe needs
  for (int threads : {128, 256, 384, 512}) {
    const int blocks = 148, iters = 20000;
    float ms;
    dmma_kernel<<<blocks, threads>>>(out, 100, 1.0000001, 1e-9);
    cudaEventRecord(e0);
    dmma_kernel<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("DMMA  1 blk/SM x %4d thr (16 independent accumulators/warp): %.2f TFLOP/s\n", threads,
           512.0 * 16 * iters * blocks * (threads / 32) / (ms * 1e-3) / 1e12);
  }
  for (int threads : {128, 256}) {
    chain<1>(out, threads);
    chain<2>(out, threads);
    chain<4>(out, threads);
    chain<6>(out, threads);
    chain<10>(out, threads);
    chain<16>(out, threads);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
