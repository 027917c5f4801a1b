// Shared device helpers for the B200 NTF hot path (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <utility>

#include "../../include/ntf_b200.h"

namespace ntf {

constexpr int kWarp = 32;

// Tuning and diagnostic environment knobs (tile geometry overrides, the
// tcgen05 kernel's skip masks and wait counters, the row update's debug
// flags, plan timing) exist only in NTF_DIAG builds made by tools/; the
// release library never reads them, so no environment setting can change
// what a timed kernel does.
inline const char* diag_env(const char* name) {
#ifdef NTF_DIAG
  return getenv(name);
#else
  (void)name;
  return nullptr;
#endif
}

#ifdef NTF_DIAG
constexpr bool kDiagBuild = true;
#else
constexpr bool kDiagBuild = false;
#endif

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// cp.async with zero-fill when `valid` is false (src-size 0 reads nothing).
template <int BYTES>
__device__ __forceinline__ void cp_async_ca(void* dst, const void* src, bool valid) {
  static_assert(BYTES == 4 || BYTES == 8 || BYTES == 16, "cp.async size");
  const uint32_t d = smem_u32(dst);
  const int n = valid ? BYTES : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(d), "l"(src), "n"(BYTES),
               "r"(n));
}

__device__ __forceinline__ void cp_async_cg16(void* dst, const void* src, bool valid) {
  const uint32_t d = smem_u32(dst);
  const int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(n));
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }

template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Overflow/underflow-safe sum of squares, (scale, ssq) with value
// scale^2 * ssq, as the reference's BLAS nrm2 under np.linalg.norm
// (solver.py:247-255): factor columns driven to ~1e-200 by large penalties
// must not square to zero and fake an exactly consistent split.
struct ScaledSq {
  double scale = 0.0, ssq = 0.0;
  __device__ __forceinline__ void add(double v) {
    const double a = fabs(v);
    if (a == 0.0) return;
    if (a > scale) {
      const double r = scale / a;
      ssq = 1.0 + ssq * r * r;
      scale = a;
    } else {
      const double r = a / scale;
      ssq += r * r;
    }
  }
  __device__ __forceinline__ void merge(double s2, double q2) {
    if (s2 == 0.0) return;
    if (s2 > scale) {
      const double r = scale / s2;
      ssq = q2 + ssq * r * r;
      scale = s2;
    } else {
      const double r = s2 / scale;
      ssq += q2 * r * r;
    }
  }
  __device__ __forceinline__ double norm() const { return scale * sqrt(ssq); }
};

// Device memory of plans and tensor splits comes from the device's default
// stream-ordered pool with a retained release threshold: repeated fit() calls
// reuse already-mapped memory instead of paying cudaMalloc/cudaFree page
// mapping each time.  Allocation and release are ordered on the legacy
// stream; callers synchronise their own streams before release.
inline void retain_pool() {
  static std::once_flag once;
  std::call_once(once, [] {
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  });
}

template <typename T>
inline cudaError_t dev_alloc(T** p, size_t bytes) {
  retain_pool();
  void* v = nullptr;
  cudaError_t e = cudaMallocAsync(&v, bytes, 0);
  if (e == cudaSuccess) e = cudaStreamSynchronize(0);
  *p = static_cast<T*>(v);
  return e;
}

inline void dev_free(void* p) {
  if (p) cudaFreeAsync(p, 0);
}

// Programmatic dependent launch (PDL).  The main-stream chain of a mode
// update (W slices -> MTTKRP -> row update -> ...) is launched with the
// programmatic-serialization attribute: every kernel lets its dependent be
// scheduled at once (pdl_trigger), and each kernel waits for its predecessor
// (pdl_wait: full completion and memory visibility) only before touching
// data that predecessor produced.  Prologues, TMEM allocation and the
// predecessor-independent X stream then overlap the previous kernel.
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

// Allow a kernel the device's whole opt-in dynamic shared memory (less its
// static shared memory) and check `need` fits.  The attribute is a per-kernel
// cap, not a reservation: setting it to the maximum once means plans of
// different sizes that share a kernel instance never undercut each other
// (setting it to each plan's own size let the last plan created win).
inline cudaError_t allow_dyn_smem(const void* kern, size_t need) {
  int dev = 0, optin = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaFuncAttributes fa{};
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, kern);
  if (e != cudaSuccess) return e;
  const int cap = optin - static_cast<int>(fa.sharedSizeBytes);
  if (need > static_cast<size_t>(cap)) return cudaErrorInvalidValue;
  return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
}

// Launches made while this (per host thread) switch is off carry no PDL
// attribute: kernels then serialise on the stream and the griddepcontrol
// instructions are no-ops.  The plan turns it off while it enqueues an
// instrumented iteration, so the CUDA events around each kernel bracket that
// kernel alone.
inline bool& pdl_switch() {
  thread_local bool on = true;
  return on;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t stream, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_switch() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// Error/status flags written by kernels (host reads them back once per run).
enum DeviceStatus : int {
  kDevOk = 0,
  kDevNotPD = 1,      // ridge system not positive definite (InvalidPenaltyError)
  kDevNonFinite = 2,  // non-finite value entering the projection (ValueError)
};

__device__ __forceinline__ void raise_status(int* status, int code) {
  if (status) atomicCAS(status, 0, code);
}

}  // namespace ntf
