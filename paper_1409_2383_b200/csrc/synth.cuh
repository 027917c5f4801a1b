// Counter-based synthetic NTF tensors generated in HBM.
#pragma once

#include "common.cuh"

namespace ntf {

struct SynthBox {
  int64_t dims[3];  // full tensor extents (the element counter is global)
  int64_t lo[3];    // box [lo, hi) of the full tensor, written row-major
  int64_t hi[3];
};

cudaError_t synth_dense_launch(int x_dtype, void* out, const SynthBox& box, const double* A,
                               const double* B, const double* C, int R, double sigma, uint64_t key,
                               cudaStream_t stream);

}  // namespace ntf
