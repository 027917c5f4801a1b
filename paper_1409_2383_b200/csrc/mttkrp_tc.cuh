// tcgen05 (5th-gen tensor core) dense MTTKRP with split-precision TF32 for
// ranks where the CUDA-core contraction leaves the HBM roof.
#pragma once

#include "common.cuh"

namespace ntf {

struct MttkrpTCLaunch {
  int mode;
  int64_t M, Q;
  int n_mtiles, splits;
  int64_t n_chunks, chunks_per_split;
  int n_pad;          // MMA N (rank padded)
  int smem_bytes;
  int threads;
};

bool mttkrp_tc_supported(int x_dtype, int R);
bool mttkrp_tc_auto(int x_dtype, int R);
MttkrpTCLaunch mttkrp_tc_plan(int mode, int x_dtype, int64_t I, int64_t J, int64_t K, int R);
size_t mttkrp_tc_workspace_bytes(const MttkrpTCLaunch& L, int R);
cudaError_t mttkrp_tc_prepare(const MttkrpTCLaunch& L);
cudaError_t mttkrp_tc_launch(int mode, int x_dtype, const void* X, int64_t I, int64_t J, int64_t K,
                             const double* A, const double* B, const double* C, int R,
                             const MttkrpTCLaunch& L, double* ws, const int* stop_flag,
                             cudaStream_t stream);

}  // namespace ntf
