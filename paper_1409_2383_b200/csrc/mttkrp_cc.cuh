// CUDA-core dense MTTKRP: parameter block and host dispatch declarations.
#pragma once

#include <algorithm>
#include <cstdint>

#include "common.cuh"

namespace ntf {

struct MttkrpCCParams {
  const void* X;
  int64_t M;            // output rows
  int64_t Q;            // reduction length (< 2^31)
  int64_t K;            // contiguous extent (KIND_Q index split)
  int64_t s_m, s_o;     // element strides of m and o
  const double* Fhi;    // KR slow factor (indexed by q / lo_extent)
  const double* Flo;    // KR fast factor (indexed by q % lo_extent)
  uint32_t lo_extent, hi_extent;
  int R, R_pad;         // R: all columns (factor / output row stride); R_pad: of one 128-column chunk
  int64_t n_chunks, chunks_per_split;
  int stage_bytes, max_hi;
  int n_stages;         // fp64 pipeline: stage ring depth (3, or 2 where 3 do not fit)
  double* ws;           // [groups][M][R] fp64 partials (one per cluster)
  const int* stop_flag;
};

struct MttkrpCCLaunch {
  int TM, TR, R_pad, threads;  // of one column chunk (<= 128 columns)
  int col_chunks;               // ceil(R / 128): grid z
  int n_mtiles, splits, cluster, groups;
  int64_t M, Q, n_chunks, chunks_per_split;
  int stage_bytes, max_hi, smem_bytes, stages;
  bool vec;
};

MttkrpCCLaunch mttkrp_cc_plan(int mode, int x_dtype, int64_t I, int64_t J, int64_t K, int R);
size_t mttkrp_cc_workspace_bytes(const MttkrpCCLaunch& L, int R);
cudaError_t mttkrp_cc_prepare(int mode, int x_dtype, const MttkrpCCLaunch& L);
cudaError_t mttkrp_cc_launch(int mode, int x_dtype, const void* X, int64_t I, int64_t J, int64_t K,
                             const double* A, const double* B, const double* C, int R,
                             const MttkrpCCLaunch& L, double* ws, const int* stop_flag,
                             cudaStream_t stream);
// out[m] = sum of the partials of row m: `groups` of them for m < tail_row0,
// `groups_tail` after (the tensor-core engine's ragged last tile)
cudaError_t mttkrp_reduce_launch(const double* ws, int groups, int64_t M, int R, double* out,
                                 const int* stop_flag, cudaStream_t stream,
                                 int64_t tail_row0 = INT64_MAX, int groups_tail = 0);

}  // namespace ntf
