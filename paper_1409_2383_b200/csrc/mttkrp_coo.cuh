// Sparse COO MTTKRP and squared error (reference tensors.py:84-132, 263-273,
// 291-301), fp64 on the CUDA cores.
#pragma once

#include "common.cuh"

namespace ntf {

// A COO tensor on the device: entries sorted lexicographically (the
// reference's CooTensor order), plus per mode a stable permutation of the
// entries by that mode's index and the row segments of that order.
struct CooView {
  int order;                 // 3 or 4 (0 means 3)
  int64_t dims[4];
  int64_t nnz;
  const int64_t* idx;        // [nnz][order]
  const double* vals;        // [nnz]
  const int64_t* perm[4];    // [nnz] entries ordered by index m (ties: entry order)
  const int64_t* rowptr[4];  // [dims[m] + 1] segments of perm[m]
};

// out[i][r] = sum over the entries of row i (entry order) of
//   F_c0[i_c0][r] * F_c1[i_c1][r] * val   (highest companion mode first,
// the association of tensors.py:266-270), accumulated sequentially per
// (row, column) exactly like np.add.at: bitwise equal to the reference.
// F: the order's factors (F[3] unused for order 3).
cudaError_t mttkrp_coo_launch(const CooView& t, int mode, const double* const F[4], int R,
                              double* out, const int* stop_flag, cudaStream_t stream);

// out2 = {sum x^2, ||X - [[A,B,C]]||^2 by the Gram identity
//   ||X||^2 - 2 <X, W> + sum((A^T A) * (B^T B) * (C^T C))}  (tensors.py:291-301)
// in fixed-order fp64 reductions.  ws: coo_sq_error_workspace_bytes.
size_t coo_sq_error_workspace_bytes(int64_t nnz, int R);
cudaError_t coo_sq_error_launch(const CooView& t, const double* const F[4], int R, double* out2,
                                void* ws, cudaStream_t stream);

}  // namespace ntf
