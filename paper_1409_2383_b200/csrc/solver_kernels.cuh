// Declarations for the per-mode update / Gram / finalize / norm kernels.
#pragma once

#include <algorithm>

#include "common.cuh"

namespace ntf {

struct FactorUpdateParams {
  int mode;                 // 1..3
  int R;
  int64_t rows;             // owned rows
  int64_t row_offset;       // first owned row within the full factor
  const double* mtt;        // [splits][rows][R] MTTKRP partials
  int splits;               // partials of rows < tail_row0
  int64_t tail_row0;        // rows >= tail_row0 have splits_tail partials
  int splits_tail;
  const double* Lg;         // ridge factor from ridge_factor_kernel
  const double* rho;        // device [3]
  double* F;                // full factor (rows written at row_offset)
  double* aux;              // owned rows
  double* dual;             // owned rows
  int last_sweep;
  int fuse_gram;
  double* norm_partials;    // [blocks][5][scale, ssq] (last sweep)
  double* gram_partials;    // [blocks][R][R] (fuse_gram)
  unsigned long long* colmax_bits;  // [R] running max |F[:, r]| as IEEE bits (fuse_gram)
  int* gram_pending;        // set to 1 (fuse_gram): partials await the next MTTKRP's ridge CTA
  int ridge_in_pred;        // 1: Lg comes from the preceding kernel (read after pdl_wait)
  int* status;
  const int* stop_flag;
  int debug;                // profiling only (NTF_UPD_DEBUG)
  // constraint of this mode (reference constraints.py): 0 nonneg, 1 nonneg
  // with a global cardinality budget (last sweep writes v = F + Y/rho to
  // cand; card_select/card_apply finish the projection), 2 row-stochastic
  // (equality-constrained row solve, per-row simplex projection)
  int kind;
  double* cand;             // [rows][R] (kind 1)
};

constexpr int kConstraintNonneg = 0, kConstraintCard = 1, kConstraintRowStochastic = 2;

// Cardinality projection (constraints.py:95-102) of a mode's owned rows:
// card_select finds the c-th largest clamped value T and the index cut among
// its ties (stable, row-major order); card_apply then does the aux / dual
// step (solver.py:311-317) with that projection and the norm partials.
// sel: [2] uint64 {T bits, idx_cut}.
// Khatri-Rao pair of two factors for the order-4 views (rows a*nb + b =
// Fa[a] * Fb[b]); cm: view column maxima [3][R] filled from the factors'
// maxima (cm_src[3] pointers, the merged view mode as the product of two),
// and cm_zero ([R], may be NULL) zeroed for the row update that follows.
struct KrMergeParams {
  const double* Fa;
  int64_t na;
  const double* Fb;
  int64_t nb;
  int R;
  double* out;
  int merged_mode;          // view mode (0..2) whose factor is out
  const double* cm_src[3];  // per view mode: factor maxima (merged: cm_src[mm] x cm_src2)
  const double* cm_src2;
  double* cm_view;          // [3][R]
  double* cm_zero;
  const int* stop_flag;
};
cudaError_t kr_merge_launch(const KrMergeParams& p, cudaStream_t stream);

cudaError_t card_select_launch(const double* cand, int64_t n, int64_t card, unsigned long long* sel,
                               const int* stop_flag, cudaStream_t stream);
cudaError_t card_apply_launch(const FactorUpdateParams& p, const unsigned long long* sel,
                              cudaStream_t stream);

struct FinalizeParams {
  const double* norm_acc;   // [parts][order][5][scale, ssq]
  int norm_parts;           // shards whose norms are merged (1 unsharded)
  int order;                // 3 or 4
  double* rho;              // [order] in/out
  int64_t dims[4];
  int R;
  double eps_abs, eps_rel, mu, tau_incr, tau_decr;
  int adapt;
  int64_t history_capacity;
  double* resid_history;    // [cap][2 * order]
  double* rho_history;      // [cap][order]
  int* counters;            // [0] iteration, [1] stop flag
  const double* rho_schedule;  // optional [cap][order] replayed penalties
};

struct RidgeParams {
  int mode, R;
  const double* Ga;         // companion Grams (highest mode first)
  const double* Gb;
  const double* Gc;         // third companion (order-4 tensors), else NULL
  const double* rho;        // device [order]
  double* L;                // out: [R*R] lower factor + [R] 1/diag
  int* status;
  const int* stop_flag;
};

int factor_update_blocks(int64_t rows, int R);
size_t ridge_factor_smem(int R);
size_t ridge_buffer_doubles(int R);
cudaError_t ridge_factor_launch(const RidgeParams& p, cudaStream_t stream);
size_t factor_update_smem(int R);
cudaError_t factor_update_prepare(int R);
cudaError_t factor_update_launch(const FactorUpdateParams& p, cudaStream_t stream);
// grams[m] = sum of the update blocks' Gram partials; norm_acc[m] likewise
cudaError_t gram_reduce_launch(const double* part, int nb, int R, double* G, const int* stop_flag,
                               cudaStream_t stream);
cudaError_t norm_reduce_launch(const double* part, int nb, double* out, const int* stop_flag,
                               cudaStream_t stream);

size_t gram_workspace_bytes(int64_t rows, int R);
cudaError_t gram_launch(const double* F, int64_t rows, int R, double* G, double* ws,
                        cudaStream_t stream);

cudaError_t finalize_launch(const FinalizeParams& p, cudaStream_t stream);

size_t sq_error_workspace_bytes(int64_t I, int64_t J, int64_t K, int R);
cudaError_t sq_error_launch(int x_dtype, const void* X, int64_t I, int64_t J, int64_t K,
                            const double* A, const double* B, const double* C, int R, double* out2,
                            void* ws, cudaStream_t stream);

}  // namespace ntf
