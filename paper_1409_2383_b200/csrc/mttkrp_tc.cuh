// tcgen05 (5th-gen tensor core) dense MTTKRP for fp32 tensors, exact
// fixed-point slicing (see mttkrp_tc.cu for the numerics).
#pragma once

#include <cuda.h>
#include <cuda_fp16.h>

#include "common.cuh"

namespace ntf {

// fp16 fixed-point split of an fp32 tensor: X ~= xscale * (S0 + S1),
// S0 integers |S0| <= 2048, S1 multiples of 2^-11 with |S1| <= 0.5, xscale a
// power of two (2^(e-11), e = ceil(log2 max|X|)), stored as ONE mode's block
// image (mttkrp_tc.cu: image_split_kernel): every X block a CTA streams is a
// contiguous no-swizzle UMMA image, and a CTA's blocks are consecutive.
// Built once per (tensor, mode plan).
struct TcTensor {
  unsigned char* img = nullptr;
  size_t img_bytes = 0;
  double* xscale = nullptr;  // device scalar
  int mode = 0;
  int64_t dims[3] = {0, 0, 0};
  const float* src = nullptr;  // the tensor the image was split from
};

struct MttkrpTCLaunch;
// same_values: an image already split (on this stream) from the same tensor
// values; its max|X| is reused instead of another pass over the tensor.
cudaError_t tc_tensor_create(const MttkrpTCLaunch& L, const float* X, const int64_t dims[3],
                             TcTensor* out, cudaStream_t stream, const TcTensor* same_values = nullptr);
void tc_tensor_destroy(TcTensor* t);
// Re-split t.src into the existing image (the tensor's values changed in place).
cudaError_t tc_tensor_fill(const MttkrpTCLaunch& L, const TcTensor& t, cudaStream_t stream,
                           const TcTensor* same_values = nullptr);

constexpr int kTcMaxSplits = 160;  // CTAs per m-tile
constexpr int kTcMaxXStages = 32;  // X ring slots

struct MttkrpTCLaunch {
  CUtensorMap map_full, map_tail, map_w;  // cg == 2: the image's blocks and the W slices (mttkrp_tc_bind)
  int mode;
  int R, N;                 // rank and MMA N (R rounded up to 16)
  int np;                   // columns of the T0 / T1 slice ranges and of ACC0 (N, or N - 8 packed)
  int64_t M, Q;
  int n_mtiles;             // m-tiles (cg == 2: even)
  int cg;                   // CTAs per MMA group: 2 = CTA pairs (tcgen05 cta_group::2)
  int n_full, splits;       // full 128-row tiles and CTAs per full tile
  int splits_tail;          // CTAs of the ragged last tile (0: none)
  int tm;                   // rows per m-tile (a multiple of 8)
  int r8_full, r8_tail;     // stored rows of a full / the ragged last tile (multiples of 8)
  int ct;                   // 8-element chunks stored for the last l block
  int64_t tile_bytes;       // image bytes of one full m-tile
  size_t img_bytes;         // image bytes of the whole mode
  int l_ext, n_o, n_lb;     // l extent, o extent, 64-wide l blocks
  int G, n_g;               // l blocks per unit (one TMEM drain), groups
  int threads, smem_bytes;
  int x_stages, h_stages;
  int slot_ks;              // K steps (16 l values, 64 tm bytes) per X ring slot
  int stage_bytes;          // X ring slot stride, 128 B aligned
  int tmem_cols;
  uint32_t ub_full[kTcMaxSplits + 1];  // unit range of each CTA of a full tile
  uint32_t ub_tail[kTcMaxSplits + 1];
  double* wscale;           // [2 * N] device: column maxima for one-shot calls
  unsigned char* wsl;       // [n_lb][3][N][128 B] W slices of F_lo (per launch)
  float2* hpair;            // [n_o][N] F_hi rows as scaled fp32 pairs (per launch)
  bool bound;
};

bool mttkrp_tc_supported(int x_dtype, int R);
bool mttkrp_tc_auto(int x_dtype, int R);
bool mttkrp_tc_shape_ok(int mode, int64_t I, int64_t J, int64_t K);
MttkrpTCLaunch mttkrp_tc_plan(int mode, int x_dtype, int64_t I, int64_t J, int64_t K, int R);
size_t mttkrp_tc_workspace_bytes(const MttkrpTCLaunch& L, int R);
cudaError_t mttkrp_tc_prepare(const MttkrpTCLaunch& L);
// Check the image matches the plan and allocate the per-launch buffers.
cudaError_t mttkrp_tc_bind(MttkrpTCLaunch& L, const TcTensor& t);
void mttkrp_tc_unbind(MttkrpTCLaunch& L);
// colmax3: [3][R] per-factor column maxima of |F| (NULL: computed here)
cudaError_t mttkrp_tc_launch(MttkrpTCLaunch& L, const TcTensor& t, const double* A,
                             const double* B, const double* C, const double* colmax3, double* ws,
                             const int* stop_flag, cudaStream_t stream);
// diagnostics (NTF_TC_DEBUG & 256): per-CTA globaltimer stamps of the last launch
int tc_debug_read_times(unsigned long long* host, int ctas);
// out[r] = max_i |F[i][r]|
cudaError_t colmax_launch(const double* F, int64_t rows, int R, double* out, cudaStream_t stream);

}  // namespace ntf
