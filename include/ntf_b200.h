/*
 * ntf_b200.h — C ABI of the B200 (sm_100a) NTF hot path.
 *
 * Drop-in boundary for the per-mode update of the reference's ADMoM
 * non-negative CP solver (package `cpadmm`, /root/reference/pkg/src/cpadmm).
 * The reference is pure Python with no FFI; its boundary is the Python call
 * `cpadmm.fit(t, rank, specs=None, config=None) -> FitResult` (solver.py:340).
 * The Python package `paper_1409_2383_b200` mirrors that call and binds the
 * entry points below with ctypes (INTEGRATION.md shows the binding).  Each
 * entry point names the reference function it replaces.
 *
 * Conventions
 *  - All pointers are DEVICE pointers unless stated; no torch types.
 *  - `stream` is a cudaStream_t passed as an opaque pointer.  Every call is
 *    stream-ordered and asynchronous; nothing synchronises the host.
 *  - Tensors are dense, order 3, row-major X[i][j][k] (tensors.py:40-48),
 *    element type NTF_F32 or NTF_F64.  Factors/aux/duals are row-major
 *    fp64 (rows x R), R <= NTF_MAX_RANK.
 *  - Return value: NTF_OK or an NTF_ERR_* code; `ntf_last_error()` gives a
 *    thread-local message.  Device-side numerical failures (Cholesky
 *    breakdown, non-finite projection input) are reported through the
 *    int status word the caller passes in and map to the reference's
 *    InvalidPenaltyError (solver.py:31-32, 167-175) and ValueError
 *    (constraints.py:108-109).
 *  - Reentrant: no global mutable state besides the thread-local message;
 *    a plan owns its own scratch memory.
 */
#ifndef NTF_B200_H
#define NTF_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NTF_ABI_VERSION 2
#define NTF_MAX_ORDER 4
/* Largest CP rank (the reference only requires rank >= 1, solver.py:355-356).
 * Ranks above 128 run the fp64-arithmetic MTTKRP in 128-column chunks, the row
 * update and the ridge Cholesky against L held in global memory (L2). */
#define NTF_MAX_RANK 256

typedef void* ntf_stream_t;

enum ntf_status {
  NTF_OK = 0,
  NTF_ERR_INVALID = 1,     /* bad argument (ValueError in the shim)          */
  NTF_ERR_NOT_PD = 2,      /* InvalidPenaltyError                           */
  NTF_ERR_NONFINITE = 3,   /* ValueError: non-finite entries                */
  NTF_ERR_CUDA = 4,        /* CUDA runtime/launch failure (RuntimeError)     */
  NTF_ERR_UNSUPPORTED = 5  /* configuration outside the kernels' envelope    */
};

enum ntf_dtype { NTF_F32 = 0, NTF_F64 = 1 };

/* MTTKRP engine selection (NTF_ENGINE_AUTO picks by rank and dtype). */
enum ntf_engine { NTF_ENGINE_AUTO = 0, NTF_ENGINE_CUDA_CORE = 1, NTF_ENGINE_TCGEN05 = 2 };

int ntf_abi_version(void);
const char* ntf_last_error(void);

/* ---------------------------------------------------------------------------
 * Dense MTTKRP, one mode:  out = X_(mode) * KR(companions, highest first).
 * Replaces tensors.mttkrp_factors dense branch (tensors.py:254-262), i.e.
 * khatri_rao (tensors.py:203-220) + the unfolding GEMM (tensors.py:262),
 * without the unfolding copy (tensors.py:63-71) or the materialised KR.
 * out: M x R fp64 (M = dims[mode-1]).  `workspace` holds split partials.
 * ------------------------------------------------------------------------- */
size_t ntf_mttkrp_workspace_bytes(int mode, int x_dtype, int64_t I, int64_t J, int64_t K, int R,
                                  int engine);
int ntf_mttkrp(int mode, int x_dtype, const void* X, int64_t I, int64_t J, int64_t K,
               const double* A, const double* B, const double* C, int R, double* out,
               void* workspace, size_t workspace_bytes, int engine, ntf_stream_t stream);

/* Gram matrix G = F^T F (R x R fp64) — the per-factor term of
 * solver.companion_gram (solver.py:196-204) / tensors.gram_hadamard
 * (tensors.py:228-240).  Deterministic fixed-order reduction. */
size_t ntf_gram_workspace_bytes(int64_t rows, int R);
int ntf_gram(const double* F, int64_t rows, int R, double* G, void* workspace,
             size_t workspace_bytes, ntf_stream_t stream);

/* Sum of squares over a dense tensor and of its residual against a Kruskal
 * model: out2[0] = sum x^2, out2[1] = sum (x - [[A,B,C]])^2, fp64
 * accumulation, fixed-order reduction.  Replaces DenseTensor.norm
 * (tensors.py:57-61) and tensors.rfe dense (tensors.py:282-290,
 * reconstruct tensors.py:276-279).  A/B/C may be NULL (only out2[0]). */
size_t ntf_sq_error_workspace_bytes(int64_t I, int64_t J, int64_t K);
int ntf_sq_error(int x_dtype, const void* X, int64_t I, int64_t J, int64_t K, const double* A,
                 const double* B, const double* C, int R, double* out2, void* workspace,
                 size_t workspace_bytes, ntf_stream_t stream);

/* Sparse COO MTTKRP, one mode: replaces tensors.mttkrp_factors' sparse branch
 * (tensors.py:263-273) for order 3 or 4.  Entries sorted lexicographically
 * (idx [nnz][order]); perm: the entries ordered by index `mode` (stable; NULL
 * for mode 1), rowptr: its row segments [dims[mode-1]+1]; factors[order]
 * (the mode's own entry unused).  Per (row, column) the products of the
 * companion rows (highest mode first) times val are summed in entry order,
 * as np.add.at: bitwise equal to the reference.  out: dims[mode-1] x R fp64. */
int ntf_mttkrp_coo(int order, const int64_t* dims, int mode, int64_t nnz, const int64_t* idx,
                   const double* vals, const int64_t* perm, const int64_t* rowptr,
                   const double* const* factors, int R, double* out, ntf_stream_t stream);

/* COO sum of squares and model residual by the Gram identity
 * (CooTensor.norm tensors.py:114-115, tensors.rfe sparse tensors.py:291-301):
 * out2[0] = sum vals^2, out2[1] = ||X||^2 - 2<X, W> + sum(Hadamard of the
 * factor Grams); factors may be NULL (only out2[0]). */
size_t ntf_sq_error_coo_workspace_bytes(int64_t nnz);
int ntf_sq_error_coo(int order, const int64_t* dims, int64_t nnz, const int64_t* idx,
                     const double* vals, const double* const* factors, int R, double* out2,
                     void* workspace, size_t workspace_bytes, ntf_stream_t stream);

/* Khatri-Rao pair out[a*nb + b][r] = Fa[a][r] * Fb[b][r] (tensors.khatri_rao,
 * tensors.py:203-220, for two factors): the merged factor of an order-4
 * tensor's reshaped views (e.g. the model [A, B, C o D] of X as I x J x KL). */
int ntf_khatri_rao_pair(const double* Fa, int64_t na, const double* Fb, int64_t nb, int R, double* out,
                        ntf_stream_t stream);

/* Synthetic dense tensor in HBM (stands in for the reference
 * generator bench.py:34-46: U[0,1) true factors, X = [[A,B,C]] + Gaussian
 * noise).  Writes the box [lo, hi) of the full dims[0] x dims[1] x dims[2]
 * tensor, row-major, to `out` (x_dtype):
 *   x[i,j,k] = sum_r (A[i,r] B[j,r]) C[k,r]  (sequential in r, fp64)
 *            + sigma * z(e),  e = (i dims[1] + j) dims[2] + k,
 * z = Box-Muller over SplitMix64 words 2e+1, 2e+2 of `key`, with ln and cos
 * as fixed polynomials in correctly rounded arithmetic: every element is a
 * pure function of its global index, so ranks generate their own slabs and
 * the bytes equal the host restatement's (oracle/synth_oracle.c).  A, B, C
 * are the full device factors (dims[m] x R fp64). */
int ntf_synth_dense(int x_dtype, void* out, const int64_t* dims, const int64_t* lo, const int64_t* hi,
                    const double* A, const double* B, const double* C, int R, double sigma,
                    uint64_t key, ntf_stream_t stream);

/* ---------------------------------------------------------------------------
 * Solver plan: device-resident ADMoM outer iterations for one order-3 or
 * order-4 tensor (dense order 3 sharded or not; dense order 4 and sparse
 * COO of either order on one GPU) and a constraint per mode.  Replaces solver.iterate
 * (solver.py:295-327) and the per-iteration part of solver.fit
 * (solver.py:375-387): Gauss-Seidel sweeps of _factor_update_core
 * (solver.py:207-219), aux/dual updates fused into each mode's last sweep
 * (as mesh.py:220-223), residuals (solver.py:247-255), check_stop
 * (solver.py:258-269) and adapt_penalties (solver.py:272-292), with the
 * penalties, histories and stop flag kept on the device.
 * ------------------------------------------------------------------------- */
typedef struct ntf_plan ntf_plan;

enum ntf_format { NTF_FORMAT_DENSE = 0, NTF_FORMAT_COO = 1 };

enum ntf_constraint {
  NTF_CONSTRAINT_NONNEG = 0,
  NTF_CONSTRAINT_CARD = 1,
  NTF_CONSTRAINT_ROW_STOCHASTIC = 2
};

typedef struct ntf_plan_desc {
  /* tensor order: 3, or 4 (dense, single GPU: each order-4 MTTKRP runs as an
   * order-3 one on a reshaped view, I x J x (K L) for modes 1-2 and
   * (I J) x K x L for modes 3-4, with the Khatri-Rao pair of the merged
   * modes formed on the device); 0 means 3.  Arrays below hold `order`
   * entries. */
  int order;
  /* problem: the tensor as seen by each mode's MTTKRP.  Single GPU: all
   * entries are the whole tensor.  Sharded (P GPUs, order 3):
   * entry m is this rank's mode-m slab (X[I_p,:,:], X[:,J_p,:], X[:,:,K_p])
   * and x_dims[m] its extents; mode-m rows [row_offset[m], +row_count[m]) of
   * the factor are owned here (blocks.PartitionPlan.uniform, blocks.py:47-61). */
  int x_dtype;
  const void* x_mode[4];
  int64_t x_dims[4][4];
  int64_t dims[4];          /* full extents (factor row counts)             */
  int64_t row_offset[4];
  int64_t row_count[4];
  int rank;
  int engine;               /* ntf_engine                                   */
  int fuse_gram;            /* 1: refresh grams[m] inside the mode update   */
  /* SolverConfig (solver.py:35-49) */
  double eps_abs, eps_rel, mu, tau_incr, tau_decr;
  int inner_sweeps;
  int adapt;
  /* state, caller-owned device buffers (fp64 row-major) */
  double* factors[4];       /* dims[m] x R  working factors (replicated)    */
  double* aux[4];           /* row_count[m] x R  auxiliary copies (owned)   */
  double* duals[4];         /* row_count[m] x R  scaled duals Y (owned)     */
  double* grams[4];         /* R x R        F_m^T F_m                       */
  double* colmax;           /* [order][R]   max_i |F_m[i][r]| (W scales of the
                               tensor-core MTTKRP), kept like the grams     */
  double* rho;              /* [order]      per-mode penalties              */
  double* norm_acc;         /* [order][5][2] per-mode scaled sums of squares of
                               the last sweep, (scale, ssq) with value
                               scale^2*ssq (nrm2-style, no under/overflow):
                               F-aux, aux-aux_prev, F, aux, Y               */
  const double* norm_all;   /* NULL, or [norm_parts][10 order]: every shard's
                               norm_acc gathered in rank order (P>1); the
                               finalize merges them instead of norm_acc     */
  int norm_parts;           /* rows of norm_all (ignored when NULL)         */
  /* per-iteration outputs: row `it` written by iteration `it` */
  int64_t history_capacity; /* rows available in the history buffers        */
  double* resid_history;    /* [cap][2 order]  primal[order], dual[order]   */
  double* rho_history;      /* [cap][order]  rho after adaptation           */
  int* counters;            /* [4]: iteration, stop flag, status, spare     */
  /* Verification hook: when non-NULL, iteration `it` sets rho to row `it`
   * of this [cap][order] device array instead of applying adapt_penalties, so a
   * trajectory can be replayed under the reference's penalty sequence. */
  const double* rho_schedule;
  /* Constraint of each mode (reference constraints.py, solver.py:182-193):
   * NTF_CONSTRAINT_NONNEG (0, the default of a zero-initialised desc),
   * NTF_CONSTRAINT_CARD with card[m] the global nonzero budget (single-GPU
   * plans only), NTF_CONSTRAINT_ROW_STOCHASTIC (rows on the simplex, the
   * equality-constrained row solve). */
  int constraint[4];
  int64_t card[4];
  /* Tensor format: NTF_FORMAT_DENSE (x_mode/x_dims as above), or
   * NTF_FORMAT_COO (reference CooTensor, tensors.py:84-132; single GPU, fp64
   * values, x_dtype = NTF_F64, x_mode[m] = coo_vals, x_dims[m] = dims):
   * nnz entries sorted lexicographically, coo_idx [nnz][order] int64, and per
   * mode m a stable order of the entries by index m (coo_perm[m], NULL for
   * mode 1 = the entry order) with its row segments coo_rowptr[m]
   * [dims[m]+1]. */
  int x_format;
  int64_t nnz;
  const int64_t* coo_idx;
  const double* coo_vals;
  const int64_t* coo_perm[4];
  const int64_t* coo_rowptr[4];
} ntf_plan_desc;

int ntf_plan_create(const ntf_plan_desc* desc, ntf_plan** out);
/* Plans draw device memory from the device's default stream-ordered pool and
 * keep it mapped after release (repeated fits of one geometry re-use it).
 * This returns every unused pool byte to the device (e.g. before allocating
 * a large tensor outside the library).  Synchronises the device. */
int ntf_trim_device_pool(void);
/* Bytes the pool holds mapped but unused right now (released plans leave
 * their memory there): the next plan allocates from them first, so they count
 * as free HBM although cudaMemGetInfo reports them as taken. */
int ntf_device_pool_idle_bytes(size_t* bytes);
/* Column maxima out[r] = max_i |F[i][r]| (sharded runs refresh colmax[m]
 * with this after gathering a factor, as they refresh grams[m]). */
int ntf_colmax(const double* F, int64_t rows, int R, double* out, ntf_stream_t stream);
/* The tensor behind desc->x_mode[] was overwritten in place with new values
 * (same shape and dtype): rebuild the plan's derived copies of it (the
 * tensor-core block images) on `stream`, so the plan, its buffers and its
 * captured graph serve another fit.  Follows reference solver.fit
 * (solver.py:340-403) being called again on new data. */
int ntf_plan_refresh_tensor(ntf_plan* plan, ntf_stream_t stream);
/* Recompute grams[m] from factors[m] (after the caller (re)initialises state). */
int ntf_plan_sync_grams(ntf_plan* plan, ntf_stream_t stream);
/* Enqueue `n_iters` outer iterations.  Iterations after the stop flag is set
 * are no-ops (kernels observe the flag), so a chunk may be enqueued ahead.
 * use_graph != 0 replays one captured outer iteration (CUDA graph). */
int ntf_plan_run(ntf_plan* plan, int n_iters, int use_graph, ntf_stream_t stream);
/* Single per-mode update, for tests and the sharded engine:  mode 1..3,
 * last_sweep != 0 also applies the projection, dual step and norm partials. */
int ntf_plan_mode_update(ntf_plan* plan, int mode, int last_sweep, ntf_stream_t stream);
/* Close one outer iteration after the sweeps: residuals, stop test, adaptation. */
int ntf_plan_finalize(ntf_plan* plan, ntf_stream_t stream);
/* Optional per-launch timing: when enabled, the plan records CUDA events
 * around every MTTKRP and every row-update launch of an outer iteration (also
 * inside the captured graph; the plain and the instrumented graph are cached
 * separately, so toggling costs nothing after the first capture of each).
 * ntf_plan_kernel_times writes, for the most recent instrumented iteration,
 * 2 floats (MTTKRP ms, update ms) per mode update in sweep order and returns
 * how many floats were written (or a negative status). */
int ntf_plan_set_timing(ntf_plan* plan, int enable);
int ntf_plan_kernel_times(ntf_plan* plan, float* ms_out, int capacity);
void ntf_plan_destroy(ntf_plan* plan);

/* ---- Row all-gather over NVLink peer memory (sharded engine) -------------
 * Replaces the broadcast of updated row blocks after every block-row mode
 * update (reference blocks.py:171-196, mesh.py:149-237; the centralized
 * equivalent is the factor assignment in solver.iterate, solver.py:305-310).
 * Every rank allocates one peer buffer per factor (ntf_peer_alloc), exchanges
 * the 64-byte IPC handles out of band and maps the peers' buffers
 * (ntf_peer_open).  ntf_peer_gather then pushes the caller's owned rows of
 * `full` into every peer's buffer with P2P stores, waits (at most timeout_ns,
 * then writes NTF_PEER_TIMEOUT to *status) for every rank's rows to arrive in
 * its own buffer and copies them into `full`.  One kernel, graph-capturable;
 * every rank must issue the same sequence of gathers per buffer with the
 * same `ctas`.  The kernel's CTAs spin-wait on the arrivals of every rank's
 * CTAs, so `ctas` is bounded by what is co-resident on the device
 * (occupancy x SM count; larger values are rejected).  A gather finding
 * *status already set does nothing (no pushes, no arrivals): after a timeout
 * the caller checks the status word and aborts the fit on every rank. */
#define NTF_MAX_PEERS 8
#define NTF_PEER_TIMEOUT 6
typedef struct ntf_peer_gather_desc {
  int nranks;                            /* 1..NTF_MAX_PEERS                   */
  int me;                                /* caller's rank                      */
  int R;
  int ctas;                              /* CTAs per rank, same on all ranks   */
  int64_t row_offset[NTF_MAX_PEERS + 1]; /* rank q owns rows [off[q], off[q+1]) */
  double* full;                          /* local factor, off[nranks] x R fp64 */
  void* peer_base[NTF_MAX_PEERS];        /* rank q's peer buffer, mapped here  */
  int* status;                           /* device int, may be NULL            */
  int64_t timeout_ns;
} ntf_peer_gather_desc;
size_t ntf_peer_buffer_bytes(int64_t rows, int R);
/* cudaMalloc'd, zeroed; handle_out receives 64 bytes (cudaIpcMemHandle_t). */
int ntf_peer_alloc(size_t bytes, void** base_out, void* handle_out);
int ntf_peer_open(const void* handle, void** base_out);
int ntf_peer_close(void* base);
int ntf_peer_free(void* base);
int ntf_peer_gather(const ntf_peer_gather_desc* desc, ntf_stream_t stream);
/* Every rank's gather in ONE cooperative launch on the current device,
 * descs[q] being rank q's (all ranks' buffers and factors on this device).
 * Ranks that wait on one another may not be separate launches on one GPU
 * (nothing makes them co-resident); this is how the protocol runs with all
 * ranks live on a single GPU (tests, single-process emulation of P ranks). */
int ntf_peer_gather_group(const ntf_peer_gather_desc* descs, int nranks, ntf_stream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* NTF_B200_H */
