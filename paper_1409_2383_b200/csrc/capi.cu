// C ABI (include/ntf_b200.h) and the solver-plan runtime.
//
// The plan owns the launch geometry, scratch memory and a captured CUDA graph
// of one outer iteration: inner_sweeps x 3 x (MTTKRP -> fused ridge/ADMM row
// update) followed by the finalize kernel, i.e. solver.iterate
// (reference solver.py:295-327) with aux/dual fused into each mode's last
// sweep exactly as mesh.py:220-223 does.  Nothing here synchronises the host.
#include <chrono>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>

#include "mttkrp_cc.cuh"
#include "mttkrp_coo.cuh"
#include "mttkrp_tc.cuh"
#include "peer_gather.cuh"
#include "solver_kernels.cuh"
#include "synth.cuh"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  g_err = std::string(where) + ": " + cudaGetErrorString(e);
  return NTF_ERR_CUDA;
}

#define NTF_CUDA_TRY(expr)                              \
  do {                                                  \
    cudaError_t _e = (expr);                            \
    if (_e != cudaSuccess) return cuda_fail(_e, #expr); \
  } while (0)

int check_dims(int mode, int x_dtype, int64_t I, int64_t J, int64_t K, int R) {
  if (mode < 1 || mode > 3) return fail(NTF_ERR_INVALID, "mode must be 1..3");
  if (x_dtype != NTF_F32 && x_dtype != NTF_F64) return fail(NTF_ERR_INVALID, "bad dtype");
  if (I < 1 || J < 1 || K < 1) return fail(NTF_ERR_INVALID, "all extents must be >= 1");
  if (R < 1 || R > NTF_MAX_RANK) return fail(NTF_ERR_UNSUPPORTED, "rank must be in 1..256 (NTF_MAX_RANK)");
  const int64_t Q = mode == 1 ? J * K : (mode == 2 ? I * K : I * J);
  if (Q >= (int64_t(1) << 31)) return fail(NTF_ERR_UNSUPPORTED, "reduction length >= 2^31");
  return NTF_OK;
}

bool tc_ok(int mode, int x_dtype, int64_t I, int64_t J, int64_t K, int R) {
  return ntf::mttkrp_tc_supported(x_dtype, R) && ntf::mttkrp_tc_shape_ok(mode, I, J, K);
}

bool use_tc(int engine, int mode, int x_dtype, int64_t I, int64_t J, int64_t K, int R) {
  if (engine == NTF_ENGINE_CUDA_CORE) return false;
  if (engine == NTF_ENGINE_TCGEN05) return tc_ok(mode, x_dtype, I, J, K, R);
  return ntf::mttkrp_tc_auto(x_dtype, R) && tc_ok(mode, x_dtype, I, J, K, R);
}

// One MTTKRP engine instance for one (mode, shape): geometry + launcher.
struct MttkrpOp {
  bool tc = false;
  bool coo = false;          // sparse COO tensor (mttkrp_coo.cu): one fp64 "split", the whole output
  ntf::CooView cv{};
  const double* f3 = nullptr;  // order-4 COO: the fourth factor
  ntf::MttkrpCCLaunch cc{};
  ntf::MttkrpTCLaunch tcl{};
  const ntf::TcTensor* tct = nullptr;  // fp16 split planes (tensor-core engine)
  int splits() const { return coo ? 1 : (tc ? tcl.splits : cc.groups); }
  // rows from tail_row0() on have splits_tail() partials (ragged last tile)
  int64_t tail_row0() const {
    return !coo && tc && tcl.splits_tail ? static_cast<int64_t>(tcl.n_full) * tcl.tm : INT64_MAX;
  }
  int splits_tail() const { return !coo && tc ? tcl.splits_tail : 0; }
  size_t ws_bytes(int R) const {
    if (coo) return 0;  // sized by the caller from the mode's row count
    return tc ? ntf::mttkrp_tc_workspace_bytes(tcl, R) : ntf::mttkrp_cc_workspace_bytes(cc, R);
  }
};

MttkrpOp make_op(int mode, int x_dtype, int64_t I, int64_t J, int64_t K, int R, int engine) {
  MttkrpOp op;
  op.tc = use_tc(engine, mode, x_dtype, I, J, K, R);
  if (op.tc)
    op.tcl = ntf::mttkrp_tc_plan(mode, x_dtype, I, J, K, R);
  else
    op.cc = ntf::mttkrp_cc_plan(mode, x_dtype, I, J, K, R);
  return op;
}

cudaError_t run_op(MttkrpOp& op, int mode, int x_dtype, const void* X, int64_t I, int64_t J,
                   int64_t K, const double* A, const double* B, const double* C, int R, double* ws,
                   const int* stop, cudaStream_t s, const double* colmax3 = nullptr) {
  if (op.coo) {  // the order's factors follow A, B, C in the plan (D: op.f3)
    const double* F[4] = {A, B, C, op.f3};
    return ntf::mttkrp_coo_launch(op.cv, mode, F, R, ws, stop, s);
  }
  if (op.tc) return ntf::mttkrp_tc_launch(op.tcl, *op.tct, A, B, C, colmax3, ws, stop, s);
  return ntf::mttkrp_cc_launch(mode, x_dtype, X, I, J, K, A, B, C, R, op.cc, ws, stop, s);
}

// Function attributes (dynamic smem opt-in) are set once, outside any capture.
cudaError_t prepare_op(const MttkrpOp& op, int mode, int x_dtype) {
  if (op.coo) return cudaSuccess;
  if (op.tc) return ntf::mttkrp_tc_prepare(op.tcl);
  return ntf::mttkrp_cc_prepare(mode, x_dtype, op.cc);
}

}  // namespace

struct ntf_plan {
  ntf_plan_desc d;
  int order = 3;
  MttkrpOp op[4];
  int blocks[4];
  double* mtt_ws = nullptr;
  double* norm_partials[4] = {};  // [blocks][5][2] per mode
  double* gram_partials[4] = {};  // [blocks][R][R] per mode
  double* card_cand[4] = {};      // [rows][R] (cardinality modes)
  unsigned long long* card_sel[4] = {};  // [2] threshold, index cut
  // order 4: each MTTKRP is an order-3 one on a reshaped view (view 0:
  // I x J x KL for modes 1-2, view 1: IJ x K x L for modes 3-4) with the
  // Khatri-Rao pair of the merged modes (C o D, A o B) formed per update
  int64_t vdims[2][3] = {};
  double* kr[2] = {};   // view 0: KL x R, view 1: IJ x R
  double* vcm[2] = {};  // [3][R] column maxima of each view's factors
  double* gram_ws = nullptr;
  bool any_tc = false;
  cudaStream_t capture_stream = nullptr;
  cudaGraphExec_t graph[2] = {nullptr, nullptr};  // [timing]: plain / with timing events
  // ridge factorisation runs on a side stream concurrently with the MTTKRP
  // Gram reductions (after each update) and the next mode's ridge run there:
  // both only feed the ridge, so neither is on the critical path.
  cudaStream_t side = nullptr;
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr, post_ev = nullptr;
  double* ridge = nullptr;  // [3R*R + R], see ridge_factor_kernel
  // fp16 split planes for the tensor-core engine, one per distinct slab
  ntf::TcTensor tct[4];
  int n_tct = 0;
  // per-launch timing events: 3 per mode update (before MTTKRP, after MTTKRP,
  // after the row update), inner_sweeps * 3 mode updates per iteration
  int timing = 0;
  int n_events = 0;
  int cursor = 0;
  cudaEvent_t* events = nullptr;
};

namespace {

// Inside stream capture an event record must be an *external* node to be
// observable from the host after the graph runs.
cudaError_t record_event(cudaEvent_t ev, cudaStream_t s) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  cudaError_t e = cudaStreamIsCapturing(s, &st);
  if (e != cudaSuccess) return e;
  if (st == cudaStreamCaptureStatusActive)
    return cudaEventRecordWithFlags(ev, s, cudaEventRecordExternal);
  return cudaEventRecord(ev, s);
}

int enqueue_row_update(ntf_plan* pl, int mode, int last, cudaStream_t s, cudaEvent_t* ev);

int enqueue_mode_update(ntf_plan* pl, int mode, int last, cudaStream_t s) {
  const ntf_plan_desc& d = pl->d;
  const int m = mode - 1;
  const int R = d.rank;
  const int N = pl->order;
  const int64_t* xd = d.x_dims[m];
  // companions, highest mode first (solver.py:196-204)
  int comp[3] = {-1, -1, -1};
  for (int q = N - 1, k = 0; q >= 0; --q)
    if (q != m) comp[k++] = q;
  // fork: ridge Cholesky (solver.py:167-175) on the side stream
  ntf::RidgeParams rp{};
  rp.mode = mode;
  rp.R = R;
  rp.Ga = d.grams[comp[0]];
  rp.Gb = d.grams[comp[1]];
  rp.Gc = N == 4 ? d.grams[comp[2]] : nullptr;
  rp.rho = d.rho;
  rp.L = pl->ridge;
  rp.status = d.counters + 2;
  rp.stop_flag = d.counters + 1;
  NTF_CUDA_TRY(cudaEventRecord(pl->fork_ev, s));
  NTF_CUDA_TRY(cudaStreamWaitEvent(pl->side, pl->fork_ev, 0));
  NTF_CUDA_TRY(ntf::ridge_factor_launch(rp, pl->side));
  NTF_CUDA_TRY(cudaEventRecord(pl->join_ev, pl->side));
  cudaEvent_t* ev = nullptr;
  if (pl->timing && pl->events) {
    ev = pl->events + 3 * pl->cursor;
    pl->cursor = (pl->cursor + 1) % (pl->n_events / 3);
    NTF_CUDA_TRY(record_event(ev[0], s));
  }
  if (N == 4 && !pl->op[m].coo) {
    // order 4: Khatri-Rao pair of the merged modes, then the order-3 MTTKRP
    // of the view (modes 1, 2: I x J x KL with C o D; 3, 4: IJ x K x L with A o B)
    const int v = m < 2 ? 0 : 1;
    const int vmode = m == 0 ? 1 : (m == 3 ? 3 : 2);
    const double* cm = d.colmax;
    ntf::KrMergeParams kp{};
    kp.R = R;
    kp.out = pl->kr[v];
    kp.cm_view = pl->vcm[v];
    kp.cm_zero = pl->any_tc ? d.colmax + m * R : nullptr;
    kp.stop_flag = d.counters + 1;
    if (v == 0) {
      kp.Fa = d.factors[2], kp.na = d.dims[2], kp.Fb = d.factors[3], kp.nb = d.dims[3];
      kp.merged_mode = 2;
      kp.cm_src[0] = cm, kp.cm_src[1] = cm + R, kp.cm_src[2] = cm + 2 * R, kp.cm_src2 = cm + 3 * R;
    } else {
      kp.Fa = d.factors[0], kp.na = d.dims[0], kp.Fb = d.factors[1], kp.nb = d.dims[1];
      kp.merged_mode = 0;
      kp.cm_src[0] = cm, kp.cm_src[1] = cm + 2 * R, kp.cm_src[2] = cm + 3 * R, kp.cm_src2 = cm + R;
    }
    NTF_CUDA_TRY(ntf::kr_merge_launch(kp, s));
    const int64_t* vd = pl->vdims[v];
    const double* F0 = v == 0 ? d.factors[0] : pl->kr[1];
    const double* F1 = v == 0 ? d.factors[1] : d.factors[2];
    const double* F2 = v == 0 ? pl->kr[0] : d.factors[3];
    NTF_CUDA_TRY(run_op(pl->op[m], vmode, d.x_dtype, d.x_mode[m], vd[0], vd[1], vd[2], F0, F1, F2, R,
                        pl->mtt_ws, d.counters + 1, s, pl->vcm[v]));
  } else {
    NTF_CUDA_TRY(run_op(pl->op[m], mode, d.x_dtype, d.x_mode[m], xd[0], xd[1], xd[2], d.factors[0],
                        d.factors[1], d.factors[2], R, pl->mtt_ws, d.counters + 1, s, d.colmax));
  }
  if (ev) NTF_CUDA_TRY(record_event(ev[1], s));
  NTF_CUDA_TRY(cudaStreamWaitEvent(s, pl->join_ev, 0));
  return enqueue_row_update(pl, mode, last, s, ev);
}

// Row update of one mode (+ Gram reduction off the critical path, + norm
// reduction in the last sweep), after its MTTKRP and ridge factor.
int enqueue_row_update(ntf_plan* pl, int mode, int last, cudaStream_t s, cudaEvent_t* ev) {
  const ntf_plan_desc& d = pl->d;
  const int m = mode - 1;
  const int R = d.rank;
  ntf::FactorUpdateParams fp{};
  fp.mode = mode;
  fp.R = R;
  fp.rows = d.row_count[m];
  fp.row_offset = d.row_offset[m];
  fp.mtt = pl->mtt_ws;
  fp.splits = pl->op[m].splits();
  fp.tail_row0 = pl->op[m].tail_row0();
  fp.splits_tail = pl->op[m].splits_tail();
  fp.Lg = pl->ridge;
  fp.rho = d.rho;
  fp.F = d.factors[m];
  fp.aux = d.aux[m];
  fp.dual = d.duals[m];
  fp.last_sweep = last;
  fp.fuse_gram = d.fuse_gram;
  fp.norm_partials = pl->norm_partials[m];
  fp.gram_partials = pl->gram_partials[m];
  // column maxima feed the tensor-core MTTKRPs only (zeroed by this mode's
  // MTTKRP, re-accumulated here)
  fp.colmax_bits = pl->any_tc ? reinterpret_cast<unsigned long long*>(d.colmax + m * R) : nullptr;
  fp.gram_pending = nullptr;
  fp.ridge_in_pred = 0;
  fp.status = d.counters + 2;
  fp.stop_flag = d.counters + 1;
  fp.kind = d.constraint[m];
  fp.cand = pl->card_cand[m];
  NTF_CUDA_TRY(ntf::factor_update_launch(fp, s));
  if (last && fp.kind == NTF_CONSTRAINT_CARD) {  // global top-c projection (constraints.py:95-102)
    NTF_CUDA_TRY(ntf::card_select_launch(pl->card_cand[m], d.row_count[m] * R, d.card[m],
                                         pl->card_sel[m], d.counters + 1, s));
    NTF_CUDA_TRY(ntf::card_apply_launch(fp, pl->card_sel[m], s));
  }
  if (ev) NTF_CUDA_TRY(record_event(ev[2], s));
  if (d.fuse_gram) {  // G_m for the coming ridges, off the critical path
    NTF_CUDA_TRY(cudaEventRecord(pl->post_ev, s));
    NTF_CUDA_TRY(cudaStreamWaitEvent(pl->side, pl->post_ev, 0));
    NTF_CUDA_TRY(ntf::gram_reduce_launch(pl->gram_partials[m], pl->blocks[m], R, d.grams[m],
                                         d.counters + 1, pl->side));
  }
  if (last)
    NTF_CUDA_TRY(ntf::norm_reduce_launch(pl->norm_partials[m], pl->blocks[m], d.norm_acc + 10 * m,
                                         d.counters + 1, s));
  return NTF_OK;
}

// main stream waits for the side stream's queued work (Gram reductions)
int join_side(ntf_plan* pl, cudaStream_t s) {
  NTF_CUDA_TRY(cudaEventRecord(pl->join_ev, pl->side));
  NTF_CUDA_TRY(cudaStreamWaitEvent(s, pl->join_ev, 0));
  return NTF_OK;
}

int enqueue_finalize(ntf_plan* pl, cudaStream_t s) {
  const ntf_plan_desc& d = pl->d;
  ntf::FinalizeParams fz{};
  fz.norm_acc = d.norm_all ? d.norm_all : d.norm_acc;
  fz.norm_parts = d.norm_all ? d.norm_parts : 1;
  fz.rho = d.rho;
  fz.order = pl->order;
  for (int m = 0; m < pl->order; ++m) fz.dims[m] = d.dims[m];
  fz.R = d.rank;
  fz.eps_abs = d.eps_abs;
  fz.eps_rel = d.eps_rel;
  fz.mu = d.mu;
  fz.tau_incr = d.tau_incr;
  fz.tau_decr = d.tau_decr;
  fz.adapt = d.adapt;
  fz.history_capacity = d.history_capacity;
  fz.resid_history = d.resid_history;
  fz.rho_history = d.rho_history;
  fz.counters = d.counters;
  fz.rho_schedule = d.rho_schedule;
  NTF_CUDA_TRY(ntf::finalize_launch(fz, s));
  return NTF_OK;
}

// An instrumented iteration (timing events around every MTTKRP / row
// update) is enqueued without PDL: its kernels serialise, so each event pair
// brackets exactly its own kernels and the per-kernel times cannot overlap.
struct PdlOff {
  bool prev;
  explicit PdlOff(bool off) : prev(ntf::pdl_switch()) {
    if (off) ntf::pdl_switch() = false;
  }
  ~PdlOff() { ntf::pdl_switch() = prev; }
};

int enqueue_iteration(ntf_plan* pl, cudaStream_t s) {
  PdlOff no_pdl(pl->timing && pl->events);
  const int sweeps = pl->d.inner_sweeps;
  for (int sw = 0; sw < sweeps; ++sw)
    for (int mode = 1; mode <= pl->order; ++mode) {
      const int rc = enqueue_mode_update(pl, mode, sw == sweeps - 1, s);
      if (rc != NTF_OK) return rc;
    }
  const int rc = join_side(pl, s);
  if (rc != NTF_OK) return rc;
  return enqueue_finalize(pl, s);
}

}  // namespace

extern "C" {

int ntf_abi_version(void) { return NTF_ABI_VERSION; }

const char* ntf_last_error(void) { return g_err.c_str(); }

size_t ntf_mttkrp_workspace_bytes(int mode, int x_dtype, int64_t I, int64_t J, int64_t K, int R,
                                  int engine) {
  if (check_dims(mode, x_dtype, I, J, K, R) != NTF_OK) return 0;
  const MttkrpOp op = make_op(mode, x_dtype, I, J, K, R, engine);
  return op.ws_bytes(R);
}

int ntf_mttkrp(int mode, int x_dtype, const void* X, int64_t I, int64_t J, int64_t K,
               const double* A, const double* B, const double* C, int R, double* out,
               void* workspace, size_t workspace_bytes, int engine, ntf_stream_t stream) {
  int rc = check_dims(mode, x_dtype, I, J, K, R);
  if (rc != NTF_OK) return rc;
  if (!X || !out || !workspace) return fail(NTF_ERR_INVALID, "null pointer");
  if ((mode != 1 && !A) || (mode != 2 && !B) || (mode != 3 && !C))
    return fail(NTF_ERR_INVALID, "missing companion factor");
  if (engine == NTF_ENGINE_TCGEN05 && !tc_ok(mode, x_dtype, I, J, K, R))
    return fail(NTF_ERR_UNSUPPORTED, "tcgen05 engine unsupported for this dtype/rank/shape");
  MttkrpOp op = make_op(mode, x_dtype, I, J, K, R, engine);
  if (workspace_bytes < op.ws_bytes(R)) return fail(NTF_ERR_INVALID, "workspace too small");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  double* ws = static_cast<double*>(workspace);
  NTF_CUDA_TRY(prepare_op(op, mode, x_dtype));
  const int64_t M = mode == 1 ? I : (mode == 2 ? J : K);
  if (op.tc) {
    // one-shot call: split the tensor into its fp16 planes for this call only
    // (a solver plan does this once); synchronises before releasing them.
    ntf::TcTensor t;
    const int64_t dims[3] = {I, J, K};
    NTF_CUDA_TRY(ntf::tc_tensor_create(op.tcl, static_cast<const float*>(X), dims, &t, s));
    cudaError_t e = ntf::mttkrp_tc_bind(op.tcl, t);
    op.tct = &t;
    if (e == cudaSuccess) e = run_op(op, mode, x_dtype, X, I, J, K, A, B, C, R, ws, nullptr, s);
    if (e == cudaSuccess)
      e = ntf::mttkrp_reduce_launch(ws, op.splits(), M, R, out, nullptr, s, op.tail_row0(),
                                    op.splits_tail());
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    ntf::mttkrp_tc_unbind(op.tcl);
    ntf::tc_tensor_destroy(&t);
    if (e != cudaSuccess) return cuda_fail(e, "tcgen05 mttkrp");
    return NTF_OK;
  }
  NTF_CUDA_TRY(run_op(op, mode, x_dtype, X, I, J, K, A, B, C, R, ws, nullptr, s));
  NTF_CUDA_TRY(ntf::mttkrp_reduce_launch(ws, op.splits(), M, R, out, nullptr, s));
  return NTF_OK;
}

size_t ntf_gram_workspace_bytes(int64_t rows, int R) { return ntf::gram_workspace_bytes(rows, R); }

int ntf_gram(const double* F, int64_t rows, int R, double* G, void* workspace,
             size_t workspace_bytes, ntf_stream_t stream) {
  if (!F || !G || !workspace) return fail(NTF_ERR_INVALID, "null pointer");
  if (rows < 1 || R < 1 || R > NTF_MAX_RANK) return fail(NTF_ERR_INVALID, "bad shape");
  if (workspace_bytes < ntf::gram_workspace_bytes(rows, R))
    return fail(NTF_ERR_INVALID, "workspace too small");
  NTF_CUDA_TRY(ntf::gram_launch(F, rows, R, G, static_cast<double*>(workspace),
                                static_cast<cudaStream_t>(stream)));
  return NTF_OK;
}

size_t ntf_sq_error_workspace_bytes(int64_t I, int64_t J, int64_t K) {
  return ntf::sq_error_workspace_bytes(I, J, K, NTF_MAX_RANK);
}

int ntf_sq_error(int x_dtype, const void* X, int64_t I, int64_t J, int64_t K, const double* A,
                 const double* B, const double* C, int R, double* out2, void* workspace,
                 size_t workspace_bytes, ntf_stream_t stream) {
  if (!X || !out2 || !workspace) return fail(NTF_ERR_INVALID, "null pointer");
  if (x_dtype != NTF_F32 && x_dtype != NTF_F64) return fail(NTF_ERR_INVALID, "bad dtype");
  if (I < 1 || J < 1 || K < 1) return fail(NTF_ERR_INVALID, "bad shape");
  if (A && (!B || !C || R < 1 || R > NTF_MAX_RANK)) return fail(NTF_ERR_INVALID, "bad model");
  if (workspace_bytes < ntf::sq_error_workspace_bytes(I, J, K, A ? R : 0))
    return fail(NTF_ERR_INVALID, "workspace too small");
  NTF_CUDA_TRY(ntf::sq_error_launch(x_dtype, X, I, J, K, A, B, C, A ? R : 0, out2, workspace,
                                    static_cast<cudaStream_t>(stream)));
  return NTF_OK;
}

int ntf_mttkrp_coo(int order, const int64_t* dims, int mode, int64_t nnz, const int64_t* idx,
                   const double* vals, const int64_t* perm, const int64_t* rowptr,
                   const double* const* factors, int R, double* out, ntf_stream_t stream) {
  if (order != 3 && order != 4) return fail(NTF_ERR_UNSUPPORTED, "tensor order must be 3 or 4");
  if (mode < 1 || mode > order) return fail(NTF_ERR_INVALID, "mode out of range");
  if (!dims || !factors || nnz < 0) return fail(NTF_ERR_INVALID, "bad shape");
  for (int m = 0; m < order; ++m)
    if (dims[m] < 1) return fail(NTF_ERR_INVALID, "bad shape");
  if (R < 1 || R > NTF_MAX_RANK) return fail(NTF_ERR_UNSUPPORTED, "rank must be in 1..256 (NTF_MAX_RANK)");
  if (!out || !rowptr || (nnz > 0 && (!idx || !vals || (mode > 1 && !perm))))
    return fail(NTF_ERR_INVALID, "null pointer");
  for (int m = 0; m < order; ++m)
    if (m != mode - 1 && !factors[m]) return fail(NTF_ERR_INVALID, "missing companion factor");
  ntf::CooView v{};
  v.order = order;
  for (int m = 0; m < order; ++m) v.dims[m] = dims[m];
  v.nnz = nnz;
  v.idx = idx;
  v.vals = vals;
  v.perm[mode - 1] = mode > 1 ? perm : nullptr;
  v.rowptr[mode - 1] = rowptr;
  const double* F[4] = {factors[0], factors[1], factors[2], order == 4 ? factors[3] : nullptr};
  NTF_CUDA_TRY(ntf::mttkrp_coo_launch(v, mode, F, R, out, nullptr, static_cast<cudaStream_t>(stream)));
  return NTF_OK;
}

size_t ntf_sq_error_coo_workspace_bytes(int64_t nnz) { return ntf::coo_sq_error_workspace_bytes(nnz, 0); }

int ntf_sq_error_coo(int order, const int64_t* dims, int64_t nnz, const int64_t* idx,
                     const double* vals, const double* const* factors, int R, double* out2,
                     void* workspace, size_t workspace_bytes, ntf_stream_t stream) {
  if (order != 3 && order != 4) return fail(NTF_ERR_UNSUPPORTED, "tensor order must be 3 or 4");
  if (!dims || nnz < 0) return fail(NTF_ERR_INVALID, "bad shape");
  for (int m = 0; m < order; ++m)
    if (dims[m] < 1) return fail(NTF_ERR_INVALID, "bad shape");
  if (!out2 || !workspace || (nnz > 0 && (!idx || !vals))) return fail(NTF_ERR_INVALID, "null pointer");
  if (factors) {
    if (R < 1 || R > NTF_MAX_RANK) return fail(NTF_ERR_INVALID, "bad model");
    for (int m = 0; m < order; ++m)
      if (!factors[m]) return fail(NTF_ERR_INVALID, "bad model");
  }
  if (workspace_bytes < ntf::coo_sq_error_workspace_bytes(nnz, R))
    return fail(NTF_ERR_INVALID, "workspace too small");
  ntf::CooView v{};
  v.order = order;
  for (int m = 0; m < order; ++m) v.dims[m] = dims[m];
  v.nnz = nnz;
  v.idx = idx;
  v.vals = vals;
  const double* F[4] = {nullptr, nullptr, nullptr, nullptr};
  if (factors)
    for (int m = 0; m < order; ++m) F[m] = factors[m];
  NTF_CUDA_TRY(ntf::coo_sq_error_launch(v, factors ? F : nullptr, factors ? R : 0, out2, workspace,
                                        static_cast<cudaStream_t>(stream)));
  return NTF_OK;
}

int ntf_synth_dense(int x_dtype, void* out, const int64_t* dims, const int64_t* lo, const int64_t* hi,
                    const double* A, const double* B, const double* C, int R, double sigma,
                    uint64_t key, ntf_stream_t stream) {
  if (x_dtype != NTF_F32 && x_dtype != NTF_F64) return fail(NTF_ERR_INVALID, "bad dtype");
  if (!out || !dims || !lo || !hi || !A || !B || !C) return fail(NTF_ERR_INVALID, "null pointer");
  if (R < 1) return fail(NTF_ERR_INVALID, "rank must be >= 1");
  if (!(sigma >= 0.0) || sigma > 1e300) return fail(NTF_ERR_INVALID, "sigma must be finite and >= 0");
  ntf::SynthBox b{};
  for (int m = 0; m < 3; ++m) {
    if (dims[m] < 1 || lo[m] < 0 || hi[m] <= lo[m] || hi[m] > dims[m])
      return fail(NTF_ERR_INVALID, "box outside the tensor");
    b.dims[m] = dims[m];
    b.lo[m] = lo[m];
    b.hi[m] = hi[m];
  }
  NTF_CUDA_TRY(ntf::synth_dense_launch(x_dtype, out, b, A, B, C, R, sigma, key,
                                       static_cast<cudaStream_t>(stream)));
  return NTF_OK;
}

int ntf_trim_device_pool(void) {
  int dev = 0;
  cudaMemPool_t pool;
  NTF_CUDA_TRY(cudaGetDevice(&dev));
  NTF_CUDA_TRY(cudaDeviceSynchronize());
  NTF_CUDA_TRY(cudaDeviceGetDefaultMemPool(&pool, dev));
  NTF_CUDA_TRY(cudaMemPoolTrimTo(pool, 0));
  return NTF_OK;
}

int ntf_device_pool_idle_bytes(size_t* bytes) {
  if (!bytes) return fail(NTF_ERR_INVALID, "null pointer");
  int dev = 0;
  cudaMemPool_t pool;
  cuuint64_t reserved = 0, used = 0;
  NTF_CUDA_TRY(cudaGetDevice(&dev));
  NTF_CUDA_TRY(cudaDeviceGetDefaultMemPool(&pool, dev));
  NTF_CUDA_TRY(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved));
  NTF_CUDA_TRY(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used));
  *bytes = reserved > used ? static_cast<size_t>(reserved - used) : 0;
  return NTF_OK;
}

int ntf_plan_create(const ntf_plan_desc* desc, ntf_plan** out) {
  if (!desc || !out) return fail(NTF_ERR_INVALID, "null pointer");
  *out = nullptr;
  const ntf_plan_desc& d = *desc;
  const int R = d.rank;
  if (R < 1 || R > NTF_MAX_RANK) return fail(NTF_ERR_UNSUPPORTED, "rank must be in 1..256 (NTF_MAX_RANK)");
  if (d.inner_sweeps < 1) return fail(NTF_ERR_INVALID, "inner_sweeps must be >= 1");
  if (d.norm_all && d.norm_parts < 1) return fail(NTF_ERR_INVALID, "norm_parts must be >= 1");
  if (!d.rho || !d.norm_acc || !d.counters || !d.resid_history || !d.rho_history || !d.colmax)
    return fail(NTF_ERR_INVALID, "null plan buffer");
  const int N = d.order == 0 ? 3 : d.order;
  if (N != 3 && N != 4) return fail(NTF_ERR_UNSUPPORTED, "tensor order must be 3 or 4");
  if (d.x_format != NTF_FORMAT_DENSE && d.x_format != NTF_FORMAT_COO)
    return fail(NTF_ERR_INVALID, "unknown tensor format");
  const bool coo = d.x_format == NTF_FORMAT_COO;
  if (coo) {
    if (d.x_dtype != NTF_F64) return fail(NTF_ERR_INVALID, "COO values are fp64");
    if (d.nnz < 0 || (d.nnz > 0 && (!d.coo_idx || !d.coo_vals)))
      return fail(NTF_ERR_INVALID, "null COO buffer");
    for (int m = 0; m < N; ++m) {
      if (!d.coo_rowptr[m] || (m > 0 && d.nnz > 0 && !d.coo_perm[m]))
        return fail(NTF_ERR_INVALID, "null COO mode order");
      if (d.row_count[m] != d.dims[m] || d.row_offset[m] != 0)
        return fail(NTF_ERR_UNSUPPORTED, "COO tensors are single-GPU");
    }
  }
  // order-4 views: I x J x KL (modes 1, 2) and IJ x K x L (modes 3, 4)
  int64_t vdims[2][3] = {};
  if (N == 4 && !coo) {
    vdims[0][0] = d.dims[0], vdims[0][1] = d.dims[1], vdims[0][2] = d.dims[2] * d.dims[3];
    vdims[1][0] = d.dims[0] * d.dims[1], vdims[1][1] = d.dims[2], vdims[1][2] = d.dims[3];
  }
  auto vmode_of = [](int m) { return m == 0 ? 1 : (m == 3 ? 3 : 2); };
  for (int m = 0; m < N; ++m) {
    if (!d.x_mode[m] || !d.factors[m] || !d.aux[m] || !d.duals[m] || !d.grams[m])
      return fail(NTF_ERR_INVALID, "null state buffer");
    if (d.row_offset[m] < 0 || d.row_offset[m] + d.row_count[m] > d.dims[m])
      return fail(NTF_ERR_INVALID, "owned rows out of range");
    const int64_t* xd = d.x_dims[m];
    if (coo) continue;  // the COO engine reads the entries directly
    if (N == 4) {
      if (d.row_count[m] != d.dims[m] || d.x_mode[m] != d.x_mode[0])
        return fail(NTF_ERR_UNSUPPORTED, "order-4 tensors are single-GPU");
      for (int a = 0; a < 4; ++a)
        if (xd[a] != d.dims[a]) return fail(NTF_ERR_INVALID, "order-4 extents");
      const int64_t* vd = vdims[m < 2 ? 0 : 1];
      int rc = check_dims(vmode_of(m), d.x_dtype, vd[0], vd[1], vd[2], R);
      if (rc != NTF_OK) return rc;
      continue;
    }
    int rc = check_dims(m + 1, d.x_dtype, xd[0], xd[1], xd[2], R);
    if (rc != NTF_OK) return rc;
    if (xd[m] != d.row_count[m]) return fail(NTF_ERR_INVALID, "slab extent != owned row count");
    for (int a = 0; a < 3; ++a)
      if (a != m && xd[a] != d.dims[a]) return fail(NTF_ERR_INVALID, "slab companion extent");
  }
  for (int m = 0; m < N; ++m) {
    if (d.constraint[m] < NTF_CONSTRAINT_NONNEG || d.constraint[m] > NTF_CONSTRAINT_ROW_STOCHASTIC)
      return fail(NTF_ERR_INVALID, "unknown constraint kind");
    if (d.constraint[m] == NTF_CONSTRAINT_CARD) {
      if (d.card[m] < 1 || d.card[m] > d.dims[m] * R)
        return fail(NTF_ERR_INVALID, "cardinality budget out of range");
      if (d.row_count[m] != d.dims[m])
        return fail(NTF_ERR_UNSUPPORTED, "cardinality constraint needs the whole factor on one GPU");
    }
  }
  for (int m = 0; m < N && !coo; ++m) {
    const int64_t* xd = N == 4 ? vdims[m < 2 ? 0 : 1] : d.x_dims[m];
    const int vm = N == 4 ? vmode_of(m) : m + 1;
    if (d.engine == NTF_ENGINE_TCGEN05 && !tc_ok(vm, d.x_dtype, xd[0], xd[1], xd[2], R))
      return fail(NTF_ERR_UNSUPPORTED, "tcgen05 engine unsupported for this dtype/rank/shape");
  }

  ntf_plan* pl = new (std::nothrow) ntf_plan();
  if (!pl) return fail(NTF_ERR_INVALID, "out of host memory");
  pl->d = d;
  pl->order = N;
  for (int v = 0; v < 2; ++v)
    for (int a = 0; a < 3; ++a) pl->vdims[v][a] = vdims[v][a];
  size_t ws = 0;
  int maxb = 1;
  int64_t max_rows = 1;
  for (int m = 0; m < N; ++m) {
    const int64_t* xd = d.x_dims[m];
    if (coo) {
      MttkrpOp op;
      op.coo = true;
      op.cv.order = N;
      for (int a = 0; a < N; ++a) op.cv.dims[a] = d.dims[a];
      op.cv.nnz = d.nnz;
      op.cv.idx = d.coo_idx;
      op.cv.vals = d.coo_vals;
      for (int a = 0; a < N; ++a) {
        op.cv.perm[a] = d.coo_perm[a];
        op.cv.rowptr[a] = d.coo_rowptr[a];
      }
      op.f3 = N == 4 ? d.factors[3] : nullptr;
      pl->op[m] = op;
      ws = std::max(ws, static_cast<size_t>(d.dims[m]) * R * sizeof(double));
    } else if (N == 4) {
      const int64_t* vd = vdims[m < 2 ? 0 : 1];
      pl->op[m] = make_op(vmode_of(m), d.x_dtype, vd[0], vd[1], vd[2], R, d.engine);
    } else {
      pl->op[m] = make_op(m + 1, d.x_dtype, xd[0], xd[1], xd[2], R, d.engine);
    }
    ws = std::max(ws, pl->op[m].ws_bytes(R));
    pl->blocks[m] = ntf::factor_update_blocks(d.row_count[m], R);
    maxb = std::max(maxb, pl->blocks[m]);
    max_rows = std::max(max_rows, d.dims[m]);
  }
  cudaError_t e = cudaSuccess;
  auto cleanup = [&](int rc) {
    ntf_plan_destroy(pl);
    return rc;
  };
  // NTF_B200_PLAN_TIMING=1: host wall time of each setup phase to stderr
  static const bool plan_timing = ntf::diag_env("NTF_B200_PLAN_TIMING") != nullptr;
  auto t_last = std::chrono::steady_clock::now();
  auto phase = [&](const char* what) {
    if (!plan_timing) return;
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "plan %s %.2f ms\n", what,
            std::chrono::duration<double, std::milli>(now - t_last).count());
    t_last = now;
  };
  if ((e = ntf::dev_alloc(&pl->mtt_ws, ws)) != cudaSuccess) return cleanup(cuda_fail(e, "cudaMalloc ws"));
  if (N == 4 && !coo) {
    if ((e = ntf::dev_alloc(&pl->kr[0], sizeof(double) * R * vdims[0][2])) != cudaSuccess ||
        (e = ntf::dev_alloc(&pl->kr[1], sizeof(double) * R * vdims[1][0])) != cudaSuccess ||
        (e = ntf::dev_alloc(&pl->vcm[0], sizeof(double) * 3 * R)) != cudaSuccess ||
        (e = ntf::dev_alloc(&pl->vcm[1], sizeof(double) * 3 * R)) != cudaSuccess)
      return cleanup(cuda_fail(e, "cudaMalloc views"));
  }
  for (int m = 0; m < N; ++m) {
    const size_t nb = static_cast<size_t>(pl->blocks[m]);
    if ((e = ntf::dev_alloc(&pl->norm_partials[m], sizeof(double) * 10 * nb)) != cudaSuccess)
      return cleanup(cuda_fail(e, "cudaMalloc norm"));
    if ((e = ntf::dev_alloc(&pl->gram_partials[m], sizeof(double) * R * R * nb)) != cudaSuccess)
      return cleanup(cuda_fail(e, "cudaMalloc gram"));
    if (d.constraint[m] == NTF_CONSTRAINT_CARD) {
      if ((e = ntf::dev_alloc(&pl->card_cand[m], sizeof(double) * R * d.row_count[m])) != cudaSuccess ||
          (e = ntf::dev_alloc(&pl->card_sel[m], 2 * sizeof(unsigned long long))) != cudaSuccess)
        return cleanup(cuda_fail(e, "cudaMalloc card"));
    }
  }
  if ((e = ntf::dev_alloc(&pl->gram_ws, ntf::gram_workspace_bytes(max_rows, R))) != cudaSuccess)
    return cleanup(cuda_fail(e, "cudaMalloc gram ws"));
  if ((e = ntf::dev_alloc(&pl->ridge, sizeof(double) * ntf::ridge_buffer_doubles(R))) != cudaSuccess)
    return cleanup(cuda_fail(e, "cudaMalloc ridge"));
  if ((e = cudaStreamCreateWithFlags(&pl->side, cudaStreamNonBlocking)) != cudaSuccess)
    return cleanup(cuda_fail(e, "cudaStreamCreate"));
  if ((e = cudaEventCreateWithFlags(&pl->fork_ev, cudaEventDisableTiming)) != cudaSuccess)
    return cleanup(cuda_fail(e, "cudaEventCreate"));
  if ((e = cudaEventCreateWithFlags(&pl->join_ev, cudaEventDisableTiming)) != cudaSuccess)
    return cleanup(cuda_fail(e, "cudaEventCreate"));
  if ((e = cudaEventCreateWithFlags(&pl->post_ev, cudaEventDisableTiming)) != cudaSuccess)
    return cleanup(cuda_fail(e, "cudaEventCreate"));
  phase("buffers");
  if ((e = ntf::factor_update_prepare(R)) != cudaSuccess) return cleanup(cuda_fail(e, "prepare"));
  for (int m = 0; m < N; ++m) {
    if ((e = prepare_op(pl->op[m], N == 4 ? vmode_of(m) : m + 1, d.x_dtype)) != cudaSuccess)
      return cleanup(cuda_fail(e, "mttkrp prepare"));
  }
  // Tensor-core engine: split each distinct slab once into its fp16 planes
  // (one-time setup; synchronous so the caller's upload stream is irrelevant).
  for (int m = 0; m < N; ++m) pl->any_tc = pl->any_tc || pl->op[m].tc;
  phase("prepare");
  if (pl->any_tc) {
    if ((e = cudaDeviceSynchronize()) != cudaSuccess) return cleanup(cuda_fail(e, "sync"));
    phase("sync");
    // one block image per mode (each is laid out for its mode's stream;
    // order 4: of the mode's reshaped view)
    for (int m = 0; m < N; ++m) {
      if (!pl->op[m].tc) continue;
      // one max|X| pass per distinct tensor (the unsharded plan's modes share one)
      const ntf::TcTensor* same = pl->n_tct > 0 ? &pl->tct[0] : nullptr;
      ntf::TcTensor& slot = pl->tct[pl->n_tct++];
      const int64_t* xd = N == 4 ? vdims[m < 2 ? 0 : 1] : d.x_dims[m];
      if ((e = ntf::tc_tensor_create(pl->op[m].tcl, static_cast<const float*>(d.x_mode[m]), xd,
                                     &slot, nullptr, same)) != cudaSuccess)
        return cleanup(cuda_fail(e, "tc split"));
      pl->op[m].tct = &slot;
      if ((e = ntf::mttkrp_tc_bind(pl->op[m].tcl, slot)) != cudaSuccess)
        return cleanup(cuda_fail(e, "tc bind"));
      phase("tc image");
    }
    if ((e = cudaDeviceSynchronize()) != cudaSuccess) return cleanup(cuda_fail(e, "sync"));
    phase("images done");
  }
  *out = pl;
  return NTF_OK;
}

int ntf_plan_refresh_tensor(ntf_plan* pl, ntf_stream_t stream) {
  if (!pl) return fail(NTF_ERR_INVALID, "null plan");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const ntf::TcTensor* first = nullptr;
  for (int m = 0; m < pl->order; ++m) {
    const MttkrpOp& op = pl->op[m];
    if (!op.tc || !op.tct) continue;
    NTF_CUDA_TRY(ntf::tc_tensor_fill(op.tcl, *op.tct, s, first));
    if (!first) first = op.tct;
  }
  return NTF_OK;
}

int ntf_plan_sync_grams(ntf_plan* pl, ntf_stream_t stream) {
  if (!pl) return fail(NTF_ERR_INVALID, "null plan");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  for (int m = 0; m < pl->order; ++m) {
    NTF_CUDA_TRY(ntf::gram_launch(pl->d.factors[m], pl->d.dims[m], pl->d.rank, pl->d.grams[m],
                                  pl->gram_ws, s));
    NTF_CUDA_TRY(ntf::colmax_launch(pl->d.factors[m], pl->d.dims[m], pl->d.rank,
                                    pl->d.colmax + m * pl->d.rank, s));
  }
  return NTF_OK;
}

int ntf_khatri_rao_pair(const double* Fa, int64_t na, const double* Fb, int64_t nb, int R, double* out,
                        ntf_stream_t stream) {
  if (!Fa || !Fb || !out) return fail(NTF_ERR_INVALID, "null pointer");
  if (na < 1 || nb < 1 || R < 1 || R > NTF_MAX_RANK) return fail(NTF_ERR_INVALID, "bad shape");
  ntf::KrMergeParams kp{};
  kp.Fa = Fa, kp.na = na, kp.Fb = Fb, kp.nb = nb, kp.R = R, kp.out = out;
  NTF_CUDA_TRY(ntf::kr_merge_launch(kp, static_cast<cudaStream_t>(stream)));
  return NTF_OK;
}

size_t ntf_peer_buffer_bytes(int64_t rows, int R) {
  if (rows < 1 || R < 1) return 0;
  return ntf::kPeerHeaderBytes + 2 * static_cast<size_t>(rows) * R * sizeof(double);
}

int ntf_peer_alloc(size_t bytes, void** base_out, void* handle_out) {
  if (!base_out || !handle_out) return fail(NTF_ERR_INVALID, "null pointer");
  if (bytes < ntf::kPeerHeaderBytes) return fail(NTF_ERR_INVALID, "peer buffer too small");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  void* p = nullptr;
  NTF_CUDA_TRY(cudaMalloc(&p, bytes));
  cudaError_t e = cudaMemset(p, 0, bytes);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();  // zeroed before any peer can map it
  cudaIpcMemHandle_t h;
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, p);
  if (e != cudaSuccess) {
    cudaFree(p);
    return cuda_fail(e, "ntf_peer_alloc");
  }
  std::memcpy(handle_out, &h, sizeof(h));
  *base_out = p;
  return NTF_OK;
}

int ntf_peer_open(const void* handle, void** base_out) {
  if (!handle || !base_out) return fail(NTF_ERR_INVALID, "null pointer");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  NTF_CUDA_TRY(cudaIpcOpenMemHandle(base_out, h, cudaIpcMemLazyEnablePeerAccess));
  return NTF_OK;
}

int ntf_peer_close(void* base) {
  if (!base) return NTF_OK;
  NTF_CUDA_TRY(cudaIpcCloseMemHandle(base));
  return NTF_OK;
}

int ntf_peer_free(void* base) {
  if (!base) return NTF_OK;
  NTF_CUDA_TRY(cudaFree(base));
  return NTF_OK;
}

namespace {
int peer_args(const ntf_peer_gather_desc* d, int ranks_in_launch, ntf::PeerGatherArgs* out) {
  static_assert(NTF_MAX_PEERS == ntf::kPeerMaxRanks, "peer limits");
  static_assert(NTF_PEER_TIMEOUT == ntf::kPeerGatherTimeout, "timeout status");
  if (!d || !d->full) return fail(NTF_ERR_INVALID, "null pointer");
  if (d->nranks < 1 || d->nranks > NTF_MAX_PEERS || d->me < 0 || d->me >= d->nranks)
    return fail(NTF_ERR_INVALID, "bad rank geometry");
  if (d->R < 1 || d->R > NTF_MAX_RANK) return fail(NTF_ERR_INVALID, "bad rank R");
  if (d->ctas < 1 || d->ctas > ntf::peer_gather_max_ctas(ranks_in_launch))
    return fail(NTF_ERR_INVALID, "ctas must be >= 1 and small enough for every CTA to be co-resident");
  if (d->timeout_ns <= 0) return fail(NTF_ERR_INVALID, "timeout_ns must be > 0");
  ntf::PeerGatherArgs& a = *out;
  a = ntf::PeerGatherArgs{};
  a.nranks = d->nranks, a.me = d->me, a.R = d->R, a.ctas = d->ctas;
  for (int q = 0; q <= d->nranks; ++q) {
    a.row_offset[q] = d->row_offset[q];
    if (q > 0 && d->row_offset[q] < d->row_offset[q - 1]) return fail(NTF_ERR_INVALID, "row offsets decrease");
  }
  if (d->row_offset[0] != 0 || d->row_offset[d->nranks] < 1) return fail(NTF_ERR_INVALID, "bad row offsets");
  for (int q = 0; q < d->nranks; ++q) {
    if (!d->peer_base[q]) return fail(NTF_ERR_INVALID, "null peer buffer");
    a.base[q] = d->peer_base[q];
  }
  a.full = d->full, a.status = d->status, a.timeout_ns = d->timeout_ns;
  return NTF_OK;
}
}  // namespace

int ntf_peer_gather(const ntf_peer_gather_desc* d, ntf_stream_t stream) {
  ntf::PeerGatherArgs a;
  const int rc = peer_args(d, 1, &a);
  if (rc != NTF_OK) return rc;
  NTF_CUDA_TRY(ntf::peer_gather_launch(a, static_cast<cudaStream_t>(stream)));
  return NTF_OK;
}

int ntf_peer_gather_group(const ntf_peer_gather_desc* descs, int nranks, ntf_stream_t stream) {
  if (!descs || nranks < 1 || nranks > NTF_MAX_PEERS) return fail(NTF_ERR_INVALID, "bad rank count");
  ntf::PeerGatherGroup g{};
  for (int q = 0; q < nranks; ++q) {
    const int rc = peer_args(descs + q, nranks, &g.args[q]);
    if (rc != NTF_OK) return rc;
    if (descs[q].me != q || descs[q].nranks != nranks || descs[q].ctas != descs[0].ctas)
      return fail(NTF_ERR_INVALID, "group: descs[q] must be rank q of nranks, same ctas");
    for (int r = 0; r <= nranks; ++r)
      if (descs[q].row_offset[r] != descs[0].row_offset[r])
        return fail(NTF_ERR_INVALID, "group: ranks disagree on the row blocks");
  }
  NTF_CUDA_TRY(ntf::peer_gather_group_launch(g, nranks, static_cast<cudaStream_t>(stream)));
  return NTF_OK;
}

int ntf_colmax(const double* F, int64_t rows, int R, double* out, ntf_stream_t stream) {
  if (!F || !out) return fail(NTF_ERR_INVALID, "null pointer");
  if (rows < 1 || R < 1 || R > NTF_MAX_RANK) return fail(NTF_ERR_INVALID, "bad shape");
  NTF_CUDA_TRY(ntf::colmax_launch(F, rows, R, out, static_cast<cudaStream_t>(stream)));
  return NTF_OK;
}

int ntf_plan_mode_update(ntf_plan* pl, int mode, int last_sweep, ntf_stream_t stream) {
  if (!pl) return fail(NTF_ERR_INVALID, "null plan");
  if (mode < 1 || mode > pl->order) return fail(NTF_ERR_INVALID, "mode out of range");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  PdlOff no_pdl(pl->timing && pl->events);
  const int rc = enqueue_mode_update(pl, mode, last_sweep ? 1 : 0, s);
  if (rc != NTF_OK) return rc;
  return join_side(pl, s);  // grams[m] is current when the stream reaches here
}

int ntf_plan_finalize(ntf_plan* pl, ntf_stream_t stream) {
  if (!pl) return fail(NTF_ERR_INVALID, "null plan");
  return enqueue_finalize(pl, static_cast<cudaStream_t>(stream));
}

int ntf_plan_run(ntf_plan* pl, int n_iters, int use_graph, ntf_stream_t stream) {
  if (!pl) return fail(NTF_ERR_INVALID, "null plan");
  if (n_iters < 0) return fail(NTF_ERR_INVALID, "n_iters < 0");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (!use_graph) {
    for (int i = 0; i < n_iters; ++i) {
      const int rc = enqueue_iteration(pl, s);
      if (rc != NTF_OK) return rc;
    }
    return NTF_OK;
  }
  cudaGraphExec_t& graph = pl->graph[pl->timing ? 1 : 0];
  if (!graph) {
    if (!pl->capture_stream)
      NTF_CUDA_TRY(cudaStreamCreateWithFlags(&pl->capture_stream, cudaStreamNonBlocking));
    NTF_CUDA_TRY(cudaStreamBeginCapture(pl->capture_stream, cudaStreamCaptureModeThreadLocal));
    const int rc = enqueue_iteration(pl, pl->capture_stream);
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture(pl->capture_stream, &g);
    if (rc != NTF_OK) {
      if (g) cudaGraphDestroy(g);
      return rc;
    }
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture");
    e = cudaGraphInstantiate(&graph, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGraphInstantiate");
  }
  for (int i = 0; i < n_iters; ++i) NTF_CUDA_TRY(cudaGraphLaunch(graph, s));
  return NTF_OK;
}

static void free_events(ntf_plan* pl) {
  if (pl->events) {
    for (int i = 0; i < pl->n_events; ++i) cudaEventDestroy(pl->events[i]);
    delete[] pl->events;
  }
  pl->events = nullptr;
  pl->n_events = 0;
  pl->cursor = 0;
}

int ntf_plan_set_timing(ntf_plan* pl, int enable) {
  if (!pl) return fail(NTF_ERR_INVALID, "null plan");
  // the two captured graphs stay cached: toggling is free once both exist
  pl->timing = enable ? 1 : 0;
  if (!enable || pl->events) return NTF_OK;
  const int n = 3 * pl->order * pl->d.inner_sweeps;
  pl->events = new (std::nothrow) cudaEvent_t[n];
  if (!pl->events) return fail(NTF_ERR_INVALID, "out of host memory");
  for (int i = 0; i < n; ++i) {
    cudaError_t e = cudaEventCreate(&pl->events[i]);
    if (e != cudaSuccess) {
      pl->n_events = i;
      free_events(pl);
      return cuda_fail(e, "cudaEventCreate");
    }
  }
  pl->n_events = n;
  return NTF_OK;
}

int ntf_plan_kernel_times(ntf_plan* pl, float* ms_out, int capacity) {
  if (!pl || !ms_out) return -fail(NTF_ERR_INVALID, "null pointer");
  if (!pl->timing || !pl->events) return -fail(NTF_ERR_INVALID, "timing not enabled");
  const int nupd = pl->n_events / 3;
  if (capacity < 2 * nupd) return -fail(NTF_ERR_INVALID, "capacity too small");
  cudaError_t e = cudaEventSynchronize(pl->events[pl->n_events - 1]);
  if (e != cudaSuccess) return -cuda_fail(e, "cudaEventSynchronize");
  for (int u = 0; u < nupd; ++u) {
    float a = 0.f, b = 0.f;
    e = cudaEventElapsedTime(&a, pl->events[3 * u], pl->events[3 * u + 1]);
    if (e != cudaSuccess) return -cuda_fail(e, "cudaEventElapsedTime");
    e = cudaEventElapsedTime(&b, pl->events[3 * u + 1], pl->events[3 * u + 2]);
    if (e != cudaSuccess) return -cuda_fail(e, "cudaEventElapsedTime");
    ms_out[2 * u] = a;
    ms_out[2 * u + 1] = b;
  }
  return 2 * nupd;
}

void ntf_plan_destroy(ntf_plan* pl) {
  if (!pl) return;
  if (pl->side) cudaStreamSynchronize(pl->side);  // pool releases are legacy-stream ordered
  free_events(pl);
  for (int k = 0; k < 2; ++k)
    if (pl->graph[k]) cudaGraphExecDestroy(pl->graph[k]);
  if (pl->capture_stream) cudaStreamDestroy(pl->capture_stream);
  if (pl->side) cudaStreamDestroy(pl->side);
  if (pl->fork_ev) cudaEventDestroy(pl->fork_ev);
  if (pl->join_ev) cudaEventDestroy(pl->join_ev);
  if (pl->post_ev) cudaEventDestroy(pl->post_ev);
  ntf::dev_free(pl->ridge);
  for (int m = 0; m < 4; ++m)
    if (pl->op[m].tc) ntf::mttkrp_tc_unbind(pl->op[m].tcl);
  for (int k = 0; k < pl->n_tct; ++k) ntf::tc_tensor_destroy(&pl->tct[k]);
  ntf::dev_free(pl->mtt_ws);
  for (int v = 0; v < 2; ++v) {
    ntf::dev_free(pl->kr[v]);
    ntf::dev_free(pl->vcm[v]);
  }
  for (int m = 0; m < 4; ++m) {
    ntf::dev_free(pl->norm_partials[m]);
    ntf::dev_free(pl->gram_partials[m]);
    ntf::dev_free(pl->card_cand[m]);
    ntf::dev_free(pl->card_sel[m]);
  }
  ntf::dev_free(pl->gram_ws);
  delete pl;
}

// Diagnostics only (not part of the reference-facing ABI): per-CTA globaltimer
// stamps of the last tcgen05 MTTKRP launched with NTF_TC_DEBUG & 256 set.
int ntf_debug_tc_times(unsigned long long* host, int ctas) {
  return ntf::tc_debug_read_times(host, ctas);
}

}  // extern "C"
