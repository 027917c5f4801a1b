// Per-mode ridge/ADMM update, Gram, iteration finalisation and residual-norm
// kernels for the B200 NTF hot path (sm_100a).  All floating-point reductions
// run in a fixed order (no float atomics; column maxima use an integer
// atomicMax on IEEE bits, which is exact and order-free), so a fit is bitwise
// run-to-run deterministic like the reference (blocks.py:130-140).
#include "solver_kernels.cuh"
#include "ridge.cuh"

namespace ntf {

namespace {

constexpr int kUpdThreads = 256;
// rows per update block.  R <= 64: the rows of a block are solved together as
// small GEMMs against the ridge inverse; few rows per block spread a mode over
// many SMs, so the latency-bound MTTKRP split reduction runs wide.  R > 64:
// one row per warp (substitution against the Cholesky factor).
#ifndef NTF_RPB_ROWS
#define NTF_RPB_ROWS 1024
#endif
#ifndef NTF_RPB_R2MAX
#define NTF_RPB_R2MAX 32
#endif
__host__ __device__ __forceinline__ int rows_per_block(int R, int64_t rows) {
  // R <= 32: two rows per block for short factors (c2's 400 rows: 200
  // blocks, 605 vs 592 it/s with four), four for long ones, which bounds the
  // Gram partials (one R x R block per CTA, reduced on the side stream) of
  // factors like c4's 5000 rows (c4 within noise, 92-93 it/s, either way)
  return R <= 32 ? ((rows > NTF_RPB_ROWS || R > NTF_RPB_R2MAX) ? 4 : 2) : (R <= 64 ? 2 : 8);
}

// One block: H = G_a o G_b + rho I, Cholesky, then L (row-major R x R, lower)
// and 1/diag(L) to global for the row-update kernel (ridge.cuh).  Runs on the
// plan's side stream concurrently with the mode's CUDA-core MTTKRP; the
// tensor-core MTTKRP runs the same code in one extra CTA.
__global__ void ridge_factor_kernel(RidgeParams p) {
  if (p.stop_flag && *p.stop_flag) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ridge_factor_block(p.Ga, p.Gb, p.rho[p.mode - 1], p.R, p.L, p.status,
                     reinterpret_cast<double*>(smem_raw), p.Gc);
}

// Row solve of X (L L^T) = rhs for one row held by a warp: lane owns entries
// r = lane + 32*t, t < RT.  Column-oriented forward then backward
// substitution (solver.solve_factor_rows / cho_solve, solver.py:182-188),
// dividing by the diagonal through its precomputed reciprocal.
template <int RT>
__device__ __forceinline__ void warp_chol_solve(double (&y)[RT], const double* L, int ldl, int R,
                                                const double* inv_diag, int lane) {
  // forward: L z = y
#pragma unroll
  for (int s = 0; s < RT; ++s) {
    for (int kk = 0; kk < 32; ++kk) {
      const int k = s * 32 + kk;
      if (k >= R) break;
      double zk = y[s] * inv_diag[k];
      zk = __shfl_sync(0xffffffffu, zk, kk);
      if (lane == kk) y[s] = zk;
#pragma unroll
      for (int t = 0; t < RT; ++t) {
        const int r = lane + 32 * t;
        if (r > k && r < R) y[t] -= L[r * ldl + k] * zk;
      }
    }
  }
  // backward: L^T x = z
#pragma unroll
  for (int s = RT - 1; s >= 0; --s) {
    for (int kk = 31; kk >= 0; --kk) {
      const int k = s * 32 + kk;
      if (k >= R) continue;
      double xk = y[s] * inv_diag[k];
      xk = __shfl_sync(0xffffffffu, xk, kk);
      if (lane == kk) y[s] = xk;
#pragma unroll
      for (int t = 0; t < RT; ++t) {
        const int r = lane + 32 * t;
        if (r < k) y[t] -= L[k * ldl + r] * xk;
      }
    }
  }
}

// Sum of the MTTKRP split partials of the block's elements [base, base+cnt)
// (rows * R contiguous values) into out[0, npm).  With npm < kUpdThreads,
// kUpdThreads / npm threads share an element, each summing a fixed strided
// subset of the splits with 8 independent loads in flight, then the subsets
// are combined in fixed order; all orders are fixed, so the sum is
// deterministic.  Ends with a barrier.
__device__ void split_sum(const FactorUpdateParams& p, int64_t base, int cnt, int npm, double* out,
                          double* scratch) {
  const int R = p.R;
  const int64_t nM = p.rows * R;
  const int K = npm >= kUpdThreads ? 1 : kUpdThreads / npm;
  auto partial = [&](int e, int k) {
    const int64_t g = base + e;
    const int ns = g / R >= p.tail_row0 ? p.splits_tail : p.splits;
    const double* src = p.mtt + g;
    double a[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    for (int s0 = k; s0 < ns; s0 += 8 * K) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int sp = s0 + u * K;
        if (sp < ns) a[u] += src[static_cast<int64_t>(sp) * nM];
      }
    }
    return ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
  };
  if (K == 1) {
    for (int e = threadIdx.x; e < npm; e += blockDim.x) out[e] = e < cnt ? partial(e, 0) : 0.0;
  } else {
    const int t = threadIdx.x, e = t % npm, k = t / npm;
    double v = 0.0;
    if (k < K && e < cnt && !(kDiagBuild && (p.debug & 1))) v = partial(e, k);
    scratch[t] = v;
    __syncthreads();
    if (t < npm) {
      double acc = 0.0;
      for (int kk = 0; kk < K; ++kk) acc += scratch[kk * npm + t];
      out[t] = acc;
    }
  }
  __syncthreads();
}

// aux = project(F + Y/rho) (solver.py:311-314, constraints.py:105-111),
// Y += rho (F - aux) (solver.py:315-317); residual terms into the scaled norms
__device__ __forceinline__ void admm_apply(const FactorUpdateParams& p, int64_t g, double x,
                                           double a, double rho, ScaledSq (&nrm)[5]) {
  const double yd = p.dual[g];
  const double a_old = p.aux[g];
  const double ynew = yd + rho * (x - a);
  p.aux[g] = a;
  p.dual[g] = ynew;
  nrm[0].add(x - a);
  nrm[1].add(a - a_old);
  nrm[2].add(x);
  nrm[3].add(a);
  nrm[4].add(ynew);
}

__device__ __forceinline__ void admm_step(const FactorUpdateParams& p, int64_t g, double x,
                                          double rho, ScaledSq (&nrm)[5]) {
  const double v = x + p.dual[g] / rho;
  if (!isfinite(v)) raise_status(p.status, kDevNonFinite);
  if (p.kind == kConstraintCard) {  // projection needs the whole matrix: card_apply
    p.cand[g] = v;
    return;
  }
  admm_apply(p, g, x, v > 0.0 ? v : 0.0, rho, nrm);
}

// Row-stochastic projection of one row (constraints.py:72-92) by one warp:
// v[0..R) in shared memory (u: R doubles of scratch) -> a[c] for the lane's
// columns c = lane + 32 t.  Sort-and-threshold: u = v sorted descending
// (rank by value, ties by index), css = running sums (in order, as
// np.cumsum), k = #{j: u_j (j+1) > css_j - 1}, theta = (css_{k-1} - 1)/k,
// a = max(v - theta, 0); a row already on the simplex (min >= 0,
// |sum - 1| <= 8 eps R) is returned unchanged.
template <int RT>
__device__ void simplex_row(const double* v, double* u, int R, int lane, double (&a)[RT]) {
#pragma unroll
  for (int t = 0; t < RT; ++t) {
    const int c = lane + 32 * t;
    if (c < R) {
      const double vc = v[c];
      int rank = 0;
      for (int j = 0; j < R; ++j) {
        const double vj = v[j];
        rank += (vj > vc || (vj == vc && j < c)) ? 1 : 0;
      }
      u[rank] = vc;
    }
  }
  __syncwarp();
  double theta = 0.0;
  int feasible = 0;
  if (lane == 0) {
    double css = 0.0, mn = v[0], sum = 0.0;
    int k = 0;
    for (int j = 0; j < R; ++j) {
      css += u[j];
      k += (u[j] * (j + 1) > css - 1.0) ? 1 : 0;  // count, as np.count_nonzero
      u[j] = css;                                 // u now holds the running sums
      mn = fmin(mn, v[j]);
      sum += v[j];
    }
    theta = (u[k - 1] - 1.0) / k;
    feasible = (mn >= 0.0 && fabs(sum - 1.0) <= 8.0 * 2.220446049250313e-16 * R) ? 1 : 0;
  }
  theta = __shfl_sync(0xffffffffu, theta, 0);
  feasible = __shfl_sync(0xffffffffu, feasible, 0);
#pragma unroll
  for (int t = 0; t < RT; ++t) {
    const int c = lane + 32 * t;
    a[t] = 0.0;
    if (c < R) {
      const double d = v[c] - theta;
      a[t] = feasible ? v[c] : (d > 0.0 ? d : 0.0);
    }
  }
  __syncwarp();
}

// Block epilogue: scaled-norm partial (last sweep), Gram partial of the
// block's new rows and the column maxima (fuse_gram).  xr: [rpb][R] new rows
// (zero for rows past the end).  red: >= 80 doubles of scratch.
__device__ void block_partials(const FactorUpdateParams& p, ScaledSq (&nrm)[5], const double* xr,
                               int rpb, double* red) {
  const int R = p.R;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int nwarps = kUpdThreads / 32;
  if (p.last_sweep && p.kind != kConstraintCard) {
#pragma unroll
    for (int c = 0; c < 5; ++c) {
      ScaledSq v = nrm[c];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double s2 = __shfl_xor_sync(0xffffffffu, v.scale, o);
        const double q2 = __shfl_xor_sync(0xffffffffu, v.ssq, o);
        v.merge(s2, q2);
      }
      if (lane == 0) {
        red[(warp * 5 + c) * 2] = v.scale;
        red[(warp * 5 + c) * 2 + 1] = v.ssq;
      }
    }
    __syncthreads();
    if (threadIdx.x < 5) {
      ScaledSq acc;
      for (int w = 0; w < nwarps; ++w)
        acc.merge(red[(w * 5 + threadIdx.x) * 2], red[(w * 5 + threadIdx.x) * 2 + 1]);
      p.norm_partials[(blockIdx.x * 5 + threadIdx.x) * 2] = acc.scale;
      p.norm_partials[(blockIdx.x * 5 + threadIdx.x) * 2 + 1] = acc.ssq;
    }
  }
  if (p.fuse_gram) {
    // G_m: recomputed from the new rows by the next MTTKRP's ridge CTA
    // (gram_pending), or from per-block partials reduced on the side stream
    if (p.gram_pending && blockIdx.x == 0 && threadIdx.x == 0) *p.gram_pending = 1;
    double* gp = p.gram_partials ? p.gram_partials + static_cast<int64_t>(blockIdx.x) * R * R : nullptr;
    for (int e = threadIdx.x; gp && e < R * R; e += blockDim.x) {
      const int r = e / R, c = e - (e / R) * R;
      double acc = 0.0;
      for (int lr = 0; lr < rpb; ++lr) acc += xr[lr * R + r] * xr[lr * R + c];
      gp[e] = acc;
    }
    // max |F[:, r]| (W scales of the next tensor-core MTTKRPs): non-negative
    // doubles order like their IEEE bits, so an integer atomicMax is exact
    if (p.colmax_bits)
      for (int r = threadIdx.x; r < R; r += blockDim.x) {
        double mx = 0.0;
        for (int lr = 0; lr < rpb; ++lr) mx = fmax(mx, fabs(xr[lr * R + r]));
        if (mx > 0.0) atomicMax(p.colmax_bits + r, static_cast<unsigned long long>(__double_as_longlong(mx)));
      }
  }
}

// R <= 64: all rows of the block at once as small GEMMs against the ridge
// inverse, with one step of iterative refinement against H itself:
//   x1 = y H^-1,  x = x1 + (y - x1 H) H^-1
// Every (row, column) pair is independent: no sequential substitution chain
// on the critical path.  Agreement with cho_solve (solver.py:188) is at the
// backward-error level.
template <int KIND>
__global__ void __launch_bounds__(kUpdThreads) factor_update_gemv_kernel(FactorUpdateParams p) {
  pdl_trigger();
  if (p.stop_flag && *p.stop_flag) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int R = p.R;
  const int rpb = rows_per_block(R, p.rows);
  const int npm = rpb * R;
  double* Hi = reinterpret_cast<double*>(smem_raw);  // [R][R] H^-1
  double* Hm = Hi + R * R;                            // [R][R] H
  double* yb = Hm + R * R;                            // [npm] rhs, then residual
  double* x1 = yb + npm;
  double* ms = x1 + npm;                              // MTTKRP row sums
  double* ax = ms + npm;                              // aux rows
  double* dl = ax + npm;                              // dual rows
  double* xr = dl + npm;                              // new rows
  double* scr = xr + npm;                             // [kUpdThreads] scratch
  double* gs = scr + kUpdThreads;                     // [R + 8]: g1 = H^-1 1, sum(g1), lambdas
  const int64_t base = static_cast<int64_t>(blockIdx.x) * npm;
  const int64_t nM = p.rows * R;
  const int cnt = static_cast<int>(nM - base < npm ? nM - base : npm);
  constexpr bool rowstoch = KIND == kConstraintRowStochastic;
  // loads that do not depend on the preceding kernel first
  for (int e = threadIdx.x; e < npm; e += blockDim.x) {
    ax[e] = e < cnt ? p.aux[base + e] : 0.0;
    dl[e] = e < cnt ? p.dual[base + e] : 0.0;
  }
  const double rho = p.rho[p.mode - 1];
  auto load_ridge = [&]() {
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
      Hi[e] = p.Lg[R * R + R + e];
      Hm[e] = p.Lg[2 * R * R + R + e];
    }
  };
  // The side-stream ridge is event-joined (complete): prefetch it.  The
  // MTTKRP partials, a ridge computed by the preceding kernel, and every
  // write below follow the preceding kernel.
  if (!p.ridge_in_pred) {
    if (*p.status == kDevNotPD) return;
    load_ridge();
  }
  pdl_wait();
  // The early stop-flag read above can precede the kernel that sets the flag
  // (eager launches overlap through PDL); re-read it here, in flight with the
  // partials, and skip every write if the fit has stopped.
  const int stopped = p.stop_flag ? *reinterpret_cast<const volatile int*>(p.stop_flag) : 0;
  if (p.ridge_in_pred) {
    if (*p.status == kDevNotPD) return;
    load_ridge();
  }
  split_sum(p, base, cnt, npm, ms, scr);
  if (stopped) return;
  if (rowstoch) {  // g1 = (G + rho I)^-1 1 (solver.py:190), refined like the rows
    for (int c = threadIdx.x; c < R; c += blockDim.x) {
      double acc = 0.0;
      for (int k = 0; k < R; ++k) acc += Hi[k * R + c];
      gs[c] = acc;
    }
    __syncthreads();
    for (int c = threadIdx.x; c < R; c += blockDim.x) {
      double acc = 1.0;
      for (int k = 0; k < R; ++k) acc = fma(-gs[k], Hm[k * R + c], acc);
      x1[c] = acc;
    }
    __syncthreads();
    for (int c = threadIdx.x; c < R; c += blockDim.x) {
      double acc = gs[c];
      for (int k = 0; k < R; ++k) acc = fma(x1[k], Hi[k * R + c], acc);
      scr[c] = acc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double sg = 0.0;
      for (int c = 0; c < R; ++c) {
        gs[c] = scr[c];
        sg += scr[c];
      }
      gs[R] = sg;
    }
  }
  for (int e = threadIdx.x; e < npm; e += blockDim.x)
    yb[e] = e < cnt ? (ms[e] + rho * ax[e]) - dl[e] : 0.0;  // ridge_rhs (solver.py:178-179)
  __syncthreads();
  for (int e = threadIdx.x; e < npm; e += blockDim.x) {
    const int lr = e / R, c = e - (e / R) * R;
    double acc = 0.0;
    for (int k = 0; k < R; ++k) acc = fma(yb[lr * R + k], Hi[k * R + c], acc);
    x1[e] = acc;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < npm; e += blockDim.x) {  // residual y - x1 H
    const int lr = e / R, c = e - (e / R) * R;
    double acc = yb[e];
    for (int k = 0; k < R; ++k) acc = fma(-x1[lr * R + k], Hm[k * R + c], acc);
    xr[e] = acc;
  }
  __syncthreads();
  ScaledSq nrm[5];
  double xv[(64 * 2 + kUpdThreads - 1) / kUpdThreads];
#pragma unroll
  for (int u = 0; u < (64 * 2 + kUpdThreads - 1) / kUpdThreads; ++u) {
    const int e = threadIdx.x + u * kUpdThreads;
    xv[u] = 0.0;
    if (e < npm) {
      const int lr = e / R, c = e - (e / R) * R;
      double acc = x1[e];
      for (int k = 0; k < R; ++k) acc = fma(xr[lr * R + k], Hi[k * R + c], acc);
      xv[u] = e < cnt ? acc : 0.0;
    }
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < (64 * 2 + kUpdThreads - 1) / kUpdThreads; ++u) {
    const int e = threadIdx.x + u * kUpdThreads;
    if (e < npm) xr[e] = xv[u];
  }
  __syncthreads();
  if (rowstoch) {
    // rows summing to one (solver.py:189-193): x += lam g1, lam = (1 - x 1)/sum(g1)
    if (threadIdx.x < rpb) {
      double sx = 0.0;
      for (int c = 0; c < R; ++c) sx += xr[threadIdx.x * R + c];
      gs[R + 1 + threadIdx.x] = (1.0 - sx) / gs[R];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < npm; e += blockDim.x) {
      const int lr = e / R, c = e - (e / R) * R;
      if (e < cnt) xr[e] = fma(gs[R + 1 + lr], gs[c], xr[e]);
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < cnt; e += blockDim.x) {
    const int64_t g = base + e;
    p.F[p.row_offset * R + g] = xr[e];
    if (p.last_sweep && !rowstoch) admm_step(p, g, xr[e], rho, nrm);
  }
  if (p.last_sweep && rowstoch) {  // per-row simplex projection, one warp per row
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int lr = warp; lr < rpb && lr * R < cnt; lr += kUpdThreads / 32) {
      double* v = x1 + lr * R;
      double* u = yb + lr * R;
      for (int c = lane; c < R; c += 32) {
        const double vc = xr[lr * R + c] + dl[lr * R + c] / rho;
        if (!isfinite(vc)) raise_status(p.status, kDevNonFinite);
        v[c] = vc;
      }
      __syncwarp();
      double a[2];
      simplex_row<2>(v, u, R, lane, a);
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int c = lane + 32 * t;
        if (c < R) admm_apply(p, base + lr * R + c, xr[lr * R + c], a[t], rho, nrm);
      }
    }
  }
  __syncthreads();
  block_partials(p, nrm, xr, rpb, scr);
}

// R > 64: one row per warp, forward/backward substitution against L.
constexpr int kUpdSmemMaxR = 128;
template <int RT, int KIND>
__global__ void __launch_bounds__(kUpdThreads) factor_update_warp_kernel(FactorUpdateParams p) {
  pdl_trigger();
  if (p.stop_flag && *p.stop_flag) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int R = p.R;
  // L in shared memory with an odd pitch (conflict-free row and column
  // walks); above kUpdSmemMaxR it is read in place from the ridge buffer
  // (global memory, L2-resident)
  const bool l_global = R > kUpdSmemMaxR;
  const int ldl = l_global ? R : R + 1;
  const int rpb = rows_per_block(R, p.rows);
  const int npm = rpb * R;
  double* Ls = reinterpret_cast<double*>(smem_raw);
  double* inv_s = Ls + R * ldl;                // [R]
  double* ms = l_global ? Ls : inv_s + R;      // [npm] MTTKRP row sums
  const double* L = l_global ? p.Lg : Ls;
  const double* inv_diag = l_global ? p.Lg + R * R : inv_s;
  double* xr = ms + npm;           // [npm] new rows
  double* scr = xr + npm;          // [kUpdThreads]
  double* gs = scr + kUpdThreads;  // [R + 8] g1 = (G + rho I)^-1 1 and its sum
  double* vb = gs + R + 8;         // [warps][R] projection input rows
  double* ub = vb + (kUpdThreads / 32) * R;  // [warps][R] projection scratch
  const int64_t base = static_cast<int64_t>(blockIdx.x) * npm;
  const int64_t nM = p.rows * R;
  const int cnt = static_cast<int>(nM - base < npm ? nM - base : npm);
  const double rho = p.rho[p.mode - 1];
  constexpr bool rowstoch = KIND == kConstraintRowStochastic;
  pdl_wait();  // MTTKRP partials and ridge factor
  const int stopped = p.stop_flag ? *reinterpret_cast<const volatile int*>(p.stop_flag) : 0;
  if (*p.status == kDevNotPD || stopped) return;
  if (!l_global) {
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
      const int i = e / R, k = e - (e / R) * R;
      Ls[i * ldl + k] = p.Lg[e];
    }
    for (int j = threadIdx.x; j < R; j += blockDim.x) inv_s[j] = p.Lg[R * R + j];
  }
  split_sum(p, base, cnt, npm, ms, scr);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (rowstoch) {  // g1 = cho_solve(ones) (solver.py:190) by warp 0
    if (warp == 0) {
      double y1[RT];
#pragma unroll
      for (int t = 0; t < RT; ++t) y1[t] = (lane + 32 * t) < R ? 1.0 : 0.0;
      warp_chol_solve<RT>(y1, L, ldl, R, inv_diag, lane);
#pragma unroll
      for (int t = 0; t < RT; ++t)
        if (lane + 32 * t < R) gs[lane + 32 * t] = y1[t];
      __syncwarp();
      if (lane == 0) {
        double sg = 0.0;
        for (int c = 0; c < R; ++c) sg += gs[c];
        gs[R] = sg;
      }
    }
    __syncthreads();
  }
  ScaledSq nrm[5];
  for (int lr = warp; lr < rpb; lr += kUpdThreads / 32) {
    const bool valid = lr * R < cnt;
    double y[RT];
#pragma unroll
    for (int t = 0; t < RT; ++t) {
      const int r = lane + 32 * t;
      y[t] = 0.0;
      if (valid && r < R) {
        const int64_t g = base + lr * R + r;
        y[t] = (ms[lr * R + r] + rho * p.aux[g]) - p.dual[g];  // ridge_rhs
      }
    }
    if (valid) warp_chol_solve<RT>(y, L, ldl, R, inv_diag, lane);
    if (rowstoch && valid) {  // rows summing to one (solver.py:189-193)
      double sx = 0.0;
#pragma unroll
      for (int t = 0; t < RT; ++t) sx += y[t];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sx += __shfl_xor_sync(0xffffffffu, sx, o);
      const double lam = (1.0 - sx) / gs[R];
#pragma unroll
      for (int t = 0; t < RT; ++t)
        if (lane + 32 * t < R) y[t] = fma(lam, gs[lane + 32 * t], y[t]);
    }
#pragma unroll
    for (int t = 0; t < RT; ++t) {
      const int r = lane + 32 * t;
      if (r < R) {
        xr[lr * R + r] = valid ? y[t] : 0.0;
        if (valid) {
          const int64_t g = base + lr * R + r;
          p.F[p.row_offset * R + g] = y[t];
          if (p.last_sweep && !rowstoch) admm_step(p, g, y[t], rho, nrm);
        }
      }
    }
    if (p.last_sweep && rowstoch && valid) {  // per-row simplex projection
      double* v = vb + warp * R;
      double* u = ub + warp * R;
#pragma unroll
      for (int t = 0; t < RT; ++t) {
        const int r = lane + 32 * t;
        if (r < R) {
          const double vc = y[t] + p.dual[base + lr * R + r] / rho;
          if (!isfinite(vc)) raise_status(p.status, kDevNonFinite);
          v[r] = vc;
        }
      }
      __syncwarp();
      double a[RT];
      simplex_row<RT>(v, u, R, lane, a);
#pragma unroll
      for (int t = 0; t < RT; ++t) {
        const int r = lane + 32 * t;
        if (r < R) admm_apply(p, base + lr * R + r, y[t], a[t], rho, nrm);
      }
    }
  }
  __syncthreads();
  block_partials(p, nrm, xr, rpb, scr);
}

// G[e] = sum_b part[b][e]: kGramSub threads per element each sum a fixed
// strided subset of the blocks (8 independent loads in flight), then the
// subsets are added in fixed order.  On the plan's side stream, it only
// feeds the next ridge factorisation.
constexpr int kGramSub = 8;

__global__ void gram_reduce_kernel(const double* __restrict__ part, int nb, int n,
                                   double* __restrict__ G, const int* stop_flag) {
  if (stop_flag && *stop_flag) return;
  __shared__ double sub[kGramSub][32];
  const int el = threadIdx.x & 31, k = threadIdx.x >> 5;  // 32 elements x kGramSub subsets
  const int e = blockIdx.x * 32 + el;
  double a[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  if (e < n) {
    for (int b0 = k; b0 < nb; b0 += 8 * kGramSub) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int b = b0 + u * kGramSub;
        if (b < nb) a[u] += part[static_cast<int64_t>(b) * n + e];
      }
    }
  }
  sub[k][el] = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
  __syncthreads();
  if (k == 0 && e < n) {
    double acc = 0.0;
    for (int kk = 0; kk < kGramSub; ++kk) acc += sub[kk][el];
    G[e] = acc;
  }
}

// norm_acc[c] = merge_b part[b][c] (5 scaled norms): 32 chains per norm, each
// merging a fixed strided subset of the blocks (loads issued first), then
// the chains merged in order.
__global__ void norm_reduce_kernel(const double* __restrict__ part, int nb, double* __restrict__ out,
                                   const int* stop_flag) {
  pdl_trigger();
  pdl_wait();
  if (stop_flag && *stop_flag) return;
  __shared__ double red[5][32][2];
  const int c = threadIdx.x >> 5, ch = threadIdx.x & 31;  // 5 warps: norm c, chain ch
  if (c < 5) {
    ScaledSq acc;
    for (int b0 = ch; b0 < nb; b0 += 4 * 32) {
      double s2[4], q2[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int b = b0 + u * 32;
        s2[u] = b < nb ? part[(b * 5 + c) * 2] : 0.0;
        q2[u] = b < nb ? part[(b * 5 + c) * 2 + 1] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) acc.merge(s2[u], q2[u]);
    }
    red[c][ch][0] = acc.scale;
    red[c][ch][1] = acc.ssq;
  }
  __syncthreads();
  if (threadIdx.x < 5) {
    ScaledSq acc;
    for (int k = 0; k < 32; ++k) acc.merge(red[threadIdx.x][k][0], red[threadIdx.x][k][1]);
    out[threadIdx.x * 2] = acc.scale;
    out[threadIdx.x * 2 + 1] = acc.ssq;
  }
}

// ---------------------------------------------------------------------------
// Gram G = F^T F, two-pass deterministic (partials per row block, then sum).
// ---------------------------------------------------------------------------
constexpr int kGramRows = 64;

__global__ void gram_partial_kernel(const double* __restrict__ F, int64_t rows, int R,
                                    double* __restrict__ part) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* fs = reinterpret_cast<double*>(smem_raw);  // [kGramRows][R]
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * kGramRows;
  for (int e = threadIdx.x; e < kGramRows * R; e += blockDim.x) {
    const int64_t row = r0 + e / R;
    fs[e] = row < rows ? F[r0 * R + e] : 0.0;
  }
  __syncthreads();
  double* gp = part + static_cast<int64_t>(blockIdx.x) * R * R;
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    const int r = e / R, s = e - (e / R) * R;
    double acc = 0.0;
    for (int lr = 0; lr < kGramRows; ++lr) acc += fs[lr * R + r] * fs[lr * R + s];
    gp[e] = acc;
  }
}

__global__ void sum_partials_kernel(const double* __restrict__ part, int64_t nparts, int64_t n,
                                    double* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t b = 0; b < nparts; ++b) s += part[b * n + e];
    out[e] = s;
  }
}

// ---------------------------------------------------------------------------
// Close one outer iteration: residuals (solver.py:247-255), stop test
// (solver.py:258-269), penalty adaptation (solver.py:272-292).
// ---------------------------------------------------------------------------
__global__ void finalize_kernel(FinalizeParams p) {
  // thread (m, c) < 5*order merges the shards' (scale, ssq) pairs of one norm
  // in rank order; thread 0 then closes the iteration
  __shared__ double nv[20];
  const int N = p.order;
  int* ctr = p.counters;
  if (ctr[1]) return;  // already stopped: iteration is a no-op
  if (threadIdx.x < 5 * N) {
    ScaledSq a;
    for (int q = 0; q < p.norm_parts; ++q) {
      const double* s = p.norm_acc + (q * 5 * N + threadIdx.x) * 2;
      a.merge(s[0], s[1]);
    }
    nv[threadIdx.x] = a.norm();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const int64_t it = ctr[0];
  double primal[4], dual[4];
  bool stop = true;
  for (int m = 0; m < N; ++m) {
    const double a[5] = {nv[m * 5], nv[m * 5 + 1], nv[m * 5 + 2], nv[m * 5 + 3], nv[m * 5 + 4]};
    primal[m] = a[0];
    dual[m] = p.rho[m] * a[1];
    const double base = sqrt(static_cast<double>(p.dims[m]) * p.R) * p.eps_abs;
    const double fn = a[2], an = a[3], yn = a[4];
    const double pthr = base + p.eps_rel * (fn > an ? fn : an);
    const double dthr = base + p.eps_rel * yn;
    if (primal[m] > pthr || dual[m] > dthr) stop = false;
  }
  double rho_new[4];
  for (int m = 0; m < N; ++m) {
    const double r = p.rho[m];
    if (p.rho_schedule && it < p.history_capacity) {
      rho_new[m] = p.rho_schedule[it * N + m];
    } else if (!p.adapt) {
      rho_new[m] = r;
    } else if (primal[m] > p.mu * dual[m]) {
      rho_new[m] = r * p.tau_incr;
    } else if (dual[m] > p.mu * primal[m] && primal[m] > 0.0) {
      rho_new[m] = r / p.tau_decr;
    } else {
      rho_new[m] = r;
    }
  }
  if (it < p.history_capacity) {
    for (int m = 0; m < N; ++m) {
      p.resid_history[it * 2 * N + m] = primal[m];
      p.resid_history[it * 2 * N + N + m] = dual[m];
      p.rho_history[it * N + m] = rho_new[m];
    }
  }
  for (int m = 0; m < N; ++m) p.rho[m] = rho_new[m];
  ctr[0] = static_cast<int>(it + 1);
  if (stop) ctr[1] = 1;
}

// ---------------------------------------------------------------------------
// sum x^2 and sum (x - [[A,B,C]])^2 with fp64 accumulation (tensors.py:57-61,
// 276-290).  Block = one i and kSqJ consecutive j; threads along k.
// ---------------------------------------------------------------------------
constexpr int kSqJ = 8;        // j values per block: narrow tensors
constexpr int kSqJWide = 32;   // ... and the others (C^T is re-read from L2 once per block: 1/4 of the traffic)
constexpr int kSqThreads = 256;

// the norm-only pass (no model) streams X: narrow tiles, more blocks per SM
__host__ __device__ constexpr int sq_jt(int64_t J, bool model) { return model && J >= 24 ? kSqJWide : kSqJ; }

template <typename XT, int JT>
__global__ void __launch_bounds__(kSqThreads) sq_error_kernel(const XT* __restrict__ X, int64_t I,
                                                              int64_t J, int64_t K,
                                                              const double* __restrict__ A,
                                                              const double* __restrict__ B,
                                                              const double* __restrict__ CT,
                                                              int R, double* __restrict__ part) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* ab = reinterpret_cast<double*>(smem_raw);  // [R][JT]: A[i, r] * B[j0 + jj, r]
  const int64_t nj_blocks = (J + JT - 1) / JT;
  const int64_t i = blockIdx.x / nj_blocks;
  const int64_t j0 = (blockIdx.x - i * nj_blocks) * JT;
  const bool model = A != nullptr;
  if (model) {
    for (int e = threadIdx.x; e < JT * R; e += blockDim.x) {
      const int r = e / JT, jj = e - r * JT;
      const int64_t j = j0 + jj;
      ab[e] = j < J ? A[i * R + r] * B[j * R + r] : 0.0;
    }
  }
  __syncthreads();
  double sx = 0.0, se = 0.0;
  for (int64_t k = threadIdx.x; k < K; k += blockDim.x) {
    double rec[JT];
#pragma unroll
    for (int jj = 0; jj < JT; ++jj) rec[jj] = 0.0;
    if (model) {
      for (int r = 0; r < R; ++r) {
        const double c = CT[static_cast<int64_t>(r) * K + k];
        const double2* abr = reinterpret_cast<const double2*>(ab + r * JT);  // 16-byte broadcasts
#pragma unroll
        for (int jj = 0; jj < JT; jj += 2) {
          const double2 v = abr[jj >> 1];
          rec[jj] = fma(v.x, c, rec[jj]);
          rec[jj + 1] = fma(v.y, c, rec[jj + 1]);
        }
      }
    }
#pragma unroll
    for (int jj = 0; jj < JT; ++jj) {
      const int64_t j = j0 + jj;
      if (j < J) {
        const double x = static_cast<double>(X[(i * J + j) * K + k]);
        const double d = x - rec[jj];
        sx += x * x;
        se += d * d;
      }
    }
  }
  __shared__ double red[2][kSqThreads / 32];
  sx = warp_sum(sx);
  se = warp_sum(se);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    red[0][warp] = sx;
    red[1][warp] = se;
  }
  __syncthreads();
  if (threadIdx.x < 2) {
    double s = 0.0;
    for (int w = 0; w < kSqThreads / 32; ++w) s += red[threadIdx.x][w];
    part[static_cast<int64_t>(blockIdx.x) * 2 + threadIdx.x] = s;
  }
}

// The same sums on the fp64 tensor pipe, for tensors at least kSqJWide wide
// with a model: a block owns one i and kSqJWide j values and walks k in tiles
// of 256; each warp reconstructs a 32 (j) x 32 (k) tile as m8n8k4 DMMA
// fragments, D[j][k] += (A[i, r] B[j, r]) C[k, r] (A operand: the A*B rows in
// shared memory, pitch 4 mod 16 doubles; B operand: C^T rows from L2, 64-byte
// pieces), then subtracts it from X in the accumulator-fragment layout (each
// lane reads two consecutive k of one j row: full 32-byte sectors).  The
// products a*b are rounded once and the sums over r run in fp64, as
// tensors.reconstruct; the order of the r sum differs from the FMA kernel's
// at the 1e-16 level.  Per-thread partial sums in a fixed order: deterministic.
template <typename XT>
__global__ void __launch_bounds__(kSqThreads, 2) sq_error_dmma_kernel(const XT* __restrict__ X, int64_t I,
                                                                      int64_t J, int64_t K,
                                                                      const double* __restrict__ A,
                                                                      const double* __restrict__ B,
                                                                      const double* __restrict__ CT,
                                                                      int R, int pitch,
                                                                      double* __restrict__ part) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* ab = reinterpret_cast<double*>(smem_raw);  // [kSqJWide][pitch]: A[i, r] * B[j0 + jj, r], zero padded
  constexpr int JT = kSqJWide;
  const int64_t nj_blocks = (J + JT - 1) / JT;
  const int64_t i = blockIdx.x / nj_blocks;
  const int64_t j0 = (blockIdx.x - i * nj_blocks) * JT;
  const int R4 = (R + 3) & ~3;
  for (int e = threadIdx.x; e < JT * R4; e += blockDim.x) {
    const int jj = e / R4, r = e - jj * R4;
    const int64_t j = j0 + jj;
    ab[jj * pitch + r] = (j < J && r < R) ? A[i * R + r] * B[j * R + r] : 0.0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  double sx = 0.0, se = 0.0;
  for (int64_t kt = static_cast<int64_t>(warp) * 32; kt < K; kt += (kSqThreads / 32) * 32) {
    double d[4][4][2];  // [j block][k block][2]
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) d[a][b][0] = d[a][b][1] = 0.0;
    // B fragment rows: C^T[r + t4][kt + 8 b + g] (zero outside K or R)
    int64_t kb[4];
    bool kv[4];
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      kb[b] = kt + 8 * b + g;
      kv[b] = kb[b] < K;
    }
    for (int r = 0; r < R4; r += 4) {
      const bool rv = r + t4 < R;
      const double* ctr = CT + static_cast<int64_t>(r + t4) * K;
      double bf[4], af[4];
#pragma unroll
      for (int b = 0; b < 4; ++b) bf[b] = (rv && kv[b]) ? ctr[kb[b]] : 0.0;
#pragma unroll
      for (int a = 0; a < 4; ++a) af[a] = ab[(8 * a + g) * pitch + r + t4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                       : "+d"(d[a][b][0]), "+d"(d[a][b][1])
                       : "d"(af[a]), "d"(bf[b]));
    }
    // D[j = 8 a + g][k = kt + 8 b + 2 t4 + {0, 1}] against X
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int64_t j = j0 + 8 * a + g;
      if (j >= J) continue;
      const XT* xr = X + (i * J + j) * K;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int64_t k = kt + 8 * b + 2 * t4;
#pragma unroll
        for (int u = 0; u < 2; ++u)
          if (k + u < K) {
            const double x = static_cast<double>(xr[k + u]);
            const double df = x - d[a][b][u];
            sx += x * x;
            se += df * df;
          }
      }
    }
  }
  __shared__ double red[2][kSqThreads / 32];
  sx = warp_sum(sx);
  se = warp_sum(se);
  if (lane == 0) {
    red[0][warp] = sx;
    red[1][warp] = se;
  }
  __syncthreads();
  if (threadIdx.x < 2) {
    double s = 0.0;
    for (int w = 0; w < kSqThreads / 32; ++w) s += red[threadIdx.x][w];
    part[static_cast<int64_t>(blockIdx.x) * 2 + threadIdx.x] = s;
  }
}

__global__ void transpose_kernel(const double* __restrict__ C, int64_t K, int R,
                                 double* __restrict__ CT) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < K * R;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = e / R;
    const int r = static_cast<int>(e - k * R);
    CT[static_cast<int64_t>(r) * K + k] = C[e];
  }
}

// fixed-order tree-free reduction of [n][2] partials into out2 (one block)
__global__ void sum_pairs_kernel(const double* __restrict__ part, int64_t n,
                                 double* __restrict__ out2) {
  __shared__ double red[2][256];
  for (int c = 0; c < 2; ++c) {
    double s = 0.0;
    for (int64_t b = threadIdx.x; b < n; b += blockDim.x) s += part[b * 2 + c];
    red[c][threadIdx.x] = s;
  }
  __syncthreads();
  if (threadIdx.x < 2) {
    double s = 0.0;
    for (int t = 0; t < static_cast<int>(blockDim.x); ++t) s += red[threadIdx.x][t];
    out2[threadIdx.x] = s;
  }
}



// ---------------------------------------------------------------------------
// Cardinality projection (constraints.py:95-102): keep the c largest clamped
// entries of the mode's matrix, ties by smaller row-major index.  Clamped
// values are non-negative, so their IEEE bits order like the values.
// ---------------------------------------------------------------------------
constexpr int kSelThreads = 1024;

__device__ __forceinline__ unsigned long long card_key(double v) {
  return v > 0.0 ? static_cast<unsigned long long>(__double_as_longlong(v)) : 0ull;
}

// One block: MSB-first radix select (8 passes of 8 bits, shared histograms)
// of the c-th largest key T, then an ordered scan for the index cut among
// the keys equal to T.  Integer counts only: deterministic.
__global__ void __launch_bounds__(kSelThreads) card_select_kernel(const double* __restrict__ cand,
                                                                  int64_t n, int64_t c,
                                                                  unsigned long long* sel,
                                                                  const int* stop_flag) {
  if (stop_flag && *stop_flag) return;
  __shared__ unsigned int hist[256];
  __shared__ unsigned long long s_prefix;
  __shared__ long long s_remaining;
  __shared__ long long scan[kSelThreads];
  if (c >= n) {  // every clamped entry is kept
    if (threadIdx.x == 0) {
      sel[0] = 0ull;
      sel[1] = static_cast<unsigned long long>(n);
    }
    return;
  }
  if (threadIdx.x == 0) {
    s_prefix = 0ull;
    s_remaining = c;
  }
  unsigned long long mask = 0ull;
  for (int pass = 7; pass >= 0; --pass) {
    for (int b = threadIdx.x; b < 256; b += blockDim.x) hist[b] = 0u;
    __syncthreads();
    const unsigned long long prefix = s_prefix;
    const int sh = pass * 8;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
      const unsigned long long k = card_key(cand[i]);
      if ((k & mask) == prefix) atomicAdd(&hist[(k >> sh) & 255ull], 1u);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      long long rem = s_remaining;
      int b = 255;
      for (; b > 0; --b) {
        if (static_cast<long long>(hist[b]) >= rem) break;
        rem -= hist[b];
      }
      s_remaining = rem;
      s_prefix = prefix | (static_cast<unsigned long long>(b) << sh);
    }
    mask |= 255ull << sh;
    __syncthreads();
  }
  const unsigned long long T = s_prefix;
  const long long want = s_remaining;  // ties with key T to keep, in index order
  // ordered scan: thread t owns the contiguous index range [t*chunk, ...)
  const int64_t chunk = (n + blockDim.x - 1) / blockDim.x;
  const int64_t i0 = threadIdx.x * chunk, i1 = i0 + chunk < n ? i0 + chunk : n;
  long long ties = 0;
  for (int64_t i = i0; i < i1; ++i) ties += card_key(cand[i]) == T ? 1 : 0;
  scan[threadIdx.x] = ties;
  __syncthreads();
  if (threadIdx.x == 0) {  // exclusive prefix, in order
    long long acc = 0;
    for (int t = 0; t < static_cast<int>(blockDim.x); ++t) {
      const long long v = scan[t];
      scan[t] = acc;
      acc += v;
    }
  }
  __syncthreads();
  const long long before = scan[threadIdx.x];
  if (before < want && before + ties >= want) {
    long long k = before;
    for (int64_t i = i0; i < i1; ++i) {
      if (card_key(cand[i]) == T && ++k == want) {
        sel[0] = T;
        sel[1] = static_cast<unsigned long long>(i + 1);
        break;
      }
    }
  }
}

// aux / dual / norms with the cardinality projection, same grid and element
// ranges as the row update (its norm partials feed norm_reduce unchanged).
__global__ void __launch_bounds__(kUpdThreads) card_apply_kernel(FactorUpdateParams p,
                                                                 const unsigned long long* sel) {
  if (p.stop_flag && *p.stop_flag) return;
  __shared__ double red[kUpdThreads / 32 * 10];
  const int R = p.R;
  const int npm = rows_per_block(R, p.rows) * R;
  const int64_t base = static_cast<int64_t>(blockIdx.x) * npm;
  const int64_t nM = p.rows * R;
  const int cnt = static_cast<int>(nM - base < npm ? nM - base : npm);
  const double rho = p.rho[p.mode - 1];
  const unsigned long long T = sel[0];
  const int64_t cut = static_cast<int64_t>(sel[1]);
  ScaledSq nrm[5];
  for (int e = threadIdx.x; e < cnt; e += blockDim.x) {
    const int64_t g = base + e;
    const double v = p.cand[g];
    const unsigned long long k = card_key(v);
    const bool keep = k > T || (k == T && p.row_offset * R + g < cut);
    admm_apply(p, g, p.F[p.row_offset * R + g], keep ? (v > 0.0 ? v : 0.0) : 0.0, rho, nrm);
  }
  FactorUpdateParams q = p;
  q.kind = kConstraintNonneg;  // write the norm partials
  q.fuse_gram = 0;
  q.last_sweep = 1;
  block_partials(q, nrm, nullptr, 0, red);
}

// Khatri-Rao pair for the order-4 views (tensors.py:203-220 restated for two
// factors, rows a*nb + b); block 0 also refreshes the view's column maxima.
__global__ void kr_merge_kernel(KrMergeParams p) {
  pdl_trigger();
  pdl_wait();  // the factors come from the preceding row updates
  if (p.stop_flag && *p.stop_flag) return;
  const int R = p.R;
  const int64_t n = p.na * p.nb * R;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(e % R);
    const int64_t row = e / R;
    const int64_t a = row / p.nb, b = row - (row / p.nb) * p.nb;
    p.out[e] = p.Fa[a * R + r] * p.Fb[b * R + r];
  }
  if (blockIdx.x == 0 && p.cm_view) {
    // max over (a, b) of |Fa Fb| is the rounded product of the maxima
    for (int e = threadIdx.x; e < 3 * R; e += blockDim.x) {
      const int vm = e / R, r = e - (e / R) * R;
      double v = p.cm_src[vm] ? p.cm_src[vm][r] : 0.0;
      if (vm == p.merged_mode) v *= p.cm_src2[r];
      p.cm_view[e] = v;
    }
    __syncthreads();
    if (p.cm_zero)
      for (int r = threadIdx.x; r < R; r += blockDim.x) p.cm_zero[r] = 0.0;
  }
}
}  // namespace

// ---------------------------------------------------------------------------
// host-side launchers
// ---------------------------------------------------------------------------
int factor_update_blocks(int64_t rows, int R) {
  const int rpb = rows_per_block(R, rows);
  return static_cast<int>((rows + rpb - 1) / rpb);
}

size_t factor_update_smem(int R) {
  const size_t npm = static_cast<size_t>(rows_per_block(R, INT64_MAX)) * R;  // the largest block
  size_t n;
  if (R <= 64)
    n = 2 * static_cast<size_t>(R) * R + 6 * npm + kUpdThreads + R + 8;
  else
    n = (R > kUpdSmemMaxR ? 0 : static_cast<size_t>(R) * (R + 1) + R) + 2 * npm + kUpdThreads + R + 8 +
        2 * (kUpdThreads / 32) * static_cast<size_t>(R);
  return n * sizeof(double);
}

size_t ridge_factor_smem(int R) { return static_cast<size_t>(ridge_smem_doubles(R)) * sizeof(double); }

size_t ridge_buffer_doubles(int R) { return 3 * static_cast<size_t>(R) * R + R; }

cudaError_t ridge_factor_launch(const RidgeParams& p, cudaStream_t stream) {
  ridge_factor_kernel<<<1, ridge_threads(p.R), ridge_factor_smem(p.R), stream>>>(p);
  return cudaGetLastError();
}

cudaError_t factor_update_prepare(int R) {
  const size_t smem = factor_update_smem(R);
  cudaError_t e = allow_dyn_smem(reinterpret_cast<const void*>(ridge_factor_kernel), ridge_factor_smem(R));
  if (e != cudaSuccess) return e;
  const void* kerns[] = {
      reinterpret_cast<const void*>(factor_update_gemv_kernel<kConstraintNonneg>),
      reinterpret_cast<const void*>(factor_update_gemv_kernel<kConstraintRowStochastic>),
      reinterpret_cast<const void*>(factor_update_warp_kernel<3, kConstraintNonneg>),
      reinterpret_cast<const void*>(factor_update_warp_kernel<3, kConstraintRowStochastic>),
      reinterpret_cast<const void*>(factor_update_warp_kernel<4, kConstraintNonneg>),
      reinterpret_cast<const void*>(factor_update_warp_kernel<4, kConstraintRowStochastic>),
      reinterpret_cast<const void*>(factor_update_warp_kernel<8, kConstraintNonneg>),
      reinterpret_cast<const void*>(factor_update_warp_kernel<8, kConstraintRowStochastic>)};
  for (const void* k : kerns) {
    e = allow_dyn_smem(k, smem);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t factor_update_launch(const FactorUpdateParams& p_in, cudaStream_t stream) {
  static int dbg = -1;
  if (dbg < 0) {
    const char* env = diag_env("NTF_UPD_DEBUG");
    dbg = env ? atoi(env) : 0;
  }
  FactorUpdateParams p = p_in;
  p.debug = dbg;
  const int blocks = factor_update_blocks(p.rows, p.R);
  const size_t smem = factor_update_smem(p.R);
  // the constraint kind is a template parameter: the nonneg kernels carry
  // no row-stochastic code
  auto launch = [&](auto kern) { return launch_pdl(kern, dim3(blocks), dim3(kUpdThreads), smem, stream, p); };
  const bool rs = p.kind == kConstraintRowStochastic;
  if (p.R <= 64)
    return rs ? launch(factor_update_gemv_kernel<kConstraintRowStochastic>)
              : launch(factor_update_gemv_kernel<kConstraintNonneg>);
  if (p.R <= 96)
    return rs ? launch(factor_update_warp_kernel<3, kConstraintRowStochastic>)
              : launch(factor_update_warp_kernel<3, kConstraintNonneg>);
  if (p.R <= 128)
    return rs ? launch(factor_update_warp_kernel<4, kConstraintRowStochastic>)
              : launch(factor_update_warp_kernel<4, kConstraintNonneg>);
  return rs ? launch(factor_update_warp_kernel<8, kConstraintRowStochastic>)
            : launch(factor_update_warp_kernel<8, kConstraintNonneg>);
}

cudaError_t kr_merge_launch(const KrMergeParams& p, cudaStream_t stream) {
  const int64_t n = p.na * p.nb * p.R;
  const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 4 * 148));
  return launch_pdl(kr_merge_kernel, dim3(blocks > 0 ? blocks : 1), dim3(256), 0, stream, p);
}

cudaError_t card_select_launch(const double* cand, int64_t n, int64_t card, unsigned long long* sel,
                               const int* stop_flag, cudaStream_t stream) {
  card_select_kernel<<<1, kSelThreads, 0, stream>>>(cand, n, card, sel, stop_flag);
  return cudaGetLastError();
}

cudaError_t card_apply_launch(const FactorUpdateParams& p, const unsigned long long* sel,
                              cudaStream_t stream) {
  card_apply_kernel<<<factor_update_blocks(p.rows, p.R), kUpdThreads, 0, stream>>>(p, sel);
  return cudaGetLastError();
}

cudaError_t gram_reduce_launch(const double* part, int nb, int R, double* G, const int* stop_flag,
                               cudaStream_t stream) {
  const int n = R * R;
  gram_reduce_kernel<<<(n + 31) / 32, 32 * kGramSub, 0, stream>>>(part, nb, n, G, stop_flag);
  return cudaGetLastError();
}

cudaError_t norm_reduce_launch(const double* part, int nb, double* out, const int* stop_flag,
                               cudaStream_t stream) {
  return launch_pdl(norm_reduce_kernel, dim3(1), dim3(160), 0, stream, part, nb, out, stop_flag);
}

size_t gram_workspace_bytes(int64_t rows, int R) {
  const int64_t nb = (rows + kGramRows - 1) / kGramRows;
  return static_cast<size_t>(nb) * R * R * sizeof(double);
}

cudaError_t gram_launch(const double* F, int64_t rows, int R, double* G, double* ws,
                        cudaStream_t stream) {
  const int64_t nb = (rows + kGramRows - 1) / kGramRows;
  const size_t smem = static_cast<size_t>(kGramRows) * R * sizeof(double);
  cudaError_t e = allow_dyn_smem(reinterpret_cast<const void*>(gram_partial_kernel), smem);
  if (e != cudaSuccess) return e;
  gram_partial_kernel<<<static_cast<unsigned>(nb), 256, smem, stream>>>(F, rows, R, ws);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int64_t n = static_cast<int64_t>(R) * R;
  sum_partials_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(ws, nb, n, G);
  return cudaGetLastError();
}

cudaError_t finalize_launch(const FinalizeParams& p, cudaStream_t stream) {
  finalize_kernel<<<1, 32, 0, stream>>>(p);
  return cudaGetLastError();
}

size_t sq_error_workspace_bytes(int64_t I, int64_t J, int64_t K, int R) {
  const int64_t nb = I * ((J + kSqJ - 1) / kSqJ);  // the narrow tiling has the most blocks
  return static_cast<size_t>(nb) * 2 * sizeof(double) + static_cast<size_t>(K) * R * sizeof(double);
}

template <typename XT, int JT>
cudaError_t sq_error_dispatch(const void* X, int64_t I, int64_t J, int64_t K, const double* A,
                              const double* B, const double* CT, int R, double* part, int64_t nb,
                              cudaStream_t stream) {
  const size_t smem = static_cast<size_t>(JT) * (R > 0 ? R : 1) * sizeof(double);
  auto kern = sq_error_kernel<XT, JT>;
  if (smem > 48 * 1024) {  // 32 j values x ranks above 192
    cudaError_t e = allow_dyn_smem(reinterpret_cast<const void*>(kern), smem);
    if (e != cudaSuccess) return e;
  }
  kern<<<static_cast<unsigned>(nb), kSqThreads, smem, stream>>>(static_cast<const XT*>(X), I, J, K, A, B, CT,
                                                               R, part);
  return cudaGetLastError();
}

cudaError_t sq_error_launch(int x_dtype, const void* X, int64_t I, int64_t J, int64_t K,
                            const double* A, const double* B, const double* C, int R, double* out2,
                            void* ws, cudaStream_t stream) {
  const int jt = sq_jt(J, A != nullptr);
  const int64_t nb = I * ((J + jt - 1) / jt);
  double* part = static_cast<double*>(ws);
  double* CT = part + nb * 2;
  if (A) {
    transpose_kernel<<<static_cast<unsigned>(std::min<int64_t>((K * R + 255) / 256, 4096)), 256, 0,
                       stream>>>(C, K, R, CT);
  }
  cudaError_t e;
  if (jt == kSqJWide) {  // wide tensors with a model: the fp64 tensor pipe
    int pitch = (R + 3) & ~3;
    while (pitch % 16 != 4 && pitch % 16 != 12) ++pitch;  // conflict-free A fragments
    const size_t smem = static_cast<size_t>(kSqJWide) * pitch * sizeof(double);
    if (x_dtype == NTF_F32) {
      auto kern = sq_error_dmma_kernel<float>;
      e = smem > 48 * 1024 ? allow_dyn_smem(reinterpret_cast<const void*>(kern), smem) : cudaSuccess;
      if (e == cudaSuccess)
        kern<<<static_cast<unsigned>(nb), kSqThreads, smem, stream>>>(static_cast<const float*>(X), I, J, K, A,
                                                                     B, CT, R, pitch, part);
    } else {
      auto kern = sq_error_dmma_kernel<double>;
      e = smem > 48 * 1024 ? allow_dyn_smem(reinterpret_cast<const void*>(kern), smem) : cudaSuccess;
      if (e == cudaSuccess)
        kern<<<static_cast<unsigned>(nb), kSqThreads, smem, stream>>>(static_cast<const double*>(X), I, J, K, A,
                                                                     B, CT, R, pitch, part);
    }
    if (e == cudaSuccess) e = cudaGetLastError();
  } else if (x_dtype == NTF_F32) {
    e = sq_error_dispatch<float, kSqJ>(X, I, J, K, A, B, CT, R, part, nb, stream);
  } else {
    e = sq_error_dispatch<double, kSqJ>(X, I, J, K, A, B, CT, R, part, nb, stream);
  }
  if (e != cudaSuccess) return e;
  sum_pairs_kernel<<<1, 256, 0, stream>>>(part, nb, out2);
  return cudaGetLastError();
}

}  // namespace ntf
