// Per-mode ridge/ADMM update, Gram, iteration finalisation and residual-norm
// kernels for the B200 NTF hot path (sm_100a).  All reductions run in a fixed
// order (no float atomics), so a fit is bitwise run-to-run deterministic like
// the reference (blocks.py:130-140).
#include "solver_kernels.cuh"

namespace ntf {

namespace {

constexpr int kUpdThreads = 256;
// rows per update block: two rows per warp keeps the dependent substitution
// chains short and spreads a mode's rows over many SMs; the per-block Gram
// partials are reduced by the last block
__host__ __device__ __forceinline__ int rows_per_block(int R) { return R <= 64 ? 16 : 8; }

// ---------------------------------------------------------------------------
// Ridge Cholesky in shared memory (solver.ridge_cholesky, solver.py:167-175):
// H = G_a o G_b + rho*I (companion Gram, solver.py:196-204), lower factor
// L with L L^T = H.  Right-looking, one barrier per column: the trailing
// update uses the unscaled column (L[i][j] L[k][j] / pivot) and columns are
// scaled at the end.  A non-positive or non-finite pivot raises NOT_PD.
// ---------------------------------------------------------------------------
__device__ void build_and_factor(double* L, int ldl, int R, const double* __restrict__ Ga,
                                 const double* __restrict__ Gb, double rho, int* status,
                                 bool* bad) {
  const int tid = threadIdx.x;
  for (int e = tid; e < R * R; e += blockDim.x) {
    const int i = e / R, k = e - (e / R) * R;
    double h = Ga[e] * Gb[e];
    if (i == k) h += rho;
    L[i * ldl + k] = h;
  }
  __syncthreads();
  for (int j = 0; j < R; ++j) {
    const double piv = L[j * ldl + j];
    if (!(piv > 0.0) || !isfinite(piv)) {
      if (tid == 0) {
        raise_status(status, kDevNotPD);
        *bad = true;
      }
      __syncthreads();
      return;
    }
    const double inv = 1.0 / piv;
    const int n = R - j - 1;  // trailing order; update the lower triangle i >= k > j
    for (int e = tid; e < n * n; e += blockDim.x) {
      const int ii = e / n, kk = e - (e / n) * n;
      if (kk > ii) continue;
      const int i = j + 1 + ii, k = j + 1 + kk;
      L[i * ldl + k] -= L[i * ldl + j] * L[k * ldl + j] * inv;
    }
    __syncthreads();
  }
  // scale: L[i][j] = U[i][j] / sqrt(U[j][j]) for i > j, L[j][j] = sqrt(U[j][j])
  for (int e = tid; e < R * R; e += blockDim.x) {
    const int i = e / R, k = e - (e / R) * R;
    if (k < i) L[i * ldl + k] = L[i * ldl + k] / sqrt(L[k * ldl + k]);
  }
  __syncthreads();
  for (int j = tid; j < R; j += blockDim.x) L[j * ldl + j] = sqrt(L[j * ldl + j]);
  __syncthreads();
}

// Fixed-order sum of n strided values with 8 independent load/add chains
// (latency-bound reductions over L2-resident partials).  The combination
// order is fixed, so results are bitwise reproducible.
__device__ __forceinline__ double strided_sum(const double* __restrict__ p, int64_t n,
                                              int64_t stride) {
  double a[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  for (int64_t s = 0; s < n; s += 8) {
#pragma unroll
    for (int u = 0; u < 8; ++u)  // static indices: the chains stay in registers
      if (s + u < n) a[u] += p[(s + u) * stride];
  }
  return ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
}

// One block: H = G_a o G_b + rho I, Cholesky, then L (row-major R x R, lower)
// and 1/diag(L) to global for the row-update kernel.  Runs concurrently with
// the mode's MTTKRP (it only depends on the companion Grams and rho).
// Output layout of the ridge buffer:
//   [0, R*R)            L, row-major lower Cholesky factor of H
//   [R*R, R*R+R)        1 / diag(L)
//   [R*R+R, 2R*R+R)     H^-1 = L^-T L^-1  (R <= 64 only)
//   [2R*R+R, 3R*R+R)    H = G_a o G_b + rho I
__global__ void ridge_factor_kernel(RidgeParams p) {
  if (p.stop_flag && *p.stop_flag) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int R = p.R;
  const int ldl = R + 1;
  double* L = reinterpret_cast<double*>(smem_raw);
  double* Li = L + R * ldl;  // L^-1 (lower), R <= 64
  __shared__ bool bad;
  if (threadIdx.x == 0) bad = false;
  __syncthreads();
  const double rho = p.rho[p.mode - 1];
  double* Hout = p.L + 2 * R * R + R;
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    const int i = e / R, k = e - (e / R) * R;
    Hout[e] = p.Ga[e] * p.Gb[e] + (i == k ? rho : 0.0);
  }
  build_and_factor(L, ldl, R, p.Ga, p.Gb, rho, p.status, &bad);
  if (bad) return;
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    const int i = e / R, k = e - (e / R) * R;
    p.L[e] = k <= i ? L[i * ldl + k] : 0.0;
  }
  for (int j = threadIdx.x; j < R; j += blockDim.x) p.L[R * R + j] = 1.0 / L[j * ldl + j];
  if (R > 64) return;
  // L^-1 by forward substitution on the identity, one column per thread
  for (int j = threadIdx.x; j < R; j += blockDim.x) {
    for (int i = 0; i < R; ++i) {
      double s = i == j ? 1.0 : 0.0;
      if (i < j) {
        Li[i * ldl + j] = 0.0;
        continue;
      }
      for (int k = j; k < i; ++k) s -= L[i * ldl + k] * Li[k * ldl + j];
      Li[i * ldl + j] = s / L[i * ldl + i];
    }
  }
  __syncthreads();
  // H^-1 = L^-T L^-1: (a, b) = sum_{i >= max(a,b)} Li[i][a] Li[i][b]
  double* Hinv = p.L + R * R + R;
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    const int a = e / R, b = e - (e / R) * R;
    double s = 0.0;
    for (int i = a > b ? a : b; i < R; ++i) s += Li[i * ldl + a] * Li[i * ldl + b];
    Hinv[e] = s;
  }
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

template <int RT>
__global__ void __launch_bounds__(kUpdThreads, 1) factor_update_kernel(FactorUpdateParams p) {
  if (p.stop_flag && *p.stop_flag) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int R = p.R;
  const int ldl = R + 1;  // odd pitch: conflict-free row and column walks
  double* L = reinterpret_cast<double*>(smem_raw);
  double* inv_diag = L + R * ldl;               // [R]
  const int kRowsPerBlock = rows_per_block(R);
  double* xrows = inv_diag + R;                 // [rows][R] new factor rows
  double* msum = xrows + kRowsPerBlock * R;     // [rows][R] reduced MTTKRP rows
  // [8 warps][5][scale, ssq], after the GEMV path's H / rhs / x1 buffers when RT <= 2
  double* red = msum + kRowsPerBlock * R + (RT <= 2 ? R * R + 2 * kRowsPerBlock * R : 0);
  __shared__ bool is_last;
  // Ridge factor from the concurrent ridge_factor_kernel (solver.py:167-175)
  if (*p.status == kDevNotPD) return;
  if constexpr (RT <= 2) {
    // H^-1 into L's slot (pitch R) and H after the MTTKRP row sums
    double* Hm = msum + kRowsPerBlock * R;
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
      L[e] = p.Lg[R * R + R + e];
      Hm[e] = p.Lg[2 * R * R + R + e];
    }
  } else {
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
      const int i = e / R, k = e - (e / R) * R;
      L[i * ldl + k] = p.Lg[e];
    }
    for (int j = threadIdx.x; j < R; j += blockDim.x) inv_diag[j] = p.Lg[R * R + j];
  }

  const int64_t row_base = static_cast<int64_t>(blockIdx.x) * kRowsPerBlock;
  const int64_t n_rows = p.rows;
  const int64_t nM = n_rows * R;
  // Sum the MTTKRP split partials of this block's rows (fixed split order),
  // all threads cooperating; rows are contiguous so the block's slice of each
  // partial is one contiguous run.
  {
    const int64_t base = row_base * R;
    int64_t cnt = nM - base;
    if (cnt > static_cast<int64_t>(kRowsPerBlock) * R) cnt = static_cast<int64_t>(kRowsPerBlock) * R;
    for (int e = threadIdx.x; e < cnt; e += blockDim.x) {
      double m = 0.0;
      const int ns = (base + e) / R >= p.tail_row0 ? p.splits_tail : p.splits;
      if (!(p.debug & 1)) m = strided_sum(p.mtt + base + e, ns, nM);
      msum[e] = m;
    }
  }

  const double rho = p.rho[p.mode - 1];
  __syncthreads();

  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nwarps = kUpdThreads / 32;

  ScaledSq nrm[5];
  if constexpr (RT <= 2) {
    // R <= 64: all rows of the block at once as small GEMMs against the
    // ridge inverse, with one step of iterative refinement against H itself:
    //   x1 = y H^-1,  x = x1 + (y - x1 H) H^-1
    // Every (row, column) pair is independent: no sequential substitution
    // chain on the critical path.  Agreement with cho_solve (solver.py:188)
    // is at the backward-error level.
    double* Hi = L;                          // reuse: [R][R] H^-1
    double* Hm = msum + kRowsPerBlock * R;   // [R][R] H   (after msum)
    double* yb = Hm + R * R;                 // [rows][R]  rhs, then residual
    double* x1 = yb + kRowsPerBlock * R;     // [rows][R]
    const int np = kRowsPerBlock * R;
    for (int e = threadIdx.x; e < np; e += blockDim.x) {
      const int lr = e / R, c = e - (e / R) * R;
      const int64_t row = row_base + lr;
      double y = 0.0;
      if (row < n_rows) {
        const int64_t g = row * R + c;
        y = (msum[e] + rho * p.aux[g]) - p.dual[g];  // ridge_rhs (solver.py:178-179)
      }
      yb[e] = y;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < np; e += blockDim.x) {
      const int lr = e / R, c = e - (e / R) * R;
      double s = 0.0;
      for (int k = 0; k < R; ++k) s = fma(yb[lr * R + k], Hi[k * R + c], s);
      x1[e] = s;
    }
    __syncthreads();
    double res[4];  // np / blockDim <= 4 (rows 16 x R <= 64 over 256 threads)
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = threadIdx.x + u * kUpdThreads;
      res[u] = 0.0;
      if (e < np) {
        const int lr = e / R, c = e - (e / R) * R;
        double s = yb[e];
        for (int k = 0; k < R; ++k) s = fma(-x1[lr * R + k], Hm[k * R + c], s);
        res[u] = s;
      }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = threadIdx.x + u * kUpdThreads;
      if (e < np) yb[e] = res[u];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < np; e += blockDim.x) {
      const int lr = e / R, c = e - (e / R) * R;
      const int64_t row = row_base + lr;
      double x = x1[e];
      for (int k = 0; k < R; ++k) x = fma(yb[lr * R + k], Hi[k * R + c], x);
      if (row >= n_rows) {
        xrows[e] = 0.0;
        continue;
      }
      const int64_t g = row * R + c;
      p.F[(p.row_offset + row) * R + c] = x;
      xrows[e] = x;
      if (p.last_sweep) {
        // aux = project(F + Y/rho), Y += rho (F - aux), residual partials
        const double yd = p.dual[g];
        const double a_old = p.aux[g];
        const double v = x + yd / rho;
        if (!isfinite(v)) raise_status(p.status, kDevNonFinite);
        const double a = v > 0.0 ? v : 0.0;
        const double ynew = yd + rho * (x - a);
        p.aux[g] = a;
        p.dual[g] = ynew;
        const double d0 = x - a, d1 = a - a_old;
        nrm[0].add(d0);
        nrm[1].add(d1);
        nrm[2].add(x);
        nrm[3].add(a);
        nrm[4].add(ynew);
      }
    }
  }
  for (int lr = warp; RT > 2 && lr < kRowsPerBlock; lr += nwarps) {
    const int64_t row = row_base + lr;
    double y[RT];
    if (row < n_rows) {
#pragma unroll
      for (int t = 0; t < RT; ++t) {
        const int r = lane + 32 * t;
        y[t] = 0.0;
        if (r < R) {
          const int64_t e = row * R + r;
          // ridge_rhs: mtt + rho*aux - dual (solver.py:178-179)
          y[t] = (msum[lr * R + r] + rho * p.aux[e]) - p.dual[e];
        }
      }
      if (!(p.debug & 2)) warp_chol_solve<RT>(y, L, ldl, R, inv_diag, lane);
#pragma unroll
      for (int t = 0; t < RT; ++t) {
        const int r = lane + 32 * t;
        if (r < R) {
          const int64_t e = row * R + r;
          const double x = y[t];
          p.F[(p.row_offset + row) * R + r] = x;
          xrows[lr * R + r] = x;
          if (p.last_sweep) {
            // aux = project(F + Y/rho) (solver.py:311-314, constraints.py:105-111),
            // Y += rho (F - aux) (solver.py:315-317), residual partials (247-255)
            const double yd = p.dual[e];
            const double a_old = p.aux[e];
            const double v = x + yd / rho;
            if (!isfinite(v)) raise_status(p.status, kDevNonFinite);
            const double a = v > 0.0 ? v : 0.0;
            const double ynew = yd + rho * (x - a);
            p.aux[e] = a;
            p.dual[e] = ynew;
            const double d0 = x - a, d1 = a - a_old;
            nrm[0].add(d0);
            nrm[1].add(d1);
            nrm[2].add(x);
            nrm[3].add(a);
            nrm[4].add(ynew);
          }
        }
      }
    } else {
#pragma unroll
      for (int t = 0; t < RT; ++t) {
        const int r = lane + 32 * t;
        if (r < R) xrows[lr * R + r] = 0.0;
      }
    }
  }

  const int nblocks = gridDim.x;
  if (p.last_sweep) {
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
  }
  __syncthreads();
  if (p.last_sweep && threadIdx.x < 5) {
    ScaledSq s;
    for (int w = 0; w < nwarps; ++w)
      s.merge(red[(w * 5 + threadIdx.x) * 2], red[(w * 5 + threadIdx.x) * 2 + 1]);
    p.norm_partials[(blockIdx.x * 5 + threadIdx.x) * 2] = s.scale;
    p.norm_partials[(blockIdx.x * 5 + threadIdx.x) * 2 + 1] = s.ssq;
  }
  if (p.fuse_gram) {
    // partial Gram of this block's new rows, fixed row order
    double* gp = p.gram_partials + static_cast<int64_t>(blockIdx.x) * R * R;
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
      const int r = e / R, s = e - (e / R) * R;
      double acc = 0.0;
      for (int lr = 0; lr < kRowsPerBlock; ++lr) acc += xrows[lr * R + r] * xrows[lr * R + s];
      gp[e] = acc;
    }
    // per-column max |F| of this block's rows (W scales of the next MTTKRPs)
    for (int r = threadIdx.x; r < R; r += blockDim.x) {
      double mx = 0.0;
      for (int lr = 0; lr < kRowsPerBlock; ++lr) mx = fmax(mx, fabs(xrows[lr * R + r]));
      p.colmax_partials[blockIdx.x * R + r] = mx;
    }
  }
  if (!p.fuse_gram && !p.last_sweep) return;

  // last block to finish reduces the per-block partials in block order
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned prev = atomicAdd(p.done_counter, 1u);
    is_last = (prev == static_cast<unsigned>(nblocks - 1));
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  if (p.fuse_gram && !(p.debug & 4)) {
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
      double s = 0.0;
      s = strided_sum(p.gram_partials + e, nblocks, static_cast<int64_t>(R) * R);
      p.G_out[e] = s;
    }
    for (int r = threadIdx.x; r < R; r += blockDim.x) {
      double mx = 0.0;  // max is order-independent: exact and deterministic
      for (int b = 0; b < nblocks; ++b) mx = fmax(mx, p.colmax_partials[b * R + r]);
      p.colmax_out[r] = mx;
    }
  }
  if (p.last_sweep) {
    // 8 interleaved merge chains per norm (fixed order), then chain 0..7 merged
    __syncthreads();
    if (threadIdx.x < 40) {
      const int c = threadIdx.x >> 3, ch = threadIdx.x & 7;
      ScaledSq s;
      for (int b = ch; b < nblocks; b += 8)
        s.merge(p.norm_partials[(b * 5 + c) * 2], p.norm_partials[(b * 5 + c) * 2 + 1]);
      red[threadIdx.x * 2] = s.scale;
      red[threadIdx.x * 2 + 1] = s.ssq;
    }
    __syncthreads();
    if (threadIdx.x < 5) {
      ScaledSq s;
      for (int ch = 0; ch < 8; ++ch)
        s.merge(red[(threadIdx.x * 8 + ch) * 2], red[(threadIdx.x * 8 + ch) * 2 + 1]);
      p.norm_acc[threadIdx.x * 2] = s.scale;
      p.norm_acc[threadIdx.x * 2 + 1] = s.ssq;
    }
  }
  if (threadIdx.x == 0) *p.done_counter = 0u;
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
  if (threadIdx.x != 0) return;
  int* ctr = p.counters;
  if (ctr[1]) return;  // already stopped: iteration is a no-op
  const int64_t it = ctr[0];
  double primal[3], dual[3];
  bool stop = true;
  for (int m = 0; m < 3; ++m) {
    // merge the shards' (scale, ssq) pairs in rank order
    ScaledSq a[5];
    for (int q = 0; q < p.norm_parts; ++q)
      for (int c = 0; c < 5; ++c) {
        const double* s = p.norm_acc + ((q * 3 + m) * 5 + c) * 2;
        a[c].merge(s[0], s[1]);
      }
    primal[m] = a[0].norm();
    dual[m] = p.rho[m] * a[1].norm();
    const double base = sqrt(static_cast<double>(p.dims[m]) * p.R) * p.eps_abs;
    const double fn = a[2].norm(), an = a[3].norm(), yn = a[4].norm();
    const double pthr = base + p.eps_rel * (fn > an ? fn : an);
    const double dthr = base + p.eps_rel * yn;
    if (primal[m] > pthr || dual[m] > dthr) stop = false;
  }
  double rho_new[3];
  for (int m = 0; m < 3; ++m) {
    const double r = p.rho[m];
    if (p.rho_schedule && it < p.history_capacity) {
      rho_new[m] = p.rho_schedule[it * 3 + m];
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
    for (int m = 0; m < 3; ++m) {
      p.resid_history[it * 6 + m] = primal[m];
      p.resid_history[it * 6 + 3 + m] = dual[m];
      p.rho_history[it * 3 + m] = rho_new[m];
    }
  }
  for (int m = 0; m < 3; ++m) p.rho[m] = rho_new[m];
  ctr[0] = static_cast<int>(it + 1);
  if (stop) ctr[1] = 1;
}

// ---------------------------------------------------------------------------
// sum x^2 and sum (x - [[A,B,C]])^2 with fp64 accumulation (tensors.py:57-61,
// 276-290).  Block = one i and kSqJ consecutive j; threads along k.
// ---------------------------------------------------------------------------
constexpr int kSqJ = 8;
constexpr int kSqThreads = 256;

template <typename XT>
__global__ void __launch_bounds__(kSqThreads) sq_error_kernel(const XT* __restrict__ X, int64_t I,
                                                              int64_t J, int64_t K,
                                                              const double* __restrict__ A,
                                                              const double* __restrict__ B,
                                                              const double* __restrict__ CT,
                                                              int R, double* __restrict__ part) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* ab = reinterpret_cast<double*>(smem_raw);  // [kSqJ][R]
  const int64_t nj_blocks = (J + kSqJ - 1) / kSqJ;
  const int64_t i = blockIdx.x / nj_blocks;
  const int64_t j0 = (blockIdx.x - i * nj_blocks) * kSqJ;
  const bool model = A != nullptr;
  if (model) {
    for (int e = threadIdx.x; e < kSqJ * R; e += blockDim.x) {
      const int jj = e / R, r = e - (e / R) * R;
      const int64_t j = j0 + jj;
      ab[e] = j < J ? A[i * R + r] * B[j * R + r] : 0.0;
    }
  }
  __syncthreads();
  double sx = 0.0, se = 0.0;
  for (int64_t k = threadIdx.x; k < K; k += blockDim.x) {
    double rec[kSqJ];
#pragma unroll
    for (int jj = 0; jj < kSqJ; ++jj) rec[jj] = 0.0;
    if (model) {
      for (int r = 0; r < R; ++r) {
        const double c = CT[static_cast<int64_t>(r) * K + k];
#pragma unroll
        for (int jj = 0; jj < kSqJ; ++jj) rec[jj] = fma(ab[jj * R + r], c, rec[jj]);
      }
    }
#pragma unroll
    for (int jj = 0; jj < kSqJ; ++jj) {
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

int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

}  // namespace

// ---------------------------------------------------------------------------
// host-side launchers
// ---------------------------------------------------------------------------
int factor_update_blocks(int64_t rows, int R) {
  const int rpb = rows_per_block(R);
  return static_cast<int>((rows + rpb - 1) / rpb);
}

size_t factor_update_smem(int R) {
  const size_t rpb = rows_per_block(R);
  size_t n = static_cast<size_t>(R) * (R + 1) + R + 2 * rpb * R + 8 * 10;
  if (R <= 64) n += static_cast<size_t>(R) * R + 2 * rpb * R;  // GEMV path buffers
  return n * sizeof(double);
}

size_t ridge_factor_smem(int R) {
  return static_cast<size_t>(R <= 64 ? 2 : 1) * R * (R + 1) * sizeof(double);
}

size_t ridge_buffer_doubles(int R) { return 3 * static_cast<size_t>(R) * R + R; }

cudaError_t ridge_factor_launch(const RidgeParams& p, cudaStream_t stream) {
  ridge_factor_kernel<<<1, 256, ridge_factor_smem(p.R), stream>>>(p);
  return cudaGetLastError();
}

cudaError_t factor_update_prepare(int R) {
  const int smem = static_cast<int>(factor_update_smem(R));
  cudaError_t e = cudaFuncSetAttribute(ridge_factor_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(ridge_factor_smem(R)));
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(factor_update_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(factor_update_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(factor_update_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(factor_update_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              smem);
}

cudaError_t factor_update_launch(const FactorUpdateParams& p_in, cudaStream_t stream) {
  static int dbg = -1;
  if (dbg < 0) {
    const char* env = getenv("NTF_UPD_DEBUG");
    dbg = env ? atoi(env) : 0;
  }
  FactorUpdateParams p = p_in;
  p.debug = dbg;
  const int blocks = factor_update_blocks(p.rows, p.R);
  const size_t smem = factor_update_smem(p.R);
  const int rt = (p.R + 31) / 32;
  switch (rt) {
    case 1: factor_update_kernel<1><<<blocks, kUpdThreads, smem, stream>>>(p); break;
    case 2: factor_update_kernel<2><<<blocks, kUpdThreads, smem, stream>>>(p); break;
    case 3: factor_update_kernel<3><<<blocks, kUpdThreads, smem, stream>>>(p); break;
    default: factor_update_kernel<4><<<blocks, kUpdThreads, smem, stream>>>(p); break;
  }
  return cudaGetLastError();
}

size_t gram_workspace_bytes(int64_t rows, int R) {
  const int64_t nb = (rows + kGramRows - 1) / kGramRows;
  return static_cast<size_t>(nb) * R * R * sizeof(double);
}

cudaError_t gram_launch(const double* F, int64_t rows, int R, double* G, double* ws,
                        cudaStream_t stream) {
  const int64_t nb = (rows + kGramRows - 1) / kGramRows;
  const size_t smem = static_cast<size_t>(kGramRows) * R * sizeof(double);
  cudaError_t e = cudaFuncSetAttribute(gram_partial_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
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
  const int64_t nb = I * ((J + kSqJ - 1) / kSqJ);
  return static_cast<size_t>(nb) * 2 * sizeof(double) + static_cast<size_t>(K) * R * sizeof(double);
}

cudaError_t sq_error_launch(int x_dtype, const void* X, int64_t I, int64_t J, int64_t K,
                            const double* A, const double* B, const double* C, int R, double* out2,
                            void* ws, cudaStream_t stream) {
  const int64_t nb = I * ((J + kSqJ - 1) / kSqJ);
  double* part = static_cast<double*>(ws);
  double* CT = part + nb * 2;
  if (A) {
    transpose_kernel<<<static_cast<unsigned>(std::min<int64_t>((K * R + 255) / 256, 4096)), 256, 0,
                       stream>>>(C, K, R, CT);
  }
  const size_t smem = static_cast<size_t>(kSqJ) * (R > 0 ? R : 1) * sizeof(double);
  if (x_dtype == NTF_F32) {
    sq_error_kernel<float><<<static_cast<unsigned>(nb), kSqThreads, smem, stream>>>(
        static_cast<const float*>(X), I, J, K, A, B, CT, R, part);
  } else {
    sq_error_kernel<double><<<static_cast<unsigned>(nb), kSqThreads, smem, stream>>>(
        static_cast<const double*>(X), I, J, K, A, B, CT, R, part);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  sum_pairs_kernel<<<1, 256, 0, stream>>>(part, nb, out2);
  return cudaGetLastError();
}

}  // namespace ntf
