// Small kernels of the H/S path (sm_100a): T-block preparation with the batched
// Cholesky (kernels.py:119-132, builder.py:284-288), the Hermitian mirror
// (matrix.py:216-226), row scaling (matrix.py:229-239) and operand preparation for the
// per-op KernelBackend entry points (kernels.py:77-116).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <cooperative_groups.h>

#include "common.cuh"

namespace hsdla {
namespace {

__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }

// Phase timers for tools/exp/tjoint_bench.cu (no-ops in the library build).
#ifndef HSDLA_PROF_POINT
#define HSDLA_PROF_POINT(i)
#define HSDLA_PROF_START()
#endif

// Column-major sweep of an n x n index space by the whole CTA: warp w takes columns w, w + nw,
// ..., its lanes go down the rows (coalesced), no integer division in the loop.
#define FOR_SQUARE(n, r, c)                                       \
  for (int c = threadIdx.x >> 5; c < (n); c += blockDim.x >> 5) \
    for (int r = threadIdx.x & 31; r < (n); r += 32)

// ---------------------------------------------------------------------------
// Cholesky of tril(T) into F (lower, zero strict upper), one CTA per matrix.
// Left-looking column algorithm, the same recurrence as the reference's portable
// backend (kernels.py:217-228): d_j = Re T_jj - sum_k |L_jk|^2, pivot fails unless
// d_j > 0 and finite; L_ij = (T_ij - sum_k L_ik conj(L_jk)) / sqrt(d_j).
// info: 0 ok, j+1 first bad pivot, -1 NaN in tril(T).
__device__ void chol_block(int n, const double2* __restrict__ T, long long ldt, double2* F,
                           long long ldf, int* info) {
  extern __shared__ double2 rowj[];  // n entries
  __shared__ double red[32];
  __shared__ int s_nan;
  __shared__ double s_d;
  const int tid = threadIdx.x, nt = blockDim.x;
  if (tid == 0) s_nan = 0;
  __syncthreads();
  FOR_SQUARE(n, r, c) {
    double2 v = make_double2(0.0, 0.0);
    if (r >= c) {
      v = T[r + c * ldt];
      if (isnan(v.x) || isnan(v.y)) s_nan = 1;
    }
    F[r + c * ldf] = v;
  }
  __syncthreads();
  if (s_nan) {
    if (tid == 0) *info = -1;
    return;
  }
  for (int j = 0; j < n; ++j) {
    double part = 0.0;
    for (int k = tid; k < j; k += nt) {
      const double2 v = F[j + (long long)k * ldf];
      rowj[k] = v;
      part += v.x * v.x + v.y * v.y;
    }
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if ((tid & 31) == 0) red[tid >> 5] = part;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int w = 0; w < (nt + 31) / 32; ++w) s += red[w];
      s_d = F[j + (long long)j * ldf].x - s;
    }
    __syncthreads();
    const double d = s_d;
    if (!(d > 0.0) || !isfinite(d)) {
      if (tid == 0) *info = j + 1;
      return;
    }
    const double ljj = sqrt(d);
    for (int i = j + 1 + tid; i < n; i += nt) {
      double2 acc = F[i + (long long)j * ldf];
      for (int k = 0; k < j; ++k) {
        const double2 a = F[i + (long long)k * ldf];
        const double2 b = rowj[k];
        // a * conj(b)
        acc.x -= a.x * b.x + a.y * b.y;
        acc.y -= a.y * b.x - a.x * b.y;
      }
      F[i + (long long)j * ldf] = make_double2(acc.x / ljj, acc.y / ljj);
    }
    if (tid == 0) F[j + (long long)j * ldf] = make_double2(ljj, 0.0);
    __syncthreads();
  }
  if (tid == 0) *info = 0;
}

// Blocked right-looking Cholesky of the lower triangle of A in place (ld lda), one CTA: a
// panel of kNB columns is staged in shared memory (rows x kNB, row stride kNB + 1 against bank
// conflicts) and factored there column by column (one barrier per column, a few updates per
// thread), written back scaled, and the trailing lower triangle takes the rank-kNB update
// A22 -= L21 L21^H in 4 x 4 register micro-tiles straight in global memory (L2-resident).
// Same pivot rule and info as chol_block (0 ok, j+1 first bad pivot, -1 NaN in tril(A));
// writes zeros to the strict upper triangle.  Dynamic shared memory: chol_blocked_smem(n).
constexpr int kNB = 16;
constexpr int kNBS = kNB + 1;
__host__ __device__ constexpr size_t chol_blocked_smem(int n) {
  return size_t(n > 0 ? n : 1) * kNBS * sizeof(double2);
}

// Staging of the current panel (rows k..n, columns k..k+nb) into P, lower part only.
__device__ __forceinline__ void chol_stage_panel(int k, int nb, int rows, const double2* A,
                                                 long long lda, double2* P) {
  const double2 zero = make_double2(0.0, 0.0);
  for (int e = threadIdx.x; e < rows * nb; e += blockDim.x) {
    const int r = e % rows, c = e / rows;
    P[r * kNBS + c] = r >= c ? A[(k + r) + (long long)(k + c) * lda] : zero;
  }
}

// Factor the staged panel in place in P (final, scaled L values) and write it back to A
// (zeros above the diagonal block's diagonal).  Returns 0, or the 1-based matrix index of the
// first pivot that is not positive and finite (uniform across the block).
__device__ int chol_factor_panel(int k, int nb, int rows, double2* A, long long lda, double2* P) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const double2 zero = make_double2(0.0, 0.0);
    // Panel factorization in steps of kSB columns: thread 0 factors the kSB x kSB diagonal
    // block in registers and publishes it, then (a) each row below it is solved against that
    // factor (L_r = P_r L_D^-H, final values in place) and (b) the panel's remaining columns
    // take the rank-kSB update; three barriers per step.
    constexpr int kSB = 4;  // 8 measured 2x slower (spills in the row solve)
    __shared__ double2 sL[kSB][kSB];
    __shared__ double sld[kSB], sli[kSB];
    __shared__ int sbad;
    for (int j0 = 0; j0 < nb; j0 += kSB) {
      const int sb = min(kSB, nb - j0);
      // registers only: fully unrolled loops over the kSB x kSB block, predicated on sb.  One
      // thread factors it (the other warps would only compete for the FP64 pipe with the same
      // dependent sqrt / reciprocal chain) and publishes it through shared memory.
      double2 L[kSB][kSB];
      double ld[kSB], li[kSB];
      int bad = 0;
      if (tid == 0) {
#pragma unroll
        for (int i = 0; i < kSB; ++i)
#pragma unroll
          for (int q = 0; q < kSB; ++q)
            L[i][q] = (q <= i && i < sb) ? P[(j0 + i) * kNBS + j0 + q] : zero;
#pragma unroll
        for (int i = 0; i < kSB; ++i) {
          double d = L[i][i].x;
#pragma unroll
          for (int q = 0; q < i; ++q) d -= L[i][q].x * L[i][q].x + L[i][q].y * L[i][q].y;
          const bool ok = i >= sb || (d > 0.0 && isfinite(d));
          if (!ok && !bad) bad = i + 1;
          ld[i] = ok && i < sb ? sqrt(d) : 1.0;
          li[i] = 1.0 / ld[i];
#pragma unroll
          for (int i2 = i + 1; i2 < kSB; ++i2) {
            double2 v = L[i2][i];
#pragma unroll
            for (int q = 0; q < i; ++q) {  // v -= L[i2][q] conj(L[i][q])
              v.x = fma(-L[i2][q].x, L[i][q].x, v.x);
              v.x = fma(-L[i2][q].y, L[i][q].y, v.x);
              v.y = fma(-L[i2][q].y, L[i][q].x, v.y);
              v.y = fma(L[i2][q].x, L[i][q].y, v.y);
            }
            L[i2][i] = make_double2(v.x * li[i], v.y * li[i]);
          }
        }
#pragma unroll
        for (int i = 0; i < kSB; ++i) {
          sld[i] = ld[i];
          sli[i] = li[i];
#pragma unroll
          for (int q = 0; q < kSB; ++q) sL[i][q] = L[i][q];
        }
        sbad = bad;
      }
      __syncthreads();  // the factor is published and thread 0 has read the block before rows are rewritten
      HSDLA_PROF_POINT(9);
      bad = sbad;
      if (bad) return k + j0 + bad;  // uniform
#pragma unroll
      for (int i = 0; i < kSB; ++i) {
        ld[i] = sld[i];
        li[i] = sli[i];
#pragma unroll
        for (int q = 0; q < kSB; ++q) L[i][q] = sL[i][q];
      }
      // (a) rows of the diagonal block take L_D; rows below solve x L_D^H = P_r
      for (int r = j0 + tid; r < rows; r += nt) {
        double2 x[kSB];
        if (r < j0 + sb) {  // a row of the diagonal block: its factor row
          const int rr = r - j0;
#pragma unroll
          for (int i = 0; i < kSB; ++i) {
            double2 v = zero;
#pragma unroll
            for (int q = 0; q < kSB; ++q)
              if (q == rr) v = i < q ? L[q][i] : (i == q ? make_double2(ld[i], 0.0) : zero);
            x[i] = v;
          }
        } else {
#pragma unroll
          for (int i = 0; i < kSB; ++i) {
            double2 v = i < sb ? P[r * kNBS + j0 + i] : zero;
#pragma unroll
            for (int q = 0; q < i; ++q) {  // v -= x_q conj(L_D[i][q])
              v.x = fma(-x[q].x, L[i][q].x, v.x);
              v.x = fma(-x[q].y, L[i][q].y, v.x);
              v.y = fma(-x[q].y, L[i][q].x, v.y);
              v.y = fma(x[q].x, L[i][q].y, v.y);
            }
            x[i] = make_double2(v.x * li[i], v.y * li[i]);
          }
        }
#pragma unroll
        for (int i = 0; i < kSB; ++i)
          if (i < sb) P[r * kNBS + j0 + i] = x[i];
      }
      __syncthreads();
      HSDLA_PROF_POINT(10);
      // (b) P[r][c] -= sum_q L[r][j0+q] conj(L[c][j0+q]) for the panel's columns c >= j0 + sb
      const int tx = tid % kNB, ty = tid / kNB, c = j0 + sb + tx;
      if (c < nb) {
        double2 lc[kSB];
#pragma unroll
        for (int q = 0; q < kSB; ++q) lc[q] = q < sb ? P[c * kNBS + j0 + q] : zero;
        const int S = nt / kNB;
        int r = j0 + sb + ty;
        if (r < c) r += (c - r + S - 1) / S * S;
        for (; r < rows; r += S) {
          double2 v = P[r * kNBS + c];
#pragma unroll
          for (int q = 0; q < kSB; ++q) {
            const double2 a = q < sb ? P[r * kNBS + j0 + q] : zero;
            v.x = fma(-a.x, lc[q].x, v.x);
            v.x = fma(-a.y, lc[q].y, v.x);
            v.y = fma(-a.y, lc[q].x, v.y);
            v.y = fma(a.x, lc[q].y, v.y);
          }
          P[r * kNBS + c] = v;
        }
      }
      __syncthreads();
      HSDLA_PROF_POINT(11);
    }
    for (int e = tid; e < rows * nb; e += nt) {
      const int r = e % rows, c = e / rows;
      A[(k + r) + (long long)(k + c) * lda] = r >= c ? P[r * kNBS + c] : zero;
    }
    __syncthreads();
    return 0;
}

// Trailing update A22 -= L21 L21^H after the panel at k (L21 = P rows nb..rows), warp tasks
// task0, task0 + task_step, ... of the 32 x 16 task grid.
__device__ void chol_trailing(int k, int nb, int rows, int n, double2* A, long long lda,
                              const double2* P, int task0, int task_step) {
  const double2 zero = make_double2(0.0, 0.0);
  const int tid = threadIdx.x;
    // trailing lower triangle, rows / columns [k + nb, n): warp tasks of 32 rows x 16 columns,
    // lane l on row i0 + l (consecutive panel rows: conflict-free shared loads), the 16
    // column rows j0..j0+15 broadcast; only tasks touching i >= j run (the diagonal-crossing
    // ones mask their upper part).
    {
      constexpr int TR = 32, TC = 16;
      const int tr = rows - nb;
      const int nrb = (tr + TR - 1) / TR, ncb = (tr + TC - 1) / TC;
      const int lane = tid & 31;
      for (int task = task0; task < nrb * ncb; task += task_step) {
        const int rb = task % nrb, cb = task / nrb;
        const int i0 = TR * rb, j0 = TC * cb;  // trailing-relative
        if (i0 + TR - 1 < j0) continue;       // strictly upper: nothing to do
        double2 acc[TC];
#pragma unroll
        for (int q = 0; q < TC; ++q) acc[q] = zero;
        const int ia = nb + i0 + lane;
        for (int c = 0; c < nb; ++c) {
          const double2 la = ia < rows ? P[ia * kNBS + c] : zero;
#pragma unroll
          for (int q = 0; q < TC; ++q) {
            const int rj = nb + j0 + q;
            const double2 lj = rj < rows ? P[rj * kNBS + c] : zero;
            acc[q].x = fma(la.x, lj.x, acc[q].x);
            acc[q].x = fma(la.y, lj.y, acc[q].x);
            acc[q].y = fma(la.y, lj.x, acc[q].y);
            acc[q].y = fma(-la.x, lj.y, acc[q].y);
          }
        }
        const int i = k + nb + i0 + lane;
#pragma unroll
        for (int q = 0; q < TC; ++q) {
          const int jj = k + nb + j0 + q;
          if (i < n && jj < n && jj <= i) {
            double2* x = A + i + (long long)jj * lda;
            const double2 v = *x;
            *x = make_double2(v.x - acc[q].x, v.y - acc[q].y);
          }
        }
      }
    }
}

// `checked`: the caller already rejected NaN input and zeroed the strict upper triangle.
__device__ void chol_blocked(int n, double2* A, long long lda, int* info, bool checked = false) {
  extern __shared__ double2 P[];  // [rows][kNBS]
  __shared__ int s_bad;
  const int tid = threadIdx.x;
  const double2 zero = make_double2(0.0, 0.0);
  if (!checked) {
    if (tid == 0) s_bad = 0;
    __syncthreads();
    FOR_SQUARE(n, r, c) {
      if (r >= c) {
        const double2 v = A[r + c * lda];
        if (isnan(v.x) || isnan(v.y)) s_bad = 1;
      }
    }
    __syncthreads();
    if (s_bad) {
      if (tid == 0) *info = -1;
      return;
    }
  }
  HSDLA_PROF_POINT(1);
  for (int k = 0; k < n; k += kNB) {
    const int nb = min(kNB, n - k), rows = n - k;
    chol_stage_panel(k, nb, rows, A, lda, P);
    __syncthreads();
    HSDLA_PROF_POINT(2);
    const int bad = chol_factor_panel(k, nb, rows, A, lda, P);
    if (bad) {
      if (tid == 0) *info = bad;
      return;
    }
    HSDLA_PROF_POINT(4);
    chol_trailing(k, nb, rows, n, A, lda, P, tid >> 5, blockDim.x >> 5);
    __syncthreads();
    HSDLA_PROF_POINT(5);
  }
  if (!checked) {
    FOR_SQUARE(n, r, c) {
      if (r < c) A[r + c * lda] = zero;
    }
  }
  if (tid == 0) *info = 0;
}

// Cluster version (one thread-block cluster of kCS CTAs per matrix): rank 0 stages and factors
// each panel; after a cluster barrier every rank copies the factored panel from global memory
// (L2) into its own shared memory and takes a 1/kCS share of the trailing update's warp tasks;
// a second barrier closes the step.  The input must be checked (no NaN, zero strict upper).
// `info` is written by rank 0; every rank returns together.
constexpr int kCS = 8;
// The cluster versions pay off from about this order on (the panel factorisation on rank 0
// stays the critical path; measured: 2m = 242 401 vs 546 us, 2m = 162 245 vs 242 us).
#ifndef HSDLA_CLUSTER_MIN_N
#define HSDLA_CLUSTER_MIN_N 192
#endif
constexpr int kClusterMinN = HSDLA_CLUSTER_MIN_N;
// HSDLA_TPREP_CLUSTER=0: one CTA per T set for the T preparation kernels.
inline bool tprep_cluster() {
  static int m = -1;
  if (m < 0) {
    const char* e = getenv("HSDLA_TPREP_CLUSTER");
    m = (e && e[0] == '0') ? 0 : 1;
  }
  return m == 1;
}

__device__ void chol_blocked_cluster(int n, double2* A, long long lda, int* info) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ double2 P[];
  __shared__ int s_bad;
  const int tid = threadIdx.x;
  const int rank = (int)cl.block_rank(), ncl = (int)cl.num_blocks();
  const int* bad0 = cl.map_shared_rank(&s_bad, 0);
  for (int k = 0; k < n; k += kNB) {
    const int nb = min(kNB, n - k), rows = n - k;
    if (rank == 0) {
      chol_stage_panel(k, nb, rows, A, lda, P);
      __syncthreads();
      const int bad = chol_factor_panel(k, nb, rows, A, lda, P);
      if (tid == 0) s_bad = bad;
      __threadfence();
    }
    cl.sync();
    const int bad = *bad0;
    if (bad) {
      if (rank == 0 && tid == 0) *info = bad;
      return;
    }
    if (rank != 0) {
      chol_stage_panel(k, nb, rows, A, lda, P);
      __syncthreads();
    }
    const int nw = blockDim.x >> 5;
    chol_trailing(k, nb, rows, n, A, lda, P, rank * nw + (tid >> 5), nw * ncl);
    __threadfence();
    cl.sync();
  }
  if (rank == 0 && tid == 0) *info = 0;
}

// Cholesky of tril(T) into F: blocked in place on a copy when its panel fits in shared memory
// (n <= kBlockedMaxN), else the column algorithm (chol_block).
constexpr int kBlockedMaxN = 768;

__global__ void __launch_bounds__(512) potrf_batched_kernel(int n, const double2* T, long long ldt, long long st,
                                     double2* F, long long ldf, long long sf, int* info) {
  const int b = blockIdx.x;
  if (n <= kBlockedMaxN) {
    const double2* Tb = T + b * st;
    double2* Fb = F + b * sf;
    FOR_SQUARE(n, r, c) {
      Fb[r + c * ldf] = r >= c ? Tb[r + c * ldt] : make_double2(0.0, 0.0);
    }
    __syncthreads();
    chol_blocked(n, Fb, ldf, info + b);
  } else {
    chol_block(n, T + b * st, ldt, F + b * sf, ldf, info + b);
  }
}

constexpr int kPotrfMaxDynSmem = 227 * 1024;  // opt-in limit per CTA (static smem comes off it)

// Per T set: forms[0] = T_AB, forms[1] = 1/2 full(T_BB), forms[2] = full(T_AA),
// forms[3] = Cholesky factor of tril(T_AA) (if do_chol), all m x m with ld mp.
// CL: one cluster of kCS CTAs per T set (launched with the cluster dimension), the copies
// split across the ranks and the factor by chol_blocked_cluster; else one CTA per set.
template <bool CL>
__global__ void __launch_bounds__(512) tprep_kernel(const int* tdim, int mp, const double2* taa, const double2* tab,
                             const double2* tbb, long long t_ld, double2* forms, int do_chol,
                             int* info) {
  namespace cg = cooperative_groups;
  const int b = CL ? blockIdx.x / kCS : blockIdx.x;
  const int rank = CL ? (int)cg::this_cluster().block_rank() : 0;
  const int nrk = CL ? kCS : 1;
  const int c0 = rank * (blockDim.x >> 5) + (threadIdx.x >> 5), cs = nrk * (blockDim.x >> 5);
  const int m = tdim[b];
  const long long tstride = t_ld * t_ld;
  const double2* Taa = taa + b * tstride;
  const double2* Tab = tab + b * tstride;
  const double2* Tbb = tbb + b * tstride;
  double2* f = forms + (long long)b * 4 * mp * mp;
  const long long fs = (long long)mp * mp;
  // columns split over the cluster's warps (rows by lanes)
  for (int c = c0; c < m; c += cs)
  for (int r = threadIdx.x & 31; r < m; r += 32) {
    f[r + (long long)c * mp] = Tab[r + c * t_ld];
    double2 bb, aa;
    if (r > c) { bb = Tbb[r + c * t_ld]; aa = Taa[r + c * t_ld]; }
    else if (r < c) { bb = cconj(Tbb[c + r * t_ld]); aa = cconj(Taa[c + r * t_ld]); }
    else { bb = make_double2(Tbb[r + r * t_ld].x, 0.0); aa = make_double2(Taa[r + r * t_ld].x, 0.0); }
    f[fs + r + (long long)c * mp] = make_double2(0.5 * bb.x, 0.5 * bb.y);
    f[2 * fs + r + (long long)c * mp] = aa;
  }
  __syncthreads();
  if (!do_chol) {
    if (threadIdx.x == 0 && rank == 0) info[b] = -2;
  } else if (!CL) {  // blocked, in place on tril(T_AA) copied into forms[3]
    double2* F = f + 3 * fs;
    FOR_SQUARE(m, r, c) {
      F[r + (long long)c * mp] = r >= c ? Taa[r + c * t_ld] : make_double2(0.0, 0.0);
    }
    __syncthreads();
    chol_blocked(m, F, mp, info + b);
  } else {
    cg::cluster_group cl = cg::this_cluster();
    __shared__ int s_nan;
    if (threadIdx.x == 0) s_nan = 0;
    cl.sync();
    int* nan0 = cl.map_shared_rank(&s_nan, 0);
    double2* F = f + 3 * fs;
    bool nan = false;
    for (int c = c0; c < m; c += cs)
      for (int r = threadIdx.x & 31; r < m; r += 32) {
        const double2 v = r >= c ? Taa[r + c * t_ld] : make_double2(0.0, 0.0);
        nan = nan || isnan(v.x) || isnan(v.y);
        F[r + (long long)c * mp] = v;
      }
    if (nan) atomicOr(nan0, 1);
    __threadfence();
    cl.sync();
    if (*nan0) {
      if (rank == 0 && threadIdx.x == 0) info[b] = -1;
    } else {
      chol_blocked_cluster(m, F, mp, info + b);
    }
  }
}

// Joint factor of one T set: the 2m x 2m Hermitian
//   T = [[T_AA, T_AB], [T_AB^H, T_BB]]
// (T_AA / T_BB from their lower triangles with real diagonals, as hermitian_product and
// cholesky_factor read them, kernels.py:198-201 / :217-228) so that per atom
//   A^H T_AA A + A^H T_AB B + B^H T_AB^H A + B^H T_BB B = W^H W,  W = L^H [A; B],  T = L L^H,
// i.e. the H of build_H_ABBA_BB + build_H_AA (builder.py:212-315) as one rank-2m update.
// Structure split: when the set's dense size d =
// (l_nonsph+1)^2 is below m and every T entry outside the leading d x d blocks is zero except
// the diagonals (what assemble_T builds, flapw.py:306-363), the joint matrix is factored in the
// order (A rows 0..d, B rows 0..d) and then one 2x2 block [[T_AA_ii, T_AB_ii], [conj, T_BB_ii]]
// per tail row i: a dense 2d x 2d factor plus per-row 2x2 factors (l11, l21, l22) stored in the
// region's last two columns (l11 + i l22, l21).  The factor is written in place over the
// assembled lower triangle (ld 2*mp); info as chol_block (0 = HPD); without the split L11
// equals the T_AA factor of tprep_kernel bit for bit.  info_host / split_host (mapped) may be
// null.
template <bool CL>
__global__ void __launch_bounds__(512) tjoint_kernel(const int* tdim, const int* tdense, int mp, const double2* taa,
                              const double2* tab, const double2* tbb, long long t_ld,
                              double2* joint, int* info, int* info_host, int* split_host,
                              const double* u2, double sigma_fixed, double* sigma_host) {
  namespace cg = cooperative_groups;
  __shared__ int s_off, s_tail_bad;
  __shared__ double s_scale, s_rho;
  HSDLA_PROF_START();
  // CL: a cluster of kCS CTAs per T set: the assembly's columns and the factorisation's trailing
  // updates are split over the ranks (chol_blocked_cluster); rank 0 owns the decisions and the
  // outputs, the other ranks reduce their flags and row sums into its shared memory.
  const int b = CL ? blockIdx.x / kCS : blockIdx.x;
  const int rank = CL ? (int)cg::this_cluster().block_rank() : 0;
  const int nrk = CL ? kCS : 1;
  const int m = tdim[b];
  const int d = tdense ? min(max(tdense[b], 0), m) : m;
  const long long lj = 2LL * mp;
  const long long tstride = t_ld * t_ld;
  const double2* Taa = taa + b * tstride;
  const double2* Tab = tab + b * tstride;
  const double2* Tbb = tbb + b * tstride;
  // Shift metric diag(I, U^2) of this set (u2 rows, < 0 = shift not allowed for this set)
  const double* U2 = u2 ? u2 + (long long)b * mp : nullptr;
  const bool can_shift = U2 && U2[0] >= 0.0;
  double2* J = joint + (long long)b * lj * lj;
  if (threadIdx.x == 0) {
    s_off = 0;
    s_scale = 0.0;
    s_rho = 0.0;
  }
  __syncthreads();
  if (can_shift)  // max |T_ii| / D_ii: the scale of the shift search (non-negative: max on the bits)
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
      const double v = fmax(fabs(Taa[i + i * t_ld].x), fabs(Tbb[i + i * t_ld].x) / fmax(U2[i], 1e-300));
      atomicMax(reinterpret_cast<unsigned long long*>(&s_scale), __double_as_longlong(v));
    }
  __syncthreads();
  // Gershgorin radius of the 2m x 2m matrix (max absolute row sum): the shift guard's scale.
  // Every thread takes whole columns' worth of entries (consecutive threads on consecutive
  // rows of a column: coalesced), row sums accumulate in shared memory.
  __shared__ double s_row[2 * (HSDLA_MAX_LSPH + 1) * (HSDLA_MAX_LSPH + 1)];
  const bool want_rho = sigma_host && sigma_fixed < 0.0;
  const bool split_cand = tdense && min(max(tdense[b], 0), m) < m;
  // without a split candidate the assembly pass sums the rows; else a separate pass (rank 0)
  const bool rho_in_assembly = want_rho && !split_cand;
  if (want_rho) {
    for (int r = threadIdx.x; r < 2 * m; r += blockDim.x) s_row[r] = 0.0;
    __syncthreads();
  }
  if (want_rho && split_cand && rank == 0) {
    const int n2 = 2 * m;
    FOR_SQUARE(n2, r, c) {
      double2 v;
      const int rr = r < m ? r : r - m, cc = c < m ? c : c - m;
      if (r < m && c < m) v = rr >= cc ? Taa[rr + cc * t_ld] : cconj(Taa[cc + rr * t_ld]);
      else if (r < m) v = Tab[rr + cc * t_ld];
      else if (c < m) v = cconj(Tab[cc + rr * t_ld]);
      else v = rr >= cc ? Tbb[rr + cc * t_ld] : cconj(Tbb[cc + rr * t_ld]);
      if (rr == cc && (r < m) == (c < m)) v.y = 0.0;
      atomicAdd(s_row + r, sqrt(v.x * v.x + v.y * v.y));
    }
    __syncthreads();
    for (int r = threadIdx.x; r < n2; r += blockDim.x)
      atomicMax(reinterpret_cast<unsigned long long*>(&s_rho), __double_as_longlong(s_row[r]));
    __syncthreads();
  }
  HSDLA_PROF_POINT(7);
  bool split = d < m;
  if (split) {  // every coupling of a tail row other than its own diagonal must vanish
    FOR_SQUARE(m, r, c) {
      if (r == c || (r < d && c < d)) continue;
      const double2 x = Tab[r + c * t_ld];
      bool nz = x.x != 0.0 || x.y != 0.0;
      if (r > c) {
        const double2 y = Taa[r + c * t_ld], z = Tbb[r + c * t_ld];
        nz = nz || y.x != 0.0 || y.y != 0.0 || z.x != 0.0 || z.y != 0.0;
      }
      if (nz) s_off = 1;
    }
    __syncthreads();
    split = s_off == 0;
  }
  const int h = split ? d : m, n = 2 * h;
  // sigma_fixed >= 0: factor T + sigma D once.  Otherwise T itself, and when that is not HPD and
  // the set may shift, T + sigma D for sigma = scale * 2^(k - 12), k = 0, 1, ... (the first that
  // is HPD, i.e. within 2x of the smallest such shift).
  if (sigma_fixed > 0.0 && !can_shift) {  // a common shift cannot apply to this set
    if (threadIdx.x == 0 && rank == 0) {
      info[b] = -3;
      if (info_host) info_host[b] = -3;
      if (split_host) split_host[b] = 0;
      if (sigma_host) sigma_host[b] = -1.0;
    }
    return;
  }
  double sigma = sigma_fixed >= 0.0 ? sigma_fixed : 0.0;
  const int attempts = (sigma_fixed < 0.0 && can_shift) ? 40 : 1;
  int* flag0 = &s_tail_bad;  // rank 0's flag (the cluster's)
  double* row0 = s_row;      // rank 0's row sums
  if constexpr (CL) {
    flag0 = cg::this_cluster().map_shared_rank(&s_tail_bad, 0);
    row0 = cg::this_cluster().map_shared_rank(s_row, 0);
  }
  for (int att = 0; att < attempts; ++att) {
    if (att > 0) sigma = s_scale * ldexp(1.0, att - 13);
    if (threadIdx.x == 0) s_tail_bad = 0;  // also the NaN flag of the assembly below
    if constexpr (CL) cg::this_cluster().sync();
    else __syncthreads();
    // (rows by lanes with whole-warp iterations: the row-sum reduction below shuffles; columns
    // split over the cluster's ranks)
    bool nan = false;
    const bool sums = rho_in_assembly && att == 0;  // Gershgorin row sums of the unshifted matrix
    // Lane l of a warp walks rows l, l + 32, ...: its share of each row's |T_rc| sum stays in
    // registers across the warp's columns and reaches shared memory once per (warp, row) at the
    // end; the mirror's |T_cr| of column c is warp-reduced (one add per column).  (Per-element
    // shared-memory double atomics here cost ~70 k cycles at 2m = 162.)
    constexpr int kRowChunks = (2 * (HSDLA_MAX_LSPH + 1) * (HSDLA_MAX_LSPH + 1) + 31) / 32;
    double rsum[kRowChunks];
#pragma unroll
    for (int i = 0; i < kRowChunks; ++i) rsum[i] = 0.0;
    for (int c = rank * (blockDim.x >> 5) + (threadIdx.x >> 5); c < n; c += nrk * (blockDim.x >> 5)) {
      double mirror = 0.0;  // the warp shares column c
#pragma unroll
      for (int i = 0; i < kRowChunks; ++i) {
        const int r0 = 32 * i;
        if (r0 >= n) break;
        const int r = r0 + (threadIdx.x & 31);
        double2 v = make_double2(0.0, 0.0);
        if (r < n && r >= c) {
          if (r < h) v = Taa[r + c * t_ld];
          else if (c < h) v = cconj(Tab[c + (r - h) * t_ld]);
          else v = Tbb[(r - h) + (c - h) * t_ld];
          nan = nan || isnan(v.x) || isnan(v.y);
          if (r == c) v.y = 0.0;
          if (sums) {
            const double av = sqrt(v.x * v.x + v.y * v.y);
            rsum[i] += av;
            if (r > c) mirror += av;
          }
          if (r == c && sigma != 0.0) v.x += sigma * (r < h ? 1.0 : U2[r - h]);
        }
        if (r < n) J[r + c * lj] = v;
      }
      if (sums) {
        for (int o = 16; o > 0; o >>= 1) mirror += __shfl_xor_sync(0xffffffffu, mirror, o);
        if ((threadIdx.x & 31) == 0 && mirror != 0.0) atomicAdd(s_row + c, mirror);
      }
    }
    if (sums) {
#pragma unroll
      for (int i = 0; i < kRowChunks; ++i) {
        const int r = 32 * i + (threadIdx.x & 31);
        if (r < n && rsum[i] != 0.0) atomicAdd(s_row + r, rsum[i]);
      }
    }
    if (nan) atomicOr(flag0, 1);
    if constexpr (CL) {  // the other ranks' partial row sums into rank 0's (one add per row)
      if (rho_in_assembly && att == 0 && rank != 0) {
        __syncthreads();
        for (int r = threadIdx.x; r < n; r += blockDim.x)
          if (s_row[r] != 0.0) atomicAdd(row0 + r, s_row[r]);
      }
    }
    __threadfence();
    if constexpr (CL) cg::this_cluster().sync();
    else __syncthreads();
    if (rho_in_assembly && att == 0 && rank == 0) {
      for (int r = threadIdx.x; r < n; r += blockDim.x)
        atomicMax(reinterpret_cast<unsigned long long*>(&s_rho), __double_as_longlong(s_row[r]));
      __syncthreads();
    }
    HSDLA_PROF_POINT(8);
    if (*flag0) {
      if (threadIdx.x == 0 && rank == 0) info[b] = -1;
    } else if constexpr (CL) {
      chol_blocked_cluster(n, J, lj, info + b);  // in place; shared memory sized for 2*mp rows
    } else {
      chol_blocked(n, J, lj, info + b, true);
    }
    __threadfence();
    if constexpr (CL) cg::this_cluster().sync();  // every rank sees info[b]
    __syncthreads();
    if (threadIdx.x == 0) s_tail_bad = 0;
    __syncthreads();
    HSDLA_PROF_POINT(6);
    if (split && info[b] == 0 && rank == 0) {
      for (int i = d + threadIdx.x; i < m; i += blockDim.x) {
        const double a = Taa[i + i * t_ld].x + sigma, c = Tbb[i + i * t_ld].x + (sigma != 0.0 ? sigma * U2[i] : 0.0);
        const double2 ab = Tab[i + i * t_ld];
        bool ok = a > 0.0 && isfinite(a);
        const double l11 = ok ? sqrt(a) : 1.0;
        const double2 l21 = make_double2(ab.x / l11, -ab.y / l11);  // T_BA_ii / l11
        const double rr = c - (l21.x * l21.x + l21.y * l21.y);
        ok = ok && rr > 0.0 && isfinite(rr);
        J[i + (lj - 2) * lj] = make_double2(l11, ok ? sqrt(rr) : 0.0);
        J[i + (lj - 1) * lj] = l21;
        if (!ok) atomicExch(&s_tail_bad, 1);
      }
      __syncthreads();
      if (threadIdx.x == 0 && s_tail_bad) info[b] = n + 1;  // a tail block is not HPD
    }
    __threadfence();
    if constexpr (CL) cg::this_cluster().sync();
    __syncthreads();
    if (info[b] == 0 || info[b] == -1) break;  // HPD, or NaN input (no shift helps)
  }
  if (threadIdx.x == 0 && rank == 0) {
    if (info_host) info_host[b] = info[b];
    if (split_host) split_host[b] = split ? 1 : 0;
    if (sigma_host) sigma_host[b] = info[b] == 0 ? sigma : -1.0;
    if (sigma_host && sigma_fixed < 0.0) sigma_host[96 + b] = s_rho;  // guard scale
  }
}

// Tail rows of split joint T sets: for atom entry e = (row offset, d, m, T set) and every
// column, W1_i = l11 A_i + conj(l21) B_i (XY slot) and W2_i = l22 B_i (Z slot), i in [d, m).
__global__ void ttail_kernel(const int4* atoms, int n_basis, const double2* __restrict__ A,
                             const double2* __restrict__ B, long long ld, double2* XY, double2* Z,
                             const double2* joint, long long lj) {
  const int4 at = atoms[blockIdx.y];
  const int t = at.z - at.y;  // tail rows
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t <= 0 || idx >= (long long)t * n_basis) return;
  const int i = at.y + (int)(idx % t);
  const long long col = idx / t;
  const double2* L = joint + (long long)at.w * lj * lj;
  const double2 l1122 = L[i + (lj - 2) * lj], l21 = L[i + (lj - 1) * lj];
  const long long e = at.x + i + col * ld;
  const double2 a = A[e], bb = B[e];
  // conj(l21) * b = (l21.x b.x + l21.y b.y) + i (l21.x b.y - l21.y b.x)
  XY[e] = make_double2(l1122.x * a.x + l21.x * bb.x + l21.y * bb.y,
                       l1122.x * a.y + l21.x * bb.y - l21.y * bb.x);
  Z[e] = make_double2(l1122.y * bb.x, l1122.y * bb.y);
}

// ---------------------------------------------------------------------------
// Mirror: 32x32 tiles over the lower triangle; tile (ti, tj), ti >= tj.
__global__ void mirror_kernel(int n, double2* C, long long ldc, int* flag) {
  __shared__ double2 tile[32][33];
  int b = blockIdx.x, tj = 0;
  const int nb = (n + 31) / 32;
  while (b >= nb - tj) { b -= nb - tj; ++tj; }
  const int ti = tj + b;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  bool bad = false;
  for (int c = ty; c < 32; c += 8) {
    const int i = ti * 32 + tx, j = tj * 32 + c;
    if (i < n && j < n && i >= j) {
      double2 v = C[i + (long long)j * ldc];
      if (i == j) { v.y = 0.0; C[i + (long long)j * ldc] = v; }
      bad |= !(isfinite(v.x) && isfinite(v.y));
      tile[c][tx] = v;  // tile[col][row]
    }
  }
  __syncthreads();
  // write upper: C[j, i] = conj(C[i, j]) for i > j; coalesced over j (tx)
  for (int r = ty; r < 32; r += 8) {
    const int i = ti * 32 + r, j = tj * 32 + tx;
    if (i < n && j < n && i > j) C[j + (long long)i * ldc] = cconj(tile[tx][r]);
  }
  if (bad) atomicOr(flag, 1);
}

__global__ void scale_rows_kernel(int m, int n, const double* d, double2* B, long long ldb) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y;
  if (i < m) {
    double2 v = B[i + (long long)j * ldb];
    const double s = d[i];
    B[i + (long long)j * ldb] = make_double2(v.x * s, v.y * s);
  }
}

__global__ void prep_kernel(int op, int rows, int cols, const double2* in, long long ldin,
                            double2* out, long long ldout, double scale) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  const int c = blockIdx.y;
  if (r >= rows) return;
  double2 v;
  switch (op) {
    case PREP_COPY: v = in[r + (long long)c * ldin]; break;
    case PREP_CONJ_TRANS: v = cconj(in[c + (long long)r * ldin]); break;
    case PREP_HERM_FULL:
      if (r > c) v = in[r + (long long)c * ldin];
      else if (r < c) v = cconj(in[c + (long long)r * ldin]);
      else v = make_double2(in[r + (long long)r * ldin].x, 0.0);
      break;
    case PREP_TRIL: v = (r >= c) ? in[r + (long long)c * ldin] : make_double2(0.0, 0.0); break;
    default: v = (r <= c) ? cconj(in[c + (long long)r * ldin]) : make_double2(0.0, 0.0); break;
  }
  if (scale != 1.0) { v.x *= scale; v.y *= scale; }
  out[r + (long long)c * ldout] = v;
}

__global__ void publish_kernel(const int* flag, const int* info, int n, int* out) {
  for (int i = threadIdx.x; i <= n; i += blockDim.x) {
    volatile int* o = out;
    o[i] = (i == 0) ? *flag : info[i - 1];
  }
  __threadfence_system();
}

__global__ void zero_rows_kernel(double2* base, long long ld, int row0, int rows) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  const int c = blockIdx.y;
  if (r < rows) base[row0 + r + (long long)c * ld] = make_double2(0.0, 0.0);
}

}  // namespace

int launch_potrf_batched(hsdla_ctx* ctx, int n, int batch, const double2* T, long long ldt,
                         long long stride_t, double2* F, long long ldf, long long stride_f,
                         int* info_dev) {
  if (batch <= 0 || n <= 0) return HSDLA_OK;
  if (size_t(n) * sizeof(double2) > size_t(kPotrfMaxDynSmem) - 1024) {
    set_error("Cholesky order above 14400 (one shared-memory row per CTA)");
    return HSDLA_ERR_UNSUPPORTED;
  }
  const size_t smem = n <= kBlockedMaxN ? chol_blocked_smem(n) : size_t(n) * sizeof(double2);
  potrf_batched_kernel<<<batch, 512, smem, ctx->stream>>>(n, T, ldt, stride_t, F, ldf, stride_f,
                                                          info_dev);
  HS_CHECK_LAUNCH();
  return HSDLA_OK;
}

int launch_tprep(hsdla_ctx* ctx, cudaStream_t stream, int n_tsets, const int* tdim_dev, int mp,
                 const double2* taa, const double2* tab, const double2* tbb, long long t_ld,
                 double2* forms, int do_chol, int* info_dev) {
  if (n_tsets <= 0) return HSDLA_OK;
  const size_t smem = chol_blocked_smem(mp);  // limit set once per device in preload_small()
  if (tprep_cluster() && mp >= kClusterMinN) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kCS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(n_tsets * kCS);
    cfg.blockDim = dim3(512);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    HS_CUDA(cudaLaunchKernelEx(&cfg, tprep_kernel<true>, tdim_dev, mp, taa, tab, tbb, t_ld, forms,
                               do_chol, info_dev));
    return HSDLA_OK;
  }
  tprep_kernel<false><<<n_tsets, 512, smem, stream>>>(tdim_dev, mp, taa, tab, tbb, t_ld, forms,
                                                      do_chol, info_dev);
  HS_CHECK_LAUNCH();
  return HSDLA_OK;
}

int launch_tjoint(cudaStream_t stream, int n_tsets, const int* tdim_dev, const int* tdense_dev,
                  int mp, const double2* taa, const double2* tab, const double2* tbb,
                  long long t_ld, double2* joint, int* info_dev, int* info_host_dev,
                  int* split_host_dev, const double* u2_dev, double sigma_fixed,
                  double* sigma_host_dev) {
  if (n_tsets <= 0) return HSDLA_OK;
  const size_t smem = chol_blocked_smem(2 * mp);
  if (tprep_cluster() && 2 * mp >= kClusterMinN) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kCS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(n_tsets * kCS);
    cfg.blockDim = dim3(512);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    HS_CUDA(cudaLaunchKernelEx(&cfg, tjoint_kernel<true>, tdim_dev, tdense_dev, mp, taa, tab, tbb,
                               t_ld, joint, info_dev, info_host_dev, split_host_dev, u2_dev,
                               sigma_fixed, sigma_host_dev));
    return HSDLA_OK;
  }
  tjoint_kernel<false><<<n_tsets, 512, smem, stream>>>(tdim_dev, tdense_dev, mp, taa, tab, tbb,
                                                       t_ld, joint, info_dev, info_host_dev,
                                                       split_host_dev, u2_dev, sigma_fixed,
                                                       sigma_host_dev);
  HS_CHECK_LAUNCH();
  return HSDLA_OK;
}

// C -= sigma * S over the full n x n matrices (both column-major, ld ldc / lds).
__global__ void axpy_shift_kernel(int n, double sigma, const double2* __restrict__ S, long long lds,
                                  double2* __restrict__ C, long long ldc) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const long long j = blockIdx.y;
  if (i >= n) return;
  const double2 s = S[i + j * lds];
  double2 c = C[i + j * ldc];
  c.x -= sigma * s.x;
  c.y -= sigma * s.y;
  C[i + j * ldc] = c;
}

int launch_axpy_shift(hsdla_ctx* ctx, int n, double sigma, const double2* S, long long lds,
                      double2* C, long long ldc) {
  if (n <= 0) return HSDLA_OK;
  axpy_shift_kernel<<<dim3((n + 255) / 256, n), 256, 0, ctx->stream>>>(n, sigma, S, lds, C, ldc);
  HS_CHECK_LAUNCH();
  return HSDLA_OK;
}

int launch_ttail(hsdla_ctx* ctx, const int4* atoms_dev, int n_atoms, int max_tail, int n_basis,
                 const double2* A, const double2* B, long long ld, double2* XY, double2* Z,
                 const double2* joint, long long lj) {
  if (n_atoms <= 0 || max_tail <= 0 || n_basis <= 0) return HSDLA_OK;
  const long long work = (long long)max_tail * n_basis;
  ttail_kernel<<<dim3((unsigned)((work + 255) / 256), n_atoms), 256, 0, ctx->stream>>>(
      atoms_dev, n_basis, A, B, ld, XY, Z, joint, lj);
  HS_CHECK_LAUNCH();
  return HSDLA_OK;
}

int launch_mirror(hsdla_ctx* ctx, int n, double2* C, long long ldc, int* flag_dev) {
  if (n <= 0) return HSDLA_OK;
  const int nb = (n + 31) / 32;
  mirror_kernel<<<nb * (nb + 1) / 2, dim3(32, 8), 0, ctx->stream>>>(n, C, ldc, flag_dev);
  HS_CHECK_LAUNCH();
  return HSDLA_OK;
}

int launch_scale_rows(hsdla_ctx* ctx, int m, int n, const double* d, double2* B, long long ldb) {
  if (m <= 0 || n <= 0) return HSDLA_OK;
  scale_rows_kernel<<<dim3((m + 127) / 128, n), 128, 0, ctx->stream>>>(m, n, d, B, ldb);
  HS_CHECK_LAUNCH();
  return HSDLA_OK;
}

int launch_prep(hsdla_ctx* ctx, int op, int rows, int cols, const double2* in, long long ldin,
                double2* out, long long ldout, double scale) {
  if (rows <= 0 || cols <= 0) return HSDLA_OK;
  prep_kernel<<<dim3((rows + 127) / 128, cols), 128, 0, ctx->stream>>>(op, rows, cols, in, ldin,
                                                                        out, ldout, scale);
  HS_CHECK_LAUNCH();
  return HSDLA_OK;
}

int launch_publish(hsdla_ctx* ctx, const int* flag, const int* info, int n, int* out_mapped) {
  publish_kernel<<<1, 128, 0, ctx->stream>>>(flag, info, n, out_mapped);
  HS_CHECK_LAUNCH();
  return HSDLA_OK;
}

// flag |= 1 if any element of the m x n window is NaN/Inf (write_hsm1's guard,
// matrix.py:244-246).  Rows are the fast index: one coalesced 16-byte load per thread.
__global__ void finite_kernel(int m, int n, const double2* __restrict__ A, long long lda,
                              int* flag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  bool bad = false;
  if (i < m)
    for (int j = blockIdx.y; j < n; j += gridDim.y) {
      const double2 v = A[i + (long long)j * lda];
      bad |= !(isfinite(v.x) && isfinite(v.y));
    }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

int launch_finite_check(hsdla_ctx* ctx, int m, int n, const double2* A, long long lda, int* flag) {
  if (m <= 0 || n <= 0) return HSDLA_OK;
  const int gy = n < 4096 ? n : 4096;
  finite_kernel<<<dim3((m + 255) / 256, gy), 256, 0, ctx->stream>>>(m, n, A, lda, flag);
  HS_CHECK_LAUNCH();
  return HSDLA_OK;
}

int launch_zero_rows(hsdla_ctx* ctx, double2* base, long long ld, int row0, int rows, int cols) {
  if (rows <= 0 || cols <= 0) return HSDLA_OK;
  zero_rows_kernel<<<dim3((rows + 127) / 128, cols), 128, 0, ctx->stream>>>(base, ld, row0, rows);
  HS_CHECK_LAUNCH();
  return HSDLA_OK;
}

int preload_small() {
  const void* fns[] = {(const void*)potrf_batched_kernel, (const void*)tprep_kernel<false>,
                       (const void*)tprep_kernel<true>, (const void*)tjoint_kernel<true>,
                       (const void*)mirror_kernel, (const void*)scale_rows_kernel,
                       (const void*)prep_kernel, (const void*)publish_kernel,
                       (const void*)zero_rows_kernel, (const void*)finite_kernel,
                       (const void*)tjoint_kernel<false>, (const void*)ttail_kernel,
                       (const void*)axpy_shift_kernel};
  for (const void* f : fns) {
    cudaFuncAttributes at;
    HS_CUDA(cudaFuncGetAttributes(&at, f));
  }
  if (first_on_device((const void*)potrf_batched_kernel)) {  // one row of n complex per CTA
    cudaFuncAttributes at;
    HS_CUDA(cudaFuncGetAttributes(&at, (const void*)potrf_batched_kernel));
    HS_CUDA(cudaFuncSetAttribute(potrf_batched_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kPotrfMaxDynSmem - (int)at.sharedSizeBytes));
  }
  for (const void* f : {(const void*)tjoint_kernel<false>, (const void*)tprep_kernel<false>,
                        (const void*)tjoint_kernel<true>, (const void*)tprep_kernel<true>})
    if (first_on_device(f)) {
      cudaFuncAttributes at;
      HS_CUDA(cudaFuncGetAttributes(&at, f));
      HS_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   kPotrfMaxDynSmem - (int)at.sharedSizeBytes));
    }
  return HSDLA_OK;
}

}  // namespace hsdla
