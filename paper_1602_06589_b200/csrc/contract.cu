// Multi-segment complex128 contraction on FP64 tensor cores (DMMA) for sm_100a.
//
//   C (+)= sum_s P_s^H Q_s        (P_s: k_s x m, Q_s: k_s x n, column-major, K-contiguous)
//
// This one kernel carries every level-3 update of the HSDLA build
// (reference builder.py:199-315 / kernels.py:56-132):
//   * S  = A*^H A* + (U B*)^H (U B*)                       two ZHERK segments
//   * H  = Z*^H B* + B*^H Z* + Y^H Y + A_nh^H X_nh          ZHER2K + ZHERK + ZGEMM segments
//   * Z_a = T_AB^H A_a + (1/2 T_BB)^H B_a, Y_a = C_a^H A_a, X_a = T_AA A_a  (batched small GEMMs)
// Triangular problems compute only lower tiles and (PROB_TRI_MIRROR) write the Hermitian
// mirror in the epilogue, replacing HermitianAccumulator.mirror_to_full (matrix.py:216-226).
//
// FP64 on sm_100a has no tcgen05 kind: the tensor path is mma.sync.m8n8k4.f64 (SASS
// DMMA.8x8x4), 128 flop/clk/SM = 37.2 TF at 1965 MHz (measured, profiles/r01_fp64_peaks.json).
// Complex arithmetic uses the real embedding over interleaved (re, im) pairs, K' = 2K:
//   Re C = P^T Q        Im C = P^T (J Q),  (J Q)[2k] = Q[2k+1], (J Q)[2k+1] = -Q[2k]
// so every complex MAC is exactly 4 real FMAs (the ledger's 8 flops), no 3M trick.
//
// CTA: 128 threads = 2x2 warps, 64x64 complex output tile, each warp 32x32 complex
// (16 DMMA blocks for Re + 16 for Im).  K is staged in chunks of 16 complex (256 B per
// column) through a 3-stage cp.async ring, 32-byte XOR swizzle (conflict-free fragment
// loads).  Persistent grid with an atomic tile counter; results are deterministic because
// each tile is owned by one CTA and its K order is fixed.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace hsdla {

namespace {

constexpr int kThreads = 128;
constexpr int kStages = 3;
constexpr int kChunk = 16;                     // complex K per stage
constexpr int kColDoubles = 2 * kChunk;        // 32 doubles per column per stage
constexpr int kOpDoubles = kTile * kColDoubles;  // 2048 doubles = 16 KB per operand
constexpr int kStageDoubles = 2 * kOpDoubles;
constexpr size_t kSmemBytes = size_t(kStages) * kStageDoubles * sizeof(double);

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc, int src_bytes) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gsrc),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ bool finite2(double2 v) {
  return isfinite(v.x) && isfinite(v.y);
}

__global__ void __launch_bounds__(kThreads, 2)
    contract_kernel(const Prob* __restrict__ probs, int nprob, const Seg* __restrict__ segs,
                    int ntiles, int* __restrict__ counter, int* __restrict__ flag) {
  extern __shared__ __align__(128) double smem[];
  __shared__ int s_tile;

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int wm = warp & 1, wn = warp >> 1;
  const int g = lane >> 2, q = lane & 3;
  const unsigned sign_hi = (q & 1) ? 0x80000000u : 0u;
  // cp.async slot of this thread: complex element lp of the chunk, columns lc + 8r.
  const int lp = tid & 15;
  const int lc = tid >> 4;
  const int dst_lane = (((lp >> 1) ^ lc) << 2) + (lp & 1) * 2;  // within a column (doubles)

  for (;;) {
    if (tid == 0) s_tile = atomicAdd(counter, 1);
    __syncthreads();
    const int t = s_tile;
    __syncthreads();
    if (t >= ntiles) break;

    int lo = 0, hi = nprob - 1;
    while (lo < hi) {
      int mid = (lo + hi + 1) >> 1;
      if (probs[mid].tile_base <= t) lo = mid; else hi = mid - 1;
    }
    const Prob pr = probs[lo];
    int local = t - pr.tile_base;
    int tm, tn;
    if (pr.kind == PROB_GENERAL) {
      tm = local % pr.tiles_m;
      tn = local / pr.tiles_m;
    } else {
      const int nb = pr.tiles_m;
      tn = pr.col_tile_lo;
      while (local >= nb - tn) { local -= nb - tn; ++tn; }
      tm = tn + local;
    }
    const int i0 = tm * kTile, j0 = tn * kTile;
    const int mP = pr.m, mQ = pr.n;

    // Count chunks of this problem and find the first non-empty segment.
    int nchunks = 0;
    for (int s = 0; s < pr.nseg; ++s) nchunks += (segs[pr.seg0 + s].k + kChunk - 1) / kChunk;

    int isi = pr.seg0;
    const int send = pr.seg0 + pr.nseg;
    while (isi < send && segs[isi].k <= 0) ++isi;
    Seg cur;
    if (isi < send) cur = segs[isi];
    int iko = 0;

    auto issue = [&](int stage) {
      double* sP = smem + stage * kStageDoubles;
      double* sQ = sP + kOpDoubles;
      const bool kval = (iko + lp) < cur.k;
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int col = lc + 8 * r;
        const int gp = i0 + col;
        const bool vp = kval && gp < mP;
        const double2* srcp = vp ? cur.P + (long long)gp * cur.ldP + iko + lp : cur.P;
        cp_async16(sP + col * kColDoubles + dst_lane, srcp, vp ? 16 : 0);
        const int gq = j0 + col;
        const bool vq = kval && gq < mQ;
        const double2* srcq = vq ? cur.Q + (long long)gq * cur.ldQ + iko + lp : cur.Q;
        cp_async16(sQ + col * kColDoubles + dst_lane, srcq, vq ? 16 : 0);
      }
      iko += kChunk;
      if (iko >= cur.k) {
        iko = 0;
        ++isi;
        while (isi < send && segs[isi].k <= 0) ++isi;
        if (isi < send) cur = segs[isi];
      }
    };

    double accR[4][4][2], accI[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        accR[a][b][0] = accR[a][b][1] = 0.0;
        accI[a][b][0] = accI[a][b][1] = 0.0;
      }

#pragma unroll
    for (int st = 0; st < kStages - 1; ++st) {
      if (st < nchunks) issue(st);
      cp_async_commit();
    }

    for (int c = 0; c < nchunks; ++c) {
      cp_async_wait<kStages - 2>();
      __syncthreads();
      const int nc = c + kStages - 1;
      if (nc < nchunks) issue(nc % kStages);
      cp_async_commit();

      const double* sP = smem + (c % kStages) * kStageDoubles;
      const double* sQ = sP + kOpDoubles;
      const double* pa = sP + (wm * 32 + g) * kColDoubles;
      const double* pb = sQ + (wn * 32 + g) * kColDoubles;
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const int off = ((s ^ g) << 2);
        double a[4], br[4], bi[4];
#pragma unroll
        for (int ib = 0; ib < 4; ++ib) a[ib] = pa[ib * 8 * kColDoubles + off + q];
#pragma unroll
        for (int jb = 0; jb < 4; ++jb) {
          br[jb] = pb[jb * 8 * kColDoubles + off + q];
          const double x = pb[jb * 8 * kColDoubles + off + (q ^ 1)];
          bi[jb] = __hiloint2double(__double2hiint(x) ^ sign_hi, __double2loint(x));
        }
#pragma unroll
        for (int ib = 0; ib < 4; ++ib)
#pragma unroll
          for (int jb = 0; jb < 4; ++jb) {
            dmma(accR[ib][jb][0], accR[ib][jb][1], a[ib], br[jb]);
            dmma(accI[ib][jb][0], accI[ib][jb][1], a[ib], bi[jb]);
          }
      }
    }
    cp_async_wait<0>();
    __syncthreads();

    // ---- epilogue
    bool bad = false;
#pragma unroll
    for (int ib = 0; ib < 4; ++ib) {
      const int i = i0 + wm * 32 + ib * 8 + g;
#pragma unroll
      for (int jb = 0; jb < 4; ++jb) {
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int j = j0 + wn * 32 + jb * 8 + 2 * q + v;
          double2 val = make_double2(accR[ib][jb][v], accI[ib][jb][v]);
          if (pr.kind == PROB_GENERAL) {
            if (i < pr.m && j < pr.n) {
              double2* cp = pr.C + i + (long long)j * pr.ldC;
              const double2 al = pr.alpha;
              double2 out;
              if (al.x == 1.0 && al.y == 0.0) {
                out = val;
              } else {
                out.x = al.x * val.x - al.y * val.y;
                out.y = al.x * val.y + al.y * val.x;
              }
              if (pr.accumulate) {
                const double2 old = *cp;
                const double2 be = pr.beta;
                out.x += be.x * old.x - be.y * old.y;
                out.y += be.x * old.y + be.y * old.x;
              }
              *cp = out;
            }
          } else if (i < pr.n && j < pr.n && i >= j) {
            double2* cl = pr.C + i + (long long)j * pr.ldC;
            if (pr.accumulate) {
              const double2 old = *cl;
              val.x += old.x;
              val.y += old.y;
            }
            if (pr.kind == PROB_TRI_MIRROR) {
              if (i == j) val.y = 0.0;
              bad |= !finite2(val);
              if (i > j) pr.C[j + (long long)i * pr.ldC] = make_double2(val.x, -val.y);
            }
            *cl = val;
          }
        }
      }
    }
    if (bad) atomicOr(flag, 1);
  }
}

}  // namespace

int prob_tile_count(const Prob& p) {
  if (p.kind == PROB_GENERAL) return p.tiles_m * p.tiles_n;
  int cnt = 0;
  for (int tn = p.col_tile_lo; tn < p.col_tile_hi; ++tn) cnt += p.tiles_m - tn;
  return cnt;
}

int launch_contract(hsdla_ctx* ctx, const std::vector<Prob>& probs_in,
                    const std::vector<Seg>& segs, int counter_slot, int* flag_dev) {
  std::vector<Prob> probs = probs_in;
  int ntiles = 0;
  for (auto& p : probs) {
    p.tiles_m = (p.m + kTile - 1) / kTile;
    p.tiles_n = (p.n + kTile - 1) / kTile;
    if (p.kind != PROB_GENERAL) {
      p.tiles_n = p.tiles_m;
      if (p.col_tile_hi <= 0 || p.col_tile_hi > p.tiles_m) p.col_tile_hi = p.tiles_m;
      if (p.col_tile_lo < 0) p.col_tile_lo = 0;
    }
    p.tile_base = ntiles;
    ntiles += (p.m > 0 && p.n > 0) ? prob_tile_count(p) : 0;
  }
  if (ntiles == 0) return HSDLA_OK;
  static bool attr_set = false;
  if (!attr_set) {
    HS_CUDA(cudaFuncSetAttribute(contract_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kSmemBytes));
    attr_set = true;
  }
  int rc = arena_begin(ctx, probs.size() * sizeof(Prob) + segs.size() * sizeof(Seg) + 256);
  if (rc) return rc;
  Prob* dprobs = static_cast<Prob*>(arena_push(ctx, probs.data(), probs.size() * sizeof(Prob), nullptr));
  Seg* dsegs = static_cast<Seg*>(
      arena_push(ctx, segs.data(), (segs.empty() ? 1 : segs.size()) * sizeof(Seg), nullptr));
  rc = arena_flush(ctx);
  if (rc) return rc;

  int* counter = ctx->scratch_dev + counter_slot;
  HS_CUDA(cudaMemsetAsync(counter, 0, sizeof(int), ctx->stream));
  int occ = 0;
  HS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, contract_kernel, kThreads, kSmemBytes));
  if (occ < 1) occ = 1;
  int grid = ctx->num_sms * occ;
  if (grid > ntiles) grid = ntiles;
  contract_kernel<<<grid, kThreads, kSmemBytes, ctx->stream>>>(dprobs, (int)probs.size(), dsegs,
                                                              ntiles, counter, flag_dev);
  HS_CHECK_LAUNCH();
  return HSDLA_OK;
}

}  // namespace hsdla
