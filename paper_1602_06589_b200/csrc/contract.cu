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
// Complex multiply, default (G3, cmul_mode() == 3): three real DMMA products per complex MAC
// (Gauss / ZHERK3M): accR = sum P_re Q_re, accX = sum P_im Q_im, accI = sum (P_re - P_im)(Q_re +
// Q_im), then Re = accR + accX, Im = accI - accR + accX; its error bound is normwise (see the
// adversarial cases in tests/test_gpu_contracts.py).  HSDLA_CMUL=4: the real embedding over
// interleaved (re, im) pairs, K' = 2K,
//   Re C = P^T Q        Im C = P^T (J Q),  (J Q)[2k] = Q[2k+1], (J Q)[2k+1] = -Q[2k]
// i.e. exactly 4 real FMAs per complex MAC (the ledger's 8 flops).
//
// CTA: 128 threads = 2x2 warps, 64x64 complex output tile, each warp 32x32 complex
// (16 DMMA blocks for Re + 16 for Im).  K is staged in chunks of 16 complex (256 B per
// column) through a 3-stage cp.async ring (zero fill by the ignore-src predicate).  Default
// shared-memory layout "pair": lane q loads complex element 4j+q whole (128-bit) and feeds
// its real part to DMMA step 2j and its imaginary part to step 2j+1 (the K order of the
// real embedding is free as long as P and Q share it); odd columns swap 32-byte units in
// pairs so a quarter-warp's two columns hit opposite bank halves.  Alternatives: "xor"
// (64-bit loads, 32-byte XOR swizzle) and "pad" (288-byte columns).  HSDLA_CP_SPREAD=1
// issues the next chunk's copies a round at a time between DMMA steps at run time; the
// default path keeps that code in the kernel (measured: with it present ptxas interleaves
// the cp.async block with the DMMA stream, 2% faster on C2 than without it).
//
// Work distribution: whole tiles dealt round-robin for floor(T/G) waves (the CTAs of a wave
// walk K in step over neighbouring tiles, so operands stay in L2), then the remaining
// (tile, K-chunk) iterations split evenly over the co-resident CTAs (stream-K, cooperative
// launch): no wave-quantisation tail.  A tile split between CTAs is finished by the CTA
// holding its first chunk, which adds the later pieces' partial tiles in a fixed order:
// results are deterministic run to run (builder.py backup invariance).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "common.cuh"

namespace hsdla {

namespace {

constexpr int kStages = 3;
constexpr int kChunk = 16;                       // complex K per stage
// Column stride in shared memory: 32 doubles of data padded to 36 (288 B).  Eight
// consecutive columns then start 8 banks apart, so a DMMA fragment load (8 columns x 4
// consecutive doubles per half-warp phase) is conflict-free with compile-time offsets.
// PAD = 0 instead keeps 256-B columns with a 32-byte XOR swizzle (k-chunk index ^ column&7).
// PL: the stage also holds the P-side (Re - Im) and Q-side (Re + Im) sum planes of the
// three-product multiply, one double per K element and column (8 KB each per stage).
// KC = complex K elements per stage (16, or 8 with planes so that four stages fit 2 CTAs/SM).
template <int PAD, bool PL = false, int ST = kStages, int KC = kChunk> struct Layout {
  static constexpr int kColDoubles = 2 * KC + (PAD == 1 ? 4 : 0);
  static constexpr int kOpDoubles = kTile * kColDoubles;
  static constexpr int kPlaneDoubles = kTile * KC;
  static constexpr int kStageDoubles = 2 * kOpDoubles + (PL ? 2 * kPlaneDoubles : 0);
  static constexpr size_t kSmemBytes = size_t(ST) * kStageDoubles * sizeof(double);
};
constexpr int kPartialDoubles = kTile * kTile * 2;  // one partial tile (64 KB)

struct SKParams {
  const Prob* probs;
  const Seg* segs;
  long long total_it;
  long long dp_it;    // iterations [0, dp_it) are whole tiles dealt round-robin (dp_waves waves)
  int dp_waves;
  int dp_nch;         // chunks per tile (uniform across problems when dp_waves > 0)
  int spread;         // issue cp.async rounds between DMMA steps (HSDLA_CP_SPREAD=1; default 0)
  int nprob;
  int grid;
  double* partials;
  int* ready;
  int* flag;
};

#ifndef HSDLA_DMMA_VOLATILE
#define HSDLA_DMMA_VOLATILE 1
#endif
// Default three-product K loop: products ordered by column block with the next K group's
// fragments requested inside the current group (0: fragments loaded at the top of each group,
// the earlier loop, kept for A/B builds: `make er ER=0`).
#ifndef HSDLA_EARLY_RELOAD
#define HSDLA_EARLY_RELOAD 1
#endif
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
#if HSDLA_DMMA_VOLATILE
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
#else
  // register-only: the compiler may interleave DMMAs of different accumulators with the
  // fragment loads and sum DADDs (each accumulator's own order is fixed by its dependence)
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
#endif
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc, int src_bytes) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gsrc),
               "r"(src_bytes));
}
// Zero-filling variant with the PTX ignore-src predicate: when !valid no global access is
// made (src may then point anywhere) and the 16 bytes are written as zeros.
__device__ __forceinline__ void cp_async16_zfill(void* smem_dst, const void* gsrc, bool valid) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile(
      "{\n .reg .pred ign;\n setp.eq.u32 ign, %2, 0;\n"
      " cp.async.cg.shared.global [%0], [%1], 16, ign;\n}\n" ::"r"(s),
      "l"(gsrc), "r"((unsigned)valid));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ bool finite2(double2 v) { return isfinite(v.x) && isfinite(v.y); }

__device__ __forceinline__ long long range_start(long long total, int grid, int g) {
  return total * g / grid;
}
// First iteration of CTA g's stream-K range (the part after the data-parallel waves).
__device__ __forceinline__ long long sk_start(const SKParams& sk, int g) {
  return sk.dp_it + range_start(sk.total_it - sk.dp_it, sk.grid, g);
}

__device__ __forceinline__ Seg load_seg(const Seg* s) {
  Seg v = *s;
  if (v.sel && *v.sel != 0) v.P = v.P_alt;
  return v;
}

// JB = 8-column DMMA blocks per warp along n: JB = 4 -> warp tile 32x32 complex, 4 warps
// (128 threads, ~250 registers, 2 warps per SM sub-partition); JB = 2 -> warp tile 32x16,
// 8 warps (256 threads, <= 128 registers, 4 warps per sub-partition).
// G3 with JB = 2 keeps three accumulator sets in 255 registers at one 8-warp CTA per SM.
// PL (G3 only, pair layout): the sums P_re - P_im and Q_re + Q_im come precomputed from global
// memory (Seg::Pd / Seg::Qs, written by their producers) and are staged with the operands, so
// the K loop issues no DADD on the FP64 pipe; ST = ring stages (2 keeps two CTAs per SM).
// MINB = CTAs per SM the register allocation must allow (JB = 2 with G3: 1 = 255 registers,
// 2 = 128 registers for two 8-warp CTAs, 16 warps per SM).
template <int JB, int PAD, bool G3 = false, bool PL = false, int ST = kStages, int KC = kChunk,
          int MINB = (G3 && JB == 2) ? 1 : 2>
__global__ void __launch_bounds__(32 * 2 * (8 / JB), MINB)
    contract_kernel(SKParams sk) {
  static_assert(!PL || (G3 && PAD == 2), "sum planes need the three-product pair layout");
  static_assert(KC == 16 || (KC == 8 && PAD == 2), "8-element chunks: pair layout only");
  constexpr int kStages = ST;
  extern __shared__ __align__(128) double smem[];
  constexpr int kColDoubles = Layout<PAD, PL, ST, KC>::kColDoubles;
  constexpr int kOpDoubles = Layout<PAD, PL, ST, KC>::kOpDoubles;
  constexpr int kStageDoubles = Layout<PAD, PL, ST, KC>::kStageDoubles;
  constexpr int kPlaneDoubles = Layout<PAD, PL, ST, KC>::kPlaneDoubles;
  constexpr int kWarpCols = 8 * JB;
  constexpr int kThreads = 32 * 2 * (kTile / kWarpCols);
  constexpr int kColStep = kThreads / KC;           // columns covered per cp.async round
  constexpr int kRounds = kTile / kColStep;         // cp.async rounds per operand per chunk

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int wm = warp & 1, wn = warp >> 1;
  const int g = lane >> 2, q = lane & 3;
  const unsigned sign_hi = (q & 1) ? 0x80000000u : 0u;
  // cp.async slot of this thread: complex element lp of the chunk, columns lc + kColStep*r.
  const int lp = tid & (KC - 1);
  const int lc = tid / KC;
  const int dst_lane = PAD == 1 ? lp * 2
                       : PAD == 2 ? ((((lp >> 1) ^ ((lc & 1) << 1)) << 2) + (lp & 1) * 2)
                                  : ((((lp >> 1) ^ (lc & 7)) << 2) + (lp & 1) * 2);
  // Sum-plane cp.async slot: 16-byte piece lp2 (K elements 2 lp2, 2 lp2 + 1) of column lc2 +
  // kColStep2 * r; the 32-byte unit u of column c is stored at u ^ sw(c) (KC = 16: c & 3,
  // KC = 8: (c >> 1) & 1), so a fragment's four consecutive K elements of eight columns are
  // read with two wavefronts.
  constexpr int kColStep2 = kThreads / (KC / 2);
  constexpr int kRounds2 = kTile / kColStep2;
  const int lp2 = tid & (KC / 2 - 1);
  const int lc2 = tid / (KC / 2);
  auto psw = [](int c) { return KC == 16 ? (c & 3) : ((c >> 1) & 1); };
  const int dst2 = ((((lp2 >> 1) ^ psw(lc2)) << 2) + ((lp2 & 1) << 1));

  const int cta = blockIdx.x;
  // Work order: dp_waves waves of whole tiles (CTA g takes tile g + w*grid, so the CTAs of
  // a wave start together and walk K in step over neighbouring tiles: the live operand
  // set stays L2-resident), then an even stream-K split of the remaining iterations.
  for (int ph = 0; ph <= sk.dp_waves; ++ph) {
  long long it, it_end;
  if (ph < sk.dp_waves) {
    it = (long long)(cta + ph * sk.grid) * sk.dp_nch;
    it_end = it + sk.dp_nch;
  } else {
    it = sk_start(sk, cta);
    it_end = sk_start(sk, cta + 1);
  }

  while (it < it_end) {
    // ---- locate (problem, tile, chunk range) of the next piece
    int lo = 0, hi = sk.nprob - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (sk.probs[mid].it_base <= it) lo = mid; else hi = mid - 1;
    }
    const Prob pr = sk.probs[lo];
    const long long local = it - pr.it_base;
    const int nch = pr.nchunks;
    int tile = (int)(local / nch);
    const int c_lo = (int)(local - (long long)tile * nch);
    const long long left = it_end - it;
    const int c_hi = (left < (long long)(nch - c_lo)) ? c_lo + (int)left : nch;
    const long long tile_it_end = pr.it_base + (long long)(tile + 1) * nch;
    int tm, tn;
    if (pr.kind == PROB_GENERAL) {
      tm = tile % pr.tiles_m;
      tn = tile / pr.tiles_m;
    } else {
      const int nb = pr.tiles_m;
      tn = pr.col_tile_lo;
      while (tile >= nb - tn) { tile -= nb - tn; ++tn; }
      tm = tn + tile;
    }
    const int i0 = tm * kTile, j0 = tn * kTile;
    const int mP = pr.m, mQ = pr.n;

    // ---- position the issue iterator at chunk c_lo
    int isi = pr.seg0;
    const int send = pr.seg0 + pr.nseg;
    int iko = 0;
    {
      int cb = 0;
      for (; isi < send; ++isi) {
        const int ncs = (sk.segs[isi].k + KC - 1) / KC;
        if (c_lo < cb + ncs) { iko = (c_lo - cb) * KC; break; }
        cb += ncs;
      }
    }
    Seg cur;
    if (isi < send) cur = load_seg(sk.segs + isi);
    else { cur = load_seg(sk.segs + pr.seg0); cur.k = 0; }
    // Per-thread cp.async bases of the current segment: column lc + kColStep*r, element lp.
    // Columns past the problem edge are zero-filled; their count is tile-constant.
    const int nvP = max(0, min(kRounds, (mP - i0 - lc + kColStep - 1) / kColStep));
    const int nvQ = max(0, min(kRounds, (mQ - j0 - lc + kColStep - 1) / kColStep));
    const double2* bP = cur.P + (long long)(i0 + lc) * cur.ldP + lp;
    const double2* bQ = cur.Q + (long long)(j0 + lc) * cur.ldQ + lp;
    long long stP = (long long)kColStep * cur.ldP, stQ = (long long)kColStep * cur.ldQ;
    const int nvP2 = max(0, min(kRounds2, (mP - i0 - lc2 + kColStep2 - 1) / kColStep2));
    const int nvQ2 = max(0, min(kRounds2, (mQ - j0 - lc2 + kColStep2 - 1) / kColStep2));
    const double* bPd = nullptr;
    const double* bQs = nullptr;
    if constexpr (PL) {
      bPd = cur.Pd + (long long)(i0 + lc2) * cur.ldP + 2 * lp2;
      bQs = cur.Qs + (long long)(j0 + lc2) * cur.ldQ + 2 * lp2;
    }

    // cp.async rounds [r0, r1) of the chunk at iko into `stage` (round r = columns
    // lc + kColStep*r of both operands), then advance() moves iko to the next chunk.
    auto issue_rounds = [&](int stage, int r0, int r1) {
      double* sP = smem + stage * kStageDoubles + lc * kColDoubles + dst_lane;
      double* sQ = sP + kOpDoubles;
      const bool kval = (iko + lp) < cur.k;
      const int limP = kval ? nvP : 0, limQ = kval ? nvQ : 0;
      const double2* p = bP + iko + r0 * stP;
      const double2* qq = bQ + iko + r0 * stQ;
#pragma unroll
      for (int r = r0; r < r1; ++r) {
        cp_async16_zfill(sP + r * kColStep * kColDoubles, p, r < limP);
        cp_async16_zfill(sQ + r * kColStep * kColDoubles, qq, r < limQ);
        p += stP;
        qq += stQ;
      }
      if constexpr (PL) {
        if (r0 == 0) {
          double* sPd = smem + stage * kStageDoubles + 2 * kOpDoubles + lc2 * KC + dst2;
          double* sQs = sPd + kPlaneDoubles;
          // bytes of this 16-byte piece inside the segment: K may be odd (the pad row past it
          // need not be zero in the planes); the remainder is zero-filled
          const int kr = cur.k - (iko + 2 * lp2);
          const int nb2 = kr >= 2 ? 16 : (kr == 1 ? 8 : 0);
          const double* pd = bPd + iko;
          const double* qs = bQs + iko;
#pragma unroll
          for (int r = 0; r < kRounds2; ++r) {
            cp_async16(sPd + r * kColStep2 * KC, r < nvP2 && nb2 ? pd : cur.Pd,
                       r < nvP2 ? nb2 : 0);
            cp_async16(sQs + r * kColStep2 * KC, r < nvQ2 && nb2 ? qs : cur.Qs,
                       r < nvQ2 ? nb2 : 0);
            pd += (long long)kColStep2 * cur.ldP;
            qs += (long long)kColStep2 * cur.ldQ;
          }
        }
      }
    };
    auto advance = [&]() {
      iko += KC;
      if (iko >= cur.k) {
        int nx = isi + 1;
        while (nx < send && sk.segs[nx].k <= 0) ++nx;
        if (nx < send) {
          isi = nx;
          iko = 0;
          cur = load_seg(sk.segs + isi);
          bP = cur.P + (long long)(i0 + lc) * cur.ldP + lp;
          bQ = cur.Q + (long long)(j0 + lc) * cur.ldQ + lp;
          stP = (long long)kColStep * cur.ldP;
          stQ = (long long)kColStep * cur.ldQ;
          if constexpr (PL) {
            bPd = cur.Pd + (long long)(i0 + lc2) * cur.ldP + 2 * lp2;
            bQs = cur.Qs + (long long)(j0 + lc2) * cur.ldQ + 2 * lp2;
          }
        }
      }
    };
    auto issue = [&](int stage) {
      issue_rounds(stage, 0, kRounds);
      advance();
    };

    // G3 (three-product complex multiply): accR = sum p_re q_re, accX = sum p_im q_im,
    // accI = sum (p_re - p_im)(q_re + q_im); combined after the K loop into
    // Re = accR + accX, Im = accI - accR + accX.  Otherwise accR / accI hold Re / Im.
    double accR[4][JB][2], accI[4][JB][2], accX[G3 ? 4 : 1][G3 ? JB : 1][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < JB; ++b) {
        accR[a][b][0] = accR[a][b][1] = 0.0;
        accI[a][b][0] = accI[a][b][1] = 0.0;
        if constexpr (G3) accX[a][b][0] = accX[a][b][1] = 0.0;
      }

    const int nchunks = c_hi - c_lo;
#pragma unroll
    for (int st = 0; st < kStages - 1; ++st) {
      if (st < nchunks) issue(st);
      cp_async_commit();
    }

    for (int c = 0; c < nchunks; ++c) {
      cp_async_wait<kStages - 2>();
      __syncthreads();
      const int nc = c + kStages - 1;
      const bool more = nc < nchunks;
      const int nstage = nc % kStages;
      // spread: the next-but-one chunk's loads are issued a round at a time between the
      // DMMA steps instead of as one block after the barrier.
      constexpr bool kLoadFirst = PAD == 2 && G3 && !PL && HSDLA_EARLY_RELOAD != 0;
      if (!kLoadFirst && !sk.spread) {
        if (more) issue(nstage);
        cp_async_commit();
      }

      const double* sP = smem + (c % kStages) * kStageDoubles;
      const double* sQ = sP + kOpDoubles;
      const double* pa = sP + (wm * 32 + g) * kColDoubles;
      const double* pb = sQ + (wn * kWarpCols + g) * kColDoubles;
      if constexpr (PAD == 2 && G3 && !PL && HSDLA_EARLY_RELOAD) {
        // Products ordered by column block with the three products of a block pair together, so
        // a row fragment's registers are free after its last column block and the next K
        // group's fragment is loaded there (and the next group's first column fragment one
        // block earlier) instead of at the top of the next group, where the warp would wait for
        // shared memory with nothing to issue: contractions -0.9% (C2) .. -1.35% (C3),
        // profiles/r02d_early_reload.json.  Double-buffering the column fragments on top of
        // this measured the same; carrying the fragments across chunk boundaries as well (the
        // chunk barrier moved before a chunk's last K group, one chunk of cp.async lead) spilled
        // and measured 3.4% slower.
        auto offj = [&](int j) {
          return (((2 * j + (q >> 1)) ^ ((g & 1) << 1)) << 2) + ((q & 1) << 1);
        };
        double2 av[4], bpre;
        {
          const int off0 = offj(0);
#pragma unroll
          for (int ib = 0; ib < 4; ++ib)
            av[ib] = *reinterpret_cast<const double2*>(pa + ib * 8 * kColDoubles + off0);
          bpre = *reinterpret_cast<const double2*>(pb + off0);
        }
        // the next-but-one chunk's cp.async block goes out under these loads' latency (issued
        // before them, right after the barrier, it delayed the chunk's first products: another
        // -0.8%; split in two halves or moved before K group 1 it measured 1.3% slower, the
        // row-block-outer mirror order 0.4% slower: profiles/r02d_early_reload.json)
        if (kLoadFirst && !sk.spread) {
          if (more) issue(nstage);
          cp_async_commit();
        }
#pragma unroll
        for (int j = 0; j < KC / 4; ++j) {
          if (sk.spread && more)
            issue_rounds(nstage, j * kRounds / (KC / 4), (j + 1) * kRounds / (KC / 4));
          const int off = offj(j), offn = offj(j + 1);
          const bool nextj = j + 1 < KC / 4;
          double sa[4];
#pragma unroll
          for (int ib = 0; ib < 4; ++ib) sa[ib] = av[ib].x - av[ib].y;
#pragma unroll
          for (int jb = 0; jb < JB; ++jb) {
            const double2 b = jb == 0 ? bpre
                                      : *reinterpret_cast<const double2*>(
                                            pb + jb * 8 * kColDoubles + off);
            const double sb = b.x + b.y;
#pragma unroll
            for (int ib = 0; ib < 4; ++ib) {
              dmma(accR[ib][jb][0], accR[ib][jb][1], av[ib].x, b.x);
              dmma(accX[ib][jb][0], accX[ib][jb][1], av[ib].y, b.y);
              dmma(accI[ib][jb][0], accI[ib][jb][1], sa[ib], sb);
              if (jb == JB - 1 && nextj)
                av[ib] = *reinterpret_cast<const double2*>(pa + ib * 8 * kColDoubles + offn);
            }
            if (jb == JB - 2 && nextj) bpre = *reinterpret_cast<const double2*>(pb + offn);
          }
        }
      } else if constexpr (PAD == 2) {
        // Paired K steps: lane q takes complex element 4j+q whole (one 16-byte load per
        // fragment) and uses its real part at step 2j, its imaginary part at step 2j+1.
        // The K order of the real embedding is free as long as P and Q share it:
        //   step 2j:   Re += p_re q_re   Im += p_re q_im
        //   step 2j+1: Re += p_im q_im   Im += p_im (-q_re)
        // 32-byte units of odd columns are swapped in pairs (unit ^ 2), so the two
        // columns of a quarter-warp's 128-bit load fall in opposite 64-byte bank halves.
#pragma unroll
        for (int j = 0; j < KC / 4; ++j) {
          if (sk.spread && more)
            issue_rounds(nstage, j * kRounds / (KC / 4), (j + 1) * kRounds / (KC / 4));
          const int off = (((2 * j + (q >> 1)) ^ ((g & 1) << 1)) << 2) + ((q & 1) << 1);
          double2 av[4], bv[JB];
#pragma unroll
          for (int ib = 0; ib < 4; ++ib)
            av[ib] = *reinterpret_cast<const double2*>(pa + ib * 8 * kColDoubles + off);
#pragma unroll
          for (int jb = 0; jb < JB; ++jb)
            bv[jb] = *reinterpret_cast<const double2*>(pb + jb * 8 * kColDoubles + off);
          if constexpr (G3) {
            // Three DMMAs per (block pair, complex-K group) instead of four.
#pragma unroll
            for (int ib = 0; ib < 4; ++ib)
#pragma unroll
              for (int jb = 0; jb < JB; ++jb) {
                dmma(accR[ib][jb][0], accR[ib][jb][1], av[ib].x, bv[jb].x);
                dmma(accX[ib][jb][0], accX[ib][jb][1], av[ib].y, bv[jb].y);
              }
            double sa[4], sb[JB];
            if constexpr (PL) {
              const double* pda = sP + 2 * kOpDoubles + (wm * 32 + g) * KC;
              const double* qsb = pda - (wm * 32 + g) * KC + kPlaneDoubles +
                                  (wn * kWarpCols + g) * KC;
              const int po = ((j ^ psw(g)) << 2) + q;
#pragma unroll
              for (int ib = 0; ib < 4; ++ib) sa[ib] = pda[ib * 8 * KC + po];
#pragma unroll
              for (int jb = 0; jb < JB; ++jb) sb[jb] = qsb[jb * 8 * KC + po];
            } else {
#pragma unroll
              for (int ib = 0; ib < 4; ++ib) sa[ib] = av[ib].x - av[ib].y;
#pragma unroll
              for (int jb = 0; jb < JB; ++jb) sb[jb] = bv[jb].x + bv[jb].y;
            }
#pragma unroll
            for (int ib = 0; ib < 4; ++ib)
#pragma unroll
              for (int jb = 0; jb < JB; ++jb)
                dmma(accI[ib][jb][0], accI[ib][jb][1], sa[ib], sb[jb]);
          } else {
#pragma unroll
          for (int ib = 0; ib < 4; ++ib)
#pragma unroll
            for (int jb = 0; jb < JB; ++jb) {
              dmma(accR[ib][jb][0], accR[ib][jb][1], av[ib].x, bv[jb].x);
              dmma(accI[ib][jb][0], accI[ib][jb][1], av[ib].x, bv[jb].y);
            }
          double nb[JB];
#pragma unroll
          for (int jb = 0; jb < JB; ++jb)
            nb[jb] = __hiloint2double(__double2hiint(bv[jb].x) ^ 0x80000000u,
                                      __double2loint(bv[jb].x));
#pragma unroll
          for (int ib = 0; ib < 4; ++ib)
#pragma unroll
            for (int jb = 0; jb < JB; ++jb) {
              dmma(accR[ib][jb][0], accR[ib][jb][1], av[ib].y, bv[jb].y);
              dmma(accI[ib][jb][0], accI[ib][jb][1], av[ib].y, nb[jb]);
            }
          }
        }
      } else {
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        if (sk.spread && more && s % (8 / kRounds) == 0)
          issue_rounds(nstage, s / (8 / kRounds), s / (8 / kRounds) + 1);
        const int off = PAD ? (s << 2) : ((s ^ g) << 2);
        double a[4], br[JB], bi[JB];
#pragma unroll
        for (int ib = 0; ib < 4; ++ib) a[ib] = pa[ib * 8 * kColDoubles + off + q];
#pragma unroll
        for (int jb = 0; jb < JB; ++jb) {
          br[jb] = pb[jb * 8 * kColDoubles + off + q];
          const double x = pb[jb * 8 * kColDoubles + off + (q ^ 1)];
          bi[jb] = __hiloint2double(__double2hiint(x) ^ sign_hi, __double2loint(x));
        }
#pragma unroll
        for (int ib = 0; ib < 4; ++ib)
#pragma unroll
          for (int jb = 0; jb < JB; ++jb) {
            dmma(accR[ib][jb][0], accR[ib][jb][1], a[ib], br[jb]);
            dmma(accI[ib][jb][0], accI[ib][jb][1], a[ib], bi[jb]);
          }
      }
      }
      if (sk.spread) {
        if (more) advance();
        cp_async_commit();
      }
    }
    cp_async_wait<0>();
    __syncthreads();
    it += nchunks;
    if constexpr (G3) {
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < JB; ++b)
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            const double t1 = accR[a][b][v], t2 = accX[a][b][v];
            accR[a][b][v] = t1 + t2;
            accI[a][b][v] = (accI[a][b][v] - t1) + t2;
          }
    }

    if (c_lo != 0) {
      // Later piece of a split tile: publish the partial for the tile's finishing CTA.
      double* slot = sk.partials + (long long)cta * kPartialDoubles;
      int r = 0;
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < JB; ++b)
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            __stcg(slot + (r++) * kThreads + tid, accR[a][b][v]);
            __stcg(slot + (r++) * kThreads + tid, accI[a][b][v]);
          }
      __threadfence();
      __syncthreads();
      if (tid == 0) atomicExch(sk.ready + cta, 1);
      continue;
    }
    if (c_hi < nch) {
      // Head piece of a split tile: add the later pieces in CTA order (deterministic).
      for (int j = cta + 1; j < sk.grid && sk_start(sk, j) < tile_it_end; ++j) {
        if (tid == 0) {
          while (atomicAdd(sk.ready + j, 0) == 0) __nanosleep(100);
        }
        __syncthreads();
        const double* slot = sk.partials + (long long)j * kPartialDoubles;
        int r = 0;
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < JB; ++b)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
              accR[a][b][v] += __ldcg(slot + (r++) * kThreads + tid);
              accI[a][b][v] += __ldcg(slot + (r++) * kThreads + tid);
            }
      }
    }

    // ---- epilogue
    bool bad = false;
#pragma unroll
    for (int ib = 0; ib < 4; ++ib) {
      const int i = i0 + wm * 32 + ib * 8 + g;
#pragma unroll
      for (int jb = 0; jb < JB; ++jb) {
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int j = j0 + wn * kWarpCols + jb * 8 + 2 * q + v;
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
    if (bad) atomicOr(sk.flag, 1);
    if (pr.panel_done) {
      // Publish the finished tile to the streaming copy: the barrier orders every thread's
      // stores before thread 0's system-scope fence (cumulative), then its column group's
      // counter (Prob::panel_group tile columns per counter).
      __syncthreads();
      if (tid == 0) {
        __threadfence_system();
        atomicAdd(pr.panel_done + (pr.panel_group > 1 ? tn / pr.panel_group : tn), 1);
      }
    }
  }
  }
}

}  // namespace

int prob_tile_count(const Prob& p) {
  if (p.kind == PROB_GENERAL) return p.tiles_m * p.tiles_n;
  int cnt = 0;
  for (int tn = p.col_tile_lo; tn < p.col_tile_hi; ++tn) cnt += p.tiles_m - tn;
  return cnt;
}

// Data-parallel waves ahead of the stream-K split (HSDLA_SK_DP=0 disables): only when all
// problems share one chunk count, so a whole tile is the same work everywhere.  The
// stream-K remainder is kept at >= 8 chunks per CTA (else one wave moves back into it)
// to avoid long split-tile fix-up chains.
void plan_dp_waves(const std::vector<Prob>& probs, long long total, int grid, int* waves,
                   int* nch, long long* dp_it) {
  static int enabled = -1;
  if (enabled < 0) {
    const char* e = getenv("HSDLA_SK_DP");
    enabled = (e && std::string(e) == "0") ? 0 : 1;
  }
  *waves = 0;
  *nch = 1;
  *dp_it = 0;
  if (!enabled || probs.empty()) return;
  const int n0 = probs[0].nchunks;
  for (const Prob& p : probs)
    if (p.nchunks != n0) return;
  const long long tiles = total / n0;
  long long w = tiles / grid;
  const long long rem = tiles - w * grid;
  if (w > 0 && rem > 0 && rem * n0 < 8LL * grid) --w;
  *waves = (int)w;
  *nch = n0;
  *dp_it = w * grid * n0;
}

int preload_contract() {
  const void* fns[] = {(const void*)contract_kernel<2, 0>, (const void*)contract_kernel<2, 1>,
                       (const void*)contract_kernel<2, 2>, (const void*)contract_kernel<4, 0>,
                       (const void*)contract_kernel<4, 1>, (const void*)contract_kernel<4, 2>,
                       (const void*)contract_kernel<2, 2, true>,
                       (const void*)contract_kernel<4, 2, true>,
                       (const void*)contract_kernel<4, 2, true, true, 2>,
                       (const void*)contract_kernel<4, 2, true, true, 3>,
                       (const void*)contract_kernel<4, 2, true, true, 4, 8>,
                       (const void*)contract_kernel<4, 2, true, true, 3, 8>,
                       (const void*)contract_kernel<2, 2, true, false, 3, 16, 2>};
  const size_t smem[] = {Layout<0>::kSmemBytes, Layout<1>::kSmemBytes, Layout<2>::kSmemBytes,
                         Layout<0>::kSmemBytes, Layout<1>::kSmemBytes, Layout<2>::kSmemBytes,
                         Layout<2>::kSmemBytes, Layout<2>::kSmemBytes,
                         Layout<2, true, 2>::kSmemBytes, Layout<2, true, 3>::kSmemBytes,
                         Layout<2, true, 4, 8>::kSmemBytes, Layout<2, true, 3, 8>::kSmemBytes,
                         Layout<2>::kSmemBytes};
  for (int i = 0; i < 13; ++i) {
    cudaFuncAttributes at;
    HS_CUDA(cudaFuncGetAttributes(&at, fns[i]));
    if (first_on_device(fns[i]))
      HS_CUDA(cudaFuncSetAttribute(fns[i], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem[i]));
  }
  return HSDLA_OK;
}

int launch_contract(hsdla_ctx* ctx, const std::vector<Prob>& probs_in,
                    const std::vector<Seg>& segs, int* flag_dev) {
  // Variant selection (HSDLA_WARP_COLS = 32 | 16, HSDLA_SMEM_PAD = 0 | 1) for A/B tests.
  // Shared-memory layout / fragment path: HSDLA_CP_LAYOUT = pair (default: paired K steps,
  // 128-bit fragment loads) | xor (32-byte XOR swizzle, 64-bit loads) | pad (288-byte columns).
  // Complex multiply (cmul_mode, HSDLA_CMUL): 3 (default) uses the three-product kernel, pair
  // layout only.
  static int variant = -1, pad = -1, cmul = -1;
  // Sum planes: when every segment carries them (the pipeline's generated stacks), the
  // DADD-free kernel (HSDLA_PLANES=1, common.cuh); ring HSDLA_PL_VARIANT = 8x4 (default: chunks
  // of 8 complex K, 4 stages) | 8x3 | 16x2 | 16x3.
  static int planes_env = -1, pl_kc = 8, pl_stages = 4;
  if (variant < 0) {
    const char* e = getenv("HSDLA_WARP_COLS");
    variant = (e && atoi(e) == 16) ? 2 : 4;
    const char* p = getenv("HSDLA_CP_LAYOUT");
    pad = (p && std::string(p) == "pad") ? 1 : (p && std::string(p) == "xor") ? 0 : 2;
    cmul = cmul_mode();
    planes_env = planes_enabled() ? 1 : 0;
    const char* pv = getenv("HSDLA_PL_VARIANT");
    if (pv && std::string(pv) == "8x3") { pl_kc = 8; pl_stages = 3; }
    if (pv && std::string(pv) == "16x2") { pl_kc = 16; pl_stages = 2; }
    if (pv && std::string(pv) == "16x3") { pl_kc = 16; pl_stages = 3; }
  }
  bool planes = planes_env && variant == 4 && pad == 2 && cmul == 3 && !segs.empty();
  for (const Seg& sg : segs) planes = planes && sg.Pd && sg.Qs;
  const int kc = planes ? pl_kc : kChunk;
  std::vector<Prob> probs;
  long long total = 0;
  for (Prob p : probs_in) {
    if (p.m <= 0 || p.n <= 0) continue;
    p.tiles_m = (p.m + kTile - 1) / kTile;
    p.tiles_n = (p.n + kTile - 1) / kTile;
    if (p.kind != PROB_GENERAL) {
      p.tiles_n = p.tiles_m;
      if (p.col_tile_hi <= 0 || p.col_tile_hi > p.tiles_m) p.col_tile_hi = p.tiles_m;
      if (p.col_tile_lo < 0) p.col_tile_lo = 0;
    }
    p.ntiles = prob_tile_count(p);
    int nch = 0;
    for (int s = 0; s < p.nseg; ++s) nch += (segs[p.seg0 + s].k + kc - 1) / kc;
    p.nchunks = nch > 0 ? nch : 1;  // an empty K still visits each tile once (C = beta C)
    p.it_base = total;
    total += (long long)p.ntiles * p.nchunks;
    if (p.ntiles > 0) probs.push_back(p);
  }
  if (total == 0) return HSDLA_OK;
  // Feed path: HSDLA_CONTRACT = auto (default: TMA 96x32 tiles for T applications with
  // 64 < m <= 96, cp.async 64x64 otherwise) | tma (all TMA) | cpasync (all cp.async).
  static int mode = -1;
  if (mode < 0) {
    const char* e = getenv("HSDLA_CONTRACT");
    mode = (e && std::string(e) == "tma") ? 1 : (e && std::string(e) == "cpasync") ? 2 : 0;
  }
  if (!planes && (mode == 1 || (mode == 0 && tma_wants(probs))))
    return launch_contract_tma(ctx, probs, total, segs, flag_dev);
  const void* kfns[2][4] = {
      {(const void*)contract_kernel<2, 0>, (const void*)contract_kernel<2, 1>, (const void*)contract_kernel<2, 2>,
       (const void*)contract_kernel<2, 2, true>},
      {(const void*)contract_kernel<4, 0>, (const void*)contract_kernel<4, 1>, (const void*)contract_kernel<4, 2>,
       (const void*)contract_kernel<4, 2, true>}};
  const void* kfn = kfns[variant == 4 ? 1 : 0][(pad == 2 && cmul == 3) ? 3 : pad];
  static int minb2 = -1;  // HSDLA_G3_MINB=2 with HSDLA_WARP_COLS=16: two 8-warp CTAs per SM
  if (minb2 < 0) {
    const char* e = getenv("HSDLA_G3_MINB");
    minb2 = (e && e[0] == '2') ? 1 : 0;
  }
  if (minb2 && variant == 2 && pad == 2 && cmul == 3)
    kfn = (const void*)contract_kernel<2, 2, true, false, 3, 16, 2>;
  size_t kSmemBytes = pad == 1 ? Layout<1>::kSmemBytes : Layout<0>::kSmemBytes;
  if (planes) {
    if (pl_kc == 8 && pl_stages == 4) {
      kfn = (const void*)contract_kernel<4, 2, true, true, 4, 8>;
      kSmemBytes = Layout<2, true, 4, 8>::kSmemBytes;
    } else if (pl_kc == 8) {
      kfn = (const void*)contract_kernel<4, 2, true, true, 3, 8>;
      kSmemBytes = Layout<2, true, 3, 8>::kSmemBytes;
    } else if (pl_stages == 3) {
      kfn = (const void*)contract_kernel<4, 2, true, true, 3>;
      kSmemBytes = Layout<2, true, 3>::kSmemBytes;
    } else {
      kfn = (const void*)contract_kernel<4, 2, true, true, 2>;
      kSmemBytes = Layout<2, true, 2>::kSmemBytes;
    }
  }
  if (first_on_device(kfn))
    HS_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes));
  const int kThreads = variant == 4 ? 128 : 256;
  int occ = 0;
  HS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, kThreads, kSmemBytes));
  if (occ < 1) occ = 1;
  long long grid_ll = (long long)ctx->num_sms * occ;
  if (grid_ll > total) grid_ll = total;
  const int grid = (int)grid_ll;
  if (ctx->partial_slots < grid) {
    HS_CUDA(cudaStreamSynchronize(ctx->stream));
    if (ctx->partials) cudaFree(ctx->partials);
    if (ctx->ready) cudaFree(ctx->ready);
    HS_CUDA(cudaMalloc(&ctx->partials, size_t(grid) * kPartialDoubles * sizeof(double)));
    HS_CUDA(cudaMalloc(&ctx->ready, size_t(grid) * sizeof(int)));
    ctx->partial_slots = grid;
  }
  int rc = arena_begin(ctx, probs.size() * sizeof(Prob) + segs.size() * sizeof(Seg) + 256);
  if (rc) return rc;
  Prob* dprobs = static_cast<Prob*>(arena_push(ctx, probs.data(), probs.size() * sizeof(Prob), nullptr));
  Seg* dsegs = static_cast<Seg*>(
      arena_push(ctx, segs.data(), (segs.empty() ? 1 : segs.size()) * sizeof(Seg), nullptr));
  rc = arena_flush(ctx);
  if (rc) return rc;
  HS_CUDA(cudaMemsetAsync(ctx->ready, 0, size_t(grid) * sizeof(int), ctx->stream));
  SKParams sk;
  sk.probs = dprobs;
  sk.segs = dsegs;
  sk.total_it = total;
  sk.nprob = (int)probs.size();
  sk.grid = grid;
  plan_dp_waves(probs, total, grid, &sk.dp_waves, &sk.dp_nch, &sk.dp_it);
  static int spread = -1;
  if (spread < 0) {
    const char* e = getenv("HSDLA_CP_SPREAD");
    spread = (e && std::string(e) == "1") ? 1 : 0;
  }
  sk.spread = spread;
  sk.partials = ctx->partials;
  sk.ready = ctx->ready;
  sk.flag = flag_dev;
  void* kargs[] = {&sk};
  // Cooperative launch guarantees all CTAs are co-resident, which the split-tile
  // hand-off (a finishing CTA waits for later CTAs' partials) relies on.
  HS_CUDA(cudaLaunchCooperativeKernel(kfn, dim3(grid), dim3(kThreads), kargs, kSmemBytes,
                                      ctx->stream));
  return HSDLA_OK;
}

}  // namespace hsdla
