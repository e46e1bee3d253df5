// TMA-fed variant of the multi-segment DMMA contraction (sm_100a).
//
// Same math, tiles, stream-K work split and epilogue as contract.cu (see there), but the
// operand K-chunks arrive by TMA (cp.async.bulk.tensor, 128-byte swizzle) into a 3-stage
// ring guarded by mbarriers instead of per-thread cp.async + __syncthreads:
//   * one elected thread (warp 0, lane 0) is the producer: it issues the four box loads of
//     chunk j+2 (P/Q x two 16-double k halves, 8 KB each) while chunk j is consumed, across
//     tile and segment boundaries of the CTA's stream-K range;
//   * consumer warps wait on the stage's `full` barrier (transaction-count completion) and
//     release it through its `empty` barrier — no CTA-wide barrier per chunk, so one slow
//     warp no longer stalls the others, and the DMMA warps execute no load-issue code.
// Each operand of each segment is a 2-D tensor map over doubles: dim0 = 2k (the segment's
// K extent, so K tails read as zeros), dim1 = columns (tile edges read as zeros).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>

#include <stdlib.h>

#include <algorithm>
#include <map>
#include <tuple>

#include "common.cuh"

namespace hsdla {
namespace {

constexpr int kStg = 3;

// Tile configuration: WM x WN warps, each 32 rows x 8*JB columns (complex); the output
// tile is TM x TN.  Cfg<2,2,4> = 64x64 (4 warps, ~250 registers, every triangular problem);
// Cfg<3,2,2> = 96x32 (6 warps, ~128 registers) for the T applications when 64 < m <= 96
// (m = 81 at l_sph = 8: 84% of the rows useful instead of 63% with 64-row tiles).
template <int WM_, int WN_, int JB_, bool PAIR_ = false, bool G3_ = false>
struct Cfg {
  static constexpr int WM = WM_, WN = WN_, JB = JB_;
  static constexpr bool PAIR = PAIR_;
  static constexpr bool G3 = G3_;  // three-product complex multiply (PAIR only), see contract.cu
  static constexpr int TM = 32 * WM, TN = 8 * JB * WN;
  static constexpr int kT = 32 * WM * WN;
  static constexpr int kPBox = TM * 128, kQBox = TN * 128;  // box = columns x 16 doubles
  static constexpr int kStageBytes = 2 * (kPBox + kQBox);
  static constexpr size_t kSmemBytes = size_t(kStg) * kStageBytes + 1024 + 128;
  static constexpr int kPartial = TM * TN * 2;
};
using Cfg64 = Cfg<2, 2, 4>;
using Cfg96 = Cfg<3, 2, 2>;
// PAIR: 128-bit fragment loads (lane q takes complex element 4j+q whole; real part at DMMA
// step 2j, imaginary part at 2j+1, as contract.cu's "pair" layout).  Under the TMA 128-byte
// swizzle (16-B unit u of row c at u ^ (c & 7)) the two rows of a quarter-warp must differ
// in bit 2 of (c & 7), so fragment row g reads tile column pi(g) = (g >> 1) | ((g & 1) << 2)
// inside each 8-column block; the epilogue maps rows and columns through pi.
using Cfg64P = Cfg<2, 2, 4, true>;
using Cfg96P = Cfg<3, 2, 2, true>;
using Cfg64G = Cfg<2, 2, 4, true, true>;
using Cfg96G = Cfg<3, 2, 2, true, true>;
// 64x64 with eight 32x16 warps (three-product): 128 registers, two CTAs / 16 warps per SM.
using Cfg64G8 = Cfg<2, 4, 2, true, true>;
__device__ __forceinline__ int pair_perm(int g) { return (g >> 1) | ((g & 1) << 2); }

struct TSeg {
  int mapP, mapPalt, mapQ;
  int k;
  const int* sel;
};

struct TKParams {
  const Prob* probs;
  const TSeg* segs;
  const CUtensorMap* maps;
  long long total_it;
  int nprob;
  int grid;
  double* partials;
  int* ready;
  int* flag;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)),
               "r"(bytes));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(b)));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity));
}
__device__ __forceinline__ bool mbar_test(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(parity));
  return ok != 0;
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, "
      "{%2, %3}], [%4];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ long long range_start(long long total, int grid, int g) {
  return total * g / grid;
}

__device__ __forceinline__ int locate_prob(const TKParams& sk, long long it) {
  int lo = 0, hi = sk.nprob - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (sk.probs[mid].it_base <= it) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ void tile_coords(const Prob& pr, int tile, int& tm, int& tn) {
  if (pr.kind == PROB_GENERAL) {
    tm = tile % pr.tiles_m;
    tn = tile / pr.tiles_m;
  } else {
    const int nb = pr.tiles_m;
    tn = pr.col_tile_lo;
    while (tile >= nb - tn) { tile -= nb - tn; ++tn; }
    tm = tn + tile;
  }
}

// Producer-side walk over the CTA's (tile, chunk) sequence: the segment and K offset of
// the next chunk to load.  Lives in one thread.
struct ProdIter {
  long long it, it_end;
  int p, tile, c, nch, i0, j0, seg, send, kofs;

  template <class C>
  __device__ void seek(const TKParams& sk, long long it0, long long it1) {
    it = it0;
    it_end = it1;
    if (it >= it_end) return;
    p = locate_prob(sk, it);
    const Prob& pr = sk.probs[p];
    nch = pr.nchunks;
    const long long local = it - pr.it_base;
    tile = (int)(local / nch);
    c = (int)(local - (long long)tile * nch);
    set_tile<C>(sk);
    // walk segments to chunk c
    int cb = 0;
    for (; seg < send; ++seg) {
      const int ncs = (sk.segs[seg].k + 15) / 16;
      if (c < cb + ncs) { kofs = (c - cb) * 16; return; }
      cb += ncs;
    }
    seg = pr.seg0;  // empty K: one chunk reading out of bounds (zeros)
    kofs = 1 << 24;
  }
  template <class C>
  __device__ void set_tile(const TKParams& sk) {
    const Prob& pr = sk.probs[p];
    int tm, tn;
    tile_coords(pr, tile, tm, tn);
    i0 = tm * C::TM;
    j0 = tn * C::TN;
    seg = pr.seg0;
    send = pr.seg0 + pr.nseg;
    kofs = 0;
  }
  __device__ void first_nonempty(const TKParams& sk) {
    const int s0 = seg;
    while (seg < send && sk.segs[seg].k <= 0) ++seg;
    if (seg >= send) { seg = s0; kofs = 1 << 24; }
  }
  template <class C>
  __device__ void next(const TKParams& sk) {
    ++it;
    if (it >= it_end) return;
    ++c;
    if (c == nch) {
      c = 0;
      ++tile;
      if (tile == sk.probs[p].ntiles) {
        ++p;
        tile = 0;
        nch = sk.probs[p].nchunks;
      }
      set_tile<C>(sk);
      first_nonempty(sk);
      return;
    }
    kofs += 16;
    if (kofs >= sk.segs[seg].k) {
      int nx = seg + 1;
      while (nx < send && sk.segs[nx].k <= 0) ++nx;
      if (nx < send) { seg = nx; kofs = 0; }
    }
  }
  template <class C>
  __device__ void issue(const TKParams& sk, char* stage, uint64_t* full) {
    const TSeg s = sk.segs[seg];
    const int mp = (s.sel && *s.sel != 0) ? s.mapPalt : s.mapP;
    const CUtensorMap* mP = sk.maps + mp;
    const CUtensorMap* mQ = sk.maps + s.mapQ;
    const int kd = 2 * kofs;
    mbar_expect_tx(full, C::kStageBytes);
    tma_load_2d(stage, mP, kd, i0, full);
    tma_load_2d(stage + C::kPBox, mP, kd + 16, i0, full);
    tma_load_2d(stage + 2 * C::kPBox, mQ, kd, j0, full);
    tma_load_2d(stage + 2 * C::kPBox + C::kQBox, mQ, kd + 16, j0, full);
  }
};

__device__ __forceinline__ bool finite2(double2 v) { return isfinite(v.x) && isfinite(v.y); }

template <class C>
__global__ void __launch_bounds__(C::kT, 2) contract_tma_kernel(TKParams sk) {
  constexpr int kT = C::kT, JB = C::JB, kStageBytes = C::kStageBytes, kPartial = C::kPartial;
  extern __shared__ __align__(1024) char smem_raw[];
  // 1024-byte alignment for the 128B-swizzled TMA boxes; indexing the shared array keeps
  // the shared address space visible to the compiler (LDS, not generic loads).
  char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStg * kStageBytes);
  uint64_t* empty = full + kStg;

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int wm = warp % C::WM, wn = warp / C::WM;
  const int g = lane >> 2, q = lane & 3;
  const unsigned sign_hi = (q & 1) ? 0x80000000u : 0u;
  // K order inside a chunk is free (P and Q use the same one): in k'-step s4 of a 16-double
  // box, lane q reads double 2*s4 + (q&1) + 8*(q>>1), so a half-warp touches 16 distinct
  // bank pairs under the TMA 128B swizzle (16-B unit u of row c stored at u ^ (c & 7)).
  // The re/im partner (double ^ 1) stays in the same 16-B unit: byte offset ^ 8.
  const int fo = (((4 * (q >> 1)) ^ g) << 4) | ((q & 1) << 3);

  const int cta = blockIdx.x;
  const long long it0 = range_start(sk.total_it, sk.grid, cta);
  const long long it_end = range_start(sk.total_it, sk.grid, cta + 1);
  const long long nchunks_cta = it_end - it0;

  if (tid == 0) {
    for (int s = 0; s < kStg; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, C::WM * C::WN);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  }
  __syncthreads();

  ProdIter pi;
  if (tid == 0) {
    pi.seek<C>(sk, it0, it_end);
    for (int s = 0; s < kStg - 1 && s < nchunks_cta; ++s) {
      pi.issue<C>(sk, smem + s * kStageBytes, full + s);
      pi.next<C>(sk);
    }
  }

  long long j = 0;  // chunks consumed by this CTA
  long long it = it0;
  while (it < it_end) {
    const int pidx = locate_prob(sk, it);
    const Prob pr = sk.probs[pidx];
    const long long local = it - pr.it_base;
    const int nch = pr.nchunks;
    int tile = (int)(local / nch);
    const int c_lo = (int)(local - (long long)tile * nch);
    const long long left = it_end - it;
    const int c_hi = (left < (long long)(nch - c_lo)) ? c_lo + (int)left : nch;
    const long long tile_it_end = pr.it_base + (long long)(tile + 1) * nch;
    int tm, tn;
    tile_coords(pr, tile, tm, tn);
    const int i0 = tm * C::TM, j0 = tn * C::TN;

    // G3: accR = sum p_re q_re, accX = sum p_im q_im, accI = sum (p_re - p_im)(q_re + q_im),
    // combined after the K loop (Re = accR + accX, Im = accI - accR + accX).
    double accR[4][JB][2], accI[4][JB][2], accX[C::G3 ? 4 : 1][C::G3 ? JB : 1][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < JB; ++b) {
        accR[a][b][0] = accR[a][b][1] = 0.0;
        accI[a][b][0] = accI[a][b][1] = 0.0;
        if constexpr (C::G3) accX[a][b][0] = accX[a][b][1] = 0.0;
      }

    for (int cc = c_lo; cc < c_hi; ++cc, ++j) {
      const int st = (int)(j % kStg);
      mbar_wait(full + st, (uint32_t)((j / kStg) & 1));
      if constexpr (C::PAIR) {
        const int pg = pair_perm(g);
        const char* sP = smem + st * kStageBytes + (wm * 32 + pg) * 128;
        const char* sQ = smem + st * kStageBytes + 2 * C::kPBox + (wn * 8 * JB + pg) * 128;
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const int off = ((((jj & 1) << 2) + q) ^ pg) << 4;
          const char* pA = sP + (jj >> 1) * C::kPBox + off;
          const char* pB = sQ + (jj >> 1) * C::kQBox + off;
          double2 av[4], bv[JB];
#pragma unroll
          for (int ib = 0; ib < 4; ++ib) av[ib] = *reinterpret_cast<const double2*>(pA + ib * 8 * 128);
#pragma unroll
          for (int jb = 0; jb < JB; ++jb) bv[jb] = *reinterpret_cast<const double2*>(pB + jb * 8 * 128);
          if constexpr (C::G3) {
#pragma unroll
            for (int ib = 0; ib < 4; ++ib)
#pragma unroll
              for (int jb = 0; jb < JB; ++jb) {
                dmma(accR[ib][jb][0], accR[ib][jb][1], av[ib].x, bv[jb].x);
                dmma(accX[ib][jb][0], accX[ib][jb][1], av[ib].y, bv[jb].y);
              }
            double sa[4], sb[JB];
#pragma unroll
            for (int ib = 0; ib < 4; ++ib) sa[ib] = av[ib].x - av[ib].y;
#pragma unroll
            for (int jb = 0; jb < JB; ++jb) sb[jb] = bv[jb].x + bv[jb].y;
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
            nb[jb] = __hiloint2double(__double2hiint(bv[jb].x) ^ 0x80000000u, __double2loint(bv[jb].x));
#pragma unroll
          for (int ib = 0; ib < 4; ++ib)
#pragma unroll
            for (int jb = 0; jb < JB; ++jb) {
              dmma(accR[ib][jb][0], accR[ib][jb][1], av[ib].y, bv[jb].y);
              dmma(accI[ib][jb][0], accI[ib][jb][1], av[ib].y, nb[jb]);
            }
          }
          if (jj == 1 && tid == 0) {
            const long long x = j + kStg - 1;
            if (x < nchunks_cta) {
              const int sx = (int)(x % kStg);
              if (x >= kStg) mbar_wait(empty + sx, (uint32_t)(((x / kStg) - 1) & 1));
              pi.issue<C>(sk, smem + sx * kStageBytes, full + sx);
              pi.next<C>(sk);
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + st);
        continue;
      }
      const char* sP = smem + st * kStageBytes + (wm * 32 + g) * 128;
      const char* sQ = smem + st * kStageBytes + 2 * C::kPBox + (wn * 8 * JB + g) * 128;
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const int off = fo ^ ((s & 3) << 4);
        const char* pA = sP + (s >> 2) * C::kPBox;
        const char* pB = sQ + (s >> 2) * C::kQBox;
        double a[4], br[JB], bi[JB];
#pragma unroll
        for (int ib = 0; ib < 4; ++ib)
          a[ib] = *reinterpret_cast<const double*>(pA + ib * 8 * 128 + off);
#pragma unroll
        for (int jb = 0; jb < JB; ++jb) {
          br[jb] = *reinterpret_cast<const double*>(pB + jb * 8 * 128 + off);
          const double x = *reinterpret_cast<const double*>(pB + jb * 8 * 128 + (off ^ 8));
          bi[jb] = __hiloint2double(__double2hiint(x) ^ sign_hi, __double2loint(x));
        }
#pragma unroll
        for (int ib = 0; ib < 4; ++ib)
#pragma unroll
          for (int jb = 0; jb < JB; ++jb) {
            dmma(accR[ib][jb][0], accR[ib][jb][1], a[ib], br[jb]);
            dmma(accI[ib][jb][0], accI[ib][jb][1], a[ib], bi[jb]);
          }
        if (s == 3 && tid == 0) {
          // Producer, mid-chunk: by now the other warps have released chunk j-1 (whose stage
          // chunk j+2 reuses), so the empty-barrier wait rarely blocks this warp.
          const long long x = j + kStg - 1;
          if (x < nchunks_cta) {
            const int sx = (int)(x % kStg);
            if (x >= kStg) mbar_wait(empty + sx, (uint32_t)(((x / kStg) - 1) & 1));
            pi.issue<C>(sk, smem + sx * kStageBytes, full + sx);
            pi.next<C>(sk);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + st);
    }
    it += c_hi - c_lo;
    if constexpr (C::G3) {
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
      double* slot = sk.partials + (long long)cta * kPartial;
      int r = 0;
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < JB; ++b)
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            __stcg(slot + (r++) * kT + tid, accR[a][b][v]);
            __stcg(slot + (r++) * kT + tid, accI[a][b][v]);
          }
      __threadfence();
      __syncthreads();
      if (tid == 0) atomicExch(sk.ready + cta, 1);
      continue;
    }
    if (c_hi < nch) {
      for (int jj = cta + 1; jj < sk.grid && range_start(sk.total_it, sk.grid, jj) < tile_it_end; ++jj) {
        if (tid == 0) {
          while (atomicAdd(sk.ready + jj, 0) == 0) __nanosleep(100);
        }
        __syncthreads();
        const double* slot = sk.partials + (long long)jj * kPartial;
        int r = 0;
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < JB; ++b)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
              accR[a][b][v] += __ldcg(slot + (r++) * kT + tid);
              accI[a][b][v] += __ldcg(slot + (r++) * kT + tid);
            }
      }
    }

    bool bad = false;
#pragma unroll
    for (int ib = 0; ib < 4; ++ib) {
      const int i = i0 + wm * 32 + ib * 8 + (C::PAIR ? pair_perm(g) : g);
#pragma unroll
      for (int jb = 0; jb < JB; ++jb) {
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int jcol = j0 + wn * 8 * JB + jb * 8 + (C::PAIR ? pair_perm(2 * q + v) : 2 * q + v);
          double2 val = make_double2(accR[ib][jb][v], accI[ib][jb][v]);
          if (pr.kind == PROB_GENERAL) {
            if (i < pr.m && jcol < pr.n) {
              double2* cp = pr.C + i + (long long)jcol * pr.ldC;
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
          } else if (i < pr.n && jcol < pr.n && i >= jcol) {
            double2* cl = pr.C + i + (long long)jcol * pr.ldC;
            if (pr.accumulate) {
              const double2 old = *cl;
              val.x += old.x;
              val.y += old.y;
            }
            if (pr.kind == PROB_TRI_MIRROR) {
              if (i == jcol) val.y = 0.0;
              bad |= !finite2(val);
              if (i > jcol) pr.C[jcol + (long long)i * pr.ldC] = make_double2(val.x, -val.y);
            }
            *cl = val;
          }
        }
      }
    }
    if (bad) atomicOr(sk.flag, 1);
    if (pr.panel_done) {  // streamed copy-out, see Prob::panel_done and contract.cu
      __syncthreads();
      if (tid == 0) {
        __threadfence_system();
        atomicAdd(pr.panel_done + (pr.panel_group > 1 ? tn / pr.panel_group : tn), 1);
      }
    }
  }
}

PFN_cuTensorMapEncodeTiled_v12000 get_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

}  // namespace

namespace {
template <class C>
int launch_cfg(hsdla_ctx* ctx, const std::vector<Prob>& probs_in, const std::vector<Seg>& segs,
               int* flag_dev) {
  auto encode = get_encoder();
  if (!encode) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return HSDLA_ERR_UNSUPPORTED;
  }
  // Stream-K iteration space with this configuration's tile shape.
  std::vector<Prob> probs;
  long long total = 0;
  for (Prob p : probs_in) {
    if (p.m <= 0 || p.n <= 0) continue;
    p.tiles_m = (p.m + C::TM - 1) / C::TM;
    p.tiles_n = (p.n + C::TN - 1) / C::TN;
    if (p.kind != PROB_GENERAL) {
      if (C::TM != C::TN) {
        set_error("triangular problems need square tiles");
        return HSDLA_ERR_UNSUPPORTED;
      }
      p.tiles_n = p.tiles_m;
      if (p.col_tile_hi <= 0 || p.col_tile_hi > p.tiles_m) p.col_tile_hi = p.tiles_m;
      if (p.col_tile_lo < 0) p.col_tile_lo = 0;
    }
    p.ntiles = prob_tile_count(p);
    int nch = 0;
    for (int s = 0; s < p.nseg; ++s) nch += (segs[p.seg0 + s].k + 15) / 16;
    p.nchunks = nch > 0 ? nch : 1;
    p.it_base = total;
    total += (long long)p.ntiles * p.nchunks;
    if (p.ntiles > 0) probs.push_back(p);
  }
  if (total == 0) return HSDLA_OK;
  // Tensor maps, deduplicated by (address, K extent, columns, leading dimension, box rows).
  std::vector<CUtensorMap> maps;
  std::map<std::tuple<const void*, long long, long long, long long, int>, int> cache;
  auto map_of = [&](const double2* base, int k, int cols, long long ld, int box_cols,
                    int* out) -> int {
    const long long kk = k > 0 ? k : 1;
    auto key = std::make_tuple((const void*)base, kk, (long long)cols, ld, box_cols);
    auto it = cache.find(key);
    if (it != cache.end()) { *out = it->second; return HSDLA_OK; }
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)(2 * kk), (cuuint64_t)cols};
    cuuint64_t strides[1] = {(cuuint64_t)ld * 16};
    cuuint32_t box[2] = {16, (cuuint32_t)box_cols};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double2*>(base), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      set_error("cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
      return HSDLA_ERR_CUDA;
    }
    *out = (int)maps.size();
    cache[key] = *out;
    maps.push_back(m);
    return HSDLA_OK;
  };
  std::vector<TSeg> tsegs(segs.size());
  for (const Prob& p : probs) {
    for (int s = p.seg0; s < p.seg0 + p.nseg; ++s) {
      const Seg& sg = segs[s];
      TSeg& t = tsegs[s];
      t.k = sg.k;
      t.sel = sg.sel;
      int rc = map_of(sg.P, sg.k, p.m, sg.ldP, C::TM, &t.mapP);
      if (rc) return rc;
      t.mapPalt = t.mapP;
      if (sg.P_alt) {
        rc = map_of(sg.P_alt, sg.k, p.m, sg.ldP, C::TM, &t.mapPalt);
        if (rc) return rc;
      }
      rc = map_of(sg.Q, sg.k, p.n, sg.ldQ, C::TN, &t.mapQ);
      if (rc) return rc;
    }
  }
  if (first_on_device((const void*)contract_tma_kernel<C>))
    HS_CUDA(cudaFuncSetAttribute(contract_tma_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)C::kSmemBytes));
  int occ = 0;
  HS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, contract_tma_kernel<C>, C::kT,
                                                        C::kSmemBytes));
  if (occ < 1) occ = 1;
  long long grid_ll = (long long)ctx->num_sms * occ;
  if (grid_ll > total) grid_ll = total;
  const int grid = (int)grid_ll;
  constexpr int kSlot = kTile * kTile * 2;  // partial slot stride covers every configuration
  static_assert(C::kPartial <= kSlot, "partial tile larger than a slot");
  if (ctx->partial_slots < grid) {
    HS_CUDA(cudaStreamSynchronize(ctx->stream));
    if (ctx->partials) cudaFree(ctx->partials);
    if (ctx->ready) cudaFree(ctx->ready);
    HS_CUDA(cudaMalloc(&ctx->partials, size_t(grid) * kSlot * sizeof(double)));
    HS_CUDA(cudaMalloc(&ctx->ready, size_t(grid) * sizeof(int)));
    ctx->partial_slots = grid;
  }
  int rc = arena_begin(ctx, probs.size() * sizeof(Prob) + tsegs.size() * sizeof(TSeg) +
                                maps.size() * sizeof(CUtensorMap) + 512);
  if (rc) return rc;
  Prob* dprobs = static_cast<Prob*>(arena_push(ctx, probs.data(), probs.size() * sizeof(Prob), nullptr));
  TSeg* dsegs = static_cast<TSeg*>(
      arena_push(ctx, tsegs.data(), (tsegs.empty() ? 1 : tsegs.size()) * sizeof(TSeg), nullptr));
  CUtensorMap* dmaps = static_cast<CUtensorMap*>(
      arena_push(ctx, maps.data(), maps.size() * sizeof(CUtensorMap), nullptr));
  rc = arena_flush(ctx);
  if (rc) return rc;
  HS_CUDA(cudaMemsetAsync(ctx->ready, 0, size_t(grid) * sizeof(int), ctx->stream));
  TKParams sk;
  sk.probs = dprobs;
  sk.segs = dsegs;
  sk.maps = dmaps;
  sk.total_it = total;
  sk.nprob = (int)probs.size();
  sk.grid = grid;
  sk.partials = ctx->partials;
  sk.ready = ctx->ready;
  sk.flag = flag_dev;
  void* kargs[] = {&sk};
  HS_CUDA(cudaLaunchCooperativeKernel((const void*)contract_tma_kernel<C>, dim3(grid), dim3(C::kT),
                                      kargs, C::kSmemBytes, ctx->stream));
  return HSDLA_OK;
}
}  // namespace

namespace {
template <class C>
int preload_cfg() {
  cudaFuncAttributes at;
  HS_CUDA(cudaFuncGetAttributes(&at, (const void*)contract_tma_kernel<C>));
  if (first_on_device((const void*)contract_tma_kernel<C>))
    HS_CUDA(cudaFuncSetAttribute(contract_tma_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)C::kSmemBytes));
  return HSDLA_OK;
}
}  // namespace

int preload_contract_tma() {
  if (int rc = preload_cfg<Cfg64>()) return rc;
  if (int rc = preload_cfg<Cfg96>()) return rc;
  if (int rc = preload_cfg<Cfg64P>()) return rc;
  if (int rc = preload_cfg<Cfg96P>()) return rc;
  if (int rc = preload_cfg<Cfg64G>()) return rc;
  if (int rc = preload_cfg<Cfg64G8>()) return rc;
  return preload_cfg<Cfg96G>();
}

bool tma_wants(const std::vector<Prob>& probs) {
  // General (T-application) problems with 64 < m <= 96 run on 96 x 32 tiles.
  static int apply_tile = -1;
  if (apply_tile < 0) {
    const char* e = getenv("HSDLA_APPLY_TILE");
    apply_tile = (e && atoi(e) == 64) ? 64 : 96;
  }
  bool general = !probs.empty();
  int max_m = 0;
  for (const Prob& p : probs) {
    general = general && p.kind == PROB_GENERAL;
    max_m = std::max(max_m, p.m);
  }
  return general && apply_tile == 96 && max_m > 64 && max_m <= 96;
}

int launch_contract_tma(hsdla_ctx* ctx, const std::vector<Prob>& probs, long long total,
                        const std::vector<Seg>& segs, int* flag_dev) {
  (void)total;
  // HSDLA_TMA_PAIR=0 selects the 64-bit fragment-load variant.
  static int pair = -1;
  if (pair < 0) {
    const char* e = getenv("HSDLA_TMA_PAIR");
    pair = (e && atoi(e) == 0) ? 0 : 1;
  }
  const bool g3 = pair && cmul_mode() == 3;
  if (tma_wants(probs))
    return g3     ? launch_cfg<Cfg96G>(ctx, probs, segs, flag_dev)
           : pair ? launch_cfg<Cfg96P>(ctx, probs, segs, flag_dev)
                  : launch_cfg<Cfg96>(ctx, probs, segs, flag_dev);
  static int w8 = -1;  // HSDLA_TMA_W8=1: eight 32x16 warps per 64x64 tile
  if (w8 < 0) {
    const char* e = getenv("HSDLA_TMA_W8");
    w8 = (e && e[0] == '1') ? 1 : 0;
  }
  if (g3 && w8) return launch_cfg<Cfg64G8>(ctx, probs, segs, flag_dev);
  return g3     ? launch_cfg<Cfg64G>(ctx, probs, segs, flag_dev)
         : pair ? launch_cfg<Cfg64P>(ctx, probs, segs, flag_dev)
                : launch_cfg<Cfg64>(ctx, probs, segs, flag_dev);
}

}  // namespace hsdla
