// Legendre-reduced A-side overlap and radial match factors for sm_100a.
//
//   S_AA[G, G'] = (4 pi)^2 / Omega * sum_a conj(p_a(G)) p_a(G')
//                 * sum_{l <= l_a} (2l+1) / (4 pi) / W_{a,l}^2 * f_{a,l}(G) f_{a,l}(G') P_l(cos g)
//
// with p_a(G) = e^{i K_G . x_a}, cos g = K^_G . K^_G' (1 when either K is zero) and f the
// A-side match factors.  This is the reference's reduced_S_AA (oracle.py:159-216, inputs
// from reduced_overlap_inputs, flapw.py:236-250): the m-sum of A*^H A* collapsed by the
// addition theorem, (l_max+1)x fewer flops than the stacked contraction
// (FLEUR's Legendre-reduced overlap).
//
// Compiled with -fmad=false: every product and sum follows the reference's numpy
// evaluation order, and the element (G', G) is computed from the same commutative
// products as (G, G'), so the output is exactly Hermitian.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <vector>

#include "bessel.cuh"
#include "common.cuh"

namespace hsdla {
namespace {

constexpr int kMfThreads = 128;

// f_A, f_B of one atom group (l_sph = L): thread per K-vector, blockIdx.y = atom
// (flapw.py:179-198 match_factors).
template <int L>
__global__ void __launch_bounds__(kMfThreads)
    mf_kernel(int n, const double* __restrict__ kv, const double* __restrict__ rmt,
              const double* __restrict__ radial, int radial_stride, const int* __restrict__ atoms,
              const long long* __restrict__ frow, double* fa, double* fb, long long ldf) {
  const int t = blockIdx.x * kMfThreads + threadIdx.x;
  if (t >= n) return;
  const int a = atoms[blockIdx.y];
  const long long r0 = frow[blockIdx.y];
  const double kx = kv[3 * t + 0], ky = kv[3 * t + 1], kz = kv[3 * t + 2];
  const double kn = sqrt(kx * kx + ky * ky + kz * kz);
  double jv[L + 2], jd[L + 1];
  bessel::bessel_jd<L>(rmt[a] * kn, jv, jd);
  const double* rad = radial + (long long)a * radial_stride * 5;
#pragma unroll
  for (int l = 0; l <= L; ++l) {
    const double u = rad[5 * l + 0], up = rad[5 * l + 1], ud = rad[5 * l + 2], udp = rad[5 * l + 3];
    if (fa) fa[(r0 + l) * ldf + t] = ud * kn * jd[l] - udp * jv[l];
    if (fb) fb[(r0 + l) * ldf + t] = -u * kn * jd[l] + up * jv[l];
  }
}

typedef int (*mf_launcher)(hsdla_ctx*, int, const double*, const double*, const double*, int,
                           const int*, const long long*, double*, double*, long long, int);

template <int L>
int launch_mf(hsdla_ctx* ctx, int n, const double* kv, const double* rmt, const double* radial,
              int stride, const int* atoms, const long long* frow, double* fa, double* fb,
              long long ldf, int count) {
  dim3 grid((n + kMfThreads - 1) / kMfThreads, count);
  mf_kernel<L><<<grid, kMfThreads, 0, ctx->stream>>>(n, kv, rmt, radial, stride, atoms, frow, fa,
                                                     fb, ldf);
  HS_CHECK_LAUNCH();
  return HSDLA_OK;
}

const mf_launcher kMfLaunchers[HSDLA_MAX_LSPH + 1] = {
    &launch_mf<0>, &launch_mf<1>, &launch_mf<2>, &launch_mf<3>, &launch_mf<4>,
    &launch_mf<5>, &launch_mf<6>, &launch_mf<7>, &launch_mf<8>, &launch_mf<9>,
    &launch_mf<10>, &launch_mf<11>, &launch_mf<12>, &launch_mf<13>, &launch_mf<14>};

// Per K-vector unit direction (w = 1 if K != 0) and per (atom, K) phase e^{i K.x_a}.
__global__ void rs_prep_kernel(int n, int n_atoms, const double* __restrict__ kv,
                               const double* __restrict__ pos, double4* unit, double2* phase) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const double kx = kv[3 * t + 0], ky = kv[3 * t + 1], kz = kv[3 * t + 2];
  const double kn = sqrt(kx * kx + ky * ky + kz * kz);
  unit[t] = kn > 0.0 ? make_double4(kx / kn, ky / kn, kz / kn, 1.0)
                     : make_double4(0.0, 0.0, 0.0, 0.0);
  for (int a = 0; a < n_atoms; ++a) {
    const double th = kx * pos[3 * a + 0] + ky * pos[3 * a + 1] + kz * pos[3 * a + 2];
    double s, c;
    sincos(th, &s, &c);
    phase[(long long)a * n + t] = make_double2(c, s);
  }
}

// E[a + t * lde] = e^{i K_t . x_a}: the phase matrix of the per-type factorised build
// (same expression and rounding as the A/B generator's phase).
__global__ void phase_matrix_kernel(int n, int n_atoms, const double* __restrict__ kv,
                                    const double* __restrict__ pos, double2* E, long long lde) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const double kx = kv[3 * t + 0], ky = kv[3 * t + 1], kz = kv[3 * t + 2];
  for (int a = 0; a < n_atoms; ++a) {
    const double th = kx * pos[3 * a + 0] + ky * pos[3 * a + 1] + kz * pos[3 * a + 2];
    double sn, cs;
    sincos(th, &sn, &cs);
    E[a + (long long)t * lde] = make_double2(cs, sn);
  }
}

// C (+)= W o G on the lower triangle (i >= j): the Hadamard combine of a type's phase Gram
// W with its template Gram G.
__global__ void hadamard_lower_kernel(int n, const double2* __restrict__ W, long long ldw,
                                      const double2* __restrict__ G, long long ldg, double2* C,
                                      long long ldc, int accumulate) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y;
  if (i >= n || i < j) return;
  const double2 w = W[i + (long long)j * ldw], g = G[i + (long long)j * ldg];
  double2 v = make_double2(__fma_rn(w.x, g.x, -__dmul_rn(w.y, g.y)), __fma_rn(w.x, g.y, __dmul_rn(w.y, g.x)));
  double2* c = C + i + (long long)j * ldc;
  if (accumulate) {
    const double2 o = *c;
    v.x = __dadd_rn(v.x, o.x);
    v.y = __dadd_rn(v.y, o.y);
  }
  *c = v;
}

struct RsParams {
  int n, tiles;
  const double4* unit;       // n: K^ and 1 (0 for K = 0)
  const double2* phase;      // n_atoms x n: e^{i K.x_a}
  const double* f;           // this type's match-factor rows l = 0..ltop, stride ldf
  long long ldf;
  int ltop;
  const double* coef;        // this type's (2l+1) / (4 pi) / W_l^2
  const int* atoms;          // atoms of this type
  int n_type_atoms;
  int accumulate;            // add to the lower triangle already in S (earlier types)
  double scale;              // (4 pi)^2 / Omega
  double2* S;
  long long lds;
};

__device__ __forceinline__ void cp_async16_rs(void* smem_dst, const void* gsrc) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gsrc));
}
__device__ __forceinline__ void cp_async_commit_rs() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_rs() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

constexpr int kRsTile = 64;
constexpr int kRsAtomChunk = 8;

// One CTA per lower 64 x 64 tile and atom type, 256 threads, each thread a 4 x 4 micro-tile
// (rows i0 + tx + 16 r, columns j0 + ty + 16 s):
//   radial(i, j) = sum_l coef_l f_l(i) f_l(j) P_l(K^_i . K^_j)      (Legendre recurrence)
//   sf(i, j)     = sum_{a in type} conj(p_a(i)) p_a(j)               (phases staged in smem)
//   S(i, j)     (+)= scale * sf * radial
// Per element: (l+1) x (recurrence + FMA) + atoms x 4 FMAs, against 8 (l+1)^2 flops per
// atom of the stacked A*^H A*.  The strict lower part is mirrored as conj and the diagonal's
// imaginary part is 0, so the result is exactly Hermitian (as the reference's is).
__global__ void __launch_bounds__(256) rs_kernel(RsParams p) {
  constexpr int MR = 4, MS = 4;
  __shared__ __align__(16) double2 sEi[2][kRsAtomChunk][kRsTile];
  __shared__ __align__(16) double2 sEj[2][kRsAtomChunk][kRsTile];
  int t = blockIdx.x, tj = 0;
  while (t >= p.tiles - tj) { t -= p.tiles - tj; ++tj; }
  const int ti = tj + t;
  const int i0 = ti * kRsTile, j0 = tj * kRsTile;
  // cp.async of chunk q's phases (kRsAtomChunk atoms x 64 rows/columns) into buffer q & 1
  auto stage = [&](int q) {
    const int a0 = q * kRsAtomChunk;
    const int na = min(kRsAtomChunk, p.n_type_atoms - a0);
    for (int e = threadIdx.x; e < na * kRsTile; e += blockDim.x) {
      const int k = e / kRsTile, x = e - k * kRsTile;
      const double2* ph = p.phase + (long long)p.atoms[a0 + k] * p.n;
      cp_async16_rs(&sEi[q & 1][k][x], ph + min(i0 + x, p.n - 1));
      cp_async16_rs(&sEj[q & 1][k][x], ph + min(j0 + x, p.n - 1));
    }
  };
  if (p.n_type_atoms > 0) stage(0);
  cp_async_commit_rs();
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  int ci[MR], cj[MS];  // clamped indices (edge tiles compute duplicates, never stored)
#pragma unroll
  for (int r = 0; r < MR; ++r) ci[r] = min(i0 + tx + 16 * r, p.n - 1);
#pragma unroll
  for (int s = 0; s < MS; ++s) cj[s] = min(j0 + ty + 16 * s, p.n - 1);
  // ---- radial part
  double rad[MR][MS] = {};
  {
    double c[MR][MS], p0[MR][MS], p1[MR][MS];
    double4 ui[MR], uj[MS];
#pragma unroll
    for (int r = 0; r < MR; ++r) ui[r] = p.unit[ci[r]];
#pragma unroll
    for (int s = 0; s < MS; ++s) uj[s] = p.unit[cj[s]];
#pragma unroll
    for (int r = 0; r < MR; ++r)
#pragma unroll
      for (int s = 0; s < MS; ++s) {
        double v = 1.0;  // a zero K-vector is parallel to everything (oracle.py:199-201)
        if (ui[r].w != 0.0 && uj[s].w != 0.0)
          v = fmin(fmax(__fma_rn(ui[r].x, uj[s].x, __fma_rn(ui[r].y, uj[s].y, __dmul_rn(ui[r].z, uj[s].z))),
                        -1.0), 1.0);
        c[r][s] = v;
        p0[r][s] = 0.0;
        p1[r][s] = 0.0;
      }
#pragma unroll 1
    for (int l = 0; l <= p.ltop; ++l) {
      const double tl = (double)(2 * l - 1), ml = (double)(l - 1), il = 1.0 / (double)l;
      const double cl = p.coef[l];
      const double* fr = p.f + l * p.ldf;
      double hi[MR], fj[MS];
#pragma unroll
      for (int r = 0; r < MR; ++r) hi[r] = __dmul_rn(cl, __ldg(fr + ci[r]));
#pragma unroll
      for (int s = 0; s < MS; ++s) fj[s] = __ldg(fr + cj[s]);
#pragma unroll
      for (int r = 0; r < MR; ++r)
#pragma unroll
        for (int s = 0; s < MS; ++s) {
          double pl;  // P_l, special.py:22-38 recurrence
          if (l == 0) pl = 1.0;
          else if (l == 1) pl = c[r][s];
          else pl = __dmul_rn(__fma_rn(__dmul_rn(tl, c[r][s]), p1[r][s], -__dmul_rn(ml, p0[r][s])), il);
          p0[r][s] = p1[r][s];
          p1[r][s] = pl;
          rad[r][s] = __fma_rn(__dmul_rn(hi[r], fj[s]), pl, rad[r][s]);
        }
    }
  }
  // ---- structure factor of the type: phases of kRsAtomChunk atoms at a time, double-
  // buffered in smem by cp.async (chunk 0 was issued before the radial loop)
  double sr[MR][MS] = {}, si[MR][MS] = {};
  const int nchunk = (p.n_type_atoms + kRsAtomChunk - 1) / kRsAtomChunk;
  for (int q = 0; q < nchunk; ++q) {
    if (q + 1 < nchunk) stage(q + 1);
    cp_async_commit_rs();
    cp_async_wait_rs<1>();
    __syncthreads();
    const int na = min(kRsAtomChunk, p.n_type_atoms - q * kRsAtomChunk);
    const int b = q & 1;
#pragma unroll 2
    for (int k = 0; k < na; ++k) {
      double2 pi_[MR], pj[MS];
#pragma unroll
      for (int r = 0; r < MR; ++r) pi_[r] = sEi[b][k][tx + 16 * r];
#pragma unroll
      for (int s = 0; s < MS; ++s) pj[s] = sEj[b][k][ty + 16 * s];
#pragma unroll
      for (int r = 0; r < MR; ++r)
#pragma unroll
        for (int s = 0; s < MS; ++s) {
          sr[r][s] = __fma_rn(pi_[r].x, pj[s].x, __fma_rn(pi_[r].y, pj[s].y, sr[r][s]));
          si[r][s] = __fma_rn(pi_[r].x, pj[s].y, __fma_rn(-pi_[r].y, pj[s].x, si[r][s]));
        }
    }
    __syncthreads();  // buffer b is refilled by the stage() of iteration q + 1
  }
  // ---- epilogue: lower tile + conjugate mirror
#pragma unroll
  for (int r = 0; r < MR; ++r)
#pragma unroll
    for (int s = 0; s < MS; ++s) {
      const int i = i0 + tx + 16 * r, j = j0 + ty + 16 * s;
      if (i >= p.n || j >= p.n || i < j) continue;
      double re = __dmul_rn(__dmul_rn(sr[r][s], rad[r][s]), p.scale);
      double im = (i == j) ? 0.0 : __dmul_rn(__dmul_rn(si[r][s], rad[r][s]), p.scale);
      double2* lo = p.S + i + (long long)j * p.lds;
      if (p.accumulate) {
        const double2 old = *lo;
        re = __dadd_rn(re, old.x);
        im = (i == j) ? 0.0 : __dadd_rn(im, old.y);
      }
      *lo = make_double2(re, im);
      if (i != j) p.S[j + (long long)i * p.lds] = make_double2(re, -im);
    }
}

}  // namespace

int phase_matrix(hsdla_ctx* ctx, int n, int n_atoms, const double* kv, const double* pos,
                 double2* E, long long lde) {
  if (n <= 0 || n_atoms <= 0) return HSDLA_OK;
  phase_matrix_kernel<<<(n + 127) / 128, 128, 0, ctx->stream>>>(n, n_atoms, kv, pos, E, lde);
  HS_CHECK_LAUNCH();
  return HSDLA_OK;
}

int hadamard_lower(hsdla_ctx* ctx, int n, const double2* W, long long ldw, const double2* G,
                   long long ldg, double2* C, long long ldc, int accumulate) {
  if (n <= 0) return HSDLA_OK;
  hadamard_lower_kernel<<<dim3((n + 127) / 128, n), 128, 0, ctx->stream>>>(n, W, ldw, G, ldg, C,
                                                                          ldc, accumulate);
  HS_CHECK_LAUNCH();
  return HSDLA_OK;
}

int match_factors(hsdla_ctx* ctx, const hsdla_ab_args* s, const int64_t* f_row, double* fa,
                  double* fb, int64_t ldf) {
  if (s->n_atoms < 1 || s->n_basis < 1) return -2;
  if (ldf < s->n_basis) return -6;
  std::vector<int> atoms;
  std::vector<long long> rows;
  std::vector<int> gl, gb, gc;
  for (int L = 0; L <= HSDLA_MAX_LSPH; ++L) {
    const int begin = (int)atoms.size();
    for (int a = 0; a < s->n_atoms; ++a)
      if (s->l_sph[a] == L) { atoms.push_back(a); rows.push_back(f_row[a]); }
    if ((int)atoms.size() > begin) { gl.push_back(L); gb.push_back(begin); gc.push_back((int)atoms.size() - begin); }
  }
  if ((int)atoms.size() != s->n_atoms) {
    set_error("l_sph above HSDLA_MAX_LSPH");
    return HSDLA_ERR_UNSUPPORTED;
  }
  int rc = arena_begin(ctx, atoms.size() * (sizeof(int) + sizeof(long long)) + 64);
  if (rc) return rc;
  int* da = static_cast<int*>(arena_push(ctx, atoms.data(), atoms.size() * sizeof(int), nullptr));
  long long* dr = static_cast<long long*>(arena_push(ctx, rows.data(), rows.size() * sizeof(long long), nullptr));
  rc = arena_flush(ctx);
  if (rc) return rc;
  for (size_t g = 0; g < gl.size(); ++g) {
    rc = kMfLaunchers[gl[g]](ctx, s->n_basis, s->k_vectors, s->mt_radius, s->radial,
                             s->radial_stride, da + gb[g], dr + gb[g], fa, fb, ldf, gc[g]);
    if (rc) return rc;
  }
  return HSDLA_OK;
}

int reduced_s_aa(hsdla_ctx* ctx, const hsdla_reduced_args* r) {
  const int n = r->n_basis, na = r->n_atoms;
  if (na < 1) return -2;
  if (n < 1) return -2;
  if (r->ld_f < n || r->lds < n) return -2;
  // Types = distinct (f_row, l_top): atoms pointing at the same match-factor rows share
  // the radial sum.
  std::vector<long long> trow;
  std::vector<int> tlt, tatoms, tbegin;
  std::vector<int> type_of(na, -1);
  for (int a = 0; a < na; ++a) {
    if (r->l_top[a] < 0 || r->l_top[a] > HSDLA_MAX_LSPH) {
      set_error("l above HSDLA_MAX_LSPH");
      return HSDLA_ERR_UNSUPPORTED;
    }
    for (size_t k = 0; k < trow.size(); ++k)
      if (trow[k] == r->f_row[a] && tlt[k] == r->l_top[a]) type_of[a] = (int)k;
    if (type_of[a] < 0) {
      type_of[a] = (int)trow.size();
      trow.push_back(r->f_row[a]);
      tlt.push_back(r->l_top[a]);
    }
  }
  for (size_t k = 0; k < trow.size(); ++k) {
    tbegin.push_back((int)tatoms.size());
    for (int a = 0; a < na; ++a)
      if (type_of[a] == (int)k) tatoms.push_back(a);
  }
  tbegin.push_back((int)tatoms.size());
  const size_t need = size_t(n) * sizeof(double4) + size_t(na) * n * sizeof(double2);
  double* scratch = nullptr;
  HS_CUDA(cudaMallocAsync(&scratch, need, ctx->stream));
  double4* unit = reinterpret_cast<double4*>(scratch);
  double2* phase = reinterpret_cast<double2*>(unit + n);
  int rc = arena_begin(ctx, trow.size() * (sizeof(long long) + sizeof(int)) +
                                (tatoms.size() + tbegin.size()) * sizeof(int) + 256);
  if (rc) return rc;
  int* dtat = static_cast<int*>(arena_push(ctx, tatoms.data(), tatoms.size() * sizeof(int), nullptr));
  rc = arena_flush(ctx);
  if (rc) return rc;
  rs_prep_kernel<<<(n + 127) / 128, 128, 0, ctx->stream>>>(n, na, r->k_vectors, r->positions,
                                                           unit, phase);
  HS_CHECK_LAUNCH();
  RsParams p;
  p.n = n;
  p.tiles = (n + kRsTile - 1) / kRsTile;
  p.unit = unit;
  p.phase = phase;
  p.ldf = r->ld_f;
  p.scale = r->scale;
  p.S = reinterpret_cast<double2*>(r->S);
  p.lds = r->lds;
  const long long ntile = (long long)p.tiles * (p.tiles + 1) / 2;
  // one launch per atom type; later types accumulate into the lower triangle
  for (size_t k = 0; k < trow.size(); ++k) {
    p.f = r->f + trow[k] * r->ld_f;
    p.coef = r->coef + trow[k];
    p.ltop = tlt[k];
    p.atoms = dtat + tbegin[k];
    p.n_type_atoms = tbegin[k + 1] - tbegin[k];
    p.accumulate = k > 0;
    rs_kernel<<<(unsigned)ntile, 256, 0, ctx->stream>>>(p);
    HS_CHECK_LAUNCH();
  }
  HS_CUDA(cudaFreeAsync(scratch, ctx->stream));
  return HSDLA_OK;
}

}  // namespace hsdla
