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

struct RsParams {
  int n, n_types, tiles;
  const double4* unit;       // n: K^ and 1 (0 for K = 0)
  const double2* phase;      // n_atoms x n: e^{i K.x_a}
  const double* f;           // match-factor rows, stride ldf
  long long ldf;
  const long long* trow;     // per type: first f row
  const int* tltop;          // per type: l_top
  const int* tatoms;         // atoms grouped by type
  const int* tbegin;         // n_types + 1
  const double* coef;        // per f row: (2l+1) / (4 pi) / W^2
  double scale;              // (4 pi)^2 / Omega
  double2* S;
  long long lds;
};

// One CTA per lower 32 x 32 tile, 128 threads, each thread a 2 x 4 micro-tile (rows
// i0 + tx + 16 r, columns j0 + ty + 8 s).  Atoms that share match factors (one type) share
// the radial sum, so per element the work is
//   types x (l+1) x (Legendre step + FMA)  +  atoms x 2 complex FMAs (structure factor),
// against 8 (l+1)^2 flops per atom of the stacked A*^H A*.  The tile's strict lower part
// is mirrored as conj into the upper triangle and the diagonal's imaginary part is 0, so the
// result is exactly Hermitian (as the reference's is).
template <int LMAX>
__global__ void __launch_bounds__(128) rs_kernel(RsParams p) {
  int t = blockIdx.x, tj = 0;
  while (t >= p.tiles - tj) { t -= p.tiles - tj; ++tj; }
  const int ti = tj + t;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // ty < 8
  constexpr int MR = 2, MS = 4;
  int gi[MR], gj[MS];
  double4 ui[MR], uj[MS];
#pragma unroll
  for (int r = 0; r < MR; ++r) {
    gi[r] = ti * 32 + tx + 16 * r;
    ui[r] = p.unit[min(gi[r], p.n - 1)];
  }
#pragma unroll
  for (int s = 0; s < MS; ++s) {
    gj[s] = tj * 32 + ty + 8 * s;
    uj[s] = p.unit[min(gj[s], p.n - 1)];
  }
  double c[MR][MS];
#pragma unroll
  for (int r = 0; r < MR; ++r)
#pragma unroll
    for (int s = 0; s < MS; ++s) {
      double v = 1.0;  // a zero K-vector is parallel to everything (oracle.py:199-201)
      if (ui[r].w != 0.0 && uj[s].w != 0.0)
        v = fmin(fmax(__fma_rn(ui[r].x, uj[s].x, __fma_rn(ui[r].y, uj[s].y, __dmul_rn(ui[r].z, uj[s].z))),
                      -1.0), 1.0);
      c[r][s] = v;
    }
  double ar[MR][MS] = {}, ai[MR][MS] = {};
  for (int ty_ = 0; ty_ < p.n_types; ++ty_) {
    const double* fr = p.f + p.trow[ty_] * p.ldf;
    const double* cf = p.coef + p.trow[ty_];
    const int lt = p.tltop[ty_];
    double rad[MR][MS] = {}, p0[MR][MS], p1[MR][MS];
#pragma unroll 1
    for (int l = 0; l <= lt; ++l) {
      const double tl = (double)(2 * l - 1), ml = (double)(l - 1), il = 1.0 / (double)l;
      double hi[MR], fj[MS];
#pragma unroll
      for (int r = 0; r < MR; ++r) hi[r] = __dmul_rn(cf[l], __ldg(fr + l * p.ldf + min(gi[r], p.n - 1)));
#pragma unroll
      for (int s = 0; s < MS; ++s) fj[s] = __ldg(fr + l * p.ldf + min(gj[s], p.n - 1));
#pragma unroll
      for (int r = 0; r < MR; ++r)
#pragma unroll
        for (int s = 0; s < MS; ++s) {
          double pl;  // P_l(c), special.py:22-38 recurrence
          if (l == 0) pl = 1.0;
          else if (l == 1) pl = c[r][s];
          else pl = __dmul_rn(__fma_rn(__dmul_rn(tl, c[r][s]), p1[r][s], -__dmul_rn(ml, p0[r][s])), il);
          if (l > 0) p0[r][s] = p1[r][s];
          p1[r][s] = pl;
          rad[r][s] = __fma_rn(__dmul_rn(hi[r], fj[s]), pl, rad[r][s]);
        }
    }
    // structure factor of the type: sum_a conj(p_a(i)) p_a(j)
    double sr[MR][MS] = {}, si[MR][MS] = {};
    for (int k = p.tbegin[ty_]; k < p.tbegin[ty_ + 1]; ++k) {
      const double2* ph = p.phase + (long long)p.tatoms[k] * p.n;
      double2 pi_[MR], pj[MS];
#pragma unroll
      for (int r = 0; r < MR; ++r) pi_[r] = __ldg(ph + min(gi[r], p.n - 1));
#pragma unroll
      for (int s = 0; s < MS; ++s) pj[s] = __ldg(ph + min(gj[s], p.n - 1));
#pragma unroll
      for (int r = 0; r < MR; ++r)
#pragma unroll
        for (int s = 0; s < MS; ++s) {
          sr[r][s] = __fma_rn(pi_[r].x, pj[s].x, __fma_rn(pi_[r].y, pj[s].y, sr[r][s]));
          si[r][s] = __fma_rn(pi_[r].x, pj[s].y, __fma_rn(-pi_[r].y, pj[s].x, si[r][s]));
        }
    }
#pragma unroll
    for (int r = 0; r < MR; ++r)
#pragma unroll
      for (int s = 0; s < MS; ++s) {
        ar[r][s] = __fma_rn(sr[r][s], rad[r][s], ar[r][s]);
        ai[r][s] = __fma_rn(si[r][s], rad[r][s], ai[r][s]);
      }
  }
#pragma unroll
  for (int r = 0; r < MR; ++r)
#pragma unroll
    for (int s = 0; s < MS; ++s) {
      const int i = gi[r], j = gj[s];
      if (i >= p.n || j >= p.n || i < j) continue;
      const double re = __dmul_rn(ar[r][s], p.scale);
      const double im = (i == j) ? 0.0 : __dmul_rn(ai[r][s], p.scale);
      p.S[i + (long long)j * p.lds] = make_double2(re, im);
      if (i != j) p.S[j + (long long)i * p.lds] = make_double2(re, -im);
    }
}

typedef void (*rs_kernel_t)(RsParams);
const rs_kernel_t kRsKernels[HSDLA_MAX_LSPH + 1] = {
    rs_kernel<0>, rs_kernel<1>, rs_kernel<2>, rs_kernel<3>, rs_kernel<4>,
    rs_kernel<5>, rs_kernel<6>, rs_kernel<7>, rs_kernel<8>, rs_kernel<9>,
    rs_kernel<10>, rs_kernel<11>, rs_kernel<12>, rs_kernel<13>, rs_kernel<14>};

}  // namespace

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
  int lmax = 0;
  for (int a = 0; a < na; ++a) {
    if (r->l_top[a] < 0 || r->l_top[a] > HSDLA_MAX_LSPH) {
      set_error("l above HSDLA_MAX_LSPH");
      return HSDLA_ERR_UNSUPPORTED;
    }
    lmax = r->l_top[a] > lmax ? r->l_top[a] : lmax;
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
  long long* dtrow = static_cast<long long*>(arena_push(ctx, trow.data(), trow.size() * sizeof(long long), nullptr));
  int* dtlt = static_cast<int*>(arena_push(ctx, tlt.data(), tlt.size() * sizeof(int), nullptr));
  int* dtat = static_cast<int*>(arena_push(ctx, tatoms.data(), tatoms.size() * sizeof(int), nullptr));
  int* dtb = static_cast<int*>(arena_push(ctx, tbegin.data(), tbegin.size() * sizeof(int), nullptr));
  rc = arena_flush(ctx);
  if (rc) return rc;
  rs_prep_kernel<<<(n + 127) / 128, 128, 0, ctx->stream>>>(n, na, r->k_vectors, r->positions,
                                                           unit, phase);
  HS_CHECK_LAUNCH();
  RsParams p;
  p.n = n;
  p.n_types = (int)trow.size();
  p.tiles = (n + 31) / 32;
  p.unit = unit;
  p.phase = phase;
  p.f = r->f;
  p.ldf = r->ld_f;
  p.trow = dtrow;
  p.tltop = dtlt;
  p.tatoms = dtat;
  p.tbegin = dtb;
  p.coef = r->coef;
  p.scale = r->scale;
  p.S = reinterpret_cast<double2*>(r->S);
  p.lds = r->lds;
  const long long ntile = (long long)p.tiles * (p.tiles + 1) / 2;
  kRsKernels[lmax]<<<(unsigned)ntile, 128, 0, ctx->stream>>>(p);
  HS_CHECK_LAUNCH();
  HS_CUDA(cudaFreeAsync(scratch, ctx->stream));
  return HSDLA_OK;
}

}  // namespace hsdla
