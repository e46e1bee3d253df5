// Fused matching-coefficient generator (compute_AB, reference flapw.py:201-233) for sm_100a.
//
// One thread per (K-vector t, atom a) evaluates, entirely in registers:
//   * |K|, K_hat (zero vector -> +z), atom-frame direction R_a K_hat renormalised
//     (flapw.py:169-176, :220-221);
//   * j_0..j_{L+1}(r_MT |K|) with the reference's three regimes — exact limits at 0,
//     power series below 0.5, upward recurrence at x >= L+1, Miller downward recurrence
//     normalised on the better-conditioned of j_0/j_1 otherwise — and j'_l
//     (special.py:49-131);
//   * f_A, f_B = the boundary-matching brackets (flapw.py:179-198);
//   * Y_lm by the normalised associated-Legendre recurrence with Condon-Shortley phase
//     (special.py:139-179), rows ordered l^2 + l + m;
//   * prefactor 4 pi / (sqrt(Omega) W_l) * i^l * e^{i K.x_a} (flapw.py:227),
// and writes its column of A, B and (optionally) ||udot|| B, the build_S row scaling
// (builder.py:207) fused into the producer.  L (= l_sph of the atom) is a template
// parameter so every recurrence array lives in registers.
//
// This translation unit is compiled with -fmad=false: the reference evaluates these
// formulas in numpy without FMA contraction, and the Wronskian / match-factor brackets
// cancel, so keeping the same rounding sequence keeps A/B within ~1 ulp of the reference.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <cmath>

#include "bessel.cuh"
#include "common.cuh"

namespace hsdla {
namespace {

// Y_lm recurrence coefficients (special.py:159-169), computed on the host with the
// reference's exact expressions (IEEE sqrt/div are correctly rounded, so the values are
// bit-identical to numpy's) instead of per thread at run time.
constexpr int kL = HSDLA_MAX_LSPH + 1;
__constant__ double c_sect[kL];    // sqrt((2m+1)/(2m))
__constant__ double c_sub[kL];     // sqrt(2m+3)
__constant__ double c_a[kL][kL];   // sqrt((4l^2-1)/(l^2-m^2))
__constant__ double c_b[kL][kL];   // sqrt(((l-1)^2-m^2)/(4(l-1)^2-1))

struct AbParams {
  int n_basis;
  const double* kv;
  const double* pos;
  const double* rot;
  const double* rmt;
  const double* radial;
  int radial_stride;
  double omega;
  double2* A;
  double2* B;
  double2* Bs;
  long long ld;
  double* udot_norms;
  int zero_phase;  // 1: e^{i K.x_a} taken as 1 (per-type templates at the origin)
};

constexpr int kAbThreads = 128;

// One thread per K-vector t (kAbThreads consecutive t per CTA), one atom per blockIdx.y.
// The Legendre recurrence runs l-outer (all m of one l at a time, same operands and
// rounding as special.py:159-169), so each l block of 2l+1 rows is complete at once: it
// is staged in shared memory as [column][row] and written out with consecutive threads
// on consecutive rows of a column — coalesced, sector-complete stores instead of one
// 16-byte store per column per thread.
template <int L>
__global__ void __launch_bounds__(kAbThreads) ab_kernel(AbParams p, const int* __restrict__ atoms,
                                                        const long long* __restrict__ row_off) {
  constexpr int S = 2 * L + 1;  // tallest l block; odd stride keeps smem conflict-free
  extern __shared__ double2 stage[];
  double2* sA = stage;
  double2* sB = stage + kAbThreads * S;
  const int t0 = blockIdx.x * kAbThreads;
  const int t = t0 + threadIdx.x;
  const bool live = t < p.n_basis;
  const int tc = live ? t : p.n_basis - 1;
  const int a = atoms[blockIdx.y];
  const long long off = row_off[blockIdx.y];
  // This atom's radial table (u, u', udot, udot', ||udot|| per l) staged in shared memory at
  // entry (the load overlaps the Bessel recurrences): uniform per CTA, read once instead of
  // an L2 round trip inside every l iteration.
  __shared__ double rad[5 * (L + 1)];
  {
    const double* src = p.radial + (long long)a * p.radial_stride * 5;
    for (int e = threadIdx.x; e < 5 * (L + 1); e += blockDim.x) rad[e] = src[e];
  }

  const double kx = p.kv[3 * tc + 0], ky = p.kv[3 * tc + 1], kz = p.kv[3 * tc + 2];
  const double kn = sqrt(kx * kx + ky * ky + kz * kz);
  double ux = 0.0, uy = 0.0, uz = 1.0;
  if (kn > 0.0) { ux = kx / kn; uy = ky / kn; uz = kz / kn; }
  const double* R = p.rot + 9 * a;
  double lx = ux * R[0] + uy * R[1] + uz * R[2];
  double ly = ux * R[3] + uy * R[4] + uz * R[5];
  double lz = ux * R[6] + uy * R[7] + uz * R[8];
  const double ln = sqrt(lx * lx + ly * ly + lz * lz);
  lx /= ln; ly /= ln; lz /= ln;
  const double ct = fmin(fmax(lz, -1.0), 1.0);
  const double st = sqrt(fmax(0.0, 1.0 - ct * ct));
  double ephr, ephi;  // e^{i phi}
  sincos(atan2(ly, lx), &ephi, &ephr);

  // Bessel values / derivatives at x = r_MT |K| (special.py:104-131).
  constexpr int LT = L + 1;
  const double x = p.rmt[a] * kn;
  double jv[LT + 1];
  double jd[L + 1];
  bessel::bessel_jd<L>(x, jv, jd);

  // Phase e^{i K.x_a}.
  const double* X = p.pos + 3 * a;
  const double th = p.zero_phase ? 0.0 : kx * X[0] + ky * X[1] + kz * X[2];
  double phs, phc;
  sincos(th, &phs, &phc);
  const double sqo = sqrt(p.omega);
  const double fourpi = 4.0 * 3.141592653589793;
  __syncthreads();  // rad[] staged at kernel entry

  // e^{i m phi} for m <= L (running product as the reference's expphi**m)
  double emr[L + 1], emi[L + 1];
  emr[0] = 1.0;
  emi[0] = 0.0;
#pragma unroll
  for (int m = 1; m <= L; ++m) {
    emr[m] = emr[m - 1] * ephr - emi[m - 1] * ephi;
    emi[m] = emr[m - 1] * ephi + emi[m - 1] * ephr;
  }
  double p1[L + 1], p2[L + 1];  // P_{l-1,m}, P_{l-2,m} (normalised)

#pragma unroll
  for (int l = 0; l <= L; ++l) {
    // prefactor 4 pi / (sqrt(Omega) W_l) * i^l * phase times the match factors (flapw.py:196-231)
    const double u = rad[5 * l + 0], up = rad[5 * l + 1], ud = rad[5 * l + 2], udp = rad[5 * l + 3];
    const double w = ud * up - u * udp;
    const double cl = fourpi / (sqo * w);
    double zr, zi;
    switch (l & 3) {
      case 0: zr = phc; zi = phs; break;
      case 1: zr = -phs; zi = phc; break;
      case 2: zr = -phc; zi = -phs; break;
      default: zr = phs; zi = -phc; break;
    }
    const double prr = cl * zr, pri = cl * zi;
    const double fa = ud * kn * jd[l] - udp * jv[l];
    const double fb = -u * kn * jd[l] + up * jv[l];
    const double par = prr * fa, pai = pri * fa;
    const double pbr = prr * fb, pbi = pri * fb;

    // P_{l,m} for all m <= l
    double pl[L + 1];
#pragma unroll
    for (int m = 0; m <= l; ++m) {
      if (m == l) pl[m] = (l == 0) ? 0.28209479177387814 : -c_sect[m] * st * p1[m - (l > 0 ? 1 : 0)];
      else if (m == l - 1) pl[m] = c_sub[m] * ct * p1[m];
      else pl[m] = c_a[l][m] * (ct * p1[m] - c_b[l][m] * p2[m]);
    }
    // rows l^2 + l + m, m = -l..l, staged [column][row]
#pragma unroll
    for (int m = 0; m <= l; ++m) {
      const double yr = pl[m] * emr[m], yi = pl[m] * emi[m];  // Y_{l,m}
      sA[threadIdx.x * S + l + m] =
          make_double2(yr * par + yi * pai, yr * pai + (-yi) * par);
      sB[threadIdx.x * S + l + m] =
          make_double2(yr * pbr + yi * pbi, yr * pbi + (-yi) * pbr);
      if (m > 0) {
        const double sg = (m & 1) ? -1.0 : 1.0;
        const double qr = sg * yr, qi = -(sg * yi);  // Y_{l,-m} = (-1)^m conj(Y_{l,m})
        sA[threadIdx.x * S + l - m] =
            make_double2(qr * par + qi * pai, qr * pai + (-qi) * par);
        sB[threadIdx.x * S + l - m] =
            make_double2(qr * pbr + qi * pbi, qr * pbi + (-qi) * pbr);
      }
    }
#pragma unroll
    for (int m = 0; m <= l; ++m) { p2[m] = p1[m]; p1[m] = pl[m]; }
    __syncthreads();
    // coalesced write-out of this l block: element e -> (column e / h, row e % h)
    const int h = 2 * l + 1;
    const double wl = rad[5 * l + 4];
    const int ncol = min(kAbThreads, p.n_basis - t0);
    for (int e = threadIdx.x; e < ncol * h; e += kAbThreads) {
      const int col = e / h, r = e - col * h;
      const long long gidx = (long long)(t0 + col) * p.ld + off + l * l + r;
      const double2 va = sA[col * S + r];
      const double2 vb = sB[col * S + r];
      p.A[gidx] = va;
      p.B[gidx] = vb;
      if (p.Bs) p.Bs[gidx] = make_double2(vb.x * wl, vb.y * wl);
    }
    __syncthreads();
  }
  (void)live;
}

// Per-type templates (zero_phase launches, a handful of atom blocks): one WARP per
// (K-vector, atom block), lane m in [0, L] evaluating the Legendre chain of its own m over
// l = m..L and writing rows l^2 + l +- m of A and B.  The per-K scalars (direction, Bessel
// values, match factors) are evaluated by every lane alike, so the dependent chain per lane is
// the prologue plus one m-chain instead of all (l, m) pairs, and C2's 2999 K-vectors give
// ~3000 warps instead of 24 CTAs with one warp per SM sub-partition (which left the unrolled
// kernel instruction-fetch bound, profiles/r02_ncu_abgen_template_stalls.txt).  Every
// value is computed by the same operations in the same order as ab_kernel (the file is built
// with -fmad=false): the templates are bitwise those of ab_kernel.
constexpr int kTplWarps = 4;
template <int L>
__global__ void __launch_bounds__(32 * kTplWarps) ab_tpl_kernel(AbParams p, const int* __restrict__ atoms,
                                                               const long long* __restrict__ row_off,
                                                               int count) {
  const int lane = threadIdx.x & 31;
  const long long item = (long long)blockIdx.x * kTplWarps + (threadIdx.x >> 5);
  if (item >= (long long)count * p.n_basis) return;  // warp-uniform
  const int blk = (int)(item / p.n_basis);
  const int t = (int)(item - (long long)blk * p.n_basis);
  const int a = atoms[blk];
  const long long off = row_off[blk];
  const int mm = lane;  // this lane's m (lanes > L idle after the shared prologue)
  const double* rad = p.radial + (long long)a * p.radial_stride * 5;

  const double kx = p.kv[3 * t + 0], ky = p.kv[3 * t + 1], kz = p.kv[3 * t + 2];
  const double kn = sqrt(kx * kx + ky * ky + kz * kz);
  double ux = 0.0, uy = 0.0, uz = 1.0;
  if (kn > 0.0) { ux = kx / kn; uy = ky / kn; uz = kz / kn; }
  const double* R = p.rot + 9 * a;
  double lx = ux * R[0] + uy * R[1] + uz * R[2];
  double ly = ux * R[3] + uy * R[4] + uz * R[5];
  double lz = ux * R[6] + uy * R[7] + uz * R[8];
  const double ln = sqrt(lx * lx + ly * ly + lz * lz);
  lx /= ln; ly /= ln; lz /= ln;
  const double ct = fmin(fmax(lz, -1.0), 1.0);
  const double st = sqrt(fmax(0.0, 1.0 - ct * ct));
  double ephr, ephi;
  sincos(atan2(ly, lx), &ephi, &ephr);
  constexpr int LT = L + 1;
  const double x = p.rmt[a] * kn;
  double jv[LT + 1];
  double jd[L + 1];
  bessel::bessel_jd<L>(x, jv, jd);
  const double* X = p.pos + 3 * a;
  const double th = p.zero_phase ? 0.0 : kx * X[0] + ky * X[1] + kz * X[2];
  double phs, phc;
  sincos(th, &phs, &phc);
  const double sqo = sqrt(p.omega);
  const double fourpi = 4.0 * 3.141592653589793;
  if (mm > L) return;

  // e^{i m phi}: the running product up to this lane's m (ab_kernel's emr / emi chain)
  double emr = 1.0, emi = 0.0;
#pragma unroll
  for (int m = 1; m <= L; ++m) {
    if (m > mm) break;
    const double r0 = emr * ephr - emi * ephi;
    const double i0 = emr * ephi + emi * ephr;
    emr = r0;
    emi = i0;
  }
  // sectoral seed P_{m,m} (ab_kernel's m == l branch, chained over m' <= m)
  double p1 = 0.0, p2 = 0.0;  // P_{l-1,m}, P_{l-2,m}
  double seed = 0.28209479177387814;
#pragma unroll
  for (int m = 1; m <= L; ++m) {
    if (m > mm) break;
    seed = -c_sect[m] * st * seed;
  }
  double2* const Ac = p.A + (long long)t * p.ld + off;
  double2* const Bc = p.B + (long long)t * p.ld + off;
  const double sg = (mm & 1) ? -1.0 : 1.0;
#pragma unroll
  for (int l = 0; l <= L; ++l) {
    if (l < mm) continue;
    const double u = rad[5 * l + 0], up = rad[5 * l + 1], ud = rad[5 * l + 2], udp = rad[5 * l + 3];
    const double w = ud * up - u * udp;
    const double cl = fourpi / (sqo * w);
    double zr, zi;
    switch (l & 3) {
      case 0: zr = phc; zi = phs; break;
      case 1: zr = -phs; zi = phc; break;
      case 2: zr = -phc; zi = -phs; break;
      default: zr = phs; zi = -phc; break;
    }
    const double prr = cl * zr, pri = cl * zi;
    const double fa = ud * kn * jd[l] - udp * jv[l];
    const double fb = -u * kn * jd[l] + up * jv[l];
    const double par = prr * fa, pai = pri * fa;
    const double pbr = prr * fb, pbi = pri * fb;
    double pl;
    if (l == mm) pl = seed;
    else if (l == mm + 1) pl = c_sub[mm] * ct * p1;
    else pl = c_a[l][mm] * (ct * p1 - c_b[l][mm] * p2);
    const double yr = pl * emr, yi = pl * emi;
    Ac[l * l + l + mm] = make_double2(yr * par + yi * pai, yr * pai + (-yi) * par);
    Bc[l * l + l + mm] = make_double2(yr * pbr + yi * pbi, yr * pbi + (-yi) * pbr);
    if (mm > 0) {
      const double qr = sg * yr, qi = -(sg * yi);
      Ac[l * l + l - mm] = make_double2(qr * par + qi * pai, qr * pai + (-qi) * par);
      Bc[l * l + l - mm] = make_double2(qr * pbr + qi * pbi, qr * pbi + (-qi) * pbr);
    }
    p2 = p1;
    p1 = pl;
  }
}

template <int L>
int launch_ab_tpl(hsdla_ctx* ctx, const AbParams& p, const int* atoms_dev, const long long* off_dev,
                  int count) {
  const long long items = (long long)count * p.n_basis;
  const int grid = (int)((items + kTplWarps - 1) / kTplWarps);
  ab_tpl_kernel<L><<<grid, 32 * kTplWarps, 0, ctx->stream>>>(p, atoms_dev, off_dev, count);
  HS_CHECK_LAUNCH();
  return HSDLA_OK;
}

template <int L>
int launch_ab_l(hsdla_ctx* ctx, const AbParams& p, const int* atoms_dev, const long long* off_dev,
                int count) {
  constexpr int S = 2 * L + 1;
  const size_t smem = size_t(2) * kAbThreads * S * sizeof(double2);
  if (smem > 48 * 1024 && first_on_device((const void*)ab_kernel<L>))
    HS_CUDA(cudaFuncSetAttribute(ab_kernel<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid((p.n_basis + kAbThreads - 1) / kAbThreads, count);
  ab_kernel<L><<<grid, kAbThreads, smem, ctx->stream>>>(p, atoms_dev, off_dev);
  HS_CHECK_LAUNCH();
  return HSDLA_OK;
}

// Standalone special functions (special.py:104-179) on the same device code as the A/B
// generator: j_l, j'_l at many x, and Y_lm at many unit directions.
template <int L>
__global__ void bessel_all_kernel(int n, const double* __restrict__ x, double* j, double* jp) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double jv[L + 2], jd[L + 1];
  bessel::bessel_jd<L>(x[i], jv, jd);
#pragma unroll
  for (int l = 0; l <= L; ++l) {
    j[(long long)l * n + i] = jv[l];
    jp[(long long)l * n + i] = jd[l];
  }
}

template <int L>
__global__ void ylm_all_kernel(int n, const double* __restrict__ d, double2* Y) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double ct = fmin(fmax(d[3 * i + 2], -1.0), 1.0);
  const double st = sqrt(fmax(0.0, 1.0 - ct * ct));
  double ephr, ephi;
  sincos(atan2(d[3 * i + 1], d[3 * i + 0]), &ephi, &ephr);
  double emr[L + 1], emi[L + 1];
  emr[0] = 1.0;
  emi[0] = 0.0;
#pragma unroll
  for (int m = 1; m <= L; ++m) {
    emr[m] = emr[m - 1] * ephr - emi[m - 1] * ephi;
    emi[m] = emr[m - 1] * ephi + emi[m - 1] * ephr;
  }
  double p1[L + 1], p2[L + 1];
#pragma unroll
  for (int l = 0; l <= L; ++l) {
    double pl[L + 1];
#pragma unroll
    for (int m = 0; m <= l; ++m) {
      if (m == l) pl[m] = (l == 0) ? 0.28209479177387814 : -c_sect[m] * st * p1[m - (l > 0 ? 1 : 0)];
      else if (m == l - 1) pl[m] = c_sub[m] * ct * p1[m];
      else pl[m] = c_a[l][m] * (ct * p1[m] - c_b[l][m] * p2[m]);
    }
#pragma unroll
    for (int m = 0; m <= l; ++m) {
      const double yr = pl[m] * emr[m], yi = pl[m] * emi[m];
      Y[(long long)(l * l + l + m) * n + i] = make_double2(yr, yi);
      if (m > 0) {
        const double sg = (m & 1) ? -1.0 : 1.0;
        Y[(long long)(l * l + l - m) * n + i] = make_double2(sg * yr, -(sg * yi));
      }
    }
#pragma unroll
    for (int m = 0; m <= l; ++m) { p2[m] = p1[m]; p1[m] = pl[m]; }
  }
}

template <int L>
int launch_special_l(hsdla_ctx* ctx, int kind, int n, const double* in, double* o1, double* o2) {
  const int grid = (n + 127) / 128;
  if (kind == 0) bessel_all_kernel<L><<<grid, 128, 0, ctx->stream>>>(n, in, o1, o2);
  else ylm_all_kernel<L><<<grid, 128, 0, ctx->stream>>>(n, in, reinterpret_cast<double2*>(o1));
  HS_CHECK_LAUNCH();
  return HSDLA_OK;
}
typedef int (*special_launcher)(hsdla_ctx*, int, int, const double*, double*, double*);
const special_launcher kSpecialLaunchers[HSDLA_MAX_LSPH + 1] = {
    &launch_special_l<0>, &launch_special_l<1>, &launch_special_l<2>, &launch_special_l<3>,
    &launch_special_l<4>, &launch_special_l<5>, &launch_special_l<6>, &launch_special_l<7>,
    &launch_special_l<8>, &launch_special_l<9>, &launch_special_l<10>, &launch_special_l<11>,
    &launch_special_l<12>, &launch_special_l<13>, &launch_special_l<14>};

template <int L>
int preload_ab_l() {
  constexpr int S = 2 * L + 1;
  const size_t smem = size_t(2) * kAbThreads * S * sizeof(double2);
  cudaFuncAttributes at;
  HS_CUDA(cudaFuncGetAttributes(&at, (const void*)ab_kernel<L>));
  if (smem > 48 * 1024 && first_on_device((const void*)ab_kernel<L>))
    HS_CUDA(cudaFuncSetAttribute(ab_kernel<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  return HSDLA_OK;
}

typedef int (*ab_launcher)(hsdla_ctx*, const AbParams&, const int*, const long long*, int);

const ab_launcher kAbLaunchers[HSDLA_MAX_LSPH + 1] = {
    &launch_ab_l<0>, &launch_ab_l<1>, &launch_ab_l<2>, &launch_ab_l<3>, &launch_ab_l<4>,
    &launch_ab_l<5>, &launch_ab_l<6>, &launch_ab_l<7>, &launch_ab_l<8>, &launch_ab_l<9>,
    &launch_ab_l<10>, &launch_ab_l<11>, &launch_ab_l<12>, &launch_ab_l<13>, &launch_ab_l<14>};
const ab_launcher kAbTplLaunchers[HSDLA_MAX_LSPH + 1] = {
    &launch_ab_tpl<0>, &launch_ab_tpl<1>, &launch_ab_tpl<2>, &launch_ab_tpl<3>, &launch_ab_tpl<4>,
    &launch_ab_tpl<5>, &launch_ab_tpl<6>, &launch_ab_tpl<7>, &launch_ab_tpl<8>, &launch_ab_tpl<9>,
    &launch_ab_tpl<10>, &launch_ab_tpl<11>, &launch_ab_tpl<12>, &launch_ab_tpl<13>, &launch_ab_tpl<14>};
// HSDLA_AB_TPL=0: the per-thread generator (ab_kernel) for the per-type templates as well.
bool ab_tpl_warp() {
  static int m = -1;
  if (m < 0) {
    const char* e = getenv("HSDLA_AB_TPL");
    m = (e && e[0] == '0') ? 0 : 1;
  }
  return m == 1;
}

__global__ void udot_rows_kernel(const double* __restrict__ radial, int stride, const int* atoms,
                                 const long long* off, int L, double* out) {
  const int a = atoms[blockIdx.x];
  const int h = (L + 1) * (L + 1);
  for (int r = threadIdx.x; r < h; r += blockDim.x) {
    int l = 0;
    while ((l + 1) * (l + 1) <= r) ++l;
    out[off[blockIdx.x] + r] = radial[((long long)a * stride + l) * 5 + 4];
  }
}

}  // namespace

int upload_ylm_tables() {
  static bool done[64] = {};
  int dev = 0;
  HS_CUDA(cudaGetDevice(&dev));
  if (dev < 64 && done[dev]) return HSDLA_OK;
  double sect[kL] = {}, sub[kL] = {}, a[kL][kL] = {}, b[kL][kL] = {};
  for (int m = 0; m < kL; ++m) {
    if (m > 0) sect[m] = std::sqrt((2 * m + 1) / (2.0 * m));
    sub[m] = std::sqrt(2 * m + 3.0);
    for (int l = m + 2; l < kL; ++l) {
      a[l][m] = std::sqrt((4.0 * l * l - 1.0) / (double)(l * l - m * m));
      const double lm1 = l - 1.0;
      b[l][m] = std::sqrt((lm1 * lm1 - (double)(m * m)) / (4.0 * (lm1 * lm1) - 1.0));
    }
  }
  HS_CUDA(cudaMemcpyToSymbol(c_sect, sect, sizeof(sect)));
  HS_CUDA(cudaMemcpyToSymbol(c_sub, sub, sizeof(sub)));
  HS_CUDA(cudaMemcpyToSymbol(c_a, a, sizeof(a)));
  HS_CUDA(cudaMemcpyToSymbol(c_b, b, sizeof(b)));
  if (dev < 64) done[dev] = true;
  return HSDLA_OK;
}

int preload_abgen() {
  int rc = HSDLA_OK;
  rc = rc ? rc : preload_ab_l<0>();
  rc = rc ? rc : preload_ab_l<1>();
  rc = rc ? rc : preload_ab_l<2>();
  rc = rc ? rc : preload_ab_l<3>();
  rc = rc ? rc : preload_ab_l<4>();
  rc = rc ? rc : preload_ab_l<5>();
  rc = rc ? rc : preload_ab_l<6>();
  rc = rc ? rc : preload_ab_l<7>();
  rc = rc ? rc : preload_ab_l<8>();
  rc = rc ? rc : preload_ab_l<9>();
  rc = rc ? rc : preload_ab_l<10>();
  rc = rc ? rc : preload_ab_l<11>();
  rc = rc ? rc : preload_ab_l<12>();
  rc = rc ? rc : preload_ab_l<13>();
  rc = rc ? rc : preload_ab_l<14>();
  if (rc) return rc;
  cudaFuncAttributes at;
  HS_CUDA(cudaFuncGetAttributes(&at, (const void*)udot_rows_kernel));
  return upload_ylm_tables();
}

int special_functions(hsdla_ctx* ctx, int kind, int l_max, int n, const double* in, double* o1,
                      double* o2) {
  if (l_max < 0 || l_max > HSDLA_MAX_LSPH) {
    set_error("l_max above HSDLA_MAX_LSPH");
    return HSDLA_ERR_UNSUPPORTED;
  }
  if (n <= 0) return HSDLA_OK;
  int rc = upload_ylm_tables();
  if (rc) return rc;
  return kSpecialLaunchers[l_max](ctx, kind, n, in, o1, o2);
}

int ab_generate(hsdla_ctx* ctx, const hsdla_ab_args* args) {
  {
    int rc0 = upload_ylm_tables();
    if (rc0) return rc0;
  }
  if (args->n_atoms < 1) return -1;
  if (args->n_basis < 1) return -1;
  for (int a = 0; a < args->n_atoms; ++a)
    if (args->l_sph[a] < 0 || args->l_sph[a] > HSDLA_MAX_LSPH) {
      set_error("l_sph above HSDLA_MAX_LSPH");
      return HSDLA_ERR_UNSUPPORTED;
    }
  AbParams p;
  p.n_basis = args->n_basis;
  p.kv = args->k_vectors;
  p.pos = args->positions;
  p.rot = args->rotations;
  p.rmt = args->mt_radius;
  p.radial = args->radial;
  p.radial_stride = args->radial_stride;
  p.omega = args->omega;
  p.A = reinterpret_cast<double2*>(args->A);
  p.B = reinterpret_cast<double2*>(args->B);
  p.Bs = reinterpret_cast<double2*>(args->B_scaled);
  p.ld = args->ld;
  p.udot_norms = args->udot_norms;
  p.zero_phase = 0;
  // Group atoms by l_sph; upload (atom, row offset) lists through the arena.
  std::vector<int> atoms;
  std::vector<long long> offs;
  std::vector<int> group_l, group_begin, group_count;
  for (int L = 0; L <= HSDLA_MAX_LSPH; ++L) {
    int begin = (int)atoms.size();
    for (int a = 0; a < args->n_atoms; ++a)
      if (args->l_sph[a] == L) { atoms.push_back(a); offs.push_back(args->row_offset[a]); }
    if ((int)atoms.size() > begin) {
      group_l.push_back(L);
      group_begin.push_back(begin);
      group_count.push_back((int)atoms.size() - begin);
    }
  }
  int rc = arena_begin(ctx, atoms.size() * (sizeof(int) + sizeof(long long)) + 64);
  if (rc) return rc;
  int* datoms = static_cast<int*>(arena_push(ctx, atoms.data(), atoms.size() * sizeof(int), nullptr));
  long long* doffs = static_cast<long long*>(
      arena_push(ctx, offs.data(), offs.size() * sizeof(long long), nullptr));
  rc = arena_flush(ctx);
  if (rc) return rc;
  for (size_t gi = 0; gi < group_l.size(); ++gi) {
    rc = kAbLaunchers[group_l[gi]](ctx, p, datoms + group_begin[gi], doffs + group_begin[gi],
                                   group_count[gi]);
    if (rc) return rc;
    if (p.udot_norms) {
      udot_rows_kernel<<<group_count[gi], 128, 0, ctx->stream>>>(
          p.radial, p.radial_stride, datoms + group_begin[gi], doffs + group_begin[gi], group_l[gi],
          p.udot_norms);
      HS_CHECK_LAUNCH();
    }
  }
  return HSDLA_OK;
}

// Per-type templates: the generator run once per type for a representative atom placed at
// the origin (phase 1), rows toff[i] of At / Bt (ld ldt).  The type's atoms differ from it
// only by the column phase e^{i K.x_a}, applied by the expansion pass (expand.cu).
int ab_generate_templates(hsdla_ctx* ctx, const hsdla_ab_args* args, const std::vector<int>& reps,
                          const std::vector<long long>& toff, double2* At, double2* Bt,
                          long long ldt) {
  int rc = upload_ylm_tables();
  if (rc) return rc;
  AbParams p;
  p.n_basis = args->n_basis;
  p.kv = args->k_vectors;
  p.pos = args->positions;
  p.rot = args->rotations;
  p.rmt = args->mt_radius;
  p.radial = args->radial;
  p.radial_stride = args->radial_stride;
  p.omega = args->omega;
  p.A = At;
  p.B = Bt;
  p.Bs = nullptr;
  p.ld = ldt;
  p.udot_norms = nullptr;
  p.zero_phase = 1;
  std::vector<int> atoms;
  std::vector<long long> offs;
  std::vector<int> group_l, group_begin, group_count;
  for (int L = 0; L <= HSDLA_MAX_LSPH; ++L) {
    const int begin = (int)atoms.size();
    for (size_t i = 0; i < reps.size(); ++i)
      if (args->l_sph[reps[i]] == L) { atoms.push_back(reps[i]); offs.push_back(toff[i]); }
    if ((int)atoms.size() > begin) {
      group_l.push_back(L);
      group_begin.push_back(begin);
      group_count.push_back((int)atoms.size() - begin);
    }
  }
  rc = arena_begin(ctx, atoms.size() * (sizeof(int) + sizeof(long long)) + 64);
  if (rc) return rc;
  int* datoms = static_cast<int*>(arena_push(ctx, atoms.data(), atoms.size() * sizeof(int), nullptr));
  long long* doffs = static_cast<long long*>(
      arena_push(ctx, offs.data(), offs.size() * sizeof(long long), nullptr));
  rc = arena_flush(ctx);
  if (rc) return rc;
  for (size_t gi = 0; gi < group_l.size(); ++gi) {
    rc = (ab_tpl_warp() ? kAbTplLaunchers : kAbLaunchers)[group_l[gi]](ctx, p, datoms + group_begin[gi], doffs + group_begin[gi],
                                   group_count[gi]);
    if (rc) return rc;
  }
  return HSDLA_OK;
}

}  // namespace hsdla
