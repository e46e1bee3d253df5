// Spherical Bessel functions j_0..j_LT(x) on the device, restating the reference's three
// regimes (special.py:49-131): power series below 0.5, upward recurrence at x >= LT,
// Miller downward recurrence normalised on the better-conditioned of j_0 / j_1 otherwise.
// Shared by the A/B generator (abgen.cu) and the reduced-overlap path (reduced.cu); both
// translation units are compiled with -fmad=false so the rounding follows numpy's.
#pragma once
#include <cuda_runtime.h>
#include <math.h>

namespace hsdla {
namespace bessel {

__device__ __forceinline__ double dbl_fact(int n) {
  double r = 1.0;
  while (n > 1) { r *= n; n -= 2; }
  return r;
}

// j_0..j_{LT}(x) for x > 0 (LT = L + 1 orders, special.py:104-131 regime switch).
template <int LT>
__device__ inline void bessel_j(double x, double (&j)[LT + 1]) {
  if (x < 0.5) {
    const double x2h = 0.5 * x * x;
#pragma unroll
    for (int l = 0; l <= LT; ++l) {
      double term = pow(x, (double)l) / dbl_fact(2 * l + 1);
      double total = term;
      for (int k = 1;; ++k) {
        term *= -x2h / (double)(k * (2 * l + 2 * k + 1));
        total += term;
        if (fabs(term) <= 1e-18 * fmax(fabs(total), 1e-300) || k > 60) break;
      }
      j[l] = total;
    }
    return;
  }
  double s, c;
  sincos(x, &s, &c);
  if (x >= (double)LT) {
    j[0] = s / x;
    if (LT >= 1) j[1] = s / (x * x) - c / x;
#pragma unroll
    for (int l = 1; l < LT; ++l) j[l + 1] = (double)(2 * l + 1) / x * j[l] - j[l - 1];
    return;
  }
  // Miller downward recurrence (special.py:77-101)
  const int ix = (int)x;
  const int start = LT + (ix > 16 ? ix : 16) + (int)(2.0 * sqrt((double)(LT + 1)));
  double scratch[LT + 1];
#pragma unroll
  for (int l = 0; l <= LT; ++l) scratch[l] = 0.0;
  double jp1 = 0.0, jl = 1e-30;
  int l = start;
  for (; l > LT + 1; --l) {  // orders above l_top are not stored
    const double jm1 = (double)(2 * l + 1) / x * jl - jp1;
    jp1 = jl;
    jl = jm1;
    if (fabs(jl) > 1e250) { jl *= 1e-250; jp1 *= 1e-250; }
  }
#pragma unroll
  for (int ll = LT + 1; ll >= 1; --ll) {
    const double jm1 = (double)(2 * ll + 1) / x * jl - jp1;
    jp1 = jl;
    jl = jm1;
    if (fabs(jl) > 1e250) {
      jl *= 1e-250;
      jp1 *= 1e-250;
#pragma unroll
      for (int q = (ll < LT ? ll : LT); q <= LT; ++q) scratch[q] *= 1e-250;
    }
    scratch[ll - 1] = jl;
  }
  const double j0 = s / x;
  const double j1 = s / (x * x) - c / x;
  double scale;
  if (fabs(j0) >= fabs(j1) && scratch[0] != 0.0) scale = j0 / scratch[0];
  else if (LT >= 1 && scratch[1] != 0.0) scale = j1 / scratch[1];
  else scale = j0 / scratch[0];
#pragma unroll
  for (int q = 0; q <= LT; ++q) j[q] = scratch[q] * scale;
}


// j_0..j_{L+1}(x) and j'_0..j'_L(x) including the exact x = 0 limits (special.py:114-130):
// j'_0 = -j_1, j'_l = j_{l-1} - (l+1)/x j_l.
template <int L>
__device__ inline void bessel_jd(double x, double (&jv)[L + 2], double (&jd)[L + 1]) {
  if (x == 0.0) {
#pragma unroll
    for (int l = 0; l <= L + 1; ++l) jv[l] = (l == 0) ? 1.0 : 0.0;
#pragma unroll
    for (int l = 0; l <= L; ++l) jd[l] = (l == 1) ? 1.0 / 3.0 : 0.0;
    return;
  }
  bessel_j<L + 1>(x, jv);
  jd[0] = -jv[1];
#pragma unroll
  for (int l = 1; l <= L; ++l) jd[l] = jv[l - 1] - (double)(l + 1) / x * jv[l];
}

}  // namespace bessel
}  // namespace hsdla
