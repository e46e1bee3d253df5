// Gaunt tensor and the Gaunt-sum T assembly on the GPU (input side):
//   G[L', L, L''] = sum_pts w conj(Y_L') Y_L Y_L''      (special.py:189-244 gaunt_tensor)
//   T[p, q]       = sum_k c[l(p), l(q), k] G[p, q, k] + diagonal terms   (flapw.py:306-363)
// over the reference's product quadrature grid (Gauss-Legendre in cos(theta) x uniform phi,
// exact for triple products up to l_max), with Y_lm from the A/B generator's device code.
// Layouts follow numpy C order: G[(i * n_row + j) * n_pot + k], c[(lp * n_l + l) * n_pot + k].
#include <cuda_runtime.h>

#include "common.cuh"

namespace hsdla {
namespace {

__global__ void gaunt_kernel(int n_row, int n_pot, int npts, int ldy, const double2* __restrict__ Y,
                             const double* __restrict__ w, double2* __restrict__ G) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long total = (long long)n_row * n_row * n_pot;
  if (idx >= total) return;
  const int k = (int)(idx % n_pot);
  const int j = (int)((idx / n_pot) % n_row);
  const int i = (int)(idx / ((long long)n_pot * n_row));
  const double2* yi = Y + (long long)i * ldy;
  const double2* yj = Y + (long long)j * ldy;
  const double2* yk = Y + (long long)k * ldy;
  double re = 0.0, im = 0.0;
  for (int p = 0; p < npts; ++p) {
    const double2 a = yi[p], b = yj[p], c = yk[p];
    // t = w conj(a) b
    const double tr = w[p] * (a.x * b.x + a.y * b.y);
    const double ti = w[p] * (a.x * b.y - a.y * b.x);
    re += tr * c.x - ti * c.y;
    im += tr * c.y + ti * c.x;
  }
  G[idx] = make_double2(re, im);
}

// One thread per (p, q) of the n_full x n_full output (column-major, ld n_full): the Gaunt sum
// on the leading n_dense block, plus the diagonal term diag[l(p)] (0 when diag is null) and
// `unit` on the diagonal (the AB block's 1).
__global__ void gaunt_sum_kernel(int n_full, int n_dense, int n_l, int n_pot,
                                 const double2* __restrict__ c, const double2* __restrict__ G,
                                 const double* __restrict__ diag, double unit,
                                 double2* __restrict__ out) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  const int q = blockIdx.y;
  if (p >= n_full) return;
  double2 v = make_double2(0.0, 0.0);
  if (p < n_dense && q < n_dense) {
    int lp = 0, lq = 0;
    while ((lp + 1) * (lp + 1) <= p) ++lp;
    while ((lq + 1) * (lq + 1) <= q) ++lq;
    const double2* cc = c + ((long long)lp * n_l + lq) * n_pot;
    const double2* gg = G + ((long long)p * n_dense + q) * n_pot;
    for (int k = 0; k < n_pot; ++k) {
      v.x += cc[k].x * gg[k].x - cc[k].y * gg[k].y;
      v.y += cc[k].x * gg[k].y + cc[k].y * gg[k].x;
    }
  }
  if (p == q) {
    int l = 0;
    while ((l + 1) * (l + 1) <= p) ++l;
    if (diag) v.x += diag[l];
    v.x += unit;
  }
  out[p + (long long)q * n_full] = v;
}

}  // namespace

int gaunt_tensor(hsdla_ctx* ctx, int n_row, int n_pot, int npts, int ldy, const double2* Y,
                 const double* w, double2* G) {
  const long long total = (long long)n_row * n_row * n_pot;
  if (total <= 0) return HSDLA_OK;
  gaunt_kernel<<<(unsigned)((total + 127) / 128), 128, 0, ctx->stream>>>(n_row, n_pot, npts, ldy,
                                                                         Y, w, G);
  HS_CHECK_LAUNCH();
  return HSDLA_OK;
}

int gaunt_sum(hsdla_ctx* ctx, int n_full, int n_dense, int n_l, int n_pot, const double2* c,
              const double2* G, const double* diag, double unit, double2* out) {
  if (n_full <= 0) return HSDLA_OK;
  gaunt_sum_kernel<<<dim3((n_full + 127) / 128, n_full), 128, 0, ctx->stream>>>(
      n_full, n_dense, n_l, n_pot, c, G, diag, unit, out);
  HS_CHECK_LAUNCH();
  return HSDLA_OK;
}

int preload_gaunt() {
  cudaFuncAttributes at;
  HS_CUDA(cudaFuncGetAttributes(&at, (const void*)gaunt_kernel));
  HS_CUDA(cudaFuncGetAttributes(&at, (const void*)gaunt_sum_kernel));
  return HSDLA_OK;
}

}  // namespace hsdla
