// Per-type template expansion for sm_100a: the HBM-bound write pass of the stacked operands.
//
// With identity-equal atoms of a type (same rotation, muffin-tin radius, radial data, T set),
// compute_AB's per-atom loop (reference flapw.py:216-232) produces blocks that differ only by
// the column phase:  A_a = A_type diag(e^{iK.x_a}),  B_a = B_type diag(e^{iK.x_a}).  The T
// applications of the build (builder.py:231-240, :284-302) act on rows, so they commute with
// that phase too:  W_a = L^H [A_a; B_a] = (L^H [A_type; B_type]) diag(e^{iK.x_a}).  The build
// therefore evaluates the recurrences and applies T once per type (tiny) and this kernel
// writes every atom's rows: template times phase, optionally times ||udot|| per row (S's
// weighting, builder.py:207), plus the two real sum planes the three-product DMMA contraction
// stages instead of forming Re - Im and Re + Im with DADDs in its K loop (contract.cu, PL).
//
// Layout: one CTA per (32-column block, atom block); the 32 phases are computed once per CTA
// (one sincos each); consecutive threads take consecutive rows of a column, so every
// template read and stacked write is a contiguous run of the column (coalesced).  Work per
// element: 16 B template read (L2-resident: the templates are n_types x m x N) and up to
// 16 + 8 + 8 B written per output stack.
#include <cuda_runtime.h>

#include "common.cuh"

namespace hsdla {
namespace {

constexpr int kExCols = 32;
constexpr int kExThreads = 256;
constexpr int kMaxRows = (HSDLA_MAX_LSPH + 1) * (HSDLA_MAX_LSPH + 1);

struct ExpandParams {
  int n_basis;
  const double* kv;
  const double* pos;
  const double* radial;
  int radial_stride;
  const int4* atoms;
  const long long* off;
  const double2* T0;
  const double2* T1;
  long long ldt;
  ExpandOut o;
  long long ld;
  int atoms_fast;  // grid x = atom blocks (else x = column blocks)
};

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

__global__ void __launch_bounds__(kExThreads) expand_kernel(ExpandParams p) {
  __shared__ double2 ph[kExCols];
  __shared__ double urow[kMaxRows];
  const int ab = p.atoms_fast ? blockIdx.x : blockIdx.y;  // atom block
  const int4 at = p.atoms[ab];
  const int a = at.x, toff = at.y, m = at.z;
  const long long off = p.off[ab];
  const int t0 = (p.atoms_fast ? blockIdx.y : blockIdx.x) * kExCols;
  const int ncol = min(kExCols, p.n_basis - t0);
  if (threadIdx.x < ncol) {
    const int t = t0 + threadIdx.x;
    const double* X = p.pos + 3 * a;
    const double th = p.kv[3 * t + 0] * X[0] + p.kv[3 * t + 1] * X[1] + p.kv[3 * t + 2] * X[2];
    double s, c;
    sincos(th, &s, &c);
    ph[threadIdx.x] = make_double2(c, s);
  }
  if (p.o.scale1) {
    for (int r = threadIdx.x; r < m; r += kExThreads) {
      int l = 0;
      while ((l + 1) * (l + 1) <= r) ++l;
      urow[r] = p.radial[((long long)a * p.radial_stride + l) * 5 + 4];
    }
  }
  __syncthreads();
  const ExpandOut& o = p.o;
  for (int e = threadIdx.x; e < ncol * m; e += kExThreads) {
    const int col = e / m, r = e - col * m;
    const int t = t0 + col;
    const double2 z = ph[col];
    const long long src = toff + r + (long long)t * p.ldt;
    const long long dst = off + r + (long long)t * p.ld;
    const double2 w0 = cmul(__ldg(p.T0 + src), z);
    __stcs(o.O0 + dst, w0);
    if (o.O0d) {
      __stcs(o.O0d + dst, w0.x - w0.y);
      __stcs(o.O0s + dst, w0.x + w0.y);
    }
    if (o.O1) {
      double2 w1 = cmul(__ldg(p.T1 + src), z);
      if (o.O2) __stcs(o.O2 + dst, w1);
      if (o.scale1) {
        const double u = urow[r];
        w1 = make_double2(w1.x * u, w1.y * u);
      }
      __stcs(o.O1 + dst, w1);
      if (o.O1d) {
        __stcs(o.O1d + dst, w1.x - w1.y);
        __stcs(o.O1s + dst, w1.x + w1.y);
      }
    }
  }
}

}  // namespace

int launch_expand(hsdla_ctx* ctx, int n_basis, const double* kv, const double* pos,
                  const double* radial, int radial_stride, const int4* atoms_dev,
                  const long long* off_dev, int n_blocks, const double2* T0, const double2* T1,
                  long long ldt, const ExpandOut& o, long long ld) {
  if (n_blocks <= 0 || n_basis <= 0) return HSDLA_OK;
  ExpandParams p;
  p.n_basis = n_basis;
  p.kv = kv;
  p.pos = pos;
  p.radial = radial;
  p.radial_stride = radial_stride;
  p.atoms = atoms_dev;
  p.off = off_dev;
  p.T0 = T0;
  p.T1 = T1;
  p.ldt = ldt;
  p.o = o;
  p.ld = ld;
  // Many atoms (> 32): atoms fastest, so the CTAs resident at a time fill whole stacked columns
  // (C4 1.82 -> 1.50 ms, C3 -4%); few atoms: column blocks fastest (C2 30 vs 36 us per pass,
  // profiles/r02_expand_variants.json).
  p.atoms_fast = n_blocks > 32 ? 1 : 0;
  const int ncb = (n_basis + kExCols - 1) / kExCols;
  dim3 grid = p.atoms_fast ? dim3(n_blocks, ncb) : dim3(ncb, n_blocks);
  expand_kernel<<<grid, kExThreads, 0, ctx->stream>>>(p);
  HS_CHECK_LAUNCH();
  return HSDLA_OK;
}

int preload_expand() {
  cudaFuncAttributes at;
  HS_CUDA(cudaFuncGetAttributes(&at, (const void*)expand_kernel));
  return HSDLA_OK;
}

}  // namespace hsdla
