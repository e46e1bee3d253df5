// DMMA issue-rate probe for realistic operand patterns (sm_100a).
// Measures chip-wide FP64 TFLOP/s of register/smem-fed DMMA streams shaped like the
// contraction kernel's warp tile (4 A fragments x 4 B fragments x {Re, Im}).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// MODE 0: operands in registers, perturbed by an integer add each step (no smem)
// MODE 1: operands loaded from shared memory each step (12 LDS.64), ib-outer order
// MODE 2: as 1, jb-outer order
// MODE 3: as 1 but loads for step s+1 issued before the DMMAs of step s (register double buffer)
template <int MODE>
__global__ void __launch_bounds__(128, 2) pattern(double* out, int iters) {
  __shared__ double sm[2][64 * 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 2 * 64 * 32; i += blockDim.x) (&sm[0][0])[i] = 1.0 + i * 1e-7;
  __syncthreads();
  const int g = lane >> 2, q = lane & 3;
  const double* pa = &sm[0][((warp & 1) * 32 + g) * 32];
  const double* pb = &sm[1][((warp >> 1) * 32 + g) * 32];
  double accR[4][4][2] = {}, accI[4][4][2] = {};
  double a[4], br[4], bi[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) { a[i] = pa[i * 256 + q]; br[i] = pb[i * 256 + q]; bi[i] = pb[i * 256 + (q ^ 1)]; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      const int off = (s ^ g) << 2;
      if (MODE == 0) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          a[i] = __hiloint2double(__double2hiint(a[i]), __double2loint(a[i]) + 1);
          br[i] = __hiloint2double(__double2hiint(br[i]), __double2loint(br[i]) + 1);
          bi[i] = __hiloint2double(__double2hiint(bi[i]), __double2loint(bi[i]) + 1);
        }
      } else if (MODE == 1 || MODE == 2) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          a[i] = pa[i * 256 + off + q];
          br[i] = pb[i * 256 + off + q];
          bi[i] = pb[i * 256 + off + (q ^ 1)];
        }
      }
      double na[4], nbr[4], nbi[4];
      if (MODE == 3) {
        const int off2 = ((s + 1) & 7 ^ g) << 2;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          na[i] = pa[i * 256 + off2 + q];
          nbr[i] = pb[i * 256 + off2 + q];
          nbi[i] = pb[i * 256 + off2 + (q ^ 1)];
        }
      }
      if (MODE == 2) {
#pragma unroll
        for (int jb = 0; jb < 4; ++jb)
#pragma unroll
          for (int ib = 0; ib < 4; ++ib) {
            dmma(accR[ib][jb][0], accR[ib][jb][1], a[ib], br[jb]);
            dmma(accI[ib][jb][0], accI[ib][jb][1], a[ib], bi[jb]);
          }
      } else {
#pragma unroll
        for (int ib = 0; ib < 4; ++ib)
#pragma unroll
          for (int jb = 0; jb < 4; ++jb) {
            dmma(accR[ib][jb][0], accR[ib][jb][1], a[ib], br[jb]);
            dmma(accI[ib][jb][0], accI[ib][jb][1], a[ib], bi[jb]);
          }
      }
      if (MODE == 3) {
#pragma unroll
        for (int i = 0; i < 4; ++i) { a[i] = na[i]; br[i] = nbr[i]; bi[i] = nbi[i]; }
      }
    }
  }
  double sum = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) sum += accR[i][j][0] + accI[i][j][1];
  if (sum == 1234.5) out[threadIdx.x] = sum;
}

template <int MODE>
void run(const char* name, double* d, int sms) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int ctas : {1, 2}) {
    int iters = 2000;
    pattern<MODE><<<sms * ctas, 128>>>(d, 10);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    pattern<MODE><<<sms * ctas, 128>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 256 * 32 * 8 * (double)iters * 4 * sms * ctas;
    printf("{\"probe\": \"%s\", \"ctas_per_sm\": %d, \"tflops\": %.2f}\n", name, ctas, flops / ms / 1e9);
  }
}

int main() {
  double* d;
  cudaMalloc(&d, 4096);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0>("regs_varying", d, sms);
  run<1>("lds_ib_outer", d, sms);
  run<2>("lds_jb_outer", d, sms);
  run<3>("lds_prefetched", d, sms);
  cudaError_t e = cudaGetLastError();
  printf("{\"status\": \"%s\"}\n", cudaGetErrorString(e));
  return 0;
}
