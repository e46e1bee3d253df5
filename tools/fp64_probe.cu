// FP64 ceiling probe for sm_100a (B200).
//
// 1. Checks the register fragment layout of mma.sync.m8n8k4.f64 against a
//    host-side 8x8x4 product (the contraction kernels depend on it).
// 2. Measures the chip-wide DMMA and DFMA issue ceilings with register-only
//    loops (no memory traffic), timed with CUDA events.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_probe fp64_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__global__ void layout_kernel(const double* A, const double* B, double* D) {
  // A: 8x4 row-major, B: 4x8 col-major (B[k + 4*n]), D: 8x8 row-major.
  int lane = threadIdx.x;
  double a = A[(lane >> 2) * 4 + (lane & 3)];
  double b = B[(lane >> 2) * 4 + (lane & 3)];  // B[k = lane%4][n = lane/4]
  double d0 = 0, d1 = 0;
  dmma(d0, d1, a, b);
  D[(lane >> 2) * 8 + (lane & 3) * 2 + 0] = d0;
  D[(lane >> 2) * 8 + (lane & 3) * 2 + 1] = d1;
}

template <int NACC>
__global__ void dmma_loop(double* out, int iters) {
  double acc[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { acc[i][0] = 0; acc[i][1] = 0; }
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) dmma(acc[i][0], acc[i][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <int NACC>
__global__ void dfma_loop(double* out, int iters) {
  double acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = threadIdx.x;
  double a = 1.0 + threadIdx.x * 1e-9, b = 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i];
  if (s == 12345.0) out[threadIdx.x] = s;
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("{\"device\": \"%s\", \"sms\": %d, \"clock_khz_attr\": %d}\n", p.name, p.multiProcessorCount, clk_khz);

  // ---- layout check
  double hA[32], hB[32], hD[64], ref[64];
  for (int i = 0; i < 32; ++i) { hA[i] = (i * 7 % 11) - 5.0; hB[i] = (i * 5 % 13) - 6.0; }
  for (int m = 0; m < 8; ++m)
    for (int n = 0; n < 8; ++n) {
      double s = 0;
      for (int k = 0; k < 4; ++k) s += hA[m * 4 + k] * hB[n * 4 + k];
      ref[m * 8 + n] = s;
    }
  double *dA, *dB, *dD, *dO;
  CK(cudaMalloc(&dA, 256)); CK(cudaMalloc(&dB, 256)); CK(cudaMalloc(&dD, 512));
  CK(cudaMalloc(&dO, 4096));
  CK(cudaMemcpy(dA, hA, 256, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, hB, 256, cudaMemcpyHostToDevice));
  layout_kernel<<<1, 32>>>(dA, dB, dD);
  CK(cudaMemcpy(hD, dD, 512, cudaMemcpyDeviceToHost));
  double maxerr = 0;
  for (int i = 0; i < 64; ++i) maxerr = fmax(maxerr, fabs(hD[i] - ref[i]));
  printf("{\"dmma_layout_max_err\": %g}\n", maxerr);

  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int sms = p.multiProcessorCount;
  for (int warps : {4, 8, 16}) {
    for (int ctas_per_sm : {1, 2}) {
      int iters = 20000;
      int grid = sms * ctas_per_sm;
      dmma_loop<8><<<grid, 32 * warps>>>(dO, 100);
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      dmma_loop<8><<<grid, 32 * warps>>>(dO, iters);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 256.0 * 8 * (double)iters * warps * grid;
      printf("{\"probe\": \"dmma_m8n8k4\", \"warps_per_cta\": %d, \"ctas_per_sm\": %d, \"ms\": %.3f, \"tflops\": %.2f}\n",
             warps, ctas_per_sm, ms, flops / ms / 1e9);
    }
  }
  for (int warps : {8, 16, 32}) {
    int iters = 20000, grid = sms * 2;
    dfma_loop<8><<<grid, 32 * warps>>>(dO, 100);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dfma_loop<8><<<grid, 32 * warps>>>(dO, iters);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 32.0 * 8 * (double)iters * warps * grid;
    printf("{\"probe\": \"dfma\", \"warps_per_cta\": %d, \"ctas_per_sm\": 2, \"ms\": %.3f, \"tflops\": %.2f}\n",
           warps, ms, flops / ms / 1e9);
  }
  // Sustained: run the DMMA loop ~3 s so the clock sampler sees FP64 load.
  {
    int warps = 8, grid = sms * 2, iters = 400000;
    cudaEventRecord(e0);
    for (int r = 0; r < 8; ++r) dmma_loop<8><<<grid, 32 * warps>>>(dO, iters);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 8 * 2.0 * 256.0 * 8 * (double)iters * warps * grid;
    printf("{\"probe\": \"dmma_sustained\", \"ms\": %.3f, \"tflops\": %.2f}\n", ms, flops / ms / 1e9);
  }
  return 0;
}
