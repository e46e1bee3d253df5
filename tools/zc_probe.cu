// Probe (GPU, not a test): how fast SM stores reach pinned host memory over PCIe, against a
// DMA copy of the same bytes.  Decides whether the contraction epilogue should store
// synchronous-call results straight to the host (zero-copy) instead of a copy after it.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/zc_probe tools/zc_probe.cu
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

// contiguous: every warp stores 512 contiguous bytes per instruction
__global__ void store_lin(double2* __restrict__ dst, long long n) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride)
    dst[i] = make_double2((double)i, 1.0);
}

// epilogue pattern: a 64x64 complex tile per CTA (column-major, ld), each warp instruction
// writes 8 columns x 8 rows (8 x 128 B segments), as the DMMA fragment layout does
__global__ void store_tiles(double2* __restrict__ dst, int n, long long ld) {
  const int tiles = (n + 63) / 64;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  for (int t = blockIdx.x; t < tiles * tiles; t += gridDim.x) {
    const int ti = t % tiles, tj = t / tiles;
    const int wm = warp & 1, wn = warp >> 1;  // 4 warps: 2 x 2 of 32 x 32
    for (int ib = 0; ib < 4; ++ib)
      for (int jb = 0; jb < 4; ++jb)
        for (int v = 0; v < 2; ++v) {
          const int i = ti * 64 + wm * 32 + ib * 8 + g;
          const int j = tj * 64 + wn * 32 + jb * 8 + 2 * q + v;
          if (i < n && j < n) dst[i + (long long)j * ld] = make_double2(i, j);
        }
  }
}

int main() {
  const int n = 2999;
  const long long elems = (long long)n * n;
  const size_t bytes = elems * sizeof(double2);
  double2 *h, *d;
  cudaHostAlloc(&h, bytes, cudaHostAllocDefault);
  cudaMalloc(&d, bytes);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto timeit = [&](const char* what, auto fn) {
    for (int w = 0; w < 2; ++w) fn();
    cudaStreamSynchronize(s);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0, s);
      fn();
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    printf("%-40s %.3f ms  %.1f GB/s\n", what, best, bytes / (best * 1e6));
  };
  timeit("DMA D2H (cudaMemcpyAsync)", [&] { cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, s); });
  for (int blocks : {sms, 2 * sms, 8 * sms})
    for (int thr : {128, 256}) {
      char lbl[64];
      snprintf(lbl, sizeof lbl, "SM linear stores %dx%d", blocks, thr);
      timeit(lbl, [&] { store_lin<<<blocks, thr, 0, s>>>(h, elems); });
    }
  for (int blocks : {sms, 2 * sms}) {
    char lbl[64];
    snprintf(lbl, sizeof lbl, "SM tile stores %dx128", blocks);
    timeit(lbl, [&] { store_tiles<<<blocks, 128, 0, s>>>(h, n, n); });
  }
  // strided runs: every column of the n x n matrix written as runs of `run` bytes (SM stores
  // and 2D DMA copies), to separate run length from address pattern
  for (long long run : {1024LL, 3072LL, 12288LL, 49152LL}) {
    const long long per_col = (long long)n * sizeof(double2) / run;  // runs per column
    char lbl[80];
    snprintf(lbl, sizeof lbl, "DMA 2D D2H, %lld-B runs, pitch 48 KB", run);
    // rows of the 2D copy = column pieces: copy piece r of every column as one 2D copy
    timeit(lbl, [&] {
      for (long long r = 0; r < per_col; ++r)
        cudaMemcpy2DAsync((char*)h + r * run, n * sizeof(double2), (char*)d + r * run,
                          n * sizeof(double2), run, n, cudaMemcpyDeviceToHost, s);
    });
  }
  // the same pieces spread over several copy streams (engines) at once
  {
    cudaStream_t ss[4];
    cudaEvent_t fk;
    cudaEventCreateWithFlags(&fk, cudaEventDisableTiming);
    std::vector<cudaEvent_t> jn(4);
    for (int k = 0; k < 4; ++k) {
      cudaStreamCreateWithFlags(&ss[k], cudaStreamNonBlocking);
      cudaEventCreateWithFlags(&jn[k], cudaEventDisableTiming);
    }
    for (long long run : {1024LL, 4096LL})
      for (int ns : {1, 2, 4}) {
        const long long per_col = (long long)n * sizeof(double2) / run;
        char lbl[80];
        snprintf(lbl, sizeof lbl, "DMA 2D %lld-B runs on %d streams (96%%+ bytes)", run, ns);
        timeit(lbl, [&] {
          cudaEventRecord(fk, s);
          for (int k = 0; k < ns; ++k) cudaStreamWaitEvent(ss[k], fk, 0);
          for (long long r = 0; r < per_col; ++r)
            cudaMemcpy2DAsync((char*)h + r * run, n * sizeof(double2), (char*)d + r * run,
                              n * sizeof(double2), run, n, cudaMemcpyDeviceToHost, ss[r % ns]);
          for (int k = 0; k < ns; ++k) {
            cudaEventRecord(jn[k], ss[k]);
            cudaStreamWaitEvent(s, jn[k], 0);
          }
        });
      }
  }
  timeit("SM tile stores to HBM 296x128", [&] { store_tiles<<<2 * sms, 128, 0, s>>>(d, n, n); });
  cudaError_t err = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(err));
  return err == cudaSuccess ? 0 : 1;
}
