// Phase timing of tjoint_kernel (joint T factor) on one T set: builds small.cu with clock64
// phase points (HSDLA_PROF_POINT) and prints cycles per phase.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/exp/tjoint_bench \
//        tools/exp_tjoint_bench.cu && tools/exp/tjoint_bench 81
#include <cstdio>
#include <cstdlib>
#include <random>
#include <string>
#include <vector>

__device__ long long g_prof[16];
__device__ long long g_last;
#define HSDLA_PROF_START() \
  do { if (threadIdx.x == 0 && blockIdx.x == 0) g_last = clock64(); } while (0)
#define HSDLA_PROF_POINT(i)                                              \
  do {                                                                   \
    if (threadIdx.x == 0 && blockIdx.x == 0) {                           \
      long long _t = clock64();                                          \
      g_prof[i] += _t - g_last;                                          \
      g_last = _t;                                                       \
    }                                                                    \
  } while (0)
#include "../paper_1602_06589_b200/csrc/small.cu"

namespace hsdla {
void set_error(const std::string&) {}
}

int main(int argc, char** argv) {
  const int m = argc > 1 ? atoi(argv[1]) : 81;
  std::mt19937_64 rng(5);
  std::normal_distribution<double> nd;
  std::vector<double2> taa(m * m), tab(m * m), tbb(m * m);
  for (auto* t : {&taa, &tbb})
    for (int c = 0; c < m; ++c)
      for (int r = 0; r < m; ++r) (*t)[r + c * m] = make_double2(nd(rng) / m + (r == c ? 2.0 : 0.0), r == c ? 0.0 : nd(rng) / m);
  for (auto& v : tab) v = make_double2(nd(rng) / m, nd(rng) / m);
  double2 *dA, *dB, *dC, *J;
  int *tdim, *info;
  double* sig;
  cudaMalloc(&dA, m * m * 16); cudaMalloc(&dB, m * m * 16); cudaMalloc(&dC, m * m * 16);
  cudaMalloc(&J, 4 * m * m * 16); cudaMalloc(&tdim, 8); cudaMalloc(&info, 8); cudaMalloc(&sig, 200 * 8);
  cudaMemcpy(dA, taa.data(), m * m * 16, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, tab.data(), m * m * 16, cudaMemcpyHostToDevice);
  cudaMemcpy(dC, tbb.data(), m * m * 16, cudaMemcpyHostToDevice);
  cudaMemcpy(tdim, &m, 4, cudaMemcpyHostToDevice);
  if (hsdla::preload_small()) { printf("preload failed\n"); return 1; }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int it = 0; it < 4; ++it) {
    long long z[16] = {};
    cudaMemcpyToSymbol(g_prof, z, sizeof(z));
    cudaEventRecord(e0);
    hsdla::launch_tjoint(0, 1, tdim, nullptr, m, dA, dB, dC, m, J, info, nullptr, nullptr, nullptr, -1.0, sig);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaMemcpyFromSymbol(z, g_prof, sizeof(z));
    int inf = 0;
    cudaMemcpy(&inf, info, 4, cudaMemcpyDeviceToHost);
    std::vector<double2> Jh(4 * m * m);
    cudaMemcpy(Jh.data(), J, 4 * m * m * 16, cudaMemcpyDeviceToHost);
    double cks = 0.0;
    for (size_t q = 0; q < Jh.size(); ++q) cks += Jh[q].x * (1.0 + 1e-3 * (q % 97)) - Jh[q].y * (1.0 + 1e-3 * (q % 89));
    printf("checksum %.17g ", cks);
    printf("m=%d n=%d: %.1f us info %d | cycles: gersh+split %lld, assemble %lld, nan %lld, stage %lld, panel %lld, writeback %lld, trailing %lld, zero+rest %lld | panel: diag %lld rows %lld update %lld\n",
           m, 2 * m, ms * 1e3, inf, z[7], z[8], z[1], z[2], z[3], z[4], z[5], z[6], z[9], z[10], z[11]);
  }
  return 0;
}
