// Bandwidth of the fused optimizer-update kernel vs the number of CTAs
// (tuning aid). Measured on B200: one SM streams at most ~44 GB/s, so the
// update needs ~all 148 SMs to approach HBM peak; it cannot hide in the SMs a
// GEMM leaves idle.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I include \
//        -o build/update_bench tests/native/update_bench.cu paper_2111_10672_b200/csrc/kernels.cu
#include <cuda_runtime.h>

#include <cstdio>

#include "../../paper_2111_10672_b200/csrc/launch.hpp"

using namespace spb;

int main() {
  const long n = 4096L * 4096;
  float *hi, *lo, *g, *m;
  cudaMalloc(&hi, n * 4), cudaMalloc(&lo, n * 4), cudaMalloc(&g, n * 4), cudaMalloc(&m, n * 4);
  cudaMemset(hi, 0, n * 4), cudaMemset(lo, 0, n * 4), cudaMemset(g, 0, n * 4), cudaMemset(m, 0, n * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a), cudaEventCreate(&b);
  const double bytes = n * 28.0;  // r: hi, lo, g, mom; w: hi, lo, mom
  for (int ctas : {8, 20, 40, 74, 148, 296, 1184}) {
    launch_sgd_update(hi, lo, g, m, n, 1e-3f, 0.9f, 1e-4f, 0, ctas);
    cudaEventRecord(a);
    for (int i = 0; i < 10; ++i) launch_sgd_update(hi, lo, g, m, n, 1e-3f, 0.9f, 1e-4f, 0, ctas);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double gbs = bytes / (ms / 10 * 1e-3) / 1e9;
    std::printf("update %5d CTAs x 256 thr: %7.1f us  %6.0f GB/s  (%5.1f GB/s per SM used) %s\n", ctas,
                1e3 * ms / 10, gbs, gbs / (ctas < 148 ? ctas : 148), cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
