// Per-shape timing of the 3xTF32 GEMM variants on the cfg3 shapes (tuning
// aid, not a test): forward (K-major x K-major), dgrad (K-major x MN-major),
// wgrad (MN-major x MN-major). Prints algorithmic TFLOP/s and the tensor-pipe
// equivalent (6x) for the 1-CTA and the CTA-pair kernels.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I include \
//        -o build/gemm_bench tests/native/gemm_bench.cu paper_2111_10672_b200/csrc/gemm.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <string>
#include <vector>

#include "../../paper_2111_10672_b200/csrc/gemm_tf32x3.cuh"
#include "../../paper_2111_10672_b200/csrc/launch.hpp"

using namespace spb;

int main(int argc, char** argv) {
  const int reps = argc > 1 ? atoi(argv[1]) : 20;
  struct Shape {
    const char* name;
    int M, N, K;
    bool am, bm;
    int epi;
  };
  std::vector<Shape> shapes;
  const bool sweep = argc > 2 && std::string(argv[2]) == "sweep";
  if (sweep) {  // plan sweep over the SPB shapes at 1 / 2 / 4 GPUs (planner calibration)
    for (int m : {256, 512, 1024}) shapes.push_back({"fwd", m, 4096, 4096, false, false, kEpiFwdTanh});
    for (int q : {1, 2, 3, 4, 5, 6, 7}) shapes.push_back({"dgrad", 128 * q, 4096, 4096, false, true, kEpiDgradTanh});
    for (int q : {1, 2, 3, 4, 5, 6, 8}) shapes.push_back({"wgrad", 4096, 4096, 128 * q, true, true, kEpiStoreScaled});
  } else {
    shapes.push_back({"fwd", 1024, 4096, 4096, false, false, kEpiFwdTanh});
    for (int q : {1, 2, 3, 4, 7}) shapes.push_back({"dgrad", 128 * q, 4096, 4096, false, true, kEpiDgradTanh});
    for (int m : {1, 2, 4, 8}) shapes.push_back({"wgrad", 4096, 4096, 128 * m, true, true, kEpiStoreScaled});
    for (int m : {1, 4, 8}) shapes.push_back({"wgupd", 4096, 4096, 128 * m, true, true, kEpiWgradUpdate});
  }
  struct P {
    int two, pn, sp;
  };
  std::vector<P> plans = {{-1, 0, 0}, {0, 0, 1}, {1, 256, 1}};
  if (sweep) {
    plans = {{-1, 0, 0}};
    for (int sp : {1, 2, 4}) plans.push_back({0, 128, sp});
    for (int pn : {192, 240, 256})
      for (int sp : {1, 2, 4}) plans.push_back({1, pn, sp});
  }
  const long big = 4096L * 4096;
  float *ah, *al, *bh, *bl, *out, *oh, *ol;
  cudaMalloc(&ah, big * 4), cudaMalloc(&al, big * 4), cudaMalloc(&bh, big * 4), cudaMalloc(&bl, big * 4);
  cudaMalloc(&out, big * 4), cudaMalloc(&oh, big * 4), cudaMalloc(&ol, big * 4);
  cudaMemset(ah, 0, big * 4), cudaMemset(al, 0, big * 4), cudaMemset(bh, 0, big * 4), cudaMemset(bl, 0, big * 4);
  cudaMemset(oh, 0, big * 4), cudaMemset(ol, 0, big * 4);
  float* ws;
  const long ws_floats = 16L << 20;
  cudaMalloc(&ws, ws_floats * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0), cudaEventCreate(&e1);
  for (auto& sh : shapes) {
    for (const P& pl : plans) {
      if (pl.two < 0) gemm_force_plan(0, 0, 0);
      else gemm_force_plan(pl.two, pl.pn, pl.sp);
      if (pl.sp > 1 && sh.epi == kEpiWgradUpdate) continue;
      Operand A{ah, al, sh.am ? sh.M : sh.K, sh.M, sh.K, sh.am};
      Operand B{bh, bl, sh.bm ? sh.N : sh.K, sh.N, sh.K, sh.bm};
      GemmEpilogue ep{};
      ep.out_hi = sh.epi == kEpiStoreScaled ? out : oh;
      ep.out_lo = ol;
      ep.ld_out = sh.N;
      ep.bias_hi = bh;
      ep.bias_lo = bl;
      ep.h_hi = ah;
      ep.h_lo = al;
      ep.ld_h = sh.N;
      ep.alpha = 1.f;
      ep.M = sh.M;
      ep.N = sh.N;
      ep.splitk_ws = ws;
      ep.splitk_ws_floats = ws_floats;
      if (sh.epi == kEpiWgradUpdate) {
        ep.out_hi = oh;
        ep.mom = out;
        ep.lr = 1e-3f;
        ep.mu = 0.9f;
        ep.wd = 1e-4f;
      }
      for (int i = 0; i < 3; ++i) gemm_tf32x3(A, B, sh.epi, ep, 0);
      cudaEventRecord(e0);
      for (int i = 0; i < reps; ++i) gemm_tf32x3(A, B, sh.epi, ep, 0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const double us = 1e3 * ms / reps;
      const double tf = 2.0 * sh.M * sh.N * sh.K / (us * 1e-6) / 1e12;
      char tag[32];
      if (pl.two < 0) std::snprintf(tag, sizeof tag, "auto");
      else std::snprintf(tag, sizeof tag, "%s pn=%d sp=%d", pl.two ? "2sm" : "1sm", pl.two ? pl.pn : 128, pl.sp);
      std::printf("%-6s %-18s M=%5d N=%5d K=%5d  %8.1f us  alg %6.1f TF/s  pipe %7.1f TF/s  %s\n", sh.name, tag, sh.M,
                  sh.N, sh.K, us, tf, 6 * tf, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
