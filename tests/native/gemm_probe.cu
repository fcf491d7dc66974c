// Standalone numerics probe of the tcgen05 3xTF32 GEMM for every operand
// majorness, against an fp64 host reference (a torch-free stand-in for the
// "plain fp32 reference" of a floating-point kernel). Built and run by
// tests/test_native.py (nvcc -gencode arch=compute_100a,code=sm_100a with
// paper_2111_10672_b200/csrc/gemm.cu).
// Prints one line per case: "case am bm M N K rel_err max_abs_err" and exits
// non-zero if any case exceeds 2e-6 norm-wise relative error.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "../../paper_2111_10672_b200/csrc/gemm_tf32x3.cuh"
#include "../../paper_2111_10672_b200/csrc/launch.hpp"

using namespace spb;

static float rna(float x) {  // host cvt.rna.tf32.f32
  uint32_t u;
  std::memcpy(&u, &x, 4);
  u = (u + 0x1000u) & ~0x1FFFu;
  float r;
  std::memcpy(&r, &u, 4);
  return r;
}

struct Dev {
  float *hi, *lo;
};

// Stores logical X[mn][k] in the requested majorness with ld padding.
static Dev upload(const std::vector<float>& X, int mn, int k, bool mn_major, long& ld) {
  const long rows = mn_major ? k : mn, cols = mn_major ? mn : k;
  ld = (cols + 3) / 4 * 4 + 4;  // deliberately padded
  std::vector<float> h(rows * ld, 0.f), l(rows * ld, 0.f);
  for (int i = 0; i < mn; ++i)
    for (int j = 0; j < k; ++j) {
      const float v = X[static_cast<long>(i) * k + j];
      const long at = mn_major ? static_cast<long>(j) * ld + i : static_cast<long>(i) * ld + j;
      h[at] = rna(v);
      l[at] = v - h[at];
    }
  Dev d;
  cudaMalloc(&d.hi, h.size() * 4);
  cudaMalloc(&d.lo, l.size() * 4);
  cudaMemcpy(d.hi, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(d.lo, l.data(), l.size() * 4, cudaMemcpyHostToDevice);
  return d;
}

int main() {
  struct Case {
    int M, N, K;
  };
  const Case cases[] = {{200, 300, 100}, {128, 128, 32}, {5, 7, 3}, {1024, 1024, 1024}, {333, 129, 517}, {256, 384, 4096}, {130, 260, 8192}};
  int bad = 0;
  float *ws, *zb, *outh, *outl;
  const long ws_floats = 16L << 20;
  cudaMalloc(&ws, ws_floats * 4);
  cudaMalloc(&zb, 16384 * 4);
  cudaMemset(zb, 0, 16384 * 4);
  cudaMalloc(&outh, 8L << 20);
  cudaMalloc(&outl, 8L << 20);
  std::mt19937_64 rng(1234);
  std::uniform_real_distribution<float> U(-1.f, 1.f);
  for (const Case& c : cases) {
    std::vector<float> A(static_cast<long>(c.M) * c.K), B(static_cast<long>(c.N) * c.K);
    for (auto& v : A) v = U(rng);
    for (auto& v : B) v = U(rng);
    std::vector<double> R(static_cast<long>(c.M) * c.N, 0.0);
    for (int i = 0; i < c.M; ++i)
      for (int j = 0; j < c.N; ++j) {
        double s = 0;
        for (int q = 0; q < c.K; ++q) s += static_cast<double>(A[static_cast<long>(i) * c.K + q]) * B[static_cast<long>(j) * c.K + q];
        R[static_cast<long>(i) * c.N + j] = s;
      }
    // variant -1 auto, 0 1-CTA, 1 pair 256; >= 2: forced plans (pair tile
    // widths 192 / 240 / 256, K-splits on both kernels).
    struct Forced {
      int two, pn, sp;
    };
    const Forced forced[] = {{1, 192, 1}, {1, 192, 3}, {1, 240, 2}, {1, 256, 4}, {0, 128, 3}};
    for (int variant = -1; variant < 2 + 5; ++variant)
    for (int am = 0; am < 2; ++am)
      for (int bm = 0; bm < 2; ++bm) {
        if (variant >= 2 && forced[variant - 2].two && forced[variant - 2].pn < 240 && am && !bm) continue;
        gemm_force_variant(variant < 2 ? variant : -1);
        if (variant >= 2) gemm_force_plan(forced[variant - 2].two, forced[variant - 2].pn, forced[variant - 2].sp);
        else gemm_force_plan(0, 0, 0);
        long lda, ldb;
        Dev a = upload(A, c.M, c.K, am, lda), b = upload(B, c.N, c.K, bm, ldb);
        float* out;
        const long ldo = (c.N + 3) / 4 * 4;
        cudaMalloc(&out, static_cast<long>(c.M) * ldo * 4);
        cudaMemset(out, 0, static_cast<long>(c.M) * ldo * 4);
        Operand OA{a.hi, a.lo, lda, c.M, c.K, am != 0}, OB{b.hi, b.lo, ldb, c.N, c.K, bm != 0};
        // variant -1: the automatic plan through the split-K path (linear
        // epilogue with zero bias == the plain product).
        GemmEpilogue ep{};
        ep.out_hi = variant < 0 ? outh : out;
        ep.out_lo = outl;
        ep.ld_out = ldo;
        ep.alpha = 1.0f;
        ep.M = c.M;
        ep.N = c.N;
        ep.bias_hi = zb;
        ep.bias_lo = zb;
        ep.splitk_ws = ws;
        ep.splitk_ws_floats = ws_floats;
        gemm_tf32x3(OA, OB, variant < 0 ? kEpiFwdLinear : kEpiStoreScaled, ep, 0);
        if (variant < 0) {  // out = hi + lo
          std::vector<float> h(static_cast<long>(c.M) * ldo), l2(h.size());
          cudaMemcpy(h.data(), outh, h.size() * 4, cudaMemcpyDeviceToHost);
          cudaMemcpy(l2.data(), outl, l2.size() * 4, cudaMemcpyDeviceToHost);
          for (size_t i = 0; i < h.size(); ++i) h[i] += l2[i];
          cudaMemcpy(out, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
        }
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<float> got(static_cast<long>(c.M) * ldo);
        cudaMemcpy(got.data(), out, got.size() * 4, cudaMemcpyDeviceToHost);
        double num = 0, den = 0, mx = 0;
        for (int i = 0; i < c.M; ++i)
          for (int j = 0; j < c.N; ++j) {
            const double d = got[static_cast<long>(i) * ldo + j] - R[static_cast<long>(i) * c.N + j];
            num += d * d;
            den += R[static_cast<long>(i) * c.N + j] * R[static_cast<long>(i) * c.N + j];
            mx = std::max(mx, std::fabs(d));
          }
        const double rel = std::sqrt(num / (den > 0 ? den : 1));
        char tag[40];
        if (variant < 2) std::snprintf(tag, sizeof tag, "%s", variant < 0 ? "auto" : variant ? "2sm" : "1sm");
        else std::snprintf(tag, sizeof tag, "%s/pn%d/sp%d", forced[variant - 2].two ? "2sm" : "1sm", forced[variant - 2].pn,
                           forced[variant - 2].sp);
        std::printf("case %s am=%d bm=%d M=%d N=%d K=%d rel_err=%.3e max_abs=%.3e %s\n", tag, am, bm,
                    c.M, c.N, c.K, rel, mx,
                    e == cudaSuccess ? "" : cudaGetErrorString(e));
        if (!(rel <= 2e-6) || e != cudaSuccess) ++bad;
        cudaFree(a.hi), cudaFree(a.lo), cudaFree(b.hi), cudaFree(b.lo), cudaFree(out);
      }
  }
  gemm_force_plan(0, 0, 0);
  std::printf("%s\n", bad ? "GEMM PROBE FAILED" : "GEMM PROBE OK");
  return bad ? 1 : 0;
}
