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
#include <thread>
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

// ---- "shapes": the exact GEMM shapes, layouts, epilogues and automatic plans
// of the benchmarked cfg3 step (4096-wide layers, k = 8 x 128 rows; 1 / 2 / 4
// GPUs give M = 1024 / 512 / 256 rows per rank), against fp64 host references
// of the full epilogue. Prints the plan the planner chose for each launch.

static void upload_exact(const std::vector<float>& X, long rows, long cols, float** hi, float** lo) {
  std::vector<float> h(rows * cols), l(rows * cols);
  for (long i = 0; i < rows * cols; ++i) h[i] = rna(X[i]), l[i] = X[i] - h[i];
  cudaMalloc(hi, h.size() * 4);
  cudaMalloc(lo, l.size() * 4);
  cudaMemcpy(*hi, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(*lo, l.data(), l.size() * 4, cudaMemcpyHostToDevice);
}

// C[i][j] = sum_q a(i, q) * b(j, q) in fp64 over all host threads.
template <class FA, class FB>
static std::vector<double> host_gemm(int M, int N, int K, FA a, FB b) {
  std::vector<double> C(static_cast<long>(M) * N);
  const int T = std::max(1u, std::thread::hardware_concurrency());
  std::vector<std::thread> pool;
  for (int t = 0; t < T; ++t)
    pool.emplace_back([&, t] {
      std::vector<double> arow(K);
      for (int i = t; i < M; i += T) {
        for (int q = 0; q < K; ++q) arow[q] = a(i, q);
        for (int j = 0; j < N; ++j) {
          double s0 = 0, s1 = 0, s2 = 0, s3 = 0;  // four chains: fp64 either way, 4x the throughput
          int q = 0;
          for (; q + 4 <= K; q += 4) {
            s0 += arow[q] * b(j, q);
            s1 += arow[q + 1] * b(j, q + 1);
            s2 += arow[q + 2] * b(j, q + 2);
            s3 += arow[q + 3] * b(j, q + 3);
          }
          for (; q < K; ++q) s0 += arow[q] * b(j, q);
          C[static_cast<long>(i) * N + j] = (s0 + s1) + (s2 + s3);
        }
      }
    });
  for (auto& th : pool) th.join();
  return C;
}

static std::vector<float> rand_vec(long n, std::mt19937_64& rng, float scale) {
  std::uniform_real_distribution<float> U(-scale, scale);
  std::vector<float> v(n);
  for (auto& x : v) x = U(rng);
  return v;
}

static std::vector<float> fetch_pair(const float* hi, const float* lo, long n) {
  std::vector<float> h(n), l(n);
  cudaMemcpy(h.data(), hi, n * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(l.data(), lo, n * 4, cudaMemcpyDeviceToHost);
  for (long i = 0; i < n; ++i) h[i] += l[i];
  return h;
}

static double rel_err(const std::vector<float>& got, const std::vector<double>& want) {
  double num = 0, den = 0;
  for (size_t i = 0; i < want.size(); ++i) {
    const double d = got[i] - want[i];
    num += d * d;
    den += want[i] * want[i];
  }
  return std::sqrt(num / (den > 0 ? den : 1));
}

static int report(const char* name, int M, int N, int K, double rel, double tol) {
  int two, pn, sp;
  gemm_last_plan(&two, &pn, &sp);
  const cudaError_t e = cudaDeviceSynchronize();
  std::printf("shape %-28s M=%d N=%d K=%d plan=%s/pn%d/sp%d rel_err=%.3e %s\n", name, M, N, K, two ? "2sm" : "1sm", pn, sp,
              rel, e == cudaSuccess ? "" : cudaGetErrorString(e));
  return (rel <= tol && e == cudaSuccess) ? 0 : 1;
}

static int run_shapes() {
  const int n = 4096;
  int bad = 0;
  gemm_prepare_device();  // the fused-bias ones boxes
  std::mt19937_64 rng(77);
  float *ws;
  const long ws_floats = 64L << 20;  // room for the forced 3-way split-K of a 4096 x 4097 wgrad
  cudaMalloc(&ws, ws_floats * 4);
  // Weights U(+-1/64) like make_random_chain_mlp's U(-1/sqrt(n), 1/sqrt(n)); activations in (-1, 1).
  std::vector<float> W = rand_vec(static_cast<long>(n) * n, rng, 1.f / 64), bias = rand_vec(n, rng, 1.f / 64);
  float *Wh, *Wl, *bh, *bl;
  upload_exact(W, n, n, &Wh, &Wl);
  upload_exact(bias, 1, n, &bh, &bl);
  for (int M : {1024, 512, 256}) {  // forward: H_l = tanh(H_{l-1} W^T + b) (kEpiFwdTanh)
    std::vector<float> H = rand_vec(static_cast<long>(M) * n, rng, 1.f);
    float *Hh, *Hl, *Oh, *Ol;
    upload_exact(H, M, n, &Hh, &Hl);
    cudaMalloc(&Oh, static_cast<long>(M) * n * 4);
    cudaMalloc(&Ol, static_cast<long>(M) * n * 4);
    GemmEpilogue ep{};
    ep.out_hi = Oh, ep.out_lo = Ol, ep.ld_out = n, ep.bias_hi = bh, ep.bias_lo = bl, ep.M = M, ep.N = n;
    ep.splitk_ws = ws, ep.splitk_ws_floats = ws_floats;
    gemm_tf32x3(Operand{Hh, Hl, n, M, n, false}, Operand{Wh, Wl, n, n, n, false}, kEpiFwdTanh, ep, 0);
    auto R = host_gemm(M, n, n, [&](int i, int q) { return static_cast<double>(H[static_cast<long>(i) * n + q]); },
                       [&](int j, int q) { return static_cast<double>(W[static_cast<long>(j) * n + q]); });
    for (long i = 0; i < static_cast<long>(M) * n; ++i) R[i] = std::tanh(R[i] + bias[i % n]);
    bad += report("forward (tanh epilogue)", M, n, n, rel_err(fetch_pair(Oh, Ol, static_cast<long>(M) * n), R), 2e-6);
    // dgrad: Delta_{l-1} = (Delta_l W_l) * (1 - H^2) (kEpiDgradTanh), Delta K-major, W MN-major.
    for (int Md : {M / 8, M / 4, M / 2}) {
      std::vector<float> D = rand_vec(static_cast<long>(Md) * n, rng, 1e-3f);
      float *Dh, *Dl;
      upload_exact(D, Md, n, &Dh, &Dl);
      GemmEpilogue ed{};
      ed.out_hi = Oh, ed.out_lo = Ol, ed.ld_out = n, ed.h_hi = Hh, ed.h_lo = Hl, ed.ld_h = n, ed.M = Md, ed.N = n;
      ed.splitk_ws = ws, ed.splitk_ws_floats = ws_floats;
      gemm_tf32x3(Operand{Dh, Dl, n, Md, n, false}, Operand{Wh, Wl, n, n, n, true}, kEpiDgradTanh, ed, 0);
      auto Rd = host_gemm(Md, n, n, [&](int i, int q) { return static_cast<double>(D[static_cast<long>(i) * n + q]); },
                          [&](int j, int q) { return static_cast<double>(W[static_cast<long>(q) * n + j]); });
      for (long i = 0; i < static_cast<long>(Md) * n; ++i) {
        const double h = H[i];  // H as stored (hi + lo == H exactly)
        Rd[i] *= 1.0 - h * h;
      }
      char nm[64];
      std::snprintf(nm, sizeof nm, "dgrad (1-H^2 epilogue)");
      bad += report(nm, Md, n, n, rel_err(fetch_pair(Oh, Ol, static_cast<long>(Md) * n), Rd), 2e-6);
      cudaFree(Dh), cudaFree(Dl);
    }
    cudaFree(Hh), cudaFree(Hl), cudaFree(Oh), cudaFree(Ol);
  }
  // wgrad over K contributor rows: dW = alpha Delta^T H (MN x MN, kEpiStoreScaled);
  // K = 1024 is the 8-contributor layer of the 1-GPU step.
  for (int K : {1024, 768, 512, 256, 128}) {
    std::vector<float> D = rand_vec(static_cast<long>(K) * n, rng, 1e-3f), H = rand_vec(static_cast<long>(K) * n, rng, 1.f);
    float *Dh, *Dl, *Hh, *Hl, *G;
    upload_exact(D, K, n, &Dh, &Dl);
    upload_exact(H, K, n, &Hh, &Hl);
    cudaMalloc(&G, static_cast<long>(n) * n * 4);
    const float alpha = 1.0f / K;
    auto R = host_gemm(n, n, K, [&](int i, int q) { return static_cast<double>(D[static_cast<long>(q) * n + i]); },
                       [&](int j, int q) { return static_cast<double>(H[static_cast<long>(q) * n + j]); });
    GemmEpilogue ep{};
    ep.out_hi = G, ep.ld_out = n, ep.alpha = alpha, ep.M = n, ep.N = n;
    ep.splitk_ws = ws, ep.splitk_ws_floats = ws_floats;
    gemm_tf32x3(Operand{Dh, Dl, n, n, K, true}, Operand{Hh, Hl, n, n, K, true}, kEpiStoreScaled, ep, 0);
    std::vector<float> got(static_cast<long>(n) * n);
    cudaDeviceSynchronize();
    cudaMemcpy(got.data(), G, got.size() * 4, cudaMemcpyDeviceToHost);
    std::vector<double> Ra(R.size());
    for (size_t i = 0; i < R.size(); ++i) Ra[i] = R[i] * alpha;
    bad += report("wgrad (alpha epilogue)", n, n, K, rel_err(got, Ra), 2e-6);
    {  // bias fused as the virtual ones column 4096 of B: [dW | db] in one GEMM, on the
       // automatic plan and forced 1-CTA split-K / pair plans (split-K routes the bias in the fixup)
      std::vector<double> Rb(n, 0.0);
      for (int q = 0; q < K; ++q)
        for (int i = 0; i < n; ++i) Rb[i] += D[static_cast<long>(q) * n + i];
      for (double& v : Rb) v *= alpha;
      float* gb;
      cudaMalloc(&gb, n * 4);
      const struct { int two, pn, sp; } fp[] = {{-1, 0, 0}, {0, 128, 3}, {0, 128, 1}, {0, 128, 1}, {1, 192, 2}, {1, 256, 1}};
      for (const auto& f : fp) {
        if (f.two >= 0 && K != 1024) continue;
        if (f.two >= 0) gemm_force_plan(f.two, f.pn, f.sp);
        cudaMemset(G, 0, static_cast<long>(n) * n * 4);
        cudaMemset(gb, 0, n * 4);
        GemmEpilogue eb{};
        eb.out_hi = G, eb.ld_out = n, eb.alpha = alpha, eb.M = n, eb.N = n, eb.gb_hi = gb;
        eb.bias_col_p1 = eb.ones_col_p1 = n + 1;
        eb.splitk_ws = ws, eb.splitk_ws_floats = ws_floats;
        Operand OB{Hh, Hl, n, n + 1, K, true, n};
        gemm_tf32x3(Operand{Dh, Dl, n, n, K, true}, OB, kEpiStoreScaled, eb, 0);
        cudaDeviceSynchronize();
        gemm_force_plan(0, 0, 0);
        std::vector<float> gw(static_cast<long>(n) * n), gbh(n);
        cudaMemcpy(gw.data(), G, gw.size() * 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(gbh.data(), gb, n * 4, cudaMemcpyDeviceToHost);
        const double e = std::max(rel_err(gw, Ra), rel_err(gbh, Rb));
        bad += report(f.two < 0 ? "wgrad + fused bias" : "wgrad + fused bias (forced)", n, n + 1, K, e, 2e-6);
      }
      cudaFree(gb);
    }
    if (K <= 512) {  // the fused optimizer epilogue of the <= 512-row layers: W -= lr (mu buf + g + wd W)
      std::vector<float> M0 = rand_vec(static_cast<long>(n) * n, rng, 1e-4f);
      float *Uh, *Ul, *Mom;
      upload_exact(W, n, n, &Uh, &Ul);
      cudaMalloc(&Mom, M0.size() * 4);
      cudaMemcpy(Mom, M0.data(), M0.size() * 4, cudaMemcpyHostToDevice);
      // with the bias fused (ones column): b -= lr (mu mb + g_b + wd b) on its split pair
      std::vector<float> b0 = rand_vec(n, rng, 1.f / 64), mb0 = rand_vec(n, rng, 1e-4f);
      float *Bh, *Bl, *Mb;
      upload_exact(b0, 1, n, &Bh, &Bl);
      cudaMalloc(&Mb, n * 4);
      cudaMemcpy(Mb, mb0.data(), n * 4, cudaMemcpyHostToDevice);
      GemmEpilogue eu{};
      eu.out_hi = Uh, eu.out_lo = Ul, eu.ld_out = n, eu.alpha = alpha, eu.M = n, eu.N = n, eu.mom = Mom;
      eu.lr = 1.0f, eu.mu = 0.9f, eu.wd = 1e-2f;
      eu.bias_col_p1 = eu.ones_col_p1 = n + 1, eu.gb_hi = Bh, eu.gb_lo = Bl, eu.gb_mom = Mb;
      gemm_tf32x3(Operand{Dh, Dl, n, n, K, true}, Operand{Hh, Hl, n, n + 1, K, true, n}, kEpiWgradUpdate, eu, 0);
      {
        std::vector<double> db(n), gsum(n, 0.0);
        for (int q = 0; q < K; ++q)
          for (int i = 0; i < n; ++i) gsum[i] += D[static_cast<long>(q) * n + i];
        std::vector<float> bn = fetch_pair(Bh, Bl, n), d(n);
        for (int i = 0; i < n; ++i) {
          const double g = gsum[i] * alpha + 1e-2 * b0[i], buf = 0.9 * mb0[i] + g;
          db[i] = -buf;
          d[i] = static_cast<float>(static_cast<double>(bn[i]) - b0[i]);
        }
        bad += report("wgrad fused update (db)", n, n + 1, K, rel_err(d, db), 1e-5);
      }
      cudaFree(Bh), cudaFree(Bl), cudaFree(Mb);
      std::vector<double> Wn(R.size()), dW(R.size());
      for (size_t i = 0; i < R.size(); ++i) {
        const double g = Ra[i] + 1e-2 * W[i], buf = 0.9 * M0[i] + g;
        Wn[i] = W[i] - 1.0 * buf;
        dW[i] = Wn[i] - W[i];
      }
      std::vector<float> w = fetch_pair(Uh, Ul, static_cast<long>(n) * n), d(w.size());
      for (size_t i = 0; i < w.size(); ++i) d[i] = static_cast<float>(static_cast<double>(w[i]) - W[i]);
      // the update's own rounding (fp32 W) bounds the change's accuracy: 1e-5 of it
      bad += report("wgrad fused update (dW)", n, n, K, rel_err(d, dW), 1e-5);
      cudaFree(Uh), cudaFree(Ul), cudaFree(Mom);
    }
    cudaFree(Dh), cudaFree(Dl), cudaFree(Hh), cudaFree(Hl), cudaFree(G);
  }
  std::printf("%s\n", bad ? "GEMM SHAPES FAILED" : "GEMM SHAPES OK");
  return bad ? 1 : 0;
}

int main(int argc, char** argv) {
  if (argc > 1 && std::strcmp(argv[1], "shapes") == 0) return run_shapes();
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
