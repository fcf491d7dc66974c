// Synthetic ChainMlp instances: make_random_chain_mlp (model.cpp:208-231) on
// the host, multi-threaded. The generator is counter-based (rng.hpp), so the
// n-th draw of the stream Rng(seed).split(0x313a) is mix(key, n) and disjoint
// counter ranges can be filled by independent threads with bit-identical
// results. Values are produced in fp64 exactly as the reference does and
// rounded to fp32 (the B200 path computes in fp32).
#include <cmath>
#include <thread>
#include <vector>

#include "../../include/spb_b200.h"
#include "planner.hpp"

namespace {

inline double unit_at(uint64_t key, uint64_t counter) {  // rng.hpp:23
  return static_cast<double>(spb::Rng::mix(key, counter) >> 11) * 0x1.0p-53;
}

inline double gaussian_at(uint64_t key, uint64_t counter) {  // rng.hpp:40-45, draws counter, counter+1
  double u1 = unit_at(key, counter);
  double u2 = unit_at(key, counter + 1);
  if (u1 <= 0.0) u1 = 0x1.0p-53;
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586476925286766559 * u2);
}

template <class F>
void parallel_for(long n, F&& f) {
  const int hw = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  const int T = static_cast<int>(std::min<long>(hw, std::max<long>(1, n / 65536)));
  if (T <= 1) {
    f(0, n);
    return;
  }
  std::vector<std::thread> pool;
  for (int t = 0; t < T; ++t) pool.emplace_back([&, t] { f(n * t / T, n * (t + 1) / T); });
  for (auto& th : pool) th.join();
}

}  // namespace

extern "C" SPB_API spb_status spb_make_random_chain_mlp(const int* widths, int n_widths, int samples, uint64_t seed,
                                                        float* X, float* Y, float* const* W) {
  if (n_widths < 2 || samples < 1) return SPB_E_ARGUMENT;
  const uint64_t key = spb::Rng::mix(seed, 0x313aULL);  // Rng(seed).split(0x313a)
  const int L = n_widths - 1;
  uint64_t counter = 0;  // the last counter consumed
  for (int l = 0; l < L; ++l) {  // model.cpp:213-218
    const long n = static_cast<long>(widths[l + 1]) * widths[l] + widths[l + 1];
    const double scale = 1.0 / std::sqrt(static_cast<double>(widths[l]));
    const uint64_t base = counter;
    float* dst = W[l];
    parallel_for(n, [&](long a, long b) {
      for (long i = a; i < b; ++i)
        dst[i] = static_cast<float>(scale * (2.0 * unit_at(key, base + 1 + static_cast<uint64_t>(i)) - 1.0));
    });
    counter += static_cast<uint64_t>(n);
  }
  // model.cpp:219-229: per sample, n_0 gaussians (2 draws each) then the
  // target noise gaussian: 2*(n_0 + 1) draws per sample.
  const int n0 = widths[0];
  const int nout = widths[L];
  const uint64_t per = 2ull * (static_cast<uint64_t>(n0) + 1);
  const uint64_t base = counter;
  parallel_for(samples, [&](long a, long b) {
    for (long s = a; s < b; ++s) {
      const uint64_t c0 = base + static_cast<uint64_t>(s) * per;
      double t = 0.0;
      for (int i = 0; i < n0; ++i) {
        const double v = gaussian_at(key, c0 + 1 + 2ull * i);
        X[s * n0 + i] = static_cast<float>(v);
        t += v;
      }
      const double y = std::tanh(t) + 0.1 * gaussian_at(key, c0 + 1 + 2ull * n0);
      for (int o = 0; o < nout; ++o) Y[s * nout + o] = static_cast<float>(y);
    }
  });
  return SPB_OK;
}
