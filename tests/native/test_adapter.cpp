// The C++ drop-in adapter (include/spb_b200/jigsaw_spb.hpp) exercised the way
// the reference's own unit tests exercise jigsaw::spb (tests/test_spb.cpp:
// suffix rule 43-56, coverage 58-67, layout 69-91, partial backprop 93-124,
// aggregate 145-207, sgd validation 209-229) -- on a B200. Built and run by
// tests/test_native.py (g++ -std=c++20 -I include ... -l:libspb_b200.so).
#include <cstdio>
#include <cstring>
#include <numeric>

#include "spb_b200/jigsaw_spb.hpp"

using namespace jigsaw;
using namespace jigsaw::spb;

static long g_checks = 0, g_fail = 0;
#define CHECK(x)                                                      \
  do {                                                                \
    ++g_checks;                                                       \
    if (!(x)) {                                                       \
      ++g_fail;                                                       \
      std::fprintf(stderr, "%s:%d CHECK failed: %s\n", __FILE__, __LINE__, #x); \
    }                                                                 \
  } while (0)
#define CHECK_THROWS_AS(expr, T)   \
  do {                             \
    bool ok_ = false;              \
    try {                          \
      (void)(expr);                \
    } catch (const T&) {           \
      ok_ = true;                  \
    } catch (...) {                \
    }                              \
    CHECK(ok_ && #T);              \
  } while (0)

static bool same_bits(const std::vector<double>& a, const std::vector<double>& b) {
  return a.size() == b.size() && (a.empty() || std::memcmp(a.data(), b.data(), a.size() * sizeof(double)) == 0);
}

int main() {
  // suffix rule
  CHECK(suffix_layers(3, 3, 9) == 9);
  CHECK(suffix_layers(1, 3, 9) == 3);
  CHECK(suffix_layers(2, 3, 9) == 6);
  CHECK(suffix_layers(1, 4, 10) == 3);
  for (int k = 1; k <= 12; ++k)
    for (int L = 1; L <= 20; ++L) {
      CHECK(suffix_layers(k, k, L) == L);
      for (int j = 2; j <= k; ++j) CHECK(suffix_layers(j, k, L) >= suffix_layers(j - 1, k, L));
    }
  CHECK_THROWS_AS(suffix_layers(0, 3, 9), ArgumentError);
  CHECK_THROWS_AS(suffix_layers(4, 3, 9), ArgumentError);
  // coverage and layout
  CHECK(chunk_coverage(1, 4) == std::vector<int>{4});
  CHECK(chunk_coverage(4, 4) == (std::vector<int>{1, 2, 3, 4}));
  CHECK_THROWS_AS(chunk_coverage(5, 4), ArgumentError);
  auto spans = chunk_layout(3, 7);
  CHECK(spans.size() == 3 && spans[0] == std::make_pair(1, 2) && spans[1] == std::make_pair(3, 4) &&
        spans[2] == std::make_pair(5, 7));

  // partial backprop == full pass on its suffix (bit-identical on the device too)
  auto mlp = make_random_chain_mlp({3, 4, 4, 4, 1}, 24, 5);
  auto x = mlp->initial_params();
  std::vector<int> batch{0, 3, 5, 7, 11, 13};
  const int L = mlp->layer_count();
  auto full = partial_backprop(*mlp, x, batch, L);
  CHECK(full.covered_from == 1);
  for (int suffix = 1; suffix <= L; ++suffix) {
    BackpropStats stats;
    auto part = partial_backprop(*mlp, x, batch, suffix, &stats);
    CHECK(part.covered_from == L - suffix + 1);
    for (int l = 1; l <= L; ++l) {
      if (l >= part.covered_from) {
        CHECK(same_bits(part.blocks[l - 1], full.blocks[l - 1]));
        CHECK(stats.layer_ops[l - 1] > 0);
      } else {
        CHECK(part.blocks[l - 1].empty());
        CHECK(stats.layer_ops[l - 1] == 0);
      }
    }
  }
  CHECK_THROWS_AS(partial_backprop(*mlp, x, batch, 0), ArgumentError);
  CHECK_THROWS_AS(partial_backprop(*mlp, x, batch, L + 1), ArgumentError);
  std::vector<int> empty;
  CHECK_THROWS_AS(partial_backprop(*mlp, x, empty, 1), ArgumentError);

  // add_sample_gradient accumulates into the caller's blocks, prefix untouched
  {
    Params acc = mlp->zeros_like();
    acc[0][0] = 42.0;
    mlp->add_sample_gradient(x, 3, 2, acc);
    CHECK(acc[0][0] == 42.0);
    double s = 0;
    for (double v : acc[L - 1]) s += v * v;
    CHECK(s > 0);
  }

  // aggregate: hand example (k = L = 3)
  {
    int k = 3, LL = 3;
    std::vector<PartialGradient> grads(k);
    for (int j = 1; j <= k; ++j) {
      auto& g = grads[j - 1];
      g.blocks.resize(LL);
      g.covered_from = LL - suffix_layers(j, k, LL) + 1;
      for (int l = g.covered_from; l <= LL; ++l) g.blocks[l - 1] = {3.0 * j};
    }
    grads[2].blocks[0] = {-2.5};
    auto agg = aggregate(grads, k);
    CHECK(std::fabs(agg[2][0] - 6.0) < 1e-6);
    CHECK(agg[0][0] == -2.5);
    auto broken = grads;
    broken[0].covered_from -= 1;
    CHECK_THROWS_AS(aggregate(broken, k), ProtocolError);
    auto missing = grads;
    missing[1].blocks[LL - 1].clear();
    CHECK_THROWS_AS(aggregate(missing, k), ProtocolError);
  }

  // sgd validation
  {
    auto m2 = make_random_chain_mlp({3, 4, 1}, 16, 3, 2, 4);
    SpbConfig cfg;
    cfg.k = 2;
    cfg.B = 8;
    cfg.lr_base = 1e-2;
    auto res = spb_sgd_run(*m2, cfg, 5, StepSchedule::Constant, 11, true);
    CHECK(res.avg_loss.size() == 5 && res.step_size.size() == 5 && res.iterates.size() == 5);
    cfg.R = 1.0;
    cfg.V = 1.0;
    CHECK_THROWS_AS(spb_sgd_run(*m2, cfg, 5, StepSchedule::Theorem1, 1), ConfigError);
    SpbConfig bad = cfg;
    bad.B = 7;
    CHECK_THROWS_AS(spb_sgd_run(*m2, bad, 5, StepSchedule::Constant, 1), ArgumentError);
  }
  std::printf("[adapter] checks: %ld | %ld failed\n", g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}
