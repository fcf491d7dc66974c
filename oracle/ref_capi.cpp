// TEST INFRASTRUCTURE ONLY. A C-ABI shim over the UNMODIFIED reference SPB
// core (/root/reference/proj/src/spb/{spb,model}.cpp), compiled by
// oracle/Makefile into oracle/_ref/libjigsaw_ref.so. It lets the Python tests
// and bench.py's reference arm drive the reference's own public API:
//   partial_backprop  spb.hpp:54-56  (spb.cpp:51-68)
//   aggregate         spb.hpp:61     (spb.cpp:70-106)
//   spb_sgd_run       spb.hpp:82-83  (spb.cpp:164-210)
//   suffix/chunk bookkeeping spb.hpp:39-49 (spb.cpp:16-49)
//   make_random_chain_mlp    model.hpp:240-241 (model.cpp:208-231)
//   empirical_variance spb.hpp:100-101 (spb.cpp:212-265) and the reference's
//   independent variance_oracle (oracle.hpp:57-62, oracle.cpp:240-326)
//   ProfileTable::from_csv + forward_time / backward_time / peak_memory /
//   task_demand  profile.hpp:43-80 (profile.cpp:67-171): parses and queries
//                the task profiles the B200 emitter writes
//                (paper_2111_10672_b200/jigsaw_profiles.py)
// Only tests/, __graft_entry__.smoke() and bench.py's CPU legs load it. It is
// built only where /root/reference exists (this container); the .so itself
// travels to the GPU box with the snapshot.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "jigsaw/cost/profile.hpp"
#include "jigsaw/errors.hpp"
#include "jigsaw/oracle/oracle.hpp"
#include "jigsaw/rng.hpp"
#include "jigsaw/spb/model.hpp"
#include "jigsaw/spb/spb.hpp"

using jigsaw::Rng;
using namespace jigsaw::spb;

namespace {

thread_local std::string g_err;

// Status convention shared with include/spb_b200.h.
enum { kOk = 0, kArgument = 1, kProtocol = 2, kConfig = 3, kOther = 9 };

template <class F>
int guard(F&& f) {
  try {
    f();
    return kOk;
  } catch (const jigsaw::ArgumentError& e) {
    g_err = e.what();
    return kArgument;
  } catch (const jigsaw::ProtocolError& e) {
    g_err = e.what();
    return kProtocol;
  } catch (const jigsaw::ConfigError& e) {
    g_err = e.what();
    return kConfig;
  } catch (const std::exception& e) {
    g_err = e.what();
    return kOther;
  }
}

struct Handle {
  std::unique_ptr<ChainMlp> model;
  Params x;  // current iterate, owned here so steps do not marshal params
};

// Same draw as the file-local draw_batch in spb.cpp:127-131.
std::vector<int> draw(Rng rng, int count, int n) {
  std::vector<int> b(count);
  for (int& s : b) s = static_cast<int>(rng.next_below(n));
  return b;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- RNG (rng.hpp) ---------------------------------------------------------
uint64_t ref_rng_mix(uint64_t a, uint64_t b) { return Rng::mix(a, b); }

// Fills out[0..n) with successive draws of Rng(key).split(tags...) where
// kind 0 = next_u64, 1 = next_below(bound), 2 = next_unit bits, 3 = gaussian bits.
void ref_rng_stream(uint64_t key, const uint64_t* tags, int ntags, int kind, uint64_t bound,
                    int n, uint64_t* out) {
  Rng r(key);
  for (int i = 0; i < ntags; ++i) r = r.split(tags[i]);
  for (int i = 0; i < n; ++i) {
    if (kind == 0) out[i] = r.next_u64();
    else if (kind == 1) out[i] = r.next_below(bound);
    else {
      double d = kind == 2 ? r.next_unit() : r.next_gaussian();
      std::memcpy(&out[i], &d, sizeof d);
    }
  }
}

// ---- bookkeeping (spb.cpp:16-49) --------------------------------------------
int ref_suffix_layers(int j, int k, int L, int* out) {
  return guard([&] { *out = suffix_layers(j, k, L); });
}
int ref_chunk_coverage(int m, int k, int* out) {
  return guard([&] {
    auto w = chunk_coverage(m, k);
    std::copy(w.begin(), w.end(), out);
  });
}
int ref_chunk_layout(int k, int L, int* out) {
  return guard([&] {
    auto s = chunk_layout(k, L);
    for (int m = 0; m < k; ++m) {
      out[2 * m] = s[m].first;
      out[2 * m + 1] = s[m].second;
    }
  });
}
int ref_layer_chunks(int k, int L, int* out) {
  return guard([&] {
    auto c = layer_chunks(k, L);
    std::copy(c.begin(), c.end(), out);
  });
}

// ---- model ------------------------------------------------------------------
// make_random_chain_mlp (model.cpp:208-231), unmodified.
void* ref_chain_random(const int* widths, int nw, int samples, uint64_t seed) {
  Handle* h = nullptr;
  int st = guard([&] {
    auto m = make_random_chain_mlp(std::vector<int>(widths, widths + nw), samples, seed);
    h = new Handle{std::move(m), {}};
    h->x = h->model->initial_params();
  });
  return st == kOk ? h : nullptr;
}

// ChainMlp from explicit data (model.cpp:86-101). X: N x n0 row-major, Y: N.
// W[l]: block l (W_l row-major then b_l), as Params block l.
void* ref_chain_new(const int* widths, int nw, const double* X, const double* Y, int N,
                    const double* const* W) {
  Handle* h = nullptr;
  int st = guard([&] {
    std::vector<int> wv(widths, widths + nw);
    std::vector<std::vector<double>> inputs(N);
    for (int s = 0; s < N; ++s) inputs[s].assign(X + static_cast<size_t>(s) * wv[0],
                                                 X + static_cast<size_t>(s + 1) * wv[0]);
    std::vector<double> targets(Y, Y + N);
    int L = nw - 1;
    Params w(L);
    for (int l = 0; l < L; ++l) w[l].assign(W[l], W[l] + (wv[l + 1] * wv[l] + wv[l + 1]));
    auto m = std::make_unique<ChainMlp>(wv, std::move(inputs), std::move(targets), std::move(w));
    h = new Handle{std::move(m), {}};
    h->x = h->model->initial_params();
  });
  return st == kOk ? h : nullptr;
}

void ref_chain_free(void* p) { delete static_cast<Handle*>(p); }

int ref_layer_count(void* p) { return static_cast<Handle*>(p)->model->layer_count(); }
int ref_block_dim(void* p, int l) { return static_cast<Handle*>(p)->model->block_dims()[l]; }

void ref_get_params(void* p, double* const* out) {
  auto* h = static_cast<Handle*>(p);
  for (size_t l = 0; l < h->x.size(); ++l)
    std::memcpy(out[l], h->x[l].data(), h->x[l].size() * sizeof(double));
}
void ref_set_params(void* p, const double* const* in) {
  auto* h = static_cast<Handle*>(p);
  for (size_t l = 0; l < h->x.size(); ++l) std::memcpy(h->x[l].data(), in[l], h->x[l].size() * sizeof(double));
}

int ref_loss(void* p, double* out) {
  auto* h = static_cast<Handle*>(p);
  return guard([&] { *out = h->model->loss(h->x); });
}

// partial_backprop (spb.cpp:51-68) at the handle's iterate. out_blocks[l] may
// be NULL for absent layers; layer_ops (nullable) accumulates like
// BackpropStats (spb.cpp:61).
int ref_partial_backprop(void* p, const int* batch, int len, int suffix, double* const* out_blocks,
                         long long* layer_ops, int* covered_from) {
  auto* h = static_cast<Handle*>(p);
  return guard([&] {
    BackpropStats stats;
    int L = h->model->layer_count();
    if (layer_ops) stats.layer_ops.assign(layer_ops, layer_ops + L);
    auto g = partial_backprop(*h->model, h->x, std::span<const int>(batch, len), suffix,
                              layer_ops ? &stats : nullptr);
    if (covered_from) *covered_from = g.covered_from;
    for (int l = 0; l < L; ++l)
      if (!g.blocks[l].empty() && out_blocks[l])
        std::memcpy(out_blocks[l], g.blocks[l].data(), g.blocks[l].size() * sizeof(double));
    if (layer_ops) std::copy(stats.layer_ops.begin(), stats.layer_ops.end(), layer_ops);
  });
}

// aggregate (spb.cpp:70-106). blocks[j*L + l] is worker j+1's block l, NULL when
// absent; dims[j*L + l] its length (0 when absent).
int ref_aggregate(int k, int L, const double* const* blocks, const int* dims, const int* covered_from,
                  double* const* out) {
  return guard([&] {
    std::vector<PartialGradient> grads(k);
    for (int j = 0; j < k; ++j) {
      grads[j].covered_from = covered_from[j];
      grads[j].blocks.resize(L);
      for (int l = 0; l < L; ++l)
        if (blocks[j * L + l]) grads[j].blocks[l].assign(blocks[j * L + l], blocks[j * L + l] + dims[j * L + l]);
    }
    auto agg = aggregate(grads, k);
    for (int l = 0; l < L; ++l) std::memcpy(out[l], agg[l].data(), agg[l].size() * sizeof(double));
  });
}

// One SPB-SGD iteration exactly as the body of spb_sgd_run (spb.cpp:187-196)
// with the Constant schedule, minus the diagnostic loss(xbar) at :202:
// every worker j draws B/k samples from Rng(seed).split(s).split(j), runs
// partial_backprop on suffix_layers(j,k,L), the results are aggregated, and
// x -= lr * g. full != 0 gives the full-backprop DP baseline
// (baseline_estimate, spb.cpp:149-160). threads > 1 runs the workers of the
// step on concurrent std::threads (a harness change: the reference's model
// methods are const and thread-safe, model.hpp:21-25); results are identical.
int ref_step(void* p, int k, int B, double lr, uint64_t seed, int s, int full, int threads) {
  auto* h = static_cast<Handle*>(p);
  return guard([&] {
    SpbConfig cfg;
    cfg.k = k;
    cfg.B = B;
    cfg.validate();
    const auto& model = *h->model;
    int L = model.layer_count();
    int per = B / k;
    Rng stream = Rng(seed).split(static_cast<std::uint64_t>(s));
    std::vector<PartialGradient> grads(k);
    auto work = [&](int j) {
      auto batch = draw(stream.split(j), per, model.dataset_size());
      grads[j - 1] = partial_backprop(model, h->x, batch, full ? L : suffix_layers(j, k, L));
    };
    if (threads <= 1) {
      for (int j = 1; j <= k; ++j) work(j);
    } else {
      std::vector<std::exception_ptr> errs(k);
      for (int base = 1; base <= k; base += threads) {
        std::vector<std::thread> pool;
        for (int j = base; j < base + threads && j <= k; ++j)
          pool.emplace_back([&, j] {
            try {
              work(j);
            } catch (...) {
              errs[j - 1] = std::current_exception();
            }
          });
        for (auto& t : pool) t.join();
      }
      for (auto& e : errs)
        if (e) std::rethrow_exception(e);
    }
    Params g;
    if (full) {
      g = model.zeros_like();
      for (int j = 1; j <= k; ++j) axpy(g, 1.0 / k, grads[j - 1].blocks);
    } else {
      g = aggregate(grads, k);
    }
    axpy(h->x, -lr, g);
  });
}

// spb_sgd_run (spb.cpp:164-210), Constant schedule, recording the final
// iterate into the handle and avg_loss[0..iters).
int ref_sgd_run(void* p, int k, int B, double lr, int iters, uint64_t seed, double* avg_loss) {
  auto* h = static_cast<Handle*>(p);
  return guard([&] {
    SpbConfig cfg;
    cfg.k = k;
    cfg.B = B;
    cfg.lr_base = lr;
    auto res = spb_sgd_run(*h->model, cfg, iters, StepSchedule::Constant, seed, true);
    h->x = res.iterates.back();
    if (avg_loss) std::copy(res.avg_loss.begin(), res.avg_loss.end(), avg_loss);
  });
}

// Wall time of `steps` ref_step calls (steady_clock), for bench.py's CPU arm.
double ref_time_steps(void* p, int k, int B, double lr, uint64_t seed, int s0, int steps, int full,
                      int threads) {
  auto t0 = std::chrono::steady_clock::now();
  for (int s = s0; s < s0 + steps; ++s)
    if (ref_step(p, k, B, lr, seed, s, full, threads) != kOk) return -1.0;
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// empirical_variance at the handle's iterate: out = {spb, spb_se, baseline,
// baseline_se, p_hat[0..k), p_se[0..k)}.
int ref_empirical_variance(void* p, int k, int B, int trials, uint64_t seed, double* out) {
  auto* h = static_cast<Handle*>(p);
  return guard([&] {
    SpbConfig cfg;
    cfg.k = k;
    cfg.B = B;
    auto e = empirical_variance(*h->model, cfg, h->x, trials, seed);
    out[0] = e.spb, out[1] = e.spb_se, out[2] = e.baseline, out[3] = e.baseline_se;
    for (int m = 0; m < k; ++m) out[4 + m] = e.p_hat[m], out[4 + k + m] = e.p_se[m];
  });
}

// variance_oracle at the handle's iterate: out = {spb, spb_se, harmonic_sum,
// harmonic_sum_se, p_hat[0..k), p_se[0..k)}.
int ref_variance_oracle(void* p, int k, int B, int trials, uint64_t seed, double* out) {
  auto* h = static_cast<Handle*>(p);
  return guard([&] {
    SpbConfig cfg;
    cfg.k = k;
    cfg.B = B;
    auto e = jigsaw::oracle::variance_oracle(*h->model, cfg, h->x, trials, seed);
    out[0] = e.spb, out[1] = e.spb_se, out[2] = e.harmonic_sum, out[3] = e.harmonic_sum_se;
    for (int m = 0; m < k; ++m) out[4 + m] = e.p_hat[m], out[4 + k + m] = e.p_se[m];
  });
}

// Parses `csv` with the reference's ProfileTable::from_csv (which validates
// every entry) and queries model `model` at `fraction`:
// out = {forward_time, backward_time, peak_memory, grad_size_mb, batch,
//        task_demand(fraction).duration_ms, task_demand.comm_mb}.
int ref_profile_query(const char* csv, const char* model, double fraction, double* out) {
  return guard([&] {
    auto table = jigsaw::cost::ProfileTable::from_csv(csv, "<b200>");
    const auto& e = table.get(model);
    out[0] = jigsaw::cost::forward_time(e, fraction);
    out[1] = jigsaw::cost::backward_time(e, fraction);
    out[2] = jigsaw::cost::peak_memory(e, fraction);
    out[3] = e.grad_size_mb;
    out[4] = e.batch_size;
    auto d = jigsaw::cost::task_demand(e, fraction);
    out[5] = d.duration_ms;
    out[6] = d.comm_mb;
  });
}

}  // extern "C"
