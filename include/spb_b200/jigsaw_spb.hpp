// jigsaw_spb.hpp -- header-only C++ adapter: the reference's SPB API
// (/root/reference/proj/include/jigsaw/{errors,spb/model,spb/spb}.hpp) on top
// of the B200 C ABI (spb_b200.h). A reference user replaces
//     #include "jigsaw/spb/spb.hpp"      with   #include "spb_b200/jigsaw_spb.hpp"
// and links libspb_b200.so; names, argument meanings, value semantics
// (results by value, absent blocks EMPTY, caller-owned accumulators, stats
// accumulated across calls) and exception types are the reference's.
//
// Differences, all documented in INTEGRATION.md: ChainMlp runs on a B200 in
// fp32 (Params stay std::vector<double> at this boundary and are converted);
// its constructor takes the device workspace size (k, per-worker batch) so
// spb_sgd_run can run whole device-resident SPB steps; the convex
// BlockQuadratic fixture and the variance estimators are not provided (out of
// scope).
#pragma once
#include <cmath>
#include <cstdint>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../spb_b200.h"

namespace jigsaw {

// errors.hpp:9-25
class ArgumentError : public std::invalid_argument {
 public:
  explicit ArgumentError(const std::string& what) : std::invalid_argument(what) {}
};
class ProtocolError : public std::runtime_error {
 public:
  explicit ProtocolError(const std::string& what) : std::runtime_error(what) {}
};
class ConfigError : public std::runtime_error {
 public:
  explicit ConfigError(const std::string& what) : std::runtime_error(what) {}
};
class DeviceError : public std::runtime_error {
 public:
  explicit DeviceError(const std::string& what) : std::runtime_error(what) {}
};

namespace detail {
inline void check(spb_status st, const spb_ctx* ctx = nullptr) {
  if (st == SPB_OK) return;
  std::string msg = spb_last_error(ctx);
  switch (st) {
    case SPB_E_ARGUMENT: throw ArgumentError(msg);
    case SPB_E_PROTOCOL: throw ProtocolError(msg);
    case SPB_E_CONFIG: throw ConfigError(msg);
    default: throw DeviceError(msg);
  }
}
}  // namespace detail

namespace spb {

using Params = std::vector<std::vector<double>>;  // model.hpp:11

enum class ModelKind { ChainMlp, ConvexQuadratic };  // model.hpp:13

struct BackpropStats {  // model.hpp:17-19
  std::vector<long long> layer_ops;
};

// model.hpp:26-60
class LayeredModel {
 public:
  virtual ~LayeredModel() = default;
  virtual ModelKind kind() const = 0;
  int layer_count() const { return static_cast<int>(block_dims_.size()); }
  const std::vector<int>& block_dims() const { return block_dims_; }
  int dataset_size() const { return dataset_size_; }
  const Params& initial_params() const { return initial_params_; }
  void set_initial_params(Params x) { initial_params_ = std::move(x); }
  virtual double loss(const Params& x) const = 0;
  virtual void add_sample_gradient(const Params& x, int sample, int suffix, Params& acc,
                                   BackpropStats* stats = nullptr) const = 0;
  virtual std::optional<double> beta() const { return std::nullopt; }
  virtual std::optional<double> optimum_value() const { return std::nullopt; }
  Params zeros_like() const {
    Params p(block_dims_.size());
    for (size_t i = 0; i < block_dims_.size(); ++i) p[i].assign(block_dims_[i], 0.0);
    return p;
  }

 protected:
  std::vector<int> block_dims_;
  int dataset_size_ = 0;
  Params initial_params_;
};

// ChainMlp (model.hpp:95-111) on one B200.
class ChainMlp final : public LayeredModel {
 public:
  ChainMlp(std::vector<int> widths, std::vector<std::vector<double>> inputs, std::vector<double> targets,
           Params weights, int k = 1, int per_worker_batch = 1, int device = 0)
      : widths_(std::move(widths)), k_(k), bw_(per_worker_batch) {
    if (widths_.size() < 2) throw ArgumentError("mlp: need at least one layer");
    if (widths_.back() != 1) throw ArgumentError("mlp: output must be scalar");
    if (inputs.empty() || inputs.size() != targets.size()) throw ArgumentError("mlp: dataset shape mismatch");
    dataset_size_ = static_cast<int>(inputs.size());
    const int L = static_cast<int>(widths_.size()) - 1;
    block_dims_.resize(L);
    for (int l = 0; l < L; ++l) block_dims_[l] = widths_[l + 1] * widths_[l] + widths_[l + 1];
    for (int l = 0; l < L; ++l)
      if (static_cast<int>(weights[l].size()) != block_dims_[l]) throw ArgumentError("mlp: weight block size mismatch");
    spb_ctx* c = nullptr;
    detail::check(spb_create(widths_.data(), static_cast<int>(widths_.size()), k, per_worker_batch, device, &c));
    ctx_.reset(c);
    std::vector<float> X(static_cast<size_t>(dataset_size_) * widths_[0]), Y(dataset_size_);
    for (int s = 0; s < dataset_size_; ++s) {
      for (int i = 0; i < widths_[0]; ++i) X[static_cast<size_t>(s) * widths_[0] + i] = static_cast<float>(inputs[s][i]);
      Y[s] = static_cast<float>(targets[s]);
    }
    detail::check(spb_set_dataset(ctx(), X.data(), Y.data(), dataset_size_), ctx());
    initial_params_ = std::move(weights);
  }

  ModelKind kind() const override { return ModelKind::ChainMlp; }

  // model.cpp:139-143 at x.
  double loss(const Params& x) const override {
    upload(x);
    double out = 0.0;
    detail::check(spb_loss(ctx(), &out), ctx());
    return out;
  }

  // model.hpp:40-46: adds sample's suffix gradient into acc; prefix blocks untouched.
  void add_sample_gradient(const Params& x, int sample, int suffix, Params& acc,
                           BackpropStats* stats = nullptr) const override {
    auto g = run_partial(x, std::span<const int>(&sample, 1), suffix, stats);
    for (size_t l = 0; l < g.size(); ++l)
      for (size_t c = 0; c < g[l].size(); ++c) acc[l][c] += g[l][c];
  }

  // partial_backprop body on the device: covered blocks (batch mean), empty otherwise.
  Params run_partial(const Params& x, std::span<const int> batch, int suffix, BackpropStats* stats) const {
    const int L = layer_count();
    if (suffix < 1 || suffix > L) throw ArgumentError("partial_backprop: suffix out of range");
    if (batch.empty()) throw ArgumentError("partial_backprop: empty batch");
    upload(x);
    std::vector<std::vector<float>> out(L);
    std::vector<float*> ptrs(L, nullptr);
    for (int l = L - suffix; l < L; ++l) {
      out[l].resize(block_dims_[l]);
      ptrs[l] = out[l].data();
    }
    if (stats && stats->layer_ops.empty()) stats->layer_ops.assign(L, 0);
    int cov = 0;
    detail::check(spb_partial_backprop(ctx(), batch.data(), static_cast<int>(batch.size()), suffix, ptrs.data(),
                                       stats ? stats->layer_ops.data() : nullptr, &cov),
                  ctx());
    Params g(L);
    for (int l = cov - 1; l < L; ++l) g[l].assign(out[l].begin(), out[l].end());
    return g;
  }

  void train_steps(std::uint64_t seed, int step0, int steps) const {
    detail::check(spb_train_steps(ctx(), seed, step0, steps, 0, nullptr), ctx());
  }
  void set_optimizer(double lr, double momentum = 0.0, double weight_decay = 0.0) const {
    detail::check(spb_set_optimizer(ctx(), static_cast<float>(lr), static_cast<float>(momentum),
                                    static_cast<float>(weight_decay)),
                  ctx());
  }
  void upload(const Params& x) const {
    std::vector<std::vector<float>> f(x.size());
    std::vector<const float*> p(x.size());
    for (size_t l = 0; l < x.size(); ++l) {
      if (x[l].size() != static_cast<size_t>(block_dims_[l])) throw ArgumentError("mlp: param block size mismatch");
      f[l].assign(x[l].begin(), x[l].end());
      p[l] = f[l].data();
    }
    detail::check(spb_set_params(ctx(), p.data()), ctx());
  }
  Params download() const {
    std::vector<std::vector<float>> f(block_dims_.size());
    std::vector<float*> p(block_dims_.size());
    for (size_t l = 0; l < f.size(); ++l) f[l].resize(block_dims_[l]), p[l] = f[l].data();
    detail::check(spb_get_params(ctx(), p.data()), ctx());
    Params x(f.size());
    for (size_t l = 0; l < f.size(); ++l) x[l].assign(f[l].begin(), f[l].end());
    return x;
  }
  int k() const { return k_; }
  int per_worker_batch() const { return bw_; }
  spb_ctx* ctx() const { return ctx_.get(); }

 private:
  struct Del {
    void operator()(spb_ctx* c) const { spb_destroy(c); }
  };
  std::vector<int> widths_;
  int k_, bw_;
  std::unique_ptr<spb_ctx, Del> ctx_;
};

// ---- spb.hpp:20-61 ------------------------------------------------------------
struct SpbConfig {
  int k = 1;
  int B = 1;
  double P = 0.0;
  double lr_base = 0.0;
  double R = 0.0;
  double V = 0.0;
  void validate() const {
    if (k < 1) throw ArgumentError("SpbConfig: k must be >= 1");
    if (B < 1 || B % k != 0) throw ArgumentError("SpbConfig: B must be positive and divisible by k");
  }
};

struct PartialGradient {
  std::vector<std::vector<double>> blocks;
  int covered_from = 1;
  bool covers(int layer_1based) const { return layer_1based >= covered_from; }
};

inline int suffix_layers(int j, int k, int L) {
  int out = 0;
  detail::check(spb_suffix_layers(j, k, L, &out));
  return out;
}

inline std::vector<int> chunk_coverage(int m, int k) {
  std::vector<int> out(m > 0 ? m : 1);
  detail::check(spb_chunk_coverage(m, k, out.data()));
  out.resize(m);
  return out;
}

inline std::vector<std::pair<int, int>> chunk_layout(int k, int L) {
  std::vector<int> raw(2 * static_cast<size_t>(k > 0 ? k : 1));
  detail::check(spb_chunk_layout(k, L, raw.data()));
  std::vector<std::pair<int, int>> out(k);
  for (int m = 0; m < k; ++m) out[m] = {raw[2 * m], raw[2 * m + 1]};
  return out;
}

inline std::vector<int> layer_chunks(int k, int L) {
  std::vector<int> out(L > 0 ? L : 1);
  detail::check(spb_layer_chunks(k, L, out.data()));
  out.resize(L);
  return out;
}

// spb.hpp:54-56: only the B200 ChainMlp is supported as the model.
inline PartialGradient partial_backprop(const LayeredModel& model, const Params& x, std::span<const int> batch,
                                        int suffix, BackpropStats* stats = nullptr) {
  auto* mlp = dynamic_cast<const ChainMlp*>(&model);
  if (!mlp) throw ConfigError("partial_backprop: the B200 build runs ChainMlp models");
  PartialGradient g;
  g.blocks = mlp->run_partial(x, batch, suffix, stats);
  g.covered_from = model.layer_count() - suffix + 1;
  return g;
}

// spb.hpp:61, validated and averaged on the device (spb_aggregate).
inline Params aggregate(const std::vector<PartialGradient>& grads, int k) {
  if (k < 1 || static_cast<int>(grads.size()) != k) throw ArgumentError("aggregate: need exactly k gradients");
  const int L = static_cast<int>(grads[0].blocks.size());
  for (const auto& g : grads)
    if (static_cast<int>(g.blocks.size()) != L) throw ProtocolError("aggregate: gradient layer counts differ");
  static std::unique_ptr<spb_ctx, void (*)(spb_ctx*)> agg_ctx(nullptr, [](spb_ctx* c) { spb_destroy(c); });
  if (!agg_ctx) {
    const int w[2] = {1, 1};
    spb_ctx* c = nullptr;
    detail::check(spb_create(w, 2, 1, 1, 0, &c));
    agg_ctx.reset(c);
  }
  std::vector<std::vector<float>> f(static_cast<size_t>(k) * L);
  std::vector<const float*> ptrs(f.size(), nullptr);
  std::vector<int> dims(f.size(), 0), cov(k);
  std::vector<int> sizes(L, 0);
  for (int j = 0; j < k; ++j) {
    cov[j] = grads[j].covered_from;
    for (int l = 0; l < L; ++l) {
      const auto& b = grads[j].blocks[l];
      if (b.empty()) continue;
      f[j * L + l].assign(b.begin(), b.end());
      ptrs[j * L + l] = f[j * L + l].data();
      dims[j * L + l] = static_cast<int>(b.size());
      sizes[l] = std::max(sizes[l], dims[j * L + l]);
    }
  }
  std::vector<std::vector<float>> out(L);
  std::vector<float*> op(L);
  for (int l = 0; l < L; ++l) out[l].resize(sizes[l] > 0 ? sizes[l] : 1), op[l] = out[l].data();
  detail::check(spb_aggregate(agg_ctx.get(), k, L, ptrs.data(), dims.data(), cov.data(), op.data()), agg_ctx.get());
  Params res(L);
  for (int l = 0; l < L; ++l) res[l].assign(out[l].begin(), out[l].begin() + sizes[l]);
  return res;
}

// ---- spb.hpp:63-83 ------------------------------------------------------------
enum class StepSchedule { Theorem1, Constant };

struct SgdResult {
  std::vector<double> avg_loss;
  std::vector<double> step_size;
  std::vector<double> avg_subopt;
  Params avg_iterate;
  std::vector<Params> iterates;
};

// spb_sgd_run (spb.cpp:164-210): each iteration is one device SPB step.
inline SgdResult spb_sgd_run(const LayeredModel& model, const SpbConfig& cfg, int iterations, StepSchedule schedule,
                             std::uint64_t seed, bool record_iterates = false) {
  cfg.validate();
  if (iterations < 1) throw ArgumentError("spb_sgd_run: iterations must be >= 1");
  if (schedule == StepSchedule::Theorem1) {
    if (model.kind() != ModelKind::ConvexQuadratic) throw ConfigError("Theorem1 schedule requires the convex model");
  }
  auto* mlp = dynamic_cast<const ChainMlp*>(&model);
  if (!mlp) throw ConfigError("spb_sgd_run: the B200 build runs ChainMlp models");
  if (cfg.k != mlp->k() || cfg.B / cfg.k != mlp->per_worker_batch())
    throw ArgumentError("spb_sgd_run: model workspace was created for a different (k, B)");
  mlp->upload(model.initial_params());
  mlp->set_optimizer(cfg.lr_base);
  Params xbar = model.zeros_like();
  SgdResult res;
  for (int s = 1; s <= iterations; ++s) {
    mlp->train_steps(seed, s, 1);
    Params x = mlp->download();
    for (size_t l = 0; l < x.size(); ++l)
      for (size_t c = 0; c < x[l].size(); ++c) xbar[l][c] += (x[l][c] - xbar[l][c]) / s;
    res.step_size.push_back(cfg.lr_base);
    res.avg_loss.push_back(mlp->loss(xbar));
    mlp->upload(x);
    if (record_iterates) res.iterates.push_back(std::move(x));
  }
  res.avg_iterate = std::move(xbar);
  return res;
}

// ---- small helpers (spb.hpp:121-122) -------------------------------------------
inline double block_distance_sq(const Params& a, const Params& b) {
  double acc = 0.0;
  for (size_t l = 0; l < a.size(); ++l)
    for (size_t c = 0; c < a[l].size(); ++c) {
      const double d = a[l][c] - b[l][c];
      acc += d * d;
    }
  return acc;
}
inline void axpy(Params& y, double alpha, const Params& x) {
  for (size_t l = 0; l < y.size(); ++l)
    for (size_t c = 0; c < y[l].size(); ++c) y[l][c] += alpha * x[l][c];
}

// model.hpp:240-241: the reference instance (fp32-rounded) on a B200.
inline std::unique_ptr<ChainMlp> make_random_chain_mlp(const std::vector<int>& widths, int samples,
                                                       std::uint64_t seed, int k = 1, int per_worker_batch = 1,
                                                       int device = 0) {
  const int L = static_cast<int>(widths.size()) - 1;
  std::vector<float> X(static_cast<size_t>(samples) * widths[0]), Y(static_cast<size_t>(samples) * widths[L]);
  std::vector<std::vector<float>> W(L);
  std::vector<float*> wp(L);
  for (int l = 0; l < L; ++l) W[l].resize(static_cast<size_t>(widths[l + 1]) * widths[l] + widths[l + 1]), wp[l] = W[l].data();
  detail::check(spb_make_random_chain_mlp(widths.data(), static_cast<int>(widths.size()), samples, seed, X.data(),
                                          Y.data(), wp.data()));
  std::vector<std::vector<double>> inputs(samples);
  std::vector<double> targets(samples);
  for (int s = 0; s < samples; ++s) {
    inputs[s].assign(X.begin() + static_cast<long>(s) * widths[0], X.begin() + static_cast<long>(s + 1) * widths[0]);
    targets[s] = Y[static_cast<size_t>(s) * widths[L]];
  }
  Params w(L);
  for (int l = 0; l < L; ++l) w[l].assign(W[l].begin(), W[l].end());
  return std::make_unique<ChainMlp>(widths, std::move(inputs), std::move(targets), std::move(w), k, per_worker_batch,
                                    device);
}

}  // namespace spb
}  // namespace jigsaw
