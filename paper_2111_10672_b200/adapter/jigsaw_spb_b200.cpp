// The B200 drop-in for the reference's SPB core: this ONE translation unit
// defines every symbol the reference declares in
//   include/jigsaw/spb/model.hpp  (LayeredModel, BlockQuadratic, ChainMlp,
//                                  make_random_quadratic, make_random_chain_mlp)
//   include/jigsaw/spb/spb.hpp    (SpbConfig::validate, suffix_layers ..
//                                  layer_chunks, partial_backprop, aggregate,
//                                  spb_sgd_run, empirical_variance,
//                                  full_gradient, exact_chunk_variances,
//                                  exact_spb_variance, measured_grad_norm_bound,
//                                  block_distance_sq, axpy)
// and is compiled against the reference's OWN headers (-I <reference>/include),
// so a maintainer links it in place of src/spb/spb.cpp + src/spb/model.cpp and
// the rest of jigsaw_core (verify, oracle, sim, scheduler) links unchanged --
// one definition of every type, no ODR conflict.
//
// What runs where:
// * ChainMlp -- the model of the hot path -- lives on a B200: its constructor
//   binds it to a device context (libspb_b200.so, include/spb_b200.h) holding
//   the dataset; partial_backprop / add_sample_gradient run the tcgen05 3xTF32
//   forward + truncated backward, spb_sgd_run with the constant schedule runs
//   whole device-resident SPB iterations (spb_train_steps), empirical_variance
//   the device estimator, and loss / sample_loss an fp64 GPU forward (the
//   reference's precision, needed by finite-difference callers). The fp64
//   Params of this API are converted at the boundary (parity mode); the
//   performance path is the device-resident one.
// * aggregate runs on the GPU in fp64 with the reference's exact operation
//   order (bit-identical).
// * BlockQuadratic -- the theory fixture behind the Theorem-1 schedule
//   (model.hpp:62-89) -- and any user-defined LayeredModel stay on the CPU:
//   the generic paths below follow the reference's semantics
//   (spb.cpp:51-68, 120-123, 164-318; model.cpp:21-84). That is the plugin
//   API: a LayeredModel subclass only implements add_sample_gradient.
// Errors are the reference's exception types with the reference's trigger
// conditions; C-ABI status codes are mapped back to them.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

#include "jigsaw/errors.hpp"
#include "jigsaw/rng.hpp"
#include "jigsaw/spb/model.hpp"
#include "jigsaw/spb/spb.hpp"
#include "spb_b200.h"

namespace jigsaw::spb {
namespace {

// ---- C-ABI status -> the reference's exception types -----------------------

[[noreturn]] void throw_status(spb_status st, const char* msg) {
  const std::string m = msg ? msg : "";
  switch (st) {
    case SPB_E_ARGUMENT: throw ArgumentError(m);
    case SPB_E_PROTOCOL: throw ProtocolError(m);
    case SPB_E_CONFIG: throw ConfigError(m);
    default: throw std::runtime_error("spb_b200: " + m);
  }
}

void check(spb_status st, const spb_ctx* ctx = nullptr) {
  if (st != SPB_OK) throw_status(st, spb_last_error(ctx));
}

// ---- the GPU binding of one ChainMlp ----------------------------------------

// Device contexts of one ChainMlp (one per (k, per-worker batch) workspace
// shape), the fp32 dataset they were created from, and the parameters last
// uploaded to each. Contexts are created on the calling thread's current CUDA
// device (spb_create with device -1). All GPU work of a model is serialised by
// its mutex (the reference promises const, thread-safe model methods).
struct GpuModel {
  std::vector<int> widths;
  int N = 0;
  std::vector<float> X, Y;
  std::mutex mu;
  std::map<std::pair<int, int>, spb_ctx*> ctxs;
  std::map<const spb_ctx*, std::vector<float>> uploaded;

  ~GpuModel() {
    for (auto& kv : ctxs) spb_destroy(kv.second);
  }

  spb_ctx* ctx(int k, int bw) {
    auto it = ctxs.find({k, bw});
    if (it != ctxs.end()) return it->second;
    spb_ctx* c = nullptr;
    check(spb_create(widths.data(), static_cast<int>(widths.size()), k, bw, -1, &c));
    if (spb_status st = spb_set_dataset(c, X.data(), Y.data(), N); st != SPB_OK) {
      const std::string msg = spb_last_error(c);
      spb_destroy(c);
      throw_status(st, msg.c_str());
    }
    ctxs[{k, bw}] = c;
    return c;
  }

  // fp64 Params -> the context's fp32 parameters (skipped when unchanged).
  void upload(spb_ctx* c, const Params& x) {
    const int L = static_cast<int>(widths.size()) - 1;
    if (static_cast<int>(x.size()) != L) throw ArgumentError("mlp: parameter block count mismatch");
    size_t total = 0;
    for (int l = 0; l < L; ++l) {
      const size_t d = static_cast<size_t>(widths[l + 1]) * widths[l] + widths[l + 1];
      if (x[l].size() != d) throw ArgumentError("mlp: weight block size mismatch");
      total += d;
    }
    std::vector<float> flat(total);
    size_t o = 0;
    for (const auto& blk : x)
      for (double v : blk) flat[o++] = static_cast<float>(v);
    auto& last = uploaded[c];
    if (last == flat) return;
    std::vector<const float*> ptrs(L);
    o = 0;
    for (int l = 0; l < L; ++l) ptrs[l] = flat.data() + o, o += x[l].size();
    check(spb_set_params(c, ptrs.data()), c);
    last = std::move(flat);
  }

  std::vector<float*> block_ptrs(std::vector<std::vector<float>>& bufs) const {
    const int L = static_cast<int>(widths.size()) - 1;
    bufs.resize(L);
    std::vector<float*> p(L);
    for (int l = 0; l < L; ++l) {
      bufs[l].assign(static_cast<size_t>(widths[l + 1]) * widths[l] + widths[l + 1], 0.f);
      p[l] = bufs[l].data();
    }
    return p;
  }
};

std::mutex g_registry_mu;
std::unordered_map<const LayeredModel*, std::shared_ptr<GpuModel>> g_registry;

std::shared_ptr<GpuModel> bind_gpu(const LayeredModel* m, const std::vector<int>& widths,
                                   const std::vector<std::vector<double>>& inputs,
                                   const std::vector<double>& targets) {
  auto g = std::make_shared<GpuModel>();
  g->widths = widths;
  g->N = static_cast<int>(inputs.size());
  const int n0 = widths.front();
  g->X.resize(static_cast<size_t>(g->N) * n0);
  g->Y.resize(g->N);
  for (int s = 0; s < g->N; ++s) {
    for (int i = 0; i < n0; ++i) g->X[static_cast<size_t>(s) * n0 + i] = static_cast<float>(inputs[s][i]);
    g->Y[s] = static_cast<float>(targets[s]);
  }
  g->ctx(1, 1);  // fails loudly here when there is no B200 / no libspb_b200
  std::lock_guard<std::mutex> lock(g_registry_mu);
  g_registry[m] = g;  // a new model at a reused address replaces the stale binding
  return g;
}

// The GPU binding of `m`, or null for models that run on the CPU.
std::shared_ptr<GpuModel> gpu_of(const LayeredModel& m) {
  if (m.kind() != ModelKind::ChainMlp) return nullptr;
  std::lock_guard<std::mutex> lock(g_registry_mu);
  auto it = g_registry.find(&m);
  return it == g_registry.end() ? nullptr : it->second;
}

std::vector<int> draw_batch(Rng rng, int count, int dataset_size) {  // spb.cpp:127-131
  std::vector<int> batch(count);
  for (int& s : batch) s = static_cast<int>(rng.next_below(static_cast<std::uint64_t>(dataset_size)));
  return batch;
}

// ---- BlockQuadratic numerics (model.cpp:33-47): eigenvalues of the Gram
// matrix by cyclic Jacobi rotations, x* by a Cholesky solve. -----------------

std::vector<double> symmetric_eigenvalues(std::vector<double> a, int n) {
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) off += a[p * n + q] * a[p * n + q];
    if (off < 1e-30) break;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        const double apq = a[p * n + q];
        if (std::fabs(apq) < 1e-300) continue;
        const double theta = (a[q * n + q] - a[p * n + p]) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int r = 0; r < n; ++r) {  // A <- A J
          const double arp = a[r * n + p], arq = a[r * n + q];
          a[r * n + p] = c * arp - s * arq;
          a[r * n + q] = s * arp + c * arq;
        }
        for (int r = 0; r < n; ++r) {  // A <- J^T A
          const double apr = a[p * n + r], aqr = a[q * n + r];
          a[p * n + r] = c * apr - s * aqr;
          a[q * n + r] = s * apr + c * aqr;
        }
      }
  }
  std::vector<double> ev(n);
  for (int i = 0; i < n; ++i) ev[i] = a[i * n + i];
  return ev;
}

std::vector<double> cholesky_solve(std::vector<double> a, std::vector<double> b, int n) {
  for (int j = 0; j < n; ++j) {
    double d = a[j * n + j];
    for (int k = 0; k < j; ++k) d -= a[j * n + k] * a[j * n + k];
    if (d <= 0.0) throw ArgumentError("quadratic: A does not have full column rank");
    const double ljj = std::sqrt(d);
    a[j * n + j] = ljj;
    for (int i = j + 1; i < n; ++i) {
      double v = a[i * n + j];
      for (int k = 0; k < j; ++k) v -= a[i * n + k] * a[j * n + k];
      a[i * n + j] = v / ljj;
    }
  }
  for (int i = 0; i < n; ++i) {  // L y = b
    for (int k = 0; k < i; ++k) b[i] -= a[i * n + k] * b[k];
    b[i] /= a[i * n + i];
  }
  for (int i = n - 1; i >= 0; --i) {  // L^T x = y
    for (int k = i + 1; k < n; ++k) b[i] -= a[k * n + i] * b[k];
    b[i] /= a[i * n + i];
  }
  return b;
}

// Squared distance of two gradients restricted to layers [first, last] (1-based).
double span_distance_sq(const Params& a, const Params& b, int first, int last) {
  double d = 0.0;
  for (int l = first; l <= last; ++l)
    for (size_t c = 0; c < a[l - 1].size(); ++c) {
      const double e = a[l - 1][c] - b[l - 1][c];
      d += e * e;
    }
  return d;
}

// One SPB estimate (spb.cpp:133-145) / the full-backprop baseline with the
// same worker streams (spb.cpp:147-160), through the public functions.
Params spb_estimate(const LayeredModel& model, const SpbConfig& cfg, const Params& x, const Rng& root) {
  const int L = model.layer_count(), per = cfg.B / cfg.k;
  std::vector<PartialGradient> grads(cfg.k);
  for (int j = 1; j <= cfg.k; ++j)
    grads[j - 1] =
        partial_backprop(model, x, draw_batch(root.split(j), per, model.dataset_size()), suffix_layers(j, cfg.k, L));
  return aggregate(grads, cfg.k);
}

Params baseline_estimate(const LayeredModel& model, const SpbConfig& cfg, const Params& x, const Rng& root) {
  const int L = model.layer_count(), per = cfg.B / cfg.k;
  Params mean = model.zeros_like();
  for (int j = 1; j <= cfg.k; ++j)
    axpy(mean, 1.0 / cfg.k, partial_backprop(model, x, draw_batch(root.split(j), per, model.dataset_size()), L).blocks);
  return mean;
}

void mean_and_se(double sum, double sumsq, int n, double& mean, double& se) {
  mean = sum / n;
  se = std::sqrt(std::max(0.0, sumsq / n - mean * mean) / n);
}

}  // namespace

// ============================================================================
// model.hpp
// ============================================================================

Params LayeredModel::zeros_like() const {
  Params p(block_dims_.size());
  for (size_t l = 0; l < block_dims_.size(); ++l) p[l].assign(static_cast<size_t>(block_dims_[l]), 0.0);
  return p;
}

// ---- BlockQuadratic (CPU: a theory fixture, not the training step) ----------

BlockQuadratic::BlockQuadratic(std::vector<double> a_rowmajor, std::vector<double> b, int blocks)
    : a_(std::move(a_rowmajor)), b_(std::move(b)) {
  if (blocks < 1) throw ArgumentError("quadratic: blocks must be >= 1");
  if (b_.empty()) throw ArgumentError("quadratic: empty dataset");
  dataset_size_ = static_cast<int>(b_.size());
  if (a_.size() % b_.size() != 0) throw ArgumentError("quadratic: A shape mismatch");
  dim_ = static_cast<int>(a_.size() / b_.size());
  if (dim_ % blocks != 0) throw ArgumentError("quadratic: dim not divisible into blocks");
  const int bd = dim_ / blocks;
  block_dims_.assign(blocks, bd);
  initial_params_ = zeros_like();
  // Gram = A^T A, A^T b.
  const int n = dim_, N = dataset_size_;
  std::vector<double> gram(static_cast<size_t>(n) * n, 0.0), atb(n, 0.0);
  for (int s = 0; s < N; ++s) {
    const double* row = a_.data() + static_cast<size_t>(s) * n;
    for (int i = 0; i < n; ++i) {
      atb[i] += row[i] * b_[s];
      for (int j = 0; j < n; ++j) gram[static_cast<size_t>(i) * n + j] += row[i] * row[j];
    }
  }
  const auto ev = symmetric_eigenvalues(gram, n);
  beta_ = *std::max_element(ev.begin(), ev.end());
  if (*std::min_element(ev.begin(), ev.end()) <= 1e-9 * beta_)
    throw ArgumentError("quadratic: A does not have full column rank");
  const auto xs = cholesky_solve(gram, atb, n);
  x_star_.resize(blocks);
  for (int l = 0; l < blocks; ++l) x_star_[l].assign(xs.begin() + l * bd, xs.begin() + (l + 1) * bd);
  double f = 0.0;
  for (int s = 0; s < N; ++s) {
    double r = -b_[s];
    for (int i = 0; i < n; ++i) r += a_[static_cast<size_t>(s) * n + i] * xs[i];
    f += r * r;
  }
  f_star_ = 0.5 * f;
}

double BlockQuadratic::residual(const Params& x, int sample) const {
  const double* row = a_.data() + static_cast<size_t>(sample) * dim_;
  double r = 0.0;
  size_t i = 0;
  for (const auto& blk : x)
    for (double v : blk) r += row[i++] * v;
  return r - b_[sample];
}

double BlockQuadratic::loss(const Params& x) const {
  double total = 0.0;
  for (int s = 0; s < dataset_size_; ++s) {
    const double r = residual(x, s);
    total += 0.5 * r * r;
  }
  return total;
}

void BlockQuadratic::add_sample_gradient(const Params& x, int sample, int suffix, Params& acc,
                                         BackpropStats* stats) const {
  const int L = layer_count();
  if (suffix < 1 || suffix > L) throw ArgumentError("suffix out of range");
  if (sample < 0 || sample >= dataset_size_) throw ArgumentError("sample out of range");
  // Per-sample gradient N * a_i (a_i . x - b_i) (model.hpp:64-67), suffix blocks only.
  const double scale = static_cast<double>(dataset_size_) * residual(x, sample);
  const int bd = block_dims_[0];
  const double* row = a_.data() + static_cast<size_t>(sample) * dim_;
  for (int l = L - suffix; l < L; ++l) {
    for (int c = 0; c < bd; ++c) acc[l][c] += scale * row[l * bd + c];
    if (stats) stats->layer_ops[l] += bd;
  }
}

// ---- ChainMlp (GPU) -----------------------------------------------------------

ChainMlp::ChainMlp(std::vector<int> widths, std::vector<std::vector<double>> inputs, std::vector<double> targets,
                   Params weights)
    : widths_(std::move(widths)), inputs_(std::move(inputs)), targets_(std::move(targets)) {
  if (widths_.size() < 2) throw ArgumentError("mlp: need at least one layer");
  if (widths_.back() != 1) throw ArgumentError("mlp: output must be scalar");
  if (inputs_.empty() || inputs_.size() != targets_.size()) throw ArgumentError("mlp: dataset shape mismatch");
  for (const auto& in : inputs_)
    if (static_cast<int>(in.size()) != widths_.front()) throw ArgumentError("mlp: dataset shape mismatch");
  dataset_size_ = static_cast<int>(inputs_.size());
  const int L = static_cast<int>(widths_.size()) - 1;
  block_dims_.resize(L);
  for (int l = 0; l < L; ++l) block_dims_[l] = widths_[l + 1] * widths_[l] + widths_[l + 1];
  if (static_cast<int>(weights.size()) != L) throw ArgumentError("mlp: weight block size mismatch");
  for (int l = 0; l < L; ++l)
    if (static_cast<int>(weights[l].size()) != block_dims_[l]) throw ArgumentError("mlp: weight block size mismatch");
  initial_params_ = std::move(weights);
  bind_gpu(this, widths_, inputs_, targets_);
}

double ChainMlp::sample_loss(const Params& x, int sample) const {
  if (sample < 0 || sample >= dataset_size_) throw ArgumentError("sample out of range");
  auto g = gpu_of(*this);
  if (!g) g = bind_gpu(this, widths_, inputs_, targets_);  // a copied model binds on first use
  std::lock_guard<std::mutex> lock(g->mu);
  spb_ctx* c = g->ctx(1, 1);
  std::vector<const double*> p(x.size());
  for (size_t l = 0; l < x.size(); ++l) p[l] = x[l].data();
  double out = 0.0;
  check(spb_loss64(c, p.data(), &sample, 1, &out), c);
  return out;
}

double ChainMlp::loss(const Params& x) const {
  auto g = gpu_of(*this);
  if (!g) g = bind_gpu(this, widths_, inputs_, targets_);
  std::lock_guard<std::mutex> lock(g->mu);
  spb_ctx* c = g->ctx(1, 1);
  std::vector<const double*> p(x.size());
  for (size_t l = 0; l < x.size(); ++l) p[l] = x[l].data();
  double out = 0.0;
  check(spb_loss64(c, p.data(), nullptr, 0, &out), c);
  return out / dataset_size_;
}

void ChainMlp::add_sample_gradient(const Params& x, int sample, int suffix, Params& acc, BackpropStats* stats) const {
  const int L = layer_count();
  if (suffix < 1 || suffix > L) throw ArgumentError("suffix out of range");
  if (sample < 0 || sample >= dataset_size_) throw ArgumentError("sample out of range");
  auto g = gpu_of(*this);
  if (!g) g = bind_gpu(this, widths_, inputs_, targets_);
  std::lock_guard<std::mutex> lock(g->mu);
  spb_ctx* c = g->ctx(1, 1);
  g->upload(c, x);
  std::vector<std::vector<float>> bufs;
  auto out = g->block_ptrs(bufs);
  std::vector<long long> ops(L, 0);
  int cov = 0;
  check(spb_partial_backprop(c, &sample, 1, suffix, out.data(), ops.data(), &cov), c);
  for (int l = cov; l <= L; ++l)
    for (size_t i = 0; i < bufs[l - 1].size(); ++i) acc[l - 1][i] += static_cast<double>(bufs[l - 1][i]);
  if (stats)
    for (int l = 0; l < L; ++l) stats->layer_ops[l] += ops[l];
}

// ---- instance generators (model.cpp:191-231: the same Rng streams and
// draw order, so instances are identical to the reference's) -----------------

std::unique_ptr<BlockQuadratic> make_random_quadratic(int blocks, int block_dim, int samples, double target_noise,
                                                      std::uint64_t seed) {
  Rng rng = Rng(seed).split(0x9A4DULL);
  const int dim = blocks * block_dim;
  std::vector<double> a(static_cast<size_t>(samples) * dim), x_true(dim), b(samples);
  for (double& v : a) v = rng.next_gaussian();
  for (double& v : x_true) v = rng.next_gaussian();
  for (int s = 0; s < samples; ++s) {
    double dot = 0.0;
    for (int c = 0; c < dim; ++c) dot += a[static_cast<size_t>(s) * dim + c] * x_true[c];
    b[s] = dot + target_noise * rng.next_gaussian();
  }
  return std::make_unique<BlockQuadratic>(std::move(a), std::move(b), blocks);
}

std::unique_ptr<ChainMlp> make_random_chain_mlp(const std::vector<int>& widths, int samples, std::uint64_t seed) {
  Rng rng = Rng(seed).split(0x313aULL);
  const int L = static_cast<int>(widths.size()) - 1;
  Params w(std::max(L, 0));
  for (int l = 0; l < L; ++l) {  // U(-1/sqrt(n_in), 1/sqrt(n_in)), weights then biases
    w[l].resize(static_cast<size_t>(widths[l + 1]) * widths[l] + widths[l + 1]);
    const double scale = 1.0 / std::sqrt(static_cast<double>(widths[l]));
    for (double& v : w[l]) v = scale * (2.0 * rng.next_unit() - 1.0);
  }
  std::vector<std::vector<double>> inputs(samples);
  std::vector<double> targets(samples);
  for (int s = 0; s < samples; ++s) {  // inputs N(0,1); target tanh(sum) + 0.1 N(0,1)
    inputs[s].resize(widths.empty() ? 0 : widths[0]);
    double t = 0.0;
    for (double& v : inputs[s]) {
      v = rng.next_gaussian();
      t += v;
    }
    targets[s] = std::tanh(t) + 0.1 * rng.next_gaussian();
  }
  return std::make_unique<ChainMlp>(widths, std::move(inputs), std::move(targets), std::move(w));
}

// ============================================================================
// spb.hpp
// ============================================================================

void SpbConfig::validate() const {  // spb.cpp:11-14
  if (k < 1) throw ArgumentError("SpbConfig: k must be >= 1");
  if (B < 1 || B % k != 0) throw ArgumentError("SpbConfig: B must be positive and divisible by k");
}

int suffix_layers(int j, int k, int L) {
  int out = 0;
  check(spb_suffix_layers(j, k, L, &out));
  return out;
}

std::vector<int> chunk_coverage(int m, int k) {
  if (k < 1) throw ArgumentError("chunk_coverage: k must be >= 1");
  if (m < 1 || m > k) throw ArgumentError("chunk_coverage: chunk index out of range");
  std::vector<int> out(m);
  check(spb_chunk_coverage(m, k, out.data()));
  return out;
}

std::vector<std::pair<int, int>> chunk_layout(int k, int L) {
  if (k < 1 || L < 1) throw ArgumentError("chunk_layout: k and L must be >= 1");
  std::vector<int> flat(2 * static_cast<size_t>(k));
  check(spb_chunk_layout(k, L, flat.data()));
  std::vector<std::pair<int, int>> spans(k);
  for (int m = 0; m < k; ++m) spans[m] = {flat[2 * m], flat[2 * m + 1]};
  return spans;
}

std::vector<int> layer_chunks(int k, int L) {
  if (k < 1 || L < 1) throw ArgumentError("chunk_layout: k and L must be >= 1");
  std::vector<int> out(L);
  check(spb_layer_chunks(k, L, out.data()));
  return out;
}

PartialGradient partial_backprop(const LayeredModel& model, const Params& x, std::span<const int> batch, int suffix,
                                 BackpropStats* stats) {
  const int L = model.layer_count();
  if (suffix < 1 || suffix > L) throw ArgumentError("partial_backprop: suffix out of range");
  if (batch.empty()) throw ArgumentError("partial_backprop: empty batch");
  PartialGradient g;
  g.covered_from = L - suffix + 1;
  g.blocks.resize(L);
  if (stats && stats->layer_ops.empty()) stats->layer_ops.assign(L, 0);
  if (auto gpu = gpu_of(model)) {
    // The batch mean over the suffix as one device pass (worker rows through
    // the tcgen05 forward + truncated backward); covered blocks are the same
    // bits for every suffix that covers them, as the reference promises.
    std::lock_guard<std::mutex> lock(gpu->mu);
    spb_ctx* c = gpu->ctx(1, 1);
    gpu->upload(c, x);
    std::vector<std::vector<float>> bufs;
    auto out = gpu->block_ptrs(bufs);
    std::vector<long long> ops(L, 0);
    int cov = 0;
    check(spb_partial_backprop(c, batch.data(), static_cast<int>(batch.size()), suffix, out.data(), ops.data(), &cov),
          c);
    for (int l = g.covered_from; l <= L; ++l) g.blocks[l - 1].assign(bufs[l - 1].begin(), bufs[l - 1].end());
    if (stats)
      for (int l = 0; l < L; ++l) stats->layer_ops[l] += ops[l];
    return g;
  }
  // Any other LayeredModel (the BlockQuadratic fixture, user models): the
  // batch mean of its per-sample gradients, accumulated in batch order.
  for (int l = g.covered_from; l <= L; ++l) g.blocks[l - 1].assign(model.block_dims()[l - 1], 0.0);
  for (int s : batch) model.add_sample_gradient(x, s, suffix, g.blocks, stats);
  const double inv = 1.0 / static_cast<double>(batch.size());
  for (int l = g.covered_from; l <= L; ++l)
    for (double& v : g.blocks[l - 1]) v *= inv;
  return g;
}

Params aggregate(const std::vector<PartialGradient>& grads, int k) {
  if (k < 1 || static_cast<int>(grads.size()) != k) throw ArgumentError("aggregate: need exactly k gradients");
  const int L = static_cast<int>(grads[0].blocks.size());
  for (const auto& g : grads)
    if (static_cast<int>(g.blocks.size()) != L) throw ProtocolError("aggregate: gradient layer counts differ");
  std::vector<const double*> blocks(static_cast<size_t>(k) * L, nullptr);
  std::vector<int> dims(static_cast<size_t>(k) * L, 0), cov(k);
  for (int j = 0; j < k; ++j) {
    cov[j] = grads[j].covered_from;
    for (int l = 0; l < L; ++l) {
      const auto& b = grads[j].blocks[l];
      blocks[static_cast<size_t>(j) * L + l] = b.empty() ? nullptr : b.data();
      dims[static_cast<size_t>(j) * L + l] = static_cast<int>(b.size());
    }
  }
  // Output sizes: the contributors' block size per layer (checked equal on the device side).
  Params out(L);
  std::vector<double*> op(L);
  for (int l = 0; l < L; ++l) {
    size_t d = 0;
    for (int j = 0; j < k; ++j) d = std::max(d, grads[j].blocks[l].size());
    out[l].assign(d, 0.0);
    op[l] = out[l].data();
  }
  check(spb_aggregate64(-1, k, L, blocks.data(), dims.data(), cov.data(), op.data()));
  return out;
}

SgdResult spb_sgd_run(const LayeredModel& model, const SpbConfig& cfg, int iterations, StepSchedule schedule,
                      std::uint64_t seed, bool record_iterates) {
  cfg.validate();
  if (iterations < 1) throw ArgumentError("spb_sgd_run: iterations must be >= 1");
  double beta = 0.0;
  if (schedule == StepSchedule::Theorem1) {
    if (model.kind() != ModelKind::ConvexQuadratic) throw ConfigError("Theorem1 schedule requires the convex model");
    if (cfg.R <= 0.0 || cfg.V <= 0.0) throw ConfigError("Theorem1 schedule requires R, V > 0");
    beta = *model.beta();
  }
  const auto f_star = model.optimum_value();
  SgdResult res;
  res.avg_loss.reserve(iterations);
  res.step_size.reserve(iterations);
  Params x = model.initial_params();
  Params xbar = model.zeros_like();
  auto record = [&](int s, double gamma) {
    // Running average of x_2 .. x_{t+1} and f(xbar_s) (spb.cpp:198-206).
    for (size_t l = 0; l < x.size(); ++l)
      for (size_t c = 0; c < x[l].size(); ++c) xbar[l][c] += (x[l][c] - xbar[l][c]) / s;
    const double fl = model.loss(xbar);
    res.avg_loss.push_back(fl);
    res.step_size.push_back(gamma);
    if (f_star) res.avg_subopt.push_back(fl - *f_star);
    if (record_iterates) res.iterates.push_back(x);
  };
  auto gpu = gpu_of(model);
  if (gpu && schedule == StepSchedule::Constant) {
    // Device-resident SPB iterations: the k workers' batches drawn on the GPU
    // from Rng(seed).split(s).split(j) (bit-exact with the reference's
    // draws), forward, truncated backward, contributor aggregation in the
    // wgrad GEMMs and x -= lr g -- one graph replay per iteration.
    std::unique_lock<std::mutex> lock(gpu->mu);
    spb_ctx* c = gpu->ctx(cfg.k, cfg.B / cfg.k);
    gpu->upload(c, x);
    gpu->uploaded.erase(c);  // the device parameters move away from the host copy
    check(spb_set_optimizer(c, static_cast<float>(cfg.lr_base), 0.f, 0.f), c);
    std::vector<std::vector<float>> bufs;
    auto out = gpu->block_ptrs(bufs);
    for (int s = 1; s <= iterations; ++s) {
      check(spb_train_steps(c, seed, s, 1, 0, nullptr), c);
      check(spb_get_params(c, out.data()), c);
      for (size_t l = 0; l < x.size(); ++l) x[l].assign(bufs[l].begin(), bufs[l].end());
      lock.unlock();  // loss() takes the model lock itself
      record(s, cfg.lr_base);
      lock.lock();
    }
  } else {
    Rng root(seed);
    for (int s = 1; s <= iterations; ++s) {
      Params g = spb_estimate(model, cfg, x, root.split(static_cast<std::uint64_t>(s)));
      double gamma = cfg.lr_base;
      if (schedule == StepSchedule::Theorem1) {  // 1 / (beta + 1/eta(s)), eta(s) = (R/V) sqrt(2/s)
        const double eta = (cfg.R / cfg.V) * std::sqrt(2.0 / static_cast<double>(s));
        gamma = 1.0 / (beta + 1.0 / eta);
      }
      axpy(x, -gamma, g);
      record(s, gamma);
    }
  }
  res.avg_iterate = std::move(xbar);
  return res;
}

VarianceEstimate empirical_variance(const LayeredModel& model, const SpbConfig& cfg, const Params& x, int trials,
                                    std::uint64_t seed) {
  cfg.validate();
  if (trials < 1) throw ArgumentError("empirical_variance: trials must be >= 1");
  VarianceEstimate est;
  if (auto gpu = gpu_of(model)) {
    // The device estimator, with the reference's sampling protocol
    // (kWorkerDrawTag / kChunkDrawTag streams) sample for sample.
    std::lock_guard<std::mutex> lock(gpu->mu);
    spb_ctx* c = gpu->ctx(cfg.k, cfg.B / cfg.k);
    gpu->upload(c, x);
    std::vector<double> out(4 + 2 * static_cast<size_t>(cfg.k));
    check(spb_empirical_variance(c, cfg.k, cfg.B, trials, seed, out.data()), c);
    est.spb = out[0], est.spb_se = out[1], est.baseline = out[2], est.baseline_se = out[3];
    est.p_hat.assign(out.begin() + 4, out.begin() + 4 + cfg.k);
    est.p_se.assign(out.begin() + 4 + cfg.k, out.end());
    return est;
  }
  const Params grad = full_gradient(model, x);
  const Rng root(seed);
  const Rng worker_draws = root.split(kWorkerDrawTag);
  double s1 = 0, s2 = 0, b1 = 0, b2 = 0;
  for (int r = 1; r <= trials; ++r) {
    const Rng stream = worker_draws.split(static_cast<std::uint64_t>(r));
    const double ds = block_distance_sq(grad, spb_estimate(model, cfg, x, stream));
    const double db = block_distance_sq(grad, baseline_estimate(model, cfg, x, stream));
    s1 += ds, s2 += ds * ds, b1 += db, b2 += db * db;
  }
  mean_and_se(s1, s2, trials, est.spb, est.spb_se);
  mean_and_se(b1, b2, trials, est.baseline, est.baseline_se);
  // p_i: one single-sample gradient per trial, restricted to chunk i's layers.
  const int L = model.layer_count();
  const auto spans = chunk_layout(cfg.k, L);
  const Rng chunk_draws = root.split(kChunkDrawTag);
  est.p_hat.assign(cfg.k, 0.0);
  est.p_se.assign(cfg.k, 0.0);
  for (int m = 1; m <= cfg.k; ++m) {
    Rng stream = chunk_draws.split(static_cast<std::uint64_t>(m));
    double p1 = 0, p2 = 0;
    for (int r = 1; r <= trials; ++r) {
      const int sample = static_cast<int>(stream.next_below(static_cast<std::uint64_t>(model.dataset_size())));
      Params g = model.zeros_like();
      model.add_sample_gradient(x, sample, L, g);
      const double d = span_distance_sq(grad, g, spans[m - 1].first, spans[m - 1].second);
      p1 += d, p2 += d * d;
    }
    mean_and_se(p1, p2, trials, est.p_hat[m - 1], est.p_se[m - 1]);
  }
  return est;
}

Params full_gradient(const LayeredModel& model, const Params& x) {
  std::vector<int> all(model.dataset_size());
  std::iota(all.begin(), all.end(), 0);
  return partial_backprop(model, x, all, model.layer_count()).blocks;
}

std::vector<double> exact_chunk_variances(const LayeredModel& model, const Params& x, int k) {
  const int L = model.layer_count(), N = model.dataset_size();
  const Params grad = full_gradient(model, x);
  const auto spans = chunk_layout(k, L);
  std::vector<double> p(k, 0.0);
  for (int s = 0; s < N; ++s) {
    Params g = model.zeros_like();
    model.add_sample_gradient(x, s, L, g);
    for (int m = 1; m <= k; ++m) p[m - 1] += span_distance_sq(grad, g, spans[m - 1].first, spans[m - 1].second);
  }
  for (double& v : p) v /= N;
  return p;
}

double exact_spb_variance(const LayeredModel& model, const SpbConfig& cfg, const Params& x) {
  // sum_i (k / (i B)) p_i(x) (spb.hpp:113-114).
  const auto p = exact_chunk_variances(model, x, cfg.k);
  double v = 0.0;
  for (int m = 1; m <= cfg.k; ++m) v += static_cast<double>(cfg.k) / (static_cast<double>(m) * cfg.B) * p[m - 1];
  return v;
}

double measured_grad_norm_bound(const LayeredModel& model, const Params& x) {
  const int N = model.dataset_size(), L = model.layer_count();
  double worst = 0.0;
  for (int s = 0; s < N; ++s) {
    Params g = model.zeros_like();
    model.add_sample_gradient(x, s, L, g);
    double n2 = 0.0;
    for (const auto& blk : g)
      for (double v : blk) n2 += v * v;
    worst = std::max(worst, n2);
  }
  return std::sqrt(worst);
}

double block_distance_sq(const Params& a, const Params& b) {
  double d = 0.0;
  for (size_t l = 0; l < a.size(); ++l)
    for (size_t c = 0; c < a[l].size(); ++c) {
      const double e = a[l][c] - b[l][c];
      d += e * e;
    }
  return d;
}

void axpy(Params& y, double alpha, const Params& x) {
  for (size_t l = 0; l < y.size(); ++l)
    for (size_t c = 0; c < y[l].size(); ++c) y[l][c] += alpha * x[l][c];
}

}  // namespace jigsaw::spb
