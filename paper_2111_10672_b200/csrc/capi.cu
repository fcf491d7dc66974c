// The extern "C" surface of include/spb_b200.h over spb::Engine: every entry
// point maps C++ exceptions to spb_status codes (guard) and records the
// message for spb_last_error.
#include "engine.hpp"

namespace spb {
namespace {
thread_local std::string g_err;
}  // namespace
}  // namespace spb

using spb::Engine;

struct spb_ctx {
  Engine e;
};

namespace {

template <class F>
spb_status guard(spb_ctx* ctx, F&& f) {
  std::string* err = ctx ? &ctx->e.err : &spb::g_err;
  try {
    if (ctx) SPB_CUDA(cudaSetDevice(ctx->e.dev));
    f();
    return SPB_OK;
  } catch (const spb::ArgumentError& x) {
    *err = x.what();
    return SPB_E_ARGUMENT;
  } catch (const spb::ProtocolError& x) {
    *err = x.what();
    return SPB_E_PROTOCOL;
  } catch (const spb::ConfigError& x) {
    *err = x.what();
    return SPB_E_CONFIG;
  } catch (const spb::CudaError& x) {
    *err = x.what();
    return SPB_E_CUDA;
  } catch (const std::invalid_argument& x) {
    *err = x.what();
    return SPB_E_ARGUMENT;
  } catch (const std::exception& x) {
    *err = x.what();
    return SPB_E_CUDA;
  }
}

}  // namespace

namespace spb {
namespace {
// aggregate (spb.cpp:70-106): the reference's protocol checks (spb.cpp:74-87,
// 91-99), before any device work. Returns the layer -> contributor counts.
template <class T>
std::vector<int> aggregate_validate(int k, int L, const T* const* blocks, const int* dims, const int* covered_from) {
  if (k < 1) throw ArgumentError("aggregate: need exactly k gradients");
  if (L < 1) throw ProtocolError("aggregate: gradient layer counts differ");
  for (int j = 1; j <= k; ++j) {
    const int expect_from = L - suffix_layers(j, k, L) + 1;
    if (covered_from[j - 1] != expect_from)
      throw ProtocolError("aggregate: worker " + std::to_string(j) + " coverage does not match the suffix rule");
    for (int l = 1; l <= L; ++l) {
      const bool present = blocks[(j - 1) * L + l - 1] != nullptr && dims[(j - 1) * L + l - 1] > 0;
      if (present != (l >= covered_from[j - 1]))
        throw ProtocolError("aggregate: block presence inconsistent with covered_from");
    }
  }
  auto chunk_of = layer_chunks(k, L);
  for (int l = 1; l <= L; ++l) {
    const int m = chunk_of[l - 1];
    const long dim = dims[(k - m) * L + l - 1];
    for (int wkr = k - m + 1; wkr <= k; ++wkr)
      if (dims[(wkr - 1) * L + l - 1] != dim) throw ProtocolError("aggregate: block dimension mismatch");
  }
  return chunk_of;
}

// Per-thread, per-device staging for the aggregator entry points: grown on
// demand and reused across calls (the reference's callers aggregate once per
// SGD iteration -- thousands of times in its verify suite).
struct AggWorkspace {
  void* stage = nullptr;
  size_t stage_bytes = 0;
  void* ptrs = nullptr;
  size_t ptr_bytes = 0;
  cudaStream_t st = nullptr;
  ~AggWorkspace() {
    if (stage) cudaFree(stage);
    if (ptrs) cudaFree(ptrs);
    if (st) cudaStreamDestroy(st);
  }
  static AggWorkspace& get(int dev) {
    thread_local std::map<int, AggWorkspace> per_device;
    return per_device[dev];
  }
  void reserve(size_t sb, size_t pb) {
    if (sb > stage_bytes) {
      if (stage) cudaFree(stage), stage = nullptr, stage_bytes = 0;
      SPB_CUDA(cudaMalloc(&stage, sb));
      stage_bytes = sb;
    }
    if (pb > ptr_bytes) {
      if (ptrs) cudaFree(ptrs), ptrs = nullptr, ptr_bytes = 0;
      SPB_CUDA(cudaMalloc(&ptrs, pb));
      ptr_bytes = pb;
    }
    if (!st) SPB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  }
};

// The per-layer contributor means of validated host blocks, on the GPU.
template <class T>
void aggregate_run(int k, int L, const std::vector<int>& chunk_of, const T* const* blocks, const int* dims,
                   T* const* out, int dev) {
  std::vector<long> base(L + 1, 0), pbase(L + 1, 0);
  for (int l = 1; l <= L; ++l) {
    const int m = chunk_of[l - 1];
    const long dim = dims[(k - m) * L + l - 1];
    base[l] = base[l - 1] + round_up(dim * (m + 1), 32);
    pbase[l] = pbase[l - 1] + m;
  }
  AggWorkspace& ws = AggWorkspace::get(dev);
  ws.reserve(std::max(1L, base[L]) * sizeof(T), std::max(1L, pbase[L]) * sizeof(T*));
  cudaStream_t st = ws.st;
  T* stage = static_cast<T*>(ws.stage);
  const T** ptrs = static_cast<const T**>(ws.ptrs);
  std::vector<const T*> hp(pbase[L]);
  for (int l = 1; l <= L; ++l) {
    const int m = chunk_of[l - 1];
    const long dim = dims[(k - m) * L + l - 1];
    for (int i = 0; i < m; ++i) hp[pbase[l - 1] + i] = stage + base[l - 1] + i * dim;
  }
  SPB_CUDA(cudaMemcpyAsync(ptrs, hp.data(), hp.size() * sizeof(T*), cudaMemcpyHostToDevice, st));
  for (int l = 1; l <= L; ++l) {
    const int m = chunk_of[l - 1];
    const long dim = dims[(k - m) * L + l - 1];
    T* sl = stage + base[l - 1];
    for (int i = 0; i < m; ++i)
      SPB_CUDA(cudaMemcpyAsync(sl + i * dim, blocks[(k - m + i) * L + l - 1], dim * sizeof(T), cudaMemcpyHostToDevice,
                               st));
    if constexpr (sizeof(T) == 8)
      launch_aggregate64(ptrs + pbase[l - 1], m, dim, sl + m * dim, st);
    else
      launch_aggregate(ptrs + pbase[l - 1], m, dim, sl + m * dim, st);
    SPB_CUDA(cudaMemcpyAsync(out[l - 1], sl + m * dim, dim * sizeof(T), cudaMemcpyDeviceToHost, st));
  }
  SPB_CUDA(cudaStreamSynchronize(st));  // the staging is reused by the next call
}
}  // namespace
}  // namespace spb

extern "C" {

const char* spb_last_error(const spb_ctx* ctx) { return ctx ? ctx->e.err.c_str() : spb::g_err.c_str(); }

spb_status spb_suffix_layers(int j, int k, int L, int* out) {
  return guard(nullptr, [&] { *out = spb::suffix_layers(j, k, L); });
}

spb_status spb_chunk_coverage(int m, int k, int* out) {
  return guard(nullptr, [&] {
    auto v = spb::chunk_coverage(m, k);
    std::copy(v.begin(), v.end(), out);
  });
}

spb_status spb_chunk_layout(int k, int L, int* out) {
  return guard(nullptr, [&] {
    auto v = spb::chunk_layout(k, L);
    for (int m = 0; m < k; ++m) out[2 * m] = v[m].first, out[2 * m + 1] = v[m].second;
  });
}

spb_status spb_layer_chunks(int k, int L, int* out) {
  return guard(nullptr, [&] {
    auto v = spb::layer_chunks(k, L);
    std::copy(v.begin(), v.end(), out);
  });
}

spb_status spb_draw_batch(uint64_t seed, int step, int worker, int count, int dataset_size, int* out) {
  return guard(nullptr, [&] {
    if (count < 0 || dataset_size < 1) throw spb::ArgumentError("draw_batch: bad size");
    spb::Rng r = spb::Rng(seed).split(static_cast<uint64_t>(step)).split(static_cast<uint64_t>(worker));
    for (int i = 0; i < count; ++i) out[i] = static_cast<int>(r.next_below(static_cast<uint64_t>(dataset_size)));
  });
}

spb_status spb_rank_workers(int k, int L, int rank, int nranks, int* out, int* count) {
  return guard(nullptr, [&] {
    auto v = spb::rank_workers(k, L, rank, nranks);
    std::copy(v.begin(), v.end(), out);
    *count = static_cast<int>(v.size());
  });
}

spb_status spb_create(const int* widths, int n_widths, int k, int per_worker_batch, int device, spb_ctx** out) {
  *out = nullptr;
  auto ctx = std::make_unique<spb_ctx>();
  spb_status s = guard(nullptr, [&] { ctx->e.init(widths, n_widths, k, per_worker_batch, device); });
  if (s == SPB_OK) *out = ctx.release();
  return s;
}

spb_status spb_create_conv(const int* geom, int nconv, int nout, int k, int per_worker_batch, int device,
                           spb_ctx** out) {
  *out = nullptr;
  auto ctx = std::make_unique<spb_ctx>();
  spb_status s = guard(nullptr, [&] { ctx->e.init_conv(geom, nconv, nout, k, per_worker_batch, device); });
  if (s == SPB_OK) *out = ctx.release();
  return s;
}

spb_status spb_destroy(spb_ctx* ctx) {
  if (ctx) {
    cudaSetDevice(ctx->e.dev);
    if (cudaStreamSynchronize(ctx->e.st) == cudaSuccess && ctx->e.loss_pin)
      ctx->e.flush_losses();  // spb_step_host_async losses not yet handed out
    delete ctx;
  }
  return SPB_OK;
}

spb_status spb_set_dataset(spb_ctx* ctx, const float* X, const float* Y, int N) {
  return guard(ctx, [&] {
    auto& e = ctx->e;
    if (N < 1) throw spb::ArgumentError("mlp: dataset shape mismatch");
    SPB_CUDA(cudaStreamSynchronize(e.st));
    if (e.X) cudaFree(e.X), cudaFree(e.Y);
    const long row = e.conv_model ? e.ldx : e.w[0];  // values per sample (ConvNet: an NHWC image)
    e.X = Engine::alloc<float>(static_cast<long>(N) * e.ldx);
    e.Y = Engine::alloc<float>(static_cast<long>(N) * e.nout);
    SPB_CUDA(cudaMemcpy2D(e.X, e.ldx * 4, X, row * 4, row * 4, N, cudaMemcpyHostToDevice));
    SPB_CUDA(cudaMemcpy(e.Y, Y, static_cast<size_t>(N) * e.nout * 4, cudaMemcpyHostToDevice));
    e.N = N;
    e.invalidate_graphs();
  });
}

spb_status spb_set_params(spb_ctx* ctx, const float* const* blocks) {
  return guard(ctx, [&] {
    auto& e = ctx->e;
    for (int l = 1; l <= e.L; ++l) {
      const int no = e.w[l], ni = e.fan[l];
      SPB_CUDA(cudaMemsetAsync(e.tmp, 0, e.tmp_n * 4, e.st));
      SPB_CUDA(cudaMemcpy2DAsync(e.tmp, e.ldf[l] * 4, blocks[l - 1], ni * 4, ni * 4, no, cudaMemcpyHostToDevice,
                                 e.st));
      spb::launch_split(e.tmp, no * e.ldf[l], e.p_hi + e.w_off[l], e.p_lo + e.w_off[l], e.st);
      SPB_CUDA(cudaMemcpyAsync(e.tmp, blocks[l - 1] + static_cast<long>(no) * ni, no * 4, cudaMemcpyHostToDevice,
                               e.st));
      spb::launch_split(e.tmp, no, e.p_hi + e.b_off[l], e.p_lo + e.b_off[l], e.st);
      SPB_CUDA(cudaStreamSynchronize(e.st));
    }
    if (e.mom) SPB_CUDA(cudaMemsetAsync(e.mom, 0, e.nflat * 4, e.st));
    SPB_CUDA(cudaStreamSynchronize(e.st));
  });
}

spb_status spb_get_params(spb_ctx* ctx, float* const* blocks) {
  return guard(ctx, [&] {
    auto& e = ctx->e;
    for (int l = 1; l <= e.L; ++l) {
      const int no = e.w[l], ni = e.fan[l];
      spb::launch_join(e.p_hi + e.w_off[l], e.p_lo + e.w_off[l], no * e.ldf[l], e.tmp, e.st);
      SPB_CUDA(cudaMemcpy2DAsync(blocks[l - 1], ni * 4, e.tmp, e.ldf[l] * 4, ni * 4, no, cudaMemcpyDeviceToHost,
                                 e.st));
      SPB_CUDA(cudaStreamSynchronize(e.st));
      spb::launch_join(e.p_hi + e.b_off[l], e.p_lo + e.b_off[l], no, e.tmp, e.st);
      SPB_CUDA(cudaMemcpyAsync(blocks[l - 1] + static_cast<long>(no) * ni, e.tmp, no * 4, cudaMemcpyDeviceToHost,
                               e.st));
      SPB_CUDA(cudaStreamSynchronize(e.st));
    }
  });
}

spb_status spb_get_grads(spb_ctx* ctx, float* const* blocks) {
  return guard(ctx, [&] {
    auto& e = ctx->e;
    for (int l = 1; l <= e.L; ++l) {
      if (!blocks[l - 1]) continue;
      const int no = e.w[l], ni = e.fan[l];
      SPB_CUDA(cudaMemcpy2DAsync(blocks[l - 1], ni * 4, e.grad + e.w_off[l], e.ldf[l] * 4, ni * 4, no,
                                 cudaMemcpyDeviceToHost, e.st));
      SPB_CUDA(cudaMemcpyAsync(blocks[l - 1] + static_cast<long>(no) * ni, e.grad + e.b_off[l], no * 4,
                               cudaMemcpyDeviceToHost, e.st));
    }
    SPB_CUDA(cudaStreamSynchronize(e.st));
  });
}

spb_status spb_set_fused_update(spb_ctx* ctx, int fused) {
  return guard(ctx, [&] {
    if (fused < 0 || fused > 2) throw spb::ArgumentError("set_fused_update: mode must be 0, 1 or 2");
    ctx->e.fused_mode = fused;
    ctx->e.invalidate_graphs();
  });
}

spb_status spb_set_chain(spb_ctx* ctx, int steps) {
  return guard(ctx, [&] {
    if (steps < 1 || steps > Engine::kMaxChain) throw spb::ArgumentError("set_chain: steps must be in [1, 16]");
    ctx->e.chain = steps;
  });
}

spb_status spb_set_optimizer(spb_ctx* ctx, float lr, float momentum, float weight_decay) {
  return guard(ctx, [&] {
    auto& e = ctx->e;
    e.lr = lr;
    e.mu = momentum;
    e.wd = weight_decay;
    if (momentum != 0.f && !e.mom) e.mom = Engine::alloc<float>(e.nflat);
    e.invalidate_graphs();
  });
}

spb_status spb_partial_backprop(spb_ctx* ctx, const int* batch, int len, int suffix, float* const* out_blocks,
                                long long* layer_ops, int* covered_from) {
  return guard(ctx, [&] {
    auto& e = ctx->e;
    const int L = e.L;
    if (suffix < 1 || suffix > L) throw spb::ArgumentError("partial_backprop: suffix out of range");
    if (len <= 0) throw spb::ArgumentError("partial_backprop: empty batch");
    if (!e.X) throw spb::ConfigError("partial_backprop: no dataset");
    for (int i = 0; i < len; ++i)
      if (batch[i] < 0 || batch[i] >= e.N) throw spb::ArgumentError("sample out of range");
    e.ensure_rows(len);
    const int stop = L - suffix + 1;
    SPB_CUDA(cudaMemcpyAsync(e.idx_in, batch, len * sizeof(int), cudaMemcpyHostToDevice, e.st));
    e.enqueue_gather(e.X, e.ldx, len, len, nullptr, 0, nullptr, 0, e.idx_in, e.st);
    std::vector<int> row0(L + 1, len);
    std::vector<float> alpha(L + 1, 1.0f / static_cast<float>(len));
    for (int l = stop; l <= L; ++l) row0[l] = 0;
    e.enqueue_pass(len, row0, alpha, e.st);
    for (int l = stop; l <= L; ++l) {
      if (!out_blocks[l - 1]) continue;
      const int no = e.w[l], ni = e.fan[l];
      SPB_CUDA(cudaMemcpy2DAsync(out_blocks[l - 1], ni * 4, e.grad + e.w_off[l], e.ldf[l] * 4, ni * 4, no,
                                 cudaMemcpyDeviceToHost, e.st));
      SPB_CUDA(cudaMemcpyAsync(out_blocks[l - 1] + static_cast<long>(no) * ni, e.grad + e.b_off[l], no * 4,
                               cudaMemcpyDeviceToHost, e.st));
    }
    SPB_CUDA(cudaStreamSynchronize(e.st));
    if (covered_from) *covered_from = stop;
    if (layer_ops)  // model.cpp:165-184, per sample
      for (int l = stop; l <= L; ++l) {
        long long ops = static_cast<long long>(e.w[l]) * (e.fan[l] + 1);
        if (l > stop) ops += static_cast<long long>(e.w[l]) * e.fan[l] + e.fan[l];
        layer_ops[l - 1] += ops * len;
      }
  });
}

spb_status spb_aggregate(spb_ctx* ctx, int k, int L, const float* const* blocks, const int* dims,
                         const int* covered_from, float* const* out) {
  return guard(ctx, [&] {
    auto chunk_of = spb::aggregate_validate(k, L, blocks, dims, covered_from);
    spb::aggregate_run(k, L, chunk_of, blocks, dims, out, ctx->e.dev);
  });
}

spb_status spb_aggregate64(int device, int k, int L, const double* const* blocks, const int* dims,
                           const int* covered_from, double* const* out) {
  return guard(nullptr, [&] {
    auto chunk_of = spb::aggregate_validate(k, L, blocks, dims, covered_from);
    if (device >= 0) SPB_CUDA(cudaSetDevice(device));
    int dev = 0;
    SPB_CUDA(cudaGetDevice(&dev));
    spb::aggregate_run(k, L, chunk_of, blocks, dims, out, dev);
  });
}

spb_status spb_train_steps(spb_ctx* ctx, uint64_t seed, int step0, int steps, int full_backprop, float* losses) {
  return guard(ctx, [&] {
    auto& e = ctx->e;
    if (!e.X) throw spb::ConfigError("train_steps: no dataset");
    if (steps < 0) throw spb::ArgumentError("train_steps: steps must be >= 0");
    e.ensure_rows(static_cast<int>(e.workers.size()) * e.bw);
    spb::Ctl c{seed, step0, 0};
    SPB_CUDA(cudaMemcpyAsync(e.ctl, &c, sizeof c, cudaMemcpyHostToDevice, e.st));
    e.run_steps(full_backprop != 0, steps, losses);
    if (losses) {
      SPB_CUDA(cudaStreamSynchronize(e.st));
      e.flush_losses();
    }
  });
}

spb_status spb_step_host(spb_ctx* ctx, const float* X_rows, const float* Y_rows, int full_backprop, float* loss_out) {
  return guard(ctx, [&] {
    auto& e = ctx->e;
    const int rows = static_cast<int>(e.workers.size()) * e.bw;
    e.ensure_rows(rows);
    cudaGraphExec_t g = e.get_graph(full_backprop != 0, true, 1, &e.last_launches);
    const size_t per = e.conv_model ? static_cast<size_t>(e.ldx) : static_cast<size_t>(e.w[0]);
    SPB_CUDA(cudaMemcpyAsync(e.xin, X_rows, static_cast<size_t>(rows) * per * 4, cudaMemcpyHostToDevice, e.st));
    SPB_CUDA(cudaMemcpyAsync(e.ybatch, Y_rows, static_cast<size_t>(rows) * e.nout * 4, cudaMemcpyHostToDevice, e.st));
    SPB_CUDA(cudaGraphLaunch(g, e.st));
    SPB_CUDA(cudaMemcpyAsync(loss_out, e.loss_dev, 4, cudaMemcpyDeviceToHost, e.st));
    SPB_CUDA(cudaStreamSynchronize(e.st));
    e.flush_losses();  // earlier spb_step_host_async steps are complete too
  });
}

spb_status spb_step_host_async(spb_ctx* ctx, const float* X_rows, const float* Y_rows, int full_backprop,
                               float* loss_out) {
  return guard(ctx, [&] {
    auto& e = ctx->e;
    const int rows = static_cast<int>(e.workers.size()) * e.bw;
    e.ensure_rows(rows);
    const long per = e.conv_model ? static_cast<long>(e.ldx) : static_cast<long>(e.w[0]);
    const long nx = rows * per, ny = static_cast<long>(rows) * e.nout;
    if (!e.hst) SPB_CUDA(cudaStreamCreateWithFlags(&e.hst, cudaStreamNonBlocking));
    if (nx > e.hx_n || ny > e.hy_n) {
      SPB_CUDA(cudaStreamSynchronize(e.st));
      SPB_CUDA(cudaStreamSynchronize(e.hst));
      for (int i = 0; i < 2; ++i) {
        if (e.hx[i]) cudaFree(e.hx[i]);
        if (e.hy[i]) cudaFree(e.hy[i]);
        e.hx[i] = Engine::alloc<float>(nx);
        e.hy[i] = Engine::alloc<float>(ny);
      }
      e.hx_n = nx, e.hy_n = ny;
    }
    int launches = 0;
    cudaGraphExec_t g = e.get_graph(full_backprop != 0, true, 1, &launches);
    const int b = static_cast<int>(e.host_calls++ & 1u);
    const int ev_done = spb::kEvP2pFork + 56 + b, ev_in = spb::kEvP2pFork + 58 + b;  // past the p2p joins (<= +47)
    // Staging slot b was last read by the step two calls ago (its D2D copy on st).
    if (e.host_calls > 2) SPB_CUDA(cudaStreamWaitEvent(e.hst, e.ev(ev_done), 0));
    SPB_CUDA(cudaMemcpyAsync(e.hx[b], X_rows, nx * 4, cudaMemcpyHostToDevice, e.hst));
    SPB_CUDA(cudaMemcpyAsync(e.hy[b], Y_rows, ny * 4, cudaMemcpyHostToDevice, e.hst));
    SPB_CUDA(cudaEventRecord(e.ev(ev_in), e.hst));
    SPB_CUDA(cudaStreamWaitEvent(e.st, e.ev(ev_in), 0));
    SPB_CUDA(cudaMemcpyAsync(e.xin, e.hx[b], nx * 4, cudaMemcpyDeviceToDevice, e.st));
    SPB_CUDA(cudaMemcpyAsync(e.ybatch, e.hy[b], ny * 4, cudaMemcpyDeviceToDevice, e.st));
    SPB_CUDA(cudaEventRecord(e.ev(ev_done), e.st));
    SPB_CUDA(cudaGraphLaunch(g, e.st));
    if (!e.loss_pin) SPB_CUDA(cudaMallocHost(&e.loss_pin, Engine::kLossRing * sizeof(float)));
    if (static_cast<int>(e.loss_pending.size()) == Engine::kLossRing) {  // ring full: drain it
      SPB_CUDA(cudaStreamSynchronize(e.st));
      e.flush_losses();
    }
    const int slot = static_cast<int>((e.host_calls - 1) % Engine::kLossRing);
    SPB_CUDA(cudaMemcpyAsync(e.loss_pin + slot, e.loss_dev, 4, cudaMemcpyDeviceToHost, e.st));
    e.loss_pending.push_back({loss_out, slot});
    e.last_launches = launches;
  });
}

spb_status spb_loss(spb_ctx* ctx, double* out) {
  return guard(ctx, [&] {
    auto& e = ctx->e;
    if (!e.X) throw spb::ConfigError("loss: no dataset");
    const int chunk = e.cap_rows;
    std::vector<int> iota(chunk);
    double total = 0.0;
    std::vector<float> rl(chunk);
    for (int s0 = 0; s0 < e.N; s0 += chunk) {
      const int rows = std::min(chunk, e.N - s0);
      for (int i = 0; i < rows; ++i) iota[i] = s0 + i;
      SPB_CUDA(cudaMemcpyAsync(e.idx_in, iota.data(), rows * sizeof(int), cudaMemcpyHostToDevice, e.st));
      e.enqueue_gather(e.X, e.ldx, rows, rows, nullptr, 0, nullptr, 0, e.idx_in, e.st);
      std::vector<int> row0(e.L + 1, rows);  // forward + head only
      std::vector<float> alpha(e.L + 1, 0.f);
      e.enqueue_pass(rows, row0, alpha, e.st);
      SPB_CUDA(cudaMemcpyAsync(rl.data(), e.row_loss, rows * 4, cudaMemcpyDeviceToHost, e.st));
      SPB_CUDA(cudaStreamSynchronize(e.st));
      for (int i = 0; i < rows; ++i) total += rl[i];
    }
    *out = total / e.N;
  });
}

spb_status spb_loss64(spb_ctx* ctx, const double* const* blocks, const int* samples, int count, double* out) {
  return guard(ctx, [&] {
    auto& e = ctx->e;
    if (!e.X) throw spb::ConfigError("loss: no dataset");
    if (e.conv_model) throw spb::ConfigError("loss64: ChainMlp contexts only");
    if (!blocks || !out) throw spb::ArgumentError("loss64: null argument");
    const int L = e.L;
    std::vector<long> off(L + 1, 0);
    long maxw = 0;
    for (int l = 1; l <= L; ++l) {
      off[l] = off[l - 1] + static_cast<long>(e.w[l]) * e.w[l - 1] + e.w[l];
      maxw = std::max<long>(maxw, std::max(e.w[l], e.w[l - 1]));
    }
    // Parameters: re-uploaded only when they changed since the last call.
    bool same = e.p64_host.size() == static_cast<size_t>(off[L]);
    for (int l = 0; same && l < L; ++l)
      same = std::memcmp(e.p64_host.data() + off[l], blocks[l], (off[l + 1] - off[l]) * sizeof(double)) == 0;
    if (!same) {
      e.p64_host.resize(off[L]);
      for (int l = 0; l < L; ++l) std::memcpy(e.p64_host.data() + off[l], blocks[l], (off[l + 1] - off[l]) * 8);
      if (e.p64) cudaFree(e.p64), e.p64 = nullptr;
      SPB_CUDA(cudaMalloc(&e.p64, off[L] * sizeof(double)));
      SPB_CUDA(cudaMemcpyAsync(e.p64, e.p64_host.data(), off[L] * sizeof(double), cudaMemcpyHostToDevice, e.st));
    }
    const int n = samples ? count : e.N;
    if (n < 0) throw spb::ArgumentError("loss64: negative count");
    for (int i = 0; samples && i < n; ++i)
      if (samples[i] < 0 || samples[i] >= e.N) throw spb::ArgumentError("sample out of range");
    const int chunk = std::max(1, std::min(n, 2048));
    const long lda = spb::round_up(maxw, 4);
    struct DevBuf {
      void* p = nullptr;
      ~DevBuf() {
        if (p) cudaFree(p);
      }
    } a, b, rl, ix;
    SPB_CUDA(cudaMalloc(&a.p, chunk * lda * sizeof(double)));
    SPB_CUDA(cudaMalloc(&b.p, chunk * lda * sizeof(double)));
    SPB_CUDA(cudaMalloc(&rl.p, chunk * sizeof(double)));
    SPB_CUDA(cudaMalloc(&ix.p, chunk * sizeof(int)));
    std::vector<int> idx(chunk);
    std::vector<double> host_rl(chunk);
    double total = 0.0;
    for (int s0 = 0; s0 < n; s0 += chunk) {
      const int rows = std::min(chunk, n - s0);
      for (int i = 0; i < rows; ++i) idx[i] = samples ? samples[s0 + i] : s0 + i;
      SPB_CUDA(cudaMemcpyAsync(ix.p, idx.data(), rows * sizeof(int), cudaMemcpyHostToDevice, e.st));
      spb::launch_loss64(e.X, e.ldx, e.Y, static_cast<int*>(ix.p), rows, e.w.data(), L, e.p64, off.data(),
                         static_cast<double*>(a.p), static_cast<double*>(b.p), lda, static_cast<double*>(rl.p), e.st);
      SPB_CUDA(cudaMemcpyAsync(host_rl.data(), rl.p, rows * sizeof(double), cudaMemcpyDeviceToHost, e.st));
      SPB_CUDA(cudaStreamSynchronize(e.st));
      for (int i = 0; i < rows; ++i) total += host_rl[i];  // sample order, as ChainMlp::loss sums
    }
    *out = total;
  });
}

spb_status spb_synchronize(spb_ctx* ctx) {
  return guard(ctx, [&] {
    SPB_CUDA(cudaStreamSynchronize(ctx->e.st));
    ctx->e.flush_losses();
  });
}

void* spb_stream(spb_ctx* ctx) { return ctx ? static_cast<void*>(ctx->e.st) : nullptr; }

spb_status spb_comm_unique_id(void* out128) {
  return guard(nullptr, [&] {
    ncclUniqueId id;
    spb::nccl_check(spb::nccl().GetUniqueId(&id));
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(out128, &id, sizeof id);
  });
}

spb_status spb_comm_init(spb_ctx* ctx, const void* unique_id128, int rank, int nranks) {
  spb_status st = guard(ctx, [&] {
    auto& e = ctx->e;
    if (nranks < 1 || rank < 0 || rank >= nranks) throw spb::ArgumentError("comm: bad rank");
    if (nranks > e.k) throw spb::ArgumentError("comm: more ranks than SPB workers");
    if (e.comm) throw spb::ConfigError("comm: already initialised");
    ncclUniqueId id;
    std::memcpy(&id, unique_id128, sizeof id);
    spb::nccl_check(spb::nccl().CommInitRank(&e.comm, nranks, id, rank));
    e.rank = rank;
    e.nranks = nranks;
    SPB_CUDA(cudaStreamCreateWithFlags(&e.cst, cudaStreamNonBlocking));
    e.buckets[0] = spb::bucket_plan(e.k, e.L, nranks, false);
    e.buckets[1] = spb::bucket_plan(e.k, e.L, nranks, true);
    e.set_workers(spb::rank_workers(e.k, e.L, rank, nranks));
    e.ensure_rows(static_cast<int>(e.workers.size()) * e.bw);
    // Aggregation mode: SPB_COMM = rh | p2p | sub | push.
    // Default by measurement (cfg3): p2p for 2 ranks (one
    // pairwise copy-engine exchange); push from 3 to 8 ranks for the MLP
    // (gradient rows stored to their owners by the wgrad epilogue: 4.47 ms
    // vs rh 5.02, p2p 5.2, sub 6.6 at 4 ranks), rh for the ConvNet at a
    // power of two (push is MLP-only); sub otherwise -- NCCL over
    // contributor sub-communicators. Every mode is parity-tested at 2 and 4
    // ranks; 8 ranks could not be run here (gpurun offers at most 4 GPUs).
    const char* cm = std::getenv("SPB_COMM");
    const bool pow2 = (nranks & (nranks - 1)) == 0;
    const std::string mode =
        cm ? cm
           : (nranks == 2 ? "p2p"
                          : (e.conv_model ? (pow2 ? "rh" : "sub") : (nranks <= spb::kMaxPeers ? "push" : "sub")));
    if (mode != "p2p" && mode != "sub" && mode != "push" && mode != "rh")
      throw spb::ArgumentError("comm: SPB_COMM must be rh, push, p2p or sub");
    // NCCL's kernels need SMs while the backward GEMMs run: keep some free
    // (the copy-engine modes' few SM kernels measured the same with 0 / 16).
    const char* rs = std::getenv("SPB_COMM_SMS");
    e.reserved_sms = rs ? std::max(0, std::atoi(rs)) : (mode == "sub" ? 16 : 0);
    if (mode == "rh" && (nranks & (nranks - 1)))
      throw spb::ArgumentError("comm: rh mode needs a power-of-two rank count");
    if (nranks > 1 && mode == "p2p") e.setup_p2p();
    if (nranks > 1 && mode == "rh") {
      int d = 0;
      while ((1 << d) < nranks) ++d;
      e.setup_p2p(2 * d);
      e.comm_mode = 5;
    }
    if (nranks > 1 && mode == "push") e.setup_push();
    if (nranks > 1 && mode == "sub") e.setup_sub();
  });
  if (st != SPB_OK && ctx && (ctx->e.err.rfind("nccl", 0) == 0 || ctx->e.err.rfind("comm: ", 0) == 0))
    return SPB_E_NCCL;
  return st;
}

spb_status spb_set_gemm_chunk(int kind, int kblocks) {
  return guard(nullptr, [&] { spb::gemm_set_chunk(kind, kblocks); });
}

spb_status spb_layer_shard(long long count, int parts, long long* shard) {
  return guard(nullptr, [&] {
    if (count < 0 || parts < 1) throw spb::ArgumentError("layer_shard: bad arguments");
    *shard = spb::Engine::layer_shard(count, parts);
  });
}

spb_status spb_comm_mode(spb_ctx* ctx, int* mode) {
  return guard(ctx, [&] { *mode = ctx->e.comm ? ctx->e.comm_mode : -1; });
}

spb_status spb_bucket_plan(int k, int L, int nranks, int full_backprop, int* kind, int* root, int* rank_mask) {
  return guard(nullptr, [&] {
    if (nranks > 31) throw spb::ArgumentError("bucket_plan: at most 31 ranks");
    auto b = spb::bucket_plan(k, L, nranks, full_backprop != 0);
    for (auto& x : b) {
      const int l = x.l_hi;
      kind[l - 1] = x.kind;
      root[l - 1] = x.root;
      int mask = 0;
      for (int r : x.ranks) mask |= 1 << r;
      rank_mask[l - 1] = mask;
    }
  });
}

spb_status spb_profile_step(spb_ctx* ctx, uint64_t seed, int step, int full_backprop, int ncls, float* ms,
                            double* work, int* launches, float* step_ms) {
  return guard(ctx, [&] {
    auto& e = ctx->e;
    if (!e.X) throw spb::ConfigError("profile_step: no dataset");
    if (ncls < spb::kNumCls) throw spb::ArgumentError("profile_step: ncls too small");
    std::vector<Engine::ProfRec> recs;
    spb::Ctl c{seed, step, 0};
    SPB_CUDA(cudaMemcpyAsync(e.ctl, &c, sizeof c, cudaMemcpyHostToDevice, e.st));
    cudaEvent_t a, b;
    SPB_CUDA(cudaEventCreate(&a));
    SPB_CUDA(cudaEventCreate(&b));
    e.prof = &recs;
    e.concurrent = false;  // serialise so each launch's events time it alone
    // 5 ms head start: the whole step is enqueued before the GPU reaches it
    // (the step enqueues in ~1 ms), so no launch's events include a wait for
    // the host to submit it.
    spb::launch_spin(5'000'000, e.st);
    SPB_CUDA(cudaEventRecord(a, e.st));
    try {
      e.enqueue_step(full_backprop != 0, false, e.st);
      e.fwd_wait.clear();
    } catch (...) {
      e.fwd_wait.clear();
      e.prof = nullptr;
      e.concurrent = true;
      throw;
    }
    SPB_CUDA(cudaEventRecord(b, e.st));
    e.prof = nullptr;
    e.concurrent = true;
    SPB_CUDA(cudaStreamSynchronize(e.st));
    for (int i = 0; i < ncls; ++i) ms[i] = 0.f, work[i] = 0.0, launches[i] = 0;
    for (auto& r : recs) {
      float t = 0.f;
      SPB_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
      ms[r.cls] += t;
      work[r.cls] += r.work;
      launches[r.cls] += 1;
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    }
    SPB_CUDA(cudaEventElapsedTime(step_ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  });
}

spb_status spb_trace_steps(spb_ctx* ctx, uint64_t seed, int step0, int steps, int full_backprop, int cap,
                           long long* t_begin, long long* t_end, int* cls, int* stream, int* sub, int* n_out) {
  return guard(ctx, [&] {
    auto& e = ctx->e;
    if (!e.X) throw spb::ConfigError("trace_steps: no dataset");
    if (steps < 1 || steps > Engine::kMaxChain) throw spb::ArgumentError("trace_steps: steps must be in [1, 16]");
    if (!e.trace_dev) e.trace_dev = e.alloc<unsigned long long>(2L * Engine::kTraceCap);
    e.invalidate_graphs();  // the traced graph must not be reused untraced
    e.trace_meta.clear();
    e.tracing = true;
    cudaGraphExec_t g = nullptr;
    try {
      g = e.get_graph(full_backprop != 0, false, steps);
    } catch (...) {
      e.tracing = false;
      throw;
    }
    e.tracing = false;
    spb::Ctl c{seed, step0, 0};
    SPB_CUDA(cudaMemcpyAsync(e.ctl, &c, sizeof c, cudaMemcpyHostToDevice, e.st));
    SPB_CUDA(cudaGraphLaunch(g, e.st));  // warm-up replay (graph upload)
    SPB_CUDA(cudaGraphLaunch(g, e.st));
    const int n = static_cast<int>(e.trace_meta.size());
    std::vector<unsigned long long> ts(2L * n);
    SPB_CUDA(cudaMemcpyAsync(ts.data(), e.trace_dev, ts.size() * 8, cudaMemcpyDeviceToHost, e.st));
    SPB_CUDA(cudaStreamSynchronize(e.st));
    e.invalidate_graphs();
    *n_out = n;
    for (int i = 0; i < n && i < cap; ++i) {
      t_begin[i] = static_cast<long long>(ts[2 * i]);
      t_end[i] = static_cast<long long>(ts[2 * i + 1]);
      cls[i] = e.trace_meta[i].cls;
      stream[i] = e.trace_meta[i].stream;
      sub[i] = e.trace_meta[i].sub;
    }
  });
}

spb_status spb_time_train_steps(spb_ctx* ctx, uint64_t seed, int step0, int steps, int full_backprop, float* ms) {
  return guard(ctx, [&] {
    auto& e = ctx->e;
    if (!e.X) throw spb::ConfigError("train_steps: no dataset");
    for (int d = 0; d < steps;) {  // instantiate every graph of the run before timing
      const int c = std::max(1, std::min({e.chain_len(), Engine::kMaxChain, steps - d}));
      e.get_graph(full_backprop != 0, false, c);
      d += c;
    }
    spb::Ctl c{seed, step0, 0};
    SPB_CUDA(cudaMemcpyAsync(e.ctl, &c, sizeof c, cudaMemcpyHostToDevice, e.st));
    cudaEvent_t a, b;
    SPB_CUDA(cudaEventCreate(&a));
    SPB_CUDA(cudaEventCreate(&b));
    SPB_CUDA(cudaEventRecord(a, e.st));
    e.run_steps(full_backprop != 0, steps, nullptr);
    SPB_CUDA(cudaEventRecord(b, e.st));
    SPB_CUDA(cudaEventSynchronize(b));
    SPB_CUDA(cudaEventElapsedTime(ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  });
}

spb_status spb_profile_task(spb_ctx* ctx, int rows, int suffix, int reps, float* forward_ms, float* backward_ms,
                            double* peak_mem_gb) {
  return guard(ctx, [&] {
    auto& e = ctx->e;
    const int L = e.L;
    if (!e.X) throw spb::ConfigError("profile_task: no dataset");
    if (rows < 1) throw spb::ArgumentError("profile_task: rows must be >= 1");
    if (suffix < 0 || suffix > L) throw spb::ArgumentError("profile_task: suffix out of range");
    if (reps < 1) throw spb::ArgumentError("profile_task: reps must be >= 1");
    e.ensure_rows(rows);
    std::vector<int> iota(rows);
    for (int i = 0; i < rows; ++i) iota[i] = i % e.N;
    SPB_CUDA(cudaMemcpyAsync(e.idx_in, iota.data(), rows * sizeof(int), cudaMemcpyHostToDevice, e.st));
    e.enqueue_gather(e.X, e.ldx, rows, rows, nullptr, 0, nullptr, 0, e.idx_in, e.st);
    // One worker task (partial_backprop, spb.cpp:51-68, on one batch): the
    // forward + head, then dgrad / wgrad of the top `suffix` layers. Each
    // variant is captured into a graph and replayed `reps` times.
    auto time_pass = [&](int suf) {
      std::vector<int> row0(L + 1, rows);
      std::vector<float> alpha(L + 1, 1.0f / static_cast<float>(rows));
      for (int l = L - suf + 1; l <= L; ++l) row0[l] = 0;
      cudaGraph_t gr;
      cudaGraphExec_t ge;
      SPB_CUDA(cudaStreamBeginCapture(e.st, cudaStreamCaptureModeThreadLocal));
      try {
        e.enqueue_pass(rows, row0, alpha, e.st);
      } catch (...) {
        cudaStreamEndCapture(e.st, &gr);
        throw;
      }
      SPB_CUDA(cudaStreamEndCapture(e.st, &gr));
      SPB_CUDA(cudaGraphInstantiate(&ge, gr, 0));
      cudaGraphDestroy(gr);
      cudaEvent_t a, b;
      SPB_CUDA(cudaEventCreate(&a));
      SPB_CUDA(cudaEventCreate(&b));
      SPB_CUDA(cudaGraphLaunch(ge, e.st));  // warm-up
      SPB_CUDA(cudaEventRecord(a, e.st));
      for (int i = 0; i < reps; ++i) SPB_CUDA(cudaGraphLaunch(ge, e.st));
      SPB_CUDA(cudaEventRecord(b, e.st));
      SPB_CUDA(cudaEventSynchronize(b));
      float ms = 0.f;
      SPB_CUDA(cudaEventElapsedTime(&ms, a, b));
      cudaEventDestroy(a);
      cudaEventDestroy(b);
      cudaGraphExecDestroy(ge);
      return ms / static_cast<float>(reps);
    };
    const float f = time_pass(0);
    const float fb = suffix > 0 ? time_pass(suffix) : f;
    *forward_ms = f;
    *backward_ms = std::max(0.f, fb - f);
    // Device working set of the task: parameters (hi + lo), the gradient
    // blocks of the covered layers, the activations (split pairs) and, when
    // backpropagating, the three Delta buffers.
    double bytes = 8.0 * static_cast<double>(e.nflat);
    for (int l = L - suffix + 1; l <= L; ++l) bytes += 4.0 * static_cast<double>(e.w[l]) * (e.fan[l] + 1);
    for (int l = 0; l < L; ++l) bytes += 8.0 * rows * e.pix[l] * static_cast<double>(e.ld[l]);
    if (e.conv_model)  // im2col pairs kept for wgrad, plus the dgrad columns when backpropagating
      for (int l = 1; l < L; ++l) bytes += 8.0 * rows * e.pix[l] * static_cast<double>(e.ldf[l]);
    bytes += 4.0 * rows * (static_cast<double>(e.ldx) + 2.0 * e.nout + 2.0);
    if (suffix > 0) {
      double dmax = e.ldd, cmax = 0;
      for (int l = 1; l < L; ++l)
        dmax = std::max(dmax, e.pix[l] * static_cast<double>(e.ld[l])), cmax = std::max(cmax, e.pix[l] * static_cast<double>(e.ldf[l]));
      bytes += 3.0 * 8.0 * rows * dmax + (e.conv_model ? 4.0 * rows * cmax : 0.0);
    }
    *peak_mem_gb = bytes / 1e9;
  });
}

spb_status spb_empirical_variance(spb_ctx* ctx, int k, int B, int trials, uint64_t seed, double* out) {
  return guard(ctx, [&] {
    auto& e = ctx->e;
    if (!e.X) throw spb::ConfigError("empirical_variance: no dataset");
    if (k < 1) throw spb::ArgumentError("SpbConfig: k must be >= 1");  // spb.cpp:11-14
    if (B < 1 || B % k != 0) throw spb::ArgumentError("SpbConfig: B must be positive and divisible by k");
    if (trials < 1) throw spb::ArgumentError("empirical_variance: trials must be >= 1");
    if (k != e.k || B / k != e.bw)
      throw spb::ArgumentError("empirical_variance: cfg.k and cfg.B / cfg.k must match the context");
    if (e.comm) throw spb::ConfigError("empirical_variance: single-GPU contexts only");
    const int L = e.L, N = e.N, rows = k * e.bw;
    e.ensure_rows(std::max(N, rows));
    float* G = Engine::alloc<float>(e.nflat);
    const long nd = static_cast<long>(2 + k) * trials;
    double* dist = Engine::alloc<double>(nd);
    int* samp = Engine::alloc<int>(static_cast<long>(k) * trials);
    cudaStream_t st = e.st;
    try {
      // grad f(x): the mean gradient over the whole dataset (full_gradient,
      // spb.cpp:267-271), one pass over all N rows.
      std::vector<int> iota(N);
      std::iota(iota.begin(), iota.end(), 0);
      SPB_CUDA(cudaMemcpyAsync(e.idx_in, iota.data(), N * sizeof(int), cudaMemcpyHostToDevice, st));
      e.enqueue_gather(e.X, e.ldx, N, N, nullptr, 0, nullptr, 0, e.idx_in, st);
      {
        std::vector<int> row0(L + 1, 0);
        std::vector<float> alpha(L + 1, 1.0f / static_cast<float>(N));
        e.enqueue_pass(N, row0, alpha, st);
      }
      SPB_CUDA(cudaMemcpyAsync(G, e.grad, e.nflat * sizeof(float), cudaMemcpyDeviceToDevice, st));
      // Trials (spb.cpp:219-229): trial r's worker j draws its batch from
      // Rng(seed).split(kWorkerDrawTag).split(r).split(j) -- the device
      // gather's Rng(seed').split(step).split(j) with seed' = the first split
      // and step = r. The SPB estimate and the full-backprop baseline use the
      // same batches.
      const uint64_t wseed = spb::Rng::mix(seed, 0x5D17);  // kWorkerDrawTag, spb.hpp:86
      e.set_workers_all();
      std::vector<int> r0s, r0f;
      std::vector<float> as, af;
      e.step_plan(false, r0s, as);
      e.step_plan(true, r0f, af);
      for (int r = 1; r <= trials; ++r) {
        e.enqueue_gather(e.X, e.ldx, rows, e.bw, nullptr, wseed, nullptr, r, nullptr, st);
        e.enqueue_pass(rows, r0s, as, st);
        spb::launch_sqdist(G, e.grad, e.nflat, dist + (r - 1), st);
        e.enqueue_pass(rows, r0f, af, st);
        spb::launch_sqdist(G, e.grad, e.nflat, dist + trials + (r - 1), st);
      }
      // Per-chunk p_i (spb.cpp:240-262): single-sample gradients drawn from
      // Rng(seed).split(kChunkDrawTag).split(m), restricted to chunk m.
      auto spans = spb::chunk_layout(k, L);
      std::vector<int> hs(static_cast<size_t>(k) * trials);
      for (int m = 1; m <= k; ++m) {
        spb::Rng cs = spb::Rng(seed).split(0xC410).split(static_cast<uint64_t>(m));  // kChunkDrawTag, spb.hpp:87
        for (int t = 0; t < trials; ++t) hs[static_cast<size_t>(m - 1) * trials + t] = static_cast<int>(cs.next_below(N));
      }
      SPB_CUDA(cudaMemcpyAsync(samp, hs.data(), hs.size() * sizeof(int), cudaMemcpyHostToDevice, st));
      for (int m = 1; m <= k; ++m) {
        const int first = spans[m - 1].first, last = spans[m - 1].second;
        if (first > last) continue;  // empty chunk: d = 0 every trial
        std::vector<int> row0(L + 1, 1);
        for (int l = first; l <= L; ++l) row0[l] = 0;
        std::vector<float> alpha(L + 1, 1.0f);
        const long a = e.w_off[first], b = e.b_off[last] + spb::round_up(e.w[last], 32);
        for (int t = 0; t < trials; ++t) {
          e.enqueue_gather(e.X, e.ldx, 1, 1, nullptr, 0, nullptr, 0, samp + static_cast<long>(m - 1) * trials + t, st);
          e.enqueue_pass(1, row0, alpha, st);
          spb::launch_sqdist(G + a, e.grad + a, b - a, dist + static_cast<long>(2 + m - 1) * trials + t, st);
        }
      }
      std::vector<double> h(nd);
      SPB_CUDA(cudaMemcpyAsync(h.data(), dist, nd * sizeof(double), cudaMemcpyDeviceToHost, st));
      SPB_CUDA(cudaStreamSynchronize(st));
      auto finish = [&](const double* d, double& mean, double& se) {  // spb.cpp:230-234
        double sum = 0.0, sumsq = 0.0;
        for (int t = 0; t < trials; ++t) sum += d[t], sumsq += d[t] * d[t];
        mean = sum / trials;
        const double var = std::max(0.0, sumsq / trials - mean * mean);
        se = std::sqrt(var / trials);
      };
      finish(h.data(), out[0], out[1]);
      finish(h.data() + trials, out[2], out[3]);
      for (int m = 0; m < k; ++m) finish(h.data() + static_cast<long>(2 + m) * trials, out[4 + m], out[4 + k + m]);
    } catch (...) {
      cudaStreamSynchronize(st);
      cudaFree(G), cudaFree(dist), cudaFree(samp);
      throw;
    }
    cudaFree(G), cudaFree(dist), cudaFree(samp);
  });
}

spb_status spb_last_batch(spb_ctx* ctx, int* out, int rows) {
  return guard(ctx, [&] {
    auto& e = ctx->e;
    if (rows > e.cap_rows) throw spb::ArgumentError("last_batch: too many rows");
    SPB_CUDA(cudaMemcpyAsync(out, e.idx, rows * sizeof(int), cudaMemcpyDeviceToHost, e.st));
    SPB_CUDA(cudaStreamSynchronize(e.st));
  });
}

spb_status spb_launches_per_step(spb_ctx* ctx, int* out) {
  return guard(ctx, [&] { *out = ctx->e.last_launches; });
}

}  // extern "C"

