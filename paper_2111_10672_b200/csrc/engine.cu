// Engine: allocation, the per-step launch program and its CUDA graphs (see
// engine.hpp for the layout; the multi-GPU exchange is in exchange.cu).
#include <dlfcn.h>

#include "engine.hpp"

namespace spb {

const NcclApi& nccl() {
  static NcclApi api{};
  static std::string fail;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = nullptr;
    if (const char* p = std::getenv("SPB_NCCL_LIB")) h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      fail = std::string("comm: cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    auto sym = [&](const char* n) {
      void* f = dlsym(h, n);
      if (!f && fail.empty()) fail = std::string("comm: missing NCCL symbol ") + n;
      return f;
    };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
    api.Broadcast = reinterpret_cast<decltype(api.Broadcast)>(sym("ncclBroadcast"));
    api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
    api.ReduceScatter = reinterpret_cast<decltype(api.ReduceScatter)>(sym("ncclReduceScatter"));
    api.CommSplit = reinterpret_cast<decltype(api.CommSplit)>(sym("ncclCommSplit"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
    api.CommFinalize = reinterpret_cast<decltype(api.CommFinalize)>(sym("ncclCommFinalize"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.CommGetAsyncError = reinterpret_cast<decltype(api.CommGetAsyncError)>(sym("ncclCommGetAsyncError"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
  });
  if (!fail.empty()) throw std::runtime_error(fail);
  return api;
}

void Engine::release() {
  // Order matters: graphs that captured NCCL collectives hold references to
  // the communicator, so they go first; then the communicator is finalized
  // (flushes outstanding work) before it is destroyed.
  if (st) cudaStreamSynchronize(st);
  if (cst) cudaStreamSynchronize(cst);
  invalidate_graphs();
  if (comm_mode == 2 || comm_mode == 4 || comm_mode == 5) {
    // Peers may still read this rank's memory until they pass this point.
    if (s3) cudaStreamSynchronize(s3);
    if (s4) cudaStreamSynchronize(s4);
    for (auto q : gpull)
      if (q) cudaStreamSynchronize(q);
    for (auto q : wpull)
      if (q) cudaStreamSynchronize(q);
    try {
      host_barrier();
    } catch (...) {
    }
    for (int p = 0; p < nranks; ++p) {
      if (p == rank) continue;
      if (peer_grad[p]) cudaIpcCloseMemHandle(peer_grad[p]);
      if (peer_w32[p]) cudaIpcCloseMemHandle(peer_w32[p]);
      if (peer_flags.p[p]) cudaIpcCloseMemHandle(peer_flags.p[p]);
      if (p < static_cast<int>(peer_pstage.size()) && peer_pstage[p]) cudaIpcCloseMemHandle(peer_pstage[p]);
    }
    peer_grad.clear(), peer_w32.clear(), peer_pstage.clear();
    for (auto q : gpull)
      if (q) cudaStreamDestroy(q);
    for (auto q : wpull)
      if (q) cudaStreamDestroy(q);
    gpull.clear(), wpull.clear();
    comm_mode = 0;
  }
  for (auto& kv : subcomms)
    if (kv.second) {
      const NcclApi& api = nccl();
      api.CommFinalize(kv.second);
      ncclResult_t state = ncclInProgress;
      while (api.CommGetAsyncError(kv.second, &state) == ncclSuccess && state == ncclInProgress) {
      }
      api.CommDestroy(kv.second);
    }
  subcomms.clear();
  if (comm) {
    const NcclApi& api = nccl();
    api.CommFinalize(comm);
    ncclResult_t state = ncclInProgress;
    while (api.CommGetAsyncError(comm, &state) == ncclSuccess && state == ncclInProgress) {
    }
    api.CommDestroy(comm);
    comm = nullptr;
  }
  if (cst) cudaStreamDestroy(cst), cst = nullptr;
  if (s4) cudaStreamDestroy(s4), s4 = nullptr;
  if (s2) cudaStreamDestroy(s2), s2 = nullptr;
  if (s3) cudaStreamDestroy(s3), s3 = nullptr;
  for (auto ev : evs) cudaEventDestroy(ev);
  evs.clear();
  auto f = [](void* p) {
    if (p) cudaFree(p);
  };
  f(splitk_ws);
  f(splitk_ws2), f(splitk_ws3), f(colsum_ws), f(colsum_cnt);
  f(p64);
  f(p_hi), f(p_lo), f(grad), f(mom), f(X), f(Y), f(delta), f(delta_lo), f(row_loss), f(ybatch), f(xin), f(idx),
      f(idx_in), f(loss_dev), f(tmp), f(ctl), f(workers_dev), f(epoch_dev), f(bar_dev), f(w32), f(flags),
      f(stage), f(pstage), f(trace_dev);
  for (int i = 0; i < 2; ++i) f(hx[i]), f(hy[i]);
  if (hst) cudaStreamDestroy(hst), hst = nullptr;
  if (loss_pin) cudaFreeHost(loss_pin), loss_pin = nullptr;
  for (auto p : Hh) f(p);
  for (auto p : Hl) f(p);
  for (auto p : Ch) f(p);
  for (auto p : Cl) f(p);
  f(Ph), f(Pl), f(Gh), f(Gl), f(dcol), f(iota_dev), f(Fh), f(Fl);
  for (int i = 0; i < kDbuf; ++i) f(Dh[i]), f(Dl[i]);
  if (st) cudaStreamDestroy(st);
  st = nullptr;
}

void Engine::init(const int* widths, int n_widths, int k_, int bw_, int device) {
  if (n_widths < 2) throw ArgumentError("mlp: need at least one layer");
  for (int i = 0; i < n_widths; ++i)
    if (widths[i] < 1) throw ArgumentError("mlp: widths must be >= 1");
  if (widths[n_widths - 1] > 16) throw ArgumentError("mlp: output width must be <= 16");
  if (k_ < 1 || bw_ < 1) throw ArgumentError("SpbConfig: k and per-worker batch must be >= 1");
  w.assign(widths, widths + n_widths);
  L = n_widths - 1;
  nout = w[L];
  k = k_;
  bw = bw_;
  if (device < 0) SPB_CUDA(cudaGetDevice(&device));  // -1: the calling thread's current device
  dev = device;
  SPB_CUDA(cudaSetDevice(dev));
  gemm_prepare_device();
  SPB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  SPB_CUDA(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  SPB_CUDA(cudaStreamCreateWithFlags(&s3, cudaStreamNonBlocking));
  ld.resize(L + 1);
  long ldmax = 0;
  for (int l = 0; l <= L; ++l) ld[l] = round_up(w[l], 4), ldmax = std::max(ldmax, ld[l]);
  ldd = ldmax;
  ldx = ld[0];
  pix.assign(L + 1, 1);
  fan.assign(L + 1, 0);
  ldf.assign(L + 1, 0);
  for (int l = 1; l <= L; ++l) fan[l] = w[l - 1], ldf[l] = ld[l - 1];
  allocate_params();
  ensure_rows(k * bw);
}

void Engine::init_conv(const int* geom, int nconv, int nout_, int k_, int bw_, int device) {
  if (nconv < 1) throw ArgumentError("convnet: need at least one convolution");
  if (geom[0] < 1 || geom[1] < 1 || geom[2] < 1) throw ArgumentError("convnet: bad input geometry");
  if (nout_ < 1 || nout_ > 16) throw ArgumentError("convnet: output width must be in [1, 16]");
  if (k_ < 1 || bw_ < 1) throw ArgumentError("SpbConfig: k and per-worker batch must be >= 1");
  conv_model = true;
  L = nconv + 1;
  nout = nout_;
  k = k_;
  bw = bw_;
  if (device < 0) SPB_CUDA(cudaGetDevice(&device));  // -1: the calling thread's current device
  dev = device;
  SPB_CUDA(cudaSetDevice(dev));
  gemm_prepare_device();
  SPB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  SPB_CUDA(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  SPB_CUDA(cudaStreamCreateWithFlags(&s3, cudaStreamNonBlocking));
  w.assign(L + 1, 0);
  pix.assign(L + 1, 1);
  cg.assign(L, ConvGeom{});
  int h = geom[0], wd_ = geom[1];
  w[0] = geom[2];
  pix[0] = static_cast<long>(h) * wd_;
  for (int l = 1; l <= nconv; ++l) {
    const int c = geom[3 + 2 * (l - 1)], stride = geom[4 + 2 * (l - 1)];
    if (c < 1 || (stride != 1 && stride != 2)) throw ArgumentError("convnet: channels >= 1, stride 1 or 2");
    ConvGeom g{h, wd_, w[l - 1], (h - 1) / stride + 1, (wd_ - 1) / stride + 1, c, stride};
    cg[l] = g;
    w[l] = c;
    h = g.out_h, wd_ = g.out_w;
    pix[l] = static_cast<long>(h) * wd_;
  }
  w[L] = nout;
  ld.resize(L + 1);
  for (int l = 0; l <= L; ++l) ld[l] = round_up(w[l], 4);
  ldd = 0;
  fan.assign(L + 1, 0);
  ldf.assign(L + 1, 0);
  for (int l = 1; l <= L; ++l) {
    fan[l] = l < L ? 9 * w[l - 1] : w[L - 1];
    ldf[l] = round_up(fan[l], 4);
  }
  ldx = pix[0] * w[0];
  allocate_params();
  ensure_rows(k * bw);
}

void Engine::allocate_params() {
  w_off.assign(L + 1, 0);
  b_off.assign(L + 1, 0);
  long cur = 0, maxblk = 0;
  for (int l = 1; l <= L; ++l) {
    w_off[l] = cur;
    cur += round_up(w[l] * ldf[l], 32);
    b_off[l] = cur;
    cur += round_up(w[l], 32);
    maxblk = std::max(maxblk, w[l] * ldf[l] + w[l]);
  }
  nflat = cur;
  p_hi = alloc<float>(nflat);
  p_lo = alloc<float>(nflat);
  grad = alloc<float>(nflat + kGradSlack);  // sub mode's reduce-scatter reads up to 4 * ranks floats past a layer
  tmp_n = maxblk;
  tmp = alloc<float>(tmp_n);
  splitk_ws = alloc<float>(kSplitkWsFloats);
  splitk_ws2 = alloc<float>(kSplitkWs2Floats);
  if (conv_model) splitk_ws3 = alloc<float>(kConvWsFloats);  // the conv wgrads' split-K (gradient stream)
  colsum_ws = alloc<float>(kColsumWsFloats);
  colsum_cnt = alloc<int>(kColsumCounters);
  ctl = alloc<Ctl>(1);
  loss_dev = alloc<float>(kMaxChain);
  workers_dev = alloc<int>(k);
  set_workers_all();
}

void Engine::ensure_rows(int rows) {
  if (rows <= cap_rows) return;
  SPB_CUDA(cudaStreamSynchronize(st));
  invalidate_graphs();
  if (conv_model) return ensure_samples_conv(rows);
  for (auto p : Hh) cudaFree(p);
  for (auto p : Hl) cudaFree(p);
  Hh.assign(L, nullptr);
  Hl.assign(L, nullptr);
  for (int i = 0; i < kDbuf; ++i) {
    if (Dh[i]) cudaFree(Dh[i]), cudaFree(Dl[i]);
  }
  for (void* p : {(void*)delta, (void*)delta_lo, (void*)row_loss, (void*)ybatch, (void*)xin, (void*)idx, (void*)idx_in})
    if (p) cudaFree(p);
  cap_rows = rows;
  for (int l = 0; l < L; ++l) {
    Hh[l] = alloc<float>(rows * ld[l]);
    Hl[l] = alloc<float>(rows * ld[l]);
  }
  for (int i = 0; i < kDbuf; ++i) {
    Dh[i] = alloc<float>(rows * ldd);
    Dl[i] = alloc<float>(rows * ldd);
  }
  ldq = round_up(nout, 4);
  delta = alloc<float>(static_cast<long>(rows) * ldq);
  delta_lo = alloc<float>(static_cast<long>(rows) * ldq);
  row_loss = alloc<float>(rows);
  ybatch = alloc<float>(static_cast<long>(rows) * nout);
  xin = alloc<float>(static_cast<long>(rows) * w[0]);
  idx = alloc<int>(rows);
  idx_in = alloc<int>(rows);
}

void Engine::ensure_samples_conv(int samples) {
  auto f = [](void* p) {
    if (p) cudaFree(p);
  };
  for (auto p : Hh) f(p);
  for (auto p : Hl) f(p);
  for (auto p : Ch) f(p);
  for (auto p : Cl) f(p);
  for (int i = 0; i < kDbuf; ++i) f(Dh[i]), f(Dl[i]);
  for (void* p : {(void*)delta, (void*)delta_lo, (void*)row_loss, (void*)ybatch, (void*)xin, (void*)idx,
                  (void*)idx_in, (void*)Ph, (void*)Pl, (void*)Gh, (void*)Gl, (void*)dcol, (void*)iota_dev})
    f(p);
  cap_rows = samples;
  const long S = samples;
  Hh.assign(L, nullptr);
  Hl.assign(L, nullptr);
  Ch.assign(L, nullptr);
  Cl.assign(L, nullptr);
  long dmax = 1, cmax = 1;
  for (int l = 0; l < L; ++l) {
    Hh[l] = alloc<float>(S * pix[l] * ld[l]);
    Hl[l] = alloc<float>(S * pix[l] * ld[l]);
    if (l >= 1) {
      if (!conv_tma(l)) {  // implicit-GEMM layers read H_{l-1} through TMA im2col maps instead
        Ch[l] = alloc<float>(S * pix[l] * ldf[l]);
        Cl[l] = alloc<float>(S * pix[l] * ldf[l]);
      }
      dmax = std::max(dmax, S * pix[l] * ld[l]);
      cmax = std::max(cmax, S * pix[l] * ldf[l]);
    }
  }
  for (int i = 0; i < kDbuf; ++i) Dh[i] = alloc<float>(dmax), Dl[i] = alloc<float>(dmax);
  dcol = alloc<float>(cmax);
  long fmax = 1;
  for (int l = 2; l < L; ++l) fmax = std::max(fmax, static_cast<long>(w[l - 1]) * round_up(9L * w[l], 4));
  if (!Fh) Fh = alloc<float>(fmax), Fl = alloc<float>(fmax);
  Ph = alloc<float>(S * ld[L - 1]);
  Pl = alloc<float>(S * ld[L - 1]);
  Gh = alloc<float>(S * ld[L - 1]);
  Gl = alloc<float>(S * ld[L - 1]);
  ldq = round_up(nout, 4);
  delta = alloc<float>(S * ldq);
  delta_lo = alloc<float>(S * ldq);
  row_loss = alloc<float>(S);
  ybatch = alloc<float>(S * nout);
  xin = alloc<float>(S * ldx);
  idx = alloc<int>(S);
  idx_in = alloc<int>(S);
  iota_dev = alloc<int>(S);
  std::vector<int> io(samples);
  std::iota(io.begin(), io.end(), 0);
  SPB_CUDA(cudaMemcpy(iota_dev, io.data(), S * sizeof(int), cudaMemcpyHostToDevice));
}

int Engine::enqueue_pass_conv(int samples, const std::vector<int>& row0, const std::vector<float>& alpha,
                              cudaStream_t s, const std::function<int(int, cudaStream_t)>& on_grad, int* step_dev,
                              const std::function<void(int, cudaStream_t)>& on_layer) {
  int n = 0;
  const int Lc = L - 1;
  for (int l = 1; l <= Lc; ++l) {
    fwd_gate(l, s);
    const int M = static_cast<int>(samples * pix[l]);
    const bool tma = conv_tma(l);
    if (conv_direct(l)) {
      pbeg(s);
      launch_conv_direct_fwd(Hh[l - 1], Hl[l - 1], ld[l - 1], cg[l], M, p_hi + w_off[l], p_lo + w_off[l], ldf[l],
                             p_hi + b_off[l], p_lo + b_off[l], Hh[l], Hl[l], ld[l], s);
      pend(kClsFwd, 2.0 * M * w[l] * fan[l], s);
      ++n;
      continue;
    }
    if (!tma) {
      pbeg(s);
      launch_im2col(Hh[l - 1], Hl[l - 1], ld[l - 1], cg[l], 0, M, Ch[l], Cl[l], ldf[l], s);
      pend(kClsGather, 0, s);
      ++n;
    }
    Operand A{Ch[l], Cl[l], ldf[l], M, fan[l], false};
    Operand B{p_hi + w_off[l], p_lo + w_off[l], ldf[l], w[l], fan[l], false};
    GemmEpilogue ep{};
    ep.out_hi = Hh[l];
    ep.out_lo = Hl[l];
    ep.ld_out = ld[l];
    ep.bias_hi = p_hi + b_off[l];
    ep.bias_lo = p_lo + b_off[l];
    ep.M = M;
    ep.N = w[l];
    ep.splitk_ws = splitk_ws;
    ep.splitk_ws_floats = kSplitkWsFloats;
    pbeg(s);
    if (tma) {
      ConvSrc src{Hh[l - 1], Hl[l - 1], ld[l - 1], samples, cg[l]};
      n += gemm_conv_fwd(src, B, ep, s);
    } else {
      n += gemm_tf32x3(A, B, kEpiFwdTanh, ep, s);
    }
    pend(kClsFwd, 2.0 * M * w[l] * fan[l], s);
  }
  const bool has_next = Lc >= 1 && row0[Lc] < samples;
  fwd_gate(L, s);
  pbeg(s);
  launch_avgpool(Hh[Lc], Hl[Lc], ld[Lc], samples, static_cast<int>(pix[Lc]), w[Lc], Ph, Pl, ld[Lc], s);
  launch_head(Ph, Pl, ld[Lc], samples, w[Lc], nout, p_hi + w_off[L], p_lo + w_off[L], ldf[L], p_hi + b_off[L],
              p_lo + b_off[L], ybatch, delta, delta_lo, ldq, row_loss, has_next ? Gh : nullptr,
              has_next ? Gl : nullptr, ld[Lc], has_next ? row0[Lc] : samples, false, s, /*dn_act=*/false);
  launch_sum_loss(row_loss, samples, 1.0f / static_cast<float>(samples), loss_dev + chain_sub, step_dev, s);
  pend(kClsHead, 0, s);
  n += 3;
  if (row0[L] < samples) {  // head wgrad + bias: alpha delta^T [P | 1] over the contributor samples
    pbeg(s);
    n += enqueue_head_wgrad(Ph, Pl, ld[Lc], row0[L], samples, w[Lc], alpha[L], false, splitk_ws, kSplitkWsFloats, s);
    pend(kClsWgrad, 2.0 * (samples - row0[L]) * nout * (w[Lc] + 1), s);
  }
  if (on_grad) n += on_grad(L, s);
  if (on_layer) on_layer(L, s);
  if (has_next) {
    launch_unpool_tanh(Gh, Gl, ld[Lc], samples, row0[Lc], static_cast<int>(pix[Lc]), w[Lc], Hh[Lc], Hl[Lc], ld[Lc],
                       Dh[Lc % kDbuf], Dl[Lc % kDbuf], ld[Lc], s);
    ++n;
  }
  // Two streams, as in the MLP pass: the Delta chain (dgrads) on s, the
  // wgrads (+ the RGB layer's column gather) on s2 with their own split-K
  // workspace; Delta is triple-buffered, so dgrad_l waits for wgrad_{l+2}.
  // (SPB_CONV_TWO_STREAM=0: one stream, for A/B.)
  static const bool one = [] {
    const char* v = std::getenv("SPB_CONV_TWO_STREAM");
    return v && std::string(v) == "0";
  }();
  const bool two = concurrent && !one;
  cudaStream_t sw = two ? s2 : s;
  float* wws = splitk_ws3;  // (used by the wgrads only, on whichever stream they run)
  // SM partition of the two streams: off by default for the ConvNet (A/B knob).
  const int dsms = part_sms(dgrad_sms, 0), wsms = part_sms(wgrad_sms, 0);
  auto ev_delta = [&](int q) { return ev(kEvLayer + 2 * q); };     // Delta_q ready (on s)
  auto ev_wgrad = [&](int q) { return ev(kEvLayer + 2 * q + 1); }; // wgrad_q done (on s2)
  if (two) {  // fork the gradient stream (also when this rank has no rows below the head)
    SPB_CUDA(cudaEventRecord(ev_delta(Lc), s));
    SPB_CUDA(cudaStreamWaitEvent(s2, ev_delta(Lc), 0));
  }
  int l = Lc;
  for (; l >= 1; --l) {
    if (row0[l] >= samples) break;
    const int b = l % kDbuf, bn = (l - 1) % kDbuf;
    const long r0 = row0[l] * pix[l], cnt = (samples - row0[l]) * pix[l];
    if (two && l > 1 && row0[l - 1] < samples && l + 2 <= Lc) SPB_CUDA(cudaStreamWaitEvent(s, ev_wgrad(l + 2), 0));
    if (l > 1 && row0[l - 1] < samples && conv_tma_dgrad(l)) {
      // Delta_{l-1} = conv(Delta_l, flipped W_l) * (1 - H_{l-1}^2), rows of the continuing samples.
      const long q0 = row0[l - 1] * pix[l - 1], qn = (samples - row0[l - 1]) * pix[l - 1];
      const long ldfl = round_up(9L * w[l], 4);
      pbeg(s);
      launch_conv_flip(p_hi + w_off[l], p_lo + w_off[l], ldf[l], w[l], w[l - 1], Fh, Fl, ldfl, s);
      ConvGeom gd{cg[l].out_h, cg[l].out_w, w[l], cg[l].in_h, cg[l].in_w, w[l - 1], 1};
      ConvSrc src{Dh[b], Dl[b], ld[l], samples, gd};
      Operand B{Fh, Fl, ldfl, w[l - 1], 9 * w[l], false};
      GemmEpilogue ep{};
      ep.out_hi = Dh[bn] + q0 * ld[l - 1];
      ep.out_lo = Dl[bn] + q0 * ld[l - 1];
      ep.ld_out = ld[l - 1];
      ep.h_hi = Hh[l - 1] + q0 * ld[l - 1];
      ep.h_lo = Hl[l - 1] + q0 * ld[l - 1];
      ep.ld_h = ld[l - 1];
      ep.M = static_cast<int>(qn);
      ep.N = w[l - 1];
      SmReserve part(two && dsms > 0 ? std::max(reserved_sms, sm_total() - dsms) : reserved_sms);
      n += 1 + gemm_conv_dgrad(src, q0, static_cast<int>(qn), B, ep, s);
      pend(kClsDgrad, 2.0 * qn * w[l] * fan[l], s);
    } else if (l > 1 && row0[l - 1] < samples) {  // dgrad into columns, then col2im * (1 - H^2)
      const long q0 = row0[l - 1] * pix[l], qn = (samples - row0[l - 1]) * pix[l];
      Operand A{Dh[b] + q0 * ld[l], Dl[b] + q0 * ld[l], ld[l], static_cast<int>(qn), w[l], false};
      Operand B{p_hi + w_off[l], p_lo + w_off[l], ldf[l], fan[l], w[l], true};
      GemmEpilogue ep{};
      ep.out_hi = dcol + q0 * ldf[l];
      ep.ld_out = ldf[l];
      ep.alpha = 1.f;
      ep.M = static_cast<int>(qn);
      ep.N = fan[l];
      ep.splitk_ws = splitk_ws;
      ep.splitk_ws_floats = kSplitkWsFloats;
      pbeg(s);
      {
        SmReserve part(two && dsms > 0 ? std::max(reserved_sms, sm_total() - dsms) : reserved_sms);
        n += gemm_tf32x3(A, B, kEpiStoreScaled, ep, s);
      }
      pend(kClsDgrad, 2.0 * qn * w[l] * fan[l], s);
      pbeg(s);
      launch_col2im_tanh(dcol, ldf[l], cg[l], static_cast<int>(row0[l - 1] * pix[l - 1]),
                         static_cast<int>((samples - row0[l - 1]) * pix[l - 1]), Hh[l - 1], Hl[l - 1], ld[l - 1],
                         Dh[bn], Dl[bn], ld[l - 1], s);
      pend(kClsDgrad, 0, s);  // the gather half of the stride-2 dgrad
      ++n;
    }
    if (two) {  // Delta_{l-1} ready / dgrad_l (last reader of W_l) done; wgrad_l needs Delta_l
      SPB_CUDA(cudaEventRecord(ev_delta(l - 1), s));
      SPB_CUDA(cudaStreamWaitEvent(s2, ev_delta(l), 0));
    }
    if (conv_direct(l)) {  // the direct forward left no columns: those of the contributor samples
      pbeg(sw);
      launch_im2col(Hh[l - 1], Hl[l - 1], ld[l - 1], cg[l], static_cast<int>(r0), static_cast<int>(cnt), Ch[l], Cl[l],
                    ldf[l], sw);
      pend(kClsGather, 0, sw);
      ++n;
    }
    {  // wgrad + bias: [dW_l | db_l] = alpha_l * Delta_l[r0:]^T [col_l[r0:] | 1]
      Operand A{Dh[b] + r0 * ld[l], Dl[b] + r0 * ld[l], ld[l], w[l], static_cast<int>(cnt), true};
      const bool tma = conv_tma(l);
      const int bc = static_cast<int>(round_up(fan[l], 32));  // the fused bias column (ones box)
      Operand B{tma ? nullptr : Ch[l] + r0 * ldf[l], tma ? nullptr : Cl[l] + r0 * ldf[l], ldf[l], bc + 1,
                static_cast<int>(cnt), true, fan[l]};
      GemmEpilogue ep{};
      ep.out_hi = grad + w_off[l];
      ep.ld_out = ldf[l];
      ep.alpha = alpha[l];
      ep.M = w[l];
      ep.N = fan[l];
      ep.bias_col_p1 = ep.ones_col_p1 = bc + 1;
      ep.gb_hi = grad + b_off[l];
      ep.colsum_ws = colsum_ws, ep.colsum_cnt = colsum_cnt;
      ep.splitk_ws = wws;  // few output tiles, K = pixel rows: split K
      ep.splitk_ws_floats = kConvWsFloats;
      pbeg(sw);
      SmReserve part(two && wsms > 0 ? std::max(reserved_sms, sm_total() - wsms) : reserved_sms);
      if (tma) {
        ConvSrc src{Hh[l - 1], Hl[l - 1], ld[l - 1], samples, cg[l]};
        n += gemm_conv_wgrad(A, src, r0, ep, sw);
      } else {
        n += gemm_tf32x3(A, B, kEpiStoreScaled, ep, sw);
      }
      pend(kClsWgrad, 2.0 * cnt * w[l] * fan[l], sw);
    }
    if (two) SPB_CUDA(cudaEventRecord(ev_wgrad(l), s2));
    if (on_grad) n += on_grad(l, sw);
    if (on_layer) on_layer(l, sw);  // grad of layer l final on sw; dgrad_l (last W_l reader) done on s
  }
  if (two) {  // join the gradient stream
    SPB_CUDA(cudaEventRecord(ev(kEvJoin), s2));
    SPB_CUDA(cudaStreamWaitEvent(s, ev(kEvJoin), 0));
  }
  for (; l >= 1 && on_grad; --l) {
    n += on_grad(l, s);
    if (on_layer) on_layer(l, s);
  }
  return n;
}

int Engine::enqueue_pass(int rows, const std::vector<int>& row0, const std::vector<float>& alpha, cudaStream_t s,
                         const std::function<int(int, cudaStream_t)>& on_grad, bool fused, int* step_dev,
                         const std::function<void(int, cudaStream_t)>& on_layer) {
  SmReserve reserve(reserved_sms);  // this context's SMs-left-free for its collectives
  if (conv_model) return enqueue_pass_conv(rows, row0, alpha, s, on_grad, step_dev, on_layer);
  int n = 0;
  // Forward, hidden layers (mlp_forward model.cpp:108-128 batched).
  for (int l = 1; l < L; ++l) {
    fwd_gate(l, s);
    Operand A{Hh[l - 1], Hl[l - 1], ld[l - 1], rows, w[l - 1], false};
    Operand B{p_hi + w_off[l], p_lo + w_off[l], ld[l - 1], w[l], w[l - 1], false};
    GemmEpilogue ep{};
    ep.out_hi = Hh[l];
    ep.out_lo = Hl[l];
    ep.ld_out = ld[l];
    ep.bias_hi = p_hi + b_off[l];
    ep.bias_lo = p_lo + b_off[l];
    ep.M = rows;
    ep.N = w[l];
    ep.splitk_ws = splitk_ws;
    ep.splitk_ws_floats = kSplitkWsFloats;
    pbeg(s);
    n += gemm_tf32x3(A, B, kEpiFwdTanh, ep, s);
    pend(kClsFwd, 2.0 * rows * w[l] * w[l - 1], s);
  }
  auto lf = [&](int l) { return fused && static_cast<int>(fuse_layer.size()) > l && fuse_layer[l]; };
  // Output head: out, delta_L = out - y (model.cpp:156), Delta_{L-1}.
  const bool has_next = L > 1 && row0[L - 1] < rows;
  fwd_gate(L, s);
  pbeg(s);
  launch_head(Hh[L - 1], Hl[L - 1], ld[L - 1], rows, w[L - 1], nout, p_hi + w_off[L], p_lo + w_off[L], ld[L - 1],
              p_hi + b_off[L], p_lo + b_off[L], ybatch, delta, delta_lo, ldq, row_loss,
              has_next ? Dh[(L - 1) % kDbuf] : nullptr,
              has_next ? Dl[(L - 1) % kDbuf] : nullptr, ldd, has_next ? row0[L - 1] : rows, false, s);
  launch_sum_loss(row_loss, rows, 1.0f / static_cast<float>(rows), loss_dev + chain_sub, step_dev, s);
  pend(kClsHead, 0, s);
  n += 2;
  // Two streams from here on: the Delta chain (head, dgrads) on s, the
  // gradient reductions (head gradients, wgrads, bias sums) on s2, so
  // dgrad_{L-1} starts right after the head kernel.
  const bool two = concurrent;
  if (two) {
    SPB_CUDA(cudaEventRecord(ev(kEvFork), s));
    SPB_CUDA(cudaStreamWaitEvent(s2, ev(kEvFork), 0));
  }
  cudaStream_t sw = two ? s2 : s;
  const int dsms = part_sms(dgrad_sms, 68), wsms = part_sms(wgrad_sms, 72);
  // Head gradients over the contributor rows of layer L: one wgrad GEMM,
  // alpha_L delta_L^T [H_{L-1} | 1] (weights and bias; never fused with the
  // optimizer -- enqueue_step keeps layer L unfused).
  if (row0[L] < rows) {
    pbeg(sw);
    n += enqueue_head_wgrad(Hh[L - 1], Hl[L - 1], ld[L - 1], row0[L], rows, w[L - 1], alpha[L], route_push,
                            two ? splitk_ws2 : splitk_ws, two ? kSplitkWs2Floats : kSplitkWsFloats, sw);
    pend(kClsWgrad, 2.0 * (rows - row0[L]) * nout * (w[L - 1] + 1), sw);
  }
  if (on_grad) n += on_grad(L, sw);
  if (on_layer) on_layer(L, sw);  // W_L: read by the head only
  // Truncated backward (model.cpp:161-185): layer l runs over its
  // contributor rows only; dgrad stops at the lowest covered layer.
  // dgrad_l on s (the Delta chain), wgrad_l (+ bias) on s2.
  // Delta is triple-buffered (Delta_l in buffer l % 3), so dgrad_l only has
  // to wait for wgrad_{l+2}, the last reader of the buffer it overwrites.
  // Fused: wgrad_l updates W_l in place, so it also waits for dgrad_l (the
  // last reader of W_l). Collectives and per-layer updates hang off the
  // events recorded here.
  auto ev_delta = [&](int l) { return ev(kEvLayer + 2 * l); };     // Delta_l ready (on s)
  auto ev_wgrad = [&](int l) { return ev(kEvLayer + 2 * l + 1); }; // wgrad_l done (on s2)
  if (two) SPB_CUDA(cudaEventRecord(ev_delta(L - 1), s));          // from the head kernel
  int l = L - 1;
  for (; l >= 1; --l) {
    if (row0[l] >= rows) break;
    const int r0 = row0[l], cnt = rows - r0;
    const int b = l % kDbuf, bn = (l - 1) % kDbuf;
    const bool has_dgrad = l > 1 && row0[l - 1] < rows;
    // dgrad: Delta_{l-1} = (Delta_l W_l) * (1 - H_{l-1}^2), on s.
    if (has_dgrad) {
      if (two && l + 2 <= L - 1) SPB_CUDA(cudaStreamWaitEvent(s, ev_wgrad(l + 2), 0));
      const int q0 = row0[l - 1], qn = rows - q0;
      Operand A{Dh[b] + q0 * ldd, Dl[b] + q0 * ldd, ldd, qn, w[l], false};
      Operand B{p_hi + w_off[l], p_lo + w_off[l], ld[l - 1], w[l - 1], w[l], true};
      GemmEpilogue ep{};
      ep.out_hi = Dh[bn] + q0 * ldd;
      ep.out_lo = Dl[bn] + q0 * ldd;
      ep.ld_out = ldd;
      ep.h_hi = Hh[l - 1] + q0 * ld[l - 1];
      ep.h_lo = Hl[l - 1] + q0 * ld[l - 1];
      ep.ld_h = ld[l - 1];
      ep.M = qn;
      ep.N = w[l - 1];
      ep.splitk_ws = splitk_ws;
      ep.splitk_ws_floats = kSplitkWsFloats;
      pbeg(s);
      {
        SmReserve part(two && dsms > 0 ? std::max(reserved_sms, sm_total() - dsms) : reserved_sms);
        n += gemm_tf32x3(A, B, kEpiDgradTanh, ep, s);
      }
      pend(kClsDgrad, 2.0 * qn * w[l] * w[l - 1], s);
    }
    if (two) {
      // Delta_{l-1} ready / dgrad_l (last reader of W_l) done.
      SPB_CUDA(cudaEventRecord(ev_delta(l - 1), s));
      SPB_CUDA(cudaStreamWaitEvent(s2, lf(l) ? ev_delta(l - 1) : ev_delta(l), 0));
    }
    {  // wgrad + bias: [dW_l | db_l] = alpha_l * Delta_l[r0:]^T [H_{l-1}[r0:] | 1] (or the fused update)
      const int bc = static_cast<int>(round_up(w[l - 1], 32));  // the fused bias column (ones box)
      Operand A{Dh[b] + r0 * ldd, Dl[b] + r0 * ldd, ldd, w[l], cnt, true};
      Operand B{Hh[l - 1] + r0 * ld[l - 1], Hl[l - 1] + r0 * ld[l - 1], ld[l - 1], bc + 1, cnt, true, w[l - 1]};
      GemmEpilogue ep{};
      ep.ld_out = ld[l - 1];
      ep.alpha = alpha[l];
      ep.M = w[l];
      ep.N = w[l - 1];
      ep.bias_col_p1 = ep.ones_col_p1 = bc + 1;
      ep.colsum_ws = colsum_ws, ep.colsum_cnt = colsum_cnt;
      if (lf(l)) {
        ep.out_hi = p_hi + w_off[l];
        ep.out_lo = p_lo + w_off[l];
        ep.mom = mom ? mom + w_off[l] : nullptr;
        ep.gb_hi = p_hi + b_off[l];
        ep.gb_lo = p_lo + b_off[l];
        ep.gb_mom = mom ? mom + b_off[l] : nullptr;
        ep.lr = lr;
        ep.mu = mu;
        ep.wd = wd;
      } else {
        ep.out_hi = grad + w_off[l];
        ep.gb_hi = grad + b_off[l];  // local even when the weight rows are routed (the push signal sends it)
        if (route_push) push_route(l, ep);  // rows stored straight to their owners
      }
      pbeg(sw);
      {
        SmReserve part(two && wsms > 0 ? std::max(reserved_sms, sm_total() - wsms) : reserved_sms);
        n += gemm_tf32x3(A, B, lf(l) ? kEpiWgradUpdate : kEpiStoreScaled, ep, sw);
      }
      pend(kClsWgrad, 2.0 * cnt * w[l] * w[l - 1], sw);
    }
    if (two) SPB_CUDA(cudaEventRecord(ev_wgrad(l), s2));
    if (on_grad) n += on_grad(l, sw);
    if (on_layer) on_layer(l, sw);  // grad of layer l final on sw; dgrad_l (last W_l reader) done on s
  }
  if (two) {  // join the side stream
    SPB_CUDA(cudaEventRecord(ev(kEvJoin), s2));
    SPB_CUDA(cudaStreamWaitEvent(s, ev(kEvJoin), 0));
  }
  for (; l >= 1 && on_grad; --l) {  // no local rows below here
    n += on_grad(l, s);
    if (on_layer) on_layer(l, s);
  }
  return n;
}

int Engine::enqueue_head_wgrad(const float* h_hi, const float* h_lo, long ldh, int r0, int rows, int n_in, float a,
                               bool /*push*/, float* ws, long ws_floats, cudaStream_t q) {
  const int cnt = rows - r0, bc = static_cast<int>(round_up(n_in, 32));
  Operand A{delta + static_cast<long>(r0) * ldq, delta_lo + static_cast<long>(r0) * ldq, ldq, nout, cnt, true};
  Operand B{h_hi + static_cast<long>(r0) * ldh, h_lo + static_cast<long>(r0) * ldh, ldh, bc + 1, cnt, true, n_in};
  GemmEpilogue ep{};
  ep.out_hi = grad + w_off[L];
  ep.ld_out = ldf[L];
  ep.alpha = a;
  ep.M = nout;
  ep.N = n_in;
  ep.bias_col_p1 = ep.ones_col_p1 = bc + 1;
  ep.gb_hi = grad + b_off[L];
  ep.colsum_ws = colsum_ws, ep.colsum_cnt = colsum_cnt;
  ep.splitk_ws = ws;
  ep.splitk_ws_floats = ws_floats;
  return gemm_tf32x3(A, B, kEpiStoreScaled, ep, q);
}

void Engine::step_plan(bool full, std::vector<int>& row0, std::vector<float>& alpha) const {
  const int rows = static_cast<int>(workers.size()) * bw;
  row0.assign(L + 1, rows);
  alpha.assign(L + 1, 0.f);
  auto chunk_of = layer_chunks(k, L);
  for (int l = 1; l <= L; ++l) {
    if (full) {
      row0[l] = 0;
      alpha[l] = 1.0f / static_cast<float>(static_cast<long>(k) * bw);
      continue;
    }
    for (size_t t = 0; t < workers.size(); ++t)
      if (worker_stop(workers[t], k, L) <= l) {
        row0[l] = static_cast<int>(t) * bw;
        break;
      }
    alpha[l] = 1.0f / static_cast<float>(static_cast<long>(chunk_of[l - 1]) * bw);
  }
}

int Engine::enqueue_step(bool full, bool host_rows, cudaStream_t s, int sub, int nsub) {
  const int rows = static_cast<int>(workers.size()) * bw;
  int n = 0;
  if (nsub < 1 || nsub > kMaxChain || sub < 0 || sub >= nsub) throw ArgumentError("enqueue_step: bad chain index");
  chain_sub = sub;
  if (sub == 0) fwd_wait.assign(L + 1, -1);
  const bool last = sub == nsub - 1;
  // The gather overwrites H_0, read by wgrad_1 of the previous step (s2,
  // joined into s by enqueue_pass), so it needs no extra wait.
  pbeg(s);
  if (host_rows && conv_model) {
    // Host images already in xin (spb_step_host): identity index, and no
    // target copy (nout = 0: ybatch was uploaded directly).
    launch_conv_gather(xin, ldx, nullptr, static_cast<int>(pix[0]), w[0], 0, rows, rows, rows, workers_dev, nullptr, 0,
                       nullptr, 0, iota_dev, nullptr, Hh[0], Hl[0], ld[0], nullptr, s);
  } else if (host_rows) {
    launch_split_rows(xin, w[0], rows, w[0], Hh[0], Hl[0], ld[0], s);
  } else {
    enqueue_gather(X, ldx, rows, bw, &ctl->seed, 0, &ctl->step, 0, nullptr, s);
  }
  pend(kClsGather, 0, s);
  ++n;
  std::vector<int> row0;
  std::vector<float> alpha;
  step_plan(full, row0, alpha);
  // Unfused optimizer: one update launch per layer on s3, issued as soon as
  // the layer's gradient is final (wgrad on s2, or its NCCL bucket on cst)
  // and its last reader dgrad_l (on s) is done, so the HBM-bound update
  // runs beside the remaining backward GEMMs instead of after them.
  // Cross-rank exchange: the layer hooks of the active mode (a context that
  // joined a 1-rank clique aggregates locally).
  const bool xch = comm && nranks > 1;
  if (xch && comm_mode != 2 && comm_mode != 3 && comm_mode != 4 && comm_mode != 5)
    throw ConfigError("comm: no exchange mode selected");
  const bool fused_ok = fused_mode != 0 && !conv_model && !xch;  // the conv pass has no fused epilogue
  fuse_layer.assign(L + 1, 0);
  bool any_unfused = !fused_ok;
  for (int l = 1; l <= L; ++l) {
    // The head (layer L) is never fused: its wgrad is a split-K GEMM, which
    // has no in-place optimizer epilogue.
    fuse_layer[l] = fused_ok && l < L && row0[l] < rows && (fused_mode == 1 || rows - row0[l] <= kFuseMaxRows);
    if (!fuse_layer[l]) any_unfused = true;
  }
  const bool per_layer = any_unfused;
  cudaStream_t us = concurrent ? s3 : s;
  auto fork = [&](cudaStream_t to, int e) {
    SPB_CUDA(cudaEventRecord(ev(e), s));
    SPB_CUDA(cudaStreamWaitEvent(to, ev(e), 0));
  };
  auto join = [&](cudaStream_t from, int e) {
    SPB_CUDA(cudaEventRecord(ev(e), from));
    SPB_CUDA(cudaStreamWaitEvent(s, ev(e), 0));
  };
  if (xch && comm_mode == 3) {
    fork(cst, kEvStepFork);
    fork(s3, kEvUpdFork);
    n += enqueue_pass(rows, row0, alpha, s,
                      [&](int l, cudaStream_t from) { return enqueue_sub_layer(l, full, from, s); }, false,
                      &ctl->step, nullptr);
    join(cst, kEvStepJoin);  // not pipelined across steps: joined every step
    join(s3, kEvUpdJoin);
    fwd_wait.assign(L + 1, -1);
    return n;
  }
  if (xch && (comm_mode == 2 || comm_mode == 5)) {
    // Per layer (top down): G signal on the gradient stream, gradient and
    // weight pulls on per-peer copy streams, shard update on s3, split on
    // s4; all joined back into s, then the epoch advances. (5 = rh: the
    // same streams, recursive-halving / -doubling pull schedule.)
    std::vector<cudaStream_t> side = {s3, s4};
    for (int p = 0; p < nranks; ++p)
      if (p != rank) side.push_back(gpull[p]), side.push_back(wpull[p]);
    for (size_t i = 0; i < side.size(); ++i) fork(side[i], kEvP2pFork + static_cast<int>(i));
    n += enqueue_pass(rows, row0, alpha, s,
                      [&](int l, cudaStream_t from) {
                        return comm_mode == 5 ? enqueue_rh_layer(l, full, from, s) : enqueue_p2p_layer(l, full, from, s);
                      },
                      false, &ctl->step, nullptr);
    if (!last) return n;  // enqueue_p2p_layer / enqueue_rh_layer set fwd_wait for the next step
    for (size_t i = 0; i < side.size(); ++i) join(side[i], kEvP2pFork + 32 + static_cast<int>(i));
    launch_p2p_epoch(epoch_dev, nsub, s);
    return n + 1;
  }
  if (xch && comm_mode == 4) {
    // Per layer (top down): gradient rows stored to their owners by the
    // wgrad epilogue, G signal on the gradient stream, owner update on s3,
    // weight pulls on per-peer copy streams, split on s4.
    std::vector<cudaStream_t> side = {s3, s4};
    for (int p = 0; p < nranks; ++p)
      if (p != rank) side.push_back(wpull[p]);
    for (size_t i = 0; i < side.size(); ++i) fork(side[i], kEvP2pFork + static_cast<int>(i));
    route_push = true;
    try {
      n += enqueue_pass(rows, row0, alpha, s,
                        [&](int l, cudaStream_t from) { return enqueue_push_layer(l, full, from, s); }, false,
                        &ctl->step, nullptr);
    } catch (...) {
      route_push = false;
      throw;
    }
    route_push = false;
    if (!last) return n;
    for (size_t i = 0; i < side.size(); ++i) join(side[i], kEvP2pFork + 32 + static_cast<int>(i));
    launch_p2p_epoch(epoch_dev, nsub, s);
    return n + 1;
  }
  if (per_layer && concurrent) fork(s3, kEvUpdFork);
  auto on_layer = [&](int l, cudaStream_t grad_stream) {
    if (fuse_layer[l]) return;  // updated inside its wgrad epilogue
    SPB_CUDA(cudaEventRecord(ev(kEvUpd + 2 * l), s));  // dgrad_l issued before this point on s
    SPB_CUDA(cudaEventRecord(ev(kEvUpd + 2 * l + 1), grad_stream));
    SPB_CUDA(cudaStreamWaitEvent(us, ev(kEvUpd + 2 * l), 0));
    SPB_CUDA(cudaStreamWaitEvent(us, ev(kEvUpd + 2 * l + 1), 0));
    const long off = w_off[l], cnt = b_off[l] + round_up(w[l], 32) - w_off[l];
    pbeg(us);
    launch_sgd_update(p_hi + off, p_lo + off, grad + off, mom ? mom + off : nullptr, cnt, lr, mu, wd, us);
    // Algorithmic bytes: read w, g (+ mom), write w
    // (+ mom), 4 B each, over the layer's real parameters. The split-pair
    // storage moves 28 B / 20 B per stored element (hi and lo for w).
    pend(kClsUpdate, static_cast<double>(w[l]) * (fan[l] + 1) * (mom ? 20.0 : 12.0), us);
    ++n;
    if (us != s) {  // W_l final on us
      SPB_CUDA(cudaEventRecord(ev(ev_ready(l)), us));
      fwd_wait[l] = ev_ready(l);
    }
  };
  n += enqueue_pass(rows, row0, alpha, s, nullptr, fused_ok, &ctl->step,
                    per_layer ? std::function<void(int, cudaStream_t)>(on_layer) : nullptr);
  if (per_layer && concurrent && last) join(s3, kEvUpdJoin);
  return n;
}

cudaGraphExec_t Engine::get_graph(bool full, bool host_rows, int nsub, int* launches) {
  auto& slot = graphs[std::make_tuple(full, host_rows, nsub)];
  if (!slot.first) {
    cudaGraph_t gr;
    SPB_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    int n = 0;
    try {
      for (int t = 0; t < nsub; ++t) n += enqueue_step(full, host_rows, st, t, nsub);
    } catch (...) {
      fwd_wait.clear();
      cudaStreamEndCapture(st, &gr);
      graphs.erase(std::make_tuple(full, host_rows, nsub));
      throw;
    }
    fwd_wait.clear();  // its events belong to this capture
    SPB_CUDA(cudaStreamEndCapture(st, &gr));
    cudaGraphExec_t g = nullptr;
    cudaError_t e = cudaGraphInstantiate(&g, gr, 0);
    cudaGraphDestroy(gr);
    if (e != cudaSuccess) {
      graphs.erase(std::make_tuple(full, host_rows, nsub));
      SPB_CUDA(e);
    }
    slot = {g, n / nsub};
  }
  if (launches) *launches = slot.second;
  return slot.first;
}

void Engine::run_steps(bool full, int steps, float* losses) {
  int done = 0;
  while (done < steps) {
    const int c = std::max(1, std::min({chain_len(), kMaxChain, steps - done}));
    cudaGraphExec_t g = get_graph(full, false, c, &last_launches);
    SPB_CUDA(cudaGraphLaunch(g, st));
    if (losses) SPB_CUDA(cudaMemcpyAsync(losses + done, loss_dev, c * sizeof(float), cudaMemcpyDeviceToHost, st));
    done += c;
  }
}

}  // namespace spb
