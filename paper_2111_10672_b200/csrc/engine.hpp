// The SPB engine behind the C ABI (include/spb_b200.h): device state for one
// ChainMlp / ConvNet on one B200. The code is split by concern:
//   engine.cu   -- allocation, the per-step launch program (forward -> head ->
//                  truncated backward -> update) and CUDA-graph capture;
//   exchange.cu -- the multi-GPU aggregation of a layer (p2p / rh / push /
//                  sub modes), enqueued per layer from the backward;
//   capi.cu     -- the extern "C" entry points (reference-facing worker /
//                  aggregator calls, tooling).
//
// HBM layout (all fp32, rows padded to a multiple of 4 elements = 16 B):
//   params  : one flat allocation per role -- p_hi, p_lo (the exact 3xTF32
//             split, W = hi + lo), grad, mom. Layer l owns W_l [n_l x ld_{l-1}]
//             at w_off[l] and b_l [n_l] at b_off[l], each segment aligned to
//             32 elements (128 B), so a single update launch covers all.
//   H_l     : activations of hidden layer l (l = 0 is the gathered input),
//             split pair [rows x ld_l].
//   Delta   : two ping-pong split pairs [rows x ld_max] (Delta_l lives in
//             buffer l % 2).
// Row order: hosted workers ascending, per_worker_batch rows each, so the
// contributors of every layer are a contiguous tail of rows (chunk_coverage,
// spb.cpp:23-29) and each layer's aggregate is ONE wgrad GEMM over that tail.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/spb_b200.h"
#include "gemm_tf32x3.cuh"
#include "conv.hpp"
#include "launch.hpp"
#include "p2p.hpp"
#include "planner.hpp"

namespace spb {

// NCCL is resolved at first use with dlopen, never at library load: the
// process may also host torch's own NCCL (a newer libnccl.so.2), and binding
// the system one at load time would shadow it. SPB_NCCL_LIB (set by the
// Python front-end to torch's bundled copy when present) wins; otherwise the
// already-loaded or system libnccl.so.2 is used.
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  ncclResult_t (*CommFinalize)(ncclComm_t);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*);
  const char* (*GetErrorString)(ncclResult_t);
};

const NcclApi& nccl();  // engine.cu

inline void nccl_check(ncclResult_t r) {
  if (r != ncclSuccess) throw std::runtime_error(std::string("nccl: ") + nccl().GetErrorString(r));
}

struct Ctl {
  uint64_t seed;
  int step;
  int pad;
};

// Event slots (Engine::ev): fork/join of the step, per-layer backward and
// per-layer bucket events.
enum { kEvStepFork = 0, kEvStepJoin = 1, kEvFork = 2, kEvJoin = 3, kEvUpdFork = 4, kEvUpdJoin = 5, kEvBucket = 8,
       kEvLayer = 8 + 1024, kEvUpd = 8 + 3072, kEvP2pFork = 8 + 5120, kEvP2pLayer = 8 + 5120 + 64 };

// Kernel classes of spb_profile_step (index into its output arrays).
enum { kClsFwd = 0, kClsWgrad, kClsDgrad, kClsHead, kClsColred, kClsUpdate, kClsGather, kClsComm, kNumCls };

struct Engine {
  int dev = 0;
  cudaStream_t st = nullptr;
  std::vector<int> w;  // widths n_0..n_L
  int L = 0, nout = 0;
  int k = 1, bw = 1;
  std::vector<long> ld;            // ld[l] = round_up(n_l, 4)
  std::vector<long> w_off, b_off;  // index 1..L
  // Weight geometry of layer l (1..L): W_l is [w[l] x fan[l]] stored with row
  // stride ldf[l]. ChainMlp: fan[l] = w[l-1], ldf[l] = ld[l-1].
  std::vector<int> fan;
  std::vector<long> ldf;
  // ConvNet (conv_model): layers 1..L-1 are 3x3 convolutions (cg[l]) over
  // NHWC pixel rows, pix[l] pixels per sample (pix[0] = the input image);
  // layer L is the affine head on the globally average-pooled features.
  bool conv_model = false;
  std::vector<ConvGeom> cg;
  std::vector<long> pix;
  std::vector<float*> Ch, Cl;  // im2col split pairs, [samples * pix[l] x ldf[l]], kept for wgrad
  float *Ph = nullptr, *Pl = nullptr, *Gh = nullptr, *Gl = nullptr;  // pooled features / their gradient
  float* dcol = nullptr;  // dgrad columns (fp32), reused per layer
  float *Fh = nullptr, *Fl = nullptr;  // flipped kernel of the current implicit dgrad
  int* iota_dev = nullptr;
  long ldx = 0;  // dataset row stride
  long nflat = 0, ldd = 0;
  float *p_hi = nullptr, *p_lo = nullptr, *grad = nullptr, *mom = nullptr;
  float lr = 0.01f, mu = 0.f, wd = 0.f;
  // dataset
  float *X = nullptr, *Y = nullptr;
  int N = 0;
  // spb_loss64: the fp64 parameters last evaluated (host copy + device copy).
  std::vector<double> p64_host;
  double* p64 = nullptr;
  // row workspace
  int cap_rows = 0;
  std::vector<float*> Hh, Hl;
  static constexpr int kDbuf = 3;  // Delta_l lives in buffer l % 3
  float *Dh[kDbuf] = {nullptr, nullptr, nullptr}, *Dl[kDbuf] = {nullptr, nullptr, nullptr};
  // delta_L (head output error) as a split pair [rows x ldq], ldq = round_up(n_L, 4):
  // the A operand of the head's wgrad GEMM.
  float *delta = nullptr, *delta_lo = nullptr, *row_loss = nullptr, *ybatch = nullptr, *xin = nullptr;
  long ldq = 4;
  int* idx = nullptr;
  int* idx_in = nullptr;
  float* loss_dev = nullptr;
  float* tmp = nullptr;
  long tmp_n = 0;
  float* splitk_ws = nullptr;  // split-K partials (forward / dgrad GEMMs, stream s only)
  static constexpr long kSplitkWsFloats = 16L << 20;
  float* splitk_ws3 = nullptr;  // ConvNet: split-K partials of the wgrads (gradient stream s2)
  // 256 MB: room for ~30-60 K-splits of the widest conv wgrads (M = 512, N = 4609)
  static constexpr long kConvWsFloats = 64L << 20;
  float* splitk_ws2 = nullptr;  // split-K partials of the head wgrad (the gradient stream s2)
  // Column-sum bias slices + counters of the 1-CTA wgrads (GemmEpilogue::
  // colsum_ws): the wgrads run in stream order (s2, or s for the ConvNet).
  float* colsum_ws = nullptr;
  int* colsum_cnt = nullptr;
  static constexpr long kSplitkWs2Floats = 1L << 20;
  Ctl* ctl = nullptr;
  int* workers_dev = nullptr;
  std::vector<int> workers;  // hosted workers, ascending
  // graphs, keyed by (full, host_rows, steps chained in the graph); value:
  // (exec, kernel launches per step)
  std::map<std::tuple<bool, bool, int>, std::pair<cudaGraphExec_t, int>> graphs;
  int last_launches = 0;
  // Cross-step pipelining (a chain of `chain` steps captured in ONE graph):
  // step t+1's forward of layer l waits only for W_l of step t (its update,
  // and in multi-GPU modes its exchange), not for the whole of step t, so the
  // exchange / update tail of step t runs beside the forward of step t+1.
  // fwd_wait[l] = event index the forward of layer l (the head for l = L)
  // must wait on, -1 = none; chain_sub = index of the step being enqueued.
  static constexpr int kMaxChain = 16;
  static constexpr long kGradSlack = 4096;
  // chain = 0: automatic = 1. Measured (cfg5 sweep, one box, chain 8 vs 1):
  // -16 % / -8 % / -1 % / +1 % at widths 1k / 2k / 4k / 8k on one GPU,
  // -2 to -7 % with a multi-GPU exchange (its tail running beside the next
  // forward slows both), and slower on the launch-bound cfg2. Kept as an
  // option (SPB_CHAIN / spb_set_chain).
  int chain = default_chain();
  int chain_sub = 0;
  static int default_chain() {
    const char* c = std::getenv("SPB_CHAIN");
    if (!c) return 0;
    const int v = std::atoi(c);
    return v < 1 ? 1 : (v > kMaxChain ? kMaxChain : v);
  }
  int chain_len() const { return chain > 0 ? chain : 1; }
  std::vector<int> fwd_wait;
  std::string err;
  // multi-GPU
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1;
  cudaStream_t cst = nullptr;  // collectives
  cudaStream_t s2 = nullptr;   // wgrad branch of the backward (runs beside dgrad)
  cudaStream_t s3 = nullptr;   // per-layer optimizer updates (run beside the backward GEMMs)
  std::vector<Bucket> buckets[2];  // [full]
  std::vector<cudaEvent_t> evs;    // fork/join events (reused)
  // Single-GPU optimizer placement: 0 = per-layer update kernels, 1 = inside
  // every wgrad epilogue, 2 = auto (the default): inside the epilogue of the
  // wgrads over <= kFuseMaxRows contributor rows, where it is cheaper than a
  // separate update pass (measured: the fused epilogue costs the same as
  // wgrad + update at 1024 rows and saves ~20 us per layer at <= 512).
  int fused_mode = default_fused_mode();
  static int default_fused_mode() {  // SPB_FUSED_MODE: A/B experiments (spb_set_fused_update sets it per context)
    const char* v = std::getenv("SPB_FUSED_MODE");
    return v ? std::max(0, std::min(2, std::atoi(v))) : 2;
  }
  static constexpr int kFuseMaxRows = 512;  // 640 / 768 measured the same; 384 slower
  std::vector<char> fuse_layer;  // per layer, set by enqueue_step for enqueue_pass / on_layer
  // Multi-GPU aggregation mode (0 = none selected yet):
  // 2 = peer-to-peer copy-engine pulls (p2p.cu), 3 = NCCL contributor
  // sub-communicators ("sub": reduce-scatter among the layer's contributing
  // ranks only, sharded update, weight broadcast to every rank).
  int comm_mode = 0;
  // sub mode: one NCCL communicator per distinct contributor-rank set
  // (ncclCommSplit of `comm`; null on ranks outside the set), keyed by the set.
  std::map<std::vector<int>, ncclComm_t> subcomms;
  // SMs the persistent GEMMs of this context leave free (spb_comm_init: 16
  // with NCCL collectives in the step, 0 for the copy-engine modes).
  int reserved_sms = 0;
  // SM partition of the concurrent backward: persistent grids of the dgrad
  // chain (stream s) and of the wgrads (s2) capped at these SM counts, so
  // the two streams (and the exchange kernels beside them) share the SMs by
  // partition instead of by whichever CTAs the scheduler places first.
  // -1 = automatic: 68 / 72 with a multi-GPU exchange (measured 4.5 -> 4.28
  // ms at 4 ranks, 4.50 -> 4.31 at 2), off on one GPU (there it costs 3-6 %);
  // SPB_DGRAD_SMS / SPB_WGRAD_SMS override (0 = off).
  int dgrad_sms = env_int("SPB_DGRAD_SMS", -1);
  int wgrad_sms = env_int("SPB_WGRAD_SMS", -1);
  static int env_int(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return v ? std::max(0, std::atoi(v)) : dflt;
  }
  int part_sms(int v, int dflt) const { return v >= 0 ? v : (comm && nranks > 1 ? dflt : 0); }
  static int sm_total() {
    int dev = 0, n = 0;
    SPB_CUDA(cudaGetDevice(&dev));
    SPB_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
    return n;
  }
  // p2p mode: fp32 weights (own shards published to the peers), epoch-stamped
  // flags [2 * (L + 1)][nranks], gradient staging [2][nranks - 1][shard], and
  // the peers' IPC-mapped grad / w32 / flags.
  float* w32 = nullptr;
  int* flags = nullptr;
  float* stage = nullptr;
  long stage_shard = 0;
  PeerPtrs<int> peer_flags{};
  std::vector<float*> peer_grad, peer_w32;
  // push mode (comm_mode 4, push.cu): layer l's rows are owned block-wise
  // (rank o: rows [o * prpo[l], (o + 1) * prpo[l])); pstage holds, per layer
  // and source rank, the source's gradient rows this rank owns (weight rows
  // then bias rows, pslot[l] floats per source), written by the sources'
  // wgrad epilogues over NVLink.
  float* pstage = nullptr;
  std::vector<int> prpo;
  std::vector<long> pstage_off, pslot;
  std::vector<float*> peer_pstage;
  int flag_slots = 2;  // flags per layer (p2p / push: 2; rh: 2 log2 N)
  bool route_push = false;  // set while enqueue_step builds a push-mode step
  // spb_step_host_async: double-buffered device staging of host batches,
  // filled on their own copy stream while the previous step runs.
  float *hx[2] = {nullptr, nullptr}, *hy[2] = {nullptr, nullptr};
  long hx_n = 0, hy_n = 0;
  cudaStream_t hst = nullptr;
  unsigned host_calls = 0;
  // Losses of async steps land in a pinned ring (a D2H copy into pageable
  // memory would block the host until the step finished) and are copied to
  // the callers' pointers at the next synchronisation.
  static constexpr int kLossRing = 64;
  float* loss_pin = nullptr;
  std::vector<std::pair<float*, int>> loss_pending;
  void flush_losses() {  // after a stream synchronisation
    for (auto& pr : loss_pending) *pr.first = loss_pin[pr.second];
    loss_pending.clear();
  }
  cudaStream_t s4 = nullptr;
  std::vector<cudaStream_t> gpull, wpull;  // per-peer copy streams (copy engines run concurrently)
  int* epoch_dev = nullptr;  // completed steps of the flag-synchronised exchange modes
  float* bar_dev = nullptr;  // host-barrier scratch
  bool concurrent = true;          // side streams (off in spb_profile_step: clean per-kernel times)

  // Eager-mode instrumentation (spb_profile_step): CUDA events around every
  // launch, tagged with a kernel class and its algorithmic work.
  struct ProfRec {
    int cls;
    double work;
    cudaEvent_t a, b;
  };
  std::vector<ProfRec>* prof = nullptr;
  cudaEvent_t prof_a = nullptr;
  // Timeline tracing (spb_trace_steps): a %globaltimer stamp kernel before
  // and after every op of a captured graph, on the op's own stream, so the
  // replayed graph's real per-stream schedule can be read back.
  static constexpr int kTraceCap = 1 << 15;  // ops
  static constexpr int kTraceWait = 100;     // class of the p2p flag waits (trace only)
  struct TraceRec {
    int cls, stream, sub;
  };
  bool tracing = false;
  unsigned long long* trace_dev = nullptr;
  std::vector<TraceRec> trace_meta;
  int trace_open = -1;
  int stream_id(cudaStream_t q) const {
    if (q == st) return 0;
    if (q == s2) return 1;
    if (q == s3) return 2;
    if (q == s4) return 3;
    if (q == cst) return 4;
    for (size_t p = 0; p < gpull.size(); ++p)
      if (q == gpull[p]) return 10 + static_cast<int>(p);
    for (size_t p = 0; p < wpull.size(); ++p)
      if (q == wpull[p]) return 20 + static_cast<int>(p);
    return 99;
  }
  void tbeg(cudaStream_t s) {
    if (!tracing) return;
    if (trace_meta.size() >= static_cast<size_t>(kTraceCap)) throw ConfigError("trace: too many ops");
    trace_open = static_cast<int>(trace_meta.size());
    trace_meta.push_back({-1, stream_id(s), chain_sub});
    launch_stamp(trace_dev + 2 * trace_open, s);
  }
  void tend(int cls, cudaStream_t s) {
    if (!tracing || trace_open < 0) return;
    trace_meta[trace_open].cls = cls;
    launch_stamp(trace_dev + 2 * trace_open + 1, s);
    trace_open = -1;
  }
  void pbeg(cudaStream_t s) {
    tbeg(s);
    if (!prof) return;
    SPB_CUDA(cudaEventCreate(&prof_a));
    SPB_CUDA(cudaEventRecord(prof_a, s));
  }
  void pend(int cls, double work, cudaStream_t s) {
    tend(cls, s);
    if (!prof) return;
    cudaEvent_t b;
    SPB_CUDA(cudaEventCreate(&b));
    SPB_CUDA(cudaEventRecord(b, s));
    prof->push_back({cls, work, prof_a, b});
  }

  ~Engine() { release(); }

  void release();

  template <class T>
  // Zeroed device allocation. cudaMemset runs on the legacy default stream,
  // which does NOT order against the context's non-blocking streams, so the
  // zeroing is waited for here: otherwise it could land after the first
  // writes on those streams (it did: spb_aggregate's staging buffer lost a
  // worker's block about once in 15 calls).
  static T* alloc(long n) {
    void* p = nullptr;
    SPB_CUDA(cudaMalloc(&p, static_cast<size_t>(n < 1 ? 1 : n) * sizeof(T)));
    SPB_CUDA(cudaMemset(p, 0, static_cast<size_t>(n < 1 ? 1 : n) * sizeof(T)));
    SPB_CUDA(cudaStreamSynchronize(0));
    return static_cast<T*>(p);
  }

  void init(const int* widths, int n_widths, int k_, int bw_, int device);

  // ConvNet: geom = {in_h, in_w, in_c, then (c_out, stride) per conv layer}.
  void init_conv(const int* geom, int nconv, int nout_, int k_, int bw_, int device);

  void allocate_params();

  void set_workers(const std::vector<int>& ws) {
    workers = ws;
    SPB_CUDA(cudaMemcpy(workers_dev, ws.data(), ws.size() * sizeof(int), cudaMemcpyHostToDevice));
    invalidate_graphs();
  }
  void set_workers_all() {
    std::vector<int> ws(k);
    std::iota(ws.begin(), ws.end(), 1);
    set_workers(ws);
  }

  void invalidate_graphs() {
    for (auto& kv : graphs)
      if (kv.second.first) cudaGraphExecDestroy(kv.second.first);
    graphs.clear();
  }

  // Event index "W_l of the current step final on this rank".
  static int ev_ready(int l) { return kEvP2pLayer + 32 * l + 2; }

  // Before the forward of layer l (the head for l = L): wait for W_l of the
  // previous step of the chain.
  void fwd_gate(int l, cudaStream_t s) {
    if (l < static_cast<int>(fwd_wait.size()) && fwd_wait[l] >= 0)
      SPB_CUDA(cudaStreamWaitEvent(s, ev(fwd_wait[l]), 0));
  }

  void ensure_rows(int rows);

  // ConvNet workspace for `samples` samples (rows = pixel rows per layer).
  void ensure_samples_conv(int samples);

  // Convolution l runs as an implicit GEMM (TMA im2col, no column matrix)
  // when its input channels fill whole 128-byte TMA boxes.
  // dgrad of convolution l as an implicit GEMM over Delta_l (stride 1, its
  // output channels filling whole TMA boxes).
  bool conv_tma_dgrad(int l) const {
    static const bool off = std::getenv("SPB_CONV_IM2COL") != nullptr;
    return !off && cg[l].stride == 1 && w[l] % 32 == 0 && ld[l] % 32 == 0;
  }

  bool conv_tma(int l) const {
    static const bool off = std::getenv("SPB_CONV_IM2COL") != nullptr;  // A/B experiments: materialise columns
    return !off && cg[l].c_in % 32 == 0 && ld[l - 1] % 32 == 0;
  }

  // Forward of convolution l as a direct fp32 kernel (the RGB layer: c_in <=
  // 4); its wgrad materialises the im2col columns of the contributor samples
  // only, in the backward. SPB_CONV_DIRECT=0: the im2col GEMM forward (A/B).
  bool conv_direct(int l) const {
    static const bool off = [] {
      const char* v = std::getenv("SPB_CONV_DIRECT");
      return v && std::string(v) == "0";
    }();
    return !off && !conv_tma(l) && conv_direct_ok(cg[l], ld[l - 1], ld[l]);
  }

  // Gathers `rows` samples (ChainMlp: rows; ConvNet: pixel rows of the
  // samples) into H_0 and ybatch: from idx_in, or drawn on the device.
  void enqueue_gather(const float* Xsrc, long ldxs, int rows, int bw_, const uint64_t* seed_dev, uint64_t seed_host,
                      const int* step_dev, int step_host, const int* idx_in_, cudaStream_t s) {
    if (conv_model)
      launch_conv_gather(Xsrc, ldxs, Y, static_cast<int>(pix[0]), w[0], nout, N, rows, bw_, workers_dev, seed_dev,
                         seed_host, step_dev, step_host, idx_in_, idx, Hh[0], Hl[0], ld[0], ybatch, s);
    else
      launch_gather(Xsrc, ldxs, Y, w[0], nout, N, rows, bw_, workers_dev, seed_dev, seed_host, step_dev, step_host,
                    idx_in_, idx, Hh[0], Hl[0], ld[0], ybatch, s);
  }

  // ConvNet pass (same contract as enqueue_pass; rows, row0 and alpha count
  // samples). Forward: im2col -> GEMM (bias + tanh) per convolution, global
  // average pool, head. Backward over the contributor samples' pixel rows:
  // wgrad = GEMM(Delta^T, im2col) scaled by alpha_l, bias column sums,
  // dgrad = GEMM(Delta, W) into columns -> col2im * (1 - H^2). One stream.
  int enqueue_pass_conv(int samples, const std::vector<int>& row0, const std::vector<float>& alpha, cudaStream_t s,
                        const std::function<int(int, cudaStream_t)>& on_grad, int* step_dev,
                        const std::function<void(int, cudaStream_t)>& on_layer);

  // ---- the per-step launch program ----------------------------------------
  // row0[l] (l = 1..L): first row contributing to layer l (rows when none).
  // alpha[l]: the averaging factor 1/(m_l * per_worker_batch) of layer l.
  // on_grad(l) runs after layer l's gradient is final on this rank (for every
  // layer, top down, including layers with no local contributor rows).
  // fused: apply the optimizer inside the backward (single-GPU step): the
  // wgrad GEMM epilogue updates W_l in place and the bias / head reductions
  // update b_l / W_L, so the gradient never round-trips through HBM. dgrad_l
  // then runs before wgrad_l, because it reads the pre-update W_l.
  // step_dev (nullable) is advanced once the gather has consumed it.
  int enqueue_pass(int rows, const std::vector<int>& row0, const std::vector<float>& alpha, cudaStream_t s,
                   const std::function<int(int, cudaStream_t)>& on_grad = nullptr, bool fused = false,
                   int* step_dev = nullptr, const std::function<void(int, cudaStream_t)>& on_layer = nullptr);

  // The head layer's wgrad over rows [r0, rows): [dW_L | db_L] =
  // alpha delta_L[r0:]^T [H[r0:] | 1] as ONE tcgen05 GEMM (M = n_L <= 16 rows
  // of one tile, N = n_{L-1} + the fused bias column, K = contributor rows;
  // split-K over `ws`). The old two column-reduction kernels are gone. In the
  // push exchange the head's rows travel with the signal, so it is never routed.
  int enqueue_head_wgrad(const float* h_hi, const float* h_lo, long ldh, int r0, int rows, int n_in, float a,
                         bool /*push*/, float* ws, long ws_floats, cudaStream_t q);

  cudaEvent_t ev(size_t i) {
    while (evs.size() <= i) {
      cudaEvent_t e;
      SPB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      evs.push_back(e);
    }
    return evs[i];
  }

  // p2p mode, layer l (see p2p.cu for the protocol). gs: the stream that
  // produced this rank's gradient of l; s: the main stream (dgrad_l, the last
  // local reader of W_l, was issued on it before this call).
  int enqueue_p2p_layer(int l, bool full, cudaStream_t gs, cudaStream_t s);

  // "rh" mode (N = 2^d ranks), layer l: Rabenseifner's all-reduce on the
  // copy engines -- recursive-halving reduce-scatter, the owner's update,
  // recursive-doubling all-gather of the fp32 weights -- so that every
  // transfer is a single-peer pull (measured ~760 GB/s per direction over
  // NVLink, against ~450 GB/s when a GPU pulls from 3 peers at once, the p2p
  // mode's pattern). Rank r owns shard r of the layer segment (the p2p
  // sharding). Reduce round k = 0..d-1 (bit b = d-1-k, partner r ^ 2^b): r
  // keeps the half of its current shard block whose bit b matches its own,
  // pulls the partner's partial sums of that half and adds them into its own
  // gradient buffer in place (the partner pulls the other half of r's buffer
  // meanwhile); the last round feeds the update kernel directly. Partial sums
  // that cover no contributor of the layer (SPB) are skipped. All-gather
  // round b = 0..d-1: pull the partner's weight block of 2^b shards. Flags
  // per layer (slot base 2d*l): +0 gradient final, +1+k reduce round k done
  // (k < d-1), +d+b weight block of 2^b shards final (b = 0: the update).
  int enqueue_rh_layer(int l, bool full, cudaStream_t gs, cudaStream_t s);

  // "sub" mode, layer l (the reference's
  // aggregate spb.cpp:89-104 restricted to the workers that reached the
  // layer): on cst, after this rank's gradient of l is final (gs) and its
  // dgrad_l -- the last local reader of W_l -- was issued on s:
  //  1. the layer's CONTRIBUTING ranks C (those hosting a worker whose suffix
  //     covers l) reduce-scatter the gradient among themselves over their
  //     sub-communicator; ranks outside C move no gradient bytes;
  //  2. each member updates its shard (momentum / wd / SGD; the 1/(m B_w)
  //     average is already in the wgrad epilogue), writing the new fp32
  //     weights of the shard to w32 (and its own hi / lo);
  //  3. every member broadcasts its shard to ALL ranks (one NCCL group), since
  //     non-contributors need the updated weights for their next forward;
  //  4. every rank splits the received fp32 weights into hi / lo.
  // A single contributor skips step 1 and updates the whole layer.
  int enqueue_sub_layer(int l, bool full, cudaStream_t gs, cudaStream_t s);

  // Shard length of a layer segment of cnt floats over `parts` ranks (a
  // multiple of 4 floats, parts * shard >= cnt; the last shards may be short
  // or empty). spb_layer_shard exports it for the protocol tests.
  static long layer_shard(long cnt, int parts) { return round_up((cnt + parts - 1) / parts, 4); }

  void setup_sub();

  // Collective over the ranks (spb_comm_init): allocate the p2p buffers and
  // map every peer's grad / w32 / flags through CUDA IPC.
  // slots_per_layer: epoch-stamped flags per layer (p2p: G and U; rh: see
  // enqueue_rh_layer).
  void setup_p2p(int slots_per_layer = 2);

  // push mode setup (collective over the ranks): staging slots, fp32 weight
  // copies for the received rows, flags; every peer's pstage / w32 / flags
  // mapped through CUDA IPC. MLP only (the conv wgrad has no row routing).
  void setup_push();

  // push mode: where the wgrad epilogue of layer l stores gradient row r
  // (GemmEpilogue::route): the owner's staging slot for this rank, or this
  // rank's own gradient buffer for its own rows.
  void push_route(int l, GemmEpilogue& ep) const;

  // push mode, layer l (protocol: push.cu). gs: the stream that produced this
  // rank's gradient of l (its wgrad already stored the weight rows to their
  // owners, except for the head layer); s: main stream (dgrad_l issued).
  int enqueue_push_layer(int l, bool full, cudaStream_t gs, cudaStream_t s);

  void host_barrier();

  // HBM bytes one update launch must move: read hi, lo, grad (+ mom), write
  // hi, lo (+ mom), 4 B each.
  double update_bytes() const { return static_cast<double>(nflat) * 4.0 * (mom ? 7 : 5); }

  // Row plan of one SPB step for the hosted workers.
  void step_plan(bool full, std::vector<int>& row0, std::vector<float>& alpha) const;

  // Step `sub` of a chain of `nsub` steps captured into one graph (sub = 0,
  // nsub = 1: a plain step). Side streams are joined back into s only after
  // the last step of the chain; before that, the next step's forward waits
  // per layer (fwd_wait) for the weights this step finalises.
  int enqueue_step(bool full, bool host_rows, cudaStream_t s, int sub = 0, int nsub = 1);

  // The graph of `nsub` chained steps (see enqueue_step); `launches` gets the
  // kernel launches per step.
  cudaGraphExec_t get_graph(bool full, bool host_rows, int nsub = 1, int* launches = nullptr);

  // Replay `steps` steps as chained graphs of up to `chain` steps each
  // (losses: the per-step loss, copied back asynchronously; may be null).
  void run_steps(bool full, int steps, float* losses);
};

}  // namespace spb
