// The SPB engine behind the C ABI (include/spb_b200.h): device state for one
// ChainMlp on one B200, the per-step launch program (forward -> head ->
// truncated backward -> update), CUDA-graph capture, and the
// reference-facing worker / aggregator entry points.
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
#include <cuda_runtime.h>
#include <dlfcn.h>
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
namespace {

thread_local std::string g_err;

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

void nccl_check(ncclResult_t r) {
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

}  // namespace

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

  void release() {
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
    f(splitk_ws2), f(colsum_ws), f(colsum_cnt);
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

  void init(const int* widths, int n_widths, int k_, int bw_, int device) {
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

  // ConvNet: geom = {in_h, in_w, in_c, then (c_out, stride) per conv layer}.
  void init_conv(const int* geom, int nconv, int nout_, int k_, int bw_, int device) {
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

  void allocate_params() {
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
    colsum_ws = alloc<float>(kColsumWsFloats);
    colsum_cnt = alloc<int>(kColsumCounters);
    ctl = alloc<Ctl>(1);
    loss_dev = alloc<float>(kMaxChain);
    workers_dev = alloc<int>(k);
    set_workers_all();
  }

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

  void ensure_rows(int rows) {
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

  // ConvNet workspace for `samples` samples (rows = pixel rows per layer).
  void ensure_samples_conv(int samples) {
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
                        const std::function<void(int, cudaStream_t)>& on_layer) {
    int n = 0;
    const int Lc = L - 1;
    for (int l = 1; l <= Lc; ++l) {
      fwd_gate(l, s);
      const int M = static_cast<int>(samples * pix[l]);
      const bool tma = conv_tma(l);
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
    int l = Lc;
    for (; l >= 1; --l) {
      if (row0[l] >= samples) break;
      const int b = l % kDbuf, bn = (l - 1) % kDbuf;
      const long r0 = row0[l] * pix[l], cnt = (samples - row0[l]) * pix[l];
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
        n += gemm_tf32x3(A, B, kEpiStoreScaled, ep, s);
        pend(kClsDgrad, 2.0 * qn * w[l] * fan[l], s);
        pbeg(s);
        launch_col2im_tanh(dcol, ldf[l], cg[l], static_cast<int>(row0[l - 1] * pix[l - 1]),
                           static_cast<int>((samples - row0[l - 1]) * pix[l - 1]), Hh[l - 1], Hl[l - 1], ld[l - 1],
                           Dh[bn], Dl[bn], ld[l - 1], s);
        pend(kClsDgrad, 0, s);  // the gather half of the stride-2 dgrad
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
        ep.splitk_ws = splitk_ws;  // few output tiles, K = pixel rows: split K (single stream)
        ep.splitk_ws_floats = kSplitkWsFloats;
        pbeg(s);
        if (tma) {
          ConvSrc src{Hh[l - 1], Hl[l - 1], ld[l - 1], samples, cg[l]};
          n += gemm_conv_wgrad(A, src, r0, ep, s);
        } else {
          n += gemm_tf32x3(A, B, kEpiStoreScaled, ep, s);
        }
        pend(kClsWgrad, 2.0 * cnt * w[l] * fan[l], s);
      }
      if (on_grad) n += on_grad(l, s);
      if (on_layer) on_layer(l, s);
    }
    for (; l >= 1 && on_grad; --l) {
      n += on_grad(l, s);
      if (on_layer) on_layer(l, s);
    }
    return n;
  }

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
                   int* step_dev = nullptr, const std::function<void(int, cudaStream_t)>& on_layer = nullptr) {
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
        n += gemm_tf32x3(A, B, kEpiDgradTanh, ep, s);
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
        n += gemm_tf32x3(A, B, lf(l) ? kEpiWgradUpdate : kEpiStoreScaled, ep, sw);
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

  // The head layer's wgrad over rows [r0, rows): [dW_L | db_L] =
  // alpha delta_L[r0:]^T [H[r0:] | 1] as ONE tcgen05 GEMM (M = n_L <= 16 rows
  // of one tile, N = n_{L-1} + the fused bias column, K = contributor rows;
  // split-K over `ws`). The old two column-reduction kernels are gone. In the
  // push exchange the head's rows travel with the signal, so it is never routed.
  int enqueue_head_wgrad(const float* h_hi, const float* h_lo, long ldh, int r0, int rows, int n_in, float a,
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
  int enqueue_p2p_layer(int l, bool full, cudaStream_t gs, cudaStream_t s) {
    const Bucket* bk = nullptr;
    for (auto& b : buckets[full])
      if (b.l_lo <= l && l <= b.l_hi) bk = &b;
    if (!bk) throw ConfigError("comm: no bucket for layer");
    unsigned contrib = 0;
    for (int r : bk->ranks) contrib |= 1u << r;
    const long off = w_off[l], cnt = b_off[l] + round_up(w[l], 32) - w_off[l], n4 = cnt / 4;
    auto lo_of = [&](int r) { return n4 * r / nranks * 4; };
    const long a = lo_of(rank), b = lo_of(rank + 1), sh = b - a;
    // Layer events: 0 dgrad_l issued (s), 1 shard updated (s3), 8+p gradient
    // pull from p done, 16+p weight pull from p done.
    auto evl = [&](int k) { return ev(kEvP2pLayer + 32 * l + k); };
    int n = 0;
    // 1. gradient of l final here -> G[l] to every rank.
    launch_p2p_signal(peer_flags, 2 * l, nranks, rank, epoch_dev, chain_sub, gs);
    SPB_CUDA(cudaEventRecord(evl(0), s));  // dgrad_l issued on s before this point
    ++n;
    // 2. copy engines, one stream per peer: wait for the peer's G[l] (every
    // peer's, contributor or not: that also orders this step's writes after
    // every peer finished the previous step), then pull its gradient of this
    // shard if it contributes.
    float* st_buf = stage + static_cast<long>(l % 2) * (nranks - 1) * stage_shard;
    PeerPtrs<const float> src{};
    int nsrc = 0, slot = 0;
    for (int r = 0; r < nranks; ++r) {
      if (r == rank) {
        if (contrib >> r & 1u) src.p[nsrc++] = grad + off + a;
        continue;
      }
      cudaStream_t cs = gpull[r];
      // Staging buffer l % 2 was last read by the shard update of layer l + 2,
      // or (top layers, chained step) of layer 1 / 2 of the previous step.
      if (l + 2 <= L)
        SPB_CUDA(cudaStreamWaitEvent(cs, ev(kEvP2pLayer + 32 * (l + 2) + 1), 0));
      else if (chain_sub > 0 && l + 2 - L >= 1 && l + 2 - L <= 2)
        SPB_CUDA(cudaStreamWaitEvent(cs, ev(kEvP2pLayer + 32 * ((l % 2) == 1 ? 1 : 2) + 1), 0));
      tbeg(cs);
      launch_p2p_wait(flags, 2 * l, nranks, 1u << r, epoch_dev, chain_sub, cs);
      tend(kTraceWait, cs);
      ++n;
      if (contrib >> r & 1u) {
        float* dst = st_buf + static_cast<long>(slot++) * stage_shard;
        pbeg(cs);
        if (sh > 0) SPB_CUDA(cudaMemcpyAsync(dst, peer_grad[r] + off + a, sh * 4, cudaMemcpyDeviceToDevice, cs));
        pend(kClsComm, static_cast<double>(sh) * 4.0, cs);
        src.p[nsrc++] = dst;
      }
      SPB_CUDA(cudaEventRecord(evl(8 + r), cs));
    }
    // 3. shard update (SMs) -> U[l].
    for (int r = 0; r < nranks; ++r)
      if (r != rank) SPB_CUDA(cudaStreamWaitEvent(s3, evl(8 + r), 0));
    SPB_CUDA(cudaStreamWaitEvent(s3, evl(0), 0));
    if (contrib >> rank & 1u) {
      SPB_CUDA(cudaEventRecord(ev(kEvBucket + l), gs));
      SPB_CUDA(cudaStreamWaitEvent(s3, ev(kEvBucket + l), 0));
    }
    pbeg(s3);
    launch_p2p_update(src, nsrc, p_hi + off + a, p_lo + off + a, mom ? mom + off + a : nullptr, w32 + off + a, sh, lr, mu,
                      wd, s3);
    pend(kClsUpdate, static_cast<double>(sh) * 4.0 * (nsrc + (mom ? 7 : 5)), s3);
    launch_p2p_signal(peer_flags, 2 * l + 1, nranks, rank, epoch_dev, chain_sub, s3);
    SPB_CUDA(cudaEventRecord(evl(1), s3));
    n += 2;
    // 4. copy engines, one stream per peer: pull its updated fp32 shard.
    for (int r = 0; r < nranks; ++r) {
      if (r == rank) continue;
      cudaStream_t cs = wpull[r];
      tbeg(cs);
      launch_p2p_wait(flags, 2 * l + 1, nranks, 1u << r, epoch_dev, chain_sub, cs);
      tend(kTraceWait, cs);
      ++n;
      const long ra = lo_of(r), rb = lo_of(r + 1);
      pbeg(cs);
      if (rb > ra)
        SPB_CUDA(cudaMemcpyAsync(w32 + off + ra, peer_w32[r] + off + ra, (rb - ra) * 4, cudaMemcpyDeviceToDevice, cs));
      pend(kClsComm, static_cast<double>(rb - ra) * 4.0, cs);
      SPB_CUDA(cudaEventRecord(evl(16 + r), cs));
      SPB_CUDA(cudaStreamWaitEvent(s4, evl(16 + r), 0));
    }
    // 5. split the pulled shards into (hi, lo) (after dgrad_l).
    SPB_CUDA(cudaStreamWaitEvent(s4, evl(0), 0));
    pbeg(s4);
    launch_p2p_split(w32 + off, p_hi + off, p_lo + off, cnt, a, b, s4);
    pend(kClsUpdate, static_cast<double>(cnt - sh) * 12.0, s4);
    ++n;
    // W_l final here: the peers' shards split (s4) and this rank's own (s3).
    SPB_CUDA(cudaStreamWaitEvent(s4, evl(1), 0));
    SPB_CUDA(cudaEventRecord(ev(ev_ready(l)), s4));
    fwd_wait[l] = ev_ready(l);
    return n;
  }

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
  int enqueue_rh_layer(int l, bool full, cudaStream_t gs, cudaStream_t s) {
    const Bucket* bk = nullptr;
    for (auto& b : buckets[full])
      if (b.l_lo <= l && l <= b.l_hi) bk = &b;
    if (!bk) throw ConfigError("comm: no bucket for layer");
    unsigned contrib = 0;
    for (int r : bk->ranks) contrib |= 1u << r;
    const int d = flag_slots / 2;
    const long off = w_off[l], cnt = b_off[l] + round_up(w[l], 32) - w_off[l], n4 = cnt / 4;
    auto lo_of = [&](int sidx) { return n4 * sidx / nranks * 4; };
    auto evl = [&](int k) { return ev(kEvP2pLayer + 32 * l + k); };
    auto slot = [&](int j) { return flag_slots * l + j; };
    // Ranks whose contributions a partial held by rank q before reduce round
    // k covers: those agreeing with q on bits 0..b (b = d-1-k).
    auto covers = [&](int q, int b) {
      unsigned m = 0;
      const int low = (1 << (b + 1)) - 1;
      for (int x = 0; x < nranks; ++x)
        if ((x & low) == (q & low)) m |= 1u << x;
      return m;
    };
    int n = 0;
    SPB_CUDA(cudaEventRecord(evl(0), s));  // dgrad_l (last reader of W_l) issued on s
    launch_p2p_signal(peer_flags, slot(0), nranks, rank, epoch_dev, chain_sub, gs);
    ++n;
    SPB_CUDA(cudaEventRecord(ev(kEvBucket + l), gs));
    SPB_CUDA(cudaStreamWaitEvent(s3, ev(kEvBucket + l), 0));
    SPB_CUDA(cudaStreamWaitEvent(s3, evl(0), 0));
    float* st_buf = stage + static_cast<long>(l % 2) * (nranks - 1) * stage_shard;
    long st_off = 0;
    bool own = contrib >> rank & 1u;  // does this rank's buffer hold a valid partial?
    PeerPtrs<const float> fin{};
    int nfin = 0;
    for (int k = 0; k < d; ++k) {
      const int b = d - 1 - k, p = rank ^ (1 << b);
      const int base = (rank >> (b + 1)) << (b + 1), s0 = base + (((rank >> b) & 1) << b), s1 = s0 + (1 << b);
      const long a0 = lo_of(s0), a1 = lo_of(s1), len = a1 - a0;
      const bool theirs = (covers(p, b) & contrib) != 0;
      cudaStream_t cs = gpull[p];
      // Staging reuse: the buffer of layer l % 2 was last read by layer l + 2's
      // update, or (top layers, chained step) by layer 1 / 2's update of the
      // previous step -- the same explicit wait as the p2p mode, instead of
      // relying on the transitive cross-rank flag ordering alone.
      if (k == 0 && l + 2 <= L)
        SPB_CUDA(cudaStreamWaitEvent(cs, ev(kEvP2pLayer + 32 * (l + 2) + 1), 0));
      else if (k == 0 && chain_sub > 0 && l + 2 - L >= 1 && l + 2 - L <= 2)
        SPB_CUDA(cudaStreamWaitEvent(cs, ev(kEvP2pLayer + 32 * ((l % 2) == 1 ? 1 : 2) + 1), 0));
      if (k > 0) SPB_CUDA(cudaStreamWaitEvent(cs, evl(3 + k - 1 + 8), 0));  // my previous round's sum done
      tbeg(cs);
      launch_p2p_wait(flags, k == 0 ? slot(0) : slot(k), nranks, 1u << p, epoch_dev, chain_sub, cs);
      tend(kTraceWait, cs);
      ++n;
      float* dst = nullptr;
      if (theirs) {
        dst = own ? st_buf + st_off : grad + off + a0;
        if (!own && k == 0) SPB_CUDA(cudaStreamWaitEvent(cs, ev(kEvBucket + l), 0));  // (own grad unused; order anyway)
        pbeg(cs);
        if (len > 0) SPB_CUDA(cudaMemcpyAsync(dst, peer_grad[p] + off + a0, len * 4, cudaMemcpyDeviceToDevice, cs));
        pend(kClsComm, static_cast<double>(len) * 4.0, cs);
      }
      SPB_CUDA(cudaEventRecord(evl(3 + k), cs));
      SPB_CUDA(cudaStreamWaitEvent(s3, evl(3 + k), 0));
      if (k < d - 1) {
        if (theirs && own) {
          pbeg(s3);
          launch_rh_add(grad + off + a0, st_buf + st_off, len, s3);
          pend(kClsUpdate, static_cast<double>(len) * 12.0, s3);
          ++n;
        }
        own = own || theirs;
        launch_p2p_signal(peer_flags, slot(1 + k), nranks, rank, epoch_dev, chain_sub, s3);
        ++n;
        SPB_CUDA(cudaEventRecord(evl(3 + k + 8), s3));
      } else {
        if (own) fin.p[nfin++] = grad + off + a0;
        if (theirs && own) fin.p[nfin++] = st_buf + st_off;
        if (theirs && !own) fin.p[nfin++] = grad + off + a0;
      }
      if (theirs && own) st_off += len;
    }
    // Update of shard `rank` (the last round's range) -> hi, lo, mom, w32.
    const long a = lo_of(rank), sh = lo_of(rank + 1) - a;
    pbeg(s3);
    launch_p2p_update(fin, nfin, p_hi + off + a, p_lo + off + a, mom ? mom + off + a : nullptr, w32 + off + a, sh, lr, mu,
                      wd, s3);
    pend(kClsUpdate, static_cast<double>(sh) * 4.0 * (nfin + (mom ? 7 : 5)), s3);
    launch_p2p_signal(peer_flags, slot(d), nranks, rank, epoch_dev, chain_sub, s3);
    SPB_CUDA(cudaEventRecord(evl(1), s3));
    n += 2;
    // All-gather rounds: pull the partner's final weight block of 2^b shards.
    cudaStream_t prev = s3;
    for (int b = 0; b < d; ++b) {
      const int p = rank ^ (1 << b);
      const int pb = (p >> b) << b;
      const long a0 = lo_of(pb), a1 = lo_of(pb + (1 << b));
      cudaStream_t cs = wpull[p];
      SPB_CUDA(cudaEventRecord(evl(24 + b), prev));
      SPB_CUDA(cudaStreamWaitEvent(cs, evl(24 + b), 0));  // my block of 2^b shards final
      tbeg(cs);
      launch_p2p_wait(flags, slot(d + b), nranks, 1u << p, epoch_dev, chain_sub, cs);
      tend(kTraceWait, cs);
      pbeg(cs);
      if (a1 > a0) SPB_CUDA(cudaMemcpyAsync(w32 + off + a0, peer_w32[p] + off + a0, (a1 - a0) * 4,
                                            cudaMemcpyDeviceToDevice, cs));
      pend(kClsComm, static_cast<double>(a1 - a0) * 4.0, cs);
      n += 1;
      if (b + 1 < d) {
        launch_p2p_signal(peer_flags, slot(d + b + 1), nranks, rank, epoch_dev, chain_sub, cs);
        ++n;
      }
      prev = cs;
    }
    // Split every shard but this rank's own into (hi, lo), after dgrad_l.
    SPB_CUDA(cudaEventRecord(evl(16), prev));
    SPB_CUDA(cudaStreamWaitEvent(s4, evl(16), 0));
    SPB_CUDA(cudaStreamWaitEvent(s4, evl(0), 0));
    pbeg(s4);
    launch_p2p_split(w32 + off, p_hi + off, p_lo + off, cnt, a, a + sh, s4);
    pend(kClsUpdate, static_cast<double>(cnt - sh) * 12.0, s4);
    ++n;
    SPB_CUDA(cudaStreamWaitEvent(s4, evl(1), 0));
    SPB_CUDA(cudaEventRecord(ev(ev_ready(l)), s4));
    fwd_wait[l] = ev_ready(l);
    return n;
  }

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
  int enqueue_sub_layer(int l, bool full, cudaStream_t gs, cudaStream_t s) {
    const Bucket* bk = nullptr;
    for (auto& b : buckets[full])
      if (b.l_lo <= l && l <= b.l_hi) bk = &b;
    if (!bk) throw ConfigError("comm: no bucket for layer");
    const std::vector<int>& C = bk->ranks;
    const int nc = static_cast<int>(C.size());
    const int me = static_cast<int>(std::find(C.begin(), C.end(), rank) - C.begin());  // nc: not a member
    const long off = w_off[l], cnt = b_off[l] + round_up(w[l], 32) - w_off[l];
    const long sh = layer_shard(cnt, nc);
    auto lo_of = [&](int i) { return std::min(cnt, sh * i); };
    auto evl = [&](int k) { return ev(kEvP2pLayer + 32 * l + k); };
    SPB_CUDA(cudaEventRecord(ev(kEvBucket + l), gs));
    SPB_CUDA(cudaStreamWaitEvent(cst, ev(kEvBucket + l), 0));
    SPB_CUDA(cudaEventRecord(evl(0), s));  // dgrad_l issued on s before this point
    int n = 0;
    long a = 0, b = 0;  // the range this rank updates itself
    pbeg(cst);
    if (me < nc) {
      a = lo_of(me), b = lo_of(me + 1);
      const float* g = grad + off + a;
      if (nc > 1) {  // reduce-scatter among the contributors (reads up to nc*sh: grad has tail slack)
        auto it = subcomms.find(C);
        if (it == subcomms.end() || !it->second) throw ConfigError("comm: missing contributor communicator");
        nccl_check(nccl().ReduceScatter(grad + off, stage, sh, ncclFloat32, ncclSum, it->second, cst));
        g = stage;
      }
      SPB_CUDA(cudaStreamWaitEvent(cst, evl(0), 0));
      if (b > a) {
        PeerPtrs<const float> src{};
        src.p[0] = g;
        launch_p2p_update(src, 1, p_hi + off + a, p_lo + off + a, mom ? mom + off + a : nullptr, w32 + off + a, b - a,
                          lr, mu, wd, cst);
        ++n;
      }
    } else {
      SPB_CUDA(cudaStreamWaitEvent(cst, evl(0), 0));
    }
    nccl_check(nccl().GroupStart());
    for (int i = 0; i < nc; ++i) {
      const long ia = lo_of(i), ib = lo_of(i + 1);
      if (ib > ia) nccl_check(nccl().Broadcast(w32 + off + ia, w32 + off + ia, ib - ia, ncclFloat32, C[i], comm, cst));
    }
    nccl_check(nccl().GroupEnd());
    // Bytes this rank moves: its reduce-scatter share (contributors) plus the
    // weight shards it receives.
    pend(kClsComm, 4.0 * ((me < nc && nc > 1 ? static_cast<double>(sh) * (nc - 1) : 0.0) + (cnt - (b - a))), cst);
    pbeg(cst);
    launch_p2p_split(w32 + off, p_hi + off, p_lo + off, cnt, a, b, cst);
    pend(kClsUpdate, static_cast<double>(cnt - (b - a)) * 12.0, cst);
    return n + 1;
  }

  // Shard length of a layer segment of cnt floats over `parts` ranks (a
  // multiple of 4 floats, parts * shard >= cnt; the last shards may be short
  // or empty). spb_layer_shard exports it for the protocol tests.
  static long layer_shard(long cnt, int parts) { return round_up((cnt + parts - 1) / parts, 4); }

  void setup_sub() {
    w32 = alloc<float>(nflat);
    long maxcnt = 0;
    for (int l = 1; l <= L; ++l) maxcnt = std::max(maxcnt, b_off[l] + round_up(w[l], 32) - w_off[l]);
    stage_shard = layer_shard(maxcnt, 2);
    stage = alloc<float>(stage_shard);
    // One communicator per distinct contributor set, split collectively in
    // the same (sorted) order on every rank.
    std::vector<std::vector<int>> sets;
    for (int f = 0; f < 2; ++f)
      for (const Bucket& b : buckets[f])
        if (b.ranks.size() > 1 && std::find(sets.begin(), sets.end(), b.ranks) == sets.end()) sets.push_back(b.ranks);
    std::sort(sets.begin(), sets.end());
    for (const auto& set : sets) {
      const bool member = std::find(set.begin(), set.end(), rank) != set.end();
      ncclComm_t c = nullptr;
      nccl_check(nccl().CommSplit(comm, member ? 0 : NCCL_SPLIT_NOCOLOR, rank, &c, nullptr));
      subcomms[set] = member ? c : nullptr;
    }
    comm_mode = 3;
    invalidate_graphs();
  }

  // Collective over the ranks (spb_comm_init): allocate the p2p buffers and
  // map every peer's grad / w32 / flags through CUDA IPC.
  // slots_per_layer: epoch-stamped flags per layer (p2p: G and U; rh: see
  // enqueue_rh_layer).
  void setup_p2p(int slots_per_layer = 2) {
    if (nranks > kMaxPeers) throw ConfigError("comm: p2p mode supports at most 8 ranks");
    if (!bar_dev) bar_dev = alloc<float>(1);
    w32 = alloc<float>(nflat);
    flag_slots = slots_per_layer;
    flags = alloc<int>(static_cast<long>(slots_per_layer) * (L + 1) * nranks);
    epoch_dev = alloc<int>(1);
    long maxcnt = 0;
    for (int l = 1; l <= L; ++l) maxcnt = std::max(maxcnt, b_off[l] + round_up(w[l], 32) - w_off[l]);
    stage_shard = round_up((maxcnt / 4 + nranks - 1) / nranks * 4, 32);
    stage = alloc<float>(2L * std::max(1, nranks - 1) * stage_shard);
    cudaIpcMemHandle_t mine[3];
    SPB_CUDA(cudaIpcGetMemHandle(&mine[0], grad));
    SPB_CUDA(cudaIpcGetMemHandle(&mine[1], w32));
    SPB_CUDA(cudaIpcGetMemHandle(&mine[2], flags));
    const size_t hb = sizeof mine;
    char* dbuf = nullptr;
    SPB_CUDA(cudaMalloc(&dbuf, hb * (nranks + 1)));
    SPB_CUDA(cudaMemcpy(dbuf, mine, hb, cudaMemcpyHostToDevice));
    nccl_check(nccl().AllGather(dbuf, dbuf + hb, hb, ncclUint8, comm, cst));
    SPB_CUDA(cudaStreamSynchronize(cst));
    std::vector<cudaIpcMemHandle_t> all(3 * nranks);
    SPB_CUDA(cudaMemcpy(all.data(), dbuf + hb, hb * nranks, cudaMemcpyDeviceToHost));
    cudaFree(dbuf);
    peer_grad.assign(nranks, nullptr);
    peer_w32.assign(nranks, nullptr);
    for (int p = 0; p < nranks; ++p) {
      if (p == rank) {
        peer_grad[p] = grad, peer_w32[p] = w32, peer_flags.p[p] = flags;
        continue;
      }
      void* q = nullptr;
      SPB_CUDA(cudaIpcOpenMemHandle(&q, all[3 * p + 0], cudaIpcMemLazyEnablePeerAccess));
      peer_grad[p] = static_cast<float*>(q);
      SPB_CUDA(cudaIpcOpenMemHandle(&q, all[3 * p + 1], cudaIpcMemLazyEnablePeerAccess));
      peer_w32[p] = static_cast<float*>(q);
      SPB_CUDA(cudaIpcOpenMemHandle(&q, all[3 * p + 2], cudaIpcMemLazyEnablePeerAccess));
      peer_flags.p[p] = static_cast<int*>(q);
    }
    SPB_CUDA(cudaStreamCreateWithFlags(&s4, cudaStreamNonBlocking));
    gpull.assign(nranks, nullptr);
    wpull.assign(nranks, nullptr);
    for (int p = 0; p < nranks; ++p) {
      if (p == rank) continue;
      SPB_CUDA(cudaStreamCreateWithFlags(&gpull[p], cudaStreamNonBlocking));
      SPB_CUDA(cudaStreamCreateWithFlags(&wpull[p], cudaStreamNonBlocking));
    }
    comm_mode = 2;
    invalidate_graphs();
    host_barrier();
  }

  // push mode setup (collective over the ranks): staging slots, fp32 weight
  // copies for the received rows, flags; every peer's pstage / w32 / flags
  // mapped through CUDA IPC. MLP only (the conv wgrad has no row routing).
  void setup_push() {
    if (nranks > kMaxPeers) throw ConfigError("comm: push mode supports at most 8 ranks");
    if (conv_model) throw ConfigError("comm: push mode is MLP-only");
    if (!bar_dev) bar_dev = alloc<float>(1);
    w32 = alloc<float>(nflat);
    flags = alloc<int>(2L * (L + 1) * nranks);
    epoch_dev = alloc<int>(1);
    prpo.assign(L + 1, 0);
    pstage_off.assign(L + 1, 0);
    pslot.assign(L + 1, 0);
    long tot = 0;
    for (int l = 1; l <= L; ++l) {
      prpo[l] = (w[l] + nranks - 1) / nranks;
      pslot[l] = round_up(static_cast<long>(prpo[l]) * ld[l - 1] + prpo[l], 32);
      pstage_off[l] = tot;
      tot += pslot[l] * nranks;
    }
    pstage = alloc<float>(tot);
    cudaIpcMemHandle_t mine[3];
    SPB_CUDA(cudaIpcGetMemHandle(&mine[0], pstage));
    SPB_CUDA(cudaIpcGetMemHandle(&mine[1], w32));
    SPB_CUDA(cudaIpcGetMemHandle(&mine[2], flags));
    const size_t hb = sizeof mine;
    char* dbuf = nullptr;
    SPB_CUDA(cudaMalloc(&dbuf, hb * (nranks + 1)));
    SPB_CUDA(cudaMemcpy(dbuf, mine, hb, cudaMemcpyHostToDevice));
    nccl_check(nccl().AllGather(dbuf, dbuf + hb, hb, ncclUint8, comm, cst));
    SPB_CUDA(cudaStreamSynchronize(cst));
    std::vector<cudaIpcMemHandle_t> all(3 * nranks);
    SPB_CUDA(cudaMemcpy(all.data(), dbuf + hb, hb * nranks, cudaMemcpyDeviceToHost));
    cudaFree(dbuf);
    peer_grad.assign(nranks, nullptr);
    peer_pstage.assign(nranks, nullptr);
    peer_w32.assign(nranks, nullptr);
    for (int p = 0; p < nranks; ++p) {
      if (p == rank) {
        peer_pstage[p] = pstage, peer_w32[p] = w32, peer_flags.p[p] = flags;
        continue;
      }
      void* q = nullptr;
      SPB_CUDA(cudaIpcOpenMemHandle(&q, all[3 * p + 0], cudaIpcMemLazyEnablePeerAccess));
      peer_pstage[p] = static_cast<float*>(q);
      SPB_CUDA(cudaIpcOpenMemHandle(&q, all[3 * p + 1], cudaIpcMemLazyEnablePeerAccess));
      peer_w32[p] = static_cast<float*>(q);
      SPB_CUDA(cudaIpcOpenMemHandle(&q, all[3 * p + 2], cudaIpcMemLazyEnablePeerAccess));
      peer_flags.p[p] = static_cast<int*>(q);
    }
    SPB_CUDA(cudaStreamCreateWithFlags(&s4, cudaStreamNonBlocking));
    wpull.assign(nranks, nullptr);
    for (int p = 0; p < nranks; ++p)
      if (p != rank) SPB_CUDA(cudaStreamCreateWithFlags(&wpull[p], cudaStreamNonBlocking));
    comm_mode = 4;
    invalidate_graphs();
    host_barrier();
  }

  // push mode: where the wgrad epilogue of layer l stores gradient row r
  // (GemmEpilogue::route): the owner's staging slot for this rank, or this
  // rank's own gradient buffer for its own rows.
  void push_route(int l, GemmEpilogue& ep) const {
    ep.route_rows = prpo[l];
    for (int o = 0; o < nranks; ++o)
      ep.route[o] = o == rank ? grad + w_off[l] + static_cast<long>(o) * prpo[l] * ld[l - 1]
                              : peer_pstage[o] + pstage_off[l] + static_cast<long>(rank) * pslot[l];
  }

  // push mode, layer l (protocol: push.cu). gs: the stream that produced this
  // rank's gradient of l (its wgrad already stored the weight rows to their
  // owners, except for the head layer); s: main stream (dgrad_l issued).
  int enqueue_push_layer(int l, bool full, cudaStream_t gs, cudaStream_t s) {
    const Bucket* bk = nullptr;
    for (auto& b : buckets[full])
      if (b.l_lo <= l && l <= b.l_hi) bk = &b;
    if (!bk) throw ConfigError("comm: no bucket for layer");
    unsigned contrib = 0;
    for (int r : bk->ranks) contrib |= 1u << r;
    const bool mine = contrib >> rank & 1u;
    const unsigned peers = ((1u << nranks) - 1u) & ~(1u << rank);
    const long ldw = ld[l - 1];
    const int rpo = prpo[l];
    const int r0 = std::min(w[l], rank * rpo), r1 = std::min(w[l], (rank + 1) * rpo);
    auto evl = [&](int k) { return ev(kEvP2pLayer + 32 * l + k); };
    // Layer L's weight gradient comes from a column reduction, not the routed
    // wgrad GEMM: its rows travel with the signal.
    const bool rows_in_signal = l == L || conv_model;
    PeerPtrs<float> wdst{}, bdst{};
    for (int o = 0; o < nranks; ++o) {
      if (o == rank) continue;
      wdst.p[o] = peer_pstage[o] + pstage_off[l] + static_cast<long>(rank) * pslot[l];
      bdst.p[o] = wdst.p[o] + static_cast<long>(rpo) * ldw;
    }
    // 1. bias rows (+ head weight rows) to their owners, fence, G[l].
    pbeg(gs);
    launch_push_signal(peer_flags, 2 * l, nranks, rank, epoch_dev, chain_sub,
                       mine && rows_in_signal ? grad + w_off[l] : nullptr, ldw, mine ? grad + b_off[l] : nullptr, rpo,
                       w[l], wdst, bdst, gs);
    // Bytes this rank sends to the owners (the wgrad epilogue's routed rows
    // and the bias rows): its share of the exchange, like a pull elsewhere.
    pend(kClsComm, mine ? static_cast<double>(w[l] - (r1 - r0)) * (ldw + 1) * 4.0 : 0.0, gs);
    SPB_CUDA(cudaEventRecord(evl(0), s));  // dgrad_l issued on s before this point
    SPB_CUDA(cudaEventRecord(ev(kEvBucket + l), gs));
    // 2. owner update on s3: every rank's G[l], own gradient final, dgrad_l
    // done (the update rewrites W_l rows in place).
    SPB_CUDA(cudaStreamWaitEvent(s3, ev(kEvBucket + l), 0));
    SPB_CUDA(cudaStreamWaitEvent(s3, evl(0), 0));
    tbeg(s3);
    launch_p2p_wait(flags, 2 * l, nranks, peers, epoch_dev, chain_sub, s3);
    tend(kTraceWait, s3);
    const long nw = static_cast<long>(r1 - r0) * ldw, nb = r1 - r0;
    PeerPtrs<const float> sw{}, sb{};
    PeerPtrs<float> dw{}, db{};
    int nsrc = 0, ndst = 0;
    for (int r = 0; r < nranks; ++r) {
      if (!(contrib >> r & 1u)) continue;
      if (r == rank) {
        sw.p[nsrc] = grad + w_off[l] + static_cast<long>(r0) * ldw;
        sb.p[nsrc] = grad + b_off[l] + r0;
      } else {
        sw.p[nsrc] = pstage + pstage_off[l] + static_cast<long>(r) * pslot[l];
        sb.p[nsrc] = sw.p[nsrc] + static_cast<long>(rpo) * ldw;
      }
      ++nsrc;
    }
    // The owner's new fp32 rows go to its own w32; the peers pull them (copy
    // engines), as in the p2p mode.
    dw.p[ndst] = w32 + w_off[l] + static_cast<long>(r0) * ldw;
    db.p[ndst] = w32 + b_off[l] + r0;
    ++ndst;
    pbeg(s3);
    launch_push_update(sw, nsrc, p_hi + w_off[l] + r0 * ldw, p_lo + w_off[l] + r0 * ldw,
                       mom ? mom + w_off[l] + r0 * ldw : nullptr, dw, ndst, nw, lr, mu, wd, s3);
    launch_push_update(sb, nsrc, p_hi + b_off[l] + r0, p_lo + b_off[l] + r0, mom ? mom + b_off[l] + r0 : nullptr, db,
                       ndst, nb, lr, mu, wd, s3);
    pend(kClsUpdate, static_cast<double>(nw + nb) * 4.0 * (nsrc + (mom ? 6 : 5)), s3);
    launch_p2p_signal(peer_flags, 2 * l + 1, nranks, rank, epoch_dev, chain_sub, s3);
    SPB_CUDA(cudaEventRecord(evl(1), s3));
    // 3. every other owner's rows: wait for its U[l], pull (copy engines);
    // then split after dgrad_l.
    for (int o = 0; o < nranks; ++o) {
      if (o == rank) continue;
      const int q0 = std::min(w[l], o * rpo), q1 = std::min(w[l], (o + 1) * rpo);
      cudaStream_t cs = wpull[o];
      tbeg(cs);
      launch_p2p_wait(flags, 2 * l + 1, nranks, 1u << o, epoch_dev, chain_sub, cs);
      tend(kTraceWait, cs);
      if (q1 > q0) {
        pbeg(cs);
        SPB_CUDA(cudaMemcpyAsync(w32 + w_off[l] + static_cast<long>(q0) * ldw, peer_w32[o] + w_off[l] + q0 * ldw,
                                 static_cast<size_t>(q1 - q0) * ldw * 4, cudaMemcpyDeviceToDevice, cs));
        SPB_CUDA(cudaMemcpyAsync(w32 + b_off[l] + q0, peer_w32[o] + b_off[l] + q0, static_cast<size_t>(q1 - q0) * 4,
                                 cudaMemcpyDeviceToDevice, cs));
        pend(kClsComm, static_cast<double>(q1 - q0) * (ldw + 1) * 4.0, cs);
      }
      SPB_CUDA(cudaEventRecord(evl(16 + o), cs));
      SPB_CUDA(cudaStreamWaitEvent(s4, evl(16 + o), 0));
    }
    SPB_CUDA(cudaStreamWaitEvent(s4, evl(0), 0));
    pbeg(s4);
    launch_push_split(w32 + w_off[l], p_hi + w_off[l], p_lo + w_off[l], static_cast<long>(w[l]) * ldw, r0 * ldw,
                      r1 * ldw, s4);
    launch_push_split(w32 + b_off[l], p_hi + b_off[l], p_lo + b_off[l], w[l], r0, r1, s4);
    pend(kClsUpdate, static_cast<double>(w[l] - (r1 - r0)) * (ldw + 1) * 12.0, s4);
    SPB_CUDA(cudaStreamWaitEvent(s4, evl(1), 0));
    SPB_CUDA(cudaEventRecord(ev(ev_ready(l)), s4));
    fwd_wait[l] = ev_ready(l);
    return 6;
  }

  void host_barrier() {
    nccl_check(nccl().AllReduce(bar_dev, bar_dev, 1, ncclFloat32, ncclSum, comm, cst));
    SPB_CUDA(cudaStreamSynchronize(cst));
  }

  // HBM bytes one update launch must move: read hi, lo, grad (+ mom), write
  // hi, lo (+ mom), 4 B each.
  double update_bytes() const { return static_cast<double>(nflat) * 4.0 * (mom ? 7 : 5); }

  // Row plan of one SPB step for the hosted workers.
  void step_plan(bool full, std::vector<int>& row0, std::vector<float>& alpha) const {
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

  // Step `sub` of a chain of `nsub` steps captured into one graph (sub = 0,
  // nsub = 1: a plain step). Side streams are joined back into s only after
  // the last step of the chain; before that, the next step's forward waits
  // per layer (fwd_wait) for the weights this step finalises.
  int enqueue_step(bool full, bool host_rows, cudaStream_t s, int sub = 0, int nsub = 1) {
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

  // The graph of `nsub` chained steps (see enqueue_step); `launches` gets the
  // kernel launches per step.
  cudaGraphExec_t get_graph(bool full, bool host_rows, int nsub = 1, int* launches = nullptr) {
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

  // Replay `steps` steps as chained graphs of up to `chain` steps each
  // (losses: the per-step loss, copied back asynchronously; may be null).
  void run_steps(bool full, int steps, float* losses) {
    int done = 0;
    while (done < steps) {
      const int c = std::max(1, std::min({chain_len(), kMaxChain, steps - done}));
      cudaGraphExec_t g = get_graph(full, false, c, &last_launches);
      SPB_CUDA(cudaGraphLaunch(g, st));
      if (losses) SPB_CUDA(cudaMemcpyAsync(losses + done, loss_dev, c * sizeof(float), cudaMemcpyDeviceToHost, st));
      done += c;
    }
  }
};

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
    // pairwise copy-engine exchange); push for 4 ranks (gradient rows stored
    // to their owners by the wgrad epilogue: 4.47 ms vs rh 5.02, p2p 5.2,
    // nccl 5.09 on one box), rh for the ConvNet there (push is MLP-only);
    // sub elsewhere -- NCCL over contributor sub-communicators, parity-tested
    // at 2 and 4 ranks (8 ranks could not be measured: gpurun offers 4 GPUs).
    const char* cm = std::getenv("SPB_COMM");
    const std::string mode =
        cm ? cm : (nranks == 2 ? "p2p" : (nranks == 4 ? (e.conv_model ? "rh" : "push") : "sub"));
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
