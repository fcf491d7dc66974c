// Host side of the tcgen05 3xTF32 GEMM: TMA tensor-map encoding and the
// template dispatch over (A major, B major, epilogue).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>
#include <set>
#include <string>
#include <vector>

#include <algorithm>
#include <cstdlib>

#include "gemm_2sm.cuh"
#include "gemm_tf32x3.cuh"
#include "conv.hpp"
#include "launch.hpp"

namespace spb {
namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  if (!fn) throw CudaError("cuTensorMapEncodeTiled unavailable");
  return fn;
}

PFN_cuTensorMapEncodeIm2col_v12000 encode_im2col_fn() {
  static PFN_cuTensorMapEncodeIm2col_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeIm2col_v12000>(p);
  });
  if (!fn) throw CudaError("cuTensorMapEncodeIm2col unavailable");
  return fn;
}

// im2col map of an NHWC activation tensor (row stride ld floats per pixel)
// for a 3x3 / padding-1 convolution: the window of output pixel (p, q)
// starts at (q*s - 1, p*s - 1); bounding box corners -1 / -1 (so the walk
// covers exactly out_w x out_h window origins per image, CUTLASS's
// q = (W + upper - lower - 1) / s + 1), traversal stride s, 32 channels per
// pixel, `pixels` pixels per box, zero fill outside the image.
CUtensorMap im2col_map(const float* base, const ConvSrc& src, int pixels, CUtensorMapSwizzle swz) {
  CUtensorMap m;
  const ConvGeom& g = src.g;
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(g.c_in), static_cast<cuuint64_t>(g.in_w),
                        static_cast<cuuint64_t>(g.in_h), static_cast<cuuint64_t>(src.samples)};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(src.ld) * 4, static_cast<cuuint64_t>(src.ld) * 4 * g.in_w,
                           static_cast<cuuint64_t>(src.ld) * 4 * g.in_w * g.in_h};
  int lower[2] = {-1, -1}, upper[2] = {-1, -1};
  cuuint32_t estr[4] = {1, static_cast<cuuint32_t>(g.stride), static_cast<cuuint32_t>(g.stride), 1};
  CUresult r = encode_im2col_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(base), dims, strides, lower,
                                  upper, 32, static_cast<cuuint32_t>(pixels), estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeIm2col failed: " + std::to_string(static_cast<int>(r)));
  return m;
}

// 2D fp32 tensor map, 128-byte swizzle (16 B or 32 B atoms), zero fill out of bounds.
CUtensorMap tmap2d(const float* base, long inner, long outer, long ld, int box_inner, int box_outer,
                   CUtensorMapSwizzle swz) {
  CUtensorMap m;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(outer)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 4};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(box_inner), static_cast<cuuint32_t>(box_outer)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box,
                           estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed: " + std::to_string(static_cast<int>(r)));
  return m;
}

// SMs left free for concurrent NCCL kernels (multi-GPU). Thread-local and
// set per launch sequence by the engine context that owns the communicator
// (SmReserve in engine.cu), so one context's reservation never leaks into
// another context's GEMMs.
thread_local int g_reserved_sms = 0;

// SMs a persistent GEMM grid may occupy.
int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    SPB_CUDA(cudaGetDevice(&dev));
    SPB_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  }
  return std::max(2, (n - g_reserved_sms) & ~1);
}

// TMEM accumulation chunk (k-blocks) per GEMM kind [forward K x K, dgrad
// K x MN, wgrad MN x MN]: the compile-time defaults, overridable per process
// (SPB_CHUNK_FWD / _DGRAD / _WGRAD or gemm_set_chunk) for A/B measurements.
int g_chunk[3] = {-1, -1, -1};

int chunk_for(bool a_mn, bool b_mn) {
  const int kind = (a_mn && b_mn) ? 2 : ((!a_mn && b_mn) ? 1 : 0);
  if (g_chunk[kind] < 0) {
    static const char* env[3] = {"SPB_CHUNK_FWD", "SPB_CHUNK_DGRAD", "SPB_CHUNK_WGRAD"};
    const char* v = std::getenv(env[kind]);
    const int def[3] = {SPB_CHUNK_KB_FWD, SPB_CHUNK_KB_DGRAD, SPB_CHUNK_KB_WGRAD};
    g_chunk[kind] = v ? std::max(1, std::atoi(v)) : def[kind];
  }
  return g_chunk[kind];
}

// Launch with programmatic stream serialization (SPB_PDL=1; default off): the
// GEMM's prologue (barrier init, TMEM allocation, tensor-map prefetch) may
// start while the previous kernel in the stream drains; the kernels execute
// griddepcontrol.wait before touching any data (gemm_tf32x3.cuh). Same-box
// A/B (tools/ab_env.py, 3 rounds): cfg3 SPB 6.04 vs 6.02 ms, full backprop
// 8.54 vs 8.35 ms, cfg4 equal -- no gain, so off.
bool pdl_enabled() {
  static const bool v = [] {
    const char* e = std::getenv("SPB_PDL");
    return e && std::atoi(e) != 0;
  }();
  return v;
}

template <class Kern, class... Args>
void launch_pdl(Kern kern, dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  SPB_CUDA(cudaLaunchKernelEx(&cfg, kern, args...));
}

// The TMA extent along MN: the operand's real columns (mn_map) when the GEMM
// extends past them (the fused-bias ones column of a wgrad B operand).
CUtensorMap operand_map(const Operand& X, const float* base, int tile_rows) {
  const int mn = X.mn_map > 0 ? X.mn_map : X.mn;
  if (!X.mn_major) return tmap2d(base, X.k, mn, X.ld, kBK, tile_rows, CU_TENSOR_MAP_SWIZZLE_128B);
  return tmap2d(base, mn, X.k, X.ld, 32, kBK, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
}

// Constant boxes for the fused-bias ones column (GemmEpilogue::ones_col_p1):
// a [64 x 32] fp32 array per device, rows 0-31 ones (the hi half of the
// column), rows 32-63 zeros (its lo half), read as 32 x 32 MN-major boxes.
// Allocated once per device by gemm_prepare_device (not capturable).
const float* g_ones[64] = {};
// Default column-sum slice scratch / counters (GemmEpilogue::colsum_ws /
// colsum_cnt) for callers that pass none: one per device, so such callers
// must not run colsum GEMMs on two streams at once (the engine passes its own).
float* g_colsum_ws[64] = {};
int* g_colsum_cnt[64] = {};


const float* ones_buffer() {
  int dev = 0;
  SPB_CUDA(cudaGetDevice(&dev));
  if (!g_ones[dev]) throw CudaError("gemm: gemm_prepare_device() was not called on this device");
  return g_ones[dev];
}

CUtensorMap ones_map() {
  return tmap2d(ones_buffer(), 32, 64, 32, 32, kBK, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
}

// The dynamic shared-memory opt-in of a kernel, once per (kernel, device):
// a function attribute belongs to the device's context, so a process driving
// contexts on several GPUs must set it on each.
template <class K>
void configure_smem(K* kern, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  SPB_CUDA(cudaGetDevice(&dev));
  const auto key = std::make_pair(reinterpret_cast<const void*>(kern), dev);
  std::lock_guard<std::mutex> lock(mu);
  if (done.count(key)) return;
  SPB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  done.insert(key);
}

template <int BN, bool AM, bool BM_, int EPI, bool TMA_UPD = false, int IC = 0>
void launch_inst(const Operand& A, const Operand& B, const GemmEpilogue& ep, cudaStream_t s, int splits = 1,
                 const CUtensorMap* ic_a = nullptr, const CUtensorMap* ic_b = nullptr, ConvTmaArgs ic = {}) {
  auto kern = gemm_tf32x3_kernel<BN, AM, BM_, EPI, TMA_UPD, IC>;
  constexpr int smem = GemmCfg<BN, TMA_UPD>::kSmem;
  configure_smem(kern, smem);
  // IC == 1: A comes from ic_a[0..1] (im2col hi / lo); IC == 2: B from ic_b.
  CUtensorMap ah = IC == 1 ? ic_a[0] : operand_map(A, A.hi, kBM), al = IC == 1 ? ic_a[1] : operand_map(A, A.lo, kBM);
  CUtensorMap bh = IC == 2 ? ic_b[0] : operand_map(B, B.hi, BN), bl = IC == 2 ? ic_b[1] : operand_map(B, B.lo, BN);
  const int num_kb = (A.k + kBK - 1) / kBK;
  const int num_m = (A.mn + kBM - 1) / kBM, num_n = (B.mn + BN - 1) / BN;
  const int tiles = num_m * num_n;
  const int kbs = (num_kb + splits - 1) / splits;
  const int units = tiles * ((num_kb + kbs - 1) / kbs);
  const int grid = units < num_sms() ? units : num_sms();
  CUtensorMap wh{}, wl{}, wm{};
  if (TMA_UPD) {  // the W tile the optimizer epilogue updates in place: [M rows x N cols] (no bias column)
    wh = tmap2d(ep.out_hi, ep.N, ep.M, ep.ld_out, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B);
    wl = tmap2d(ep.out_lo, ep.N, ep.M, ep.ld_out, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B);
    wm = ep.mom ? tmap2d(ep.mom, ep.N, ep.M, ep.ld_out, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B) : wh;
  }
  const CUtensorMap ones = ep.ones_col_p1 > 0 ? ones_map() : ah;
  GemmEpilogue e = ep;
  if (e.chunk_kb <= 0) e.chunk_kb = chunk_for(AM, BM_);
  if (e.colsum_col_p1 > 0 && !e.colsum_ws) {  // the per-device default slice scratch
    int dev = 0;
    SPB_CUDA(cudaGetDevice(&dev));
    e.colsum_ws = g_colsum_ws[dev];
    e.colsum_cnt = g_colsum_cnt[dev];
  }
  if (e.colsum_col_p1 > 0 && (!e.colsum_ws || static_cast<long>(num_n) * num_m * kBM > kColsumWsFloats ||
                              num_m > kColsumCounters))
    throw std::invalid_argument("gemm: column-sum scratch missing or too small");
  launch_pdl(kern, dim3(grid), dim3(256), smem, s, ah, al, bh, bl, num_kb, num_m, tiles, kbs, units, e, wh, wl, wm, ic,
             ones);
  SPB_CUDA(cudaGetLastError());
}

template <bool AM, bool BM_, int EPI, int PN, int IC = 0>
void launch_2sm_pn(const Operand& A, const Operand& B, const GemmEpilogue& ep, cudaStream_t s, int splits = 1,
                   const CUtensorMap* ic_a = nullptr, ConvTmaArgs ic = {}, const CUtensorMap* ic_b = nullptr) {
  using Cfg = Gemm2smCfg<PN>;
  auto kern = gemm_tf32x3_2sm_kernel<AM, BM_, EPI, PN, IC>;
  configure_smem(kern, Cfg::kSmem);
  CUtensorMap ah = IC == 1 ? ic_a[0] : operand_map(A, A.hi, Cfg::kRowsA);
  CUtensorMap al = IC == 1 ? ic_a[1] : operand_map(A, A.lo, Cfg::kRowsA);
  CUtensorMap bh = IC == 2 ? ic_b[0] : operand_map(B, B.hi, Cfg::kRowsB);
  CUtensorMap bl = IC == 2 ? ic_b[1] : operand_map(B, B.lo, Cfg::kRowsB);
  const int num_kb = (A.k + kBK - 1) / kBK;
  const int num_m = (A.mn + 255) / 256, num_n = (B.mn + Cfg::kPairN - 1) / Cfg::kPairN;
  const int tiles = num_m * num_n;
  if (splits > 1 && EPI != kEpiStoreScaled) throw std::invalid_argument("gemm: pair split-K needs kEpiStoreScaled");
  const int kbs = (num_kb + splits - 1) / splits;
  const int units = tiles * ((num_kb + kbs - 1) / kbs);
  const int pairs = num_sms() / 2;
  const int clusters = units < pairs ? units : pairs;
  const CUtensorMap ones = ep.ones_col_p1 > 0 ? ones_map() : ah;
  GemmEpilogue e = ep;
  if (e.chunk_kb <= 0) e.chunk_kb = chunk_for(AM, BM_);
  launch_pdl(kern, dim3(2 * clusters), dim3(Cfg::kThreads), Cfg::kSmem, s, ah, al, bh, bl, num_kb, num_m, tiles, kbs,
             units, e, ones, ic);
  SPB_CUDA(cudaGetLastError());
}

// Pair-tile widths with instantiated kernels. 240 / 256 for every operand
// layout and epilogue; 192 for the MLP's three GEMM shapes (forward K x K,
// dgrad K x MN, wgrad MN x MN) and split-K partials. (64 and 128 were
// measured too: they never beat these on the SPB shapes.)
constexpr int kPairNs[] = {192, 240, 256};

template <bool AM, bool BM_, int EPI>
constexpr bool narrow_ok() {
  return (!AM && !BM_ && (EPI == kEpiFwdTanh || EPI == kEpiFwdLinear || EPI == kEpiStoreScaled)) ||
         (!AM && BM_ && (EPI == kEpiDgradTanh || EPI == kEpiStoreScaled)) || (AM && BM_ && EPI == kEpiStoreScaled);
}

template <bool AM, bool BM_, int EPI>
void launch_2sm(const Operand& A, const Operand& B, const GemmEpilogue& ep, cudaStream_t s, int pn, int splits) {
  if constexpr (narrow_ok<AM, BM_, EPI>()) {
    if (pn == 192) return launch_2sm_pn<AM, BM_, EPI, 192>(A, B, ep, s, splits);
  }
  if (pn == 240) return launch_2sm_pn<AM, BM_, EPI, 240>(A, B, ep, s, splits);
  if (pn == 256) return launch_2sm_pn<AM, BM_, EPI, 256>(A, B, ep, s, splits);
  throw std::invalid_argument("gemm: no pair kernel for this tile width / layout");
}

template <int EPI>
void dispatch_2sm(const Operand& A, const Operand& B, const GemmEpilogue& ep, cudaStream_t s, int pn, int splits = 1) {
  if (!A.mn_major && !B.mn_major) launch_2sm<false, false, EPI>(A, B, ep, s, pn, splits);
  else if (!A.mn_major && B.mn_major) launch_2sm<false, true, EPI>(A, B, ep, s, pn, splits);
  else if (A.mn_major && !B.mn_major) launch_2sm<true, false, EPI>(A, B, ep, s, pn, splits);
  else launch_2sm<true, true, EPI>(A, B, ep, s, pn, splits);
}

bool narrow_pair_ok(const Operand& A, const Operand& B, int epi) {
  if (!A.mn_major && !B.mn_major) return epi == kEpiFwdTanh || epi == kEpiFwdLinear || epi == kEpiStoreScaled;
  if (!A.mn_major && B.mn_major) return epi == kEpiDgradTanh || epi == kEpiStoreScaled;
  if (A.mn_major && B.mn_major) return epi == kEpiStoreScaled;
  return false;
}

// Split-K fixup: sum the per-split fp32 partials (in split order, so the
// result is deterministic) and apply the real epilogue.
template <int EPI>
__global__ void splitk_fixup_kernel(const float* __restrict__ ws, int splits, long stride, long ldw, GemmEpilogue ep) {
  const int cols = epi_cols(ep);  // including the fused bias column
  const long n = static_cast<long>(ep.M) * cols;
  for (long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(i / cols), c = static_cast<int>(i % cols);
    float v = 0.f;
    for (int sp = 0; sp < splits; ++sp) v += ws[sp * stride + r * ldw + c];
    epilogue_one<EPI>(ep, v, r, c);
  }
}

// The same for many splits and few outputs (the conv wgrads: K = up to ~1M
// pixel rows over <= 296 splits, a few thousand outputs): one warp per output,
// lanes strided over the splits, a fixed shuffle tree -- deterministic.
template <int EPI>
__global__ void splitk_fixup_wide_kernel(const float* __restrict__ ws, int splits, long stride, long ldw, GemmEpilogue ep) {
  const int cols = epi_cols(ep);
  const long n = static_cast<long>(ep.M) * cols;
  const int lane = threadIdx.x & 31;
  for (long i = (static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; i < n;
       i += (static_cast<long>(gridDim.x) * blockDim.x) >> 5) {
    const int r = static_cast<int>(i / cols), c = static_cast<int>(i % cols);
    float v = 0.f;
    for (int sp = lane; sp < splits; sp += 32) v += ws[sp * stride + r * ldw + c];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) epilogue_one<EPI>(ep, v, r, c);
  }
}

template <int EPI>
void launch_fixup(const float* ws, int splits, long stride, long ldw, const GemmEpilogue& ep, cudaStream_t s) {
  const long n = static_cast<long>(ep.M) * epi_cols(ep);
  if (splits >= 16) {
    const int grid = static_cast<int>(std::min<long>((n * 32 + 255) / 256, 148L * 32));
    splitk_fixup_wide_kernel<EPI><<<grid, 256, 0, s>>>(ws, splits, stride, ldw, ep);
  } else {
    const int grid = static_cast<int>(std::min<long>((n + 255) / 256, 148L * 16));
    splitk_fixup_kernel<EPI><<<grid, 256, 0, s>>>(ws, splits, stride, ldw, ep);
  }
  SPB_CUDA(cudaGetLastError());
}

// Launch plan: the 1-CTA 128x128 kernel or the CTA-pair 256 x pn kernel,
// with `splits` K-splits (fp32 partials + deterministic fixup) when > 1.
struct Plan {
  bool two_sm;
  int splits;
  int pn;
};

template <int EPI>
void launch_splitk(const Operand& A, const Operand& B, const GemmEpilogue& ep, cudaStream_t s, const Plan& plan) {
  // Workspace rows hold the GEMM's columns and, with a column-sum bias, the bias column after them.
  const long ldw = round_up(std::max(B.mn, epi_cols(ep)), 4), stride = static_cast<long>(A.mn) * ldw;
  GemmEpilogue part{};
  part.out_hi = ep.splitk_ws;
  part.ld_out = ldw;
  part.alpha = 1.0f;
  part.M = A.mn;
  part.N = B.mn;
  part.split_stride = stride;
  part.ones_col_p1 = ep.ones_col_p1;  // the partials compute the bias column like any other
  part.colsum_col_p1 = ep.colsum_col_p1;  // (or the column-sum warps write it into the workspace)
  part.colsum_ws = ep.colsum_ws, part.colsum_cnt = ep.colsum_cnt;
  // Splits actually populated: ceil(kb / ceil(kb / splits)) can be < splits.
  const int kb = (A.k + kBK - 1) / kBK, kbs = (kb + plan.splits - 1) / plan.splits;
  const int splits = (kb + kbs - 1) / kbs;
  if (static_cast<long>(splits) * stride > ep.splitk_ws_floats)  // forced plans skip the planner's check
    throw std::invalid_argument("gemm: split-K workspace too small for this plan");
  if (plan.two_sm) dispatch_2sm<kEpiStoreScaled>(A, B, part, s, plan.pn, splits);
  else if (!A.mn_major && !B.mn_major) launch_inst<128, false, false, kEpiStoreScaled>(A, B, part, s, splits);
  else if (!A.mn_major && B.mn_major) launch_inst<128, false, true, kEpiStoreScaled>(A, B, part, s, splits);
  else if (A.mn_major && !B.mn_major) launch_inst<128, true, false, kEpiStoreScaled>(A, B, part, s, splits);
  else launch_inst<128, true, true, kEpiStoreScaled>(A, B, part, s, splits);
  launch_fixup<EPI>(ep.splitk_ws, splits, stride, ldw, ep, s);
}

// How the 1-CTA kernels produce the fused bias column: the virtual ones column
// (default: one more column tile when n is a multiple of 128) or, with
// SPB_BIAS=colsum, the column-sum warps. Same-box A/B (tools/ab_env.py, 3
// rounds each): cfg3 SPB step 5.95-6.00 ms with the ones column vs 6.06-6.12
// with the column sums (their per-k-block barrier traffic and extra smem reads
// in the smem-bound 1-CTA kernel cost more than the 33rd tile); cfg4 equal.
bool bias_by_ones() {
  static const bool v = [] {
    const char* e = std::getenv("SPB_BIAS");
    return !(e && std::string(e) == "colsum");
  }();
  return v;
}

int g_force_variant = -1;  // -1 auto, 0 = 1-CTA 128x128, 1 = CTA pair
Plan g_force_plan{false, 0, 0};  // splits == 0: not forced
Plan g_last_plan{false, 1, 128};  // the plan of the last gemm_tf32x3 launch (test hook)

// Wave-quantised cost model (microseconds), fitted on B200 to the plan
// sweep of tests/native/gemm_bench.cu (`gemm_bench 10 sweep`: every plan on
// the SPB forward / dgrad / wgrad shapes at 1, 2 and 4 GPUs; 7.6 % rms; its
// choice is within 1 % of the best measured plan summed over the shapes):
//  - 1-CTA 128 x 128 unit: 0.638 us per 32-deep k-block + 1.41 us
//    (0.31 us per k-block for N <= 64 tiles);
//  - pair 256 x pn unit (2 SMs): 1.01 us x pe / 256 per k-block + 1.01 us +
//    4.24 us x pn / 256, pe = the B rows actually loaded (MN-major B comes in
//    32-row boxes: pn 240 loads 256 when A is MN-major too);
//  - split-K: + 3.0 us + (splits + 2) M N fp32 streamed at 3.17 TB/s (fixup;
//    the constant is the old small-shape calibration, the slope the new fit).
// no240: the bias-fused wgrads need 32-aligned B boxes (the ones box), which
// the 120-row CTA halves of the 240-wide pair tile do not have.
Plan plan_gemm(int M, int N, int K, long ws_floats, bool can_split, bool narrow_ok, bool allow_pair = true,
               bool both_mn = false, bool no240 = false) {
  const int sms = num_sms();
  const int kb = (K + kBK - 1) / kBK;
  const long t1 = static_cast<long>((M + 127) / 128) * ((N + 127) / 128);
  if (allow_pair && g_force_plan.splits > 0 && !(no240 && g_force_plan.pn == 240)) return g_force_plan;
  if (g_force_variant >= 0) return {allow_pair && g_force_variant == 1, 1, 256};
  Plan best{false, 1, 256};
  double best_t = 1e30;
  auto fixup = [&](int sp) { return sp > 1 ? 3.0 + (sp + 2.0) * M * static_cast<double>(N) * 4.0 / 3.17e6 : 0.0; };
  auto split_ok = [&](int sp) {
    return sp == 1 || (can_split && static_cast<long>(sp) * M * round_up(N, 4) <= ws_floats && kb >= 8 * sp);
  };
  // Split counts: up to 8 for the MLP shapes; far more for the few-tile,
  // huge-K wgrad GEMMs of the conv model (K = pixel rows, up to ~1M).
  static const int kSplits[] = {1, 2, 3, 4, 5, 6, 7, 8, 12, 16, 24, 32, 48, 64, 96, 128, 148, 192, 256, 296};
  auto try_split = [&](int sp) {
    const int kbs = (kb + sp - 1) / sp, eff = (kb + kbs - 1) / kbs;
    const long units = t1 * eff;
    const double t =
        static_cast<double>((units + sms - 1) / sms) * ((N <= 64 && sp == 1 ? 0.31 : 0.638) * kbs + 1.41) + fixup(eff);
    if (t < best_t) best_t = t, best = {false, sp, 256};
  };
  // Few output tiles over a huge K (the conv wgrads: K = pixel rows): every
  // split count, so that tiles x splits can land just under a whole number
  // of waves (38 tiles: 35 splits = 8.99 waves, where the list's 32 / 48 fill
  // 8.2 / 12.3); the MLP shapes keep the fitted list.
  const bool fine = t1 < sms / 2 && kb >= 512;
  for (int sp : kSplits) {
    if (!split_ok(sp)) break;
    try_split(sp);
  }
  for (int sp = 9; fine && sp <= 296; ++sp) {
    if (!split_ok(sp)) break;
    try_split(sp);
  }
  const int pairs = sms / 2;
  for (int pn : kPairNs) {
    if (!allow_pair) break;
    if (pn < 240 && !narrow_ok) continue;
    if (pn == 240 && no240) continue;
    const int pe = both_mn ? 64 * ((pn + 63) / 64) : pn;
    for (int sp : {1, 2, 3, 4, 6, 8}) {
      if (!split_ok(sp)) break;
      const int kbs = (kb + sp - 1) / sp, eff = (kb + kbs - 1) / kbs;
      const long units = static_cast<long>((M + 255) / 256) * ((N + pn - 1) / pn) * eff;
      const double t = static_cast<double>((units + pairs - 1) / pairs) *
                           (1.01 * pe / 256.0 * kbs + 1.01 + 4.24 * pn / 256.0) +
                       fixup(eff);
      if (t < best_t) best_t = t, best = {true, sp, pn};
    }
  }
  return best;
}

template <int BN, int EPI>
void dispatch_major(const Operand& A, const Operand& B, const GemmEpilogue& ep, cudaStream_t s) {
  if (!A.mn_major && !B.mn_major) launch_inst<BN, false, false, EPI>(A, B, ep, s);
  else if (!A.mn_major && B.mn_major) launch_inst<BN, false, true, EPI>(A, B, ep, s);
  else if (A.mn_major && !B.mn_major) launch_inst<BN, true, false, EPI>(A, B, ep, s);
  else launch_inst<BN, true, true, EPI>(A, B, ep, s);
}

}  // namespace

void gemm_force_variant(int v) { g_force_variant = v; }

void gemm_set_chunk(int kind, int kb) {
  if (kind < 0 || kind > 2) throw std::invalid_argument("gemm_set_chunk: kind 0 (forward), 1 (dgrad), 2 (wgrad)");
  g_chunk[kind] = kb < 1 ? -1 : kb;
}

void gemm_prepare_device() {
  int dev = 0;
  SPB_CUDA(cudaGetDevice(&dev));
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  if (g_ones[dev]) return;
  float* p = nullptr;
  SPB_CUDA(cudaMalloc(&p, 64 * 32 * sizeof(float)));
  std::vector<float> h(64 * 32, 0.f);
  std::fill(h.begin(), h.begin() + 32 * 32, 1.f);
  SPB_CUDA(cudaMemcpy(p, h.data(), h.size() * sizeof(float), cudaMemcpyHostToDevice));
  g_ones[dev] = p;
  SPB_CUDA(cudaMalloc(&g_colsum_ws[dev], kColsumWsFloats * sizeof(float)));
  SPB_CUDA(cudaMalloc(&g_colsum_cnt[dev], kColsumCounters * sizeof(int)));
  SPB_CUDA(cudaMemset(g_colsum_cnt[dev], 0, kColsumCounters * sizeof(int)));
  SPB_CUDA(cudaDeviceSynchronize());
}

void gemm_force_plan(int two_sm, int pn, int splits) { g_force_plan = {two_sm != 0, splits, pn}; }

// Implicit-GEMM convolution (forward / stride-1 dgrad) on the 1-CTA kernel,
// or -- output channels >= 128 and >= 2 pixel-row tiles -- on the CTA pair
// (256 pixels x 128 / 256 channels per SM pair: half the shared-memory bytes
// per FLOP of the 1-CTA tile, which is smem-bandwidth bound at 45 % tensor
// activity on these shapes). SPB_CONV_PAIR=0 keeps the 1-CTA kernel (A/B).
template <int EPI>
int launch_conv_implicit(const Operand& A, const Operand& B, const GemmEpilogue& ep, cudaStream_t s,
                         const CUtensorMap* a, const ConvTmaArgs& ic) {
  static const bool pair_off = [] {
    const char* v = std::getenv("SPB_CONV_PAIR");
    return v && std::atoi(v) == 0;
  }();
  if (!pair_off && B.mn >= 128 && A.mn >= 256) {
    if (B.mn <= 128) launch_2sm_pn<false, false, EPI, 128, 1>(A, B, ep, s, 1, a, ic);
    else launch_2sm_pn<false, false, EPI, 256, 1>(A, B, ep, s, 1, a, ic);
    return 1;
  }
  if (B.mn <= 64)
    launch_inst<64, false, false, EPI, false, 1>(A, B, ep, s, 1, a, nullptr, ic);
  else
    launch_inst<128, false, false, EPI, false, 1>(A, B, ep, s, 1, a, nullptr, ic);
  return 1;
}

int gemm_conv_fwd(const ConvSrc& src, const Operand& B, const GemmEpilogue& ep, cudaStream_t s) {
  const ConvGeom& g = src.g;
  if (g.c_in % 32 || src.ld % 32) throw std::invalid_argument("gemm_conv_fwd: c_in and ld must be multiples of 32");
  const int M = src.samples * g.out_h * g.out_w, K = 9 * g.c_in;
  if (B.k != K || B.mn_major) throw std::invalid_argument("gemm_conv_fwd: B must be K-major [c_out x 9 c_in]");
  CUtensorMap a[2] = {im2col_map(src.hi, src, kBM, CU_TENSOR_MAP_SWIZZLE_128B),
                      im2col_map(src.lo, src, kBM, CU_TENSOR_MAP_SWIZZLE_128B)};
  const ConvTmaArgs ic{g.out_h * g.out_w, g.out_w, g.stride, g.c_in, 0, 0};
  Operand A{nullptr, nullptr, 4, M, K, false};  // shape only: tiles come from the im2col maps
  return launch_conv_implicit<kEpiFwdTanh>(A, B, ep, s, a, ic);
}

int gemm_conv_dgrad(const ConvSrc& src, long pixel0, int rows, const Operand& B, const GemmEpilogue& ep, cudaStream_t s) {
  const ConvGeom& g = src.g;
  if (g.c_in % 32 || src.ld % 32 || g.stride != 1)
    throw std::invalid_argument("gemm_conv_dgrad: stride 1, c_in and ld multiples of 32");
  const int K = 9 * g.c_in;
  if (B.k != K || B.mn_major) throw std::invalid_argument("gemm_conv_dgrad: B must be K-major [c_out x 9 c_in]");
  CUtensorMap a[2] = {im2col_map(src.hi, src, kBM, CU_TENSOR_MAP_SWIZZLE_128B),
                      im2col_map(src.lo, src, kBM, CU_TENSOR_MAP_SWIZZLE_128B)};
  const ConvTmaArgs ic{g.out_h * g.out_w, g.out_w, 1, g.c_in, 0, pixel0};
  Operand A{nullptr, nullptr, 4, rows, K, false};
  return launch_conv_implicit<kEpiDgradTanh>(A, B, ep, s, a, ic);
}

// The conv wgrads with >= 256 output channels run on the CTA pair (each CTA
// loads half of the im2col B columns, the pair shares the 256-row A tile):
// cfg4 SPB 6.35 -> 5.92 ms, wgrad phase 2.28 -> 1.72 ms on one B200 against
// the 1-CTA 128 x 128 kernel. SPB_CONV_WGRAD_PAIR=0: the 1-CTA kernel (A/B).
bool conv_wgrad_pair() {
  static const bool on = [] {
    const char* v = std::getenv("SPB_CONV_WGRAD_PAIR");
    return !(v && std::string(v) == "0");
  }();
  return on;
}

int gemm_conv_wgrad(const Operand& A, const ConvSrc& src, long pixel0, const GemmEpilogue& ep, cudaStream_t s) {
  const ConvGeom& g = src.g;
  if (g.c_in % 32 || src.ld % 32) throw std::invalid_argument("gemm_conv_wgrad: c_in and ld must be multiples of 32");
  if (!A.mn_major) throw std::invalid_argument("gemm_conv_wgrad: A (Delta) must be MN-major");
  // N = 9 c_in weight columns; with ep.bias_col_p1 = 9 c_in + 1 the bias is
  // produced by the kernel's column-sum warps as output column 9 c_in.
  const int Nw = 9 * g.c_in;
  if (ep.bias_col_p1 > 0 && ep.bias_col_p1 != Nw + 1)
    throw std::invalid_argument("gemm_conv_wgrad: the bias column must follow the 9 c_in weights");
  GemmEpilogue e = ep;
  const bool ones = ep.bias_col_p1 > 0 && bias_by_ones();
  const int N = ones ? Nw + 1 : Nw;  // the ones column (A/B knob) is one more GEMM column
  e.ones_col_p1 = ones ? ep.bias_col_p1 : 0;
  e.colsum_col_p1 = ones ? 0 : ep.bias_col_p1;
  CUtensorMap b[2] = {im2col_map(src.hi, src, 32, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B),
                      im2col_map(src.lo, src, 32, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B)};
  const ConvTmaArgs ic{g.out_h * g.out_w, g.out_w, g.stride, g.c_in, pixel0, 0};
  Operand B{nullptr, nullptr, 4, N, A.k, true};  // shape only
  if (conv_wgrad_pair() && A.mn >= 256 && ep.splitk_ws) {
    // CTA pair, 256 x 256 tiles (each CTA half of B's columns): over the
    // huge K the split count is chosen so pair tiles x splits fill whole
    // waves of the SM pairs (same cost model as plan_gemm's pair branch).
    const int pairs = num_sms() / 2, kb = (A.k + kBK - 1) / kBK;
    const int cols = epi_cols(e) > N ? epi_cols(e) : N;
    const long tiles = static_cast<long>((A.mn + 255) / 256) * ((cols + 255) / 256);
    const long ldw = round_up(cols, 4), stride = static_cast<long>(A.mn) * ldw;
    int best_sp = 1;
    double best_t = 1e300;
    for (int sp = 1; sp <= 128; ++sp) {
      if (sp > 1 && (static_cast<long>(sp) * stride > ep.splitk_ws_floats || kb < 8 * sp)) break;
      const int kbs = (kb + sp - 1) / sp, eff = (kb + kbs - 1) / kbs;
      const long units = tiles * eff;
      const double t = static_cast<double>((units + pairs - 1) / pairs) * (1.01 * kbs + 1.01 + 4.24) +
                       (eff > 1 ? 3.0 + (eff + 2.0) * A.mn * static_cast<double>(cols) * 4.0 / 3.17e6 : 0.0);
      if (t < best_t) best_t = t, best_sp = sp;
    }
    const int kbs = (kb + best_sp - 1) / best_sp, eff = (kb + kbs - 1) / kbs;
    if (eff > 1) {
      GemmEpilogue part{};
      part.out_hi = ep.splitk_ws;
      part.ld_out = ldw;
      part.alpha = 1.0f;
      part.M = A.mn;
      part.N = N;
      part.split_stride = stride;
      part.ones_col_p1 = e.ones_col_p1;
      part.colsum_col_p1 = 0;
      launch_2sm_pn<true, true, kEpiStoreScaled, 256, 2>(A, B, part, s, eff, nullptr, ic, b);
      launch_fixup<kEpiStoreScaled>(ep.splitk_ws, eff, stride, ldw, e, s);
      return 2;
    }
    launch_2sm_pn<true, true, kEpiStoreScaled, 256, 2>(A, B, e, s, 1, nullptr, ic, b);
    return 1;
  }
  const Plan plan = plan_gemm(A.mn, epi_cols(e) > N ? epi_cols(e) : N, A.k, ep.splitk_ws ? ep.splitk_ws_floats : 0,
                              ep.splitk_ws != nullptr, false, false);  // the im2col-B wgrad has a 1-CTA kernel only
  if (plan.splits > 1) {
    const long ldw = round_up(epi_cols(e) > N ? epi_cols(e) : N, 4), stride = static_cast<long>(A.mn) * ldw;
    GemmEpilogue part{};
    part.out_hi = ep.splitk_ws;
    part.ld_out = ldw;
    part.alpha = 1.0f;
    part.M = A.mn;
    part.N = N;
    part.split_stride = stride;
    part.ones_col_p1 = e.ones_col_p1;      // the partials compute the bias column like any other,
    part.colsum_col_p1 = e.colsum_col_p1;  // or the column-sum warps write it into the workspace
    part.colsum_ws = e.colsum_ws, part.colsum_cnt = e.colsum_cnt;
    launch_inst<128, true, true, kEpiStoreScaled, false, 2>(A, B, part, s, plan.splits, nullptr, b, ic);
    const int kb = (A.k + kBK - 1) / kBK, kbs = (kb + plan.splits - 1) / plan.splits;
    // (the fixup's epilogue `e` routes column 9 c_in to the bias)
    launch_fixup<kEpiStoreScaled>(ep.splitk_ws, (kb + kbs - 1) / kbs, stride, ldw, e, s);
    return 2;
  }
  launch_inst<128, true, true, kEpiStoreScaled, false, 2>(A, B, e, s, 1, nullptr, b, ic);
  return 1;
}

int gemm_reserve_sms(int n) {
  const int prev = g_reserved_sms;
  g_reserved_sms = n < 0 ? 0 : n;
  return prev;
}

void gemm_last_plan(int* two_sm, int* pn, int* splits) {
  *two_sm = g_last_plan.two_sm ? 1 : 0;
  *pn = g_last_plan.pn;
  *splits = g_last_plan.splits;
}

int gemm_tf32x3_planned(const Operand& A, const Operand& B, int epi, const GemmEpilogue& ep, cudaStream_t s,
                        const Plan& plan);

int gemm_tf32x3(const Operand& A, const Operand& B, int epi, const GemmEpilogue& ep, cudaStream_t s) {
  if (A.k != B.k) throw std::invalid_argument("gemm: K mismatch");
  if (epi == kEpiWgradUpdate && !(A.mn_major && B.mn_major)) throw std::invalid_argument("gemm: wgrad-update is MN/MN");
  if (A.mn <= 0 || B.mn <= 0 || A.k <= 0) return 0;
  if ((A.ld % 4) || (B.ld % 4)) throw std::invalid_argument("gemm: ld must be a multiple of 4");
  constexpr int BN = 128;
  static const bool no_split = std::getenv("SPB_NO_SPLITK") != nullptr;  // tuning experiments
  const bool can_split = ep.splitk_ws != nullptr && (epi == kEpiFwdTanh || epi == kEpiDgradTanh ||
                                                     epi == kEpiFwdLinear || epi == kEpiStoreScaled);
  if (ep.ones_col_p1 > 0) {  // fused bias: a 32-aligned ones box at or beyond the real MN extent
    const int oc = ep.ones_col_p1 - 1;
    if (!B.mn_major || oc % 32 || oc < (B.mn_map > 0 ? B.mn_map : B.mn) || B.mn != oc + 1)
      throw std::invalid_argument("gemm: bad fused-bias column");
  }
  // Routed epilogues (the push exchange) stage rows through shared memory in
  // the 1-CTA kernel only: the pair kernel would store 16-byte pieces row by
  // row over NVLink.
  const Plan plan = plan_gemm(A.mn, B.mn, A.k, ep.splitk_ws && !no_split ? ep.splitk_ws_floats : 0, can_split,
                              narrow_pair_ok(A, B, epi), ep.route_rows == 0, A.mn_major && B.mn_major,
                              ep.ones_col_p1 > 0);
  g_last_plan = plan;
  if (ep.ones_col_p1 > 0 && !bias_by_ones() && (!plan.two_sm || (epi == kEpiWgradUpdate && g_force_variant != 1))) {
    // 1-CTA kernel: the column-sum warps produce the bias (no extra column tile).
    Operand B2 = B;
    B2.mn = B.mn_map > 0 ? B.mn_map : B.mn - 1;
    B2.mn_map = 0;
    GemmEpilogue e2 = ep;
    e2.ones_col_p1 = 0;
    e2.colsum_col_p1 = ep.bias_col_p1;
    return gemm_tf32x3_planned(A, B2, epi, e2, s, plan);
  }
  return gemm_tf32x3_planned(A, B, epi, ep, s, plan);
}

int gemm_tf32x3_planned(const Operand& A, const Operand& B, int epi, const GemmEpilogue& ep, cudaStream_t s,
                        const Plan& plan) {
  constexpr int BN = 128;
  if (plan.splits > 1) {
    switch (epi) {
      case kEpiFwdTanh: launch_splitk<kEpiFwdTanh>(A, B, ep, s, plan); break;
      case kEpiDgradTanh: launch_splitk<kEpiDgradTanh>(A, B, ep, s, plan); break;
      case kEpiFwdLinear: launch_splitk<kEpiFwdLinear>(A, B, ep, s, plan); break;
      case kEpiStoreScaled: launch_splitk<kEpiStoreScaled>(A, B, ep, s, plan); break;
      default: throw std::invalid_argument("gemm: split-K not supported for this epilogue");
    }
    return 2;
  }
  // The in-place optimizer epilogue is HBM bound: it always takes the 1-CTA
  // kernel with TMA-staged W / momentum tiles (unless a test forces the pair kernel).
  if (epi == kEpiWgradUpdate && g_force_variant != 1) {
    g_last_plan = {false, 1, BN};
    launch_inst<BN, true, true, kEpiWgradUpdate, true>(A, B, ep, s);
    return 1;
  }
  if (plan.two_sm) {
    const int pn = epi == kEpiWgradUpdate && plan.pn < 240 ? 256 : plan.pn;
    switch (epi) {
      case kEpiFwdTanh: dispatch_2sm<kEpiFwdTanh>(A, B, ep, s, pn); break;
      case kEpiStoreScaled: dispatch_2sm<kEpiStoreScaled>(A, B, ep, s, pn); break;
      case kEpiDgradTanh: dispatch_2sm<kEpiDgradTanh>(A, B, ep, s, pn); break;
      case kEpiFwdLinear: dispatch_2sm<kEpiFwdLinear>(A, B, ep, s, pn); break;
      case kEpiWgradUpdate: launch_2sm<true, true, kEpiWgradUpdate>(A, B, ep, s, pn, 1); break;
      default: throw std::invalid_argument("gemm: bad epilogue");
    }
    return 1;
  }
  g_last_plan.pn = B.mn <= 64 && epi != kEpiWgradUpdate ? 64 : BN;
  if (B.mn <= 64 && epi != kEpiWgradUpdate) {  // narrow outputs (64-channel convs): 128 x 64 tiles, no idle MMA half
    switch (epi) {
      case kEpiFwdTanh: dispatch_major<64, kEpiFwdTanh>(A, B, ep, s); break;
      case kEpiStoreScaled: dispatch_major<64, kEpiStoreScaled>(A, B, ep, s); break;
      case kEpiDgradTanh: dispatch_major<64, kEpiDgradTanh>(A, B, ep, s); break;
      case kEpiFwdLinear: dispatch_major<64, kEpiFwdLinear>(A, B, ep, s); break;
      default: throw std::invalid_argument("gemm: bad epilogue");
    }
    return 1;
  }
  switch (epi) {
    case kEpiFwdTanh: dispatch_major<BN, kEpiFwdTanh>(A, B, ep, s); break;
    case kEpiStoreScaled: dispatch_major<BN, kEpiStoreScaled>(A, B, ep, s); break;
    case kEpiDgradTanh: dispatch_major<BN, kEpiDgradTanh>(A, B, ep, s); break;
    case kEpiFwdLinear: dispatch_major<BN, kEpiFwdLinear>(A, B, ep, s); break;
    case kEpiWgradUpdate: launch_inst<BN, true, true, kEpiWgradUpdate>(A, B, ep, s); break;
    default: throw std::invalid_argument("gemm: bad epilogue");
  }
  return 1;
}

}  // namespace spb
