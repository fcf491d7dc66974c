// Host side of the tcgen05 3xTF32 GEMM: TMA tensor-map encoding and the
// template dispatch over (A major, B major, epilogue).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include <cstdlib>

#include "gemm_2sm.cuh"
#include "gemm_tf32x3.cuh"
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

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    SPB_CUDA(cudaGetDevice(&dev));
    SPB_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  }
  return n;
}

CUtensorMap operand_map(const Operand& X, const float* base, int tile_rows) {
  if (!X.mn_major) return tmap2d(base, X.k, X.mn, X.ld, kBK, tile_rows, CU_TENSOR_MAP_SWIZZLE_128B);
  return tmap2d(base, X.mn, X.k, X.ld, 32, kBK, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
}

template <int BN, bool AM, bool BM_, int EPI>
void launch_inst(const Operand& A, const Operand& B, const GemmEpilogue& ep, cudaStream_t s) {
  auto kern = gemm_tf32x3_kernel<BN, AM, BM_, EPI>;
  constexpr int smem = GemmCfg<BN>::kSmem;
  static bool configured = false;
  if (!configured) {
    SPB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    configured = true;
  }
  CUtensorMap ah = operand_map(A, A.hi, kBM), al = operand_map(A, A.lo, kBM);
  CUtensorMap bh = operand_map(B, B.hi, BN), bl = operand_map(B, B.lo, BN);
  const int num_kb = (A.k + kBK - 1) / kBK;
  const int num_m = (A.mn + kBM - 1) / kBM, num_n = (B.mn + BN - 1) / BN;
  const int tiles = num_m * num_n;
  const int grid = tiles < num_sms() ? tiles : num_sms();
  kern<<<grid, 256, smem, s>>>(ah, al, bh, bl, num_kb, num_m, tiles, ep);
  SPB_CUDA(cudaGetLastError());
}

template <bool AM, bool BM_, int EPI>
void launch_2sm(const Operand& A, const Operand& B, const GemmEpilogue& ep, cudaStream_t s) {
  using Cfg = Gemm2smCfg;
  auto kern = gemm_tf32x3_2sm_kernel<AM, BM_, EPI>;
  static bool configured = false;
  if (!configured) {
    SPB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem));
    configured = true;
  }
  CUtensorMap ah = operand_map(A, A.hi, Cfg::kRowsA), al = operand_map(A, A.lo, Cfg::kRowsA);
  CUtensorMap bh = operand_map(B, B.hi, Cfg::kRowsB), bl = operand_map(B, B.lo, Cfg::kRowsB);
  const int num_kb = (A.k + kBK - 1) / kBK;
  const int num_m = (A.mn + 255) / 256, num_n = (B.mn + Cfg::kPairN - 1) / Cfg::kPairN;
  const int tiles = num_m * num_n;
  const int pairs = num_sms() / 2;
  const int clusters = tiles < pairs ? tiles : pairs;
  kern<<<2 * clusters, Cfg::kThreads, Cfg::kSmem, s>>>(ah, al, bh, bl, num_kb, num_m, tiles, ep);
  SPB_CUDA(cudaGetLastError());
}

template <int EPI>
void dispatch_2sm(const Operand& A, const Operand& B, const GemmEpilogue& ep, cudaStream_t s) {
  if (!A.mn_major && !B.mn_major) launch_2sm<false, false, EPI>(A, B, ep, s);
  else if (!A.mn_major && B.mn_major) launch_2sm<false, true, EPI>(A, B, ep, s);
  else if (A.mn_major && !B.mn_major) launch_2sm<true, false, EPI>(A, B, ep, s);
  else launch_2sm<true, true, EPI>(A, B, ep, s);
}

int g_force_variant = -1;  // -1 auto, 0 = 1-CTA 128x128, 1 = CTA pair 256x256

// Wave-quantised cost of each variant, in units of one 1-CTA 128x128 tile.
// A pair tile is 4 such tiles on 2 SMs at kPairSpeedup x the per-SM rate.
bool use_2sm(int M, int N) {
  if (g_force_variant >= 0) return g_force_variant == 1;
  static const double ratio = [] {
    const char* e = std::getenv("SPB_2SM_COST");
    return e ? std::atof(e) : 0.7;
  }();
  const int sms = num_sms();
  const long t1 = static_cast<long>((M + 127) / 128) * ((N + 127) / 128);
  const long t2 = static_cast<long>((M + 255) / 256) * ((N + 255) / 256);
  const double c1 = static_cast<double>((t1 + sms - 1) / sms);
  const double c2 = static_cast<double>((t2 + sms / 2 - 1) / (sms / 2)) * 2.0 * ratio;
  return c2 < c1;
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

int gemm_tf32x3(const Operand& A, const Operand& B, int epi, const GemmEpilogue& ep, cudaStream_t s) {
  if (A.k != B.k) throw std::invalid_argument("gemm: K mismatch");
  if (epi == kEpiWgradUpdate && !(A.mn_major && B.mn_major)) throw std::invalid_argument("gemm: wgrad-update is MN/MN");
  if (A.mn <= 0 || B.mn <= 0 || A.k <= 0) return 0;
  if ((A.ld % 4) || (B.ld % 4)) throw std::invalid_argument("gemm: ld must be a multiple of 4");
  constexpr int BN = 128;
  if (use_2sm(A.mn, B.mn)) {
    switch (epi) {
      case kEpiFwdTanh: dispatch_2sm<kEpiFwdTanh>(A, B, ep, s); break;
      case kEpiStoreScaled: dispatch_2sm<kEpiStoreScaled>(A, B, ep, s); break;
      case kEpiDgradTanh: dispatch_2sm<kEpiDgradTanh>(A, B, ep, s); break;
      case kEpiFwdLinear: dispatch_2sm<kEpiFwdLinear>(A, B, ep, s); break;
      case kEpiWgradUpdate: launch_2sm<true, true, kEpiWgradUpdate>(A, B, ep, s); break;
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
