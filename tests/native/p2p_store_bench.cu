// NVLink write paths from one B200 into a peer's memory (tuning aid for the
// push exchange, not a test): the same 48 MB of fp32 rows, 4096 wide, written
//   (a) by SM stores of 128-byte row segments (the push epilogue today),
//   (b) by TMA tensor stores of 32 x 32 tiles staged in shared memory,
//   (c) by the copy engine (cudaMemcpyPeerAsync of the same bytes),
// while (optionally) the peer does the same towards us. Prints GB/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I include \
//        -o build/p2p_store_bench tests/native/p2p_store_bench.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <thread>
#include <vector>

#include "../../paper_2111_10672_b200/csrc/ptx.cuh"

using namespace spb;

constexpr int kCols = 4096;
constexpr int kRows = 3072;  // 48 MB of fp32

__global__ void sm_store_kernel(const float* __restrict__ src, float* __restrict__ dst) {
  // one warp per 32 x 32 block: 8 row segments of 128 B per warp store
  const int warps = blockDim.x / 32, lane = threadIdx.x & 31;
  const long nblk = static_cast<long>(kRows / 32) * (kCols / 32);
  for (long b = blockIdx.x * warps + threadIdx.x / 32; b < nblk; b += static_cast<long>(gridDim.x) * warps) {
    const int r0 = static_cast<int>(b / (kCols / 32)) * 32, c0 = static_cast<int>(b % (kCols / 32)) * 32;
    const int cc = 4 * (lane & 7);
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      const int r = r0 + it * 4 + (lane >> 3);
      const float4 v = *reinterpret_cast<const float4*>(src + static_cast<long>(r) * kCols + c0 + cc);
      *reinterpret_cast<float4*>(dst + static_cast<long>(r) * kCols + c0 + cc) = v;
    }
  }
}

__global__ void tma_store_kernel(const float* __restrict__ src, const __grid_constant__ CUtensorMap dmap) {
  // one warp per 32 x 32 block: stage in smem (SW128), one TMA tensor store
  extern __shared__ __align__(1024) uint8_t sm[];
  const int warps = blockDim.x / 32, w = threadIdx.x / 32, lane = threadIdx.x & 31;
  uint8_t* buf = sm + w * 2 * 4096;
  int k = 0;
  const long nblk = static_cast<long>(kRows / 32) * (kCols / 32);
  for (long b = blockIdx.x * warps + w; b < nblk; b += static_cast<long>(gridDim.x) * warps, ++k) {
    const int r0 = static_cast<int>(b / (kCols / 32)) * 32, c0 = static_cast<int>(b % (kCols / 32)) * 32;
    uint8_t* t = buf + (k & 1) * 4096;
    if (lane == 0 && k >= 2) bulk_wait_read_all();
    __syncwarp();
    const float* row = src + static_cast<long>(r0 + lane) * kCols + c0;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const float4 v = *reinterpret_cast<const float4*>(row + 4 * c);
      *reinterpret_cast<float4*>(t + lane * 128 + ((c ^ (lane & 7)) << 4)) = v;
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      tma_store_2d(&dmap, t, c0, r0);
      bulk_commit();
    }
  }
  if (lane == 0) bulk_wait_all();
}

static CUtensorMap make_map(float* base) {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  CUtensorMap m;
  cuuint64_t dims[2] = {kCols, kRows};
  cuuint64_t strides[1] = {kCols * 4};
  cuuint32_t box[2] = {32, 32}, es[2] = {1, 1};
  fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return m;
}

int main() {
  int n = 0;
  cudaGetDeviceCount(&n);
  if (n < 2) {
    std::printf("needs 2 GPUs\n");
    return 1;
  }
  const size_t bytes = static_cast<size_t>(kRows) * kCols * 4;
  float *src[2], *dst[2];
  for (int d = 0; d < 2; ++d) {
    cudaSetDevice(d);
    cudaDeviceEnablePeerAccess(1 - d, 0);
    cudaMalloc(&src[d], bytes);
    cudaMalloc(&dst[d], bytes);
    cudaMemset(src[d], 0, bytes);
  }
  const int smem = 8 * 2 * 4096;
  for (int d = 0; d < 2; ++d) {
    cudaSetDevice(d);
    cudaFuncSetAttribute(tma_store_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  }
  for (int both = 0; both < 2; ++both)
    for (int mode = 0; mode < 3; ++mode)
      for (int ctas : {16, 32, 74, 148}) {
        if (mode == 2 && ctas != 148) continue;
        float ms[2] = {0, 0};
        auto run = [&](int d) {
          cudaSetDevice(d);
          cudaStream_t s;
          cudaStreamCreate(&s);
          float* peer_dst = dst[1 - d];
          CUtensorMap m = make_map(peer_dst);
          cudaEvent_t a, b;
          cudaEventCreate(&a), cudaEventCreate(&b);
          for (int rep = 0; rep < 6; ++rep) {
            if (rep == 1) cudaEventRecord(a, s);
            if (mode == 0) sm_store_kernel<<<ctas, 256, 0, s>>>(src[d], peer_dst);
            if (mode == 1) tma_store_kernel<<<ctas, 256, smem, s>>>(src[d], m);
            if (mode == 2) cudaMemcpyPeerAsync(peer_dst, 1 - d, src[d], d, bytes, s);
          }
          cudaEventRecord(b, s);
          cudaEventSynchronize(b);
          cudaEventElapsedTime(&ms[d], a, b);
          cudaError_t e = cudaGetLastError();
          if (e != cudaSuccess) std::printf("error %s\n", cudaGetErrorString(e));
          cudaStreamDestroy(s);
        };
        if (both) {
          std::thread t0(run, 0), t1(run, 1);
          t0.join(), t1.join();
        } else {
          run(0);
        }
        const char* names[3] = {"sm-store", "tma-store", "copy-engine"};
        std::printf("%-12s %s ctas=%3d  %.1f GB/s per direction\n", names[mode], both ? "bidir" : "one-way", ctas,
                    5.0 * bytes / (ms[0] * 1e-3) / 1e9);
      }
  return 0;
}
