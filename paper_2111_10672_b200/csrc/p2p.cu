// Peer-to-peer per-layer aggregation for the multi-GPU SPB step (the default
// multi-GPU path, engine.cu "p2p" mode).
//
// Every layer's parameters are sharded over the ranks (rank r owns the r-th
// 1/N of the layer's flat segment). Per layer l, top down:
//   1. the rank's gradient of l is final -> signal G[l] to every rank;
//   2. wait for G[l] of the contributing ranks, then PULL their gradients of
//      this rank's shard over NVLink with the copy engines (cudaMemcpyAsync
//      from IPC-mapped peer memory: no SMs, ~750 GB/s per direction);
//   3. shard update kernel: sum the contributions in rank order, momentum /
//      weight decay / SGD, write hi / lo / momentum and the fp32 weights w32
//      the peers will pull; signal U[l];
//   4. wait for U[l] of every rank, PULL their w32 shards (copy engines);
//   5. split kernel: w32 -> (hi, lo) for the pulled shards.
// Signals are epoch-stamped flags written into the peers' flag arrays with
// st.release.sys and polled with ld.acquire.sys; step t of a replayed graph
// uses the value epoch + t + 1, and the epoch advances by the graph's step
// count after its last step, identically on all ranks (values only grow, so
// a wait is a >= compare).
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>

#include "launch.hpp"
#include "p2p.hpp"

namespace spb {
namespace {

__device__ __forceinline__ void spin_ge(const int* flag, int target) {
  int v = 0;
  uint64_t t0 = 0;
  for (uint32_t spin = 0;; ++spin) {
    asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    if (v >= target) return;
    if ((spin & 0x3FFu) == 0x3FFu) {
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t0 == 0) t0 = t;
      else if (t - t0 > 30000000000ull) __trap();  // a missing rank must fail, not hang the GPU
    }
  }
}

// flags layout (every rank): [slot][src rank] int.
// Flag value of step `sub` of the graph being replayed: epoch + sub + 1 (the
// epoch advances by the graph's step count after its last step).
__global__ void p2p_signal_kernel(PeerPtrs<int> flags, int slot, int nranks, int rank, const int* epoch, int sub) {
  __threadfence_system();
  const int v = *epoch + sub + 1;
  for (int p = threadIdx.x; p < nranks; p += blockDim.x) {
    int* f = flags.p[p] + slot * nranks + rank;
    asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(f), "r"(v) : "memory");
  }
}

__global__ void p2p_wait_kernel(const int* flags, int slot, int nranks, unsigned mask, const int* epoch, int sub) {
  const int target = *epoch + sub + 1;
  for (int p = threadIdx.x; p < nranks; p += blockDim.x)
    if (mask >> p & 1u) spin_ge(flags + slot * nranks + p, target);
}

__global__ void p2p_epoch_kernel(int* epoch, int add) { *epoch += add; }

// Shard update: g = sum of the contributions (fixed rank order), then
// g' = g + wd*w; buf = mu*buf + g'; w -= lr*buf; hi, lo = split(w); w32 = w.
__global__ void __launch_bounds__(256) p2p_update_kernel(PeerPtrs<const float> src, int nsrc, float* __restrict__ hi,
                                                         float* __restrict__ lo, float* __restrict__ mom,
                                                         float* __restrict__ w32, long n4, float lr, float mu,
                                                         float wd) {
  const long stride = static_cast<long>(gridDim.x) * blockDim.x;
  for (long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride) {
    float g[4] = {0.f, 0.f, 0.f, 0.f};
    for (int s = 0; s < nsrc; ++s) {
      const float4 v = reinterpret_cast<const float4*>(src.p[s])[i];
      g[0] += v.x, g[1] += v.y, g[2] += v.z, g[3] += v.w;
    }
    const float4 h = reinterpret_cast<const float4*>(hi)[i];
    const float4 l = reinterpret_cast<const float4*>(lo)[i];
    float w[4] = {h.x + l.x, h.y + l.y, h.z + l.z, h.w + l.w};
    float b[4] = {0.f, 0.f, 0.f, 0.f};
    if (mom) {
      const float4 m = reinterpret_cast<const float4*>(mom)[i];
      b[0] = m.x, b[1] = m.y, b[2] = m.z, b[3] = m.w;
    }
    float nh[4], nl[4], nw[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float gg = fmaf(wd, w[j], g[j]);
      if (mom) {
        b[j] = fmaf(mu, b[j], gg);
        gg = b[j];
      }
      nw[j] = w[j] - lr * gg;
      uint32_t r;
      asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(nw[j]));
      nh[j] = __uint_as_float(r);
      nl[j] = nw[j] - nh[j];
    }
    reinterpret_cast<float4*>(hi)[i] = make_float4(nh[0], nh[1], nh[2], nh[3]);
    reinterpret_cast<float4*>(lo)[i] = make_float4(nl[0], nl[1], nl[2], nl[3]);
    reinterpret_cast<float4*>(w32)[i] = make_float4(nw[0], nw[1], nw[2], nw[3]);
    if (mom) reinterpret_cast<float4*>(mom)[i] = make_float4(b[0], b[1], b[2], b[3]);
  }
}

// (hi, lo) = split(w32) over [0, n4) minus the hole [h0, h1) (in float4s).
__global__ void __launch_bounds__(256) p2p_split_kernel(const float* __restrict__ w32, float* __restrict__ hi,
                                                        float* __restrict__ lo, long n4, long h0, long h1) {
  const long stride = static_cast<long>(gridDim.x) * blockDim.x;
  const long m = n4 - (h1 - h0);
  for (long t = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; t < m; t += stride) {
    const long i = t < h0 ? t : t + (h1 - h0);
    const float4 v = reinterpret_cast<const float4*>(w32)[i];
    float x[4] = {v.x, v.y, v.z, v.w}, nh[4], nl[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint32_t r;
      asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x[j]));
      nh[j] = __uint_as_float(r);
      nl[j] = x[j] - nh[j];
    }
    reinterpret_cast<float4*>(hi)[i] = make_float4(nh[0], nh[1], nh[2], nh[3]);
    reinterpret_cast<float4*>(lo)[i] = make_float4(nl[0], nl[1], nl[2], nl[3]);
  }
}

// dst += src over n floats (n % 4 == 0): one recursive-halving reduce round.
__global__ void __launch_bounds__(256) rh_add_kernel(float* __restrict__ dst, const float* __restrict__ src, long n4) {
  const long stride = static_cast<long>(gridDim.x) * blockDim.x;
  for (long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4 a = reinterpret_cast<float4*>(dst)[i];
    const float4 b = reinterpret_cast<const float4*>(src)[i];
    a.x += b.x, a.y += b.y, a.z += b.z, a.w += b.w;
    reinterpret_cast<float4*>(dst)[i] = a;
  }
}

int grid_for(long n4) { return static_cast<int>(std::max<long>(1, std::min<long>((n4 + 255) / 256, 148L * 8))); }

}  // namespace

void launch_p2p_signal(const PeerPtrs<int>& flags, int slot, int nranks, int rank, const int* epoch, int sub,
                       cudaStream_t s) {
  p2p_signal_kernel<<<1, 32, 0, s>>>(flags, slot, nranks, rank, epoch, sub);
  SPB_CUDA(cudaGetLastError());
}

void launch_p2p_wait(const int* flags, int slot, int nranks, unsigned mask, const int* epoch, int sub, cudaStream_t s) {
  p2p_wait_kernel<<<1, 32, 0, s>>>(flags, slot, nranks, mask, epoch, sub);
  SPB_CUDA(cudaGetLastError());
}

void launch_p2p_epoch(int* epoch, int add, cudaStream_t s) {
  p2p_epoch_kernel<<<1, 1, 0, s>>>(epoch, add);
  SPB_CUDA(cudaGetLastError());
}

void launch_p2p_update(const PeerPtrs<const float>& src, int nsrc, float* hi, float* lo, float* mom, float* w32, long n,
                       float lr, float mu, float wd, cudaStream_t s) {
  if (n <= 0) return;
  if (n % 4) throw std::invalid_argument("p2p: shard must be a multiple of 4 floats");
  if (nsrc > kMaxPeers) throw std::invalid_argument("p2p: too many sources");
  p2p_update_kernel<<<grid_for(n / 4), 256, 0, s>>>(src, nsrc, hi, lo, mom, w32, n / 4, lr, mu, wd);
  SPB_CUDA(cudaGetLastError());
}

void launch_rh_add(float* dst, const float* src, long n, cudaStream_t s) {
  if (n <= 0) return;
  if (n % 4) throw std::invalid_argument("rh: ranges must be multiples of 4 floats");
  rh_add_kernel<<<grid_for(n / 4), 256, 0, s>>>(dst, src, n / 4);
  SPB_CUDA(cudaGetLastError());
}

void launch_p2p_split(const float* w32, float* hi, float* lo, long n, long hole0, long hole1, cudaStream_t s) {
  if (n % 4 || hole0 % 4 || hole1 % 4) throw std::invalid_argument("p2p: split ranges must be multiples of 4");
  const long m = (n - (hole1 - hole0)) / 4;
  if (m <= 0) return;
  p2p_split_kernel<<<grid_for(m), 256, 0, s>>>(w32, hi, lo, n / 4, hole0 / 4, hole1 / 4);
  SPB_CUDA(cudaGetLastError());
}

}  // namespace spb
