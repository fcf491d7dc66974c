// "push" per-layer aggregation for the multi-GPU SPB step (engine.cu
// comm_mode 4): the exchange rides on NVLink STORES issued by the kernels
// that produce the data, instead of copy-engine pulls.
//
// Layer l's rows are owned block-wise: rank o owns output rows
// [o * rpo, (o + 1) * rpo) of W_l and b_l (rpo = ceil(n_l / N)). Per layer,
// top down:
//   1. the wgrad GEMM's epilogue stores each gradient row straight into its
//      owner's staging slot for this rank (peer memory mapped through CUDA
//      IPC; own rows stay in the local gradient buffer), so the transfer
//      overlaps the GEMM tile by tile;
//   2. push_signal_kernel: the bias-gradient rows (and, for the head layer,
//      whose gradient comes from a column reduction rather than the GEMM, the
//      weight rows) are copied to the owners the same way, then a system
//      fence and the epoch-stamped G[l] flag at every rank;
//   3. the owner waits for every rank's G[l], then push_update_kernel sums
//      the contributions in rank order (the p2p mode's order: identical bits),
//      applies momentum / weight decay / SGD to its rows (hi, lo, momentum)
//      and writes the new fp32 rows to its w32, then signals U[l];
//   4. every rank waits for each owner's U[l], pulls its rows with the copy
//      engines (as in the p2p mode; the first version stored them into every
//      peer from the update kernel, which ran at ~130 GB/s) and splits them
//      w32 -> (hi, lo) (p2p_split_kernel / push_split_kernel).
// The GEMM epilogue stages each 32 x 32 block in shared memory so that the
// NVLink stores are 128-byte row segments (gemm_tf32x3.cuh; the first version
// stored row-per-lane 16-byte pieces at ~115 GB/s).
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>

#include "launch.hpp"
#include "p2p.hpp"

namespace spb {
namespace {

// 1 block: copy this rank's gradient rows owned by each peer o into o's
// staging slot (bias rows always when gb != null, weight rows when gw !=
// null), then fence and signal flags[slot][rank] = epoch + sub + 1 everywhere.
__global__ void __launch_bounds__(512) push_signal_kernel(PeerPtrs<int> flags, int slot, int nranks, int rank,
                                                          const int* epoch, int sub, const float* __restrict__ gw,
                                                          long ldw, const float* __restrict__ gb, int rpo,
                                                          int n_rows, PeerPtrs<float> wdst, PeerPtrs<float> bdst) {
  for (int o = 0; o < nranks; ++o) {
    if (o == rank) continue;
    const int r0 = o * rpo, r1 = min(n_rows, r0 + rpo);
    if (r1 <= r0) continue;
    if (gb)
      for (int i = threadIdx.x; i < r1 - r0; i += blockDim.x) bdst.p[o][i] = gb[r0 + i];
    if (gw) {
      const long n = static_cast<long>(r1 - r0) * ldw;
      const float* src = gw + static_cast<long>(r0) * ldw;
      for (long i = threadIdx.x; i < n; i += blockDim.x) wdst.p[o][i] = src[i];
    }
  }
  __syncthreads();
  __threadfence_system();
  const int v = *epoch + sub + 1;
  for (int p = threadIdx.x; p < nranks; p += blockDim.x) {
    int* f = flags.p[p] + slot * nranks + rank;
    asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(f), "r"(v) : "memory");
  }
}

// Owner update of n contiguous parameters: g = sum of the nsrc contributions
// (rank order), g' = g + wd*w; buf = mu*buf + g'; w -= lr*buf; hi, lo =
// split(w) in place; w stored to the ndst peers' w32 copies.
template <bool VEC>
__global__ void __launch_bounds__(256) push_update_kernel(PeerPtrs<const float> src, int nsrc, float* __restrict__ hi,
                                                          float* __restrict__ lo, float* __restrict__ mom,
                                                          PeerPtrs<float> dst, int ndst, long n, float lr, float mu,
                                                          float wd) {
  constexpr int V = VEC ? 4 : 1;
  const long nv = n / V;
  const long stride = static_cast<long>(gridDim.x) * blockDim.x;
  for (long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; i < nv; i += stride) {
    float g[V], h[V], l[V], b[V];
#pragma unroll
    for (int j = 0; j < V; ++j) g[j] = 0.f, b[j] = 0.f;
    for (int s = 0; s < nsrc; ++s) {
      if constexpr (VEC) {
        const float4 v = reinterpret_cast<const float4*>(src.p[s])[i];
        g[0] += v.x, g[1] += v.y, g[2] += v.z, g[3] += v.w;
      } else {
        g[0] += src.p[s][i];
      }
    }
    if constexpr (VEC) {
      const float4 a = reinterpret_cast<const float4*>(hi)[i], c = reinterpret_cast<const float4*>(lo)[i];
      h[0] = a.x, h[1] = a.y, h[2] = a.z, h[3] = a.w, l[0] = c.x, l[1] = c.y, l[2] = c.z, l[3] = c.w;
      if (mom) {
        const float4 m = reinterpret_cast<const float4*>(mom)[i];
        b[0] = m.x, b[1] = m.y, b[2] = m.z, b[3] = m.w;
      }
    } else {
      h[0] = hi[i], l[0] = lo[i];
      if (mom) b[0] = mom[i];
    }
    float nh[V], nl[V], nw[V];
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const float w = h[j] + l[j];
      float gg = fmaf(wd, w, g[j]);
      if (mom) {
        b[j] = fmaf(mu, b[j], gg);
        gg = b[j];
      }
      nw[j] = w - lr * gg;
      uint32_t r;
      asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(nw[j]));
      nh[j] = __uint_as_float(r);
      nl[j] = nw[j] - nh[j];
    }
    if constexpr (VEC) {
      reinterpret_cast<float4*>(hi)[i] = make_float4(nh[0], nh[1], nh[2], nh[3]);
      reinterpret_cast<float4*>(lo)[i] = make_float4(nl[0], nl[1], nl[2], nl[3]);
      if (mom) reinterpret_cast<float4*>(mom)[i] = make_float4(b[0], b[1], b[2], b[3]);
      const float4 o = make_float4(nw[0], nw[1], nw[2], nw[3]);
      for (int d = 0; d < ndst; ++d) reinterpret_cast<float4*>(dst.p[d])[i] = o;
    } else {
      hi[i] = nh[0], lo[i] = nl[0];
      if (mom) mom[i] = b[0];
      for (int d = 0; d < ndst; ++d) dst.p[d][i] = nw[0];
    }
  }
}

// (hi, lo) = split(w32) on [0, n) except [h0, h1), any alignment.
__global__ void push_split_kernel(const float* __restrict__ w32, float* __restrict__ hi, float* __restrict__ lo,
                                  long n, long h0, long h1) {
  const long stride = static_cast<long>(gridDim.x) * blockDim.x;
  for (long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    if (i >= h0 && i < h1) continue;
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(w32[i]));
    hi[i] = __uint_as_float(r);
    lo[i] = w32[i] - __uint_as_float(r);
  }
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace

void launch_push_signal(const PeerPtrs<int>& flags, int slot, int nranks, int rank, const int* epoch, int sub,
                        const float* gw, long ldw, const float* gb, int rpo, int n_rows, const PeerPtrs<float>& wdst,
                        const PeerPtrs<float>& bdst, cudaStream_t s) {
  push_signal_kernel<<<1, 512, 0, s>>>(flags, slot, nranks, rank, epoch, sub, gw, ldw, gb, rpo, n_rows, wdst, bdst);
  SPB_CUDA(cudaGetLastError());
}

void launch_push_update(const PeerPtrs<const float>& src, int nsrc, float* hi, float* lo, float* mom,
                        const PeerPtrs<float>& dst, int ndst, long n, float lr, float mu, float wd, cudaStream_t s) {
  if (n <= 0) return;
  if (nsrc > kMaxPeers || ndst > kMaxPeers) throw std::invalid_argument("push: too many peers");
  bool vec = n % 4 == 0 && aligned16(hi) && aligned16(lo) && (!mom || aligned16(mom));
  for (int i = 0; i < nsrc; ++i) vec = vec && aligned16(src.p[i]);
  for (int i = 0; i < ndst; ++i) vec = vec && aligned16(dst.p[i]);
  const long nv = vec ? n / 4 : n;
  const int grid = static_cast<int>(std::max<long>(1, std::min<long>((nv + 255) / 256, 148L * 8)));
  if (vec)
    push_update_kernel<true><<<grid, 256, 0, s>>>(src, nsrc, hi, lo, mom, dst, ndst, n, lr, mu, wd);
  else
    push_update_kernel<false><<<grid, 256, 0, s>>>(src, nsrc, hi, lo, mom, dst, ndst, n, lr, mu, wd);
  SPB_CUDA(cudaGetLastError());
}

void launch_push_split(const float* w32, float* hi, float* lo, long n, long hole0, long hole1, cudaStream_t s) {
  if (n - (hole1 - hole0) <= 0) return;
  if (n % 4 == 0 && hole0 % 4 == 0 && hole1 % 4 == 0 && aligned16(w32) && aligned16(hi) && aligned16(lo))
    return launch_p2p_split(w32, hi, lo, n, hole0, hole1, s);
  const int grid = static_cast<int>(std::max<long>(1, std::min<long>((n + 255) / 256, 148L * 8)));
  push_split_kernel<<<grid, 256, 0, s>>>(w32, hi, lo, n, hole0, hole1);
  SPB_CUDA(cudaGetLastError());
}

}  // namespace spb
