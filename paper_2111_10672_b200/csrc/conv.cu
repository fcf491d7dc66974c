// Data-movement kernels of the convolutional SPB model (ConvNet, engine.cu):
// the GEMM work (forward, wgrad, dgrad) runs on the same tcgen05 3xTF32
// kernels as the MLP; these kernels lower the 3x3 convolutions onto them.
//
// Layout: activations NHWC, one GEMM row per pixel ([samples * h * w, ld(c)],
// split pairs hi + lo). im2col rows: [samples * h_out * w_out, ld(9 c_in)],
// column (ky * 3 + kx) * c_in + ci. Padding 1, stride 1 or 2.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <stdexcept>

#include "conv.hpp"
#include "launch.hpp"

namespace spb {
namespace {

__device__ __forceinline__ float tf32r(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__device__ __forceinline__ uint64_t mix64(uint64_t a, uint64_t b) {  // rng.hpp:47-53
  uint64_t z = a ^ (b + 0x9E3779B97F4A7C15ULL + (a << 6) + (a >> 2));
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// One block per sample slot: draw (or take) the sample index, copy its
// h*w*c NHWC image into pixel rows of H0 (split pair, row stride ldh) and its
// target into ybatch.
__global__ void conv_gather_kernel(const float* __restrict__ X, long ldx, const float* __restrict__ Y, int pix, int c0,
                                   int nout, int N, int bw, const int* __restrict__ workers,
                                   const uint64_t* __restrict__ seed_dev, uint64_t seed_host,
                                   const int* __restrict__ step_dev, int step_host, const int* __restrict__ idx_in,
                                   int* __restrict__ idx_out, float* __restrict__ h_hi, float* __restrict__ h_lo,
                                   long ldh, float* __restrict__ ybatch) {
  const int r = blockIdx.x;
  int idx;
  if (idx_in) {
    idx = idx_in[r];
  } else {  // Rng(seed).split(step).split(worker), draw r % bw (same as gather_kernel)
    const int step = step_dev ? *step_dev : step_host;
    const uint64_t seed = seed_dev ? *seed_dev : seed_host;
    const uint64_t key = mix64(mix64(seed, static_cast<uint64_t>(step)), static_cast<uint64_t>(workers[r / bw]));
    const uint64_t u = mix64(key, static_cast<uint64_t>(r % bw) + 1);
    idx = static_cast<int>(__umul64hi(u, static_cast<uint64_t>(N)));
  }
  if (threadIdx.x == 0 && idx_out) idx_out[r] = idx;
  const float* src = X + static_cast<long>(idx) * ldx;
  const long base = static_cast<long>(r) * pix;
  for (int e = threadIdx.x; e < pix * c0; e += blockDim.x) {
    const int p = e / c0, c = e - p * c0;
    const float v = src[e];
    const float h = tf32r(v);
    h_hi[(base + p) * ldh + c] = h;
    h_lo[(base + p) * ldh + c] = v - h;
  }
  if (threadIdx.x < nout) ybatch[r * nout + threadIdx.x] = Y[static_cast<long>(idx) * nout + threadIdx.x];
}

// Flat over (output row, tap, channel vector): consecutive threads move
// consecutive VEC-channel vectors, coalesced on both sides. VEC = 4 when
// c_in % 4 == 0 (every layer but the RGB input).
template <int VEC>
__global__ void __launch_bounds__(256) im2col_kernel(const float* __restrict__ in_hi, const float* __restrict__ in_lo,
                                                     long ldin, ConvGeom g, long row0, long rows,
                                                     float* __restrict__ col_hi, float* __restrict__ col_lo, long ldk) {
  const int cv = g.c_in / VEC;
  const long total = rows * 9 * cv;
  const int opix = g.out_h * g.out_w;
  for (long t = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
       t += static_cast<long>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(t % cv);
    const long rt = t / cv;
    const int tap = static_cast<int>(rt % 9);
    const long orow = row0 + rt / 9;
    const long s = orow / opix;
    const int rem = static_cast<int>(orow - s * opix);
    const int oy = rem / g.out_w, ox = rem - oy * g.out_w;
    const int ky = tap / 3, kx = tap - ky * 3;
    const int iy = oy * g.stride + ky - 1, ix = ox * g.stride + kx - 1;
    const bool inside = iy >= 0 && iy < g.in_h && ix >= 0 && ix < g.in_w;
    const long src = ((s * g.in_h + iy) * g.in_w + ix) * ldin + c * VEC;
    const long dst = orow * ldk + tap * g.c_in + c * VEC;
    if constexpr (VEC == 4) {
      const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
      *reinterpret_cast<float4*>(col_hi + dst) = inside ? *reinterpret_cast<const float4*>(in_hi + src) : z;
      *reinterpret_cast<float4*>(col_lo + dst) = inside ? *reinterpret_cast<const float4*>(in_lo + src) : z;
    } else {
      col_hi[dst] = inside ? in_hi[src] : 0.f;
      col_lo[dst] = inside ? in_lo[src] : 0.f;
    }
  }
}

// Delta_{l-1}[(s, y, x), ci] = (1 - H^2) * sum over taps of dcol[(s, oy, ox),
// tap * c_in + ci] for the output pixels (oy, ox) whose window covers (y, x);
// fixed tap order (deterministic). Flat over (input row, channel vector).
template <int VEC>
__global__ void __launch_bounds__(256) col2im_tanh_kernel(const float* __restrict__ dcol, long ldk, ConvGeom g,
                                                          long row0, long rows, const float* __restrict__ h_hi,
                                                          const float* __restrict__ h_lo, long ldh,
                                                          float* __restrict__ d_hi, float* __restrict__ d_lo,
                                                          long ldd) {
  const int cv = g.c_in / VEC;
  const long total = rows * cv;
  const int ipix = g.in_h * g.in_w;
  for (long t = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
       t += static_cast<long>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(t % cv);
    const long irow = row0 + t / cv;
    const long s = irow / ipix;
    const int rem = static_cast<int>(irow - s * ipix);
    const int y = rem / g.in_w, x = rem - y * g.in_w;
    float acc[VEC];
#pragma unroll
    for (int v = 0; v < VEC; ++v) acc[v] = 0.f;
    for (int ky = 0; ky < 3; ++ky) {
      const int ty = y + 1 - ky;
      if (ty < 0 || ty % g.stride) continue;
      const int oy = ty / g.stride;
      if (oy >= g.out_h) continue;
      for (int kx = 0; kx < 3; ++kx) {
        const int tx = x + 1 - kx;
        if (tx < 0 || tx % g.stride) continue;
        const int ox = tx / g.stride;
        if (ox >= g.out_w) continue;
        const float* src = dcol + ((s * g.out_h + oy) * g.out_w + ox) * ldk + (ky * 3 + kx) * g.c_in + c * VEC;
        if constexpr (VEC == 4) {
          const float4 q = *reinterpret_cast<const float4*>(src);
          acc[0] += q.x, acc[1] += q.y, acc[2] += q.z, acc[3] += q.w;
        } else {
          acc[0] += src[0];
        }
      }
    }
    const long at = irow * ldh + c * VEC, ad = irow * ldd + c * VEC;
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      const float h = h_hi[at + v] + h_lo[at + v];
      const float r = acc[v] * (1.0f - h * h);
      const float rh = tf32r(r);
      d_hi[ad + v] = rh;
      d_lo[ad + v] = r - rh;
    }
  }
}

// Wf[ci, (ky*3 + kx) * c_out + co] = W[co, ((2-ky)*3 + (2-kx)) * c_in + ci]
// for both halves of the split pair (a permutation: exact).
__global__ void conv_flip_kernel(const float* __restrict__ w_hi, const float* __restrict__ w_lo, long ldw, int c_out,
                                 int c_in, float* __restrict__ f_hi, float* __restrict__ f_lo, long ldf) {
  const long total = static_cast<long>(c_in) * 9 * c_out;
  for (long t = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
       t += static_cast<long>(gridDim.x) * blockDim.x) {
    const int co = static_cast<int>(t % c_out);
    const long r = t / c_out;
    const int tap = static_cast<int>(r % 9), ci = static_cast<int>(r / 9);
    const long src = static_cast<long>(co) * ldw + (8 - tap) * c_in + ci;
    const long dst = static_cast<long>(ci) * ldf + tap * c_out + co;
    f_hi[dst] = w_hi[src];
    f_lo[dst] = w_lo[src];
  }
}

// Direct 3x3 convolution of a narrow input (c_in <= 4, stored 4-wide: the RGB
// layer), the forward of a layer whose im2col GEMM would have K = 27: one
// thread per output pixel computes all c_out (<= kDirectMaxOut) channels in
// fp32 FMAs over the 9 taps x c_in inputs, with x = hi + lo and w = hi + lo
// (both exact), then bias + tanh + split like the GEMM's forward epilogue.
// The 9 taps are loaded up front (18 independent 16-byte loads); the weights
// sit in shared memory tap-major ([9 * 4][c_out]) and are read as warp-wide
// broadcasts; each warp stages its 32 output rows in shared memory so the
// stores are contiguous 512-byte runs. Memory-bound on the split output
// (8 B per output element), where the im2col GEMM wrote 9 c_in columns first
// and then ran a K = 32 GEMM at a few % of the tensor peak.
constexpr int kDirectMaxOut = 64;
constexpr int kDirectThreads = 128;
constexpr int kDirectPad = kDirectMaxOut + 4;  // staging row stride (floats)

template <int CIN>
__global__ void __launch_bounds__(kDirectThreads, 3) conv_direct_fwd_kernel(
    const float* __restrict__ in_hi, const float* __restrict__ in_lo, long ldin, ConvGeom g, long rows,
    const float* __restrict__ w_hi, const float* __restrict__ w_lo, long ldw, const float* __restrict__ b_hi,
    const float* __restrict__ b_lo, float* __restrict__ o_hi, float* __restrict__ o_lo, long ldo) {
  // [36][kDirectMaxOut] weights (tap * 4 + c; zero for c >= c_in), [kDirectMaxOut] bias,
  // then per warp a [32][kDirectPad] staging tile.
  extern __shared__ __align__(16) float ws[];
  float* bias = ws + 36 * kDirectMaxOut;
  const int C = g.c_out;
  for (int i = threadIdx.x; i < 36 * kDirectMaxOut; i += blockDim.x) {
    const int k = i / kDirectMaxOut, co = i - k * kDirectMaxOut;
    const int tap = k >> 2, c = k & 3;
    const long at = static_cast<long>(co) * ldw + tap * g.c_in + c;
    ws[i] = (co < C && c < g.c_in) ? w_hi[at] + w_lo[at] : 0.f;
  }
  for (int co = threadIdx.x; co < kDirectMaxOut; co += blockDim.x) bias[co] = co < C ? b_hi[co] + b_lo[co] : 0.f;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* stage = bias + kDirectMaxOut + warp * 32 * kDirectPad;
  const int opix = g.out_h * g.out_w;
  const long step = static_cast<long>(gridDim.x) * blockDim.x;
  for (long base = static_cast<long>(blockIdx.x) * blockDim.x + warp * 32; base < rows; base += step) {
    const long r = base + lane;
    const bool live = r < rows;
    float x[9 * CIN];
    {
      const long s = live ? r / opix : 0;
      const int rem = live ? static_cast<int>(r - s * opix) : 0;
      const int oy = rem / g.out_w, ox = rem - oy * g.out_w;
#pragma unroll
      for (int tap = 0; tap < 9; ++tap) {
        const int iy = oy * g.stride + tap / 3 - 1, ix = ox * g.stride + tap % 3 - 1;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (live && iy >= 0 && iy < g.in_h && ix >= 0 && ix < g.in_w) {  // else zero padding
          const long src = ((s * g.in_h + iy) * g.in_w + ix) * ldin;
          const float4 h = *reinterpret_cast<const float4*>(in_hi + src);
          const float4 l = *reinterpret_cast<const float4*>(in_lo + src);
          v = make_float4(h.x + l.x, h.y + l.y, h.z + l.z, h.w + l.w);
        }
        const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int c = 0; c < CIN; ++c) x[tap * CIN + c] = vv[c];
      }
    }
    float acc[kDirectMaxOut];
#pragma unroll
    for (int j = 0; j < kDirectMaxOut; ++j) acc[j] = bias[j];
#pragma unroll
    for (int tap = 0; tap < 9; ++tap) {
#pragma unroll
      for (int c = 0; c < CIN; ++c) {  // the 4th (padding) channel of an RGB input is skipped
        const float xc = x[tap * CIN + c];
        const float* wk = ws + (tap * 4 + c) * kDirectMaxOut;
#pragma unroll
        for (int j = 0; j < kDirectMaxOut; j += 4) {
          const float4 w4 = *reinterpret_cast<const float4*>(wk + j);
          acc[j] = fmaf(xc, w4.x, acc[j]);
          acc[j + 1] = fmaf(xc, w4.y, acc[j + 1]);
          acc[j + 2] = fmaf(xc, w4.z, acc[j + 2]);
          acc[j + 3] = fmaf(xc, w4.w, acc[j + 3]);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < kDirectMaxOut; ++j) acc[j] = tanhf(acc[j]);
    // hi then lo through the staging tile: lane-row writes, then the warp
    // stores its 32 rows x C channels as contiguous float4 runs.
    const int n = static_cast<int>(rows - base < 32 ? rows - base : 32);
    const int cv = C / 4;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
#pragma unroll
      for (int j = 0; j < kDirectMaxOut; j += 4) {
        float4 v;
        float* vp = &v.x;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float h = tf32r(acc[j + q]);
          vp[q] = half == 0 ? h : acc[j + q] - h;
        }
        *reinterpret_cast<float4*>(stage + lane * kDirectPad + j) = v;
      }
      __syncwarp();
      float* out = half == 0 ? o_hi : o_lo;
      for (int e = lane; e < n * cv; e += 32) {
        const int row = e / cv, q = e - row * cv;
        *reinterpret_cast<float4*>(out + (base + row) * ldo + 4 * q) =
            *reinterpret_cast<const float4*>(stage + row * kDirectPad + 4 * q);
      }
      __syncwarp();
    }
  }
}

int flat_grid(long total) { return static_cast<int>(std::max<long>(1, std::min<long>((total + 255) / 256, 148L * 16))); }

// pooled[s, c] = mean over the pix pixel rows of sample s (split pair out).
__global__ void avgpool_kernel(const float* __restrict__ h_hi, const float* __restrict__ h_lo, long ldh, int pix,
                               int c, float* __restrict__ p_hi, float* __restrict__ p_lo, long ldp) {
  const int s = blockIdx.x;
  const float inv = 1.0f / static_cast<float>(pix);
  for (int ch = threadIdx.x; ch < c; ch += blockDim.x) {
    float acc = 0.f;
    for (int p = 0; p < pix; ++p) {
      const long r = static_cast<long>(s) * pix + p;
      acc += h_hi[r * ldh + ch] + h_lo[r * ldh + ch];
    }
    const float v = acc * inv;
    const float vh = tf32r(v);
    p_hi[static_cast<long>(s) * ldp + ch] = vh;
    p_lo[static_cast<long>(s) * ldp + ch] = v - vh;
  }
}

// Delta[(s, p), c] = g[s, c] / pix * (1 - H[(s, p), c]^2) for samples >= s0.
__global__ void unpool_tanh_kernel(const float* __restrict__ g_hi, const float* __restrict__ g_lo, long ldg, int pix,
                                   int c, int s0, const float* __restrict__ h_hi, const float* __restrict__ h_lo,
                                   long ldh, float* __restrict__ d_hi, float* __restrict__ d_lo, long ldd) {
  const long r = static_cast<long>(s0) * pix + blockIdx.x;
  const long s = r / pix;
  const float inv = 1.0f / static_cast<float>(pix);
  for (int ch = threadIdx.x; ch < c; ch += blockDim.x) {
    const float gv = (g_hi[s * ldg + ch] + g_lo[s * ldg + ch]) * inv;
    const float h = h_hi[r * ldh + ch] + h_lo[r * ldh + ch];
    const float v = gv * (1.0f - h * h);
    const float vh = tf32r(v);
    d_hi[r * ldd + ch] = vh;
    d_lo[r * ldd + ch] = v - vh;
  }
}

int threads_for(int c) { return c >= 256 ? 256 : (c >= 128 ? 128 : (c >= 64 ? 64 : 32)); }

}  // namespace

void launch_conv_gather(const float* X, long ldx, const float* Y, int pix, int c0, int nout, int N, int samples, int bw,
                        const int* workers, const uint64_t* seed_dev, uint64_t seed_host, const int* step_dev,
                        int step_host, const int* idx_in, int* idx_out, float* h_hi, float* h_lo, long ldh,
                        float* ybatch, cudaStream_t s) {
  if (samples <= 0) return;
  conv_gather_kernel<<<samples, 256, 0, s>>>(X, ldx, Y, pix, c0, nout, N, bw, workers, seed_dev, seed_host, step_dev,
                                             step_host, idx_in, idx_out, h_hi, h_lo, ldh, ybatch);
  SPB_CUDA(cudaGetLastError());
}

void launch_im2col(const float* in_hi, const float* in_lo, long ldin, const ConvGeom& g, int row0, int rows,
                   float* col_hi, float* col_lo, long ldk, cudaStream_t s) {
  if (rows <= 0) return;
  if (g.c_in % 4 == 0 && ldin % 4 == 0 && ldk % 4 == 0)
    im2col_kernel<4><<<flat_grid(static_cast<long>(rows) * 9 * (g.c_in / 4)), 256, 0, s>>>(in_hi, in_lo, ldin, g, row0,
                                                                                          rows, col_hi, col_lo, ldk);
  else
    im2col_kernel<1><<<flat_grid(static_cast<long>(rows) * 9 * g.c_in), 256, 0, s>>>(in_hi, in_lo, ldin, g, row0, rows,
                                                                                   col_hi, col_lo, ldk);
  SPB_CUDA(cudaGetLastError());
}

bool conv_direct_ok(const ConvGeom& g, long ldin, long ldo) {
  return g.c_in <= 4 && ldin == 4 && g.c_out <= kDirectMaxOut && g.c_out % 4 == 0 && ldo % 4 == 0;
}

void launch_conv_direct_fwd(const float* in_hi, const float* in_lo, long ldin, const ConvGeom& g, long rows,
                            const float* w_hi, const float* w_lo, long ldw, const float* b_hi, const float* b_lo,
                            float* o_hi, float* o_lo, long ldo, cudaStream_t s) {
  if (rows <= 0) return;
  if (!conv_direct_ok(g, ldin, ldo)) throw std::invalid_argument("conv_direct_fwd: unsupported geometry");
  const int smem = static_cast<int>((37 * kDirectMaxOut + (kDirectThreads / 32) * 32 * kDirectPad) * sizeof(float));
  static_assert((37 * kDirectMaxOut + (kDirectThreads / 32) * 32 * kDirectPad) * sizeof(float) <= 48 * 1024,
                "conv_direct_fwd: static shared-memory budget");
  const int grid = static_cast<int>(std::max<long>(1, std::min<long>((rows + kDirectThreads - 1) / kDirectThreads,
                                                                     148L * 3)));
  auto kern = g.c_in == 3 ? conv_direct_fwd_kernel<3>
                          : (g.c_in == 4 ? conv_direct_fwd_kernel<4>
                                         : (g.c_in == 2 ? conv_direct_fwd_kernel<2> : conv_direct_fwd_kernel<1>));
  kern<<<grid, kDirectThreads, smem, s>>>(in_hi, in_lo, ldin, g, rows, w_hi, w_lo, ldw, b_hi, b_lo, o_hi, o_lo, ldo);
  SPB_CUDA(cudaGetLastError());
}

void launch_col2im_tanh(const float* dcol, long ldk, const ConvGeom& g, int row0, int rows, const float* h_hi,
                        const float* h_lo, long ldh, float* d_hi, float* d_lo, long ldd, cudaStream_t s) {
  if (rows <= 0) return;
  if (g.c_in % 4 == 0 && ldk % 4 == 0)
    col2im_tanh_kernel<4><<<flat_grid(static_cast<long>(rows) * (g.c_in / 4)), 256, 0, s>>>(
        dcol, ldk, g, row0, rows, h_hi, h_lo, ldh, d_hi, d_lo, ldd);
  else
    col2im_tanh_kernel<1><<<flat_grid(static_cast<long>(rows) * g.c_in), 256, 0, s>>>(dcol, ldk, g, row0, rows, h_hi,
                                                                                    h_lo, ldh, d_hi, d_lo, ldd);
  SPB_CUDA(cudaGetLastError());
}

void launch_conv_flip(const float* w_hi, const float* w_lo, long ldw, int c_out, int c_in, float* f_hi, float* f_lo,
                      long ldf, cudaStream_t s) {
  const long total = static_cast<long>(c_in) * 9 * c_out;
  conv_flip_kernel<<<flat_grid(total), 256, 0, s>>>(w_hi, w_lo, ldw, c_out, c_in, f_hi, f_lo, ldf);
  SPB_CUDA(cudaGetLastError());
}

void launch_avgpool(const float* h_hi, const float* h_lo, long ldh, int samples, int pix, int c, float* p_hi,
                    float* p_lo, long ldp, cudaStream_t s) {
  if (samples <= 0) return;
  avgpool_kernel<<<samples, threads_for(c), 0, s>>>(h_hi, h_lo, ldh, pix, c, p_hi, p_lo, ldp);
  SPB_CUDA(cudaGetLastError());
}

void launch_unpool_tanh(const float* g_hi, const float* g_lo, long ldg, int samples, int s0, int pix, int c,
                        const float* h_hi, const float* h_lo, long ldh, float* d_hi, float* d_lo, long ldd,
                        cudaStream_t s) {
  const long rows = static_cast<long>(samples - s0) * pix;
  if (rows <= 0) return;
  unpool_tanh_kernel<<<static_cast<unsigned>(rows), threads_for(c), 0, s>>>(g_hi, g_lo, ldg, pix, c, s0, h_hi, h_lo,
                                                                             ldh, d_hi, d_lo, ldd);
  SPB_CUDA(cudaGetLastError());
}

}  // namespace spb
