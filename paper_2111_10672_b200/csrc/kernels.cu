// Non-GEMM kernels of the SPB step: dataset gather with the on-device
// counter-based Rng, the fused output head, the optimizer update, and the
// per-layer contributor averages of the aggregator entry points (fp32, and
// fp64 with the reference's exact operation order). The bias / head gradient
// reductions of round 1 now live inside the wgrad GEMMs (gemm_tf32x3.cuh).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <stdexcept>

#include "launch.hpp"
#include "ptx.cuh"

namespace spb {
namespace {

// rng.hpp:47-53, bit-exact.
__device__ __forceinline__ uint64_t rng_mix(uint64_t a, uint64_t b) {
  uint64_t z = a ^ (b + 0x9E3779B97F4A7C15ULL + (a << 6) + (a >> 2));
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// One CTA per row: draw (or read) the sample index, split its input row into
// the H0 pair and copy its target row.
__global__ void gather_kernel(const float* __restrict__ X, long ldx, const float* __restrict__ Y, int n0, int nout,
                              int N, int bw, const int* __restrict__ workers, const uint64_t* __restrict__ seed_dev,
                              uint64_t seed_host, const int* __restrict__ step_dev, int step_host, const int* __restrict__ idx_in,
                              int* __restrict__ idx_out, float* __restrict__ h_hi, float* __restrict__ h_lo,
                              long ldh, float* __restrict__ ybatch) {
  const int r = blockIdx.x;
  int idx;
  if (idx_in) {
    idx = idx_in[r];
  } else {
    // Rng(seed).split(step).split(worker): keys chain through mix
    // (rng.hpp:18); draw p is next_u64 at counter p+1 (rng.hpp:20) and
    // next_below is the high half of the 128-bit product (rng.hpp:26-29).
    const int step = step_dev ? *step_dev : step_host;
    const uint64_t seed = seed_dev ? *seed_dev : seed_host;
    const uint64_t key = rng_mix(rng_mix(seed, static_cast<uint64_t>(step)), static_cast<uint64_t>(workers[r / bw]));
    const uint64_t u = rng_mix(key, static_cast<uint64_t>(r % bw) + 1);
    idx = static_cast<int>(__umul64hi(u, static_cast<uint64_t>(N)));
  }
  if (threadIdx.x == 0 && idx_out) idx_out[r] = idx;
  const float* src = X + idx * ldx;
  float* dh = h_hi + r * ldh;
  float* dl = h_lo + r * ldh;
  for (int c = threadIdx.x; c < n0; c += blockDim.x) {
    const float v = src[c];
    const float h = tf32_rna(v);
    dh[c] = h;
    dl[c] = v - h;
  }
  if (threadIdx.x < nout) ybatch[r * nout + threadIdx.x] = Y[static_cast<long>(idx) * nout + threadIdx.x];
}

__global__ void split_rows_kernel(const float* __restrict__ x, long ldx, int cols, float* __restrict__ hi,
                                  float* __restrict__ lo, long ld) {
  const int r = blockIdx.x;
  for (int c = threadIdx.x; c < cols; c += blockDim.x) {
    const float v = x[r * ldx + c];
    const float h = tf32_rna(v);
    hi[r * ld + c] = h;
    lo[r * ld + c] = v - h;
  }
}

constexpr int kMaxOut = 16;

// One warp per row (model.cpp:121-126 for layer L, :156 for the output
// delta, :172-183 for the delta entering layer L-1). Rows are read as float4
// over the padded width ld (padding columns of H and W are zero), 4 chunks per
// lane in flight.
__global__ void head_kernel(const float* __restrict__ h_hi, const float* __restrict__ h_lo, long ldh, int rows,
                            int n_in, int n_out, const float* __restrict__ w_hi, const float* __restrict__ w_lo,
                            long ldw, const float* __restrict__ b_hi, const float* __restrict__ b_lo,
                            const float* __restrict__ y, float* __restrict__ delta, float* __restrict__ delta_lo,
                            long ldq, float* __restrict__ row_loss, float* __restrict__ dn_hi,
                            float* __restrict__ dn_lo, long ldd, int cont_row0, int tanh_out, int dn_act) {
  const int warps = blockDim.x / 32;
  const int r = blockIdx.x * warps + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const int n4 = static_cast<int>((n_in + 3) / 4);
  const float4* hh = reinterpret_cast<const float4*>(h_hi + r * ldh);
  const float4* hl = reinterpret_cast<const float4*>(h_lo + r * ldh);
  float acc[kMaxOut];
#pragma unroll
  for (int o = 0; o < kMaxOut; ++o) acc[o] = 0.f;
#pragma unroll 4
  for (int c = lane; c < n4; c += 32) {
    const float4 a = hh[c], b = hl[c];
    const float4 h = make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
#pragma unroll
    for (int o = 0; o < kMaxOut; ++o) {
      if (o >= n_out) break;
      const float4 wa = __ldg(reinterpret_cast<const float4*>(w_hi + o * ldw) + c);
      const float4 wb = __ldg(reinterpret_cast<const float4*>(w_lo + o * ldw) + c);
      acc[o] = fmaf(wa.x + wb.x, h.x, acc[o]);
      acc[o] = fmaf(wa.y + wb.y, h.y, acc[o]);
      acc[o] = fmaf(wa.z + wb.z, h.z, acc[o]);
      acc[o] = fmaf(wa.w + wb.w, h.w, acc[o]);
    }
  }
  float d[kMaxOut];
  float loss = 0.f;
#pragma unroll
  for (int o = 0; o < kMaxOut; ++o) {
    d[o] = 0.f;
    if (o < n_out) {
      float z = warp_sum(acc[o]) + (b_hi[o] + b_lo[o]);
      if (tanh_out) z = tanhf(z);
      d[o] = z - y[r * n_out + o];
      loss += 0.5f * d[o] * d[o];
    }
  }
  if (lane == 0) {  // delta_L as a split pair (the head wgrad GEMM's A operand), row stride ldq
    for (int o = 0; o < n_out; ++o) {
      const float dh = tf32_rna(d[o]);
      delta[r * ldq + o] = dh;
      delta_lo[r * ldq + o] = d[o] - dh;
    }
    row_loss[r] = loss;
  }
  if (dn_hi && r >= cont_row0) {
    float4* oh = reinterpret_cast<float4*>(dn_hi + r * ldd);
    float4* ol = reinterpret_cast<float4*>(dn_lo + r * ldd);
#pragma unroll 4
    for (int c = lane; c < n4; c += 32) {
      float4 sv = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int o = 0; o < kMaxOut; ++o) {
        if (o >= n_out) break;
        const float4 wa = __ldg(reinterpret_cast<const float4*>(w_hi + o * ldw) + c);
        const float4 wb = __ldg(reinterpret_cast<const float4*>(w_lo + o * ldw) + c);
        sv.x = fmaf(d[o], wa.x + wb.x, sv.x);
        sv.y = fmaf(d[o], wa.y + wb.y, sv.y);
        sv.z = fmaf(d[o], wa.z + wb.z, sv.z);
        sv.w = fmaf(d[o], wa.w + wb.w, sv.w);
      }
      const float4 a = hh[c], b = hl[c];
      float v[4] = {sv.x, sv.y, sv.z, sv.w};
      if (dn_act) {
        v[0] *= 1.0f - (a.x + b.x) * (a.x + b.x);
        v[1] *= 1.0f - (a.y + b.y) * (a.y + b.y);
        v[2] *= 1.0f - (a.z + b.z) * (a.z + b.z);
        v[3] *= 1.0f - (a.w + b.w) * (a.w + b.w);
      }
      const float4 vh = make_float4(tf32_rna(v[0]), tf32_rna(v[1]), tf32_rna(v[2]), tf32_rna(v[3]));
      oh[c] = vh;
      ol[c] = make_float4(v[0] - vh.x, v[1] - vh.y, v[2] - vh.z, v[3] - vh.w);
    }
  }
}


// Fused optimizer over the flat parameter pair, float4-vectorised, grid-stride:
//   w = hi + lo; g' = g + wd*w; buf = mu*buf + g' (when mu != 0); w -= lr*buf
//   hi = rna_tf32(w); lo = w - hi  (the split the next forward's GEMMs read)
// With mu = wd = 0 this is the reference's x -= gamma*g (spb.cpp:196). The
// first momentum step sees buf = 0, so buf = g' exactly as in PyTorch SGD.
// <= 32 registers (launch bounds) so one block can sit beside a 1-CTA GEMM
// CTA on the same SM and stream the update while the GEMMs run.
__global__ void __launch_bounds__(256, 8) sgd_update_kernel(float4* __restrict__ p_hi, float4* __restrict__ p_lo,
                                  const float4* __restrict__ grad, float4* __restrict__ mom, long n4, float lr,
                                  float mu, float wd) {
  const long stride = static_cast<long>(gridDim.x) * blockDim.x;
  for (long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride) {
    const float4 h = p_hi[i], l = p_lo[i], g = __ldg(&grad[i]);
    float w[4] = {h.x + l.x, h.y + l.y, h.z + l.z, h.w + l.w};
    float gg[4] = {g.x, g.y, g.z, g.w};
    if (wd != 0.f) {
#pragma unroll
      for (int j = 0; j < 4; ++j) gg[j] = fmaf(wd, w[j], gg[j]);
    }
    if (mom) {
      float4 b = mom[i];
      float bb[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        bb[j] = fmaf(mu, bb[j], gg[j]);
        gg[j] = bb[j];
      }
      mom[i] = make_float4(bb[0], bb[1], bb[2], bb[3]);
    }
    float nh[4], nl[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float wn = w[j] - lr * gg[j];
      nh[j] = tf32_rna(wn);
      nl[j] = wn - nh[j];
    }
    p_hi[i] = make_float4(nh[0], nh[1], nh[2], nh[3]);
    p_lo[i] = make_float4(nl[0], nl[1], nl[2], nl[3]);
  }
}

__global__ void aggregate_kernel(const float* const* __restrict__ srcs, int m, long n, float* __restrict__ out) {
  const long stride = static_cast<long>(gridDim.x) * blockDim.x;
  const double inv = 1.0 / static_cast<double>(m);
  for (long c = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; c < n; c += stride) {
    double s = 0.0;
    for (int w = 0; w < m; ++w) s += static_cast<double>(srcs[w][c]);
    out[c] = static_cast<float>(s * inv);
  }
}

// fp64 aggregate with the reference's exact operation sequence (spb.cpp:97-103):
// dst += src for the contributors in ascending worker order, then dst *= inv
// (inv = 1.0 / m from the host); explicit round-to-nearest ops, no FMA
// contraction, so results are bit-identical to the CPU code.
__global__ void aggregate64_kernel(const double* const* __restrict__ srcs, int m, long n, double inv,
                                   double* __restrict__ out) {
  const long stride = static_cast<long>(gridDim.x) * blockDim.x;
  for (long c = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; c < n; c += stride) {
    double s = 0.0;
    for (int w = 0; w < m; ++w) s = __dadd_rn(s, srcs[w][c]);
    out[c] = __dmul_rn(s, inv);
  }
}

__global__ void split_kernel(const float* __restrict__ in, long n, float* __restrict__ hi, float* __restrict__ lo) {
  const long stride = static_cast<long>(gridDim.x) * blockDim.x;
  for (long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const float v = in[i], h = tf32_rna(v);
    hi[i] = h;
    lo[i] = v - h;
  }
}

__global__ void join_kernel(const float* __restrict__ hi, const float* __restrict__ lo, long n, float* __restrict__ out) {
  const long stride = static_cast<long>(gridDim.x) * blockDim.x;
  for (long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) out[i] = hi[i] + lo[i];
}

// Deterministic single-CTA sum of the per-row losses (warp-shuffle tree).
__global__ void sum_loss_kernel(const float* __restrict__ row_loss, int rows, float scale, float* __restrict__ out,
                                int* step_dev) {
  if (step_dev && threadIdx.x == 0) *step_dev += 1;  // the gather already read this step's Rng stream
  __shared__ float part[32];
  float s = 0.f;
  for (int r = threadIdx.x; r < rows; r += blockDim.x) s += row_loss[r];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x / 32] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < blockDim.x / 32 ? part[threadIdx.x] : 0.f;
    v = warp_sum(v);
    if (threadIdx.x == 0) *out = v * scale;
  }
}

int grid_for(long n, int threads) {
  long b = (n + threads - 1) / threads;
  long cap = 148L * 8;
  return static_cast<int>(b < 1 ? 1 : (b > cap ? cap : b));
}

}  // namespace

void launch_gather(const float* X, long ldx, const float* Y, int n0, int nout, int N, int rows, int bw,
                   const int* workers, const uint64_t* seed_dev, uint64_t seed_host, const int* step_dev,
                   int step_host, const int* idx_in, int* idx_out, float* h_hi, float* h_lo, long ldh, float* ybatch,
                   cudaStream_t s) {
  if (rows <= 0) return;
  gather_kernel<<<rows, 256, 0, s>>>(X, ldx, Y, n0, nout, N, bw, workers, seed_dev, seed_host, step_dev, step_host,
                                     idx_in, idx_out,
                                     h_hi, h_lo, ldh, ybatch);
  SPB_CUDA(cudaGetLastError());
}

void launch_split_rows(const float* x, long ldx_in, int rows, int cols, float* hi, float* lo, long ld,
                       cudaStream_t s) {
  if (rows <= 0) return;
  split_rows_kernel<<<rows, 256, 0, s>>>(x, ldx_in, cols, hi, lo, ld);
  SPB_CUDA(cudaGetLastError());
}

void launch_head(const float* h_hi, const float* h_lo, long ldh, int rows, int n_in, int n_out, const float* w_hi,
                 const float* w_lo, long ldw, const float* b_hi, const float* b_lo, const float* y, float* delta,
                 float* delta_lo, long ldq, float* row_loss, float* dn_hi, float* dn_lo, long ldd, int cont_row0,
                 bool tanh_out, cudaStream_t s, bool dn_act) {
  if (rows <= 0) return;
  if (n_out > kMaxOut) throw std::invalid_argument("head: n_out > 16");
  const int warps = 8;
  head_kernel<<<(rows + warps - 1) / warps, warps * 32, 0, s>>>(h_hi, h_lo, ldh, rows, n_in, n_out, w_hi, w_lo, ldw,
                                                                b_hi, b_lo, y, delta, delta_lo, ldq, row_loss, dn_hi,
                                                                dn_lo, ldd,
                                                                cont_row0, tanh_out ? 1 : 0, dn_act ? 1 : 0);
  SPB_CUDA(cudaGetLastError());
}

void launch_sgd_update(float* p_hi, float* p_lo, const float* grad, float* mom, long n, float lr, float momentum,
                       float wd, cudaStream_t s, int ctas) {
  if (n % 4) throw std::invalid_argument("update: n must be a multiple of 4");
  const long n4 = n / 4;
  sgd_update_kernel<<<ctas > 0 ? ctas : grid_for(n4, 256), 256, 0, s>>>(
      reinterpret_cast<float4*>(p_hi), reinterpret_cast<float4*>(p_lo), reinterpret_cast<const float4*>(grad),
      reinterpret_cast<float4*>(mom), n4, lr, momentum, wd);
  SPB_CUDA(cudaGetLastError());
}

// out[slot] += sum_i (a_i - b_i)^2 over [0, n), fp64 accumulation
// (block_distance_sq, spb.cpp:110-118).
__global__ void __launch_bounds__(256) sqdist_kernel(const float* __restrict__ a, const float* __restrict__ b, long n4,
                                                     double* __restrict__ out) {
  double acc = 0.0;
  const long stride = static_cast<long>(gridDim.x) * blockDim.x;
  for (long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride) {
    const float4 x = reinterpret_cast<const float4*>(a)[i];
    const float4 y = reinterpret_cast<const float4*>(b)[i];
    const double d0 = static_cast<double>(x.x) - y.x, d1 = static_cast<double>(x.y) - y.y;
    const double d2 = static_cast<double>(x.z) - y.z, d3 = static_cast<double>(x.w) - y.w;
    acc += d0 * d0 + d1 * d1 + d2 * d2 + d3 * d3;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  __shared__ double part[8];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += part[w];
    atomicAdd(out, t);
  }
}

void launch_sqdist(const float* a, const float* b, long n, double* out, cudaStream_t s) {
  if (n <= 0) return;
  if (n % 4) throw std::invalid_argument("sqdist: n must be a multiple of 4");
  sqdist_kernel<<<static_cast<int>(std::min<long>((n / 4 + 255) / 256, 148L * 4)), 256, 0, s>>>(a, b, n / 4, out);
  SPB_CUDA(cudaGetLastError());
}

void launch_aggregate(const float* const* srcs_dev, int m, long n, float* out, cudaStream_t s) {
  if (n <= 0) return;
  aggregate_kernel<<<grid_for(n, 256), 256, 0, s>>>(srcs_dev, m, n, out);
  SPB_CUDA(cudaGetLastError());
}

void launch_aggregate64(const double* const* srcs_dev, int m, long n, double* out, cudaStream_t s) {
  if (n <= 0) return;
  aggregate64_kernel<<<grid_for(n, 256), 256, 0, s>>>(srcs_dev, m, n, 1.0 / static_cast<double>(m), out);
  SPB_CUDA(cudaGetLastError());
}

void launch_split(const float* in, long n, float* hi, float* lo, cudaStream_t s) {
  if (n <= 0) return;
  split_kernel<<<grid_for(n, 256), 256, 0, s>>>(in, n, hi, lo);
  SPB_CUDA(cudaGetLastError());
}

void launch_join(const float* hi, const float* lo, long n, float* out, cudaStream_t s) {
  if (n <= 0) return;
  join_kernel<<<grid_for(n, 256), 256, 0, s>>>(hi, lo, n, out);
  SPB_CUDA(cudaGetLastError());
}

__global__ void stamp_kernel(unsigned long long* slot) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *slot = t;
}

void launch_stamp(unsigned long long* slot, cudaStream_t s) {
  stamp_kernel<<<1, 1, 0, s>>>(slot);
  SPB_CUDA(cudaGetLastError());
}

// One thread idles on the stream for ns nanoseconds (%globaltimer).
__global__ void spin_kernel(long long ns) {
  long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    __nanosleep(2000);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}

void launch_spin(long long ns, cudaStream_t s) {
  spin_kernel<<<1, 1, 0, s>>>(ns);
  SPB_CUDA(cudaGetLastError());
}

void launch_sum_loss(const float* row_loss, int rows, float scale, float* out, int* step_dev, cudaStream_t s) {
  sum_loss_kernel<<<1, 1024, 0, s>>>(row_loss, rows, scale, out, step_dev);
  SPB_CUDA(cudaGetLastError());
}

}  // namespace spb
