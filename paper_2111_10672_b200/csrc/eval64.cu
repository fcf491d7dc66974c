// fp64 evaluation of the ChainMlp loss on the GPU (ChainMlp::sample_loss /
// ChainMlp::loss, model.cpp:130-143): the reference's own precision, for the
// callers that difference losses -- the verify suite's finite-difference
// gradient check (verify.cpp:217-248, h = 1e-5) cannot work on an fp32 loss.
// Not on the training path: the SPB step stays fp32 (3xTF32 tcgen05).
//
// Layer by layer over a chunk of samples: H_l = act(H_{l-1} W_l^T + b_l) with
// a shared-memory tiled fp64 kernel, then per-row 0.5 ||out - y||^2.
#include <cuda_runtime.h>

#include <cstdint>

#include "launch.hpp"

namespace spb {
namespace {

constexpr int kT = 16;  // tile edge (rows x outputs), and the K step

__global__ void gather64_kernel(const float* __restrict__ X, long ldx, const int* __restrict__ idx, int rows, int n,
                                double* __restrict__ H, long ldh) {
  for (long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; i < static_cast<long>(rows) * n;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    const long r = i / n, c = i % n;
    H[r * ldh + c] = static_cast<double>(X[static_cast<long>(idx[r]) * ldx + c]);
  }
}

// Hout[r, o] = act(b[o] + sum_i W[o, i] Hin[r, i]); W row-major [n_out x n_in]
// followed by b (the reference's parameter block layout, model.hpp:93-94).
template <bool TANH>
__global__ void dense64_kernel(const double* __restrict__ Hin, long ldi, int rows, int n_in,
                               const double* __restrict__ block, int n_out, double* __restrict__ Hout, long ldo) {
  __shared__ double hs[kT][kT + 1];
  __shared__ double ws[kT][kT + 1];
  const int tr = threadIdx.y, to = threadIdx.x;
  const int r = blockIdx.y * kT + tr, o = blockIdx.x * kT + to;
  double acc = 0.0;
  for (int i0 = 0; i0 < n_in; i0 += kT) {
    const int ih = i0 + to, iw = i0 + tr;
    hs[tr][to] = (r < rows && ih < n_in) ? Hin[static_cast<long>(r) * ldi + ih] : 0.0;
    const int ow = blockIdx.x * kT + to;  // ws[i][o] = W[o, i0 + i]
    ws[tr][to] = (ow < n_out && iw < n_in) ? block[static_cast<long>(ow) * n_in + iw] : 0.0;
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kT; ++i) acc = fma(hs[tr][i], ws[i][to], acc);
    __syncthreads();
  }
  if (r < rows && o < n_out) {
    const double z = block[static_cast<long>(n_out) * n_in + o] + acc;
    Hout[static_cast<long>(r) * ldo + o] = TANH ? tanh(z) : z;
  }
}

__global__ void sqerr64_kernel(const double* __restrict__ H, long ldh, int rows, int n_out, const float* __restrict__ Y,
                               const int* __restrict__ idx, double* __restrict__ row_loss) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  double s = 0.0;
  for (int o = 0; o < n_out; ++o) {
    const double d = H[static_cast<long>(r) * ldh + o] - static_cast<double>(Y[static_cast<long>(idx[r]) * n_out + o]);
    s += 0.5 * d * d;
  }
  row_loss[r] = s;
}

}  // namespace

void launch_loss64(const float* X, long ldx, const float* Y, const int* idx, int rows, const int* widths, int L,
                   const double* params, const long* block_off, double* act_a, double* act_b, long ld_act,
                   double* row_loss, cudaStream_t s) {
  if (rows <= 0) return;
  gather64_kernel<<<256, 256, 0, s>>>(X, ldx, idx, rows, widths[0], act_a, ld_act);
  SPB_CUDA(cudaGetLastError());
  double* in = act_a;
  double* out = act_b;
  const dim3 blk(kT, kT);
  for (int l = 1; l <= L; ++l) {
    const dim3 grid((widths[l] + kT - 1) / kT, (rows + kT - 1) / kT);
    if (l < L)
      dense64_kernel<true><<<grid, blk, 0, s>>>(in, ld_act, rows, widths[l - 1], params + block_off[l - 1], widths[l],
                                                out, ld_act);
    else
      dense64_kernel<false><<<grid, blk, 0, s>>>(in, ld_act, rows, widths[l - 1], params + block_off[l - 1],
                                                 widths[l], out, ld_act);
    SPB_CUDA(cudaGetLastError());
    double* t = in;
    in = out;
    out = t;
  }
  sqerr64_kernel<<<(rows + 255) / 256, 256, 0, s>>>(in, ld_act, rows, widths[L], Y, idx, row_loss);
  SPB_CUDA(cudaGetLastError());
}

}  // namespace spb
