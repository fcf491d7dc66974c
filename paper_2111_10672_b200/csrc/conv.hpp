// Lowering kernels of the convolutional SPB model (conv.cu). Internal.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace spb {

// One 3x3 convolution, padding 1.
struct ConvGeom {
  int in_h, in_w, c_in;
  int out_h, out_w, c_out;
  int stride;
};

void launch_conv_gather(const float* X, long ldx, const float* Y, int pix, int c0, int nout, int N, int samples, int bw,
                        const int* workers, const uint64_t* seed_dev, uint64_t seed_host, const int* step_dev,
                        int step_host, const int* idx_in, int* idx_out, float* h_hi, float* h_lo, long ldh,
                        float* ybatch, cudaStream_t s);
// col rows [row0, row0 + rows) (output pixels) from the input split pair.
void launch_im2col(const float* in_hi, const float* in_lo, long ldin, const ConvGeom& g, int row0, int rows,
                   float* col_hi, float* col_lo, long ldk, cudaStream_t s);
// Direct forward (bias + tanh + split) of a narrow-input convolution (the RGB
// layer): output pixel rows [0, rows). conv_direct_ok: the geometries it takes.
bool conv_direct_ok(const ConvGeom& g, long ldin, long ldo);
void launch_conv_direct_fwd(const float* in_hi, const float* in_lo, long ldin, const ConvGeom& g, long rows,
                            const float* w_hi, const float* w_lo, long ldw, const float* b_hi, const float* b_lo,
                            float* o_hi, float* o_lo, long ldo, cudaStream_t s);
// Delta of the layer below for input pixel rows [row0, row0 + rows).
void launch_col2im_tanh(const float* dcol, long ldk, const ConvGeom& g, int row0, int rows, const float* h_hi,
                        const float* h_lo, long ldh, float* d_hi, float* d_lo, long ldd, cudaStream_t s);
// Spatially flipped, channel-transposed kernel for the stride-1 implicit dgrad.
void launch_conv_flip(const float* w_hi, const float* w_lo, long ldw, int c_out, int c_in, float* f_hi, float* f_lo,
                      long ldf, cudaStream_t s);
void launch_avgpool(const float* h_hi, const float* h_lo, long ldh, int samples, int pix, int c, float* p_hi,
                    float* p_lo, long ldp, cudaStream_t s);
// Pixel rows of samples [s0, samples).
void launch_unpool_tanh(const float* g_hi, const float* g_lo, long ldg, int samples, int s0, int pix, int c,
                        const float* h_hi, const float* h_lo, long ldh, float* d_hi, float* d_lo, long ldd,
                        cudaStream_t s);

}  // namespace spb
