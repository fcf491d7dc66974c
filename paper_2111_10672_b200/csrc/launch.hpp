// Internal launcher interface shared by the kernel translation units and the
// engine (C-ABI). Not part of the public boundary (include/spb_b200.h).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

namespace spb {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define SPB_CUDA(expr)                                                                            \
  do {                                                                                            \
    cudaError_t e_ = (expr);                                                                      \
    if (e_ != cudaSuccess)                                                                        \
      throw ::spb::CudaError(std::string(#expr) + ": " + cudaGetErrorString(e_) + " @" __FILE__); \
  } while (0)

inline long round_up(long x, long a) { return (x + a - 1) / a * a; }

// A GEMM operand as an exact split pair (hi + lo) in HBM.
//   K-major : memory rows are MN indices (mn rows of k contiguous elements)
//   MN-major: memory rows are K indices  (k rows of mn contiguous elements)
struct Operand {
  const float* hi;
  const float* lo;
  long ld;  // elements between memory rows (multiple of 4)
  int mn;   // extent along the GEMM M (for A) / N (for B) dimension
  int k;    // extent along K
  bool mn_major;
  int mn_map = 0;  // > 0: the stored MN extent when mn runs past it (TMA zero-fills beyond)
};

struct GemmEpilogue;  // gemm_tf32x3.cuh

// D = epi(A * B^T) over M = A.mn, N = B.mn, K = A.k. Returns kernels launched.
// Picks the 1-CTA 128x128 or the CTA-pair 256x256 kernel by wave-quantised cost.
int gemm_tf32x3(const Operand& A, const Operand& B, int epi, const GemmEpilogue& ep, cudaStream_t s);
// Implicit-GEMM 3x3 convolutions straight from the NHWC split pair through
// TMA im2col maps (c_in and ld multiples of 32; conv.hpp ConvGeom).
struct ConvGeom;
struct ConvSrc {
  const float* hi;
  const float* lo;
  long ld;      // floats per pixel row
  int samples;  // images in the tensor
  const ConvGeom& g;
};
// Forward: out = tanh(im2col(src) W^T + b) (kEpiFwdTanh epilogue `ep`).
int gemm_conv_fwd(const ConvSrc& src, const Operand& B, const GemmEpilogue& ep, cudaStream_t s);
// wgrad: D[c_out x 9 c_in] = A^T im2col(src) over pixel rows [pixel0, pixel0 + A.k)
// (A = Delta, MN-major; kEpiStoreScaled epilogue, split-K when ep has a workspace).
int gemm_conv_wgrad(const Operand& A, const ConvSrc& src, long pixel0, const GemmEpilogue& ep, cudaStream_t s);
// dgrad of a stride-1 convolution as a convolution of Delta: out rows
// [pixel0, pixel0 + rows) of the layer below = (im2col(Delta) Wf^T) * (1 - H^2)
// (kEpiDgradTanh), Wf = the spatially flipped, channel-transposed kernel
// [c_below x 9 c_out] (launch_conv_flip). src.g describes Delta as input.
int gemm_conv_dgrad(const ConvSrc& src, long pixel0, int rows, const Operand& B, const GemmEpilogue& ep, cudaStream_t s);
// Column-sum bias scratch a caller passes in GemmEpilogue::colsum_ws /
// colsum_cnt (floats / zeroed counters); gemm_prepare_device makes a default.
constexpr long kColsumWsFloats = 4L << 20;
constexpr int kColsumCounters = 4096;
// Per-device constants of the GEMMs (the fused-bias ones boxes); call once
// per device before capturing any GEMM with a fused bias column.
void gemm_prepare_device();
// Tuning aid: TMEM accumulation chunk (k-blocks) of GEMM kind 0 (forward),
// 1 (dgrad) or 2 (wgrad); kb < 1 restores the default. Captured graphs keep
// the value they were captured with.
void gemm_set_chunk(int kind, int kb);
// Test hook: -1 automatic choice, 0 force 1-CTA, 1 force CTA pair.
void gemm_force_variant(int v);
// Tuning aid: force every GEMM onto one plan (two_sm: CTA-pair kernel of
// width pn; splits K-splits); splits = 0 restores the planner.
void gemm_force_plan(int two_sm, int pn, int splits);
// Test hook: the plan of the last gemm_tf32x3 call (CTA pair?, tile width, K-splits).
void gemm_last_plan(int* two_sm, int* pn, int* splits);
// Persistent GEMM grids launched by this thread leave n SMs free (for NCCL
// kernels running beside them); returns the previous value.
int gemm_reserve_sms(int n);
// Scoped reservation: the engine wraps each launch sequence of a context.
struct SmReserve {
  int prev;
  explicit SmReserve(int n) : prev(gemm_reserve_sms(n)) {}
  ~SmReserve() { gemm_reserve_sms(prev); }
};

// ---- non-GEMM kernels (kernels.cu) ----
// H0 / Ybatch rows from the dataset. Indices come from `idx` (host-provided,
// device pointer) or, when idx_in == nullptr, from the counter-based Rng
// (rng.hpp) : row r -> slot r / bw, worker workers[slot], draw r % bw of
// Rng(seed).split(*step).split(worker). Drawn indices are stored to idx_out.
void launch_gather(const float* X, long ldx, const float* Y, int n0, int nout, int N, int rows, int bw,
                   const int* workers, const uint64_t* seed_dev, uint64_t seed_host, const int* step_dev, int step_host,
                   const int* idx_in,
                   int* idx_out, float* h_hi, float* h_lo, long ldh, float* ybatch, cudaStream_t s);
// Rows already on device (spb_step_host): split X rows into H0 hi/lo.
void launch_split_rows(const float* x, long ldx_in, int rows, int cols, float* hi, float* lo, long ld,
                       cudaStream_t s);
// Head layer L (n_out <= 16): out = H W^T + b, delta = out - y, row_loss,
// and for rows >= cont_row0: dnext = (delta W) * (1 - H^2) as a split pair
// (dn_act = false: dnext = delta W, for the pooled conv features).
// delta_L is written as a split pair (delta, delta_lo) with row stride ldq.
void launch_head(const float* h_hi, const float* h_lo, long ldh, int rows, int n_in, int n_out, const float* w_hi,
                 const float* w_lo, long ldw, const float* b_hi, const float* b_lo, const float* y,
                 float* delta, float* delta_lo, long ldq, float* row_loss, float* dn_hi, float* dn_lo, long ldd,
                 int cont_row0, bool tanh_out, cudaStream_t s, bool dn_act = true);
// Optimizer over the flat parameter pair (see engine.cu).
// ctas > 0 fixes the grid (measurement tools); 0 sizes it to the SM count.
void launch_sgd_update(float* p_hi, float* p_lo, const float* grad, float* mom, long n, float lr, float momentum,
                       float wd, cudaStream_t s, int ctas = 0);
// out[c] = (sum_{w} src[w][c]) / m for w ascending (aggregate, spb.cpp:97-103).
void launch_aggregate(const float* const* srcs_dev, int m, long n, float* out, cudaStream_t s);
// fp64 variant with the reference's exact sum-then-scale sequence (bit-identical).
void launch_aggregate64(const double* const* srcs_dev, int m, long n, double* out, cudaStream_t s);
// *out += sum over [0, n) of (a - b)^2 in fp64 (n a multiple of 4).
void launch_sqdist(const float* a, const float* b, long n, double* out, cudaStream_t s);
void launch_split(const float* in, long n, float* hi, float* lo, cudaStream_t s);
void launch_join(const float* hi, const float* lo, long n, float* out, cudaStream_t s);
// Also advances *step_dev (nullable): the next step's Rng stream.
void launch_sum_loss(const float* row_loss, int rows, float scale, float* out, int* step_dev, cudaStream_t s);
// fp64 ChainMlp loss rows (eval64.cu): row_loss[r] = 0.5 ||out - y||^2 of
// sample idx[r], params in the reference block layout (block l-1 at
// params + block_off[l-1]); act_a / act_b: [rows x ld_act] fp64 scratch.
void launch_loss64(const float* X, long ldx, const float* Y, const int* idx, int rows, const int* widths, int L,
                   const double* params, const long* block_off, double* act_a, double* act_b, long ld_act,
                   double* row_loss, cudaStream_t s);
// One thread writes %globaltimer (ns) to *slot (timeline tracing).
void launch_stamp(unsigned long long* slot, cudaStream_t s);
// One thread idles the stream for ns nanoseconds: gives the host a head start
// to enqueue a whole eager step before the GPU reaches it (spb_profile_step),
// so per-launch event timings carry no host-submission gaps.
void launch_spin(long long ns, cudaStream_t s);

}  // namespace spb
