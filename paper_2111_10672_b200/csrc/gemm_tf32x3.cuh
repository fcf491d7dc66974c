// fp32-accurate GEMM on the 5th-gen tensor cores: tcgen05.mma kind::tf32 with
// the 3xTF32 split, operands staged by TMA into 128B-swizzled shared memory,
// accumulators in TMEM, fused epilogues.
//
//   D[M x N] = epi( sum_k A[m,k] * B[n,k] )
//
// Every operand X (A or B) is held in HBM as an exact split pair
// X = X_hi + X_lo, X_hi = rna_tf32(X), X_lo = X - X_hi (both fp32 words), written
// by whichever kernel produced X (forward / dgrad epilogues, the update
// kernel, the dataset gather). The MMA pipe computes
//   A_lo*B_hi + A_hi*B_lo + A_hi*B_hi
// which loses only the A_lo*B_lo term (~2^-22 relative): fp32-class products,
// needed for the 1e-5 parity bar that plain TF32 (2^-11) cannot meet.
//
// An operand is K-major (memory rows = MN index, K contiguous) or MN-major
// (memory rows = K index, MN contiguous); tcgen05 accepts both for tf32, so
// wgrad (Delta^T H) and dgrad (Delta W) need no transposed copies.
//
// Roles (256 threads, 1 CTA/SM): warp 0 = TMA producer, warp 1 = MMA issuer
// (one elected lane), warp 2 = TMEM allocator, warps 4..7 = epilogue
// (TMEM lanes 32*(warp%4)..+31).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "ptx.cuh"

namespace spb {

enum Epi : int {
  kEpiFwdTanh = 0,     // out = split(tanh(acc + bias[n]))
  kEpiStoreScaled = 1, // out_f32 = alpha * acc
  kEpiDgradTanh = 2,   // out = split(acc * (1 - h[m,n]^2)), h = h_hi + h_lo
  kEpiFwdLinear = 3,   // out = split(acc + bias[n])
  kEpiWgradUpdate = 4, // W (= out_hi + out_lo) -= lr * sgd_dir(alpha * acc), in place (single-GPU step)
};

struct GemmEpilogue {
  float* out_hi;  // kEpiStoreScaled: the fp32 output
  float* out_lo;
  long ld_out;
  const float* bias_hi;
  const float* bias_lo;
  const float* h_hi;
  const float* h_lo;
  long ld_h;
  float alpha;
  int M, N;  // valid output extent
  // kEpiWgradUpdate: momentum buffer (nullable) and optimizer constants.
  float* mom;
  float lr, mu, wd;
  // Split-K: work unit u covers K-split u / num_tiles and writes its partial
  // sums at out_hi + split * split_stride (kEpiStoreScaled only).
  long split_stride;
  // Workspace the host launcher may use for split-K partials (nullable).
  float* splitk_ws;
  long splitk_ws_floats;
  // kEpiStoreScaled row routing (multi-GPU "push" exchange): when
  // route_rows > 0, output row r belongs to owner o = r / route_rows and is
  // stored at route[o] + (r - o * route_rows) * ld_out + col -- the owner's
  // staging slot in peer memory (NVLink stores), or this rank's own buffer.
  float* route[8];
  int route_rows;
  // Fused bias gradient (wgrad GEMMs): the B operand carries a virtual column
  // of ones at output column bias_col_p1 - 1 (a 32-aligned column >= N: the
  // producer TMA-loads a constant ones box there, gemm.cu), so that column of
  // the product is sum_k A[m, k] = the bias gradient of output row m
  // (model.cpp:169, gb[o] += delta). The epilogue routes it to gb_hi[row]
  // (kEpiStoreScaled, scaled by alpha) or applies the optimizer to the bias
  // split pair gb_hi / gb_lo (+ gb_mom) in place (kEpiWgradUpdate). Columns
  // in [N, bias col) are padding and never stored. bias_col_p1 = 0: no bias.
  // ones_col_p1 (same encoding) is where the PRODUCER puts the ones box: equal
  // to bias_col_p1, except in split-K partial GEMMs, which compute the column
  // like any other into the workspace and leave the routing to the fixup.
  int bias_col_p1;
  int ones_col_p1;
  // k-blocks per TMEM accumulation chunk (see kChunkKb below); 0 = the
  // compile-time default of this GEMM kind. The host launcher resolves it.
  int chunk_kb;
  // 1-CTA kernel, MN-major A (wgrad): the bias gradient without a ones column
  // -- warps 2-3 sum the A tile (Delta^T) over K straight from shared memory
  // as the stages stream by (Kahan-compensated fp32), in the units of column
  // tile 0, and emit the sum as output column colsum_col_p1 - 1 (the bias
  // column: bias_store; in split-K partials: the workspace column). Keeps the
  // N tile count at n (no extra 128-wide tile for one column); the CTA-pair
  // kernel uses the ones column instead (its CTA 1 cannot see the stage
  // barrier, which lives on the leader).
  int colsum_col_p1;
  // Without K-splits every column tile of an m-tile sums a 1/(column tiles)
  // slice of the k-blocks (so no CTA carries all of it); the slices meet in
  // colsum_ws [column tiles x m-tiles*128] and the last tile to finish (per
  // m-tile counter colsum_cnt, zero between launches) adds them in tile
  // order -- deterministic.
  float* colsum_ws;
  int* colsum_cnt;
  float* gb_hi;
  float* gb_lo;
  float* gb_mom;
};

__host__ __device__ __forceinline__ int epi_bias_col(const GemmEpilogue& ep) { return ep.bias_col_p1 - 1; }
// The bias column as a TILE column of the accumulator (the ones-column
// scheme), or -1 when the column-sum warps produce it (colsum_col_p1).
__host__ __device__ __forceinline__ int epi_tile_bias_col(const GemmEpilogue& ep) {
  return ep.colsum_col_p1 > 0 ? -1 : ep.bias_col_p1 - 1;
}
// Output columns a GEMM with this epilogue computes (N, or up to the bias column).
__host__ __device__ __forceinline__ int epi_cols(const GemmEpilogue& ep) {
  return ep.bias_col_p1 > 0 ? ep.bias_col_p1 : ep.N;
}

// Address of output element (row, col) of a kEpiStoreScaled epilogue.
__device__ __forceinline__ float* store_addr(const GemmEpilogue& ep, int row, int col, long out_shift) {
  if (ep.route_rows > 0) {
    const int o = row / ep.route_rows;
    return ep.route[o] + static_cast<long>(row - o * ep.route_rows) * ep.ld_out + col;
  }
  return ep.out_hi + out_shift + static_cast<long>(row) * ep.ld_out + col;
}

// The optimizer step on one weight (PyTorch SGD semantics, see kernels.cu
// sgd_update_kernel): g' = g + wd*w; buf = mu*buf + g'; w -= lr*buf.
__device__ __forceinline__ float sgd_apply(float w, float g, float* buf, float lr, float mu, float wd) {
  g = fmaf(wd, w, g);
  if (buf) {
    *buf = fmaf(mu, *buf, g);
    g = *buf;
  }
  return w - lr * g;
}

constexpr int kBM = 128;
constexpr int kBK = 32;  // 32 fp32 = one 128-byte swizzle row

template <int BN, bool TMA_UPD = false>
struct GemmCfg {
  static constexpr int kABytes = kBM * kBK * 4;
  static constexpr int kBBytes = BN * kBK * 4;
  static constexpr int kStageBytes = 2 * kABytes + 2 * kBBytes;
  static constexpr int kStages = TMA_UPD ? 2 : ((BN >= 256) ? 2 : 3);
  // TMA-staged optimizer epilogue: per epilogue warp, 2 buffers x {W_hi,
  // W_lo, mom} x one 32 x 32 fp32 tile (4 KB, 128B-swizzled).
  static constexpr int kEpiTile = 32 * 32 * 4;
  static constexpr int kEpiBytes = TMA_UPD ? 4 * 2 * 3 * kEpiTile : 0;
  // Routed kEpiStoreScaled epilogue (GemmEpilogue::route): per epilogue warp
  // one 32 x 32 fp32 block staged with a 33-float row pitch.
  static constexpr int kRouteBytes = 4 * 32 * 33 * 4;
  // stages | barrier page (1 KB) | epilogue tiles | + 1 KB alignment slack
  static constexpr int kSmem = kStages * kStageBytes + 1024 + (TMA_UPD ? kEpiBytes : kRouteBytes) + 1024;
  static_assert(kSmem <= 232448, "exceeds 227 KB of dynamic shared memory");
};

// Element (r, c) of a 32 x 32 fp32 tile stored with the 128B swizzle.
__device__ __forceinline__ uint32_t sw128_off(int r, int chunk16) {
  return static_cast<uint32_t>(r * 128 + ((chunk16 ^ (r & 7)) << 4));
}

// TMA for one operand tile of ROWS (MN) x kBK (K) elements. MN-major B
// operands of bias-fused wgrads: the 32-column box starting at ones_col (the
// virtual ones column, GemmEpilogue::bias_col_p1) comes from the constant map
// t_ones instead: rows 0-31 of it are ones (the hi half), rows 32-63 zeros
// (the lo half: ones are exact in tf32). ones_col < 0: none.
template <bool MN_MAJOR, int ROWS>
__device__ __forceinline__ void load_operand(uint8_t* dst, const CUtensorMap* tm, uint64_t* bar, int mn0, int k0,
                                             const CUtensorMap* t_ones = nullptr, int ones_col = -1,
                                             int ones_row = 0) {
  if constexpr (!MN_MAJOR) {
    tma_load_2d(dst, tm, bar, k0, mn0);  // box {32 (K), ROWS (MN)}
  } else {
#pragma unroll
    for (int c = 0; c < (ROWS + 31) / 32; ++c) {  // boxes {32 (MN), 32 (K)}, 4 KB apart
      if (mn0 + c * 32 == ones_col)
        tma_load_2d(dst + c * 4096, t_ones, bar, 0, ones_row);
      else
        tma_load_2d(dst + c * 4096, tm, bar, mn0 + c * 32, k0);
    }
  }
}

// UMMA descriptor for the kk-th K=8 slice of an operand tile.
template <bool MN_MAJOR>
__device__ __forceinline__ uint64_t operand_desc(uint32_t base, int kk) {
  if constexpr (!MN_MAJOR) {
    // K-major SW128: rows of 128 B, 8-row atoms 1024 B apart (SBO); K slice = +32 B.
    return sdesc(base + kk * 32, 16, 1024, kLayoutSw128);
  } else {
    // MN-major SW128_BASE32B: 32-element MN chunks 4 KB apart (LBO), 4-K-row
    // atoms 512 B apart (SBO); a K=8 slice is 8 rows = +1 KB.
    return sdesc(base + kk * 1024, 4096, 512, kLayoutSw128Base32);
  }
}

__device__ __forceinline__ void store_split4(float* hi, float* lo, float4 v) {
  float4 h = make_float4(tf32_rna(v.x), tf32_rna(v.y), tf32_rna(v.z), tf32_rna(v.w));
  float4 l = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
  *reinterpret_cast<float4*>(hi) = h;
  *reinterpret_cast<float4*>(lo) = l;
}

// The bias column of a wgrad GEMM (GemmEpilogue::bias_col_p1): v = sum_k A[row, k].
template <int EPI>
__device__ __forceinline__ void bias_store(const GemmEpilogue& ep, float v, int row) {
  if (row >= ep.M) return;
  if constexpr (EPI == kEpiStoreScaled) {
    ep.gb_hi[row] = ep.alpha * v;
  } else if constexpr (EPI == kEpiWgradUpdate) {
    const float b = sgd_apply(ep.gb_hi[row] + ep.gb_lo[row], ep.alpha * v, ep.gb_mom ? ep.gb_mom + row : nullptr, ep.lr,
                              ep.mu, ep.wd);
    const float bh = tf32_rna(b);
    ep.gb_hi[row] = bh;
    ep.gb_lo[row] = b - bh;
  }
}

// The epilogue of one output element (split-K fixup path).
template <int EPI>
__device__ __forceinline__ void epilogue_one(const GemmEpilogue& ep, float v, int row, int col) {
  if (col >= ep.N) {  // the fused bias column, or padding before it
    if (col == epi_bias_col(ep)) bias_store<EPI>(ep, v, row);
    return;
  }
  const long at = row * ep.ld_out + col;
  if constexpr (EPI == kEpiStoreScaled) {
    *store_addr(ep, row, col, 0) = ep.alpha * v;
  } else if constexpr (EPI == kEpiFwdTanh || EPI == kEpiFwdLinear) {
    float z = v + (ep.bias_hi[col] + ep.bias_lo[col]);
    if (EPI == kEpiFwdTanh) z = tanhf(z);
    const float h = tf32_rna(z);
    ep.out_hi[at] = h;
    ep.out_lo[at] = z - h;
  } else if constexpr (EPI == kEpiDgradTanh) {
    const float h = ep.h_hi[row * ep.ld_h + col] + ep.h_lo[row * ep.ld_h + col];
    const float d = v * (1.0f - h * h);
    const float dh = tf32_rna(d);
    ep.out_hi[at] = dh;
    ep.out_lo[at] = d - dh;
  } else {
    const float w = sgd_apply(ep.out_hi[at] + ep.out_lo[at], ep.alpha * v, ep.mom ? ep.mom + at : nullptr, ep.lr,
                              ep.mu, ep.wd);
    const float wh = tf32_rna(w);
    ep.out_hi[at] = wh;
    ep.out_lo[at] = w - wh;
  }
}

// out_shift: split-K slice offset applied to out_hi (kEpiStoreScaled only).
// n_lim: first column NOT to write (the output width, or the end of a tile
// narrower than the 32-column chunk grid).
template <int EPI>
__device__ __forceinline__ void epilogue_chunk(const GemmEpilogue& ep, const float* v, int row, int col0,
                                               long out_shift = 0, int n_lim = -1) {
  if (n_lim < 0) n_lim = ep.N;
  if (row >= ep.M) return;
  const bool full = (col0 + 32 <= n_lim);
  if constexpr (EPI == kEpiStoreScaled) {
    float* o = store_addr(ep, row, col0, out_shift);
    if (full) {
#pragma unroll
      for (int j = 0; j < 32; j += 4)
        *reinterpret_cast<float4*>(o + j) =
            make_float4(ep.alpha * v[j], ep.alpha * v[j + 1], ep.alpha * v[j + 2], ep.alpha * v[j + 3]);
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (col0 + j < n_lim) o[j] = ep.alpha * v[j];
    }
  } else if constexpr (EPI == kEpiWgradUpdate) {
    float* oh = ep.out_hi + row * ep.ld_out + col0;
    float* ol = ep.out_lo + row * ep.ld_out + col0;
    float* mb = ep.mom ? ep.mom + row * ep.ld_out + col0 : nullptr;
    if (full) {
      // 8-column slices, software-pipelined: the loads of slice j+1 are issued
      // before the math and stores of slice j, so each thread keeps up to 12
      // x 16 B in flight (x 512 epilogue threads per SM in the pair kernel).
      float4 h0 = *reinterpret_cast<const float4*>(oh), h1 = *reinterpret_cast<const float4*>(oh + 4);
      float4 l0 = *reinterpret_cast<const float4*>(ol), l1 = *reinterpret_cast<const float4*>(ol + 4);
      float4 b0 = make_float4(0.f, 0.f, 0.f, 0.f), b1 = b0;
      if (mb) b0 = *reinterpret_cast<const float4*>(mb), b1 = *reinterpret_cast<const float4*>(mb + 4);
#pragma unroll
      for (int j = 0; j < 32; j += 8) {
        float4 nh0, nh1, nl0, nl1, nb0 = make_float4(0.f, 0.f, 0.f, 0.f), nb1 = nb0;
        if (j + 8 < 32) {
          nh0 = *reinterpret_cast<const float4*>(oh + j + 8);
          nh1 = *reinterpret_cast<const float4*>(oh + j + 12);
          nl0 = *reinterpret_cast<const float4*>(ol + j + 8);
          nl1 = *reinterpret_cast<const float4*>(ol + j + 12);
          if (mb) nb0 = *reinterpret_cast<const float4*>(mb + j + 8), nb1 = *reinterpret_cast<const float4*>(mb + j + 12);
        }
        float4 w0, w1;
        w0.x = sgd_apply(h0.x + l0.x, ep.alpha * v[j + 0], mb ? &b0.x : nullptr, ep.lr, ep.mu, ep.wd);
        w0.y = sgd_apply(h0.y + l0.y, ep.alpha * v[j + 1], mb ? &b0.y : nullptr, ep.lr, ep.mu, ep.wd);
        w0.z = sgd_apply(h0.z + l0.z, ep.alpha * v[j + 2], mb ? &b0.z : nullptr, ep.lr, ep.mu, ep.wd);
        w0.w = sgd_apply(h0.w + l0.w, ep.alpha * v[j + 3], mb ? &b0.w : nullptr, ep.lr, ep.mu, ep.wd);
        w1.x = sgd_apply(h1.x + l1.x, ep.alpha * v[j + 4], mb ? &b1.x : nullptr, ep.lr, ep.mu, ep.wd);
        w1.y = sgd_apply(h1.y + l1.y, ep.alpha * v[j + 5], mb ? &b1.y : nullptr, ep.lr, ep.mu, ep.wd);
        w1.z = sgd_apply(h1.z + l1.z, ep.alpha * v[j + 6], mb ? &b1.z : nullptr, ep.lr, ep.mu, ep.wd);
        w1.w = sgd_apply(h1.w + l1.w, ep.alpha * v[j + 7], mb ? &b1.w : nullptr, ep.lr, ep.mu, ep.wd);
        store_split4(oh + j, ol + j, w0);
        store_split4(oh + j + 4, ol + j + 4, w1);
        if (mb) {
          *reinterpret_cast<float4*>(mb + j) = b0;
          *reinterpret_cast<float4*>(mb + j + 4) = b1;
        }
        if (j + 8 < 32) h0 = nh0, h1 = nh1, l0 = nl0, l1 = nl1, b0 = nb0, b1 = nb1;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        if (col0 + j >= n_lim) continue;
        const float w = sgd_apply(oh[j] + ol[j], ep.alpha * v[j], mb ? mb + j : nullptr, ep.lr, ep.mu, ep.wd);
        const float wh = tf32_rna(w);
        oh[j] = wh;
        ol[j] = w - wh;
      }
    }
  } else if constexpr (EPI == kEpiFwdTanh || EPI == kEpiFwdLinear) {
    float* oh = ep.out_hi + row * ep.ld_out + col0;
    float* ol = ep.out_lo + row * ep.ld_out + col0;
    if (full) {
#pragma unroll
      for (int j = 0; j < 32; j += 4) {
        float4 bh = __ldg(reinterpret_cast<const float4*>(ep.bias_hi + col0 + j));
        float4 bl = __ldg(reinterpret_cast<const float4*>(ep.bias_lo + col0 + j));
        float4 z = make_float4(v[j] + (bh.x + bl.x), v[j + 1] + (bh.y + bl.y), v[j + 2] + (bh.z + bl.z),
                               v[j + 3] + (bh.w + bl.w));
        if (EPI == kEpiFwdTanh) z = make_float4(tanhf(z.x), tanhf(z.y), tanhf(z.z), tanhf(z.w));
        store_split4(oh + j, ol + j, z);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        if (col0 + j >= n_lim) continue;
        float z = v[j] + (ep.bias_hi[col0 + j] + ep.bias_lo[col0 + j]);
        if (EPI == kEpiFwdTanh) z = tanhf(z);
        float h = tf32_rna(z);
        oh[j] = h;
        ol[j] = z - h;
      }
    }
  } else {  // kEpiDgradTanh
    float* oh = ep.out_hi + row * ep.ld_out + col0;
    float* ol = ep.out_lo + row * ep.ld_out + col0;
    const float* hh = ep.h_hi + row * ep.ld_h + col0;
    const float* hl = ep.h_lo + row * ep.ld_h + col0;
    if (full) {
#pragma unroll
      for (int j = 0; j < 32; j += 4) {
        float4 a = *reinterpret_cast<const float4*>(hh + j);
        float4 b = *reinterpret_cast<const float4*>(hl + j);
        float4 h = make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
        float4 d = make_float4(v[j] * (1.0f - h.x * h.x), v[j + 1] * (1.0f - h.y * h.y),
                               v[j + 2] * (1.0f - h.z * h.z), v[j + 3] * (1.0f - h.w * h.w));
        store_split4(oh + j, ol + j, d);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        if (col0 + j >= n_lim) continue;
        float h = hh[j] + hl[j];
        float d = v[j] * (1.0f - h * h);
        float dh = tf32_rna(d);
        oh[j] = dh;
        ol[j] = d - dh;
      }
    }
  }
}

// Persistent CTAs (grid <= #SMs) walk the output tiles m-fastest, so the
// CTAs running side by side share one B tile (read from HBM once).
//
// fp32-faithful accumulation: the tensor core rounds its fp32 accumulator
// toward zero after every tcgen05.mma, so a single TMEM accumulator drifts by
// ~(3K/8) * 2^-25 relative over K (7e-6 at K=1024, measured). The MMA warp
// therefore accumulates only kChunkKb k-blocks (K = 32*kChunkKb) per TMEM
// buffer; the epilogue warps drain each chunk into fp32 registers
// (round-to-nearest adds) while the MMA warp fills the other buffer. The error
// is then bounded independently of K.
// k-blocks per TMEM chunk, per GEMM kind (told apart by operand majorness:
// forward K x K, dgrad K x MN, wgrad MN x MN -- split-K partials included).
#ifndef SPB_CHUNK_KB
#define SPB_CHUNK_KB 4
#endif
#ifndef SPB_CHUNK_KB_FWD
#define SPB_CHUNK_KB_FWD SPB_CHUNK_KB
#endif
// dgrad: 2 (64 of K per chunk). The dgrad chain carries the truncation bias
// through every layer of the backward (Delta_{l-1} from Delta_l): at the full
// cfg3 depth (16 layers) chunk 4 leaves layer 1's aggregate at 1.12e-5 of the
// fp64 reference, chunk 2 at 7.2e-6, at the same step time (5.73 vs 5.78 ms;
// the dgrads are split-K / HBM-heavy, the TMEM drains hide). Forward and
// wgrad chunk size barely moves the error (tools/chunk_experiment.py,
// profiles/r02_chunk_experiment.jsonl).
#ifndef SPB_CHUNK_KB_DGRAD
#define SPB_CHUNK_KB_DGRAD 2
#endif
#ifndef SPB_CHUNK_KB_WGRAD
#define SPB_CHUNK_KB_WGRAD SPB_CHUNK_KB
#endif
template <bool A_MN, bool B_MN>
__host__ __device__ constexpr int chunk_kb() {
  return (A_MN && B_MN) ? SPB_CHUNK_KB_WGRAD : ((!A_MN && B_MN) ? SPB_CHUNK_KB_DGRAD : SPB_CHUNK_KB_FWD);
}

// Implicit-GEMM convolution operands (3x3, padding 1, NHWC, c_in % 32 == 0):
// the tensor maps are TMA im2col maps of the activation tensor and the tile
// loads compute window origins and filter-tap offsets instead of reading a
// materialised column matrix.
//   IC == 1: A = columns of the output-pixel rows [m0, m0 + 128) (forward:
//            K-major, K = tap * c_in + ci), one 128-pixel box per k-block.
//   IC == 2: B = columns of the pixel rows k_base + [kb*32, kb*32 + 32)
//            (wgrad: MN-major, N = tap * c_in + ci), one 32 x 32 box per
//            32-column chunk.
struct ConvTmaArgs {
  int opix, out_w, stride, c_in;
  long k_base;  // IC == 2: first pixel row of K
  long m_base;  // IC == 1: first pixel row of M
};

__device__ __forceinline__ void conv_origin(const ConvTmaArgs& ic, long pixel, int& w, int& h, int& n) {
  n = static_cast<int>(pixel / ic.opix);
  const int rem = static_cast<int>(pixel - static_cast<long>(n) * ic.opix);
  const int p = rem / ic.out_w, q = rem - p * ic.out_w;
  w = q * ic.stride - 1;
  h = p * ic.stride - 1;
}

template <int BN, bool A_MN, bool B_MN, int EPI, bool TMA_UPD = false, int IC = 0>
__global__ void __launch_bounds__(256, 1)
    gemm_tf32x3_kernel(const __grid_constant__ CUtensorMap ta_hi, const __grid_constant__ CUtensorMap ta_lo,
                       const __grid_constant__ CUtensorMap tb_hi, const __grid_constant__ CUtensorMap tb_lo,
                       int num_kb, int num_m_tiles, int num_tiles, int kb_per_split, int num_units,
                       const __grid_constant__ GemmEpilogue ep, const __grid_constant__ CUtensorMap tw_hi,
                       const __grid_constant__ CUtensorMap tw_lo, const __grid_constant__ CUtensorMap tw_mom,
                       const ConvTmaArgs ic, const __grid_constant__ CUtensorMap t_ones) {
  using Cfg = GemmCfg<BN, TMA_UPD>;
  const int kChunkKb = ep.chunk_kb > 0 ? ep.chunk_kb : chunk_kb<A_MN, B_MN>();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + Cfg::kStages * Cfg::kStageBytes);
  uint64_t* empty_bar = full_bar + Cfg::kStages;
  uint64_t* tfull_bar = empty_bar + Cfg::kStages;  // [2]
  uint64_t* tempty_bar = tfull_bar + 2;            // [2]
  uint64_t* eload_bar = tempty_bar + 2;            // [4 warps][2 buffers] (TMA_UPD)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(eload_bar + 8);
  uint8_t* epi_smem = smem + Cfg::kStages * Cfg::kStageBytes + 1024;  // after the barriers page

  const uint32_t warp = warp_idx_sync();
  const uint32_t lane = threadIdx.x & 31u;
  const bool colsum = A_MN && IC != 1 && ep.colsum_col_p1 > 0;
  // Work unit u -> output tile u % num_tiles, K-split u / num_tiles.
  auto unit = [&](int u, int& m0, int& n0, int& kb0, int& kb1, int& split) {
    const int t = u % num_tiles;
    split = u / num_tiles;
    m0 = (t % num_m_tiles) * kBM;
    n0 = (t / num_m_tiles) * BN;
    kb0 = split * kb_per_split;
    kb1 = min(num_kb, kb0 + kb_per_split);
  };

  if (warp == 0 && elect_one()) {
    tma_prefetch(&ta_hi);
    tma_prefetch(&ta_lo);
    tma_prefetch(&tb_hi);
    tma_prefetch(&tb_lo);
  }
  if (warp == 1 && elect_one()) {
    for (int s = 0; s < Cfg::kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], colsum ? 3 : 1);  // the MMA commit (+ the two column-sum warps)
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull_bar[b], 1);
      mbar_init(&tempty_bar[b], 4);  // one arrive per epilogue warp
    }
    for (int i = 0; i < 8; ++i) mbar_init(&eload_bar[i], 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 2 * BN);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // Programmatic dependent launch (gemm.cu, SPB_PDL): the prologue above ran
  // beside the previous kernel's tail; everything below reads its outputs.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");

  if (warp == 0) {
    if (elect_one()) {
      const int ones_col = B_MN ? ep.ones_col_p1 - 1 : -1;
      int it = 0;
      for (int u = blockIdx.x; u < num_units; u += gridDim.x) {
        int m0, n0, kb0, kb1, split;
        unit(u, m0, n0, kb0, kb1, split);
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % Cfg::kStages;
          const uint32_t ph = (it / Cfg::kStages) & 1u;
          mbar_wait(&empty_bar[s], ph ^ 1u);
          mbar_arrive_expect_tx(&full_bar[s], Cfg::kStageBytes);
          uint8_t* base = smem + s * Cfg::kStageBytes;
          if constexpr (IC == 1) {
            const int k = kb * kBK, tap = k / ic.c_in, c = k - tap * ic.c_in;
            int w, h, n;
            conv_origin(ic, ic.m_base + m0, w, h, n);
            const uint16_t ox = static_cast<uint16_t>(tap % 3), oy = static_cast<uint16_t>(tap / 3);
            tma_load_im2col_4d(base, &ta_hi, &full_bar[s], c, w, h, n, ox, oy);
            tma_load_im2col_4d(base + Cfg::kABytes, &ta_lo, &full_bar[s], c, w, h, n, ox, oy);
          } else {
            load_operand<A_MN, kBM>(base, &ta_hi, &full_bar[s], m0, kb * kBK);
            load_operand<A_MN, kBM>(base + Cfg::kABytes, &ta_lo, &full_bar[s], m0, kb * kBK);
          }
          if constexpr (IC == 2) {
            int w, h, n;
            conv_origin(ic, ic.k_base + kb * kBK, w, h, n);
#pragma unroll
            for (int cc = 0; cc < BN / 32; ++cc) {
              const int col = n0 + cc * 32, tap = col / ic.c_in, c = col - tap * ic.c_in;
              uint8_t* dh = base + 2 * Cfg::kABytes + cc * 4096;
              if (col == ones_col) {  // the fused bias column: constant ones / zeros boxes
                tma_load_2d(dh, &t_ones, &full_bar[s], 0, 0);
                tma_load_2d(dh + Cfg::kBBytes, &t_ones, &full_bar[s], 0, 32);
                continue;
              }
              const uint16_t ox = static_cast<uint16_t>(tap % 3), oy = static_cast<uint16_t>(tap / 3);
              tma_load_im2col_4d(dh, &tb_hi, &full_bar[s], c, w, h, n, ox, oy);
              tma_load_im2col_4d(dh + Cfg::kBBytes, &tb_lo, &full_bar[s], c, w, h, n, ox, oy);
            }
          } else {
            load_operand<B_MN, BN>(base + 2 * Cfg::kABytes, &tb_hi, &full_bar[s], n0, kb * kBK, &t_ones, ones_col, 0);
            load_operand<B_MN, BN>(base + 2 * Cfg::kABytes + Cfg::kBBytes, &tb_lo, &full_bar[s], n0, kb * kBK, &t_ones,
                                   ones_col, 32);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      constexpr uint32_t idesc = idesc_tf32(kBM, BN, A_MN, B_MN);
      int it = 0, g = 0;
      for (int u = blockIdx.x; u < num_units; u += gridDim.x) {
        int m0, n0, kb0, kb1, split;
        unit(u, m0, n0, kb0, kb1, split);
        const int num_chunks = (kb1 - kb0 + kChunkKb - 1) / kChunkKb;
        for (int c = 0; c < num_chunks; ++c, ++g) {
          const uint32_t b = g & 1, tph = (g >> 1) & 1;
          mbar_wait(&tempty_bar[b], tph ^ 1u);  // epilogue drained this buffer
          tc_fence_after();
          const uint32_t acc_addr = tmem + b * BN;
          const int kb_beg = kb0 + c * kChunkKb, kb_end = min(kb1, kb_beg + kChunkKb);
          for (int kb = kb_beg; kb < kb_end; ++kb, ++it) {
            const int s = it % Cfg::kStages;
            const uint32_t ph = (it / Cfg::kStages) & 1u;
            mbar_wait(&full_bar[s], ph);
            tc_fence_after();
            const uint32_t base = smem_u32(smem + s * Cfg::kStageBytes);
            const uint32_t a_hi = base, a_lo = base + Cfg::kABytes;
            const uint32_t b_hi = base + 2 * Cfg::kABytes, b_lo = b_hi + Cfg::kBBytes;
#pragma unroll
            for (int kk = 0; kk < kBK / 8; ++kk) {
              const uint32_t acc = (kb != kb_beg) || kk != 0;
              umma_tf32(acc_addr, operand_desc<A_MN>(a_lo, kk), operand_desc<B_MN>(b_hi, kk), idesc, acc);
              umma_tf32(acc_addr, operand_desc<A_MN>(a_hi, kk), operand_desc<B_MN>(b_lo, kk), idesc, 1u);
              umma_tf32(acc_addr, operand_desc<A_MN>(a_hi, kk), operand_desc<B_MN>(b_hi, kk), idesc, 1u);
            }
            umma_commit(&empty_bar[s]);  // frees the smem stage once these MMAs retire
          }
          umma_commit(&tfull_bar[b]);  // chunk accumulated
        }
      }
    }
  } else if (warp == 2 || warp == 3) {
    if (colsum) {
      // Column sums of A (MN-major: 32 x 32 boxes, K rows of 128 B, SW128 with
      // 32 B atoms: the 8-float granule g of row k sits at g ^ (k & 3)).
      // Warp 2 sums boxes 0-1 (m0 + [0, 64)), warp 3 boxes 2-3. Lane l reads
      // the float4 p = l & 7 (m = 4p .. 4p + 3 of the box) of the rows
      // k = 4 kk + (l >> 3): 16-byte loads, one fp32 partial per k-block,
      // Kahan-compensated across k-blocks, the four row-phase lanes combined
      // at the end. With K-splits, the unit of split s whose column tile is
      // s mod (column tiles) sums its whole k-range (the fixup adds the
      // splits); without, column tile j sums the k-blocks kb = j mod (column
      // tiles) and the per-m-tile counter combines the slices (colsum_ws).
      const int box0 = static_cast<int>(warp - 2) * 2;
      const int col = ep.colsum_col_p1 - 1;
      const int num_n_tiles = num_tiles / num_m_tiles;
      const bool split_k = num_units > num_tiles;
      const int p = static_cast<int>(lane & 7u), r4 = static_cast<int>(lane >> 3);
      int it = 0, uflip = 0;
      for (int u = blockIdx.x; u < num_units; u += gridDim.x) {
        int m0, n0, kb0, kb1, split;
        unit(u, m0, n0, kb0, kb1, split);
        const int nt = n0 / BN;
        const bool mine = split_k ? nt == split % num_n_tiles : true;
        float sum[2][4] = {}, cmp[2][4] = {};
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % Cfg::kStages;
          const uint32_t ph = (it / Cfg::kStages) & 1u;
          mbar_wait(&full_bar[s], ph);
          if (mine && (split_k || (kb - kb0) % num_n_tiles == nt)) {
            const uint8_t* base = smem + s * Cfg::kStageBytes;
#pragma unroll
            for (int b = 0; b < 2; ++b) {
              const uint8_t* hi = base + (box0 + b) * 4096;
              const uint8_t* lo = hi + Cfg::kABytes;
              float4 part = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
              for (int kk = 0; kk < kBK / 4; ++kk) {
                const int k = kk * 4 + r4;
                const uint32_t off = k * 128 + ((((p >> 1) ^ (k & 3)) & 3) << 5) + (p & 1) * 16;
                const float4 vh = *reinterpret_cast<const float4*>(hi + off);
                const float4 vl = *reinterpret_cast<const float4*>(lo + off);
                part.x += vh.x + vl.x, part.y += vh.y + vl.y, part.z += vh.z + vl.z, part.w += vh.w + vl.w;
              }
              const float pv[4] = {part.x, part.y, part.z, part.w};
#pragma unroll
              for (int i = 0; i < 4; ++i) {  // Kahan
                const float y = pv[i] - cmp[b][i], t = sum[b][i] + y;
                cmp[b][i] = (t - sum[b][i]) - y;
                sum[b][i] = t;
              }
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty_bar[s]);
        }
        if (!mine) continue;
        float tot[2][4];
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            float v = sum[b][i] - cmp[b][i];
            v += __shfl_xor_sync(0xffffffffu, v, 8);
            v += __shfl_xor_sync(0xffffffffu, v, 16);
            tot[b][i] = v;
          }
        bool emit = true;
        const long mpad = static_cast<long>(num_m_tiles) * kBM;
        if (!split_k && num_n_tiles > 1) {
          // Publish this tile's slice, count it; the last of the m-tile's
          // column tiles adds all slices in tile order.
          if (r4 == 0)
#pragma unroll
            for (int b = 0; b < 2; ++b)
#pragma unroll
              for (int i = 0; i < 4; ++i)
                ep.colsum_ws[nt * mpad + m0 + (box0 + b) * 32 + 4 * p + i] = tot[b][i];
          // bar.sync then ONE gpu-scope acq_rel atomic by warp 2's lane 0
          // publishes every lane's slice (the barrier orders the 64 threads'
          // stores before the release) -- no per-thread fences -- and tells
          // warp 3 through a barrier-ordered flag (two slots, alternating by
          // unit, next to the TMEM slot in the barrier page).
          asm volatile("bar.sync 1, 64;" ::: "memory");
          volatile int* flag = reinterpret_cast<volatile int*>(tmem_slot + 1 + (uflip & 1));
          if (warp == 2 && lane == 0) {
            const int mt = m0 / kBM;
            int old;
            asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(old) : "l"(ep.colsum_cnt + mt) : "memory");
            const bool last = old == num_n_tiles - 1;
            if (last) ep.colsum_cnt[mt] = 0;  // ready for the next launch
            *flag = last ? 1 : 0;
          }
          asm volatile("bar.sync 1, 64;" ::: "memory");
          emit = *flag != 0;
          ++uflip;
          if (emit) {
#pragma unroll
            for (int b = 0; b < 2; ++b)
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const long row = m0 + (box0 + b) * 32 + 4 * p + i;
                float v = 0.f;
                for (int j = 0; j < num_n_tiles; ++j) v += __ldcg(ep.colsum_ws + j * mpad + row);
                tot[b][i] = v;
              }
          }
        }
        if (!emit || r4 != 0) continue;
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int row = m0 + (box0 + b) * 32 + 4 * p + i;
            if (ep.bias_col_p1 > 0) {
              bias_store<EPI>(ep, tot[b][i], row);
            } else if (EPI == kEpiStoreScaled && row < ep.M) {  // split-K partial: the workspace column
              ep.out_hi[split * ep.split_stride + static_cast<long>(row) * ep.ld_out + col] = ep.alpha * tot[b][i];
            }
          }
      }
    }
  } else if (warp >= 4) {
    const uint32_t q = warp & 3u;
    const uint32_t lane_addr = (q * 32u) << 16;
    int g = 0;
    int eload_phase[2] = {0, 0};
    for (int u = blockIdx.x; u < num_units; u += gridDim.x) {
      int m0, n0, kb0, kb1, split;
      unit(u, m0, n0, kb0, kb1, split);
      const int num_chunks = (kb1 - kb0 + kChunkKb - 1) / kChunkKb;
      const long out_shift = EPI == kEpiStoreScaled ? split * ep.split_stride : 0;
      float acc[BN];
#pragma unroll
      for (int j = 0; j < BN; ++j) acc[j] = 0.f;
      for (int c = 0; c < num_chunks; ++c, ++g) {
        const uint32_t b = g & 1, tph = (g >> 1) & 1;
        mbar_wait(&tfull_bar[b], tph);
        tc_fence_after();
#pragma unroll
        for (int c0 = 0; c0 < BN; c0 += 32) {
          float v[32];
          tmem_ld_32x32b_x32(tmem + lane_addr + b * BN + c0, v);
#pragma unroll
          for (int j = 0; j < 32; ++j) acc[c0 + j] += v[j];
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty_bar[b]);
      }
      const int row = m0 + static_cast<int>(q * 32 + lane);
      if constexpr (TMA_UPD) {
        // In-place optimizer on the W tile rows [m0 + 32q, +32), columns
        // [n0, n0 + BN): {W_hi, W_lo, mom} 32 x 32 tiles are TMA-loaded into
        // this warp's smem (double-buffered: chunk c+1 loads while chunk c
        // computes), updated row-per-lane from the fp32 accumulators, and
        // TMA-stored back. TMA clips rows / columns outside W.
        uint8_t* wbuf = epi_smem + q * (2 * 3 * Cfg::kEpiTile);
        const int gr = m0 + static_cast<int>(q * 32);
        const bool has_mom = ep.mom != nullptr;
        const uint32_t tx = (has_mom ? 3 : 2) * Cfg::kEpiTile;
        auto issue = [&](int c) {
          uint8_t* bb = wbuf + (c & 1) * 3 * Cfg::kEpiTile;
          uint64_t* bar = &eload_bar[q * 2 + (c & 1)];
          mbar_arrive_expect_tx(bar, tx);
          tma_load_2d(bb, &tw_hi, bar, n0 + c * 32, gr);
          tma_load_2d(bb + Cfg::kEpiTile, &tw_lo, bar, n0 + c * 32, gr);
          if (has_mom) tma_load_2d(bb + 2 * Cfg::kEpiTile, &tw_mom, bar, n0 + c * 32, gr);
        };
        if (lane == 0) {
          bulk_wait_read_all();  // previous tile's stores have left these buffers
          issue(0);
          if (BN / 32 > 1) issue(1);
        }
        __syncwarp();
#pragma unroll
        for (int c = 0; c < BN / 32; ++c) {
          const int bsel = c & 1;
          uint8_t* bb = wbuf + bsel * 3 * Cfg::kEpiTile;
          mbar_wait(&eload_bar[q * 2 + bsel], static_cast<uint32_t>(eload_phase[bsel]));
          eload_phase[bsel] ^= 1;
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint32_t off = sw128_off(static_cast<int>(lane), k);
            float4* ph = reinterpret_cast<float4*>(bb + off);
            float4* pl = reinterpret_cast<float4*>(bb + Cfg::kEpiTile + off);
            float4* pm = reinterpret_cast<float4*>(bb + 2 * Cfg::kEpiTile + off);
            const float4 h = *ph, l = *pl;
            float4 b = has_mom ? *pm : make_float4(0.f, 0.f, 0.f, 0.f);
            const float* a = acc + c * 32 + 4 * k;
            float4 w;
            w.x = sgd_apply(h.x + l.x, ep.alpha * a[0], has_mom ? &b.x : nullptr, ep.lr, ep.mu, ep.wd);
            w.y = sgd_apply(h.y + l.y, ep.alpha * a[1], has_mom ? &b.y : nullptr, ep.lr, ep.mu, ep.wd);
            w.z = sgd_apply(h.z + l.z, ep.alpha * a[2], has_mom ? &b.z : nullptr, ep.lr, ep.mu, ep.wd);
            w.w = sgd_apply(h.w + l.w, ep.alpha * a[3], has_mom ? &b.w : nullptr, ep.lr, ep.mu, ep.wd);
            const float4 wh = make_float4(tf32_rna(w.x), tf32_rna(w.y), tf32_rna(w.z), tf32_rna(w.w));
            *ph = wh;
            *pl = make_float4(w.x - wh.x, w.y - wh.y, w.z - wh.z, w.w - wh.w);
            if (has_mom) *pm = b;
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&tw_hi, bb, n0 + c * 32, gr);
            tma_store_2d(&tw_lo, bb + Cfg::kEpiTile, n0 + c * 32, gr);
            if (has_mom) tma_store_2d(&tw_mom, bb + 2 * Cfg::kEpiTile, n0 + c * 32, gr);
            bulk_commit();
            if (c + 2 < BN / 32) {
              bulk_wait_read_all();  // this buffer's store has read smem
              issue(c + 2);
            }
          }
          __syncwarp();
        }
        // The fused bias column in this tile (its W box was out of bounds);
        // static indices only, so acc stays in registers.
        const int tbc = epi_tile_bias_col(ep);
#pragma unroll
        for (int c0 = 0; c0 < BN; c0 += 32)
          if (n0 + c0 == tbc) bias_store<EPI>(ep, acc[c0], row);
      } else if (EPI == kEpiStoreScaled && ep.route_rows > 0) {
        // Rows routed to peer memory (multi-GPU push exchange): stage each
        // 32 x 32 block in shared memory so that one warp store writes four
        // 128-byte row segments over NVLink instead of 32 scattered 16-byte
        // pieces (row-per-lane order).
        float* stg = reinterpret_cast<float*>(epi_smem) + q * (32 * 33);
        const int rbase = m0 + static_cast<int>(q * 32);
        const int cc = 4 * static_cast<int>(lane & 7);
#pragma unroll
        for (int c0 = 0; c0 < BN; c0 += 32) {
          if (n0 + c0 == epi_tile_bias_col(ep)) {
            bias_store<EPI>(ep, acc[c0], row);  // the bias row stays local (it travels with the push signal)
          } else if (n0 + c0 < ep.N) {
#pragma unroll
            for (int j = 0; j < 32; ++j) stg[lane * 33 + j] = ep.alpha * acc[c0 + j];
            __syncwarp();
            const int gcol = n0 + c0 + cc;
#pragma unroll
            for (int it = 0; it < 8; ++it) {
              const int r = it * 4 + static_cast<int>(lane >> 3);
              const int grow = rbase + r;
              if (grow < ep.M && gcol < ep.N) {
                const float* sp = stg + r * 33 + cc;
                float* dp = store_addr(ep, grow, gcol, 0);
                if (gcol + 3 < ep.N) {
                  *reinterpret_cast<float4*>(dp) = make_float4(sp[0], sp[1], sp[2], sp[3]);
                } else {
                  for (int t = 0; t < 4 && gcol + t < ep.N; ++t) dp[t] = sp[t];
                }
              }
            }
            __syncwarp();
          }
        }
      } else {
#pragma unroll
        for (int c0 = 0; c0 < BN; c0 += 32) {
          if (n0 + c0 == epi_tile_bias_col(ep)) bias_store<EPI>(ep, acc[c0], row);
          else if (n0 + c0 < ep.N) epilogue_chunk<EPI>(ep, acc + c0, row, n0 + c0, out_shift);
        }
      }
    }
    if constexpr (TMA_UPD) {
      if (lane == 0) bulk_wait_all();
      __syncwarp();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 2 * BN);
  }
}

}  // namespace spb
