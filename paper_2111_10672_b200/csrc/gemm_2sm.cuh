// CTA-pair (cta_group::2) variant of the 3xTF32 GEMM: one 256 x 256 output
// tile per SM pair. Each CTA stages its 128 rows of A and its 128 rows of B
// (hi + lo, 64 KB per k-block) and the leader CTA issues
// tcgen05.mma.cta_group::2 M=256 N=256 K=8, which reads A from each CTA's own
// smem and B from both halves. Per SM this moves half the shared-memory and
// L2 bytes per FLOP of the 1-CTA 128 x 128 tile, which is what bounds the
// 1-CTA kernel (tensor pipe ~60% active, profiles/r01_*).
//
// Roles (640 threads = 5 warpgroups, 1 CTA/SM): warp 0 TMA producer (both
// CTAs), warp 1 MMA issuer (leader only), warp 2 TMEM allocator, warp 3
// idle; warps 4..19 epilogue: warp w drains TMEM lanes 32*(w%4)..+31 and
// columns 64*((w-4)/4)..+63 of its CTA's 128 x 256 accumulator (16 warps:
// enough memory-level parallelism for the HBM-heavy fused epilogues).
// The whole kernel fits 96 registers/thread (640 x 96 = 61440 of 64 K), so
// no setmaxnreg rebalancing (a .dec below what ptxas allocated for the
// producer / MMA code corrupts it).
// Accumulation is chunked exactly as in gemm_tf32x3.cuh (kChunkKb k-blocks
// per TMEM buffer, drained into fp32 registers), so numerics match.
#pragma once
#include "gemm_tf32x3.cuh"

namespace spb {

// PN: the pair tile's N (a multiple of 16 in [64, 256]): 256 for large
// outputs, 240 so that e.g. 4096 columns make 18 tiles and a 1024-row forward
// fills 72 of the 74 SM pairs in one wave, and 64 / 128 / 192 so that the
// few-row GEMMs (the multi-GPU forward, the SPB dgrads) fill a wave instead of
// leaving half the SM pairs idle (the host planner picks by wave-quantised cost).
template <int PN = 256>
struct Gemm2smCfg {
  static constexpr int kRowsA = 128;      // per CTA
  static constexpr int kPairN = PN;
  static constexpr int kRowsB = PN / 2;   // per CTA
  static constexpr int kABytes = kRowsA * kBK * 4;
  static constexpr int kBBytes = 128 * kBK * 4;  // smem slot (MN-major loads whole 32-row boxes)
  static constexpr int kStageBytes = 2 * kABytes + 2 * kBBytes;  // 64 KB
  static constexpr int kStages = 3;
  static constexpr int kSmem = kStages * kStageBytes + 1024 + 256;
  static constexpr int kThreads = 640;
  static constexpr int kEpiWarps = 16;
  static constexpr int kEpiCols = 64;  // accumulator columns per epilogue thread
};

// ones_col / t_ones / ones_row: the fused-bias ones box (load_operand in gemm_tf32x3.cuh).
template <bool MN_MAJOR, int ROWS>
__device__ __forceinline__ void load_operand_2sm(uint8_t* dst, const CUtensorMap* tm, uint64_t* bar, int mn0, int k0,
                                                 const CUtensorMap* t_ones = nullptr, int ones_col = -1,
                                                 int ones_row = 0) {
  if constexpr (!MN_MAJOR) {
    tma_load_2d_2sm(dst, tm, bar, k0, mn0);
  } else {
#pragma unroll
    for (int c = 0; c < (ROWS + 31) / 32; ++c) {
      if (mn0 + c * 32 == ones_col)
        tma_load_2d_2sm(dst + c * 4096, t_ones, bar, 0, ones_row);
      else
        tma_load_2d_2sm(dst + c * 4096, tm, bar, mn0 + c * 32, k0);
    }
  }
}

// IC == 1: A is the implicit im2col operand of a 3x3 convolution (forward or
// stride-1 dgrad), loaded through TMA im2col maps exactly as in the 1-CTA
// kernel (gemm_tf32x3.cuh, ConvTmaArgs), each CTA its own 128 output pixels.
// IC == 2: B is (the conv wgrad), each CTA its own PN / 2 columns.
template <bool A_MN, bool B_MN, int EPI, int PN = 256, int IC = 0>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(640, 1)
    gemm_tf32x3_2sm_kernel(const __grid_constant__ CUtensorMap ta_hi, const __grid_constant__ CUtensorMap ta_lo,
                           const __grid_constant__ CUtensorMap tb_hi, const __grid_constant__ CUtensorMap tb_lo,
                           int num_kb, int num_m_pairs, int num_tiles, int kb_per_split, int num_units,
                           const __grid_constant__ GemmEpilogue ep, const __grid_constant__ CUtensorMap t_ones,
                           const ConvTmaArgs ic) {
  using Cfg = Gemm2smCfg<PN>;
  const int kChunkKb = ep.chunk_kb > 0 ? ep.chunk_kb : chunk_kb<A_MN, B_MN>();
  // TMA bytes one CTA brings per k-block (A hi/lo + B hi/lo).
  constexpr uint32_t kBLoaded = B_MN ? ((Cfg::kRowsB + 31) / 32) * 4096 : Cfg::kRowsB * 128;
  constexpr uint32_t kCtaBytes = 2 * Cfg::kABytes + 2 * kBLoaded;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + Cfg::kStages * Cfg::kStageBytes);
  uint64_t* empty_bar = full_bar + Cfg::kStages;
  uint64_t* tfull_bar = empty_bar + Cfg::kStages;  // [2]
  uint64_t* tempty_bar = tfull_bar + 2;            // [2], leader's copy is the live one
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const uint32_t warp = warp_idx_sync();
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t cta = cluster_ctarank();
  const bool leader = cta == 0;
  const int cluster_id = static_cast<int>(blockIdx.x >> 1), nclusters = static_cast<int>(gridDim.x >> 1);
  // Work unit u -> pair tile u % num_tiles, K-split u / num_tiles (split-K:
  // kEpiStoreScaled partials at out_hi + split * split_stride, summed by the
  // host launcher's fixup kernel).
  // Only kEpiStoreScaled instantiations take K-splits (the partials); the
  // others compile to the plain tile loop (registers are tight at 96/thread).
  constexpr bool kSplit = EPI == kEpiStoreScaled;
  auto unit = [&](int u, int& t, int& kb0, int& kb1, int& split) {
    if constexpr (kSplit) {
      t = u % num_tiles;
      split = u / num_tiles;
      kb0 = split * kb_per_split;
      kb1 = min(num_kb, kb0 + kb_per_split);
    } else {
      t = u, split = 0, kb0 = 0, kb1 = num_kb;
    }
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
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull_bar[b], 1);
      mbar_init(&tempty_bar[b], 2 * Cfg::kEpiWarps);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc_2sm(tmem_slot, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // Programmatic dependent launch (see gemm_tf32x3.cuh).
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");

  if (warp < 4) {
    if (warp == 0) {
      if (elect_one()) {
        const int ones_col = B_MN ? ep.ones_col_p1 - 1 : -1;
        int it = 0;
        for (int u = cluster_id; u < num_units; u += nclusters) {
          int t, kb0, kb1, split;
          unit(u, t, kb0, kb1, split);
          const int m0 = (t % num_m_pairs) * 256 + static_cast<int>(cta) * Cfg::kRowsA;
          const int n0 = (t / num_m_pairs) * Cfg::kPairN + static_cast<int>(cta) * Cfg::kRowsB;
          for (int kb = kb0; kb < kb1; ++kb, ++it) {
            const int s = it % Cfg::kStages;
            const uint32_t ph = (it / Cfg::kStages) & 1u;
            mbar_wait(&empty_bar[s], ph ^ 1u);
            if (leader) mbar_arrive_expect_tx(&full_bar[s], 2 * kCtaBytes);
            uint8_t* base = smem + s * Cfg::kStageBytes;
            if constexpr (IC == 1) {
              const int k = kb * kBK, tap = k / ic.c_in, c = k - tap * ic.c_in;
              int w, h, n;
              conv_origin(ic, ic.m_base + m0, w, h, n);
              const uint16_t ox = static_cast<uint16_t>(tap % 3), oy = static_cast<uint16_t>(tap / 3);
              tma_load_im2col_4d_2sm(base, &ta_hi, &full_bar[s], c, w, h, n, ox, oy);
              tma_load_im2col_4d_2sm(base + Cfg::kABytes, &ta_lo, &full_bar[s], c, w, h, n, ox, oy);
            } else {
              load_operand_2sm<A_MN, Cfg::kRowsA>(base, &ta_hi, &full_bar[s], m0, kb * kBK);
              load_operand_2sm<A_MN, Cfg::kRowsA>(base + Cfg::kABytes, &ta_lo, &full_bar[s], m0, kb * kBK);
            }
            if constexpr (IC == 2) {
              // B = im2col columns (conv wgrad, MN-major): this CTA's kRowsB
              // columns as 32-channel x 32-pixel boxes (N = tap * c_in + ci),
              // as in the 1-CTA kernel; the fused bias column loads ones.
              int w, h, n;
              conv_origin(ic, ic.k_base + kb * kBK, w, h, n);
#pragma unroll
              for (int cc = 0; cc < (Cfg::kRowsB + 31) / 32; ++cc) {
                const int col = n0 + cc * 32, tap = col / ic.c_in, c = col - tap * ic.c_in;
                uint8_t* dh = base + 2 * Cfg::kABytes + cc * 4096;
                if (col == ones_col) {
                  tma_load_2d_2sm(dh, &t_ones, &full_bar[s], 0, 0);
                  tma_load_2d_2sm(dh + Cfg::kBBytes, &t_ones, &full_bar[s], 0, 32);
                  continue;
                }
                const uint16_t ox = static_cast<uint16_t>(tap % 3), oy = static_cast<uint16_t>(tap / 3);
                tma_load_im2col_4d_2sm(dh, &tb_hi, &full_bar[s], c, w, h, n, ox, oy);
                tma_load_im2col_4d_2sm(dh + Cfg::kBBytes, &tb_lo, &full_bar[s], c, w, h, n, ox, oy);
              }
            } else {
              load_operand_2sm<B_MN, Cfg::kRowsB>(base + 2 * Cfg::kABytes, &tb_hi, &full_bar[s], n0, kb * kBK,
                                                  &t_ones, ones_col, 0);
              load_operand_2sm<B_MN, Cfg::kRowsB>(base + 2 * Cfg::kABytes + Cfg::kBBytes, &tb_lo, &full_bar[s], n0,
                                                  kb * kBK, &t_ones, ones_col, 32);
            }
          }
        }
      }
    } else if (warp == 1 && leader) {
      if (elect_one()) {
        constexpr uint32_t idesc = idesc_tf32(256, Cfg::kPairN, A_MN, B_MN);
        int it = 0, g = 0;
        for (int u = cluster_id; u < num_units; u += nclusters) {
          int t, kb0, kb1, split;
          unit(u, t, kb0, kb1, split);
          const int num_chunks = (kb1 - kb0 + kChunkKb - 1) / kChunkKb;
          for (int c = 0; c < num_chunks; ++c, ++g) {
            const uint32_t b = g & 1, tph = (g >> 1) & 1;
            mbar_wait(&tempty_bar[b], tph ^ 1u);  // both CTAs' epilogues drained buffer b
            tc_fence_after();
            const uint32_t acc_addr = tmem + b * Cfg::kPairN;
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
                umma_tf32_2sm(acc_addr, operand_desc<A_MN>(a_lo, kk), operand_desc<B_MN>(b_hi, kk), idesc, acc);
                umma_tf32_2sm(acc_addr, operand_desc<A_MN>(a_hi, kk), operand_desc<B_MN>(b_lo, kk), idesc, 1u);
                umma_tf32_2sm(acc_addr, operand_desc<A_MN>(a_hi, kk), operand_desc<B_MN>(b_hi, kk), idesc, 1u);
              }
              umma_commit_2sm(&empty_bar[s], 0x3);  // frees this stage in both CTAs
            }
            umma_commit_2sm(&tfull_bar[b], 0x3);  // chunk ready in both CTAs' TMEM
          }
        }
      }
    }
    __syncwarp();
  } else {
    const uint32_t q = warp & 3u;
    const int colbase = static_cast<int>((warp - 4) >> 2) * Cfg::kEpiCols;
    const int width = min(Cfg::kEpiCols, PN - colbase);  // this warp's accumulator columns
    const uint32_t lane_addr = (q * 32u) << 16;
    const uint32_t tempty_leader0 = mapa_shared(smem_u32(&tempty_bar[0]), 0);
    int g = 0;
    for (int u = cluster_id; u < num_units; u += nclusters) {
      int t, kb0, kb1, split;
      unit(u, t, kb0, kb1, split);
      const int num_chunks = (kb1 - kb0 + kChunkKb - 1) / kChunkKb;
      const long out_shift = EPI == kEpiStoreScaled ? split * ep.split_stride : 0;
      const int m0 = (t % num_m_pairs) * 256 + static_cast<int>(cta) * Cfg::kRowsA;
      const int n_pair0 = (t / num_m_pairs) * Cfg::kPairN;
      const int n0 = n_pair0 + colbase;
      const int n_lim = min(ep.N, n_pair0 + PN);
      const int bias_col = epi_bias_col(ep);
      float acc[Cfg::kEpiCols];
#pragma unroll
      for (int j = 0; j < Cfg::kEpiCols; ++j) acc[j] = 0.f;
      for (int c = 0; c < num_chunks; ++c, ++g) {
        const uint32_t b = g & 1, tph = (g >> 1) & 1;
        mbar_wait(&tfull_bar[b], tph);
        tc_fence_after();
#pragma unroll
        for (int c0 = 0; c0 < Cfg::kEpiCols; c0 += 16) {
          if (c0 >= width) break;
          float v[16];
          tmem_ld_32x32b_x16(tmem + lane_addr + b * Cfg::kPairN + colbase + c0, v);
#pragma unroll
          for (int j = 0; j < 16; ++j) acc[c0 + j] += v[j];
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(tempty_leader0 + b * 8);
      }
      const int row = m0 + static_cast<int>(q * 32 + lane);
#pragma unroll
      for (int c0 = 0; c0 < Cfg::kEpiCols; c0 += 32) {
        if (n0 + c0 == bias_col && c0 < width) bias_store<EPI>(ep, acc[c0], row);
        else if (n0 + c0 < n_lim) epilogue_chunk<EPI>(ep, acc + c0, row, n0 + c0, out_shift, n_lim);
      }
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_2sm(tmem, 512);
  }
}

}  // namespace spb
