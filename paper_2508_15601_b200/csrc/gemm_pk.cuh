// gemm_pk.cuh -- persistent W4A16 prefill GEMM for sm_100a (§8(a) rows a3-a10 at large M).
//
// Same data path as the tiled kernel (gemm_w4a16.cuh: PAPER.md §3.1 steps i-iv, P:179-182;
// §4.3's overlap of loads, I2F and tensor cores): LAYOUT v1 blobs and activation
// tiles arrive by bulk copy / TMA, four dequant warps turn each 64-k stage into the bf16/fp16
// operand (reading R6) in TMEM, one thread issues tcgen05.mma (M = 128 weight columns,
// N = NT tokens, K = 16) with fp32 accumulators in TMEM.  What changes (measured on the tiled
// kernel, profiles/r02: ~21K of ~54K cycles per 128 x 256 tile were outside the MMA -- CTA
// prologue, pipeline fill and epilogue -- so the tensor pipe was 62 % active):
//   * persistent CTAs (one per SM) walk the tiles p, p + P, ... of the banded raster order, so
//     the prologue is paid once and the producers run ahead into the next tile;
//   * two TMEM accumulators (tile t uses buffer t & 1): the MMA of tile t + 1 runs while four
//     dedicated epilogue warps drain tile t (tcgen05.ld -> RNE -> SMEM -> TMA 2-D store);
//   * NT = 192 tokens per tile so 2 x 192 accumulator columns + 4 x 32 operand columns fill
//     the 512 TMEM columns exactly.
//   * two dequant sets of four warps take alternate 64-k stages (one set's per-stage chain --
//     LDS, I2F, tcgen05.st x32 -- is about as long as a stage's MMAs at N = 192).
// Warps: 0 producer W (weights + s/z boxes), 1 MMA issuer (+ TMEM allocator), 2-5 dequant set
// 0, 6 producer A (activations), 7 spare, 8-11 epilogue, 12-15 dequant set 1.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "dequant.cuh"
#include "gemm_w4a16.cuh"
#include "ptx.cuh"

namespace w4k {

template <int NT, bool BF16>
struct PkCfg {
  static constexpr int STAGES = 5;
  static constexpr int ASTAGES = 4;
  static constexpr int NDS = 2;                      // dequant sets (4 warps each), alternate stages
  static constexpr int THREADS = 512;                // 16 warps
  static constexpr int ACT_BYTES = NT * 128;          // NT rows x 64 k (SW128)
  static constexpr int C_BYTES = NT * kBN * 2;        // bf16/fp16 C tile staging [NT][128]
  static constexpr int HDR = 1024;
  static constexpr int OFF_ACT = HDR;
  static constexpr int OFF_BLOB = OFF_ACT + STAGES * ACT_BYTES;
  static constexpr int OFF_SZ = OFF_BLOB + STAGES * kBlobBytes;
  static constexpr int OFF_C = OFF_SZ + kSZSlots * 2 * kSZBox;
  static constexpr int SMEM = 1024 + OFF_C + C_BYTES;
  static constexpr int TMEM_COLS = 512;
  static_assert(2 * NT + ASTAGES * 32 <= TMEM_COLS, "two accumulators + operand stages");
  static_assert(ACT_BYTES % 1024 == 0 && OFF_BLOB % 1024 == 0, "SW128 stages");
  static_assert(SMEM <= 227 * 1024, "shared memory");
  static_assert(NT % 16 == 0 && NT <= 256, "UMMA N");
};

// tile index -> (n-tile, first row) in the banded raster order of the tiled kernel: `band`
// m-tiles per n-tile, n-tiles fastest within a band
__device__ __forceinline__ void pk_tile(int tile, int n_tiles, int m_tiles, int band, int NT, int& nt, int& m0) {
  const int b0 = (tile / (band * n_tiles)) * band;
  const int rows = min(band, m_tiles - b0);
  const int within = tile - b0 * n_tiles;
  nt = within / rows;
  m0 = (b0 + within % rows) * NT;
}

template <int NT, bool BF16>
__global__ void __launch_bounds__(PkCfg<NT, BF16>::THREADS, 1)
    w4a16_gemm_pk_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_c,
                         const __grid_constant__ CUtensorMap tmap_s, const __grid_constant__ CUtensorMap tmap_z,
                         const GemmArgs args, const int n_tiles, const int m_tiles) {
  using Cfg = PkCfg<NT, BF16>;
  constexpr int STAGES = Cfg::STAGES, ASTAGES = Cfg::ASTAGES;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* const base_ptr = smem_raw + (base - smem_u32(smem_raw));
  const uint32_t bar_full = base;                          // STAGES (W + A producers, tx)
  const uint32_t bar_empty = bar_full + 8 * STAGES;        // STAGES (128 dequant + 1 MMA commit)
  const uint32_t bar_afull = bar_empty + 8 * STAGES;       // ASTAGES (128 dequant)
  const uint32_t bar_aempty = bar_afull + 8 * ASTAGES;     // ASTAGES (MMA commit)
  const uint32_t bar_szfull = bar_aempty + 8 * ASTAGES;    // kSZSlots (tx)
  const uint32_t bar_szempty = bar_szfull + 8 * kSZSlots;  // kSZSlots (128 dequant)
  const uint32_t bar_accf = bar_szempty + 8 * kSZSlots;    // 2 (MMA commit)
  const uint32_t bar_acce = bar_accf + 16;                 // 2 (128 epilogue)
  const uint32_t tmem_slot = bar_acce + 16;
  uint32_t* const tmem_slot_ptr = reinterpret_cast<uint32_t*>(base_ptr + (tmem_slot - base));
  const uint32_t act0 = base + Cfg::OFF_ACT, blob0 = base + Cfg::OFF_BLOB, sz0 = base + Cfg::OFF_SZ;
  const uint32_t cst = base + Cfg::OFF_C;
  const uint8_t* const blob_ptr0 = base_ptr + Cfg::OFF_BLOB;
  const uint8_t* const sz_ptr0 = base_ptr + Cfg::OFF_SZ;
  uint8_t* const c_ptr = base_ptr + Cfg::OFF_C;

  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
  const uint32_t lane = threadIdx.x & 31;
  const int P = gridDim.x, p = blockIdx.x;
  const int tiles = n_tiles * m_tiles;
  const int KS = args.K / kBK;
  const int gshift = args.group == 64 ? 6 : 7;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmap_a);
    prefetch_tmap(&tmap_c);
    prefetch_tmap(&tmap_s);
    prefetch_tmap(&tmap_z);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(bar_full + 8 * s, 2);
      mbar_init(bar_empty + 8 * s, 128 + 1);
    }
    for (int a = 0; a < ASTAGES; ++a) {
      mbar_init(bar_afull + 8 * a, 128);
      mbar_init(bar_aempty + 8 * a, 1);
    }
    for (int j = 0; j < kSZSlots; ++j) {
      mbar_init(bar_szfull + 8 * j, 1);
      mbar_init(bar_szempty + 8 * j, 128 * Cfg::NDS);  // every set releases every box once
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(bar_accf + 8 * b, 1);
      mbar_init(bar_acce + 8 * b, 128);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot_ptr;
  const uint32_t tmem_a0 = tmem_base + 2 * NT;  // ASTAGES x 32 operand columns after the accumulators
  grid_dependency_wait();  // A may be the previous kernel's output

  if (warp == 0) {
    // ------------------------------------------------------------ producer W: weights + s/z
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      const bool stream_weights = m_tiles == 1;
      int i = 0, gb = 0;  // global stage / s/z box counters
      for (int tile = p; tile < tiles; tile += P) {
        int nt, m0;
        pk_tile(tile, n_tiles, m_tiles, args.band, NT, nt, m0);
        const uint8_t* blob_g = args.packed + static_cast<size_t>(nt) * KS * kBlobBytes;
        for (int k = 0; k < KS; ++k, ++i) {
          if (((k * kBK) >> gshift) % 8 == 0 && ((k * kBK) & ((1 << gshift) - 1)) == 0) {  // first stage of a box
            const int j = gb % kSZSlots;
            mbar_wait(bar_szempty + 8 * j, ((gb / kSZSlots) & 1) ^ 1);
            const uint32_t fb = bar_szfull + 8 * j;
            mbar_arrive_expect_tx(fb, 2 * kSZBox);
            const int grow = (k * kBK) >> gshift;
            tma_load_2d(sz0 + j * 2 * kSZBox, &tmap_s, nt * kBN, grow, fb);
            tma_load_2d(sz0 + j * 2 * kSZBox + kSZBox, &tmap_z, nt * kBN, grow, fb);
            ++gb;
          }
          const int s = i % STAGES;
          mbar_wait(bar_empty + 8 * s, ((i / STAGES) & 1) ^ 1);
          const uint32_t fb = bar_full + 8 * s;
          mbar_arrive_expect_tx(fb, kBlobBytes);
          if (stream_weights)
            bulk_g2s_hint(blob0 + s * kBlobBytes, blob_g + static_cast<size_t>(k) * kBlobBytes, kBlobBytes, fb, pol);
          else
            bulk_g2s(blob0 + s * kBlobBytes, blob_g + static_cast<size_t>(k) * kBlobBytes, kBlobBytes, fb);
        }
      }
    }
    __syncwarp();
  } else if (warp == 6) {
    // ------------------------------------------------------------ producer A: activations
    if (lane == 0) {
      int i = 0;
      for (int tile = p; tile < tiles; tile += P) {
        int nt, m0;
        pk_tile(tile, n_tiles, m_tiles, args.band, NT, nt, m0);
        for (int k = 0; k < KS; ++k, ++i) {
          const int s = i % STAGES;
          mbar_wait(bar_empty + 8 * s, ((i / STAGES) & 1) ^ 1);
          const uint32_t fb = bar_full + 8 * s;
          mbar_arrive_expect_tx(fb, Cfg::ACT_BYTES);
          const int aks = k >= args.a_ks ? k - args.a_ks : k;  // W8: low planes reuse A
          tma_load_2d(act0 + s * Cfg::ACT_BYTES, &tmap_a, aks * kBK, m0, fb);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_f16(BF16, 128, NT);
      int i = 0, it = 0;
      for (int tile = p; tile < tiles; tile += P, ++it) {
        const int b = it & 1;
        mbar_wait(bar_acce + 8 * b, ((it >> 1) & 1) ^ 1);  // the epilogue drained this buffer
        tc_fence_after();
        const uint32_t acc = tmem_base + b * NT;
        for (int k = 0; k < KS; ++k, ++i) {
          const int s = i % STAGES, a = i % ASTAGES;
          mbar_wait(bar_full + 8 * s, (i / STAGES) & 1);
          mbar_wait(bar_afull + 8 * a, (i / ASTAGES) & 1);
          tc_fence_after();
          const uint32_t act = act0 + s * Cfg::ACT_BYTES;
#pragma unroll
          for (int j = 0; j < kBK / 16; ++j)
            mma_ts(acc, tmem_a0 + a * 32 + 8 * j, umma_desc_sw128(act + 32 * j), idesc, (k | j) != 0 ? 1u : 0u);
          tc_commit(bar_empty + 8 * s);
          tc_commit(bar_aempty + 8 * a);
        }
        tc_commit(bar_accf + 8 * b);
      }
    }
    __syncwarp();
  } else if ((warp >= 2 && warp < 6) || warp >= 12) {
    // ------------------------------------------------------------ dequant (set `set`: stages i % NDS == set)
    const int set = warp >= 12 ? 1 : 0;
    const int quarter = warp & 3;
    const int row = quarter * 32 + static_cast<int>(lane);
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    int i = 0, gb = -1, seen = -1;  // gb: global box counter (every box), seen: last box this set used
    for (int tile = p; tile < tiles; tile += P) {
      for (int k = 0; k < KS; ++k, ++i) {
        const int gl = (k * kBK) >> gshift;  // group of this stage within the tile
        if ((gl & 7) == 0 && ((k * kBK) & ((1 << gshift) - 1)) == 0) ++gb;  // first stage of a new box
        if (i % Cfg::NDS != set) continue;
        const int s = i % STAGES, a = i % ASTAGES;
        if (gb != seen) {
          if (seen >= 0) mbar_arrive(bar_szempty + 8 * (seen % kSZSlots));
          seen = gb;
          mbar_wait(bar_szfull + 8 * (gb % kSZSlots), (gb / kSZSlots) & 1);
        }
        mbar_wait(bar_full + 8 * s, (i / STAGES) & 1);
        const uint8_t* blob = blob_ptr0 + s * kBlobBytes;
        const uint4 w0 = *reinterpret_cast<const uint4*>(blob + row * 16);
        const uint4 w1 = *reinterpret_cast<const uint4*>(blob + 2048 + row * 16);
        const uint8_t* szb = sz_ptr0 + (gb % kSZSlots) * 2 * kSZBox + ((gl & 7) * kBN + row) * 2;
        const uint16_t sb = *reinterpret_cast<const uint16_t*>(szb);
        const uint16_t zb = *reinterpret_cast<const uint16_t*>(szb + kSZBox);
        mbar_arrive(bar_empty + 8 * s);
        uint32_t s2, z2;
        deq_prepare<BF16>(sb, zb, s2, z2);
        uint32_t r[32];
        deq_word<BF16>(w0.x, s2, z2, r + 0);
        deq_word<BF16>(w0.y, s2, z2, r + 4);
        deq_word<BF16>(w0.z, s2, z2, r + 8);
        deq_word<BF16>(w0.w, s2, z2, r + 12);
        deq_word<BF16>(w1.x, s2, z2, r + 16);
        deq_word<BF16>(w1.y, s2, z2, r + 20);
        deq_word<BF16>(w1.z, s2, z2, r + 24);
        deq_word<BF16>(w1.w, s2, z2, r + 28);
        mbar_wait(bar_aempty + 8 * a, ((i / ASTAGES) & 1) ^ 1);
        tc_fence_after();
        tmem_st_32x32b_x32(tmem_a0 + a * 32 + lane_off, r);
        tc_wait_st();
        tc_fence_before();
        mbar_arrive(bar_afull + 8 * a);
      }
    }
    if (seen >= 0) mbar_arrive(bar_szempty + 8 * (seen % kSZSlots));
  } else if (warp >= 8) {
    // ------------------------------------------------------------ epilogue
    const int quarter = warp & 3;
    const int row = quarter * 32 + static_cast<int>(lane);
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    const bool leader = warp == 8 && lane == 0;
    int it = 0;
    for (int tile = p; tile < tiles; tile += P, ++it) {
      int nt, m0;
      pk_tile(tile, n_tiles, m_tiles, args.band, NT, nt, m0);
      const int b = it & 1;
      mbar_wait(bar_accf + 8 * b, (it >> 1) & 1);
      tc_fence_after();
      if (leader) bulk_wait_group_read0();  // the previous tile's store has read the staging tile
      asm volatile("bar.sync 2, 128;" ::: "memory");
      const uint32_t acc = tmem_base + b * NT + lane_off;
#pragma unroll 1
      for (int c0 = 0; c0 < NT; c0 += 16) {
        uint32_t v[16];
        tmem_ld_32x32b_x16(acc + c0, v);
        tc_wait_ld();
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          uint8_t* dst = c_ptr + (static_cast<size_t>(c0 + c) * kBN + row) * 2;
          const float x = __uint_as_float(v[c]);
          if constexpr (BF16)
            *reinterpret_cast<__nv_bfloat16*>(dst) = __float2bfloat16_rn(x);
          else
            *reinterpret_cast<__half*>(dst) = __float2half_rn(x);
        }
      }
      tc_fence_before();
      mbar_arrive(bar_acce + 8 * b);  // the MMA may reuse this accumulator
      fence_proxy_async_shared();
      asm volatile("bar.sync 2, 128;" ::: "memory");
      if (leader) {
        tma_store_2d(&tmap_c, cst, nt * kBN, m0);  // rows >= M are clipped by the map
        bulk_commit_group();
      }
    }
    if (leader) bulk_wait_group_read0();  // shared memory must outlive the last store's read
  }
  __syncwarp();
  grid_dependency_launch();
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
}

}  // namespace w4k
