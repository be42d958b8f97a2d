// gemm_w4a16.cuh -- the online W4A16 GEMM for sm_100a (§8(a) rows a3-a10).
//
// PAPER.md §3.1: (i) load INT4 weights + fp16 scales to shared memory,
// (ii) move them to registers, (iii) I2F + scales, (iv) tensor-core MMA with the
// activations; §4.3: overlap tensor cores, I2F ALUs and async loads.
// B200 form, one CTA = 128 weight columns n x NT tokens x a K range:
//
//   warp 0      producer : per 64-k stage, cp.async.bulk of the 4 KB LAYOUT v1 blob,
//                          of the s and z rows (256 B each) and a TMA 2-D SW128 tile of
//                          NT x 64 activations -> SMEM ring slot, mbarrier full[s]
//   warp 1      MMA      : one thread issues 4 x tcgen05.mma.kind::f16 (M=128, N=NT,
//                          K=16) with A = dequantised weights in TMEM, B = activations
//                          (SMEM descriptor); tcgen05.commit frees the ring slot and
//                          the TMEM A stage; fp32 accumulator in TMEM
//   warps 2..5  dequant  : thread = weight column n (= TMEM lane): 2 x LDS.128 of its 64
//                          codes, LOP3 + sub.rn + mul.rn (dequant.cuh), tcgen05.st of 32
//                          bf16x2 columns into the TMEM A stage; after the mainloop they
//                          are the epilogue (tcgen05.ld -> RNE -> C[m][n])
//   split-K (S > 1, decode): the S CTAs of a cluster own disjoint K ranges of the same
//                          tile; ranks 1..S-1 push fp32 partials into rank 0's shared
//                          memory (DSMEM) and rank 0 sums them in rank order.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "dequant.cuh"
#include "ptx.cuh"

namespace w4k {

constexpr int kBN = 128;          // weight columns per CTA tile (= TMEM lanes)
constexpr int kBK = 64;           // k per pipeline stage
constexpr int kBlobBytes = 4096;  // packed bytes per (n-tile, k-stage)
constexpr int kSZBox = 8 * kBN * 2;  // one TMA box: 8 groups x 128 columns of fp16 (s or z)
constexpr int kSZSlots = 2;          // s/z box ring
constexpr int kThreads = 256;        // 8 warps (registers are allocated per SM sub-partition)

enum OutKind { OUT_ACT = 0, OUT_F32 = 1 };

struct GemmArgs {
  const uint8_t* packed;
  const uint16_t* scales;  // fp16 bits [K/g][N]
  const uint16_t* zeros;   // fp16 bits [K/g][N]
  void* out;               // [M][N] bf16/fp16 or fp32
  int M, N, K, group;
  int split;  // S: CTAs per tile along K (cluster size)
  int band;   // m-tiles per raster band (tile order below); >= 1
  int a_ks;   // 64-k stages of A along K: K / 64, or K / 128 for W8 bit planes (A reused)
  uint32_t* trace;  // optional per-CTA timeline (debug; nullptr in production)
};

constexpr int kTraceSlots = 160;
// trace slot layout per CTA: 0 globaltimer(ns) at start, 1 setup done, 2 producer start,
// 3+i producer issue of stage i, 35+i dequant full-wait done, 67+i dequant A-stage arrive,
// 99+i MMA issue, 131 epilogue start, 132 epilogue end, 133 kernel end (clock cycles since start)
#define TM_TRACE(slot)                                                                        \
  do {                                                                                        \
    if (args.trace)                                                                           \
      args.trace[(blockIdx.y * gridDim.x + blockIdx.x) * kTraceSlots + (slot)] =               \
          static_cast<uint32_t>(clock64() - t_start);                                         \
  } while (0)

template <int NT>
struct GemmCfg {
  static constexpr int STAGES = NT <= 32 ? 8 : (NT <= 64 ? 6 : 4);
  static constexpr int ASTAGES = NT >= 256 ? 4 : 2;
  static constexpr int ACT_BYTES = NT * 128;  // NT rows x 64 bf16
  static constexpr int ACC_COLS = NT < 32 ? 32 : NT;
  static constexpr int TMEM_NEED = ACC_COLS + ASTAGES * 32;
  static constexpr int TMEM_COLS = TMEM_NEED <= 32 ? 32 : TMEM_NEED <= 64 ? 64 : TMEM_NEED <= 128 ? 128 : TMEM_NEED <= 256 ? 256 : 512;
  static constexpr int HDR = 1024;  // barriers + tmem pointer
  static constexpr int RING = STAGES * (ACT_BYTES + kBlobBytes) + kSZSlots * 2 * kSZBox;
  // largest split-K whose DSMEM reduction buffer fits next to the header (<= ~200 KB)
  static constexpr int MAX_SPLIT = (1 + (200 * 1024) / (NT * kBN * 4)) < 8 ? (1 + (200 * 1024) / (NT * kBN * 4)) : 8;
  static int smem_bytes(int split) {
    const int red = (split - 1) * NT * kBN * 4;
    return 1024 /*align slack*/ + HDR + (RING > red ? RING : red);
  }
  static_assert(ACT_BYTES % 1024 == 0, "SW128 atoms need 1024-B aligned stages");
  // epilogue staging of the C tile (NT rows m x 128 n) for the TMA store, in the drained ring
  static_assert(RING >= NT * kBN * 4, "C staging fits the ring (fp32 worst case)");
  static_assert(TMEM_NEED <= 512, "TMEM overflow");
};

template <int NT, bool BF16, int OUT>
__global__ void __launch_bounds__(kThreads, 1)
    w4a16_gemm_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_c,
                      const __grid_constant__ CUtensorMap tmap_s, const __grid_constant__ CUtensorMap tmap_z,
                      const GemmArgs args) {
  using Cfg = GemmCfg<NT>;
  constexpr int STAGES = Cfg::STAGES;
  constexpr int ASTAGES = Cfg::ASTAGES;

  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* const base_ptr = smem_raw + (base - smem_u32(smem_raw));
  // header
  const uint32_t bar_full = base;                         // STAGES x 8 B
  const uint32_t bar_empty = bar_full + 8 * STAGES;       // STAGES x 8 B
  const uint32_t bar_afull = bar_empty + 8 * STAGES;      // ASTAGES x 8 B
  const uint32_t bar_aempty = bar_afull + 8 * ASTAGES;    // ASTAGES x 8 B
  const uint32_t bar_acc = bar_aempty + 8 * ASTAGES;      // 8 B
  const uint32_t bar_szfull = bar_acc + 8;                // kSZSlots x 8 B (producer W, tx)
  const uint32_t bar_szempty = bar_szfull + 8 * kSZSlots; // kSZSlots x 8 B (128 dequant threads)
  const uint32_t tmem_slot = bar_szempty + 8 * kSZSlots;  // 4 B
  uint32_t* const tmem_slot_ptr = reinterpret_cast<uint32_t*>(base_ptr + (tmem_slot - base));
  // ring
  const uint32_t ring = base + Cfg::HDR;
  const uint32_t act0 = ring;                                    // STAGES x ACT_BYTES
  const uint32_t blob0 = act0 + STAGES * Cfg::ACT_BYTES;         // STAGES x 4096
  const uint32_t sz0 = blob0 + STAGES * kBlobBytes;              // kSZSlots x [s box | z box]
  uint8_t* const ring_ptr = base_ptr + Cfg::HDR;
  const uint8_t* const blob_ptr0 = ring_ptr + STAGES * Cfg::ACT_BYTES;
  const uint8_t* const sz_ptr0 = blob_ptr0 + STAGES * kBlobBytes;

  const int warp = threadIdx.x >> 5;
  const uint32_t lane = threadIdx.x & 31;
  const long long t_start = clock64();
  if (args.trace && threadIdx.x == 0) {
    uint64_t gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    args.trace[(blockIdx.y * gridDim.x + blockIdx.x) * kTraceSlots] = static_cast<uint32_t>(gt);
  }

  // Tile order (L2 reuse): consecutive tiles walk a band of `band` m-tiles for one n-tile, then
  // the next n-tile, so the CTAs resident at one time read each weight column from DRAM once per
  // band (the band's activations, band x NT x K x 2 B, stay in L2); a CTA's split-K rank stays
  // the fastest index so the S CTAs of a cluster take consecutive block ids.
  const int S = args.split;
  const int rank = blockIdx.x % S;
  const int n_tiles = gridDim.x / S;
  const int m_tiles = gridDim.y;
  const int tile = (blockIdx.y * gridDim.x + blockIdx.x) / S;
  const int band = args.band;
  const int b0 = (tile / (band * n_tiles)) * band;           // first m-tile of this band
  const int rows = min(band, m_tiles - b0);                   // m-tiles in this band
  const int within = tile - b0 * n_tiles;
  const int nt = within / rows;
  const int m0 = (b0 + within % rows) * NT;
  const int KS = args.K / kBK;
  const int ks0 = static_cast<int>((static_cast<long long>(rank) * KS) / S);
  const int ks1 = static_cast<int>((static_cast<long long>(rank + 1) * KS) / S);
  const int nks = ks1 - ks0;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmap_a);
    prefetch_tmap(&tmap_s);
    prefetch_tmap(&tmap_z);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(bar_full + 8 * s, 2);         // weight producer + activation producer
      mbar_init(bar_empty + 8 * s, 128 + 1);  // 128 dequant threads + 1 MMA commit
    }
    for (int j = 0; j < kSZSlots; ++j) {
      mbar_init(bar_szfull + 8 * j, 1);
      mbar_init(bar_szempty + 8 * j, 128);
    }
    for (int a = 0; a < ASTAGES; ++a) {
      mbar_init(bar_afull + 8 * a, 128);
      mbar_init(bar_aempty + 8 * a, 1);
    }
    mbar_init(bar_acc, 1);
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
  if (threadIdx.x == 0) TM_TRACE(1);
  const uint32_t tmem_acc = tmem_base;
  const uint32_t tmem_a0 = tmem_base + Cfg::ACC_COLS;

  // PDL: everything above overlaps the previous kernel's tail; global reads start below.
  grid_dependency_wait();

  // groups of this CTA's K range; s/z arrive as 8-group x 128-column TMA boxes
  const int gshift = args.group == 64 ? 6 : 7;
  const int g_start = (ks0 * kBK) >> gshift;
  if (warp == 0) {
    // ------------------------------------------------------------ producer W: weights + s/z
    // (one request per stage here and one per stage on the activation producer: a bulk/TMA
    // request costs its issuing warp ~300 cycles, four per stage on one warp paced the loop)
    if (lane == 0) {
      const uint8_t* blob_g = args.packed + (static_cast<size_t>(nt) * KS + ks0) * kBlobBytes;
      const uint64_t pol_stream = policy_evict_first();
      const bool stream_weights = gridDim.y == 1;  // weights read once: do not keep them in L2
      TM_TRACE(2);
      int box = -1;
      for (int i = 0; i < nks; ++i) {
        const int s = i % STAGES;
        const uint32_t ph = (i / STAGES) & 1;
        const int gb = ((((ks0 + i) * kBK) >> gshift) - g_start) >> 3;  // box of this stage
        if (gb != box) {
          box = gb;
          const int j = box % kSZSlots;
          mbar_wait(bar_szempty + 8 * j, ((box / kSZSlots) & 1) ^ 1);
          const uint32_t fb = bar_szfull + 8 * j;
          mbar_arrive_expect_tx(fb, 2 * kSZBox);
          tma_load_2d(sz0 + j * 2 * kSZBox, &tmap_s, nt * kBN, g_start + 8 * box, fb);
          tma_load_2d(sz0 + j * 2 * kSZBox + kSZBox, &tmap_z, nt * kBN, g_start + 8 * box, fb);
        }
        mbar_wait(bar_empty + 8 * s, ph ^ 1);
        if (i < 32) TM_TRACE(3 + i);
        const uint32_t fb = bar_full + 8 * s;
        mbar_arrive_expect_tx(fb, kBlobBytes);
        if (stream_weights)
          bulk_g2s_hint(blob0 + s * kBlobBytes, blob_g + static_cast<size_t>(i) * kBlobBytes, kBlobBytes, fb,
                        pol_stream);
        else
          bulk_g2s(blob0 + s * kBlobBytes, blob_g + static_cast<size_t>(i) * kBlobBytes, kBlobBytes, fb);
      }
    }
    __syncwarp();
  } else if (warp == 6) {
    // ------------------------------------------------------------ producer A: activations
    if (lane == 0) {
      for (int i = 0; i < nks; ++i) {
        const int s = i % STAGES;
        const uint32_t ph = (i / STAGES) & 1;
        mbar_wait(bar_empty + 8 * s, ph ^ 1);
        const uint32_t fb = bar_full + 8 * s;
        mbar_arrive_expect_tx(fb, Cfg::ACT_BYTES);
        const int aks = ks0 + i >= args.a_ks ? ks0 + i - args.a_ks : ks0 + i;  // W8: low planes reuse A
        tma_load_2d(act0 + s * Cfg::ACT_BYTES, &tmap_a, aks * kBK, m0, fb);
      }
    }
    __syncwarp();
  } else if (warp == 7) {
    // spare warp (keeps the CTA a multiple of 4 warps)
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_f16(BF16, 128, NT);
      for (int i = 0; i < nks; ++i) {
        const int s = i % STAGES;
        const uint32_t ph = (i / STAGES) & 1;
        const int a = i % ASTAGES;
        const uint32_t aph = (i / ASTAGES) & 1;
        mbar_wait(bar_full + 8 * s, ph);
        mbar_wait(bar_afull + 8 * a, aph);
        tc_fence_after();
        if (i < 32) TM_TRACE(99 + i);
        const uint32_t act = act0 + s * Cfg::ACT_BYTES;
#pragma unroll
        for (int j = 0; j < kBK / 16; ++j) {
          const uint64_t bdesc = umma_desc_sw128(act + 32 * j);
          mma_ts(tmem_acc, tmem_a0 + a * 32 + 8 * j, bdesc, idesc, (i | j) != 0 ? 1u : 0u);
        }
        tc_commit(bar_empty + 8 * s);
        tc_commit(bar_aempty + 8 * a);
      }
      tc_commit(bar_acc);
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ dequant warps
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    const int row = quarter * 32 + static_cast<int>(lane);
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    int box = -1;
    for (int i = 0; i < nks; ++i) {
      const int s = i % STAGES;
      const uint32_t ph = (i / STAGES) & 1;
      const int a = i % ASTAGES;
      const uint32_t aph = (i / ASTAGES) & 1;
      const int gl = (((ks0 + i) * kBK) >> gshift) - g_start;  // group within this CTA's range
      if ((gl >> 3) != box) {
        if (box >= 0) mbar_arrive(bar_szempty + 8 * (box % kSZSlots));
        box = gl >> 3;
        mbar_wait(bar_szfull + 8 * (box % kSZSlots), (box / kSZSlots) & 1);
      }
      mbar_wait(bar_full + 8 * s, ph);
      if (i < 32 && warp == 2 && lane == 0) TM_TRACE(35 + i);
      const uint8_t* blob = blob_ptr0 + s * kBlobBytes;
      const uint4 w0 = *reinterpret_cast<const uint4*>(blob + row * 16);
      const uint4 w1 = *reinterpret_cast<const uint4*>(blob + 2048 + row * 16);
      const uint8_t* szb = sz_ptr0 + (box % kSZSlots) * 2 * kSZBox + ((gl & 7) * kBN + row) * 2;
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
      mbar_wait(bar_aempty + 8 * a, aph ^ 1);
      tc_fence_after();
      tmem_st_32x32b_x32(tmem_a0 + a * 32 + lane_off, r);
      tc_wait_st();
      tc_fence_before();
      mbar_arrive(bar_afull + 8 * a);
      if (i < 32 && warp == 2 && lane == 0) TM_TRACE(67 + i);
    }

    if (box >= 0) mbar_arrive(bar_szempty + 8 * (box % kSZSlots));

    // ------------------------------------------------------------ epilogue
    mbar_wait(bar_acc, 0);
    tc_fence_after();
    if (warp == 2 && lane == 0) TM_TRACE(131);
    const int n = nt * kBN + row;
    if (S > 1 && rank != 0) {
      // wait until rank 0 has drained its ring, then push fp32 partials into its SMEM
      cluster_arrive();
      cluster_wait();
      const uint32_t red_remote = mapa_shared(ring, 0) + static_cast<uint32_t>((rank - 1) * NT * kBN * 4);
#pragma unroll
      for (int c0 = 0; c0 < NT; c0 += 16) {
        uint32_t v[16];
        tmem_ld_32x32b_x16(tmem_acc + lane_off + c0, v);
        tc_wait_ld();
#pragma unroll
        for (int c = 0; c < 16; ++c)
          st_cluster_f32(red_remote + static_cast<uint32_t>(((c0 + c) * kBN + row) * 4), __uint_as_float(v[c]));
      }
      cluster_arrive();
      cluster_wait();
    } else if (S == 1) {
      // C tile -> shared memory [m][128 n] (row = 256 B bf16 / 512 B fp32; each warp writes 64 or
      // 128 contiguous bytes per m) -> one TMA 2-D store; rows m >= M are clipped by the map.
      // (Direct 2-byte global stores per (m, n) were measured at ~18k cycles per 256 x 128 tile,
      // a quarter of the CTA's time.)
      constexpr int ES = OUT == OUT_F32 ? 4 : 2;
      uint8_t* const stage = ring_ptr;
#pragma unroll 1
      for (int c0 = 0; c0 < NT; c0 += 16) {
        uint32_t v[16];
        tmem_ld_32x32b_x16(tmem_acc + lane_off + c0, v);
        tc_wait_ld();
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          uint8_t* dst = stage + (static_cast<size_t>(c0 + c) * kBN + row) * ES;
          const float x = __uint_as_float(v[c]);
          if constexpr (OUT == OUT_F32) {
            *reinterpret_cast<float*>(dst) = x;
          } else if constexpr (BF16) {
            *reinterpret_cast<__nv_bfloat16*>(dst) = __float2bfloat16_rn(x);
          } else {
            *reinterpret_cast<__half*>(dst) = __float2half_rn(x);
          }
        }
      }
      fence_proxy_async_shared();
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (warp == 2 && lane == 0) {
        constexpr int BOXM = NT < 256 ? NT : 256;
        constexpr int ROWS_PER_STORE = ES == 4 && NT > 128 ? 128 : BOXM;  // fp32 map box is 128 rows
        for (int r0 = 0; r0 < NT; r0 += ROWS_PER_STORE)
          if (m0 + r0 < args.M) tma_store_2d(&tmap_c, ring + r0 * kBN * ES, nt * kBN, m0 + r0);
        bulk_commit_group();
        bulk_wait_group_read0();  // the ring must stay intact until the store has read it
      }
    } else {
      if (S > 1) {
        cluster_arrive();
        cluster_wait();
        cluster_arrive();
        cluster_wait();
      }
      const float* red = reinterpret_cast<const float*>(ring_ptr);
#pragma unroll 1
      for (int c0 = 0; c0 < NT; c0 += 16) {
        uint32_t v[16];
        tmem_ld_32x32b_x16(tmem_acc + lane_off + c0, v);
        tc_wait_ld();
        float acc[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) acc[c] = __uint_as_float(v[c]);
        for (int r2 = 1; r2 < S; ++r2) {
#pragma unroll
          for (int c = 0; c < 16; ++c) acc[c] += red[((r2 - 1) * NT + c0 + c) * kBN + row];
        }
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          const int m = m0 + c0 + c;
          if (m < args.M) {
            const size_t idx = static_cast<size_t>(m) * args.N + n;
            if constexpr (OUT == OUT_F32) {
              reinterpret_cast<float*>(args.out)[idx] = acc[c];
            } else if constexpr (BF16) {
              reinterpret_cast<__nv_bfloat16*>(args.out)[idx] = __float2bfloat16_rn(acc[c]);
            } else {
              reinterpret_cast<__half*>(args.out)[idx] = __float2half_rn(acc[c]);
            }
          }
        }
      }
    }
  }

  if (S > 1 && (warp < 2 || warp >= 6)) {
    // producer, MMA and spare warps take part in the two cluster barriers of the epilogue
    cluster_arrive();
    cluster_wait();
    cluster_arrive();
    cluster_wait();
  }
  if (warp == 2 && lane == 0) TM_TRACE(132);
  grid_dependency_launch();
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) TM_TRACE(133);
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
}

}  // namespace w4k
