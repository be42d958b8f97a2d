// gemm_sk.cuh -- persistent stream-K W4A16 GEMM for sm_100a (§8(a) rows a3-a10).
//
// Same method as PAPER.md §3.1 steps i-iv and §4.3's overlap of loads, I2F and
// tensor cores, organised for B200 after measuring:
//   * a bulk/TMA request costs its issuing warp ~250-360 cycles, so the kernel moves
//     weights in 16 KB chunks (4 LAYOUT v1 blobs, one contiguous cp.async.bulk), the
//     activations of a chunk with one 3-D TMA box, and s/z for 8 groups per 2-D TMA box,
//     from two producer warps;
//   * every CTA is persistent and owns an equal contiguous range of the (tile, k-chunk)
//     sequence (stream-K), so all SMs stream the same number of weight bytes; tiles split
//     between CTAs are reduced through a global fp32 workspace in fixed k order by the
//     last-arriving contributor (deterministic, no float atomics).
//
// Warp roles (352 threads):
//   0      producer W : weight chunks (1-D bulk, may start before griddepcontrol.wait since
//                       weights never depend on the previous kernel) + s/z boxes (2-D TMA)
//   1      MMA        : one thread; 4 x tcgen05.mma.kind::f16 (M=128 weights from TMEM,
//                       N=NT tokens from SMEM, K=16) per 64-k blob; commits free the SMEM
//                       stage, the TMEM A stage, and signal the accumulator
//   2..5   dequant    : thread = weight column = TMEM lane; LDS.128 x 2 per blob, LOP3 magic
//                       I2F + exact sub + one rounding mul (dequant.cuh), tcgen05.st
//   6      producer A : activation chunk (3-D TMA, SW128), after griddepcontrol.wait
//   7..10  epilogue   : tcgen05.ld of a finished accumulator (double-buffered), RNE store of
//                       C, or fp32 partial + stream-K fix-up
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "dequant.cuh"
#include "ptx.cuh"

namespace w4k {

constexpr int kSkThreads = 352;

struct SkArgs {
  const uint8_t* packed;   // LAYOUT v1
  void* out;               // [M][N] bf16/fp16 or fp32
  float* workspace;        // [2 * P][NT][128] fp32 partial slots
  int* counters;           // [m_tiles * n_tiles] arrival counters (zero between launches)
  int M, N, K, group;
  int n_tiles, m_tiles;
  int kc;                  // chunks per tile = ceil(K / CH)
  long long total;         // m_tiles * n_tiles * kc
  uint32_t* trace;         // optional timeline (debug)
};

template <int NT>
struct SkCfg {
  static constexpr int CH = NT <= 64 ? 256 : (NT <= 128 ? 128 : 64);  // k per chunk
  static constexpr int BLOBS = CH / 64;
  static constexpr int ACT_BYTES = NT * CH * 2;
  static constexpr int W_BYTES = BLOBS * 4096;
  static constexpr int STAGE_BYTES = ACT_BYTES + W_BYTES;
  static constexpr int STAGES = NT <= 16 ? 4 : (NT <= 32 ? 3 : (NT <= 64 ? 2 : 3));
  static constexpr int SZG = 8;                       // groups per s/z box
  static constexpr int SZ_BOX = SZG * 128 * 2;        // bytes of one s (or z) box
  static constexpr int SZ_SLOTS = 2;
  static constexpr int ASTAGES = NT <= 64 ? 12 : 8;   // TMEM A stages (one blob = 32 columns): deep
                                                      // enough to cover the MMA commit round trip
  static constexpr int ACC_COLS = NT < 32 ? 32 : NT;  // one accumulator buffer
  static constexpr int ACC_BUFS = NT <= 128 ? 2 : 1;
  static constexpr int TMEM_NEED = ACC_BUFS * ACC_COLS + ASTAGES * 32;
  static constexpr int TMEM_COLS = TMEM_NEED <= 64 ? 64 : TMEM_NEED <= 128 ? 128 : TMEM_NEED <= 256 ? 256 : 512;
  static constexpr int HDR = 1024;
  static constexpr int SMEM = 1024 + HDR + STAGES * STAGE_BYTES + SZ_SLOTS * 2 * SZ_BOX;
  static_assert(ACT_BYTES % 1024 == 0 && (NT * 128) % 1024 == 0, "SW128 sub-tiles must be 1 KB aligned");
  static_assert(SMEM <= 227 * 1024, "shared memory");
};

// owner CTA of linear chunk u when T chunks are split into P contiguous ranges
__device__ __forceinline__ int sk_owner(long long u, long long T, int P) {
  return static_cast<int>(((u + 1) * P - 1) / T);
}
__device__ __forceinline__ long long sk_start(int p, long long T, int P) { return (static_cast<long long>(p) * T) / P; }

// store 16 fp32 accumulator columns (tokens m0..m0+15 of weight column n) as the output dtype
template <bool BF16, int OUT>
__device__ __forceinline__ void sk_store16(void* out, int N, int m0, int n, int valid, const uint32_t (&v)[16]) {
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    if (c < valid) {
      const size_t idx = static_cast<size_t>(m0 + c) * N + n;
      const float x = __uint_as_float(v[c]);
      if constexpr (OUT == 1) {
        reinterpret_cast<float*>(out)[idx] = x;
      } else if constexpr (BF16) {
        reinterpret_cast<__nv_bfloat16*>(out)[idx] = __float2bfloat16_rn(x);
      } else {
        reinterpret_cast<__half*>(out)[idx] = __float2half_rn(x);
      }
    }
  }
}

#define SK_TRACE(slot)                                                                          \
  do {                                                                                          \
    if (args.trace) args.trace[blockIdx.x * 160 + (slot)] = static_cast<uint32_t>(clock64() - t_start); \
  } while (0)

template <int NT, bool BF16, int OUT>
__global__ void __launch_bounds__(kSkThreads, 1)
    w4a16_sk_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_s,
                    const __grid_constant__ CUtensorMap tmap_z, const SkArgs args) {
  using Cfg = SkCfg<NT>;
  constexpr int STAGES = Cfg::STAGES;
  constexpr int ASTAGES = Cfg::ASTAGES;
  constexpr int CH = Cfg::CH;
  constexpr int ACC_BUFS = Cfg::ACC_BUFS;

  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* const base_ptr = smem_raw + (base - smem_u32(smem_raw));
  const uint32_t bar_full = base;                              // STAGES (count 2: W + A producers)
  const uint32_t bar_empty = bar_full + 8 * STAGES;            // STAGES (128 dequant + 1 MMA commit)
  const uint32_t bar_afull = bar_empty + 8 * STAGES;           // ASTAGES (128)
  const uint32_t bar_aempty = bar_afull + 8 * ASTAGES;         // ASTAGES (1 commit)
  const uint32_t bar_szfull = bar_aempty + 8 * ASTAGES;        // SZ_SLOTS (1)
  const uint32_t bar_szempty = bar_szfull + 8 * Cfg::SZ_SLOTS;  // SZ_SLOTS (128)
  const uint32_t bar_accfull = bar_szempty + 8 * Cfg::SZ_SLOTS;  // ACC_BUFS (1 commit)
  const uint32_t bar_accempty = bar_accfull + 8 * ACC_BUFS;    // ACC_BUFS (128 epilogue)
  const uint32_t tmem_slot = bar_accempty + 8 * ACC_BUFS;
  int* const bcast = reinterpret_cast<int*>(base_ptr + (tmem_slot - base) + 16);
  uint32_t* const tmem_slot_ptr = reinterpret_cast<uint32_t*>(base_ptr + (tmem_slot - base));
  const uint32_t stage0 = base + Cfg::HDR;                     // STAGES x [act | weights]
  const uint32_t sz0 = stage0 + STAGES * Cfg::STAGE_BYTES;     // SZ_SLOTS x [s box | z box]
  const uint8_t* const stage_ptr0 = base_ptr + Cfg::HDR;
  const uint8_t* const sz_ptr0 = stage_ptr0 + STAGES * Cfg::STAGE_BYTES;

  const int warp = threadIdx.x >> 5;
  const uint32_t lane = threadIdx.x & 31;
  const long long t_start = clock64();

  const int P = gridDim.x;
  const int p = blockIdx.x;
  const long long T = args.total;
  const long long u0 = sk_start(p, T, P);
  const long long u1 = sk_start(p + 1, T, P);
  const int KS = args.K / 64;
  const int kc = args.kc;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmap_a);
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
    for (int j = 0; j < Cfg::SZ_SLOTS; ++j) {
      mbar_init(bar_szfull + 8 * j, 1);
      mbar_init(bar_szempty + 8 * j, 128);
    }
    for (int b = 0; b < ACC_BUFS; ++b) {
      mbar_init(bar_accfull + 8 * b, 1);
      mbar_init(bar_accempty + 8 * b, 128);
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
  const uint32_t tmem_a0 = tmem_base + ACC_BUFS * Cfg::ACC_COLS;

  // chunks per s/z box (boxes are segment-relative, 8 groups each; a box spans whole chunks)
  const int gshift = args.group == 64 ? 6 : 7;
  const int chunks_per_box = (Cfg::SZG << gshift) / CH;

  if (warp == 0) {
    // ---------------------------------------------------------------- producer W (+ s/z)
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int i = 0, box = 0;
      for (long long u = u0; u < u1;) {
        const int t = static_cast<int>(u / kc);
        const long long cend = (static_cast<long long>(t) + 1) * kc < u1 ? (static_cast<long long>(t) + 1) * kc : u1;
        const int nt = t % args.n_tiles;
        const int c0 = static_cast<int>(u - static_cast<long long>(t) * kc);
        const int c1 = static_cast<int>(cend - static_cast<long long>(t) * kc);
        for (int c = c0; c < c1; ++c, ++i) {
          if ((c - c0) % chunks_per_box == 0) {
            const int j = box % Cfg::SZ_SLOTS;
            mbar_wait(bar_szempty + 8 * j, ((box / Cfg::SZ_SLOTS) & 1) ^ 1);
            const uint32_t fb = bar_szfull + 8 * j;
            mbar_arrive_expect_tx(fb, 2 * Cfg::SZ_BOX);
            const int g0 = (c * CH) >> gshift;
            tma_load_2d(sz0 + j * 2 * Cfg::SZ_BOX, &tmap_s, nt * 128, g0, fb);
            tma_load_2d(sz0 + j * 2 * Cfg::SZ_BOX + Cfg::SZ_BOX, &tmap_z, nt * 128, g0, fb);
            ++box;
          }
          const int s = i % STAGES;
          mbar_wait(bar_empty + 8 * s, ((i / STAGES) & 1) ^ 1);
          const int kb0 = c * Cfg::BLOBS;
          const int nb = (KS - kb0) < Cfg::BLOBS ? (KS - kb0) : Cfg::BLOBS;
          const uint32_t fb = bar_full + 8 * s;
          mbar_arrive_expect_tx(fb, nb * 4096);
          bulk_g2s_hint(stage0 + s * Cfg::STAGE_BYTES + Cfg::ACT_BYTES,
                        args.packed + (static_cast<size_t>(nt) * KS + kb0) * 4096, nb * 4096, fb, pol);
          if (i < 32) SK_TRACE(3 + i);
        }
        u = cend;
      }
    }
    __syncwarp();
  } else if (warp == 6) {
    // ---------------------------------------------------------------- producer A
    if (lane == 0) {
      grid_dependency_wait();  // activations may be produced by the previous kernel
      int i = 0;
      for (long long u = u0; u < u1;) {
        const int t = static_cast<int>(u / kc);
        const long long cend = (static_cast<long long>(t) + 1) * kc < u1 ? (static_cast<long long>(t) + 1) * kc : u1;
        const int mt = t / args.n_tiles;
        const int c0 = static_cast<int>(u - static_cast<long long>(t) * kc);
        const int c1 = static_cast<int>(cend - static_cast<long long>(t) * kc);
        for (int c = c0; c < c1; ++c, ++i) {
          const int s = i % STAGES;
          mbar_wait(bar_empty + 8 * s, ((i / STAGES) & 1) ^ 1);
          const uint32_t fb = bar_full + 8 * s;
          mbar_arrive_expect_tx(fb, Cfg::ACT_BYTES);
          tma_load_3d(stage0 + s * Cfg::STAGE_BYTES, &tmap_a, 0, mt * NT, c * Cfg::BLOBS, fb);
        }
        u = cend;
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_f16(BF16, 128, NT);
      int i = 0, ia = 0, seg = 0;
      for (long long u = u0; u < u1; ++seg) {
        const int t = static_cast<int>(u / kc);
        const long long cend = (static_cast<long long>(t) + 1) * kc < u1 ? (static_cast<long long>(t) + 1) * kc : u1;
        const int c0 = static_cast<int>(u - static_cast<long long>(t) * kc);
        const int c1 = static_cast<int>(cend - static_cast<long long>(t) * kc);
        const int b = seg % ACC_BUFS;
        mbar_wait(bar_accempty + 8 * b, ((seg / ACC_BUFS) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + b * Cfg::ACC_COLS;
        bool first = true;
        for (int c = c0; c < c1; ++c, ++i) {
          const int s = i % STAGES;
          mbar_wait(bar_full + 8 * s, (i / STAGES) & 1);
          const int kb0 = c * Cfg::BLOBS;
          const int nb = (KS - kb0) < Cfg::BLOBS ? (KS - kb0) : Cfg::BLOBS;
          const uint32_t act = stage0 + s * Cfg::STAGE_BYTES;
          for (int bb = 0; bb < nb; ++bb, ++ia) {
            const int a = ia % ASTAGES;
            mbar_wait(bar_afull + 8 * a, (ia / ASTAGES) & 1);
            tc_fence_after();
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const uint64_t bdesc = umma_desc_sw128(act + bb * (NT * 128) + 32 * j);
              mma_ts(d_tmem, tmem_a0 + a * 32 + 8 * j, bdesc, idesc, first ? 0u : 1u);
              first = false;
            }
            tc_commit(bar_aempty + 8 * a);
          }
          tc_commit(bar_empty + 8 * s);
          if (i < 32) SK_TRACE(99 + i);
        }
        tc_commit(bar_accfull + 8 * b);
        u = cend;
      }
    }
    __syncwarp();
  } else if (warp >= 2 && warp <= 5) {
    // ---------------------------------------------------------------- dequant
    const int quarter = warp & 3;
    const int row = quarter * 32 + static_cast<int>(lane);
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    int i = 0, ia = 0, box = -1;
    for (long long u = u0; u < u1;) {
      const int t = static_cast<int>(u / kc);
      const long long cend = (static_cast<long long>(t) + 1) * kc < u1 ? (static_cast<long long>(t) + 1) * kc : u1;
      const int c0 = static_cast<int>(u - static_cast<long long>(t) * kc);
      const int c1 = static_cast<int>(cend - static_cast<long long>(t) * kc);
      int g_base = 0;
      for (int c = c0; c < c1; ++c, ++i) {
        if ((c - c0) % chunks_per_box == 0) {
          if (box >= 0) mbar_arrive(bar_szempty + 8 * (box % Cfg::SZ_SLOTS));
          ++box;
          mbar_wait(bar_szfull + 8 * (box % Cfg::SZ_SLOTS), (box / Cfg::SZ_SLOTS) & 1);
          g_base = (c * CH) >> gshift;
        }
        const uint8_t* szs = sz_ptr0 + (box % Cfg::SZ_SLOTS) * 2 * Cfg::SZ_BOX;
        const int s = i % STAGES;
        mbar_wait(bar_full + 8 * s, (i / STAGES) & 1);
        if (i < 32 && warp == 2 && lane == 0) SK_TRACE(35 + i);
        const uint8_t* wst = stage_ptr0 + s * Cfg::STAGE_BYTES + Cfg::ACT_BYTES;
        const int kb0 = c * Cfg::BLOBS;
        const int nb = (KS - kb0) < Cfg::BLOBS ? (KS - kb0) : Cfg::BLOBS;
        uint4 wv[2 * Cfg::BLOBS];
#pragma unroll
        for (int bb = 0; bb < Cfg::BLOBS; ++bb) {
          if (bb < nb) {
            wv[2 * bb] = *reinterpret_cast<const uint4*>(wst + bb * 4096 + row * 16);
            wv[2 * bb + 1] = *reinterpret_cast<const uint4*>(wst + bb * 4096 + 2048 + row * 16);
          }
        }
        mbar_arrive(bar_empty + 8 * s);  // codes are in registers; the MMA commit covers the activations
        // software pipeline: the tcgen05.st of blob b completes while blob b+1 is dequantised
        uint32_t ra[32], rb[32];
        int pend = -1;
#pragma unroll
        for (int bb = 0; bb < Cfg::BLOBS; ++bb) {
          if (bb < nb) {
            uint32_t(&r)[32] = (bb & 1) ? rb : ra;
            const int gi = (((kb0 + bb) * 64) >> gshift) - g_base;
            const uint16_t sb = *reinterpret_cast<const uint16_t*>(szs + gi * 256 + row * 2);
            const uint16_t zb = *reinterpret_cast<const uint16_t*>(szs + Cfg::SZ_BOX + gi * 256 + row * 2);
            uint32_t s2, z2;
            deq_prepare<BF16>(sb, zb, s2, z2);
            deq_word<BF16>(wv[2 * bb].x, s2, z2, r + 0);
            deq_word<BF16>(wv[2 * bb].y, s2, z2, r + 4);
            deq_word<BF16>(wv[2 * bb].z, s2, z2, r + 8);
            deq_word<BF16>(wv[2 * bb].w, s2, z2, r + 12);
            deq_word<BF16>(wv[2 * bb + 1].x, s2, z2, r + 16);
            deq_word<BF16>(wv[2 * bb + 1].y, s2, z2, r + 20);
            deq_word<BF16>(wv[2 * bb + 1].z, s2, z2, r + 24);
            deq_word<BF16>(wv[2 * bb + 1].w, s2, z2, r + 28);
            if (pend >= 0) {
              tc_wait_st();
              tc_fence_before();
              mbar_arrive(bar_afull + 8 * pend);
            }
            const int a = ia % ASTAGES;
            mbar_wait(bar_aempty + 8 * a, ((ia / ASTAGES) & 1) ^ 1);
            tc_fence_after();
            tmem_st_32x32b_x32(tmem_a0 + a * 32 + lane_off, r);
            pend = a;
            ++ia;
          }
        }
        if (pend >= 0) {
          tc_wait_st();
          tc_fence_before();
          mbar_arrive(bar_afull + 8 * pend);
        }
        if (i < 32 && warp == 2 && lane == 0) SK_TRACE(67 + i);
      }
      u = cend;
    }
    if (box >= 0) mbar_arrive(bar_szempty + 8 * (box % Cfg::SZ_SLOTS));
  } else if (warp >= 7) {
    // ---------------------------------------------------------------- epilogue
    const int quarter = warp & 3;
    const int row = quarter * 32 + static_cast<int>(lane);
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    const int et = threadIdx.x - 7 * 32;  // 0..127
    int seg = 0;
    for (long long u = u0; u < u1; ++seg) {
      const int t = static_cast<int>(u / kc);
      const long long cend = (static_cast<long long>(t) + 1) * kc < u1 ? (static_cast<long long>(t) + 1) * kc : u1;
      const int nt = t % args.n_tiles;
      const int mt = t / args.n_tiles;
      const long long tile_lo = static_cast<long long>(t) * kc;
      const long long tile_hi = tile_lo + kc;
      const bool full = (u == tile_lo) && (cend == tile_hi);
      const int b = seg % ACC_BUFS;
      mbar_wait(bar_accfull + 8 * b, (seg / ACC_BUFS) & 1);
      tc_fence_after();
      const int n = nt * 128 + row;
      const int m0 = mt * NT;
      const int mcount = (args.M - m0) < NT ? (args.M - m0) : NT;
      const uint32_t tacc = tmem_base + b * Cfg::ACC_COLS + lane_off;
      if (full) {
#pragma unroll 1
        for (int c0 = 0; c0 < NT; c0 += 16) {
          uint32_t v[16];
          tmem_ld_32x32b_x16(tacc + c0, v);
          tc_wait_ld();
          sk_store16<BF16, OUT>(args.out, args.N, m0 + c0, n, mcount - c0, v);
        }
        tc_fence_before();
        mbar_arrive(bar_accempty + 8 * b);
      } else {
        // stream-K partial: slot 2p (CTA's first tile) or 2p+1 (its last tile)
        const bool is_first_tile = (u == u0);
        float* ws = args.workspace + (static_cast<size_t>(2 * p + (is_first_tile ? 0 : 1)) * NT) * 128;
#pragma unroll 1
        for (int c0 = 0; c0 < NT; c0 += 16) {
          uint32_t v[16];
          tmem_ld_32x32b_x16(tacc + c0, v);
          tc_wait_ld();
#pragma unroll
          for (int c = 0; c < 16; ++c) ws[(c0 + c) * 128 + row] = __uint_as_float(v[c]);
        }
        tc_fence_before();
        mbar_arrive(bar_accempty + 8 * b);
        __threadfence();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (et == 0) {
          const int p_lo = sk_owner(tile_lo, T, P);
          const int p_hi = sk_owner(tile_hi - 1, T, P);
          const int old = atomicAdd(args.counters + t, 1);
          const int last = (old == p_hi - p_lo) ? 1 : 0;
          if (last) args.counters[t] = 0;  // every contributor has arrived: reset for the next launch
          bcast[0] = last;
          bcast[1] = p_lo;
          bcast[2] = p_hi;
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        const int last = bcast[0], p_lo = bcast[1], p_hi = bcast[2];
        asm volatile("bar.sync 1, 128;" ::: "memory");  // bcast may be rewritten by the next segment
        if (last) {
          __threadfence();
#pragma unroll 1
          for (int c0 = 0; c0 < NT; c0 += 16) {
            float acc[16];
#pragma unroll
            for (int c = 0; c < 16; ++c) acc[c] = 0.f;
            for (int q = p_lo; q <= p_hi; ++q) {  // fixed k order: deterministic
              const long long qs = sk_start(q, T, P);
              const int slot = 2 * q + ((qs >= tile_lo) ? 0 : 1);  // t is q's first tile iff q starts inside t
              const float* wq = args.workspace + (static_cast<size_t>(slot) * NT) * 128;
#pragma unroll
              for (int c = 0; c < 16; ++c) acc[c] += __ldcg(wq + (c0 + c) * 128 + row);
            }
            uint32_t v[16];
#pragma unroll
            for (int c = 0; c < 16; ++c) v[c] = __float_as_uint(acc[c]);
            sk_store16<BF16, OUT>(args.out, args.N, m0 + c0, n, mcount - c0, v);
          }
        }
      }
      u = cend;
    }
  }

  if (threadIdx.x == 0) SK_TRACE(133);
  grid_dependency_launch();
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
}

}  // namespace w4k
