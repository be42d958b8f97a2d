// gemm_dec.cuh -- decode (M <= 64) W4A16 GEMM for sm_100a: persistent stream-K, integer-exact
// weight operand, per-group fp32 scaling of the tensor-core result.  §8(a) rows a3-a10.
//
// The method (§3.1 steps i-iv; §4.3) dequantises
// w = (q - z) * s before the MMA.  On sm_100a the decode path is bounded by the SM's issue
// pipes, not by the tensor core, so this kernel factors the group scale out of the k-sum
// (DESIGN.md §4 reading R6b):
//     C[m][n] = sum_g s[g][n] * D_g[n][m],   D_g[n][m] = sum_{k in g} (q[k][n] - z[g][n]) * A[m][k]
// (q - z) is an integer in [-15, 15], exact in bf16/fp16 (LOP3 magic + one exact HSUB2), the
// tensor core accumulates D_g in fp32 (bf16 x small-integer products are exact), and the
// scale warps apply s in fp32 (FFMA) once per group instead of once per weight.  Same
// algebra, no weight rounding (more accurate than rounding w to bf16), half the dequant work.
//
// Measured constraints this layout answers:
//   * a bulk/TMA request costs its issuing warp ~250-360 cycles: 16 KB weight chunks (one
//     cp.async.bulk of 4 LAYOUT v1 blobs), 3-D TMA activation tiles, 8-group s/z boxes, and
//     separate producer warps for weights and activations;
//   * a tcgen05.mma (M=128, N<=64, K=16) costs its issuing thread ~46-55 cycles, so two MMA
//     warps split the groups of a chunk (each group accumulates in its own TMEM D slot).
//
//   * every mbarrier handshake costs the waiting/committing thread ~100+ cycles, so the
//     TMEM operand is handed over once per 256-k chunk, the activation producer folds its
//     own TMA completion into that hand-over, and the weight ring (freed by the dequant
//     warps alone) is decoupled from the activation/TMEM ring (freed by the MMA commits).
//
// Warps (512 threads):
//   0       producer W : weight chunks (1-D bulk, before griddepcontrol.wait) + s/z boxes
//   1, 2    MMA        : issuer j takes every other chunk (all its groups); D_g -> TMEM slots
//   3       producer A : activation chunk (3-D TMA, SW128) after griddepcontrol.wait; when
//                        it lands, arrives on the chunk's "operands ready" barrier
//   4..7    dequant 0  : blobs 0,1 of every chunk; thread = weight column = TMEM lane;
//   12..15  dequant 1  : blobs 2,3.  LDS.128, LOP3 magic + exact sub, tcgen05.st
//   8..11   scale/epi  : tcgen05.ld D_g, acc[m] += s * D_g[m] (fp32 registers); at a segment
//                        end: RNE store of C, or fp32 partial + deterministic stream-K fix-up
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "dequant.cuh"
#include "ptx.cuh"

namespace w4k {

constexpr int kDecThreads = 512;

struct DecArgs {
  const uint8_t* packed;  // LAYOUT v1
  void* out;              // [M][N] bf16/fp16 or fp32
  float* workspace;       // [2 * P][NT][128] fp32 partial slots
  int* counters;          // [m_tiles * n_tiles] arrival counters (zero between launches)
  int M, N, K, group;
  int n_tiles, m_tiles;
  int kc;                 // chunks per tile = ceil(K / 256)
  long long total;        // m_tiles * n_tiles * kc
  uint32_t* trace;
};

template <int NT>
struct DecCfg {
  static constexpr int CH = 256;                         // k per chunk
  static constexpr int BLOBS = 4;                        // LAYOUT v1 blobs per chunk
  static constexpr int ACT_BYTES = NT * CH * 2;          // activation chunk (4 SW128 sub-tiles)
  static constexpr int W_BYTES = BLOBS * 4096;           // packed weight chunk
  static constexpr int STAGE_BYTES = ACT_BYTES + W_BYTES;
  static constexpr int NR = NT <= 32 ? 6 : 4;            // stage ring = per-chunk barrier ring
  static constexpr int AC = NT <= 16 ? 3 : 2;            // TMEM operand ring (chunks of 128 columns)
  static constexpr int DCOLS = NT;                       // one D_g slot
  static constexpr int DCHUNK_MAX = 4 * NT;              // D columns of one chunk (g = 64: 4 groups)
  static constexpr int DR = (512 - AC * BLOBS * 32) / DCHUNK_MAX >= 2 ? 2 : 1;  // D ring (chunks)
  static constexpr int SZG = 8;
  static constexpr int SZ_BOX = SZG * 128 * 2;
  static constexpr int SZ_SLOTS = 2;
  static constexpr int TMEM_COLS = 512;
  static constexpr int HDR = 1024;
  static constexpr int SMEM = 1024 + HDR + NR * STAGE_BYTES + SZ_SLOTS * 2 * SZ_BOX;
  static_assert(AC * BLOBS * 32 + DR * DCHUNK_MAX <= TMEM_COLS, "TMEM");
  static_assert(NR >= AC, "barrier ring must cover the TMEM ring");
  static_assert(SMEM <= 227 * 1024, "shared memory");
};

__device__ __forceinline__ int dec_owner(long long u, long long T, int P) {
  return static_cast<int>(((u + 1) * P - 1) / T);
}
__device__ __forceinline__ long long dec_start(int p, long long T, int P) {
  return (static_cast<long long>(p) * T) / P;
}

// operand for the integer-exact MMA: x - (MAGIC + z) for the 4 pairs of one LAYOUT v1 word
template <bool BF16>
__device__ __forceinline__ void deq_word_int(uint32_t w, uint32_t z2, uint32_t* out) {
  constexpr uint32_t MAGIC = BF16 ? 0x43004300u : 0x64006400u;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    // w >> 4i: i = 1, 2 on the ALU pipe (SHF), i = 3 as IMAD.HI (w * 2^20) >> 32 on the FMA pipe,
    // which balances the two pipes (6 ALU + 5 FMA-pipe ops per word)
    uint32_t ws = w;
    if (i == 1) ws = w >> 4;
    if (i == 2) ws = w >> 8;
    if (i == 3) asm("mul.hi.u32 %0, %1, %2;" : "=r"(ws) : "r"(w), "r"(1u << 20));
    uint32_t x;
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(x) : "r"(ws), "r"(0x000F000Fu), "r"(MAGIC));
    uint32_t d;
    if constexpr (BF16)
      asm("sub.rn.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(x), "r"(z2));
    else
      asm("sub.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(x), "r"(z2));
    out[i] = d;
  }
}

template <bool BF16>
__device__ __forceinline__ uint32_t zero_operand(uint16_t z_bits) {
  const float zf = __half2float(__ushort_as_half(z_bits));
  const uint16_t zb = BF16 ? __bfloat16_as_ushort(__float2bfloat16_rn(128.0f + zf))
                           : __half_as_ushort(__float2half_rn(1024.0f + zf));
  return static_cast<uint32_t>(zb) | (static_cast<uint32_t>(zb) << 16);
}

template <bool BF16, int OUT>
__device__ __forceinline__ void dec_store(void* out, int N, int m, int n, float x) {
  const size_t idx = static_cast<size_t>(m) * N + n;
  if constexpr (OUT == 1) {
    reinterpret_cast<float*>(out)[idx] = x;
  } else if constexpr (BF16) {
    reinterpret_cast<__nv_bfloat16*>(out)[idx] = __float2bfloat16_rn(x);
  } else {
    reinterpret_cast<__half*>(out)[idx] = __float2half_rn(x);
  }
}

#define DEC_TRACE(slot)                                                                               \
  do {                                                                                                \
    if (args.trace) args.trace[blockIdx.x * 160 + (slot)] = static_cast<uint32_t>(clock64() - t_start); \
  } while (0)

// Iterate the CTA's segments: a segment is the part of one (m-tile, n-tile) inside [u0, u1).
#define DEC_FOR_SEGMENTS                                                                            \
  for (long long u = u0, cend = 0; u < u1; u = cend)                                                \
    if (const int t = static_cast<int>(u / kc); true)                                              \
      if ((cend = ((static_cast<long long>(t) + 1) * kc < u1 ? (static_cast<long long>(t) + 1) * kc : u1)), true)

template <int NT, bool BF16, int OUT>
__global__ void __launch_bounds__(kDecThreads, 1)
    w4a16_dec_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_s,
                     const __grid_constant__ CUtensorMap tmap_z, const DecArgs args) {
  using Cfg = DecCfg<NT>;
  constexpr int NR = Cfg::NR;  // stages and per-chunk full/ready/done barriers
  constexpr int AC = Cfg::AC;
  constexpr int DR = Cfg::DR;

  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* const base_ptr = smem_raw + (base - smem_u32(smem_raw));
  const uint32_t bar_full = base;                               // NR (W + A producers, tx)
  const uint32_t bar_ready = bar_full + 8 * NR;                 // NR (128: the chunk's dequant set)
  const uint32_t bar_done = bar_ready + 8 * NR;                 // NR (1 commit of the chunk's MMA issuer)
  const uint32_t bar_dfree = bar_done + 8 * NR;                 // DR (128 scale: D slots of a chunk read)
  const uint32_t bar_szfull = bar_dfree + 8 * DR;               // SZ_SLOTS (1)
  const uint32_t bar_szempty = bar_szfull + 8 * Cfg::SZ_SLOTS;  // SZ_SLOTS (256 dequant + 128 scale)
  const uint32_t tmem_slot = bar_szempty + 8 * Cfg::SZ_SLOTS;
  uint32_t* const tmem_slot_ptr = reinterpret_cast<uint32_t*>(base_ptr + (tmem_slot - base));
  int* const bcast = reinterpret_cast<int*>(base_ptr + (tmem_slot - base) + 16);
  const uint32_t st0 = base + Cfg::HDR;                         // NR x [act | packed weights]
  const uint32_t sz0 = st0 + NR * Cfg::STAGE_BYTES;             // SZ_SLOTS x [s box | z box]
  const uint8_t* const st_ptr0 = base_ptr + Cfg::HDR;
  const uint8_t* const sz_ptr0 = st_ptr0 + NR * Cfg::STAGE_BYTES;

  const int warp = threadIdx.x >> 5;
  const uint32_t lane = threadIdx.x & 31;
  const long long t_start = clock64();

  const int P = gridDim.x;
  const int p = blockIdx.x;
  const long long T = args.total;
  const long long u0 = dec_start(p, T, P);
  const long long u1 = dec_start(p + 1, T, P);
  const int KS = args.K / 64;
  const int kc = args.kc;
  const int gshift = args.group == 64 ? 6 : 7;
  const int bpg = args.group >> 6;  // blobs per group (1 or 2)
  const int chunks_per_box = (Cfg::SZG << gshift) / Cfg::CH;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmap_a);
    prefetch_tmap(&tmap_s);
    prefetch_tmap(&tmap_z);
    for (int r = 0; r < NR; ++r) {
      mbar_init(bar_full + 8 * r, 2);
      mbar_init(bar_ready + 8 * r, 128);
      mbar_init(bar_done + 8 * r, 1);
    }
    for (int d = 0; d < DR; ++d) mbar_init(bar_dfree + 8 * d, 128);
    for (int j = 0; j < Cfg::SZ_SLOTS; ++j) {
      mbar_init(bar_szfull + 8 * j, 1);
      mbar_init(bar_szempty + 8 * j, 256 + 128);
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
  const uint32_t tmem_a0 = tmem_base;                         // AC x 4 blobs x 32 columns
  const uint32_t tmem_d0 = tmem_base + AC * Cfg::BLOBS * 32;  // DR x (groups of a chunk) x NT columns

  if (warp == 0) {
    // ---------------------------------------------------------------- producer W (+ s/z)
    const uint64_t pol = policy_evict_first();
    int i = 0, box = 0;
    DEC_FOR_SEGMENTS {
      const int nt = t % args.n_tiles;
      const int c0 = static_cast<int>(u - static_cast<long long>(t) * kc);
      const int c1 = static_cast<int>(cend - static_cast<long long>(t) * kc);
      for (int c = c0; c < c1; ++c, ++i) {
        if ((c - c0) % chunks_per_box == 0) {
          const int j = box % Cfg::SZ_SLOTS;
          mbar_wait(bar_szempty + 8 * j, ((box / Cfg::SZ_SLOTS) & 1) ^ 1);
          const uint32_t fb = bar_szfull + 8 * j;
          const int g0 = (c * Cfg::CH) >> gshift;
          if (elect_one()) {
            mbar_arrive_expect_tx(fb, 2 * Cfg::SZ_BOX);
            tma_load_2d(sz0 + j * 2 * Cfg::SZ_BOX, &tmap_s, nt * 128, g0, fb);
            tma_load_2d(sz0 + j * 2 * Cfg::SZ_BOX + Cfg::SZ_BOX, &tmap_z, nt * 128, g0, fb);
          }
          __syncwarp();
          ++box;
        }
        const int r = i % NR;
        if (i >= NR) mbar_wait(bar_done + 8 * r, ((i - NR) / NR) & 1);  // chunk i - NR fully consumed
        const int kb0 = c * Cfg::BLOBS;
        const int nb = (KS - kb0) < Cfg::BLOBS ? (KS - kb0) : Cfg::BLOBS;
        const uint32_t fb = bar_full + 8 * r;
        if (elect_one()) {
          mbar_arrive_expect_tx(fb, nb * 4096);
          bulk_g2s_hint(st0 + r * Cfg::STAGE_BYTES + Cfg::ACT_BYTES,
                        args.packed + (static_cast<size_t>(nt) * KS + kb0) * 4096, nb * 4096, fb, pol);
        }
        __syncwarp();
        if (lane == 0 && i < 32) DEC_TRACE(3 + i);
      }
    }
  } else if (warp == 3) {
    // ---------------------------------------------------------------- producer A
    grid_dependency_wait();  // activations may come from the previous kernel
    int i = 0;
    DEC_FOR_SEGMENTS {
      const int mt = t / args.n_tiles;
      const int c0 = static_cast<int>(u - static_cast<long long>(t) * kc);
      const int c1 = static_cast<int>(cend - static_cast<long long>(t) * kc);
      for (int c = c0; c < c1; ++c, ++i) {
        const int r = i % NR;
        if (i >= NR) mbar_wait(bar_done + 8 * r, ((i - NR) / NR) & 1);
        const uint32_t fb = bar_full + 8 * r;
        if (elect_one()) {
          mbar_arrive_expect_tx(fb, Cfg::ACT_BYTES);
          tma_load_3d(st0 + r * Cfg::STAGE_BYTES, &tmap_a, 0, mt * NT, c * Cfg::BLOBS, fb);
        }
        __syncwarp();
      }
    }
  } else if (warp == 1 || warp == 2) {
    // ---------------------------------------------------------------- MMA issuers
    // whole warp runs the loop (warp-uniform operands); one elected lane issues.  Per chunk:
    // wait ready, wait D ring slot, MMAs of my groups, one commit on done.
    const int me = warp - 1;
    constexpr int NISSUE = DR >= 2 ? 2 : 1;
    constexpr uint32_t idesc = umma_idesc_f16(BF16, 128, NT);
    int i = 0;
    DEC_FOR_SEGMENTS {
      const int c0 = static_cast<int>(u - static_cast<long long>(t) * kc);
      const int c1 = static_cast<int>(cend - static_cast<long long>(t) * kc);
      for (int c = c0; c < c1; ++c, ++i) {
        // issuer j takes chunks i with i % NISSUE == j (all groups); two alternating issuers need
        // two D ring entries, otherwise a fast issuer could alias a dfree phase
        if (i % NISSUE != me) continue;
        const int r = i % NR;
        const int ac = i % AC;
        const int dr = i % DR;
        const int kb0 = c * Cfg::BLOBS;
        const int nb = (KS - kb0) < Cfg::BLOBS ? (KS - kb0) : Cfg::BLOBS;
        const int ng = nb / bpg;
        const uint32_t act = st0 + r * Cfg::STAGE_BYTES;
        const long long q0 = clock64();
        mbar_wait(bar_ready + 8 * r, (i / NR) & 1);        // operands in TMEM, activations in SMEM
        const long long q1 = clock64();
        mbar_wait(bar_dfree + 8 * dr, ((i / DR) & 1) ^ 1);  // D slots of this ring entry read
        tc_fence_after();
        const long long q2 = clock64();
        long long q3 = q2;
        if (elect_one()) {
          for (int g = 0; g < ng; ++g) {
            const uint32_t d_tmem = tmem_d0 + (dr * 4 + g) * Cfg::DCOLS;
            for (int bb = 0; bb < bpg; ++bb) {
              const int blob = g * bpg + bb;
              const uint32_t a_tmem = tmem_a0 + (ac * Cfg::BLOBS + blob) * 32;
              const uint64_t bdesc0 = umma_desc_sw128(act + blob * (NT * 128));
#pragma unroll
              for (int j = 0; j < 4; ++j)
                mma_ts(d_tmem, a_tmem + 8 * j, bdesc0 + 2 * j, idesc, (bb | j) != 0 ? 1u : 0u);
            }
          }
          q3 = clock64();
          tc_commit(bar_done + 8 * r);
        }
        __syncwarp();
        if (args.trace && me == 0 && lane == 0) {  // per-role cycle accounting (debug)
          uint32_t* tr = args.trace + blockIdx.x * 160;
          tr[136] += static_cast<uint32_t>(q1 - q0);
          tr[137] += static_cast<uint32_t>(q2 - q1);
          tr[138] += static_cast<uint32_t>(q3 - q2);
          tr[139] += static_cast<uint32_t>(clock64() - q3);
          tr[140] += 1;
        }
        if (me == 0 && lane == 0 && i < 32) DEC_TRACE(99 + i);
      }
    }
  } else if ((warp >= 4 && warp <= 7) || warp >= 12) {
    // ---------------------------------------------------------------- dequant (2 sets)
    // set j takes whole chunks i with i % 2 == j, so one set's waits overlap the other's work
    const int set = warp >= 12 ? 1 : 0;
    const int quarter = warp & 3;
    const int row = quarter * 32 + static_cast<int>(lane);
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    int i = 0, box = -1;
    DEC_FOR_SEGMENTS {
      const int c0 = static_cast<int>(u - static_cast<long long>(t) * kc);
      const int c1 = static_cast<int>(cend - static_cast<long long>(t) * kc);
      int g_base = 0;
      for (int c = c0; c < c1; ++c, ++i) {
        if ((c - c0) % chunks_per_box == 0) {
          if (box >= 0) mbar_arrive(bar_szempty + 8 * (box % Cfg::SZ_SLOTS));
          ++box;
          mbar_wait(bar_szfull + 8 * (box % Cfg::SZ_SLOTS), (box / Cfg::SZ_SLOTS) & 1);
          g_base = (c * Cfg::CH) >> gshift;
        }
        if ((i & 1) != set) continue;
        const uint8_t* zs = sz_ptr0 + (box % Cfg::SZ_SLOTS) * 2 * Cfg::SZ_BOX + Cfg::SZ_BOX;
        const int r = i % NR;
        const int ac = i % AC;
        const int kb0 = c * Cfg::BLOBS;
        const int nb = (KS - kb0) < Cfg::BLOBS ? (KS - kb0) : Cfg::BLOBS;
        const long long q0 = clock64();
        mbar_wait(bar_full + 8 * r, (i / NR) & 1);  // weights and activations of the chunk landed
        const long long q1 = clock64();
        if (i < 32 && warp == 4 && lane == 0) DEC_TRACE(35 + i);
        const uint8_t* wst = st_ptr0 + r * Cfg::STAGE_BYTES + Cfg::ACT_BYTES + row * 16;
        // codes of blob 0 now; each later blob is loaded one step ahead of its use, so only
        // two 16-byte vectors are live and the two 32-register operand buffers get their own
        // ranges (tcgen05.st reads its source registers asynchronously)
        uint4 wa = *reinterpret_cast<const uint4*>(wst);
        uint4 wb = *reinterpret_cast<const uint4*>(wst + 2048);
        const long long q2 = clock64();
        if (i >= AC) mbar_wait(bar_done + 8 * ((i - AC) % NR), ((i - AC) / NR) & 1);  // TMEM slot free
        tc_fence_after();
        const long long q3 = clock64();
        uint32_t ra[32], rb[32];
        long long qa = q3, qb = q3;
#pragma unroll
        for (int bb = 0; bb < 4; ++bb) {
          if (bb < nb) {
            uint32_t(&rr)[32] = (bb & 1) ? rb : ra;
            if (bb == 2) {
              qa = clock64();
              tc_wait_st();  // ra is rewritten: its tcgen05.st must have completed
              qb = clock64();
            }
            const uint4 xa = wa, xb = wb;
            if (bb + 1 < nb) {
              wa = *reinterpret_cast<const uint4*>(wst + (bb + 1) * 4096);
              wb = *reinterpret_cast<const uint4*>(wst + (bb + 1) * 4096 + 2048);
            }
            const int gi = (((kb0 + bb) * 64) >> gshift) - g_base;
            const uint32_t z2 = zero_operand<BF16>(*reinterpret_cast<const uint16_t*>(zs + gi * 256 + row * 2));
            deq_word_int<BF16>(xa.x, z2, rr + 0);
            deq_word_int<BF16>(xa.y, z2, rr + 4);
            deq_word_int<BF16>(xa.z, z2, rr + 8);
            deq_word_int<BF16>(xa.w, z2, rr + 12);
            deq_word_int<BF16>(xb.x, z2, rr + 16);
            deq_word_int<BF16>(xb.y, z2, rr + 20);
            deq_word_int<BF16>(xb.z, z2, rr + 24);
            deq_word_int<BF16>(xb.w, z2, rr + 28);
            tmem_st_32x32b_x32(tmem_a0 + (ac * Cfg::BLOBS + bb) * 32 + lane_off, rr);
            if (bb >= 1) keep_alive_32((bb & 1) ? ra : rb);  // previous buffer: live until here
          }
        }
        const long long qc = clock64();
        tc_wait_st();
        tc_fence_before();
        const long long q4 = clock64();
        mbar_arrive(bar_ready + 8 * r);
        if (args.trace && warp == 4 && lane == 0) {
          uint32_t* tr = args.trace + blockIdx.x * 160;
          tr[143] += static_cast<uint32_t>(q1 - q0);  // wait stage
          tr[144] += static_cast<uint32_t>(q2 - q1);  // LDS
          tr[145] += static_cast<uint32_t>(q3 - q2);  // wait TMEM slot
          tr[146] += static_cast<uint32_t>(q4 - q3);  // dequant + st
          tr[147] += static_cast<uint32_t>(clock64() - q4);
          tr[148] += static_cast<uint32_t>((qa - q3) + (qc - qb));  // dequant math + st issue
          tr[149] += static_cast<uint32_t>((qb - qa) + (q4 - qc));  // tcgen05.wait::st
        }
        if (i < 32 && warp == 4 && lane == 0) DEC_TRACE(67 + i);
      }
    }
    if (box >= 0) mbar_arrive(bar_szempty + 8 * (box % Cfg::SZ_SLOTS));
  } else {
    // ---------------------------------------------------------------- scale + epilogue
    const int quarter = warp & 3;
    const int row = quarter * 32 + static_cast<int>(lane);
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    const int et = threadIdx.x - 8 * 32;  // 0..127
    int ci = 0, box = -1;
    DEC_FOR_SEGMENTS {
      const int nt = t % args.n_tiles;
      const int mt = t / args.n_tiles;
      const int c0 = static_cast<int>(u - static_cast<long long>(t) * kc);
      const int c1 = static_cast<int>(cend - static_cast<long long>(t) * kc);
      float acc[NT];
#pragma unroll
      for (int m = 0; m < NT; ++m) acc[m] = 0.f;
      int g_base = 0;
      for (int c = c0; c < c1; ++c) {
        if ((c - c0) % chunks_per_box == 0) {
          if (box >= 0) mbar_arrive(bar_szempty + 8 * (box % Cfg::SZ_SLOTS));
          ++box;
          mbar_wait(bar_szfull + 8 * (box % Cfg::SZ_SLOTS), (box / Cfg::SZ_SLOTS) & 1);
          g_base = (c * Cfg::CH) >> gshift;
        }
        const uint8_t* ss = sz_ptr0 + (box % Cfg::SZ_SLOTS) * 2 * Cfg::SZ_BOX;
        const int kb0 = c * Cfg::BLOBS;
        const int nb = (KS - kb0) < Cfg::BLOBS ? (KS - kb0) : Cfg::BLOBS;
        const int ng = nb / bpg;
        const int r = ci % NR;
        const int dr = ci % DR;
        const long long q0 = clock64();
        mbar_wait(bar_done + 8 * r, (ci / NR) & 1);
        tc_fence_after();
        const long long q1 = clock64();
        for (int g = 0; g < ng; ++g) {
          const int gi = ((kb0 * 64) >> gshift) + g - g_base;
          const float sc = __half2float(__ushort_as_half(*reinterpret_cast<const uint16_t*>(ss + gi * 256 + row * 2)));
#pragma unroll
          for (int m0 = 0; m0 < NT; m0 += 16) {
            uint32_t v[16];
            tmem_ld_32x32b_x16(tmem_d0 + (dr * 4 + g) * Cfg::DCOLS + lane_off + m0, v);
            tc_wait_ld();
#pragma unroll
            for (int m = 0; m < 16; ++m) acc[m0 + m] = fmaf(sc, __uint_as_float(v[m]), acc[m0 + m]);
          }
        }
        tc_fence_before();
        mbar_arrive(bar_dfree + 8 * dr);
        if (args.trace && et == 0) {
          uint32_t* tr = args.trace + blockIdx.x * 160;
          tr[141] += static_cast<uint32_t>(q1 - q0);
          tr[142] += static_cast<uint32_t>(clock64() - q1);
        }
        ++ci;
      }
      // ---- segment end: store (whole tile) or stream-K partial + fix-up
      const long long tile_lo = static_cast<long long>(t) * kc;
      const long long tile_hi = tile_lo + kc;
      const bool full = (u == tile_lo) && (cend == tile_hi);
      const int n = nt * 128 + row;
      const int mb = mt * NT;
      const int mcount = (args.M - mb) < NT ? (args.M - mb) : NT;
      if (full) {
#pragma unroll
        for (int m = 0; m < NT; ++m)
          if (m < mcount) dec_store<BF16, OUT>(args.out, args.N, mb + m, n, acc[m]);
      } else {
        const bool is_first_tile = (u == u0);
        float* ws = args.workspace + (static_cast<size_t>(2 * p + (is_first_tile ? 0 : 1)) * NT) * 128;
#pragma unroll
        for (int m = 0; m < NT; ++m) ws[m * 128 + row] = acc[m];
        __threadfence();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (et == 0) {
          const int p_lo = dec_owner(tile_lo, T, P);
          const int p_hi = dec_owner(tile_hi - 1, T, P);
          const int old = atomicAdd(args.counters + t, 1);
          const int last = (old == p_hi - p_lo) ? 1 : 0;
          if (last) args.counters[t] = 0;  // all contributors arrived: ready for the next launch
          bcast[0] = last;
          bcast[1] = p_lo;
          bcast[2] = p_hi;
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        const int last = bcast[0], p_lo = bcast[1], p_hi = bcast[2];
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (last) {
          __threadfence();
#pragma unroll
          for (int m = 0; m < NT; ++m) acc[m] = 0.f;
          for (int q = p_lo; q <= p_hi; ++q) {  // fixed k order: deterministic
            const long long qs = dec_start(q, T, P);
            const int slot = 2 * q + ((qs >= tile_lo) ? 0 : 1);
            const float* wq = args.workspace + (static_cast<size_t>(slot) * NT) * 128;
#pragma unroll
            for (int m = 0; m < NT; ++m) acc[m] += __ldcg(wq + m * 128 + row);
          }
#pragma unroll
          for (int m = 0; m < NT; ++m)
            if (m < mcount) dec_store<BF16, OUT>(args.out, args.N, mb + m, n, acc[m]);
        }
      }
    }
    if (box >= 0) mbar_arrive(bar_szempty + 8 * (box % Cfg::SZ_SLOTS));
  }

  if (threadIdx.x == 0) DEC_TRACE(133);
  grid_dependency_launch();
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
}

#undef DEC_FOR_SEGMENTS

}  // namespace w4k
