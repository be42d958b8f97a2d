// gemm_rf.cuh -- decode (M <= 16) W4A16 GEMM for sm_100a with a register-fed tensor path.
// §8(a) rows a3-a10 for the decode band; the kernel the bench's decode mix runs.
//
// Why not tcgen05 at M <= 16: the GEMM is HBM-bound, a tcgen05.mma reads its
// weight operand from TMEM or shared memory, so the dequantised weights (2 B each, 4x the packed
// bytes) must be staged there and handed between warp roles through mbarriers; the round-1 TMEM
// kernel was bound by exactly that staging and hand-over chain.  Here the operand never leaves
// the registers of the thread that produced it (§3.1 steps i-iv, and the
// register-resident pipeline of §4.3): packed codes stream HBM -> shared memory
// (cp.async.bulk, mbarrier ring), each consumer warp turns them into warp-level MMA fragments
// (ldmatrix + LOP3 magic I2F) and feeds mma.sync m16n8k16 with fp32 accumulators in
// registers.  Measured (scripts/microbench_hmma.cu): the legacy HMMA pipe runs 0.5 m16n8k16 per
// clock per SM; the I2F + HMMA inner loop sustains 58 weights/clk/SM at 8 tokens and 46 at 16
// (7.7 / 6.3 TB/s of packed codes) -- at or above HBM.
//
// Algebra (reading R6c): the operand is the exact magic value V + q (V = 128 for
// bf16, 1024 for fp16: one LOP3 per pair, no subtraction), so per group g and token m
//     D'_g[n][m] = sum_{k in g} (V + q[k][n]) A[m][k] = D_g[n][m] + (V + z_g[n]) R_g[m],
//     R_g[m] = sum_{k in g} A[m][k]  (on the tensor core: an all-ones A fragment x the same B)
//     C[m][n] = sum_g s_g[n] D'_g[n][m] - s_g[n] (V + z_g[n]) R_g[m]           (fp32 FFMAs)
// Products (V + q) A are exact in fp32; the group sums are fp32 (the MMA's accumulation), then
// one output rounding (RNE).
//
// Fragment mapping onto LAYOUT v1 (no re-pack).  MMA rows = 16 weight columns n
// of a row group rg (row r <-> column 16 rg + r), k16 slices in a permuted k order (the MMA is
// indifferent to the order of k as long as A and B agree):
//   * ldmatrix.x4 on a blob viewed as 16-bit elements: matrix (half j, rows 8h..8h+7) is 8 rows
//     x 16 B, lane (g, c) receives bytes 4c..4c+3 of row g = the word wj = c of that column and
//     half (k = 32 j + 8 c .. +7); conflict-free (128 contiguous bytes per matrix);
//   * pairs 2h, 2h+1 of that word are the A fragment's k-slots (2c, 2c+1) and (2c+8, 2c+9) of
//     fragment (j, h): k = 32 j + 8 c + 4 h + {0,1} and + {2,3};
//   * B fragment of lane (g', c): A[token][32 j + 8 c + 4 h .. +3] -- one LDS.128 per (j, token
//     octet) from the SW128 activation tile, token sigma(g') = (g' >> 1) | ((g' & 1) << 2)
//     so the 8 lanes of a quarter-warp hit 8 distinct 16-B chunks; D column 2c <-> token c,
//     2c + 1 <-> token c + 4.
//
// Work split: CTA = (128-column tile, contiguous range of 256-k chunks), `split` CTAs per tile.
// A unit is one quantisation group (g = 128: 2 blobs, g = 64: 1 blob); the CTA's units are dealt
// round-robin to its 4 consumer warps, each accumulating its own partial for all 128 columns; at
// the end the 4 partials are added in warp order in shared memory and, with split > 1, the
// tile's CTAs add theirs through a global workspace in CTA order (the last CTA to arrive on the
// tile's counter does it): deterministic.
//
// Warps: 0 = weight producer (1-D bulk, before griddepcontrol.wait -- weights are layer
// constants), 1 = activation producer (3-D TMA after griddepcontrol.wait), 2 = s/z producer
// (2-D TMA boxes of the chunk's groups, before the wait), 3..6 = consumers.  Small footprint
// (224 threads, ~110 KB shared memory, no TMEM): two CTAs per SM, and under PDL the next
// launch's CTAs start on an SM while this launch's CTAs finish there.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "ptx.cuh"

namespace w4k {

#ifndef TM_RF_NW
#define TM_RF_NW 4
#endif
#ifndef TM_RF_NA
#define TM_RF_NA 4
#endif
#ifndef TM_RF_SPIN
#define TM_RF_SPIN 0  // 1: spin on try_wait (no suspend hint) in every role
#endif
#ifndef TM_RF_CHAIN
#define TM_RF_CHAIN 0  // 1: consumers keep one accumulator chain per (row group, k half)
#endif
#ifndef TM_RF_DIAG
#define TM_RF_DIAG 0  // timing experiments only (wrong results): 1 consumers skip the math, 2 no R step
#endif

struct RfArgs {
  const uint8_t* packed;  // LAYOUT v1
  void* out;              // [M][N] bf16/fp16 or fp32
  float* partials;        // stream-K: [grid][NT][128] words ~bits(fp32 partial) of each CTA's first
                          // segment; 0 = not written (zero between launches)
  int M, N, K;
  int kc;                 // 256-k chunks per tile
  uint32_t total;         // tiles x kc
  int split;              // 0: stream-K; S >= 1: S CTAs per tile (a cluster when S > 1)
  int a_ks;               // 64-k blobs of A: K / 64, or K / 128 for W8 bit planes (A reused)
  uint32_t* trace;        // debug timeline (tm_set_trace; nullptr in production): [cta][64] ns
};

// debug timeline: %globaltimer (ns, low 32 bits) of event `slot` of this CTA
__device__ __forceinline__ void rf_mark(uint32_t* trace, int slot) {
  if (trace) {
    uint64_t gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    trace[blockIdx.x * 64 + slot] = static_cast<uint32_t>(gt);
  }
}

template <int NT, int GROUP>
struct RfCfg {
  static constexpr int NOCT = NT / 8;                 // token octets (B fragments per k16)
  static constexpr int U = 256 / GROUP;               // units (groups) per chunk
  static constexpr int BPG = GROUP / 64;              // LAYOUT v1 blobs per unit
  static constexpr int W_BYTES = 16384;               // packed weight chunk: 4 blobs
  static constexpr int A_BYTES = NT * 512;            // activation chunk: 4 SW128 [NT][64] tiles
  static constexpr int SZ_BYTES = U * 128 * 2;        // s (or z) rows of the chunk's groups
  static constexpr int R_BYTES = U * NT * 4;          // activation sums R_g[m] of the chunk
  static constexpr int AS_BYTES = (A_BYTES + 2 * SZ_BYTES + R_BYTES + 1023) / 1024 * 1024;  // act | s | z | R
  static constexpr int NW = TM_RF_NW;                 // weight ring
  static constexpr int NA = TM_RF_NA;                 // activation stage ring
  static constexpr int NCW = 4;                       // consumer warps
  static constexpr int THREADS = 32 * (3 + NCW);
  static constexpr int HDR = 1024;
  static constexpr int OFF_W = HDR;
  static constexpr int OFF_A = OFF_W + NW * W_BYTES;
  static constexpr int SMEM = 1024 + OFF_A + NA * AS_BYTES;  // + alignment slack
  static constexpr int MAX_SPLIT = 8;                 // portable cluster size
  static_assert(A_BYTES % 1024 == 0, "SW128 tiles need 1024-B alignment");
  static_assert(MAX_SPLIT * NT * 64 * 4 <= NW * W_BYTES, "cluster landing area (the idle weight ring)");
  static_assert(NCW == 4, "a consumer warp owns 32 columns of the 128-column tile");
  static constexpr int MINB = SMEM <= 113 * 1024 ? 2 : 1;  // CTAs per SM
  static_assert(3 * (NW + NA) * 8 <= HDR, "barrier header");
};

template <bool BF16>
__device__ __forceinline__ void rf_hmma(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  if constexpr (BF16)
    asm(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  else
    asm(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// I2F of one LAYOUT v1 word: p[i] = (V + e_{2i}, V + e_{2i+1}) as an exact bf16/fp16 pair
// (one SHF + one LOP3 per pair; LUT 0xEA = (a & b) | c)
#ifndef TM_RF_MULHI
#define TM_RF_MULHI 0  // number of the 3 nibble shifts done as mul.hi on the FMA pipe (ALU relief)
#endif
template <bool BF16>
__device__ __forceinline__ void rf_magic(uint32_t w, uint32_t (&p)[4]) {
  constexpr uint32_t MAGIC = BF16 ? 0x43004300u : 0x64006400u;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    uint32_t x = w >> (4 * i);
    if (i > 0 && i <= TM_RF_MULHI) asm("mul.hi.u32 %0, %1, %2;" : "=r"(x) : "r"(w), "r"(1u << (32 - 4 * i)));
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(p[i]) : "r"(x), "r"(0x000F000Fu), "r"(MAGIC));
  }
}

__device__ __forceinline__ void rf_ldmatrix_x4(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr)
               : "memory");
}

__device__ __forceinline__ uint4 rf_lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ float rf_lds_h2f(uint32_t addr) {
  unsigned short h;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(h) : "r"(addr) : "memory");
  return __half2float(__ushort_as_half(h));
}
__device__ __forceinline__ void rf_wait(uint32_t bar, uint32_t parity) {
  if (TM_RF_SPIN) {
    while (!mbar_try_wait(bar, parity)) {
    }
  } else {
    mbar_wait(bar, parity);
  }
}
__device__ __forceinline__ void rf_named_bar(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

template <bool BF16, int OUT>
__device__ __forceinline__ void rf_store(void* out, size_t idx, float v) {
  if constexpr (OUT == 1)
    reinterpret_cast<float*>(out)[idx] = v;
  else if constexpr (BF16)
    reinterpret_cast<__nv_bfloat16*>(out)[idx] = __float2bfloat16_rn(v);
  else
    reinterpret_cast<__half*>(out)[idx] = __float2half_rn(v);
}

// One 256-k chunk for consumer warp cw (columns 32 cw .. 32 cw + 31 of the tile): B fragments
// from the activation stage, weight fragments by ldmatrix from the weight stage, I2F magic,
// mma.sync per group, then acc += s D' - s (V + z) R in fp32 (reading R6c).  nbv = valid blobs.
template <int NT, int GROUP, bool BF16>
__device__ __forceinline__ void rf_chunk(float (&acc)[2][NT / 8][4], uint32_t ast, uint32_t wst, const float* R,
                                         int nbv, int cw, int lane) {
  using Cfg = RfCfg<NT, GROUP>;
  constexpr int NOCT = Cfg::NOCT, U = Cfg::U, BPG = Cfg::BPG;
  constexpr float V = BF16 ? 128.0f : 1024.0f;
  const int g = lane >> 2, c = lane & 3;
  const int sig = (g >> 1) | ((g & 1) << 2);
  const uint32_t lm_off =
      static_cast<uint32_t>((lane >> 4) * 2048 + (((lane >> 3) & 1) * 8 + (lane & 7)) * 16 + cw * 2 * 256);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (u * BPG < nbv) {
        constexpr int NCH = TM_RF_CHAIN ? 2 : 1;  // accumulator chains per row group
        float dd[NCH][2][NOCT][4];
#pragma unroll
        for (int q = 0; q < NCH; ++q)
#pragma unroll
          for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int o = 0; o < NOCT; ++o)
#pragma unroll
              for (int e = 0; e < 4; ++e) dd[q][r][o][e] = 0.f;
#pragma unroll
        for (int bb = 0; bb < BPG; ++bb) {
          const int blob = u * BPG + bb;
          uint4 bfr[2][NOCT];
#pragma unroll
          for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int o = 0; o < NOCT; ++o) {
              const int row = sig + 8 * o;
              bfr[j][o] = rf_lds128(ast + blob * (NT * 128) + row * 128 + (((4 * j + c) ^ (row & 7)) << 4));
            }
          uint32_t wv[2][4];
#pragma unroll
          for (int r = 0; r < 2; ++r)
            rf_ldmatrix_x4(wst + blob * 4096 + lm_off + r * 256, wv[r]);
#pragma unroll
          for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int r = 0; r < 2; ++r) {
              uint32_t p0[4], p1[4];
              rf_magic<BF16>(wv[r][2 * j], p0);      // column 16 rg + g
              rf_magic<BF16>(wv[r][2 * j + 1], p1);  // column 16 rg + g + 8
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const uint32_t a[4] = {p0[2 * h], p1[2 * h], p0[2 * h + 1], p1[2 * h + 1]};
#pragma unroll
                for (int o = 0; o < NOCT; ++o)
                  rf_hmma<BF16>(dd[j % NCH][r][o], a, h ? bfr[j][o].z : bfr[j][o].x, h ? bfr[j][o].w : bfr[j][o].y);
              }
            }
        }
        float d[2][NOCT][4];
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
          for (int o = 0; o < NOCT; ++o)
#pragma unroll
            for (int e = 0; e < 4; ++e) d[r][o][e] = NCH == 2 ? dd[0][r][o][e] + dd[NCH - 1][r][o][e] : dd[0][r][o][e];
        // group end: C += s D' - s (V + z) R  (fp32)
        float rr[NOCT][2];
#pragma unroll
        for (int o = 0; o < NOCT; ++o) {
          const float2 tv = *reinterpret_cast<const float2*>(R + ((u * 4 + c) * NOCT + o) * 2);
          rr[o][0] = tv.x;  // token c + 8 o
          rr[o][1] = tv.y;  // token c + 4 + 8 o
        }
        const uint32_t ssm = ast + Cfg::A_BYTES + u * 256;  // fp16 s[col] of group u
        const uint32_t zsm = ssm + Cfg::SZ_BYTES;
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const uint32_t col0 = static_cast<uint32_t>(16 * (2 * cw + r) + g) * 2;
          const float s0 = rf_lds_h2f(ssm + col0), s1 = rf_lds_h2f(ssm + col0 + 16);
          const float sv0 = -s0 * (V + rf_lds_h2f(zsm + col0)), sv1 = -s1 * (V + rf_lds_h2f(zsm + col0 + 16));
#pragma unroll
          for (int o = 0; o < NOCT; ++o) {
            acc[r][o][0] = fmaf(s0, d[r][o][0], fmaf(sv0, rr[o][0], acc[r][o][0]));
            acc[r][o][1] = fmaf(s0, d[r][o][1], fmaf(sv0, rr[o][1], acc[r][o][1]));
            acc[r][o][2] = fmaf(s1, d[r][o][2], fmaf(sv1, rr[o][0], acc[r][o][2]));
            acc[r][o][3] = fmaf(s1, d[r][o][3], fmaf(sv1, rr[o][1], acc[r][o][3]));
          }
        }
      }
    }
}

// ring position of the i-th chunk of a CTA in an N-slot ring
template <int N>
struct RfSlot {
  int slot;
  uint32_t phase;
  __device__ __forceinline__ explicit RfSlot(int i) : slot(i % N), phase(static_cast<uint32_t>(i / N) & 1u) {}
};

template <int NT, int GROUP, bool BF16, int OUT>
__global__ void __launch_bounds__(RfCfg<NT, GROUP>::THREADS, RfCfg<NT, GROUP>::MINB)
    w4a16_rf_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_s,
                    const __grid_constant__ CUtensorMap tmap_z, const RfArgs args) {
  using Cfg = RfCfg<NT, GROUP>;
  constexpr int NOCT = Cfg::NOCT, U = Cfg::U, BPG = Cfg::BPG;
  constexpr int NW = Cfg::NW, NA = Cfg::NA, NCW = Cfg::NCW;
  constexpr uint32_t ONES = BF16 ? 0x3F803F80u : 0x3C003C00u;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* const base_ptr = smem_raw + (base - smem_u32(smem_raw));
  const uint32_t bar_fullw = base, bar_emptyw = base + 8 * NW;
  const uint32_t bar_fulla = base + 16 * NW, bar_emptya = bar_fulla + 8 * NA, bar_acta = bar_emptya + 8 * NA;
  const uint32_t wring = base + Cfg::OFF_W, aring = base + Cfg::OFF_A;

  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
  const int lane = static_cast<int>(threadIdx.x & 31);
  const int g = lane >> 2, c = lane & 3;
  const int sig = (g >> 1) | ((g & 1) << 2);  // token row of B column g (conflict-free LDS.128)
  // Work: chunk units u = tile * kc + chunk, tile-major.  split == 0: stream-K, CTA p takes
  // [p T / P, (p + 1) T / P) of T = tiles x kc (host: T * P < 2^32, P <= T); split = S >= 1: the S
  // CTAs of a tile (one cluster) take [r kc / S, (r + 1) kc / S) of its chunks.
  const uint32_t P = gridDim.x, p = blockIdx.x, T = args.total;
  const uint32_t kc = static_cast<uint32_t>(args.kc);
  const int S = args.split;
  uint32_t u0, u1;
  if (S > 0) {
    const uint32_t tile = p / static_cast<uint32_t>(S), r = p - tile * static_cast<uint32_t>(S);
    u0 = tile * kc + (r * kc) / static_cast<uint32_t>(S);
    u1 = tile * kc + ((r + 1) * kc) / static_cast<uint32_t>(S);
  } else {
    u0 = (p * T) / P;
    u1 = ((p + 1) * T) / P;
  }
  const int n = static_cast<int>(u1 - u0);  // >= 1 (host: P <= T, S <= kc)
  const int KS = args.K >> 6;

  if (threadIdx.x == 0) {
    rf_mark(args.trace, 0);
#pragma unroll
    for (int i = 0; i < NW; ++i) {
      mbar_init(bar_fullw + 8 * i, 1);
      mbar_init(bar_emptyw + 8 * i, NCW);  // every consumer warp reads every chunk
    }
#pragma unroll
    for (int i = 0; i < NA; ++i) {
      mbar_init(bar_fulla + 8 * i, 4 + 1);  // the 4 lanes writing R + the s/z producer's expect_tx
      mbar_init(bar_emptya + 8 * i, NCW);
      mbar_init(bar_acta + 8 * i, 1);       // activation TMA (the activation warp waits on it)
    }
    fence_mbar_init();
  }
  if (warp == 1 && lane == 0) {
    prefetch_tmap(&tmap_a);
    prefetch_tmap(&tmap_s);
    prefetch_tmap(&tmap_z);
  }
  __syncthreads();
  grid_dependency_launch();
  if (threadIdx.x == 0) rf_mark(args.trace, 1);

  float keep[2][NOCT][4];  // consumers, cluster mode: this CTA's partial until the DSMEM reduction
  if (warp == 0) {
    // ---- weight producer: 16 KB chunks (a tile's K range is contiguous in LAYOUT v1); layer
    // constants, streamed before griddepcontrol.wait (overlaps the previous kernel under PDL)
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      uint32_t t = u0 / kc, cc = u0 - t * kc;
      for (int i = 0; i < n; ++i) {
        const RfSlot<NW> st(i);
        rf_wait(bar_emptyw + 8 * st.slot, st.phase ^ 1u);
        const int kb = static_cast<int>(cc) * 4;
        const int nb = KS - kb < 4 ? KS - kb : 4;
        mbar_arrive_expect_tx(bar_fullw + 8 * st.slot, nb * 4096);
        bulk_g2s_hint(wring + st.slot * Cfg::W_BYTES,
                      args.packed + (static_cast<size_t>(t) * KS + static_cast<size_t>(kb)) * 4096, nb * 4096,
                      bar_fullw + 8 * st.slot, pol);
        if (++cc == kc) cc = 0, ++t;
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---- activation warp: one 3-D TMA (4 SW128 [NT][64] tiles) per chunk after the previous
    // kernel has completed (its output may be this GEMM's input), issued NA - 2 chunks ahead; once
    // a chunk has landed, its activation sums R_u[m] = sum_{k in group u} A[m][k] on the tensor
    // core (all-ones A fragment x the chunk's B fragments), written next to it:
    // R[u][c][o][t] = R_u[token c + 4 t + 8 o]
    grid_dependency_wait();
    if (lane == 0) rf_mark(args.trace, 2);
    int issued = 0;
    uint32_t icc = u0 % kc;
    for (int i = 0; i < n; ++i) {
      for (; issued < n && issued <= i + NA - 2; ++issued) {
        const RfSlot<NA> st(issued);
        if (lane == 0) {
          rf_wait(bar_emptya + 8 * st.slot, st.phase ^ 1u);
          int kb = static_cast<int>(icc) * 4;
          if (kb >= args.a_ks) kb -= args.a_ks;  // W8 bit planes: the low planes reuse A
          mbar_arrive_expect_tx(bar_acta + 8 * st.slot, Cfg::A_BYTES);
          tma_load_3d(aring + st.slot * Cfg::AS_BYTES, &tmap_a, 0, 0, kb, bar_acta + 8 * st.slot);
        }
        if (++icc == kc) icc = 0;
        __syncwarp();
      }
      const RfSlot<NA> st(i);
      const uint32_t ast = aring + st.slot * Cfg::AS_BYTES;
      rf_wait(bar_acta + 8 * st.slot, st.phase);
      const uint32_t ones[4] = {ONES, ONES, ONES, ONES};
      float d[U][NOCT][4];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int o = 0; o < NOCT; ++o)
#pragma unroll
          for (int e = 0; e < 4; ++e) d[u][o][e] = 0.f;
      if (!(TM_RF_DIAG & 2)) {
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
          for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int o = 0; o < NOCT; ++o) {
              const int row = sig + 8 * o;
              const uint4 bf = rf_lds128(ast + b * (NT * 128) + row * 128 + (((4 * j + c) ^ (row & 7)) << 4));
              rf_hmma<BF16>(d[b / BPG][o], ones, bf.x, bf.y);
              rf_hmma<BF16>(d[b / BPG][o], ones, bf.z, bf.w);
            }
      }
      if (g == 0) {
        float* const R = reinterpret_cast<float*>(base_ptr + Cfg::OFF_A + st.slot * Cfg::AS_BYTES + Cfg::A_BYTES +
                                                  2 * Cfg::SZ_BYTES);
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int o = 0; o < NOCT; ++o)
            *reinterpret_cast<float2*>(R + ((u * 4 + c) * NOCT + o) * 2) = make_float2(d[u][o][0], d[u][o][1]);
        mbar_arrive(bar_fulla + 8 * st.slot);
      }
      __syncwarp();
    }
  } else if (warp == 2) {
    // ---- s/z producer: the chunk's U group rows x 128 columns of s and z (layer constants)
    if (lane == 0) {
      uint32_t t = u0 / kc, cc = u0 - t * kc;
      for (int i = 0; i < n; ++i) {
        const RfSlot<NA> st(i);
        rf_wait(bar_emptya + 8 * st.slot, st.phase ^ 1u);
        const uint32_t dst = aring + st.slot * Cfg::AS_BYTES + Cfg::A_BYTES;
        mbar_arrive_expect_tx(bar_fulla + 8 * st.slot, 2 * Cfg::SZ_BYTES);
        tma_load_2d(dst, &tmap_s, static_cast<int>(t) * 128, static_cast<int>(cc) * U, bar_fulla + 8 * st.slot);
        tma_load_2d(dst + Cfg::SZ_BYTES, &tmap_z, static_cast<int>(t) * 128, static_cast<int>(cc) * U,
                    bar_fulla + 8 * st.slot);
        if (++cc == kc) cc = 0, ++t;
      }
    }
    __syncwarp();
  } else {
  // -------------------------------------------------------------- consumers
  // Warp cw owns columns 32 cw .. 32 cw + 31 of every tile (row groups 2 cw, 2 cw + 1) and reads
  // every chunk: no cross-warp reduction.  A segment = the CTA's consecutive chunks of one tile.
  const int cw = warp - 3;
  // ldmatrix row address of this lane inside a blob: half (lane >> 4), row (lane & 15) of rg 2 cw
  const uint32_t lm_off =
      static_cast<uint32_t>((lane >> 4) * 2048 + (((lane >> 3) & 1) * 8 + (lane & 7)) * 16 + cw * 2 * 256);
  const int mcount = args.M < NT ? args.M : NT;
  float acc[2][NOCT][4];
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int o = 0; o < NOCT; ++o)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[r][o][e] = 0.f;

  uint32_t t = u0 / kc, cc = u0 - t * kc;
  uint32_t seg_c0 = cc;  // first chunk of the current segment
  for (int i = 0; i < n; ++i) {
    const RfSlot<NW> sw(i);
    const RfSlot<NA> sa(i);
    rf_wait(bar_fulla + 8 * sa.slot, sa.phase);
    rf_wait(bar_fullw + 8 * sw.slot, sw.phase);
    if (!(TM_RF_DIAG & 1)) {
      const uint32_t ast = aring + sa.slot * Cfg::AS_BYTES;
      const float* const R = reinterpret_cast<const float*>(base_ptr + Cfg::OFF_A + sa.slot * Cfg::AS_BYTES +
                                                            Cfg::A_BYTES + 2 * Cfg::SZ_BYTES);
      rf_chunk<NT, GROUP, BF16>(acc, ast, wring + sw.slot * Cfg::W_BYTES, R, KS - static_cast<int>(cc) * 4, cw, lane);
    }
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(bar_emptyw + 8 * sw.slot);
      mbar_arrive(bar_emptya + 8 * sa.slot);
      if (cw == 0 && i < 48) rf_mark(args.trace, 8 + i);
    }
    // ---- segment end: the tile's last chunk or the CTA's last chunk (cluster mode with S > 1:
    // after the loop, in distributed shared memory)
    if ((cc + 1 == kc || i + 1 == n) && S <= 1) {
      const size_t colbase = static_cast<size_t>(t) * 128 + cw * 32 + g;
      if (seg_c0 == 0 && cc + 1 == kc) {
        // whole tile in this CTA: store (RNE to the output dtype, or fp32)
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
          for (int o = 0; o < NOCT; ++o)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int m = c + 4 * (e & 1) + 8 * o;
              if (m < mcount)
                rf_store<BF16, OUT>(args.out, static_cast<size_t>(m) * args.N + colbase + 16 * r + 8 * (e >> 1),
                                    acc[r][o][e]);
            }
      } else if (seg_c0 > 0) {
        // contributor: this is the CTA's first segment (its range starts inside tile t).  Its
        // fp32 partial goes to the CTA's slot as self-validating words: ~bits(x) is never 0 for
        // a finite x (0xFFFFFFFF is a NaN), so a zero word means "not written yet" -- no fence,
        // no flag, nothing stalls (a release after the stores costs ~2 us under HBM load).
        uint32_t* const part = reinterpret_cast<uint32_t*>(args.partials) + static_cast<size_t>(p) * NT * 128;
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
          for (int o = 0; o < NOCT; ++o)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int m = c + 4 * (e & 1) + 8 * o;
              st_relaxed_gpu(part + m * 128 + cw * 32 + g + 16 * r + 8 * (e >> 1), ~__float_as_uint(acc[r][o][e]));
            }
      } else {
        // owner: the segment holds the tile's first chunk and is the CTA's last segment (the
        // owner reaches tile t at the end of its range, its contributors at the start of theirs,
        // so their partials are normally written long before).  Add them in CTA order
        // (deterministic), waiting per word until it is written, re-zero the words, store.
        const uint32_t q1 = ((t + 1) * kc * P - 1) / T;  // last CTA holding part of tile t
        for (uint32_t q = p + 1; q <= q1; ++q) {
          uint32_t* const pq = reinterpret_cast<uint32_t*>(args.partials) + static_cast<size_t>(q) * NT * 128;
          uint32_t x[2][NOCT][4];  // all loads in flight at once, then the (rare) re-polls
#pragma unroll
          for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int o = 0; o < NOCT; ++o)
#pragma unroll
              for (int e = 0; e < 4; ++e)
                x[r][o][e] = ld_relaxed_gpu(pq + (c + 4 * (e & 1) + 8 * o) * 128 + cw * 32 + g + 16 * r + 8 * (e >> 1));
#pragma unroll
          for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int o = 0; o < NOCT; ++o)
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                uint32_t* const w = pq + (c + 4 * (e & 1) + 8 * o) * 128 + cw * 32 + g + 16 * r + 8 * (e >> 1);
                while (x[r][o][e] == 0u) x[r][o][e] = ld_relaxed_gpu(w);
                acc[r][o][e] += __uint_as_float(~x[r][o][e]);
                st_relaxed_gpu(w, 0u);  // ready for the next launch (ordered by its griddepcontrol.wait)
              }
        }
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
          for (int o = 0; o < NOCT; ++o)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int m = c + 4 * (e & 1) + 8 * o;
              if (m < mcount)
                rf_store<BF16, OUT>(args.out, static_cast<size_t>(m) * args.N + colbase + 16 * r + 8 * (e >> 1),
                                    acc[r][o][e]);
            }
      }
#pragma unroll
      for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int o = 0; o < NOCT; ++o)
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[r][o][e] = 0.f;
      seg_c0 = 0;
    }
    if (++cc == kc) cc = 0, ++t;
  }
  if (lane == 0 && cw == 0) rf_mark(args.trace, 3);
  if (S > 1) {  // this CTA's partial of its tile's columns, kept for the cluster reduction
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int o = 0; o < NOCT; ++o)
#pragma unroll
        for (int e = 0; e < 4; ++e) keep[r][o][e] = acc[r][o][e];
  }
  }  // consumers

  if (S > 1) {
    // ---- split-K over the tile's cluster (DSMEM): CTA r owns columns [lo(r), lo(r + 1)),
    // lo(r) = 128 r / S; every CTA pushes its partial of those columns into the owner's idle weight
    // ring (landing [src rank][m][64]), the owner adds them in rank order (deterministic) and
    // stores.  Barrier 1: every CTA of the cluster is done with its rings; barrier 2: landed.
    const uint32_t rank = cluster_ctarank();
    const uint32_t tile = p / static_cast<uint32_t>(S);
    float* const land = reinterpret_cast<float*>(base_ptr + Cfg::OFF_W);
    if (threadIdx.x == 96) rf_mark(args.trace, 5);
    cluster_arrive();
    cluster_wait();
    if (threadIdx.x == 96) rf_mark(args.trace, 6);
    if (warp >= 3) {
      const int cw = warp - 3;
#pragma unroll
      for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int eh = 0; eh < 2; ++eh) {
          const int col = cw * 32 + 16 * r + g + 8 * eh;
          const int owner = ((col + 1) * S - 1) >> 7;
          const int lo = (owner * 128) / S;
          const uint32_t dst = mapa_shared(smem_u32(land + rank * NT * 64 + (col - lo)), static_cast<uint32_t>(owner));
#pragma unroll
          for (int o = 0; o < NOCT; ++o)
#pragma unroll
            for (int el = 0; el < 2; ++el) {
              const int m = c + 4 * el + 8 * o;
              st_cluster_f32(dst + m * 64 * 4, keep[r][o][2 * eh + el]);
            }
        }
    }
    cluster_arrive();
    cluster_wait();
    if (threadIdx.x == 96) rf_mark(args.trace, 7);
    const int mcount = args.M < NT ? args.M : NT;
    const int lo = (static_cast<int>(rank) * 128) / S, hi = ((static_cast<int>(rank) + 1) * 128) / S;
    const int w = hi - lo;
    for (int q = static_cast<int>(threadIdx.x); q < w * NT; q += Cfg::THREADS) {
      const int m = q / w, col = q - (q / w) * w;
      if (m < mcount) {
        float s = land[m * 64 + col];
        for (int r = 1; r < S; ++r) s += land[(r * NT + m) * 64 + col];
        rf_store<BF16, OUT>(args.out, static_cast<size_t>(m) * args.N + static_cast<size_t>(tile) * 128 + lo + col, s);
      }
    }
  }
  if (threadIdx.x == 96) rf_mark(args.trace, 4);
}



}  // namespace w4k
