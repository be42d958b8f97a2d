// gemm_rf.cuh -- decode (M <= 16) W4A16 GEMM for sm_100a with a register-fed tensor path:
// packed codes stream HBM -> shared memory (cp.async.bulk, mbarrier ring), every consumer warp
// dequantises them in registers straight into warp-level MMA fragments (mma.sync m16n8k16,
// fp32 accumulators in registers).  §8(a) rows a3-a10 for M <= 16.
//
// Why not tcgen05 here (measured): at M <= 16 the GEMM is HBM-bound and the
// tensor core is nearly idle, but a tcgen05.mma reads its weight operand from TMEM or shared
// memory, so the dequantised weights (2 B each) must first be staged there (tcgen05.st: 64 KB
// per 16 KB of codes) and handed between warp roles through mbarriers; round 1's TMEM decode
// kernel was bound by exactly that staging and hand-over chain (0.42 of HBM on the bench mix).
// Here the dequantised operand never leaves the registers of the thread that produced it:
// microbenchmark (scripts/microbench_hmma.cu, B200): LDS + LOP3 I2F + HSUB2 + mma.sync sustains
// 39 weights/clk/SM at 16 tokens and more at 8 tokens, i.e. >= 5 TB/s of packed codes, while
// the legacy HMMA pipe (0.5 m16n8k16/clk/SM) is far from saturated at M <= 8.
//
// Algebra (reading R6b): the group scale is factored out of the k-sum,
//     C[m][n] = sum_g s[g][n] * D_g[n][m],   D_g[n][m] = sum_{k in g} (q[k][n] - z[g][n]) * A[m][k],
// with the exact integer (q - z) as the bf16/fp16 MMA operand (LOP3 magic + one exact sub) and
// s applied in fp32 once per group (FFMA).
//
// Fragment mapping onto LAYOUT v1 (no re-pack): the MMA's A operand is the weight
// tile (rows = 16 output columns n, k16), B = activations (k16 x 8 tokens).  Lane (g, c)
// (g = lane / 4, c = lane % 4) loads with LDS.32 the words wj = c of half j of rows g and g+8 of
// its row group: 8 k-consecutive codes each, the 4 lanes of a quad cover 32 k of a row
// (conflict-free: 8 rows x 16 contiguous bytes per warp load).  Word j, pairs 2h and 2h+1 form
// fragment f = 2j + h: MMA k-slots (2c, 2c+1) <- k = 32j + 8c + 4h + {0,1}, (2c+8, 2c+9) <-
// +{2,3}.  The MMA is indifferent to the order of k, so the B fragment of lane (g, c) is the
// 4 activations A[token][32j + 8c + 4h .. +3]: one LDS.128 per (j, token octet) covers h = 0, 1.
// Token of B column g: sigma(g) = (g >> 1) | ((g & 1) << 2) (keeps those LDS.128 conflict-free
// on the SW128 activation tile).
//
// Work split: persistent stream-K.  T = n_tiles * kc units of (128 columns, 256 k); CTA p owns
// [p*T/P, (p+1)*T/P); a tile shared by several CTAs is finalised by the CTA holding its head
// from the fp32 partials of the others (caller/library workspace, gpu-scope flags, fixed CTA
// order -> deterministic).
//
// Warps: 0 = weight producer (1-D bulk, may run ahead of griddepcontrol.wait), 1 = activation
// producer (3-D TMA, one request per chunk), 2 = s/z producer (two 2-D TMA boxes per chunk, into
// the same stage as the activations), 3.. = NG consumer groups of 4 warps.  Group j takes the
// CTA's chunks i = j, j + NG, ...; warp rb of a group owns rows 32 rb .. 32 rb + 31 (two 16-row
// MMA groups) of the tile; the NG groups' partial sums are added in fixed order at a segment end.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "dequant.cuh"
#include "ptx.cuh"

namespace w4k {

struct RfArgs {
  const uint8_t* packed;  // LAYOUT v1
  const uint16_t* scales; // fp16 [K/group][N]
  const uint16_t* zeros;  // fp16 [K/group][N]
  void* out;              // [M][N] bf16/fp16 or fp32
  float* workspace;       // [P][NT][128] fp32 partial slots (a CTA's first segment)
  int* flags;             // [P], zero between launches
  uint32_t* trace;        // debug timeline (tm_set_trace) or null: [cta][32] %globaltimer low words
  int M, N, K, group;
  int n_tiles;
  int kc;                 // chunks (256 k) per tile
  uint32_t total;         // n_tiles * kc
};

#ifndef TM_RF_DIAG
#define TM_RF_DIAG 0  // timing experiments only (results wrong): 1 = consumers skip the math
#endif
#ifndef TM_RF_LDS64
#define TM_RF_LDS64 0  // lane word mapping: 0 = LDS.32 per word (conflict-free), 1 = LDS.64 pairs
#endif
// token of D column 2c (T0) and 2c + 1 (T1), and the token row of B column g (SIG)
#if TM_RF_LDS64
#define RF_T0(c) (2 * (c))
#define RF_T1(c) (2 * (c) + 1)
#define RF_SIG(g) (g)
#else
#define RF_T0(c) (c)
#define RF_T1(c) ((c) + 4)
#define RF_SIG(g) (((g) >> 1) | (((g) & 1) << 2))
#endif
#ifndef TM_RF_NSA
#define TM_RF_NSA 8
#endif
#ifndef TM_RF_NSW
#define TM_RF_NSW 10
#endif

#ifndef TM_RF_NG
#define TM_RF_NG 2
#endif

template <int NT, int NG>
struct RfCfg {
  static constexpr int TO = NT / 8;               // token octets (B fragments per k16)
  static constexpr int CH = 256;                  // k per chunk
  static constexpr int W_CODES = 16384;           // 4 LAYOUT v1 blobs
  static constexpr int SZ_BYTES = 4 * 128 * 2;    // s or z of one chunk: <= 4 groups x 128 columns
  static constexpr int W_BYTES = W_CODES + 2 * SZ_BYTES;  // weight stage: codes, s box, z box
  static constexpr int A_BYTES = NT * CH * 2;     // activation stage: 4 SW128 sub-tiles [NT][64]
  static constexpr int NCW = 4 * NG;              // consumer warps: NG groups of 4
  static constexpr int NPW = 3;                   // producer warps: weights, activations, s/z
  static constexpr int THREADS = 32 * (NPW + NCW);
  static constexpr int RS = 136;                  // red row stride (floats): conflict-free stores
  static constexpr int RED_BYTES = NG * NT * RS * 4;
  static constexpr int NSA = TM_RF_NSA > NG ? TM_RF_NSA : NG + 1;  // activation ring
  // weight ring: everything else.  A group copies a chunk's codes to registers and frees the
  // stage at once, so all NSW stages are HBM requests in flight (bandwidth x latency ~ 50+ KB/SM)
  static constexpr int NSW_FIT = (227 * 1024 - 2048 - NSA * A_BYTES - RED_BYTES - NG * 2 * 4 * NT * 4) / W_BYTES;
  static constexpr int NSW = NSW_FIT < TM_RF_NSW ? NSW_FIT : TM_RF_NSW;
  static constexpr int OFF_W = 1024;              // after the barrier header (1024-aligned)
  static constexpr int OFF_A = OFF_W + NSW * W_BYTES;
  static constexpr int OFF_RED = OFF_A + NSA * A_BYTES;
  static constexpr int SA_BYTES = NG * 2 * 4 * NT * 4;  // per group, 2 buffers: [blob][token] fp32
  static constexpr int OFF_SA = OFF_RED + RED_BYTES;
  static constexpr int SMEM = OFF_SA + SA_BYTES + 1024;  // + alignment slack
  static_assert(SMEM <= 227 * 1024, "shared memory");
  static_assert(2 * (NSW + NSA) * 8 <= 1024, "barrier header");
  static_assert(NG <= NSA && NG <= NSW, "rings");
};

template <bool BF16>
__device__ __forceinline__ void hmma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  if constexpr (BF16)
    asm("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  else
    asm("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// mbarrier wait that fails loudly instead of hanging: each probe parks the warp until the phase
// completes or the suspend hint expires, so 2^16 failed probes mean a broken pipeline.
__device__ __forceinline__ void rf_wait(uint32_t bar, uint32_t parity) {
  for (uint32_t i = 0; !mbar_try_wait_sleep(bar, parity);)
    if (++i == (1u << 16)) __trap();
}

__device__ __forceinline__ void rf_mark(uint32_t* trace, int slot) {
  if (trace) {
    uint64_t gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    trace[blockIdx.x * 32 + slot] = static_cast<uint32_t>(gt);
  }
}

__device__ __forceinline__ void named_bar(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

template <bool BF16, int OUT>
__device__ __forceinline__ void rf_store8(void* out, size_t idx, const float (&v)[8]) {
  if constexpr (OUT == 1) {
    float4* o = reinterpret_cast<float4*>(reinterpret_cast<float*>(out) + idx);
    o[0] = make_float4(v[0], v[1], v[2], v[3]);
    o[1] = make_float4(v[4], v[5], v[6], v[7]);
  } else {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if constexpr (BF16) {
        const __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
        w[i] = *reinterpret_cast<const uint32_t*>(&h);
      } else {
        const __half2 h = __floats2half2_rn(v[2 * i], v[2 * i + 1]);
        w[i] = *reinterpret_cast<const uint32_t*>(&h);
      }
    }
    *reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(out) + idx) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// One chunk (4 LAYOUT v1 blobs = 256 k x 128 columns) for one consumer warp: its 32 rows (two
// 16-row MMA groups r), all tokens.  NB = 4: full chunk, straight-line; NB = 3: K tail (nb < 4).
//
// Zero point folded out of the operand (reading R6b'): the MMA operand is the exact magic value
// V + q (V = 128 for bf16, 1024 for fp16: one LOP3 per pair, no subtraction), so
//     D_g = sum_{k in g} (V + q) A = sum (q - z) A + (V + z) SA_g,   SA_g[m] = sum_{k in g} A[m][k]
// and the group-end step is  acc += s * (D_g - (V + z) * SA_g)  in fp32.  SA is computed on the
// tensor core (an all-ones A fragment times the same B fragments): warp rb of the group sums blob
// rb of the chunk and the four warps exchange their sums through shared memory (named barrier
// per group and chunk, double-buffered by chunk parity).
template <int NT, int GROUP, bool BF16, int NB>
__device__ __forceinline__ void rf_chunk(float (&acc)[2][NT / 8][4], const uint8_t* wst, const uint8_t* ast,
                                         float* sa, int bar_id, int nb, int rb, int g, int c, int sig) {
  const uint16_t* ssm = reinterpret_cast<const uint16_t*>(wst + RfCfg<NT, 1>::W_CODES);  // [group][128]
  const uint16_t* zsm = ssm + 4 * 128;
  constexpr int TO = NT / 8;
  constexpr int BPG = GROUP / 64;  // blobs per group
  constexpr uint32_t ONES = BF16 ? 0x3F803F80u : 0x3C003C00u;
  constexpr float V = BF16 ? 128.0f : 1024.0f;
  const auto load_b = [&](int b, uint4 (&bfr)[2][TO]) {
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int o = 0; o < TO; ++o) {
        const int row = sig + 8 * o;
#if TM_RF_LDS64
        bfr[j][o] =
            *reinterpret_cast<const uint4*>(ast + b * (NT * 128) + row * 128 + (((2 * c + j) ^ (row & 7)) << 4));
#else
        bfr[j][o] =
            *reinterpret_cast<const uint4*>(ast + b * (NT * 128) + row * 128 + (((4 * j + c) ^ (row & 7)) << 4));
#endif
      }
  };
  // ---- activation sums of blob rb (this warp's share of the chunk)
  if ((TM_RF_DIAG & 2) == 0 && (NB == 4 || rb < nb)) {
    uint4 bfr[2][TO];
    load_b(rb, bfr);
    float ds[TO][4];
#pragma unroll
    for (int o = 0; o < TO; ++o)
#pragma unroll
      for (int e = 0; e < 4; ++e) ds[o][e] = 0.f;
    const uint32_t ones[4] = {ONES, ONES, ONES, ONES};
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int o = 0; o < TO; ++o) {
        hmma16816<BF16>(ds[o], ones, bfr[j][o].x, bfr[j][o].y);
        hmma16816<BF16>(ds[o], ones, bfr[j][o].z, bfr[j][o].w);
      }
    if (g == 0) {
#pragma unroll
      for (int o = 0; o < TO; ++o) {
        sa[rb * NT + RF_T0(c) + 8 * o] = ds[o][0];
        sa[rb * NT + RF_T1(c) + 8 * o] = ds[o][1];
      }
    }
  }
  if ((TM_RF_DIAG & 2) == 0) named_bar(bar_id, 128);
  float dg[2][TO][4];
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    if (NB == 4 || b < nb) {
      const int gi = b / BPG;
      if (b % BPG == 0) {
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
          for (int o = 0; o < TO; ++o)
#pragma unroll
            for (int e = 0; e < 4; ++e) dg[r][o][e] = 0.f;
      }
      uint4 bfr[2][TO];
      load_b(b, bfr);
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        uint32_t w0[2], w1[2];
        if (TM_RF_DIAG & 8) {
          w0[0] = b * 0x9E3779B9u + r;  // diagnostic: no weight loads
          w0[1] = w0[0] ^ 0x5555u;
          w1[0] = w0[0] * 3u;
          w1[1] = w1[0] ^ 0x3333u;
        } else {
          // ldmatrix.x4 on the packed blob viewed as 16-bit elements: matrix q = (row half q & 1,
          // k half q >> 1) is 8 rows x 16 B; lane (g, c) receives bytes 4c..4c+3 of row g, i.e.
          // the LAYOUT v1 word wj = c of that row and half (conflict-free: 128 contiguous B each)
          const int l = threadIdx.x & 31;
          const uint32_t addr = smem_u32(wst) + b * 4096 + (l >> 4) * 2048 +
                                (32 * rb + 16 * r + ((l >> 3) & 1) * 8 + (l & 7)) * 16;
          asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
                       : "=r"(w0[0]), "=r"(w1[0]), "=r"(w0[1]), "=r"(w1[1])
                       : "r"(addr)
                       : "memory");
        }
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          uint32_t p0[4], p1[4];
          deq_word_magic<BF16>(w0[j], p0);
          deq_word_magic<BF16>(w1[j], p1);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint32_t a[4] = {p0[2 * h], p1[2 * h], p0[2 * h + 1], p1[2 * h + 1]};
#pragma unroll
            for (int o = 0; o < TO; ++o) {
              const uint32_t b0 = h ? bfr[j][o].z : bfr[j][o].x;
              const uint32_t b1 = h ? bfr[j][o].w : bfr[j][o].y;
              if (TM_RF_DIAG & 16)  // diagnostic: no MMA
                dg[r][o][0] = __uint_as_float(__float_as_uint(dg[r][o][0]) ^ a[0] ^ a[1] ^ a[2] ^ a[3] ^ b0 ^ b1);
              else
                hmma16816<BF16>(dg[r][o], a, b0, b1);
            }
          }
        }
      }
      // group end: fold the zero point back in and apply the scale (fp32), once per group
      if ((TM_RF_DIAG & 4) && (b % BPG == BPG - 1 || (NB != 4 && b + 1 == nb))) {
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
          for (int o = 0; o < TO; ++o)
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[r][o][e] += dg[r][o][e];  // diagnostic: no scale step
      } else if (b % BPG == BPG - 1 || (NB != 4 && b + 1 == nb)) {
        float sam[TO][2];
#pragma unroll
        for (int o = 0; o < TO; ++o) {
          sam[o][0] = sa[(gi * BPG) * NT + RF_T0(c) + 8 * o];
          sam[o][1] = sa[(gi * BPG) * NT + RF_T1(c) + 8 * o];
          if (BPG == 2 && (NB == 4 || gi * BPG + 1 < nb)) {
            sam[o][0] += sa[(gi * BPG + 1) * NT + RF_T0(c) + 8 * o];
            sam[o][1] += sa[(gi * BPG + 1) * NT + RF_T1(c) + 8 * o];
          }
        }
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const int row0 = 32 * rb + 16 * r + g;
          const float s0 = __half2float(__ushort_as_half(ssm[gi * 128 + row0]));
          const float s1 = __half2float(__ushort_as_half(ssm[gi * 128 + row0 + 8]));
          const float v0 = V + __half2float(__ushort_as_half(zsm[gi * 128 + row0]));
          const float v1 = V + __half2float(__ushort_as_half(zsm[gi * 128 + row0 + 8]));
#pragma unroll
          for (int o = 0; o < TO; ++o) {
            acc[r][o][0] = fmaf(s0, fmaf(-v0, sam[o][0], dg[r][o][0]), acc[r][o][0]);
            acc[r][o][1] = fmaf(s0, fmaf(-v0, sam[o][1], dg[r][o][1]), acc[r][o][1]);
            acc[r][o][2] = fmaf(s1, fmaf(-v1, sam[o][0], dg[r][o][2]), acc[r][o][2]);
            acc[r][o][3] = fmaf(s1, fmaf(-v1, sam[o][1], dg[r][o][3]), acc[r][o][3]);
          }
        }
      }
    }
  }
}

template <int NT, int NG, int GROUP, bool BF16, int OUT>
__global__ void __launch_bounds__(RfCfg<NT, NG>::THREADS, 1)
    w4a16_rf_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_s,
                    const __grid_constant__ CUtensorMap tmap_z, const RfArgs args) {
  using Cfg = RfCfg<NT, NG>;
  constexpr int TO = Cfg::TO;
  constexpr int NSW = Cfg::NSW, NSA = Cfg::NSA;
  constexpr int NCW = Cfg::NCW;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* base_ptr = smem_raw + (base - raw);  // (keeps the shared address space: LDS, not LD)
  const uint32_t bar_fullw = base, bar_emptyw = base + 8 * NSW;
  const uint32_t bar_fulla = base + 16 * NSW, bar_emptya = bar_fulla + 8 * NSA;
  const uint32_t sw = base + Cfg::OFF_W, sa = base + Cfg::OFF_A;
  float* red = reinterpret_cast<float*>(base_ptr + Cfg::OFF_RED);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t P = gridDim.x, p = blockIdx.x, T = args.total;
  const uint32_t u0 = (p * T) / P, u1 = ((p + 1) * T) / P;  // host: T * P < 2^32
  const uint32_t kc = static_cast<uint32_t>(args.kc);
  const int kstages = args.K >> 6;  // 64-k blobs per tile

  if (threadIdx.x == 0) {
    rf_mark(args.trace, 0);
    for (int i = 0; i < NSW; ++i) {
      mbar_init(bar_fullw + 8 * i, 2);  // code + s/z producers
      mbar_init(bar_emptyw + 8 * i, 4);  // the 4 warps of the owning group
    }
    for (int i = 0; i < NSA; ++i) {
      mbar_init(bar_fulla + 8 * i, 1);
      mbar_init(bar_emptya + 8 * i, 4);
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

  if (warp == 0) {
    // ---------------------------------------------------------------- weight producer
    // Packed weights are constant inputs of the layer: streamed before griddepcontrol.wait
    // (overlaps the previous kernel's tail under PDL).
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      uint32_t t = u0 / kc, kq = u0 - (u0 / kc) * kc;
      int stage = 0;
      uint32_t phase = 0;
      for (uint32_t u = u0; u < u1; ++u) {
        rf_wait(bar_emptyw + 8 * stage, phase ^ 1);
        const int nb = min(4, kstages - static_cast<int>(kq) * 4);
        mbar_arrive_expect_tx(bar_fullw + 8 * stage, nb * 4096);
        const uint8_t* src = args.packed + (static_cast<size_t>(t) * kstages + kq * 4) * 4096;
        bulk_g2s_hint(sw + stage * Cfg::W_BYTES, src, nb * 4096, bar_fullw + 8 * stage, pol);
        if (++stage == NSW) {
          stage = 0;
          phase ^= 1;
        }
        if (++kq == kc) {
          kq = 0;
          ++t;
        }
      }
    }
    return;
  }
  if (warp == 1) {
    // ---------------------------------------------------------------- activation producer
    if (lane == 0) {
      grid_dependency_wait();  // activations may be written by the previous kernel
      uint32_t kq = u0 - (u0 / kc) * kc;
      int stage = 0;
      uint32_t phase = 0;
      for (uint32_t u = u0; u < u1; ++u) {
        rf_wait(bar_emptya + 8 * stage, phase ^ 1);
        mbar_arrive_expect_tx(bar_fulla + 8 * stage, Cfg::A_BYTES);
        tma_load_3d(sa + stage * Cfg::A_BYTES, &tmap_a, 0, 0, static_cast<int>(kq) * 4, bar_fulla + 8 * stage);
        if (++stage == NSA) {
          stage = 0;
          phase ^= 1;
        }
        if (++kq == kc) kq = 0;
      }
    }
    return;
  }
  if (warp == 2) {
    // ---------------------------------------------------------------- s/z producer
    if (lane == 0) {
      grid_dependency_wait();
      constexpr int GPC = 256 / GROUP;  // groups per chunk
      uint32_t t = u0 / kc, kq = u0 - (u0 / kc) * kc;
      int stage = 0;
      uint32_t phase = 0;
      for (uint32_t u = u0; u < u1; ++u) {
        rf_wait(bar_emptyw + 8 * stage, phase ^ 1);
        mbar_arrive_expect_tx(bar_fullw + 8 * stage, 2 * GPC * 128 * 2);
        const uint32_t dst = sw + stage * Cfg::W_BYTES + Cfg::W_CODES;
        tma_load_2d(dst, &tmap_s, static_cast<int>(t) * 128, static_cast<int>(kq) * GPC, bar_fullw + 8 * stage);
        tma_load_2d(dst + Cfg::SZ_BYTES, &tmap_z, static_cast<int>(t) * 128, static_cast<int>(kq) * GPC,
                    bar_fullw + 8 * stage);
        if (++stage == NSW) {
          stage = 0;
          phase ^= 1;
        }
        if (++kq == kc) {
          kq = 0;
          ++t;
        }
      }
    }
    return;
  }
  // ---------------------------------------------------------------- consumers
  grid_dependency_wait();  // workspace and flags after the previous kernel
  if (threadIdx.x == 32 * Cfg::NPW) rf_mark(args.trace, 2);
  bool first_chunk = true;
  int sabuf = 0;
  const int cw = warp - Cfg::NPW;
  const int grp = cw >> 2, rb = cw & 3;
  const int g = lane >> 2, c = lane & 3;
  const int sig = RF_SIG(g);  // token of B column g (within an octet)
  const int ct = threadIdx.x - 32 * Cfg::NPW;  // 0 .. 32 * NCW - 1
  float acc[2][TO][4];
  // ring position of this group's next chunk (chunk index i = u - u0, i = grp, grp + NG, ...)
  int wstage = grp, astage = grp;  // (NG <= NSW, NSA)
  uint32_t wphase = 0, aphase = 0;
  uint32_t um = u0 + grp;  // next chunk owned by this warp group
  uint32_t t = u0 / kc;
  uint32_t u = u0;
  while (u < u1) {
    // ---- one segment: units [u, seg_end) of tile t
    const uint32_t seg_u0 = u;
    const uint32_t tile_lo = t * kc, tile_hi = tile_lo + kc;
    const uint32_t seg_end = u1 < tile_hi ? u1 : tile_hi;
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int o = 0; o < TO; ++o)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[r][o][e] = 0.f;
    for (; um < seg_end; um += NG) {
      const int kq = static_cast<int>(um - tile_lo);
      const int nb = min(4, kstages - kq * 4);
      rf_wait(bar_fullw + 8 * wstage, wphase);
      if (first_chunk && threadIdx.x == 32 * Cfg::NPW) rf_mark(args.trace, 3);
      rf_wait(bar_fulla + 8 * astage, aphase);
      if (first_chunk && threadIdx.x == 32 * Cfg::NPW) rf_mark(args.trace, 4);
      first_chunk = false;
      {
        const uint8_t* wst = base_ptr + Cfg::OFF_W + wstage * Cfg::W_BYTES;
        const uint8_t* ast = base_ptr + Cfg::OFF_A + astage * Cfg::A_BYTES;
        float* sa = reinterpret_cast<float*>(base_ptr + Cfg::OFF_SA) + (grp * 2 + sabuf) * 4 * NT;
        sabuf ^= 1;
        if (TM_RF_DIAG & 1) {
        } else if (nb == 4)
          rf_chunk<NT, GROUP, BF16, 4>(acc, wst, ast, sa, 2 + grp, 4, rb, g, c, sig);
        else
          rf_chunk<NT, GROUP, BF16, 3>(acc, wst, ast, sa, 2 + grp, nb, rb, g, c, sig);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_emptyw + 8 * wstage);
      wstage += NG;
      if (wstage >= NSW) {
        wstage -= NSW;
        wphase ^= 1;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_emptya + 8 * astage);
      astage += NG;
      if (astage >= NSA) {
        astage -= NSA;
        aphase ^= 1;
      }
    }
    u = seg_end;
    if (lane == 0) rf_mark(args.trace, 5 + cw);  // last chunk of this warp in the segment (overwritten)
    // ---- segment end: add the NG groups' partials (fixed order), then store / hand off / fix up
    {
      float* rk = red + grp * NT * Cfg::RS;
#pragma unroll
      for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int o = 0; o < TO; ++o) {
          const int n0 = 32 * rb + 16 * r + g;
          const int m0 = RF_T0(c) + 8 * o, m1 = RF_T1(c) + 8 * o;
          rk[m0 * Cfg::RS + n0] = acc[r][o][0];
          rk[m1 * Cfg::RS + n0] = acc[r][o][1];
          rk[m0 * Cfg::RS + n0 + 8] = acc[r][o][2];
          rk[m1 * Cfg::RS + n0 + 8] = acc[r][o][3];
        }
    }
    named_bar(1, 32 * NCW);
    const int mcount = args.M < NT ? args.M : NT;
    // consumer thread ct < NT * 16 owns 8 consecutive columns of one token
    const bool active = ct < NT * 16;
    const int m = ct >> 4, nv = (ct & 15) * 8;
    float v[8];
    if (active) {
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = 0.f;
#pragma unroll
      for (int q = 0; q < NG; ++q) {
        const float4* rr = reinterpret_cast<const float4*>(red + (q * NT + m) * Cfg::RS + nv);
        const float4 a0 = rr[0], a1 = rr[1];
        v[0] += a0.x; v[1] += a0.y; v[2] += a0.z; v[3] += a0.w;
        v[4] += a1.x; v[5] += a1.y; v[6] += a1.z; v[7] += a1.w;
      }
    }
    if (seg_u0 != tile_lo) {
      // tail or middle piece of a shared tile: always this CTA's first segment -> slot p
      if (active) {
        float4* ws = reinterpret_cast<float4*>(args.workspace + (static_cast<size_t>(p) * NT + m) * 128 + nv);
        __stcg(ws, make_float4(v[0], v[1], v[2], v[3]));
        __stcg(ws + 1, make_float4(v[4], v[5], v[6], v[7]));
      }
      // bar.sync orders every consumer's partial stores before thread 0's release (cumulative)
      named_bar(1, 32 * NCW);
      if (ct == 0) st_release_gpu(args.flags + p, 1);
    } else {
      if (seg_end != tile_hi) {
        // head of a shared tile (this CTA's last segment): add the later contributors' partials.
        // Lanes of the first consumer warp poll one flag each (in parallel), then every thread
        // issues all of its partial loads before adding them in fixed CTA order (deterministic).
        const uint32_t p_hi = static_cast<uint32_t>((static_cast<uint64_t>(tile_hi) * P - 1) / T);
        if (ct < 32) {
          for (uint32_t q0 = p + 1; q0 <= p_hi; q0 += 32) {
            const uint32_t q = q0 + ct;
            bool ok = q > p_hi;
            for (uint32_t spins = 0; !__all_sync(0xffffffffu, ok);) {
              if (!ok) ok = ld_acquire_gpu(args.flags + q) != 0;
              if (++spins == (1u << 26)) __trap();  // a contributor never arrived: fail, do not hang
            }
          }
        }
        named_bar(1, 32 * NCW);
        for (uint32_t q0 = p + 1; q0 <= p_hi; q0 += 4) {
          float4 part[4][2];
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (active && q0 + i <= p_hi) {
              const float4* wq = reinterpret_cast<const float4*>(
                  args.workspace + (static_cast<size_t>(q0 + i) * NT + m) * 128 + nv);
              part[i][0] = __ldcg(wq);
              part[i][1] = __ldcg(wq + 1);
            }
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (active && q0 + i <= p_hi) {
              v[0] += part[i][0].x; v[1] += part[i][0].y; v[2] += part[i][0].z; v[3] += part[i][0].w;
              v[4] += part[i][1].x; v[5] += part[i][1].y; v[6] += part[i][1].z; v[7] += part[i][1].w;
            }
        }
        if (ct < 32)
          for (uint32_t q = p + 1 + ct; q <= p_hi; q += 32) args.flags[q] = 0;  // consumed: zero for the next launch
      }
      if (active && m < mcount) rf_store8<BF16, OUT>(args.out, static_cast<size_t>(m) * args.N + t * 128 + nv, v);
    }
    named_bar(1, 32 * NCW);  // red is reused by the next segment
    ++t;
  }
  if (ct == 0) rf_mark(args.trace, 31);
}

}  // namespace w4k
