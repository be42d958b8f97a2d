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
// Warps (32 x (8 + 4 NDS) threads; ids ordered by issue priority, see DecCfg):
//   4j..4j+3   dequant j  : NDS sets of 4 warps; set j takes chunks i with i % NDS == j and owns
//                           TMEM operand slot j; thread = weight column = TMEM lane; LDS.128,
//                           LOP3 magic + exact sub, tcgen05.st
//   4NDS..+3   scale/epi  : tcgen05.ld D_g, acc[m] += s * D_g[m] (fp32 registers); at a segment
//                           end: RNE store of C, or fp32 partial + deterministic stream-K fix-up
//   4NDS+4,+5  MMA        : issuer j takes chunks i with i % NISSUE == j (all groups); D_g -> TMEM
//   4NDS+6     producer A : s/z boxes (2-D TMA), activation chunks (3-D TMA, SW128) after
//                           griddepcontrol.wait, freed by the MMA commit
//   4NDS+7     producer W : weight chunks (1-D bulk, before griddepcontrol.wait), freed by the
//                           dequant
// Per chunk: one full wait and one ready arrive (dequant), one ready wait + one D-slot wait +
// one commit (MMA), one done wait + one D-slot release (scale).
//
// FS variant (cluster split-K, group 128): no scale warps.  Dequant set j waits for
// the completion of its own chunk's MMAs, reads that chunk's D_g from its 32-column TMEM region
// and accumulates s * D_g in registers; at the segment end sets 1..NDS-1 deposit their partial
// sums in shared memory and set 0 adds them in set order (deterministic).
// Operands go to TMEM as two 16-column tcgen05.st halves per blob, each issued as soon as its 4
// words are dequantised (staging the operand is the largest single cost).
#pragma once
#include <cstdint>
#include <type_traits>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "dequant.cuh"
#include "ptx.cuh"

namespace w4k {

#ifndef TM_CLUSTER_PUSH
#define TM_CLUSTER_PUSH 0
#endif
#ifndef TM_SZS
#define TM_SZS 4
#endif
#ifndef TM_NW16
#define TM_NW16 6
#endif
#ifndef TM_NA16
#define TM_NA16 6
#endif
#ifndef TM_ST_HALF
#define TM_ST_HALF 1
#endif
#ifndef TM_PRE_BLOB
#define TM_PRE_BLOB 1
#endif
#ifndef TM_EARLY_W
#define TM_EARLY_W 0
#endif
#ifndef TM_SCALE_TOP
#define TM_SCALE_TOP 0
#endif


constexpr int kMaxExperts = 64;

struct DecArgs {
  const uint8_t* packed;  // LAYOUT v1
  void* out;              // [M][N] bf16/fp16 or fp32
  float* workspace;       // [P][NT][128] fp32 partial slots (one per CTA: its first segment)
  int* counters;          // [P] partial-ready flags (zero between launches)
  int M, N, K, group;
  int n_tiles, m_tiles;
  int kc;                 // chunks per tile = ceil(K / 256)
  long long total;        // m_tiles * n_tiles * kc
  int cluster;            // 0: persistent stream-K over [0, total); CS >= 1: CS CTAs per tile
                          // (a thread-block cluster when CS > 1), tile = blockIdx.x / CS
  int a_ks;               // 64-k blobs of A along K: K / 64, or K / 128 for W8 bit planes (A reused)
  uint32_t* trace;
};

// Grouped launch (MoE, §8(f) NEXT-3; the kernel's GROUPED instantiation only, so the plain
// launches keep a small parameter block): n_experts problems share one launch.  Expert e owns
// tiles [tile_start[e], tile_start[e + 1]) (local tile index mt * n_tiles + nt), rows
// [row_start[e], row_start[e] + m_count[e]) of A and C, packed weights at blob offset
// e * n_tiles * (K / 64) and s/z group rows from e * K / group.
struct DecGroups {
  int n_experts;
  int tile_start[kMaxExperts + 1];
  int row_start[kMaxExperts];
  int m_count[kMaxExperts];
};
struct DecNoGroups {};

// Where tile t lives: its n-tile, first A/C row, valid rows (<= NT) and the expert's weight blob
// and s/z group-row offsets.
struct DecTile {
  int nt, row0, mcount;
  long long blob0;  // first 4 KB blob of the expert's packed weight
  int g0;           // first s/z group row of the expert
};
template <int NT, typename GA>
__device__ __forceinline__ DecTile dec_tile(const DecArgs& a, const GA& ga, int t) {
  DecTile r;
  int e = 0, local = t, rows = a.M, row_base = 0;
  if constexpr (std::is_same<GA, DecGroups>::value) {
    while (e + 1 < ga.n_experts && ga.tile_start[e + 1] <= t) ++e;
    local = t - ga.tile_start[e];
    rows = ga.m_count[e];
    row_base = ga.row_start[e];
  }
  const int mt = static_cast<int>(static_cast<unsigned>(local) / static_cast<unsigned>(a.n_tiles));
  r.nt = local - mt * a.n_tiles;
  r.row0 = row_base + mt * NT;
  r.mcount = rows - mt * NT < NT ? rows - mt * NT : NT;
  r.blob0 = static_cast<long long>(e) * a.n_tiles * (a.K >> 6);
  r.g0 = e * (a.K / a.group);
  return r;
}

template <int NT, bool FS = false>
struct DecCfg {
  static constexpr int CH = 256;                         // k per chunk
  static constexpr int BLOBS = 4;                        // LAYOUT v1 blobs per chunk
  static constexpr int ACT_BYTES = NT * CH * 2;          // activation chunk (4 SW128 sub-tiles)
  static constexpr int W_BYTES = BLOBS * 4096;           // packed weight chunk
  static constexpr int NW = NT <= 16 ? TM_NW16 : (NT <= 32 ? 6 : 5);   // weight ring (freed after the dequant's LDS)
  static constexpr int NA = NT <= 16 ? TM_NA16 : (NT <= 32 ? 6 : 4);   // activation ring = per-chunk ready/done ring
  static constexpr int NDS = NT <= 16 ? 3 : 2;           // dequant sets = TMEM operand slots
  static constexpr int DCOLS = NT;                       // one D_g slot
  static constexpr int DAVAIL = 512 - NDS * BLOBS * 32;  // TMEM columns left for the D ring
  static constexpr int DR_MAX = 4;                       // D ring entries (chunks); runtime: dec_dring()
  // FS (fused scale, group 128): no scale warps -- dequant set j also applies the group scales
  // to the D of its own chunks (its D region: 2 groups x NT columns after the operand slots)
  static constexpr int THREADS = 32 * ((FS ? 4 : 8) + 4 * NDS);   // a multiple of 4 warps
  // warp roles.  The producers and the TMEM allocator come first: an SM starts a CTA's warps
  // one after another (measured: the last of 20 warps reached the barrier initialisation ~1800
  // cycles after warp 0 started), so the setup and the first weight requests go to warp 0.
  // (Issue priority does not follow warp ids -- reordering roles by id was measured neutral.)
  static constexpr int W_PRODW = 0;                      // weight producer + barrier init
  static constexpr int W_PRODA = 1;                      // activation + s/z producer
  static constexpr int W_MMA = 2;                        // 2 MMA issuer warps (also TMEM allocator)
  // TM_SCALE_TOP: scale warps take the highest ids (the SMSP arbiter favours high warp ids)
  static constexpr int W_SCALE = FS ? 4 : (TM_SCALE_TOP ? 4 + 4 * NDS : 4);   // 4 scale / epilogue warps
  static constexpr int W_DEQ = (FS || TM_SCALE_TOP) ? 4 : 8;               // 4 * NDS dequant warps
  static constexpr int SZG = 8;
  static constexpr int SZ_BOX = SZG * 128 * 2;
  static constexpr int SZ_SLOTS = TM_SZS;                // s/z boxes in flight (4: 16 chunks of look-ahead)
  static constexpr int TMEM_COLS = 512;
  // cluster split: the leader receives CS - 1 fp32 partials (NT x 128) in its weight ring
  static constexpr int MAX_CLUSTER = 1 + (NW * W_BYTES) / (NT * 512) < 8 ? 1 + (NW * W_BYTES) / (NT * 512) : 8;
  static constexpr int HDR = 1024;
  // FS: segment-end deposit of sets 1..NDS-1 (fp32 NT x 128 each)
  // cluster split-K "push" reduction (NT = 16, CS <= 4): a dedicated landing area for the fp32
  // partials of ranks 1..3, written through DSMEM as soon as each rank's sum is final
  static constexpr int RED_MAX = (TM_CLUSTER_PUSH && NT == 16 && FS) ? 3 : 0;  // (FS = the cluster-mode kernels)
  static constexpr int RED_BYTES = RED_MAX * NT * 128 * 4;
  static constexpr int SMEM = 1024 + HDR + NW * W_BYTES + NA * ACT_BYTES + SZ_SLOTS * 2 * SZ_BOX + RED_BYTES;
  // FS (cluster split-K only: one segment per CTA): the segment-end deposits of sets 1..NDS-1
  // go to the weight ring, idle once every set has finished the CTA's chunks
  static_assert(!FS || (NDS - 1) * NT * 128 * 4 <= NW * W_BYTES, "FS deposit area");
  static_assert(DAVAIL >= 4 * NT, "TMEM: one chunk of g = 64 D slots");
  static_assert(!FS || DAVAIL >= NDS * 2 * NT, "TMEM: FS D regions (group 128)");
  // a ready/done ring entry must be reused by the same dequant set (NA % NDS == 0: that set's
  // previous use is gated by the MMA completion it waits for) -- measured: NA = 4 with 3 sets
  // let a set arrive on an entry whose previous phase the MMA had not yet consumed
  static_assert(NA >= NDS && NA % NDS == 0, "rings");
  static_assert(SMEM <= 227 * 1024, "shared memory");
  // barrier block [fullw NW][emptyw NW][fulla NA][ready NA][done NA][dfree DR_MAX][szfull][szempty]
  // (+ TMEM slot word) fits the header
  static_assert((2 * NW + 3 * NA + DR_MAX + 2 * SZ_SLOTS) * 8 + 64 <= HDR, "barrier header");
};

// D ring depth for this launch: a chunk's D slots take (256 / group) * NT columns, so g = 128
// fits twice the ring of g = 64 (more slack between the MMA and the scale warps)
template <int NT>
__device__ __forceinline__ int dec_dring(int group) {
  // a chunk's D slots: (256 / group) * NT columns (compile-time per group: no runtime division)
  constexpr int n64 = DecCfg<NT>::DAVAIL / (4 * NT), n128 = DecCfg<NT>::DAVAIL / (2 * NT);
  const int n = group == 64 ? n64 : n128;
  return n >= 4 ? 4 : (n >= 2 ? 2 : 1);
}
// MMA issuers: two when each owns whole D ring entries and whole ready/done barriers (NA even:
// chunks sharing a barrier then share an issuer, so no parity aliasing), else one
template <int NT>
__device__ __forceinline__ int dec_nissue(int dring) {
  return (dring >= 2 && DecCfg<NT>::NA % 2 == 0) ? 2 : 1;
}

// 32-bit unsigned arithmetic (the host guarantees T * P < 2^32): a 64-bit division is a
// ~100-instruction subroutine and sat on every warp's prologue
__device__ __forceinline__ int dec_owner(uint32_t u, uint32_t T, uint32_t P) {
  return static_cast<int>(((u + 1) * P - 1) / T);
}
__device__ __forceinline__ uint32_t dec_start(uint32_t p, uint32_t T, uint32_t P) {
  return (p * T) / P;
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

// ring position (slot, phase) advanced without division
struct RingPos {
  int slot = 0;
  uint32_t phase = 0;
  __device__ __forceinline__ void advance(int n) {
    if (++slot == n) {
      slot = 0;
      phase ^= 1u;
    }
  }
};


// Iterate the CTA's segments: a segment is the part of one (m-tile, n-tile) inside [u0, u1).
#define DEC_FOR_SEGMENTS                                                                            \
  for (uint32_t u = u0, cend = 0; u < u1; u = cend)                                                  \
    if (const int t = static_cast<int>(u / kc); true)                                              \
      if ((cend = ((static_cast<uint32_t>(t) + 1) * kc < u1 ? (static_cast<uint32_t>(t) + 1) * kc : u1)), true)

template <int NT, bool BF16, int OUT, bool FS = false, typename GA = DecNoGroups>
__global__ void __launch_bounds__(DecCfg<NT, FS>::THREADS, 1)
    w4a16_dec_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_s,
                     const __grid_constant__ CUtensorMap tmap_z, const DecArgs args, const __grid_constant__ GA groups) {
  using Cfg = DecCfg<NT, FS>;
  constexpr int NR = Cfg::NA;  // activation slots and per-chunk ready/done barriers
  constexpr int NW = Cfg::NW;
  constexpr int NDS = Cfg::NDS;
  constexpr int DR_MAX = Cfg::DR_MAX;

  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* const base_ptr = smem_raw + (base - smem_u32(smem_raw));
  const uint32_t bar_fullw = base;                              // NW (W producer, tx)
  const uint32_t bar_emptyw = bar_fullw + 8 * NW;               // NW (128: the chunk's dequant set)
  const uint32_t bar_fulla = bar_emptyw + 8 * NW;               // NR (A producer, tx)
  const uint32_t bar_ready = bar_fulla + 8 * NR;                // NR (128: the chunk's dequant set)
  const uint32_t bar_done = bar_ready + 8 * NR;                 // NR (1 commit: the chunk's MMA issuer)
  const uint32_t bar_dfree = bar_done + 8 * NR;                 // DR_MAX (128 scale threads)
  const uint32_t bar_szfull = bar_dfree + 8 * DR_MAX;           // SZ_SLOTS (1)
  const uint32_t bar_szempty = bar_szfull + 8 * Cfg::SZ_SLOTS;  // SZ_SLOTS (128 NDS dequant + 128 scale)
  const uint32_t tmem_slot = bar_szempty + 8 * Cfg::SZ_SLOTS;
  uint32_t* const tmem_slot_ptr = reinterpret_cast<uint32_t*>(base_ptr + (tmem_slot - base));
  const uint32_t bar_red = tmem_slot + 16;  // cluster split: partials of ranks 1..CS-1 ready (leader)
  const uint32_t w0 = base + Cfg::HDR;                          // NW x 16 KB packed weights
  const uint32_t a0 = w0 + NW * Cfg::W_BYTES;                   // NR x activation chunk (1 KB aligned)
  const uint32_t sz0 = a0 + NR * Cfg::ACT_BYTES;                // SZ_SLOTS x [s box | z box]
  const uint8_t* const w_ptr0 = base_ptr + Cfg::HDR;
  const uint8_t* const sz_ptr0 = w_ptr0 + NW * Cfg::W_BYTES + NR * Cfg::ACT_BYTES;
  float* const dep_ptr0 = reinterpret_cast<float*>(base_ptr + Cfg::HDR);  // FS: the (idle) weight ring
  const uint32_t red0 = sz0 + Cfg::SZ_SLOTS * 2 * Cfg::SZ_BOX;             // push reduction area

  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);  // warp-uniform
  const uint32_t lane = threadIdx.x & 31;

  const int P = gridDim.x;
  const int p = blockIdx.x;
  const uint32_t T = static_cast<uint32_t>(args.total);
  const int CS = args.cluster;
  // cluster split-K, push mode: every thread arrives on the cluster barrier in the setup and waits
  // before its first remote access (or at its end), ranks > 0 push their partials into the
  // leader's landing area and arrive on its bar_red, the leader waits there -- no cluster-wide
  // barrier in the tail (vs two in the classic reduction)
  const bool push = TM_CLUSTER_PUSH && Cfg::RED_MAX > 0 && CS > 1 && CS <= Cfg::RED_MAX + 1;
  uint32_t u0, u1;
  if (CS > 0) {  // CS CTAs per tile: rank r takes chunks [r kc / CS, (r + 1) kc / CS) of tile p / CS
    // (unsigned 32-bit: a signed division is a called subroutine, an i-cache miss in the prologue)
    const uint32_t ucs = static_cast<uint32_t>(CS), ukc = static_cast<uint32_t>(args.kc);
    const uint32_t tile = static_cast<uint32_t>(p) / ucs, r = static_cast<uint32_t>(p) - tile * ucs;
    u0 = tile * ukc + (r * ukc) / ucs;
    u1 = tile * ukc + ((r + 1) * ukc) / ucs;
  } else {
    u0 = dec_start(p, T, P);
    u1 = dec_start(p + 1, T, P);
  }
  float acc_keep[NT];  // scale warps, cluster split: this CTA's partial until the cluster reduction
  const int KS = args.K / 64;
  const int kc = args.kc;
  const int gshift = args.group == 64 ? 6 : 7;
  const int bpg = args.group >> 6;  // blobs per group (1 or 2)
  const int bshift = gshift - 6;    // log2(bpg)
  const int box_mask = ((Cfg::SZG << gshift) / Cfg::CH) - 1;  // chunks per s/z box - 1 (2 or 4 chunks)
  const int DR = dec_dring<NT>(args.group);           // D ring entries (1, 2 or 4)
  const int dr_mask = DR - 1, dr_shift = DR == 4 ? 2 : DR - 1;
  const int NISSUE = dec_nissue<NT>(DR);  // 1 or 2
  const int is_mask = NISSUE - 1;
  const int DSTRIDE = (Cfg::CH >> gshift) * NT;        // D columns per ring entry

  // ---- weight producer: one lane per barrier initialises them (the mbarriers are contiguous
  // from bar_fullw); produce_w issues the weight chunks of this CTA's range
  const uint64_t w_policy = policy_evict_first();
  RingPos w_st;
  int w_i = 0;
  const auto produce_w = [&](int i_end) {  // weight chunks [w_i, i_end) of this CTA's range
    int i = 0;
    DEC_FOR_SEGMENTS {
      const DecTile dt = dec_tile<NT>(args, groups, t);
      const int nt = dt.nt;
      const int c0 = static_cast<int>(u - static_cast<uint32_t>(t) * kc);
      const int c1 = static_cast<int>(cend - static_cast<uint32_t>(t) * kc);
      for (int c = c0; c < c1; ++c, ++i) {
        if (i < w_i) continue;
        if (i >= i_end) return;
        mbar_wait(bar_emptyw + 8 * w_st.slot, w_st.phase ^ 1u);  // the dequant of chunk i - NW read it
        const int kb0 = c * Cfg::BLOBS;
        const int nb = (KS - kb0) < Cfg::BLOBS ? (KS - kb0) : Cfg::BLOBS;
        const uint32_t fb = bar_fullw + 8 * w_st.slot;
        if (elect_one()) {
          mbar_arrive_expect_tx(fb, nb * 4096);
          bulk_g2s_hint(w0 + w_st.slot * Cfg::W_BYTES,
                        args.packed + (static_cast<size_t>(dt.blob0) + static_cast<size_t>(nt) * KS + kb0) * 4096,
                        nb * 4096, fb, w_policy);
        }
        __syncwarp();
        w_st.advance(NW);
        w_i = i + 1;
      }
    }
  };
  if (warp == Cfg::W_PRODW) {
    constexpr int NBAR = 2 * NW + 3 * NR + DR_MAX + 2 * Cfg::SZ_SLOTS;
    for (int b = static_cast<int>(lane); b < NBAR; b += 32) {
      uint32_t cnt;
      if (b < NW) cnt = 1;                                   // fullw
      else if (b < 2 * NW) cnt = 128;                        // emptyw
      else if (b < 2 * NW + NR) cnt = 1;                     // fulla
      else if (b < 2 * NW + 2 * NR) cnt = 128;               // ready
      else if (b < 2 * NW + 3 * NR) cnt = 1;                 // done
      else if (b < 2 * NW + 3 * NR + DR_MAX) cnt = 128;      // dfree
      else if (b < NBAR - Cfg::SZ_SLOTS) cnt = 1;            // szfull
      else cnt = 128 * NDS + (FS ? 0 : 128);                 // szempty
      mbar_init(bar_fullw + 8 * b, cnt);
    }
    if (push && lane == 0) {  // one arrival (this one) + the ranks' st.async bytes
      mbar_init(bar_red, 1);
      mbar_arrive_expect_tx(bar_red, static_cast<uint32_t>((CS - 1) * 128 * NT * 4));
    }
    fence_mbar_init();
    __syncwarp();
    if (lane == 0) {
      prefetch_tmap(&tmap_a);
      prefetch_tmap(&tmap_s);
      prefetch_tmap(&tmap_z);
    }
    // (requesting all NW first chunks here was measured slower: the setup grew by ~1500 cycles
    // and the first chunk still landed ~5900 cycles after the CTA start -- HBM latency)
    if (TM_EARLY_W > 0) produce_w(TM_EARLY_W);
  }
  if (warp == Cfg::W_MMA) {
    tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // cluster split: every thread arrives now and waits at its end, so the leader's bar_red is
  // initialised before any remote arrive without a cluster-wide stall in the setup
  if (push) cluster_arrive_relaxed();
  bool cl_waited = false;  // push mode: this thread has consumed its setup cluster arrive
  const uint32_t tmem_base = *tmem_slot_ptr;
  // PDL: let the next kernel in the stream start launching now; its CTAs take SMs as ours exit,
  // and it waits (griddepcontrol.wait) before reading anything this kernel writes.
  grid_dependency_launch();
  const uint32_t tmem_a0 = tmem_base;                          // NDS x 4 blobs x 32 columns
  const uint32_t tmem_d0 = tmem_base + NDS * Cfg::BLOBS * 32;  // DR x (256 / g) groups x NT columns

  // ---- segment end (scale warps, or dequant set 0 in FS mode: thread `row` = weight column, et =
  // its index among the 128 finishing threads).  acc = this CTA's sum over the segment's chunks.
  const auto seg_end = [&](float (&acc)[NT], int t, uint32_t u, uint32_t cend, int row, int et) {
    const DecTile dt = dec_tile<NT>(args, groups, t);
    const int nt = dt.nt;
    // ---- segment end.  A CTA's range [u0, u1) meets a shared tile only at its two ends: its
    // first segment may be the tile's tail (or a middle piece), its last segment the tile's
    // head.  The tail is computed first in time (start of the contributor's range), the head
    // last (end of the head holder's range), so the head holder finalises: it waits for the
    // contributors' flags (long set by then), adds their partials in fixed CTA order
    // (deterministic) and stores.  A tail only stores its partial and raises its flag.
    const uint32_t tile_lo = static_cast<uint32_t>(t) * kc;
    const uint32_t tile_hi = tile_lo + kc;
    const int n = nt * 128 + row;
    const int mb = dt.row0;
    const int mcount = dt.mcount;
    if (push) {
      const uint32_t rank = cluster_ctarank();
      cluster_wait();  // pairs the setup arrive: the leader's bar_red is initialised
      cl_waited = true;
      if (rank > 0) {
        // landing area [rank - 1][row][NT]: 4 x 16-byte st.async per thread, counted on the
        // leader's bar_red (a release.cluster arrive here cost ~1000 cycles under HBM load)
        const uint32_t dst = mapa_shared(red0 + ((rank - 1) * 128 + row) * NT * 4, 0);
        const uint32_t rbar = mapa_shared(bar_red, 0);
#pragma unroll
        for (int m = 0; m < NT; m += 4) st_async_v4_f32(dst + m * 4, acc[m], acc[m + 1], acc[m + 2], acc[m + 3], rbar);
      } else {
        mbar_wait_cluster(bar_red, 0);
        const float* red = reinterpret_cast<const float*>(base_ptr + (red0 - base));
        for (int q = 1; q < CS; ++q) {  // rank order: deterministic
          const float4* rq = reinterpret_cast<const float4*>(red + ((q - 1) * 128 + row) * NT);
#pragma unroll
          for (int m = 0; m < NT; m += 4) {
            const float4 v = rq[m / 4];
            acc[m] += v.x;
            acc[m + 1] += v.y;
            acc[m + 2] += v.z;
            acc[m + 3] += v.w;
          }
        }
#pragma unroll
        for (int m = 0; m < NT; ++m)
          if (m < mcount) dec_store<BF16, OUT>(args.out, args.N, mb + m, n, acc[m]);
      }
    } else if (CS > 1) {
      // cluster split: reduced through distributed shared memory after the CTA-wide sync
#pragma unroll
      for (int m = 0; m < NT; ++m) acc_keep[m] = acc[m];
    } else if (u != tile_lo) {
      // tail / middle piece: always this CTA's first segment -> partial slot p, flag p
      float* ws = args.workspace + static_cast<size_t>(p) * NT * 128;
#pragma unroll
      for (int m = 0; m < NT; ++m) __stcg(ws + m * 128 + row, acc[m]);
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (et == 0) st_release_gpu(args.counters + p, 1);  // cumulative over the barrier
    } else {
      if (cend != tile_hi) {
        // head of a shared tile (this CTA's last segment): add the later contributors' partials
        const int p_hi = dec_owner(tile_hi - 1, T, P);
        if (et == 0)
          for (int q = p + 1; q <= p_hi; ++q)
            for (uint32_t spins = 0; ld_acquire_gpu(args.counters + q) == 0;)
              if (++spins == (1u << 24)) __trap();  // a contributor never arrived: fail, do not hang
        asm volatile("bar.sync 1, 128;" ::: "memory");
        for (int q = p + 1; q <= p_hi; ++q) {  // fixed k order: deterministic
          const float* wq = args.workspace + static_cast<size_t>(q) * NT * 128;
#pragma unroll
          for (int m = 0; m < NT; ++m) acc[m] += __ldcg(wq + m * 128 + row);
        }
        if (et == 0)
          for (int q = p + 1; q <= p_hi; ++q) args.counters[q] = 0;  // consumed: zero for the next launch
      }
#pragma unroll
      for (int m = 0; m < NT; ++m)
        if (m < mcount) dec_store<BF16, OUT>(args.out, args.N, mb + m, n, acc[m]);
    }
  };
  if (warp == Cfg::W_PRODW) {
    // ---------------------------------------------------------------- producer W (the rest)
    produce_w(1 << 30);
  } else if (warp == Cfg::W_PRODA) {
    // ---------------------------------------------------------------- producer A (+ s/z boxes)
    RingPos st, prev;
    int i = 0, box = 0;
    bool waited_dep = false;
    DEC_FOR_SEGMENTS {
      const DecTile dt = dec_tile<NT>(args, groups, t);
      const int nt = dt.nt;
      const int c0 = static_cast<int>(u - static_cast<uint32_t>(t) * kc);
      const int c1 = static_cast<int>(cend - static_cast<uint32_t>(t) * kc);
      for (int c = c0; c < c1; ++c, ++i) {
        if (((c - c0) & box_mask) == 0) {  // s/z do not depend on the previous kernel
          const int j = box % Cfg::SZ_SLOTS;
          mbar_wait(bar_szempty + 8 * j, ((box / Cfg::SZ_SLOTS) & 1) ^ 1);
          const uint32_t fb = bar_szfull + 8 * j;
          const int g0 = dt.g0 + ((c * Cfg::CH) >> gshift);
          if (elect_one()) {
            mbar_arrive_expect_tx(fb, 2 * Cfg::SZ_BOX);
            tma_load_2d(sz0 + j * 2 * Cfg::SZ_BOX, &tmap_s, nt * 128, g0, fb);
            tma_load_2d(sz0 + j * 2 * Cfg::SZ_BOX + Cfg::SZ_BOX, &tmap_z, nt * 128, g0, fb);
          }
          __syncwarp();
          ++box;
        }
        if (!waited_dep) {
          grid_dependency_wait();  // activations may come from the previous kernel
          waited_dep = true;
        }
        if (i >= NR) {
          mbar_wait(bar_done + 8 * prev.slot, prev.phase);  // MMA of chunk i - NR read the slot
          prev.advance(NR);
        }
        const uint32_t fb = bar_fulla + 8 * st.slot;
        if (elect_one()) {
          mbar_arrive_expect_tx(fb, Cfg::ACT_BYTES);
          // W8 bit planes: the low planes (k >= K_A) reuse the activations of the high planes
          const int akb = c * Cfg::BLOBS >= args.a_ks ? c * Cfg::BLOBS - args.a_ks : c * Cfg::BLOBS;
          tma_load_3d(a0 + st.slot * Cfg::ACT_BYTES, &tmap_a, 0, dt.row0, akb, fb);
        }
        __syncwarp();
        st.advance(NR);
      }
    }
  } else if (warp == Cfg::W_MMA || warp == Cfg::W_MMA + 1) {
    // ---------------------------------------------------------------- MMA issuers
    // whole warp runs the loop (warp-uniform operands); one elected lane issues.  Issuer j takes
    // chunks i % NISSUE == j (all groups) and so always the D ring entries dr = j (mod NISSUE).
    // (Splitting a chunk's MMAs between both issuers was measured slower: concurrent issuers
    // each slow to ~87 cycles per MMA, i.e. the SM completes one M=128,N=16 MMA per ~44 cycles.)
    const int me = warp - Cfg::W_MMA;
    constexpr uint32_t idesc = umma_idesc_f16(BF16, 128, NT);
    if (me < NISSUE) {
      // per-chunk ring positions by counting (no integer division in the loop)
      int i = 0, ac = 0;
      RingPos rp;
      DEC_FOR_SEGMENTS {
        const int c0 = static_cast<int>(u - static_cast<uint32_t>(t) * kc);
        const int c1 = static_cast<int>(cend - static_cast<uint32_t>(t) * kc);
        for (int c = c0; c < c1; ++c, ++i, rp.advance(NR), ac = (ac + 1 == NDS) ? 0 : ac + 1) {
          if ((i & is_mask) != me) continue;
          const int r = rp.slot;
          const uint32_t rph = rp.phase;
          const int dr = i & dr_mask;
          const int kb0 = c * Cfg::BLOBS;
          const int nb = (KS - kb0) < Cfg::BLOBS ? (KS - kb0) : Cfg::BLOBS;
          const int ng = nb >> bshift;
          const uint32_t act = a0 + r * Cfg::ACT_BYTES;
          mbar_wait(bar_fulla + 8 * r, rph);  // activations in SMEM
          mbar_wait(bar_ready + 8 * r, rph);  // operands in TMEM
          // D slots read (FS: the set's D region is free once the set arrived ready for this chunk)
          if (!FS) mbar_wait(bar_dfree + 8 * dr, ((i >> dr_shift) & 1) ^ 1);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t d_base = tmem_d0 + (FS ? ac : dr) * DSTRIDE;
            const uint32_t a_base = tmem_a0 + ac * Cfg::BLOBS * 32;
            // full chunk: 16 MMAs with compile-time operand offsets (no loop-carried address math)
            const auto issue_full = [&](auto bpg_c) {
              constexpr int BPG = decltype(bpg_c)::value;
              const uint64_t bdesc = umma_desc_sw128(act);
#pragma unroll
              for (int blob = 0; blob < Cfg::BLOBS; ++blob)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  mma_ts(d_base + (blob / BPG) * Cfg::DCOLS, a_base + blob * 32 + 8 * j,
                         bdesc + ((blob * NT * 128) >> 4) + 2 * j, idesc, ((blob % BPG) | j) != 0 ? 1u : 0u);
                }
            };
            if (nb == Cfg::BLOBS && bpg == 2) {
              issue_full(std::integral_constant<int, 2>{});
            } else if (nb == Cfg::BLOBS) {
              issue_full(std::integral_constant<int, 1>{});
            } else {
              for (int g = 0; g < ng; ++g) {  // K tail: partial chunk
                for (int bb = 0; bb < bpg; ++bb) {
                  const int blob = g * bpg + bb;
                  const uint64_t bdesc0 = umma_desc_sw128(act + blob * (NT * 128));
#pragma unroll
                  for (int j = 0; j < 4; ++j)
                    mma_ts(d_base + g * Cfg::DCOLS, a_base + blob * 32 + 8 * j, bdesc0 + 2 * j, idesc,
                           (bb | j) != 0 ? 1u : 0u);
                }
              }
            }
            tc_commit(bar_done + 8 * r);
          }
          __syncwarp();
        }
      }
    }
  } else if (warp >= Cfg::W_DEQ && warp < Cfg::W_DEQ + 4 * NDS) {
    // ---------------------------------------------------------------- dequant (NDS sets)
    const int set = (warp - Cfg::W_DEQ) >> 2;  // takes chunks i % NDS == set, TMEM operand slot `set`
    const int quarter = warp & 3;
    const int row = quarter * 32 + static_cast<int>(lane);
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    const uint32_t a_slot = tmem_a0 + set * Cfg::BLOBS * 32 + lane_off;
    int box = -1, mine = 0, sel = 0;
    RingPos wp, rp, rp_prev;  // weight ring, ready/done ring, and the set's previous chunk's entry
    bool box_ready = false;
    DEC_FOR_SEGMENTS {
      const int c0 = static_cast<int>(u - static_cast<uint32_t>(t) * kc);
      const int c1 = static_cast<int>(cend - static_cast<uint32_t>(t) * kc);
      int g_base = 0;
      float acc[FS ? NT : 1];  // FS: this set's part of the segment's sum
#pragma unroll
      for (int m = 0; m < (FS ? NT : 1); ++m) acc[m] = 0.f;
      for (int c = c0; c < c1; ++c, wp.advance(NW), rp.advance(NR), sel = (sel + 1 == NDS) ? 0 : sel + 1) {
        if (((c - c0) & box_mask) == 0) {
          if (box >= 0) mbar_arrive(bar_szempty + 8 * (box % Cfg::SZ_SLOTS));  // leaving box
          ++box;
          box_ready = false;
          g_base = (c * Cfg::CH) >> gshift;
        }
        if (sel != set) continue;
        if (!box_ready) {  // wait for the box only before a chunk this set owns
          mbar_wait(bar_szfull + 8 * (box % Cfg::SZ_SLOTS), (box / Cfg::SZ_SLOTS) & 1);
          box_ready = true;
        }
        const uint8_t* zs = sz_ptr0 + (box % Cfg::SZ_SLOTS) * 2 * Cfg::SZ_BOX + Cfg::SZ_BOX;
        const int r = rp.slot;
        const int ws = wp.slot;
        const int kb0 = c * Cfg::BLOBS;
        const int nb = (KS - kb0) < Cfg::BLOBS ? (KS - kb0) : Cfg::BLOBS;
        mbar_wait(bar_fullw + 8 * ws, wp.phase);  // the chunk's packed weights landed
        const uint8_t* wst = w_ptr0 + ws * Cfg::W_BYTES + row * 16;
        // zero operands of the chunk's groups (g = 128: 2, g = 64: 4), before the slot wait
        const int gi0 = ((kb0 * 64) >> gshift) - g_base;
        const auto zop = [&](int g) {
          return zero_operand<BF16>(*reinterpret_cast<const uint16_t*>(zs + (gi0 + g) * 256 + row * 2));
        };
        // this set's TMEM slot was last read by the MMA of chunk i - NDS (FS: waited at the end of
        // the set's previous chunk already)
        const auto wait_slot = [&]() {
          if (!FS && mine > 0) mbar_wait(bar_done + 8 * rp_prev.slot, rp_prev.phase);
          tc_fence_after();
        };
        // one blob: 8 LAYOUT v1 words (two LDS.128) -> 32 operand registers -> tcgen05.st x32
        const auto blob_regs = [&](int bb, uint32_t z2, uint32_t (&rr)[32]) {
          const uint4 xa = *reinterpret_cast<const uint4*>(wst + bb * 4096);
          const uint4 xb = *reinterpret_cast<const uint4*>(wst + bb * 4096 + 2048);
          deq_word_int<BF16>(xa.x, z2, rr + 0);
          deq_word_int<BF16>(xa.y, z2, rr + 4);
          deq_word_int<BF16>(xa.z, z2, rr + 8);
          deq_word_int<BF16>(xa.w, z2, rr + 12);
          deq_word_int<BF16>(xb.x, z2, rr + 16);
          deq_word_int<BF16>(xb.y, z2, rr + 20);
          deq_word_int<BF16>(xb.z, z2, rr + 24);
          deq_word_int<BF16>(xb.w, z2, rr + 28);
        };
        const auto blob_st = [&](int bb, const uint32_t (&rr)[32]) { tmem_st_32x32b_x32(a_slot + bb * 32, rr); };
        const auto blob_to_tmem = [&](int bb, uint32_t z2) {
          if (TM_ST_HALF) {
            // two halves (16 k-pairs each): the second half's LDS + math overlaps the first store
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const uint4 x = *reinterpret_cast<const uint4*>(wst + bb * 4096 + h * 2048);
              uint32_t rr[16];
              deq_word_int<BF16>(x.x, z2, rr + 0);
              deq_word_int<BF16>(x.y, z2, rr + 4);
              if (TM_ST_HALF == 2) tmem_st_32x32b_x8(a_slot + bb * 32 + h * 16, rr);
              deq_word_int<BF16>(x.z, z2, rr + 8);
              deq_word_int<BF16>(x.w, z2, rr + 12);
              if (TM_ST_HALF == 2)
                tmem_st_32x32b_x8(a_slot + bb * 32 + h * 16 + 8, rr + 8);
              else
                tmem_st_32x32b_x16(a_slot + bb * 32 + h * 16, rr);
            }
          } else {
            uint32_t rr[32];
            blob_regs(bb, z2, rr);
            blob_st(bb, rr);
          }
        };
        if (nb == Cfg::BLOBS && bpg == 2) {  // full chunk, g = 128 (straight-line)
          const uint32_t z0 = zop(0), z1 = zop(1);
          // the first blob's operands are computed before the slot wait: the set's previous MMA
          // is still completing (measured ~400 cycles of slot wait per owned chunk)
          // (FS: the slot is already free -- the set waited for its previous MMA -- so no early
          // blob: it would only hold 32 more registers live)
          constexpr bool pre = TM_PRE_BLOB && !FS;
          uint32_t r0[32];
          if (pre) blob_regs(0, z0, r0);
          wait_slot();
          if (!pre) blob_regs(0, z0, r0);
          if (TM_ST_HALF) {
            tmem_st_32x32b_x16(a_slot, r0);
            tmem_st_32x32b_x16(a_slot + 16, r0 + 16);
          } else {
            blob_st(0, r0);
          }
          blob_to_tmem(1, z0);
          blob_to_tmem(2, z1);
          blob_to_tmem(3, z1);
        } else if (nb == Cfg::BLOBS) {      // full chunk, g = 64
          wait_slot();
          blob_to_tmem(0, zop(0));
          blob_to_tmem(1, zop(1));
          blob_to_tmem(2, zop(2));
          blob_to_tmem(3, zop(3));
        } else {                            // K tail
          wait_slot();
          for (int bb = 0; bb < nb; ++bb) blob_to_tmem(bb, zop(bb >> bshift));
        }
        rp_prev = rp;
        mbar_arrive(bar_emptyw + 8 * ws);  // all LDS of the chunk's codes have completed
        tc_wait_st();
        tc_fence_before();
        mbar_arrive(bar_ready + 8 * r);
        ++mine;
        if constexpr (FS) {
          // fused scale: once this chunk's MMAs completed, C += s_g * D_g for its groups (the D
          // region and the operand slot are then free for the set's next chunk)
          mbar_wait(bar_done + 8 * r, rp.phase);
          tc_fence_after();
          const uint8_t* ss = zs - Cfg::SZ_BOX;
          const auto scale_of = [&](int g) {
            return __half2float(__ushort_as_half(*reinterpret_cast<const uint16_t*>(ss + (gi0 + g) * 256 + row * 2)));
          };
          const uint32_t d_row = tmem_d0 + set * DSTRIDE + lane_off;
          if constexpr (NT >= 32) {
            const int ng = nb >> 1;  // group 128: 2 blobs per group (K % 128 == 0)
            for (int g = 0; g < ng; ++g) {
              const float sg = scale_of(g);
#pragma unroll
              for (int m0 = 0; m0 < NT; m0 += 16) {  // 16-column loads: acc[NT] is live here
                uint32_t v[16];
                tmem_ld_32x32b_x16(d_row + g * NT + m0, v);
                tc_wait_ld();
#pragma unroll
                for (int j = 0; j < 16; ++j) acc[m0 + j] = fmaf(sg, __uint_as_float(v[j]), acc[m0 + j]);
              }
            }
          } else if (nb == Cfg::BLOBS) {
            uint32_t v[32];
            tmem_ld_32x32b_x32(d_row, v);
            const float s0 = scale_of(0), s1 = scale_of(1);
            tc_wait_ld();
#pragma unroll
            for (int j = 0; j < 32; ++j) acc[j % NT] = fmaf(j < NT ? s0 : s1, __uint_as_float(v[j]), acc[j % NT]);
          } else {  // K tail: one group
            uint32_t v[16];
            tmem_ld_32x32b_x16(d_row, v);
            const float s0 = scale_of(0);
            tc_wait_ld();
#pragma unroll
            for (int j = 0; j < 16; ++j) acc[j] = fmaf(s0, __uint_as_float(v[j]), acc[j]);
          }
          tc_fence_before();
        }
      }
      if constexpr (FS) {
        // segment end (the CTA's only one: FS is cluster split-K): once every set is done with
        // the weight ring, sets 1..NDS-1 deposit their parts there and set 0 adds them in set
        // order (deterministic)
        asm volatile("bar.sync 3, %0;" ::"r"(128 * NDS) : "memory");
        if (set > 0) {
          float* dep = dep_ptr0 + (set - 1) * NT * 128 + row;
#pragma unroll
          for (int m = 0; m < NT; ++m) dep[m * 128] = acc[m];
        }
        asm volatile("bar.sync 4, %0;" ::"r"(128 * NDS) : "memory");
        if (set == 0) {
          for (int q = 1; q < NDS; ++q) {
            const float* dep = dep_ptr0 + (q - 1) * NT * 128 + row;
#pragma unroll
            for (int m = 0; m < NT; ++m) acc[m] += dep[m * 128];
          }
          seg_end(acc, t, u, cend, row, row);
        }
      }
    }
    if (box >= 0) mbar_arrive(bar_szempty + 8 * (box % Cfg::SZ_SLOTS));
  } else if (warp >= Cfg::W_SCALE && warp < Cfg::W_SCALE + 4) {
    // ---------------------------------------------------------------- scale + epilogue
    const int quarter = warp & 3;
    const int row = quarter * 32 + static_cast<int>(lane);
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    const int et = threadIdx.x - Cfg::W_SCALE * 32;  // 0..127
    int ci = 0, box = -1;
    RingPos rps;
    DEC_FOR_SEGMENTS {
      const int c0 = static_cast<int>(u - static_cast<uint32_t>(t) * kc);
      const int c1 = static_cast<int>(cend - static_cast<uint32_t>(t) * kc);
      float acc[NT];
#pragma unroll
      for (int m = 0; m < NT; ++m) acc[m] = 0.f;
      int g_base = 0;
      for (int c = c0; c < c1; ++c) {
        if (((c - c0) & box_mask) == 0) {
          if (box >= 0) mbar_arrive(bar_szempty + 8 * (box % Cfg::SZ_SLOTS));
          ++box;
          mbar_wait(bar_szfull + 8 * (box % Cfg::SZ_SLOTS), (box / Cfg::SZ_SLOTS) & 1);
          g_base = (c * Cfg::CH) >> gshift;
        }
        const uint8_t* ss = sz_ptr0 + (box % Cfg::SZ_SLOTS) * 2 * Cfg::SZ_BOX;
        const int kb0 = c * Cfg::BLOBS;
        const int nb = (KS - kb0) < Cfg::BLOBS ? (KS - kb0) : Cfg::BLOBS;
        const int ng = nb >> bshift;
        const int r = rps.slot;
        const int dr = ci & dr_mask;
        mbar_wait(bar_done + 8 * r, rps.phase);
        tc_fence_after();
        const uint32_t d_row = tmem_d0 + dr * DSTRIDE + lane_off;
        const int gi0 = ((kb0 * 64) >> gshift) - g_base;
        const auto scale_of = [&](int g) {
          return __half2float(__ushort_as_half(*reinterpret_cast<const uint16_t*>(ss + (gi0 + g) * 256 + row * 2)));
        };
        if (NT <= 32 && (ng * NT) % 32 == 0) {
          // whole 32-column loads (NT = 16: two groups per load), one wait per load
          for (int c0 = 0; c0 < ng * NT; c0 += 32) {
            uint32_t v[32];
            tmem_ld_32x32b_x32(d_row + c0, v);
            const float s0 = scale_of(c0 / NT);
            const float s1 = NT == 16 ? scale_of(c0 / NT + 1) : s0;
            tc_wait_ld();
#pragma unroll
            for (int j = 0; j < 32; ++j) acc[j % NT] = fmaf(j < NT ? s0 : s1, __uint_as_float(v[j]), acc[j % NT]);
          }
        } else {
          for (int g = 0; g < ng; ++g) {
            const float sc = scale_of(g);
#pragma unroll
            for (int m0 = 0; m0 < NT; m0 += 16) {
              uint32_t v[16];
              tmem_ld_32x32b_x16(d_row + g * Cfg::DCOLS + m0, v);
              tc_wait_ld();
#pragma unroll
              for (int m = 0; m < 16; ++m) acc[m0 + m] = fmaf(sc, __uint_as_float(v[m]), acc[m0 + m]);
            }
          }
        }
        tc_fence_before();
        mbar_arrive(bar_dfree + 8 * dr);
        ++ci;
        rps.advance(NR);
      }
      seg_end(acc, t, u, cend, row, et);
    }
    if (box >= 0) mbar_arrive(bar_szempty + 8 * (box % Cfg::SZ_SLOTS));
  }

  tc_fence_before();
  __syncthreads();
  if (warp == Cfg::W_MMA) {
    tc_fence_after();
    tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
  if (push) {
    if (!cl_waited) cluster_wait();  // pairs the setup arrive (threads outside the reduction)
  } else if (CS > 1) {
    // ---- cluster split-K reduction (DSMEM): ranks 1..CS-1 write their fp32 partials into the
    // leader's (now idle) weight ring, the leader adds them in rank order (deterministic) and
    // stores.  Barrier 1: every CTA is done with its rings; barrier 2: partials landed.
    const uint32_t rank = cluster_ctarank();
    const bool scale = warp >= Cfg::W_SCALE && warp < Cfg::W_SCALE + 4;
    const int row = (warp & 3) * 32 + static_cast<int>(lane);
    cluster_arrive();
    cluster_wait();
    if (scale && rank > 0) {
      const uint32_t dst = mapa_shared(w0 + ((rank - 1) * NT * 128 + row) * 4, 0);
#pragma unroll
      for (int m = 0; m < NT; ++m) st_cluster_f32(dst + m * 128 * 4, acc_keep[m]);
    }
    cluster_arrive();
    cluster_wait();
    if (scale && rank == 0) {
      const float* red = reinterpret_cast<const float*>(w_ptr0);
      for (int q = 1; q < CS; ++q) {
#pragma unroll
        for (int m = 0; m < NT; ++m) acc_keep[m] += red[(q - 1) * NT * 128 + m * 128 + row];
      }
      const DecTile dt = dec_tile<NT>(args, groups, p / CS);
      const int n = dt.nt * 128 + row;
      const int mb = dt.row0;
      const int mcount = dt.mcount;
#pragma unroll
      for (int m = 0; m < NT; ++m)
        if (m < mcount) dec_store<BF16, OUT>(args.out, args.N, mb + m, n, acc_keep[m]);
    }
  }
}

#undef DEC_FOR_SEGMENTS

}  // namespace w4k
