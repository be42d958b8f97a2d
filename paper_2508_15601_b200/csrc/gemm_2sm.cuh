// gemm_2sm.cuh -- W4A16 prefill GEMM on CTA pairs (tcgen05 cta_group::2), §8(a) rows a3-a10 at
// large M.  Same data path as the tiled kernel (gemm_w4a16.cuh; §3.1 steps i-iv,
// P:179-182; §4.3): each CTA dequantises its own 128 weight columns (reading R6) into
// its TMEM, but the pair shares one 256-token activation tile -- each CTA stages half of it (128
// tokens x 64 k, 16 KB) -- and the pair's leader issues M = 256 MMAs (cta_group::2) that read the
// A operands from both CTAs' TMEM and B from both CTAs' shared memory.  Why: the
// 128 x 256 tiled kernel's stage needs 36 KB of L2->SM ingress per 512 MMA cycles (~70 B/clk
// against a measured ~75-85 B/clk per SM), while one thread issues at most one MMA per ~118
// cycles, so N must stay 256; here each SM ingests 20 KB per stage for the same tensor work.
// Warps: 0 producer W (weights + s/z, local), 1 MMA issuer (leader) + TMEM allocator (both),
// 2-5 and 8-11 dequant (even / odd k-stages) + epilogue, 6 producer A (this CTA's activation
// half, counted on the leader's barrier), 7 stage-ready relay (leader).
// What the measured timeline (scripts/pre_trace.py history, profiles/r02_2sm_trace.log) taught:
//  * a cluster-scope release arrive costs ~1000 cycles under HBM load -> the peer's dequant
//    warps arrive on the leader's barrier with CTA-scope release after tcgen05.wait::st;
//  * the single MMA thread's budget is 512 cycles per stage for 4 MMAs (~75 cycles to issue
//    each) -> one commit per stage (TMEM operand slot), no barrier waits of its own: warp 7
//    waits on the stage barriers and publishes sequence flags the MMA thread polls 4 at a time;
//  * one warp's dequant + TMEM store chain is ~600 cycles per stage -> two dequant sets;
//  * activation loads see ~4000 cycles of latency under load -> an 11-slot activation ring,
//    released by a dequant warp when it observes MMA(i - STAGES) done.
// Mid M (args.split = S > 1): a cluster holds S pairs (rank = 2 split + pair member), split s
// takes stages [s KS / S, (s + 1) KS / S), and the splits exchange partial token slices through
// distributed shared memory (bulk copies) before each stores its slice.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "dequant.cuh"
#include "gemm_w4a16.cuh"
#include "ptx.cuh"

namespace w4k {

template <int NT_>
struct PairCfg {
  static constexpr int NT = NT_;                  // tokens per pair tile (N of the MMA): 256 or 64
  static constexpr int HALF = NT / 2;             // tokens staged per CTA
  static constexpr int STAGES = 8;    // weight + TMEM operand slots (a multiple of 4: go-flag groups)
  static constexpr int ASTAGES = 11;  // activation slots (L2 latency under load ~4000 cycles)
  static constexpr int THREADS = 384;
  static constexpr int ACT_BYTES = HALF * 128;    // 16 KB (NT = 256): 128 tokens x 64 k (SW128)
  static constexpr int HDR = 1024;
  static constexpr int OFF_ACT = HDR;
  static constexpr int OFF_W = OFF_ACT + ASTAGES * ACT_BYTES;
  static constexpr int OFF_SZ = OFF_W + STAGES * kBlobBytes;
  static constexpr int SMEM_USED = 1024 + OFF_SZ + kSZSlots * 2 * kSZBox;
  // one CTA per SM: each allocates all 512 TMEM columns (NT = 64 pads its request past half)
  static constexpr int SMEM = SMEM_USED > 117 * 1024 ? SMEM_USED : 117 * 1024;
  static constexpr int TMEM_COLS = 512;           // accumulator NT + 8 x 32 operand columns
  static_assert(NT + STAGES * 32 <= TMEM_COLS, "TMEM");
  static_assert(ASTAGES * ACT_BYTES >= NT * kBN * 4, "C staging (fp32) fits the drained activation ring");
  // split-K: landing (S - 1 blocks of [128][slice + 4] fp32) + outgoing staging (S - 1 blocks) in
  // the drained activation + weight + s/z rings (contiguous): <= 208 KB at NT = 256, S = 4
  static_assert(ASTAGES * ACT_BYTES + STAGES * kBlobBytes + kSZSlots * 2 * kSZBox >= 2 * 3 * 128 * (NT / 4 + 4) * 4,
                "split-K");
  static_assert(SMEM <= 227 * 1024, "shared memory");
};
using Pair2Cfg = PairCfg<256>;

__device__ __forceinline__ void mma_ts_2sm(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_commit_2sm(uint32_t bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
      "h"(mask)
      : "memory");
}
// 2-D TMA into this CTA's shared memory, transaction bytes counted on the pair leader's mbarrier
// (same offset; the peer bit of the shared::cluster address cleared)
__device__ __forceinline__ void tma_load_2d_2sm(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(bar & 0xFEFFFFFFu)
      : "memory");
}

// debug timeline (tm_set_trace): %globaltimer (ns, low 32 bits) of event `slot` of this CTA --
// 0 start, 1 accumulator complete, 2 split-K cluster barrier, 3 partials sent, 4 landed, 5 end
__device__ __forceinline__ void p2_stamp(const GemmArgs& a, int slot) {
  if (a.trace && threadIdx.x == 64) {
    uint64_t gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    a.trace[(blockIdx.y * gridDim.x + blockIdx.x) * kTraceSlots + slot] = static_cast<uint32_t>(gt);
  }
}

// OUT: OUT_ACT (bf16/fp16 C) or OUT_F32 (fp32 partials for the row-parallel TP reduce; bf16 A)
template <int NT_, bool BF16, int OUT>
__global__ void __launch_bounds__(PairCfg<NT_>::THREADS, 1)
    w4a16_gemm_2sm_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_c,
                          const __grid_constant__ CUtensorMap tmap_s, const __grid_constant__ CUtensorMap tmap_z,
                          const GemmArgs args) {
  using Cfg = PairCfg<NT_>;
  constexpr int NT = Cfg::NT, HALF = Cfg::HALF, STAGES = Cfg::STAGES, ASTAGES = Cfg::ASTAGES;
  constexpr int NCH = NT / 16;  // 16-token chunks of a tile (split-K token slices)
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* const base_ptr = smem_raw + (base - smem_u32(smem_raw));
  // Per stage the leader's MMA thread waits on ONE barrier and commits to ONE (its issue
  // budget is 512 cycles for 4 MMAs; every extra wait or commit costs ~65-100 cycles):
  const uint32_t bar_wfull = base;                       // STAGES: local weights (tx)
  const uint32_t bar_wempty = bar_wfull + 8 * STAGES;    // STAGES: 128 local dequant threads read the blob
  const uint32_t bar_full = bar_wempty + 8 * STAGES;     // STAGES, leader: 8 dequant warps (the leader's
                                                         //   wait for the activation first)
  const uint32_t bar_empty = bar_full + 8 * STAGES;      // STAGES: the leader's commit (TMEM slot free)
  const uint32_t bar_afull = bar_empty + 8 * STAGES;     // ASTAGES, leader: both activation halves (tx)
  const uint32_t bar_aempty = bar_afull + 8 * ASTAGES;   // ASTAGES: MMA(i) done, relayed by a dequant warp
  const uint32_t bar_szfull = bar_aempty + 8 * ASTAGES;  // kSZSlots (tx)
  const uint32_t bar_szempty = bar_szfull + 8 * kSZSlots;  // kSZSlots (128 dequant)
  const uint32_t bar_acc = bar_szempty + 8 * kSZSlots;     // 1: the leader's commit
  const uint32_t tmem_slot = bar_acc + 8;
  uint32_t* const tmem_slot_ptr = reinterpret_cast<uint32_t*>(base_ptr + (tmem_slot - base));
  // STAGES sequence flags (leader): warp 7 waits on bar_full and publishes i + 1 here; the MMA
  // thread polls the flag with a plain shared load -- its own mbarrier waits queue behind its
  // outstanding tcgen05.commit (they returned only when the previous stage's MMAs completed,
  // serialising the tensor pipe; gemm_2sm trace)
  const uint32_t go_flags = tmem_slot + 8;
  // split-K (S > 1): the other splits' partials of this CTA's token slice land here (tx)
  const uint32_t bar_land = go_flags + 4 * Cfg::STAGES;
  static_assert(8 * (6 * Cfg::STAGES + 2 * Cfg::ASTAGES + 2 * kSZSlots + 2) + 8 + 4 * Cfg::STAGES <= Cfg::HDR, "header");
  const uint32_t act0 = base + Cfg::OFF_ACT, w0 = base + Cfg::OFF_W, sz0 = base + Cfg::OFF_SZ;
  const uint8_t* const w_ptr0 = base_ptr + Cfg::OFF_W;
  const uint8_t* const sz_ptr0 = base_ptr + Cfg::OFF_SZ;
  uint8_t* const ring_ptr = base_ptr + Cfg::OFF_ACT;

  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
  const uint32_t lane = threadIdx.x & 31;
  // cluster of 2 S CTAs: rank = 2 sp + pr -- split sp (its K range) of pair member pr (pr = 0:
  // the pair's leader, which issues the MMAs); S = 1 is one pair per cluster
  const int S = args.split;
  p2_stamp(args, 0);
  const uint32_t rank = cluster_ctarank();
  const uint32_t pr = rank & 1u, lead_rank = rank & ~1u;
  const int sp = static_cast<int>(rank >> 1);
  const uint16_t pair_mask = static_cast<uint16_t>(0x3u << lead_rank);  // multicast commits: the pair
  int nt, m0;
  if (S == 1) {
    // banded raster over (n-tile pair, m-tile); CTA (2 j + pr) owns n-tile 2 j + pr
    const int n_pairs = gridDim.x / 2, m_tiles = gridDim.y;
    const int tile = blockIdx.y * n_pairs + static_cast<int>(blockIdx.x >> 1);
    const int band = args.band;
    const int b0 = (tile / (band * n_pairs)) * band;
    const int rows = min(band, m_tiles - b0);
    const int within = tile - b0 * n_pairs;
    nt = 2 * (within / rows) + static_cast<int>(pr);
    m0 = (b0 + within % rows) * NT;
  } else {
    nt = 2 * static_cast<int>(blockIdx.x / (2 * S)) + static_cast<int>(pr);
    m0 = static_cast<int>(blockIdx.y) * NT;
  }
  const int KS_ALL = args.K / kBK;
  const int ks0 = sp * KS_ALL / S;                 // this split's 64-k stages [ks0, ks0 + KS)
  const int KS = (sp + 1) * KS_ALL / S - ks0;
  // split-K token slices: split o finalises 16-token chunks [16 o / S, 16 (o + 1) / S) of the tile
  const int own_lo = NCH * sp / S, own_hi = NCH * (sp + 1) / S;
  const int gshift = args.group == 64 ? 6 : 7;
  // s/z boxes (8 groups each) of this split, ring slots and phases relative to its first box
  const int box0 = ((ks0 * kBK) >> gshift) >> 3;


  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmap_a);
    prefetch_tmap(&tmap_c);
    prefetch_tmap(&tmap_s);
    prefetch_tmap(&tmap_z);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(bar_wfull + 8 * s, 1);
      mbar_init(bar_wempty + 8 * s, 128);
      mbar_init(bar_full + 8 * s, 8);
      mbar_init(bar_empty + 8 * s, 1);
    }
    for (int s = 0; s < ASTAGES; ++s) {
      mbar_init(bar_afull + 8 * s, 1);
      mbar_init(bar_aempty + 8 * s, 1);
    }
    for (int j = 0; j < kSZSlots; ++j) {
      mbar_init(bar_szfull + 8 * j, 1);
      mbar_init(bar_szempty + 8 * j, 256);  // both dequant sets
    }
    mbar_init(bar_acc, 1);
    mbar_init(bar_land, 1);
    if (S > 1)  // (S - 1) senders x one [128 columns][slice tokens + 4] fp32 block each
      mbar_arrive_expect_tx(bar_land, static_cast<uint32_t>((S - 1) * 128 * (16 * (own_hi - own_lo) + 4) * 4));
    for (int s = 0; s < STAGES; ++s) st_shared_u32(go_flags + 4 * s, 0u);
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tmem_slot),
                 "r"(Cfg::TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_arrive();  // both CTAs' barriers and TMEM exist before any cross-CTA traffic
  cluster_wait();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot_ptr;
  const uint32_t tmem_a0 = tmem_base + NT;  // STAGES x 32 operand columns after the accumulator
  grid_dependency_wait();  // A may be the previous kernel's output

  if (warp == 0) {
    // ------------------------------------------------------------ producer W: weights + s/z (local)
    if (lane == 0) {
      const uint8_t* blob_g = args.packed + (static_cast<size_t>(nt) * KS_ALL + ks0) * kBlobBytes;
      int box = -1;
      for (int i = 0; i < KS; ++i) {
        const int s = i % STAGES;
        const int gb = (((ks0 + i) * kBK) >> gshift) >> 3;
        if (gb - box0 != box) {
          box = gb - box0;
          const int j = box % kSZSlots;
          mbar_wait(bar_szempty + 8 * j, ((box / kSZSlots) & 1) ^ 1);
          const uint32_t fb = bar_szfull + 8 * j;
          mbar_arrive_expect_tx(fb, 2 * kSZBox);
          tma_load_2d(sz0 + j * 2 * kSZBox, &tmap_s, nt * kBN, 8 * gb, fb);
          tma_load_2d(sz0 + j * 2 * kSZBox + kSZBox, &tmap_z, nt * kBN, 8 * gb, fb);
        }
        mbar_wait(bar_wempty + 8 * s, ((i / STAGES) & 1) ^ 1);
        const uint32_t fb = bar_wfull + 8 * s;
        mbar_arrive_expect_tx(fb, kBlobBytes);
        bulk_g2s(w0 + s * kBlobBytes, blob_g + static_cast<size_t>(i) * kBlobBytes, kBlobBytes, fb);
      }
    }
    __syncwarp();
  } else if (warp == 6) {
    // ------------------------------------------------------------ producer A: this CTA's half
    if (lane == 0) {
      for (int i = 0; i < KS; ++i) {
        const int s = i % ASTAGES;
        mbar_wait(bar_aempty + 8 * s, ((i / ASTAGES) & 1) ^ 1);
        if (pr == 0) mbar_arrive_expect_tx(bar_afull + 8 * s, 2 * Cfg::ACT_BYTES);  // both halves
        const int g = ks0 + i;
        const int aks = g >= args.a_ks ? g - args.a_ks : g;  // W8: low planes reuse A
        tma_load_2d_2sm(act0 + s * Cfg::ACT_BYTES, &tmap_a, aks * kBK, m0 + static_cast<int>(pr) * HALF,
                        bar_afull + 8 * s);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader CTA only)
    if (pr == 0 && lane == 0) {
      constexpr uint32_t idesc = umma_idesc_f16(BF16, 256, NT);
      for (int i = 0; i < KS; ++i) {
        const int s = i % STAGES;
        if ((i & 3) == 0) {
          // one round trip for 4 stages: a shared load from this thread takes ~220 cycles under
          // the kernel's TMA + operand traffic; stage i + 3's operands never wait on MMA(i)
          // (they need MMA(i + 3 - STAGES) only), so waiting for all four cannot deadlock
          const int n = min(4, KS - i);
          for (;;) {
            uint32_t f[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) f[q] = q < n ? ld_acquire_shared_u32(go_flags + 4 * (s + q)) : 0u;
            bool ok = true;
#pragma unroll
            for (int q = 0; q < 4; ++q) ok = ok && (q >= n || f[q] == static_cast<uint32_t>(i + 1 + q));
            if (ok) break;
          }
        }
        tc_fence_after();
        const uint32_t act = act0 + (i % ASTAGES) * Cfg::ACT_BYTES;
#pragma unroll
        for (int j = 0; j < kBK / 16; ++j)
          mma_ts_2sm(tmem_base, tmem_a0 + s * 32 + 8 * j, umma_desc_sw128(act + 32 * j), idesc, (i | j) != 0 ? 1u : 0u);
        tc_commit_2sm(bar_empty + 8 * s, pair_mask);  // both CTAs: TMEM operand slot (and act slot) free
      }
      tc_commit_2sm(bar_acc, pair_mask);
    }
    __syncwarp();
  } else if (warp == 7) {
    // ------------------------------------------------------------ stage-ready relay (leader)
    if (pr == 0 && lane == 0)
      for (int i = 0; i < KS; ++i) {
        const int s = i % STAGES;
        mbar_spin(bar_full + 8 * s, (i / STAGES) & 1);  // (peer arrivals do not wake a try_wait)
        st_release_shared_u32(go_flags + 4 * s, static_cast<uint32_t>(i + 1));
      }
    __syncwarp();
  } else if ((warp >= 2 && warp < 6) || warp >= 8) {
    // ------------------------------------------------------------ dequant (this CTA's columns)
    // two sets of 4 warps (2-5: even stages, 8-11: odd): one warp's dequant + TMEM store chain
    // is ~600 cycles per stage, above the 512-cycle MMA budget
    const int dset = warp >= 8 ? 1 : 0;
    const bool relay = warp == 2 || warp == 10;  // relays activation-slot release
    const int quarter = warp & 3;
    const int row = quarter * 32 + static_cast<int>(lane);
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    int box = -1;
    for (int i = dset; i < KS; i += 2) {
      const int s = i % STAGES;
      const int gl = ((ks0 + i) * kBK) >> gshift;
      if ((gl >> 3) - box0 != box) {
        if (box >= 0) mbar_arrive(bar_szempty + 8 * (box % kSZSlots));
        // a box this set has no stage of (a split's first box can hold a single stage): release
        // it too, or the producer would wait for its 256 arrivals when it reuses the slot
        for (int k = box + 1; k < (gl >> 3) - box0; ++k) mbar_arrive(bar_szempty + 8 * (k % kSZSlots));
        box = (gl >> 3) - box0;
        mbar_wait(bar_szfull + 8 * (box % kSZSlots), (box / kSZSlots) & 1);
      }
      mbar_wait(bar_wfull + 8 * s, (i / STAGES) & 1);
      const uint8_t* blob = w_ptr0 + s * kBlobBytes;
      const uint4 x0 = *reinterpret_cast<const uint4*>(blob + row * 16);
      const uint4 x1 = *reinterpret_cast<const uint4*>(blob + 2048 + row * 16);
      const uint8_t* szb = sz_ptr0 + (box % kSZSlots) * 2 * kSZBox + ((gl & 7) * kBN + row) * 2;
      const uint16_t sb = *reinterpret_cast<const uint16_t*>(szb);
      const uint16_t zb = *reinterpret_cast<const uint16_t*>(szb + kSZBox);
      mbar_arrive(bar_wempty + 8 * s);
      uint32_t s2, z2;
      deq_prepare<BF16>(sb, zb, s2, z2);
      uint32_t r[32];
      deq_word<BF16>(x0.x, s2, z2, r + 0);
      deq_word<BF16>(x0.y, s2, z2, r + 4);
      deq_word<BF16>(x0.z, s2, z2, r + 8);
      deq_word<BF16>(x0.w, s2, z2, r + 12);
      deq_word<BF16>(x1.x, s2, z2, r + 16);
      deq_word<BF16>(x1.y, s2, z2, r + 20);
      deq_word<BF16>(x1.z, s2, z2, r + 24);
      deq_word<BF16>(x1.w, s2, z2, r + 28);
      mbar_wait(bar_empty + 8 * s, ((i / STAGES) & 1) ^ 1);  // MMA(i - STAGES) done with the slot
      if (relay && lane == 0 && i >= STAGES)  // relay: MMA(i - STAGES)'s activation slot is free
        mbar_arrive(bar_aempty + 8 * ((i - STAGES) % ASTAGES));
      tc_fence_after();
      tmem_st_32x32b_x32(tmem_a0 + s * 32 + lane_off, r);
      tc_wait_st();
      tc_fence_before();
      if (pr == 0) mbar_wait(bar_afull + 8 * (i % ASTAGES), (i / ASTAGES) & 1);  // both halves landed
      __syncwarp();
      if (lane == 0) {  // the leader's barrier
        if (pr == 0)
          mbar_arrive(bar_full + 8 * s);
        else
          mbar_arrive_remote_cta(mapa_shared(bar_full + 8 * s, lead_rank));
      }
    }
    if (box >= 0) mbar_arrive(bar_szempty + 8 * (box % kSZSlots));

    constexpr int ES = OUT == OUT_F32 ? 4 : 2;
    mbar_wait(bar_acc, 0);
    tc_fence_after();
    p2_stamp(args, 1);
    if (S > 1) {
      // ---- split-K reduction over the cluster.  Every CTA of the cluster is past its MMAs
      // (so its activation ring is drained) after this barrier; then each split sends its
      // partial of every other split's token slice into that CTA's ring with st.async (16-byte
      // vectors counted on its bar_land), and finalises its own slice: C = sum_s partial_s in
      // split order (deterministic), stored straight from registers (row = weight column:
      // 128 consecutive outputs per token, coalesced).  Landing layout at split o:
      // [sender slot][column][slice tokens + 4 pad floats] (conflict-free 16-byte reads).
      cluster_arrive();
      cluster_wait();
      p2_stamp(args, 2);
      // stage this CTA's partials of the other slices in its own drained rings (after its
      // landing area), each destination's block in the receiver's layout, then one bulk DSMEM
      // copy per destination (scattered 16-byte st.async ran at ~2K cycles per chunk)
      // slice bounds bnd(k) = 16 k / S (k = 0..S; 16 past S) and staging offsets, computed once
      // (integer divisions by the runtime S in the per-chunk loop cost ~1K cycles per chunk)
      const int b1 = S > 1 ? NCH / S : NCH, b2 = S > 2 ? 2 * NCH / S : NCH, b3 = S > 3 ? 3 * NCH / S : NCH;
      const auto bnd = [&](int k) { return k <= 0 ? 0 : k == 1 ? b1 : k == 2 ? b2 : k == 3 ? b3 : NCH; };
      const uint32_t land_bytes = static_cast<uint32_t>((S - 1) * 128 * (16 * (own_hi - own_lo) + 4) * 4);
      const auto blk = [&](int o) { return static_cast<uint32_t>(128 * (16 * (bnd(o + 1) - bnd(o)) + 4) * 4); };
      const uint32_t off1 = land_bytes + (sp != 0 ? blk(0) : 0u);
      const uint32_t off2 = off1 + (sp != 1 ? blk(1) : 0u);
      const uint32_t off3 = off2 + (sp != 2 ? blk(2) : 0u);
      const auto out_off = [&](int o) { return o <= 0 ? land_bytes : o == 1 ? off1 : o == 2 ? off2 : off3; };
      for (int c = dset; c < NCH; c += 2) {
        // the chunk's owner: bnd(o) <= c < bnd(o + 1) (the same bounds as own_lo/hi)
        const int o = (c >= b1 ? 1 : 0) + (c >= b2 ? 1 : 0) + (c >= b3 ? 1 : 0);
        if (o == sp) continue;
        uint32_t v[16];
        tmem_ld_32x32b_x16(tmem_base + lane_off + 16 * c, v);
        tc_wait_ld();
        const int o_lo = bnd(o), o_hi = bnd(o + 1);
        const int stride = 16 * (o_hi - o_lo) + 4;
        const uint32_t dst = act0 + out_off(o) + static_cast<uint32_t>((row * stride + 16 * (c - o_lo)) * 4);
#pragma unroll
        for (int q = 0; q < 16; q += 4)
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(dst + 4 * q), "r"(v[q]), "r"(v[q + 1]),
                       "r"(v[q + 2]), "r"(v[q + 3])
                       : "memory");
      }
      fence_proxy_async_shared();  // generic-proxy writes -> the bulk copy (async proxy)
      asm volatile("bar.sync 1, 256;" ::: "memory");
      if (threadIdx.x == 64) {
        for (int o = 0; o < S; ++o) {
          if (o == sp) continue;
          const uint32_t bytes = blk(o);
          const uint32_t dst_rank = 2u * static_cast<uint32_t>(o) + pr;
          const int slot = sp < o ? sp : sp - 1;
          bulk_s2cluster(mapa_shared(act0 + static_cast<uint32_t>(slot) * bytes, dst_rank), act0 + out_off(o), bytes,
                         mapa_shared(bar_land, dst_rank));
        }
      }
      // one thread polls (256 spinning threads would compete with the incoming copies for the
      // barrier unit), the other epilogue threads wait on a named barrier
      p2_stamp(args, 3);
      if (threadIdx.x == 64) mbar_spin_cluster(bar_land, 0);  // (remote complete_tx does not wake a try_wait)
      asm volatile("bar.sync 1, 256;" ::: "memory");
      mbar_spin_cluster(bar_land, 0);  // (completed: orders this thread's reads after the bytes)
      p2_stamp(args, 4);
      const int stride = 16 * (own_hi - own_lo) + 4;
      const int n = nt * kBN + row;
#pragma unroll 1
      for (int c = own_lo; c < own_hi; ++c) {
        if ((c & 1) != dset || m0 + 16 * c >= args.M) continue;
        uint32_t v[16];
        tmem_ld_32x32b_x16(tmem_base + lane_off + 16 * c, v);
        tc_wait_ld();
        // partials in split order: x = p_0 + p_1 + ... (own p_sp from TMEM, the others landed)
        float x16[16];
#pragma unroll
        for (int cc = 0; cc < 16; ++cc) x16[cc] = 0.0f;
        for (int t = 0; t < S; ++t) {
          if (t == sp) {
#pragma unroll
            for (int cc = 0; cc < 16; ++cc) x16[cc] += __uint_as_float(v[cc]);
          } else {
            const uint32_t src =
                act0 + static_cast<uint32_t>((((t < sp ? t : t - 1) * 128 + row) * stride + 16 * (c - own_lo)) * 4);
#pragma unroll
            for (int q = 0; q < 16; q += 4) {
              float a0, a1, a2, a3;
              asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                           : "=f"(a0), "=f"(a1), "=f"(a2), "=f"(a3)
                           : "r"(src + 4 * q));
              x16[q] += a0;
              x16[q + 1] += a1;
              x16[q + 2] += a2;
              x16[q + 3] += a3;
            }
          }
        }
#pragma unroll
        for (int cc = 0; cc < 16; ++cc) {
          const float x = x16[cc];
          const int m = m0 + 16 * c + cc;
          if (m < args.M) {
            const size_t off = static_cast<size_t>(m) * args.N + n;
            if constexpr (OUT == OUT_F32)
              reinterpret_cast<float*>(args.out)[off] = x;
            else if constexpr (BF16)
              reinterpret_cast<__nv_bfloat16*>(args.out)[off] = __float2bfloat16_rn(x);
            else
              reinterpret_cast<__half*>(args.out)[off] = __float2half_rn(x);
          }
        }
      }
    } else {
    // epilogue: this CTA's accumulator (128 weight columns x 256 tokens) -> C tile [256][128]
    // staged in the drained activation ring; set d drains tokens [128 d, 128 d + 128)
#pragma unroll 1
    for (int c0 = dset * (NT / 2); c0 < (dset + 1) * (NT / 2); c0 += 16) {
      uint32_t v[16];
      tmem_ld_32x32b_x16(tmem_base + lane_off + c0, v);
      tc_wait_ld();
#pragma unroll
      for (int cc = 0; cc < 16; ++cc) {
        uint8_t* dst = ring_ptr + (static_cast<size_t>(c0 + cc) * kBN + row) * ES;
        const float x = __uint_as_float(v[cc]);
        if constexpr (OUT == OUT_F32)
          *reinterpret_cast<float*>(dst) = x;
        else if constexpr (BF16)
          *reinterpret_cast<__nv_bfloat16*>(dst) = __float2bfloat16_rn(x);
        else
          *reinterpret_cast<__half*>(dst) = __float2half_rn(x);
      }
    }
    fence_proxy_async_shared();
    asm volatile("bar.sync 1, 256;" ::: "memory");
    if (warp == 2 && lane == 0) {
      constexpr int ROWS = ES == 4 && NT > 128 ? 128 : NT;  // the fp32 map's box is <= 128 rows
      for (int r0 = 0; r0 < NT; r0 += ROWS)
        if (m0 + r0 < args.M) tma_store_2d(&tmap_c, act0 + r0 * kBN * ES, nt * kBN, m0 + r0);
      bulk_commit_group();
      bulk_wait_group_read0();
    }
    }
  }
  if (S > 1 && !((warp >= 2 && warp < 6) || warp >= 8)) {
    cluster_arrive();  // the split-K reduction's barrier (every thread of the cluster takes part)
    cluster_wait();
  }
  p2_stamp(args, 5);
  grid_dependency_launch();
  tc_fence_before();
  __syncthreads();
  cluster_arrive();  // the peer is done with our TMEM / barriers before either deallocates
  cluster_wait();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(Cfg::TMEM_COLS)
                 : "memory");
  }
}

}  // namespace w4k
