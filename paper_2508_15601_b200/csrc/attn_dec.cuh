// attn_dec.cuh -- low-bit-KV decode attention for sm_100a (§8(f) NEXT-2): the paper's attention
// pipeline (§3.4 "Attention pipeline") for one decode step over an 8-bit KV cache.
//
//   S[t][h] = scale * Q[h] . K[t],  P = softmax_t(S),  O[h] = sum_t P[t][h] V[t]
//   K[t] = (kq[t] - kz[t]) ks[t],   V[t] = (vq[t] - vz[t]) vs[t]   (one (scale, zero) per token, KV head)
//
// Pipeline (one CTA = one (sequence, KV head, token split); 8 consumer + 2 producer warps):
//  * KV loading (§4.4): 64-token macro-tiles of K and V codes stream through a
//    4-stage shared-memory ring by TMA (2-D, SWIZZLE_128B) plus 1-D bulk copies of their (scale,
//    zero) words; two producer warps (K, V) issue them, full/empty mbarriers hand the stages to
//    two consumer groups of 4 warps (tile i -> group i % 2), each warp taking one 16-token
//    micro-tile.  The host sizes the split so the grid holds ~2 CTAs per SM: long contexts are
//    streamed by a few long-lived CTAs instead of many short ones.
//  * Q x K^T on the tensor core with the codes as the operand (§4.2 "adaptive head alignment",
//    Alg. 1): mma.sync m16n8k16, A = 16 tokens x 16 channels of K, B = the
//    G query heads of this KV head (grouped-query attention, G <= 8 = the MMA's N).  A lane loads
//    16 contiguous code bytes of a token row with one LDS.128 and turns each byte pair into the
//    exact fp16 pair (1024 + code) with one PRMT (I2F) -- so, as in the paper, Q is the
//    operand that is rearranged: the B fragment of lane (g, c) for k-slice 4q + r holds
//    Q[h][16(4q + c) + 4r .. +3], matching the K bytes that lane holds.  The zero point and scale
//    are applied after the MMA in fp32:  S = ks (acc - (1024 + kz) sum_d Q[h][d]).
//  * softmax streams over the micro-tiles (running max / sum per head, base 2), P is staged in
//    shared memory scaled by vs, and P x V runs on the FMA pipe: lane l owns channels 4l .. 4l+3
//    of every head; O = sum_t P'[t] (1024 + vq[t]) - sum_t P'[t] (1024 + vz[t]).
//  * the four warps' partial states merge in shared memory; several splits of one sequence merge
//    through a caller workspace (fixed split order, the last split to finish adds them:
//    deterministic).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "ptx.cuh"

namespace w4k {

constexpr int kAttnD = 128;     // head dimension
constexpr int kAttnMT = 64;     // tokens per macro-tile (PAPER Fig. 9)
#ifndef TM_ATTN_TILES
#define TM_ATTN_TILES 4
#endif
constexpr int kAttnTiles = TM_ATTN_TILES;  // macro-tile ring depth (stages)
#ifndef TM_ATTN_WARPS
#define TM_ATTN_WARPS 8
#endif
constexpr int kAttnWarps = TM_ATTN_WARPS;     // 4 or 8: warp w takes micro-tile w % 4 of the macro-tiles
                                              // i = w / 4 (mod kAttnWarps / 4)
constexpr int kAttnThreads = 32 * (kAttnWarps + 2);  // + 2 producer warps (K tiles, V tiles)
// a ring stage is always reused by the same consumer group (tile i -> group i % groups, stage
// i % stages): a group can then never run a full ring lap ahead of the phase it waits for
static_assert(kAttnTiles % (kAttnWarps / 4) == 0, "ring stages must be a multiple of the consumer groups");

struct AttnArgs {
  const uint16_t* q;        // [B][Hq][D] bf16 / fp16
  const uint32_t* ksz;      // [B][Hkv][Lmax] (fp16 scale | fp16 zero << 16)
  const uint32_t* vsz;
  const int* seq_lens;      // [B]
  uint16_t* out;            // [B][Hq][D]
  float* part;              // [B][Hkv][splits][G][D + 2] (m, l, O) partials
  int* counters;            // [B][Hkv], zero between launches
  int B, Hq, Hkv, Lmax, splits;
  int split_tokens;         // tokens per CTA (multiple of 64; host-chosen so the grid fills the GPU)
  float scale_log2;         // softmax scale * log2(e)
};

template <int G>
struct AttnCfg {
  static constexpr int KV_TILE = kAttnMT * kAttnD;          // bytes of one 8-bit macro-tile
  static constexpr int SZ_TILE = kAttnMT * 4;
  static constexpr int STAGE = (2 * KV_TILE + 2 * SZ_TILE + 1023) / 1024 * 1024;  // K, V, K sz, V sz (1 KB aligned: SW128)
  static constexpr int OFF_TILES = 1024;
  static constexpr int OFF_P = OFF_TILES + kAttnTiles * STAGE;          // per warp [16][8] P' + [8] alpha
  static constexpr int P_BYTES = kAttnWarps * (16 * 8 + 8) * 4;
  static constexpr int OFF_MERGE = OFF_P + P_BYTES;                     // per warp [G][D + 3]
  static constexpr int MERGE_BYTES = kAttnWarps * G * (kAttnD + 4) * 4;
  static constexpr int SMEM = OFF_MERGE + MERGE_BYTES + 1024;
};

__device__ __forceinline__ void hmma_f16(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// bytes (b0, b1) of w at positions sel -> fp16 pair (1024 + b0, 1024 + b1), exact
__device__ __forceinline__ uint32_t i2f_pair(uint32_t w, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(w), "r"(0x64646464u), "r"(sel));
  return r;
}

__device__ __forceinline__ float f16lo(uint32_t x) { return __half2float(__ushort_as_half(static_cast<uint16_t>(x))); }
__device__ __forceinline__ float f16hi(uint32_t x) {
  return __half2float(__ushort_as_half(static_cast<uint16_t>(x >> 16)));
}

template <bool BF16>
__device__ __forceinline__ float act_to_float(uint16_t x) {
  if constexpr (BF16)
    return __bfloat162float(__ushort_as_bfloat16(x));
  else
    return __half2float(__ushort_as_half(x));
}

template <int G, bool BF16>
__global__ void __launch_bounds__(kAttnThreads)
    attn_dec_kernel(const __grid_constant__ CUtensorMap tmap_k, const __grid_constant__ CUtensorMap tmap_v,
                    const AttnArgs args) {
  using Cfg = AttnCfg<G>;
  constexpr int D = kAttnD;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* const base_ptr = smem_raw + (base - raw);
  const int split = blockIdx.x, hk = blockIdx.y, b = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // every input (KV cache, Q, seq_lens) may be written by the previous kernel on the stream: no
  // global read before griddepcontrol.wait (PDL lets this grid start before that kernel ends)
  grid_dependency_wait();
  // (clamped to the cache capacity: a bad length must not index past the workspace sized for Lmax)
  const int L = min(args.seq_lens[b], args.Lmax);
  const int t0 = split * args.split_tokens;
  if (t0 >= L) return;  // this split holds no tokens of the sequence
  const int nsplit = (L + args.split_tokens - 1) / args.split_tokens;
  const int ntiles = min(args.split_tokens, L - t0 + kAttnMT - 1) / kAttnMT;
  const long long row0 = (static_cast<long long>(b) * args.Hkv + hk) * args.Lmax + t0;  // cache row of token t0
  const uint32_t bar_full = base, bar_empty = base + 8 * kAttnTiles;  // ring of kAttnTiles macro-tiles

  if (threadIdx.x == 0) {
    for (int i = 0; i < kAttnTiles; ++i) {
      mbar_init(bar_full + 8 * i, 2);   // K producer + V producer
      mbar_init(bar_empty + 8 * i, 4);  // the 4 warps of the tile's consumer group
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp >= kAttnWarps) {
    // ---- producers (§4.4 KV loading pipeline): warp kAttnWarps streams K tiles + K (scale, zero)
    // words, the next warp V; a bulk/TMA request costs its issuing thread ~300 cycles, so the
    // two tensors get separate issuers
    if (lane == 0) {
      const bool isv = warp == kAttnWarps + 1;
      for (int i = 0; i < ntiles; ++i) {
        const int stg = i % kAttnTiles;
        mbar_wait(bar_empty + 8 * stg, ((i / kAttnTiles) & 1) ^ 1);
        const uint32_t st = base + Cfg::OFF_TILES + stg * Cfg::STAGE;
        const uint32_t fb = bar_full + 8 * stg;
        mbar_arrive_expect_tx(fb, Cfg::KV_TILE + Cfg::SZ_TILE);
        const int r = static_cast<int>(row0 + i * kAttnMT);
        tma_load_2d(st + (isv ? Cfg::KV_TILE : 0), isv ? &tmap_v : &tmap_k, 0, r, fb);
        bulk_g2s(st + 2 * Cfg::KV_TILE + (isv ? Cfg::SZ_TILE : 0), (isv ? args.vsz : args.ksz) + row0 + i * kAttnMT,
                 Cfg::SZ_TILE, fb);
      }
    }
    return;
  }

  const int g = lane >> 2, c = lane & 3;
  const int sig = (g >> 1) | ((g & 1) << 2);  // token row of MMA row g (conflict-free LDS.128)
  const int h0 = hk * G;                      // first query head of this KV head
  // ---- Q fragments (the rearrangement): slice 4q + r, lane (g = head, c): Q[g][16(4q + c) + 4r ..]
  uint32_t qf[8][2];
  {
    const uint16_t* qh = args.q + (static_cast<size_t>(b) * args.Hq + h0 + (g < G ? g : 0)) * D;
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int d = 16 * (4 * q + c) + 4 * r;
        float x[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) x[e] = g < G ? act_to_float<BF16>(qh[d + e]) : 0.f;
        const __half2 lo = __floats2half2_rn(x[0], x[1]), hi = __floats2half2_rn(x[2], x[3]);
        qf[4 * q + r][0] = *reinterpret_cast<const uint32_t*>(&lo);
        qf[4 * q + r][1] = *reinterpret_cast<const uint32_t*>(&hi);
      }
  }
  // sum_d Q[h][d] of the fp16 operand, for every head h < G (lane l sums channels 4l .. 4l+3)
  float sq[G];
#pragma unroll
  for (int h = 0; h < G; ++h) {
    const uint16_t* qh = args.q + (static_cast<size_t>(b) * args.Hq + h0 + h) * D + 4 * lane;
    float v = 0.f;
#pragma unroll
    for (int e = 0; e < 4; ++e) v += __half2float(__float2half_rn(act_to_float<BF16>(qh[e])));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    sq[h] = v;
  }
  float sq0 = 0.f, sq1 = 0.f;  // heads 2c, 2c + 1 of this lane (selects: no local-memory indexing)
#pragma unroll
  for (int h = 0; h < G; ++h) {
    sq0 = h == 2 * c ? sq[h] : sq0;
    sq1 = h == 2 * c + 1 ? sq[h] : sq1;
  }

  // ---- per-warp streaming state: heads 2c, 2c + 1 (softmax), channels 4 lane .. +3 (output)
  float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f}, c_run[2] = {0.f, 0.f};
  float o[8][4];  // P.V accumulators, tile 2P + u: (channel row g | g + 8) x (head 2c | 2c + 1)
#pragma unroll
  for (int tt = 0; tt < 8; ++tt)
#pragma unroll
    for (int e = 0; e < 4; ++e) o[tt][e] = 0.f;
  float* const pw = reinterpret_cast<float*>(base_ptr + Cfg::OFF_P) + warp * (16 * 8 + 8);  // P'[16][8], alpha[8]

  const int mtw = warp & 3;  // micro-tile of this warp in each of its macro-tiles
  float al2[2];
  for (int i = warp >> 2; i < ntiles; i += kAttnWarps / 4) {
    const int tm = t0 + i * kAttnMT + 16 * mtw;  // first token of this warp's micro-tile
    const int stg = i % kAttnTiles;
    if (tm >= L) {  // micro-tile past the sequence end (last tile): release the stage only
      if (lane == 0) mbar_arrive(bar_empty + 8 * stg);
      continue;
    }
    mbar_wait(bar_full + 8 * stg, (i / kAttnTiles) & 1);
    const uint8_t* st = base_ptr + Cfg::OFF_TILES + stg * Cfg::STAGE;
    const uint8_t* kt = st;
    const uint8_t* vt = st + Cfg::KV_TILE;
    const uint32_t* kz = reinterpret_cast<const uint32_t*>(st + 2 * Cfg::KV_TILE);
    const uint32_t* vz = kz + kAttnMT;
    // ---- S^T = K . Q^T for 16 tokens x 8 heads
    float acc[4] = {0.f, 0.f, 0.f, 0.f}, acc1[4] = {0.f, 0.f, 0.f, 0.f};  // two MMA chains
    const int ra = 16 * mtw + sig, rb = ra + 8;  // token rows of MMA rows g, g + 8
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int ch = 4 * q + c;  // 16-byte chunk of the row
      const uint4 wa = *reinterpret_cast<const uint4*>(kt + ra * 128 + ((ch ^ (ra & 7)) << 4));
      const uint4 wb = *reinterpret_cast<const uint4*>(kt + rb * 128 + ((ch ^ (rb & 7)) << 4));
      const uint32_t xa[4] = {wa.x, wa.y, wa.z, wa.w}, xb[4] = {wb.x, wb.y, wb.z, wb.w};
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const uint32_t a[4] = {i2f_pair(xa[r], 0x5140), i2f_pair(xb[r], 0x5140), i2f_pair(xa[r], 0x7362),
                               i2f_pair(xb[r], 0x7362)};
        if (q == 0)
          hmma_f16(acc, a, qf[4 * q + r][0], qf[4 * q + r][1]);
        else
          hmma_f16(acc1, a, qf[4 * q + r][0], qf[4 * q + r][1]);
      }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[e] += acc1[e];
    // ---- scores (fold the zero point and scale back in, base-2 units), mask, streaming softmax
    const uint32_t sza = kz[ra], szb = kz[rb];
    const float ksa = f16lo(sza), kza = 1024.f + f16hi(sza), ksb = f16lo(szb), kzb = 1024.f + f16hi(szb);
    const bool va = tm - 16 * mtw + ra < L, vb = tm - 16 * mtw + rb < L;
    float s[4];
    s[0] = va ? ksa * fmaf(-kza, sq0, acc[0]) * args.scale_log2 : -INFINITY;
    s[1] = va ? ksa * fmaf(-kza, sq1, acc[1]) * args.scale_log2 : -INFINITY;
    s[2] = vb ? ksb * fmaf(-kzb, sq0, acc[2]) * args.scale_log2 : -INFINITY;
    s[3] = vb ? ksb * fmaf(-kzb, sq1, acc[3]) * args.scale_log2 : -INFINITY;
    const uint32_t vsa = vz[ra], vsb = vz[rb];
    const float vva = f16lo(vsa), vvb = f16lo(vsb);
    const float vza = 1024.f + f16hi(vsa), vzb = 1024.f + f16hi(vsb);
#pragma unroll
    for (int j = 0; j < 2; ++j) {  // head 2c + j
      float mx = fmaxf(s[j], s[2 + j]);
#pragma unroll
      for (int off = 4; off < 32; off <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
      const float m_new = fmaxf(m_run[j], mx);
      const float alpha = m_new == -INFINITY ? 1.f : exp2f(m_run[j] - m_new);
      const float pa = m_new == -INFINITY ? 0.f : exp2f(s[j] - m_new);
      const float pb = m_new == -INFINITY ? 0.f : exp2f(s[2 + j] - m_new);
      // P' = p vs, rounded once to the fp16 MMA operand; the zero-point term uses the same values
      const __half qa = __float2half_rn(pa * vva), qb = __float2half_rn(pb * vvb);
      float ps = pa + pb;
      float pc = __half2float(qa) * vza + __half2float(qb) * vzb;
#pragma unroll
      for (int off = 4; off < 32; off <<= 1) {
        ps += __shfl_xor_sync(0xffffffffu, ps, off);
        pc += __shfl_xor_sync(0xffffffffu, pc, off);
      }
      m_run[j] = m_new;
      l_run[j] = l_run[j] * alpha + ps;
      c_run[j] = c_run[j] * alpha + pc;
      __half* pt = reinterpret_cast<__half*>(pw);  // P'^T [8 heads][16 tokens] fp16
      pt[(2 * c + j) * 16 + sig] = qa;
      pt[(2 * c + j) * 16 + sig + 8] = qb;
      al2[j] = alpha;
    }
    __syncwarp();
    // ---- O^T += V^T . P' on the tensor core: D[channel][head], A = V codes transposed (16
    // channels x 16 tokens, exact fp16 1024 + code), B = P'^T^T (16 tokens x 8 heads, fp16).
    // Lane (g, c) loads tokens 4c .. 4c + 3 of channels 32 P + 4g .. +3 (one LDS.32 each) and
    // transposes the 4 x 4 bytes with PRMT: channel 32 P + 4g + e feeds row g (e = 0, 2) or row
    // g + 8 (e = 1, 3) of tile 2P + e / 2; k-slots (2c, 2c + 1, 2c + 8, 2c + 9) are tokens
    // 4c .. 4c + 3 in both operands.  Each lane accumulates its heads 2c, 2c + 1.
    {
#pragma unroll
      for (int tt = 0; tt < 8; ++tt) {
        o[tt][0] *= al2[0];
        o[tt][1] *= al2[1];
        o[tt][2] *= al2[0];
        o[tt][3] *= al2[1];
      }
      const uint2 pb2 = *reinterpret_cast<const uint2*>(reinterpret_cast<const __half*>(pw) + g * 16 + 4 * c);
#pragma unroll
      for (int P = 0; P < 4; ++P) {
        const int cb = 32 * P + 4 * g;  // first channel of this lane's 4
        uint32_t r[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int row = 16 * mtw + 4 * c + i;
          r[i] = *reinterpret_cast<const uint32_t*>(vt + row * 128 + (((cb >> 4) ^ (row & 7)) << 4) + (cb & 15));
        }
        uint32_t pr[4][2];  // channel e: fp16 pairs (tokens 4c, 4c+1), (4c+2, 4c+3)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          uint32_t x01, x23;
          asm("prmt.b32 %0, %1, %2, %3;" : "=r"(x01) : "r"(r[0]), "r"(r[1]), "r"(e | ((4 + e) << 4)));
          asm("prmt.b32 %0, %1, %2, %3;" : "=r"(x23) : "r"(r[2]), "r"(r[3]), "r"(e | ((4 + e) << 4)));
          pr[e][0] = i2f_pair(x01, 0x5140);
          pr[e][1] = i2f_pair(x23, 0x5140);
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {  // tile 2P + u: rows g <- channel e = 2u, g + 8 <- e = 2u + 1
          const uint32_t afr[4] = {pr[2 * u][0], pr[2 * u + 1][0], pr[2 * u][1], pr[2 * u + 1][1]};
          hmma_f16(o[2 * P + u], afr, pb2.x, pb2.y);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(bar_empty + 8 * stg);
  }
  // ---- merge the warps: (m, l, O - corr) per head, fixed warp order
  float* mg = reinterpret_cast<float*>(base_ptr + Cfg::OFF_MERGE) + warp * G * (D + 4);
#pragma unroll
  for (int P = 0; P < 4; ++P)
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int j = 0; j < 2; ++j)
        if (2 * c + j < G) {
          const int ch = 32 * P + 4 * g + 2 * u;  // channel of row g; row g + 8 is ch + 1
          mg[(2 * c + j) * (D + 4) + ch] = o[2 * P + u][j] - c_run[j];
          mg[(2 * c + j) * (D + 4) + ch + 1] = o[2 * P + u][2 + j] - c_run[j];
        }
  if (g == 0) {
#pragma unroll
    for (int j = 0; j < 2; ++j)
      if (2 * c + j < G) {
        mg[(2 * c + j) * (D + 4) + D] = m_run[j];
        mg[(2 * c + j) * (D + 4) + D + 1] = l_run[j];
      }
  }
  asm volatile("bar.sync 1, %0;" ::"r"(32 * kAttnWarps) : "memory");  // consumers only
  const float* mall = reinterpret_cast<const float*>(base_ptr + Cfg::OFF_MERGE);
  // thread layout for the output: G heads x 128 channels over 128 threads
  for (int idx = threadIdx.x; idx < G * D; idx += 32 * kAttnWarps) {
    const int h = idx / D, d = idx - (idx / D) * D;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < kAttnWarps; ++w) M = fmaxf(M, mall[(w * G + h) * (D + 4) + D]);
    float Lsum = 0.f, O = 0.f;
#pragma unroll
    for (int w = 0; w < kAttnWarps; ++w) {
      const float mw = mall[(w * G + h) * (D + 4) + D];
      const float f = mw == -INFINITY ? 0.f : exp2f(mw - M);
      Lsum += f * mall[(w * G + h) * (D + 4) + D + 1];
      O += f * mall[(w * G + h) * (D + 4) + d];
    }
    const size_t oidx = (static_cast<size_t>(b) * args.Hq + h0 + h) * D + d;
    if (nsplit == 1) {
      const float y = O / Lsum;
      args.out[oidx] = BF16 ? __bfloat16_as_ushort(__float2bfloat16_rn(y)) : __half_as_ushort(__float2half_rn(y));
    } else {
      float* pp = args.part + ((static_cast<size_t>(b) * args.Hkv + hk) * args.splits + split) * G * (D + 2) + h * (D + 2);
      pp[d] = O;
      if (d == 0) {
        pp[D] = M;
        pp[D + 1] = Lsum;
      }
    }
  }
  if (nsplit == 1) return;
  // ---- split merge: the last split of (b, hk) to finish adds all splits in split order
  __shared__ int last;
  asm volatile("bar.sync 1, %0;" ::"r"(32 * kAttnWarps) : "memory");
  if (threadIdx.x == 0) {
    __threadfence();  // cumulative over the barrier: every consumer's partial stores
    last = atomicAdd(args.counters + b * args.Hkv + hk, 1) == nsplit - 1;
  }
  asm volatile("bar.sync 1, %0;" ::"r"(32 * kAttnWarps) : "memory");
  if (!last) return;
  __threadfence();
  for (int idx = threadIdx.x; idx < G * D; idx += 32 * kAttnWarps) {
    const int h = idx / D, d = idx - (idx / D) * D;
    const float* p0 = args.part + (static_cast<size_t>(b) * args.Hkv + hk) * args.splits * G * (D + 2) + h * (D + 2);
    // all of a thread's loads are issued before they are combined (L2 latency paid once per 8)
    float M = -INFINITY, Lsum = 0.f, O = 0.f;
    for (int s0 = 0; s0 < nsplit; s0 += 8) {
      float ms[8], ls[8], os[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float* ps = p0 + (s0 + j) * G * (D + 2);
        const bool ok = s0 + j < nsplit;
        ms[j] = ok ? __ldcg(ps + D) : -INFINITY;
        ls[j] = ok ? __ldcg(ps + D + 1) : 0.f;
        os[j] = ok ? __ldcg(ps + d) : 0.f;
      }
      float mb = M;
#pragma unroll
      for (int j = 0; j < 8; ++j) mb = fmaxf(mb, ms[j]);
      const float fo = M == -INFINITY ? 0.f : exp2f(M - mb);  // rescale the running sums (split order kept)
      Lsum *= fo;
      O *= fo;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float f = ms[j] == -INFINITY ? 0.f : exp2f(ms[j] - mb);
        Lsum += f * ls[j];
        O += f * os[j];
      }
      M = mb;
    }
    const float y = O / Lsum;
    args.out[(static_cast<size_t>(b) * args.Hq + h0 + h) * D + d] =
        BF16 ? __bfloat16_as_ushort(__float2bfloat16_rn(y)) : __half_as_ushort(__float2half_rn(y));
  }
  if (threadIdx.x == 0) args.counters[b * args.Hkv + hk] = 0;  // zero for the next launch
}

}  // namespace w4k
