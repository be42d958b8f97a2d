/*
 * tm_w4a16.h -- C ABI of libtm_w4a16.so: the B200 (sm_100a) hot path of the
 * TurboMind mixed-precision GEMM pipeline (arXiv 2508.15601, §3.4
 * "GEMM pipeline"): offline low-bit weight packing followed by an
 * online W4A16 GEMM with in-kernel dequantisation.
 *
 * Conventions for every entry point
 *   - All tensor pointers are DEVICE pointers (cudaMalloc / torch CUDA tensors)
 *     owned by the caller; the library keeps no reference after the call returns.
 *     tm_gemm_w4a16_ws takes a caller-owned workspace and allocates nothing.  The
 *     convenience entry points tm_gemm_w4a16 / _f16 / _partial_f32 instead use a
 *     library-owned workspace, one per (device, stream), allocated with cudaMalloc on
 *     the first call that needs it (a decode shape routed to the stream-K kernel) and
 *     kept for the process lifetime; that first call must not be made inside CUDA-graph
 *     capture (it returns TM_ERR_CUDA there).  All other state (TMA descriptors, kernel
 *     attributes, SM counts, occupancy) is host-side and cached per device.
 *   - Weights are read early: packed, scales and zeros may be read before the previous
 *     kernel on `stream` has completed (programmatic dependent launch: the GEMM streams
 *     its first weight chunks while the preceding kernel drains).  They must therefore not
 *     be written by the kernel that immediately precedes the GEMM on its stream; tm_pack_w4
 *     ends with a no-op kernel, so pack -> GEMM on one stream is safe.  Activations are
 *     read only after the previous kernel has completed.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *     Every call only enqueues work on `stream` and returns; the caller keeps the
 *     buffers alive until the stream has completed.
 *   - Errors are returned as tm_status; no exception crosses the ABI.  Arguments are
 *     validated before anything is launched; TM_ERR_CUDA wraps a launch failure.
 *   - Matrices are row-major and dense (leading dimension = row length).
 *   - Shapes (DESIGN.md §4 reading R9): N % 128 == 0, K % 64 == 0, K % group == 0,
 *     group in {64, 128}; M >= 0 is arbitrary and M == 0 is a no-op.
 *   - All tensor pointers must be 16-byte aligned (TMA / bulk-copy requirement).
 *   - Quantisation (readings R1-R4): codes are unsigned 0..15 (only the low nibble
 *     of each input byte is used); W[k][n] = (q[k][n] - z[k/g][n]) * s[k/g][n] with
 *     fp16 scales s and fp16 zeros z stored [K/group][N] row-major, z integer-valued.
 */
#ifndef TM_W4A16_H
#define TM_W4A16_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  TM_OK = 0,
  TM_ERR_INVALID_ARG = -1,       /* null pointer, negative size, descriptor mismatch   */
  TM_ERR_UNSUPPORTED_SHAPE = -2, /* N % 128, K % 64, K % group, group not in {64,128}  */
  TM_ERR_MISALIGNED = -3,        /* a pointer is not 16-byte aligned                   */
  TM_ERR_CUDA = -4,              /* a CUDA call or kernel launch failed                */
  TM_ERR_NO_DEVICE = -5          /* no sm_100 device is current                        */
} tm_status;

/* LAYOUT v1: BN = 128 weight columns per tile, BK = 64 k per stage,
 * one contiguous 4096-byte blob per (n-tile, k-stage), nibble order 0,2,4,6,1,3,5,7
 * inside each 32-bit word.  Realises PAPER.md §4.1 ("hardware-aware weight packing",
 * P:317-326) for the sm_100a data path.                                            */
#define TM_LAYOUT_V1 1u
/* W8 weights as LAYOUT v1 bit planes (tm_pack_w8): the [2K][N] nibble matrix of high planes
 * (rows 0..K-1) then low planes (rows K..2K-1); only tm_gemm_w8a16 accepts it.             */
#define TM_LAYOUT_V1_W8 2u

/* Element types of tm_gemm_w4a16_ws. */
#define TM_DTYPE_BF16 0
#define TM_DTYPE_FP16 1
#define TM_DTYPE_F32 2

/* Host-side descriptor of a packed weight.  `data` is caller-owned device memory of
 * tm_pack_w4_bytes(K, N, group) bytes; tm_pack_w4 fills K, N, group and layout.    */
typedef struct {
  void*    data;   /* in : device buffer, 16-byte aligned                         */
  int64_t  bytes;  /* in : size of `data` in bytes                                 */
  int32_t  K;      /* out: reduction length                                        */
  int32_t  N;      /* out: output columns                                          */
  int32_t  group;  /* out: quantisation group along K (64 or 128)                 */
  uint32_t layout; /* out: TM_LAYOUT_V1                                            */
} tm_packed_w4;

/* Size in bytes of the packed buffer (= K*N/2), or a negative tm_status if the shape
 * is unsupported.                                                                   */
int64_t tm_pack_w4_bytes(int K, int N, int group);

/* Offline packing (§4.1 steps i-iv; §8(a) row a2).
 *   q      : uint8 [K][N], one code per byte (low nibble used)                    (in)
 *   scales : fp16 [K/group][N]                                                    (in)
 *   zeros  : fp16 [K/group][N]                                                    (in)
 *   packed : descriptor; packed->data / packed->bytes set by the caller; on success
 *            K, N, group and layout are filled in                                 (in/out)
 * scales/zeros are validated for null/alignment only and are not read in LAYOUT v1
 * (the GEMM consumes the raw [K/group][N] arrays).  Bit-exact to oracle/layout_v1.  */
tm_status tm_pack_w4(const uint8_t* q, const void* scales, const void* zeros,
                     int K, int N, int group, tm_packed_w4* packed, void* stream);

/* Checkpoint converters (§8(f) NEXT-4; AWQ/GPTQ checkpoints, §5):
 * int4 checkpoints straight into LAYOUT v1 plus the fp16 zero points the GEMM takes; the
 * checkpoint's fp16 scales [K/group][N] are used as they are.  Bit-exact to oracle/formats.py.
 *   tm_pack_awq  : qweight int32 [K][N/8], qzeros int32 [K/group][N/8], nibble i of a word
 *                  holds column 8j + (0,2,4,6,1,3,5,7)[i]
 *   tm_pack_gptq : qweight int32 [K/8][N] (nibble i = row 8kb + i), qzeros int32 [K/group][N/8]
 *                  (nibble i = column 8j + i, stored value = zero - zero_offset; zero_offset 1
 *                  for GPTQ-v1 checkpoints, 0 for v2); no act-order (g_idx[k] = k / group)
 *   packed    : as tm_pack_w4 (caller buffer of K*N/2 bytes; K, N, group, layout filled in)
 *   zeros_out : fp16 [K/group][N] (device, caller-owned)                                   */
tm_status tm_pack_awq(const int32_t* qweight, const int32_t* qzeros, int K, int N, int group,
                      tm_packed_w4* packed, void* zeros_out, void* stream);
tm_status tm_pack_gptq(const int32_t* qweight, const int32_t* qzeros, int K, int N, int group,
                       int zero_offset, tm_packed_w4* packed, void* zeros_out, void* stream);

/* 8-bit weights (W8A16; 4- and 8-bit weights, §2; §8(f) NEXT-4) by bit planes:
 * with q8 = 16 hi + lo and z8 = 16 zh + zl, (q8 - z8) s = (hi - zh)(16 s) + (lo - zl) s exactly,
 * so the W8 weight is packed as the W4 weight of 2K rows (high planes, then low planes) and
 * multiplied by the activations twice along K (R17).
 *   tm_pack_w8_bytes : K * N (K % 256 == 0 besides the W4 shape rules), or a negative status
 *   tm_pack_w8  : q8 uint8 [K][N], scales fp16 [K/group][N], zeros8 fp16 [K/group][N] holding
 *                 integers 0..255 -> packed (descriptor K = 2K, layout TM_LAYOUT_V1_W8),
 *                 scales_out / zeros_out fp16 [2K/group][N] (caller buffers; 16 s must be finite)
 *   tm_gemm_w8a16 : C bf16 [M][N] = A bf16 [M][K] . W8, with the tm_pack_w8 outputs; the
 *                 decode/prefill kernels run over 2K and re-read A for the low planes.     */
int64_t   tm_pack_w8_bytes(int K, int N, int group);
tm_status tm_pack_w8(const uint8_t* q8, const void* scales, const void* zeros8, int K, int N, int group,
                     tm_packed_w4* packed, void* scales_out, void* zeros_out, void* stream);
tm_status tm_gemm_w8a16(const void* A, const tm_packed_w4* packed, const void* scales, const void* zeros,
                        void* C, int M, int N, int K, void* stream);

/* Online W4A16 GEMM (§3.1 steps i-iv P:179-182, §3.4, §4.3 P:420-426;
 * §8(a) rows a3-a10):
 *     C[m][n] = RNE_bf16( sum_k A[m][k] * (q[k][n] - z[k/g][n]) * s[k/g][n] )
 * with fp32 accumulation (the result is tolerance-checked, not bit-exact; R7, R12).
 *   A      : bf16 [M][K]                                                           (in)
 *   packed : descriptor filled by tm_pack_w4 (packed->K == K, packed->N == N)       (in)
 *   scales, zeros : fp16 [K/group][N] (group from the descriptor)                  (in)
 *   C      : bf16 [M][N]                                                           (out)
 * Kernels (chosen on the host from M, N, K; tm_query_gemm_kind in tm_w4a16_debug.h):
 *   M <= 64 : decode kernel (TMEM operand), reading R6b: the tensor-core operand is the
 *             exact integer (q - z) in bf16 and the group scale s is applied in fp32 to the
 *             per-group MMA result (C = sum_g s_g * sum_{k in g} (q - z) A); no weight
 *             rounding.  K is split over a thread-block cluster reduced in distributed shared
 *             memory when the tiles are few, else over a persistent stream-K grid whose
 *             shared tiles are reduced through the workspace (fixed order: deterministic).
 *   M > 64  : prefill kernels, reading R6: weights rounded once to bf16,
 *             RNE_bf16((q - z) * RNE_bf16(s)), before the MMA.  N % 256 == 0: CTA pairs
 *             (tcgen05 cta_group::2; 256 weight columns x 256 tokens per pair) -- unsplit
 *             where the tiles fill the GPU, for 65 <= M <= 512 K split over up to 4 pairs of
 *             one cluster (partials exchanged by bulk DSMEM copies, summed in split order).
 *             Otherwise the single-CTA tiled kernel (128 columns x 128/256 tokens; for
 *             65 <= M <= 512 K may be split over a cluster, DSMEM reduction).  Unsplit, the
 *             two prefill kernels take the same MMA order along K (identical results); a
 *             split changes only the fp32 summation order of the per-split partials.
 * Results are deterministic run to run.  Uses the library-owned workspace (see above).    */
tm_status tm_gemm_w4a16(const void* A, const tm_packed_w4* packed,
                        const void* scales, const void* zeros, void* C,
                        int M, int N, int K, void* stream);

/* Same with fp16 activations and fp16 output (decode: exact (q - z) operand in fp16;
 * prefill: deq = RNE_fp16((q - z) * s)).  Library-owned workspace.              */
tm_status tm_gemm_w4a16_f16(const void* A, const tm_packed_w4* packed,
                            const void* scales, const void* zeros, void* C,
                            int M, int N, int K, void* stream);

/* Row-parallel tensor parallelism (§8(e)): bf16 A, fp32 output C_partial [M][N]
 * (no output rounding), to be summed across ranks (fp32 all-reduce, reading R13)
 * and finalised with tm_tp_finalize.                                                 */
tm_status tm_gemm_w4a16_partial_f32(const void* A, const tm_packed_w4* packed,
                                    const void* scales, const void* zeros, float* C_partial,
                                    int M, int N, int K, void* stream);

/* Workspace for tm_gemm_w4a16_ws: bytes needed for this shape (0 when the chosen kernel needs
 * none), or a negative tm_status for an unsupported shape.                             */
int64_t tm_gemm_workspace_bytes(int M, int N, int K, int group);

/* The same GEMM with explicit element types and a caller-owned workspace (allocates nothing).
 *   a_dtype   : TM_DTYPE_BF16 or TM_DTYPE_FP16 (A)
 *   c_dtype   : a_dtype (rounded output) or TM_DTYPE_F32 (fp32 partial, bf16 A only)
 *   workspace : device buffer of >= tm_gemm_workspace_bytes(M, N, K, group) bytes, 16-byte
 *               aligned, ZERO-FILLED once before its first use; a buffer used by the
 *               register-fed decode path (tm_set_decode_path(2, ...)) must not be shared with
 *               calls that run the other kernels (its partial words must stay zero between launches);
 *               may be NULL (with workspace_bytes 0) when that size is 0.  One workspace
 *               must not be used by two calls that can run concurrently.
 * Errors: TM_ERR_INVALID_ARG for a missing/too small workspace or a dtype pair not listed. */
tm_status tm_gemm_w4a16_ws(const void* A, const tm_packed_w4* packed,
                           const void* scales, const void* zeros, void* C,
                           int M, int N, int K, int a_dtype, int c_dtype,
                           void* workspace, int64_t workspace_bytes, void* stream);

/* Grouped W4A16 GEMM for mixture-of-experts layers (§8(f) NEXT-3; MoE models are evaluated
 * in PAPER.md §5): n_experts independent problems of the same (N, K, group) in ONE
 * launch,  C[r] = A[r] . W_e  for the rows r of expert e.
 *   A            : bf16 [sum_e m_e][K], the tokens routed to expert 0 first, then expert 1, ...
 *   packed       : the experts' LAYOUT v1 weights back to back (expert e at byte offset
 *                  e * K * N / 2; pack each with tm_pack_w4 into its slice), descriptor
 *                  K, N, group of ONE expert, bytes >= n_experts * K * N / 2
 *   scales/zeros : fp16 [n_experts][K/group][N]
 *   C            : bf16 [sum_e m_e][N], rows in the order of A
 *   m_per_expert : HOST array [n_experts] of token counts m_e >= 0 (experts with m_e = 0 get
 *                  no tiles: their weights are not read)
 *   n_experts    : 1 .. 64
 * The decode kernel (reading R6b) runs over the union of the experts' output tiles (cluster
 * split-K or stream-K as for one GEMM, token tile = 16/32/64 from max m_e); deterministic.
 * Library-owned workspace (see above).                                                      */
tm_status tm_gemm_w4a16_grouped(const void* A, const tm_packed_w4* packed,
                                const void* scales, const void* zeros, void* C,
                                const int32_t* m_per_expert, int n_experts, int N, int K,
                                void* stream);

/* Low-bit-KV decode attention (§8(f) NEXT-2; the paper's attention pipeline, §3.4 P:276-280,
 * §4.2, §4.4): one decode step, 8-bit KV cache, head_dim 128,
 *     O[b][h] = sum_t softmax_t(scale Q[b][h] . K[t]) V[t],   t < seq_lens[b],
 *     K[t] = (k_codes[t] - kz[t]) ks[t] (one fp16 (scale, zero) per token and KV head; V alike),
 * KV head h / G serves query head h (grouped-query attention, G = Hq / Hkv in {1, 2, 4, 8}).
 *   Q        : [B][Hq][128] bf16 (q_dtype TM_DTYPE_BF16) or fp16; O : same shape and dtype
 *   k_codes, v_codes : uint8 [B][Hkv][Lmax][128], Lmax % 64 == 0 (cache capacity)
 *   k_sz, v_sz : uint32 [B][Hkv][Lmax], fp16 scale in the low half, fp16 zero in the high half
 *   seq_lens : int32 [B] on the device, 1 <= seq_lens[b] <= Lmax
 *   workspace: tm_attn_workspace_bytes(B, Hq, Hkv, Lmax) bytes (0 when Lmax <= 256: NULL is
 *              fine), zero-filled once before first use, left zeroed; not shared by concurrent calls
 * Deterministic; fp32 softmax and accumulation, one rounding of O (R18).          */
int64_t   tm_attn_workspace_bytes(int B, int Hq, int Hkv, int Lmax);
tm_status tm_attn_decode_kv8(const void* Q, const void* k_codes, const void* v_codes, const void* k_sz,
                             const void* v_sz, const int32_t* seq_lens, void* O, int B, int Hq, int Hkv,
                             int Lmax, float softmax_scale, int q_dtype, void* workspace,
                             int64_t workspace_bytes, void* stream);

/* out_bf16[i] = RNE_bf16(in_f32[i]) for i < count (TP epilogue after the all-reduce). */
tm_status tm_tp_finalize(const float* in_f32, void* out_bf16, int64_t count, void* stream);

/* Fused row-parallel epilogue over symmetric memory (§8(f) NEXT-1):
 * replaces the fp32 all-reduce + tm_tp_finalize pair with one kernel.
 *   out_bf16[i] = RNE_bf16( sum_{r < world} partials[r][i] ),  i < count
 *   partials : host array of `world` device pointers -- rank r's fp32 partial [count] as mapped
 *              in THIS process (a symmetric buffer: entry `rank` is local, the others are peer
 *              memory reachable over NVLink; 16-byte aligned).  Written by each rank's
 *              tm_gemm_w4a16_partial_f32 earlier on its stream.
 *   signals  : host array of `world` device pointers -- rank r's signal pad (uint32 words,
 *              >= TM_TP_SIGNAL_WORDS * world, zero-filled once; used exclusively by this call
 *              while it runs).
 *   multicast: NVLS multicast address of the partial buffers (the switch adds the ranks'
 *              words, multimem.ld_reduce), or NULL: the sum runs over partials[] in rank order
 *              (deterministic, bit-identical on every rank).
 * Every rank of the group must make the matching call (the kernel contains two barriers over
 * the signal pads: entry -- all partials complete; exit -- no rank reuses its partial buffer
 * before every peer has read it).  world in 1..8.  Errors: TM_ERR_INVALID_ARG, TM_ERR_MISALIGNED. */
#define TM_TP_SIGNAL_WORDS 64
tm_status tm_tp_allreduce_finalize(const float* const* partials, uint32_t* const* signals,
                                   const float* multicast, int rank, int world, int64_t count,
                                   void* out_bf16, void* stream);

/* Test / debug entry points ---------------------------------------------------------
 * tm_unpack_w4  : packed -> uint8 [K][N] codes 0..15 (inverse of tm_pack_w4, bit-exact).
 * tm_dequant_w4 : packed + scales + zeros -> W [K][N] in the activation dtype using the
 *                 GEMM's own dequantisation code (bit-exact to oracle/quant.dequant_rounded).
 *                 dtype: 0 = bf16, 1 = fp16.                                          */
tm_status tm_unpack_w4(const tm_packed_w4* packed, uint8_t* q_out, void* stream);
tm_status tm_dequant_w4(const tm_packed_w4* packed, const void* scales, const void* zeros,
                        void* W_out, int dtype, void* stream);

/* Human-readable status; library version string.                                     */
const char* tm_status_string(tm_status status);
const char* tm_version(void);

#ifdef __cplusplus
}
#endif

#endif /* TM_W4A16_H */
