/*
 * tm_w4a16.h -- C ABI of libtm_w4a16.so: the B200 (sm_100a) hot path of the
 * TurboMind mixed-precision GEMM pipeline (arXiv 2508.15601, §3.4
 * "GEMM pipeline"): offline low-bit weight packing followed by an
 * online W4A16 GEMM with in-kernel dequantisation.
 *
 * Conventions for every entry point
 *   - All tensor pointers are DEVICE pointers (cudaMalloc / torch CUDA tensors)
 *     owned by the caller; the library keeps no reference after the call returns.
 *     The only device memory the library allocates is the per-stream stream-K
 *     workspace of tm_gemm_* (see below).
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

/* Online W4A16 GEMM (§3.1 steps i-iv P:179-182, §3.4, §4.3 P:420-426;
 * §8(a) rows a3-a10):
 *     C[m][n] = RNE_bf16( sum_k A[m][k] * deq(q[k][n]) )   fp32 accumulation,
 * deq per reading R6 (weights rounded once to bf16 before the tensor-core MMA).
 *   A      : bf16 [M][K]                                                           (in)
 *   packed : descriptor filled by tm_pack_w4 (packed->K == K, packed->N == N)       (in)
 *   scales, zeros : fp16 [K/group][N] (group from the descriptor)                  (in)
 *   C      : bf16 [M][N]                                                           (out)
 * M <= 64 uses a persistent stream-K kernel (one CTA per SM, equal k-chunk ranges);
 * tiles shared by several CTAs are reduced in fixed k order through a library-owned
 * per-stream fp32 workspace (allocated on first use -- do that first call outside CUDA
 * graph capture).  Results are deterministic run to run.                              */
tm_status tm_gemm_w4a16(const void* A, const tm_packed_w4* packed,
                        const void* scales, const void* zeros, void* C,
                        int M, int N, int K, void* stream);

/* Same with fp16 activations and fp16 output; deq = RNE_fp16((q - z) * s). */
tm_status tm_gemm_w4a16_f16(const void* A, const tm_packed_w4* packed,
                            const void* scales, const void* zeros, void* C,
                            int M, int N, int K, void* stream);

/* Row-parallel tensor parallelism (§8(e)): bf16 A, fp32 output C_partial [M][N]
 * (no output rounding), to be summed across ranks (fp32 all-reduce, reading R13)
 * and finalised with tm_tp_finalize.                                                 */
tm_status tm_gemm_w4a16_partial_f32(const void* A, const tm_packed_w4* packed,
                                    const void* scales, const void* zeros, float* C_partial,
                                    int M, int N, int K, void* stream);

/* out_bf16[i] = RNE_bf16(in_f32[i]) for i < count (TP epilogue after the all-reduce). */
tm_status tm_tp_finalize(const float* in_f32, void* out_bf16, int64_t count, void* stream);

/* Test / debug entry points ---------------------------------------------------------
 * tm_unpack_w4  : packed -> uint8 [K][N] codes 0..15 (inverse of tm_pack_w4, bit-exact).
 * tm_dequant_w4 : packed + scales + zeros -> W [K][N] in the activation dtype using the
 *                 GEMM's own dequantisation code (bit-exact to oracle/quant.dequant_rounded).
 *                 dtype: 0 = bf16, 1 = fp16.                                          */
tm_status tm_unpack_w4(const tm_packed_w4* packed, uint8_t* q_out, void* stream);
tm_status tm_dequant_w4(const tm_packed_w4* packed, const void* scales, const void* zeros,
                        void* W_out, int dtype, void* stream);

/* Force a launch configuration (tests / benchmarking only).  tile_m in {16,32,64,128,256}
 * (<= 0: automatic).  split_k > 0: tiled kernel with split_k CTAs per tile along K (cluster
 * DSMEM reduction); split_k < 0: persistent stream-K kernel with -split_k CTAs; 0: automatic
 * (stream-K with one CTA per SM for tile_m <= 64, tiled kernel otherwise).
 * tm_query_gemm_config reports split_k < 0 for the stream-K kernel (its CTA count).      */
tm_status tm_set_gemm_override(int tile_m, int split_k);

/* Launch configuration the next tm_gemm_* call with these sizes would use. */
tm_status tm_query_gemm_config(int M, int N, int K, int* tile_m, int* split_k, int* grid_ctas);

/* Which kernel that configuration runs: 0 = tiled (prefill; split_k > 1 = CTAs per tile along
 * K in one cluster, chosen for 65 <= M <= 512 while tiles * split_k <= 128), 1 = persistent
 * stream-K decode, 2 = decode with split_k CTAs per tile reduced in distributed shared memory
 * over a thread-block cluster (chosen when few output tiles would leave SMs idle; split_k = 1:
 * one CTA per tile, no split, when 70-100 % of the SMs get a whole tile).              */
tm_status tm_query_gemm_kind(int M, int N, int K, int* kind);

/* Decode cluster mode (tests / benchmarking only): 0 automatic (default), 1 never (always
 * stream-K), 2..8 force that many CTAs per tile (capped by shared memory and K), -1 one CTA
 * per tile without a split.                                                            */
tm_status tm_set_decode_cluster(int cs);

/* Debug timeline: when buf != NULL every GEMM CTA writes 160 uint32 events (clock cycles
 * since CTA start; slot 0 = %globaltimer ns) at buf[cta * 160 + slot].  The buffer must
 * hold grid_ctas * 160 * 4 bytes.  NULL disables tracing (the default).               */
tm_status tm_set_trace(void* buf, int64_t bytes);

/* Human-readable status; library version string.                                     */
const char* tm_status_string(tm_status status);
const char* tm_version(void);

#ifdef __cplusplus
}
#endif

#endif /* TM_W4A16_H */
