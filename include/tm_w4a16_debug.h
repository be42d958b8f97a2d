/*
 * tm_w4a16_debug.h -- test and measurement hooks of libtm_w4a16.so (not part of the product
 * ABI in tm_w4a16.h).  The setters change process-global state read at launch time: call
 * them only from single-threaded test or benchmark code, never while another thread issues
 * GEMMs.  Everything here is exported by the same library.
 */
#ifndef TM_W4A16_DEBUG_H
#define TM_W4A16_DEBUG_H

#include "tm_w4a16.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Force a launch configuration.  tile_m in {16,32,64,128,256} (<= 0: automatic).  split_k > 0:
 * tiled kernel with split_k CTAs per tile along K (cluster DSMEM reduction); split_k < 0 (tile_m
 * <= 64): persistent stream-K decode kernel with -split_k CTAs; 0: automatic.                */
tm_status tm_set_gemm_override(int tile_m, int split_k);

/* Launch configuration the next tm_gemm_* call with these sizes would use (split_k < 0: the
 * stream-K kernel's CTA count).                                                             */
tm_status tm_query_gemm_config(int M, int N, int K, int* tile_m, int* split_k, int* grid_ctas);

/* Which kernel that configuration runs: 0 = tiled (prefill; split_k > 1 = CTAs per tile along
 * K in one cluster, chosen for 65 <= M <= 512 while tiles * split_k <= 128), 1 = persistent
 * stream-K decode, 2 = decode with split_k CTAs per tile reduced in distributed shared memory
 * over a thread-block cluster (split_k = 1: one CTA per tile), 3 = register-fed decode
 * (M <= 16; split_k CTAs per tile reduced through the workspace in CTA order), 4 = persistent
 * prefill (opt-in), 5 = prefill on CTA pairs (cta_group::2; grid_ctas CTAs = grid_ctas / 2
 * pairs of 256 weight columns x 256 tokens).                                                 */
tm_status tm_query_gemm_kind(int M, int N, int K, int* kind);

/* Decode kernel for M <= 16: path 0 = automatic (the TMEM decode kernel, kinds 1/2), 1 = the
 * TMEM decode kernel, 2 = the register-fed kernel (kind 3, gemm_rf.cuh).  split in 1..8 forces the
 * register-fed kernel's cluster mode with that many CTAs per tile (capped at the tile's 256-k
 * chunks), split < 0 its stream-K mode with -split CTAs, 0 = automatic.                     */
tm_status tm_set_decode_path(int path, int split);

/* Prefill (M >= 1024, bf16/fp16 output): on != 0 runs the persistent kernel (gemm_pk.cuh: one
 * CTA per SM over 128 x 192 tiles, double-buffered TMEM accumulator, kind 4) instead of the
 * tiled kernel (kind 0) or the pair kernel (kind 5) -- both measured faster on every CFG#2
 * shape.                                                                                     */
tm_status tm_set_prefill_persistent(int on);

/* Prefill on CTA pairs (gemm_2sm.cuh, kind 5, tcgen05 cta_group::2): chosen by default where
 * the tiled kernel would run 256-token tiles without split-K and N % 256 == 0 (bf16/fp16
 * outputs and fp32 partials).  on = 0 restores the tiled kernel (kind 0)
 * there -- A/B measurements and tests; on = 2 additionally runs 17 <= M <= 64 on 64-token
 * pair tiles with split-K (experiment); on = 3 is 1 with 256-token instead of 128-token pair
 * tiles at 65 <= M <= 128 (A/B).  Default 1; other values: TM_ERR_INVALID_ARG.             */
tm_status tm_set_prefill_pair(int on);

/* Decode cluster mode: 0 automatic (default), 1 never (always stream-K), 2..8 force that many
 * CTAs per tile (capped by shared memory and K), -1 one CTA per tile without a split.        */
tm_status tm_set_decode_cluster(int cs);

/* Debug timeline: when buf != NULL the CTAs of the tiled (prefill) kernel write 160 uint32
 * events at buf[cta * 160 + slot] (slot 0 = %globaltimer ns at start, others clock cycles
 * since start) and those of the register-fed decode kernel 64 %globaltimer (ns) events at
 * buf[cta * 64 + slot].  NULL disables tracing (the default).                               */
tm_status tm_set_trace(void* buf, int64_t bytes);

/* The decode kernel's MMA operand for every weight (reading R6b), through the kernel's own
 * dequantisation code: W_out[k][n] = (MAGIC + q) - (MAGIC + z) in bf16 (dtype 0) or fp16
 * (dtype 1) -- exactly q - z for integer zeros.  zeros: fp16 [K/group][N].                  */
tm_status tm_debug_dequant_int(const tm_packed_w4* packed, const void* zeros, void* W_out, int dtype,
                               void* stream);

#ifdef __cplusplus
}
#endif

#endif /* TM_W4A16_DEBUG_H */
