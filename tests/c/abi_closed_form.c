/* Pure-C consumer of the C ABI (include/tm_w4a16.h): no Python, no torch.  Packs a seeded
 * weight with tm_pack_w4, runs tm_gemm_w4a16 on one-hot activation rows and checks the
 * closed form C[m][n] = RNE_bf16((q[k_m][n] - z) * s) (R6b: one rounding of an
 * exactly representable product), then the error paths.  Exit code 0 = pass.
 *   gcc -O2 -I include abi_closed_form.c -L<lib dir> -ltm_w4a16 -lcudart */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime_api.h>

#include "tm_w4a16.h"

static uint16_t f2h(float f) { /* fp32 -> fp16 RNE, finite normal range only (test values) */
  uint32_t x;
  memcpy(&x, &f, 4);
  const uint32_t sign = (x >> 16) & 0x8000u;
  int e = (int)((x >> 23) & 0xff) - 127 + 15;
  uint32_t m = x & 0x7fffffu;
  if (e <= 0) return (uint16_t)sign; /* not used by the test values */
  uint32_t h = sign | ((uint32_t)e << 10) | (m >> 13);
  const uint32_t rem = m & 0x1fffu;
  if (rem > 0x1000u || (rem == 0x1000u && (h & 1u))) h += 1u;
  return (uint16_t)h;
}
static float h2f(uint16_t h) {
  const uint32_t sign = (uint32_t)(h & 0x8000u) << 16, e = (h >> 10) & 0x1f, m = h & 0x3ffu;
  uint32_t x = e ? (sign | ((e - 15 + 127) << 23) | (m << 13)) : sign;
  float f;
  memcpy(&f, &x, 4);
  return f;
}
static uint16_t f2bf(float f) { /* fp32 -> bf16 RNE */
  uint32_t x;
  memcpy(&x, &f, 4);
  x += 0x7fffu + ((x >> 16) & 1u);
  return (uint16_t)(x >> 16);
}

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e_ = (x);                                                        \
    if (e_ != cudaSuccess) {                                                     \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      return 2;                                                                  \
    }                                                                            \
  } while (0)

int main(void) {
  const int K = 512, N = 256, G = 128, M = 16;
  uint8_t* q = malloc((size_t)K * N);
  uint16_t* s = malloc((size_t)(K / G) * N * 2);
  uint16_t* z = malloc((size_t)(K / G) * N * 2);
  uint16_t* a = calloc((size_t)M * K, 2);
  uint16_t* c = malloc((size_t)M * N * 2);
  uint32_t st = 12345u;
  for (int i = 0; i < K * N; ++i) {
    st = st * 1664525u + 1013904223u;
    q[i] = (uint8_t)(st >> 24); /* high nibble must be ignored */
  }
  for (int i = 0; i < (K / G) * N; ++i) {
    st = st * 1664525u + 1013904223u;
    s[i] = f2h(ldexpf(1.0f + (float)((st >> 9) & 1023u) / 1024.0f, -6)); /* [2^-6, 2^-5) */
    z[i] = f2h((float)((st >> 20) & 15u));
  }
  int km[16];
  for (int m = 0; m < M; ++m) {
    km[m] = (m * 37 + 5) % K; /* row m of A is one-hot at k = km[m] */
    a[(size_t)m * K + km[m]] = 0x3f80u; /* bf16 1.0 */
  }
  void *dq, *ds, *dz, *da, *dc, *dp;
  const int64_t pbytes = tm_pack_w4_bytes(K, N, G);
  if (pbytes != (int64_t)K * N / 2) return fprintf(stderr, "pack bytes %lld\n", (long long)pbytes), 1;
  CK(cudaMalloc(&dq, (size_t)K * N));
  CK(cudaMalloc(&ds, (size_t)(K / G) * N * 2));
  CK(cudaMalloc(&dz, (size_t)(K / G) * N * 2));
  CK(cudaMalloc(&da, (size_t)M * K * 2));
  CK(cudaMalloc(&dc, (size_t)M * N * 2));
  CK(cudaMalloc(&dp, (size_t)pbytes));
  CK(cudaMemcpy(dq, q, (size_t)K * N, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(ds, s, (size_t)(K / G) * N * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dz, z, (size_t)(K / G) * N * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(da, a, (size_t)M * K * 2, cudaMemcpyHostToDevice));
  tm_packed_w4 pk;
  memset(&pk, 0, sizeof(pk));
  pk.data = dp;
  pk.bytes = pbytes;
  int rc = tm_pack_w4(dq, ds, dz, K, N, G, &pk, NULL);
  if (rc != TM_OK || pk.K != K || pk.N != N || pk.group != G || pk.layout != TM_LAYOUT_V1)
    return fprintf(stderr, "pack: %s\n", tm_status_string(rc)), 1;
  rc = tm_gemm_w4a16(da, &pk, ds, dz, dc, M, N, K, NULL);
  if (rc != TM_OK) return fprintf(stderr, "gemm: %s\n", tm_status_string(rc)), 1;
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(c, dc, (size_t)M * N * 2, cudaMemcpyDeviceToHost));
  int bad = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      const int k = km[m], g = k / G;
      const float w = ((float)(q[(size_t)k * N + n] & 15u) - h2f(z[g * N + n])) * h2f(s[g * N + n]); /* exact */
      if (c[(size_t)m * N + n] != f2bf(w) && bad++ < 5)
        fprintf(stderr, "C[%d][%d] = 0x%04x, closed form 0x%04x\n", m, n, c[(size_t)m * N + n], f2bf(w));
    }
  /* error paths: validated before any launch */
  tm_packed_w4 bad_pk = pk;
  bad_pk.K = K + 64;
  const int e1 = tm_gemm_w4a16(da, &bad_pk, ds, dz, dc, M, N, K, NULL);             /* descriptor mismatch */
  const int e2 = tm_gemm_w4a16((char*)da + 2, &pk, ds, dz, dc, M, N, K, NULL);      /* misaligned A        */
  const int e3 = tm_pack_w4(dq, ds, dz, K, 100, G, &pk, NULL);                      /* N % 128 != 0        */
  const int e4 = tm_gemm_w4a16(NULL, &pk, ds, dz, NULL, 0, N, K, NULL);              /* M == 0: no-op       */
  if (e1 != TM_ERR_INVALID_ARG || e2 != TM_ERR_MISALIGNED || e3 != TM_ERR_UNSUPPORTED_SHAPE || e4 != TM_OK) {
    fprintf(stderr, "error paths: %d %d %d %d\n", e1, e2, e3, e4);
    return 1;
  }
  printf("%s: %d mismatches of %d (closed form, bit-exact); error paths ok\n", bad ? "FAIL" : "ok", bad, M * N);
  return bad ? 1 : 0;
}
