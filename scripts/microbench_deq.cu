// Microbenchmark: throughput of the decode dequant word sequence (deq_word_int) in registers,
// 1..8 warps per SMSP, with and without tcgen05.st of the results.
#include <cuda_runtime.h>

#include <cstdio>

#include "../paper_2508_15601_b200/csrc/gemm_dec.cuh"

using namespace w4k;

template <int MODE>  // 0: math only (xor-reduce results), 1: math + tcgen05.st x32 per 8 words
__global__ void kern(int iters, unsigned long long* out, uint32_t seed) {
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    tmem_alloc(smem_u32(&tslot), 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot + ((static_cast<uint32_t>(warp & 3) * 32) << 16) + (warp >> 2) * 32;
  uint32_t w[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) w[j] = seed * (threadIdx.x + 1) + j * 0x9E3779B9u;
  uint32_t acc = 0;
  const uint32_t z2 = zero_operand<true>(0x4000);
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t r[32];
#pragma unroll
    for (int j = 0; j < 8; ++j) deq_word_int<true>(w[j] ^ it, z2, r + 4 * j);
    if (MODE == 1) {
      tmem_st_32x32b_x32(tmem, r);
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) acc ^= r[j];
    }
  }
  if (MODE == 1) tc_wait_st();
  const long long t1 = clock64();
  if ((threadIdx.x & 31) == 0) out[blockIdx.x * 32 + warp] = t1 - t0;
  if (acc == 0x12345678u) out[0] = 1;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tslot, 512);
  }
}

template <int MODE>
void run(int warps) {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 32 * 8);
  const int iters = 2048;
  kern<MODE><<<148, 32 * warps>>>(iters, d, 7);
  kern<MODE><<<148, 32 * warps>>>(iters, d, 7);
  cudaDeviceSynchronize();
  unsigned long long h[32];
  cudaMemcpy(h, d, 32 * 8, cudaMemcpyDeviceToHost);
  double c = 0;
  for (int i = 0; i < warps; ++i) c += h[i];
  c /= warps;
  // words per SMSP: warps/4 warps x 8 words per iteration
  const double wps = (warps / 4.0) * 8.0 * iters;
  printf("mode %d warps %2d (%.1f/SMSP): cycles/iter/warp %.1f -> SMSP cycles per word %.2f  %s\n", MODE, warps,
         warps / 4.0, c / iters, c / wps, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  for (int w : {4, 8, 12, 16, 32}) run<0>(w);
  for (int w : {4, 8, 12, 16}) run<1>(w);
  return 0;
}
