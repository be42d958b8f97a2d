// Microbenchmark: tcgen05.mma kind::f16 issue/throughput, M=128, cta_group::1, A from TMEM (TS)
// or SMEM (SS), various N; one elected thread issues R MMAs into one accumulator, then commits.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "../paper_2508_15601_b200/csrc/ptx.cuh"

using namespace w4k;

__device__ __forceinline__ void mma_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(acc)
      : "memory");
}

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) kern(int reps, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t base = (smem_u32(smem) + 1023) & ~1023u;
  const uint32_t bar = base;
  const uint32_t tslot = base + 16;
  const uint32_t a_smem = base + 1024;            // 128 x 64 bf16 (16 KB)
  const uint32_t b_smem = a_smem + 16384;         // N x 64 bf16
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    tmem_alloc(tslot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<uint32_t*>(smem + (tslot - smem_u32(smem)));
  unsigned long long t = 0;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = umma_idesc_f16(true, 128, N);
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (TS)
          mma_ts(tmem, tmem + 256 + 8 * j, umma_desc_sw128(b_smem + 32 * j), idesc, (r | j) != 0);
        else
          mma_ss(tmem, umma_desc_sw128(a_smem + 32 * j), umma_desc_sw128(b_smem + 32 * j), idesc, (r | j) != 0);
      }
    }
    const long long t1 = clock64();
    tc_commit(bar);
    mbar_wait(bar, 0);
    const long long t2 = clock64();
    t = (t1 - t0) | ((unsigned long long)(t2 - t0) << 32);
    out[blockIdx.x] = t;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int N, bool TS>
void run(int reps) {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  auto k = kern<N, TS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  k<<<148, 128, 100 * 1024>>>(reps, d);
  k<<<148, 128, 100 * 1024>>>(reps, d);
  cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double issue = 0, total = 0;
  for (int i = 0; i < 148; ++i) {
    issue += (double)(h[i] & 0xffffffffull);
    total += (double)(h[i] >> 32);
  }
  issue /= 148;
  total /= 148;
  const double n_mma = 4.0 * reps;
  printf("%s N=%3d reps=%5d  issue cyc/mma %7.1f  total cyc/mma %7.1f  (floor %5.1f)  %s\n", TS ? "TS" : "SS", N, reps,
         issue / n_mma, total / n_mma, 128.0 * N / 256.0, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  for (int reps : {4, 64, 1024}) {
    run<16, true>(reps);
    run<16, false>(reps);
    run<32, true>(reps);
    run<64, true>(reps);
    run<64, false>(reps);
    run<128, true>(reps);
    run<256, true>(reps);
    run<256, false>(reps);
  }
  return 0;
}
