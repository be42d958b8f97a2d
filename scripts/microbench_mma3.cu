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

template <int N, bool TS, int NACC>
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
    tmem_alloc(tslot, 256);
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
        const uint32_t d = tmem + (j % NACC) * 32;
        if (TS)
          mma_ts(d, tmem + 128 + 8 * j, umma_desc_sw128(b_smem + 32 * j), idesc, r != 0);
        else
          mma_ss(d, umma_desc_sw128(a_smem + 32 * j), umma_desc_sw128(b_smem + 32 * j), idesc, r != 0);
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
    tmem_dealloc(tmem, 256);
  }
}

template <int N, bool TS, int NACC = 1>
void run(int reps, int cps = 1, int M = 128) {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  auto k = kern<N, TS, NACC>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaMalloc(&d, 148 * 4 * 8);
  k<<<148 * cps, 128, 100 * 1024 / cps>>>(reps, d);
  k<<<148 * cps, 128, 100 * 1024 / cps>>>(reps, d);
  cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);  // first 148 CTAs
  double issue = 0, total = 0;
  for (int i = 0; i < 148; ++i) {
    issue += (double)(h[i] & 0xffffffffull);
    total += (double)(h[i] >> 32);
  }
  issue /= 148;
  total /= 148;
  const double n_mma = 4.0 * reps;
  printf("cps=%d %s nacc=%d N=%3d reps=%5d  issue cyc/mma %7.1f  total cyc/mma %7.1f  (floor %5.1f)  %s\n", cps, TS ? "TS" : "SS", NACC, N, reps,
         issue / n_mma, total / n_mma, 128.0 * N / 256.0, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<16, true, 1>(1024, 1);
  run<16, true, 1>(1024, 2);
  run<16, true, 1>(1024, 3);
  run<16, false, 1>(1024, 2);
  run<32, true, 1>(1024, 2);
  return 0;
}
