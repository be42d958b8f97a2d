// Microbenchmark: tcgen05.mma kind::f16 M=128 K=16 rate, TS form (A from TMEM: the prefill and
// decode kernels) vs SS form (A from shared memory), N in {128, 256}.  One CTA per SM, one thread
// issues ITER back-to-back groups of 4 MMAs (one 64-k stage), commit + wait every `per` groups.
#include <cuda_runtime.h>

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

// MODE 0: commit + wait every `per` stages; 1: per stage 2 commits (no wait), like the prefill
// MMA thread; 2: per stage 2 try_waits on completed barriers + fence + 2 commits (the full loop)
template <int N, bool TS, int MODE = 0>
__global__ void __launch_bounds__(128, 1) kern(int iters, int per, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t base = (smem_u32(smem) + 1023) & ~1023u;
  const uint32_t bar = base, tslot = base + 64, a_s = base + 1024, b_s = a_s + 16384;
  const int warp = threadIdx.x >> 5;
  const uint32_t done0 = base + 8, done1 = base + 16, ready = base + 24, empt0 = base + 32, empt1 = base + 40;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init(done0, 1);
    mbar_init(done1, 1);
    mbar_init(ready, 1);
    mbar_init(empt0, 1 << 20);  // never completes: commits just arrive
    mbar_init(empt1, 1 << 20);
    fence_mbar_init();
  }
  if (warp == 1) {
    tmem_alloc(tslot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(smem + (tslot - smem_u32(smem)));
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = umma_idesc_f16(true, 128, N);
    const long long t0 = clock64();
    uint32_t ph = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint64_t bd = umma_desc_sw128(b_s + 32 * j);
        if (TS)
          mma_ts(tmem, tmem + 256 + 8 * j, bd, idesc, (it | j) != 0);
        else
          mma_ss(tmem, umma_desc_sw128(a_s + 32 * j), bd, idesc, (it | j) != 0);
      }
      if (MODE == 0 && (it + 1) % per == 0) {
        tc_commit(bar);
        mbar_wait(bar, ph);
        ph ^= 1;
      } else if (MODE >= 1) {
        tc_commit(empt0);
        tc_commit(empt1);
      }
      if (MODE == 2) {
        mbar_try_wait(done0, 1);  // a fresh barrier: parity 1 completes immediately (like a ready stage)
        mbar_try_wait(done1, 1);
        tc_fence_after();
      }
    }
    tc_commit(bar);
    mbar_wait(bar, ph);
    out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int N, bool TS, int MODE = 0>
void run(int sms, int per) {
  unsigned long long* d;
  cudaMalloc(&d, sms * 8);
  const int smem = 2048 + 16384 + 32768 + 1024;
  cudaFuncSetAttribute(kern<N, TS, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4096;
  kern<N, TS, MODE><<<sms, 128, smem>>>(64, per, d);
  kern<N, TS, MODE><<<sms, 128, smem>>>(iters, per, d);
  cudaDeviceSynchronize();
  unsigned long long h[256];
  cudaMemcpy(h, d, sms * 8, cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("mode %d %s N=%3d commit/wait every %4d stages: %.1f cycles per 64-k stage (4 MMAs; floor %d)  %s\n", MODE, TS ? "TS" : "SS",
         N, per, mx / iters, 4 * 128 * N / 256, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<256, true, 0>(sms, 1000000);
  run<256, true, 1>(sms, 1000000);
  run<256, true, 2>(sms, 1000000);
  return 0;
}
