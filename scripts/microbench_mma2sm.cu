// Microbenchmark: tcgen05.mma.cta_group::2 kind::f16 (M = 256 across a CTA pair, N = 256, K = 16),
// TS form (A from both CTAs' TMEM) and SS form, issued back to back by the leader's thread.
// MODE (TS only): 0 plain; 1 + a tcgen05.commit per 64-k stage; 2 + commit and a shared-flag
// poll (flag already set) per stage; 3 + commit and an mbarrier test_wait on an already
// completed barrier per stage -- does the issuing thread's per-stage bookkeeping serialise the
// tensor pipe?
#include <cuda_runtime.h>

#include <cstdio>

#include "../paper_2508_15601_b200/csrc/ptx.cuh"
using namespace w4k;

template <bool TS, int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) kern(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t base = (smem_u32(smem) + 1023) & ~1023u;
  const uint32_t bar = base, bar2 = base + 8, bar3 = base + 16, flag = base + 32, tslot = base + 64,
                 a_s = base + 1024, b_s = a_s + 16384;
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = cluster_ctarank();
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init(bar2, 1);
    mbar_init(bar3, 1);
    st_shared_u32(flag, 1u);
    fence_mbar_init();
    mbar_arrive(bar3);  // phase 0 of bar3 completed
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tslot), "r"(512) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_arrive();
  cluster_wait();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(smem + (tslot - smem_u32(smem)));
  if (rank == 0 && threadIdx.x == 0) {
    constexpr uint32_t idesc = umma_idesc_f16(true, 256, 256);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint64_t bd = umma_desc_sw128(b_s + 32 * j);
        if (TS)
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
              "r"(tmem + 256 + 8 * j), "l"(bd), "r"(idesc), "r"((it | j) != 0 ? 1u : 0u)
              : "memory");
        else
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
              "l"(umma_desc_sw128(a_s + 32 * j)), "l"(bd), "r"(idesc), "r"((it | j) != 0 ? 1u : 0u)
              : "memory");
      }
      if (MODE >= 1)
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar2),
                     "h"((uint16_t)1)
                     : "memory");
      if (MODE == 2)
        while (ld_acquire_shared_u32(flag) != 1u) {
        }
      if (MODE == 3) mbar_spin(bar3, 0);
    }
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
                 "h"((uint16_t)1)
                 : "memory");
    mbar_wait(bar, 0);
    out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  cluster_arrive();
  cluster_wait();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
  }
}

template <bool TS, int MODE>
void run(int sms) {
  unsigned long long* d;
  cudaMalloc(&d, sms * 8);
  cudaMemset(d, 0, sms * 8);
  const int smem = 2048 + 16384 + 32768 + 1024;
  cudaFuncSetAttribute(kern<TS, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  kern<TS, MODE><<<sms, 128, smem>>>(64, d);
  kern<TS, MODE><<<sms, 128, smem>>>(4096, d);
  cudaDeviceSynchronize();
  unsigned long long h[256];
  cudaMemcpy(h, d, sms * 8, cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("2SM %s mode %d M=256 N=256: %.1f cycles per 64-k stage (4 MMAs; per-SM floor 512)  %s\n", TS ? "TS" : "SS", MODE, mx / 4096,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<true, 0>(sms);
  run<false, 0>(sms);
  run<true, 1>(sms);
  run<true, 2>(sms);
  run<true, 3>(sms);
  return 0;
}
