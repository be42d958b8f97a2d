// MMA (M=128, N=16, K=16) throughput with concurrent tcgen05.st traffic from other warps.
#include <cuda_runtime.h>
#include <cstdio>
#include "../paper_2508_15601_b200/csrc/ptx.cuh"
using namespace w4k;
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
               :: "r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
// warps: 0 = MMA issuer; 4..4+NST-1 = STTM writers (each x32 into its own 32 columns)
template <bool TS>
__global__ void __launch_bounds__(384, 1) kern(int reps, int nst, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t base = (smem_u32(smem) + 1023) & ~1023u;
  const uint32_t bar = base, tslot = base + 64, a_smem = base + 1024, b_smem = a_smem + 16384;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { mbar_init(bar, 1); fence_mbar_init(); }
  if (warp == 1) { tmem_alloc(tslot, 512); tmem_relinquish(); }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<uint32_t*>(smem + (tslot - smem_u32(smem)));
  volatile __shared__ int stop;
  if (threadIdx.x == 0) stop = 0;
  __syncthreads();
  if (warp == 0) {
    constexpr uint32_t idesc = umma_idesc_f16(true, 128, 16);
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      if (elect_one()) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (TS) mma_ts(tmem, tmem + 128 + 8 * j, umma_desc_sw128(b_smem + 32 * j), idesc, (r | j) != 0);
          else mma_ss(tmem, umma_desc_sw128(a_smem + 32 * j), umma_desc_sw128(b_smem + 32 * j), idesc, (r | j) != 0);
        }
      }
      __syncwarp();
    }
    if (elect_one()) tc_commit(bar);
    __syncwarp();
    mbar_wait(bar, 0);
    const long long t1 = clock64();
    if (threadIdx.x == 0) { out[blockIdx.x] = t1 - t0; stop = 1; }
  } else if (warp >= 4 && warp < 4 + nst) {
    uint32_t r[32];
    for (int j = 0; j < 32; ++j) r[j] = threadIdx.x * 3 + j;
    const uint32_t taddr = tmem + 256 + ((warp - 4) / 4) * 32 + ((uint32_t)((warp & 3) * 32) << 16);
    long long n = 0;
    const long long t0 = clock64();
    while (!stop) { tmem_st_32x32b_x32(taddr, r); ++n; if ((n & 7) == 0) tc_wait_st(); }
    tc_wait_st();
    const long long t1 = clock64();
    if ((threadIdx.x & 31) == 0 && warp == 4) out[148 + blockIdx.x] = (t1 - t0) / (n ? n : 1);
  }
  tc_fence_before(); __syncthreads();
  if (warp == 1) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}
template <bool TS> void run(int nst) {
  unsigned long long* d; cudaMalloc(&d, 400 * 8);
  auto k = kern<TS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const int reps = 2048;
  k<<<148, 384, 64 * 1024>>>(reps, nst, d); k<<<148, 384, 64 * 1024>>>(reps, nst, d);
  cudaDeviceSynchronize();
  unsigned long long h[400]; cudaMemcpy(h, d, 400 * 8, cudaMemcpyDeviceToHost);
  printf("%s  sttm warps %2d: cycles per MMA %.1f  (sttm x32 per warp every %llu cycles)  %s\n", TS ? "TS" : "SS", nst,
         (double)h[0] / (4.0 * reps), nst ? h[148] : 0ull, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}
int main() { for (int n : {0, 4, 8}) { run<true>(n); run<false>(n); } return 0; }
