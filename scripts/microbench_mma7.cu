// Does mbarrier polling by other warps slow tcgen05.mma?  One MMA warp issues 16-MMA chunks
// (M=128, N=16, K=16, TS) with commit + wait per chunk; NSPIN other warps poll an mbarrier
// (try_wait loop, optionally with a suspend-time hint or nanosleep back-off) that completes at
// the end.
#include <cuda_runtime.h>
#include <cstdio>
#include "../paper_2508_15601_b200/csrc/ptx.cuh"
using namespace w4k;

__device__ __forceinline__ bool try_wait_hint(uint32_t bar, uint32_t parity, uint32_t ns) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity), "r"(ns)
      : "memory");
  return ok != 0;
}

template <int SPIN, int FILL = 0, int BOFF = 0>  // BOFF: B operand offset in KB; FILL: 0 leave TMEM/SMEM as found, 1 zeros, 2 random bf16 in [-8, 8]; 0 plain try_wait, 1 try_wait with 1 us suspend hint, 2 nanosleep(64) back-off
__global__ void __launch_bounds__(1024, 1) kern(int chunks, int nspin, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t base = (smem_u32(smem) + 1023) & ~1023u;
  uint8_t* const bptr = smem + (base - smem_u32(smem));
  const uint32_t bar = base, endbar = base + 8, tslot = base + 64, b0 = base + 1024 + BOFF * 1024;
  const int warp = __shfl_sync(0xffffffff, threadIdx.x >> 5, 0);
  if (threadIdx.x == 0) { mbar_init(bar, 1); mbar_init(endbar, 1); fence_mbar_init(); }
  if (warp == 1) { tmem_alloc(tslot, 512); tmem_relinquish(); }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<uint32_t*>(bptr + 64);
  if (FILL) {
    // SMEM B region (6 x 8 KB) and TMEM columns 0..511 of all 128 lanes
    uint32_t h = threadIdx.x * 0x9E3779B9u + 12345u;
    auto rnd = [&]() {
      h ^= h << 13; h ^= h >> 17; h ^= h << 5;
      if (FILL == 1) return 0u;
      const uint32_t lo = 0x4000u | ((h & 0x7F)) | ((h >> 7) & 1) << 15;   // +-[2, 4)
      const uint32_t hi = 0x3F80u | ((h >> 8) & 0x7F) | ((h >> 15) & 1) << 15;  // +-[1, 2)
      return lo | (hi << 16);
    };
    uint32_t* bw = reinterpret_cast<uint32_t*>(bptr + 1024);
    for (int k = threadIdx.x; k < 6 * 8192 / 4; k += blockDim.x) bw[k] = rnd();
    if (warp < 4) {
      for (int c0 = 0; c0 < 512; c0 += 32) {
        uint32_t r[32];
        for (int j = 0; j < 32; ++j) r[j] = rnd();
        tmem_st_32x32b_x32(tmem + c0 + ((uint32_t)(warp * 32) << 16), r);
      }
      tc_wait_st();
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before(); __syncthreads(); tc_fence_after();
  }
  if (warp == 0) {
    constexpr uint32_t idesc = umma_idesc_f16(true, 128, 16);
    uint32_t ph = 0;
    const long long t0 = clock64();
    for (int i = 0; i < chunks; ++i) {
      const uint32_t dbase = tmem + 384 + (i & 3) * 32;
      const uint32_t abase = tmem + (i % 3) * 128;
      if (elect_one()) {
        for (int g = 0; g < 2; ++g)
          for (int bb = 0; bb < 2; ++bb) {
            const int blob = g * 2 + bb;
            const uint64_t bd = umma_desc_sw128(b0 + (i % 6) * 8192 + blob * 2048);
#pragma unroll
            for (int j = 0; j < 4; ++j) mma_ts(dbase + g * 16, abase + blob * 32 + 8 * j, bd + 2 * j, idesc, (bb | j) != 0);
          }
        tc_commit(bar);
      }
      __syncwarp();
      mbar_wait(bar, ph);
      ph ^= 1;
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) { out[blockIdx.x] = t1 - t0; mbar_arrive(endbar); }
  } else if (warp >= 2 && warp < 2 + nspin) {
    if (SPIN == 0) { while (!mbar_try_wait(endbar, 0)) {} }
    if (SPIN == 1) { while (!try_wait_hint(endbar, 0, 1000)) {} }
    if (SPIN == 2) { while (!mbar_try_wait(endbar, 0)) __nanosleep(64); }
  }
  tc_fence_before(); __syncthreads();
  if (warp == 1) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int SPIN, int FILL = 0, int BOFF = 0> void run(int nspin, int smem_kb = 64) {
  unsigned long long* d; cudaMalloc(&d, 400 * 8);
  auto k = kern<SPIN, FILL, BOFF>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_kb * 1024);
  const int chunks = 512;
  k<<<148, 32 * (2 + nspin), smem_kb * 1024>>>(chunks, nspin, d); k<<<148, 32 * (2 + nspin), smem_kb * 1024>>>(chunks, nspin, d);
  cudaDeviceSynchronize();
  unsigned long long h[400]; cudaMemcpy(h, d, 400 * 8, cudaMemcpyDeviceToHost);
  const char* names[] = {"try_wait", "try_wait+hint", "nanosleep"};
  printf("boff %3d smem %3d fill %d spin %-14s warps %2d: cycles per 16-MMA chunk %.1f  %s\n", BOFF, smem_kb, FILL, names[SPIN], nspin, (double)h[0] / chunks,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}
int main() {
  run<0, 2>(4); run<0, 2>(18, 200); run<0, 2, 132>(4, 200); run<0, 2, 132>(18, 200); run<0, 2, 150>(18, 210);
  return 0;
}
