// MMA issue/execution (16 x M=128,N=16,K=16 TS MMAs + commit + wait per chunk) while other warps
// load the SM: BG=0 idle, 1 ALU (lop3 chains), 2 LDS.128 streams, 3 dequant words + tcgen05.st,
// 4 FMA-pipe (fma.f32 chains).  Isolates what slows the decode kernel's MMA warp.
#include <cuda_runtime.h>
#include <cstdio>
#include "../paper_2508_15601_b200/csrc/gemm_dec.cuh"
using namespace w4k;

template <int BG>
__global__ void __launch_bounds__(512, 1) kern(int chunks, int nbg, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t base = (smem_u32(smem) + 1023) & ~1023u;
  uint8_t* const bptr = smem + (base - smem_u32(smem));
  const uint32_t bar = base, tslot = base + 64, b0 = base + 1024;  // B: 8 KB; LDS source: 64 KB after
  volatile int* stop = reinterpret_cast<volatile int*>(bptr + 128);
  const int warp = __shfl_sync(0xffffffff, threadIdx.x >> 5, 0);
  const uint32_t lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { mbar_init(bar, 1); fence_mbar_init(); *stop = 0; }
  if (warp == 1) { tmem_alloc(tslot, 512); tmem_relinquish(); }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<uint32_t*>(bptr + 64);
  if (warp == 0) {
    constexpr uint32_t idesc = umma_idesc_f16(true, 128, 16);
    uint32_t ph = 0;
    const long long t0 = clock64();
    for (int i = 0; i < chunks; ++i) {
      const uint32_t dbase = tmem + 384 + (i & 1) * 64;
      const uint32_t abase = tmem + (i % 3) * 128;
      if (elect_one()) {
        for (int g = 0; g < 2; ++g)
          for (int bb = 0; bb < 2; ++bb) {
            const int blob = g * 2 + bb;
            const uint64_t bd = umma_desc_sw128(b0 + blob * 2048);
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
    if (threadIdx.x == 0) { out[blockIdx.x] = t1 - t0; *stop = 1; }
  } else if (warp >= 4 && warp < 4 + nbg) {
    const int q = warp & 3;
    long long n = 0;
    const long long t0 = clock64();
    if (BG == 1 || BG == 4) {
      uint32_t v[8];
      for (int j = 0; j < 8; ++j) v[j] = threadIdx.x * 7 + j;
      while (!*stop) {
        for (int it = 0; it < 64; ++it)
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            if (BG == 1) asm volatile("lop3.b32 %0, %0, %1, %2, 0xEA;" : "+r"(v[j]) : "r"(0x000F000Fu), "r"(0x43004300u));
            else asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+r"(v[j]));
          }
        n += 64 * 8;
      }
      if (v[0] == 0x1234567u) out[300] = v[1];
    } else if (BG == 2) {
      uint32_t acc = 0;
      const uint8_t* src = bptr + 1024 + 8192 + (warp - 4) * 4096;
      while (!*stop) {
        for (int it = 0; it < 8; ++it) {
          uint32_t x0, x1, x2, x3;
          asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(x0), "=r"(x1), "=r"(x2), "=r"(x3)
                       : "r"(smem_u32(src + ((it * 512 + lane * 16) & 4095))));
          acc ^= x0 ^ x3;
        }
        n += 8;
      }
      if (acc == 0x1234567u) out[300] = acc;
    } else if (BG == 5 || BG == 6) {
      const uint32_t z2 = zero_operand<true>(0x4000);
      const uint32_t taddr = tmem + 256 + ((uint32_t)(q * 32) << 16);
      uint32_t w = threadIdx.x * 0x9E3779B9u;
      uint32_t acc = 0;
      while (!*stop) {
        uint32_t r[32];
        if (BG == 5) {
#pragma unroll
          for (int j = 0; j < 32; ++j) r[j] = w + j;
          tmem_st_32x32b_x32(taddr, r);
          tc_wait_st();
        } else {
#pragma unroll
          for (int j = 0; j < 8; ++j) deq_word_int<true>(w ^ j, z2, r + 4 * j);
#pragma unroll
          for (int j = 0; j < 32; ++j) acc ^= r[j];
        }
        w += 0x1234567u;
        n += 8;
      }
      if (acc == 0x1234567u) out[300] = acc;
    } else if (BG == 7) {
      const uint32_t taddr = tmem + 448 + ((uint32_t)(q * 32) << 16);
      uint32_t acc = 0;
      while (!*stop) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(taddr, r);
        tc_wait_ld();
#pragma unroll
        for (int j = 0; j < 32; ++j) acc += r[j];
        n += 8;
      }
      if (acc == 0x1234567u) out[300] = acc;
    } else if (BG == 3) {
      const uint32_t z2 = zero_operand<true>(0x4000);
      const uint32_t taddr = tmem + 256 + ((uint32_t)(q * 32) << 16);  // reads of A use cols 0..383 too; harmless
      uint32_t w = threadIdx.x * 0x9E3779B9u;
      while (!*stop) {
        uint32_t r[32];
#pragma unroll
        for (int j = 0; j < 8; ++j) deq_word_int<true>(w ^ j, z2, r + 4 * j);
        tmem_st_32x32b_x32(taddr, r);
        w += 0x1234567u;
        n += 8;
      }
      tc_wait_st();
    }
    const long long t1 = clock64();
    if (lane == 0 && warp == 4) out[148 + blockIdx.x] = n ? (t1 - t0) * 1000 / n : 0;
  }
  tc_fence_before(); __syncthreads();
  if (warp == 1) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int BG> void run(int nbg) {
  unsigned long long* d; cudaMalloc(&d, 400 * 8);
  auto k = kern<BG>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
  const int chunks = 512;
  k<<<148, 512, 128 * 1024>>>(chunks, nbg, d); k<<<148, 512, 128 * 1024>>>(chunks, nbg, d);
  cudaDeviceSynchronize();
  unsigned long long h[400]; cudaMemcpy(h, d, 400 * 8, cudaMemcpyDeviceToHost);
  const char* names[] = {"idle", "ALU lop3", "LDS.128", "dequant+STTM", "FMA", "STTM only", "dequant only", "LDTM"};
  printf("bg %-13s warps %2d: cycles per chunk %.1f  (bg: %.2f cycles per unit per warp)  %s\n", names[BG], nbg,
         (double)h[0] / chunks, h[148] / 1000.0, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}
int main() {
  run<0>(0);
  for (int n : {4, 12}) { run<3>(n); run<5>(n); run<6>(n); run<7>(n); }
  return 0;
}
