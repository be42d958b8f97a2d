// MMA issue pattern of the decode kernel: per "chunk" 16 MMAs (4 blobs x 4 k-steps) into D slots,
// A rotating over TMEM slots, B over SMEM stages, then commit + mbarrier wait (or not).
#include <cuda_runtime.h>
#include <cstdio>
#include "../paper_2508_15601_b200/csrc/ptx.cuh"
using namespace w4k;
// MODE bit0: commit+wait per chunk; bit1: D at 16-col offsets per group (else 32); bit2: rotate A slot
template <int MODE>
__global__ void __launch_bounds__(128, 1) kern(int chunks, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t base = (smem_u32(smem) + 1023) & ~1023u;
  const uint32_t bar = base, tslot = base + 64, b0 = base + 1024;  // 6 act stages x 8 KB
  const int warp = __shfl_sync(0xffffffff, threadIdx.x >> 5, 0);
  if (threadIdx.x == 0) { mbar_init(bar, 1); fence_mbar_init(); }
  if (warp == 1) { tmem_alloc(tslot, 512); tmem_relinquish(); }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<uint32_t*>(smem + (tslot - smem_u32(smem)));
  if (warp == 0) {
    constexpr uint32_t idesc = umma_idesc_f16(true, 128, 16);
    const long long t0 = clock64();
    uint32_t ph = 0;
    for (int i = 0; i < chunks; ++i) {
      const int ac = (MODE & 4) ? i % 3 : 0;
      const uint32_t act = b0 + (i % 6) * 8192;
      const uint32_t dbase = tmem + 384 + (i & 1) * 64;
      if (elect_one()) {
        for (int g = 0; g < 2; ++g) {
          const uint32_t d = dbase + g * ((MODE & 2) ? 16 : 32);
          for (int bb = 0; bb < 2; ++bb) {
            const int blob = g * 2 + bb;
            const uint32_t a = tmem + (ac * 4 + blob) * 32;
            const uint64_t bd = umma_desc_sw128(act + blob * 2048);
#pragma unroll
            for (int j = 0; j < 4; ++j) mma_ts(d, a + 8 * j, bd + 2 * j, idesc, (bb | j) != 0);
          }
        }
        if (MODE & 1) tc_commit(bar);
      }
      __syncwarp();
      if (MODE & 1) { mbar_wait(bar, ph); ph ^= 1; }
    }
    if (!(MODE & 1)) { if (elect_one()) tc_commit(bar); __syncwarp(); mbar_wait(bar, 0); }
    const long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before(); __syncthreads();
  if (warp == 1) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}
template <int MODE> void run() {
  unsigned long long* d; cudaMalloc(&d, 148 * 8);
  auto k = kern<MODE>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 60 * 1024);
  const int chunks = 512;
  k<<<148, 128, 60 * 1024>>>(chunks, d); k<<<148, 128, 60 * 1024>>>(chunks, d);
  cudaDeviceSynchronize();
  unsigned long long h[148]; cudaMemcpy(h, d, 148 * 8, cudaMemcpyDeviceToHost);
  printf("mode %d (commit/wait=%d d16=%d rotA=%d): cycles per chunk %.1f -> per MMA %.1f  %s\n", MODE, MODE & 1,
         (MODE >> 1) & 1, (MODE >> 2) & 1, (double)h[0] / chunks, (double)h[0] / chunks / 16, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}
int main() { run<0>(); run<1>(); run<2>(); run<3>(); run<4>(); run<5>(); run<7>(); return 0; }
