// tcgen05.st throughput: W warps (4 per lane quarter group) each store x16 / x32 columns of
// 32-bit data in a loop into their own TMEM columns; SM-wide bytes per cycle.  One CTA per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -o scripts/mb_sttm scripts/microbench_sttm.cu
#include <cuda_runtime.h>

#include <cstdio>

#include "../paper_2508_15601_b200/csrc/ptx.cuh"

using namespace w4k;

template <int X>
__global__ void __launch_bounds__(512, 1) kern(int reps, int nwarps, unsigned long long* out) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    tmem_alloc(smem_u32(&slot), 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  uint32_t r[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) r[j] = threadIdx.x * 33 + j;
  __syncthreads();
  const long long t0 = clock64();
  if (warp < nwarps) {
    // warp w: lanes 32*(w%4).., columns 32*(w/4)..  (distinct 32-column block per warp)
    const uint32_t addr = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16) + (warp >> 2) * 32;
    for (int i = 0; i < reps; ++i) {
      if (X == 32) {
        tmem_st_32x32b_x32(addr, r);
      } else {
        tmem_st_32x32b_x16(addr, r);
        tmem_st_32x32b_x16(addr + 16, r + 16);
      }
      r[0] += 1;
    }
    tc_wait_st();
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int X>
void run(int nwarps) {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  const int reps = 2000;
  kern<X><<<148, 512>>>(reps, nwarps, d);
  kern<X><<<148, 512>>>(reps, nwarps, d);
  cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double c = 0;
  for (int i = 0; i < 148; ++i) c += h[i];
  c /= 148;
  const double bytes = 4096.0 * reps * nwarps;  // 32 lanes x 32 columns x 4 B per warp per rep
  printf("x%-2d %2d warps: %.1f B/cycle/SM (%.1f cycles per 4 KB warp-store)  %s\n", X, nwarps, bytes / c,
         c / reps * 1.0, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  for (int w : {1, 4, 8, 12, 16}) {
    run<32>(w);
    run<16>(w);
  }
  return 0;
}
