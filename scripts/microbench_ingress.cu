// Microbenchmark: per-SM ingress bandwidth L2 -> shared memory with 1-D bulk copies (the prefill
// kernel's stage loads come from L2: activations are reused across n-tiles).  One CTA per SM,
// one producer lane, an NST-slot ring of CH-byte chunks, consumers free a slot as soon as it
// lands; the source is an L2-resident buffer of `src_mb` MB read round-robin.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

template <int NST, int CH>
__global__ void __launch_bounds__(64) ingress(const uint8_t* src, long long src_bytes, int iters, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const uint32_t base = (smem_u32(sm) + 1023u) & ~1023u;
  const uint32_t full = base, empty = base + 8 * NST, ring = base + 1024;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x < NST) {
    mbar_init(full + 8 * threadIdx.x, 1);
    mbar_init(empty + 8 * threadIdx.x, 1);
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  const long long t0 = clock64();
  const long long nchunk = src_bytes / CH;
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < iters; ++i) {
      const int s = i % NST;
      mbar_wait(empty + 8 * s, ((i / NST) & 1) ^ 1);
      mbar_expect(full + 8 * s, CH);
      const long long c = (blockIdx.x * 7 + i) % nchunk;
      bulk_g2s(ring + s * CH, src + c * CH, CH, full + 8 * s);
    }
  } else if (warp == 1 && lane == 0) {
    for (int i = 0; i < iters; ++i) {
      const int s = i % NST;
      mbar_wait(full + 8 * s, (i / NST) & 1);
      mbar_arrive(empty + 8 * s);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

template <int NST, int CH>
void run(const uint8_t* src, long long bytes, int sms) {
  unsigned long long* cyc;
  cudaMalloc(&cyc, sms * 8);
  const int smem = 2048 + NST * CH;
  cudaFuncSetAttribute(ingress<NST, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = (256 << 20) / CH;  // 256 MB per CTA
  ingress<NST, CH><<<sms, 64, smem>>>(src, bytes, 64, cyc);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  ingress<NST, CH><<<sms, 64, smem>>>(src, bytes, iters, cyc);
  cudaEventRecord(e1);
  cudaDeviceSynchronize();
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[256];
  cudaMemcpy(h, cyc, sms * 8, cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
  const double per_sm = static_cast<double>(iters) * CH / mx;
  printf("NST %2d chunk %6d B ring %3d KB: %.1f B/clk per SM, %.1f TB/s aggregate (%.2f ms) %s\n", NST, CH,
         NST * CH / 1024, per_sm, static_cast<double>(iters) * CH * sms / (ms * 1e-3) / 1e12, ms,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(cyc);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (long long mb : {16LL, 64LL}) {
    const long long bytes = mb << 20;
    uint8_t* src;
    cudaMalloc(&src, bytes);
    cudaMemset(src, 1, bytes);
    printf("-- source %lld MB (L2-resident)\n", mb);
    run<4, 36864>(src, bytes, sms);
    run<5, 36864>(src, bytes, sms);
    run<4, 16384>(src, bytes, sms);
    run<8, 16384>(src, bytes, sms);
    run<12, 16384>(src, bytes, sms);
    run<6, 32768>(src, bytes, sms);
    cudaFree(src);
  }
  return 0;
}
