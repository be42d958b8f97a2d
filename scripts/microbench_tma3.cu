// Microbenchmark 3: 16 KB weight bulk stream (HBM) per stage, optionally with an L2 cache
// hint, plus an activation-like 3-D TMA tile (L2-resident source) issued by a second warp
// into the same stage (development aid for the stream-K decode kernel).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait_bar(uint32_t bar, uint32_t par) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                 : "=r"(ok)
                 : "r"(bar), "r"(par)
                 : "memory");
}

// mode bit0: evict_first hint on weights; bit1: add 3-D act TMA (8 KB) per stage from warp 1;
// bit2: act TMA is 2-D (four 2 KB boxes) instead of 3-D; bit3: consumer warp releases slots
__global__ void __launch_bounds__(128, 1) kern(const __grid_constant__ CUtensorMap m3, const __grid_constant__ CUtensorMap m2,
                                               const uint8_t* src, size_t per_cta, int depth, int mode,
                                               unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t base = (smem_u32(smem) + 1023) & ~1023u;
  const uint32_t full = base, empty = base + 8 * 16;
  const uint32_t ring = base + 1024;
  const int req = 16384, act = 8192, stage = req + act;
  const int nreq = (int)(per_cta / req);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < depth; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(full + 8 * i), "r"((mode & 2) ? 2 : 1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(empty + 8 * i));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const long long t0 = clock64();
  const uint8_t* w = src + blockIdx.x * per_cta;
  if (warp == 0 && lane == 0) {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    for (int i = 0; i < nreq; ++i) {
      const int s = i % depth;
      wait_bar(empty + 8 * s, ((i / depth) & 1) ^ 1);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(full + 8 * s), "r"(req) : "memory");
      if (mode & 1)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
                ring + s * stage + act),
            "l"(w + (size_t)i * req), "r"(req), "r"(full + 8 * s), "l"(pol)
            : "memory");
      else
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         ring + s * stage + act),
                     "l"(w + (size_t)i * req), "r"(req), "r"(full + 8 * s)
                     : "memory");
    }
  } else if (warp == 1 && lane == 0 && (mode & 2)) {
    for (int i = 0; i < nreq; ++i) {
      const int s = i % depth;
      wait_bar(empty + 8 * s, ((i / depth) & 1) ^ 1);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(full + 8 * s), "r"(act) : "memory");
      const int kc = (i * 4) % 64;
      if (mode & 4) {
        for (int b = 0; b < 4; ++b)
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                  ring + s * stage + b * 2048),
              "l"(&m2), "r"((kc + b) * 64), "r"(0), "r"(full + 8 * s)
              : "memory");
      } else {
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
                ring + s * stage),
            "l"(&m3), "r"(0), "r"(0), "r"(kc), "r"(full + 8 * s)
            : "memory");
      }
    }
  } else if (warp == 2 && lane == 0) {
    for (int i = 0; i < nreq; ++i) {
      const int s = i % depth;
      wait_bar(full + 8 * s, (i / depth) & 1);
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(empty + 8 * s) : "memory");
    }
    cyc[blockIdx.x] = clock64() - t0;
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t total = (size_t)1 << 30;
  uint8_t* src;
  cudaMalloc(&src, total);
  cudaMemset(src, 1, total);
  const int K = 4096, M = 16;
  uint16_t* A;
  cudaMalloc(&A, (size_t)M * K * 2);
  cudaMemset(A, 0, (size_t)M * K * 2);
  unsigned long long* cyc;
  cudaMalloc(&cyc, 4096 * 8);
  void* fnp = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &qr);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fnp;
  CUtensorMap m3, m2;
  {
    const cuuint64_t dims[3] = {64, (cuuint64_t)M, (cuuint64_t)K / 64};
    const cuuint64_t str[2] = {(cuuint64_t)K * 2, 128};
    const cuuint32_t box[3] = {64, 16, 4};
    const cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(&m3, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, A, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("enc3 %d\n", (int)r);
  }
  {
    const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)M};
    const cuuint64_t str[1] = {(cuuint64_t)K * 2};
    const cuuint32_t box[2] = {64, 16};
    const cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&m2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, A, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("enc2 %d\n", (int)r);
  }
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  printf("mode depth GB/s(weights) cycles_per_stage\n");
  for (int mode : {0, 1, 2, 3, 6, 7}) {
    for (int depth : {4, 6, 8}) {
      const int smem = 2048 + depth * (16384 + 8192);
      if (smem > 200 * 1024) continue;
      const size_t per = (total / sms) / 16384 * 16384;
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      kern<<<sms, 128, smem>>>(m3, m2, src, per, depth, mode, cyc);
      cudaEventRecord(e0);
      for (int r = 0; r < 3; ++r) kern<<<sms, 128, smem>>>(m3, m2, src, per, depth, mode, cyc);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      unsigned long long h[4096];
      cudaMemcpy(h, cyc, sms * 8, cudaMemcpyDeviceToHost);
      double a = 0;
      for (int i = 0; i < sms; ++i) a += h[i];
      a /= sms;
      printf("%4d %4d %8.1f %8.1f %s\n", mode, depth, 3.0 * per * sms / (ms * 1e-3) / 1e9, a / (per / 16384),
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
