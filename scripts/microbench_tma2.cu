// Microbenchmark: streaming HBM -> SMEM with 1-D bulk copies of various request sizes,
// issued by one thread per CTA into an mbarrier ring (development aid).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb scripts/microbench_tma.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(128, 1) stream_kernel(const uint8_t* src, size_t bytes_per_cta, int req, int depth,
                                                        unsigned long long* cycles_out, int nissue) {
  // nissue > 0: issuers are warps 0..nissue-1 (lane 0); nissue < 0: issuers are lanes 0..-nissue-1 of warp 0
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);  // full[depth]
  uint8_t* buf = smem + 1024;
  const int ni = nissue > 0 ? nissue : -nissue;
  const int me = nissue > 0 ? ((threadIdx.x & 31) == 0 ? (int)(threadIdx.x >> 5) : 99) : (threadIdx.x < 32 ? (int)threadIdx.x : 99);
  const uint8_t* base = src + blockIdx.x * bytes_per_cta + (me < ni ? (size_t)me * (bytes_per_cta / ni) : 0);
  const int nreq = (int)(bytes_per_cta / ni / req);
  bars += (me < ni ? me : 0) * depth;
  buf += (me < ni ? me : 0) * (size_t)depth * req;
  if (me < ni) {
    for (int i = 0; i < depth; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  long long t0 = clock64();
  if (me < ni) {
    for (int i = 0; i < nreq; ++i) {
      const int s = i % depth;
      if (i >= depth) {
        // wait for the previous use of slot s to have landed (phase of use i-depth)
        const uint32_t par = ((i / depth) - 1) & 1;
        uint32_t ok = 0;
        while (!ok)
          asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                       : "=r"(ok) : "r"(smem_u32(&bars[s])), "r"(par) : "memory");
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bars[s])), "r"(req)
                   : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_u32(buf + (size_t)s * req)),
                   "l"(base + (size_t)i * req), "r"(req), "r"(smem_u32(&bars[s]))
                   : "memory");
    }
    // drain
    for (int i = nreq > depth ? nreq - depth : 0; i < nreq; ++i) {
      const int s = i % depth;
      const uint32_t par = (i / depth) & 1;
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                     : "=r"(ok) : "r"(smem_u32(&bars[s])), "r"(par) : "memory");
    }
    if (me == 0) cycles_out[blockIdx.x] = clock64() - t0;
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t total = (size_t)1 << 30;
  uint8_t* src;
  cudaMalloc(&src, total);
  cudaMemset(src, 1, total);
  unsigned long long* cyc;
  cudaMalloc(&cyc, 4096 * sizeof(unsigned long long));
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  printf("req nissue depth GB/s cycles_per_req_per_issuer\n");
  for (int req : {2048, 4096, 8192, 16384}) {
    for (int nissue : {1, 2, 4, -2, -4}) {
      for (int depth : {4, 8}) {
        const int ni = nissue > 0 ? nissue : -nissue;
        const size_t ring = (size_t)req * depth * ni;
        if (ring + 1024 > 200 * 1024) continue;
        const int grid = sms;
        const size_t per_cta = (total / grid) / (req * ni) * (req * ni);
        const int smem = (int)(ring + 1024);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        stream_kernel<<<grid, 128, smem>>>(src, per_cta, req, depth, cyc, nissue);
        cudaEventRecord(e0);
        for (int r = 0; r < 3; ++r) stream_kernel<<<grid, 128, smem>>>(src, per_cta, req, depth, cyc, nissue);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        unsigned long long h[4096];
        cudaMemcpy(h, cyc, grid * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
        double avgc = 0;
        for (int i = 0; i < grid; ++i) avgc += h[i];
        avgc /= grid;
        const double gbs = 3.0 * per_cta * grid / (ms * 1e-3) / 1e9;
        printf("%6d %3d %3d %8.1f %8.1f\n", req, nissue, depth, gbs, avgc / (per_cta / ni / req));
        cudaError_t err = cudaGetLastError();
        if (err != cudaSuccess) printf("err %s\n", cudaGetErrorString(err));
      }
    }
  }
  return 0;
}
