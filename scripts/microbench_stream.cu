// Microbenchmark: the streaming floor of the bench's decode mix.  A kernel with the decode
// GEMM's load structure but no math (one producer lane issues 16 KB cp.async.bulk chunks into an
// NST-slot mbarrier ring, 4 consumer warps touch each chunk and free the slot) runs the bench's
// sequence of 48 launches (4 layers x {qkv, o, gate_up, down} x M in {1, 8, 16}, codes + s/z
// bytes, every layer a distinct buffer, 464 MB > L2) as one CUDA graph, with and without PDL.
// The achieved GB/s is the ceiling any decode kernel with this launch structure can reach on
// the mix (per-launch head/tail included).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

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
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity), "r"(0x989680u)
        : "memory");
  }
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar), "l"(pol)
      : "memory");
}

template <int NST>
__global__ void __launch_bounds__(160) stream_kernel(const uint8_t* src, long long chunks, uint32_t* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const uint32_t base = (smem_u32(sm) + 1023u) & ~1023u;
  uint8_t* bp = sm + (base - smem_u32(sm));
  const uint32_t full = base, empty = base + 8 * NST, ring = base + 1024;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const long long c0 = chunks * blockIdx.x / gridDim.x, c1 = chunks * (blockIdx.x + 1) / gridDim.x;
  if (threadIdx.x < NST) {
    mbar_init(full + 8 * threadIdx.x, 1);
    mbar_init(empty + 8 * threadIdx.x, 4);
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  uint32_t x = 0;
  if (warp == 0) {
    if (lane == 0) {
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      int slot = 0;
      uint32_t ph = 0;
      for (long long c = c0; c < c1; ++c) {
        if (c - c0 == NST) asm volatile("griddepcontrol.wait;" ::: "memory");
        mbar_wait(empty + 8 * slot, ph ^ 1u);
        mbar_expect(full + 8 * slot, 16384);
        bulk_g2s(ring + slot * 16384, src + c * 16384, 16384, full + 8 * slot, pol);
        if (++slot == NST) slot = 0, ph ^= 1u;
      }
      if (c1 - c0 <= NST) asm volatile("griddepcontrol.wait;" ::: "memory");
    }
  } else {
    int slot = 0;
    uint32_t ph = 0;
    for (long long c = c0; c < c1; ++c) {
      mbar_wait(full + 8 * slot, ph);
      x ^= *reinterpret_cast<const uint32_t*>(bp + 1024 + slot * 16384 + (warp - 1) * 4096 + lane * 128);
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + 8 * slot);
      if (++slot == NST) slot = 0, ph ^= 1u;
    }
  }
  if (x == 0x12345678u) out[threadIdx.x] = x;
}

template <int NST>
void run(const std::vector<std::pair<const uint8_t*, long long>>& launches, double total_bytes, int ctas_per_sm,
         bool pdl, int sms) {
  const int smem = 1024 + 1024 + NST * 16384;
  cudaFuncSetAttribute(stream_kernel<NST>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  uint32_t* out;
  cudaMalloc(&out, 4096);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (auto& l : launches) {
    cudaLaunchConfig_t cfg = {};
    long long chunks = l.second / 16384;
    int grid = sms * ctas_per_sm;
    if (grid > chunks) grid = static_cast<int>(chunks);
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(160);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, stream_kernel<NST>, l.first, chunks, out);
  }
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  for (int i = 0; i < 3; ++i) cudaGraphLaunch(ge, s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int reps = 20;
  cudaEventRecord(e0, s);
  for (int i = 0; i < reps; ++i) cudaGraphLaunch(ge, s);
  cudaEventRecord(e1, s);
  cudaStreamSynchronize(s);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double us = ms * 1e3 / reps;
  printf("NST %2d (%3d KB) ctas/SM %d pdl %d: %8.1f us per mix of %zu launches  %7.1f GB/s  (%.2f us/launch)  %s\n", NST,
         smem / 1024, ctas_per_sm, pdl, us, launches.size(), total_bytes / us * 1e-3, us / launches.size(),
         cudaGetErrorString(cudaGetLastError()));
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  cudaFree(out);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  // codes + fp16 s/z at g = 128 (A and C are < 1 % of the bytes): qkv, o, gate_up, down
  const long long NK[4][2] = {{6144, 4096}, {4096, 4096}, {28672, 4096}, {4096, 14336}};
  std::vector<std::pair<const uint8_t*, long long>> launches;
  double total = 0;
  for (int layer = 0; layer < 4; ++layer) {
    for (int sh = 0; sh < 4; ++sh) {
      const long long bytes = NK[sh][0] * NK[sh][1] / 2 + 4 * (NK[sh][1] / 128) * NK[sh][0];
      const long long padded = (bytes + 16383) / 16384 * 16384;
      uint8_t* p;
      cudaMalloc(&p, padded);
      cudaMemset(p, layer + sh, padded);
      for (int m = 0; m < 3; ++m) {
        launches.push_back({p, padded});
        total += static_cast<double>(bytes);
      }
    }
  }
  // reorder like the bench: for each M, each layer's four shapes
  std::vector<std::pair<const uint8_t*, long long>> seq;
  for (int m = 0; m < 3; ++m)
    for (int layer = 0; layer < 4; ++layer)
      for (int sh = 0; sh < 4; ++sh) seq.push_back(launches[(layer * 4 + sh) * 3 + m]);
  for (int pdl = 0; pdl < 2; ++pdl) {
    run<12>(seq, total, 1, pdl, sms);
    run<6>(seq, total, 1, pdl, sms);
    run<6>(seq, total, 2, pdl, sms);
    run<4>(seq, total, 2, pdl, sms);
    run<4>(seq, total, 3, pdl, sms);
    run<3>(seq, total, 4, pdl, sms);
  }
  // one big stream for reference (gate_up only, 16 launches)
  std::vector<std::pair<const uint8_t*, long long>> big;
  double tb = 0;
  for (int i = 0; i < 16; ++i) {
    big.push_back(seq[(i % 4) * 4 + 2]);
    tb += 28672.0 * 4096 / 2 + 4.0 * 32 * 28672;
  }
  for (int pdl = 0; pdl < 2; ++pdl) {
    run<12>(big, tb, 1, pdl, sms);
    run<6>(big, tb, 2, pdl, sms);
  }
  return 0;
}
