// Inter-kernel gap inside a CUDA graph: per-CTA %globaltimer at start/end for L back-to-back
// launches of a trivial persistent-style kernel, with/without TMEM allocation, large dynamic
// SMEM, PDL and clusters.  Prints per-launch first start, last end and gap to the previous end.
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -o scripts/mb_gap scripts/microbench_gap.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#include "../paper_2508_15601_b200/csrc/ptx.cuh"

using namespace w4k;

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <bool TMEM>
__global__ void kern(unsigned long long* trace, int spin_ns) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint64_t t0 = gtimer();
  if (TMEM && threadIdx.x < 32) {
    tmem_alloc(smem_u32(smem), 512);
    tmem_relinquish();
  }
  __syncthreads();
  grid_dependency_launch();
  grid_dependency_wait();
  while (gtimer() - t0 < static_cast<uint64_t>(spin_ns)) {
  }
  smem[64 + threadIdx.x] = 1;
  __syncthreads();
  if (threadIdx.x == 0) {
    trace[2 * blockIdx.x] = t0;
    trace[2 * blockIdx.x + 1] = gtimer();
  }
  if (TMEM && threadIdx.x < 32) {
    const uint32_t base = *reinterpret_cast<uint32_t*>(smem);
    __syncwarp();
    tmem_dealloc(base, 512);
  }
}

template <bool TMEM>
void run(const char* name, int threads, int smem, bool pdl, int cluster, int grid, int spin_ns) {
  const int L = 8;
  auto k = kern<TMEM>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  std::vector<unsigned long long*> bufs(L);
  for (auto& b : bufs) cudaMalloc(&b, grid * 16);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  auto launch = [&](int i) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    cfg.attrs = at;
    cfg.numAttrs = 0;
    if (pdl) {
      at[cfg.numAttrs].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[cfg.numAttrs].val.programmaticStreamSerializationAllowed = 1;
      ++cfg.numAttrs;
    }
    if (cluster > 1) {
      at[cfg.numAttrs].id = cudaLaunchAttributeClusterDimension;
      at[cfg.numAttrs].val.clusterDim.x = cluster;
      at[cfg.numAttrs].val.clusterDim.y = 1;
      at[cfg.numAttrs].val.clusterDim.z = 1;
      ++cfg.numAttrs;
    }
    cudaLaunchKernelEx(&cfg, k, bufs[i], spin_ns);
  };
  for (int i = 0; i < L; ++i) launch(i);
  cudaStreamSynchronize(s);
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < L; ++i) launch(i);
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  for (int r = 0; r < 3; ++r) cudaGraphLaunch(ge, s);
  cudaStreamSynchronize(s);
  std::vector<unsigned long long> h(2 * grid);
  unsigned long long prev_end = 0, t_first = 0;
  double gap_sum = 0, dur_sum = 0;
  for (int i = 0; i < L; ++i) {
    cudaMemcpy(h.data(), bufs[i], grid * 16, cudaMemcpyDeviceToHost);
    unsigned long long s0 = ~0ull, e1 = 0;
    for (int c = 0; c < grid; ++c) {
      s0 = h[2 * c] < s0 ? h[2 * c] : s0;
      e1 = h[2 * c + 1] > e1 ? h[2 * c + 1] : e1;
    }
    if (i == 0) t_first = s0;
    if (i > 0) gap_sum += static_cast<double>(static_cast<long long>(s0 - prev_end));
    // the last start (CTAs that could not launch early)
    unsigned long long slast = 0;
    for (int c = 0; c < grid; ++c) slast = h[2 * c] > slast ? h[2 * c] : slast;
    if (i > 0) dur_sum += static_cast<double>(e1 - prev_end);
    prev_end = e1;
    (void)slast;
  }
  printf("%-44s L=%d: total %.2f us, mean (end_i - end_{i-1}) %.2f us, mean first-start gap %.2f us  %s\n", name, L,
         (prev_end - t_first) / 1e3, dur_sum / (L - 1) / 1e3, gap_sum / (L - 1) / 1e3,
         cudaGetErrorString(cudaGetLastError()));
  for (auto& b : bufs) cudaFree(b);
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  cudaStreamDestroy(s);
}

int main() {
  const int spin = 2000;  // each CTA lives >= 2 us
  run<false>("640 thr, 1 KB smem, no PDL", 640, 1024, false, 1, 148, spin);
  run<false>("640 thr, 1 KB smem, PDL", 640, 1024, true, 1, 148, spin);
  run<false>("640 thr, 200 KB smem, no PDL", 640, 200 * 1024, false, 1, 148, spin);
  run<false>("640 thr, 200 KB smem, PDL", 640, 200 * 1024, true, 1, 148, spin);
  run<true>("640 thr, 200 KB smem, TMEM 512, no PDL", 640, 200 * 1024, false, 1, 148, spin);
  run<true>("640 thr, 200 KB smem, TMEM 512, PDL", 640, 200 * 1024, true, 1, 148, spin);
  run<true>("640 thr, 200 KB, TMEM, PDL, cluster 2, 64 CTAs", 640, 200 * 1024, true, 2, 64, spin);
  run<true>("640 thr, 200 KB, TMEM, PDL, cluster 2, 96 CTAs", 640, 200 * 1024, true, 2, 96, spin);
  run<true>("640 thr, 200 KB, TMEM, PDL, cluster 4, 128 CTAs", 640, 200 * 1024, true, 4, 128, spin);
  run<true>("640 thr, 200 KB, TMEM, no PDL, cluster 2, 64", 640, 200 * 1024, false, 2, 64, spin);
  run<true>("640 thr, 100 KB, TMEM 512, PDL", 640, 100 * 1024, true, 1, 148, spin);
  return 0;
}
