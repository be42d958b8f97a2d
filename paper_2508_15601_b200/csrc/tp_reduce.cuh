// tp_reduce.cuh -- fused row-parallel epilogue for tensor parallelism over symmetric memory
// (§8(f) NEXT-1; §5 P:471 "we utilize tensor parallelism", App. I).
//
// A row-parallel layer (o, down) leaves one fp32 partial C_r [M][N] per rank (K-shard,
// tm_gemm_w4a16_partial_f32) in a symmetric buffer: the same allocation mapped on every rank,
// peers' copies reachable over NVLink (torch symmetric memory supplies the mappings).  One
// kernel replaces the NCCL all-reduce + tm_tp_finalize pair:
//   1. entry barrier over the ranks' signal pads (block b, channel b): every rank's partial is
//      complete before anyone reads it;
//   2. C[i] = RNE_bf16( sum_r C_r[i] ) -- with an NVLS multicast address the switch adds the
//      ranks' words (multimem.ld_reduce .add.f32, one request per 16 B); without one the sum
//      runs over the peers' mappings in rank order r = 0..P-1 (deterministic, reading R13);
//   3. exit barrier (channel P_blocks + b): no rank reuses its partial buffer (the next
//      row-parallel GEMM writes it) before every peer has read it.
// Barrier protocol per (channel, pair): the sender CASes its word in the receiver's pad 0 -> 1
// (release, system scope), the receiver CASes it back 1 -> 0 (acquire): a pad word is only
// reused after its previous signal was consumed, so back-to-back layers cannot alias.
#pragma once
#include <cstdint>
#include <cuda_bf16.h>

namespace w4k {

constexpr int kTpMaxRanks = 8;
constexpr int kTpBlocks = 32;  // channels per barrier phase (signal words: 2 x 32 x world)

struct TpReduceArgs {
  const float* partials[kTpMaxRanks];  // rank r's fp32 partial (this process's mapping)
  uint32_t* signals[kTpMaxRanks];      // rank r's signal pad (this process's mapping)
  const float* multicast;              // NVLS multicast address of the partials, or nullptr
  __nv_bfloat16* out;                  // this rank's bf16 output
  long long count;                     // elements
  int rank, world;
};

__device__ __forceinline__ uint32_t cas_release_sys(uint32_t* p, uint32_t cmp, uint32_t val) {
  uint32_t old;
  asm volatile("atom.release.sys.global.cas.b32 %0, [%1], %2, %3;" : "=r"(old) : "l"(p), "r"(cmp), "r"(val) : "memory");
  return old;
}
__device__ __forceinline__ uint32_t cas_acquire_sys(uint32_t* p, uint32_t cmp, uint32_t val) {
  uint32_t old;
  asm volatile("atom.acquire.sys.global.cas.b32 %0, [%1], %2, %3;" : "=r"(old) : "l"(p), "r"(cmp), "r"(val) : "memory");
  return old;
}

// one barrier phase on channel `ch`: thread t < world signals rank t and waits for rank t
__device__ __forceinline__ void tp_barrier(const TpReduceArgs& a, int ch) {
  const int t = static_cast<int>(threadIdx.x);
  if (t < a.world) {
    uint32_t* const to = a.signals[t] + ch * a.world + a.rank;
    while (cas_release_sys(to, 0u, 1u) != 0u) {
    }
    uint32_t* const from = a.signals[a.rank] + ch * a.world + t;
    while (cas_acquire_sys(from, 1u, 0u) != 1u) {
    }
  }
  __syncthreads();
}

__device__ __forceinline__ float4 tp_sum4(const TpReduceArgs& a, long long i4) {
  float4 s;
  if (a.multicast) {
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(s.x), "=f"(s.y), "=f"(s.z), "=f"(s.w)
                 : "l"(a.multicast + 4 * i4)
                 : "memory");
    return s;
  }
  s = __ldcv(reinterpret_cast<const float4*>(a.partials[0]) + i4);
  for (int r = 1; r < a.world; ++r) {
    const float4 v = __ldcv(reinterpret_cast<const float4*>(a.partials[r]) + i4);
    s.x += v.x;
    s.y += v.y;
    s.z += v.z;
    s.w += v.w;
  }
  return s;
}

__global__ void __launch_bounds__(256) tp_allreduce_finalize_kernel(const TpReduceArgs a) {
  __threadfence_system();  // (the partials were written by the previous kernel on this stream)
  tp_barrier(a, static_cast<int>(blockIdx.x));
  const long long n4 = a.count / 4;
  for (long long i = blockIdx.x * 256ll + threadIdx.x; i < n4; i += gridDim.x * 256ll) {
    const float4 v = tp_sum4(a, i);
    const __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y);
    const __nv_bfloat162 hi = __floats2bfloat162_rn(v.z, v.w);
    reinterpret_cast<uint2*>(a.out)[i] = make_uint2(*reinterpret_cast<const uint32_t*>(&lo),
                                                    *reinterpret_cast<const uint32_t*>(&hi));
  }
  if (blockIdx.x == 0) {  // count % 4 tail (multicast requests are 16 B: the tail reads peers)
    for (long long i = 4 * n4 + threadIdx.x; i < a.count; i += 256) {
      float s = __ldcv(a.partials[0] + i);
      for (int r = 1; r < a.world; ++r) s += __ldcv(a.partials[r] + i);
      a.out[i] = __float2bfloat16_rn(s);
    }
  }
  __syncthreads();
  tp_barrier(a, kTpBlocks + static_cast<int>(blockIdx.x));
}

}  // namespace w4k
