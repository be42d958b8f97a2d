// aux_kernels.cuh -- offline packing (§8(a) row a2) and the test/TP helper kernels.
//
// pack_w4_kernel realises PAPER.md §4.1 for sm_100a: one thread builds one
// 16-byte chunk of LAYOUT v1 = the 4 words (32 k-consecutive codes) a
// GEMM dequant thread later reads with one LDS.128.  A warp writes 512 contiguous bytes
// and reads 32 consecutive bytes of q per k row: the pass is HBM-bound (offline).
#pragma once
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "dequant.cuh"

namespace w4k {

// chunk c (16 bytes) -> (n-tile, k-stage, half j, column t)
struct ChunkCoord {
  int nt, ks, j, t;
};
__device__ __forceinline__ ChunkCoord chunk_coord(long long c, int KS) {
  ChunkCoord r;
  const long long blob = c >> 8;  // 256 chunks per 4 KB blob
  const int within = static_cast<int>(c & 255);
  r.j = within >> 7;
  r.t = within & 127;
  r.nt = static_cast<int>(blob / KS);
  r.ks = static_cast<int>(blob % KS);
  return r;
}

// nibble position of the e-th k-consecutive code inside a word: [e0 e2 e4 e6 e1 e3 e5 e7]
__device__ __forceinline__ int nibble_of(int e) { return (e & 1) * 4 + (e >> 1); }

__global__ void pack_w4_kernel(const uint8_t* __restrict__ q, uint4* __restrict__ out, int K, int N) {
  const int KS = K / 64;
  const long long nchunks = static_cast<long long>(K) * N / 32;
  for (long long c = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; c < nchunks;
       c += static_cast<long long>(gridDim.x) * blockDim.x) {
    const ChunkCoord cc = chunk_coord(c, KS);
    const int n = cc.nt * 128 + cc.t;
    const int kbase = cc.ks * 64 + cc.j * 32;
    uint32_t w[4];
#pragma unroll
    for (int wj = 0; wj < 4; ++wj) {
      uint32_t word = 0;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const uint32_t code = __ldg(q + static_cast<size_t>(kbase + wj * 8 + e) * N + n) & 0xFu;
        word |= code << (4 * nibble_of(e));
      }
      w[wj] = word;
    }
    out[c] = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

__global__ void unpack_w4_kernel(const uint4* __restrict__ in, uint8_t* __restrict__ q, int K, int N) {
  const int KS = K / 64;
  const long long nchunks = static_cast<long long>(K) * N / 32;
  for (long long c = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; c < nchunks;
       c += static_cast<long long>(gridDim.x) * blockDim.x) {
    const ChunkCoord cc = chunk_coord(c, KS);
    const int n = cc.nt * 128 + cc.t;
    const int kbase = cc.ks * 64 + cc.j * 32;
    const uint4 v = in[c];
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int wj = 0; wj < 4; ++wj)
#pragma unroll
      for (int e = 0; e < 8; ++e)
        q[static_cast<size_t>(kbase + wj * 8 + e) * N + n] = static_cast<uint8_t>((w[wj] >> (4 * nibble_of(e))) & 0xFu);
  }
}

// Dense dequantisation with the GEMM's own code path (dequant.cuh) -> W[K][N].
template <bool BF16>
__global__ void dequant_w4_kernel(const uint4* __restrict__ in, const uint16_t* __restrict__ scales,
                                  const uint16_t* __restrict__ zeros, uint16_t* __restrict__ W, int K, int N,
                                  int group) {
  const int KS = K / 64;
  const long long nchunks = static_cast<long long>(K) * N / 32;
  for (long long c = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; c < nchunks;
       c += static_cast<long long>(gridDim.x) * blockDim.x) {
    const ChunkCoord cc = chunk_coord(c, KS);
    const int n = cc.nt * 128 + cc.t;
    const int kbase = cc.ks * 64 + cc.j * 32;
    const int g = kbase / group;  // 32 k-consecutive codes never straddle a group (group % 64 == 0)
    uint32_t s2, z2;
    deq_prepare<BF16>(scales[static_cast<size_t>(g) * N + n], zeros[static_cast<size_t>(g) * N + n], s2, z2);
    const uint4 v = in[c];
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int wj = 0; wj < 4; ++wj) {
      uint32_t d[4];
      deq_word<BF16>(w[wj], s2, z2, d);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int k = kbase + wj * 8 + 2 * i;
        W[static_cast<size_t>(k) * N + n] = static_cast<uint16_t>(d[i] & 0xFFFFu);
        W[static_cast<size_t>(k + 1) * N + n] = static_cast<uint16_t>(d[i] >> 16);
      }
    }
  }
}

// The decode kernel's MMA operand (reading R6b): (MAGIC + q) - (MAGIC + z) per weight, through
// its own deq_word_int / zero_operand code (debug entry tm_debug_dequant_int) -> W[K][N].
template <bool BF16>
__global__ void dequant_int_kernel(const uint4* __restrict__ in, const uint16_t* __restrict__ zeros,
                                   uint16_t* __restrict__ W, int K, int N, int group) {
  const int KS = K / 64;
  const long long nchunks = static_cast<long long>(K) * N / 32;
  for (long long c = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; c < nchunks;
       c += static_cast<long long>(gridDim.x) * blockDim.x) {
    const ChunkCoord cc = chunk_coord(c, KS);
    const int n = cc.nt * 128 + cc.t;
    const int kbase = cc.ks * 64 + cc.j * 32;
    const int g = kbase / group;
    const uint32_t z2 = zero_operand<BF16>(zeros[static_cast<size_t>(g) * N + n]);
    const uint4 v = in[c];
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int wj = 0; wj < 4; ++wj) {
      uint32_t d[4];
      deq_word_int<BF16>(w[wj], z2, d);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int k = kbase + wj * 8 + 2 * i;
        W[static_cast<size_t>(k) * N + n] = static_cast<uint16_t>(d[i] & 0xFFFFu);
        W[static_cast<size_t>(k + 1) * N + n] = static_cast<uint16_t>(d[i] >> 16);
      }
    }
  }
}

__global__ void noop_kernel() {}

// fp32 -> bf16 RNE (row-parallel TP epilogue after the fp32 all-reduce, reading R13).
__global__ void tp_finalize_kernel(const float4* __restrict__ in, uint2* __restrict__ out, long long n4) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const float4 v = in[i];
    const __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y);
    const __nv_bfloat162 b = __floats2bfloat162_rn(v.z, v.w);
    out[i] = make_uint2(*reinterpret_cast<const uint32_t*>(&a), *reinterpret_cast<const uint32_t*>(&b));
  }
}
__global__ void tp_finalize_tail_kernel(const float* __restrict__ in, __nv_bfloat16* __restrict__ out, long long start,
                                        long long count) {
  const long long i = start + blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i < count) out[i] = __float2bfloat16_rn(in[i]);
}

}  // namespace w4k
