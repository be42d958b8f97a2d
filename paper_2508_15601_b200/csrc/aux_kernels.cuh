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

// ---------------------------------------------------------------- checkpoint converters (§8(f) NEXT-4)
// LAYOUT v1 chunks straight from AWQ / GPTQ int4 checkpoints (formats: DESIGN.md §3, "checkpoint formats").
// AWQ qweight int32 [K][N/8]: column n's code is nibble kAwqRev[n % 8] of word [k][n / 8].
__device__ __forceinline__ int awq_rev(int c) { return (c & 1) * 4 + (c >> 1); }  // inverse of (0,2,4,6,1,3,5,7)

__global__ void pack_awq_kernel(const uint32_t* __restrict__ qw, uint4* __restrict__ out, int K, int N) {
  const int KS = K / 64;
  const int NW = N / 8;
  const long long nchunks = static_cast<long long>(K) * N / 32;
  for (long long c = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; c < nchunks;
       c += static_cast<long long>(gridDim.x) * blockDim.x) {
    const ChunkCoord cc = chunk_coord(c, KS);
    const int n = cc.nt * 128 + cc.t;
    const int kbase = cc.ks * 64 + cc.j * 32;
    const int sh = 4 * awq_rev(n & 7);
    uint32_t w[4];
#pragma unroll
    for (int wj = 0; wj < 4; ++wj) {
      uint32_t word = 0;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const uint32_t code = (__ldg(qw + static_cast<size_t>(kbase + wj * 8 + e) * NW + (n >> 3)) >> sh) & 0xFu;
        word |= code << (4 * nibble_of(e));
      }
      w[wj] = word;
    }
    out[c] = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// GPTQ qweight int32 [K/8][N]: word [kb][n] holds rows 8 kb .. 8 kb + 7 of column n in nibbles
// 0..7 -- exactly one LAYOUT v1 word, nibbles permuted to (e0 e2 e4 e6 e1 e3 e5 e7).
__global__ void pack_gptq_kernel(const uint32_t* __restrict__ qw, uint4* __restrict__ out, int K, int N) {
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
      const uint32_t src = __ldg(qw + static_cast<size_t>((kbase + wj * 8) >> 3) * N + n);
      uint32_t word = 0;
#pragma unroll
      for (int e = 0; e < 8; ++e) word |= ((src >> (4 * e)) & 0xFu) << (4 * nibble_of(e));
      w[wj] = word;
    }
    out[c] = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// zeros int32 [G][N/8] -> fp16 [G][N]: AWQ order (awq = 1) or sequential + offset (GPTQ)
__global__ void unpack_zeros_kernel(const uint32_t* __restrict__ qz, uint16_t* __restrict__ z, long long count, int N,
                                    int awq, int offset) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int n = static_cast<int>(i % N);
    const long long g = i / N;
    const int nib = awq ? awq_rev(n & 7) : (n & 7);
    const int v = static_cast<int>((__ldg(qz + g * (N / 8) + (n >> 3)) >> (4 * nib)) & 0xFu) + offset;
    z[i] = __half_as_ushort(__int2half_rn(v));
  }
}

// W8 bit planes (reading R17): LAYOUT v1 of the [2K][N] nibble matrix whose row k < K is
// q8[k] >> 4 and row K + k is q8[k] & 15.
__global__ void pack_w8_kernel(const uint8_t* __restrict__ q8, uint4* __restrict__ out, int K, int N) {
  const int K2 = 2 * K;
  const int KS = K2 / 64;
  const long long nchunks = static_cast<long long>(K2) * N / 32;
  for (long long c = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; c < nchunks;
       c += static_cast<long long>(gridDim.x) * blockDim.x) {
    const ChunkCoord cc = chunk_coord(c, KS);
    const int n = cc.nt * 128 + cc.t;
    const int kbase = cc.ks * 64 + cc.j * 32;  // row of the [2K][N] plane matrix
    const bool hi = kbase < K;
    const int k8 = hi ? kbase : kbase - K;
    uint32_t w[4];
#pragma unroll
    for (int wj = 0; wj < 4; ++wj) {
      uint32_t word = 0;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const uint32_t v = __ldg(q8 + static_cast<size_t>(k8 + wj * 8 + e) * N + n);
        word |= (hi ? (v >> 4) : (v & 0xFu)) << (4 * nibble_of(e));
      }
      w[wj] = word;
    }
    out[c] = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// W8 scales / zeros -> the planes' [2G][N]: high planes (16 s, z8 >> 4), low planes (s, z8 & 15)
__global__ void w8_sz_kernel(const uint16_t* __restrict__ s, const uint16_t* __restrict__ z8, uint16_t* __restrict__ s4,
                             uint16_t* __restrict__ z4, long long count) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const __half sv = __ushort_as_half(s[i]);
    const int zv = __half2int_rn(__ushort_as_half(z8[i]));
    s4[i] = __half_as_ushort(__hmul(sv, __float2half(16.0f)));  // exact (power of two) unless overflow
    s4[count + i] = s[i];
    z4[i] = __half_as_ushort(__int2half_rn((zv >> 4) & 0xF));
    z4[count + i] = __half_as_ushort(__int2half_rn(zv & 0xF));
  }
}

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
