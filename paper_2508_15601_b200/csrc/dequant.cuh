// dequant.cuh -- the I2F + zero/scale step of the W4A16 path (§3.1 step iii,
// P:181; §3.4 "Integer-to-Float (I2F)"; §4.3) on the LAYOUT v1 word order.
//
// A LAYOUT v1 word holds 8 k-consecutive codes in nibble order [e0 e2 e4 e6 e1 e3 e5 e7]
// (DESIGN.md §3), so for i = 0..3
//     x_i = ((w >> 4i) & 0x000F000F) | MAGIC          (one SHF + one LOP3)
// is the 16-bit pair (MAGIC + e_{2i}, MAGIC + e_{2i+1}) with MAGIC = 0x4300 (bf16 128.0,
// whose ulp is 1) or 0x6400 (fp16 1024.0, ulp 1): an exact int->float conversion.
// Then (reading R6):
//     t = x - (MAGIC_VALUE + z)      sub.rn  -- exact for integer z
//     d = t * s                      mul.rn  -- the one rounding (s pre-rounded to bf16 on
//                                               the bf16 path: RNE_bf16((q-z)*RNE_bf16(s)))
// Both the GEMM and tm_dequant_w4 use exactly these functions.
#pragma once
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

namespace w4k {

__device__ __forceinline__ uint32_t pack_u16x2(uint16_t lo, uint16_t hi) {
  return static_cast<uint32_t>(lo) | (static_cast<uint32_t>(hi) << 16);
}

// Per-(row, group) constants: s2 = {s', s'}, z2 = {MAGIC + z, MAGIC + z} in the operand dtype.
template <bool BF16>
__device__ __forceinline__ void deq_prepare(uint16_t s_bits, uint16_t z_bits, uint32_t& s2, uint32_t& z2) {
  const float sf = __half2float(__ushort_as_half(s_bits));
  const float zf = __half2float(__ushort_as_half(z_bits));
  if constexpr (BF16) {
    const uint16_t sb = __bfloat16_as_ushort(__float2bfloat16_rn(sf));
    const uint16_t zb = __bfloat16_as_ushort(__float2bfloat16_rn(128.0f + zf));
    s2 = pack_u16x2(sb, sb);
    z2 = pack_u16x2(zb, zb);
  } else {
    const uint16_t zh = __half_as_ushort(__float2half_rn(1024.0f + zf));
    s2 = pack_u16x2(s_bits, s_bits);
    z2 = pack_u16x2(zh, zh);
  }
}

// One packed word -> 4 operand pairs (k-consecutive: out[i] = (k0+2i, k0+2i+1)).
template <bool BF16>
__device__ __forceinline__ void deq_word(uint32_t w, uint32_t s2, uint32_t z2, uint32_t* out) {
  constexpr uint32_t MAGIC = BF16 ? 0x43004300u : 0x64006400u;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    // one LOP3: (w' & 0x000F000F) | MAGIC  (LUT 0xEA = (a & b) | c)
    uint32_t x;
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(x) : "r"(w >> (4 * i)), "r"(0x000F000Fu), "r"(MAGIC));
    uint32_t d;
    if constexpr (BF16) {
      asm("{\n\t.reg .b32 t;\n\tsub.rn.bf16x2 t, %1, %2;\n\tmul.rn.bf16x2 %0, t, %3;\n\t}"
          : "=r"(d)
          : "r"(x), "r"(z2), "r"(s2));
    } else {
      asm("{\n\t.reg .b32 t;\n\tsub.rn.f16x2 t, %1, %2;\n\tmul.rn.f16x2 %0, t, %3;\n\t}"
          : "=r"(d)
          : "r"(x), "r"(z2), "r"(s2));
    }
    out[i] = d;
  }
}

#ifndef TM_DEQ_MULHI
#define TM_DEQ_MULHI 0
#endif
// operand for the integer-exact MMA: x - (MAGIC + z) for the 4 pairs of one LAYOUT v1 word
template <bool BF16>
__device__ __forceinline__ void deq_word_int(uint32_t w, uint32_t z2, uint32_t* out) {
  constexpr uint32_t MAGIC = BF16 ? 0x43004300u : 0x64006400u;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    // w >> 4i.  The dequant phase is ALU-pipe bound (3 SHF + 4 LOP3 = 14 ALU cycles per word vs
    // 4 HSUB = 8 FMA cycles), so the last shift runs on the FMA pipe as mul.hi (half rate, 4
    // cycles): 12 ALU / 12 FMA cycles per word.
    uint32_t ws;
    if (TM_DEQ_MULHI && i == 3)
      asm("mul.hi.u32 %0, %1, %2;" : "=r"(ws) : "r"(w), "r"(1u << 20));
    else
      ws = w >> (4 * i);
    uint32_t x;
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(x) : "r"(ws), "r"(0x000F000Fu), "r"(MAGIC));
    uint32_t d;
    if constexpr (BF16)
      asm("sub.rn.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(x), "r"(z2));
    else
      asm("sub.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(x), "r"(z2));
    out[i] = d;
  }
}

template <bool BF16>
__device__ __forceinline__ uint32_t zero_operand(uint16_t z_bits) {
  const float zf = __half2float(__ushort_as_half(z_bits));
  const uint16_t zb = BF16 ? __bfloat16_as_ushort(__float2bfloat16_rn(128.0f + zf))
                           : __half_as_ushort(__float2half_rn(1024.0f + zf));
  return static_cast<uint32_t>(zb) | (static_cast<uint32_t>(zb) << 16);
}

}  // namespace w4k
