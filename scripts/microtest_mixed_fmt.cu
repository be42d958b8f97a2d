// Correctness probe: does tcgen05.mma kind::f16 honour different A/B formats in the instruction
// descriptor (a_format bits 7-9, b_format bits 10-12)?  A (M=128 x K=16) from TMEM, B (N=16 x K=16)
// from SMEM (SW128 K-major), one MMA, D read back and compared with a host fp64 product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -o mt_mixed scripts/microtest_mixed_fmt.cu
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>

#include "../paper_2508_15601_b200/csrc/ptx.cuh"

using namespace w4k;

__host__ __device__ constexpr uint32_t idesc_mixed(int afmt, int bfmt, int M, int N) {
  return (1u << 4) | (static_cast<uint32_t>(afmt) << 7) | (static_cast<uint32_t>(bfmt) << 10) |
         (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(M >> 4) << 24);
}

// a_bits[n][k] (16-bit patterns), b_bits[m][k]; out[n][m]
__global__ void __launch_bounds__(128, 1) kern(const uint16_t* a_bits, const uint16_t* b_bits, float* out,
                                                uint32_t idesc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t base = (smem_u32(smem) + 1023) & ~1023u;
  uint8_t* bptr = smem + (base - smem_u32(smem));
  const uint32_t bar = base + 4096;
  const uint32_t tslot = base + 4096 + 16;
  const int warp = threadIdx.x >> 5;
  const int n = threadIdx.x;
  // B: 16 rows x 64 k (only k < 16 non-zero), SW128: row m at m*128, 16-B chunk c at (c ^ (m & 7))*16
  for (int i = threadIdx.x; i < 16 * 64; i += 128) {
    const int m = i / 64, k = i % 64;
    const uint16_t v = k < 16 ? b_bits[m * 16 + k] : 0;
    const int c = k / 8, e = k % 8;
    *reinterpret_cast<uint16_t*>(bptr + m * 128 + ((c ^ (m & 7)) * 16) + e * 2) = v;
  }
  fence_proxy_async_shared();
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    tmem_alloc(tslot, 64);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<uint32_t*>(smem + (tslot - smem_u32(smem)));
  // A operand: lane n, columns 32..39 hold k pairs (k0,k1),(k2,k3),...
  uint32_t r[32];
  for (int j = 0; j < 32; ++j) r[j] = 0;
  for (int j = 0; j < 8; ++j)
    r[j] = static_cast<uint32_t>(a_bits[n * 16 + 2 * j]) | (static_cast<uint32_t>(a_bits[n * 16 + 2 * j + 1]) << 16);
  const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
  tmem_st_32x32b_x32(tmem + 32 + lane_off, r);
  tc_wait_st();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    mma_ts(tmem, tmem + 32, umma_desc_sw128(base), idesc, 0u);
    tc_commit(bar);
  }
  __syncwarp();
  mbar_wait(bar, 0);
  tc_fence_after();
  uint32_t v[16];
  tmem_ld_32x32b_x16(tmem + lane_off, v);
  tc_wait_ld();
  for (int m = 0; m < 16; ++m) out[n * 16 + m] = __uint_as_float(v[m]);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 64);
  }
}

static double dec(uint16_t b, int fmt) {
  if (fmt == 0) return static_cast<double>(__half2float(__ushort_as_half(b)));
  uint32_t u = static_cast<uint32_t>(b) << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}
static uint16_t enc(double x, int fmt) {
  if (fmt == 0) return __half_as_ushort(__float2half_rn(static_cast<float>(x)));
  return __bfloat16_as_ushort(__float2bfloat16_rn(static_cast<float>(x)));
}

int main() {
  uint16_t ha[128 * 16], hb[16 * 16];
  uint16_t *da, *db;
  float* dout;
  cudaMalloc(&da, sizeof(ha));
  cudaMalloc(&db, sizeof(hb));
  cudaMalloc(&dout, 128 * 16 * 4);
  float hout[128 * 16];
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 1024);
  int fails = 0;
  for (int afmt = 0; afmt < 2; ++afmt)
    for (int bfmt = 0; bfmt < 2; ++bfmt) {
      unsigned s = 12345;
      auto rnd = [&]() { s = s * 1103515245u + 12345u; return static_cast<int>((s >> 16) & 0x7fff); };
      // A: integers -15..15 and fp16-only values (1024+q) when afmt = f16; B: random values
      for (int i = 0; i < 128 * 16; ++i) ha[i] = enc((rnd() % 31) - 15 + (afmt == 0 ? 1024.0 * (i % 3 == 0) : 0.0), afmt);
      for (int i = 0; i < 16 * 16; ++i) hb[i] = enc(((rnd() % 2001) - 1000) / 256.0, bfmt);
      cudaMemcpy(da, ha, sizeof(ha), cudaMemcpyHostToDevice);
      cudaMemcpy(db, hb, sizeof(hb), cudaMemcpyHostToDevice);
      kern<<<1, 128, 16 * 1024>>>(da, db, dout, idesc_mixed(afmt, bfmt, 128, 16));
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(hout, dout, sizeof(hout), cudaMemcpyDeviceToHost);
      double maxerr = 0, maxref = 0;
      for (int n = 0; n < 128; ++n)
        for (int m = 0; m < 16; ++m) {
          double ref = 0;
          for (int k = 0; k < 16; ++k) ref += dec(ha[n * 16 + k], afmt) * dec(hb[m * 16 + k], bfmt);
          maxerr = fmax(maxerr, fabs(ref - hout[n * 16 + m]));
          maxref = fmax(maxref, fabs(ref));
        }
      const bool ok = e == cudaSuccess && maxerr <= 1e-6 * maxref + 1e-6;
      fails += !ok;
      printf("a=%s b=%s: %s max|err| %.3g (max|ref| %.3g) %s\n", afmt ? "bf16" : "f16", bfmt ? "bf16" : "f16",
             cudaGetErrorString(e), maxerr, maxref, ok ? "EXACT" : "MISMATCH");
    }
  return fails;
}
