// Per-instruction throughput on sm_100a: SMSP cycles per warp-instruction at saturation
// (16 warps per SM, 8 independent chains per thread).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#define N_CHAIN 8

template <int OP>
__global__ void kern(int iters, unsigned long long* out, uint32_t seed) {
  uint32_t v[N_CHAIN];
#pragma unroll
  for (int j = 0; j < N_CHAIN; ++j) v[j] = seed * (threadIdx.x + 7 * j + 1);
  const uint32_t k1 = seed ^ 0x3C003C00u, k2 = seed | 0x000F000Fu;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < N_CHAIN; ++j) {
      uint32_t x = v[j], d;
      if (OP == 0) asm volatile("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(x), "r"(k2), "r"(k1));
      if (OP == 1) asm volatile("shr.b32 %0, %1, 4;" : "=r"(d) : "r"(x));
      if (OP == 2) asm volatile("sub.rn.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(x), "r"(k1));
      if (OP == 3) asm volatile("sub.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(x), "r"(k1));
      if (OP == 4) asm volatile("mul.hi.u32 %0, %1, %2;" : "=r"(d) : "r"(x), "r"(k1));
      if (OP == 5) asm volatile("fma.rn.f32 %0, %1, %2, %1;" : "=r"(d) : "r"(x), "r"(k1));
      if (OP == 6) asm volatile("prmt.b32 %0, %1, %2, 0x5140;" : "=r"(d) : "r"(x), "r"(k1));
      if (OP == 7) asm volatile("fma.rn.bf16x2 %0, %1, %2, %1;" : "=r"(d) : "r"(x), "r"(k1));
      if (OP == 8) asm volatile("add.u32 %0, %1, %2;" : "=r"(d) : "r"(x), "r"(k1));
      if (OP == 9) asm volatile("mul.rn.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(x), "r"(k1));
      if (OP == 10) asm volatile("sub.rn.f32 %0, %1, %2;" : "=r"(d) : "r"(x), "r"(k1));
      if (OP == 11) asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "r"(x), "r"(k1));
      v[j] = d;
    }
  }
  const long long t1 = clock64();
  uint32_t acc = 0;
#pragma unroll
  for (int j = 0; j < N_CHAIN; ++j) acc ^= v[j];
  if ((threadIdx.x & 31) == 0) out[blockIdx.x * 64 + (threadIdx.x >> 5)] = t1 - t0;
  if (acc == 0x1234567u) out[0] = 0;
}

const char* NAMES[] = {"lop3", "shr", "sub.bf16x2", "sub.f16x2", "mul.hi.u32", "fma.f32", "prmt",
                       "fma.bf16x2", "add.u32", "mul.bf16x2", "sub.f32", "cvt.bf16x2.f32"};

template <int OP>
void run() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 64 * 8);
  const int iters = 4096, warps = 16;
  kern<OP><<<148, 32 * warps>>>(iters, d, 3);
  kern<OP><<<148, 32 * warps>>>(iters, d, 3);
  cudaDeviceSynchronize();
  unsigned long long h[64];
  cudaMemcpy(h, d, 64 * 8, cudaMemcpyDeviceToHost);
  double c = 0;
  for (int i = 0; i < warps; ++i) c += h[i];
  c /= warps;
  const double instr_per_smsp = (warps / 4.0) * N_CHAIN * iters;
  printf("%-16s SMSP cycles per warp-instruction %.2f\n", NAMES[OP], c / instr_per_smsp);
  cudaFree(d);
}

int main() {
  run<0>(); run<1>(); run<2>(); run<3>(); run<4>(); run<5>(); run<6>(); run<7>(); run<8>(); run<9>(); run<10>(); run<11>();
  return 0;
}
