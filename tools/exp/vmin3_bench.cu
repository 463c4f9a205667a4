// vmin3_bench.cu -- issue rate of VIMNMX3.S16x2 (3 registers) vs VIMNMX.S16x2
// (does a 3-input min cost one ALU slot or two?).  8 independent chains per
// thread, full occupancy; SASS checked with cuobjdump.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define ITERS 4096
#define CH 8
__global__ void k_min2(uint32_t* out, uint32_t k1, uint32_t k2) {
  uint32_t r[CH];
  for (int c = 0; c < CH; ++c) r[c] = threadIdx.x * 7 + c;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) asm volatile("{min.s16x2 %0, %0, %1; max.s16x2 %0, %0, %2;}" : "+r"(r[c]) : "r"(k1 ^ i), "r"(k2 + i));
  }
  uint32_t acc = 0;
  for (int c = 0; c < CH; ++c) acc ^= r[c];
  if (acc == 0x12345678u) out[0] = acc;
}
__global__ void k_min3(uint32_t* out, uint32_t k1, uint32_t k2) {
  uint32_t r[CH];
  for (int c = 0; c < CH; ++c) r[c] = threadIdx.x * 7 + c;
  for (int i = 0; i < ITERS; ++i) {
    const uint32_t x = k1 ^ i, y = k2 + i;
#pragma unroll
    for (int c = 0; c < CH; ++c) asm volatile("{.reg .b32 t; min.s16x2 t, %0, %1; min.s16x2 %0, t, %2;}" : "+r"(r[c]) : "r"(x), "r"(y));
  }
  uint32_t acc = 0;
  for (int c = 0; c < CH; ++c) acc ^= r[c];
  if (acc == 0x12345678u) out[0] = acc;
}
int main() {
  uint32_t* d; cudaMalloc(&d, 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int v = 0; v < 2; ++v) {
    auto k = v == 0 ? k_min2 : k_min3;
    k<<<sms * 8, 256>>>(d, 3, 5);
    cudaEventRecord(a);
    k<<<sms * 8, 256>>>(d, 3, 5);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double instr = (double)sms * 8 * 256 / 32 * ITERS * CH * (v == 0 ? 2 : 1);   // warp-level SASS instructions
    printf("{\"kernel\": \"%s\", \"ms\": %.3f, \"warp_instr_per_clk_per_sm\": %.3f}\n", v ? "VIMNMX3 (min of 3, 1 per step)" : "VIMNMX (min then max, 2 per step)",
           ms, instr / (ms * 1e-3) / sms / (1965e6));
  }
  return 0;
}
