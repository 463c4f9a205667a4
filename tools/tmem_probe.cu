// tmem_probe.cu -- check tcgen05 TMEM alloc / st / ld semantics used by the
// decoder's message store: 32x32b shapes x1..x8 at unaligned column offsets,
// several warps per lane quarter, round trip and timing.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tmem_probe tools/tmem_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void tm_st4(uint32_t taddr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr), "r"(a), "r"(b), "r"(c), "r"(d));
}
__device__ __forceinline__ void tm_st2(uint32_t taddr, uint32_t a, uint32_t b) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(taddr), "r"(a), "r"(b));
}
__device__ __forceinline__ void tm_st1(uint32_t taddr, uint32_t a) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(taddr), "r"(a));
}
__device__ __forceinline__ void tm_ld4(uint32_t taddr, uint32_t& a, uint32_t& b, uint32_t& c, uint32_t& d) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "r"(taddr));
}
__device__ __forceinline__ void tm_ld2(uint32_t taddr, uint32_t& a, uint32_t& b) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(a), "=r"(b) : "r"(taddr));
}
__device__ __forceinline__ void tm_ld1(uint32_t taddr, uint32_t& a) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(a) : "r"(taddr));
}
__device__ __forceinline__ void tm_wait_ld7(uint32_t& a, uint32_t& b, uint32_t& c, uint32_t& d, uint32_t& e, uint32_t& f, uint32_t& g) {
  asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(a), "+r"(b), "+r"(c), "+r"(d), "+r"(e), "+r"(f), "+r"(g)::"memory");
}
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// 12 warps (384 threads); warp w uses lane quarter w%4 and column slot w/4 * 76
__global__ void probe(uint32_t* out, int rounds, int stride, int slot) {
  __shared__ uint32_t s_taddr;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"((uint32_t)__cvta_generic_to_shared(&s_taddr)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = s_taddr + ((uint32_t)(32 * (w & 3)) << 16) + (uint32_t)((w >> 2) * slot);
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  long long t0 = clock64();
  uint32_t bad = 0;
  for (int r = 0; r < rounds; ++r) {
    for (int t = 0; t < 12; ++t) {          // 12 "tiers" of 7 columns at offsets 0, 7, 14, ... (unaligned)
      const uint32_t col = base + (uint32_t)(t * stride);
      const uint32_t v = tid * 1000u + (uint32_t)(t * 10 + r);
      tm_st4(col, v, v + 1, v + 2, v + 3);
      tm_st2(col + 4, v + 4, v + 5);
      tm_st1(col + 6, v + 6);
      tm_wait_st();
    }
    for (int t = 0; t < 12; ++t) {
      const uint32_t col = base + (uint32_t)(t * stride);
      uint32_t a, b, c, d, e, f, g;
      tm_ld4(col, a, b, c, d);
      tm_ld2(col + 4, e, f);
      tm_ld1(col + 6, g);
      tm_wait_ld7(a, b, c, d, e, f, g);
      const uint32_t v = tid * 1000u + (uint32_t)(t * 10 + r);
      bad += (a != v) + (b != v + 1) + (c != v + 2) + (d != v + 3) + (e != v + 4) + (f != v + 5) + (g != v + 6);
    }
  }
  long long t1 = clock64();
  out[tid * 2] = bad;
  out[tid * 2 + 1] = (uint32_t)(t1 - t0);
  (void)lane;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(s_taddr));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 2, threads = 384, rounds = 100;
  uint32_t* d;
  cudaMalloc(&d, (size_t)blocks * threads * 8);
  int cfg[][2] = {{7, 76}, {8, 76}, {8, 80}, {8, 84}, {7, 84}};
  for (auto& c : cfg) {
  probe<<<blocks, threads>>>(d, rounds, c[0], c[1]);
  cudaError_t e = cudaDeviceSynchronize();
  printf("stride %d slot %d: ", c[0], c[1]);
  uint32_t* h = (uint32_t*)malloc((size_t)blocks * threads * 8);
  cudaMemcpy(h, d, (size_t)blocks * threads * 8, cudaMemcpyDeviceToHost);
  unsigned long long bad = 0, cyc = 0;
  for (int i = 0; i < blocks * threads; ++i) { bad += h[2 * i]; cyc += h[2 * i + 1]; }
  printf("{\"err\": \"%s\", \"mismatches\": %llu, \"avg_cycles_per_round\": %.1f, "
         "\"cycles_per_tier_ldst_pair\": %.1f}\n", cudaGetErrorString(e), bad,
         (double)cyc / (blocks * threads) / rounds, (double)cyc / (blocks * threads) / rounds / 24.0);
  }
  return 0;
}
