// pipebench.cu -- measure sm_100a issue rates of the instructions the decoder
// is built from (lane-ops per clock per SM), to pick pipe-balanced
// formulations and to record the ALU roofline denominator.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pipebench tools/pipebench.cu
//   ./tools/pipebench            (prints one JSON line per instruction mix)
//
// Each kernel runs 8 independent dependency chains per thread (enough ILP to
// hide the 4-cycle latency) at full occupancy; the chains are written with
// inline PTX so the measured SASS is the intended instruction (checked with
// cuobjdump -sass).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 4096
#define CH 8

#define KERNEL(name, init, body, fin)                                               \
  __global__ void name(uint32_t* out, uint32_t k1, uint32_t k2) {                   \
    uint32_t r[CH];                                                                 \
    _Pragma("unroll") for (int c = 0; c < CH; ++c) r[c] = init;                     \
    for (int i = 0; i < ITERS; ++i) {                                               \
      _Pragma("unroll") for (int c = 0; c < CH; ++c) { body; }                      \
    }                                                                               \
    uint32_t acc = 0;                                                               \
    _Pragma("unroll") for (int c = 0; c < CH; ++c) acc ^= fin;                      \
    if (acc == 0x12345678u) out[0] = acc;                                           \
  }

#define A(x) asm volatile(x : "+r"(r[c]) : "r"(k1 + (uint32_t)i), "r"(k2))

KERNEL(k_iadd3, threadIdx.x + c, A("add.u32 %0, %0, %1;"), r[c])
KERNEL(k_lop3, threadIdx.x + c, A("xor.b32 %0, %0, %1;"), r[c])
KERNEL(k_imad, threadIdx.x + c, A("mad.lo.u32 %0, %0, %1, %2;"), r[c])
KERNEL(k_imadhi, threadIdx.x + c, A("mad.hi.u32 %0, %0, %1, %2;"), r[c])
KERNEL(k_vadd2, threadIdx.x + c, A("add.s16x2 %0, %0, %1;"), r[c])
KERNEL(k_vmin2, threadIdx.x + c, A("min.s16x2 %0, %0, %1;"), r[c])
KERNEL(k_umin, threadIdx.x + c, A("min.u32 %0, %0, %1;"), r[c])
KERNEL(k_prmt, threadIdx.x + c, A("prmt.b32 %0, %0, %1, 0x3210;"), r[c])
KERNEL(k_shf, threadIdx.x + c, A("shf.l.wrap.b32 %0, %0, %1, 3;"), r[c])
KERNEL(k_sel, threadIdx.x + c,
       asm volatile("{.reg .pred p; setp.ne.u32 p, %1, 0; selp.b32 %0, %0, %2, p;}" : "+r"(r[c]) : "r"(k1 & (uint32_t)i), "r"(k2)),
       r[c])
KERNEL(k_fadd, __float_as_uint((float)(threadIdx.x + c)),
       asm volatile("{.reg .f32 t; mov.b32 t, %0; add.rn.f32 t, t, 0f3F800000; mov.b32 %0, t;}" : "+r"(r[c]) : "r"(k1), "r"(k2)),
       r[c])
KERNEL(k_fmnmx, __float_as_uint((float)(threadIdx.x + c)),
       asm volatile("{.reg .f32 t, u; mov.b32 t, %0; mov.b32 u, %1; min.f32 t, t, u; mov.b32 %0, t;}" : "+r"(r[c]) : "r"(k1 + (uint32_t)i), "r"(k2)),
       r[c])
KERNEL(k_iadd_fadd, threadIdx.x + c,
       if (c & 1) { A("add.u32 %0, %0, %1;"); } else {
         asm volatile("{.reg .f32 t; mov.b32 t, %0; add.rn.f32 t, t, 0f3F800000; mov.b32 %0, t;}" : "+r"(r[c]) : "r"(k1), "r"(k2)); },
       r[c])
KERNEL(k_lop3_imad, threadIdx.x + c,
       if (c & 1) { A("xor.b32 %0, %0, %1;"); } else { A("mad.lo.u32 %0, %0, %1, %2;"); },
       r[c])
KERNEL(k_vadd2_imad, threadIdx.x + c,
       if (c & 1) { A("add.s16x2 %0, %0, %1;"); } else { A("mad.lo.u32 %0, %0, %1, %2;"); },
       r[c])
KERNEL(k_vmin2_fadd, threadIdx.x + c,
       if (c & 1) { A("min.s16x2 %0, %0, %1;"); } else {
         asm volatile("{.reg .f32 t; mov.b32 t, %0; add.rn.f32 t, t, 0f3F800000; mov.b32 %0, t;}" : "+r"(r[c]) : "r"(k1), "r"(k2)); },
       r[c])
KERNEL(k_imad_fadd, threadIdx.x + c,
       if (c & 1) { A("mad.lo.u32 %0, %0, %1, %2;"); } else {
         asm volatile("{.reg .f32 t; mov.b32 t, %0; add.rn.f32 t, t, 0f3F800000; mov.b32 %0, t;}" : "+r"(r[c]) : "r"(k1), "r"(k2)); },
       r[c])

typedef void (*kern_t)(uint32_t*, uint32_t, uint32_t);

int main() {
  struct { const char* name; kern_t k; } ks[] = {
      {"IADD3(add.u32)", k_iadd3}, {"LOP3(xor)", k_lop3}, {"IMAD", k_imad}, {"IMAD.HI", k_imadhi},
      {"VIADD.16x2", k_vadd2}, {"VIMNMX.S16x2", k_vmin2}, {"IMNMX.U32", k_umin}, {"PRMT", k_prmt},
      {"SHF", k_shf}, {"ISETP+SEL", k_sel}, {"FADD", k_fadd}, {"FMNMX", k_fmnmx},
      {"IADD3|FADD", k_iadd_fadd}, {"LOP3|IMAD", k_lop3_imad}, {"VIADD2|IMAD", k_vadd2_imad},
      {"VIMNMX2|FADD", k_vmin2_fadd}, {"IMAD|FADD", k_imad_fadd},
  };
  int dev = 0, sms = 0, clk_khz = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  uint32_t* out;
  cudaMalloc(&out, 64);
  const int threads = 1024, blocks = sms * 2;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (auto& k : ks) {
    k.k<<<blocks, threads>>>(out, 3u, 5u);
    cudaEventRecord(a);
    for (int rep = 0; rep < 3; ++rep) k.k<<<blocks, threads>>>(out, 3u, 5u);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double ops = 3.0 * blocks * threads * (double)ITERS * CH;   // lane-ops
    const double per_s = ops / (ms * 1e-3);
    const double per_clk_sm = per_s / (clk_khz * 1e3) / sms;
    printf("{\"op\": \"%s\", \"lane_ops_per_s\": %.4g, \"lane_ops_per_clk_per_sm_at_max_clock\": %.1f, \"ms\": %.3f}\n",
           k.name, per_s, per_clk_sm, ms);
  }
  printf("{\"sms\": %d, \"clock_khz_max\": %d, \"err\": \"%s\"}\n", sms, clk_khz, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
