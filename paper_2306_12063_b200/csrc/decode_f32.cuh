// decode_f32.cuh -- float32 layered min-sum, one thread per check row per
// codeword, pipe-balanced for sm_100a.
//
// Reference: /root/reference/pkg/src/qcldpc/_kernels.py:17-100.  Bit-exact:
// every value the reference computes (zz = post - L_old, |zz|, min1/min2,
// L_new, post = zz + L_new, hard = post <= 0) is computed by the same IEEE
// float32 operation on the same operands; only *how* the selections are made
// differs.
//
// Why this shape (measured with ncu on B200, profiles/):
//  * the decoder is issue bound; compare/select/logic/min-max instructions
//    run on the half-rate ALU pipe (64 lanes/clk/SM) while FADD and IMAD run
//    on the full-rate FMA pipe, so selections that are not comparisons are
//    routed to the FMA pipe: sign flips of L_old / L_new are integer adds of
//    2^31 to the float bit pattern (IMAD with the sign bit of a bit stream),
//    bit streams advance with IMAD.HI, and the sign/argmin bitmaps are built
//    with predicated IMADs;
//  * min1/min2 are tracked two edges at a time (lo/hi of the pair, then one
//    3-input min): 2.5 min/max instructions per edge instead of 3, NaN
//    handled like the reference's if/elif (max.NaN keeps NaN out of min2);
//  * L_new's magnitude is nm2 exactly when |zz_j| == nm1 (on a tie nm2 ==
//    nm1), so no argmin index is tracked in pass 1;
//  * compressed check-node state per row stays in registers:
//      m1s, m2s : min1 / min2 bit patterns with the row's sign parity in bit 31
//      wa       : bit j set when edge j took min2 (argmin, any on ties)
//      ws       : bit j = (zz_j < 0) of the last update (packed into wa's
//                 upper half when the row degree is <= 16)
//    so L_old_j = (wa_j ? m2s : m1s) + ws_j * 2^31  (mod 2^32);
//  * one codeword per thread keeps the fully unrolled tier loop inside the
//    32 KB L1.5 instruction cache (two codewords per thread thrashed it:
//    "no_instructions" was the top stall reason);
//  * native codes (the 18 base matrices at their own Z) get compile-time Z
//    and shifts: an edge address is one ISETP + one SEL, the circulant offset
//    is the LDS immediate.
#pragma once
#include <cstdlib>
#include <utility>

#include "common.cuh"
#include "kernels.h"

namespace qcb {

#ifndef QCB_F32_MAXT
#define QCB_F32_MAXT 384
#endif
constexpr int kF32MaxThreads = QCB_F32_MAXT;
constexpr int kF32MaxCw = 16;

// integer ops kept on the FMA pipe: the multipliers come from the parameter
// block (constant bank), so ptxas cannot strength-reduce them into ALU shifts
__device__ __forceinline__ uint32_t imad(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ uint32_t imulhi(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("mul.hi.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
// acc += bit if z < 0 (exact "< 0": -0.0 and NaN do not count, _kernels.py:73)
__device__ __forceinline__ void add_if_neg(uint32_t& acc, float z, uint32_t bit, uint32_t one) {
  asm("{\n\t.reg .pred p;\n\tsetp.lt.f32 p, %1, 0f00000000;\n\t@p mad.lo.u32 %0, %2, %3, %0;\n\t}"
      : "+r"(acc) : "f"(z), "r"(bit), "r"(one));
}
// |z| == nm1 ? n2 : n1   (nm2 exactly when edge k was the/an argmin; on a tie
// nm2 == nm1, so this equals the reference's (k == argmin) choice)
__device__ __forceinline__ uint32_t sel_eq(float z, float nm1, uint32_t n1, uint32_t n2) {
  return fabsf(z) == nm1 ? n2 : n1;
}

// One check row's update with explicit check-to-variable messages.
// msg[k] holds L_mn of edge k from the previous sweep (L_old); it is
// replaced by L_new.  The reference keeps the same information compressed
// (min1, min2, argmin, sign bitmap, parity; _kernels.py:80-84) and
// reconstructs L_old from it (:62-63); holding the reconstructed values in
// registers instead removes that reconstruction from the inner loop and is
// bit-identical: L_old_k of sweep i+1 *is* L_new_k of sweep i.
template <int D>
__device__ __forceinline__ void row_update_f32(const float (&p)[D], float (&o)[D], float* msg,
                                               uint32_t one, uint32_t sign, uint32_t shr) {
  float zz[D];
  uint32_t nsb = 0;
  // ---- pass 1: zz = post - L_old, sign bits (_kernels.py:61-75) -------------
#pragma unroll
  for (int k = 0; k < D; ++k) {
    zz[k] = f_sub(p[k], msg[k]);
    add_if_neg(nsb, zz[k], 1u << k, one);
  }
  // ---- min1 / min2 over |zz| (two edges per step) ---------------------------
  float nm1 = f_inf(), nm2 = f_inf();
#pragma unroll
  for (int k = 0; k + 1 < D; k += 2) {
    const float x = fabsf(zz[k]), y = fabsf(zz[k + 1]);
    const float lo = fminf(x, y), hi = f_max_nan(x, y);
    nm2 = fminf(nm2, fminf(hi, f_max_nan(nm1, lo)));
    nm1 = fminf(nm1, lo);
  }
  if (D & 1) {
    const float x = fabsf(zz[D - 1]);
    nm2 = fminf(nm2, f_max_nan(nm1, x));
    nm1 = fminf(nm1, x);
  }
  // ---- pass 2: L_new and post = zz + L_new (_kernels.py:76-79) -------------
  const uint32_t ps = imad(__popc(nsb), sign, 0u);      // sign-product parity in bit 31
  const uint32_t n1s = __float_as_uint(nm1) + ps, n2s = __float_as_uint(nm2) + ps;
  uint32_t vn = nsb;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    const uint32_t msel = sel_eq(zz[k], nm1, n1s, n2s);
    const float lnew = __uint_as_float(imad(vn, sign, msel));   // sign = parity ^ (zz_k < 0)
    vn = imulhi(vn, shr);
    msg[k] = lnew;
    o[k] = f_add(zz[k], lnew);
  }
}

// byte offset of cell (c, j) inside a codeword's block: row stride 25 words
constexpr int kRsF32 = kRowStrideUnits * 4;

template <class S, int ZS, int E>
__device__ __forceinline__ uint32_t edge_addr_f32(const SpecArgs& a, int r, uint32_t b0, uint32_t b1) {
  if constexpr (ZS > 0) {
    constexpr int sh = S::SHIFT0[E];
    constexpr uint32_t off = (uint32_t)((sh * kRowStrideUnits + S::COL[E]) * 4);
    if constexpr (sh == 0) return b0 + off;
    else return (r >= ZS - sh ? b1 : b0) + off;
  } else {
    return (r >= a.thr[E] ? b1 : b0) + (uint32_t)a.off[E];
  }
}

template <class S, int ZS, int E0, int... Ks>
__device__ __forceinline__ void tier_addrs(const SpecArgs& a, int r, uint32_t b0, uint32_t b1, uint32_t* addr,
                                           std::integer_sequence<int, Ks...>) {
  ((addr[Ks] = edge_addr_f32<S, ZS, E0 + Ks>(a, r, b0, b1)), ...);
}

template <class S, int ZS, bool ET>
struct F32Decoder {
  template <int T>
  __device__ __forceinline__ static void tier(const SpecArgs& a, int r, uint32_t b0, uint32_t b1,
                                              float (&msg)[S::NE]) {
    constexpr int D = S::DEG[T];
    constexpr int E0 = S::START[T];
    uint32_t addr[D];
    float p[D], o[D];
    tier_addrs<S, ZS, E0>(a, r, b0, b1, addr, std::make_integer_sequence<int, D>{});
#pragma unroll
    for (int k = 0; k < D; ++k) asm volatile("ld.shared.f32 %0, [%1];" : "=f"(p[k]) : "r"(addr[k]));
    row_update_f32<D>(p, o, msg + E0, a.k_one, a.k_sign, a.k_shr);
#pragma unroll
    for (int k = 0; k < D; ++k) asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr[k]), "f"(o[k]) : "memory");
  }

  template <int T>
  __device__ __forceinline__ static uint32_t parity(const SpecArgs& a, int r, uint32_t b0, uint32_t b1) {
    constexpr int D = S::DEG[T];
    constexpr int E0 = S::START[T];
    uint32_t addr[D];
    tier_addrs<S, ZS, E0>(a, r, b0, b1, addr, std::make_integer_sequence<int, D>{});
    uint32_t par = 0;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      float v;
      asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr[k]));
      par ^= v <= 0.0f ? 1u : 0u;
    }
    return par;
  }

  template <int... Ts>
  __device__ __forceinline__ static void sweep(const SpecArgs& a, int r, uint32_t b0, uint32_t b1,
                                               float (&msg)[S::NE], bool work, std::integer_sequence<int, Ts...>) {
    ((work ? tier<Ts>(a, r, b0, b1, msg) : void(), __syncthreads()), ...);
  }

  template <int... Ts>
  __device__ __forceinline__ static uint32_t parity_all(const SpecArgs& a, int r, uint32_t b0, uint32_t b1,
                                                        std::integer_sequence<int, Ts...>) {
    return (parity<Ts>(a, r, b0, b1) | ...);
  }
};

// Register cap: the messages (S::NE floats) plus ~52 for the widest tier's
// transients.  Measured on C2 (NE = 76): 161 regs uncapped -> 4 CTAs of 96
// threads per SM, 45.9 Gb/s; capped at 128 -> 5 CTAs, 50.3 Gb/s; capped at
// 96 -> spills, 43.0 Gb/s.
#ifndef QCB_F32_REG_SLACK
#define QCB_F32_REG_SLACK 52
#endif
template <class S>
constexpr int f32_reg_cap() {
  return (S::NE + QCB_F32_REG_SLACK + 7) / 8 * 8 > 255 ? 255 : (S::NE + QCB_F32_REG_SLACK + 7) / 8 * 8;
}
template <class S, int ZS, bool ET>
__global__ void __launch_bounds__(kF32MaxThreads) __maxnreg__(f32_reg_cap<S>()) decode_f32_kernel(const __grid_constant__ SpecArgs a) {
  using Dec = F32Decoder<S, ZS, ET>;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int s_fail[kF32MaxCw], s_done[kF32MaxCw], s_iters[kF32MaxCw];
  __shared__ int s_active;

  const int Z = ZS > 0 ? ZS : a.z;
  const int N = S::NB * Z;
  const int G = a.pairs;                       // codewords per CTA (one per thread row group)
  const int tid = threadIdx.x;
  const int g = tid / Z, r = tid - g * Z;
  const int64_t cw0 = (int64_t)blockIdx.x * G;
  const int ncw = (int)(a.w - cw0 < (int64_t)G ? a.w - cw0 : (int64_t)G);
  const bool act = g < ncw;
  const uint32_t cws = (uint32_t)(Z * kRsF32);   // bytes per codeword block
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  // opaque copies: keeps the row bases in registers instead of letting the
  // compiler rematerialise them (S2R + LEA + IMAD) in every tier
  uint32_t b0 = sbase + (uint32_t)g * cws + (uint32_t)(r * kRsF32), b1;
  asm volatile("mov.b32 %0, %0;" : "+r"(b0));
  asm volatile("sub.u32 %0, %1, %2;" : "=r"(b1) : "r"(b0), "r"(cws));

  // ---- load channel LLRs (coalesced) into [cw][c][j] ------------------------
  {
    const int nthr = blockDim.x;
    const int dj = nthr / Z, dc = nthr - dj * Z;
    const float* src = reinterpret_cast<const float*>(a.llr) + cw0 * N;
    for (int q = 0; q < ncw; ++q) {
      const uint32_t cb = sbase + (uint32_t)q * cws;
      int j = tid / Z, c = tid - (tid / Z) * Z;
      for (int n = tid; n < N; n += nthr) {
        const float v = __ldcs(src + (int64_t)q * N + n);
        asm volatile("st.shared.f32 [%0], %1;" ::"r"(cb + c * kRsF32 + j * 4), "f"(v));
        c += dc; j += dj;
        if (c >= Z) { c -= Z; ++j; }
      }
    }
    for (int q = tid; q < kF32MaxCw; q += blockDim.x) {
      s_fail[q] = 1; s_done[q] = q >= ncw; s_iters[q] = 0;
    }
  }
  __syncthreads();

  // check-to-variable messages of this thread's rows, all tiers (registers);
  // the reference starts from min1 = min2 = 0 with no signs: L = +0.0
  float msg[S::NE];
#pragma unroll
  for (int e = 0; e < S::NE; ++e) msg[e] = 0.0f;

  const auto tiers = std::make_integer_sequence<int, S::MB>{};
  for (int k = 0; k < a.max_iters; ++k) {
    const bool work = act && !(ET && s_done[g]);
    Dec::sweep(a, r, b0, b1, msg, work, tiers);
    const bool last = (k + 1 == a.max_iters);
    if (ET || last) {
      if (tid < kF32MaxCw) s_fail[tid] = 0;
      __syncthreads();
      if (work && Dec::parity_all(a, r, b0, b1, tiers)) s_fail[g] = 1;
      __syncthreads();
    }
    if (tid == 0) s_active = 0;
    __syncthreads();
    if (tid < ncw && !s_done[tid]) {
      s_iters[tid] = k + 1;
      if (ET && !s_fail[tid]) s_done[tid] = 1;
      else s_active = 1;
    }
    __syncthreads();
    if (!s_active) break;
  }

  // ---- outputs ----------------------------------------------------------------
  if (tid < ncw) {
    a.iters[cw0 + tid] = s_iters[tid];
    a.conv[cw0 + tid] = (a.max_iters > 0 && !s_fail[tid]) ? 1 : 0;
  }
  const int nthr = blockDim.x;
  if (a.hard_packed) {
    const int nbytes = (N + 7) >> 3;
    uint8_t* hp = reinterpret_cast<uint8_t*>(a.hard) + cw0 * nbytes;
    for (int i = tid; i < ncw * nbytes; i += nthr) {
      const int q = i / nbytes, b = i - q * nbytes;
      const uint32_t cb = sbase + (uint32_t)q * cws;
      uint32_t byte = 0;
      int n = b * 8;
      int j = n / Z, c = n - j * Z;
#pragma unroll
      for (int u = 0; u < 8; ++u, ++n) {
        float v = 1.0f;
        if (n < N) asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(cb + c * kRsF32 + j * 4));
        byte = (byte << 1) | (v <= 0.0f ? 1u : 0u);
        if (++c == Z) { c = 0; ++j; }
      }
      hp[i] = (uint8_t)byte;
    }
  } else {
    uint8_t* h = reinterpret_cast<uint8_t*>(a.hard) + cw0 * N;
    for (int q = 0; q < ncw; ++q) {
      const uint32_t cb = sbase + (uint32_t)q * cws;
      for (int n4 = tid * 4; n4 < N; n4 += nthr * 4) {
        int j = n4 / Z, c = n4 - j * Z;
        uint32_t word = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          float v = 1.0f;
          if (n4 + u < N) asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(cb + c * kRsF32 + j * 4));
          word |= (v <= 0.0f ? 1u : 0u) << (8 * u);
          if (++c == Z) { c = 0; ++j; }
        }
        uint8_t* dst = h + (int64_t)q * N + n4;
        if (n4 + 4 <= N && (reinterpret_cast<uintptr_t>(dst) & 3u) == 0) *reinterpret_cast<uint32_t*>(dst) = word;
        else for (int u = 0; n4 + u < N; ++u) dst[u] = (uint8_t)(word >> (8 * u));
      }
    }
  }
  if (a.post) {
    float* po = reinterpret_cast<float*>(a.post) + cw0 * N;
    for (int q = 0; q < ncw; ++q) {
      const uint32_t cb = sbase + (uint32_t)q * cws;
      for (int n = tid; n < N; n += nthr) {
        const int j = n / Z, c = n - j * Z;
        float v;
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(cb + c * kRsF32 + j * 4));
        po[(int64_t)q * N + n] = v;
      }
    }
  }
}

inline int f32_cw_per_cta(int z) {
  if (const char* env = getenv("QCB_F32_CW")) {   // tuning knob (benchmarks only)
    const int v = atoi(env);
    if (v >= 1 && v <= kF32MaxCw && v * z <= kF32MaxThreads) return v;
  }
  int best = 1;
  double best_eff = 0.0;
  for (int p = 1; p <= kF32MaxCw; ++p) {
    const int thr = p * z;
    if (thr > kF32MaxThreads) break;
    const int padded = (thr + 31) / 32 * 32;
    double eff = (double)thr / padded;
    if (thr > 160) eff *= 0.97;      // small CTAs: one barrier per tier costs less
    if (eff > best_eff + 1e-9) { best_eff = eff; best = p; }
  }
  return best;
}

template <class S, int ZS, bool ET>
inline cudaError_t launch_f32(const SpecArgs& a, cudaStream_t s) {
  const int z = ZS > 0 ? ZS : a.z;
  const int threads = (a.pairs * z + 31) / 32 * 32;
  const size_t smem = (size_t)a.pairs * z * kRsF32;
  auto kern = decode_f32_kernel<S, ZS, ET>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int64_t blocks = (a.w + a.pairs - 1) / a.pairs;
  if (blocks <= 0) return cudaSuccess;
  kern<<<(unsigned)blocks, threads, smem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace qcb
