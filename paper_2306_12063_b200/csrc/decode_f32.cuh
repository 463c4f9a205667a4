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

constexpr int kF32MaxThreads = 384;
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
// e = (|z| == nm1); sel = e ? n2 : n1; am += e ? bit : 0
__device__ __forceinline__ uint32_t sel_eq(float z, float nm1, uint32_t n1, uint32_t n2, uint32_t& am,
                                           uint32_t bit, uint32_t one) {
  uint32_t s;
  asm("{\n\t.reg .pred p;\n\t.reg .f32 t;\n\tabs.f32 t, %2;\n\tsetp.eq.f32 p, t, %3;\n\t"
      "selp.b32 %0, %5, %4, p;\n\t@p mad.lo.u32 %1, %6, %7, %1;\n\t}"
      : "=r"(s), "+r"(am) : "f"(z), "f"(nm1), "r"(n1), "r"(n2), "r"(bit), "r"(one));
  return s;
}

struct RowF32 {
  uint32_t m1s, m2s, wa, ws;
};

template <int D, bool PACK>
__device__ __forceinline__ void row_update_f32(const float (&p)[D], float (&o)[D], RowF32& s,
                                               uint32_t one, uint32_t sign, uint32_t shr) {
  const uint32_t wa = s.wa;
  uint32_t vs = PACK ? (s.wa >> 16) : s.ws;
  float zz[D];
  uint32_t nsb = 0;
  // ---- pass 1: L_old, zz = post - L_old, sign bits (_kernels.py:61-75) -----
#pragma unroll
  for (int k = 0; k < D; ++k) {
    const uint32_t msel = ((wa >> k) & 1u) ? s.m2s : s.m1s;
    const uint32_t lold = imad(vs, sign, msel);        // + ws_k * 2^31: sign of L_old
    vs = imulhi(vs, shr);                               // next bit
    zz[k] = f_sub(p[k], __uint_as_float(lold));
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
  uint32_t vn = nsb, am = 0;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    const uint32_t msel = sel_eq(zz[k], nm1, n1s, n2s, am, 1u << k, one);
    const uint32_t lnew = imad(vn, sign, msel);         // sign = parity ^ (zz_k < 0)
    vn = imulhi(vn, shr);
    o[k] = f_add(zz[k], __uint_as_float(lnew));
  }
  s.m1s = n1s;
  s.m2s = n2s;
  if (PACK) {
    s.wa = am | (nsb << 16);
  } else {
    s.wa = am;
    s.ws = nsb;
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
  static constexpr bool PACK = S::MAXDEG <= 16;

  template <int T>
  __device__ __forceinline__ static void tier(const SpecArgs& a, int r, uint32_t b0, uint32_t b1,
                                              RowF32 (&st)[S::MB]) {
    constexpr int D = S::DEG[T];
    constexpr int E0 = S::START[T];
    uint32_t addr[D];
    float p[D], o[D];
    tier_addrs<S, ZS, E0>(a, r, b0, b1, addr, std::make_integer_sequence<int, D>{});
#pragma unroll
    for (int k = 0; k < D; ++k) asm volatile("ld.shared.f32 %0, [%1];" : "=f"(p[k]) : "r"(addr[k]));
    row_update_f32<D, PACK>(p, o, st[T], a.k_one, a.k_sign, a.k_shr);
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
                                               RowF32 (&st)[S::MB], bool work, std::integer_sequence<int, Ts...>) {
    ((work ? tier<Ts>(a, r, b0, b1, st) : void(), __syncthreads()), ...);
  }

  template <int... Ts>
  __device__ __forceinline__ static uint32_t parity_all(const SpecArgs& a, int r, uint32_t b0, uint32_t b1,
                                                        std::integer_sequence<int, Ts...>) {
    return (parity<Ts>(a, r, b0, b1) | ...);
  }
};

#ifndef QCB_F32_MINB
#define QCB_F32_MINB 1
#endif
template <class S, int ZS, bool ET>
__global__ void __launch_bounds__(kF32MaxThreads, QCB_F32_MINB) decode_f32_kernel(const __grid_constant__ SpecArgs a) {
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

  RowF32 st[S::MB];
#pragma unroll
  for (int t = 0; t < S::MB; ++t) st[t] = RowF32{0u, 0u, 0u, 0u};  // min1 = min2 = 0, no signs

  const auto tiers = std::make_integer_sequence<int, S::MB>{};
  for (int k = 0; k < a.max_iters; ++k) {
    const bool work = act && !(ET && s_done[g]);
    Dec::sweep(a, r, b0, b1, st, work, tiers);
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
