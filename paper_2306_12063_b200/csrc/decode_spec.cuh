// decode_spec.cuh -- specialised layered min-sum kernels for the 18 standard
// base-matrix structures (12 Wi-Fi, 6 WiMAX), float32 and int16.
//
// Reference: /root/reference/pkg/src/qcldpc/_kernels.py:17-100 (float32),
// :103-186 (int16).  Results are bit-identical: every per-edge operation is
// the reference's, in the reference's order, and rows of one tier touch
// disjoint columns so running them concurrently changes nothing.
//
// Layout and mapping (B200, sm_100a):
//  * one thread = one check row r of every tier, for TWO codewords at once
//    (a "pair"); a CTA holds `pairs` pairs, i.e. pairs*Z threads;
//  * posteriors of a pair live in shared memory as [c][j] x {cw0, cw1}
//    (c = position inside the circulant, j = block column, row stride padded
//    to 25 elements so the Z lanes of a tier hit distinct banks); the cyclic
//    shift of edge (j, e) is an indexed shared-memory read at
//    j + ((r + e) mod Z) * 25 -- no expanded H anywhere;
//  * compressed check-node state (min1, min2, argmin, sign bitmap) stays in
//    registers for all tiers: the tier loop is unrolled at compile time from
//    the structure tables (structures_gen.cuh), shifts come from the kernel
//    parameter block (constant bank);
//  * one CTA barrier per tier (layered schedule).
#pragma once
#include <utility>

#include "common.cuh"
#include "kernels.h"

namespace qcb {

constexpr int kSpecMaxThreads = 384;
constexpr int kMaxPairsPerCta = 16;

// ---------------------------------------------------------------------------
// float32: exact reference row update for one codeword
// ---------------------------------------------------------------------------
struct F32Pair {
  static constexpr int ES = 8;        // bytes per (c, j) cell: float x 2 codewords
  using Cell = float2;
  struct State { float m1, m2; uint32_t sa; };  // sa: bits 0..26 sign bits ^ parity, 27..31 argmin
  using Val = float;
  // reference init: min1 = min2 = 0, argmin 0, no signs (_kernels.py:38-43)
  __device__ static State init_state() { return State{0.0f, 0.0f, 0u}; }

  __device__ static Val get(const Cell& c, int q) { return q ? c.y : c.x; }
  __device__ static void put(Cell& c, int q, Val v) { if (q) c.y = v; else c.x = v; }
  __device__ static bool hard(Val p) { return p <= 0.0f; }

  template <int D>
  __device__ __forceinline__ static void row(const Val (&p)[D], Val (&out)[D], State& s) {
    const int am = (int)(s.sa >> 27);
    Val zz[D];
    float nm1 = f_inf(), nm2 = f_inf();
    uint32_t nsb = 0;
#pragma unroll
    for (int k = 0; k < D; ++k) {                       // _kernels.py:61-75
      const float mag = (am == k) ? s.m2 : s.m1;
      const float lold = ((s.sa >> k) & 1u) ? -mag : mag;
      zz[k] = f_sub(p[k], lold);
      const float av = fabsf(zz[k]);
      nm2 = fminf(nm2, f_max_nan(nm1, av));              // == the if/elif update, NaN included
      nm1 = fminf(nm1, av);
      nsb |= (zz[k] < 0.0f) ? (1u << k) : 0u;
    }
    const uint32_t nsbx = nsb ^ (0u - (__popc(nsb) & 1u));  // sign of L_new_j = sp ^ bit j
    int nam = 0;
#pragma unroll
    for (int k = D - 1; k >= 0; --k) {                  // _kernels.py:76-79
      // |zz_k| == nm1 picks nm2; on ties nm2 == nm1 so the value equals the
      // reference's (k == argmin) choice
      const bool eq = fabsf(zz[k]) == nm1;
      const float mag = eq ? nm2 : nm1;
      nam = eq ? k : nam;
      const float lnew = ((nsbx >> k) & 1u) ? -mag : mag;
      out[k] = f_add(zz[k], lnew);
    }
    s.m1 = nm1;
    s.m2 = nm2;
    s.sa = (nsbx & 0x07FFFFFFu) | ((uint32_t)nam << 27);
  }
};

// ---------------------------------------------------------------------------
// int16 (wrap-around fixed point): values carried sign-extended in 32 bits
// ---------------------------------------------------------------------------
struct I16Pair {
  static constexpr int ES = 4;        // int16 x 2 codewords
  using Cell = uint32_t;
  struct State { uint32_t mk; uint32_t sa; };  // mk: key(min1) | key(min2) << 16
  using Val = int;
  // reference init min1 = min2 = 0 (_kernels.py:124-129); key(0) = 0x8000
  __device__ static State init_state() { return State{0x80008000u, 0u}; }

  __device__ static Val get(const Cell& c, int q) { return q ? ((int)c >> 16) : sext16((int)c); }
  __device__ static void put(Cell& c, int q, Val v) {
    c = q ? ((c & 0xFFFFu) | ((uint32_t)v << 16)) : ((c & 0xFFFF0000u) | ((uint32_t)v & 0xFFFFu));
  }
  __device__ static bool hard(Val p) { return p <= 0; }

  template <int D>
  __device__ __forceinline__ static void row(const Val (&p)[D], Val (&out)[D], State& s) {
    const int am = (int)(s.sa >> 27);
    const int v1 = i16_val_of_key(s.mk & 0xFFFFu), v2 = i16_val_of_key(s.mk >> 16);
    int zz[D];
    uint32_t key[D];
    uint32_t nm1 = kI16KeyInit, nm2 = kI16KeyInit;
    uint32_t nsb = 0;
#pragma unroll
    for (int k = 0; k < D; ++k) {                       // _kernels.py:147-161
      const int mag = (am == k) ? v2 : v1;
      const int lold = ((s.sa >> k) & 1u) ? -mag : mag;
      zz[k] = sext16(p[k] - lold);                      // np.int16(post - lold)
      key[k] = i16_key_of(zz[k]);                       // np.int16(abs(zz)) in unsigned order
      nm2 = min(nm2, max(nm1, key[k]));
      nm1 = min(nm1, key[k]);
      nsb |= (zz[k] < 0) ? (1u << k) : 0u;
    }
    const uint32_t nsbx = nsb ^ (0u - (__popc(nsb) & 1u));
    const int w1 = i16_val_of_key(nm1), w2 = i16_val_of_key(nm2);
    int nam = 0;
#pragma unroll
    for (int k = D - 1; k >= 0; --k) {                  // _kernels.py:162-165
      const bool eq = key[k] == nm1;
      const int mag = eq ? w2 : w1;
      nam = eq ? k : nam;
      const int lnew = ((nsbx >> k) & 1u) ? -mag : mag;
      out[k] = zz[k] + lnew;                            // wrapped at the 16-bit store
    }
    s.mk = nm1 | (nm2 << 16);
    s.sa = (nsbx & 0x07FFFFFFu) | ((uint32_t)nam << 27);
  }
};

template <class A>
__device__ __forceinline__ typename A::Cell lds_cell(uint32_t addr) {
  typename A::Cell c;
  if constexpr (sizeof(c) == 8) {
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(c.x), "=f"(c.y) : "r"(addr));
  } else {
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(c) : "r"(addr));
  }
  return c;
}
template <class A>
__device__ __forceinline__ void sts_cell(uint32_t addr, const typename A::Cell& c) {
  if constexpr (sizeof(c) == 8) {
    asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(addr), "f"(c.x), "f"(c.y) : "memory");
  } else {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(c) : "memory");
  }
}

template <class A>
__device__ __forceinline__ typename A::Val lds_val(uint32_t addr);
template <>
__device__ __forceinline__ float lds_val<F32Pair>(uint32_t addr) {
  float v; asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr)); return v;
}
template <>
__device__ __forceinline__ int lds_val<I16Pair>(uint32_t addr) {
  short v; asm volatile("ld.shared.s16 %0, [%1];" : "=h"(v) : "r"(addr)); return (int)v;
}

// address of edge `e` (tier-major entry index) of row r for this thread
__device__ __forceinline__ uint32_t edge_addr(const SpecArgs& a, int e, int r, uint32_t base) {
  const uint32_t u = base + (uint32_t)a.off[e];
  return r >= a.thr[e] ? u - (uint32_t)a.zrs : u;
}

template <class S, class A, bool ET>
struct SpecDecoder {
  using State = typename A::State;
  using Val = typename A::Val;
  using Cell = typename A::Cell;

  template <int T>
  __device__ __forceinline__ static void tier(const SpecArgs& a, int r, uint32_t base,
                                              State (&st)[2][S::MB], bool fz0, bool fz1) {
    constexpr int D = S::DEG[T];
    constexpr int E0 = S::START[T];
    uint32_t addr[D];
    Cell cell[D];
#pragma unroll
    for (int k = 0; k < D; ++k) {
      addr[k] = edge_addr(a, E0 + k, r, base);
      cell[k] = lds_cell<A>(addr[k]);
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      Val p[D], o[D];
#pragma unroll
      for (int k = 0; k < D; ++k) p[k] = A::get(cell[k], q);
      State s = st[q][T];
      A::template row<D>(p, o, s);
      const bool fz = q ? fz1 : fz0;
      if (!ET || !fz) {
        st[q][T] = s;
#pragma unroll
        for (int k = 0; k < D; ++k) A::put(cell[k], q, o[k]);
      }
    }
#pragma unroll
    for (int k = 0; k < D; ++k) sts_cell<A>(addr[k], cell[k]);
  }

  template <int T>
  __device__ __forceinline__ static uint32_t tier_parity(const SpecArgs& a, int r, uint32_t base) {
    constexpr int D = S::DEG[T];
    constexpr int E0 = S::START[T];
    uint32_t par = 0;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const Cell c = lds_cell<A>(edge_addr(a, E0 + k, r, base));
      par ^= (A::hard(A::get(c, 0)) ? 1u : 0u) | (A::hard(A::get(c, 1)) ? 2u : 0u);
    }
    return par;
  }

};

// per-tier sweep with barriers: expanded by hand via a fold over tiers
template <class S, class A, bool ET, int... Ts>
__device__ __forceinline__ void sweep_all(const SpecArgs& a, int r, uint32_t base,
                                          typename A::State (&st)[2][S::MB], bool act, bool fz0, bool fz1,
                                          std::integer_sequence<int, Ts...>) {
  ((act ? SpecDecoder<S, A, ET>::template tier<Ts>(a, r, base, st, fz0, fz1) : void(), __syncthreads()), ...);
}

template <class S, class A, int... Ts>
__device__ __forceinline__ uint32_t parity_all(const SpecArgs& a, int r, uint32_t base,
                                               std::integer_sequence<int, Ts...>) {
  return (SpecDecoder<S, A, false>::template tier_parity<Ts>(a, r, base) | ...);
}

template <class S, class A, bool ET>
__global__ void __launch_bounds__(kSpecMaxThreads) decode_spec_kernel(const __grid_constant__ SpecArgs a) {
  using State = typename A::State;
  using Val = typename A::Val;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int s_fail[2 * kMaxPairsPerCta];
  __shared__ int s_done[2 * kMaxPairsPerCta];
  __shared__ int s_iters[2 * kMaxPairsPerCta];
  __shared__ int s_active;

  constexpr int RS = kRowStrideUnits * A::ES;
  constexpr int TS = A::ES / 2;  // bytes per value
  const int Z = a.z, N = a.n;
  const int tid = threadIdx.x;
  const int g = tid / Z, r = tid - g * Z;
  const bool act = g < a.pairs;
  const int64_t cw0 = (int64_t)blockIdx.x * a.pairs * 2;
  const int ncw = (int)(a.w - cw0 < (int64_t)a.pairs * 2 ? a.w - cw0 : (int64_t)a.pairs * 2);
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t base = sbase + (uint32_t)(g * a.ps + r * RS);

  // ---- load channel LLRs into the transposed [pair][c][j] layout ----------
  {
    const int nthr = blockDim.x;
    const int dj = nthr / Z, dc = nthr - dj * Z;
    for (int q = 0; q < ncw; ++q) {
      const uint32_t cwbase = sbase + (uint32_t)((q >> 1) * a.ps + (q & 1) * TS);
      int j = tid / Z, c = tid - (tid / Z) * Z;
      if (TS == 4) {
        const float* src = reinterpret_cast<const float*>(a.llr) + (cw0 + q) * N;
        for (int n = tid; n < N; n += nthr) {
          const float v = __ldcs(src + n);
          asm volatile("st.shared.f32 [%0], %1;" ::"r"(cwbase + c * RS + j * A::ES), "f"(v));
          c += dc; j += dj;
          if (c >= Z) { c -= Z; ++j; }
        }
      } else {
        const short* src = reinterpret_cast<const short*>(a.llr) + (cw0 + q) * N;
        for (int n = tid; n < N; n += nthr) {
          const short v = __ldcs(src + n);
          asm volatile("st.shared.s16 [%0], %1;" ::"r"(cwbase + c * RS + j * A::ES), "h"(v));
          c += dc; j += dj;
          if (c >= Z) { c -= Z; ++j; }
        }
      }
    }
    // codeword slots past the end of the batch decode zeros (outputs dropped)
    for (int q = ncw; q < a.pairs * 2; ++q) {
      const uint32_t cwbase = sbase + (uint32_t)((q >> 1) * a.ps + (q & 1) * TS);
      for (int n = tid; n < N; n += blockDim.x) {
        const int j = n / Z, c = n - (n / Z) * Z;
        if (TS == 4) asm volatile("st.shared.f32 [%0], %1;" ::"r"(cwbase + c * RS + j * A::ES), "f"(0.0f));
        else asm volatile("st.shared.s16 [%0], %1;" ::"r"(cwbase + c * RS + j * A::ES), "h"((short)0));
      }
    }
    for (int q = tid; q < 2 * kMaxPairsPerCta; q += blockDim.x) {
      s_fail[q] = 1; s_done[q] = q >= ncw; s_iters[q] = 0;
    }
  }
  __syncthreads();

  State st[2][S::MB];
#pragma unroll
  for (int t = 0; t < S::MB; ++t) {
    st[0][t] = A::init_state();
    st[1][t] = A::init_state();
  }

  const auto tiers = std::make_integer_sequence<int, S::MB>{};
  for (int k = 0; k < a.max_iters; ++k) {
    bool fz0 = false, fz1 = false;
    if (ET) { fz0 = s_done[2 * g] != 0 && act; fz1 = s_done[2 * g + 1] != 0 && act; }
    sweep_all<S, A, ET>(a, r, base, st, act, fz0, fz1, tiers);
    const bool last = (k + 1 == a.max_iters);
    if (ET || last) {
      for (int q = tid; q < 2 * a.pairs; q += blockDim.x) s_fail[q] = 0;
      __syncthreads();
      if (act) {
        const uint32_t par = parity_all<S, A>(a, r, base, tiers);
        if (par & 1u) s_fail[2 * g] = 1;
        if (par & 2u) s_fail[2 * g + 1] = 1;
      }
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

  // ---- outputs --------------------------------------------------------------
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
      const uint32_t cwbase = sbase + (uint32_t)((q >> 1) * a.ps + (q & 1) * TS);
      uint32_t byte = 0;
      int n = b * 8;
      int j = n / Z, c = n - j * Z;
#pragma unroll
      for (int u = 0; u < 8; ++u, ++n) {
        const bool h = n < N && A::hard(lds_val<A>(cwbase + c * RS + j * A::ES));
        byte = (byte << 1) | (h ? 1u : 0u);
        if (++c == Z) { c = 0; ++j; }
      }
      hp[i] = (uint8_t)byte;
    }
  } else {
    uint8_t* h = reinterpret_cast<uint8_t*>(a.hard) + cw0 * N;
    for (int q = 0; q < ncw; ++q) {
      const uint32_t cwbase = sbase + (uint32_t)((q >> 1) * a.ps + (q & 1) * TS);
      for (int n4 = tid * 4; n4 < N; n4 += nthr * 4) {
        int j = n4 / Z, c = n4 - j * Z;
        uint32_t word = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const bool hb = (n4 + u) < N && A::hard(lds_val<A>(cwbase + c * RS + j * A::ES));
          word |= (hb ? 1u : 0u) << (8 * u);
          if (++c == Z) { c = 0; ++j; }
        }
        uint8_t* dst = h + (int64_t)q * N + n4;
        if (n4 + 4 <= N && (reinterpret_cast<uintptr_t>(dst) & 3u) == 0) *reinterpret_cast<uint32_t*>(dst) = word;
        else for (int u = 0; n4 + u < N; ++u) h[(int64_t)q * N + n4 + u] = (uint8_t)(word >> (8 * u));
      }
    }
  }
  if (a.post) {
    for (int q = 0; q < ncw; ++q) {
      const uint32_t cwbase = sbase + (uint32_t)((q >> 1) * a.ps + (q & 1) * TS);
      for (int n = tid; n < N; n += nthr) {
        const int j = n / Z, c = n - j * Z;
        const Val v = lds_val<A>(cwbase + c * RS + j * A::ES);
        if (TS == 4) reinterpret_cast<float*>(a.post)[(cw0 + q) * N + n] = (float)v;
        else reinterpret_cast<int16_t*>(a.post)[(cw0 + q) * N + n] = (int16_t)v;
      }
    }
  }
}

template <class S, class A, bool ET>
inline cudaError_t launch_one(const SpecArgs& a, cudaStream_t s) {
  const int threads = (a.pairs * a.z + 31) / 32 * 32;
  const size_t smem = (size_t)a.pairs * a.ps;
  auto kern = decode_spec_kernel<S, A, ET>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int64_t blocks = (a.w + 2 * a.pairs - 1) / (2 * a.pairs);
  if (blocks <= 0) return cudaSuccess;
  kern<<<(unsigned)blocks, threads, smem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace qcb
