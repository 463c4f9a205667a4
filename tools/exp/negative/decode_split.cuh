// NEGATIVE RESULT, NOT BUILT (kept for the record).
// Measured on B200, all parity tests passing (QCB_SPLIT=1): C1 (Wi-Fi 648 R1/2,
// 1024 codewords) 21.8 Gb/s against 29.3 for one lane per row: the two lanes of
// a row read different block columns, so a warp's 32 accesses are two
// unrelated 16-row bank patterns (28 % of shared wavefronts were conflicts,
// short-scoreboard stalls 40 %), and the address table adds a dependent load.
// decode_split.cuh -- small-batch float32 layered decoder: TWO lanes per
// check row.
//
// Same bit-exact row update as decode_layered.cuh (_kernels.py:49-84), for
// batches too small to fill the GPU (BASELINE C1: 1024 codewords = 7
// one-warp CTAs per SM, latency-bound).  Lanes 2r and 2r+1 of a warp share
// row r of every tier: each takes half of the row's edges (lane 0 the first
// ceil(D/2), lane 1 the rest plus, for odd D, a dummy slot reading a cell that
// holds +inf and is never written).  Each lane forms the leave-one-out minima
// of its own half, the lanes swap their half-minimum and sign parity with one
// __shfl_xor each, and |L_new_k| = min(own leave-one-out, partner's minimum)
// -- the same min over j != k, NaN-ignoring and +inf seeded, so the result is
// the reference's.  Twice the threads, half the dependent chain per tier and
// half the message registers per thread.  Addresses come from a per-thread
// shared-memory table (the two lanes of a pair touch different edges).
#pragma once
#include "decode_layered.cuh"

namespace qcb {

template <class S>
struct SplitPlan {
  static constexpr int half(int t) { return (S::DEG[t] + 1) / 2; }   // slots per lane in tier t
  static constexpr int slot0(int t) {
    int s = 0;
    for (int i = 0; i < t; ++i) s += half(i);
    return s;
  }
  static constexpr int slots() { return slot0(S::MB); }
  static constexpr int unit0(int t) {
    int u = 0;
    for (int i = 0; i < t; ++i) u += (half(i) + 1) / 2;
    return u;
  }
  static constexpr int units() { return unit0(S::MB) | 1; }          // odd: conflict-free LDS.64
  static constexpr int maxhalf() {
    int m = 1;
    for (int t = 0; t < S::MB; ++t) m = half(t) > m ? half(t) : m;
    return m;
  }
};

template <class S, int ZS, int T, int I>
__device__ __forceinline__ uint32_t split_pick(const SpecArgs& a, int r, uint32_t b0, uint32_t b1, int h,
                                               uint32_t dummy) {
  using SP = SplitPlan<S>;
  constexpr int H = SP::half(T);
  const uint32_t x0 = edge_addr<S, ArithF32, ZS, S::START[T] + I>(a, r, b0, b1);
  if constexpr (H + I < S::DEG[T]) {
    const uint32_t x1 = edge_addr<S, ArithF32, ZS, S::START[T] + H + I>(a, r, b0, b1);
    return h ? x1 : x0;
  } else {
    return h ? dummy : x0;
  }
}
template <class S, int ZS, int T, int... Is>
__device__ __forceinline__ void split_fill_tier(const SpecArgs& a, int r, uint32_t b0, uint32_t b1, int h,
                                                uint32_t dummy, uint32_t* ent, std::integer_sequence<int, Is...>) {
  ((ent[2 * SplitPlan<S>::unit0(T) + Is] = split_pick<S, ZS, T, Is>(a, r, b0, b1, h, dummy)), ...);
}
template <class S, int ZS, int... Ts>
__device__ __forceinline__ void split_fill(const SpecArgs& a, int r, uint32_t b0, uint32_t b1, int h,
                                           uint32_t dummy, uint32_t tab, std::integer_sequence<int, Ts...>) {
  constexpr int NU = SplitPlan<S>::units();
  uint32_t ent[2 * NU];
#pragma unroll
  for (int i = 0; i < 2 * NU; ++i) ent[i] = dummy;
  (split_fill_tier<S, ZS, Ts>(a, r, b0, b1, h, dummy, ent,
                              std::make_integer_sequence<int, SplitPlan<S>::half(Ts)>{}), ...);
#pragma unroll
  for (int u = 0; u < NU; ++u) sts64(tab + (uint32_t)(u * 8), ent[2 * u], ent[2 * u + 1]);
}

template <class S>
struct SplitRow {
  using SP = SplitPlan<S>;

  static constexpr int MA = SP::maxhalf() + 1;

  template <int T>
  __device__ __forceinline__ static void fetch(uint32_t tab, uint32_t (&addr)[MA]) {
    if constexpr (T < S::MB) {
    constexpr int H = SP::half(T);
#pragma unroll
    for (int u = 0; u < (H + 1) / 2; ++u) {
      const uint2 v = lds64(tab + (uint32_t)((SP::unit0(T) + u) * 8));
      addr[2 * u] = v.x;
      addr[2 * u + 1] = v.y;
    }
    }
  }

  // tier T for this lane's H slots; h = lane parity (0: first half of the row);
  // addr = this tier's addresses (fetched a tier ahead), an = the next tier's
  template <int T>
  __device__ __forceinline__ static void tier(const RtK& K, int h, uint32_t tab, float* msg, uint32_t (&addr)[MA],
                                              uint32_t (&an)[MA]) {
    constexpr int H = SP::half(T);
    constexpr bool ODD = (S::DEG[T] & 1) != 0;
    float p[H], zz[H];
#pragma unroll
    for (int i = 0; i < H; ++i) p[i] = ArithF32::lds(addr[i]);
    fetch<T + 1>(tab, an);
#pragma unroll
    for (int i = 0; i + 1 < H; i += 2) f_sub2(p[i], p[i + 1], msg[i], msg[i + 1], zz[i], zz[i + 1]);
    if (H & 1) zz[H - 1] = f_sub(p[H - 1], msg[H - 1]);
    uint32_t sx = 0;
#pragma unroll
    for (int i = 0; i < H; ++i) sx ^= __float_as_uint(zz[i]);
    // own leave-one-out minima and own minimum (+inf seeded, NaN-ignoring)
    float ex[H], pre[H + 1];
    pre[0] = f_inf();
#pragma unroll
    for (int i = 0; i < H; ++i) pre[i + 1] = fminf(pre[i], fabsf(zz[i]));
    float suf = f_inf();
#pragma unroll
    for (int i = H - 1; i >= 0; --i) {
      ex[i] = fminf(pre[i], suf);
      suf = fminf(suf, fabsf(zz[i]));
    }
    const float mo = __shfl_xor_sync(0xffffffffu, pre[H], 1);        // partner's half-minimum
    const uint32_t so = __shfl_xor_sync(0xffffffffu, sx, 1);         // partner's sign parity
    const uint32_t sxm = (sx ^ so) & 0x80000000u;
#pragma unroll
    for (int i = 0; i < H; ++i) {
      const float e = fminf(ex[i], mo);
      uint32_t t;
      asm("lop3.b32 %0, %1, %2, 0x80000000, 0x28;" : "=r"(t) : "r"(__float_as_uint(zz[i])), "r"(sxm));
      msg[i] = __uint_as_float(imad(t, K.one, __float_as_uint(e)));
    }
    float o[H];
#pragma unroll
    for (int i = 0; i + 1 < H; i += 2) f_add2(zz[i], zz[i + 1], msg[i], msg[i + 1], o[i], o[i + 1]);
    if (H & 1) o[H - 1] = f_add(zz[H - 1], msg[H - 1]);
#pragma unroll
    for (int i = 0; i < H; ++i) {
      if (ODD && i == H - 1) {
        if (!h) ArithF32::sts(addr[i], o[i]);                        // lane 1's slot is the dummy
      } else {
        ArithF32::sts(addr[i], o[i]);
      }
    }
  }

  template <int T>
  __device__ __forceinline__ static uint32_t parity(uint32_t tab) {
    constexpr int H = SP::half(T);
    uint32_t addr[MA];
    fetch<T>(tab, addr);
    uint32_t par = 0;
#pragma unroll
    for (int i = 0; i < H; ++i) par ^= ArithF32::hard(ArithF32::lds(addr[i])) ? 1u : 0u;   // dummy: +inf -> 0
    return par;
  }

  template <bool ET, int... Ts>
  __device__ __forceinline__ static void sweep(const RtK& K, int h, uint32_t tab, float (&msg)[SP::slots()],
                                               bool work, std::integer_sequence<int, Ts...>) {
    uint32_t aa[MA], ab[MA];
    fetch<0>(tab, aa);
    (void)work;
    ((tier<Ts>(K, h, tab, msg + SP::slot0(Ts), (Ts & 1) ? ab : aa, (Ts & 1) ? aa : ab), __syncthreads()), ...);
  }
  // bit T = this lane's parity share of its row in tier T (the row's check is
  // the XOR with the partner lane's share, tier by tier)
  template <int... Ts>
  __device__ __forceinline__ static uint32_t parity_all(uint32_t tab, std::integer_sequence<int, Ts...>) {
    return ((parity<Ts>(tab) << Ts) | ...);
  }
};

template <class S>
constexpr int split_reg_cap() {
  const int want = SplitPlan<S>::slots() + 56;
  return (want + 7) / 8 * 8 > 255 ? 255 : (want + 7) / 8 * 8;
}

// one codeword per CTA, 2 lanes per row: blockDim = 32 * ceil(2Z / 32)
template <class S, int ZS, bool ET>
__global__ void __launch_bounds__(kLayMaxThreads) __maxnreg__((split_reg_cap<S>()))
    decode_split_kernel(const __grid_constant__ SpecArgs a) {
  using SR = SplitRow<S>;
  constexpr int RS = row_stride_bytes<ArithF32>();
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int s_fail;

  const RtK K{a.k_one, a.k_sign, a.k_shr, a.k_neg1, a.k_lane1};
  const int Z = ZS > 0 ? ZS : a.z;
  const int N = S::NB * Z;
  const int tid = threadIdx.x;
  const int64_t cw = blockIdx.x;
  const uint32_t cws = (uint32_t)((Z * RS + 15) & ~15);
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  // padding lanes shadow same-warp lanes of the same parity (see decode_layered_kernel)
  const int twin = tid < 2 * Z ? tid : (tid & ~31) + ((tid & 31) % (2 * Z - (tid & ~31)));
  const int h = twin & 1, rs = twin >> 1;
  uint32_t b0 = sbase + (uint32_t)(rs * RS), b1;
  asm volatile("mov.b32 %0, %0;" : "+r"(b0));
  asm volatile("sub.u32 %0, %1, %2;" : "=r"(b1) : "r"(b0), "r"((uint32_t)(Z * RS)));
  const uint32_t dummy = sbase + cws;                              // one +inf cell, never written
  const uint32_t tab = sbase + cws + 16u + (uint32_t)(tid * SplitPlan<S>::units() * 8);
  split_fill<S, ZS>(a, rs, b0, b1, h, dummy, tab, std::make_integer_sequence<int, S::MB>{});
  if (tid == 0) {
    sts32(dummy, 0x7f800000u);
    s_fail = 1;
  }
  load_llrs_f32(reinterpret_cast<const float*>(a.llr) + cw * N, 1, N, Z, sbase, cws, RS);
  __syncthreads();

  float msg[SplitPlan<S>::slots()];
#pragma unroll
  for (int e = 0; e < SplitPlan<S>::slots(); ++e) msg[e] = 0.0f;
  const auto tiers = std::make_integer_sequence<int, S::MB>{};
  int iters = a.max_iters;
  if constexpr (!ET) {
    for (int k = 0; k < a.max_iters; ++k) SR::template sweep<false>(K, h, tab, msg, true, tiers);
    if (a.max_iters > 0) {
      if (tid == 0) s_fail = 0;
      __syncthreads();
      const uint32_t par = SR::parity_all(tab, tiers);
      const uint32_t row = par ^ __shfl_xor_sync(0xffffffffu, par, 1);
      if (row) s_fail = 1;
      __syncthreads();
    }
  } else {
    bool done = false;
    iters = 0;
    for (int k = 0; k < a.max_iters && !done; ++k) {
      SR::template sweep<true>(K, h, tab, msg, true, tiers);
      if (tid == 0) s_fail = 0;                  // syndrome (_kernels.py:85-96)
      __syncthreads();
      const uint32_t par = SR::parity_all(tab, tiers);
      const uint32_t row = par ^ __shfl_xor_sync(0xffffffffu, par, 1);
      if (row) s_fail = 1;
      __syncthreads();
      iters = k + 1;
      done = !s_fail;                            // uniform: read after the barrier
      __syncthreads();
    }
  }
  if (tid == 0) {
    a.iters[cw] = iters;
    a.conv[cw] = (a.max_iters > 0 && !s_fail) ? 1 : 0;
  }
  uint8_t* hard = reinterpret_cast<uint8_t*>(a.hard) + cw * (a.hard_packed ? (N + 7) >> 3 : N);
  float* post = a.post ? reinterpret_cast<float*>(a.post) + cw * N : nullptr;
  store_outputs_cell32(hard, a.hard_packed, post, 1, N, Z, sbase, cws, RS,
                       [](uint32_t v) { return __uint_as_float(v) <= 0.0f; },
                       [](uint32_t v) { return __uint_as_float(v); });
}

template <class S, int ZS, bool ET>
inline cudaError_t launch_split(const SpecArgs& a, cudaStream_t s) {
  constexpr int RS = row_stride_bytes<ArithF32>();
  const int z = ZS > 0 ? ZS : a.z;
  auto kern = decode_split_kernel<S, ZS, ET>;
  const int threads = (2 * z + 31) / 32 * 32;
  if (threads > kLayMaxThreads) return cudaErrorInvalidValue;
  const size_t smem = (size_t)((z * RS + 15) & ~15) + 16 + (size_t)threads * SplitPlan<S>::units() * 8;
  cudaError_t e = ensure_dyn_smem((const void*)kern, smem);
  if (e != cudaSuccess) return e;
  if (a.w <= 0) return cudaSuccess;
  kern<<<(unsigned)a.w, threads, smem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace qcb
