// NEGATIVE RESULT, NOT BUILT (kept for the record; see DESIGN.md 3.3 (4b)).
// Round 2, B200, parity green (Wi-Fi 648, all four rates, fixed iterations and
// early termination, hostile values).  Time per launch against the iteration
// count (tools/exp/c1_iters.py, 40 back-to-back launches in one CUDA graph):
//   one lane per row:  148 codewords 136 cycles per tier, 1024 codewords 179
//   this kernel:       148 codewords 143 cycles per tier, 1024 codewords 266
// Halving the in-order instruction stream (34 instead of 64 instructions per
// tier) does not shorten the tier: the shuffle and the two-warp CTA barrier put
// as much latency back into the chain as the shorter stream removes, and with
// 1024 codewords the doubled warp count is issue-bound.  C1: 20.6 us per launch
// against 15.0 us.
//
// decode_split.cuh -- small-batch float32 layered min-sum: TWO lanes per check
// row, for batches that leave the GPU latency-bound (BASELINE C1: 1024
// codewords of Wi-Fi 648 = 1.7 one-warp CTAs per SM sub-partition).
//
// Reference: /root/reference/pkg/src/qcldpc/_kernels.py:17-100 -- the same
// bit-exact row update as decode_layered.cuh (ArithF32::row).
//
// Why.  With one lane per row a tier is ~64 in-order instructions of ONE warp;
// measured (tools/exp/c1_scaling.py) the C1 kernel takes the same ~16 us for
// 148, 296 or 592 codewords and 17.4 us for 1024: the time is one warp's
// dependency chain (120 tiers x ~255 cycles), with half of every sub-partition's
// issue slots idle.  Splitting a row's D edges over two lanes halves the
// in-order stream per tier (ceil(D/2) slots per lane).
//
// Mapping.  Warp w, lane l: half h = l >> 4, row r = 16 w + (l & 15); a CTA is
// one codeword, ceil(Z / 16) warps.  The two lanes of a row sit 16 lanes
// apart in the SAME warp, so they exchange their half-minimum and sign parity
// with one __shfl_xor (the half-minimum is >= +0 or +inf, so the parity rides
// in its sign bit).  |L_new_k| = min(leave-one-out minimum of the lane's own
// slots, partner's half-minimum) is the same NaN-ignoring, +inf-seeded minimum
// over j != k as the reference's `k == argmin ? min2 : min1`.
//
// A tier's edges are ordered late-first (columns the previous tier writes) and
// dealt out alternately, so a slot is (late, late) or (early, early) wherever
// possible: early slots are loaded before the previous tier's barrier exactly
// as in decode_layered.cuh.  Odd D: half 1's last slot is a dummy that loads a
// cell holding +inf (never written; its store is predicated off): |zz| = +inf
// or NaN never wins a minimum and its sign bit is clear (canonical NaN), so it
// changes neither the minima nor the parity.
//
// Every slot's address is a per-lane constant (it depends on r and h): kept in
// registers for the whole decode.  Padding lanes (r >= Z) shadow a real lane of
// the same warp and half (same words, same values, lockstep).
//
// An earlier version (tools/exp/negative/decode_split.cuh: halves interleaved
// on lanes 2r / 2r+1, per-thread address table in shared memory, [c][j]
// layout) measured slower than one lane per row; this one keeps the halves
// 16 lanes apart (each half's accesses are 16 consecutive cells), has no table
// and runs on the bit-order layout.
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
  static constexpr int maxhalf() {
    int m = 1;
    for (int t = 0; t < S::MB; ++t) m = half(t) > m ? half(t) : m;
    return m;
  }
  // edge k of tier t reads a column tier t-1 does not write (see early_mask_of)
  static constexpr bool early(int t, int k) {
    if (t <= 0 || !QCB_EARLY_LOADS) return false;
    const int j = S::COL[S::START[t] + k];
    for (int e = S::START[t - 1]; e < S::START[t]; ++e)
      if (S::COL[e] == j) return false;
    return true;
  }
  // i-th edge of tier t, late edges first
  static constexpr int ordered(int t, int i) {
    int n = 0;
    for (int k = 0; k < S::DEG[t]; ++k)
      if (!early(t, k)) { if (n == i) return k; ++n; }
    for (int k = 0; k < S::DEG[t]; ++k)
      if (early(t, k)) { if (n == i) return k; ++n; }
    return -1;
  }
  static constexpr int edge(int t, int s, int h) {        // edge of slot s for half h, -1 = dummy
    const int i = 2 * s + h;
    return i < S::DEG[t] ? ordered(t, i) : -1;
  }
  static constexpr bool slot_early(int t, int s) {
    const int a = edge(t, s, 0), b = edge(t, s, 1);
    return early(t, a) && (b < 0 || early(t, b));
  }
  static constexpr uint32_t early_slots(int t) {           // bit s: slot s of tier t is early
    if (t >= S::MB) return 0u;
    uint32_t m = 0;
    for (int s = 0; s < half(t); ++s)
      if (slot_early(t, s)) m |= 1u << s;
    return m;
  }
};
// compile-time constants (the plan's tables are host constexpr data: device code
// must only see values folded through template arguments)
template <class S, int T>
struct SplitTier {
  static constexpr int H = T < S::MB ? SplitPlan<S>::half(T < S::MB ? T : 0) : 0;
  static constexpr int SLOT0 = SplitPlan<S>::slot0(T < S::MB ? T : S::MB);
  static constexpr uint32_t EARLY = SplitPlan<S>::early_slots(T);
  static constexpr bool ODD = T < S::MB && (S::DEG[T < S::MB ? T : 0] & 1) != 0;
};

template <class S, int ZS>
struct SplitRow {
  using SP = SplitPlan<S>;
  using A = ArithF32;
  static constexpr int MH = SP::maxhalf();

  template <int T, int I>
  __device__ __forceinline__ static uint32_t slot_addr(const SpecArgs& a, int r, uint32_t b0, uint32_t b1, int h,
                                                       uint32_t dummy) {
    constexpr int ka = SP::edge(T, I, 0), kb = SP::edge(T, I, 1);
    const uint32_t xa = edge_addr<S, A, ZS, S::START[T] + ka>(a, r, b0, b1);
    if constexpr (kb >= 0) {
      const uint32_t xb = edge_addr<S, A, ZS, S::START[T] + kb>(a, r, b0, b1);
      return h ? xb : xa;
    } else {
      return h ? dummy : xa;
    }
  }
  template <int T, int... Is>
  __device__ __forceinline__ static void fill_tier(const SpecArgs& a, int r, uint32_t b0, uint32_t b1, int h,
                                                   uint32_t dummy, uint32_t* addr, std::integer_sequence<int, Is...>) {
    ((addr[SplitTier<S, T>::SLOT0 + Is] = slot_addr<T, Is>(a, r, b0, b1, h, dummy)), ...);
  }
  template <int... Ts>
  __device__ __forceinline__ static void fill(const SpecArgs& a, int r, uint32_t b0, uint32_t b1, int h,
                                              uint32_t dummy, uint32_t* addr, std::integer_sequence<int, Ts...>) {
    (fill_tier<Ts>(a, r, b0, b1, h, dummy, addr, std::make_integer_sequence<int, SP::half(Ts)>{}), ...);
  }

  // tier T for this lane's H slots; pe = its early-loaded posteriors, pn = the
  // next tier's (loaded here, before the barrier that follows)
  template <int T>
  __device__ __forceinline__ static void tier(const RtK& K, bool h, const uint32_t* addr, float* msg,
                                              float (&pe)[MH], float (&pn)[MH]) {
    using ST = SplitTier<S, T>;
    using SN = SplitTier<S, T + 1>;
    constexpr int H = ST::H;
    constexpr bool ODD = ST::ODD;
    constexpr uint32_t EARLY = ST::EARLY, EARLY_N = SN::EARLY;
    const uint32_t* ad = addr + ST::SLOT0;
    float* m = msg + ST::SLOT0;
    float p[H], zz[H];
#pragma unroll
    for (int i = 0; i < H; ++i) p[i] = ((EARLY >> i) & 1u) ? pe[i] : A::lds(ad[i]);
#pragma unroll
    for (int i = 0; i + 1 < H; i += 2) f_sub2(p[i], p[i + 1], m[i], m[i + 1], zz[i], zz[i + 1]);
    if (H & 1) zz[H - 1] = f_sub(p[H - 1], m[H - 1]);
    uint32_t sx = 0;
#pragma unroll
    for (int i = 0; i < H; ++i) sx ^= __float_as_uint(zz[i]);
    // own leave-one-out minima and own minimum (+inf seeded, NaN-ignoring)
    float az[H], ex[H];
#pragma unroll
    for (int i = 0; i < H; ++i) az[i] = fabsf(zz[i]);
    loo_minima3<H>(az, ex, [](float x, float y) { return fminf(x, y); },
                   [](float x, float y, float z) { return f_min3(x, y, z); }, f_inf());
    const float hm = fminf(ex[0], az[0]);                  // >= +0, +inf if every |zz| is NaN / +inf
    uint32_t pk;                                           // half-minimum | own parity in the sign bit
    asm("lop3.b32 %0, %1, %2, 0x80000000, 0xF8;" : "=r"(pk) : "r"(__float_as_uint(hm)), "r"(sx));   // a | (b & c)
    const uint32_t po = __shfl_xor_sync(0xffffffffu, pk, 16);
    const float mo = fabsf(__uint_as_float(po));
    const uint32_t sxm = (sx ^ po) & 0x80000000u;          // the row's sign parity
#pragma unroll
    for (int i = 0; i < H; ++i) {
      const float e = fminf(ex[i], mo);
      uint32_t t;
      asm("lop3.b32 %0, %1, %2, 0x80000000, 0x28;" : "=r"(t) : "r"(__float_as_uint(zz[i])), "r"(sxm));  // (zz ^ sxm) & sign
      m[i] = __uint_as_float(imad(t, K.one, __float_as_uint(e)));
    }
    float o[H];
#pragma unroll
    for (int i = 0; i + 1 < H; i += 2) f_add2(zz[i], zz[i + 1], m[i], m[i + 1], o[i], o[i + 1]);
    if (H & 1) o[H - 1] = f_add(zz[H - 1], m[H - 1]);
#pragma unroll
    for (int i = 0; i < H; ++i) {
      if (ODD && i == H - 1) {
        if (!h) A::sts(ad[i], o[i]);                       // half 1's slot is the dummy
      } else {
        A::sts(ad[i], o[i]);
      }
    }
    if constexpr (EARLY_N != 0u) {
      const uint32_t* an = addr + SN::SLOT0;
#pragma unroll
      for (int i = 0; i < SN::H; ++i)
        if ((EARLY_N >> i) & 1u) pn[i] = A::lds(an[i]);
    }
  }

  template <int... Ts>
  __device__ __forceinline__ static void sweep(const RtK& K, bool h, const uint32_t* addr, float* msg,
                                               std::integer_sequence<int, Ts...>) {
    float pa[MH], pb[MH];
    ((tier<Ts>(K, h, addr, msg, (Ts & 1) ? pb : pa, (Ts & 1) ? pa : pb), split_sync()), ...);
  }
  __device__ __forceinline__ static void split_sync() {
    if constexpr (ZS <= 16) __syncwarp();
    else __syncthreads();
  }

  // bit T = this lane's share of its row's parity in tier T (dummy: +inf -> 0)
  template <int T>
  __device__ __forceinline__ static uint32_t parity(const uint32_t* addr) {
    using ST = SplitTier<S, T>;
    uint32_t par = 0;
#pragma unroll
    for (int i = 0; i < ST::H; ++i) par ^= A::hard(A::lds(addr[ST::SLOT0 + i])) ? 1u : 0u;
    return par << T;
  }
  template <int... Ts>
  __device__ __forceinline__ static uint32_t parity_all(const uint32_t* addr, std::integer_sequence<int, Ts...>) {
    return (parity<Ts>(addr) | ...);
  }
};

// min CTAs per SM for the register budget: 8 two-warp CTAs = 128 registers per
// thread = 4 warps per sub-partition, so 1024 two-warp CTAs stay one wave
#ifndef QCB_SPLIT_MIN_CTAS
#define QCB_SPLIT_MIN_CTAS 8
#endif

// one codeword per CTA, two lanes per row: blockDim = 32 ceil(Z / 16)
template <class S, int ZS, bool ET>
__global__ void __launch_bounds__(64, QCB_SPLIT_MIN_CTAS)
    decode_split_kernel(const __grid_constant__ SpecArgs a) {
  using SR = SplitRow<S, ZS>;
  using SP = SplitPlan<S>;
  static_assert(ZS > 0 && ZS <= 32, "two warps at most");
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int s_fail;

  const RtK K{a.k_one, a.k_sign, a.k_shr, a.k_neg1, a.k_lane1};
  constexpr int Z = ZS;
  constexpr int N = S::NB * Z;
  const int tid = threadIdx.x;
  const int64_t cw = blockIdx.x;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  dbg_check(cw < a.w, 23);
  dbg_poison_smem();
  dbg_inject_probe(a.dbg_inject, sbase);
  const int lane = tid & 31, wrp = tid >> 5;
  const bool h = (lane >> 4) != 0;
  const int q = lane & 15, rows = Z - 16 * wrp < 16 ? Z - 16 * wrp : 16;   // rows of this warp
  const int rs = 16 * wrp + (q < rows ? q : q % rows);
  uint32_t b0 = sbase + (uint32_t)(rs * kCellBytes), b1;
  asm volatile("mov.b32 %0, %0;" : "+r"(b0));
  asm volatile("sub.u32 %0, %1, %2;" : "=r"(b1) : "r"(b0), "r"((uint32_t)(Z * kCellBytes)));
  const uint32_t dummy = sbase + (uint32_t)cw_block_bytes(Z);          // one +inf cell, never written
  constexpr int NS = SP::slots();
  uint32_t addr[NS];
  SR::fill(a, rs, b0, b1, h ? 1 : 0, dummy, addr, std::make_integer_sequence<int, S::MB>{});
#pragma unroll
  for (int i = 0; i < NS; ++i) asm volatile("mov.b32 %0, %0;" : "+r"(addr[i]));   // stay in registers
  if (tid == 0) {
    sts32(dummy, 0x7f800000u);
    s_fail = 1;
  }
  load_llrs_f32<io_cells8<ZS>()>(reinterpret_cast<const float*>(a.llr) + cw * N, 1, N, sbase);
  __syncthreads();

  float msg[NS];
#pragma unroll
  for (int e = 0; e < NS; ++e) msg[e] = 0.0f;
  const auto tiers = std::make_integer_sequence<int, S::MB>{};
  int iters = a.max_iters;
  if constexpr (!ET) {
    for (int k = 0; k < a.max_iters; ++k) SR::sweep(K, h, addr, msg, tiers);
    if (a.max_iters > 0) {
      if (tid == 0) s_fail = 0;
      __syncthreads();
      const uint32_t par = SR::parity_all(addr, tiers);
      if (par ^ __shfl_xor_sync(0xffffffffu, par, 16)) s_fail = 1;
      __syncthreads();
    }
  } else {
    iters = 0;
    int fail = 1;
    while (iters < a.max_iters) {
      SR::sweep(K, h, addr, msg, tiers);
      ++iters;
      const uint32_t par = SR::parity_all(addr, tiers);
      fail = __syncthreads_or((par ^ __shfl_xor_sync(0xffffffffu, par, 16)) != 0u);
      if (!fail) break;
    }
    if (tid == 0) s_fail = fail;
    __syncthreads();
  }
  if (tid == 0) {
    a.iters[cw] = iters;
    a.conv[cw] = (a.max_iters > 0 && !s_fail) ? 1 : 0;
  }
  uint8_t* hard = reinterpret_cast<uint8_t*>(a.hard) + cw * (a.hard_packed ? (N + 7) >> 3 : N);
  float* post = a.post ? reinterpret_cast<float*>(a.post) + cw * N : nullptr;
  store_outputs_cell32<io_cells8<ZS>()>(hard, a.hard_packed, post, 1, N, sbase,
                                        [](uint32_t v) { return __uint_as_float(v) <= 0.0f; },
                                        [](uint32_t v) { return __uint_as_float(v); });
}

// Batches up to this many codewords take the split kernel (native Z <= 32,
// float32): measured crossover against one lane per row, see DESIGN 3.1b.
#ifndef QCB_SPLIT_MAX_W
#define QCB_SPLIT_MAX_W 2368
#endif
inline int64_t split_max_w() {
  static const int64_t v = [] {
    const char* e = getenv("QCB_SPLIT_MAX_W");           // tuning knob (benchmarks only)
    return e ? (int64_t)atoll(e) : (int64_t)QCB_SPLIT_MAX_W;
  }();
  return v;
}

template <class S, int ZS, bool ET>
inline cudaError_t launch_split(const SpecArgs& a, cudaStream_t s) {
  auto kern = decode_split_kernel<S, ZS, ET>;
  constexpr int threads = 32 * ((ZS + 15) / 16);
  const size_t smem = (size_t)cw_block_bytes(ZS) + 16;
  cudaError_t e = ensure_dyn_smem((const void*)kern, smem);
  if (e != cudaSuccess) return e;
  if (a.w <= 0) return cudaSuccess;
  kern<<<(unsigned)a.w, threads, smem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace qcb
