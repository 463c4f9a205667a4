// decode_tmem.cuh -- the layered decoder with its check-to-variable messages
// resident in Tensor Memory (tcgen05 TMEM) instead of registers.
//
// Same row update, addressing and outputs as decode_layered.cuh (and the same
// bit-exact contract with /root/reference/pkg/src/qcldpc/_kernels.py).  What
// changes is where the explicit messages live between sweeps:
//
//  * register-resident (decode_layered_kernel): S::NE registers per thread ->
//    ~128-150 registers, 4-5 CTAs (12-15 warps) per SM;
//  * TMEM-resident (this kernel): thread t of warp w owns TMEM lane
//    32*(w%4) + (t%32) and the S::NE consecutive columns of slot w/4; tier T's
//    messages are columns [START[T], START[T+1]).  Registers drop to the
//    transients of one tier, so 2 CTAs x 12 warps fit per SM: 8 codewords
//    (Z=96) resident per SM instead of 5, and the 256 KB of TMEM per SM --
//    otherwise idle in a non-GEMM kernel -- holds the decoder state.
//
// Per tier each warp issues one tcgen05.ld per power-of-two piece of the
// tier's messages for the NEXT tier (prefetch; waited on at the start of that
// tier) and one tcgen05.st per piece for the current tier's new messages.
// tcgen05.ld/st are warp-collective (.sync.aligned), so every warp executes
// them unconditionally; frozen / absent codewords just store back what they
// loaded.
#pragma once
#include "decode_layered.cuh"

namespace qcb {

// ---- 32x32b TMEM pieces: lane = the thread's lane, N consecutive columns ----
template <int N>
__device__ __forceinline__ void tm_ld(uint32_t t, uint32_t* r);
template <>
__device__ __forceinline__ void tm_ld<1>(uint32_t t, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r[0]) : "r"(t));
}
template <>
__device__ __forceinline__ void tm_ld<2>(uint32_t t, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(r[0]), "=r"(r[1]) : "r"(t));
}
template <>
__device__ __forceinline__ void tm_ld<4>(uint32_t t, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(t));
}
template <>
__device__ __forceinline__ void tm_ld<8>(uint32_t t, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(t));
}
template <int N>
__device__ __forceinline__ void tm_st(uint32_t t, const uint32_t* r);
template <>
__device__ __forceinline__ void tm_st<1>(uint32_t t, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(t), "r"(r[0]));
}
template <>
__device__ __forceinline__ void tm_st<2>(uint32_t t, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(t), "r"(r[0]), "r"(r[1]));
}
template <>
__device__ __forceinline__ void tm_st<4>(uint32_t t, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(t), "r"(r[0]), "r"(r[1]),
               "r"(r[2]), "r"(r[3]));
}
template <>
__device__ __forceinline__ void tm_st<8>(uint32_t t, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(t), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]));
}

// D columns starting at column offset OFF, decomposed into 8/4/2/1 pieces
template <int OFF, int D>
__device__ __forceinline__ void tm_ld_n(uint32_t base, uint32_t* r) {
  if constexpr (D >= 8) { tm_ld<8>(base + OFF, r); tm_ld_n<OFF + 8, D - 8>(base, r + 8); }
  else if constexpr (D >= 4) { tm_ld<4>(base + OFF, r); tm_ld_n<OFF + 4, D - 4>(base, r + 4); }
  else if constexpr (D >= 2) { tm_ld<2>(base + OFF, r); tm_ld_n<OFF + 2, D - 2>(base, r + 2); }
  else if constexpr (D == 1) { tm_ld<1>(base + OFF, r); }
}
template <int OFF, int D>
__device__ __forceinline__ void tm_st_n(uint32_t base, const uint32_t* r) {
  if constexpr (D >= 8) { tm_st<8>(base + OFF, r); tm_st_n<OFF + 8, D - 8>(base, r + 8); }
  else if constexpr (D >= 4) { tm_st<4>(base + OFF, r); tm_st_n<OFF + 4, D - 4>(base, r + 4); }
  else if constexpr (D >= 2) { tm_st<2>(base + OFF, r); tm_st_n<OFF + 2, D - 2>(base, r + 2); }
  else if constexpr (D == 1) { tm_st<1>(base + OFF, r); }
}

// wait for this thread's outstanding TMEM loads; the empty asm statements make
// every later use of the loaded registers depend on the wait
template <int D>
__device__ __forceinline__ void tm_wait_ld(uint32_t* r) {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int k = 0; k < D; ++k) asm volatile("" : "+r"(r[k]));
}
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

template <class S, class A, int ZS>
struct LayeredTm {
  using Val = typename A::Val;
  static_assert(S::MB % 2 == 0, "double-buffered prefetch assumes an even number of tiers");

  // tier T: messages arrived in buf[T&1] (prefetched); prefetch tier T+1 into
  // buf[(T+1)&1]; update; store back
  template <int T>
  __device__ __forceinline__ static void tier(const SpecArgs& a, const RtK& K, int r, uint32_t b0, uint32_t b1,
                                              uint32_t tb, uint32_t (&bufA)[S::MAXDEG],
                                              uint32_t (&bufB)[S::MAXDEG], bool work) {
    constexpr int D = S::DEG[T];
    constexpr int E0 = S::START[T];
    constexpr int TN = (T + 1) % S::MB;
    uint32_t* cur = (T & 1) ? bufB : bufA;
    uint32_t* nxt = (T & 1) ? bufA : bufB;
    tm_wait_st();                                // previous tier's store (issued a tier ago)
    tm_wait_ld<D>(cur);
    tm_ld_n<S::START[TN], S::DEG[TN]>(tb, nxt);
    if (work) {
      uint32_t addr[D];
      Val p[D], o[D], m[D];
      tier_addrs<S, A, ZS, E0>(a, r, b0, b1, addr, std::make_integer_sequence<int, D>{});
#pragma unroll
      for (int k = 0; k < D; ++k) p[k] = A::lds(addr[k]);
#pragma unroll
      for (int k = 0; k < D; ++k) m[k] = from_bits(cur[k]);
      A::template row<D>(p, o, m, K);
#pragma unroll
      for (int k = 0; k < D; ++k) cur[k] = to_bits(m[k]);
#pragma unroll
      for (int k = 0; k < D; ++k) A::sts(addr[k], o[k]);
    }
    tm_st_n<E0, D>(tb, cur);                     // waited on at the start of the next tier
  }

  __device__ __forceinline__ static Val from_bits(uint32_t b) {
    if constexpr (A::kElem == 4) return __uint_as_float(b); else return b;
  }
  __device__ __forceinline__ static uint32_t to_bits(Val v) {
    if constexpr (A::kElem == 4) return __float_as_uint(v); else return v;
  }

  template <int T>
  __device__ __forceinline__ static uint32_t parity(const SpecArgs& a, int r, uint32_t b0, uint32_t b1) {
    constexpr int D = S::DEG[T];
    uint32_t addr[D];
    tier_addrs<S, A, ZS, S::START[T]>(a, r, b0, b1, addr, std::make_integer_sequence<int, D>{});
    uint32_t par = 0;
#pragma unroll
    for (int k = 0; k < D; ++k) par ^= A::hard(A::lds(addr[k])) ? 1u : 0u;
    return par;
  }
  template <int... Ts>
  __device__ __forceinline__ static uint32_t parity_all(const SpecArgs& a, int r, uint32_t b0, uint32_t b1,
                                                        std::integer_sequence<int, Ts...>) {
    return (parity<Ts>(a, r, b0, b1) | ...);
  }

  template <int... Ts>
  __device__ __forceinline__ static void sweep(const SpecArgs& a, const RtK& K, int r, uint32_t b0, uint32_t b1,
                                               uint32_t tb, uint32_t (&bufA)[S::MAXDEG],
                                               uint32_t (&bufB)[S::MAXDEG], bool work,
                                               std::integer_sequence<int, Ts...>) {
    ((tier<Ts>(a, K, r, b0, b1, tb, bufA, bufB, work), __syncthreads()), ...);
  }
};

#ifndef QCB_TM_REG_BASE
#define QCB_TM_REG_BASE 40
#endif
template <class S, class A>
constexpr int tm_reg_cap() {
  constexpr int want = QCB_TM_REG_BASE + 5 * S::MAXDEG;
  return (want + 7) / 8 * 8 > 255 ? 255 : (want + 7) / 8 * 8;
}

template <class S, class A, int ZS, bool ET>
__global__ void __launch_bounds__(kLayMaxThreads) __maxnreg__((tm_reg_cap<S, A>()))
    decode_tmem_kernel(const __grid_constant__ SpecArgs a) {
  using LT = LayeredTm<S, A, ZS>;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int s_fail[kLayMaxCw], s_done[kLayMaxCw], s_iters[kLayMaxCw];
  __shared__ int s_active;
  __shared__ uint32_t s_taddr;

  const RtK K{a.k_one, a.k_sign, a.k_shr, a.k_neg1, a.k_lane1};
  const int Z = ZS > 0 ? ZS : a.z;
  const int N = S::NB * Z;
  const int G = a.pairs;
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int g = tid / Z, r = tid - g * Z;
  const int64_t cw0 = (int64_t)blockIdx.x * G;
  const int ncw = (int)(a.w - cw0 < (int64_t)G ? a.w - cw0 : (int64_t)G);
  const bool act = g < ncw;
  const uint32_t cws = (uint32_t)cw_block_bytes(Z);
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  dbg_check(cw0 < a.w && ncw >= 1 && ncw <= G, 23);           // the CTA's chunk lies inside the batch
  dbg_poison_smem();
  dbg_inject_probe(a.dbg_inject, sbase);
  uint32_t b0 = sbase + (uint32_t)g * cws + (uint32_t)(r * kCellBytes), b1;
  asm volatile("mov.b32 %0, %0;" : "+r"(b0));
  asm volatile("sub.u32 %0, %1, %2;" : "=r"(b1) : "r"(b0), "r"((uint32_t)(Z * kCellBytes)));

  // ---- TMEM: one warp allocates a.tmem_cols columns for the CTA ----------------
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"((uint32_t)__cvta_generic_to_shared(&s_taddr)), "r"((uint32_t)a.tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }

  // ---- channel LLRs -> [cw][c][j] ------------------------------------------------
  static_assert(A::kElem == 4, "float32 cells");
  {
    load_llrs_f32<io_cells8<ZS>()>(reinterpret_cast<const float*>(a.llr) + cw0 * N, ncw, N, sbase);
    for (int q = tid; q < kLayMaxCw; q += blockDim.x) {
      s_fail[q] = 1; s_done[q] = q >= ncw; s_iters[q] = 0;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // this thread's lane and column slot
  const uint32_t tb = s_taddr + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * S::NE);

  // messages start at +0 (reference: min1 = min2 = 0, no signs)
  uint32_t bufA[S::MAXDEG], bufB[S::MAXDEG];
#pragma unroll
  for (int k = 0; k < S::MAXDEG; ++k) { bufA[k] = 0u; bufB[k] = 0u; }
  {
    uint32_t z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int c = 0; c + 8 <= S::NE; c += 8) tm_st<8>(tb + c, z);
    if constexpr (S::NE % 8 >= 4) tm_st<4>(tb + (S::NE / 8) * 8, z);
    if constexpr (S::NE % 4 >= 2) tm_st<2>(tb + (S::NE / 4) * 4, z);
    if constexpr (S::NE % 2 == 1) tm_st<1>(tb + S::NE - 1, z);
    tm_wait_st();
  }
  tm_ld_n<S::START[0], S::DEG[0]>(tb, bufA);    // prefetch tier 0

  const auto tiers = std::make_integer_sequence<int, S::MB>{};
  if constexpr (!ET) {
    // fixed iterations: every codeword runs max_iters sweeps; one syndrome at the end
    for (int k = 0; k < a.max_iters; ++k) LT::sweep(a, K, r, b0, b1, tb, bufA, bufB, act, tiers);
    if (a.max_iters > 0) {
      if (tid < kLayMaxCw) s_fail[tid] = 0;
      __syncthreads();
      if (act && LT::parity_all(a, r, b0, b1, tiers)) s_fail[g] = 1;
      __syncthreads();
    }
    if (tid < ncw) s_iters[tid] = a.max_iters;
  } else {
    for (int k = 0; k < a.max_iters; ++k) {
      const bool work = act && !s_done[g];
      LT::sweep(a, K, r, b0, b1, tb, bufA, bufB, work, tiers);
      if (tid < kLayMaxCw) s_fail[tid] = 0;       // syndrome (_kernels.py:85-96)
      __syncthreads();
      if (work && LT::parity_all(a, r, b0, b1, tiers)) s_fail[g] = 1;
      if (tid == 0) s_active = 0;
      __syncthreads();
      if (tid < ncw && !s_done[tid]) {
        s_iters[tid] = k + 1;
        if (!s_fail[tid]) s_done[tid] = 1;
        else s_active = 1;
      }
      __syncthreads();
      if (!s_active) break;
    }
  }
  tm_wait_st();
  tm_wait_ld<S::DEG[0]>(bufA);                  // drain the last prefetch

  // ---- outputs ---------------------------------------------------------------------
  if (tid < ncw) {
    a.iters[cw0 + tid] = s_iters[tid];
    a.conv[cw0 + tid] = (a.max_iters > 0 && !s_fail[tid]) ? 1 : 0;
  }
  uint8_t* hard = reinterpret_cast<uint8_t*>(a.hard) + cw0 * (a.hard_packed ? (N + 7) >> 3 : N);
  float* post = a.post ? reinterpret_cast<float*>(a.post) + cw0 * N : nullptr;
  store_outputs_cell32<io_cells8<ZS>()>(hard, a.hard_packed, post, ncw, N, sbase,
                       [](uint32_t v) { return __uint_as_float(v) <= 0.0f; },
                       [](uint32_t v) { return __uint_as_float(v); });
  // ---- release TMEM ------------------------------------------------------------------
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_taddr), "r"((uint32_t)a.tmem_cols));
}

// Pick codewords per CTA for the TMEM kernel: maximise codewords resident per
// SM under TMEM (512 columns, power-of-two allocations of slots x NE),
// registers, shared memory and the 384-thread CTA limit.  Returns 0 if no
// configuration holds at least as many codewords per SM as the register kernel.
inline int tmem_plan(int z, int ne, int regs_per_thread, int smem_per_cw, int64_t w, int* cols_out) {
  int best_g = 0, best_cw = 0, best_cols = 0;
  for (int g = 1; g <= kLayMaxCw && g * z <= kLayMaxThreads; ++g) {
    if (g > 1 && w < (int64_t)g * 148 * 2) break;
    const int warps = (g * z + 31) / 32;
    const int slots = (warps + 3) / 4;
    int cols = 32;
    while (cols < slots * ne) cols <<= 1;
    if (cols > 512) continue;
    const int by_tmem = 512 / cols;
    const int by_regs = 65536 / (warps * 32 * regs_per_thread);
    const int by_smem = (227 * 1024) / (g * smem_per_cw + 1024);
    const int by_warps = 64 / warps;
    const int ctas = std::min(std::min(by_tmem, by_regs), std::min(std::min(by_smem, by_warps), 32));
    const int cw = ctas * g;
    if (cw > best_cw) { best_cw = cw; best_g = g; best_cols = cols; }
  }
  if (cols_out) *cols_out = best_cols;
  return best_g;
}

template <class S, class A, int ZS, bool ET>
inline cudaError_t launch_tmem(const SpecArgs& a, cudaStream_t s) {
  const int z = ZS > 0 ? ZS : a.z;
  const int threads = (a.pairs * z + 31) / 32 * 32;
  const size_t smem = (size_t)a.pairs * cw_block_bytes(z);
  auto kern = decode_tmem_kernel<S, A, ZS, ET>;
  cudaError_t e = ensure_dyn_smem((const void*)kern, smem);
  if (e != cudaSuccess) return e;
  // the register count is only known after ptxas: shrink the CTA if this
  // kernel cannot launch the planned one (the decode result does not depend
  // on the CTA size)
  cudaFuncAttributes fa;
  e = kernel_attributes((const void*)kern, &fa);
  if (e != cudaSuccess) return e;
  if (threads > fa.maxThreadsPerBlock) {
    SpecArgs b = a;
    b.pairs = fa.maxThreadsPerBlock / z;
    if (b.pairs < 1) return cudaErrorLaunchOutOfResources;
    if (b.tmem_cols > 0) return cudaErrorLaunchOutOfResources;   // TMEM plan is per CTA shape
    return launch_layered_fixed(kern, b, z, s);
  }
  return launch_layered_fixed(kern, a, z, s);
}


}  // namespace qcb
