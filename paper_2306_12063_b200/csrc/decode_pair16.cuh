// decode_pair16.cuh -- int16 layered min-sum, two codewords per thread in
// 16x2 SIMD lanes (sm_100a).
//
// Reference: /root/reference/pkg/src/qcldpc/_kernels.py:103-186 (int16 with
// two's-complement wrap after every op).  The reference's int16 values are
// 16 bits wide, so one 32-bit register carries the same row of TWO
// codewords: the low lane belongs to codeword 2g, the high lane to 2g+1.
// Every per-edge operation is a lane-wise 16-bit operation with the
// reference's wrap (VIADD.16x2 adds wrap per lane; VIMNMX.S16x2 compares in
// signed int16 order, so abs(-32768) = -32768 sorts lowest exactly as in the
// reference).  One instruction therefore advances two codewords, and one
// 32-bit shared-memory access moves both codewords' posterior.
//
// Messages are kept NEGATED (nm = -L_mn) so that zz = post - L_old is a
// single lane-wise add.  Lane-wise negation / sign application use
// -x = ~x + 1 with ~x = x * (-1) + (-1) on the FMA pipe (a 32-bit IMAD
// cannot carry across lanes for this operand), so the row update splits
// about evenly between the half-rate ALU and FMA-heavy pipes:
//   pass 1  d = p + nm                                   (VIADD.16x2)
//           a = max(d, ~d + 0x10001) = |d| (wrapping)    (IMAD, VIADD, VIMNMX)
//   minima  ex_k = min_{j != k} a_j (prefix / suffix anchors, loo_minima3: VIMNMX3)
//   pass 2  m    = lane sign mask of d ^ parity          (LOP3, PRMT)
//           nex  = ~ex + 0x10001 = -ex                   (IMAD, VIADD)
//           post = d + (m ? nex : ex), nm = m ? ex : nex (LOP3, VIADD, LOP3)
//           (Wi-Fi 1944 R5/6: L_new = (ex + m) ^ m, nm = -L_new, measured faster)
// Shared memory layout, addressing and tier schedule are the float32
// kernel's (4-byte cells, decode_layered.cuh).
#pragma once
#include <mutex>

#include "decode_layered.cuh"
#include "decode_tmem.cuh"

#ifndef QCB_P16_XORSIGN
#define QCB_P16_XORSIGN 0   // 0: per-structure choice, 1: everywhere, 2: nowhere (experiments)
#endif
#ifndef QCB_P16_MIN3
#define QCB_P16_MIN3 2
#endif
#ifndef QCB_P16_TAB_LATE
#define QCB_P16_TAB_LATE 0
#endif

// Native-Z kernels: address table in global memory (read through L1) instead
// of shared memory.  Measured on C5 (round 2, tools/exp/ab_r02_tmem.sh): 68.8
// vs 82.5 Gb/s -- LDG latency on every tier's prefetch costs more than the
// freed shared memory buys; kept as an option for the TMEM experiments.
#ifndef QCB_P16_GTAB
#define QCB_P16_GTAB 0
#endif
// Row parity applied to the sign test with a lane-wise add of the parity's
// sign bits (VIADD.16x2, FMA-heavy pipe) instead of an XOR (LOP3, ALU pipe):
// the ALU pipe carries ~7.4 of ~15.2 instructions per pair-edge and is the
// binding pipe (ncu: ALU 64 % at 66 % issue); this moves one op per edge.
#ifndef QCB_P16_ADDSIGN
#define QCB_P16_ADDSIGN 1
#endif
// Messages of the first TMT tiers in TMEM instead of registers (native Z > 32,
// one pair per CTA), the register cap lowered to QCB_P16_TM_CAP: fewer
// registers -> 5 CTAs (15 warps) per SM instead of 4.  Measured per structure
// (round 2, tools/exp/p16_sweep_r02.sh, int16 coded Gb/s at 262144 codewords,
// TMT 0 / 2 / 3 / 4): Wi-Fi 1944 R5/6 (C3) 65.5 / 73.3 / 73.9 / 73.9, R3/4
// 72.4 / 73.5 / 74.3 / 73.5, WiMAX 3/4A (C5) 87.0 / 87.6 / 87.6 / 87.6, 5/6
// 90.3 / 92.3 / 89.1 / 89.2; Wi-Fi 1296 loses 2-8 %, WiMAX 1/2, 2/3B, 3/4B
// lose 1-3 %, the rest are within 1 %.  QCB_P16_TMT >= 0 forces one value
// for every eligible structure (experiments).
#ifndef QCB_P16_TMT
#define QCB_P16_TMT -1
#endif
#ifndef QCB_P16_TM_CAP
#define QCB_P16_TM_CAP 0        // 0: per structure (p16_tm_cap), else one cap for every TMEM-tier kernel (experiments)
#endif
// Re-swept on the final kernels (round 2, tools/exp/r02_call52.sh, r02_call53.sh; 128 / 120 /
// 112 / 108 / 104, all four warps per sub-partition): WiMAX 3/4A (C5) 87.84 / 87.87 / 88.33 /
// 86.6 / 85.6 Gb/s, Wi-Fi 1944 R3/4 78.2 -> 80.3 at 112; Wi-Fi 1944 R5/6 (C3) 105.2 / 102.5 /
// 104.1 and WiMAX 5/6 91.6 -> 88.1 keep 128 (ptxas schedules differently under the cap).
constexpr int p16_tm_cap(int id) { return (id == 15 || id == 6) ? 112 : 128; }
#ifndef QCB_P16_TM_WAIT0
#define QCB_P16_TM_WAIT0 1      // tcgen05.wait::st once per sweep (tier 0) instead of every TMEM tier
#endif
// Wi-Fi 1944 R2/3 (5) dropped its TMEM tiers in round 2: without them it packs
// three pairs per CTA (native_fill_cw), 88.9 -> 93.2 Gb/s (r02_call10.sh).
constexpr int p16_tmt_default(int id) {
  return (id == 6 || id == 7 || id == 15) ? 3 : (id == 17 ? 2 : 0);
}

namespace qcb {

// The pair kernel's dynamic shared memory (same region as the kernel's own
// `extern __shared__ smem`): its window address is a per-kernel constant that
// ptxas keeps in a uniform register and folds into LDS/STS [R + UR] addressing.
extern __shared__ __align__(16) unsigned char qcb_p16_dyn[];
__device__ __forceinline__ uint32_t p16_sbase() { return (uint32_t)__cvta_generic_to_shared(qcb_p16_dyn); }

// Global address tables of the native-Z pair kernels.  With one codeword pair
// per CTA every CTA's thread t has the same table: its edges' cell offsets
// (wrap included) relative to the dynamic shared-memory base.  It is filled
// once per device by fill_p16_gtab_kernel and read through L1 (LDG.64, a tier
// ahead): 33 KB shared by all CTAs of an SM instead of 33 KB of shared memory
// per CTA (C5), which is what capped the kernel at 4 CTAs per SM.
template <class S, int ZS>
constexpr int p16_gtab_units() { return AddrTab<S, ZS, true>::units(); }
template <class S, int ZS>
__device__ uint2 g_p16_tab[kLayMaxThreads * (p16_gtab_units<S, ZS>() > 0 ? p16_gtab_units<S, ZS>() : 1)];

__device__ __forceinline__ uint32_t vadd2(uint32_t a, uint32_t b) {
  uint32_t d; asm("add.s16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b)); return d;
}
__device__ __forceinline__ uint32_t vmin2(uint32_t a, uint32_t b) {
  uint32_t d; asm("min.s16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b)); return d;
}
__device__ __forceinline__ uint32_t vmax2(uint32_t a, uint32_t b) {
  uint32_t d; asm("max.s16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b)); return d;
}
// min of three in ONE asm block, so that ptxas forms VIMNMX3 (see loo_minima3)
__device__ __forceinline__ uint32_t vmin3(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("{\n\t.reg .b32 t;\n\tmin.s16x2 t, %1, %2;\n\tmin.s16x2 %0, t, %3;\n\t}" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
// lane sign bit set exactly where the lane's int16 is <= 0 (the hard decision):
// min(x - 1, x) -- add + min in one asm block so that ptxas forms VIADDMNMX
__device__ __forceinline__ uint32_t hard_sign2(uint32_t x) {
  uint32_t d;
  asm("{\n\t.reg .b32 t;\n\tadd.s16x2 t, %1, %2;\n\tmin.s16x2 %0, t, %1;\n\t}" : "=r"(d) : "r"(x), "r"(0xFFFFFFFFu));
  return d;
}
// lane sign masks: 0xFFFF in a lane whose bit 15 is set
__device__ __forceinline__ uint32_t lane_signs(uint32_t x) {
  uint32_t d; asm("prmt.b32 %0, %1, 0, 0xBB99;" : "=r"(d) : "r"(x)); return d;
}

struct ArithI16x2 {
  using Val = uint32_t;
  static constexpr int kElem = 4;        // one cell = the two codewords' int16 posteriors
  static constexpr int kKind = 2;        // address-table policy key (use_addr_tab)

  __device__ static Val lds(uint32_t a) {
    dbg_smem(a, 4, 11);
    uint32_t v; asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a)); return v;
  }
  __device__ static void sts(uint32_t a, Val v) {
    dbg_smem(a, 4, 12);
    asm volatile("st.shared.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
  }

  // One row of D edges: posteriors p[] in, new posteriors o[] out, negated
  // messages nm[] updated in place (both codewords' lanes).
  template <int D, bool ANCHOR = false, bool XORSIGN = false>
  __device__ __forceinline__ static void row(const Val (&p)[D], Val (&o)[D], Val* nm, const RtK& K) {
    static_assert(D >= 2, "row degree >= 2");
    uint32_t d[D], a[D];
#pragma unroll
    for (int k = 0; k < D; ++k) {
      d[k] = vadd2(p[k], nm[k]);                                   // zz = post - L_old
      a[k] = vmax2(d[k], vadd2(imad(d[k], K.neg1, K.neg1), K.lane1));   // |zz| (wrapping)
    }
    uint32_t sx = 0;                                               // lane parities in bits 15 / 31
#pragma unroll
    for (int k = 0; k + 1 < D; k += 2) sx ^= d[k] ^ d[k + 1];
    if (D & 1) sx ^= d[D - 1];
    // lane parities only in the sign bits (for the lane-wise sign flip below)
    const uint32_t sxm = QCB_P16_ADDSIGN ? (sx & 0x80008000u) : sx;
    uint32_t exa[D];
    if constexpr (QCB_P16_MIN3 == 2 || (QCB_P16_MIN3 == 1 && ANCHOR)) {
      loo_minima3<D>(a, exa, [](uint32_t x, uint32_t y) { return vmin2(x, y); },
                     [](uint32_t x, uint32_t y, uint32_t z) { return vmin3(x, y, z); }, 0x7FFF7FFFu);
    } else if constexpr (ANCHOR) {
      loo_minima<D>(a, exa, [](uint32_t x, uint32_t y) { return vmin2(x, y); }, 0x7FFF7FFFu);
    } else {
      // suffix / prefix chains step two edges at a time (VIMNMX3.S16x2)
      uint32_t suf[D], pre[D];
      suf[D - 2] = a[D - 1];
#pragma unroll
      for (int k = D - 3; k >= 0; --k) {
        const int m = D - 1 - k;
        if (k == D - 3 || (m & 1)) suf[k] = vmin2(suf[k + 1], a[k + 1]);
        else suf[k] = vmin2(vmin2(suf[k + 2], a[k + 2]), a[k + 1]);
      }
      pre[1] = a[0];
#pragma unroll
      for (int k = 2; k < D; ++k) {
        if (k == 2 || (k & 1)) pre[k] = vmin2(pre[k - 1], a[k - 1]);
        else pre[k] = vmin2(vmin2(pre[k - 2], a[k - 2]), a[k - 1]);
      }
#pragma unroll
      for (int k = 0; k < D; ++k) exa[k] = k == 0 ? suf[0] : (k == D - 1 ? pre[D - 1] : vmin2(pre[k], suf[k]));
    }
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const uint32_t ex = exa[k];
      // sign of L_new per lane = sign(zz) ^ parity: the parity bit added to
      // bit 15 / 31 lane-wise (no carry leaves a lane) flips exactly that bit
      const uint32_t m = QCB_P16_ADDSIGN ? lane_signs(vadd2(d[k], sxm)) : lane_signs(d[k] ^ sx);
      if constexpr (XORSIGN) {
        // L_new = (ex + m) ^ m: a lane with m = 0xFFFF gets ~(ex - 1) = -ex
        // (wrapping: -(-32768) = -32768); the message's negation on the FMA pipe
        const uint32_t ln = vadd2(ex, m) ^ m;
        o[k] = vadd2(d[k], ln);                                    // post = zz + L_new
        nm[k] = vadd2(imad(ln, K.neg1, K.neg1), K.lane1);          // -L_new
      } else {
        const uint32_t nex = vadd2(imad(ex, K.neg1, K.neg1), K.lane1);   // -ex (wrapping)
        o[k] = vadd2(d[k], (nex & m) | (ex & ~m));                 // post = zz + L_new
        nm[k] = (ex & m) | (nex & ~m);                             // -L_new
      }
    }
  }
};

template <class S, int ZS>
struct Layered2 {
  using A = ArithI16x2;

  static constexpr bool TAB = use_addr_tab<S, A>();
  static constexpr int ME = tab_max_entries<S, ZS, TAB>();
  // table in global memory (native Z, one pair per CTA): `tab` is then the
  // thread's byte offset into g_p16_tab<S, ZS> and entries are relative to
  // the dynamic shared-memory base
  static constexpr bool GT = QCB_P16_GTAB && TAB && ZS > 0 && p16_gtab_units<S, ZS>() > 0;
  // tiers [0, TMT) keep their messages in TMEM columns [START[T], START[T+1])
  // of the thread's lane; the rest in registers (nm[e - TMC])
  static constexpr int kTmtWant = QCB_P16_TMT >= 0 ? QCB_P16_TMT : p16_tmt_default(S::ID);
  // (measured on the native codes only: scaled Z keep every message in registers)
  static constexpr int TMT = (ZS == S::Z0 && ZS > 32 && ZS <= 128) ? (kTmtWant < S::MB ? kTmtWant : S::MB - 1) : 0;
  static constexpr int TMC = S::START[TMT];
  static constexpr int NR = S::NE - TMC;
  static constexpr int TCOLS = TMC <= 32 ? 32 : (TMC <= 64 ? 64 : (TMC <= 128 ? 128 : 256));
  // several pairs per CTA (fixed iterations): warps w and w + 4 share TMEM
  // lanes (a warp reaches lanes 32 (w mod 4) ..), so each group of four warps
  // takes its own TMC columns; the allocation is the next power of two
  __host__ __device__ static constexpr int tm_cols(int warps) {
    const int need = ((warps + 3) / 4) * TMC;
    int c = 32;
    while (c < need) c *= 2;
    return c;
  }

  template <int T>
  __device__ __forceinline__ static void fetch(uint32_t tab, uint32_t* ent) {
    if constexpr (GT) {
      using AT = AddrTab<S, ZS, true>;
      if constexpr (T < S::MB) {
        constexpr int NU = (AT::count(T) + 1) / 2;
        const uint2* g = g_p16_tab<S, ZS> + (tab >> 3) + AT::unit0(T);
        const uint32_t sb = p16_sbase();
#pragma unroll
        for (int u = 0; u < NU; ++u) {
          const uint2 v = __ldg(g + u);
          ent[2 * u] = v.x + sb;
          ent[2 * u + 1] = v.y + sb;
        }
      }
    } else {
      tab_fetch<S, ZS, TAB, T>(tab, ent);
    }
  }
  template <int E0>
  __device__ __forceinline__ static void addrs(const SpecArgs& a, int r, uint32_t b0, uint32_t b1, uint32_t tab,
                                               uint32_t* addr) {
    constexpr int D = S::DEG[AddrTab<S, ZS, TAB>::tier_of(E0)];
    if constexpr (GT) {
      constexpr int T = AddrTab<S, ZS, TAB>::tier_of(E0);
      uint32_t ent[ME];
      fetch<T>(tab, ent);
      tab_compose<S, A, ZS, TAB, T>(a, r, b0, b1, ent, addr, std::make_integer_sequence<int, D>{});
    } else {
      tier_addrs_tab<S, A, ZS, TAB, E0>(a, r, b0, b1, tab, addr, std::make_integer_sequence<int, D>{});
    }
  }

  // keep: lanes of converged codewords (early termination) keep their posteriors;
  // pe / pn: this / the next tier's early-loaded posteriors (early_edge);
  // ec / en: this / the next tier's address-table entries
  template <int T, bool ET>
  __device__ __forceinline__ static void tier(const SpecArgs& a, const RtK& K, int r, uint32_t b0, uint32_t b1,
                                              uint32_t tab, uint32_t tb, uint32_t (&nm)[NR > 0 ? NR : 1],
                                              uint32_t keep, uint32_t (&pe)[S::MAXDEG], uint32_t (&pn)[S::MAXDEG],
                                              uint32_t (&ec)[ME], uint32_t (&en)[ME]) {
    constexpr int D = S::DEG[T];
    constexpr int E0 = S::START[T];
    constexpr bool XS = QCB_P16_XORSIGN == 1 || (QCB_P16_XORSIGN == 0 && S::ID == 7);
    uint32_t addr[D], p[D], o[D];
    uint32_t mt[T < TMT ? D : 1];
    if constexpr (T < TMT) {
      (void)tb;
      // Tier T reads the columns tier T stored one sweep ago.  One wait at tier
      // 0 covers every store of the previous sweep; waiting again at tiers 1..
      // TMT-1 would also wait for the store tier T-1 issued just before the
      // barrier (ncu, C5: those two waits held 5.8 % of all stall samples).
      if constexpr (T == 0 || !QCB_P16_TM_WAIT0) tm_wait_st();
      tm_ld_n<E0, D>(tb, mt);                    // overlaps the posterior loads below
    }
    tab_compose<S, A, ZS, TAB, T>(a, r, b0, b1, ec, addr, std::make_integer_sequence<int, D>{});
#pragma unroll
    for (int k = 0; k < D; ++k) p[k] = early_edge<S, T>(k) ? pe[k] : A::lds(addr[k]);
    if constexpr (!QCB_P16_TAB_LATE) fetch<T + 1>(tab, en);
    // sign application: two selects, or (ex + m) ^ m with the message negated
    // on the FMA pipe where measured faster (tools/exp/pc16_run.sh: Wi-Fi 1944
    // R5/6 = C3 +2.8 %; WiMAX 1/2 -4.8 %, 3/4A -2 %; others within +-1 %)
    if constexpr (T < TMT) {
      tm_wait_ld<D>(mt);
      A::template row<D, (S::ID >= 12), XS>(p, o, mt, K);
      tm_st_n<E0, D>(tb, mt);
    } else {
      A::template row<D, (S::ID >= 12), XS>(p, o, nm + (E0 - TMC), K);
    }
    // late: the next tier's table entries are not live across the row update
    if constexpr (QCB_P16_TAB_LATE) fetch<T + 1>(tab, en);
#pragma unroll
    for (int k = 0; k < D; ++k) {
      uint32_t v = o[k];
      if constexpr (ET) v = (v & ~keep) | (p[k] & keep);       // converged lanes keep their posteriors
      A::sts(addr[k], v);
    }
    if constexpr (T + 1 < S::MB && EarlyMask<S, T + 1>::value != 0) {
      constexpr int DN = S::DEG[T + 1];
      uint32_t an[DN];
      tab_compose<S, A, ZS, TAB, T + 1>(a, r, b0, b1, en, an, std::make_integer_sequence<int, DN>{});
#pragma unroll
      for (int k = 0; k < DN; ++k)
        if (early_edge<S, T + 1>(k)) pn[k] = A::lds(an[k]);
    }
  }

  template <int T>
  __device__ __forceinline__ static uint32_t parity(const SpecArgs& a, int r, uint32_t b0, uint32_t b1, uint32_t tab) {
    constexpr int D = S::DEG[T];
    constexpr int E0 = S::START[T];
    uint32_t addr[D];
    addrs<E0>(a, r, b0, b1, tab, addr);
    // hard = post <= 0 per lane: min(post - 1, post) is negative exactly for
    // post <= 0 (-32768 - 1 wraps to 32767, and the min then takes -32768 itself);
    // one VIADDMNMX.  XOR of the lane sign bits (15, 31) = the two codewords' row
    // parities
    uint32_t par = 0;
#pragma unroll
    for (int k = 0; k < D; ++k) par ^= hard_sign2(A::lds(addr[k]));
    return ((par >> 15) & 1u) | ((par >> 30) & 2u);
  }

  template <bool ET, int... Ts>
  __device__ __forceinline__ static void sweep(const SpecArgs& a, const RtK& K, int r, uint32_t b0, uint32_t b1,
                                               uint32_t tab, uint32_t tb, uint32_t (&nm)[NR > 0 ? NR : 1], bool work,
                                               uint32_t keep, std::integer_sequence<int, Ts...>) {
    uint32_t pa[S::MAXDEG], pb[S::MAXDEG];
    uint32_t ea[ME], eb[ME];
    fetch<0>(tab, ea);
    if constexpr (ET) {
      ((work ? tier<Ts, true>(a, K, r, b0, b1, tab, tb, nm, keep, (Ts & 1) ? pb : pa, (Ts & 1) ? pa : pb,
                              (Ts & 1) ? eb : ea, (Ts & 1) ? ea : eb)
             : void(),
        tier_sync<ZS, 2>()), ...);
    } else {
      (void)work; (void)keep;
      ((tier<Ts, false>(a, K, r, b0, b1, tab, tb, nm, 0u, (Ts & 1) ? pb : pa, (Ts & 1) ? pa : pb,
                        (Ts & 1) ? eb : ea, (Ts & 1) ? ea : eb),
        tier_sync<ZS, 2>()), ...);
    }
  }

  template <int... Ts>
  __device__ __forceinline__ static uint32_t parity_all(const SpecArgs& a, int r, uint32_t b0, uint32_t b1,
                                                        uint32_t tab, std::integer_sequence<int, Ts...>) {
    return (parity<Ts>(a, r, b0, b1, tab) | ...);
  }

  // Early-exit syndrome in QCB_ET_CHUNKS groups of tiers (see
  // Layered::parity_any): lane bits found odd are ORed into `flag`; a thread
  // stops once every lane in `need` is known to fail.  Returns this thread's
  // bits | the flag's (a set flag bit means some thread found that lane odd).
  static constexpr int kEtChunk = QCB_ET_CHUNKS > 0 ? (S::MB + QCB_ET_CHUNKS - 1) / QCB_ET_CHUNKS : 1;
  // QCB_ET_FIRST > 0: a first group of that many tiers (a cheap reject of a
  // codeword that has not converged), then all remaining tiers in one group
  template <int T0>
  static constexpr int et_len() {
    return QCB_ET_FIRST > 0 ? (T0 == 0 ? QCB_ET_FIRST : S::MB - QCB_ET_FIRST) : kEtChunk;
  }
  template <int T0, int... Is>
  __device__ __forceinline__ static uint32_t parity_group(const SpecArgs& a, int r, uint32_t b0, uint32_t b1,
                                                          uint32_t tab, std::integer_sequence<int, Is...>) {
    return ((T0 + Is < S::MB ? parity<(T0 + Is < S::MB ? T0 + Is : 0)>(a, r, b0, b1, tab) : 0u) | ...);
  }
  // QCB_ET_CHUNKS == 0: per tier, software-pipelined (see Layered::parity_pipe)
  template <int T>
  __device__ __forceinline__ static void parity_load(const SpecArgs& a, int r, uint32_t b0, uint32_t b1, uint32_t tab,
                                                     uint32_t (&v)[S::DEG[T]]) {
    constexpr int D = S::DEG[T];
    uint32_t addr[D];
    addrs<S::START[T]>(a, r, b0, b1, tab, addr);
#pragma unroll
    for (int k = 0; k < D; ++k) v[k] = A::lds(addr[k]);
  }
  template <int T>
  __device__ __forceinline__ static uint32_t lane_parity(const uint32_t (&v)[S::DEG[T]]) {
    constexpr int D = S::DEG[T];
    uint32_t par = 0;
#pragma unroll
    for (int k = 0; k < D; ++k) par ^= hard_sign2(v[k]);
    return ((par >> 15) & 1u) | ((par >> 30) & 2u);
  }
  template <int T>
  __device__ __forceinline__ static uint32_t parity_pipe(const SpecArgs& a, int r, uint32_t b0, uint32_t b1,
                                                         uint32_t tab, volatile int* flag, uint32_t need, uint32_t acc,
                                                         const uint32_t (&cur)[S::DEG[T]], uint32_t f_prev) {
    if constexpr (T + 1 < S::MB) {
      uint32_t nxt[S::DEG[T + 1]];
      parity_load<T + 1>(a, r, b0, b1, tab, nxt);
      const uint32_t f = (uint32_t)*flag;
      const uint32_t p = lane_parity<T>(cur) & need;
      if (p & ~acc) atomicOr((int*)flag, (int)p);
      acc |= p;
      if (((acc | f_prev) & need) == need) return acc | (f_prev & need);
      return parity_pipe<T + 1>(a, r, b0, b1, tab, flag, need, acc, nxt, f);
    } else {
      const uint32_t p = lane_parity<T>(cur) & need;
      if (p & ~acc) atomicOr((int*)flag, (int)p);           // published like every other tier's bits
      return acc | p | (f_prev & need);
    }
  }
  template <int T0>
  __device__ __forceinline__ static uint32_t parity_any(const SpecArgs& a, int r, uint32_t b0, uint32_t b1,
                                                        uint32_t tab, volatile int* flag, uint32_t need,
                                                        uint32_t acc = 0) {
#if QCB_ET_CHUNKS == 0
    uint32_t v0[S::DEG[0]];
    parity_load<0>(a, r, b0, b1, tab, v0);
    return parity_pipe<0>(a, r, b0, b1, tab, flag, need, 0u, v0, 0u);
#endif
    if constexpr (T0 >= S::MB) {
      return acc;
    } else {
      if (((acc | (uint32_t)*flag) & need) == need) return acc | ((uint32_t)*flag & need);
      const uint32_t p = parity_group<T0>(a, r, b0, b1, tab, std::make_integer_sequence<int, et_len<T0>()>{}) & need;
      if (p & ~acc) atomicOr((int*)flag, (int)p);
      return parity_any<T0 + et_len<T0>()>(a, r, b0, b1, tab, flag, need, acc | p);
    }
  }
};

#ifndef QCB_P16_SLACK
#define QCB_P16_SLACK 52
#endif
template <class S, int ZS>
constexpr int p16_reg_cap() {
  if constexpr (Layered2<S, ZS>::TMT > 0) return QCB_P16_TM_CAP > 0 ? QCB_P16_TM_CAP : p16_tm_cap(S::ID);
  const int z = ZS > 0 ? ZS : 96;
  const int cap = raise_cap(z, S::NE + QCB_P16_SLACK, cw_block_bytes(z), true, smsp_raise<S, ArithI16x2>());
  // 128 registers = 4 warps per sub-partition, paid for with spills; measured
  // per structure (tools/exp/pc16_ab.sh, Gb/s): Wi-Fi 1296 R1/2 75.1 -> 78.9,
  // 1944 R1/2 71.3 -> 74.1, R2/3 66.3 -> 67.1, R5/6 (C3) 65.4 -> 68.6, WiMAX
  // 2/3A 86.8 -> 88.4, 2/3B 86.4 -> 90.2; the other int16 codes lose 1..11 %.
#ifdef QCB_P16_CAP_MAX                                 // tuning experiments
  constexpr int kMax = QCB_P16_CAP_MAX;
#else
  constexpr int kMax =
      ((((1u << 0) | (1u << 4) | (1u << 5) | (1u << 7) | (1u << 13) | (1u << 14)) >> S::ID) & 1u) ? 128 : 255;
#endif
#ifdef QCB_P16_SCALED_CAP                              // tuning experiments: scaled Z only
  if constexpr (ZS > 0 && ZS != S::Z0) return cap > QCB_P16_SCALED_CAP ? QCB_P16_SCALED_CAP : cap;
#endif
  constexpr int kScaled = (ZS > 0 && ZS != S::Z0) ? scaled_reg_cap(S::ID, 2, ZS) : 0;   // see reg_cap
  if constexpr (kScaled > 0) return cap > kScaled ? kScaled : cap;
  return cap > kMax ? kMax : cap;
}

// Bytes between consecutive pair blocks in shared memory: the block itself
// (24 Z cells), padded to a multiple of 128 bytes (32 banks) when a CTA holds
// several pairs.  Z = 81: 1944 -> 1952 cells; measured on C3 (three pairs per
// CTA): shared-memory bank conflicts 25 % -> see DESIGN 3.2.  The scaled WiMAX Z
// (multiples of 4) are aligned already.
__host__ __device__ constexpr int p16_block_stride(int z, int pairs) {
  return blk_stride_bytes(z, pairs, true);     // chunked pairs: m banks apart (map_row)
}

// a.pairs = codeword PAIRS per CTA; codeword 2q of the CTA is lane 0 of pair q
template <class S, int ZS, bool ET>
__global__ void __launch_bounds__(kLayMaxThreads) __maxnreg__((p16_reg_cap<S, ZS>()))
    decode_pair16_kernel(const __grid_constant__ SpecArgs a) {
  using L = Layered2<S, ZS>;
  constexpr int MAXC = 2 * kLayMaxCw;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int s_fail[MAXC + 2], s_done[MAXC + 2], s_iters[MAXC + 2];   // + scratch pair
  __shared__ int s_active;
  __shared__ int s_odd2[2];                     // early-exit syndrome lane bits, per sweep parity (G == 1 with ET)
  __shared__ uint32_t s_taddr;                  // TMEM base (L::TMT > 0)

  const RtK K{a.k_one, a.k_sign, a.k_shr, a.k_neg1, a.k_lane1};
  const int Z = ZS > 0 ? ZS : a.z;
  const int N = S::NB * Z;
  const int G = a.pairs;
  const int tid = threadIdx.x;
  const int g = tid / Z, r = tid - g * Z;
  const int64_t cw0 = (int64_t)blockIdx.x * (2 * G);
  const int ncw = (int)(a.w - cw0 < (int64_t)(2 * G) ? a.w - cw0 : (int64_t)(2 * G));
  const int npairs = (ncw + 1) >> 1;
  // pair blocks: with several pairs per CTA the block stride is padded to a
  // multiple of 32 banks (p16_block_stride), so rows of two pairs in one warp
  // fall on banks offset only by their cells (C3's Z = 81: 24-bank offset)
  constexpr bool kPad = ZS != S::Z0 || ZS % 32 != 0;   // WiMAX native: compile-time stride (see decode_layered)
  const uint32_t cws = kPad ? (uint32_t)p16_block_stride(Z, G) : (uint32_t)cw_block_bytes(Z);
  const uint32_t cpad = kPad ? cws - (uint32_t)cw_block_bytes(Z) : 0u;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  dbg_check(cw0 < a.w && ncw >= 1 && ncw <= 2 * G, 22);       // the CTA's chunk lies inside the batch
  dbg_poison_smem();
  dbg_inject_probe(a.dbg_inject, sbase);
  // Padding lanes of the last warp (tid >= G*Z) shadow real lanes of the SAME
  // warp: same row, same inputs, same instruction stream, so in lockstep they
  // load and store the very words their twins do (same-word accesses: no bank
  // conflict, identical values).  A separate scratch block costs a 2-way bank
  // conflict on every access of that warp (measured: 48 % of Wi-Fi 648's
  // shared-memory wavefronts).
  const RowMap rm = map_row(tid, G, Z, kPad);
  const int gs = rm.g, rs = rm.r;
  const bool act = gs < npairs;
  uint32_t b0 = sbase + (uint32_t)gs * cws + (uint32_t)(rs * kCellBytes), b1;
  asm volatile("mov.b32 %0, %0;" : "+r"(b0));
  asm volatile("sub.u32 %0, %1, %2;" : "=r"(b1) : "r"(b0), "r"((uint32_t)(Z * kCellBytes)));
  constexpr int kTabB = L::GT ? 0 : addr_tab_bytes_per_thread<S, ZS, L::TAB>();   // shared-memory table bytes
  const uint32_t tab = L::GT ? (uint32_t)(tid * 8 * p16_gtab_units<S, ZS>())
                             : sbase + (uint32_t)G * cws + (uint32_t)(tid * kTabB);
  // early-termination snapshot block (G == 1), after the address tables
  const uint32_t snap_offset = ((uint32_t)G * cws + blockDim.x * (uint32_t)kTabB + 15u) & ~15u;
  if constexpr (!L::GT) fill_addr_tab<S, ArithI16x2, ZS, L::TAB>(a, rs, b0, b1, tab, std::make_integer_sequence<int, S::NE>{});

  if constexpr (L::TMT > 0) {                   // one warp allocates the CTA's message columns
    if (tid < 32) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                   ::"r"((uint32_t)__cvta_generic_to_shared(&s_taddr)), "r"((uint32_t)L::tm_cols(blockDim.x >> 5)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }

  // ---- channel LLRs of codewords 2q, 2q+1 -> lanes of [pair][c][j] ----------
  {
    if (kPad && cpad) load_llrs_pair16<true>(reinterpret_cast<const int16_t*>(a.llr) + cw0 * N, ncw, N, sbase, cpad);
    else load_llrs_pair16(reinterpret_cast<const int16_t*>(a.llr) + cw0 * N, ncw, N, sbase);
    for (int q = tid; q < MAXC + 2; q += blockDim.x) {
      s_fail[q] = 1; s_done[q] = q >= ncw; s_iters[q] = 0;
    }
    if (tid == 0) s_odd2[0] = s_odd2[1] = 0;
  }
  if constexpr (L::TMT > 0) asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  uint32_t tb = 0;                              // this thread's TMEM lane, column 0
  if constexpr (L::TMT > 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    tb = s_taddr + ((uint32_t)(32 * ((tid >> 5) & 3)) << 16) + (uint32_t)((tid >> 7) * L::TMC);
    uint32_t z8[8] = {0, 0, 0, 0, 0, 0, 0, 0};   // messages start at 0 (reference init)
#pragma unroll
    for (int c = 0; c + 8 <= L::TMC; c += 8) tm_st<8>(tb + c, z8);
    if constexpr (L::TMC % 8 >= 4) tm_st<4>(tb + (L::TMC / 8) * 8, z8);
    if constexpr (L::TMC % 4 >= 2) tm_st<2>(tb + (L::TMC / 4) * 4, z8);
    if constexpr (L::TMC % 2 == 1) tm_st<1>(tb + L::TMC - 1, z8);
  }

  uint32_t nm[L::NR > 0 ? L::NR : 1];
#pragma unroll
  for (int e = 0; e < (L::NR > 0 ? L::NR : 1); ++e) nm[e] = 0u;

  const auto tiers = std::make_integer_sequence<int, S::MB>{};
  if constexpr (!ET) {
    // fixed iterations: every codeword runs max_iters sweeps; one syndrome at the end
    for (int k = 0; k < a.max_iters; ++k) L::template sweep<false>(a, K, rs, b0, b1, tab, tb, nm, act, 0u, tiers);
    if (a.max_iters > 0) {
      if (tid < MAXC) s_fail[tid] = 0;
      __syncthreads();
      if (act) {
        const uint32_t par = L::parity_all(a, rs, b0, b1, tab, tiers);
        if (par & 1u) s_fail[2 * gs] = 1;
        if (par & 2u) s_fail[2 * gs + 1] = 1;
      }
      __syncthreads();
    }
    if (tid < ncw) s_iters[tid] = a.max_iters;
  } else if (G == 1) {
    // One pair per CTA.  Both lanes sweep unconditionally (no per-edge keep
    // blending); when one lane converges while the other continues, its
    // posteriors are saved to a snapshot block (that lane's halves only) and
    // restored before the outputs -- exactly the reference's frozen codeword.
    // The lanes' syndromes are reduced with __syncthreads_or.
    const uint32_t snap = sbase + (uint32_t)snap_offset;
    const int nwords = (int)(cws >> 2);
    int k = 0, it_a = 0, it_b = 0;
    int fail_a = 1, fail_b = 1;
    bool done_a = false, done_b = ncw < 2;
    uint32_t saved = 0;                                   // lane masks held in the snapshot
    while (k < a.max_iters && !(done_a && done_b)) {
      L::template sweep<false>(a, K, rs, b0, b1, tab, tb, nm, act, 0u, tiers);
      ++k;
#if QCB_ET_EARLY_EXIT
      // every odd lane bit a thread finds is published to this sweep's flag
      // (parity_any), so one barrier makes the flag the CTA-wide OR; the flags
      // alternate between sweeps, and the other one -- last read before this
      // sweep's tier barriers -- is cleared for the next sweep
      volatile int* fl = &s_odd2[k & 1];
      const uint32_t need = (done_a ? 0u : 1u) | (done_b ? 0u : 2u);
      if (act) L::template parity_any<0>(a, rs, b0, b1, tab, fl, need);
      __syncthreads();
      const uint32_t all = (uint32_t)*fl;
      if (tid == 0) s_odd2[(k + 1) & 1] = 0;
      const int fa = (int)(all & 1u), fb = (int)((all >> 1) & 1u);
#else
      const uint32_t par = act ? L::parity_all(a, rs, b0, b1, tab, tiers) : 0u;
      const int fa = __syncthreads_or((int)(par & 1u));
      const int fb = __syncthreads_or((int)(par & 2u));
#endif
      uint32_t newly = 0;
      if (!done_a) { it_a = k; fail_a = fa; done_a = !fa; if (done_a) newly |= 0x0000FFFFu; }
      if (!done_b) { it_b = k; fail_b = fb; done_b = !fb; if (done_b) newly |= 0xFFFF0000u; }
      if (newly && !(done_a && done_b)) {                 // freeze: save the converged lane
        for (int i = tid; i < nwords; i += blockDim.x) {
          const uint32_t live = lds32(sbase + 4u * i), old = lds32(snap + 4u * i);
          sts32(snap + 4u * i, (live & newly) | (old & ~newly));
        }
        saved |= newly;
        __syncthreads();
      }
    }
    if (saved) {                                          // restore the frozen lanes
      for (int i = tid; i < nwords; i += blockDim.x) {
        const uint32_t live = lds32(sbase + 4u * i), old = lds32(snap + 4u * i);
        sts32(sbase + 4u * i, (old & saved) | (live & ~saved));
      }
    }
    if (tid == 0) {
      s_iters[0] = it_a; s_fail[0] = fail_a;
      s_iters[1] = it_b; s_fail[1] = fail_b;
    }
    __syncthreads();
  } else if constexpr (L::TMT == 0) {           // several pairs per CTA (TMEM kernels launch one)
    for (int k = 0; k < a.max_iters; ++k) {
      const bool da = s_done[2 * gs], db = s_done[2 * gs + 1];
      const bool work = act && !(da && db);
      const uint32_t keep = (da ? 0x0000FFFFu : 0u) | (db ? 0xFFFF0000u : 0u);
      L::template sweep<true>(a, K, rs, b0, b1, tab, tb, nm, work, keep, tiers);
      if (tid < MAXC) s_fail[tid] = 0;          // syndrome (_kernels.py:85-96)
      __syncthreads();
      if (work) {
        const uint32_t par = L::parity_all(a, rs, b0, b1, tab, tiers);
        if (par & 1u) s_fail[2 * gs] = 1;
        if (par & 2u) s_fail[2 * gs + 1] = 1;
      }
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

  // ---- outputs ---------------------------------------------------------------
  if (tid < ncw) {
    a.iters[cw0 + tid] = s_iters[tid];
    a.conv[cw0 + tid] = (a.max_iters > 0 && !s_fail[tid]) ? 1 : 0;
  }
  {
    uint8_t* hard_out = reinterpret_cast<uint8_t*>(a.hard) + cw0 * (a.hard_packed ? (N + 7) >> 3 : N);
    int16_t* post_out = a.post ? reinterpret_cast<int16_t*>(a.post) + cw0 * N : nullptr;
    if (kPad && cpad) store_outputs_pair16<true>(hard_out, a.hard_packed, post_out, ncw, N, sbase, cpad);
    else store_outputs_pair16(hard_out, a.hard_packed, post_out, ncw, N, sbase);
  }
  if constexpr (L::TMT > 0) {                   // release the message columns
    tm_wait_st();
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (tid < 32)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_taddr),
                   "r"((uint32_t)L::tm_cols(blockDim.x >> 5)));
  }
}

template <class S, int ZS, int... Es>
__device__ __forceinline__ void p16_gtab_entries(const SpecArgs& a, int r, uint32_t b0, uint32_t b1, uint32_t* ent,
                                                 std::integer_sequence<int, Es...>) {
  using AT = AddrTab<S, ZS, true>;
#pragma unroll
  for (int i = 0; i < 2 * AT::units(); ++i) ent[i] = 0u;
  ((AT::in_tab(Es) ? (void)(ent[AT::entry(Es)] = edge_addr<S, ArithI16x2, ZS, Es>(a, r, b0, b1)) : void()), ...);
}

// g_p16_tab<S, ZS> for one pair per CTA: thread t's table entries relative to
// the dynamic shared-memory base (the decode kernel adds its base)
template <class S, int ZS>
__global__ void fill_p16_gtab_kernel(const __grid_constant__ SpecArgs a) {
  using AT = AddrTab<S, ZS, true>;
  constexpr int NU = AT::units();
  const int tid = threadIdx.x;
  const RowMap rm = map_row(tid, 1, ZS);
  const uint32_t b0 = (uint32_t)(rm.r * kCellBytes), b1 = b0 - (uint32_t)(ZS * kCellBytes);
  uint32_t ent[2 * NU];
  p16_gtab_entries<S, ZS>(a, rm.r, b0, b1, ent, std::make_integer_sequence<int, S::NE>{});
#pragma unroll
  for (int u = 0; u < NU; ++u) g_p16_tab<S, ZS>[tid * NU + u] = make_uint2(ent[2 * u], ent[2 * u + 1]);
}

// Fill g_p16_tab<S, ZS> on the current device before its first decode there.
// The fill is a stream-ordered kernel launch (capturable); a device is marked
// done only after a fill launched outside a graph capture (a captured fill
// that is never replayed must not count).
template <class S, int ZS>
inline cudaError_t ensure_p16_gtab(const SpecArgs& a, int threads, cudaStream_t s) {
  static std::mutex m;
  static unsigned done = 0;                               // bit per device (< 32 devices)
  const int dev = current_device();
  {
    std::lock_guard<std::mutex> lk(m);
    if (dev < 32 && ((done >> dev) & 1u)) return cudaSuccess;
  }
  fill_p16_gtab_kernel<S, ZS><<<1, threads, 0, s>>>(a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  e = cudaStreamIsCapturing(s, &cs);
  if (e != cudaSuccess) return e;
  if (cs == cudaStreamCaptureStatusNone && dev < 32) {
    std::lock_guard<std::mutex> lk(m);
    done |= 1u << dev;
  }
  return cudaSuccess;
}

template <class S, int ZS, bool ET>
inline cudaError_t launch_pair16(const SpecArgs& a, cudaStream_t s) {
  const int z = ZS > 0 ? ZS : a.z;
  auto kern = decode_pair16_kernel<S, ZS, ET>;
  cudaFuncAttributes fa;
  cudaError_t e = kernel_attributes((const void*)kern, &fa);
  if (e != cudaSuccess) return e;
  SpecArgs b = a;
  b.pairs = layered_cw_per_cta(z, (a.w + 1) / 2, fa.numRegs, 4,
                               ZS == S::Z0 ? native_fill_cw(2, S::ID) : lane_fill_cw(z, 2, S::ID));
  if constexpr (one_warp_cta<ZS, 2>()) b.pairs = 1;         // tier_sync is a warp barrier
  // per-thread global table: one pair; TMEM tiers: several pairs only with fixed
  // iterations (the multi-pair early-termination loop skips tiers per pair, and
  // tcgen05.ld/st are warp-collective)
  if constexpr (Layered2<S, ZS>::GT) b.pairs = 1;
  if constexpr (Layered2<S, ZS>::TMT > 0) {
    if (ET) b.pairs = 1;
  }
  while (b.pairs > 1 && (b.pairs * z + 31) / 32 * 32 > fa.maxThreadsPerBlock) --b.pairs;
  if ((b.pairs * z + 31) / 32 * 32 > fa.maxThreadsPerBlock) return cudaErrorLaunchOutOfResources;
  const int thr = (b.pairs * z + 31) / 32 * 32;
  const size_t cwsb = (ZS != S::Z0 || ZS % 32 != 0) ? (size_t)p16_block_stride(z, b.pairs) : (size_t)cw_block_bytes(z);
  constexpr int kTabB = Layered2<S, ZS>::GT ? 0 : addr_tab_bytes_per_thread<S, ZS, use_addr_tab<S, ArithI16x2>()>();
  const size_t smem = (((size_t)b.pairs * cwsb + (size_t)thr * kTabB + 15) & ~(size_t)15) +
                      (ET && b.pairs == 1 ? cwsb : 0);   // + snapshot block
  e = ensure_dyn_smem((const void*)kern, smem);
  if (e != cudaSuccess) return e;
  if constexpr (Layered2<S, ZS>::GT) {
    e = ensure_p16_gtab<S, ZS>(b, thr, s);
    if (e != cudaSuccess) return e;
  }
  const int64_t per = 2 * (int64_t)b.pairs;
  const int64_t blocks = (a.w + per - 1) / per;
  if (blocks <= 0) return cudaSuccess;
  kern<<<(unsigned)blocks, thr, smem, s>>>(b);
  return cudaGetLastError();
}

}  // namespace qcb
