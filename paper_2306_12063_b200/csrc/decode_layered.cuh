// decode_layered.cuh -- float32 layered single-scan min-sum on sm_100a for
// the 18 standard base-matrix structures (the int16 kernel, two codewords per
// thread in 16x2 lanes, is decode_pair16.cuh and reuses the addressing,
// address tables and early loads defined here).
//
// Reference: /root/reference/pkg/src/qcldpc/_kernels.py:17-100.  Bit-exact:
// every value the reference computes (zz = post - L_old, |zz|, min1/min2,
// L_new, post = zz + L_new, hard = post <= 0, the syndrome) is produced by the
// same float32 operation on the same operands; only the way selections are
// made differs.
//
// Mapping (why, with the ncu evidence):
//  * one thread = one check row r of every tier of ONE codeword; a CTA holds
//    one codeword (ceil(Z/32) warps); tiers run in sequence with one CTA
//    barrier between them (layered schedule); the Z rows of a tier touch
//    disjoint columns, so running them concurrently equals the reference's
//    row loop;
//  * posteriors live in shared memory in the codeword's own bit order: cell
//    (c, j) -- bit n = j Z + c, c = position inside the circulant, j = block
//    column -- at byte 4 n (the layout of the codeword's LLR row in HBM, so
//    prologue and epilogue are streaming 16-byte copies); the cyclic shift of
//    edge (j, e) is the indexed shared-memory read of cell ((r + e) mod Z, j)
//    -- no expanded H anywhere.  For the 18 native
//    codes Z and the shifts are compile-time constants; scaled WiMAX codes
//    take them from the kernel parameter block; the per-edge base select is
//    kept in registers or in a per-thread shared-memory address table,
//    whichever measured faster for the structure (use_addr_tab);
//  * the check-to-variable messages of a thread's rows are held explicitly,
//    one register per edge (the reference keeps them compressed as
//    min1/min2/argmin/sign bits and rebuilds L_old every sweep,
//    _kernels.py:62-63; keeping the rebuilt values is bit-identical and
//    removes that work from the inner loop);
//  * instruction mix is chosen for the measured pipe rates (tools/pipebench):
//    FADD/FADD2 are full rate, IMAD / VIADD.16x2 share the half-rate
//    FMA-heavy pipe, compare / select / logic / min-max share the half-rate
//    ALU pipe and IMAD.HI is quarter rate, so sign handling rides on IMAD and
//    the leave-one-out minima step two edges at a time with 3-input min.
//  A persistent variant that prefetched the next codeword's LLRs by bulk
//  copy was measured slower on C2 (68-74 vs 84 Gb/s: the outer block loop
//  cost registers and spills), so each CTA decodes one codeword.
#pragma once
#include <algorithm>
#include <cstdlib>
#include <utility>

#include "common.cuh"
#include "decode_io.cuh"
#include "kernels.h"
#include "launch_cache.h"
#include "scaled_plan_gen.h"

// early-termination syndrome with early exit (measured: tools/exp/ab_et.sh)
#ifndef QCB_ET_EARLY_EXIT
#define QCB_ET_EARLY_EXIT 1
#endif
#ifndef QCB_ET_FIRST
#define QCB_ET_FIRST 1
#endif
#ifndef QCB_ET_CHUNKS
#define QCB_ET_CHUNKS 2
#endif

namespace qcb {

constexpr int kLayMaxThreads = 384;
constexpr int kLayMaxCw = 16;

// Thread -> (codeword g, row r).  Rows are dealt out contiguously (lane l of
// warp w: row 32w + l) except for one codeword per CTA with W = ceil(Z/32) odd
// warps and W | Z (Wi-Fi Z = 81, WiMAX Z = 72, 84): then warp w takes rows
// w, w+W, w+2W, ...  Every tier reads cells c = (r + e) mod Z, so a warp's
// cells are then a whole residue class mod W, {y + W k}, whose 32-bank
// residues W k mod 32 are distinct (W odd): no bank conflicts, where 32
// consecutive rows wrapping at Z put up to two lanes on one bank.  Padding
// lanes shadow a real lane of the same warp (same row, same words, lockstep).
//
// Several codewords per CTA whose count G divides 32 and with m = 32 / G
// dividing Z ("chunked"): lane l of warp w takes row w m + (l mod m) of
// codeword l / m, and consecutive codeword blocks sit m banks apart
// (blk_stride_bytes).  Every lane of a warp then reads the same m cells
// (consecutive mod Z, so distinct mod m) of its own codeword, at bank
// (g m + c) mod 32: conflict-free for every shift, no idle lanes, Z / m warps
// (Z = 24, 40: G = 4; 48, 80: G = 2).  The contiguous mapping of several
// codewords put up to 0.5-1 extra wavefronts on every access (bank model over
// all shifts; ncu: 33 % of WiMAX 864 R3/4A's shared wavefronts).
struct RowMap {
  int g, r;
};
__host__ __device__ constexpr int chunk_m(int Z, int G) {
  return (G > 1 && 32 % G == 0 && Z % (32 / G) == 0) ? 32 / G : 0;
}
// bytes between consecutive codeword (pair) blocks in shared memory: the block
// (24 Z cells), offset to m banks for the chunked mapping, or (align32, several
// blocks) padded to a multiple of 32 banks
__host__ __device__ constexpr int blk_stride_bytes(int Z, int G, bool align32) {
  const int w = 24 * Z;
  return chunk_m(Z, G) ? 4 * (w + ((chunk_m(Z, G) - w % 32) % 32 + 32) % 32)
                       : ((align32 && G > 1) ? 4 * ((w + 31) / 32 * 32) : 4 * w);
}
#ifndef QCB_CHUNKED_ROWS
#define QCB_CHUNKED_ROWS 1
#endif
__device__ __forceinline__ RowMap map_row(int tid, int G, int Z, bool chunked = true) {
  if (QCB_CHUNKED_ROWS && chunked && chunk_m(Z, G)) {
    const int m = chunk_m(Z, G), lane = tid & 31;
    return RowMap{lane / m, (tid >> 5) * m + lane % m};
  }
  const int W = (Z + 31) >> 5;
  if (G == 1 && W > 1 && (W & 1) && Z % W == 0) {
    const int per = Z / W, lane = tid & 31;
    return RowMap{0, (tid >> 5) + W * (lane < per ? lane : lane % per)};
  }
  const int twin = tid < G * Z ? tid : (tid & ~31) + ((tid & 31) % (G * Z - (tid & ~31)));
  return RowMap{twin / Z, twin % Z};
}

// ---------------------------------------------------------------------------
// small PTX helpers: multipliers come from the parameter block (constant bank)
// so ptxas keeps them as IMAD (FMA-heavy pipe) instead of ALU shifts
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t imad(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// 3-input float min (PTX min.f32 with three sources -> FMNMX3): fminf
// semantics, NaN inputs ignored unless all are NaN
__device__ __forceinline__ float f_min3(float a, float b, float c) {
  float d;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
#ifndef QCB_F32_MIN3
#define QCB_F32_MIN3 1
#endif

// packed float32x2 add/sub (FADD2: two IEEE float32 ops in one instruction)
__device__ __forceinline__ void f_sub2(float a0, float a1, float b0, float b1, float& r0, float& r1) {
  asm("{\n\t.reg .b64 x, y, z;\n\tmov.b64 x, {%2, %3};\n\tmov.b64 y, {%4, %5};\n\t"
      "sub.rn.f32x2 z, x, y;\n\tmov.b64 {%0, %1}, z;\n\t}"
      : "=f"(r0), "=f"(r1) : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}
__device__ __forceinline__ void f_mul2(float a0, float a1, float b0, float b1, float& r0, float& r1) {
  asm("{\n\t.reg .b64 x, y, z;\n\tmov.b64 x, {%2, %3};\n\tmov.b64 y, {%4, %5};\n\t"
      "mul.rn.f32x2 z, x, y;\n\tmov.b64 {%0, %1}, z;\n\t}"
      : "=f"(r0), "=f"(r1) : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}
// measured (C2 / C4 Gb/s): 86.7 / 65.7 against 88.6 / 65.8 with the IMAD sign
// add -- 4 % fewer instructions, but FMUL2 lengthens the row's dependency
// chain in a kernel that is as much latency- as issue-bound: off
#ifndef QCB_F32_FMUL_SIGN
#define QCB_F32_FMUL_SIGN 0
#endif
// packed fused multiply-add: (a * b + c) per lane, one rounding each (FFMA2)
__device__ __forceinline__ void f_fma2(float a0, float a1, float b0, float b1, float c0, float c1, float& r0,
                                       float& r1) {
  asm("{\n\t.reg .b64 x, y, w, z;\n\tmov.b64 x, {%2, %3};\n\tmov.b64 y, {%4, %5};\n\tmov.b64 w, {%6, %7};\n\t"
      "fma.rn.f32x2 z, x, y, w;\n\tmov.b64 {%0, %1}, z;\n\t}"
      : "=f"(r0), "=f"(r1) : "f"(a0), "f"(a1), "f"(b0), "f"(b1), "f"(c0), "f"(c1));
}
// Sign application without the per-edge IMAD: c = copysign(ex, zz) (one LOP3),
// post = fma(c, +-1, zz) (FFMA2: the product is exact, so this is zz +- c with
// the one rounding of the reference's add) and the message c * +-1 (FMUL2, off
// the store's dependency chain): 2.5 instead of 3 instructions per edge.
// Measured per structure (round 2, tools/exp/r02_call40.sh, coded Gb/s at 65536
// codewords, IMAD -> FFMA2): Wi-Fi 1296 R1/2 63.3 -> 64.2, R3/4 60.3 -> 61.3, Wi-Fi
// 1944 R5/6 59.6 -> 60.4, WiMAX 2/3A 80.5 -> 81.2, 3/4A 69.7 -> 70.7, C1 43.5 ->
// 44.1; the rest within +-0.5 % except WiMAX 1/2 (C2: 88.3 -> 85.8, spills at its
// 128-register cap) and Wi-Fi 1944 R2/3 (57.2 -> 55.6), which keep the IMAD.
#ifndef QCB_F32_FMA_SIGN
#define QCB_F32_FMA_SIGN 1
#endif
template <class S>
constexpr bool f32_fma_sign() { return S::ID != 12 && S::ID != 5; }
__device__ __forceinline__ void f_add2(float a0, float a1, float b0, float b1, float& r0, float& r1) {
  asm("{\n\t.reg .b64 x, y, z;\n\tmov.b64 x, {%2, %3};\n\tmov.b64 y, {%4, %5};\n\t"
      "add.rn.f32x2 z, x, y;\n\tmov.b64 {%0, %1}, z;\n\t}"
      : "=f"(r0), "=f"(r1) : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}

// Leave-one-out minima ex[k] = min_{j != k} a[j] with prefix / suffix minima
// kept only at "anchor" positions two edges apart (3-input mins) and the
// remaining terms folded into each ex[k]: 2D - 2 mins for even D instead of
// 3D - 6 (D = 14: 26 vs 36).  `inf` seeds the anchors (int16: 32767, the
// reference's initial min, which every |zz| <= 32767 beats).  Used by the
// int16 kernel where measured faster (WiMAX structures: C5 +1.4 %; Wi-Fi 1944
// R5/6 -2.7 %, float32 C2 flat).
template <int D, class V, class Min>
__device__ __forceinline__ void loo_minima(const V (&a)[D], V (&ex)[D], Min mn, V inf) {
  static_assert(D >= 2, "row degree >= 2");
  if constexpr (D == 2) {
    ex[0] = mn(a[1], inf);
    ex[1] = mn(a[0], inf);
  } else {
    V P[D + 1], S[D + 1];
    P[2] = mn(mn(a[0], a[1]), inf);                       // P[k] = min a[0..k-1], k even
#pragma unroll
    for (int k = 4; k <= D - 1; k += 2) P[k] = mn(mn(P[k - 2], a[k - 2]), a[k - 1]);
    S[D - 3] = mn(mn(a[D - 2], a[D - 1]), inf);           // S[k] = min a[k+1..D-1], D-1-k even
#pragma unroll
    for (int k = D - 5; k >= 0; k -= 2) S[k] = mn(mn(S[k + 2], a[k + 2]), a[k + 1]);
#pragma unroll
    for (int k = 0; k < D; ++k) {
      // prefix part: none (k = 0) | a0 (k = 1) | P[k] (k even) | P[k-1], a[k-1]
      // suffix part: none (k = D-1) | a[D-1] (k = D-2) | S[k] (D-1-k even) | S[k+1], a[k+1]
      const bool p_anchor = k >= 2, s_anchor = k <= D - 3;
      V v;
      if (k == 0) v = ((D - 1) % 2 == 0) ? S[0] : mn(S[1], a[1]);
      else if (k == D - 1) v = (k % 2 == 0) ? P[k] : mn(P[k - 1], a[k - 1]);
      else {
        const V pp = (k == 1) ? a[0] : ((k % 2 == 0) ? P[k] : mn(P[k - 1], a[k - 1]));
        const V ss = (k == D - 2) ? a[D - 1] : (((D - 1 - k) % 2 == 0) ? S[k] : mn(S[k + 1], a[k + 1]));
        v = mn(pp, ss);
        if (!p_anchor && !s_anchor) v = mn(v, inf);       // D = 3, k = 1: no seeded anchor involved
      }
      ex[k] = v;
    }
  }
}

// The same leave-one-out minima with every 3-term minimum handed to ptxas as
// ONE inline-asm block (min3).  Composed from separate 2-input asm mins, the
// compiler CSEs the shared inner terms (P[k-1] min a[k-1] feeds both P[k+1] and
// ex[k]), after which ptxas cannot form VIMNMX3 and emits ~3D - 6 two-input
// mins; as separate blocks every term becomes one VIMNMX3 (same issue cost as
// a VIMNMX, measured: tools/exp/vmin3_bench.cu): 28 instead of 37 instructions
// for D = 14.
template <int D, class V, class Min, class Min3>
__device__ __forceinline__ void loo_minima3(const V (&a)[D], V (&ex)[D], Min mn, Min3 mn3, V inf) {
  static_assert(D >= 2, "row degree >= 2");
  if constexpr (D == 2) {
    ex[0] = mn(a[1], inf);
    ex[1] = mn(a[0], inf);
  } else if constexpr (D == 3) {
    ex[0] = mn3(a[1], a[2], inf);
    ex[1] = mn3(a[0], a[2], inf);
    ex[2] = mn3(a[0], a[1], inf);
  } else {
    V P[D + 1], S[D + 1];
    P[2] = mn3(a[0], a[1], inf);                          // P[k] = min a[0..k-1], k even
#pragma unroll
    for (int k = 4; k <= D - 1; k += 2) P[k] = mn3(P[k - 2], a[k - 2], a[k - 1]);
    S[D - 3] = mn3(a[D - 2], a[D - 1], inf);              // S[k] = min a[k+1..D-1], D-1-k even
#pragma unroll
    for (int k = D - 5; k >= 0; k -= 2) S[k] = mn3(S[k + 2], a[k + 2], a[k + 1]);
#pragma unroll
    for (int k = 0; k < D; ++k) {
      V v;
      if (k == 0) v = ((D - 1) % 2 == 0) ? S[0] : mn(S[1], a[1]);
      else if (k == D - 1) v = (k % 2 == 0) ? P[k] : mn(P[k - 1], a[k - 1]);
      else if (k == 1) v = ((D - 2) % 2 == 0) ? mn(a[0], S[1]) : mn3(a[0], S[2], a[2]);
      else if (k == D - 2) v = (k % 2 == 0) ? mn(P[k], a[D - 1]) : mn3(P[k - 1], a[k - 1], a[D - 1]);
      else if (k % 2 == 0) v = ((D - 1 - k) % 2 == 0) ? mn(P[k], S[k]) : mn3(P[k], S[k + 1], a[k + 1]);
      else v = ((D - 1 - k) % 2 == 0) ? mn3(P[k - 1], a[k - 1], S[k]) : mn(mn3(P[k - 1], a[k - 1], S[k + 1]), a[k + 1]);
      ex[k] = v;
    }
  }
}

struct RtK {              // runtime constants (kernel parameters)
  uint32_t one, sign, shr, neg1, lane1;   // lane1 = 0x00010001 (16x2 kernels)
};

// ---------------------------------------------------------------------------
// float32 row update (_kernels.py:49-84), messages msg[k] = L_mn of edge k
// ---------------------------------------------------------------------------
struct ArithF32 {
  using Val = float;                     // posterior / message value
  static constexpr int kElem = 4;        // bytes per shared-memory cell
  static constexpr int kKind = 0;        // address-table policy key (use_addr_tab)

  __device__ static Val lds(uint32_t a) {
    dbg_smem(a, 4, 9);
    float v; asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a)); return v;
  }
  __device__ static void sts(uint32_t a, Val v) {
    dbg_smem(a, 4, 10);
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
  }
  __device__ static bool hard(Val v) { return v <= 0.0f; }
  __device__ static Val zero() { return 0.0f; }   // reference init: min1 = min2 = 0, no signs -> L = +0.0
  // Channel LLRs enter shared memory as v + 0.0f: -0.0 becomes +0.0 and any
  // NaN becomes the GPU's canonical NaN (sign bit clear).  From then on no
  // posterior and no zz = post - L_old is ever -0.0 (IEEE: x - y = -0 needs
  // x = -0, x + y = -0 needs both -0) and no NaN carries a sign, so the sign
  // bit of zz equals the reference's `zz < 0` (_kernels.py:73) and can be used
  // directly.  The only observable difference is the sign of an exactly-zero
  // posterior (compares equal; hard decisions, messages and iteration counts
  // are identical).
  __device__ static float canon(float v) { return f_add(v, 0.0f); }

  // Leave-one-out formulation: |L_new_k| = min_{j != k} |zz_j| (prefix and
  // suffix minima).  This is the reference's (k == argmin ? min2 : min1)
  // exactly: for k != argmin the minimum over j != k still contains min1; for
  // k == argmin it is the second smallest with multiplicity (= min2, ties
  // included).  NaN |zz| never wins (fminf ignores NaN, as the reference's
  // `a < nm1` / `a < nm2` do) and the chains are seeded with +inf, the
  // reference's initial min1 / min2.  3*D - 6 min instructions per row
  // instead of ~2.1*D for min1/min2 plus 2*D for the per-edge min1/min2 pick.
  template <int D, bool FMA = false>
  __device__ __forceinline__ static void row(const Val (&p)[D], Val (&o)[D], Val* msg, const RtK& K) {
    static_assert(D >= 2, "row degree >= 2");
    float zz[D];
    // pass 1: zz = post - L_old (_kernels.py:61-75); sign parity = xor of sign bits
#pragma unroll
    for (int k = 0; k + 1 < D; k += 2) f_sub2(p[k], p[k + 1], msg[k], msg[k + 1], zz[k], zz[k + 1]);
    if (D & 1) zz[D - 1] = f_sub(p[D - 1], msg[D - 1]);
    uint32_t sx = 0;
#pragma unroll
    for (int k = 0; k + 1 < D; k += 2) sx ^= __float_as_uint(zz[k]) ^ __float_as_uint(zz[k + 1]);
    if (D & 1) sx ^= __float_as_uint(zz[D - 1]);
    const uint32_t sxm = sx & 0x80000000u;
    // leave-one-out minima of |zz|
    // chains step two edges at a time through 3-input mins (FMNMX3), odd
    // entries hang off them: depth ~D/2 instead of D, same instruction count
    float ex[D];
#if QCB_F32_MIN3
    {
      float az[D];
#pragma unroll
      for (int k = 0; k < D; ++k) az[k] = fabsf(zz[k]);      // |.| folds into FMNMX3 operand modifiers
      loo_minima3<D>(az, ex, [](float x, float y) { return fminf(x, y); },
                     [](float x, float y, float z) { return f_min3(x, y, z); }, f_inf());
    }
#else
    float pre[D], suf[D];
    pre[1] = fabsf(zz[0]);
#pragma unroll
    for (int k = 2; k < D; ++k) {
      if (k == 2) pre[2] = fminf(fminf(fabsf(zz[0]), fabsf(zz[1])), f_inf());
      else if (k & 1) pre[k] = fminf(pre[k - 1], fabsf(zz[k - 1]));
      else pre[k] = fminf(fminf(pre[k - 2], fabsf(zz[k - 2])), fabsf(zz[k - 1]));
    }
    suf[D - 2] = fabsf(zz[D - 1]);
#pragma unroll
    for (int k = D - 3; k >= 0; --k) {
      const int m = D - 1 - k;                  // number of |zz| folded into suf[k]
      if (k == D - 3) suf[k] = fminf(fminf(fabsf(zz[D - 1]), fabsf(zz[D - 2])), f_inf());
      else if (m & 1) suf[k] = fminf(suf[k + 1], fabsf(zz[k + 1]));
      else suf[k] = fminf(fminf(suf[k + 2], fabsf(zz[k + 2])), fabsf(zz[k + 1]));
    }
    ex[0] = D == 2 ? fminf(suf[0], f_inf()) : suf[0];
    ex[D - 1] = D == 2 ? fminf(pre[D - 1], f_inf()) : pre[D - 1];
#pragma unroll
    for (int k = 1; k < D - 1; ++k) ex[k] = fminf(pre[k], suf[k]);
#endif
    // pass 2 (_kernels.py:76-79): L_new = +-ex, sign = parity ^ sign(zz_k)
    if constexpr (FMA && QCB_F32_FMA_SIGN) {
      const float sp = __uint_as_float(0x3F800000u | sxm);   // -1.0f for an odd row, else +1.0f
      float cs[D];
#pragma unroll
      for (int k = 0; k < D; ++k) {
        uint32_t t;
        asm("lop3.b32 %0, %1, %2, 0x80000000, 0xF8;" : "=r"(t) : "r"(__float_as_uint(ex[k])), "r"(__float_as_uint(zz[k])));  // ex | (zz & sign)
        cs[k] = __uint_as_float(t);
      }
#pragma unroll
      for (int k = 0; k + 1 < D; k += 2) f_fma2(cs[k], cs[k + 1], sp, sp, zz[k], zz[k + 1], o[k], o[k + 1]);
      if (D & 1) o[D - 1] = __fmaf_rn(cs[D - 1], sp, zz[D - 1]);
#pragma unroll
      for (int k = 0; k + 1 < D; k += 2) f_mul2(cs[k], cs[k + 1], sp, sp, msg[k], msg[k + 1]);
      if (D & 1) msg[D - 1] = __fmul_rn(cs[D - 1], sp);
      return;
    }
#if QCB_F32_FMUL_SIGN
    // copysign(ex, zz) in one LOP3 (ex >= 0), then the row parity applied to
    // two edges at once by FMUL2 with (+-1, +-1): multiplying by -1 flips the
    // sign bit exactly (zeros and infinities included; ex is never NaN, the
    // minima are seeded with +inf), 0.5 FMA-pipe instructions per edge where
    // the sign-bit add needed one IMAD
    const float sp = __uint_as_float(0x3F800000u | sxm);   // -1.0f for an odd row, else +1.0f
    float cs[D];
#pragma unroll
    for (int k = 0; k < D; ++k) {
      uint32_t t;
      asm("lop3.b32 %0, %1, %2, 0x80000000, 0xF8;" : "=r"(t) : "r"(__float_as_uint(ex[k])), "r"(__float_as_uint(zz[k])));  // ex | (zz & sign)
      cs[k] = __uint_as_float(t);
    }
#pragma unroll
    for (int k = 0; k + 1 < D; k += 2) f_mul2(cs[k], cs[k + 1], sp, sp, msg[k], msg[k + 1]);
    if (D & 1) msg[D - 1] = __fmul_rn(cs[D - 1], sp);
#else
    // ex >= 0, so the sign is added to the bit pattern (IMAD, FMA pipe)
#pragma unroll
    for (int k = 0; k < D; ++k) {
      uint32_t t;
      asm("lop3.b32 %0, %1, %2, 0x80000000, 0x28;" : "=r"(t) : "r"(__float_as_uint(zz[k])), "r"(sxm));  // (zz ^ sxm) & sign
      msg[k] = __uint_as_float(imad(t, K.one, __float_as_uint(ex[k])));
    }
#endif
#pragma unroll
    for (int k = 0; k + 1 < D; k += 2) f_add2(zz[k], zz[k + 1], msg[k], msg[k + 1], o[k], o[k + 1]);
    if (D & 1) o[D - 1] = f_add(zz[D - 1], msg[D - 1]);
  }
};

// ---------------------------------------------------------------------------
// addressing
// ---------------------------------------------------------------------------

template <class S, class A, int ZS, int E>
__device__ __forceinline__ uint32_t edge_addr(const SpecArgs& a, int r, uint32_t b0, uint32_t b1) {
  if constexpr (ZS > 0) {
    constexpr int sh = zshift<S, ZS>(E);
    constexpr uint32_t off = (uint32_t)((S::COL[E] * ZS + sh) * A::kElem);   // cell (c = r + sh, j)
    if constexpr (sh == 0) return b0 + off;
    else return (r >= ZS - sh ? b1 : b0) + off;
  } else {
    return (r >= a.thr[E] ? b1 : b0) + (uint32_t)a.off[E];
  }
}

template <class S, class A, int ZS, int E0, int... Ks>
__device__ __forceinline__ void tier_addrs(const SpecArgs& a, int r, uint32_t b0, uint32_t b1, uint32_t* addr,
                                           std::integer_sequence<int, Ks...>) {
  ((addr[Ks] = edge_addr<S, A, ZS, E0 + Ks>(a, r, b0, b1)), ...);
}

// Per-thread shared-memory address table.  Every edge whose circulant shift
// is not a compile-time zero needs `(r >= Z - e) ? b1 : b0` (ISETP + SEL on
// the half-rate ALU pipe: 21 % of the float32 kernel's ALU instructions on
// C2, measured); the addresses are the same in every sweep, so each thread
// computes them once and keeps them in shared memory, and a tier fetches its
// addresses with one LDS.64 per two edges (the LSU pipe has the headroom).
// Layout [thread][unit], unit = 2 addresses, an odd number of units per
// thread so that a half-warp's LDS.64 hits 16 distinct bank pairs.
#ifndef QCB_ADDR_TAB
#define QCB_ADDR_TAB 1
#endif
// Measured per structure (tools/exp/percode.py, round 1, table vs selects):
// float32 gains on WiMAX 2/3B, 3/4A, 3/4B (+7..11 %) and Wi-Fi 1944 R2/3, R3/4
// (+3 %, re-measured after the shadow-lane change) and loses elsewhere (up to
// -11 %: those keep enough addresses hoisted in registers); the int16 pair
// kernel gains on all WiMAX codes (+5..24 %) and Wi-Fi 1944 R2/3, R3/4
// (+16 %), loses on Wi-Fi 648 R3/4, R5/6 and 1296 R5/6.
template <class S, class A>
constexpr bool use_addr_tab() {
#ifdef QCB_F32_TAB_MASK
  constexpr unsigned kF32 = QCB_F32_TAB_MASK;   // tuning experiments
#else
  constexpr unsigned kF32 = (1u << 5) | (1u << 6) | (1u << 14) | (1u << 15) | (1u << 16);
#endif
#ifdef QCB_P16_TAB_MASK
  constexpr unsigned kPair16 = QCB_P16_TAB_MASK;   // tuning experiments
#else
  // re-measured after the 3-input minima and register caps (tools/exp/tab_ab.sh):
  // Wi-Fi 648 R1/2 drops its table (+2.7 %), 648 R3/4 and 1296 R2/3 take one
  // (+6.9 / +1.8 %); float32 unchanged (all / none within 1 % of this policy)
  // round 2: Wi-Fi 1944 R5/6 (C3) takes one too now that its first tiers'
  // messages sit in TMEM: 89.7 -> 97.8 Gb/s (tools/exp/r02_call4.sh)
  constexpr unsigned kPair16 = 0x7u | (0xFu << 4) | (0x3u << 9) | (0x3Fu << 12);
#endif
  return QCB_ADDR_TAB && ((A::kKind == 0 && ((kF32 >> S::ID) & 1u)) || (A::kKind == 2 && ((kPair16 >> S::ID) & 1u)));
}

template <class S, int ZS, bool TAB>
struct AddrTab {
  static constexpr bool in_tab(int e) { return TAB && (ZS == 0 || zshift<S, ZS>(e) != 0); }
  static constexpr int tier_of(int e) {
    int t = 0;
    while (S::START[t + 1] <= e) ++t;
    return t;
  }
  static constexpr int count(int t) {
    int c = 0;
    for (int e = S::START[t]; e < S::START[t + 1]; ++e) c += in_tab(e) ? 1 : 0;
    return c;
  }
  static constexpr int unit0(int t) {
    int u = 0;
    for (int i = 0; i < t; ++i) u += (count(i) + 1) / 2;
    return u;
  }
  static constexpr int units() {
    const int u = unit0(S::MB);
    return u == 0 ? 0 : (u | 1);
  }
  static constexpr int entry(int e) {           // index in the thread's flat table
    const int t = tier_of(e);
    int c = 0;
    for (int x = S::START[t]; x < e; ++x) c += in_tab(x) ? 1 : 0;
    return 2 * unit0(t) + c;
  }
};

__device__ __forceinline__ uint2 lds64(uint32_t a) {
  uint2 v;
  dbg_smem(a, 8, 5);
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts64(uint32_t a, uint32_t x, uint32_t y) {
  dbg_smem(a, 8, 6);
  asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(a), "r"(x), "r"(y) : "memory");
}

template <class S, class A, int ZS, bool TAB, int E>
__device__ __forceinline__ uint32_t tab_pick(const SpecArgs& a, int r, uint32_t b0, uint32_t b1, const uint32_t* ent,
                                             int base) {
  if constexpr (AddrTab<S, ZS, TAB>::in_tab(E)) return ent[AddrTab<S, ZS, TAB>::entry(E) - base];
  else return edge_addr<S, A, ZS, E>(a, r, b0, b1);
}

// addresses of tier T's edges: table entries + the compile-time zero-shift ones
template <class S, class A, int ZS, bool TAB, int E0, int... Ks>
__device__ __forceinline__ void tier_addrs_tab(const SpecArgs& a, int r, uint32_t b0, uint32_t b1, uint32_t tab,
                                               uint32_t* addr, std::integer_sequence<int, Ks...>) {
  using AT = AddrTab<S, ZS, TAB>;
  constexpr int T = AT::tier_of(E0);
  constexpr int NU = (AT::count(T) + 1) / 2;
  uint32_t ent[2 * NU + 2];
#pragma unroll
  for (int u = 0; u < NU; ++u) {
    const uint2 v = lds64(tab + (uint32_t)((AT::unit0(T) + u) * 8));
    ent[2 * u] = v.x;
    ent[2 * u + 1] = v.y;
  }
  ((addr[Ks] = tab_pick<S, A, ZS, TAB, E0 + Ks>(a, r, b0, b1, ent, 2 * AT::unit0(T))), ...);
}

// split form: fetch tier T's table entries (issued a tier ahead), then compose
template <class S, int ZS, bool TAB>
constexpr int tab_max_entries() {
  int m = 2;
  for (int t = 0; t < S::MB; ++t) {
    const int e = 2 * ((AddrTab<S, ZS, TAB>::count(t) + 1) / 2);
    if (e > m) m = e;
  }
  return m;
}
template <class S, int ZS, bool TAB, int T>
__device__ __forceinline__ void tab_fetch(uint32_t tab, uint32_t* ent) {
  using AT = AddrTab<S, ZS, TAB>;
  if constexpr (T < S::MB) {
    constexpr int NU = (AT::count(T) + 1) / 2;
#pragma unroll
    for (int u = 0; u < NU; ++u) {
      const uint2 v = lds64(tab + (uint32_t)((AT::unit0(T) + u) * 8));
      ent[2 * u] = v.x;
      ent[2 * u + 1] = v.y;
    }
  }
}
template <class S, class A, int ZS, bool TAB, int T, int... Ks>
__device__ __forceinline__ void tab_compose(const SpecArgs& a, int r, uint32_t b0, uint32_t b1, const uint32_t* ent,
                                            uint32_t* addr, std::integer_sequence<int, Ks...>) {
  ((addr[Ks] = tab_pick<S, A, ZS, TAB, S::START[T] + Ks>(a, r, b0, b1, ent, 2 * AddrTab<S, ZS, TAB>::unit0(T))), ...);
}

template <class S, class A, int ZS, bool TAB, int... Es>
__device__ __forceinline__ void fill_addr_tab(const SpecArgs& a, int r, uint32_t b0, uint32_t b1, uint32_t tab,
                                              std::integer_sequence<int, Es...>) {
  using AT = AddrTab<S, ZS, TAB>;
  constexpr int NU = AT::units();
  if constexpr (NU > 0) {
    uint32_t ent[2 * NU];
#pragma unroll
    for (int i = 0; i < 2 * NU; ++i) ent[i] = 0u;
    ((AT::in_tab(Es) ? (void)(ent[AT::entry(Es)] = edge_addr<S, A, ZS, Es>(a, r, b0, b1)) : void()), ...);
#pragma unroll
    for (int u = 0; u < NU; ++u) sts64(tab + (uint32_t)(u * 8), ent[2 * u], ent[2 * u + 1]);
  }
}
template <class S, int ZS, bool TAB>
constexpr int addr_tab_bytes_per_thread() { return AddrTab<S, ZS, TAB>::units() * 8; }

// Edge k of tier T reads a block column that tier T-1 does not write: its
// posterior is final once tier T-2's barrier has passed, so it can be loaded
// before tier T-1's barrier (a tier writes exactly its own block
// columns).  WiMAX R1/2: 48 of 70 tier-to-tier loads; R3/4A: 29 of 71.
// float32 row parity from sign bits of post - 2^-149 (FADD) instead of
// compare-and-select: measured 84.0 vs 83.5 Gb/s with fixed iterations but
// 66 vs 72 under early termination (WiMAX 1/2, 1.5 dB), so off by default
#ifndef QCB_F32_SIGN_PARITY
#define QCB_F32_SIGN_PARITY 0
#endif
#ifndef QCB_EARLY_LOADS
#define QCB_EARLY_LOADS 1
#endif
template <class S, int T>
constexpr uint32_t early_mask_of() {
  if (T <= 0 || T >= S::MB || !QCB_EARLY_LOADS) return 0u;
  uint32_t m = 0;
  for (int k = 0; k < S::DEG[T]; ++k) {
    const int j = S::COL[S::START[T] + k];
    bool early = true;
    for (int e = S::START[T - 1]; e < S::START[T]; ++e)
      if (S::COL[e] == j) early = false;
    if (early) m |= 1u << k;
  }
  return m;
}
template <class S, int T>
struct EarlyMask { static constexpr uint32_t value = early_mask_of<S, T>(); };
template <class S, int T>
__device__ __forceinline__ constexpr bool early_edge(int k) { return (EarlyMask<S, T>::value >> k) & 1u; }

// Shared-memory message slots: the messages of the first SMT tiers can live in
// shared memory instead of registers (whole tiers, 16-byte aligned per tier,
// an odd number of 16-byte units per thread so quarter-warp LDS.128 / STS.128
// are conflict-free); fewer registers per thread, more resident CTAs.
// Measured on B200 (C2 / C4 / C1 Gb/s): SMT = 0: 83.7 / 58.2 / 29.5;
// 2: 78.8 / 54.6 / 28.8; 4 (7 CTAs/SM instead of 5): 74.5 / 48.2 / 29.0;
// 6: 70.0 / 42.3 / 26.8 -- the row update is not occupancy-bound, so the
// default keeps every message in registers.
#ifndef QCB_SMEM_MSG_TIERS
#define QCB_SMEM_MSG_TIERS 0
#endif
template <class S>
struct SmemMsg {
  static constexpr int SMT = QCB_SMEM_MSG_TIERS < S::MB ? QCB_SMEM_MSG_TIERS : S::MB;
  static constexpr int r4(int d) { return (d + 3) / 4 * 4; }
  static constexpr int off(int t) {            // word offset of tier t's slots
    int o = 0;
    for (int i = 0; i < t; ++i) o += r4(S::DEG[i]);
    return o;
  }
  static constexpr int words() {                // per-thread stride in words (0 if unused)
    const int w = off(SMT);
    if (w == 0) return 0;
    int u = w / 4;
    if ((u & 1) == 0) ++u;
    return 4 * u;
  }
  static constexpr int in_regs() { return S::NE - S::START[SMT]; }   // messages still in registers
};

__device__ __forceinline__ float4 lds128f(uint32_t a) {
  float4 v;
  dbg_smem(a, 16, 7);
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts128f(uint32_t a, float x, float y, float z, float w) {
  dbg_smem(a, 16, 8);
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(x), "f"(y), "f"(z), "f"(w) : "memory");
}

// The layered schedule runs the Z rows of a tier concurrently (one thread
// per row, one barrier per tier).  That equals the reference's sequential row
// loop (_kernels.py:47-48) only if no two rows of a tier touch the same
// posterior cell: each circulant is a permutation of the Z cells of its block
// column, so it suffices that a tier holds every block column at most once
// (codebook.py:249).  Checked here at compile time for every
// structure, together with the shift ranges at the native Z0 and at every
// scaled Z the per-Z decoders are compiled for.
template <class S>
constexpr bool tiers_column_disjoint() {
  for (int t = 0; t < S::MB; ++t)
    for (int e = S::START[t]; e < S::START[t + 1]; ++e)
      for (int f = e + 1; f < S::START[t + 1]; ++f)
        if (S::COL[e] == S::COL[f]) return false;
  return true;
}
template <class S, int Z>
constexpr bool shifts_in_range() {
  for (int e = 0; e < S::NE; ++e)
    if (zshift<S, Z>(e) < 0 || zshift<S, Z>(e) >= Z) return false;
  return true;
}
template <class S>
constexpr bool scaled_shifts_in_range() {
  if constexpr (S::Z0 != 96) return true;
  else
    return shifts_in_range<S, 24>() && shifts_in_range<S, 28>() && shifts_in_range<S, 32>() &&
           shifts_in_range<S, 36>() && shifts_in_range<S, 40>() && shifts_in_range<S, 44>() &&
           shifts_in_range<S, 48>() && shifts_in_range<S, 52>() && shifts_in_range<S, 56>() &&
           shifts_in_range<S, 60>() && shifts_in_range<S, 64>() && shifts_in_range<S, 68>() &&
           shifts_in_range<S, 72>() && shifts_in_range<S, 76>() && shifts_in_range<S, 80>() &&
           shifts_in_range<S, 84>() && shifts_in_range<S, 88>() && shifts_in_range<S, 92>();
}
#define QCB_STRUCT_CHECKS(STRUCT)                                                            \
  static_assert(tiers_column_disjoint<STRUCT>(), "a tier holds a block column twice");     \
  static_assert(shifts_in_range<STRUCT, STRUCT::Z0>(), "native shift outside [0, Z0)");    \
  static_assert(scaled_shifts_in_range<STRUCT>(), "scaled shift outside [0, Z)");
QCB_FOR_EACH_STRUCTURE(QCB_STRUCT_CHECKS)
#undef QCB_STRUCT_CHECKS

// Tier barrier.  A one-warp CTA (native Z <= 32: Wi-Fi 648, one codeword per
// CTA, forced at launch) needs no CTA barrier between tiers: __syncwarp
// orders the warp's shared-memory stores before its lanes' next loads.
#ifndef QCB_WARP_SYNC
#define QCB_WARP_SYNC 1
#endif
#ifndef QCB_Z24_CTA
#define QCB_Z24_CTA 0      // 1: Z = 24 codes take CTA barriers (several codewords per CTA) instead
#endif
// KIND = the arithmetic's kKind.  The int16 pair kernel at Z = 24 (scaled
// WiMAX N = 576) instead packs four codeword pairs into three full warps with
// CTA barriers: 90.7 vs 78.7 Gb/s (WiMAX 576 R1/2; +10..21 % on all six
// rates), where float32 keeps the one-warp CTA (72.2 vs 61.8 at G = 1, 60.6
// at G = 4; round 2, tools/exp/r02_call4.sh).
template <int ZS, int KIND = 0>
constexpr bool one_warp_cta() {
  return QCB_WARP_SYNC && ZS > 0 && ZS <= 32 && !((QCB_Z24_CTA || KIND == 2) && ZS == 24);
}
template <int ZS, int KIND = 0>
__device__ __forceinline__ void tier_sync() {
  if constexpr (one_warp_cta<ZS, KIND>()) __syncwarp();
  else __syncthreads();
}

template <class S, class A, int ZS>
struct Layered {
  using Val = typename A::Val;

  static constexpr bool TAB = use_addr_tab<S, A>();
  static constexpr int ME = tab_max_entries<S, ZS, TAB>();

  // tier T: its table entries arrived in ec (fetched during tier T-1); fetch
  // tier T+1's into en, load the late posteriors, update, store, then load
  // tier T+1's early posteriors (early_edge) before the barrier
  template <int T>
  __device__ __forceinline__ static void tier(const SpecArgs& a, const RtK& K, int r, uint32_t b0, uint32_t b1,
                                              uint32_t tab, uint32_t mbase, Val (&msg)[S::NE], Val (&pe)[S::MAXDEG],
                                              Val (&pn)[S::MAXDEG], uint32_t (&ec)[ME], uint32_t (&en)[ME]) {
    constexpr int D = S::DEG[T];
    constexpr int E0 = S::START[T];
    uint32_t addr[D];
    Val p[D], o[D];
    tab_compose<S, A, ZS, TAB, T>(a, r, b0, b1, ec, addr, std::make_integer_sequence<int, D>{});
#pragma unroll
    for (int k = 0; k < D; ++k) p[k] = early_edge<S, T>(k) ? pe[k] : A::lds(addr[k]);
    tab_fetch<S, ZS, TAB, T + 1>(tab, en);
    if constexpr (T < SmemMsg<S>::SMT) {
      constexpr int D4 = SmemMsg<S>::r4(D);
      const uint32_t ma = mbase + (uint32_t)(SmemMsg<S>::off(T) * 4);
      Val m[D4];
#pragma unroll
      for (int q = 0; q < D4 / 4; ++q) {
        const float4 v = lds128f(ma + 16u * q);
        m[4 * q] = v.x; m[4 * q + 1] = v.y; m[4 * q + 2] = v.z; m[4 * q + 3] = v.w;
      }
      A::template row<D, f32_fma_sign<S>()>(p, o, m, K);
#pragma unroll
      for (int q = 0; q < D4 / 4; ++q) sts128f(ma + 16u * q, m[4 * q], m[4 * q + 1], m[4 * q + 2], m[4 * q + 3]);
    } else {
      A::template row<D, f32_fma_sign<S>()>(p, o, msg + E0, K);
    }
#pragma unroll
    for (int k = 0; k < D; ++k) A::sts(addr[k], o[k]);
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
    tier_addrs_tab<S, A, ZS, TAB, E0>(a, r, b0, b1, tab, addr, std::make_integer_sequence<int, D>{});
#if QCB_F32_SIGN_PARITY
    // hard = post <= 0: the sign bit of post - 2^-149 (smallest denormal, IEEE
    // arithmetic) is set exactly for post <= 0 (incl. +-0, -inf), clear for
    // the canonical (positive) NaN; XOR of sign bits = row parity
    const float tiny = __uint_as_float(1u);
    uint32_t par = 0;
#pragma unroll
    for (int k = 0; k < D; ++k) par ^= __float_as_uint(f_sub(A::lds(addr[k]), tiny));
    return par >> 31;
#else
    uint32_t par = 0;
#pragma unroll
    for (int k = 0; k < D; ++k) par ^= A::hard(A::lds(addr[k])) ? 1u : 0u;
    return par;
#endif
  }

  // without early termination every thread runs every tier (threads beyond
  // the batch work on scratch / unused slots): no branch around the tier body
  template <bool ET, int... Ts>
  __device__ __forceinline__ static void sweep(const SpecArgs& a, const RtK& K, int r, uint32_t b0, uint32_t b1,
                                               uint32_t tab, uint32_t mbase, Val (&msg)[S::NE], bool work,
                                               std::integer_sequence<int, Ts...>) {
    Val pa[S::MAXDEG], pb[S::MAXDEG];
    uint32_t ea[ME], eb[ME];
    tab_fetch<S, ZS, TAB, 0>(tab, ea);
    if constexpr (ET) {
      ((work ? tier<Ts>(a, K, r, b0, b1, tab, mbase, msg, (Ts & 1) ? pb : pa, (Ts & 1) ? pa : pb,
                        (Ts & 1) ? eb : ea, (Ts & 1) ? ea : eb)
             : void(),
        tier_sync<ZS>()), ...);
    } else {
      (void)work;
      ((tier<Ts>(a, K, r, b0, b1, tab, mbase, msg, (Ts & 1) ? pb : pa, (Ts & 1) ? pa : pb, (Ts & 1) ? eb : ea,
                 (Ts & 1) ? ea : eb),
        tier_sync<ZS>()), ...);
    }
  }

  template <int... Ts>
  __device__ __forceinline__ static uint32_t parity_all(const SpecArgs& a, int r, uint32_t b0, uint32_t b1,
                                                        uint32_t tab, std::integer_sequence<int, Ts...>) {
    return (parity<Ts>(a, r, b0, b1, tab) | ...);
  }

  // Early-termination syndrome with early exit: the CTA only needs the OR of
  // all row parities, so the tiers are checked in QCB_ET_CHUNKS groups; a
  // thread stops after the first group holding an odd row and publishes it in
  // `flag`, the others stop at their next group once they see the flag.  (A
  // poll per tier serialises the tiers' loads: measured slower at 3 iterations.)
  // Returns 1 if this thread saw an odd row or the flag (the OR is 1 either way).
  static constexpr int kEtChunk = QCB_ET_CHUNKS > 0 ? (S::MB + QCB_ET_CHUNKS - 1) / QCB_ET_CHUNKS : 1;
  // QCB_ET_FIRST > 0: a first group of that many tiers (a cheap reject of a
  // codeword that has not converged: one tier's Z rows almost surely hold an
  // odd row), then all remaining tiers in one group.  Measured (et_perf.py, ET
  // Gb/s at 1.5 / 2.5 / 3.5 dB): two halves f32 78.0 / 142.1 / 194.0, int16
  // 69.0 / 68.0 / 140.2; first = 1 tier 83.5 / 146.6 / 197.6 and 72.3 / 70.7 /
  // 140.5; first = 2 tiers 82.3 / 146.5 / 198.0 and 70.2 / 69.1 / 140.1.
  template <int T0>
  static constexpr int et_len() {
    return QCB_ET_FIRST > 0 ? (T0 == 0 ? QCB_ET_FIRST : S::MB - QCB_ET_FIRST) : kEtChunk;
  }
  template <int T0, int... Is>
  __device__ __forceinline__ static uint32_t parity_group(const SpecArgs& a, int r, uint32_t b0, uint32_t b1,
                                                          uint32_t tab, std::integer_sequence<int, Is...>) {
    return ((T0 + Is < S::MB ? parity<(T0 + Is < S::MB ? T0 + Is : 0)>(a, r, b0, b1, tab) : 0u) | ...);
  }
  // QCB_ET_CHUNKS == 0: per tier, software-pipelined -- tier T+1's loads and
  // the flag poll are issued before tier T's parity is tested, so the early
  // exit does not serialise the loads.
  template <int T>
  __device__ __forceinline__ static void parity_load(const SpecArgs& a, int r, uint32_t b0, uint32_t b1, uint32_t tab,
                                                     Val (&v)[S::DEG[T]]) {
    constexpr int D = S::DEG[T];
    uint32_t addr[D];
    tier_addrs_tab<S, A, ZS, TAB, S::START[T]>(a, r, b0, b1, tab, addr, std::make_integer_sequence<int, D>{});
#pragma unroll
    for (int k = 0; k < D; ++k) v[k] = A::lds(addr[k]);
  }
  template <int T>
  __device__ __forceinline__ static uint32_t parity_pipe(const SpecArgs& a, int r, uint32_t b0, uint32_t b1,
                                                         uint32_t tab, volatile int* flag, const Val (&cur)[S::DEG[T]],
                                                         int f_prev) {
    constexpr int D = S::DEG[T];
    uint32_t par = 0;
    if constexpr (T + 1 < S::MB) {
      Val nxt[S::DEG[T + 1]];
      parity_load<T + 1>(a, r, b0, b1, tab, nxt);
      const int f = *flag;
#pragma unroll
      for (int k = 0; k < D; ++k) par ^= A::hard(cur[k]) ? 1u : 0u;
      if (par) { *flag = 1; return 1u; }
      if (f_prev) return 1u;
      return parity_pipe<T + 1>(a, r, b0, b1, tab, flag, nxt, f);
    } else {
#pragma unroll
      for (int k = 0; k < D; ++k) par ^= A::hard(cur[k]) ? 1u : 0u;
      return par | (f_prev ? 1u : 0u);
    }
  }
  template <int T0>
  __device__ __forceinline__ static uint32_t parity_any(const SpecArgs& a, int r, uint32_t b0, uint32_t b1,
                                                        uint32_t tab, volatile int* flag) {
#if QCB_ET_CHUNKS == 0
    Val v0[S::DEG[0]];
    parity_load<0>(a, r, b0, b1, tab, v0);
    return parity_pipe<0>(a, r, b0, b1, tab, flag, v0, 0);
#endif
    if constexpr (T0 >= S::MB) {
      return 0u;
    } else {
      if (*flag) return 1u;
      if (parity_group<T0>(a, r, b0, b1, tab, std::make_integer_sequence<int, et_len<T0>()>{})) {
        *flag = 1;
        return 1u;
      }
      return parity_any<T0 + et_len<T0>()>(a, r, b0, b1, tab, flag);
    }
  }
};

// CTA shape.  A CTA holds p codewords (p*Z threads, padded to whole warps).
// Measured on B200 (tools/exp/ctasweep.py, 16384 f32 / 65536 int16
// codewords, 10 iterations), coded Gbit/s for p = 1 / 2 / 3 / 4:
//   f32  Wi-Fi 648 R1/2   38.0 / 39.5 / 39.4 / 38.5
//   f32  Wi-Fi 1296 R1/2  46.6 / 44.8 / 39.4 / 27.9
//   f32  Wi-Fi 1944 R1/2  47.8 / 41.4 / 32.3 / 34.0
//   f32  WiMAX 2304 R1/2  71.9 / 60.9 / 40.7 / 47.3
//   i16  Wi-Fi 1296 R1/2  58.8 / 57.0 / 47.1 / 34.7
//   i16  WiMAX 2304 R3/4A 64.5 / 58.2 / 43.0 / 49.6
// i.e. one codeword (pair) per CTA: the per-tier barrier then spans only the
// codeword's own ceil(Z/32) warps, which beats every "more resident rows"
// arrangement of bigger CTAs.  plan_ctas() sizes the register budget.
constexpr int kSmemPerSm = 227 * 1024;
constexpr int plan_ctas(int z, int p, int regs, int cw_smem) {
  const int threads = (p * z + 31) / 32 * 32;
  const int r8 = (regs + 7) / 8 * 8;
  int c = 65536 / (threads * r8);
  const int cw = 64 / (threads / 32);
  if (cw < c) c = cw;
  if (c > 32) c = 32;
  const int cs = kSmemPerSm / ((p + 1) * cw_smem + 1024);   // + scratch slot + static/reserved
  if (cs < c) c = cs;
  return c;
}
constexpr int plan_cw_per_cta(int, int, int, double) { return 1; }

// Register cap: the messages (S::NE) plus a slack for the widest tier's
// transients and hoisted edge addresses; the CTA shape is planned for that
// budget and int16 kernels then take every register that keeps the same
// number of resident CTAs.  Measured on C2 (NE = 76): uncapped 161 regs ->
// 4 CTAs of 96 threads per SM, 45.9 Gb/s; 128 -> 5 CTAs, 50.3; raising
// float32 to 136 at the same CTA count costs 10 % (67.3 vs 75.6 Gb/s), so
// float32 keeps its minimum.
#ifndef QCB_REG_SLACK
#define QCB_REG_SLACK 52
#endif
// Registers are allocated per warp (in 8-register steps per thread) from the
// 16K-register file of the SM sub-partition the warp runs on, so a kernel
// with r registers fits floor(16384 / (32 r)) warps per sub-partition: every
// cap between 129 and 170 gives 3 warps (12 per SM), 103..128 gives 4.  With
// `smsp` the cap is raised to the largest value with the same warp count --
// the same occupancy, fewer spills.  It is not uniformly faster (ptxas then
// schedules differently), so it is a per-structure choice measured with
// tools/exp/regmask_ab.sh (round 1, after the 3-input minima; none -> all
// raised, coded Gb/s): float32 Wi-Fi 648 +4..8 %, 1296 +2..5 %, 1944 R1/2
// +1.5 %, WiMAX 2/3A +1.7 % (Wi-Fi 1944 R2/3 -4 %); int16 Wi-Fi 648 +2..7 %,
// 1296 R3/4, 5/6 +7 / +10 %, WiMAX 1/2, 5/6 +7 / +10 % (Wi-Fi 1944 R5/6 = C3
// -5 %, 1296 R2/3 -4 %); unlisted structures are within +-1 % either way.
#ifndef QCB_REG_SMSP
#define QCB_REG_SMSP 1
#endif
template <class S, class A>
constexpr bool smsp_raise() {
#ifdef QCB_SMSP_F32                               // tuning experiments (both masks)
  constexpr unsigned kF32 = QCB_SMSP_F32, kPair16 = QCB_SMSP_P16;
#else
  constexpr unsigned kF32 = 0xFu | (1u << 4) | (1u << 7) | (0xFu << 8) | (1u << 13) | (1u << 15) | (1u << 17);
  constexpr unsigned kPair16 = (1u << 2) | (1u << 3) | (0xFu << 8) | (1u << 12) | (1u << 17);
#endif
  return QCB_REG_SMSP && ((((A::kKind == 0) ? kF32 : kPair16) >> S::ID) & 1u);
}
constexpr int raise_cap(int z, int want, int cw_smem, bool raise, bool smsp) {
  const int p = plan_cw_per_cta(z, want, cw_smem, -1.0);
  const int threads = (p * z + 31) / 32 * 32;
  const int ctas = plan_ctas(z, p, want, cw_smem);
  int cap = (want + 7) / 8 * 8;
  if (smsp) {
    const int wps = 16384 / (32 * (cap > 255 ? 255 : cap));
    if (wps > 0) {
      const int r = 16384 / (32 * wps) / 8 * 8;
      if (r > cap) cap = r;
    }
  } else if (raise && ctas > 0) {
    const int r = 65536 / (threads * ctas) / 8 * 8;
    if (r > cap) cap = r;
  }
  return cap > 255 ? 255 : cap;
}

template <class S, class A, int ZS>
constexpr int reg_cap() {
  const int want = SmemMsg<S>::in_regs() + QCB_REG_SLACK;
  const int z = ZS > 0 ? ZS : 96;
  const int cap = raise_cap(z, want, cw_block_bytes(z), false, smsp_raise<S, A>());
  // the other direction: 128 registers = 4 warps per sub-partition (5 CTAs of
  // 3 warps instead of 4), paid for with spills.  Measured per structure
  // (tools/exp/cap128_ab.sh, Gb/s): WiMAX 2/3A 75.8 -> 79.3, 3/4A 66.7 -> 69.0,
  // Wi-Fi 1944 R3/4 56.3 -> 57.3; every other float32 code loses up to 6 %.
#ifdef QCB_F32_CAP_MAX                                 // tuning experiments
  constexpr int kMax = QCB_F32_CAP_MAX;
#else
  constexpr int kMax = ((((1u << 6) | (1u << 13) | (1u << 15)) >> S::ID) & 1u) ? 128 : 255;
#endif
#ifdef QCB_F32_SCALED_CAP                              // tuning experiments: scaled Z only
  if constexpr (ZS > 0 && ZS != S::Z0) return cap > QCB_F32_SCALED_CAP ? QCB_F32_SCALED_CAP : cap;
#endif
  // scaled Z: a 128-register cap where the per-code sweep measured it ahead
  // (4 warps per sub-partition, so CTAs of several codewords stay co-resident)
  constexpr int kScaled = (ZS > 0 && ZS != S::Z0 && A::kKind == 0) ? scaled_reg_cap(S::ID, 4, ZS) : 0;
  if constexpr (kScaled > 0) return cap > kScaled ? kScaled : cap;
  return cap > kMax ? kMax : cap;
}

template <class S, class A, int ZS, bool ET>
__global__ void __launch_bounds__(kLayMaxThreads) __maxnreg__((reg_cap<S, A, ZS>()))
    decode_layered_kernel(const __grid_constant__ SpecArgs a) {
  using L = Layered<S, A, ZS>;
  using Val = typename A::Val;
  static_assert(A::kElem == kCellBytes, "4-byte cells");
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int s_fail[kLayMaxCw], s_done[kLayMaxCw], s_iters[kLayMaxCw];
  __shared__ int s_active;
  __shared__ int s_odd;                         // early-exit syndrome flag (G == 1 with ET)

  const RtK K{a.k_one, a.k_sign, a.k_shr, a.k_neg1, a.k_lane1};
  const int Z = ZS > 0 ? ZS : a.z;
  const int N = S::NB * Z;
  const int G = a.pairs;                        // codewords per CTA
  const int tid = threadIdx.x;
  const int g = tid / Z, r = tid - g * Z;
  const int64_t cw0 = (int64_t)blockIdx.x * G;
  const int ncw = (int)(a.w - cw0 < (int64_t)G ? a.w - cw0 : (int64_t)G);
  // bank-offset block stride + chunked rows for the scaled Z only: the native
  // kernels keep compile-time strides (a runtime pad kept live across the sweep
  // loop cost C2 1.6 % at the 128-register cap)
  constexpr bool kPad = ZS != S::Z0;
  const uint32_t cws = kPad ? (uint32_t)blk_stride_bytes(Z, G, false) : (uint32_t)cw_block_bytes(Z);
  const uint32_t cpad = kPad ? cws - (uint32_t)cw_block_bytes(Z) : 0u;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
  dbg_check(cw0 < a.w && ncw >= 1 && ncw <= G, 21);           // the CTA's chunk lies inside the batch
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
  const bool act = gs < ncw;
  // opaque copies keep the row bases in registers (no per-tier rematerialisation)
  uint32_t b0 = sbase + (uint32_t)gs * cws + (uint32_t)(rs * kCellBytes), b1;
  asm volatile("mov.b32 %0, %0;" : "+r"(b0));
  asm volatile("sub.u32 %0, %1, %2;" : "=r"(b1) : "r"(b0), "r"((uint32_t)(Z * kCellBytes)));   // c = r + e - Z
  // this thread's address table (after the G posterior blocks)
  const uint32_t tab = sbase + (uint32_t)G * cws + (uint32_t)(tid * addr_tab_bytes_per_thread<S, ZS, L::TAB>());
  fill_addr_tab<S, A, ZS, L::TAB>(a, rs, b0, b1, tab, std::make_integer_sequence<int, S::NE>{});
  // this thread's shared-memory message slots (first SMT tiers), after the tables
  const uint32_t mbase = ((sbase + (uint32_t)G * cws + blockDim.x * (uint32_t)addr_tab_bytes_per_thread<S, ZS, L::TAB>()
                           + 15u) & ~15u) + (uint32_t)(tid * SmemMsg<S>::words() * 4);
#pragma unroll
  for (int q = 0; q < SmemMsg<S>::words() / 4; ++q) sts128f(mbase + 16u * q, 0.0f, 0.0f, 0.0f, 0.0f);

  // ---- channel LLRs -> the codewords' blocks (bit order) ----------------------
  // Programmatic dependent launch (launch_layered_fixed): nothing above touches
  // global memory; wait here for the previous kernel of the stream, and let the
  // next one start its own setup (a no-op pair for an ordinary launch).
  asm volatile("griddepcontrol.wait;" ::: "memory");
  {
    if (kPad && cpad) load_llrs_f32<io_cells8<ZS>(), true>(reinterpret_cast<const float*>(a.llr) + cw0 * N, ncw, N, sbase, cpad);
    else load_llrs_f32<io_cells8<ZS>()>(reinterpret_cast<const float*>(a.llr) + cw0 * N, ncw, N, sbase);
    for (int q = tid; q < kLayMaxCw; q += blockDim.x) {
      s_fail[q] = 1; s_done[q] = q >= ncw; s_iters[q] = 0;
    }
    if (tid == 0) s_odd = 0;
  }
  __syncthreads();

  Val msg[S::NE];
#pragma unroll
  for (int e = 0; e < S::NE; ++e) msg[e] = A::zero();

  const auto tiers = std::make_integer_sequence<int, S::MB>{};
  if constexpr (!ET) {
    // fixed iterations: every codeword runs max_iters sweeps; one syndrome at the end
    for (int k = 0; k < a.max_iters; ++k) L::template sweep<false>(a, K, rs, b0, b1, tab, mbase, msg, act, tiers);
    if (a.max_iters > 0) {
      if (tid < kLayMaxCw) s_fail[tid] = 0;
      __syncthreads();
      if (act && L::parity_all(a, rs, b0, b1, tab, tiers)) s_fail[gs] = 1;
      __syncthreads();
    }
    if (tid < ncw) s_iters[tid] = a.max_iters;
  } else if (G == 1) {
    // one codeword per CTA: full sweeps, then the syndrome (_kernels.py:85-96)
    // reduced with a single __syncthreads_or; stop at the first zero syndrome
    // (the reference's break), iterations = sweeps done
    int k = 0;
    int fail = 1;
    while (k < a.max_iters) {
      L::template sweep<false>(a, K, rs, b0, b1, tab, mbase, msg, act, tiers);
      ++k;
#if QCB_ET_EARLY_EXIT
      fail = __syncthreads_or(act && L::template parity_any<0>(a, rs, b0, b1, tab, &s_odd));
      if (tid == 0) s_odd = 0;                  // read again only after the next sweep's barriers
#else
      fail = __syncthreads_or(act && L::parity_all(a, rs, b0, b1, tab, tiers));
#endif
      if (!fail) break;
    }
    if (tid == 0) {
      s_iters[0] = k;
      s_fail[0] = fail;
    }
  } else {
    for (int k = 0; k < a.max_iters; ++k) {
      const bool work = act && !s_done[gs];
      L::template sweep<true>(a, K, rs, b0, b1, tab, mbase, msg, work, tiers);
      if (tid < kLayMaxCw) s_fail[tid] = 0;     // syndrome (_kernels.py:85-96)
      __syncthreads();
      if (work && L::parity_all(a, rs, b0, b1, tab, tiers)) s_fail[gs] = 1;
      if (tid == 0) s_active = 0;
      __syncthreads();
      if (tid < ncw && !s_done[tid]) {
        s_iters[tid] = k + 1;
        if (!s_fail[tid]) s_done[tid] = 1;      // converged: frozen from now on
        else s_active = 1;
      }
      __syncthreads();
      if (!s_active) break;
    }
  }

  // ---- outputs: iterations, converged, hard decisions, posteriors -------------
  // (the next launch of the stream may begin its setup while this grid stores its outputs)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (tid < ncw) {
    a.iters[cw0 + tid] = s_iters[tid];
    a.conv[cw0 + tid] = (a.max_iters > 0 && !s_fail[tid]) ? 1 : 0;
  }
  uint8_t* hard = reinterpret_cast<uint8_t*>(a.hard) + cw0 * (a.hard_packed ? (N + 7) >> 3 : N);
  float* post = a.post ? reinterpret_cast<float*>(a.post) + cw0 * N : nullptr;
  const auto is_hard = [](uint32_t v) { return __uint_as_float(v) <= 0.0f; };
  const auto post_bits = [](uint32_t v) { return __uint_as_float(v); };
  if (kPad && cpad) store_outputs_cell32<io_cells8<ZS>(), true>(hard, a.hard_packed, post, ncw, N, sbase, is_hard, post_bits, cpad);
  else store_outputs_cell32<io_cells8<ZS>()>(hard, a.hard_packed, post, ncw, N, sbase, is_hard, post_bits);
}

// codewords per CTA for a kernel with `regs` registers per thread
// Codewords (int16 kernel: codeword pairs) per CTA where Z leaves lanes of the
// last warp idle (the scaled WiMAX codes): G codewords' rows are dealt out
// contiguously over ceil(G Z / 32) warps, so a G with G Z near a multiple of
// 32 busies more lanes, at the price of a tier barrier over more warps.
// Measured per scaled code for G = 1, 2, 3, 4, 8 (scaled_plan_gen.h): G = 2
// or 4 where the chunked mapping applies (Z = 24, 40, 48, 80: conflict-free,
// no idle lanes; float32 WiMAX 960 R2/3B 55.0 -> 68.2, 1152 R3/4A 54.7 -> 67.8
// Gb/s), G = 3 at Z = 36 and on the lower-degree structures at Z = 68-84;
// full or nearly full Z keep G = 1.
inline const ScaledPlan* scaled_plan(int structure_id, int elem, int z) {
  for (int i = 0; i < kScaledPlans; ++i)
    if (kScaledPlan[i].id == structure_id && kScaledPlan[i].elem == elem && kScaledPlan[i].z == z) return &kScaledPlan[i];
  return nullptr;
}
// The native Z = 81 int16 codes: three pairs (243 rows) in eight warps busy 95 %
// of the lanes where one pair keeps 81 of 96: Wi-Fi 1944 R1/2 96.0 -> 102.3,
// R2/3 88.9 -> 93.2 Gb/s (without TMEM tiers), R3/4 89.1 -> 93.1 and R5/6 (C3)
// 96.1 -> 102.4 (TMEM tiers, one column group per four warps; fixed iterations
// only) (round 2, tools/exp/r02_call10.sh, r02_call12.sh).  WiMAX (Z = 96, no
// idle lanes) loses 9-32 % with G > 1, float32 loses everywhere.
inline int native_fill_cw(int kind, int structure_id) {
  return (kind == 2 && structure_id >= 4 && structure_id <= 7) ? 3 : 1;
}
inline int lane_fill_cw(int z, int kind, int structure_id) {
  const ScaledPlan* p = scaled_plan(structure_id, kind == 2 ? 2 : 4, z);
  return p ? p->g : 1;
}

inline int layered_cw_per_cta(int z, int64_t w, int regs, int cell_bytes, int fill = 1) {
  static const int env_v = [] {                        // tuning knob (benchmarks only)
    const char* env = getenv("QCB_CW_PER_CTA");
    return env ? atoi(env) : 0;
  }();
  if (env_v >= 1 && env_v <= kLayMaxCw && env_v * z <= kLayMaxThreads) return env_v;
  if (fill > 1 && fill * z <= kLayMaxThreads && w >= (int64_t)fill * 148 * 4) return fill;
  const int sms = device_sm_count();
  (void)cell_bytes;
  const int cw_smem = cw_block_bytes(z);
  return plan_cw_per_cta(z, regs, cw_smem, (double)w / sms);
}

template <class K>
inline cudaError_t launch_layered_fixed(K kern, const SpecArgs& a, int z, cudaStream_t s, int tab_bytes = 0,
                                        int msg_bytes = 0, int blk_bytes = 0, bool kernel_waits = false) {
  const int threads = (a.pairs * z + 31) / 32 * 32;
  const size_t blk = blk_bytes > 0 ? (size_t)blk_bytes : (size_t)cw_block_bytes(z);
  const size_t smem = (((size_t)a.pairs * blk + (size_t)threads * tab_bytes + 15) & ~(size_t)15) +
                      (size_t)threads * msg_bytes;
  cudaError_t e = ensure_dyn_smem((const void*)kern, smem);
  if (e != cudaSuccess) return e;
  const int64_t blocks = (a.w + a.pairs - 1) / a.pairs;
  if (blocks <= 0) return cudaSuccess;
  // Small batches (a grid of at most a few CTAs per SM, BASELINE C1) are launched
  // with programmatic stream serialization: the grid may start while the previous
  // kernel of the stream drains, runs its address setup, and blocks at
  // griddepcontrol.wait (before its first global access) until that kernel has
  // completed and flushed -- stream order as the caller sees it is unchanged.
  // C1 (1024 codewords, back-to-back launches): QCB_PDL=0/1, see DESIGN 3.1.
  static const bool pdl = [] {
    const char* e = getenv("QCB_PDL");
    return !(e && e[0] == '0');
  }();
  // (kernel_waits: only kernels that execute griddepcontrol.wait may be launched this way)
  if (pdl && kernel_waits && blocks <= (int64_t)device_sm_count() * 16) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)blocks);
    cfg.blockDim = dim3((unsigned)threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, a);
  }
  kern<<<(unsigned)blocks, threads, smem, s>>>(a);
  return cudaGetLastError();
}

template <class S, class A, int ZS, bool ET>
inline cudaError_t launch_layered(const SpecArgs& a, cudaStream_t s) {
  const int z = ZS > 0 ? ZS : a.z;
  auto kern = decode_layered_kernel<S, A, ZS, ET>;
  // the CTA shape is planned from the register count ptxas actually gave
  // this kernel (the decode result does not depend on the CTA size)
  cudaFuncAttributes fa;
  cudaError_t e = kernel_attributes((const void*)kern, &fa);
  if (e != cudaSuccess) return e;
  SpecArgs b = a;
  b.pairs = layered_cw_per_cta(z, a.w, fa.numRegs, A::kElem, ZS == S::Z0 ? 1 : lane_fill_cw(z, A::kKind, S::ID));
  if constexpr (one_warp_cta<ZS>()) b.pairs = 1;            // tier_sync is a warp barrier
  while (b.pairs > 1 && (b.pairs * z + 31) / 32 * 32 > fa.maxThreadsPerBlock) --b.pairs;
  if ((b.pairs * z + 31) / 32 * 32 > fa.maxThreadsPerBlock) return cudaErrorLaunchOutOfResources;
  return launch_layered_fixed(kern, b, z, s, addr_tab_bytes_per_thread<S, ZS, use_addr_tab<S, A>()>(),
                              SmemMsg<S>::words() * 4,
                              ZS != S::Z0 ? blk_stride_bytes(z, b.pairs, false) : cw_block_bytes(z), true);
}

}  // namespace qcb
