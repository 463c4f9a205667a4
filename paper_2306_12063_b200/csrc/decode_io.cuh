// decode_io.cuh -- prologue / epilogue of the layered decoders: channel LLRs
// HBM -> shared-memory cells, and cells -> hard decisions / posteriors in HBM.
//
// Shared-memory layout (common.cuh): cell (c, j) = bit n = j Z + c of a
// codeword sits at byte 4 n of the codeword's block, and a CTA's blocks are
// contiguous, exactly like the CTA's chunk of the (W, N) LLR block in HBM.
// The prologue is therefore a streaming copy (16-byte global loads, 16-byte
// shared stores at consecutive addresses: conflict-free) and the epilogue
// reads 16-byte groups of consecutive cells.  (The previous [c][j] layout
// with a 25-cell row stride made the same loops 4- to 8-way bank-conflicted:
// ncu, C3: 7.9x the ideal shared-memory wavefronts in prologue and epilogue,
// 13 % of the kernel's warp samples.)
//
// Cell formats: Cell32 = one float32 per cell; Pair16 = the int16 posteriors
// of codewords 2q (low lane) and 2q+1 (high lane) in one 32-bit cell.
#pragma once
#include "common.cuh"

namespace qcb {

// units in flight per thread; measured (C5 / C3 / C2 Gb/s): 2: 80.1 / 84.4 /
// 88.0, 4: 82.6 / 84.9 / 88.4, 8: 81.1 / 81.4 / 88.3
#ifndef QCB_IO_UNROLL
#define QCB_IO_UNROLL 4
#endif
constexpr int kIoUnroll = QCB_IO_UNROLL;
// float32 I/O unit: 8 cells (two 16-byte groups, swizzled) or 4 cells (one
// group).  Measured (C2 / C1 / C4 Gb/s): 4 + 4: 85.3 / 29.6 / 61.4;
// 8 + 8: 84.7 / 30.6 / 62.0 -- so the kernels pick 8-cell units for the
// Wi-Fi sizes (Z not a multiple of 32) and 4-cell units for WiMAX.
template <int ZS>
constexpr bool io_cells8() { return ZS > 0 && ZS % 32 != 0; }

__device__ __forceinline__ void sts32(uint32_t a, uint32_t v) {
  dbg_smem(a, 4, 1);
  asm volatile("st.shared.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  dbg_smem(a, 4, 2);
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts128(uint32_t a, uint4 v) {
  dbg_smem(a, 16, 3);
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  dbg_smem(a, 16, 4);
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
// cells 8u .. 8u+7 (two 16-byte groups).  A quarter-warp's eight lanes read
// groups 2u (+1) at a 32-byte stride, i.e. only four distinct bank quads: the
// lanes with bit 2 of u set read their second group first, which makes both
// loads conflict-free; the groups are swapped back in registers.
__device__ __forceinline__ void lds_cells8(uint32_t blk, int u, uint32_t (&v)[8]) {
  const int f = (u >> 2) & 1;
  const uint4 a = lds128(blk + (uint32_t)(32 * u + 16 * f));
  const uint4 b = lds128(blk + (uint32_t)(32 * u + 16 * (1 - f)));
  const uint4 lo = f ? b : a, hi = f ? a : b;
  v[0] = lo.x; v[1] = lo.y; v[2] = lo.z; v[3] = lo.w;
  v[4] = hi.x; v[5] = hi.y; v[6] = hi.z; v[7] = hi.w;
}

__device__ __forceinline__ void sts_cells8(uint32_t blk, int u, const uint4& lo, const uint4& hi) {
  const int f = (u >> 2) & 1;                   // the quarter-warp swizzle of lds_cells8
  sts128(blk + (uint32_t)(32 * u + 16 * f), f ? hi : lo);
  sts128(blk + (uint32_t)(32 * u + 16 * (1 - f)), f ? lo : hi);
}

// ---- float32: one codeword per 4-byte cell ----------------------------------------
// LLRs are canonicalised on the way in (v + 0.0f, see ArithF32::canon).
// The CTA's ncw codewords (ncw * n floats) land at sbase + 4 e.
// cpad: bytes of padding after each codeword's block (blk_stride_bytes)
template <bool IO8, bool PAD = false>
__device__ __forceinline__ void load_llrs_f32(const float* chunk, int ncw, int n, uint32_t sbase, uint32_t cpad = 0) {
  const int total = ncw * n;
  const int tid = threadIdx.x, nthr = blockDim.x;
  if ((reinterpret_cast<uintptr_t>(chunk) & 15) == 0) {
    const float4* src = reinterpret_cast<const float4*>(chunk);
    if constexpr (!IO8) {
      const int total4 = total / 4;
      for (int base = 0; base < total4; base += kIoUnroll * nthr) {
        float4 v[kIoUnroll];
#pragma unroll
        for (int u = 0; u < kIoUnroll; ++u) {
          const int i = base + u * nthr + tid;
          if (i < total4) v[u] = __ldcs(src + i);
        }
#pragma unroll
        for (int u = 0; u < kIoUnroll; ++u) {
          const int i = base + u * nthr + tid;
          if (i < total4)
            sts128(sbase + 16u * (uint32_t)i + (PAD ? (uint32_t)((4 * i) / n) * cpad : 0u),
                   make_uint4(__float_as_uint(__fadd_rn(v[u].x, 0.0f)), __float_as_uint(__fadd_rn(v[u].y, 0.0f)),
                              __float_as_uint(__fadd_rn(v[u].z, 0.0f)), __float_as_uint(__fadd_rn(v[u].w, 0.0f))));
        }
      }
      return;
    }
    const int units = total / 8;                  // n is a multiple of 8 (N = 24 Z)
    for (int base = 0; base < units; base += kIoUnroll * nthr) {
      float4 v[kIoUnroll], w[kIoUnroll];
#pragma unroll
      for (int u = 0; u < kIoUnroll; ++u) {
        const int i = base + u * nthr + tid;
        if (i < units) { v[u] = __ldcs(src + 2 * i); w[u] = __ldcs(src + 2 * i + 1); }
      }
#pragma unroll
      for (int u = 0; u < kIoUnroll; ++u) {
        const int i = base + u * nthr + tid;
        if (i < units)
          sts_cells8(sbase + (PAD ? (uint32_t)((8 * i) / n) * cpad : 0u), i,
                     make_uint4(__float_as_uint(__fadd_rn(v[u].x, 0.0f)), __float_as_uint(__fadd_rn(v[u].y, 0.0f)),
                                __float_as_uint(__fadd_rn(v[u].z, 0.0f)), __float_as_uint(__fadd_rn(v[u].w, 0.0f))),
                     make_uint4(__float_as_uint(__fadd_rn(w[u].x, 0.0f)), __float_as_uint(__fadd_rn(w[u].y, 0.0f)),
                                __float_as_uint(__fadd_rn(w[u].z, 0.0f)), __float_as_uint(__fadd_rn(w[u].w, 0.0f))));
      }
    }
  } else {
    for (int e = tid; e < total; e += nthr)
      sts32(sbase + 4u * (uint32_t)e + (PAD ? (uint32_t)(e / n) * cpad : 0u),
            __float_as_uint(__fadd_rn(__ldcs(chunk + e), 0.0f)));
  }
}

// hard decisions (post <= 0) of ncw codewords: unpacked (n bytes each) or
// packed (np.packbits, MSB first); optional float32 posteriors
template <bool IO8, bool PAD = false, class HardFn, class PostFn>
__device__ __forceinline__ void store_outputs_cell32(uint8_t* hard, int packed, float* post, int ncw, int n,
                                                     uint32_t sbase, HardFn is_hard, PostFn post_bits,
                                                     uint32_t cpad = 0) {
  const int tid = threadIdx.x, nthr = blockDim.x;
  const bool al = ((reinterpret_cast<uintptr_t>(hard) | reinterpret_cast<uintptr_t>(post)) & 15) == 0;
  if (!IO8 && !packed) {                                 // 4 consecutive cells per unit
    const int units4 = ncw * n / 4;
    for (int base = 0; base < units4; base += kIoUnroll * nthr) {
#pragma unroll
      for (int k = 0; k < kIoUnroll; ++k) {
        const int u = base + k * nthr + tid;
        if (u >= units4) continue;
        const uint4 c = lds128(sbase + 16u * (uint32_t)u + (PAD ? (uint32_t)((4 * u) / n) * cpad : 0u));
        const uint32_t v[4] = {c.x, c.y, c.z, c.w};
        uint32_t word = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) word |= (is_hard(v[i]) ? 1u : 0u) << (8 * i);
        uint8_t* hd = hard + 4 * (int64_t)u;
        if (al) *reinterpret_cast<uint32_t*>(hd) = word;
        else for (int i = 0; i < 4; ++i) hd[i] = (uint8_t)((word >> (8 * i)) & 1u);
        if (post) {
          float* dst = post + 4 * (int64_t)u;
          const float4 f = make_float4(post_bits(v[0]), post_bits(v[1]), post_bits(v[2]), post_bits(v[3]));
          if (al) *reinterpret_cast<float4*>(dst) = f;
          else { dst[0] = f.x; dst[1] = f.y; dst[2] = f.z; dst[3] = f.w; }
        }
      }
    }
    return;
  }
  const int units = ncw * n / 8;                 // 8 consecutive bits of one codeword (n % 8 == 0)
  for (int base = 0; base < units; base += kIoUnroll * nthr) {
#pragma unroll
    for (int k = 0; k < kIoUnroll; ++k) {
      const int u = base + k * nthr + tid;
      if (u >= units) continue;
      uint32_t v[8];
      lds_cells8(sbase + (PAD ? (uint32_t)((8 * u) / n) * cpad : 0u), u, v);
      const int e = 8 * u;
      if (packed) {
        uint32_t byte = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) byte = (byte << 1) | (is_hard(v[i]) ? 1u : 0u);
        const int q = e / n;
        hard[(int64_t)q * ((n + 7) >> 3) + ((e - q * n) >> 3)] = (uint8_t)byte;
      } else {
        uint32_t lo = 0, hi = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          lo |= (is_hard(v[i]) ? 1u : 0u) << (8 * i);
          hi |= (is_hard(v[i + 4]) ? 1u : 0u) << (8 * i);
        }
        uint8_t* hd = hard + (int64_t)e;
        if (al) *reinterpret_cast<uint2*>(hd) = make_uint2(lo, hi);
        else for (int i = 0; i < 8; ++i) hd[i] = (uint8_t)(((i < 4 ? lo : hi) >> (8 * (i & 3))) & 1u);
      }
      if (post) {
        float* dst = post + (int64_t)e;
        if (al) {
          reinterpret_cast<float4*>(dst)[0] = make_float4(post_bits(v[0]), post_bits(v[1]), post_bits(v[2]), post_bits(v[3]));
          reinterpret_cast<float4*>(dst)[1] = make_float4(post_bits(v[4]), post_bits(v[5]), post_bits(v[6]), post_bits(v[7]));
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) dst[i] = post_bits(v[i]);
        }
      }
    }
  }
}

// ---- int16 pairs: codewords 2q / 2q+1 in the low / high lane of one cell -------------
// pair q's block (n cells) at sbase + 4 q n.  Units of eight cells: two
// 16-byte loads per codeword keep as many bytes in flight as the float32 path
// (units of four halved them and cost C5 1.3 %), stored with sts_cells8.
// cpad: bytes of padding after each pair's block (several pairs per CTA, p16_block_stride)
template <bool PAD = false>
__device__ __forceinline__ void load_llrs_pair16(const int16_t* chunk, int ncw, int n, uint32_t sbase,
                                                 uint32_t cpad = 0) {
  const int npairs = (ncw + 1) >> 1;
  const int units = npairs * n / 8;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const bool al16 = (reinterpret_cast<uintptr_t>(chunk) & 15) == 0;   // rows are 2 n = 48 Z bytes
  for (int base = 0; base < units; base += kIoUnroll * nthr) {
    uint4 x[kIoUnroll], y[kIoUnroll];
#pragma unroll
    for (int k = 0; k < kIoUnroll; ++k) {
      const int u = base + k * nthr + tid;
      if (u >= units) continue;
      const int e = 8 * u, q = e / n, nn = e - q * n;
      const int16_t* a = chunk + (int64_t)(2 * q) * n + nn;
      const bool hasb = 2 * q + 1 < ncw;
      if (al16) {
        x[k] = __ldcs(reinterpret_cast<const uint4*>(a));
        y[k] = hasb ? __ldcs(reinterpret_cast<const uint4*>(a + n)) : make_uint4(0, 0, 0, 0);
      } else {
        uint32_t w[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) w[i] = (uint16_t)a[i] | ((hasb ? (uint32_t)(uint16_t)a[n + i] : 0u) << 16);
        x[k] = make_uint4(w[0], w[1], w[2], w[3]);   // already paired: (a_i | b_i << 16)
        y[k] = make_uint4(w[4], w[5], w[6], w[7]);
      }
    }
#pragma unroll
    for (int k = 0; k < kIoUnroll; ++k) {
      const int u = base + k * nthr + tid;
      if (u >= units) continue;
      if (al16) {
        const uint4 lo = make_uint4(__byte_perm(x[k].x, y[k].x, 0x5410), __byte_perm(x[k].x, y[k].x, 0x7632),
                                    __byte_perm(x[k].y, y[k].y, 0x5410), __byte_perm(x[k].y, y[k].y, 0x7632));
        const uint4 hi = make_uint4(__byte_perm(x[k].z, y[k].z, 0x5410), __byte_perm(x[k].z, y[k].z, 0x7632),
                                    __byte_perm(x[k].w, y[k].w, 0x5410), __byte_perm(x[k].w, y[k].w, 0x7632));
        sts_cells8(sbase + (PAD ? (uint32_t)((8 * u) / n) * cpad : 0u), u, lo, hi);
      } else {
        sts_cells8(sbase + (PAD ? (uint32_t)((8 * u) / n) * cpad : 0u), u, x[k], y[k]);
      }
    }
  }
}

template <bool PAD = false>
__device__ __forceinline__ void store_outputs_pair16(uint8_t* hard, int packed, int16_t* post, int ncw, int n,
                                                     uint32_t sbase, uint32_t cpad = 0) {
  const int npairs = (ncw + 1) >> 1;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const bool al = ((reinterpret_cast<uintptr_t>(hard) | reinterpret_cast<uintptr_t>(post)) & 15) == 0;
  const int nbytes = (n + 7) >> 3;
  if (packed) {
    const int units = npairs * n / 8;
    for (int base = 0; base < units; base += kIoUnroll * nthr) {
#pragma unroll
      for (int k = 0; k < kIoUnroll; ++k) {
        const int u = base + k * nthr + tid;
        if (u >= units) continue;
        uint32_t v[8];
        const int e = 8 * u, q = e / n, nn = e - q * n;
        lds_cells8(sbase + (PAD ? (uint32_t)q * cpad : 0u), u, v);
#pragma unroll
        for (int lane = 0; lane < 2; ++lane) {
          const int cw = 2 * q + lane;
          if (cw >= ncw) break;
          uint32_t byte = 0;
#pragma unroll
          for (int i = 0; i < 8; ++i) byte = (byte << 1) | (((lane ? (int)v[i] >> 16 : sext16((int)v[i])) <= 0) ? 1u : 0u);
          hard[(int64_t)cw * nbytes + (nn >> 3)] = (uint8_t)byte;
          if (post) {
            int16_t* dst = post + (int64_t)cw * n + nn;
            uint32_t w[4];
#pragma unroll
            for (int i = 0; i < 4; ++i)
              w[i] = lane ? __byte_perm(v[2 * i], v[2 * i + 1], 0x7632) : __byte_perm(v[2 * i], v[2 * i + 1], 0x5410);
            if (al) *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
            else for (int i = 0; i < 8; ++i) dst[i] = (int16_t)(w[i >> 1] >> (16 * (i & 1)));
          }
        }
      }
    }
    return;
  }
  const int units = npairs * n / 4;
  for (int base = 0; base < units; base += kIoUnroll * nthr) {
#pragma unroll
    for (int k = 0; k < kIoUnroll; ++k) {
      const int u = base + k * nthr + tid;
      if (u >= units) continue;
      const int e = 4 * u, q = e / n, nn = e - q * n;
      const uint4 c = lds128(sbase + 16u * (uint32_t)u + (PAD ? (uint32_t)q * cpad : 0u));
      const uint32_t v[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
      for (int lane = 0; lane < 2; ++lane) {
        const int cw = 2 * q + lane;
        if (cw >= ncw) break;
        uint32_t word = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i)
          word |= (((lane ? (int)v[i] >> 16 : sext16((int)v[i])) <= 0) ? 1u : 0u) << (8 * i);
        uint8_t* hd = hard + (int64_t)cw * n + nn;
        if (al) *reinterpret_cast<uint32_t*>(hd) = word;
        else for (int i = 0; i < 4; ++i) hd[i] = (uint8_t)((word >> (8 * i)) & 1u);
        if (post) {
          int16_t* dst = post + (int64_t)cw * n + nn;
          const uint32_t w0 = lane ? __byte_perm(v[0], v[1], 0x7632) : __byte_perm(v[0], v[1], 0x5410);
          const uint32_t w1 = lane ? __byte_perm(v[2], v[3], 0x7632) : __byte_perm(v[2], v[3], 0x5410);
          if (al) *reinterpret_cast<uint2*>(dst) = make_uint2(w0, w1);
          else for (int i = 0; i < 4; ++i) dst[i] = (int16_t)((i < 2 ? w0 : w1) >> (16 * (i & 1)));
        }
      }
    }
  }
}

}  // namespace qcb
