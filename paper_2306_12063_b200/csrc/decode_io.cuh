// decode_io.cuh -- prologue / epilogue of the layered decoders: channel LLRs
// HBM -> shared-memory cells, and cells -> hard decisions / posteriors in HBM.
//
// The CTA's codewords are one contiguous chunk of the (W, N) LLR block, so
// the chunk is streamed with 16-byte loads (8 int16 or 4 float32 per load),
// several loads in flight per thread before any is consumed; outputs leave in
// 8-byte units (8 hard-decision bytes or 8 consecutive bits' posteriors).
// N = 24 Z is a multiple of 8 for every code, so an 8-element unit never
// straddles two codewords.  Measured motivation (ncu source view, C2 before
// this change): the element-at-a-time load loop held 13 % of the kernel's
// warp samples and the byte-wise hard-decision loop 10 %, both latency-bound.
//
// Cell formats: Cell32 = one float32 per cell; Pair16 = the int16 posteriors
// of codewords 2q (low lane) and 2q+1 (high lane) in one 32-bit cell.
#pragma once
#include "common.cuh"

namespace qcb {

constexpr int kIoUnroll = 4;

// (j, c) of element n of a codeword, advanced by one element
struct CellPos {
  int j, c;
  __device__ __forceinline__ void next(int z) { if (++c == z) { c = 0; ++j; } }
};
__device__ __forceinline__ CellPos cell_pos(int n, int z) {
  const int j = n / z;
  return CellPos{j, n - j * z};
}
__device__ __forceinline__ uint32_t cell_addr(uint32_t blk, const CellPos& p, int rs) {
  return blk + (uint32_t)(p.c * rs + p.j * 4);
}
__device__ __forceinline__ void sts32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}

// ---- float32: one codeword per 4-byte cell ----------------------------------------
// LLRs are canonicalised on the way in (v + 0.0f, see ArithF32::canon)
__device__ __forceinline__ void load_llrs_f32(const float* chunk, int ncw, int n, int z, uint32_t sbase,
                                              uint32_t cws, int rs) {
  const int total4 = ncw * n / 4;
  const int tid = threadIdx.x, nthr = blockDim.x;
  if ((reinterpret_cast<uintptr_t>(chunk) & 15) == 0) {
    const float4* src = reinterpret_cast<const float4*>(chunk);
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
        if (i < total4) {
          const int e = 4 * i, q = e / n;
          CellPos p = cell_pos(e - q * n, z);
          const uint32_t blk = sbase + (uint32_t)q * cws;
          const float f[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            sts32(cell_addr(blk, p, rs), __float_as_uint(__fadd_rn(f[k], 0.0f)));
            p.next(z);
          }
        }
      }
    }
  } else {
    for (int e = tid; e < ncw * n; e += nthr) {
      const int q = e / n;
      const CellPos p = cell_pos(e - q * n, z);
      sts32(cell_addr(sbase + (uint32_t)q * cws, p, rs), __float_as_uint(__fadd_rn(__ldcs(chunk + e), 0.0f)));
    }
  }
}

// hard decisions (post <= 0) of ncw codewords: unpacked (n bytes each) or packed
template <class HardFn, class PostFn>
__device__ __forceinline__ void store_outputs_cell32(uint8_t* hard, int packed, float* post, int ncw, int n, int z,
                                                     uint32_t sbase, uint32_t cws, int rs, HardFn is_hard,
                                                     PostFn post_bits) {
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int units = ncw * n / 8;                 // 8 consecutive bits of one codeword
  const bool al8 = ((reinterpret_cast<uintptr_t>(hard) | reinterpret_cast<uintptr_t>(post)) & 15) == 0;
  for (int base = 0; base < units; base += kIoUnroll * nthr) {
#pragma unroll
    for (int u = 0; u < kIoUnroll; ++u) {
      const int i = base + u * nthr + tid;
      if (i >= units) continue;
      const int e = 8 * i, q = e / n, nn = e - q * n;
      CellPos p = cell_pos(nn, z);
      const uint32_t blk = sbase + (uint32_t)q * cws;
      uint32_t v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        v[k] = lds32(cell_addr(blk, p, rs));
        p.next(z);
      }
      if (packed) {
        uint32_t byte = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) byte = (byte << 1) | (is_hard(v[k]) ? 1u : 0u);
        hard[(int64_t)q * ((n + 7) >> 3) + (nn >> 3)] = (uint8_t)byte;
      } else {
        uint32_t lo = 0, hi = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          lo |= (is_hard(v[k]) ? 1u : 0u) << (8 * k);
          hi |= (is_hard(v[k + 4]) ? 1u : 0u) << (8 * k);
        }
        uint8_t* dst = hard + (int64_t)e;
        if (al8) *reinterpret_cast<uint2*>(dst) = make_uint2(lo, hi);
        else for (int k = 0; k < 8; ++k) dst[k] = (uint8_t)(((k < 4 ? lo : hi) >> (8 * (k & 3))) & 1u);
      }
      if (post) {
        float* dst = post + (int64_t)e;
        if (al8) {
          reinterpret_cast<float4*>(dst)[0] = make_float4(post_bits(v[0]), post_bits(v[1]), post_bits(v[2]), post_bits(v[3]));
          reinterpret_cast<float4*>(dst)[1] = make_float4(post_bits(v[4]), post_bits(v[5]), post_bits(v[6]), post_bits(v[7]));
        } else {
#pragma unroll
          for (int k = 0; k < 8; ++k) dst[k] = post_bits(v[k]);
        }
      }
    }
  }
}

// ---- int16 pairs: codewords 2q / 2q+1 in the low / high lane of one cell -------------
__device__ __forceinline__ void load_llrs_pair16(const int16_t* chunk, int ncw, int n, int z, uint32_t sbase,
                                                 uint32_t cws, int rs) {
  const int npairs = (ncw + 1) >> 1;
  const int units = npairs * n / 8;              // 8 consecutive bits of one pair
  const int tid = threadIdx.x, nthr = blockDim.x;
  const bool al16 = (reinterpret_cast<uintptr_t>(chunk) & 15) == 0;
  for (int base = 0; base < units; base += kIoUnroll * nthr) {
    uint4 x[kIoUnroll], y[kIoUnroll];
#pragma unroll
    for (int u = 0; u < kIoUnroll; ++u) {
      const int i = base + u * nthr + tid;
      if (i >= units) continue;
      const int e = 8 * i, q = e / n, nn = e - q * n;
      const int16_t* a = chunk + (int64_t)(2 * q) * n + nn;
      const bool hasb = 2 * q + 1 < ncw;
      if (al16) {
        x[u] = __ldcs(reinterpret_cast<const uint4*>(a));
        y[u] = hasb ? __ldcs(reinterpret_cast<const uint4*>(a + n)) : make_uint4(0, 0, 0, 0);
      } else {
        uint32_t w[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) w[k] = (uint16_t)a[k] | ((hasb ? (uint32_t)(uint16_t)a[n + k] : 0u) << 16);
        x[u] = make_uint4(w[0], w[1], w[2], w[3]);   // already paired: (a_k | b_k << 16)
        y[u] = make_uint4(w[4], w[5], w[6], w[7]);
      }
    }
#pragma unroll
    for (int u = 0; u < kIoUnroll; ++u) {
      const int i = base + u * nthr + tid;
      if (i >= units) continue;
      const int e = 8 * i, q = e / n, nn = e - q * n;
      CellPos p = cell_pos(nn, z);
      const uint32_t blk = sbase + (uint32_t)q * cws;
      uint32_t cell[8];
      if (al16) {
        const uint32_t xa[4] = {x[u].x, x[u].y, x[u].z, x[u].w}, ya[4] = {y[u].x, y[u].y, y[u].z, y[u].w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          cell[2 * k] = __byte_perm(xa[k], ya[k], 0x5410);       // element 2k of a | of b << 16
          cell[2 * k + 1] = __byte_perm(xa[k], ya[k], 0x7632);
        }
      } else {
        const uint32_t w[8] = {x[u].x, x[u].y, x[u].z, x[u].w, y[u].x, y[u].y, y[u].z, y[u].w};
#pragma unroll
        for (int k = 0; k < 8; ++k) cell[k] = w[k];
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        sts32(cell_addr(blk, p, rs), cell[k]);
        p.next(z);
      }
    }
  }
}

__device__ __forceinline__ void store_outputs_pair16(uint8_t* hard, int packed, int16_t* post, int ncw, int n, int z,
                                                     uint32_t sbase, uint32_t cws, int rs) {
  const int npairs = (ncw + 1) >> 1;
  const int units = npairs * n / 8;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const bool al16 = ((reinterpret_cast<uintptr_t>(hard) | reinterpret_cast<uintptr_t>(post)) & 15) == 0;
  const int nbytes = (n + 7) >> 3;
  for (int base = 0; base < units; base += kIoUnroll * nthr) {
#pragma unroll
    for (int u = 0; u < kIoUnroll; ++u) {
      const int i = base + u * nthr + tid;
      if (i >= units) continue;
      const int e = 8 * i, q = e / n, nn = e - q * n;
      CellPos p = cell_pos(nn, z);
      const uint32_t blk = sbase + (uint32_t)q * cws;
      uint32_t v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        v[k] = lds32(cell_addr(blk, p, rs));
        p.next(z);
      }
#pragma unroll
      for (int lane = 0; lane < 2; ++lane) {
        const int cw = 2 * q + lane;
        if (cw >= ncw) break;
        bool h[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) h[k] = (lane ? (int)v[k] >> 16 : sext16((int)v[k])) <= 0;
        if (packed) {
          uint32_t byte = 0;
#pragma unroll
          for (int k = 0; k < 8; ++k) byte = (byte << 1) | (h[k] ? 1u : 0u);
          hard[(int64_t)cw * nbytes + (nn >> 3)] = (uint8_t)byte;
        } else {
          uint32_t lo = 0, hi = 0;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            lo |= (h[k] ? 1u : 0u) << (8 * k);
            hi |= (h[k + 4] ? 1u : 0u) << (8 * k);
          }
          uint8_t* dst = hard + (int64_t)cw * n + nn;
          if (al16) *reinterpret_cast<uint2*>(dst) = make_uint2(lo, hi);
          else for (int k = 0; k < 8; ++k) dst[k] = h[k] ? 1 : 0;
        }
        if (post) {
          int16_t* dst = post + (int64_t)cw * n + nn;
          uint32_t w[4];
#pragma unroll
          for (int k = 0; k < 4; ++k)
            w[k] = lane ? __byte_perm(v[2 * k], v[2 * k + 1], 0x7632) : __byte_perm(v[2 * k], v[2 * k + 1], 0x5410);
          if (al16) *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
          else for (int k = 0; k < 8; ++k) dst[k] = (int16_t)(w[k >> 1] >> (16 * (k & 1)));
        }
      }
    }
  }
}

}  // namespace qcb
