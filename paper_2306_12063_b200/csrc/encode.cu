// encode.cu -- bit-packed direct QC-LDPC encoder (byte-aligned Z), sm_100a.
//
// Algorithm: /root/reference/pkg/src/qcldpc/encoder.py:166-199 (encode_packed),
// i.e. the paper's Eqs. 12-15 on MSB-first packed blocks:
//   S_i     = XOR_j P_{e_ij} u_j          (P_e = gather (r + e) mod Z: rotate left)
//   v_0     = rot_fwd(XOR_i S_i, hb_y)    (cyclic_shift_packed, encoder.py:72-90)
//   v_1     = S_0 ^ P_{hb_0} v_0          (hb_0 < 0 acts as (hb_0 mod Z), encoder.py:93-100)
//   v_{i+1} = v_i ^ S_i ^ [hb_i >= 0] P_{hb_i} v_0
// The reference's word_bits choice (8/16/32) only changes how the same bits
// are grouped; the encoded bytes are identical for every choice.
//
// Data path (HBM-bound: K/8 bytes in + N/8 bytes out per codeword): a CTA
// stages 128 codewords of info bytes into shared memory with coalesced
// 4-byte loads, one thread encodes one codeword, the CTA writes the 128
// codewords back with coalesced 4-byte stores; grid-stride over tiles.
//
// Three encoders, chosen per code:
//  * encode_z96_kernel<S>    native WiMAX Z = 96 codes (structure's own
//    SHIFT0): a block is three big-endian 32-bit words, every circulant
//    rotation has a compile-time shift and costs three funnel shifts; the
//    tier structure is unrolled from structures_gen.cuh, all S_i in registers;
//  * encode_struct_kernel<S> other codes of a known structure: same unrolled
//    structure, runtime shifts, blocks in unsigned __int128 registers;
//  * encode_generic_kernel   any other shift table: runtime loops, the S_i
//    accumulate in the shared-memory output row (no local-memory arrays).
#include <utility>

#include "encode_common.cuh"

namespace qcb {

// ---- staging ----------------------------------------------------------------------
__device__ __forceinline__ void stage_in(const uint8_t* gin, uint8_t* sin, int ncw, int kbytes, int stride) {
  const int total = ncw * kbytes;
  if ((kbytes & 3) == 0 && (reinterpret_cast<uintptr_t>(gin) & 3) == 0) {
    const uint32_t* g4 = reinterpret_cast<const uint32_t*>(gin);
    const int kw = kbytes >> 2;
    for (int i = threadIdx.x; i < total >> 2; i += blockDim.x) {
      const int q = i / kw, o = i - q * kw;
      *reinterpret_cast<uint32_t*>(sin + q * stride + 4 * o) = __ldcs(g4 + i);
    }
  } else {
    for (int i = threadIdx.x; i < total; i += blockDim.x) {
      const int q = i / kbytes, o = i - q * kbytes;
      sin[q * stride + o] = gin[i];
    }
  }
}

__device__ __forceinline__ void stage_out(uint8_t* gout, const uint8_t* sout, int ncw, int nbytes, int stride) {
  const int total = ncw * nbytes;
  if ((nbytes & 3) == 0 && (reinterpret_cast<uintptr_t>(gout) & 3) == 0) {
    uint32_t* g4 = reinterpret_cast<uint32_t*>(gout);
    const int nw = nbytes >> 2;
    for (int i = threadIdx.x; i < total >> 2; i += blockDim.x) {
      const int q = i / nw, o = i - q * nw;
      __stcs(g4 + i, *reinterpret_cast<const uint32_t*>(sout + q * stride + 4 * o));
    }
  } else {
    for (int i = threadIdx.x; i < total; i += blockDim.x) {
      const int q = i / nbytes, o = i - q * nbytes;
      gout[i] = sout[q * stride + o];
    }
  }
}

// ---- Z = 96 with compile-time shifts: a block is 3 big-endian words ----------------
struct B96 { uint32_t w[3]; };

template <int E>
__device__ __forceinline__ B96 rotl96(const B96& x) {   // out bit p = in bit (p + E) mod 96
  constexpr int sw = E / 32, sb = E % 32;
  B96 o;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const uint32_t hi = x.w[(i + sw) % 3], lo = x.w[(i + sw + 1) % 3];
    o.w[i] = sb == 0 ? hi : __funnelshift_l(lo, hi, sb);
  }
  return o;
}
__device__ __forceinline__ void xor_into(B96& a, const B96& b) {
  a.w[0] ^= b.w[0]; a.w[1] ^= b.w[1]; a.w[2] ^= b.w[2];
}

template <class S, int T, int J>
__device__ __forceinline__ void acc96(B96& s, const B96 (&u)[S::KB]) {
  constexpr int e = entry_at<S>(T, J);
  if constexpr (e >= 0) xor_into(s, rotl96<S::SHIFT0[e]>(u[J]));
}
template <class S, int T, int... Js>
__device__ __forceinline__ void row96(B96& s, const B96 (&u)[S::KB], std::integer_sequence<int, Js...>) {
  s = B96{{0u, 0u, 0u}};
  (acc96<S, T, Js>(s, u), ...);
}
template <class S, int... Ts>
__device__ __forceinline__ void rows96(B96 (&s)[S::MB], const B96 (&u)[S::KB], std::integer_sequence<int, Ts...>) {
  (row96<S, Ts>(s[Ts], u, std::make_integer_sequence<int, S::KB>{}), ...);
}
template <class S, int T>
__device__ __forceinline__ void hb96(B96& v, const B96& v0) {   // v ^= P_{hb_T} v0 when hb_T >= 0
  constexpr int e = entry_at<S>(T, S::KB);
  if constexpr (e >= 0) xor_into(v, rotl96<S::SHIFT0[e]>(v0));
}
template <class S, int T>
__device__ __forceinline__ void chain96(B96 (&v)[S::MB], const B96 (&s)[S::MB]) {   // encoder.py:193-197
  if constexpr (T + 1 < S::MB) {
    v[T + 1] = v[T];
    xor_into(v[T + 1], s[T]);
    hb96<S, T>(v[T + 1], v[0]);
    chain96<S, T + 1>(v, s);
  }
}

// Bulk-copy (TMA) pipeline: info tiles arrive by cp.async.bulk into a double
// buffer completing on an mbarrier, codeword tiles leave by one bulk store
// per tile.  While a CTA encodes tile i, tile i+1 (and i+2) is in flight in
// and tile i-1 is draining out, so the kernel streams at HBM rate with only
// two 128-thread CTAs per SM.


template <class S>
struct Z96Tile {
  static constexpr int KW = S::KB * 3, NW = S::NB * 3;          // 32-bit words per codeword
  static constexpr int IN_BYTES = kEncThreads * KW * 4, OUT_BYTES = kEncThreads * NW * 4;
  static constexpr size_t SMEM = 2 * (size_t)IN_BYTES + OUT_BYTES + 16;
  static_assert(KW % 2 == 0 && NW % 4 == 0, "8-byte loads / 16-byte stores");
};

// One codeword: raw (byte-order) info words in, full codeword words out.
template <class S>
__device__ __forceinline__ void encode96_words(const uint32_t (&raw)[S::KB * 3], uint32_t (&o)[S::NB * 3]) {
  B96 u[S::KB];
#pragma unroll
  for (int j = 0; j < S::KB; ++j)
#pragma unroll
    for (int q = 0; q < 3; ++q) u[j].w[q] = bswap32(raw[3 * j + q]);
  B96 s[S::MB];
  rows96<S>(s, u, std::make_integer_sequence<int, S::MB>{});
  B96 ssum = s[0];
#pragma unroll
  for (int i = 1; i < S::MB; ++i) xor_into(ssum, s[i]);
  B96 v[S::MB];
  v[0] = rotl96<(96 - hb_y_shift<S>()) % 96>(ssum);     // cyclic_shift_packed(ssum, hb_y)
  v[1] = s[0];
  hb96<S, 0>(v[1], v[0]);                                // encoder.py:192
  chain96<S, 1>(v, s);                                   // encoder.py:193-197
#pragma unroll
  for (int k = 0; k < S::KB * 3; ++k) o[k] = raw[k];     // systematic bytes unchanged
#pragma unroll
  for (int i = 0; i < S::MB; ++i)
#pragma unroll
    for (int q = 0; q < 3; ++q) o[3 * S::KB + 3 * i + q] = bswap32(v[i].w[q]);
}

// a.w must be a multiple of kEncThreads here (the host runs the tail through
// encode_struct_kernel); a.info / a.cw 16-byte aligned.
template <class S>
__global__ void __launch_bounds__(kEncThreads, 2) encode_z96_kernel(const __grid_constant__ EncodeArgs a) {
  using T = Z96Tile<S>;
  static_assert(entry_at<S>(0, S::KB) >= 0, "h_b column must start with a non-zero block");
  extern __shared__ __align__(128) uint8_t sm[];
  uint8_t* inbuf = sm;                                    // 2 x IN_BYTES, dense rows of KW words
  uint8_t* outbuf = sm + 2 * T::IN_BYTES;                 // OUT_BYTES, dense rows of NW words
  uint64_t* bar = reinterpret_cast<uint64_t*>(outbuf + T::OUT_BYTES);
  const int64_t tiles = a.w / kEncThreads;
  const int tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      const int64_t tl = blockIdx.x + (int64_t)b * gridDim.x;
      if (tl < tiles) bulk_load(inbuf + b * T::IN_BYTES, a.info + tl * T::IN_BYTES, T::IN_BYTES, &bar[b]);
    }
  }
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++it) {
    const int b = it & 1;
    mbar_wait(&bar[b], (uint32_t)((it >> 1) & 1));
    uint32_t raw[T::KW], o[T::NW];
    const uint2* in2 = reinterpret_cast<const uint2*>(inbuf + b * T::IN_BYTES + tid * T::KW * 4);
#pragma unroll
    for (int k = 0; k < T::KW / 2; ++k) {                 // LDS.64: odd 8-byte stride, no conflicts
      const uint2 x = in2[k];
      raw[2 * k] = x.x;
      raw[2 * k + 1] = x.y;
    }
    encode96_words<S>(raw, o);
    if (tid == 0) bulk_wait_read();                       // previous tile's store has left outbuf
    __syncthreads();                                      // everyone is done with inbuf[b]
    if (tid == 0) {
      const int64_t nxt = tile + 2 * (int64_t)gridDim.x;
      if (nxt < tiles) {
        fence_async_smem();
        bulk_load(inbuf + b * T::IN_BYTES, a.info + nxt * T::IN_BYTES, T::IN_BYTES, &bar[b]);
      }
    }
    uint4* out4 = reinterpret_cast<uint4*>(outbuf + tid * T::NW * 4);
#pragma unroll
    for (int k = 0; k < T::NW / 4; ++k) out4[k] = make_uint4(o[4 * k], o[4 * k + 1], o[4 * k + 2], o[4 * k + 3]);
    fence_async_smem();                                   // generic-proxy writes -> bulk store
    __syncthreads();
    if (tid == 0) bulk_store(a.cw + tile * T::OUT_BYTES, outbuf, T::OUT_BYTES);
  }
  if (tid == 0) bulk_wait_all();
}

// ---- runtime shifts, blocks right-aligned in unsigned __int128 ----------------------
__device__ __forceinline__ u128 rotl_z(u128 b, int e, int z, u128 mask) {
  if (e == 0) return b;
  return ((b << e) | (b >> (z - e))) & mask;
}
__device__ __forceinline__ u128 load_block(const uint8_t* p, int zb) {
  u128 v = 0;
  for (int i = 0; i < zb; ++i) v = (v << 8) | p[i];
  return v;
}
__device__ __forceinline__ void store_block(uint8_t* p, u128 v, int zb) {
  for (int i = zb - 1; i >= 0; --i) { p[i] = (uint8_t)v; v >>= 8; }
}
__device__ __forceinline__ u128 z_mask(int z) { return z == 128 ? ~u128(0) : ((u128(1) << z) - 1); }

// Bit-granular blocks (Z % 8 != 0): block j of a row is the
// MSB-first bit field [j Z, (j + 1) Z) of the np.packbits byte row, read and
// written through the row's big-endian 32-bit words (rows are 4-byte aligned;
// the field plus its offset in the first word spans <= 4 words for Z <= 97).
__device__ __forceinline__ u128 load_bits(const uint8_t* row, int off, int z) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(row) + (off >> 5);
  const int sh = off & 31, nw = (sh + z + 31) >> 5;
  u128 v = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i)
    if (i < nw) v = (v << 32) | bswap32(w[i]);
  return (v >> (nw * 32 - sh - z)) & z_mask(z);
}
__device__ __forceinline__ void store_bits(uint8_t* row, int off, int z, u128 v) {   // replaces the field
  uint32_t* w = reinterpret_cast<uint32_t*>(row) + (off >> 5);
  const int sh = off & 31, nw = (sh + z + 31) >> 5, pad = nw * 32 - sh - z;
  const u128 m = z_mask(z) << pad;
  v = (v & z_mask(z)) << pad;
#pragma unroll
  for (int i = 0; i < 4; ++i)
    if (i < nw) {
      const int s = (nw - 1 - i) * 32;
      const uint32_t mi = (uint32_t)(m >> s), vi = (uint32_t)(v >> s);
      w[i] = bswap32((bswap32(w[i]) & ~mi) | vi);
    }
}
// the K info bits of a bit-granular row, copied word by word (+ a partial field)
__device__ __forceinline__ void copy_info_bits(uint8_t* out, const uint8_t* u, int k) {
  const int full = k >> 5;
  for (int i = 0; i < full; ++i)
    reinterpret_cast<uint32_t*>(out)[i] = reinterpret_cast<const uint32_t*>(u)[i];
  if (k & 31) store_bits(out, full << 5, k & 31, load_bits(u, full << 5, k & 31));
}
// Block access for either layout: byte-aligned (BITS = false) or bit-granular.
template <bool BITS>
__device__ __forceinline__ u128 get_block(const uint8_t* row, int j, int z) {
  if constexpr (BITS) return load_bits(row, j * z, z);
  else return load_block(row + j * (z >> 3), z >> 3);
}
template <bool BITS>
__device__ __forceinline__ void put_block(uint8_t* row, int j, int z, u128 v) {
  if constexpr (BITS) store_bits(row, j * z, z, v);
  else store_block(row + j * (z >> 3), v, z >> 3);
}
__host__ __device__ constexpr int bytes_of_bits(int bits) { return (bits + 7) >> 3; }

template <class S, int T, int J>
__device__ __forceinline__ void acc_rt(u128& s, const u128& uj, const EncodeArgs& a, u128 mask) {
  if constexpr (entry_at<S>(T, J) >= 0) s ^= rotl_z(uj, a.shifts[T * S::NB + J], a.z, mask);
}
template <class S, int J, int... Ts>
__device__ __forceinline__ void col_rt(u128 (&s)[S::MB], const u128& uj, const EncodeArgs& a, u128 mask,
                                       std::integer_sequence<int, Ts...>) {
  (acc_rt<S, Ts, J>(s[Ts], uj, a, mask), ...);
}
template <class S, bool BITS, int... Js>
__device__ __forceinline__ void cols_rt(u128 (&s)[S::MB], const uint8_t* u, int z, const EncodeArgs& a,
                                        u128 mask, std::integer_sequence<int, Js...>) {
  (col_rt<S, Js>(s, get_block<BITS>(u, Js, z), a, mask, std::make_integer_sequence<int, S::MB>{}), ...);
}

// BITS: Z % 8 != 0, rows are np.packbits of K / N bits
template <class S, bool BITS>
__global__ void __launch_bounds__(kEncThreads) encode_struct_kernel(const __grid_constant__ EncodeArgs a) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int z = a.z, k = S::KB * z;
  const int kbytes = bytes_of_bits(k), nbytes = bytes_of_bits(S::NB * z);
  const int in_stride = enc_stride(kbytes), out_stride = enc_stride(nbytes);
  uint8_t* sin = sm;
  uint8_t* sout = sm + kEncThreads * in_stride;
  const u128 mask = z_mask(z);
  for (int64_t tile = blockIdx.x; tile * kEncThreads < a.w; tile += gridDim.x) {
    const int64_t cw0 = tile * kEncThreads;
    const int ncw = (int)(a.w - cw0 < kEncThreads ? a.w - cw0 : kEncThreads);
    stage_in(a.info + cw0 * kbytes, sin, ncw, kbytes, in_stride);
    __syncthreads();
    if (threadIdx.x < ncw) {
      const uint8_t* u = sin + threadIdx.x * in_stride;
      uint8_t* out = sout + threadIdx.x * out_stride;
      if constexpr (BITS) {
        reinterpret_cast<uint32_t*>(out)[(nbytes - 1) >> 2] = 0;   // np.packbits pads with zeros
        copy_info_bits(out, u, k);
      }
      u128 s[S::MB];
#pragma unroll
      for (int i = 0; i < S::MB; ++i) s[i] = 0;
      cols_rt<S, BITS>(s, u, z, a, mask, std::make_integer_sequence<int, S::KB>{});
      u128 ssum = 0;
#pragma unroll
      for (int i = 0; i < S::MB; ++i) ssum ^= s[i];
      const u128 v0 = rotl_z(ssum, (z - a.hb_shift) % z, z, mask);
      put_block<BITS>(out, S::KB, z, v0);
      u128 v = s[0] ^ rotl_z(v0, (a.shifts[S::KB] % z + z) % z, z, mask);
      put_block<BITS>(out, S::KB + 1, z, v);
#pragma unroll
      for (int i = 1; i < S::MB - 1; ++i) {
        v ^= s[i];
        const int hb = a.shifts[i * S::NB + S::KB];
        if (hb >= 0) v ^= rotl_z(v0, hb, z, mask);
        put_block<BITS>(out, S::KB + i + 1, z, v);
      }
      if constexpr (!BITS)
        for (int b = 0; b < kbytes; ++b) out[b] = u[b];
    }
    __syncthreads();
    stage_out(a.cw + cw0 * nbytes, sout, ncw, nbytes, out_stride);
    __syncthreads();
  }
}

template <bool BITS>
__global__ void __launch_bounds__(kEncThreads) encode_generic_kernel(const __grid_constant__ EncodeArgs a) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int z = a.z, mb = a.mb, nb = a.nb, kb = nb - mb;
  const int kbytes = bytes_of_bits(kb * z), nbytes = bytes_of_bits(nb * z);
  const int in_stride = enc_stride(kbytes), out_stride = enc_stride(nbytes);
  uint8_t* sin = sm;
  uint8_t* sout = sm + kEncThreads * in_stride;
  const u128 mask = z_mask(z);
  for (int64_t tile = blockIdx.x; tile * kEncThreads < a.w; tile += gridDim.x) {
    const int64_t cw0 = tile * kEncThreads;
    const int ncw = (int)(a.w - cw0 < kEncThreads ? a.w - cw0 : kEncThreads);
    stage_in(a.info + cw0 * kbytes, sin, ncw, kbytes, in_stride);
    __syncthreads();
    if (threadIdx.x < ncw) {
      const uint8_t* u = sin + threadIdx.x * in_stride;
      uint8_t* out = sout + threadIdx.x * out_stride;   // S_i accumulate in the parity blocks
      if constexpr (BITS) {
        reinterpret_cast<uint32_t*>(out)[(nbytes - 1) >> 2] = 0;
        copy_info_bits(out, u, kb * z);
      }
      for (int i = 0; i < mb; ++i) put_block<BITS>(out, kb + i, z, 0);
      for (int j = 0; j < kb; ++j) {
        const u128 uj = get_block<BITS>(u, j, z);
        for (int i = 0; i < mb; ++i) {
          const int e = a.shifts[i * nb + j];
          if (e >= 0) put_block<BITS>(out, kb + i, z, get_block<BITS>(out, kb + i, z) ^ rotl_z(uj, e, z, mask));
        }
      }
      u128 ssum = 0;
      for (int i = 0; i < mb; ++i) ssum ^= get_block<BITS>(out, kb + i, z);
      const u128 v0 = rotl_z(ssum, (z - a.hb_shift) % z, z, mask);
      const u128 s0 = get_block<BITS>(out, kb, z);
      put_block<BITS>(out, kb, z, v0);
      u128 v = s0 ^ rotl_z(v0, (a.shifts[kb] % z + z) % z, z, mask);
      for (int i = 1; i < mb - 1; ++i) {
        const u128 si = get_block<BITS>(out, kb + i, z);
        put_block<BITS>(out, kb + i, z, v);
        v ^= si;
        const int hb = a.shifts[i * nb + kb];
        if (hb >= 0) v ^= rotl_z(v0, hb, z, mask);
      }
      put_block<BITS>(out, kb + mb - 1, z, v);
      if constexpr (!BITS)
        for (int b = 0; b < kbytes; ++b) out[b] = u[b];
    }
    __syncthreads();
    stage_out(a.cw + cw0 * nbytes, sout, ncw, nbytes, out_stride);
    __syncthreads();
  }
}

template <class K>
static cudaError_t launch_enc(K kern, const EncodeArgs& a, cudaStream_t s) {
  const int kbytes = bytes_of_bits((a.nb - a.mb) * a.z), nbytes = bytes_of_bits(a.nb * a.z);
  const size_t smem = (size_t)kEncThreads * (enc_stride(kbytes) + enc_stride(nbytes));
  cudaError_t e = cudaSuccess;
  const int64_t grid = enc_grid((const void*)kern, smem, (a.w + kEncThreads - 1) / kEncThreads, &e);
  if (e != cudaSuccess) return e;
  kern<<<(unsigned)grid, kEncThreads, smem, s>>>(a);
  return cudaGetLastError();
}

// native Z = 96: full tiles through the bulk-copy pipeline, the ragged tail
// (and misaligned buffers) through the staged kernel.
template <class S>
static cudaError_t launch_z96(const EncodeArgs& a, cudaStream_t s) {
  using T = Z96Tile<S>;
  const bool aligned = ((reinterpret_cast<uintptr_t>(a.info) | reinterpret_cast<uintptr_t>(a.cw)) & 15) == 0;
  const int64_t full = aligned ? a.w / kEncThreads * kEncThreads : 0;
  if (full > 0) {
    cudaError_t e = cudaSuccess;
    const int64_t grid = enc_grid((const void*)encode_z96_kernel<S>, T::SMEM, full / kEncThreads, &e);
    if (e != cudaSuccess) return e;
    EncodeArgs b = a;
    b.w = full;
    encode_z96_kernel<S><<<(unsigned)grid, kEncThreads, T::SMEM, s>>>(b);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  if (full == a.w) return cudaSuccess;
  EncodeArgs r = a;
  r.info = a.info + full * (T::KW * 4);
  r.cw = a.cw + full * (T::NW * 4);
  r.w = a.w - full;
  return launch_enc(encode_struct_kernel<S, false>, r, s);
}

cudaError_t launch_zbits_scaled(const EncodeArgs& a, int structure_id, cudaStream_t s) {
  if (structure_id == S_wimax_r12::ID) return launch_zbits_scaled_r12(a, s);
  if (structure_id == S_wimax_r23a::ID) return launch_zbits_scaled_r23a(a, s);
  if (structure_id == S_wimax_r23b::ID) return launch_zbits_scaled_r23b(a, s);
  if (structure_id == S_wimax_r34a::ID) return launch_zbits_scaled_r34a(a, s);
  if (structure_id == S_wimax_r34b::ID) return launch_zbits_scaled_r34b(a, s);
  if (structure_id == S_wimax_r56::ID) return launch_zbits_scaled_r56(a, s);
  return cudaErrorNotSupported;
}

cudaError_t launch_encode_packed(const EncodeArgs& a, int structure_id, cudaStream_t s) {
  if (a.w <= 0) return cudaSuccess;
  if (a.mb < 2) return cudaErrorInvalidValue;
  const bool bits = (a.z & 7) != 0;
  if (bits && a.z > 97) return cudaErrorInvalidValue;
#define QCB_ENC(STRUCT)                                                                    \
  if (structure_id == STRUCT::ID && STRUCT::NB == a.nb && STRUCT::MB == a.mb) {            \
    if constexpr (STRUCT::Z0 == 96)                                                        \
      if (a.native && a.z == 96) return launch_z96<STRUCT>(a, s);                          \
    if constexpr (STRUCT::Z0 % 8 != 0)                                                     \
      if (a.native && a.z == STRUCT::Z0) return launch_zbits<STRUCT, STRUCT::Z0>(a, s);    \
    if constexpr (STRUCT::Z0 == 96)                                                        \
      if (a.scaled && a.z < 96) {                                                          \
        const cudaError_t e = launch_zbits_scaled(a, structure_id, s);                     \
        if (e != cudaErrorNotSupported) return e;                                          \
      }                                                                                    \
    return bits ? launch_enc(encode_struct_kernel<STRUCT, true>, a, s)                     \
                : launch_enc(encode_struct_kernel<STRUCT, false>, a, s);                   \
  }
  QCB_FOR_EACH_STRUCTURE(QCB_ENC)
#undef QCB_ENC
  return bits ? launch_enc(encode_generic_kernel<true>, a, s) : launch_enc(encode_generic_kernel<false>, a, s);
}

}  // namespace qcb
