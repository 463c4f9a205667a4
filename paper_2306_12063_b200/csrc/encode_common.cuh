// encode_common.cuh -- pieces shared by the packed encoders (encode.cu) and the
// per-structure instantiations of the compile-time-shift bit-granular encoder
// at scaled WiMAX Z (enc_scaled_*.cu).
#pragma once
#include <type_traits>
#include <utility>

#include "bulk_copy.cuh"
#include "common.cuh"
#include "kernels.h"
#include "launch_cache.h"

namespace qcb {

constexpr int kEncThreads = 128;
typedef unsigned __int128 u128;

__host__ __device__ constexpr int enc_stride(int bytes) { return ((bytes + 3) & ~3) | 4; }

// ---- compile-time structure queries -----------------------------------------------
template <class S>
constexpr int entry_at(int t, int j) {   // entry index of block (t, j); -1 = zero block
  for (int e = S::START[t]; e < S::START[t + 1]; ++e)
    if (S::COL[e] == j) return e;
  return -1;
}


template <class S, int Z = S::Z0>
constexpr int hb_y_shift() {             // the single interior h_b entry (find_y, encoder.py:39-46)
  for (int t = 1; t < S::MB - 1; ++t)
    if (entry_at<S>(t, S::KB) >= 0) return zshift<S, Z>(entry_at<S>(t, S::KB));
  return 0;
}

__device__ __forceinline__ uint32_t bswap32(uint32_t v) { return __byte_perm(v, 0, 0x0123); }

inline int64_t enc_grid(const void* kern, size_t smem, int64_t tiles, cudaError_t* err) {
  int per_sm = 0;
  if ((*err = ensure_dyn_smem(kern, smem)) != cudaSuccess) return 0;
  if ((*err = kernel_occupancy(kern, kEncThreads, smem, &per_sm)) != cudaSuccess) return 0;
  if (per_sm < 1) { *err = cudaErrorLaunchOutOfResources; return 0; }
  const int64_t cap = (int64_t)device_sm_count() * per_sm;
  return tiles < cap ? tiles : cap;
}

// ---- compile-time shifts at any Z (Wi-Fi Z0 = 27/54/81, scaled WiMAX Z = 24..92) -----
// A Z-bit block is W = ceil(Z/32) big-endian words (bit 0 = MSB of word 0, pad
// bits zero).  Thread c loads its np.packbits info row from a linear copy of the
// tile into registers (one runtime funnel shift per word: the row starts at
// bit 8 c ceil(K/8)); from there every block offset, rotation and output
// position is a compile-time constant, so the XOR work is funnel shifts on
// registers.  The codeword row is streamed into a linear output tile at its
// own byte offset: interior words are plain stores, the two words shared with
// the neighbouring rows are ORed in (atomicOr on the zeroed tile).
template <int Z>
struct BZ {
  static constexpr int W = (Z + 31) / 32;
  static constexpr uint32_t LAST = (Z % 32) ? ~0u << (32 - Z % 32) : ~0u;
  uint32_t w[W];
};
template <int Z, int E>
__device__ __forceinline__ BZ<Z> rotlz(const BZ<Z>& x) {   // out bit p = in bit (p + E) mod Z
  if constexpr (E == 0) {
    return x;
  } else {
    constexpr int W = BZ<Z>::W, la = E / 32, lr = E % 32, ra = (Z - E) / 32, rr = (Z - E) % 32;
    auto get = [&](int i) { return (i >= 0 && i < W) ? x.w[i] : 0u; };
    BZ<Z> o;
#pragma unroll
    for (int q = 0; q < W; ++q) {
      const uint32_t l = lr == 0 ? get(q + la) : __funnelshift_l(get(q + la + 1), get(q + la), lr);
      const uint32_t r = rr == 0 ? get(q - ra) : __funnelshift_r(get(q - ra), get(q - ra - 1), rr);
      o.w[q] = l | r;
    }
    o.w[W - 1] &= BZ<Z>::LAST;
    return o;
  }
}
template <int Z>
__device__ __forceinline__ void bz_xor(BZ<Z>& a, const BZ<Z>& b) {
#pragma unroll
  for (int q = 0; q < BZ<Z>::W; ++q) a.w[q] ^= b.w[q];
}

template <class S, int ZZ>
struct ZBitsTile {
  static constexpr int Z = ZZ, K = S::KB * Z, N = S::NB * Z;
  static constexpr int KBYTES = (K + 7) / 8, NBYTES = (N + 7) / 8;
  static constexpr int KW = (K + 31) / 32, NW = (N + 31) / 32;   // row words (info / codeword)
  static constexpr int K0 = K / 32;                               // codeword words holding only info bits
  static constexpr int IN_BYTES = kEncThreads * KBYTES, OUT_BYTES = kEncThreads * NBYTES;
  static constexpr int IN_ALLOC = (IN_BYTES + 16 + 15) & ~15, OUT_ALLOC = (OUT_BYTES + 16 + 15) & ~15;
  static constexpr size_t SMEM = (size_t)IN_ALLOC + OUT_ALLOC;
};

template <class S, int Z, int KW, int OFF>
__device__ __forceinline__ BZ<Z> block_of(const uint32_t (&R)[KW]) {   // bits [OFF, OFF + Z) of the row
  constexpr int a = OFF / 32, r = OFF % 32;
  auto get = [&](int i) { return i < KW ? R[i] : 0u; };
  BZ<Z> x;
#pragma unroll
  for (int q = 0; q < BZ<Z>::W; ++q) x.w[q] = r == 0 ? get(a + q) : __funnelshift_l(get(a + q + 1), get(a + q), r);
  x.w[BZ<Z>::W - 1] &= BZ<Z>::LAST;
  return x;
}
// Periodic expansion of a block: PZ.w[k] = bits [32k, 32k + 32) of the
// infinite string S[i] = x[i mod Z], so a rotation by E is one funnel shift
// per word (S[E + 32q ..]); bits past Z in the last word are garbage until the
// accumulated S_i is masked once (Z >= 16: one wrap per word suffices).
template <int Z>
struct PZ {
  static constexpr int W = BZ<Z>::W, NW = (Z - 1 + 32 * W) / 32 + 1;
  uint32_t w[NW];
};
template <int Z, int O>
__device__ __forceinline__ uint32_t word_at(const BZ<Z>& x) {   // S[O .. O + 32), 0 <= O < Z
  static_assert(Z >= 16, "one wrap per word");
  constexpr int W = BZ<Z>::W, a = O / 32, r = O % 32;
  auto get = [&](int i) { return i < W ? x.w[i] : 0u; };
  const uint32_t head = r == 0 ? get(a) : __funnelshift_l(get(a + 1), get(a), r);
  if constexpr (O + 32 <= Z) return head;
  else return head | (x.w[0] >> (Z - O));
}
template <int Z, int... Ks>
__device__ __forceinline__ PZ<Z> periodic(const BZ<Z>& x, std::integer_sequence<int, Ks...>) {
  return PZ<Z>{{word_at<Z, (32 * Ks) % Z>(x)...}};
}
template <int Z, int E>
__device__ __forceinline__ void xor_rot(BZ<Z>& s, const PZ<Z>& p) {   // s ^= rotl(x, E), unmasked
#pragma unroll
  for (int q = 0; q < BZ<Z>::W; ++q) {
    constexpr int r = E % 32;
    const int a = (E + 32 * q) / 32;
    s.w[q] ^= r == 0 ? p.w[a] : __funnelshift_l(p.w[a + 1], p.w[a], r);
  }
}
template <class S, int Z, int T, int J>
__device__ __forceinline__ void accz(BZ<Z>& s, const PZ<Z>& pj) {
  constexpr int e = entry_at<S>(T, J);
  if constexpr (e >= 0) xor_rot<Z, zshift<S, Z>(e)>(s, pj);
}
template <class S, int Z, int J, int... Ts>
__device__ __forceinline__ void colz(BZ<Z> (&s)[S::MB], const PZ<Z>& pj, std::integer_sequence<int, Ts...>) {
  (accz<S, Z, Ts, J>(s[Ts], pj), ...);
}
template <class S, int Z, int KW, int... Js>
__device__ __forceinline__ void colsz(BZ<Z> (&s)[S::MB], const uint32_t (&R)[KW], std::integer_sequence<int, Js...>) {
  (colz<S, Z, Js>(s, periodic<Z>(block_of<S, Z, KW, Js * Z>(R), std::make_integer_sequence<int, PZ<Z>::NW>{}),
                  std::make_integer_sequence<int, S::MB>{}),
   ...);
#pragma unroll
  for (int i = 0; i < S::MB; ++i) s[i].w[BZ<Z>::W - 1] &= BZ<Z>::LAST;
}
template <class S, int Z, int T>
__device__ __forceinline__ void hbz(BZ<Z>& v, const BZ<Z>& v0) {
  constexpr int e = entry_at<S>(T, S::KB);
  if constexpr (e >= 0) bz_xor(v, rotlz<Z, zshift<S, Z>(e)>(v0));
}
// OR block v into the codeword words O at row bit offset OFF
template <int Z, int OFF, int NW>
__device__ __forceinline__ void put_z(uint32_t (&O)[NW], const BZ<Z>& v) {
  constexpr int wi = OFF / 32, sh = OFF % 32;
#pragma unroll
  for (int q = 0; q < BZ<Z>::W; ++q) {
    if (wi + q < NW) O[wi + q] |= sh == 0 ? v.w[q] : v.w[q] >> sh;
    if (sh != 0 && wi + q + 1 < NW) O[wi + q + 1] |= v.w[q] << (32 - sh);
  }
}
template <class S, int Z, int T, int NW>
__device__ __forceinline__ void chainz(BZ<Z>& v, const BZ<Z>& v0, const BZ<Z> (&s)[S::MB], uint32_t (&O)[NW]) {
  if constexpr (T + 1 < S::MB) {                           // v_{T+1} = v_T ^ S_T ^ [hb_T] P v_0
    bz_xor(v, s[T]);
    hbz<S, Z, T>(v, v0);
    put_z<Z, S::KB * Z + (T + 1) * Z>(O, v);
    chainz<S, Z, T + 1>(v, v0, s, O);
  }
}

// One codeword: thread `c` of the tile reads its info row from the linear
// input tile `lin` and streams the codeword row into the zeroed linear output
// tile `lout` (interior words stored, the two shared words ORed in).
template <class S, int Z>
__device__ __forceinline__ void zbits_row(const uint32_t* lin, uint32_t* lout, int c) {
  using T = ZBitsTile<S, Z>;
  const uint32_t b0 = (uint32_t)c * T::KBYTES, a0 = b0 >> 2, sh_in = 8 * (b0 & 3);
  uint32_t R[T::KW];                                       // the info row as big-endian words
#pragma unroll
  for (int m = 0; m < T::KW; ++m) R[m] = __funnelshift_l(bswap32(lin[a0 + m + 1]), bswap32(lin[a0 + m]), sh_in);
  if constexpr (T::K % 32 != 0) R[T::KW - 1] &= ~0u << (32 - T::K % 32);
  BZ<Z> s[S::MB];
#pragma unroll
  for (int i = 0; i < S::MB; ++i)
#pragma unroll
    for (int q = 0; q < BZ<Z>::W; ++q) s[i].w[q] = 0;
  colsz<S, Z, T::KW>(s, R, std::make_integer_sequence<int, S::KB>{});
  BZ<Z> ssum = s[0];
#pragma unroll
  for (int i = 1; i < S::MB; ++i) bz_xor(ssum, s[i]);
  uint32_t O[T::NW];
#pragma unroll
  for (int m = 0; m < T::NW; ++m) O[m] = m < T::KW ? R[m] : 0u;   // systematic bits
  const BZ<Z> v0 = rotlz<Z, (Z - hb_y_shift<S, Z>()) % Z>(ssum);
  put_z<Z, T::K>(O, v0);
  BZ<Z> v = s[0];
  hbz<S, Z, 0>(v, v0);
  put_z<Z, T::K + Z>(O, v);
  chainz<S, Z, 1>(v, v0, s, O);
  const uint32_t ob = (uint32_t)c * T::NBYTES, w0 = ob >> 2, sh = 8 * (ob & 3);
#pragma unroll
  for (int t = 0; t <= T::NW; ++t) {                       // words t = 0 .. NW touched when sh != 0
    const uint32_t hi = t > 0 ? O[t - 1] : 0u, lo = t < T::NW ? O[t] : 0u;
    const uint32_t y = bswap32(__funnelshift_r(lo, hi, sh));
    const bool edge = t == 0 || t >= (int)((sh + 8 * T::NBYTES) >> 5);   // may hold a neighbour's bytes
    if (edge) {
      if (y) atomicOr(lout + w0 + t, y);
    } else {
      lout[w0 + t] = y;
    }
  }
}

// staged kernel: any alignment, ragged last tile
template <class S, int Z>
__global__ void __launch_bounds__(kEncThreads) encode_zbits_kernel(const __grid_constant__ EncodeArgs a) {
  using T = ZBitsTile<S, Z>;
  extern __shared__ __align__(16) uint8_t sm[];
  uint32_t* lin = reinterpret_cast<uint32_t*>(sm);                  // the tile's info rows, contiguous
  uint32_t* lout = reinterpret_cast<uint32_t*>(sm + T::IN_ALLOC);   // the tile's codeword rows, contiguous
  const int tid = threadIdx.x;
  const bool in_al = (reinterpret_cast<uintptr_t>(a.info) & 15) == 0;
  const bool out_al = (reinterpret_cast<uintptr_t>(a.cw) & 15) == 0;
  for (int64_t tile = blockIdx.x; tile * kEncThreads < a.w; tile += gridDim.x) {
    const int64_t cw0 = tile * kEncThreads;
    const int ncw = (int)(a.w - cw0 < kEncThreads ? a.w - cw0 : kEncThreads);
    const bool full = ncw == kEncThreads;
    const uint8_t* gin = a.info + cw0 * T::KBYTES;
    if (in_al && full) {
      const uint4* g = reinterpret_cast<const uint4*>(gin);
      for (int i = tid; i < T::IN_BYTES / 16; i += kEncThreads) reinterpret_cast<uint4*>(lin)[i] = __ldcs(g + i);
    } else {
      for (int i = tid; i < ncw * T::KBYTES; i += kEncThreads) sm[i] = gin[i];
    }
    for (int i = tid; i < T::OUT_ALLOC / 16; i += kEncThreads) reinterpret_cast<uint4*>(lout)[i] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    if (tid < ncw) zbits_row<S, Z>(lin, lout, tid);
    __syncthreads();
    uint8_t* gout = a.cw + cw0 * T::NBYTES;
    if (out_al && full) {
      uint4* g = reinterpret_cast<uint4*>(gout);
      for (int i = tid; i < T::OUT_BYTES / 16; i += kEncThreads) __stcs(g + i, reinterpret_cast<const uint4*>(lout)[i]);
    } else {
      const uint8_t* lb = reinterpret_cast<const uint8_t*>(lout);
      for (int i = tid; i < ncw * T::NBYTES; i += kEncThreads) gout[i] = lb[i];
    }
    __syncthreads();
  }
}

// Bulk-copy pipeline (whole 16-byte-aligned tiles): info tiles arrive by
// cp.async.bulk into a double buffer completing on mbarriers, codeword tiles
// leave by one bulk store each, so tile i+1's load and tile i-1's store
// overlap tile i's encoding (as encode_z96_kernel).
template <class S, int Z>
struct ZBitsPipe {
  using T = ZBitsTile<S, Z>;
  static constexpr int IN_ALLOC = T::IN_ALLOC, OUT_ALLOC = T::OUT_ALLOC;
  static constexpr size_t SMEM = 2 * (size_t)IN_ALLOC + OUT_ALLOC + 16;
};
template <class S, int Z>
__global__ void __launch_bounds__(kEncThreads) encode_zbits_tma_kernel(const __grid_constant__ EncodeArgs a) {
  using T = ZBitsTile<S, Z>;
  using PP = ZBitsPipe<S, Z>;
  extern __shared__ __align__(128) uint8_t sm[];
  uint8_t* inbuf = sm;                                     // 2 x IN_ALLOC
  uint32_t* lout = reinterpret_cast<uint32_t*>(sm + 2 * PP::IN_ALLOC);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 2 * PP::IN_ALLOC + PP::OUT_ALLOC);
  const int64_t tiles = a.w / kEncThreads;
  const int tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0)
    for (int b = 0; b < 2; ++b) {
      const int64_t tl = blockIdx.x + (int64_t)b * gridDim.x;
      if (tl < tiles) bulk_load(inbuf + b * PP::IN_ALLOC, a.info + tl * T::IN_BYTES, T::IN_BYTES, &bar[b]);
    }
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++it) {
    const int b = it & 1;
    if (tid == 0) bulk_wait_read();                        // the previous store has left lout
    __syncthreads();
    for (int i = tid; i < PP::OUT_ALLOC / 16; i += kEncThreads) reinterpret_cast<uint4*>(lout)[i] = make_uint4(0, 0, 0, 0);
    mbar_wait(&bar[b], (uint32_t)((it >> 1) & 1));
    __syncthreads();
    zbits_row<S, Z>(reinterpret_cast<const uint32_t*>(inbuf + b * PP::IN_ALLOC), lout, tid);
    fence_async_smem();                                    // generic-proxy writes -> bulk store
    __syncthreads();                                       // lout complete, inbuf[b] consumed
    if (tid == 0) {
      bulk_store(a.cw + tile * T::OUT_BYTES, lout, T::OUT_BYTES);
      const int64_t nxt = tile + 2 * (int64_t)gridDim.x;
      if (nxt < tiles) bulk_load(inbuf + b * PP::IN_ALLOC, a.info + nxt * T::IN_BYTES, T::IN_BYTES, &bar[b]);
    }
  }
  if (tid == 0) bulk_wait_all();
}

template <class S, int Z>
inline cudaError_t launch_zbits(const EncodeArgs& a, cudaStream_t s) {
  using T = ZBitsTile<S, Z>;
  cudaError_t e = cudaSuccess;
  const bool aligned = ((reinterpret_cast<uintptr_t>(a.info) | reinterpret_cast<uintptr_t>(a.cw)) & 15) == 0;
  const int64_t full = aligned ? a.w / kEncThreads * kEncThreads : 0;
  if (full > 0) {
    const size_t smem = ZBitsPipe<S, Z>::SMEM;
    const int64_t grid = enc_grid((const void*)encode_zbits_tma_kernel<S, Z>, smem, full / kEncThreads, &e);
    if (e != cudaSuccess) return e;
    EncodeArgs b = a;
    b.w = full;
    encode_zbits_tma_kernel<S, Z><<<(unsigned)grid, kEncThreads, smem, s>>>(b);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  if (full == a.w) return cudaSuccess;
  EncodeArgs r = a;
  r.info = a.info + full * T::KBYTES;
  r.cw = a.cw + full * T::NBYTES;
  r.w = a.w - full;
  const int64_t grid = enc_grid((const void*)encode_zbits_kernel<S, Z>, T::SMEM, (r.w + kEncThreads - 1) / kEncThreads, &e);
  if (e != cudaSuccess) return e;
  encode_zbits_kernel<S, Z><<<(unsigned)grid, kEncThreads, T::SMEM, s>>>(r);
  return cudaGetLastError();
}


// scaled WiMAX codes (standard zero pattern, shifts = the 802.16e scaling of
// the Z0 = 96 table, any Z = 24..92 step 4): one instantiation per (structure,
// Z), split over enc_scaled_*.cu; returns cudaErrorNotSupported for other Z.
cudaError_t launch_zbits_scaled(const EncodeArgs& a, int structure_id, cudaStream_t s);
#define QCB_SCALED_Z(X) X(24) X(28) X(32) X(36) X(40) X(44) X(48) X(52) X(56) X(60) X(64) X(68) X(72) X(76) X(80) X(84) X(88) X(92)
cudaError_t launch_zbits_scaled_r12(const EncodeArgs& a, cudaStream_t s);
cudaError_t launch_zbits_scaled_r23a(const EncodeArgs& a, cudaStream_t s);
cudaError_t launch_zbits_scaled_r23b(const EncodeArgs& a, cudaStream_t s);
cudaError_t launch_zbits_scaled_r34a(const EncodeArgs& a, cudaStream_t s);
cudaError_t launch_zbits_scaled_r34b(const EncodeArgs& a, cudaStream_t s);
cudaError_t launch_zbits_scaled_r56(const EncodeArgs& a, cudaStream_t s);

}  // namespace qcb
