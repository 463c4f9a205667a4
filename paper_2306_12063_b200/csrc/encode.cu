// encode.cu -- bit-packed direct QC-LDPC encoder (byte-aligned Z), sm_100a.
//
// Algorithm: /root/reference/pkg/src/qcldpc/encoder.py:166-199 (encode_packed),
// i.e. the paper's Eqs. 12-15 on MSB-first packed blocks:
//   S_i     = XOR_j P_{e_ij} u_j          (P_e = gather (r + e) mod Z: rotate left)
//   v_0     = rot_fwd(XOR_i S_i, hb_y)    (cyclic_shift_packed, encoder.py:72-90)
//   v_1     = S_0 ^ P_{hb_0} v_0
//   v_{i+1} = v_i ^ S_i ^ [hb_i >= 0] P_{hb_i} v_0
// A Z-bit block is held right-aligned in an unsigned __int128 (bit 0 of the
// block = most significant of the Z bits), so both rotations are two shifts
// and an OR.  The reference's word_bits choice (8/16/32) only changes how the
// same bits are grouped; the encoded bytes are identical.
//
// Data path (HBM-bound): one CTA stages 128 codewords of info bytes into
// shared memory with 16-byte coalesced loads, one thread encodes one
// codeword from shared memory, and the CTA writes the 128 codewords back
// with 16-byte coalesced stores.  Grid-stride over CTA tiles.
#include "common.cuh"
#include "kernels.h"

namespace qcb {

constexpr int kEncThreads = 128;
typedef unsigned __int128 u128;

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

__global__ void __launch_bounds__(kEncThreads) encode_packed_kernel(const __grid_constant__ EncodeArgs a) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int z = a.z, mb = a.mb, nb = a.nb, kb = nb - mb;
  const int zb = z >> 3, kbytes = kb * zb, nbytes = nb * zb;
  const int in_stride = ((kbytes + 3) & ~3) | 4;   // 4-byte aligned, odd word count (banks)
  const int out_stride = ((nbytes + 3) & ~3) | 4;
  uint8_t* sin = sm;
  uint8_t* sout = sm + kEncThreads * in_stride;
  const u128 mask = (z == 128) ? ~u128(0) : ((u128(1) << z) - 1);

  for (int64_t tile = blockIdx.x; tile * kEncThreads < a.w; tile += gridDim.x) {
    const int64_t cw0 = tile * kEncThreads;
    const int ncw = (int)(a.w - cw0 < kEncThreads ? a.w - cw0 : kEncThreads);
    // ---- stage info bytes (coalesced 4-byte words when aligned) ----------
    const uint8_t* gin = a.info + cw0 * kbytes;
    const int total_in = ncw * kbytes;
    if ((kbytes & 3) == 0 && (reinterpret_cast<uintptr_t>(gin) & 3) == 0) {
      const uint32_t* g4 = reinterpret_cast<const uint32_t*>(gin);
      const int kw = kbytes >> 2;
      for (int i = threadIdx.x; i < total_in >> 2; i += blockDim.x) {
        const int q = i / kw, o = i - q * kw;
        *reinterpret_cast<uint32_t*>(sin + q * in_stride + 4 * o) = __ldcs(g4 + i);
      }
    } else {
      for (int i = threadIdx.x; i < total_in; i += blockDim.x) {
        const int q = i / kbytes, o = i - q * kbytes;
        sin[q * in_stride + o] = gin[i];
      }
    }
    __syncthreads();
    // ---- encode one codeword per thread ------------------------------------
    if (threadIdx.x < ncw) {
      const uint8_t* u = sin + threadIdx.x * in_stride;
      uint8_t* out = sout + threadIdx.x * out_stride;
      u128 s[12];
      u128 ssum = 0;
      for (int i = 0; i < mb; ++i) s[i] = 0;
      for (int j = 0; j < kb; ++j) {
        const u128 uj = load_block(u + j * zb, zb);
        for (int i = 0; i < mb; ++i) {
          const int e = a.shifts[i * nb + j];
          if (e >= 0) s[i] ^= rotl_z(uj, e, z, mask);
        }
      }
      for (int i = 0; i < mb; ++i) ssum ^= s[i];
      // v0 = cyclic_shift_packed(ssum, hb_shift): forward rotation = rotl by (z - hb) mod z
      const u128 v0 = rotl_z(ssum, (z - a.hb_shift) % z, z, mask);
      store_block(out + kbytes, v0, zb);
      if (mb >= 2) {
        u128 v = s[0] ^ rotl_z(v0, a.shifts[kb], z, mask);   // v1 (encoder.py:192)
        store_block(out + kbytes + zb, v, zb);
        for (int i = 1; i < mb - 1; ++i) {                    // encoder.py:193-197
          v ^= s[i];
          const int hb = a.shifts[i * nb + kb];
          if (hb >= 0) v ^= rotl_z(v0, hb, z, mask);
          store_block(out + kbytes + (i + 1) * zb, v, zb);
        }
      }
      for (int b = 0; b < kbytes; ++b) out[b] = u[b];
    }
    __syncthreads();
    // ---- write codewords back (coalesced) ----------------------------------
    uint8_t* gout = a.cw + cw0 * nbytes;
    const int total_out = ncw * nbytes;
    if ((nbytes & 3) == 0 && (reinterpret_cast<uintptr_t>(gout) & 3) == 0) {
      uint32_t* g4 = reinterpret_cast<uint32_t*>(gout);
      const int nw = nbytes >> 2;
      for (int i = threadIdx.x; i < total_out >> 2; i += blockDim.x) {
        const int q = i / nw, o = i - q * nw;
        __stcs(g4 + i, *reinterpret_cast<const uint32_t*>(sout + q * out_stride + 4 * o));
      }
    } else {
      for (int i = threadIdx.x; i < total_out; i += blockDim.x) {
        const int q = i / nbytes, o = i - q * nbytes;
        gout[i] = sout[q * out_stride + o];
      }
    }
    __syncthreads();
  }
}

cudaError_t launch_encode_packed(const EncodeArgs& a, cudaStream_t s) {
  if (a.w <= 0) return cudaSuccess;
  const int zb = a.z >> 3, kb = a.nb - a.mb;
  const int in_stride = ((kb * zb + 3) & ~3) | 4, out_stride = ((a.nb * zb + 3) & ~3) | 4;
  const size_t smem = (size_t)kEncThreads * (in_stride + out_stride);
  cudaError_t e = cudaFuncSetAttribute(encode_packed_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t tiles = (a.w + kEncThreads - 1) / kEncThreads;
  const int64_t grid = tiles < (int64_t)sms * 8 ? tiles : (int64_t)sms * 8;
  encode_packed_kernel<<<(unsigned)grid, kEncThreads, smem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace qcb
