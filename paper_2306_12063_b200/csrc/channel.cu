// channel.cu -- the callers either side of the decoder, on the device
// (SURVEY.md §8f rows 1-3): frame generation, the bit-per-byte encoder,
// BPSK/AWGN channel + LLR + fixed-point quantizer, error counting for the
// waterfall loop, and the packed decode-record writer.
//
// Reference:
//   encode_array          /root/reference/pkg/src/qcldpc/encoder.py:133-163
//   _llr_batch            /root/reference/pkg/src/qcldpc/chansim.py:136-143
//     bpsk_modulate :45-47, llr_from_samples :57-62, quantize_llr
//     (decoder.py:165-171)
//   run_waterfall counting chansim.py:166-173
//   decode records        cli.py:180-183
//
// Exactness: with the reference's noise samples supplied (noise != NULL) the
// LLRs are the reference's, bit for bit: every float64 operation is the
// same IEEE operation in the same order (explicit __dmul_rn / __dadd_rn, no
// FMA contraction), the float32 cast is round-to-nearest-even like
// ndarray.astype(float32), and the quantizer's rint is round-half-even like
// np.rint.  Without noise samples the kernel draws its own Gaussian noise
// from a counter-based Philox4x32-10 stream keyed by (seed, point, frame) --
// independent of launch shape and GPU count, but a different stream than
// numpy's, so parity there is statistical (tests/test_gpu_channel.py).
#include <cmath>

#include "common.cuh"
#include "kernels.h"
#include "launch_cache.h"

namespace qcb {

// ---- Philox4x32-10 (Salmon et al., SC'11) ------------------------------------------
struct U4 { uint32_t x, y, z, w; };

__device__ __forceinline__ U4 philox4x32_10(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

// stream 0 = info bits, 1 = noise; chunk = 128-bit block index inside the frame
__device__ __forceinline__ U4 frame_block(uint64_t seed, uint32_t point, uint64_t frame, uint32_t stream,
                                          uint32_t chunk) {
  const U4 ctr{chunk, (uint32_t)frame, (uint32_t)(frame >> 32) ^ (stream << 31), point};
  return philox4x32_10(ctr, (uint32_t)seed, (uint32_t)(seed >> 32));
}

// two standard normals (Box-Muller, float64) from one 128-bit block
__device__ __forceinline__ void normal_pair(const U4& b, double& z0, double& z1) {
  const double u1 = ((double)(((uint64_t)(b.x >> 5) << 26) | (b.y >> 6)) + 1.0) * 0x1.0p-53;   // (0, 1]
  const double u2 = (double)(((uint64_t)(b.z >> 5) << 26) | (b.w >> 6)) * 0x1.0p-53;           // [0, 1)
  const double r = sqrt(-2.0 * log(u1));
  double s, c;
  sincospi(2.0 * u2, &s, &c);
  z0 = r * c;
  z1 = r * s;
}

// ---- device frame generator: info bits ---------------------------------------------
__global__ void frames_info_kernel(uint64_t seed, uint32_t point, int64_t frame0, int64_t w, int32_t k,
                                   uint8_t* info) {
  const int chunks = (k + 127) / 128;
  const int64_t total = w * chunks;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t f = t / chunks;
    const int c = (int)(t - f * chunks);
    const U4 b = frame_block(seed, point, (uint64_t)(frame0 + f), 0u, (uint32_t)c);
    const uint32_t wd[4] = {b.x, b.y, b.z, b.w};
    uint8_t* dst = info + f * k + c * 128;
    const int nbits = k - c * 128 < 128 ? k - c * 128 : 128;
#pragma unroll 4
    for (int i = 0; i < nbits; ++i) dst[i] = (uint8_t)((wd[i >> 5] >> (i & 31)) & 1u);
  }
}

// ---- bit-per-byte encoder (any Z): one CTA per codeword ----------------------------
// encoder.py:133-163: S_i = XOR_j P_{e_ij} u_j, P_e gathers u[(r+e) mod Z];
// v_0 = roll(XOR_i S_i, hb_y); v_1 = S_0 ^ P_{hb_0} v_0;
// v_{i+1} = v_i ^ S_i ^ [hb_i >= 0] P_{hb_i} v_0.
__global__ void encode_array_kernel(const __grid_constant__ EncodeArgs a) {
  extern __shared__ uint8_t sm[];
  const int z = a.z, mb = a.mb, nb = a.nb, kb = nb - mb, k = kb * z, n = nb * z;
  uint8_t* u = sm;                 // k
  uint8_t* s = u + k;              // mb x z
  uint8_t* v0 = s + mb * z;        // z
  for (int64_t cw = blockIdx.x; cw < a.w; cw += gridDim.x) {
    const uint8_t* in = a.info + cw * k;
    uint8_t* out = a.cw + cw * n;
    for (int i = threadIdx.x; i < k; i += blockDim.x) {
      const uint8_t b = in[i];
      u[i] = b;
      out[i] = b;
    }
    __syncthreads();
    for (int r = threadIdx.x; r < z; r += blockDim.x) {
      uint8_t ssum = 0;
      for (int i = 0; i < mb; ++i) {
        uint8_t acc = 0;
        for (int j = 0; j < kb; ++j) {
          const int e = a.shifts[i * nb + j];
          if (e >= 0) acc ^= u[j * z + (r + e) % z];
        }
        s[i * z + r] = acc;
        ssum ^= acc;
      }
      v0[((r + a.hb_shift) % z)] = ssum;          // np.roll(ssum, hb_y): out[r + hb] = in[r]
    }
    __syncthreads();
    const int hb0 = ((a.shifts[kb] % z) + z) % z;  // hb_0 < 0 rolls like np.roll(-e)
    for (int r = threadIdx.x; r < z; r += blockDim.x) {
      uint8_t* par = out + k;
      par[r] = v0[r];
      uint8_t v = s[r] ^ v0[(r + hb0) % z];
      if (mb >= 2) par[z + r] = v;
      for (int i = 1; i < mb - 1; ++i) {
        v ^= s[i * z + r];
        const int hb = a.shifts[i * nb + kb];
        if (hb >= 0) v ^= v0[(r + hb) % z];
        par[(i + 1) * z + r] = v;
      }
    }
    __syncthreads();
  }
}

// ---- channel: codeword bits -> LLRs --------------------------------------------------
template <bool NOISE_IN, bool Q16>
__global__ void channel_kernel(const __grid_constant__ ChannelArgs a) {
  const int64_t pairs = a.w * (int64_t)(a.n >> 1);
  const int hn = a.n >> 1;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < pairs; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t f = t / hn;
    const int p = (int)(t - f * hn);
    const int64_t idx = f * a.n + 2 * p;
    double g0, g1;
    if constexpr (NOISE_IN) {
      g0 = a.noise[idx];
      g1 = a.noise[idx + 1];
    } else {
      normal_pair(frame_block(a.seed, a.point, (uint64_t)(a.frame0 + f), 1u, (uint32_t)p), g0, g1);
    }
    const double gs[2] = {g0, g1};
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const double sym = 1.0 - 2.0 * (double)a.bits[idx + q];                 // bpsk_modulate
      const double y = __dadd_rn(sym, __dmul_rn(a.sqrt_sigma2, gs[q]));       // + sqrt(s2) * noise
      const float l = __double2float_rn(__dmul_rn(a.two_over_sigma2, y));    // (2/s2) * y -> f32
      if constexpr (Q16) {
        double v = rint(__dmul_rn((double)l, a.q_scale));                     // rint(x * (lim / l_clip))
        v = v < -a.q_lim ? -a.q_lim : (v > a.q_lim ? a.q_lim : v);
        reinterpret_cast<int16_t*>(a.llr)[idx + q] = (int16_t)v;
      } else {
        reinterpret_cast<float*>(a.llr)[idx + q] = l;
      }
    }
  }
}

__global__ void quantize_kernel(const float* x, int64_t count, double scale, double lim, int16_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    double v = rint(__dmul_rn((double)x[i], scale));
    v = v < -lim ? -lim : (v > lim ? lim : v);      // np.clip; NaN stays NaN -> see below
    out[i] = (int16_t)(v != v ? 0.0 : v);
  }
}

// ---- waterfall counters: per 256-frame batch (bit errors, frame errors, iterations)
__global__ void count_errors_kernel(const uint8_t* hard, int32_t packed, const uint8_t* info, const int32_t* iters,
                                    int64_t w, int32_t n, int32_t k, int32_t batch, unsigned long long* sums) {
  __shared__ int red[32];
  for (int64_t f = blockIdx.x; f < w; f += gridDim.x) {
    int err = 0;
    const uint8_t* in = info + f * k;
    if (packed) {
      const uint8_t* h = hard + f * ((n + 7) >> 3);
      for (int b = threadIdx.x; b < k; b += blockDim.x) err += ((h[b >> 3] >> (7 - (b & 7))) & 1) != in[b];
    } else {
      const uint8_t* h = hard + f * n;
      for (int b = threadIdx.x; b < k; b += blockDim.x) err += (h[b] != 0) != (in[b] != 0);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) err += __shfl_down_sync(0xffffffffu, err, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = err;
    __syncthreads();
    if (threadIdx.x == 0) {
      int tot = 0;
      for (int i = 0; i < (int)(blockDim.x >> 5); ++i) tot += red[i];
      unsigned long long* s = sums + 3 * (f / batch);
      atomicAdd(s + 0, (unsigned long long)tot);
      atomicAdd(s + 1, tot ? 1ull : 0ull);
      atomicAdd(s + 2, (unsigned long long)iters[f]);
    }
    __syncthreads();
  }
}

// ---- decode records (cli.py:180-183): packbits(hard) | min(iters,255) | conv ---------
__global__ void pack_records_kernel(const uint8_t* hard_packed, const int32_t* iters, const uint8_t* conv,
                                    int64_t w, int32_t nbytes, uint8_t* out) {
  const int64_t rec = nbytes + 2, total = w * rec;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t cw = o / rec;
    const int b = (int)(o - cw * rec);
    uint8_t v;
    if (b < nbytes) v = hard_packed[cw * nbytes + b];
    else if (b == nbytes) v = (uint8_t)(iters[cw] > 255 ? 255 : (iters[cw] < 0 ? 0 : iters[cw]));
    else v = conv[cw] ? 1 : 0;
    out[o] = v;
  }
}

// ---- launchers -------------------------------------------------------------------
static unsigned grid_for(int64_t items, int threads) {
  const int sms = device_sm_count();
  const int64_t want = (items + threads - 1) / threads, cap = (int64_t)sms * 16;
  return (unsigned)(want < 1 ? 1 : (want < cap ? want : cap));
}

cudaError_t launch_frames_info(uint64_t seed, uint32_t point, int64_t frame0, int64_t w, int32_t k, uint8_t* info,
                               cudaStream_t s) {
  if (w <= 0) return cudaSuccess;
  frames_info_kernel<<<grid_for(w * ((k + 127) / 128), 256), 256, 0, s>>>(seed, point, frame0, w, k, info);
  return cudaGetLastError();
}

cudaError_t launch_encode_array(const EncodeArgs& a, cudaStream_t s) {
  if (a.w <= 0) return cudaSuccess;
  const int k = (a.nb - a.mb) * a.z;
  const size_t smem = (size_t)k + (size_t)a.mb * a.z + a.z;
  cudaError_t e = ensure_dyn_smem((const void*)encode_array_kernel, smem);
  if (e != cudaSuccess) return e;
  const int threads = a.z >= 256 ? 256 : (a.z + 31) / 32 * 32;
  const int sms = device_sm_count();
  const int64_t grid = a.w < (int64_t)sms * 32 ? a.w : (int64_t)sms * 32;
  encode_array_kernel<<<(unsigned)grid, threads, smem, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_channel(const ChannelArgs& a, cudaStream_t s) {
  if (a.w <= 0) return cudaSuccess;
  const unsigned g = grid_for(a.w * (int64_t)(a.n >> 1), 256);
  if (a.noise) {
    if (a.q_lim > 0) channel_kernel<true, true><<<g, 256, 0, s>>>(a);
    else channel_kernel<true, false><<<g, 256, 0, s>>>(a);
  } else {
    if (a.q_lim > 0) channel_kernel<false, true><<<g, 256, 0, s>>>(a);
    else channel_kernel<false, false><<<g, 256, 0, s>>>(a);
  }
  return cudaGetLastError();
}

cudaError_t launch_quantize(const float* x, int64_t count, double scale, double lim, int16_t* out, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  quantize_kernel<<<grid_for(count, 256), 256, 0, s>>>(x, count, scale, lim, out);
  return cudaGetLastError();
}

cudaError_t launch_count_errors(const uint8_t* hard, int32_t packed, const uint8_t* info, const int32_t* iters,
                                int64_t w, int32_t n, int32_t k, int32_t batch, unsigned long long* sums,
                                cudaStream_t s) {
  const int64_t nbatch = (w + batch - 1) / batch;
  cudaError_t e = cudaMemsetAsync(sums, 0, (size_t)nbatch * 3 * sizeof(unsigned long long), s);
  if (e != cudaSuccess || w <= 0) return e;
  const int sms = device_sm_count();
  const int64_t grid = w < (int64_t)sms * 16 ? w : (int64_t)sms * 16;
  count_errors_kernel<<<(unsigned)grid, 128, 0, s>>>(hard, packed, info, iters, w, n, k, batch, sums);
  return cudaGetLastError();
}

cudaError_t launch_pack_records(const uint8_t* hard_packed, const int32_t* iters, const uint8_t* conv, int64_t w,
                                int32_t nbytes, uint8_t* out, cudaStream_t s) {
  if (w <= 0) return cudaSuccess;
  pack_records_kernel<<<grid_for(w * (nbytes + 2), 256), 256, 0, s>>>(hard_packed, iters, conv, w, nbytes, out);
  return cudaGetLastError();
}

}  // namespace qcb
