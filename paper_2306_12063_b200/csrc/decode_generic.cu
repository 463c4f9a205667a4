// decode_generic.cu -- layered single-scan min-sum for ANY quasi-cyclic code.
//
// Correctness path behind the specialised kernels (decode_spec.cu): runtime
// tier tables, row state in shared memory, the reference's literal
// if/elif update order.  Used for codes whose block structure is not one of
// the 18 standard base matrices (e.g. the toy codes of the reference tests)
// or whose row degree exceeds what the specialised kernels unroll.
//
// Follows /root/reference/pkg/src/qcldpc/_kernels.py:17-100 (float32) and
// :103-186 (int16).  Parallel schedule: within a tier the Z rows touch
// pairwise-disjoint columns (every circulant is a permutation), so the Z rows
// run concurrently with results identical to the reference's sequential row
// loop; tiers stay sequential (layered schedule) behind a CTA barrier.
#include "common.cuh"
#include "kernels.h"

namespace qcb {

template <typename T>
struct GenericArith;

template <>
struct GenericArith<float> {
  using Acc = float;
  __device__ static float init() { return f_inf(); }
  __device__ static float load(const float* p) { return *p; }
  __device__ static void store(float* p, float v) { *p = v; }
  __device__ static float neg(float m) { return -m; }
  __device__ static float sub(float a, float b) { return f_sub(a, b); }
  __device__ static float add(float a, float b) { return f_add(a, b); }
  __device__ static float absv(float x) { return fabsf(x); }
};

template <>
struct GenericArith<int16_t> {
  using Acc = int16_t;
  __device__ static int16_t init() { return 32767; }
  __device__ static int16_t load(const int16_t* p) { return *p; }
  __device__ static void store(int16_t* p, int16_t v) { *p = v; }
  // every op wraps through sext16 (PTX cvt), see common.cuh
  __device__ static int16_t neg(int16_t m) { return (int16_t)sext16(-(int)m); }
  __device__ static int16_t sub(int16_t a, int16_t b) { return (int16_t)sext16((int)a - (int)b); }
  __device__ static int16_t add(int16_t a, int16_t b) { return (int16_t)sext16((int)a + (int)b); }
  __device__ static int16_t absv(int16_t x) { return (int16_t)sext16(x < 0 ? -(int)x : (int)x); }
};

template <typename T>
__global__ void __launch_bounds__(256) decode_generic_kernel(GenericArgs a) {
  using A = GenericArith<T>;
  extern __shared__ __align__(16) unsigned char smem[];
  const int N = a.n, Z = a.z, MB = a.mb, M = MB * Z, G = a.cw_per_cta;
  const int64_t cw0 = (int64_t)blockIdx.x * G;
  const int gcount = (int)(a.w - cw0 < (int64_t)G ? a.w - cw0 : (int64_t)G);

  T* post = reinterpret_cast<T*>(smem);
  T* min1 = post + (size_t)G * N;
  T* min2 = min1 + (size_t)G * M;
  uint32_t* sbits = reinterpret_cast<uint32_t*>(
      (reinterpret_cast<uintptr_t>(min2 + (size_t)G * M) + 3) & ~uintptr_t(3));
  uint8_t* amin = reinterpret_cast<uint8_t*>(sbits + (size_t)G * M);
  uint8_t* sprod = amin + (size_t)G * M;
  __shared__ int s_fail[64], s_done[64], s_iters[64], s_any_active;

  const T* llr = reinterpret_cast<const T*>(a.llr) + cw0 * N;
  for (int i = threadIdx.x; i < gcount * N; i += blockDim.x) post[i] = llr[i];
  for (int i = threadIdx.x; i < G * M; i += blockDim.x) {
    min1[i] = T(0); min2[i] = T(0); sbits[i] = 0; amin[i] = 0; sprod[i] = 0;
  }
  for (int g = threadIdx.x; g < G; g += blockDim.x) {
    s_done[g] = g >= gcount; s_iters[g] = 0; s_fail[g] = 1;
  }
  __syncthreads();

  for (int k = 0; k < a.max_iters; ++k) {
    for (int t = 0; t < MB; ++t) {
      const int e0 = a.tier_start[t], deg = a.tier_start[t + 1] - e0;
      for (int idx = threadIdx.x; idx < gcount * Z; idx += blockDim.x) {
        const int g = idx / Z, r = idx - g * Z;
        if (s_done[g]) continue;
        const int m = g * M + t * Z + r;
        T* pg = post + (size_t)g * N;
        int col[kMaxDeg];
        T zrow[kMaxDeg];
        const T m1 = min1[m], m2 = min2[m];
        const int am = amin[m];
        const uint32_t sb = sbits[m];
        const uint32_t sp = sprod[m];
        T nm1 = A::init(), nm2 = A::init();
        int nam = 0;
        uint32_t nsb = 0, nsp = 0;
        for (int j = 0; j < deg; ++j) {                       // _kernels.py:61-75
          int c = r + a.ent_e[e0 + j];
          c = c >= Z ? c - Z : c;
          col[j] = a.ent_j[e0 + j] * Z + c;
          const T mag = (j == am) ? m2 : m1;
          const T lold = ((sp ^ ((sb >> j) & 1u)) == 1u) ? A::neg(mag) : mag;
          const T zz = A::sub(pg[col[j]], lold);
          zrow[j] = zz;
          const T av = A::absv(zz);
          if (av < nm1) { nm2 = nm1; nm1 = av; nam = j; }
          else if (av < nm2) { nm2 = av; }
          if (zz < T(0)) { nsb |= 1u << j; nsp ^= 1u; }
        }
        for (int j = 0; j < deg; ++j) {                       // _kernels.py:76-79
          const T mag = (j == nam) ? nm2 : nm1;
          const T lnew = ((nsp ^ ((nsb >> j) & 1u)) == 1u) ? A::neg(mag) : mag;
          pg[col[j]] = A::add(zrow[j], lnew);
        }
        min1[m] = nm1; min2[m] = nm2; amin[m] = (uint8_t)nam;
        sbits[m] = nsb; sprod[m] = (uint8_t)nsp;
      }
      __syncthreads();
    }
    // syndrome after every super-iteration (_kernels.py:85-96); without early
    // termination only the last one is observable, so it is computed once.
    const bool last = (k + 1 == a.max_iters);
    if (a.early_term || last) {
      for (int g = threadIdx.x; g < G; g += blockDim.x) s_fail[g] = 0;
      __syncthreads();
      for (int idx = threadIdx.x; idx < gcount * M; idx += blockDim.x) {
        const int g = idx / M, m = idx - g * M;
        if (s_done[g]) continue;
        const int t = m / Z, r = m - t * Z;
        const int e0 = a.tier_start[t], deg = a.tier_start[t + 1] - e0;
        const T* pg = post + (size_t)g * N;
        uint32_t par = 0;
        for (int j = 0; j < deg; ++j) {
          int c = r + a.ent_e[e0 + j];
          c = c >= Z ? c - Z : c;
          par ^= pg[a.ent_j[e0 + j] * Z + c] <= T(0);
        }
        if (par) s_fail[g] = 1;
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) s_any_active = 0;
    __syncthreads();
    for (int g = threadIdx.x; g < gcount; g += blockDim.x) {
      if (!s_done[g]) {
        s_iters[g] = k + 1;
        if (a.early_term && !s_fail[g]) s_done[g] = 1;
        else s_any_active = 1;
      }
    }
    __syncthreads();
    if (!s_any_active) break;
  }

  // outputs: hard decisions (post <= 0, _kernels.py:97-100), iterations, converged
  for (int g = threadIdx.x; g < gcount; g += blockDim.x) {
    a.iters[cw0 + g] = s_iters[g];
    a.conv[cw0 + g] = (a.max_iters > 0 && !s_fail[g]) ? 1 : 0;
  }
  if (a.hard_packed) {
    const int nbytes = (N + 7) / 8;
    uint8_t* hp = reinterpret_cast<uint8_t*>(a.hard) + cw0 * nbytes;
    for (int i = threadIdx.x; i < gcount * nbytes; i += blockDim.x) {
      const int g = i / nbytes, b = i - g * nbytes;
      uint32_t byte = 0;
      for (int q = 0; q < 8; ++q) {
        const int n = b * 8 + q;
        byte = (byte << 1) | (n < N && post[(size_t)g * N + n] <= T(0) ? 1u : 0u);
      }
      hp[i] = (uint8_t)byte;
    }
  } else {
    uint8_t* h = reinterpret_cast<uint8_t*>(a.hard) + cw0 * N;
    for (int i = threadIdx.x; i < gcount * N; i += blockDim.x) h[i] = post[i] <= T(0);
  }
  if (a.post) {
    T* po = reinterpret_cast<T*>(a.post) + cw0 * N;
    for (int i = threadIdx.x; i < gcount * N; i += blockDim.x) po[i] = post[i];
  }
}

size_t generic_smem_bytes(int cw_per_cta, int n, int m, int elem) {
  size_t b = (size_t)cw_per_cta * n * elem + 2 * (size_t)cw_per_cta * m * elem;
  b = (b + 3) & ~size_t(3);
  b += (size_t)cw_per_cta * m * (4 + 1 + 1);
  return (b + 15) & ~size_t(15);
}

cudaError_t launch_generic(const GenericArgs& a, int elem, cudaStream_t s) {
  const size_t smem = generic_smem_bytes(a.cw_per_cta, a.n, a.mb * a.z, elem);
  const int64_t blocks = (a.w + a.cw_per_cta - 1) / a.cw_per_cta;
  if (blocks <= 0) return cudaSuccess;
  if (elem == 4) {
    cudaFuncSetAttribute(decode_generic_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    decode_generic_kernel<float><<<(unsigned)blocks, 256, smem, s>>>(a);
  } else {
    cudaFuncSetAttribute(decode_generic_kernel<int16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    decode_generic_kernel<int16_t><<<(unsigned)blocks, 256, smem, s>>>(a);
  }
  return cudaGetLastError();
}

}  // namespace qcb
