// common.cuh -- shared device definitions for the qcb200 QC-LDPC kernels (sm_100a).
//
// Arithmetic traits reproduce the reference kernels' per-edge operations
// bit for bit (/root/reference/pkg/src/qcldpc/_kernels.py:61-84 float32,
// :147-170 int16 with two's-complement wrap after every op).
#pragma once
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

#include "debug_checks.cuh"
#include "structures_gen.cuh"

namespace qcb {

constexpr int kMaxDeg = 32;          // sign bitmap width (reference decoder.py:185-186)
constexpr int kMaxGenericTiers = 256;
// Shared-memory posterior layout of the specialised decoders: cell (c, j),
// i.e. bit n = j Z + c of a codeword, at byte 4 n of the codeword's block --
// the codeword's own bit order, so the prologue / epilogue are streaming
// copies.  A tier's Z rows read cells (c = (r + e) mod Z, j): consecutive c,
// consecutive words, one bank each (the same property the previous [c][j]
// layout with an odd row stride had).  Every standard structure has nb = 24.
constexpr int kCellBytes = 4;
constexpr int kStdNb = 24;
__host__ __device__ constexpr int cw_block_bytes(int z) { return kStdNb * z * kCellBytes; }   // multiple of 16

// Circulant shift of structure entry e at lifting size Z: the structure's own
// table at Z0, else the 802.16e scaling of the Z0 = 96 WiMAX table
// (reference codebook.py:217-229 / scale_model_matrix: p mod Z for rate 2/3A,
// floor(p Z / 96) otherwise; p <= 0 unchanged).  Used by the encoders and by
// the decoders compiled for a scaled WiMAX code's Z.
template <class S, int Z>
constexpr int zshift(int e) {
  const int p = S::SHIFT0[e];
  if (Z == S::Z0 || p <= 0) return p;
  return std::is_same<S, S_wimax_r23a>::value ? p % Z : p * Z / 96;
}

// ---- exact float32 helpers -------------------------------------------------
__device__ __forceinline__ float f_inf() { return __int_as_float(0x7f800000); }
__device__ __forceinline__ float f_sub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float f_add(float a, float b) { return __fadd_rn(a, b); }
// NaN-propagating max: max.NaN(nm1, NaN) = NaN so that min(nm2, .) keeps nm2,
// matching the reference's `elif a < nm2` (false for NaN).
__device__ __forceinline__ float f_max_nan(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}

// ---- int16 wrap helpers -----------------------------------------------------
// Wrap to int16 and sign-extend.  Done in PTX on purpose: NVVM folds C++
// narrowing casts of out-of-range values using value-range facts (e.g. it
// turns `(int16_t)abs(x) < 32767` into `abs(x) != 32767`, losing the
// abs(-32768) == -32768 wrap the reference relies on).
__device__ __forceinline__ int sext16(int x) {
  int r;
  asm("cvt.s32.s16 %0, %1;" : "=r"(r) : "r"(x));
  return r;
}

// Magnitude "key": a = |wrap16(zz)| lies in [0, 32768]; the reference keeps it
// as int16, so 32768 wraps to -32768 and sorts below everything.
// key = a ^ 0x8000 maps that signed-int16 order onto unsigned [0, 0xFFFF].
__device__ __forceinline__ unsigned i16_key_of(int zz_wrapped) {
  return (unsigned)abs(zz_wrapped) ^ 0x8000u;
}
// key -> magnitude value (as a 32-bit int; 32768 stands for int16 -32768,
// harmless because every use is followed by a wrapped add/sub or a 16-bit store)
__device__ __forceinline__ int i16_val_of_key(unsigned k) { return (int)(k ^ 0x8000u); }
constexpr unsigned kI16KeyInit = 32767u ^ 0x8000u;  // nm1 = nm2 = 32767 (ref _kernels.py:142-143)

}  // namespace qcb
