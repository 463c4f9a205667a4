// decode_scaled.cuh -- the layered decoders compiled for the scaled WiMAX codes.
//
// The 802.16e codes of every length N = 24 Z (Z = 24, 28, ..., 92) share
// their rate's Z0 = 96 base-matrix structure; their circulant shifts are the
// standard scaling of the Z0 table (reference codebook.py:217-229,
// scale_model_matrix).  Each (structure, Z) gets its own instantiation of the
// native kernels with Z and the scaled shifts as compile-time constants
// (zshift in common.cuh): every cell offset and wrap threshold is an
// immediate, as for the 18 native codes, where the runtime-Z kernels read
// both from the parameter block (one more integer op per edge, runtime row
// mapping).  capi.cu routes a code here after spec_is_scaled has checked its
// table really is that scaling; any other shift table keeps the runtime-Z
// kernels.
#pragma once
#include <utility>

#include "decode_pair16.cuh"
#include "decode_tmem.cuh"

namespace qcb {

template <class S, int ZS>
inline cudaError_t launch_scaled_z(int elem, const SpecArgs& a, cudaStream_t s) {
  if (elem == 4) {
    if constexpr (S::MAXDEG >= 18) {                 // degree-20 codes may take the TMEM kernel
      if (a.tmem_cols > 0)
        return a.early_term ? launch_tmem<S, ArithF32, ZS, true>(a, s) : launch_tmem<S, ArithF32, ZS, false>(a, s);
    }
    return a.early_term ? launch_layered<S, ArithF32, ZS, true>(a, s) : launch_layered<S, ArithF32, ZS, false>(a, s);
  }
  return a.early_term ? launch_pair16<S, ZS, true>(a, s) : launch_pair16<S, ZS, false>(a, s);
}

// cudaErrorInvalidValue when z is not in Zs (the caller then takes the runtime-Z kernels)
template <class S, int... Zs>
inline cudaError_t launch_scaled_list(int z, int elem, const SpecArgs& a, cudaStream_t s,
                                      std::integer_sequence<int, Zs...>) {
  cudaError_t e = cudaErrorInvalidValue;
  ((z == Zs ? (void)(e = launch_scaled_z<S, Zs>(elem, a, s)) : void()), ...);
  return e;
}

// the two halves of the Z range, compiled in separate translation units
using ScaledZLo = std::integer_sequence<int, 24, 28, 32, 36, 40, 44, 48, 52, 56>;
using ScaledZHi = std::integer_sequence<int, 60, 64, 68, 72, 76, 80, 84, 88, 92>;

cudaError_t launch_scaled(int structure_id, int elem, const SpecArgs& a, cudaStream_t s);

}  // namespace qcb
