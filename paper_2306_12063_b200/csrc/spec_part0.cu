// spec_part0.cu -- instantiations of the layered decoders for the
// structures with ID % 6 == 0 (see decode_spec.cu): float32 (register or
// TMEM messages) and int16 (two codewords per thread), each for the native
// Z / shifts and for runtime Z, with and without early termination.
#include "decode_pair16.cuh"
#include "decode_tmem.cuh"

namespace qcb {

template <class S>
static cudaError_t launch_f32(const SpecArgs& a, cudaStream_t s) {
  if (a.tmem_cols > 0) {
    if (a.native)
      return a.early_term ? launch_tmem<S, ArithF32, S::Z0, true>(a, s) : launch_tmem<S, ArithF32, S::Z0, false>(a, s);
    return a.early_term ? launch_tmem<S, ArithF32, 0, true>(a, s) : launch_tmem<S, ArithF32, 0, false>(a, s);
  }
  if (a.native)
    return a.early_term ? launch_layered<S, ArithF32, S::Z0, true>(a, s) : launch_layered<S, ArithF32, S::Z0, false>(a, s);
  return a.early_term ? launch_layered<S, ArithF32, 0, true>(a, s) : launch_layered<S, ArithF32, 0, false>(a, s);
}

template <class S>
static cudaError_t launch_i16(const SpecArgs& a, cudaStream_t s) {
  if (a.native)
    return a.early_term ? launch_pair16<S, S::Z0, true>(a, s) : launch_pair16<S, S::Z0, false>(a, s);
  return a.early_term ? launch_pair16<S, 0, true>(a, s) : launch_pair16<S, 0, false>(a, s);
}

cudaError_t launch_spec_part0(int structure_id, int elem, const SpecArgs& a, cudaStream_t s) {
#define QCB_DISPATCH(STRUCT)                                                          \
  if constexpr (STRUCT::ID % 6 == 0) {                                              \
    if (structure_id == STRUCT::ID) return elem == 4 ? launch_f32<STRUCT>(a, s) : launch_i16<STRUCT>(a, s); \
  }
  QCB_FOR_EACH_STRUCTURE(QCB_DISPATCH)
#undef QCB_DISPATCH
  return cudaErrorInvalidValue;
}

}  // namespace qcb
