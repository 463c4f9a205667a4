// spec_part5.cu -- instantiations of the layered decoder for the
// structures with ID % 6 == 5 (see decode_spec.cu / decode_layered.cuh).
#include "decode_pair16.cuh"
#include "decode_tmem.cuh"

namespace qcb {

template <class S, class A>
static cudaError_t launch_arith(const SpecArgs& a, cudaStream_t s) {
  if constexpr (A::kElem == 2) {
    if (a.pair16) {
      if (a.native)
        return a.early_term ? launch_pair16<S, S::Z0, true>(a, s) : launch_pair16<S, S::Z0, false>(a, s);
      return a.early_term ? launch_pair16<S, 0, true>(a, s) : launch_pair16<S, 0, false>(a, s);
    }
  }
  if (a.tmem_cols > 0) {
    if (a.native)
      return a.early_term ? launch_tmem<S, A, S::Z0, true>(a, s) : launch_tmem<S, A, S::Z0, false>(a, s);
    return a.early_term ? launch_tmem<S, A, 0, true>(a, s) : launch_tmem<S, A, 0, false>(a, s);
  }
  if (a.native)
    return a.early_term ? launch_layered<S, A, S::Z0, true>(a, s) : launch_layered<S, A, S::Z0, false>(a, s);
  return a.early_term ? launch_layered<S, A, 0, true>(a, s) : launch_layered<S, A, 0, false>(a, s);
}

cudaError_t launch_spec_part5(int structure_id, int elem, const SpecArgs& a, cudaStream_t s) {
#define QCB_DISPATCH(STRUCT)                                                              \
  if constexpr (STRUCT::ID % 6 == 5) {                                                 \
    if (structure_id == STRUCT::ID)                                                       \
      return elem == 4 ? launch_arith<STRUCT, ArithF32>(a, s) : launch_arith<STRUCT, ArithI16>(a, s); \
  }
  QCB_FOR_EACH_STRUCTURE(QCB_DISPATCH)
#undef QCB_DISPATCH
  return cudaErrorInvalidValue;
}

}  // namespace qcb
