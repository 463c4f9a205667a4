// spec_part5.cu -- instantiations of the specialised decoder for the
// structures with ID % 6 == 5 (see decode_spec.cu).
#include "decode_f32.cuh"
#include "decode_spec.cuh"

namespace qcb {

cudaError_t launch_spec_part5(int structure_id, int elem, const SpecArgs& a, cudaStream_t s) {
#define QCB_DISPATCH(STRUCT)                                                                \
  if constexpr (STRUCT::ID % 6 == 5) {                                                   \
    if (structure_id == STRUCT::ID) {                                                      \
      if (elem == 4) {                                                                    \
        if (a.z == STRUCT::Z0)                                                            \
          return a.early_term ? launch_f32<STRUCT, STRUCT::Z0, true>(a, s)                \
                              : launch_f32<STRUCT, STRUCT::Z0, false>(a, s);              \
        return a.early_term ? launch_f32<STRUCT, 0, true>(a, s)                           \
                            : launch_f32<STRUCT, 0, false>(a, s);                         \
      }                                                                                   \
      return a.early_term ? launch_one<STRUCT, I16Pair, true>(a, s)                         \
                          : launch_one<STRUCT, I16Pair, false>(a, s);                       \
    }                                                                                      \
  }
  QCB_FOR_EACH_STRUCTURE(QCB_DISPATCH)
#undef QCB_DISPATCH
  return cudaErrorInvalidValue;
}

}  // namespace qcb
