// dec_scaled_r23a_hi.cu -- S_wimax_r23a decoders for the scaled Z of ScaledZHi
// (decode_scaled.cuh); one translation unit per structure and Z half so they
// compile in parallel.
#include "decode_scaled.cuh"

namespace qcb {

cudaError_t launch_scaled_r23a_hi(int z, int elem, const SpecArgs& a, cudaStream_t s) {
  return launch_scaled_list<S_wimax_r23a>(z, elem, a, s, ScaledZHi{});
}

}  // namespace qcb
