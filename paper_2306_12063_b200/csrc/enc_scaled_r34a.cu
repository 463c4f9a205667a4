// enc_scaled_r34a.cu -- compile-time-shift bit-granular encoders (encode_common.cuh)
// for the WiMAX r34a structure at every scaled Z = 24..92 (one translation unit
// per structure keeps the parallel build balanced).
#include "encode_common.cuh"

namespace qcb {

cudaError_t launch_zbits_scaled_r34a(const EncodeArgs& a, cudaStream_t s) {
  switch (a.z) {
#define QCB_Z(Z) \
  case Z:        \
    return launch_zbits<S_wimax_r34a, Z>(a, s);
    QCB_SCALED_Z(QCB_Z)
#undef QCB_Z
  }
  return cudaErrorNotSupported;
}

}  // namespace qcb
