// decode_spec.cu -- host-side dispatch to the specialised layered decoders.
// The kernel template lives in decode_layered.cuh; its 18 structures x
// {float32, int16} x {native Z, runtime Z} x {early termination on, off}
// instantiations are split over spec_part{0..5}.cu so they compile in parallel.
#include "decode_layered.cuh"

namespace qcb {

cudaError_t launch_spec_part0(int, int, const SpecArgs&, cudaStream_t);
cudaError_t launch_spec_part1(int, int, const SpecArgs&, cudaStream_t);
cudaError_t launch_spec_part2(int, int, const SpecArgs&, cudaStream_t);
cudaError_t launch_spec_part3(int, int, const SpecArgs&, cudaStream_t);
cudaError_t launch_spec_part4(int, int, const SpecArgs&, cudaStream_t);
cudaError_t launch_spec_part5(int, int, const SpecArgs&, cudaStream_t);

cudaError_t launch_spec(int structure_id, int elem, const SpecArgs& a, cudaStream_t s) {
  switch (structure_id % 6) {
    case 0: return launch_spec_part0(structure_id, elem, a, s);
    case 1: return launch_spec_part1(structure_id, elem, a, s);
    case 2: return launch_spec_part2(structure_id, elem, a, s);
    case 3: return launch_spec_part3(structure_id, elem, a, s);
    case 4: return launch_spec_part4(structure_id, elem, a, s);
    default: return launch_spec_part5(structure_id, elem, a, s);
  }
}

int spec_row_stride_bytes(int elem) {
  return elem == 4 ? row_stride_bytes<ArithF32>() : row_stride_bytes<ArithI16>();
}

int spec_cw_per_cta(int z, int64_t w) { return layered_cw_per_cta(z, w); }

}  // namespace qcb
