// decode_spec.cu -- host-side dispatch to the specialised decoders.
// The kernel template lives in decode_spec.cuh; its 18 structures x 2
// arithmetics x 2 (early termination on/off) instantiations are split over
// spec_part{0..5}.cu so they compile in parallel.
#include "decode_f32.cuh"
#include "decode_spec.cuh"

namespace qcb {

constexpr int kSpecParts = 6;
cudaError_t launch_spec_part0(int, int, const SpecArgs&, cudaStream_t);
cudaError_t launch_spec_part1(int, int, const SpecArgs&, cudaStream_t);
cudaError_t launch_spec_part2(int, int, const SpecArgs&, cudaStream_t);
cudaError_t launch_spec_part3(int, int, const SpecArgs&, cudaStream_t);
cudaError_t launch_spec_part4(int, int, const SpecArgs&, cudaStream_t);
cudaError_t launch_spec_part5(int, int, const SpecArgs&, cudaStream_t);

cudaError_t launch_spec(int structure_id, int elem, const SpecArgs& a, cudaStream_t s) {
  switch (structure_id % kSpecParts) {
    case 0: return launch_spec_part0(structure_id, elem, a, s);
    case 1: return launch_spec_part1(structure_id, elem, a, s);
    case 2: return launch_spec_part2(structure_id, elem, a, s);
    case 3: return launch_spec_part3(structure_id, elem, a, s);
    case 4: return launch_spec_part4(structure_id, elem, a, s);
    default: return launch_spec_part5(structure_id, elem, a, s);
  }
}

int spec_row_stride_bytes(int elem) { return elem == 4 ? kRsF32 : kRowStrideUnits * I16Pair::ES; }

int spec_group_per_cta(int elem, int z) {
  if (elem == 4) return f32_cw_per_cta(z);
  // pick pairs so that pairs*Z fills whole warps well, 96..384 threads
  int best = 1;
  double best_eff = 0.0;
  for (int p = 1; p <= kMaxPairsPerCta; ++p) {
    const int thr = p * z;
    if (thr > kSpecMaxThreads) break;
    const int padded = (thr + 31) / 32 * 32;
    double eff = (double)thr / padded;
    if (thr < 96) eff *= 0.9;  // too few warps per CTA to hide barrier cost
    if (eff > best_eff + 1e-9) { best_eff = eff; best = p; }
  }
  return best;
}

}  // namespace qcb
