// kernels.h -- internal launch interface between the C-ABI layer (capi.cu)
// and the device kernels.  Not part of the public ABI (that is include/qcb200.h).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "structures_gen.cuh"

namespace qcb {

struct GenericArgs {
  const void* llr;
  void* hard;
  int32_t* iters;
  uint8_t* conv;
  void* post;
  int64_t w;
  int32_t n, z, mb, max_iters, early_term, hard_packed, cw_per_cta;
  const int32_t* tier_start;  // device, mb+1
  const int32_t* ent_j;       // device, block column per nonzero entry (tier-major, ascending j)
  const int32_t* ent_e;       // device, shift per nonzero entry
};

size_t generic_smem_bytes(int cw_per_cta, int n, int m, int elem);
cudaError_t launch_generic(const GenericArgs& a, int elem, cudaStream_t s);

// Specialised kernels: structure (block columns per tier) is a template
// parameter, shifts are kernel parameters.  Two codewords per thread.
struct SpecArgs {
  const void* llr;
  void* hard;
  int32_t* iters;
  uint8_t* conv;
  void* post;
  int64_t w;
  int32_t n, z, max_iters, early_term, hard_packed;
  int32_t pairs;   // codewords per CTA
  int32_t tmem_cols;  // TMEM columns per CTA (TMEM-resident message kernel), 0 = register kernel
  int32_t native;     // 1: z == S::Z0 and shifts == S::SHIFT0 (compile-time shift kernel)
  int32_t scaled;     // 1: WiMAX structure at z in 24..92 with the 802.16e-scaled shifts
                      //    (compile-time kernel for that z, decode_scaled.cuh)
  uint32_t k_one, k_sign, k_shr, k_neg1;  // 1, 2^31, 2^31+1, -1: IMAD multipliers kept out of ptxas' reach
  uint32_t k_lane1;   // 0x00010001 (16x2 lane constant)
  int32_t pair16;     // int16 only: 1 = two codewords per thread in 16x2 lanes (pairs = codeword pairs per CTA)
  int32_t dbg_inject; // debug builds only (QCB_DEBUG_CHECKS): 1 = make one out-of-bounds shared access (negative control)
  int32_t off[kMaxStructEntries];  // per entry: e*RS + j*ES (bytes, relative to the thread's row)
  int32_t thr[kMaxStructEntries];  // per entry: Z - e (row r wraps when r >= thr)
};

// returns cudaErrorInvalidValue if no specialised kernel exists for (structure, elem)
cudaError_t launch_spec(int structure_id, int elem, const SpecArgs& a, cudaStream_t s);
void spec_plan(int structure_id, int elem, int z, int native, int64_t w, int32_t* cw_per_cta, int32_t* tmem_cols,
               int32_t* pair16);
// true when (z, tier-major shifts) equal the structure's native Z0 / SHIFT0 tables
bool spec_is_native(int structure_id, int z, const int32_t* ent_e, int ne);
// a WiMAX structure whose shifts are the standard scaling of its Z0 = 96 table to z
bool spec_is_scaled(int structure_id, int z, const int32_t* ent_e, int ne);

// Packed direct encoder (encoder.py:166-199), byte-aligned Z.
struct EncodeArgs {
  const uint8_t* info;   // W x K/8
  uint8_t* cw;           // W x N/8
  int64_t w;
  int32_t mb, nb, z, hb_shift;
  int32_t native;           // 1: shifts are the structure's native SHIFT0 at Z0
  int32_t scaled;           // 1: WiMAX structure, shifts = the 802.16e scaling of SHIFT0 to z
  int32_t shifts[12 * 24];  // mb x nb, -1 = zero block
};
// structure_id: index into kStructureMasks, -1 = generic
cudaError_t launch_encode_packed(const EncodeArgs& a, int structure_id, cudaStream_t s);

// ---- channel / waterfall / records (channel.cu) -----------------------------------
struct ChannelArgs {
  const uint8_t* bits;     // W x N codeword bits, one per byte
  const double* noise;     // W x N standard normal samples, or NULL: device Philox stream
  void* llr;               // W x N float32 (q_lim == 0) or int16
  int64_t w;
  int32_t n;
  uint32_t point;
  int64_t frame0;
  uint64_t seed;
  double sqrt_sigma2, two_over_sigma2;   // math.sqrt(sigma2), 2.0 / sigma2 (host-computed, as the reference)
  double q_scale, q_lim;                 // lim / l_clip and lim (q_lim == 0: float32 LLRs out)
};
cudaError_t launch_frames_info(uint64_t seed, uint32_t point, int64_t frame0, int64_t w, int32_t k, uint8_t* info,
                               cudaStream_t s);
cudaError_t launch_encode_array(const EncodeArgs& a, cudaStream_t s);
cudaError_t launch_channel(const ChannelArgs& a, cudaStream_t s);
cudaError_t launch_quantize(const float* x, int64_t count, double scale, double lim, int16_t* out, cudaStream_t s);
cudaError_t launch_count_errors(const uint8_t* hard, int32_t packed, const uint8_t* info, const int32_t* iters,
                                int64_t w, int32_t n, int32_t k, int32_t batch, unsigned long long* sums,
                                cudaStream_t s);
cudaError_t launch_pack_records(const uint8_t* hard_packed, const int32_t* iters, const uint8_t* conv, int64_t w,
                                int32_t nbytes, uint8_t* out, cudaStream_t s);

}  // namespace qcb
