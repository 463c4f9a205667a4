// decode_spec.cu -- host-side dispatch to the specialised layered decoders.
// The kernel template lives in decode_layered.cuh; its 18 structures x
// {float32, int16} x {native Z, runtime Z} x {early termination on, off}
// instantiations are split over spec_part{0..5}.cu so they compile in parallel;
// the scaled WiMAX codes' per-Z instantiations are in dec_scaled_*.cu.
#include "decode_pair16.cuh"
#include "decode_tmem.cuh"

namespace qcb {

cudaError_t launch_spec_part0(int, int, const SpecArgs&, cudaStream_t);
cudaError_t launch_spec_part1(int, int, const SpecArgs&, cudaStream_t);
cudaError_t launch_spec_part2(int, int, const SpecArgs&, cudaStream_t);
cudaError_t launch_spec_part3(int, int, const SpecArgs&, cudaStream_t);
cudaError_t launch_spec_part4(int, int, const SpecArgs&, cudaStream_t);
cudaError_t launch_spec_part5(int, int, const SpecArgs&, cudaStream_t);

#ifndef QCB_SCALED_KERNELS
#define QCB_SCALED_KERNELS 1      // 0: scaled codes take the runtime-Z kernels (experiment builds skip dec_scaled_*.cu)
#endif

#if QCB_SCALED_KERNELS
#define QCB_SCALED_DECL(R) \
  cudaError_t launch_scaled_##R##_lo(int, int, const SpecArgs&, cudaStream_t); \
  cudaError_t launch_scaled_##R##_hi(int, int, const SpecArgs&, cudaStream_t);
QCB_SCALED_DECL(r12) QCB_SCALED_DECL(r23a) QCB_SCALED_DECL(r23b)
QCB_SCALED_DECL(r34a) QCB_SCALED_DECL(r34b) QCB_SCALED_DECL(r56)
#undef QCB_SCALED_DECL

// scaled WiMAX codes: the kernels compiled for their Z (decode_scaled.cuh)
cudaError_t launch_scaled(int structure_id, int elem, const SpecArgs& a, cudaStream_t s) {
  const int z = a.z;
  const bool lo = z <= 56;
#define QCB_SCALED_CASE(R, S) \
  if (structure_id == S::ID) return lo ? launch_scaled_##R##_lo(z, elem, a, s) : launch_scaled_##R##_hi(z, elem, a, s);
  QCB_SCALED_CASE(r12, S_wimax_r12)
  QCB_SCALED_CASE(r23a, S_wimax_r23a)
  QCB_SCALED_CASE(r23b, S_wimax_r23b)
  QCB_SCALED_CASE(r34a, S_wimax_r34a)
  QCB_SCALED_CASE(r34b, S_wimax_r34b)
  QCB_SCALED_CASE(r56, S_wimax_r56)
#undef QCB_SCALED_CASE
  return cudaErrorInvalidValue;
}
#else
cudaError_t launch_scaled(int, int, const SpecArgs&, cudaStream_t) { return cudaErrorInvalidValue; }
#endif

cudaError_t launch_spec(int structure_id, int elem, const SpecArgs& a, cudaStream_t s) {
  static const bool scaled_env = [] {
    const char* e = getenv("QCB_SCALED");
    return !(e && e[0] == '0');
  }();
  if (QCB_SCALED_KERNELS && scaled_env && a.scaled && !a.native) {
    const cudaError_t e = launch_scaled(structure_id, elem, a, s);
    if (e != cudaErrorInvalidValue) return e;
  }
  switch (structure_id % 6) {
    case 0: return launch_spec_part0(structure_id, elem, a, s);
    case 1: return launch_spec_part1(structure_id, elem, a, s);
    case 2: return launch_spec_part2(structure_id, elem, a, s);
    case 3: return launch_spec_part3(structure_id, elem, a, s);
    case 4: return launch_spec_part4(structure_id, elem, a, s);
    default: return launch_spec_part5(structure_id, elem, a, s);
  }
}



// Choose between the register-resident and the TMEM-resident message store.
// QCB_TMEM=0/1 forces one (benchmarks); default: TMEM when it keeps more
// codewords resident per SM.
bool spec_is_native(int structure_id, int z, const int32_t* ent_e, int ne) {
  bool native = false;
#define QCB_NAT(STRUCT)                                                   \
  if (structure_id == STRUCT::ID && z == STRUCT::Z0 && ne == STRUCT::NE) { \
    native = true;                                                        \
    for (int i = 0; i < ne; ++i) native = native && ent_e[i] == STRUCT::SHIFT0[i]; \
  }
  QCB_FOR_EACH_STRUCTURE(QCB_NAT)
#undef QCB_NAT
  return native;
}

bool spec_is_scaled(int structure_id, int z, const int32_t* ent_e, int ne) {
  bool scaled = false;
#define QCB_SCL(STRUCT)                                                                 \
  if (structure_id == STRUCT::ID && STRUCT::Z0 == 96 && z >= 24 && z <= 96 && z % 4 == 0 && \
      ne == STRUCT::NE) {                                                                \
    scaled = true;                                                                       \
    for (int i = 0; i < ne; ++i) {                                                       \
      const int p = STRUCT::SHIFT0[i];                                                   \
      const int want = p <= 0 ? p : (STRUCT::ID == S_wimax_r23a::ID ? p % z : p * z / 96); \
      scaled = scaled && ent_e[i] == want;                                               \
    }                                                                                    \
  }
  QCB_FOR_EACH_STRUCTURE(QCB_SCL)
#undef QCB_SCL
  return scaled;
}

void spec_plan(int structure_id, int elem, int z, int native, int64_t w, int32_t* cw_per_cta, int32_t* tmem_cols,
               int32_t* pair16) {
  int ne = 0, maxdeg = 0;
  *pair16 = 0;

  if (elem == 2) {                          // int16: two codewords per thread in 16x2 lanes
    *pair16 = 1;
    *cw_per_cta = 1;                        // planned at launch from the kernel's registers
    *tmem_cols = 0;
    return;
  }
#define QCB_NE(STRUCT) if (structure_id == STRUCT::ID) { ne = STRUCT::NE; maxdeg = STRUCT::MAXDEG; }
  QCB_FOR_EACH_STRUCTURE(QCB_NE)
#undef QCB_NE
  const int regs_reg = ne + 52 + (elem == 2 ? maxdeg : 0);
  const int reg_g = layered_cw_per_cta(z, w, regs_reg, elem);
  *cw_per_cta = reg_g;
  *tmem_cols = 0;
  static const int tmem_env = [] {
    const char* e = getenv("QCB_TMEM");
    return e ? (e[0] == '0' ? 0 : (e[0] == '1' ? 1 : -1)) : -1;
  }();
  if (tmem_env == 0) return;
  const int regs_tm = QCB_TM_REG_BASE + (elem == 2 ? 6 : 5) * maxdeg;
  const int smem_cw = cw_block_bytes(z);
  int cols = 0;
  const int g = tmem_plan(z, ne, (regs_tm + 7) / 8 * 8, smem_cw, w, &cols);
  if (g <= 0) return;
  // measured on B200 (round 1, tools/exp/tmem_ab.py, f32 coded Gb/s register / TMEM):
  // row degree 20 gains (Wi-Fi 1944 R5/6 43.2 / 46.5, WiMAX 2304 R5/6 52.7 / 55.8,
  // WiMAX 1152 R5/6 34.7 / 43.7); degree 22 loses (Wi-Fi 648 R5/6 39.7 / 35.4,
  // Wi-Fi 1296 R5/6 43.8 / 33.5) and so do the low-degree codes (5-6 %):
  // TMEM reads (64 B/clk/SM) only pay where the register kernel is starved
  // Re-measured at the end of round 1 (3-input minima, register caps at the
  // sub-partition boundary): the register kernel now wins on the native
  // degree-20 codes (Wi-Fi 1944 R5/6 59.6 vs 55.7, WiMAX 2304 R5/6 70.0 vs
  // 66.0 Gb/s, tools/exp/deg20_ab.sh); TMEM stays preferred for the scaled
  // (runtime-Z) degree-20 codes with Z >= 40, where it measured ahead
  // (tools/exp/tmem_scaled_ab.sh: WiMAX 1152 R5/6 54.4 vs 52.5, 1728 R5/6
  // 51.7 vs 45.5; 576 R5/6 48.4 vs 51.7 keeps the register kernel).
#ifndef QCB_TMEM_SCALED
#define QCB_TMEM_SCALED 1
#endif
  // compile-time kernels (native or scaled Z): TMEM where the per-code sweep
  // measured it ahead (scaled_plan_gen.h: WiMAX R5/6 at Z = 68..76)
  const ScaledPlan* sp = native ? scaled_plan(structure_id, elem, z) : nullptr;
  const bool prefer = elem == 4 && maxdeg >= 18 && maxdeg <= 20 && QCB_TMEM_SCALED &&
                      (native ? (sp && sp->tmem) : z >= 40);
  if (tmem_env == 1 || prefer) {
    *cw_per_cta = g;
    *tmem_cols = cols;
  }
}

}  // namespace qcb
