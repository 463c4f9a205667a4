// debug_checks.cuh -- device-side checks for a debug build of libqcb200
// (QCB_DEBUG_CHECKS=1; tools/debug_checks.sh builds lib_debug.so and runs the
// GPU tests and tools/sanitize_cases.py against it).  compute-sanitizer is
// closed on this GPU pool, so the decoders check their own invariants:
//   * every shared-memory access made through the cell / table / I/O helpers
//     lies inside the CTA's dynamic shared memory and is naturally aligned
//     (bounds of the posterior blocks, address tables, ET snapshot block);
//   * dynamic shared memory is poisoned (0x5A5A5A5A) before the prologue, so
//     a cell read before it is written changes the decode and shows up as a
//     mismatch against the CPU oracle (initcheck's question);
//   * a CTA never starts past the batch (global row bounds of the prologue /
//     epilogue chunk).
// A failed check prints the site and traps (the launch then fails with
// cudaErrorLaunchFailure / an illegal-instruction error, surfacing in the
// calling test).  With QCB_DEBUG_CHECKS=0 (the product build) every helper
// compiles to nothing.
#pragma once
#include <cstdint>
#include <cstdio>

#ifndef QCB_DEBUG_CHECKS
#define QCB_DEBUG_CHECKS 0
#endif

namespace qcb {

extern __shared__ __align__(16) unsigned char qcb_dbg_dyn[];

__device__ __forceinline__ void dbg_smem(uint32_t a, uint32_t bytes, int site) {
#if QCB_DEBUG_CHECKS
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(qcb_dbg_dyn);
  uint32_t size;
  asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(size));
  if (a < base || a + bytes > base + size || (a & (bytes - 1u)) != 0u) {
    printf("qcb debug: shared access site %d addr 0x%x bytes %u outside [0x%x, 0x%x) block %d thread %d\n", site, a,
           bytes, base, base + size, (int)blockIdx.x, (int)threadIdx.x);
    __trap();
  }
#else
  (void)a; (void)bytes; (void)site;
#endif
}

// fill the dynamic shared memory with a poison pattern (call before the prologue)
__device__ __forceinline__ void dbg_poison_smem() {
#if QCB_DEBUG_CHECKS
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(qcb_dbg_dyn);
  uint32_t size;
  asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(size));
  for (uint32_t o = 4u * threadIdx.x; o + 4u <= size; o += 4u * blockDim.x)
    asm volatile("st.shared.b32 [%0], %1;" ::"r"(base + o), "r"(0x5A5A5A5Au) : "memory");
  __syncthreads();
#endif
}

// negative control: with QCB_DEBUG_INJECT set, the decoders make one access
// past their dynamic shared memory, which the bounds check must catch
__device__ __forceinline__ void dbg_inject_probe(int inject, uint32_t sbase) {
#if QCB_DEBUG_CHECKS
  uint32_t size;
  asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(size));
  if (inject && threadIdx.x == 0) dbg_smem(sbase + size, 4, 99);
#else
  (void)inject; (void)sbase;
#endif
}

__device__ __forceinline__ void dbg_check(bool ok, int site) {
#if QCB_DEBUG_CHECKS
  if (!ok) {
    printf("qcb debug: check %d failed, block %d thread %d\n", site, (int)blockIdx.x, (int)threadIdx.x);
    __trap();
  }
#else
  (void)ok; (void)site;
#endif
}

}  // namespace qcb
