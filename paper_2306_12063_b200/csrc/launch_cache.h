// launch_cache.h -- host-side cache of per-kernel launch facts.
//
// cudaFuncGetAttributes / cudaFuncSetAttribute / cudaDeviceGetAttribute cost
// microseconds each; on small batches (BASELINE C1: an 18 us kernel) doing them
// on every call left the GPU idle between steps.  They are queried once per
// (kernel, device) and remembered here.
#pragma once
#include <cuda_runtime.h>

#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>

namespace qcb {

struct KernelFacts {
  cudaFuncAttributes attr{};
  bool have_attr = false;
  int dyn_smem = -1;      // largest MaxDynamicSharedMemorySize set so far
  int occ_threads = -1, occ_smem = -1, occ = 0;   // last occupancy query
};

inline std::mutex& launch_cache_mutex() {
  static std::mutex m;
  return m;
}
inline std::map<std::pair<const void*, int>, KernelFacts>& launch_cache() {
  static std::map<std::pair<const void*, int>, KernelFacts> m;
  return m;
}

inline int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}

inline int device_sm_count() {
  static std::mutex m;
  static std::map<int, int> sms;
  const int d = current_device();
  std::lock_guard<std::mutex> lk(m);
  auto it = sms.find(d);
  if (it != sms.end()) return it->second;
  int n = 148;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d);
  sms[d] = n;
  return n;
}

// attributes of kernel k on the current device (queried once)
inline cudaError_t kernel_attributes(const void* k, cudaFuncAttributes* out) {
  const auto key = std::make_pair(k, current_device());
  std::lock_guard<std::mutex> lk(launch_cache_mutex());
  KernelFacts& f = launch_cache()[key];
  if (!f.have_attr) {
    cudaError_t e = cudaFuncGetAttributes(&f.attr, k);
    if (e != cudaSuccess) return e;
    f.have_attr = true;
  }
  *out = f.attr;
  return cudaSuccess;
}

// make sure kernel k may use `bytes` of dynamic shared memory (set once, grown on demand)
inline cudaError_t ensure_dyn_smem(const void* k, size_t bytes) {
  const auto key = std::make_pair(k, current_device());
  std::lock_guard<std::mutex> lk(launch_cache_mutex());
  KernelFacts& f = launch_cache()[key];
  if ((int)bytes <= f.dyn_smem) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) f.dyn_smem = (int)bytes;
  return e;
}

// resident CTAs per SM for (threads, dynamic smem) (queried once per shape)
inline cudaError_t kernel_occupancy(const void* k, int threads, size_t smem, int* out) {
  const auto key = std::make_pair(k, current_device());
  std::lock_guard<std::mutex> lk(launch_cache_mutex());
  KernelFacts& f = launch_cache()[key];
  if (f.occ_threads != threads || f.occ_smem != (int)smem) {
    int occ = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, threads, smem);
    if (e != cudaSuccess) return e;
    f.occ_threads = threads;
    f.occ_smem = (int)smem;
    f.occ = occ;
  }
  *out = f.occ;
  return cudaSuccess;
}


}  // namespace qcb
