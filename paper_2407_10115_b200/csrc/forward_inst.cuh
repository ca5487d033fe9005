// Per-storage-type instantiation of K1 (included once per forward_<dtype>.cu
// so the three table types compile in parallel).
#pragma once

#include <mutex>
#include <unordered_map>

#include "forward_kernel.cuh"

namespace dffm {

using FwdKernel = void (*)(FwdParams);

template <typename T>
static FwdKernel select_fwd(int K, int MU) {
#define DFFM_SEL(KK)                                   \
  if (K == KK) {                                       \
    if (MU == 1) return fwd_kernel<KK, 1, T>;          \
    if (MU == 4) return fwd_kernel<KK, 4, T>;          \
    return fwd_kernel<KK, 0, T>;                       \
  }
  DFFM_SEL(4)
  DFFM_SEL(8)
  DFFM_SEL(16)
  DFFM_SEL(32)
  DFFM_SEL(0)
#undef DFFM_SEL
  return nullptr;
}

template <typename T>
int launch_forward_t(const FwdParams& p, int K, int MU, int smem, cudaStream_t s) {
  FwdKernel kern = select_fwd<T>(K, MU);
  if (!kern) { set_error("no forward kernel for k=%d", p.k); return DFFM_SIZING; }
  static std::mutex mu;
  static std::unordered_map<uint64_t, int> occ_cache;  // (kernel, smem, device) -> blocks/SM
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t key = ((uint64_t)(uintptr_t)kern * 1315423911u) ^ ((uint64_t)smem << 8) ^ dev;
  int occ = 0;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = occ_cache.find(key);
    if (it != occ_cache.end()) {
      occ = it->second;
    } else {
      DFFM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem),
                    "cudaFuncSetAttribute(forward)");
      DFFM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, FWD_THREADS, smem),
                    "occupancy(forward)");
      if (occ < 1) occ = 1;
      occ_cache[key] = occ;
    }
  }
  const int64_t ntiles = (p.n + p.TE - 1) / p.TE;
  const int64_t grid = std::min<int64_t>(ntiles, (int64_t)sm_count_current() * occ);
  kern<<<(unsigned)grid, FWD_THREADS, smem, s>>>(p);
  DFFM_CUDA_TRY(cudaGetLastError(), "launch(forward)");
  return DFFM_OK;
}

template int launch_forward_t<DFFM_INST_T>(const FwdParams&, int, int, int, cudaStream_t);

}  // namespace dffm
