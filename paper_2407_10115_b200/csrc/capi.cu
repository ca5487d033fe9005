#include <atomic>
// Library-wide C ABI helpers: error text, device queries.
#include <stdarg.h>
#include <stdio.h>

#include <mutex>
#include <unordered_map>

#include "common.cuh"

namespace dffm {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_fail(cudaError_t e, const char* what) {
  set_error("%s: %s", what, cudaGetErrorString(e));
  return DFFM_CUDA;
}

static std::mutex g_mu;
static std::unordered_map<int, int> g_sms, g_smem;

static std::atomic<long long> g_launches{0};
void note_launches(int k) { g_launches.fetch_add(k, std::memory_order_relaxed); }

int sm_count_current() {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_sms.find(dev);
  if (it != g_sms.end()) return it->second;
  int v = 0;
  cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
  g_sms[dev] = v;
  return v;
}

int max_smem_optin_current() {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_smem.find(dev);
  if (it != g_smem.end()) return it->second;
  int v = 0;
  cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  g_smem[dev] = v;
  return v;
}

int kernel_occupancy(const void* func, int threads, int smem, int* occ) {
  static std::mutex mu;
  static std::unordered_map<uint64_t, int> attr_set, occ_cache;
  int dev = 0;
  cudaGetDevice(&dev);
  const int smax = max_smem_optin_current();
  std::lock_guard<std::mutex> lk(mu);
  const uint64_t fkey = ((uint64_t)(uintptr_t)func << 8) ^ (uint64_t)dev;
  if (!attr_set.count(fkey)) {
    cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, smax);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
    attr_set[fkey] = 1;
  }
  const uint64_t okey = fkey * 1315423911ull ^ ((uint64_t)smem << 40) ^ (uint64_t)threads;
  auto it = occ_cache.find(okey);
  if (it != occ_cache.end()) {
    *occ = it->second;
    return DFFM_OK;
  }
  int v = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, func, threads, smem);
  if (e != cudaSuccess) return cuda_fail(e, "occupancy");
  if (v < 1) v = 1;
  occ_cache[okey] = v;
  *occ = v;
  return DFFM_OK;
}

}  // namespace dffm

extern "C" {

int dffm_abi_version(void) { return 1; }

#ifndef DFFM_SRC_DIGEST
#define DFFM_SRC_DIGEST "unknown"
#endif
// sha256 (first 16 hex) of the sources this library was built from (Makefile):
// deterministic, unlike the .so bytes, so a committed ncu capture can be tied to it
const char* dffm_build_id(void) { return DFFM_SRC_DIGEST; }

const char* dffm_last_error(void) { return dffm::g_err; }

int dffm_device_sm_count(int device) {
  int v = 0;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
  return v;
}

}  // extern "C"

extern "C" int64_t dffm_launch_count(void) { return (int64_t)dffm::g_launches.load(); }
