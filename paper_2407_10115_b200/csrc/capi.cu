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

}  // namespace dffm

extern "C" {

int dffm_abi_version(void) { return 1; }

const char* dffm_last_error(void) { return dffm::g_err; }

int dffm_device_sm_count(int device) {
  int v = 0;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
  return v;
}

}  // extern "C"
