// Per-storage-type instantiation of K1 (included once per forward_<dtype>.cu
// so the three table types compile in parallel).
#pragma once

#include <mutex>
#include <unordered_map>

#include "forward_kernel.cuh"
#include "forward_ws.cuh"
#include "forward_rsw.cuh"

namespace dffm {

using FwdKernel = void (*)(FwdParams);

template <typename T>
static FwdKernel select_fwd(int K, int MU) {
#define DFFM_SEL(KK)                                   \
  if (K == KK) {                                       \
    if (MU == 1) return fwd_kernel<KK, 1, T>;          \
    if (MU == 2) return fwd_kernel<KK, 2, T>;          \
    if (MU == 3) return fwd_kernel<KK, 3, T>;          \
    if (MU == 4) return fwd_kernel<KK, 4, T>;          \
    return fwd_kernel<KK, 0, T>;                       \
  }
  DFFM_SEL(4)
  DFFM_SEL(8)
  DFFM_SEL(16)
  DFFM_SEL(0)
#undef DFFM_SEL
  return nullptr;
}

template <typename T>
int launch_forward_t(const FwdParams& p, int K, int MU, int smem, cudaStream_t s) {
  FwdKernel kern = select_fwd<T>(K, MU);
  if (!kern) { set_error("no forward kernel for k=%d", p.k); return DFFM_SIZING; }
  int occ = 0;
  int rc = kernel_occupancy((const void*)kern, FWD_THREADS, smem, &occ);
  if (rc) return rc;
  const int64_t ntiles = (p.n + p.TE - 1) / p.TE;
  const int64_t grid = std::min<int64_t>(ntiles, (int64_t)sm_count_current() * occ);
  note_launches(1), kern<<<(unsigned)grid, FWD_THREADS, smem, s>>>(p);
  DFFM_CUDA_TRY(cudaGetLastError(), "launch(forward)");
  return DFFM_OK;
}

template int launch_forward_t<DFFM_INST_T>(const FwdParams&, int, int, int, cudaStream_t);

// ---------------------------------------------------------------- K1 v3 (warp-specialised)
template <typename T>
static FwdKernel select_ws(int K, int MU) {
#define DFFM_SEL(KK)                                   \
  if (K == KK) {                                       \
    if (MU == 1) return fwd_ws_kernel<KK, 1, T>;       \
    if (MU == 2) return fwd_ws_kernel<KK, 2, T>;       \
    if (MU == 3) return fwd_ws_kernel<KK, 3, T>;       \
    if (MU == 4) return fwd_ws_kernel<KK, 4, T>;       \
    return fwd_ws_kernel<KK, 0, T>;                    \
  }
  DFFM_SEL(4)
  DFFM_SEL(8)
  DFFM_SEL(16)
  DFFM_SEL(0)
#undef DFFM_SEL
  return nullptr;
}

template <typename T>
int launch_forward_ws_t(const FwdParams& p, int K, int MU, int smem, cudaStream_t s) {
  FwdKernel kern = select_ws<T>(K, MU);
  if (!kern) { set_error("no forward kernel for k=%d", p.k); return DFFM_SIZING; }
  int occ = 0;
  int rc = kernel_occupancy((const void*)kern, WS_THREADS, smem, &occ);
  if (rc) return rc;
  const int64_t ntiles = (p.n + p.TE - 1) / p.TE;
  const int64_t grid = std::min<int64_t>(ntiles, (int64_t)sm_count_current() * occ);
  note_launches(1), kern<<<(unsigned)grid, WS_THREADS, smem, s>>>(p);
  DFFM_CUDA_TRY(cudaGetLastError(), "launch(forward_ws)");
  return DFFM_OK;
}

template int launch_forward_ws_t<DFFM_INST_T>(const FwdParams&, int, int, int, cudaStream_t);

// ---------------------------------------------------------------- K1 v8 (warp-specialised row ring)
using RswKernel = void (*)(FwdParams, RswSmem);
template <typename T>
static RswKernel select_rsw(int K, int MU) {
#define DFFM_SEL(KK)                                          \
  if (K == KK) {                                              \
    if (MU == 1) return fwd_rsw_kernel<KK, T, 1>;             \
    if (MU == 2) return fwd_rsw_kernel<KK, T, 2>;             \
    if (MU == 3) return fwd_rsw_kernel<KK, T, 3>;             \
    if (MU == 4) return fwd_rsw_kernel<KK, T, 4>;             \
  }
  if constexpr (sizeof(T) == 4) { DFFM_SEL(4) }
  DFFM_SEL(8)
  DFFM_SEL(16)
#undef DFFM_SEL
  return nullptr;
}

template <typename T>
int launch_forward_rsw_t(const FwdParams& p, const RswSmem& L, int K, cudaStream_t s) {
  RswKernel kern = select_rsw<T>(K, p.M);
  if (!kern) { set_error("no row-ring kernel for k=%d M=%d", K, p.M); return DFFM_SIZING; }
  int occ = 0;
  const int threads = (L.npw + RSW_NPROD + L.nmw) * 32;
  int rc = kernel_occupancy((const void*)kern, threads, L.total, &occ);
  if (rc) return rc;
  static int grid_env = -1;  // DFFM_RSW_GRID: SMs given to the gather (measurement knob)
  if (grid_env < 0) {
    const char* v = getenv("DFFM_RSW_GRID");
    grid_env = v ? atoi(v) : 0;
  }
  const int64_t sms = grid_env > 0 ? std::min(grid_env, sm_count_current()) : sm_count_current();
  const int64_t grid = std::min<int64_t>(p.n, sms);
  if (grid <= 0) return DFFM_OK;
  note_launches(1), kern<<<(unsigned)grid, threads, L.total, s>>>(p, L);
  DFFM_CUDA_TRY(cudaGetLastError(), "launch(forward_rsw)");
  return DFFM_OK;
}

template int launch_forward_rsw_t<DFFM_INST_T>(const FwdParams&, const RswSmem&, int, cudaStream_t);

}  // namespace dffm
