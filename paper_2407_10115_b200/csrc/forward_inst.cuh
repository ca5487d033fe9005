// Per-storage-type instantiation of K1 (included once per forward_<dtype>.cu
// so the three table types compile in parallel).
#pragma once

#include <mutex>
#include <unordered_map>

#include "forward_kernel.cuh"
#include "forward_tma.cuh"
#include "forward_ws.cuh"
#include "forward_rows.cuh"
#include "forward_g4.cuh"
#include "forward_rowstage.cuh"
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

// ---------------------------------------------------------------- K1 v2 (TMA ring)
using TmaKernel = void (*)(TmaParams);

template <typename T>
static TmaKernel select_tma(int K) {
  if constexpr (sizeof(T) == 4) {
    if (K == 4) return fwd_tma_kernel<4, T>;
  }
  if (K == 8) return fwd_tma_kernel<8, T>;
  if (K == 16) return fwd_tma_kernel<16, T>;
  return nullptr;
}

template <typename T>
int launch_forward_tma_t(const TmaParams& q, int K, int smem, cudaStream_t s) {
  TmaKernel kern = select_tma<T>(K);
  if (!kern) { set_error("no TMA forward kernel for k=%d", K); return DFFM_SIZING; }
  int occ = 0;
  int rc = kernel_occupancy((const void*)kern, TMA_THREADS, smem, &occ);
  if (rc) return rc;
  const int64_t ntiles = (q.f.n + q.f.TE - 1) / q.f.TE;
  const int64_t grid = std::min<int64_t>(ntiles, (int64_t)sm_count_current() * occ);
  note_launches(1), kern<<<(unsigned)grid, TMA_THREADS, smem, s>>>(q);
  DFFM_CUDA_TRY(cudaGetLastError(), "launch(forward_tma)");
  return DFFM_OK;
}

template int launch_forward_tma_t<DFFM_INST_T>(const TmaParams&, int, int, cudaStream_t);

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

// ---------------------------------------------------------------- K1 v4 (row-coalesced)
template <int K, typename T>
static FwdKernel select_rows_m(int MU) {
  switch (MU) {
    case 1: return fwd_rows_kernel<K, 1, T>;
    case 2: return fwd_rows_kernel<K, 2, T>;
    case 3: return fwd_rows_kernel<K, 3, T>;
    case 4: return fwd_rows_kernel<K, 4, T>;
    default: return nullptr;
  }
}

template <typename T>
static FwdKernel select_rows(int K, int MU) {
  if constexpr (sizeof(T) == 4) {
    if (K == 4) return select_rows_m<4, T>(MU);
  }
  if (K == 8) return select_rows_m<8, T>(MU);
  if (K == 16) return select_rows_m<16, T>(MU);
  return nullptr;
}

template <typename T>
int launch_forward_rows_t(const FwdParams& p, int K, int smem, cudaStream_t s) {
  FwdKernel kern = select_rows<T>(K, p.M);
  if (!kern) { set_error("no row-coalesced kernel for k=%d", K); return DFFM_SIZING; }
  int occ = 0;
  int rc = kernel_occupancy((const void*)kern, RW_THREADS, smem, &occ);
  if (rc) return rc;
  const int64_t ntiles = (p.n + p.TE - 1) / p.TE;
  const int64_t grid = std::min<int64_t>(ntiles, (int64_t)sm_count_current() * occ);
  note_launches(1), kern<<<(unsigned)grid, RW_THREADS, smem, s>>>(p);
  DFFM_CUDA_TRY(cudaGetLastError(), "launch(forward_rows)");
  return DFFM_OK;
}

template int launch_forward_rows_t<DFFM_INST_T>(const FwdParams&, int, int, cudaStream_t);

// ---------------------------------------------------------------- K1 v5 (TMA gather4)
using G4Kernel = void (*)(const CUtensorMap, G4Params);

template <typename T>
static G4Kernel select_g4(int K) {
  if constexpr (sizeof(T) == 4) {
    if (K == 4) return fwd_g4_kernel<4, T>;
  }
  if (K == 8) return fwd_g4_kernel<8, T>;
  if (K == 16) return fwd_g4_kernel<16, T>;
  return nullptr;
}

template <typename T>
int launch_forward_g4_t(const CUtensorMap& tm, const G4Params& q, int K, int smem,
                        cudaStream_t s) {
  G4Kernel kern = select_g4<T>(K);
  if (!kern) { set_error("no gather4 kernel for k=%d", K); return DFFM_SIZING; }
  int occ = 0;
  int rc = kernel_occupancy((const void*)kern, G4_THREADS, smem, &occ);
  if (rc) return rc;
  const int64_t ntiles = (q.f.n + q.f.TE - 1) / q.f.TE;
  const int64_t grid = std::min<int64_t>(ntiles, (int64_t)sm_count_current());
  note_launches(1), kern<<<(unsigned)grid, G4_THREADS, smem, s>>>(tm, q);
  DFFM_CUDA_TRY(cudaGetLastError(), "launch(forward_g4)");
  return DFFM_OK;
}

template int launch_forward_g4_t<DFFM_INST_T>(const CUtensorMap&, const G4Params&, int, int,
                                              cudaStream_t);

// ---------------------------------------------------------------- K1 v7 (row staging, M == 1)
template <typename T>
static FwdKernel select_rowstage(int K, int NB) {
#define DFFM_SEL(KK)                                          \
  if (K == KK) {                                              \
    if (NB == 2) return fwd_rowstage_kernel<KK, T, 2>;        \
    if (NB == 3) return fwd_rowstage_kernel<KK, T, 3>;        \
    if (NB == 4) return fwd_rowstage_kernel<KK, T, 4>;        \
  }
  if constexpr (sizeof(T) == 4) { DFFM_SEL(4) }
  DFFM_SEL(8)
  DFFM_SEL(16)
#undef DFFM_SEL
  return nullptr;
}

template <typename T>
int launch_forward_rowstage_t(const FwdParams& p, int K, int NB, int smem, cudaStream_t s) {
  FwdKernel kern = select_rowstage<T>(K, NB);
  if (!kern) { set_error("no row-staging kernel for k=%d", K); return DFFM_SIZING; }
  int occ = 0;
  int rc = kernel_occupancy((const void*)kern, RS_THREADS, smem, &occ);
  if (rc) return rc;
  const int64_t grid = std::min<int64_t>(p.n, (int64_t)sm_count_current() * occ);
  note_launches(1), kern<<<(unsigned)grid, RS_THREADS, smem, s>>>(p);
  DFFM_CUDA_TRY(cudaGetLastError(), "launch(forward_rowstage)");
  return DFFM_OK;
}

template int launch_forward_rowstage_t<DFFM_INST_T>(const FwdParams&, int, int, int, cudaStream_t);


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
  int rc = kernel_occupancy((const void*)kern, RSW_THREADS, L.total, &occ);
  if (rc) return rc;
  const int64_t grid = std::min<int64_t>(p.n, (int64_t)sm_count_current());
  if (grid <= 0) return DFFM_OK;
  note_launches(1), kern<<<(unsigned)grid, RSW_THREADS, L.total, s>>>(p, L);
  DFFM_CUDA_TRY(cudaGetLastError(), "launch(forward_rsw)");
  return DFFM_OK;
}

template int launch_forward_rsw_t<DFFM_INST_T>(const FwdParams&, const RswSmem&, int, cudaStream_t);

}  // namespace dffm
