// K1 MLP stage on the 5th-generation tensor cores (tcgen05, kind::tf32, 3xTF32).
// Shared between mlp_tc.cu (kernels) and forward.cu (slicing / dispatch).
#pragma once

#include <cuda.h>

#include "common.cuh"

namespace dffm {

constexpr int TC_M = 128;       // examples per tile = UMMA M (one TMEM lane per example)
constexpr int TC_KC = 16;       // K elements per pipeline stage (64 B per row)
constexpr int TC_MAXH = 4;      // hidden layers (M:70-71)
#ifndef DFFM_TC_PARTS
#define DFFM_TC_PARTS 4
#endif
constexpr int TC_PARTS = DFFM_TC_PARTS;  // epilogue warps per TMEM lane quadrant (column parts)
constexpr int TC_EPI_WARPS = 4 * TC_PARTS;
#ifndef DFFM_TC_SPLIT_WARPS
#define DFFM_TC_SPLIT_WARPS 2
#endif
constexpr int TC_SPLIT_WARPS = DFFM_TC_SPLIT_WARPS;  // layer-0 A_lo producers
// warp 0 TMA, warp 1 MMA, then the epilogue warps, then the split warps
constexpr int TC_THREADS = 64 + 32 * (TC_EPI_WARPS + TC_SPLIT_WARPS);
constexpr int TC_PART_MAX = 256 / TC_PARTS;  // accumulator columns per epilogue thread
constexpr int TC_WIDTH_MULT = 16;            // hidden widths: multiples of this, <= 256
#ifndef DFFM_TC_GROUP
#define DFFM_TC_GROUP 16
#endif
constexpr int TC_GROUP = DFFM_TC_GROUP;  // K chunks per TMEM accumulation group
constexpr int TC_MAX_STAGES = 8;

struct MlpTcParams {
  const double* resid;  // [rows] lr_out + sum(pairs)            (M:377 residual)
  const int* flags;     // [rows] non-finite stage bits 1 lr, 2 ffm, 4 merge
  float* prob;          // [rows]
  float* logit;         // [rows] or null
  uint64_t* status;
  int64_t rows;
  int64_t status_base;
  int n_hidden;
  int kin[TC_MAXH];     // layer l input width, padded to a multiple of 16
  int nout[TC_MAXH];    // layer l output width (multiple of 16, <= 256)
  const float* wblk[TC_MAXH];  // per layer, kin/16 chunks of [hi N x 16][lo N x 16] (core-matrix blocked)
  const float* bias[TC_MAXH];
  const float* w_out;   // [nout[n_hidden-1]] output layer column (M:372)
  const float* b_out;   // [1]
  int stages;
  int stage_bytes;      // 16 KB (A hi + lo) + nmax * 128 B (W hi + lo), 1 KB aligned
  int tmem_cols;        // power of two >= 2 * nmax: two accumulator regions
};

__host__ __device__ inline int tc_stage_bytes(int nmax) {
  return (16384 + nmax * 128 + 1023) & ~1023;
}
// dynamic shared memory: 1 KB alignment slack, stages, barriers
// (full/aready/empty/lready per stage, accf/tempty per TMEM region), TMEM
// slot, and the parts' row exchange (double-buffered by tile)
__host__ __device__ inline int tc_smem_bytes(int stages, int stage_bytes) {
  return 1024 + stages * stage_bytes + (4 * stages + 4) * 8 + 16 + 2 * TC_PARTS * TC_M * 8;
}

int launch_mlp_tc(const CUtensorMap& tmx, const MlpTcParams& p, int smem, cudaStream_t s);

// Host plan for "stage rows, then tensor-core MLP" over slices (forward.cu):
// eligibility, per-stream workspace, blocked hi/lo weights.
struct TcPlan {
  MlpTcParams q;
  int smem;
  int Kp;
  int64_t slice_rows;
  float* X;       // [slice_rows][Kp] staged MergeNorm rows
  double* resid;  // [slice_rows]
  int* flags;     // [slice_rows]
};
struct FwdParams;
bool tc_eligible(const FwdParams& p, int smax);
int tc_plan(const FwdParams& p, int smax, int64_t slice_rows, cudaStream_t s, TcPlan* plan);
int tc_mlp_slice(TcPlan& plan, int64_t rows, int64_t status_base, float* prob, float* logit,
                 cudaStream_t s);
int64_t tc_default_slice_rows();
int launch_tc_prep_weights(const float* W, int K, int N, int Kp, float* dst, cudaStream_t s);

}  // namespace dffm
