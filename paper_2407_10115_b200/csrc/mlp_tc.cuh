// K1 MLP stage on the 5th-generation tensor cores (tcgen05, kind::f16 with an
// fp16 hi/lo operand split, f32 accumulation).  Shared between mlp_tc.cu
// (kernels) and forward.cu (slicing / dispatch).
#pragma once

#include <cuda.h>

#include <cuda_fp16.h>

#include "common.cuh"

namespace dffm {

constexpr int TC_M = 128;       // examples per tile = UMMA M (one TMEM lane per example)
constexpr int TC_KC = 16;       // K elements per pipeline stage = one kind::f16 MMA's K
constexpr int TC_MAXH = 4;      // hidden layers (M:70-71)
#ifndef DFFM_TC_PARTS
#define DFFM_TC_PARTS 4
#endif
constexpr int TC_PARTS = DFFM_TC_PARTS;  // epilogue warps per TMEM lane quadrant (column parts)
constexpr int TC_EPI_WARPS = 4 * TC_PARTS;
// warp 0 TMA, warp 1 MMA, then the epilogue warps
constexpr int TC_THREADS = 64 + 32 * TC_EPI_WARPS;
constexpr int TC_WIDTH_MULT = 16;            // hidden widths: multiples of this, <= 256
#ifndef DFFM_TC_GROUP
#define DFFM_TC_GROUP 64
#endif
constexpr int TC_GROUP = DFFM_TC_GROUP;  // max K chunks of a layer (one TMEM accumulation)
constexpr int TC_MAX_STAGES = 8;
// stage layout (bytes): A0 A1 fp16 tiles (layer 0: one TMA of the staged hi/lo
// planes) | B0 B1 fp16 tiles.  Later layers read A from TMEM: the epilogue
// rewrites the previous layer's accumulator region in place as packed fp16
// pieces (chunk c: hi at column 16c, lo at 16c + 8).
constexpr int TC_OFF_A = 0;           // 2 tiles of 128 x 16 fp16 (4 KB each)
constexpr int TC_OFF_B = 8192;
constexpr int TC_HEXP = 14;           // operands are scaled to a maximum in [2^14, 2^15)
// per-launch constants staged in shared memory: every hidden layer's bias
// (<= 256 each), the output column (<= 256), its bias and the weight scales
constexpr int TC_CONST_FLOATS = 4 * 256 + 256 + 8;

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
  const __half* wblk[TC_MAXH];  // per layer, kin/16 chunks of [B0 N x 16][B1 N x 16] fp16
                                // (K-major core-matrix blocked, see tc_prep_weights_kernel)
  const int* wexp;      // [TC_MAXH] per-layer power-of-two scale of the blocked weights
  const float* bias[TC_MAXH];
  const float* w_out;   // [nout[n_hidden-1]] output layer column (M:372)
  const float* b_out;   // [1]
  int stages;
  int stage_bytes;      // 8 KB (A tiles) + nmax * 64 B (B tiles), 1 KB aligned
  int tmem_cols;        // power of two >= 2 * nmax: two accumulator regions
};

__host__ __device__ inline int tc_stage_bytes(int nmax) {
  return (TC_OFF_B + nmax * 64 + 1023) & ~1023;
}
// dynamic shared memory: 1 KB alignment slack, stages, barriers (full/empty
// per stage, abar, accf/tempty per TMEM region),
// TMEM slot, the parts' row exchange (double-buffered by tile) and the row
// exponent exchange (double-buffered by layer)
__host__ __device__ inline int tc_smem_bytes(int stages, int stage_bytes) {
  return 1024 + stages * stage_bytes + (2 * stages + 6) * 8 + 16 +
         2 * TC_PARTS * TC_M * 8 + 2 * TC_PARTS * TC_M * 4 + TC_CONST_FLOATS * 4;
}

int launch_mlp_tc(const CUtensorMap& tmx, const MlpTcParams& p, int smem, cudaStream_t s);

// Host plan for "stage rows, then tensor-core MLP" over slices (forward.cu):
// eligibility, per-stream workspace, blocked hi/lo weights.
struct TcPlan {
  MlpTcParams q;
  int smem;
  int Kp;
  int64_t slice_rows;
  __half* X;      // [2][slice_rows][Kp] staged MergeNorm rows: fp16 hi plane, lo plane
  int64_t xplane; // halfs per plane
  double* resid;  // [slice_rows]
  int* flags;     // [slice_rows]
};
struct FwdParams;
bool tc_eligible(const FwdParams& p, int smax);
int tc_plan(const FwdParams& p, int smax, int64_t slice_rows, cudaStream_t s, TcPlan* plan);
int tc_mlp_slice(TcPlan& plan, int64_t rows, int64_t status_base, float* prob, float* logit,
                 cudaStream_t s);
int64_t tc_default_slice_rows();
// W [K][N] f32 -> fp16 hi/lo blocks (dst: Kp/16 chunks of 64 N bytes) with the
// layer's power-of-two scale in *wexp; wmax: device int scratch (max |w| bits)
int launch_tc_prep_weights(const float* W, int K, int N, int Kp, __half* dst, int* wmax,
                           int* wexp, cudaStream_t s);

}  // namespace dffm
