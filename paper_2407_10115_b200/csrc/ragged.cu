// K9: ragged (CSR) example batch -> the padded [n][F][M] layout K1 reads.
//
// The reference's canonical example (Fe:121-172) is ragged: per present field
// a strictly increasing index array and its values.  A batch of them is sent
// from the host as
//   ex_off int64 [n+1]   start of example e in idx/val (absolute; chunks of a
//                        larger batch pass their slice and nnz_base = ex_off[0])
//   cnt    u8    [n][F]  features of field f in example e (0 = absent field)
//   idx    i32   [nnz]   bucket indices, example-major, field-major, slot order
//   val    f32   [nnz]
// which is ~30% fewer host->device bytes than the padded layout at cfg2
// (47.4 of 72 slots present).  One warp per example: an exclusive scan of the
// field counts gives each field's start, then every padded slot (f, m) is
// written with coalesced stores (-1 / 0 for m >= cnt).  A count above M or a
// count sum that disagrees with ex_off is a ContractError at that example.
#include "common.cuh"

namespace dffm {

constexpr int RG_WARPS = 8;
constexpr int RG_MAXF = 256;

__global__ void __launch_bounds__(RG_WARPS * 32) unpack_ragged_kernel(
    const int64_t* __restrict__ ex_off, const uint8_t* __restrict__ cnt,
    const int32_t* __restrict__ idx, const float* __restrict__ val, int64_t n, int F, int M,
    int64_t nnz_base, int32_t* __restrict__ oidx, float* __restrict__ oval, uint64_t* status,
    int64_t status_base) {
  __shared__ int foff[RG_WARPS][RG_MAXF + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int* fo = foff[warp];
  const int FM = F * M;
  for (int64_t e = (int64_t)blockIdx.x * RG_WARPS + warp; e < n;
       e += (int64_t)gridDim.x * RG_WARPS) {
    const int64_t b = __ldg(ex_off + e) - nnz_base, len = __ldg(ex_off + e + 1) - nnz_base - b;
    int run = 0, bad = 0;
    for (int f0 = 0; f0 < F; f0 += 32) {
      const int f = f0 + lane;
      const int c = f < F ? (int)__ldg(cnt + e * F + f) : 0;
      bad |= c > M;
      int x = c;  // inclusive warp scan
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (f < F) { fo[f] = run + x - c; }
      run += __shfl_sync(0xffffffffu, x, 31);
    }
    if (lane == 0) fo[F] = run;
    __syncwarp();
    bad = __any_sync(0xffffffffu, bad) || run != len;
    if (bad && lane == 0)
      atomicMin((unsigned long long*)status,
                (unsigned long long)status_key(status_base + e, DFFM_BLOCK_NONE, DFFM_CONTRACT));
    for (int s = lane; s < FM; s += 32) {
      const int f = s / M, m = s - f * M;
      const int o = fo[f] + m;
      const bool live = !bad && o < fo[f + 1];
      oidx[e * FM + s] = live ? __ldg(idx + b + o) : -1;
      oval[e * FM + s] = live ? __ldg(val + b + o) : 0.f;
    }
    __syncwarp();
  }
}

}  // namespace dffm

using namespace dffm;

extern "C" int dffm_unpack_ragged(const int64_t* ex_off, const uint8_t* cnt, const int32_t* idx,
                                  const float* val, int64_t n, int32_t n_fields,
                                  int32_t max_per_field, int64_t nnz_base, int32_t* out_idx,
                                  float* out_val, int64_t status_base, uint64_t* status,
                                  void* stream) {
  if (n < 0 || n_fields < 1 || n_fields > RG_MAXF || max_per_field < 1 || max_per_field > 64) {
    set_error("bad ragged batch shape n=%lld F=%d M=%d", (long long)n, n_fields, max_per_field);
    return DFFM_CONTRACT;
  }
  if (!n) return DFFM_OK;
  if (!ex_off || !cnt || !out_idx || !out_val || !status) { set_error("null buffer"); return DFFM_CONTRACT; }
  const int64_t sms = sm_count_current();
  const unsigned grid =
      (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + RG_WARPS - 1) / RG_WARPS, sms * 8));
  note_launches(1), unpack_ragged_kernel<<<grid, RG_WARPS * 32, 0, (cudaStream_t)stream>>>(
      ex_off, cnt, idx, val, n, n_fields, max_per_field, nnz_base, out_idx, out_val, status,
      status_base);
  DFFM_CUDA_TRY(cudaGetLastError(), "launch(dffm_unpack_ragged)");
  return DFFM_OK;
}

// ---- K9b: packed wire format (fewer host->device bytes than the ragged batch)
//   idx as `ib` little-endian bytes per feature (3 when hash_bits <= 24: exact),
//   values equal to 1.0 elided: vbits bit t (global feature t, LSB first) set
//   <=> feature t carries an explicit f32 in vals (in feature order, example
//   e's from voff[e]).  Same per-example field counts and ex_off as K9.
namespace dffm {

constexpr int PK_MAXFM = 128;  // padded slots per example (as K1 v8)

__global__ void __launch_bounds__(RG_WARPS * 32) unpack_packed_kernel(
    const int64_t* __restrict__ ex_off, const uint8_t* __restrict__ cnt,
    const uint8_t* __restrict__ idxb, int ib, const uint8_t* __restrict__ vbits,
    const float* __restrict__ vals, const int64_t* __restrict__ voff, int64_t n, int F, int M,
    int64_t nnz_base, int64_t bit_base, int64_t val_base, int32_t* __restrict__ oidx,
    float* __restrict__ oval, uint64_t* status, int64_t status_base) {
  __shared__ int foff[RG_WARPS][RG_MAXF + 1];
  __shared__ int fidx[RG_WARPS][PK_MAXFM];
  __shared__ float fval[RG_WARPS][PK_MAXFM];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int* fo = foff[warp];
  const int FM = F * M;
  for (int64_t e = (int64_t)blockIdx.x * RG_WARPS + warp; e < n;
       e += (int64_t)gridDim.x * RG_WARPS) {
    const int64_t b = __ldg(ex_off + e) - nnz_base, len = __ldg(ex_off + e + 1) - nnz_base - b;
    int run = 0, bad = 0;
    for (int f0 = 0; f0 < F; f0 += 32) {
      const int f = f0 + lane;
      const int c = f < F ? (int)__ldg(cnt + e * F + f) : 0;
      bad |= c > M;
      int x = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (f < F) fo[f] = run + x - c;
      run += __shfl_sync(0xffffffffu, x, 31);
    }
    if (lane == 0) fo[F] = run;
    bad = __any_sync(0xffffffffu, bad) || run != len || len > FM;
    // the example's features: index bytes, explicit-value bits, ranks among them
    const int64_t v0 = __ldg(voff + e) - val_base;
    int vr = 0;
    for (int t0 = 0; t0 < (bad ? 0 : (int)len); t0 += 32) {
      const int t = t0 + lane;
      int64_t g = b + t;  // feature number within this call's buffers
      bool has = false;
      int j = -1;
      if (t < len) {
        const uint8_t* q = idxb + g * ib;
        j = (int)q[0] | ((int)q[1] << 8) | ((int)q[2] << 16) | (ib == 4 ? ((int)q[3] << 24) : 0);
        const int64_t bit = bit_base + g;
        has = (vbits[bit >> 3] >> (bit & 7)) & 1;
      }
      const uint32_t bm = __ballot_sync(0xffffffffu, has);
      if (t < len) {
        fidx[warp][t] = j;
        fval[warp][t] = has ? __ldg(vals + v0 + vr + __popc(bm & ((1u << lane) - 1u))) : 1.0f;
      }
      vr += __popc(bm);
    }
    __syncwarp();
    if (bad && lane == 0)
      atomicMin((unsigned long long*)status,
                (unsigned long long)status_key(status_base + e, DFFM_BLOCK_NONE, DFFM_CONTRACT));
    for (int s = lane; s < FM; s += 32) {
      const int f = s / M, m = s - f * M;
      const int o = fo[f] + m;
      const bool live = !bad && o < fo[f + 1];
      oidx[e * FM + s] = live ? fidx[warp][o] : -1;
      oval[e * FM + s] = live ? fval[warp][o] : 0.f;
    }
    __syncwarp();
  }
}

}  // namespace dffm

extern "C" int dffm_unpack_packed(const int64_t* ex_off, const uint8_t* cnt, const uint8_t* idx_bytes,
                                  int32_t idx_width, const uint8_t* vbits, const float* vals,
                                  const int64_t* voff, int64_t n, int32_t n_fields,
                                  int32_t max_per_field, int64_t nnz_base, int64_t bit_base,
                                  int64_t val_base, int32_t* out_idx, float* out_val,
                                  int64_t status_base, uint64_t* status, void* stream) {
  if (n < 0 || n_fields < 1 || max_per_field < 1 || n_fields * max_per_field > PK_MAXFM ||
      (idx_width != 3 && idx_width != 4)) {
    set_error("bad packed batch shape n=%lld F=%d M=%d width=%d", (long long)n, n_fields,
              max_per_field, idx_width);
    return DFFM_CONTRACT;
  }
  if (!n) return DFFM_OK;
  if (!ex_off || !cnt || !voff || !out_idx || !out_val || !status) {
    set_error("null buffer");
    return DFFM_CONTRACT;
  }
  const int64_t sms = sm_count_current();
  const unsigned grid =
      (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + RG_WARPS - 1) / RG_WARPS, sms * 8));
  note_launches(1), unpack_packed_kernel<<<grid, RG_WARPS * 32, 0, (cudaStream_t)stream>>>(
      ex_off, cnt, idx_bytes, idx_width, vbits, vals, voff, n, n_fields, max_per_field, nnz_base,
      bit_base, val_base, out_idx, out_val, status, status_base);
  DFFM_CUDA_TRY(cudaGetLastError(), "launch(dffm_unpack_packed)");
  return DFFM_OK;
}
