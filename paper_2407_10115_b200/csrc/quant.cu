// K4: bit-exact 16-bit quantisation / dequantisation (SPEC S:313-328,
// PAPER.md:291-305), with the precision choices pinned in SURVEY 8(a) row Q:
//   header   : max rounded up at alpha decimals, min down at beta, in f64;
//              bucket = (max_r - min_r)/65536; both rounded to f32; bucket = 0
//              iff max_r == min_r
//   quantise : idx = clamp(rint((f64(w) - f64(hmin)) / f64(hbucket)), 0, 65535)
//              (IEEE f64 sub + div, round-half-even: identical to numpy)
//   dequant  : hmin + idx*hbucket as an f32 multiply then an f32 add, each
//              rounded to nearest (no FMA contraction)
// All three kernels are HBM-streaming: 16-byte vector loads/stores, grid a
// multiple of the SM count, grid-stride loops.
#include <math.h>

#include "common.cuh"

namespace dffm {

__device__ __forceinline__ uint32_t f2key(float f) {
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float key2f(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k);
}

__global__ void minmax_init(uint32_t* mm) {
  mm[0] = 0xFFFFFFFFu;  // min key
  mm[1] = 0u;           // max key
}

__global__ void __launch_bounds__(256) minmax_kernel(const float* __restrict__ w, int64_t n,
                                                      uint32_t* mm, uint64_t* first_bad) {
  uint32_t kmin = 0xFFFFFFFFu, kmax = 0u;
  uint64_t bad = ~0ull;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t n4 = ((uintptr_t)w & 15) ? 0 : n / 4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
    const float4 v = __ldg((const float4*)w + i);
    const float a[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (!isfinite(a[c])) { bad = min(bad, (uint64_t)(4 * i + c)); continue; }
      const uint32_t k = f2key(a[c]);
      kmin = min(kmin, k);
      kmax = max(kmax, k);
    }
  }
  for (int64_t i = 4 * n4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const float a = __ldg(w + i);
    if (!isfinite(a)) { bad = min(bad, (uint64_t)i); continue; }
    const uint32_t k = f2key(a);
    kmin = min(kmin, k);
    kmax = max(kmax, k);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
    kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
    bad = min(bad, __shfl_xor_sync(0xffffffffu, bad, o));
  }
  __shared__ uint32_t smin[8], smax[8];
  __shared__ uint64_t sbad[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { smin[warp] = kmin; smax[warp] = kmax; sbad[warp] = bad; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i) {
      kmin = min(kmin, smin[i]);
      kmax = max(kmax, smax[i]);
      bad = min(bad, sbad[i]);
    }
    atomicMin(mm, kmin);
    atomicMax(mm + 1, kmax);
    if (bad != ~0ull) atomicMin((unsigned long long*)first_bad, (unsigned long long)bad);
  }
}

__global__ void minmax_finish(uint32_t* mm) {
  float* out = (float*)mm;
  const float lo = key2f(mm[0]), hi = key2f(mm[1]);
  out[0] = lo;
  out[1] = hi;
}

__device__ __forceinline__ uint32_t quant1(float w, double hmin, double hb) {
  if (hb == 0.0) return 0u;
  const double r = rint(__ddiv_rn(__dsub_rn((double)w, hmin), hb));
  return (uint32_t)fmin(fmax(r, 0.0), 65535.0);
}

__global__ void __launch_bounds__(256) quant_kernel(const float* __restrict__ w, int64_t n,
                                                     double hmin, double hb, uint16_t* q) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const bool vec = !(((uintptr_t)w & 15) || ((uintptr_t)q & 7));
  const int64_t n4 = vec ? n / 4 : 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
    const float4 v = __ldg((const float4*)w + i);
    uint2 o;
    o.x = quant1(v.x, hmin, hb) | (quant1(v.y, hmin, hb) << 16);
    o.y = quant1(v.z, hmin, hb) | (quant1(v.w, hmin, hb) << 16);
    ((uint2*)q)[i] = o;
  }
  for (int64_t i = 4 * n4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    q[i] = (uint16_t)quant1(__ldg(w + i), hmin, hb);
}

__global__ void __launch_bounds__(256) dequant_kernel(const uint16_t* __restrict__ q, int64_t n,
                                                       float hmin, float hb, float* out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const Deq d{hmin, hb};
  const bool vec = !(((uintptr_t)q & 7) || ((uintptr_t)out & 15));
  const int64_t n4 = vec ? n / 4 : 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
    const uint2 v = __ldg((const uint2*)q + i);
    float4 o;
    o.x = deq(v.x & 0xFFFF, d);
    o.y = deq(v.x >> 16, d);
    o.z = deq(v.y & 0xFFFF, d);
    o.w = deq(v.y >> 16, d);
    ((float4*)out)[i] = o;
  }
  for (int64_t i = 4 * n4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = deq(__ldg(q + i), d);
}

static unsigned stream_grid(int64_t n) {
  const int64_t sms = sm_count_current();
  const int64_t want = (n / 4 + 255) / 256;
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(want, sms * 8));
}

}  // namespace dffm

using namespace dffm;

extern "C" int fwq_minmax(const float* w, int64_t n, float* minmax_out, uint64_t* first_nonfinite,
                          void* stream) {
  if (n <= 0) { set_error("quantize of an empty table"); return DFFM_CONTRACT; }
  if (!w || !minmax_out || !first_nonfinite) { set_error("null buffer"); return DFFM_CONTRACT; }
  cudaStream_t s = (cudaStream_t)stream;
  uint32_t* mm = (uint32_t*)minmax_out;
  note_launches(1), minmax_init<<<1, 1, 0, s>>>(mm);
  note_launches(1), minmax_kernel<<<stream_grid(n), 256, 0, s>>>(w, n, mm, first_nonfinite);
  note_launches(1), minmax_finish<<<1, 1, 0, s>>>(mm);
  DFFM_CUDA_TRY(cudaGetLastError(), "launch(fwq_minmax)");
  return DFFM_OK;
}

extern "C" int fwq_header(float wmin, float wmax, int32_t alpha, int32_t beta, float* hmin_host,
                          float* hbucket_host) {
  if (!hmin_host || !hbucket_host) { set_error("null header out"); return DFFM_CONTRACT; }
  if (!isfinite(wmin) || !isfinite(wmax) || wmin > wmax) {
    set_error("bad min/max");
    return DFFM_NUMERIC;
  }
  if (alpha < 0 || alpha > 15 || beta < 0 || beta > 15) {
    set_error("alpha/beta outside [0, 15]");
    return DFFM_CONTRACT;
  }
  const double sa = pow(10.0, (double)alpha), sb = pow(10.0, (double)beta);
  const double max_r = ceil((double)wmax * sa) / sa;
  const double min_r = floor((double)wmin * sb) / sb;
  const double bucket = (max_r == min_r) ? 0.0 : (max_r - min_r) / 65536.0;
  *hmin_host = (float)min_r;
  *hbucket_host = (float)bucket;
  return DFFM_OK;
}

extern "C" int fwq_quantize(const float* w, int64_t n, float hmin, float hbucket, uint16_t* q,
                            void* stream) {
  if (n < 0 || (n && (!w || !q))) { set_error("bad quantize args"); return DFFM_CONTRACT; }
  if (!n) return DFFM_OK;
  note_launches(1), quant_kernel<<<stream_grid(n), 256, 0, (cudaStream_t)stream>>>(w, n, (double)hmin,
                                                                  (double)hbucket, q);
  DFFM_CUDA_TRY(cudaGetLastError(), "launch(fwq_quantize)");
  return DFFM_OK;
}

extern "C" int fwq_dequantize(const uint16_t* q, int64_t n, float hmin, float hbucket, float* out,
                              void* stream) {
  if (n < 0 || (n && (!q || !out))) { set_error("bad dequantize args"); return DFFM_CONTRACT; }
  if (!n) return DFFM_OK;
  note_launches(1), dequant_kernel<<<stream_grid(n), 256, 0, (cudaStream_t)stream>>>(q, n, hmin, hbucket, out);
  DFFM_CUDA_TRY(cudaGetLastError(), "launch(fwq_dequantize)");
  return DFFM_OK;
}
