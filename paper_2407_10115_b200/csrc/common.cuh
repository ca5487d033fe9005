// Shared device/host helpers for libdffm (sm_100a).
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/dffm.h"

namespace dffm {

// ------------------------------------------------------------------ host side
void set_error(const char* fmt, ...);
int cuda_fail(cudaError_t e, const char* what);
int sm_count_current();
int max_smem_optin_current();
// Raise the kernel's dynamic-smem limit to the device opt-in maximum (once per
// kernel and device) and return resident blocks/SM for this smem size (cached).
int kernel_occupancy(const void* func, int threads, int smem, int* occ);
// Count of kernels this library has launched (all devices, all threads):
// dffm_launch_count() reports it, so a bench can state its own launches.
void note_launches(int k);

#define DFFM_CUDA_TRY(expr, what)                 \
  do {                                            \
    cudaError_t _e = (expr);                      \
    if (_e != cudaSuccess) return cuda_fail(_e, what); \
  } while (0)

// status word: (example << 8) | (block << 4) | code   (see dffm.h)
__host__ __device__ inline uint64_t status_key(int64_t example, int block, int code) {
  return ((uint64_t)example << 8) | ((uint64_t)(block & 0xF) << 4) | (uint64_t)(code & 0xF);
}

// ------------------------------------------------------------------ device side
struct Deq {
  float qmin, qb;  // u16 header (ignored for f32/bf16)
};

// Read-only streaming loads of table rows (L1::no_allocate keeps L1 for the
// MLP weights).  Not volatile: the tables are immutable during a launch, so
// the compiler may batch these loads ahead of their uses.
__device__ __forceinline__ uint4 ldg_stream16(const void* p) {
  uint4 r;
  asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
      : "l"(p));
  return r;
}
// 256-bit load (sm_100: LDG.E.ENL2.256): one k=8 f32 / k=16 bf16 segment
__device__ __forceinline__ void ldg_stream32(const void* p, uint4& a, uint4& b) {
  asm("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
      : "l"(p));
}
// Predicated, branch-free variants: outputs are zero when !pred, so a whole
// pair's slot loads are straight-line code the scheduler issues back to back.
__device__ __forceinline__ void ldg_stream32_pred(const void* p, int pred, uint4& a, uint4& b) {
  asm("{\n\t.reg .pred q;\n\t"
      "setp.ne.b32 q, %9, 0;\n\t"
      "mov.b32 %0, 0; mov.b32 %1, 0; mov.b32 %2, 0; mov.b32 %3, 0;\n\t"
      "mov.b32 %4, 0; mov.b32 %5, 0; mov.b32 %6, 0; mov.b32 %7, 0;\n\t"
      "@q ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n\t}"
      : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
      : "l"(p), "r"(pred));
}
__device__ __forceinline__ uint4 ldg_stream16_pred(const void* p, int pred) {
  uint4 r;
  asm("{\n\t.reg .pred q;\n\t"
      "setp.ne.b32 q, %5, 0;\n\t"
      "mov.b32 %0, 0; mov.b32 %1, 0; mov.b32 %2, 0; mov.b32 %3, 0;\n\t"
      "@q ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];\n\t}"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
      : "l"(p), "r"(pred));
  return r;
}
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
__device__ __forceinline__ uint2 ldg_stream8(const void* p) {
  uint2 r;
  asm("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];"
      : "=r"(r.x), "=r"(r.y)
      : "l"(p));
  return r;
}

// ---- mbarrier / TMA-bulk / cp.async primitives (sm_90+, used on sm_100a)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;"
               ::"r"(smem_u32(bar)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// Blocking wait for phase `parity` of `bar`.  DFFM_MBAR_HINT (ns, 0 = none) is the
// try_wait suspend-time hint: a waiting warp sleeps until the phase completes (or
// the hint expires) instead of re-issuing the probe, which frees issue slots for
// the warps doing work.
#ifndef DFFM_MBAR_HINT
#define DFFM_MBAR_HINT 0
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
#if DFFM_MBAR_HINT > 0
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity), "n"(DFFM_MBAR_HINT)
      : "memory");
#else
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
#endif
}
// 1-D TMA bulk copy global -> shared, completion counted on `bar` (bytes % 16 == 0)
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
// arrive on `bar` once all of this thread's prior cp.async copies have landed
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

__device__ __forceinline__ float bf16lo(uint32_t u) { return __uint_as_float(u << 16); }
__device__ __forceinline__ float bf16hi(uint32_t u) { return __uint_as_float(u & 0xFFFF0000u); }
// inline dequantisation: w = qmin + q*qb, f32 multiply then f32 add.
// float(q) for q < 2^16 through the 2^23 magic constant (bit pattern 0x4B000000 | q
// is exactly 2^23 + q): one logic op and one exact FADD instead of an I2F on the
// quarter-rate conversion pipe -- the hottest opcode of the K3 pair warps.
__device__ __forceinline__ float deq(uint32_t q, const Deq& d) {
  const float fq = __fadd_rn(__uint_as_float(0x4B000000u | q), -8388608.f);
  return __fadd_rn(d.qmin, __fmul_rn(fq, d.qb));
}

// Scalar table element -> float
template <typename T>
__device__ __forceinline__ float load_elem(const T* p, const Deq& d);
template <>
__device__ __forceinline__ float load_elem<float>(const float* p, const Deq&) {
  return __ldg(p);
}
template <>
__device__ __forceinline__ float load_elem<__nv_bfloat16>(const __nv_bfloat16* p, const Deq&) {
  return __bfloat162float(*p);
}
template <>
__device__ __forceinline__ float load_elem<uint16_t>(const uint16_t* p, const Deq& d) {
  return deq(*p, d);
}

// Raw table element -> float (the conversion split from the load, so a warp can
// keep the load in flight and convert where the value is consumed)
template <typename T>
__device__ __forceinline__ float elem_to_float(T raw, const Deq& d);
template <>
__device__ __forceinline__ float elem_to_float<float>(float raw, const Deq&) { return raw; }
template <>
__device__ __forceinline__ float elem_to_float<__nv_bfloat16>(__nv_bfloat16 raw, const Deq&) {
  return __bfloat162float(raw);
}
template <>
__device__ __forceinline__ float elem_to_float<uint16_t>(uint16_t raw, const Deq& d) {
  return deq(raw, d);
}

// Unpack one 16-byte chunk of T into floats
template <typename T>
__device__ __forceinline__ void unpack16(const uint4& u, float* o, const Deq& d);
template <>
__device__ __forceinline__ void unpack16<float>(const uint4& u, float* o, const Deq&) {
  o[0] = __uint_as_float(u.x); o[1] = __uint_as_float(u.y);
  o[2] = __uint_as_float(u.z); o[3] = __uint_as_float(u.w);
}
template <>
__device__ __forceinline__ void unpack16<__nv_bfloat16>(const uint4& u, float* o, const Deq&) {
  o[0] = bf16lo(u.x); o[1] = bf16hi(u.x); o[2] = bf16lo(u.y); o[3] = bf16hi(u.y);
  o[4] = bf16lo(u.z); o[5] = bf16hi(u.z); o[6] = bf16lo(u.w); o[7] = bf16hi(u.w);
}
template <>
__device__ __forceinline__ void unpack16<uint16_t>(const uint4& u, float* o, const Deq& d) {
  o[0] = deq(u.x & 0xFFFF, d); o[1] = deq(u.x >> 16, d);
  o[2] = deq(u.y & 0xFFFF, d); o[3] = deq(u.y >> 16, d);
  o[4] = deq(u.z & 0xFFFF, d); o[5] = deq(u.z >> 16, d);
  o[6] = deq(u.w & 0xFFFF, d); o[7] = deq(u.w >> 16, d);
}
template <typename T>
__device__ __forceinline__ void unpack8(const uint2& u, float* o, const Deq& d) {
  uint4 w = make_uint4(u.x, u.y, 0, 0);
  float t[16 / sizeof(T)];
  unpack16<T>(w, t, d);
#pragma unroll
  for (int i = 0; i < (int)(8 / sizeof(T)); ++i) o[i] = t[i];
}

// d + <a, b> over one 16-byte chunk of T values, f32 sequential in element
// order; bf16 uses the mixed-precision FMA (FHFMA.BF16: exact bf16 products,
// one f32 rounding per step -- the same bits as widening first)
template <typename T>
__device__ __forceinline__ float dot16_acc(const uint4& a, const uint4& b, float d, const Deq& q) {
  constexpr int PER = 16 / (int)sizeof(T);
  float x[PER], y[PER];
  unpack16<T>(a, x, q);
  unpack16<T>(b, y, q);
#pragma unroll
  for (int t = 0; t < PER; ++t) d = fmaf(x[t], y[t], d);
  return d;
}
template <>
__device__ __forceinline__ float dot16_acc<__nv_bfloat16>(const uint4& a, const uint4& b, float d,
                                                          const Deq&) {
  const uint32_t xa[4] = {a.x, a.y, a.z, a.w}, xb[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
  for (int i = 0; i < 4; ++i)
    asm("{.reg .b16 al, ah, bl, bh;\n\t"
        "mov.b32 {al, ah}, %1;\n\t"
        "mov.b32 {bl, bh}, %2;\n\t"
        "fma.rn.f32.bf16 %0, al, bl, %0;\n\t"
        "fma.rn.f32.bf16 %0, ah, bh, %0;\n\t}"
        : "+f"(d)
        : "r"(xa[i]), "r"(xb[i]));
  return d;
}

// Load one k-vector segment (K elements of T, naturally aligned) as floats.
// K == 0 selects the runtime-k scalar path (tests / unusual k).
template <int K, typename T>
struct Seg {
  static constexpr int BYTES = K * (int)sizeof(T);
  __device__ __forceinline__ static void load(const T* p, float* o, const Deq& d, int) {
    if constexpr (BYTES >= 32) {
      constexpr int PER = 16 / sizeof(T);
      uint4 u[BYTES / 16];
#pragma unroll
      for (int c = 0; c < BYTES / 32; ++c) ldg_stream32(p + 2 * c * PER, u[2 * c], u[2 * c + 1]);
#pragma unroll
      for (int c = 0; c < BYTES / 16; ++c) unpack16<T>(u[c], o + c * PER, d);
    } else if constexpr (BYTES == 16) {
      constexpr int PER = 16 / sizeof(T);
      uint4 u[BYTES / 16];
#pragma unroll
      for (int c = 0; c < BYTES / 16; ++c) u[c] = ldg_stream16(p + c * PER);
#pragma unroll
      for (int c = 0; c < BYTES / 16; ++c) unpack16<T>(u[c], o + c * PER, d);
    } else if constexpr (BYTES == 8) {
      unpack8<T>(ldg_stream8(p), o, d);
    } else {
#pragma unroll
      for (int c = 0; c < K; ++c) o[c] = load_elem<T>(p + c, d);
    }
  }
};

// Runtime-k segment load for the K == 0 instantiation.
template <typename T>
struct Seg<0, T> {
  __device__ __forceinline__ static void load(const T* p, float* o, const Deq& d, int k) {
    for (int c = 0; c < k; ++c) o[c] = load_elem<T>(p + c, d);
  }
};

// np.maximum(z, 0.0) semantics (M:370): NaN propagates (fmaxf would drop it)
// Staged MergeNorm rows for the tensor-core MLP (mlp_tc.cu): two fp16 planes,
// x = hi + lo with hi = fp16(x), lo = fp16(x - hi) (22 significant bits), each
// plane row-major [rows][Kp] halfs, lo plane `plane` halfs after hi.
__device__ __forceinline__ void xstore1(__half* x, int64_t plane, int64_t i, float v) {
  const __half h = __float2half_rn(v);
  x[i] = h;
  x[plane + i] = __float2half_rn(v - __half2float(h));
}
__device__ __forceinline__ void xstore4(__half* x, int64_t plane, int64_t i, const float* v) {
  uint32_t h[2], l[2];
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    const __half a = __float2half_rn(v[2 * t]), b = __float2half_rn(v[2 * t + 1]);
    const __half al = __float2half_rn(v[2 * t] - __half2float(a));
    const __half bl = __float2half_rn(v[2 * t + 1] - __half2float(b));
    h[t] = (uint32_t)__half_as_ushort(a) | ((uint32_t)__half_as_ushort(b) << 16);
    l[t] = (uint32_t)__half_as_ushort(al) | ((uint32_t)__half_as_ushort(bl) << 16);
  }
  *(uint2*)(x + i) = make_uint2(h[0], h[1]);
  *(uint2*)(x + plane + i) = make_uint2(l[0], l[1]);
}

__device__ __forceinline__ float relu_nan(float z) { return z != z ? z : fmaxf(z, 0.f); }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_sumf(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Stable clamped sigmoid (M:293-305), f64.
__device__ __forceinline__ double sigmoid_clamped(double logit) {
  double p;
  if (logit >= 0.0) {
    p = 1.0 / (1.0 + exp(-fmin(logit, 60.0)));
  } else {
    double e = exp(fmax(logit, -60.0));
    p = e / (1.0 + e);
  }
  return fmin(fmax(p, 1e-7), 1.0 - 1e-7);
}

}  // namespace dffm
