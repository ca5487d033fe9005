// K1 v7 gather for the tensor-core MLP path, single-slot fields (M == 1:
// cfg1/4/5-style data): CTA-cooperative whole-row staging.
//
// With one feature per field an example reads its F latent rows in full
// (every segment but the diagonal, M:339-351), so instead of scattered 32-B
// segment loads held in registers (K1 v3), the whole CTA copies the example's
// rows -- contiguous F*k*sizeof(T) bytes each, 1280 B at cfg5 -- into a
// shared-memory ring with one bulk (TMA) copy per row, NB examples deep; a
// buffer is refilled as soon as its example's pairs are formed (before the
// MergeNorm reductions), and two CTAs share each SM, so ~4 examples' rows
// (~200 KB at cfg5) are resident or in flight per SM and every DRAM access
// is a whole contiguous row.
//
// Per example (one CTA, persistent over examples blockIdx.x + i*gridDim.x):
//   pairs    <S[f1][f2], S[f2][f1]> from shared memory (M:344-351), inactive
//            pairs exactly 0; raw values into a row buffer
//   lr       bias + sum of the field weights (M:327, M:338), 4-byte cp.async
//            of the aligned word holding each lr element
//   merge    f64 block reductions for mean / population std (M:355-360)
//   out      the standardised row (zero padded to Kp), lr_out + sum(pairs)
//            and the non-finite stage bits -> the staging buffers read by
//            mlp_tc_kernel
// Same arithmetic as K1 v3 (f32 pair dots in slot order, f64 statistics).
#pragma once

#include <type_traits>

#include "forward_kernel.cuh"

namespace dffm {

#ifndef DFFM_RS_THREADS
#define DFFM_RS_THREADS 256
#endif
constexpr int RS_THREADS = DFFM_RS_THREADS;
constexpr int RS_WARPS = RS_THREADS / 32;
constexpr int RS_MAXF = 128;

struct RsSmem {
  int off_ring, off_pair, off_xv, off_sidx, off_sval, off_lrw, off_red, off_bar, total;
  int row_stride;  // row bytes + 16 (rotates banks row to row)
  int nb;          // ring depth (examples)
};

__host__ __device__ inline RsSmem rs_smem_layout(int F, int P, int row_bytes, int nb) {
  RsSmem s;
  s.row_stride = row_bytes + 16;
  s.nb = nb;
  int o = 0;
  s.off_ring = o; o = align16(o + nb * F * s.row_stride);
  s.off_pair = o; o = align16(o + P * 2);
  s.off_xv = o; o = align16(o + (P + 1) * 4);
  s.off_sidx = o; o = align16(o + nb * F * 4);
  s.off_sval = o; o = align16(o + nb * F * 4);
  s.off_lrw = o; o = align16(o + nb * F * 4);
  s.off_red = o; o = align16(o + 2 * 3 * RS_WARPS * 8 + 16);
  s.off_bar = o; o = align16(o + nb * 8);
  s.total = o;
  return s;
}


// CTA-wide f64 sums of NV values per thread, results in every thread (one
// barrier; fixed order: deterministic)
template <int NV>
__device__ __forceinline__ void rs_block_sum(double* v, double* red, int& ctr) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < NV; ++q) v[q] = warp_sum(v[q]);
  double* slot = red + (++ctr & 1) * 3 * RS_WARPS;
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < NV; ++q) slot[q * RS_WARPS + warp] = v[q];
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    double t = lane < RS_WARPS ? slot[q * RS_WARPS + lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    v[q] = t;
  }
}

template <int K, typename T, int NB>
__global__ void __launch_bounds__(RS_THREADS, 2) fwd_rowstage_kernel(FwdParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int F = p.F, P = p.P, D = p.D;
  constexpr int SEGB = K * (int)sizeof(T);
  const int row_bytes = F * SEGB;
  const RsSmem L = rs_smem_layout(F, P, row_bytes, NB);
  const int RSB = L.row_stride;
  unsigned char* ring = smem + L.off_ring;
  uint16_t* pairtab = (uint16_t*)(smem + L.off_pair);
  float* xv = (float*)(smem + L.off_xv);
  int* sidx = (int*)(smem + L.off_sidx);     // [NB][F]
  float* sval = (float*)(smem + L.off_sval); // [NB][F]
  uint32_t* lrw = (uint32_t*)(smem + L.off_lrw);  // [NB][F] aligned words holding lr[j]
  double* red = (double*)(smem + L.off_red);
  uint64_t* full = (uint64_t*)(smem + L.off_bar);  // [NB] rows landed (F arrivals + tx bytes)
  const int tid = threadIdx.x;
  const T* lrt = (const T*)p.lr;
  const float bias = load_elem<T>(lrt + p.n_buckets, p.dlr);
  int bsc = 0;

  for (int f1 = tid; f1 < F; f1 += RS_THREADS) {
    const int base = f1 * F - f1 * (f1 + 1) / 2;
    for (int f2 = f1 + 1; f2 < F; ++f2) pairtab[base + f2 - f1 - 1] = (uint16_t)(f1 | (f2 << 8));
  }
  if (tid == 0) {
    for (int b = 0; b < NB; ++b) mbar_init(&full[b], F);
    mbar_fence_init();
  }
  __syncthreads();

  const int64_t my_n = p.n > blockIdx.x ? (p.n - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  // issue the copies of local example i into ring buffer i % NB: thread f < F
  // moves field f's whole row with one bulk copy (completion counted on
  // full[b]: F arrivals + the row bytes) and its lr word with a 4-byte
  // cp.async (one commit group per example, possibly empty)
  // idx / val of the next example to issue are loaded one issue ahead
  // (registers of threads f < F), so issuing never waits on global memory
  int nj = -1;
  float nx = 0.f;
  auto load_slot = [&](int64_t i) {
    if (i < my_n && tid < F) {
      const int64_t e = blockIdx.x + i * gridDim.x;
      nj = __ldg(p.idx + e * F + tid);
      nx = __ldg(p.val + e * F + tid);
    }
  };
  auto issue = [&](int64_t i) {
    if (i < my_n && tid < F) {
      const int b = (int)(i % NB);
      const int64_t e = blockIdx.x + i * gridDim.x;
      int j = nj;
      if (j >= p.n_buckets || j < -1) {  // ContractError (bad index)
        atomicMin((unsigned long long*)p.status,
                  (unsigned long long)status_key(p.status_base + e, DFFM_BLOCK_NONE,
                                                 DFFM_CONTRACT));
        j = -1;
      }
      sidx[b * F + tid] = j;
      sval[b * F + tid] = nx;
      if (j >= 0) {
        const uintptr_t a = (uintptr_t)(lrt + j) & ~(uintptr_t)3;
        cp_async4(&lrw[b * F + tid], (const void*)a);
        mbar_arrive_expect_tx(&full[b], (uint32_t)row_bytes);
        tma_load_1d(ring + ((size_t)b * F + tid) * RSB,
                    (const unsigned char*)p.ffm + (int64_t)j * row_bytes, (uint32_t)row_bytes,
                    &full[b]);
      } else {
        mbar_arrive(&full[b]);
      }
    }
    cp_async_commit();
    load_slot(i + 1);
  };

  load_slot(0);
#pragma unroll 1
  for (int i = 0; i < NB; ++i) issue(i);

  for (int64_t i = 0; i < my_n; ++i) {
    const int b = (int)(i % NB);
    cp_async_wait<NB - 1>();
    mbar_wait(&full[b], (uint32_t)((i / NB) & 1));
    __syncthreads();  // example i's rows, slots and lr words are in shared memory
    const int64_t e = blockIdx.x + i * gridDim.x;
    const int* si = sidx + b * F;
    const float* sv = sval + b * F;
    const unsigned char* rb = ring + (size_t)b * F * RSB;
    // ---- pairs (M:344-351)
    double s1 = 0.0;
    int pbad = 0;
    for (int pp = tid; pp < P; pp += RS_THREADS) {
      const uint32_t pr = pairtab[pp];
      const int f1 = pr & 0xFF, f2 = pr >> 8;
      float pv = 0.f;
      if (si[f1] >= 0 && si[f2] >= 0) {
        const float x1 = sv[f1], x2 = sv[f2];
        float a[K], bb[K];
        constexpr int PER = 16 / (int)sizeof(T);
#pragma unroll
        for (int c = 0; c < SEGB / 16; ++c) {
          unpack16<T>(*(const uint4*)(rb + f1 * RSB + f2 * SEGB + c * 16), a + c * PER, p.dffm);
          unpack16<T>(*(const uint4*)(rb + f2 * RSB + f1 * SEGB + c * 16), bb + c * PER, p.dffm);
        }
#pragma unroll
        for (int c = 0; c < K; ++c) pv = fmaf(x1 * a[c], x2 * bb[c], pv);
      }
      xv[1 + pp] = pv;
      s1 += (double)pv;
      pbad |= !isfinite(pv);
    }
    // ---- lr (M:327, M:338): thread f holds field f's term
    double lrs = 0.0;
    if (tid < F && si[tid] >= 0) {
      const uint32_t w = lrw[b * F + tid];
      float lv;
      if constexpr (sizeof(T) == 4) {
        lv = __uint_as_float(w);
      } else {
        const uint32_t h = (si[tid] & 1) ? (w >> 16) : (w & 0xFFFFu);  // little-endian half
        if constexpr (std::is_same<T, uint16_t>::value) lv = deq(h, p.dlr);
        else lv = __uint_as_float(h << 16);  // bf16
      }
      lrs = (double)sv[tid] * (double)lv;
    }
    double sums[3] = {s1, lrs, (double)pbad};
    rs_block_sum<3>(sums, red, bsc);  // its barrier also ends every read of ring buffer b
    issue(i + NB);                    // so the buffer refills while this example finishes
    const double psum = sums[0];
    double lr_out = (double)bias + sums[1];
    pbad = sums[2] != 0.0;
    // ---- MergeNorm (M:355-360)
    const double mu = (psum + lr_out) / D;
    double s2 = 0.0;
    for (int pp = tid; pp < P; pp += RS_THREADS) {
      const double d = (double)xv[1 + pp] - mu;
      s2 += d * d;
    }
    rs_block_sum<1>(&s2, red, bsc);
    s2 += (lr_out - mu) * (lr_out - mu);
    const double denom = sqrt(s2 / D) + 1e-6;
    const double rden = 1.0 / denom;  // one f64 division per example (<= 1 f64 ulp vs dividing)
    int mbad = 0;
    float* row = p.xout + e * p.Kp;
    for (int c = tid; c < p.Kp; c += RS_THREADS) {
      float m = 0.f;
      if (c == 0) m = (float)((lr_out - mu) * rden);
      else if (c < D) m = (float)(((double)xv[c] - mu) * rden);
      mbad |= !isfinite(m);
      row[c] = m;
    }
    mbad = __syncthreads_or(mbad);  // also: every xv / ring read of this example is done
    if (tid == 0) {
      p.rout[e] = lr_out + psum;
      p.fout[e] = (!isfinite(lr_out) ? 1 : 0) | (pbad ? 2 : 0) | (mbad ? 4 : 0);
    }
  }
  cp_async_wait<0>();
}

}  // namespace dffm
