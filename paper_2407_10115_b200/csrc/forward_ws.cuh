// K1 v3 (default): warp-specialised fused DeepFFM forward, one CTA per SM.
//
// Same math as fwd_kernel (forward_kernel.cuh; M:293-397).  Roles:
//   WS_NG gather warps: each owns one example at a time -- stages its padded
//     slots, gathers the LR weights, forms the DiagMask pairs with
//     branch-free predicated 256-bit row-segment loads (every slot load of a
//     pair in flight together), reduces MergeNorm in f64 and writes the
//     standardised column into a double-buffered X tile; then arrives on the
//     tile's `xfull` mbarrier.  Gather warps never stop for the MLP: they
//     only wait when both X buffers are still being consumed.
//   WS_NM MLP warps: per tile, register-tiled GEMMs (4 outputs x 4 examples
//     per thread) through the hidden layers with the weights L1-resident
//     (the CTA's shared footprint is kept small for that), the output unit,
//     residual logit and clamped sigmoid; then release the buffer (`xempty`).
// This removes v1's CTA-wide barrier between gathering and the MLP, and the
// single-producer issue ceiling of the TMA-ring variant (forward_tma.cuh).
#pragma once

#include "forward_kernel.cuh"

namespace dffm {

#ifndef DFFM_WS_NG
#define DFFM_WS_NG 16
#endif
constexpr int WS_NG = DFFM_WS_NG;
constexpr int WS_NM = 4;
constexpr int WS_THREADS = (WS_NG + WS_NM) * 32;

struct WsSmem {
  int off_bar, off_pair, off_sidx, off_sval, off_pres, off_exd, off_flag, off_X, off_Ha, off_Hb,
      total;
};

__host__ __device__ inline WsSmem ws_smem_layout(int F, int M, int P, int D, int TE, int XS,
                                                 int hmax) {
  WsSmem s;
  const int FM = F * M;
  int o = 0;
  s.off_bar = o; o = align16(o + 8 * 4);
  s.off_pair = o; o = align16(o + P * 2);
  s.off_sidx = o; o = align16(o + WS_NG * FM * 4);
  s.off_sval = o; o = align16(o + WS_NG * FM * 4);
  s.off_pres = o; o = align16(o + WS_NG * F);
  s.off_exd = o; o = align16(o + 2 * 2 * TE * 8);
  s.off_flag = o; o = align16(o + 2 * TE * 4);
  s.off_X = o; o = align16(o + 2 * D * XS * 4);
  s.off_Ha = o; o = align16(o + hmax * XS * 4);
  s.off_Hb = o; o = align16(o + hmax * XS * 4);
  s.total = o;
  return s;
}

template <int K, int MU, typename T>
__global__ void __launch_bounds__(WS_THREADS, 1)
fwd_ws_kernel(FwdParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int F = p.F, M = p.M, FM = F * M, P = p.P, D = p.D, TE = p.TE, XS = p.XS;
  const WsSmem L = ws_smem_layout(F, M, P, D, TE, XS, p.hmax);
  uint64_t* xfull = (uint64_t*)(smem + L.off_bar);
  uint64_t* xempty = xfull + 2;
  uint16_t* pairtab = (uint16_t*)(smem + L.off_pair);
  double* exd_all = (double*)(smem + L.off_exd);
  int* flag_all = (int*)(smem + L.off_flag);
  float* X_all = (float*)(smem + L.off_X);
  float* Ha = (float*)(smem + L.off_Ha);
  float* Hb = (float*)(smem + L.off_Hb);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int KA = K ? K : 32;
  const int k = K ? K : p.k;

  for (int f1 = threadIdx.x; f1 < F; f1 += WS_THREADS) {
    const int base = f1 * F - f1 * (f1 + 1) / 2;
    for (int f2 = f1 + 1; f2 < F; ++f2) pairtab[base + f2 - f1 - 1] = (uint16_t)(f1 | (f2 << 8));
  }
  if (threadIdx.x == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(&xfull[b], TE);
      mbar_init(&xempty[b], WS_NM);
    }
    mbar_fence_init();
  }
  __syncthreads();

  const int64_t ntiles = (p.n + TE - 1) / TE;
  const int64_t my_tiles = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t my_ex = my_tiles * TE;

  if (warp < WS_NG) {
    // ======================================================== gather warps
    int* sidx = (int*)(smem + L.off_sidx) + warp * FM;
    float* sval = (float*)(smem + L.off_sval) + warp * FM;
    unsigned char* spres = smem + L.off_pres + warp * F;
    const T* lrt = (const T*)p.lr;
    const float bias = load_elem<T>(lrt + p.n_buckets, p.dlr);
    // Software pipeline across this warp's examples: the NEXT example's
    // padded slots are loaded into registers while the current one's pairs
    // are formed, and each example's LR loads are issued at its start but
    // consumed only at MergeNorm, so only the pair gathers sit on the
    // critical path.  FM <= 128 -> at most 4 slots per lane.
    constexpr int SPL = 4;
    int nidx[SPL];
    float nval[SPL];
    auto ex_of = [&](int64_t le) {
      return ((int64_t)blockIdx.x + (le / TE) * gridDim.x) * TE + le % TE;
    };
    auto prefetch = [&](int64_t le) {
      const int64_t e = le < my_ex ? ex_of(le) : p.n;
#pragma unroll
      for (int c = 0; c < SPL; ++c) {
        const int s = lane + 32 * c;
        const bool ok = e < p.n && s < FM;
        nidx[c] = ok ? __ldg(p.idx + e * FM + s) : -1;
        nval[c] = ok ? __ldg(p.val + e * FM + s) : 0.f;
      }
    };
    prefetch(warp);
    for (int64_t le = warp; le < my_ex; le += WS_NG) {
      const int64_t ti = le / TE;
      const int el = (int)(le % TE);
      const int b = (int)(ti & 1);
      const int64_t e = ex_of(le);
      int cidx[SPL];
      float cval[SPL];
#pragma unroll
      for (int c = 0; c < SPL; ++c) { cidx[c] = nidx[c]; cval[c] = nval[c]; }
      prefetch(le + WS_NG);
      if (ti >= 2) mbar_wait(&xempty[b], (uint32_t)(((ti >> 1) - 1) & 1));
      float* X = X_all + b * D * XS;
      double* exd = exd_all + b * 2 * TE;
      int* flag = flag_all + b * TE;
      if (e >= p.n) {
        zero_column(X, exd, flag, el, TE, XS, D, lane);
      } else {
        int bad = 0;
        float lrw[SPL];
#pragma unroll
        for (int c = 0; c < SPL; ++c) {
          const int s = lane + 32 * c;
          int j = cidx[c];
          if (j >= p.n_buckets || j < -1) { bad = 1; j = -1; }
          if (s < FM) { sidx[s] = j; sval[s] = cval[c]; }
          lrw[c] = j >= 0 ? load_elem<T>(lrt + j, p.dlr) : 0.f;  // consumed at merge time
          cidx[c] = j;
        }
        __syncwarp();
        for (int f = lane; f < F; f += 32) {
          unsigned char pr = 0;
          for (int m = 0; m < M; ++m) pr |= (sidx[f * M + m] >= 0);
          spres[f] = pr;
        }
        if (__any_sync(0xffffffffu, bad) && lane == 0)
          atomicMin((unsigned long long*)p.status,
                    (unsigned long long)status_key(p.status_base + e, DFFM_BLOCK_NONE,
                                                   DFFM_CONTRACT));
        __syncwarp();
        double s1 = 0.0;
        int pbad = 0;
        if constexpr (MU == 1 && K > 0 && (K * sizeof(T)) % 16 == 0) {
          // single-slot fields: two pairs per lane, loads first (same sums, same order)
          for (int pp = lane; pp < P; pp += 64) {
            const int pq = pp + 32;
            const uint32_t pr = pairtab[pp];
            const int f1 = pr & 0xFF, f2 = pr >> 8;
            int g1 = 0, g2 = 0;
            bool actq = false;
            if (pq < P) {
              const uint32_t pr2 = pairtab[pq];
              g1 = pr2 & 0xFF;
              g2 = pr2 >> 8;
              actq = spres[g1] & spres[g2];
            }
            const float2 v = pair_dot_x2<K, T>(p, sidx, sval, spres[f1] & spres[f2], f1, f2,
                                               actq, g1, g2);
            X[(pp + 1) * XS + el] = v.x;
            s1 += (double)v.x;
            pbad |= !isfinite(v.x);
            if (pq < P) {
              X[(pq + 1) * XS + el] = v.y;
              s1 += (double)v.y;
              pbad |= !isfinite(v.y);
            }
          }
        } else
        for (int pp = lane; pp < P; pp += 32) {
          const uint32_t pr = pairtab[pp];
          const int f1 = pr & 0xFF, f2 = pr >> 8;
          float pv = 0.f;
          if (spres[f1] & spres[f2]) {  // inactive pairs stay exactly 0 (M:346-351)
            if constexpr (K > 0 && MU > 0 && (K * sizeof(T)) % 16 == 0) {
              pv = pair_dot_batched<K, MU, T>(p, sidx + f1 * M, sval + f1 * M, sidx + f2 * M,
                                              sval + f2 * M, M, f1, f2);
            } else {
              float a[KA], bb[KA];
#pragma unroll
              for (int c = 0; c < KA; ++c) { a[c] = 0.f; bb[c] = 0.f; }
              accum_slots<K, MU, T>(p, sidx + f1 * M, sval + f1 * M, M, f2, a);
              accum_slots<K, MU, T>(p, sidx + f2 * M, sval + f2 * M, M, f1, bb);
#pragma unroll
              for (int c = 0; c < KA; ++c)
                if (K || c < k) pv = fmaf(a[c], bb[c], pv);
            }
          }
          X[(pp + 1) * XS + el] = pv;
          s1 += (double)pv;
          pbad |= !isfinite(pv);
        }
        double lrs = 0.0;
#pragma unroll
        for (int c = 0; c < SPL; ++c)
          if (cidx[c] >= 0) lrs += (double)cval[c] * (double)lrw[c];  // M:338
        const double lr_out = (double)bias + warp_sum(lrs);          // M:327
        merge_finish(X, exd, flag, el, TE, XS, P, D, lane, lr_out, s1, pbad);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&xfull[b]);
    }
  } else {
    // ======================================================== MLP warps
    const int mt = threadIdx.x - WS_NG * 32;
    for (int64_t ti = 0; ti < my_tiles; ++ti) {
      const int b = (int)(ti & 1);
      mbar_wait(&xfull[b], (uint32_t)((ti >> 1) & 1));
      const int64_t base = ((int64_t)blockIdx.x + ti * gridDim.x) * TE;
      mlp_warps_tile<WS_NM>(p, X_all + b * D * XS, exd_all + b * 2 * TE, flag_all + b * TE, Ha,
                            Hb, base, mt);
      if ((mt & 31) == 0) mbar_arrive(&xempty[b]);
    }
  }
}

}  // namespace dffm
