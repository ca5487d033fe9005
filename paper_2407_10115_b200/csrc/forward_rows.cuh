// K1 v4 (default for F <= 32): row-coalesced warp-specialised DeepFFM forward.
//
// Same math as fwd_kernel (M:293-397).  Measured on B200 (tools/gather_bench):
// random 32-byte segment reads from a multi-GB table reach only ~1.2 TB/s of
// useful bandwidth, while row-coalesced reads reach ~6.5 TB/s.  The
// pair-per-lane gather (v1/v3) reads half of every row as scattered 32-byte
// sectors, so it is DRAM-inefficient no matter how many loads are in flight.
//
// Here every latent row is read whole and contiguously: lane g loads segment
// g of the row (one 128/256-bit load per lane, 24 x 32 B = 768 B contiguous
// per warp instruction at cfg2), W rows per wave in flight.  Rows arrive in
// field order, so lane g accumulates S[f][g] = sum_{j in f} x_j ffm[j][g][:]
// in registers; when field f is complete:
//   lanes g > f park S[f][g] in the warp's upper-triangle buffer U[pair(f,g)]
//   lanes g < f finish pair (g,f) = <U[pair(g,f)] = S[g][f], S[f][g]>   (M:344-351)
// so no (F,F,k) tensor is ever held and no latent byte is read twice.  The
// MergeNorm / MLP / sigmoid stages are those of K1 v3 (forward_ws.cuh).
#pragma once

#include "forward_ws.cuh"

namespace dffm {

constexpr int RW_NG = 8;  // gather warps
constexpr int RW_NM = 4;  // MLP warps
constexpr int RW_THREADS = (RW_NG + RW_NM) * 32;

struct RwSmem {
  int off_bar, off_sidx, off_sval, off_pres, off_U, off_exd,
      off_flag, off_X, off_Ha, off_Hb, total;
};

__host__ __device__ inline RwSmem rw_smem_layout(int F, int M, int P, int D, int k, int TE, int XS,
                                                 int hmax) {
  RwSmem s;
  const int FM = F * M;
  int o = 0;
  s.off_bar = o; o = align16(o + 8 * 4);
  s.off_sidx = o; o = align16(o + RW_NG * FM * 4);
  s.off_sval = o; o = align16(o + RW_NG * FM * 4);
  s.off_pres = o; o = align16(o + RW_NG * 32);
  s.off_U = o; o = align16(o + RW_NG * P * k * 4);
  s.off_exd = o; o = align16(o + 2 * 2 * TE * 8);
  s.off_flag = o; o = align16(o + 2 * TE * 4);
  s.off_X = o; o = align16(o + 2 * D * XS * 4);
  s.off_Ha = o; o = align16(o + hmax * XS * 4);
  s.off_Hb = o; o = align16(o + hmax * XS * 4);
  s.total = o;
  return s;
}

__device__ __forceinline__ int pair_pos(int a, int b, int F) {  // a < b, M:113-117 order
  return a * F - a * (a + 1) / 2 + (b - a - 1);
}

template <int K, int MU, typename T>
__global__ void __launch_bounds__(RW_THREADS, 1)
fwd_rows_kernel(FwdParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int SEGB = K * (int)sizeof(T);
  constexpr int NU = SEGB / 16;         // 16-byte chunks per segment
  constexpr int PER = 16 / (int)sizeof(T);
  constexpr int FW = (24 / NU) / MU > 0 ? (24 / NU) / MU : 1;  // fields per wave (~96 regs)
  const int F = p.F, FM = F * MU, P = p.P, D = p.D, TE = p.TE, XS = p.XS;
  const RwSmem L = rw_smem_layout(F, MU, P, D, K, TE, XS, p.hmax);
  uint64_t* xfull = (uint64_t*)(smem + L.off_bar);
  uint64_t* xempty = xfull + 2;
  double* exd_all = (double*)(smem + L.off_exd);
  int* flag_all = (int*)(smem + L.off_flag);
  float* X_all = (float*)(smem + L.off_X);
  float* Ha = (float*)(smem + L.off_Ha);
  float* Hb = (float*)(smem + L.off_Hb);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(&xfull[b], TE);
      mbar_init(&xempty[b], RW_NM);
    }
    mbar_fence_init();
  }
  __syncthreads();

  const int64_t ntiles = (p.n + TE - 1) / TE;
  const int64_t my_tiles = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t my_ex = my_tiles * TE;

  if (warp < RW_NG) {
    // ======================================================== gather warps
    int* sidx = (int*)(smem + L.off_sidx) + warp * FM;
    float* sval = (float*)(smem + L.off_sval) + warp * FM;
    unsigned char* spres = smem + L.off_pres + warp * 32;
    float* U = (float*)(smem + L.off_U) + (size_t)warp * P * K;
    const T* lrt = (const T*)p.lr;
    const T* ffm = (const T*)p.ffm;
    const float bias = load_elem<T>(lrt + p.n_buckets, p.dlr);
    constexpr int SPL = 4;  // FM <= 128
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
    for (int64_t le = warp; le < my_ex; le += RW_NG) {
      const int64_t ti = le / TE;
      const int el = (int)(le % TE);
      const int b = (int)(ti & 1);
      const int64_t e = ex_of(le);
      int cidx[SPL];
      float cval[SPL];
#pragma unroll
      for (int c = 0; c < SPL; ++c) { cidx[c] = nidx[c]; cval[c] = nval[c]; }
      prefetch(le + RW_NG);
      if (ti >= 2) mbar_wait(&xempty[b], (uint32_t)(((ti >> 1) - 1) & 1));
      float* X = X_all + b * D * XS;
      double* exd = exd_all + b * 2 * TE;
      int* flag = flag_all + b * TE;
      if (e >= p.n) {
        zero_column(X, exd, flag, el, TE, XS, D, lane);
      } else {
        // ---- stage slots; LR loads issued now, consumed at MergeNorm
        int bad = 0;
        float lrw[SPL];
#pragma unroll
        for (int c = 0; c < SPL; ++c) {
          const int s = lane + 32 * c;
          int j = cidx[c];
          if (j >= p.n_buckets || j < -1) { bad = 1; j = -1; }
          if (s < FM) { sidx[s] = j; sval[s] = j >= 0 ? cval[c] : 0.f; }
          lrw[c] = j >= 0 ? load_elem<T>(lrt + j, p.dlr) : 0.f;
          cidx[c] = j;
        }
        if (__any_sync(0xffffffffu, bad) && lane == 0)
          atomicMin((unsigned long long*)p.status,
                    (unsigned long long)status_key(p.status_base + e, DFFM_BLOCK_NONE,
                                                   DFFM_CONTRACT));
        __syncwarp();
        if (lane < F) {
          unsigned char pr = 0;
#pragma unroll
          for (int m = 0; m < MU; ++m) pr |= (sidx[lane * MU + m] >= 0);
          spres[lane] = pr;
        }
        __syncwarp();
        const bool my_pres = lane < F && spres[lane];
        const int gl = lane < F ? lane : 0;
        double s1 = 0.0;
        int pbad = 0;
        // ---- stream whole rows, FW fields (FW*MU slots) per wave; lane g
        // owns target segment g; one flush per completed field
        for (int f0 = 0; f0 < F; f0 += FW) {
          uint4 raw[FW][MU][NU];
#pragma unroll
          for (int fw = 0; fw < FW; ++fw) {
#pragma unroll
            for (int m = 0; m < MU; ++m) {
              const int f = f0 + fw;
              const int j = f < F ? sidx[f * MU + m] : -1;
              ldg_chunks_pred<NU>(ffm + ((int64_t)(j > 0 ? j : 0) * F + gl) * K,
                                  j >= 0 && lane < F, raw[fw][m]);
            }
          }
#pragma unroll
          for (int fw = 0; fw < FW; ++fw) {
            const int f = f0 + fw;
            if (f >= F) break;
            float acc[K];
#pragma unroll
            for (int c = 0; c < K; ++c) acc[c] = 0.f;
#pragma unroll
            for (int m = 0; m < MU; ++m) {
              const float x = sval[f * MU + m];
              float seg[K];
#pragma unroll
              for (int c = 0; c < NU; ++c) unpack16<T>(raw[fw][m][c], seg + c * PER, p.dffm);
#pragma unroll
              for (int c = 0; c < K; ++c) acc[c] = fmaf(x, seg[c], acc[c]);  // M:339
            }
            // field f complete: acc = S[f][lane]
            if (lane < F && lane > f) {
              float* u = U + pair_pos(f, lane, F) * K;
#pragma unroll
              for (int c = 0; c < K; c += 4)
                *(float4*)(u + c) = make_float4(acc[c], acc[c + 1], acc[c + 2], acc[c + 3]);
            } else if (lane < f) {
              const int pp = pair_pos(lane, f, F);
              float pv = 0.f;
              if (spres[f] && my_pres) {  // inactive pairs stay exactly 0 (M:346-351)
                const float* u = U + pp * K;  // S[lane][f]
#pragma unroll
                for (int c = 0; c < K; c += 4) {
                  const float4 a = *(const float4*)(u + c);
                  pv = fmaf(a.x, acc[c], pv);
                  pv = fmaf(a.y, acc[c + 1], pv);
                  pv = fmaf(a.z, acc[c + 2], pv);
                  pv = fmaf(a.w, acc[c + 3], pv);
                }
              }
              X[(pp + 1) * XS + el] = pv;
              s1 += (double)pv;
              pbad |= !isfinite(pv);
            }
          }
        }
        __syncwarp();
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
    const int mt = threadIdx.x - RW_NG * 32;
    for (int64_t ti = 0; ti < my_tiles; ++ti) {
      const int b = (int)(ti & 1);
      mbar_wait(&xfull[b], (uint32_t)((ti >> 1) & 1));
      const int64_t base = ((int64_t)blockIdx.x + ti * gridDim.x) * TE;
      mlp_warps_tile<RW_NM>(p, X_all + b * D * XS, exd_all + b * 2 * TE, flag_all + b * TE, Ha,
                            Hb, base, mt);
      if ((mt & 31) == 0) mbar_arrive(&xempty[b]);
    }
  }
}

}  // namespace dffm
