// K1 v5: TMA tile::gather4 fused DeepFFM forward (sm_100a), one CTA per SM.
//
// Same math as fwd_kernel (M:293-397).  Design drivers (profiles/r01_*):
//   * row-coalesced reads reach ~6.5 TB/s from HBM, scattered 32-B segment
//     reads only ~1.2 TB/s  -> fetch whole latent rows;
//   * per-row 1-D TMA copies cap at ~18 M rows/s per issuing warp
//     -> use the 2-D tensor-map gather4 form: ONE TMA op brings 4 whole rows
//        (4 x 768 B at cfg2) given their 4 bucket indices.
// Roles:
//   warp 0 (producer): two-stage lookahead.  Stage 1 TMA-copies example
//     le+LA's padded idx/val slots into its slot; stage 2 reads example le's
//     landed slots, compacts its valid rows, allocates ceil(rows/4) "quads" in a
//     shared-memory ring and issues one gather4 per quad on the example's
//     `full` mbarrier (expect_tx = quads x 4 rows x row bytes).
//   warps 1..NC (consumers): issue the example's LR loads, wait `full`, form
//     the P DiagMask pairs from the ring (pair order along diagonals f2-f1 so
//     both sides' segment reads are bank-conflict free), release the ring
//     quads and the slot (`empty`) right after the pairs, then MergeNorm into
//     the double-buffered X tile and arrive on `xfull`.
//   MLP warps: the tile GEMMs / logit / sigmoid of K1 v3 (mlp_warps_tile).
// Requirements (host-checked; else K1 v3): F*k <= 256 elements (one TMA box
// per row), k*sizeof(T) % 16 == 0, F*M % 4 == 0 and <= 128, hidden % 4 == 0.
#pragma once

#include <cuda.h>

#include "forward_tma.cuh"
#include "forward_ws.cuh"

namespace dffm {

#ifndef DFFM_G4_NC
#define DFFM_G4_NC 10
#endif
constexpr int G4_NC = DFFM_G4_NC;  // consumer warps
constexpr int G4_NM = 4;           // MLP warps
constexpr int G4_THREADS = (1 + G4_NC + G4_NM) * 32;
constexpr int G4_NS = 16;          // example slots
constexpr int G4_LA = 6;           // idx/val lookahead (examples)

struct G4Params {
  FwdParams f;
  int row_bytes;
  int quad_bytes;
  int ring_quads;
};

struct G4Smem {
  int off_bar, off_pcode, off_ppos, off_sidx, off_sval, off_srow, off_end, off_valid, off_plist,
      off_pres, off_exd, off_flag, off_X, off_Ha, off_Hb, off_ring, total;
};

__host__ __device__ inline G4Smem g4_smem_layout(int F, int M, int P, int D, int TE, int XS,
                                                 int hmax, int quad_bytes, int ring_quads) {
  G4Smem s;
  const int FM = F * M;
  int o = 0;
  s.off_bar = o; o = align16(o + 8 * (3 * G4_NS + 4));
  s.off_pcode = o; o = align16(o + P * 2);
  s.off_ppos = o; o = align16(o + P * 2);
  s.off_sidx = o; o = align16(o + G4_NS * FM * 4);
  s.off_sval = o; o = align16(o + G4_NS * FM * 4);
  s.off_srow = o; o = align16(o + G4_NS * FM * 2);
  s.off_end = o; o = align16(o + G4_NS * 8);
  s.off_valid = o; o = align16(o + G4_NS * 4);
  s.off_plist = o; o = align16(o + (FM + 4) * 4);
  s.off_pres = o; o = align16(o + G4_NC * F);
  s.off_exd = o; o = align16(o + 2 * 2 * TE * 8);
  s.off_flag = o; o = align16(o + 2 * TE * 4);
  s.off_X = o; o = align16(o + 2 * D * XS * 4);
  s.off_Ha = o; o = align16(o + hmax * XS * 4);
  s.off_Hb = o; o = align16(o + hmax * XS * 4);
  o = (o + 127) & ~127;
  s.off_ring = o; o += ring_quads * quad_bytes;
  s.total = o;
  return s;
}

// gather4: rows r0..r3 of the 2-D tensor map (whole rows, box = row), 4 x box
// bytes land contiguously at dst; completion counted on bar.
__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* tm, int col, int r0,
                                            int r1, int r2, int r3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3),
      "r"(smem_u32(bar))
      : "memory");
}

template <int K, typename T>
__global__ void __launch_bounds__(G4_THREADS, 1)
fwd_g4_kernel(const __grid_constant__ CUtensorMap tm, G4Params q) {
  extern __shared__ __align__(128) unsigned char smem[];
  const FwdParams& p = q.f;
  const int F = p.F, M = p.M, FM = F * M, P = p.P, D = p.D, TE = p.TE, XS = p.XS;
  const G4Smem L = g4_smem_layout(F, M, P, D, TE, XS, p.hmax, q.quad_bytes, q.ring_quads);
  uint64_t* full = (uint64_t*)(smem + L.off_bar);
  uint64_t* empty = full + G4_NS;
  uint64_t* metaf = empty + G4_NS;
  uint64_t* xfull = metaf + G4_NS;
  uint64_t* xempty = xfull + 2;
  uint16_t* pcode = (uint16_t*)(smem + L.off_pcode);
  uint16_t* ppos = (uint16_t*)(smem + L.off_ppos);
  int* sidx_all = (int*)(smem + L.off_sidx);
  float* sval_all = (float*)(smem + L.off_sval);
  int16_t* srow_all = (int16_t*)(smem + L.off_srow);
  int64_t* slot_end = (int64_t*)(smem + L.off_end);
  int* svalid = (int*)(smem + L.off_valid);
  int* plist = (int*)(smem + L.off_plist);
  double* exd_all = (double*)(smem + L.off_exd);
  int* flag_all = (int*)(smem + L.off_flag);
  float* X_all = (float*)(smem + L.off_X);
  float* Ha = (float*)(smem + L.off_Ha);
  float* Hb = (float*)(smem + L.off_Hb);
  unsigned char* ring = smem + L.off_ring;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int RQ = q.ring_quads, QB = q.quad_bytes, RB = q.row_bytes;
  constexpr int SEGB = K * (int)sizeof(T);

  if (threadIdx.x == 0) {
    // DiagMask pairs (M:113-117) enumerated along diagonals d = f2 - f1: 32
    // consecutive lanes then read consecutive segment indices on BOTH sides
    int t = 0;
    for (int d = 1; d < F; ++d)
      for (int f1 = 0; f1 + d < F; ++f1, ++t) {
        const int f2 = f1 + d;
        pcode[t] = (uint16_t)(f1 | (f2 << 8));
        ppos[t] = (uint16_t)(f1 * F - f1 * (f1 + 1) / 2 + (f2 - f1 - 1));
      }
    for (int s = 0; s < G4_NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&metaf[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&xfull[b], TE);
      mbar_init(&xempty[b], G4_NM);
    }
    mbar_fence_init();
  }
  __syncthreads();

  const int64_t ntiles = (p.n + TE - 1) / TE;
  const int64_t my_tiles = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t my_ex = my_tiles * TE;
  const T* lrt = (const T*)p.lr;
  auto ex_of = [&](int64_t le) {
    return ((int64_t)blockIdx.x + (le / TE) * gridDim.x) * TE + le % TE;
  };

  if (warp == 0) {
    // ======================================================== producer
    const uint32_t slot_bytes = (uint32_t)FM * 4u;
    int64_t head = 0, tail = 0, ole = 0;  // ring counters in quads
    for (int64_t step = 0; step < my_ex + G4_LA; ++step) {
      const int64_t le1 = step;
      if (le1 < my_ex && lane == 0) {
        const int s1 = (int)(le1 % G4_NS);
        if (le1 >= G4_NS) mbar_wait(&empty[s1], (uint32_t)(((le1 / G4_NS) - 1) & 1));
        const int64_t e1 = ex_of(le1);
        const bool v1 = e1 < p.n;
        svalid[s1] = v1;
        mbar_arrive_expect_tx(&metaf[s1], v1 ? 2u * slot_bytes : 0u);
        if (v1) {
          tma_load_1d(sidx_all + s1 * FM, p.idx + e1 * FM, slot_bytes, &metaf[s1]);
          tma_load_1d(sval_all + s1 * FM, p.val + e1 * FM, slot_bytes, &metaf[s1]);
        }
      }
      __syncwarp();
      const int64_t le = step - G4_LA;
      if (le < 0) continue;
      const int s = (int)(le % G4_NS);
      mbar_wait(&metaf[s], (uint32_t)((le / G4_NS) & 1));
      const int64_t e = ex_of(le);
      const int* sidx = sidx_all + s * FM;
      const bool valid = svalid[s];
      int ci[4];
      int cnt = 0, bad = 0;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int sl = lane + 32 * c;
        ci[c] = (valid && sl < FM) ? sidx[sl] : -1;
        if (ci[c] >= p.n_buckets || ci[c] < -1) { bad = 1; ci[c] = -1; }
        cnt += ci[c] >= 0;
      }
      if (__any_sync(0xffffffffu, bad) && lane == 0)
        atomicMin((unsigned long long*)p.status,
                  (unsigned long long)status_key(p.status_base + e, DFFM_BLOCK_NONE,
                                                 DFFM_CONTRACT));
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      const int total = __shfl_sync(0xffffffffu, incl, 31);
      const int nq = (total + 3) >> 2;
      // retire bookkeeping of the example whose slot this one reuses (its
      // `empty` already completed in stage 1), then wait for ring space
      while (ole + G4_NS <= le || head + nq - tail > RQ) {
        mbar_wait(&empty[ole % G4_NS], (uint32_t)((ole / G4_NS) & 1));
        tail = slot_end[ole % G4_NS];
        ++ole;
      }
      int16_t* srow = srow_all + s * FM;
      int rank = incl - cnt;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int sl = lane + 32 * c;
        if (sl < FM) {
          if (ci[c] >= 0) {
            const int qd = (int)((head + (rank >> 2)) % RQ);
            srow[sl] = (int16_t)(qd * 4 + (rank & 3));
            plist[rank] = ci[c];
            ++rank;
          } else {
            srow[sl] = (int16_t)-1;
          }
        }
      }
      __syncwarp();
      if (lane == 0) {
        for (int r = total; r < nq * 4; ++r) plist[r] = plist[total - 1];  // pad the last quad
        slot_end[s] = head + nq;
        mbar_arrive_expect_tx(&full[s], (uint32_t)nq * (uint32_t)QB);
      }
      __syncwarp();
      for (int u = lane; u < nq; u += 32) {
        const int qd = (int)((head + u) % RQ);
        tma_gather4(ring + (size_t)qd * QB, &tm, 0, plist[4 * u], plist[4 * u + 1],
                    plist[4 * u + 2], plist[4 * u + 3], &full[s]);
      }
      __syncwarp();  // plist is reused by the next example
      head += nq;
    }
  } else if (warp <= G4_NC) {
    // ======================================================== consumers
    const int cw = warp - 1;
    unsigned char* spres = smem + L.off_pres + cw * F;
    const float bias = load_elem<T>(lrt + p.n_buckets, p.dlr);
    for (int64_t le = cw; le < my_ex; le += G4_NC) {
      const int s = (int)(le % G4_NS);
      const int64_t ti = le / TE;
      const int el = (int)(le % TE);
      const int b = (int)(ti & 1);
      const uint32_t ph = (uint32_t)((le / G4_NS) & 1);
      mbar_wait(&metaf[s], ph);
      const int* sidx = sidx_all + s * FM;
      const float* sval = sval_all + s * FM;
      // LR loads now (slots visible); consumed after the pairs
      float lrw[4], xv[4];
      int jv[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int sl = lane + 32 * c;
        int j = (svalid[s] && sl < FM) ? sidx[sl] : -1;
        if (j >= p.n_buckets || j < -1) j = -1;
        jv[c] = j;
        xv[c] = j >= 0 ? sval[sl] : 0.f;
        lrw[c] = j >= 0 ? load_elem<T>(lrt + j, p.dlr) : 0.f;
      }
      if (ti >= 2) mbar_wait(&xempty[b], (uint32_t)(((ti >> 1) - 1) & 1));
      mbar_wait(&full[s], ph);
      float* X = X_all + b * D * XS;
      double* exd = exd_all + b * 2 * TE;
      int* flag = flag_all + b * TE;
      if (!svalid[s]) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        zero_column(X, exd, flag, el, TE, XS, D, lane);
      } else {
        const int16_t* srow = srow_all + s * FM;
        for (int f = lane; f < F; f += 32) {
          unsigned char pr = 0;
          for (int m = 0; m < M; ++m) pr |= (srow[f * M + m] >= 0);
          spres[f] = pr;
        }
        __syncwarp();
        double s1 = 0.0;
        int pbad = 0;
        for (int t = lane; t < P; t += 32) {
          const uint32_t pc = pcode[t];
          const int f1 = pc & 0xFF, f2 = pc >> 8;
          float pv = 0.f;
          if (spres[f1] & spres[f2]) {  // inactive pairs stay exactly 0 (M:346-351)
            float a[K], bb[K];
#pragma unroll
            for (int c = 0; c < K; ++c) { a[c] = 0.f; bb[c] = 0.f; }
            for (int m = 0; m < M; ++m) {
              const int ra = srow[f1 * M + m];
              if (ra >= 0) {
                float seg[K];
                lds_seg<K, T>(ring + (size_t)(ra >> 2) * QB + (ra & 3) * RB + f2 * SEGB, seg,
                              p.dffm);
                const float x = sval[f1 * M + m];
#pragma unroll
                for (int c = 0; c < K; ++c) a[c] = fmaf(x, seg[c], a[c]);  // S[f1][f2] (M:339)
              }
              const int rb = srow[f2 * M + m];
              if (rb >= 0) {
                float seg[K];
                lds_seg<K, T>(ring + (size_t)(rb >> 2) * QB + (rb & 3) * RB + f1 * SEGB, seg,
                              p.dffm);
                const float x = sval[f2 * M + m];
#pragma unroll
                for (int c = 0; c < K; ++c) bb[c] = fmaf(x, seg[c], bb[c]);  // S[f2][f1]
              }
            }
#pragma unroll
            for (int c = 0; c < K; ++c) pv = fmaf(a[c], bb[c], pv);
          }
          X[(ppos[t] + 1) * XS + el] = pv;
          s1 += (double)pv;
          pbad |= !isfinite(pv);
        }
        __syncwarp();  // ring quads + slot are free again
        if (lane == 0) mbar_arrive(&empty[s]);
        double lrs = 0.0;
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (jv[c] >= 0) lrs += (double)xv[c] * (double)lrw[c];  // M:338
        const double lr_out = (double)bias + warp_sum(lrs);      // M:327
        merge_finish(X, exd, flag, el, TE, XS, P, D, lane, lr_out, s1, pbad);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&xfull[b]);
    }
  } else {
    // ======================================================== MLP warps
    const int mt = threadIdx.x - (1 + G4_NC) * 32;
    for (int64_t ti = 0; ti < my_tiles; ++ti) {
      const int b = (int)(ti & 1);
      mbar_wait(&xfull[b], (uint32_t)((ti >> 1) & 1));
      const int64_t base = ((int64_t)blockIdx.x + ti * gridDim.x) * TE;
      mlp_warps_tile<G4_NM>(p, X_all + b * D * XS, exd_all + b * 2 * TE, flag_all + b * TE, Ha,
                            Hb, base, mt);
      if ((mt & 31) == 0) mbar_arrive(&xempty[b]);
    }
  }
}

}  // namespace dffm
