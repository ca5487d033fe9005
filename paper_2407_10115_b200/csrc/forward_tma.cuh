// K1 v2: warp-specialised, TMA-fed fused DeepFFM forward (sm_100a).
//
// Same math as fwd_kernel (forward_kernel.cuh) -- gather, field-aware latent
// sums, DiagMask pairs, MergeNorm, MLP, residual logit, clamped sigmoid
// (M:293-397) -- but with HBM latency fully decoupled from compute:
//
//   warp 0 (producer): per example, reads the padded idx/val slots (one
//     example ahead, in registers), allocates ring rows, and issues one 1-D
//     TMA bulk copy (cp.async.bulk ... mbarrier::complete_tx) per feature:
//     the feature's whole [F][k] latent row (768 B at cfg2) lands in a
//     shared-memory ring.  The 4-byte LR weights ride along as cp.async
//     copies that arrive on the same mbarrier.  Up to NS examples (bounded
//     by the ring) are in flight per SM.
//   warps 1..NC (consumers): one example each at a time; wait on the
//     example's "full" barrier, form the P pair dots from the ring rows in
//     shared memory (each row byte was fetched from HBM exactly once, in one
//     contiguous transfer), reduce MergeNorm statistics in f64, write the
//     standardised column into the double-buffered X tile, release the
//     slot ("empty") and arrive on the tile's "xfull" barrier.
//   warps NC+1.. (MLP): per tile of TE examples, register-tiled GEMMs
//     (4 outputs x 4 examples per thread) through the hidden layers, the
//     output unit, logit and sigmoid; then release the X buffer ("xempty").
//
// One CTA per SM, persistent over tiles.  Requirements (host-checked; other
// shapes take fwd_kernel): segment bytes k*sizeof(T) a multiple of 16, F*M
// <= 128, hidden sizes multiples of 4.
#pragma once

#include "forward_kernel.cuh"

namespace dffm {

constexpr int TMA_NC = 12;                          // consumer warps
constexpr int TMA_NM = 4;                           // MLP warps
constexpr int TMA_WARPS = 1 + TMA_NC + TMA_NM;
constexpr int TMA_THREADS = TMA_WARPS * 32;
constexpr int TMA_NS = 16;                          // example slots in flight
constexpr int TMA_MAX_FM = 128;                     // padded slots per example
constexpr int TMA_LA = TMA_NS / 2;                  // producer idx/val lookahead

struct TmaParams {
  FwdParams f;
  int row_bytes;  // F * k * sizeof(T)
  int rs;         // ring row stride (row_bytes + 16: rotates banks row to row)
  int ring_rows;
  int copy_mode;  // 0 = TMA bulk row copies, 1 = warp-cooperative cp.async 16 B
};

struct TmaSmem {
  int off_bar, off_pair, off_sidx, off_sval, off_srow, off_slr, off_end, off_valid, off_plist, off_pres,
      off_exd, off_flag, off_X, off_Ha, off_Hb, off_ring, total;
};

__host__ __device__ inline TmaSmem tma_smem_layout(int F, int M, int P, int D, int TE, int XS,
                                                   int hmax, int rs, int ring_rows) {
  TmaSmem s;
  const int FM = F * M;
  int o = 0;
  s.off_bar = o; o = align16(o + 8 * (3 * TMA_NS + 4));
  s.off_pair = o; o = align16(o + P * 2);
  s.off_sidx = o; o = align16(o + TMA_NS * FM * 4);
  s.off_sval = o; o = align16(o + TMA_NS * FM * 4);
  s.off_srow = o; o = align16(o + TMA_NS * FM * 2);
  s.off_slr = o; o = align16(o + TMA_NS * FM * 4);
  s.off_end = o; o = align16(o + TMA_NS * 8);
  s.off_valid = o; o = align16(o + TMA_NS * 4);
  s.off_plist = o; o = align16(o + FM * 8);
  s.off_pres = o; o = align16(o + TMA_NC * F);
  s.off_exd = o; o = align16(o + 2 * 2 * TE * 8);
  s.off_flag = o; o = align16(o + 2 * TE * 4);
  s.off_X = o; o = align16(o + 2 * D * XS * 4);
  s.off_Ha = o; o = align16(o + hmax * XS * 4);
  s.off_Hb = o; o = align16(o + hmax * XS * 4);
  o = (o + 127) & ~127;
  s.off_ring = o; o += ring_rows * rs;
  s.total = o;
  return s;
}

template <typename T>
__device__ __forceinline__ float lr_from_word(uint32_t w, int j, const Deq& d);
template <>
__device__ __forceinline__ float lr_from_word<float>(uint32_t w, int, const Deq&) {
  return __uint_as_float(w);
}
template <>
__device__ __forceinline__ float lr_from_word<__nv_bfloat16>(uint32_t w, int j, const Deq&) {
  return (j & 1) ? bf16hi(w) : bf16lo(w);
}
template <>
__device__ __forceinline__ float lr_from_word<uint16_t>(uint32_t w, int j, const Deq& d) {
  return deq((j & 1) ? (w >> 16) : (w & 0xFFFF), d);
}

// segment of K elements of T from shared memory -> floats (16-byte chunks)
template <int K, typename T>
__device__ __forceinline__ void lds_seg(const unsigned char* p, float* o, const Deq& d) {
  constexpr int BYTES = K * (int)sizeof(T);
  constexpr int PER = 16 / sizeof(T);
#pragma unroll
  for (int c = 0; c < BYTES / 16; ++c) {
    const uint4 u = *(const uint4*)(p + 16 * c);
    unpack16<T>(u, o + c * PER, d);
  }
}

template <int K, typename T>
__global__ void __launch_bounds__(TMA_THREADS, 1)
fwd_tma_kernel(TmaParams q) {
  extern __shared__ __align__(128) unsigned char smem[];
  const FwdParams& p = q.f;
  const int F = p.F, M = p.M, FM = F * M, P = p.P, D = p.D, TE = p.TE, XS = p.XS;
  const TmaSmem L = tma_smem_layout(F, M, P, D, TE, XS, p.hmax, q.rs, q.ring_rows);
  uint64_t* full = (uint64_t*)(smem + L.off_bar);
  uint64_t* empty = full + TMA_NS;
  uint64_t* metaf = empty + TMA_NS;
  uint64_t* xfull = metaf + TMA_NS;
  uint64_t* xempty = xfull + 2;
  uint16_t* pairtab = (uint16_t*)(smem + L.off_pair);
  int* sidx_all = (int*)(smem + L.off_sidx);
  float* sval_all = (float*)(smem + L.off_sval);
  int16_t* srow_all = (int16_t*)(smem + L.off_srow);
  uint32_t* slr_all = (uint32_t*)(smem + L.off_slr);
  int64_t* slot_end = (int64_t*)(smem + L.off_end);
  int* svalid = (int*)(smem + L.off_valid);
  int2* plist = (int2*)(smem + L.off_plist);
  double* exd_all = (double*)(smem + L.off_exd);
  int* flag_all = (int*)(smem + L.off_flag);
  float* X_all = (float*)(smem + L.off_X);
  float* Ha = (float*)(smem + L.off_Ha);
  float* Hb = (float*)(smem + L.off_Hb);
  unsigned char* ring = smem + L.off_ring;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int RR = q.ring_rows, RS = q.rs;
  constexpr int SEGB = K * (int)sizeof(T);

  for (int f1 = threadIdx.x; f1 < F; f1 += TMA_THREADS) {
    const int base = f1 * F - f1 * (f1 + 1) / 2;
    for (int f2 = f1 + 1; f2 < F; ++f2) pairtab[base + f2 - f1 - 1] = (uint16_t)(f1 | (f2 << 8));
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < TMA_NS; ++s) {
      mbar_init(&full[s], 1 + 32);  // producer lane 0 (expect_tx) + 32 cp.async arrivals
      mbar_init(&empty[s], 1);
      mbar_init(&metaf[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&xfull[b], TE);
      mbar_init(&xempty[b], TMA_NM);
    }
    mbar_fence_init();
  }
  __syncthreads();

  const int64_t ntiles = (p.n + TE - 1) / TE;
  const int64_t my_tiles = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t my_ex = my_tiles * TE;
  const T* lrt = (const T*)p.lr;
  const float bias = load_elem<T>(lrt + p.n_buckets, p.dlr);

  if (warp == 0) {
    // ======================================================== producer
    // Two-stage lookahead: stage 1 TMA-copies example (le+LA)'s padded
    // idx/val slots into its slot; stage 2 reads example le's (landed) slots,
    // allocates ring rows and issues one bulk copy per feature row plus the
    // cp.async LR words.  No dependent global load on the issue path.
    const T* ffm = (const T*)p.ffm;
    const int64_t row_elems = (int64_t)F * K;
    const uint32_t slot_bytes = (uint32_t)FM * 4u;
    int64_t head = 0, tail = 0, ole = 0;
    for (int64_t step = 0; step < my_ex + TMA_LA; ++step) {
      const int64_t le1 = step;
      if (le1 < my_ex && lane == 0) {
        const int s1 = (int)(le1 % TMA_NS);
        if (le1 >= TMA_NS) mbar_wait(&empty[s1], (uint32_t)(((le1 / TMA_NS) - 1) & 1));
        const int64_t e1 = ((int64_t)blockIdx.x + (le1 / TE) * gridDim.x) * TE + le1 % TE;
        const bool v1 = e1 < p.n;
        svalid[s1] = v1;
        mbar_arrive_expect_tx(&metaf[s1], v1 ? 2u * slot_bytes : 0u);
        if (v1) {
          tma_load_1d(sidx_all + s1 * FM, p.idx + e1 * FM, slot_bytes, &metaf[s1]);
          tma_load_1d(sval_all + s1 * FM, p.val + e1 * FM, slot_bytes, &metaf[s1]);
        }
      }
      __syncwarp();
      const int64_t le = step - TMA_LA;
      if (le < 0) continue;
      const int s = (int)(le % TMA_NS);
      mbar_wait(&metaf[s], (uint32_t)((le / TMA_NS) & 1));
      const int64_t e = ((int64_t)blockIdx.x + (le / TE) * gridDim.x) * TE + le % TE;
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
      while (ole + TMA_NS <= le || head + total - tail > RR) {
        mbar_wait(&empty[ole % TMA_NS], (uint32_t)((ole / TMA_NS) & 1));
        tail = slot_end[ole % TMA_NS];
        ++ole;
      }
      int16_t* srow = srow_all + s * FM;
      uint32_t* slr = slr_all + s * FM;
      int64_t r = head + (incl - cnt);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int sl = lane + 32 * c;
        if (sl < FM) {
          srow[sl] = ci[c] >= 0 ? (int16_t)(r % RR) : (int16_t)-1;
          if (ci[c] >= 0) ++r;
        }
      }
      if (lane == 0) slot_end[s] = head + total;
      __syncwarp();
      r = head + (incl - cnt);
      if (q.copy_mode == 0) {
        // one 1-D TMA bulk copy per feature row
        if (lane == 0) mbar_arrive_expect_tx(&full[s], (uint32_t)total * (uint32_t)q.row_bytes);
        __syncwarp();
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int sl = lane + 32 * c;
          if (sl < FM && ci[c] >= 0) {
            const int j = ci[c];
            tma_load_1d(ring + (size_t)(r % RR) * RS, ffm + (int64_t)j * row_elems,
                        (uint32_t)q.row_bytes, &full[s]);
            cp_async4(slr + sl, (const void*)((uintptr_t)(lrt + j) & ~(uintptr_t)3));
            ++r;
          }
        }
      } else {
        // warp-cooperative 16-byte cp.async: all 32 lanes stream the rows'
        // chunks (fully coalesced 512 B per warp instruction, no registers)
        int pos = incl - cnt;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int sl = lane + 32 * c;
          if (sl < FM && ci[c] >= 0) {
            plist[pos++] = make_int2(ci[c], (int)(r % RR));
            cp_async4(slr + sl, (const void*)((uintptr_t)(lrt + ci[c]) & ~(uintptr_t)3));
            ++r;
          }
        }
        __syncwarp();
        const int CH = q.row_bytes >> 4;
        int rr = lane / CH, ch = lane % CH;
        for (int qd = lane; qd < total * CH; qd += 32) {
          const int2 jr = plist[rr];
          cp_async16(ring + (size_t)jr.y * RS + ch * 16,
                     (const unsigned char*)(ffm + (int64_t)jr.x * row_elems) + ch * 16);
          ch += 32;
          while (ch >= CH) { ch -= CH; ++rr; }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[s]);
      }
      cp_async_arrive_noinc(&full[s]);
      head += total;
    }
  } else if (warp <= TMA_NC) {
    // ======================================================== consumers
    const int cw = warp - 1;
    unsigned char* spres = smem + L.off_pres + cw * F;
    for (int64_t le = cw; le < my_ex; le += TMA_NC) {
      const int s = (int)(le % TMA_NS);
      const int64_t ti = le / TE;
      const int el = (int)(le % TE);
      const int b = (int)(ti & 1);
      if (ti >= 2) mbar_wait(&xempty[b], (uint32_t)(((ti >> 1) - 1) & 1));
      mbar_wait(&full[s], (uint32_t)((le / TMA_NS) & 1));
      float* X = X_all + b * D * XS;
      double* exd = exd_all + b * 2 * TE;
      int* flag = flag_all + b * TE;
      if (!svalid[s]) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        zero_column(X, exd, flag, el, TE, XS, D, lane);
      } else {
        // srow >= 0 marks a slot whose row (and LR word) the producer fetched
        const int* sidx = sidx_all + s * FM;
        const float* sval = sval_all + s * FM;
        const int16_t* srow = srow_all + s * FM;
        const uint32_t* slr = slr_all + s * FM;
        double lrs = 0.0;
        for (int sl = lane; sl < FM; sl += 32) {
          if (srow[sl] >= 0)
            lrs += (double)sval[sl] *
                   (double)lr_from_word<T>(slr[sl], sidx[sl], p.dlr);  // M:338
        }
        for (int f = lane; f < F; f += 32) {
          unsigned char pr = 0;
          for (int m = 0; m < M; ++m) pr |= (srow[f * M + m] >= 0);
          spres[f] = pr;
        }
        const double lr_out = (double)bias + warp_sum(lrs);
        __syncwarp();
        double s1 = 0.0;
        int pbad = 0;
        for (int pp = lane; pp < P; pp += 32) {
          const uint32_t pr = pairtab[pp];
          const int f1 = pr & 0xFF, f2 = pr >> 8;
          float pv = 0.f;
          if (spres[f1] & spres[f2]) {
            float a[K], bb[K];
#pragma unroll
            for (int c = 0; c < K; ++c) { a[c] = 0.f; bb[c] = 0.f; }
            for (int m = 0; m < M; ++m) {
              const int ra = srow[f1 * M + m];
              if (ra >= 0) {
                float seg[K];
                lds_seg<K, T>(ring + (size_t)ra * RS + f2 * SEGB, seg, p.dffm);
                const float x = sval[f1 * M + m];
#pragma unroll
                for (int c = 0; c < K; ++c) a[c] = fmaf(x, seg[c], a[c]);
              }
              const int rb = srow[f2 * M + m];
              if (rb >= 0) {
                float seg[K];
                lds_seg<K, T>(ring + (size_t)rb * RS + f1 * SEGB, seg, p.dffm);
                const float x = sval[f2 * M + m];
#pragma unroll
                for (int c = 0; c < K; ++c) bb[c] = fmaf(x, seg[c], bb[c]);
              }
            }
#pragma unroll
            for (int c = 0; c < K; ++c) pv = fmaf(a[c], bb[c], pv);
          }
          X[(pp + 1) * XS + el] = pv;
          s1 += (double)pv;
          pbad |= !isfinite(pv);
        }
        __syncwarp();  // ring rows and slot no longer read: hand them back early
        if (lane == 0) mbar_arrive(&empty[s]);
        merge_finish(X, exd, flag, el, TE, XS, P, D, lane, lr_out, s1, pbad);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&xfull[b]);
    }
  } else {
    // ======================================================== MLP warps
    const int mt = threadIdx.x - (1 + TMA_NC) * 32;  // 0 .. 32*NM-1
    for (int64_t ti = 0; ti < my_tiles; ++ti) {
      const int b = (int)(ti & 1);
      mbar_wait(&xfull[b], (uint32_t)((ti >> 1) & 1));
      const int64_t base = ((int64_t)blockIdx.x + ti * gridDim.x) * TE;
      mlp_warps_tile<TMA_NM>(p, X_all + b * D * XS, exd_all + b * 2 * TE, flag_all + b * TE, Ha,
                             Hb, base, mt);
      if ((mt & 31) == 0) mbar_arrive(&xempty[b]);
    }
  }
}

}  // namespace dffm
