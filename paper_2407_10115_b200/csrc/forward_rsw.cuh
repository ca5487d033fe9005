// K1 v8 gather for the tensor-core MLP path: warp-specialised whole-row
// staging through one circular shared-memory row ring per SM (any M <= 4).
//
// Why (profiles/r01_k1_cfg5_rowstage_mlp_tc_ncu.json): the CTA-synchronous
// row-staging kernel (forward_rowstage.cuh) spends ~55% of its warp cycles in
// barrier / mbarrier waits -- three CTA barriers per example -- while DRAM
// is 31% busy.  Here no CTA barrier is left on the per-example path:
//
//   1 allocator warp  reads example i's padded slots (streamed IDXD examples
//       ahead into shared memory by cp.async), allocates its present rows in
//       a circular ring of R row slots (allocation and release in example
//       order) and publishes the slot metadata on meta[i]; the ring is shared
//       by all in-flight examples, so multi-slot data (cfg2: ~47 of 72 slots
//       present) packs densely and ~4-6 examples are resident or in flight.
//   NISS issue warps    one 1-D bulk (TMA) copy per present row, slot s by
//       warp s % NISS (full[i] counts their bytes).
//   NPW pair warps      process 32-pair chunks: npg = min(NPW, nch) warps,
//       warp w takes chunks w, w+npg, ... of every example (a group of G
//       warp sets could take alternate examples -- RSW_GT -- but one group
//       measured best).  Each chunk writes its raw pair values
//       and arrives on pdone[i]; the last chunk of an example frees its ring
//       rows.  With one slot per field a pair is x1*x2*<w1, w2>: bf16 rows
//       are dotted with the mixed-precision FMA (FHFMA.BF16, no unpacking).
//   NMW merge warps     (example i on warp i % NMW) load the LR weights
//       while the pairs are formed, then: sum(pairs) and the non-finite
//       check, lr_out (M:327, M:338), f64 mean /
//       population std over [lr_out, pairs] (M:355-360), the standardised row
//       (zero padded to Kp) written with 16-byte stores, lr_out + sum(pairs)
//       and the stage bits -> the staging buffers read by mlp_tc_kernel.
//
// Same arithmetic as the other K1 families: per pair the slot rows are summed
// in f32 in slot order (S[f1][f2] = sum_m x_m w_m[f2], M:339) and dotted in
// f32; statistics in f64 with a fixed reduction order (deterministic).
#pragma once

#include "forward_kernel.cuh"

namespace dffm {

#ifndef DFFM_RSW_NPW
#define DFFM_RSW_NPW 16
#endif
#ifndef DFFM_RSW_NISS
#define DFFM_RSW_NISS 4
#endif
#ifndef DFFM_RSW_IDXD
#define DFFM_RSW_IDXD 4
#endif
#ifndef DFFM_RSW_PAD
#define DFFM_RSW_PAD 16
#endif
#ifndef DFFM_RSW_GT
#define DFFM_RSW_GT 1
#endif
#ifndef DFFM_RSW_NMW
#define DFFM_RSW_NMW 6
#endif
constexpr int RSW_NPW = DFFM_RSW_NPW;
constexpr int RSW_NISS = DFFM_RSW_NISS;  // TMA issue warps (plus one allocator warp)
constexpr int RSW_NPROD = 1 + RSW_NISS;
constexpr int RSW_NMW = DFFM_RSW_NMW;
constexpr int RSW_GT = DFFM_RSW_GT;  // example groups of pair warps (power of 2)
constexpr int RSW_IDXD = DFFM_RSW_IDXD;  // examples of idx/val in flight per producer (power of 2)
static_assert((RSW_IDXD & (RSW_IDXD - 1)) == 0, "RSW_IDXD must be a power of two");
constexpr int RSW_THREADS = (RSW_NPW + RSW_NPROD + RSW_NMW) * 32;  // default role layout
constexpr int RSW_MAXWARPS = 28;  // CTA size bound (the role layout is chosen per shape, below)
constexpr int RSW_MAXX = 8;     // example slots (metadata + pair values)
constexpr int RSW_MAXFM = 128;  // padded slots per example (4 per producer lane)

struct RswSmem {
  int off_bar, off_pair, off_cnt, off_pidx, off_slot, off_ring, total;
  int slot_bytes, off_sidx, off_sval, off_rpos, off_xv;  // within a slot
  int row_stride, R, NX, nch;
  int npw, nmw;  // pair warps (= the allocator's warp number) and merge warps of this launch
};

// Example-slot block: sidx[FM] i32, sval[FM] f32, rpos[FM] u16, xv[P+1] f32;
// the ring takes the rest of `smem_max`.
__host__ __device__ inline RswSmem rsw_smem_layout(int F, int M, int P, int row_bytes, int NX,
                                                   int smem_max) {
  RswSmem s;
  const int FM = F * M;
  s.NX = NX;
  s.nch = (P + 31) / 32;
  s.row_stride = row_bytes + DFFM_RSW_PAD;  // +16 rotates banks row to row
  int q = 0;
  s.off_sidx = q; q = align16(q + FM * 4);
  s.off_sval = q; q = align16(q + FM * 4);
  s.off_rpos = q; q = align16(q + FM * 2);
  s.off_xv = q; q = align16(q + (P + 1) * 4);
  s.slot_bytes = q;
  int o = 0;
  s.off_bar = o; o = align16(o + 4 * RSW_MAXX * 8);
  s.off_pair = o; o = align16(o + P * 2);
  s.off_cnt = o; o = align16(o + RSW_MAXX * 4);
  s.off_pidx = o; o = align16(o + RSW_IDXD * 2 * FM * 4);
  s.off_slot = o; o = align16(o + NX * s.slot_bytes);
  s.off_ring = o;
  s.R = (smem_max - o) / s.row_stride;
  if (s.R > 65535) s.R = 65535;
  s.total = o + (s.R > 0 ? s.R : 0) * s.row_stride;
  s.npw = RSW_NPW;
  s.nmw = RSW_NMW;
  return s;
}

// Role layout per shape.  A warp's SMSP is its number mod 4, so the layout decides which
// warps share an issue port with the allocator warp -- the one serial stage of the kernel.
// Measured on B200 (tools/fwd_quick.py, ms per 1,048,576 cfg2 / 2,424,832 cfg5 examples):
//   pair / merge warps   16 / 6   17 / 6   16 / 7   17 / 7   21 / 6
//   cfg2 (9 chunks)       5.62     5.13     5.60     5.48     5.26
//   cfg5 (25 chunks)     20.68    20.85    19.99    20.58    21.40
// With few pair chunks only the first nch pair warps work (the others exit), and moving
// the allocator from warp 16 (SMSP 0, beside pair warps 0, 4, 8) to warp 17 (SMSP 1,
// beside 1 and 5) is worth 9%; with every pair warp busy a seventh merge warp (28 warps:
// seven per SMSP) is worth 3%.
__host__ __device__ inline void rsw_role_layout(int nch, int* npw, int* nmw) {
  if (nch < RSW_NPW) { *npw = RSW_NPW + 1; *nmw = RSW_NMW; }
  else { *npw = RSW_NPW; *nmw = RSW_NMW + 1; }
}

template <int K, typename T, int MU>
__global__ void __launch_bounds__(RSW_MAXWARPS * 32, 1) fwd_rsw_kernel(FwdParams p, RswSmem L) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int F = p.F, P = p.P, D = p.D;
  constexpr int M = MU;
  const int FM = F * M;
  constexpr int SEGB = K * (int)sizeof(T);
  const int row_bytes = F * SEGB;
  const int RSB = L.row_stride, R = L.R, NX = L.NX, nch = L.nch;
  const int NPW = L.npw, NMW = L.nmw;  // role layout of this launch (rsw_role_layout)
  uint64_t* full = (uint64_t*)(smem + L.off_bar);  // [NX] producers -> pair/merge warps
  uint64_t* pdone = full + RSW_MAXX;               // [NX] pair chunks -> producers/merge
  uint64_t* mfree = pdone + RSW_MAXX;              // [NX] merge warp -> producers
  uint64_t* meta = mfree + RSW_MAXX;               // [NX] allocator -> issue warps
  uint16_t* pairtab = (uint16_t*)(smem + L.off_pair);
  int* my_cnt = (int*)(smem + L.off_cnt);  // [MAXX] rows per slot (allocator-private)
  unsigned char* slots = smem + L.off_slot;
  unsigned char* ring = smem + L.off_ring;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const T* lrt = (const T*)p.lr;

  for (int f1 = threadIdx.x; f1 < F; f1 += blockDim.x) {
    const int base = f1 * F - f1 * (f1 + 1) / 2;
    for (int f2 = f1 + 1; f2 < F; ++f2) pairtab[base + f2 - f1 - 1] = (uint16_t)(f1 | (f2 << 8));
  }
  if (threadIdx.x == 0) {
    for (int b = 0; b < NX; ++b) {
      mbar_init(&full[b], RSW_NISS);
      mbar_init(&meta[b], 1);
      mbar_init(&pdone[b], nch);
      mbar_init(&mfree[b], 1);
    }
    mbar_fence_init();
  }
  __syncthreads();

  const int64_t my_n = p.n > blockIdx.x ? (p.n - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  auto slot = [&](int xs) { return slots + (size_t)xs * L.slot_bytes; };

  if (warp >= NPW + RSW_NPROD) {
    // ================================================================ merge warps
    const int mw = warp - NPW - RSW_NPROD;
    const float bias = load_elem<T>(lrt + p.n_buckets, p.dlr);
    int xs = mw % NX;
    uint32_t par = (uint32_t)((mw / NX) & 1);
    for (int64_t i = mw; i < my_n; i += NMW) {
      const int64_t e = blockIdx.x + i * gridDim.x;
      unsigned char* sb = slot(xs);
      const int* sidx = (const int*)(sb + L.off_sidx);
      const float* sval = (const float*)(sb + L.off_sval);
      // metadata published (meta[i]; before the rows are even requested): the
      // LR loads start a whole row-copy latency before the pairs are formed.
      // Phase-safe like the pair warps: pdone(i - NMW) complete means every
      // pair warp -- hence every full/meta phase up to i - NMW -- is done.
      mbar_wait(&meta[xs], par);
      // LR terms (M:338) in flight while the rows land and the pairs are formed
      float lw[RSW_MAXFM / 32], lx[RSW_MAXFM / 32];
#pragma unroll
      for (int c = 0; c < RSW_MAXFM / 32; ++c) {
        const int s = lane + 32 * c;
        const int j = s < FM ? sidx[s] : -1;
        lx[c] = j >= 0 ? sval[s] : 0.f;
        lw[c] = j >= 0 ? load_elem<T>(lrt + j, p.dlr) : 0.f;
      }
      mbar_wait(&pdone[xs], par);
      const float* xv = (const float*)(sb + L.off_xv);
      double ps = 0.0;
      int pbad = 0;
      for (int pp = lane; pp < P; pp += 32) {  // sum(pairs) (M:351, M:377) in f64
        const float v = xv[1 + pp];
        ps += (double)v;
        pbad |= !isfinite(v);
      }
      const double psum = warp_sum(ps);
      pbad = __any_sync(0xffffffffu, pbad);
      double lrs = 0.0;
#pragma unroll
      for (int c = 0; c < RSW_MAXFM / 32; ++c) lrs += (double)lx[c] * (double)lw[c];
      const double lr_out = (double)bias + warp_sum(lrs);  // M:327
      // MergeNorm (M:355-360): population std + MERGE_EPS
      const double mu = (psum + lr_out) / D;
      double s2 = 0.0;
      for (int pp = lane; pp < P; pp += 32) {
        const double d = (double)xv[1 + pp] - mu;
        s2 += d * d;
      }
      s2 = warp_sum(s2) + (lr_out - mu) * (lr_out - mu);
      const double denom = sqrt(s2 / D) + 1e-6;
      const double rden = 1.0 / denom;  // one f64 division per example
      const float m0 = (float)((lr_out - mu) * rden);
      int mbad = 0;
      for (int q = lane; q < (p.Kp >> 2); q += 32) {
        float v[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int c = 4 * q + t;
          float m = 0.f;
          if (c == 0) m = m0;
          else if (c < D) m = (float)(((double)xv[c] - mu) * rden);
          mbad |= !isfinite(m);
          v[t] = m;
        }
        xstore4(p.xout, p.xplane, e * p.Kp + 4 * q, v);
      }
      mbad = __any_sync(0xffffffffu, mbad);
      if (lane == 0) {
        p.rout[e] = lr_out + psum;
        p.fout[e] = (!isfinite(lr_out) ? 1 : 0) | (pbad ? 2 : 0) | (mbad ? 4 : 0);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&mfree[xs]);
      xs += NMW;
      while (xs >= NX) { xs -= NX; par ^= 1u; }
    }
  } else if (warp > NPW) {
    // ================================================================ TMA issue warps
    // Slot s of example i is issued by warp s % NISS, lane s / NISS, from the
    // metadata the allocator published on meta[i]; each warp arrives on
    // full[i] once with the bytes of its rows.  Issuing is spread over several
    // warps because a 1-D bulk copy per row is the step that limits how fast
    // the ring refills (measured: 2 -> 4 issuing warps, cfg5 +5%, cfg2 +20%).
    const int iw = warp - NPW - 1;
    int xs = 0;
    uint32_t par = 0;
    for (int64_t i = 0; i < my_n; ++i) {
      mbar_wait(&meta[xs], par);
      const unsigned char* sb = slot(xs);
      const int* sidx = (const int*)(sb + L.off_sidx);
      const uint16_t* rpos = (const uint16_t*)(sb + L.off_rpos);
      constexpr int SPW = (RSW_MAXFM + 32 * RSW_NISS - 1) / (32 * RSW_NISS);  // slots per lane
      int rr[SPW];
      int mine = 0;
#pragma unroll
      for (int t = 0; t < SPW; ++t) {
        const int s = iw + RSW_NISS * (lane + 32 * t);
        rr[t] = s < FM ? (int)rpos[s] : 0xFFFF;
        mine += __popc(__ballot_sync(0xffffffffu, rr[t] != 0xFFFF));
      }
      if (lane == 0) {
        if (mine) mbar_arrive_expect_tx(&full[xs], (uint32_t)(mine * row_bytes));
        else mbar_arrive(&full[xs]);
      }
      __syncwarp();
#pragma unroll
      for (int t = 0; t < SPW; ++t) {
        const int s = iw + RSW_NISS * (lane + 32 * t);
        if (rr[t] != 0xFFFF)
          tma_load_1d(ring + (size_t)rr[t] * RSB,
                      (const unsigned char*)p.ffm + (int64_t)sidx[s] * row_bytes,
                      (uint32_t)row_bytes, &full[xs]);
      }
      if (++xs == NX) { xs = 0; par ^= 1u; }
    }
  } else if (warp == NPW) {
    // ================================================================ allocator warp
    constexpr int SPL = RSW_MAXFM / 32;
    // idx / val of examples i+1 .. i+IDXD-1 stream into a shared ring by
    // 4-byte cp.async (one commit group per example), so the allocator never
    // waits a global-load latency per example
    int* pidx = (int*)(smem + L.off_pidx);  // [IDXD][idx FM | val FM]
    auto issue_ex = [&](int64_t i) {
      if (i < my_n) {
        const int64_t e = blockIdx.x + i * gridDim.x;
        int* d = pidx + (int)(i & (RSW_IDXD - 1)) * 2 * FM;
#pragma unroll
        for (int c = 0; c < SPL; ++c) {
          const int s = lane + 32 * c;
          if (s < FM) {
            cp_async4(d + s, p.idx + e * FM + s);
            cp_async4(d + FM + s, p.val + e * FM + s);
          }
        }
      }
      cp_async_commit();
    };
#pragma unroll 1
    for (int d = 0; d < RSW_IDXD; ++d) issue_ex(d);
    int head = 0, tail = 0;  // ring rows allocated / released (mod R)
    int used = 0;            // rows currently allocated
    int64_t tail_ex = 0;     // oldest example whose rows are still allocated
    const uint32_t lt = (1u << lane) - 1u;
    int xs = 0, ts = 0;         // slot of example i / of tail_ex
    uint32_t fpar = 1, tpar = 0;  // mfree parity for example i - NX / pdone parity of tail_ex
    for (int64_t i = 0; i < my_n; ++i) {
      const int64_t e = blockIdx.x + i * gridDim.x;
      int cj[SPL];
      float cx[SPL];
      int bad = 0;
      cp_async_wait<RSW_IDXD - 1>();  // this lane's copies of example i have landed
      {
        const int* d = pidx + (int)(i & (RSW_IDXD - 1)) * 2 * FM;
#pragma unroll
        for (int c = 0; c < SPL; ++c) {
          const int s = lane + 32 * c;
          int j = s < FM ? d[s] : -1;
          if (j >= p.n_buckets || j < -1) { bad = 1; j = -1; }  // ContractError (bad index)
          cj[c] = j;
          cx[c] = s < FM ? __int_as_float(d[FM + s]) : 0.f;
        }
      }
      issue_ex(i + RSW_IDXD);
      if (__any_sync(0xffffffffu, bad) && lane == 0)
        atomicMin((unsigned long long*)p.status,
                  (unsigned long long)status_key(p.status_base + e, DFFM_BLOCK_NONE,
                                                 DFFM_CONTRACT));
      uint32_t mask[SPL];
      int cnt = 0;
#pragma unroll
      for (int c = 0; c < SPL; ++c) {
        mask[c] = __ballot_sync(0xffffffffu, cj[c] >= 0);
        cnt += __popc(mask[c]);
      }
      // example slot free (its merge of example i - NX is done, so are its
      // pairs): retire that example's rows now, before the slot is reused
      if (i >= NX) {
        mbar_wait(&mfree[xs], fpar);
        if (tail_ex == i - NX) {
          const int tc = my_cnt[xs];
          tail += tc;
          if (tail >= R) tail -= R;
          used -= tc;
          ++tail_ex;
          if (++ts == NX) { ts = 0; tpar ^= 1u; }
        }
      }
      // ring space: release the oldest examples' rows once their pairs are
      // formed (examples i-NX+1 .. i-1: their slots are not reused yet)
      while (used + cnt > R) {
        mbar_wait(&pdone[ts], tpar);
        const int tc = my_cnt[ts];
        tail += tc;
        if (tail >= R) tail -= R;
        used -= tc;
        ++tail_ex;
        if (++ts == NX) { ts = 0; tpar ^= 1u; }
      }
      // slot metadata -> meta[xs] (release): the issue warps copy the rows
      unsigned char* sb = slot(xs);
      int* sidx = (int*)(sb + L.off_sidx);
      float* sval = (float*)(sb + L.off_sval);
      uint16_t* rpos = (uint16_t*)(sb + L.off_rpos);
      int before = 0;
#pragma unroll
      for (int c = 0; c < SPL; ++c) {
        const int s = lane + 32 * c;
        int r = head + before + __popc(mask[c] & lt);
        if (r >= R) r -= R;
        before += __popc(mask[c]);
        if (s < FM) {
          sidx[s] = cj[c];
          sval[s] = cx[c];
          rpos[s] = (uint16_t)(cj[c] >= 0 ? r : 0xFFFF);
        }
      }
      if (lane == 0) my_cnt[xs] = cnt;
      __syncwarp();
      if (lane == 0) mbar_arrive(&meta[xs]);
      head += cnt;
      if (head >= R) head -= R;
      used += cnt;
      if (++xs == NX) { xs = 0; fpar ^= 1u; }
    }
    cp_async_wait<0>();
  } else {
    // ================================================================ pair warps
    // G groups of npg = min(NPW / G, nch) pair warps; group g takes examples
    // g, g+G, ... and chunk c of an example goes to warp c % npg of the group,
    // so every active warp has a chunk in each of its group's examples.
    // Phase-safe waits: G divides NX, so a group revisits a slot only through
    // its own examples (it saw example i-NX complete before waiting on i), and
    // slot i is not reissued before the group's chunks of i are done.  (The
    // merge warps wait on meta[i], published only after the merge of i-NX.)
    int G = 1;
    while (2 * G <= RSW_GT && NX % (2 * G) == 0) G *= 2;
    const int npg = NPW / G < nch ? NPW / G : nch;
    const int gw = warp / npg, wi = warp - gw * npg;
    int64_t i = gw < G ? gw : my_n;
    int c = wi;
    int xs = gw < G ? gw : 0;
    uint32_t par = 0;
    int64_t cur = -1;
    const unsigned char* sb = nullptr;
    const int* sidx = nullptr;
    const float* sval = nullptr;
    const uint16_t* rpos = nullptr;
    for (; i < my_n;) {
      if (i != cur) {
        mbar_wait(&full[xs], par);
        cur = i;
        sb = slot(xs);
        sidx = (const int*)(sb + L.off_sidx);
        sval = (const float*)(sb + L.off_sval);
        rpos = (const uint16_t*)(sb + L.off_rpos);
      }
      const int pp = c * 32 + lane;
      if (pp < P) {
        const uint32_t pr = pairtab[pp];
        const int f1 = pr & 0xFF, f2 = pr >> 8;
        float pv = 0.f;
        if constexpr (M == 1) {
          // one row per field: pair = x1*x2*<w1[f2], w2[f1]> -- the raw segment
          // dot in f32 (bf16: FHFMA, exact products of the stored values), then
          // one scale (x = 1.0 for categorical fields: the same bits as
          // scaling each side first)
          const int r1 = rpos[f1], r2 = rpos[f2];
          if (r1 != 0xFFFF && r2 != 0xFFFF) {  // inactive pairs stay exactly 0 (M:346-351)
            const unsigned char* q1 = ring + (size_t)r1 * RSB + f2 * SEGB;
            const unsigned char* q2 = ring + (size_t)r2 * RSB + f1 * SEGB;
            float d = 0.f;
#pragma unroll
            for (int u = 0; u < SEGB / 16; ++u) {
              const uint4 w1 = *(const uint4*)(q1 + u * 16);
              const uint4 w2 = *(const uint4*)(q2 + u * 16);
              d = dot16_acc<T>(w1, w2, d, p.dffm);
            }
            const float x1 = sval[f1], x2 = sval[f2];
            pv = (x1 == 1.f && x2 == 1.f) ? d : (x1 * x2) * d;
          }
        } else {
          float a[K], bb[K];
#pragma unroll
          for (int t = 0; t < K; ++t) { a[t] = 0.f; bb[t] = 0.f; }
          bool p1 = false, p2 = false;
          constexpr int PER = 16 / (int)sizeof(T);
#pragma unroll
          for (int m = 0; m < M; ++m) {
            const int r1 = rpos[f1 * M + m];
            if (r1 != 0xFFFF) {
              p1 = true;
              const float x1 = sval[f1 * M + m];
              const unsigned char* q1 = ring + (size_t)r1 * RSB + f2 * SEGB;
#pragma unroll
              for (int u = 0; u < SEGB / 16; ++u) {
                float w[PER];
                unpack16<T>(*(const uint4*)(q1 + u * 16), w, p.dffm);
#pragma unroll
                for (int t = 0; t < PER; ++t) a[u * PER + t] = fmaf(x1, w[t], a[u * PER + t]);
              }
            }
            const int r2 = rpos[f2 * M + m];
            if (r2 != 0xFFFF) {
              p2 = true;
              const float x2 = sval[f2 * M + m];
              const unsigned char* q2 = ring + (size_t)r2 * RSB + f1 * SEGB;
#pragma unroll
              for (int u = 0; u < SEGB / 16; ++u) {
                float w[PER];
                unpack16<T>(*(const uint4*)(q2 + u * 16), w, p.dffm);
#pragma unroll
                for (int t = 0; t < PER; ++t) bb[u * PER + t] = fmaf(x2, w[t], bb[u * PER + t]);
              }
            }
          }
          if (p1 && p2) {  // inactive pairs stay exactly 0 (M:346-351)
#pragma unroll
            for (int t = 0; t < K; ++t) pv = fmaf(a[t], bb[t], pv);
          }
        }
        float* xv = (float*)(sb + L.off_xv);
        xv[1 + pp] = pv;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&pdone[xs]);
      c += npg;
      if (c >= nch) {
        c = wi;
        i += G;
        xs += G;
        if (xs >= NX) { xs -= NX; par ^= 1u; }
      }
    }
  }
}

}  // namespace dffm
