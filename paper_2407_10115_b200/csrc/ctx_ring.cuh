// K3 v2: context-cached candidate scorer on the K1 v8 row ring (staging mode:
// the candidates' MergeNorm rows go to the tcgen05 MLP, mlp_tc.cu).
//
// SPEC S:239-296 (no reference code; truth = model.forward on the merged
// example).  Context fields are 0..Fc-1, candidate fields Fc..F-1
// (disjoint).  The examples of the ring are the candidates of this
// CTA's requests, in order (request r = blockIdx.x + t*gridDim.x).  A candidate
// is only Fd * Md rows (8 at cfg4), so the single-warp stages -- allocator and
// issue warps -- handle a BUNDLE of B consecutive candidates per step with
// B * Fd * Md lanes active (ncu, round 2: with one candidate per step the
// allocator warp never waited and every other role waited on it):
//   allocator warp   streams candidate slots (cp.async, IDXD ahead), allocates
//                    their present rows in the ring, publishes meta[i]
//   issue warps      one 1-D bulk copy per candidate row (full[i])
//   builder warp     build_context_cache per request, one or two requests
//                    ahead of the candidates, double-buffered by request parity:
//                    Sctx[x][g][:] = sum_m x_m w_m[g] (f32 fma over the context
//                    slots, as K3 v1), the ctx x ctx pair values and their moments,
//                    the context lr partial; published on cready[t & 1]
//   pair warps       per candidate the pairs that involve a candidate field
//                    (S:263-265): <S[c][x], Sctx[x][c]> and <S[c1][c2], S[c2][c1]>, in
//                    32-pair chunks; G groups of warps take alternate bundles
//                    (phase-safe waits: G divides NX)
//   merge warps      lr_out = bias + ctx lr partial + candidate lr terms;
//                    MergeNorm over [lr_out, all P pairs] (ctx x ctx from the
//                    cache: never cached past MergeNorm) in f64 ->
//                    staged row, residual, stage bits.
// The cache of request t is built (buffer t & 1) only after every candidate of request
// t - 2 is merged (cfree[t & 1] counts the merge warps' arrivals), so no pair or merge
// warp still reads a buffer that is being rebuilt.
#pragma once

#include "forward_kernel.cuh"
#include "forward_rsw.cuh"

namespace dffm {

#ifndef DFFM_CR_GT
#define DFFM_CR_GT 2
#endif
#ifndef DFFM_CR_NPW
#define DFFM_CR_NPW 10
#endif
#ifndef DFFM_CR_NMW
#define DFFM_CR_NMW 10
#endif
#ifndef DFFM_CR_NISS
#define DFFM_CR_NISS 2
#endif
constexpr int CR_NPW = DFFM_CR_NPW, CR_NISS = DFFM_CR_NISS, CR_NMW = DFFM_CR_NMW;
constexpr int CR_GT = DFFM_CR_GT;  // candidate groups of pair warps (power of 2)
constexpr int CR_THREADS = (CR_NPW + 1 + CR_NISS + CR_NMW + 1) * 32;  // + the context builder warp
constexpr int CR_MAXX = 64;   // candidate slots in flight
constexpr int CR_MAXFM = 32;  // candidate slots per candidate (Fd * Md)
constexpr int CR_CHUNK = 32;  // pairs per chunk (lane per pair)
constexpr int CR_IDXD = 8;    // candidates of slot data streamed ahead

struct CrSmem {
  int off_bar, off_ptab, off_stab, off_cnt, off_pidx, off_cache, off_slot, off_ring, total;
  int cache_bytes, c_S, c_cpx, c_lr, c_pres, c_sidx, c_sval;  // within a cache buffer
  int slot_bytes, s_sidx, s_sval, s_rpos, s_xv, xv_stride;     // within a slot (one bundle)
  int row_stride, R, NX, nch, Pc;
  int B, lgB;  // candidates per bundle (power of two)
};

// Candidates per bundle: the largest power of two B <= 4 with B * FM <= 32 lanes
// that divides the candidates per request (bundles never straddle requests).
__host__ __device__ inline int cr_bundle(int FM, int C) {
  int B = 1;
  while (2 * B <= 4 && 2 * B * FM <= CR_MAXFM && C % (2 * B) == 0) B *= 2;
  return B;
}

// NX = bundle slots in flight (CR_MAXX / B: the same 64 candidates for every B)
__host__ __device__ inline CrSmem cr_smem_layout(int F, int Fc, int Mc, int Fd, int Md, int k,
                                                 int esz, int B, int smem_max) {
  CrSmem s;
  const int P = F * (F - 1) / 2;
  s.Pc = Fc * Fd + Fd * (Fd - 1) / 2;
  s.nch = (s.Pc + CR_CHUNK - 1) / CR_CHUNK;
  s.B = B;
  s.lgB = B == 4 ? 2 : B == 2 ? 1 : 0;
  s.NX = CR_MAXX / B;
  const int FMB = Fd * Md * B;
  const int Kp = (P + 1 + 15) & ~15;  // staged row width (tc_plan)
  s.row_stride = F * k * esz + 16;
  int q = 0;
  s.c_S = q; q = align16(q + Fc * F * k * 4);
  s.c_cpx = q; q = align16(q + P * 4);
  s.c_lr = q; q = align16(q + 32);  // lr partial, sum and sum of squares of ctx pairs, bad flag
  s.c_pres = q; q = align16(q + Fc);
  s.c_sidx = q; q = align16(q + Fc * Mc * 4);
  s.c_sval = q; q = align16(q + Fc * Mc * 4);
  s.cache_bytes = q;
  q = 0;
  s.s_sidx = q; q = align16(q + FMB * 4);
  s.s_sval = q; q = align16(q + FMB * 4);
  s.s_rpos = q; q = align16(q + FMB * 2);
  s.xv_stride = s.Pc;
  s.s_xv = q; q = align16(q + B * s.Pc * 4);
  s.slot_bytes = q;
  int o = 0;
  s.off_bar = o; o = align16(o + (4 * CR_MAXX + 4) * 8);  // + cready[2], cfree[2]
  s.off_ptab = o; o = align16(o + s.Pc * 4);
  s.off_stab = o; o = align16(o + Kp * 2);
  s.off_cnt = o; o = align16(o + CR_MAXX * 4);
  s.off_pidx = o; o = align16(o + CR_IDXD * 2 * FMB * 4);
  s.off_cache = o; o = align16(o + 2 * s.cache_bytes);
  s.off_slot = o; o = align16(o + s.NX * s.slot_bytes);
  s.off_ring = o;
  s.R = (smem_max - o) / s.row_stride;
  if (s.R > 65535) s.R = 65535;
  s.total = o + (s.R > 0 ? s.R : 0) * s.row_stride;
  return s;
}


// build_context_cache for request r into the cache blob wb (shared
// memory): context slots, lr partial, Sctx[x][g][:] (f32 fma over the slots
// in slot order), ctx x ctx pair values and their f64 sum / sum of squares.
// Called by nthr threads (tid < nthr) that share named barrier 1; ends with it.
template <typename T>
__device__ __forceinline__ void cr_build_cache(unsigned char* wb, const CtxParams& q,
                                             const CrSmem& L, int64_t r, int64_t status_ex,
                                             int tid, int nthr) {
  const FwdParams& p = q.f;
  const int F = p.F, P = p.P, Fc = q.Fc, Mc = q.Mc;
  const int lane = tid & 31;
  const T* lrt = (const T*)p.lr;
  float* S = (float*)(wb + L.c_S);
  float* cpx = (float*)(wb + L.c_cpx);
  unsigned char* cpres = wb + L.c_pres;
  int* csidx = (int*)(wb + L.c_sidx);
  float* csval = (float*)(wb + L.c_sval);
  for (int s = tid; s < Fc * Mc; s += nthr) {
    int j = __ldg(q.cidx + r * Fc * Mc + s);
    if (j >= p.n_buckets || j < -1) {
      atomicMin((unsigned long long*)p.status,
                (unsigned long long)status_key(status_ex, DFFM_BLOCK_NONE,
                                               DFFM_CONTRACT));
      j = -1;
    }
    csidx[s] = j;
    csval[s] = __ldg(q.cval + r * Fc * Mc + s);
  }
  named_bar_sync(1, nthr);
  if (tid < 32) {
    double lrs = 0.0;
    for (int s = lane; s < Fc * Mc; s += 32)
      if (csidx[s] >= 0) lrs += (double)csval[s] * (double)load_elem<T>(lrt + csidx[s], p.dlr);
    lrs = warp_sum(lrs);
    if (lane == 0) *(double*)(wb + L.c_lr) = lrs;
  }
  for (int x = tid; x < Fc; x += nthr) {
    unsigned char pr = 0;
    for (int m = 0; m < Mc; ++m) pr |= (csidx[x * Mc + m] >= 0);
    cpres[x] = pr;
  }
  // 16-byte vectors of the context rows (one load per slot per vector,
  // all in flight together); same f32 fma over the slots in slot order
  const int Fk = F * p.k;
  constexpr int PER = 16 / (int)sizeof(T);
  const int nvec = Fk / PER;  // rows are whole 16-byte vectors (k * esz % 16 == 0)
  for (int t2 = tid; t2 < Fc * nvec; t2 += nthr) {
    const int x = t2 / nvec, v = t2 - x * nvec;
    float acc[PER];
#pragma unroll
    for (int u = 0; u < PER; ++u) acc[u] = 0.f;
    for (int m = 0; m < Mc; ++m) {
      const int j = csidx[x * Mc + m];
      if (j >= 0) {
        float w[PER];
        unpack16<T>(*(const uint4*)((const unsigned char*)p.ffm +
                                    ((int64_t)j * Fk + v * PER) * (int64_t)sizeof(T)),
                    w, p.dffm);
        const float xv = csval[x * Mc + m];
#pragma unroll
        for (int u = 0; u < PER; ++u) acc[u] = fmaf(xv, w[u], acc[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < PER; ++u) S[x * Fk + v * PER + u] = acc[u];
  }
  named_bar_sync(1, nthr);
  for (int pp = tid; pp < P; pp += nthr) cpx[pp] = 0.f;
  named_bar_sync(1, nthr);
  for (int x1 = 0; x1 < Fc; ++x1)
    for (int x2 = x1 + 1 + tid; x2 < Fc; x2 += nthr) {
      float pv = 0.f;
      if (cpres[x1] & cpres[x2]) {
        const float* a = S + (x1 * F + x2) * p.k;
        const float* b = S + (x2 * F + x1) * p.k;
        for (int kk = 0; kk < p.k; ++kk) pv = fmaf(a[kk], b[kk], pv);
      }
      cpx[x1 * F - x1 * (x1 + 1) / 2 + x2 - x1 - 1] = pv;
    }
  named_bar_sync(1, nthr);
  if (tid < 32) {  // moments of the ctx x ctx block (fixed order: deterministic)
    double s1 = 0.0, sq = 0.0;
    int bad = 0;
    for (int pp = lane; pp < P; pp += 32) {
      const double v = cpx[pp];
      s1 += v;
      sq += v * v;
      bad |= !isfinite(cpx[pp]);
    }
    s1 = warp_sum(s1);
    sq = warp_sum(sq);
    bad = __any_sync(0xffffffffu, bad);
    if (lane == 0) {
      double* cm = (double*)(wb + L.c_lr);
      cm[1] = s1;
      cm[2] = sq;
      cm[3] = bad ? 1.0 : 0.0;
    }
  }
  named_bar_sync(1, nthr);
}

// Position of a stream of candidates that advances by a fixed step: request
// ordinal t of this CTA (request blockIdx.x + t * gridDim.x) and the candidate
// number within it -- no per-candidate division.
struct CrCursor {
  int64_t t;
  int w;
  __device__ __forceinline__ void advance(int step, int C) {
    w += step;
    while (w >= C) { w -= C; ++t; }
  }
  __device__ __forceinline__ int64_t cand(int C) const {  // global candidate number
    return ((int64_t)blockIdx.x + t * gridDim.x) * C + w;
  }
};

template <int K, typename T, int MD>
__global__ void __launch_bounds__(CR_THREADS, 1) ctx_ring_kernel(CtxParams q, CrSmem L) {
  extern __shared__ __align__(128) unsigned char smem[];
  const FwdParams& p = q.f;
  const int F = p.F, P = p.P, D = p.D, Fc = q.Fc, Mc = q.Mc, Fd = q.Fd;
  constexpr int M = MD;
  const int FM = Fd * M;
  const int C = q.C;
  // B candidates (a bundle: consecutive candidates of one request, B | C) share a
  // slot: the allocator / issue warps work per bundle with B * FM lanes active
  const int B = L.B, lgB = L.lgB, FMB = FM * B;
  const int CB = C >> lgB;  // bundles per request
  constexpr int SEGB = K * (int)sizeof(T);
  const int row_bytes = F * SEGB;
  const int RSB = L.row_stride, R = L.R, NX = L.NX, nch = L.nch, Pc = L.Pc;
  const int nchB = nch * B;
  uint64_t* full = (uint64_t*)(smem + L.off_bar);
  uint64_t* pdone = full + CR_MAXX;
  uint64_t* mfree = pdone + CR_MAXX;
  uint64_t* meta = mfree + CR_MAXX;
  uint64_t* cready = meta + CR_MAXX;  // [2] builder -> pair / merge warps: cache buffer built
  uint64_t* cfree = cready + 2;       // [2] merge warps -> builder: every candidate of the request merged
  uint32_t* ptab = (uint32_t*)(smem + L.off_ptab);  // candidate pairs: f1 | f2 << 8 | pos << 16
  uint16_t* stab = (uint16_t*)(smem + L.off_stab);  // staged column -> source (see merge warps)
  int* my_cnt = (int*)(smem + L.off_cnt);
  unsigned char* slots = smem + L.off_slot;
  unsigned char* ring = smem + L.off_ring;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const T* lrt = (const T*)p.lr;

  // candidate-pair table in global pair order (position = index into pairs) and
  // the staged row's source per column: 0x6000 = lr_out, 0x4000 = zero padding,
  // 0x8000 | pos = cached ctx x ctx pair, else the candidate pair's index
  // pair warps per bundle (each arrives on pdone once): as computed by the pair warps
  int pd_count;
  {
    int G = 1;
    while (2 * G <= CR_GT && NX % (2 * G) == 0 && 2 * G <= CB) G *= 2;
    pd_count = CR_NPW / G < nchB ? CR_NPW / G : nchB;
  }
  if (threadIdx.x == 0) {
    int n = 0, pos = 0;
    stab[0] = 0x6000;
    for (int f1 = 0; f1 < F; ++f1)
      for (int f2 = f1 + 1; f2 < F; ++f2, ++pos) {
        if (f2 >= Fc) {
          stab[1 + pos] = (uint16_t)n;
          ptab[n++] = (uint32_t)f1 | ((uint32_t)f2 << 8) | ((uint32_t)pos << 16);
        } else {
          stab[1 + pos] = (uint16_t)(0x8000 | pos);
        }
      }
    for (int c = D; c < p.Kp; ++c) stab[c] = 0x4000;
    for (int b = 0; b < NX; ++b) {
      mbar_init(&full[b], CR_NISS);
      mbar_init(&meta[b], 1);
      mbar_init(&pdone[b], pd_count);
      mbar_init(&mfree[b], B);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&cready[b], 1);
      mbar_init(&cfree[b], C);
    }
    mbar_fence_init();
  }
  __syncthreads();

  const int64_t my_req = q.R > blockIdx.x ? (q.R - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t my_n = my_req * C;    // candidates of this CTA
  const int64_t my_nb = my_req * CB;  // bundles
  auto slot = [&](int xs) { return slots + (size_t)xs * L.slot_bytes; };
  auto cache = [&](int64_t t) { return smem + L.off_cache + (size_t)(t & 1) * L.cache_bytes; };

  if (warp == CR_NPW + 1 + CR_NISS + CR_NMW) {
    // ================================================================ context builder warp
    // build_context_cache one or two requests AHEAD of the candidates: the
    // cache of request t goes to buffer t & 1 as soon as every candidate of request
    // t - 2 is merged (cfree), and is published on cready.  (Built by the pair warps
    // at each request boundary it was ~10% of their time -- they are the stage the
    // merge warps wait on.)
    for (int64_t t = 0; t < my_req; ++t) {
      if (t >= 2) mbar_wait(&cfree[t & 1], (uint32_t)(((t >> 1) - 1) & 1));
      const int64_t r = (int64_t)blockIdx.x + t * gridDim.x;
      unsigned char* wb = cache(t);
      if (q.cache_in) {  // prebuilt (dffm_ctx_build): copy the request's cache blob
        const uint4* src = (const uint4*)(q.cache_in + (size_t)r * L.cache_bytes);
        for (int v = lane; v < L.cache_bytes / 16; v += 32) ((uint4*)wb)[v] = __ldg(src + v);
      } else {
        cr_build_cache<T>(wb, q, L, r, p.status_base + r * C, lane, 32);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&cready[t & 1]);
    }
  } else if (warp >= CR_NPW + 1 + CR_NISS) {
    // ================================================================ merge warps
    // one candidate per warp; its bundle's slot / phase follow from the bundle
    // number (a warp never waits on a phase it has no candidate in, and a slot
    // cannot advance past a phase before every candidate of it is merged).
    // The warp is a latency chain per candidate (LR loads -> f64 reductions ->
    // sqrt / reciprocal -> row), so the next candidate's LR terms are loaded
    // before this candidate's row is written (its metadata only depends on
    // merges of older candidates: no cycle).
    const int mw = warp - CR_NPW - 1 - CR_NISS;
    const float bias = load_elem<T>(lrt + p.n_buckets, p.dlr);
    const int lgNX = 31 - __clz(NX);
    const double rD = 1.0 / (double)D;
    CrCursor cu{0, 0};
    cu.advance(mw, C);
    T lraw = T();  // this lane's LR weight as stored (converted where it is consumed)
    float lx = 0.f;
    bool lp = false;
    auto lr_terms = [&](int64_t i) {  // LR weight / value of lane's slot of candidate i
      const int64_t ib = i >> lgB;
      const int xs = (int)(ib & (NX - 1));
      const unsigned char* sb = slot(xs);
      mbar_wait(&meta[xs], (uint32_t)((ib >> lgNX) & 1));
      lp = false;
      if (lane < FM) {
        const int sub = (int)(i & (B - 1));
        const int j = ((const int*)(sb + L.s_sidx))[sub * FM + lane];
        if (j >= 0) {
          lp = true;
          lx = ((const float*)(sb + L.s_sval))[sub * FM + lane];
          lraw = __ldg(lrt + j);
        }
      }
    };
    if (mw < my_n) lr_terms(mw);
    for (int64_t i = mw; i < my_n; i += CR_NMW, cu.advance(CR_NMW, C)) {
      const int64_t e = cu.cand(C);
      const int64_t ib = i >> lgB;
      const int sub = (int)(i & (B - 1));
      const int xs = (int)(ib & (NX - 1));
      const uint32_t par = (uint32_t)((ib >> lgNX) & 1);
      unsigned char* sb = slot(xs);
      mbar_wait(&pdone[xs], par);
      const unsigned char* cb = cache(cu.t);
      const float* cpx = (const float*)(cb + L.c_cpx);
      const float* xv = (const float*)(sb + L.s_xv) + sub * L.xv_stride;
      // candidate pairs land in xv in ptab order; the ctx x ctx pairs' sum and
      // sum of squares come from the cache (f64, computed once per request)
      const double* cst = (const double*)(cb + L.c_lr);  // lr partial, sum v, sum v^2, bad
      double ps = 0.0;
      int pbad = 0;
      for (int t = lane; t < Pc; t += 32) {
        const float v = xv[t];
        ps += (double)v;
        pbad |= !isfinite(v);
      }
      const double lrc =
          warp_sum(lp ? (double)lx * (double)elem_to_float<T>(lraw, p.dlr) : 0.0);
      const double psum = warp_sum(ps) + cst[1];
      pbad = __any_sync(0xffffffffu, pbad) | (cst[3] != 0.0);
      const double lr_out = (double)bias + cst[0] + lrc;  // M:327
      const double mu = (psum + lr_out) * rD;
      // population variance (M:359): candidate deviations two-pass, the ctx x ctx
      // block through its cached moments: sum (v-mu)^2 = S2 - 2 mu S1 + n mu^2
      double s2 = 0.0;
      for (int t = lane; t < Pc; t += 32) {
        const double d = (double)xv[t] - mu;
        s2 += d * d;
      }
      const int nctx = P - Pc;
      s2 = warp_sum(s2) + (cst[2] - 2.0 * mu * cst[1] + (double)nctx * mu * mu) +
           (lr_out - mu) * (lr_out - mu);
      const double rden = 1.0 / (sqrt(s2 * rD) + 1e-6);
      const float m0 = (float)((lr_out - mu) * rden);
      if (i + CR_NMW < my_n) lr_terms(i + CR_NMW);  // next candidate's LR loads in flight
      // The standardised row in global pair order, four columns per lane.  The
      // element arithmetic is two-float f32: (v - mu_hi) - mu_lo keeps the
      // cancellation exact to 2^-24 of the difference, so the row carries more
      // bits than the fp16 hi/lo planes it is staged in (22).
      const float muh = (float)mu, mul = (float)(mu - (double)muh), rdf = (float)rden;
      int mbad = 0;
      for (int qd = lane; qd < (p.Kp >> 2); qd += 32) {
        const uint2 cd = *(const uint2*)(stab + 4 * qd);
        const uint32_t code[4] = {cd.x & 0xFFFFu, cd.x >> 16, cd.y & 0xFFFFu, cd.y >> 16};
        float v[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const float* src = (code[t] & 0x8000u) ? cpx : xv;
          const float raw = src[code[t] & 0x3FFu];
          float m = ((raw - muh) - mul) * rdf;
          if (code[t] & 0x4000u) m = (code[t] & 0x2000u) ? m0 : 0.f;
          mbad |= !isfinite(m);
          v[t] = m;
        }
        xstore4(p.xout, p.xplane, e * p.Kp + 4 * qd, v);
      }
      mbad = __any_sync(0xffffffffu, mbad);
      if (lane == 0) {
        p.rout[e] = lr_out + psum;
        p.fout[e] = (!isfinite(lr_out) ? 1 : 0) | (pbad ? 2 : 0) | (mbad ? 4 : 0);
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&mfree[xs]);
        mbar_arrive(&cfree[cu.t & 1]);  // one of the request's C candidates is done with the cache
      }
    }
  } else if (warp > CR_NPW) {
    // ================================================================ TMA issue warps
    // (measured alternative, not kept: the bundle's rows as 16-byte cp.async chunks,
    // lanes along the row, completing on full[xs] through
    // cp.async.mbarrier.arrive.noinc -- cfg4 2.43 ms per step against 2.20 ms with
    // one bulk copy per 384-byte row, 2 and 4 issue warps alike)
    const int iw = warp - CR_NPW - 1;
    int xs = 0;
    uint32_t par = 0;
    for (int64_t i = 0; i < my_nb; ++i) {
      mbar_wait(&meta[xs], par);
      const unsigned char* sb = slot(xs);
      const int* sidx = (const int*)(sb + L.s_sidx);
      const uint16_t* rpos = (const uint16_t*)(sb + L.s_rpos);
      const int s = iw + CR_NISS * lane;
      const int r = s < FMB ? (int)rpos[s] : 0xFFFF;
      const int mine = __popc(__ballot_sync(0xffffffffu, r != 0xFFFF));
      if (lane == 0) {
        if (mine) mbar_arrive_expect_tx(&full[xs], (uint32_t)(mine * row_bytes));
        else mbar_arrive(&full[xs]);
      }
      __syncwarp();
      if (r != 0xFFFF)
        tma_load_1d(ring + (size_t)r * RSB, (const unsigned char*)p.ffm + (int64_t)sidx[s] * row_bytes,
                    (uint32_t)row_bytes, &full[xs]);
      if (++xs == NX) { xs = 0; par ^= 1u; }
    }
  } else if (warp == CR_NPW) {
    // ================================================================ allocator warp
    int* pidx = (int*)(smem + L.off_pidx);  // [IDXD][idx FMB | val FMB]
    CrCursor ahead{0, 0};  // bundle being streamed in
    auto issue_ex = [&](int64_t i) {
      if (i < my_nb && lane < FMB) {
        const int64_t e0 = ahead.cand(C);
        int* d = pidx + (int)(i & (CR_IDXD - 1)) * 2 * FMB;
        cp_async4(d + lane, q.didx + e0 * FM + lane);
        cp_async4(d + FMB + lane, q.dval + e0 * FM + lane);
      }
      ahead.advance(B, C);
      cp_async_commit();
    };
#pragma unroll 1
    for (int d = 0; d < CR_IDXD; ++d) issue_ex(d);
    int head = 0, tail = 0, used = 0;
    int64_t tail_ex = 0;
    const uint32_t lt = (1u << lane) - 1u;
    int xs = 0, ts = 0;
    uint32_t fpar = 1, tpar = 0;
    CrCursor cu{0, 0};
    for (int64_t i = 0; i < my_nb; ++i, cu.advance(B, C)) {
      cp_async_wait<CR_IDXD - 1>();
      const int* d = pidx + (int)(i & (CR_IDXD - 1)) * 2 * FMB;
      int j = lane < FMB ? d[lane] : -1;
      const float x = lane < FMB ? __int_as_float(d[FMB + lane]) : 0.f;
      if (j >= p.n_buckets || j < -1) {  // ContractError at this lane's candidate
        atomicMin((unsigned long long*)p.status,
                  (unsigned long long)status_key(p.status_base + cu.cand(C) + lane / FM,
                                                 DFFM_BLOCK_NONE, DFFM_CONTRACT));
        j = -1;
      }
      issue_ex(i + CR_IDXD);
      const uint32_t mask = __ballot_sync(0xffffffffu, j >= 0);
      const int cnt = __popc(mask);
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
      while (used + cnt > R) {
        mbar_wait(&pdone[ts], tpar);
        const int tc = my_cnt[ts];
        tail += tc;
        if (tail >= R) tail -= R;
        used -= tc;
        ++tail_ex;
        if (++ts == NX) { ts = 0; tpar ^= 1u; }
      }
      unsigned char* sb = slot(xs);
      if (lane < FMB) {
        int r = head + __popc(mask & lt);
        if (r >= R) r -= R;
        ((int*)(sb + L.s_sidx))[lane] = j;
        ((float*)(sb + L.s_sval))[lane] = x;
        ((uint16_t*)(sb + L.s_rpos))[lane] = (uint16_t)(j >= 0 ? r : 0xFFFF);
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
    // G groups of npg warps; group g takes bundles g, g+G, ... (chunk c of a
    // bundle -- chunk c % nch of its candidate c / nch -- on warp c % npg of the
    // group; each warp arrives on pdone once per bundle).  Phase-safe: G divides
    // NX, so a group revisits a slot only through its own bundles, and every warp
    // of a group has a chunk in each of them.
    int G = 1;
    while (2 * G <= CR_GT && NX % (2 * G) == 0 && 2 * G <= CB) G *= 2;
    const int npg = CR_NPW / G < nchB ? CR_NPW / G : nchB;
    const int gw = warp / npg, wi = warp - gw * npg;
    if (gw >= G) return;
    int xs = gw;
    uint32_t par = 0;
    int64_t cur_req = -1;
    CrCursor cu{0, 0};  // in bundles: w = bundle within the request
    cu.advance(gw, CB);
    const unsigned char* cb = nullptr;
    constexpr int PER = 16 / (int)sizeof(T);
    // One slot per candidate field and one warp per chunk (npg == nch): warp wi
    // owns pairs wi*32 .. wi*32+31 of EVERY candidate, so the pair's fields and,
    // for a context x candidate pair, the cached S[x][c] segment stay in registers
    // for the whole request; per candidate only the candidate row's segment is
    // read.  pair = x_c * <S[x][c], w_c[x]> (x_c = 1.0 for categorical fields:
    // the same bits as scaling the row first, as K1 v8 does for M == 1).
    const bool fixed = (M == 1) && npg == nch;
    const int tf = wi * CR_CHUNK + lane;
    const bool valid = fixed && tf < Pc;
    const uint32_t prf = valid ? ptab[tf] : 0u;
    const int ff1 = prf & 0xFF, ff2 = (prf >> 8) & 0xFF;
    const bool isctx = ff1 < Fc;
    const bool allctx = __all_sync(0xffffffffu, isctx || !valid);
    float areg[K];
    bool p1c = false;
#pragma unroll
    for (int u = 0; u < K; ++u) areg[u] = 0.f;
    for (int64_t i = gw; i < my_nb; i += G, cu.advance(G, CB)) {
      if (cu.t != cur_req) {  // the builder warp has request t's cache in buffer t & 1
        cur_req = cu.t;
        mbar_wait(&cready[cur_req & 1], (uint32_t)((cur_req >> 1) & 1));
        cb = cache(cur_req);
        if (valid && isctx) {
          const float* sc = (const float*)(cb + L.c_S) + (ff1 * F + ff2) * K;
#pragma unroll
          for (int u = 0; u < K; ++u) areg[u] = sc[u];
          p1c = (cb + L.c_pres)[ff1] != 0;
        }
      }
      mbar_wait(&full[xs], par);
      const unsigned char* sb = slot(xs);
      if (fixed) {
        if (valid) {
          const int c2 = ff2 - Fc, c1 = ff1 - Fc;
          if (allctx) {
#pragma unroll 4
            for (int sub = 0; sub < B; ++sub) {
              const int r2 = ((const uint16_t*)(sb + L.s_rpos))[sub * FM + c2];
              const float x2 = ((const float*)(sb + L.s_sval))[sub * FM + c2];
              const bool p2 = r2 != 0xFFFF;
              const unsigned char* q2 = ring + (size_t)(p2 ? r2 : 0) * RSB + ff1 * SEGB;
              float d = 0.f;
#pragma unroll
              for (int u = 0; u < SEGB / 16; ++u) {
                float w[PER];
                unpack16<T>(*(const uint4*)(q2 + u * 16), w, p.dffm);
#pragma unroll
                for (int v = 0; v < PER; ++v) d = fmaf(areg[u * PER + v], w[v], d);
              }
              // inactive pairs stay exactly 0 (M:346-351)
              ((float*)(sb + L.s_xv))[sub * L.xv_stride + tf] =
                  (p1c && p2) ? (x2 == 1.f ? d : x2 * d) : 0.f;
            }
          } else {
            for (int sub = 0; sub < B; ++sub) {
              const uint16_t* rpos = (const uint16_t*)(sb + L.s_rpos) + sub * FM;
              const float* sval = (const float*)(sb + L.s_sval) + sub * FM;
              const int r2 = rpos[c2];
              const bool p2 = r2 != 0xFFFF;
              const unsigned char* q2 = ring + (size_t)(p2 ? r2 : 0) * RSB + ff1 * SEGB;
              float w2[K];
#pragma unroll
              for (int u = 0; u < SEGB / 16; ++u)
                unpack16<T>(*(const uint4*)(q2 + u * 16), w2 + u * PER, p.dffm);
              float d = 0.f, xs_ = sval[c2];
              bool p1 = p1c;
              if (isctx) {
#pragma unroll
                for (int u = 0; u < K; ++u) d = fmaf(areg[u], w2[u], d);
              } else {
                const int r1 = rpos[c1];
                p1 = r1 != 0xFFFF;
                xs_ *= sval[c1];
                const unsigned char* q1 = ring + (size_t)(p1 ? r1 : 0) * RSB + ff2 * SEGB;
#pragma unroll
                for (int u = 0; u < SEGB / 16; ++u) {
                  float w[PER];
                  unpack16<T>(*(const uint4*)(q1 + u * 16), w, p.dffm);
#pragma unroll
                  for (int v = 0; v < PER; ++v) d = fmaf(w[v], w2[u * PER + v], d);
                }
              }
              ((float*)(sb + L.s_xv))[sub * L.xv_stride + tf] =
                  (p1 && p2) ? (xs_ == 1.f ? d : xs_ * d) : 0.f;
            }
          }
        }
      } else {
        const float* S = (const float*)(cb + L.c_S);
        const unsigned char* cpres = cb + L.c_pres;
        int sub = wi / nch, cc = wi - sub * nch;
        for (int c = wi; c < nchB; c += npg) {
          const float* sval = (const float*)(sb + L.s_sval) + sub * FM;
          const uint16_t* rpos = (const uint16_t*)(sb + L.s_rpos) + sub * FM;
          float* xv = (float*)(sb + L.s_xv) + sub * L.xv_stride;
          const int t = cc * CR_CHUNK + lane;
          if (t < Pc) {
            const uint32_t pr = ptab[t];
            const int f1 = pr & 0xFF, f2 = (pr >> 8) & 0xFF;
            float a[K], bb[K];
#pragma unroll
            for (int u = 0; u < K; ++u) { a[u] = 0.f; bb[u] = 0.f; }
            bool p1 = false, p2 = false;
            const int c2 = f2 - Fc;
#pragma unroll
            for (int m = 0; m < M; ++m) {  // candidate field f2: its slots' segment f1
              const int r2 = rpos[c2 * M + m];
              if (r2 != 0xFFFF) {
                p2 = true;
                const float x2 = sval[c2 * M + m];
                const unsigned char* q2 = ring + (size_t)r2 * RSB + f1 * SEGB;
#pragma unroll
                for (int u = 0; u < SEGB / 16; ++u) {
                  float w[PER];
                  unpack16<T>(*(const uint4*)(q2 + u * 16), w, p.dffm);
#pragma unroll
                  for (int v = 0; v < PER; ++v) bb[u * PER + v] = fmaf(x2, w[v], bb[u * PER + v]);
                }
              }
            }
            if (f1 < Fc) {  // context field: the cached S[x][c]
              p1 = cpres[f1] != 0;
              const float* sc = S + (f1 * F + f2) * K;
#pragma unroll
              for (int u = 0; u < K; ++u) a[u] = sc[u];
            } else {
              const int c1 = f1 - Fc;
#pragma unroll
              for (int m = 0; m < M; ++m) {
                const int r1 = rpos[c1 * M + m];
                if (r1 != 0xFFFF) {
                  p1 = true;
                  const float x1 = sval[c1 * M + m];
                  const unsigned char* q1 = ring + (size_t)r1 * RSB + f2 * SEGB;
#pragma unroll
                  for (int u = 0; u < SEGB / 16; ++u) {
                    float w[PER];
                    unpack16<T>(*(const uint4*)(q1 + u * 16), w, p.dffm);
#pragma unroll
                    for (int v = 0; v < PER; ++v) a[u * PER + v] = fmaf(x1, w[v], a[u * PER + v]);
                  }
                }
              }
            }
            float pv = 0.f;
            if (p1 && p2) {  // inactive pairs stay exactly 0 (M:346-351)
#pragma unroll
              for (int u = 0; u < K; ++u) pv = fmaf(a[u], bb[u], pv);
            }
            xv[t] = pv;
          }
          cc += npg;
          while (cc >= nch) { cc -= nch; ++sub; }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&pdone[xs]);
      xs += G;
      if (xs >= NX) { xs -= NX; par ^= 1u; }
    }
  }
}

}  // namespace dffm
