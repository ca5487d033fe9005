// K1: fused DeepFFM forward (gather -> field-aware latent sums -> DiagMask
// pairs -> MergeNorm -> MLP -> residual logit -> clamped sigmoid).
//
// Replaces model.forward + predict_proba (M:293-397) for a batch.
//
// Work decomposition (one CTA = 8 warps, persistent over tiles of TE examples):
//   phase A (gather-bound): one warp per example.  Lane l owns pair slots
//     p = l, l+32, ...  For pair (f1,f2) it sums the k-segments
//     S[f1][f2] = sum_{j in f1} x_j * ffm[j][f2][:]  and  S[f2][f1], and
//     dots them (M:339, M:344-351).  Every latent segment of every gathered
//     row belongs to exactly one pair, so each row byte is read once and no
//     (F,F,k) latent tensor is ever materialised; the diagonal S[f][f] is
//     never loaded (DiagMask).  Rows are read with L1::no_allocate so L1
//     stays free for the MLP weights.  Lanes then reduce mean/std in f64 and
//     write the standardised merged vector (M:355-360) into a shared-memory
//     tile X[D][TE] (transposed: one column per example).
//   phase B (compute): the CTA runs the MLP over the whole tile as small
//     register-tiled GEMMs (4 outputs x 2 examples per thread, W read
//     through L1, X from shared memory), ReLU between layers (M:367-371),
//     then the output unit, the residual logit = nn + lr + sum(pairs) (M:377)
//     and the clamped sigmoid (M:300-305).
// Non-finite logits report the first example and the first non-finite block
// in lr -> ffm -> merge -> nn -> logit order (M:308-318) via the status word.
#pragma once

#include "common.cuh"

namespace dffm {

constexpr int FWD_THREADS = 256;
constexpr int FWD_WARPS = FWD_THREADS / 32;
#ifndef FWD_MIN_BLOCKS
#define FWD_MIN_BLOCKS 2  // lets ptxas keep a whole pair's slot loads in flight (<=128 regs)
#endif

struct FwdParams {
  const int32_t* idx;
  const float* val;
  float* prob;
  float* logit;
  uint64_t* status;
  int64_t n;
  int64_t n_buckets;
  int64_t status_base;  // added to example numbers in the status word
  int F, M, P, D, k;
  int TE, XS, hmax;
  int n_layers;
  int dims[DFFM_MAX_LAYERS + 1];
  const float* W[DFFM_MAX_LAYERS];
  const float* b[DFFM_MAX_LAYERS];
  const void* lr;
  const void* ffm;
  Deq dlr, dffm;
  // staging mode (tensor-core MLP, mlp_tc.cu): when xout is set the MLP warps
  // do not run the MLP; they write each example's MergeNorm row to
  // xout[e][0..Kp) as fp16 hi / lo planes (xstore*, zero padded), lr_out +
  // sum(pairs) to rout[e] and the non-finite stage bits to fout[e]
  __half* xout;
  int64_t xplane;  // halfs between the hi and the lo plane
  double* rout;
  int* fout;
  int Kp;
};

struct FwdSmem {
  int off_pair, off_X, off_Ha, off_Hb, off_exd, off_flag, off_pres, off_sidx, off_sval, total;
};

__host__ __device__ inline int align16(int x) { return (x + 15) & ~15; }

__host__ __device__ inline FwdSmem fwd_smem_layout(int F, int M, int P, int D, int TE, int XS,
                                                   int hmax) {
  FwdSmem s;
  int o = 0;
  s.off_pair = o; o = align16(o + P * 2);
  s.off_X = o; o = align16(o + D * XS * 4);
  s.off_Ha = o; o = align16(o + hmax * XS * 4);
  s.off_Hb = o; o = align16(o + hmax * XS * 4);
  s.off_exd = o; o = align16(o + 2 * TE * 8);
  s.off_flag = o; o = align16(o + TE * 4);
  s.off_pres = o; o = align16(o + FWD_WARPS * F);
  s.off_sidx = o; o = align16(o + FWD_WARPS * F * M * 4);
  s.off_sval = o; o = align16(o + FWD_WARPS * F * M * 4);
  s.total = o;
  return s;
}

// acc[0..k) += sum over the M slots (si, sv) of one field of x * ffm[j][fb][:]
template <int K, int MU, typename T>
__device__ __forceinline__ void accum_slots(const FwdParams& p, const int* si, const float* sv,
                                            int M, int fb, float* acc) {
  constexpr int KA = K ? K : 32;
  const int k = K ? K : p.k;
  const T* ffm = (const T*)p.ffm;
  if constexpr (MU > 0 && K > 0) {
    // all slot loads first (predicated, zero-filled), then the FMAs: the
    // segment loads of both sides of a pair are in flight together
    float seg[MU][KA];
    float xs[MU];
#pragma unroll
    for (int m = 0; m < MU; ++m) {
      const int j = (m < M) ? si[m] : -1;
      xs[m] = 0.f;
#pragma unroll
      for (int c = 0; c < KA; ++c) seg[m][c] = 0.f;
      if (j >= 0) {
        xs[m] = sv[m];
        Seg<K, T>::load(ffm + ((int64_t)j * p.F + fb) * k, seg[m], p.dffm, k);
      }
    }
#pragma unroll
    for (int m = 0; m < MU; ++m)
#pragma unroll
      for (int c = 0; c < KA; ++c) acc[c] = fmaf(xs[m], seg[m][c], acc[c]);
  } else {
    const int mlim = MU ? MU : M;
    for (int m = 0; m < mlim; ++m) {
      if (MU && m >= M) break;
      const int j = si[m];
      if (j < 0) continue;
      const float x = sv[m];
      float seg[KA];
      Seg<K, T>::load(ffm + ((int64_t)j * p.F + fb) * k, seg, p.dffm, k);
#pragma unroll
      for (int c = 0; c < KA; ++c)
        if (K || c < k) acc[c] = fmaf(x, seg[c], acc[c]);
    }
  }
}

template <int NU>
__device__ __forceinline__ void ldg_chunks_pred(const void* p, int pred, uint4* u) {
  if constexpr (NU == 1) {
    u[0] = ldg_stream16_pred(p, pred);
  } else {
#pragma unroll
    for (int c = 0; c < NU; c += 2)
      ldg_stream32_pred((const unsigned char*)p + 16 * c, pred, u[c], u[c + 1]);
  }
}

// <S[fa][fb], S[fb][fa]> for one pair with every slot load of BOTH sides issued
// before the first FMA (branch-free predicated 128/256-bit loads): one memory
// round trip per pair instead of one per slot.
template <int K, int MU, typename T>
__device__ __forceinline__ float pair_dot_batched(const FwdParams& p, const int* sia,
                                                  const float* sva, const int* sib,
                                                  const float* svb, int M, int fa, int fb) {
  constexpr int SEGB = K * (int)sizeof(T);
  constexpr int NU = SEGB / 16;
  constexpr int PER = 16 / (int)sizeof(T);
  const T* ffm = (const T*)p.ffm;
  uint4 ra[MU][NU], rb[MU][NU];
  float xa[MU], xb[MU];
#pragma unroll
  for (int m = 0; m < MU; ++m) {
    const int ja = (m < M) ? sia[m] : -1;
    const int jb = (m < M) ? sib[m] : -1;
    xa[m] = ja >= 0 ? sva[m] : 0.f;
    xb[m] = jb >= 0 ? svb[m] : 0.f;
    ldg_chunks_pred<NU>(ffm + ((int64_t)(ja > 0 ? ja : 0) * p.F + fb) * K, ja >= 0, ra[m]);
    ldg_chunks_pred<NU>(ffm + ((int64_t)(jb > 0 ? jb : 0) * p.F + fa) * K, jb >= 0, rb[m]);
  }
  float a[K], b[K];
#pragma unroll
  for (int c = 0; c < K; ++c) { a[c] = 0.f; b[c] = 0.f; }
#pragma unroll
  for (int m = 0; m < MU; ++m) {
    float sa[K], sb[K];
#pragma unroll
    for (int c = 0; c < NU; ++c) {
      unpack16<T>(ra[m][c], sa + c * PER, p.dffm);
      unpack16<T>(rb[m][c], sb + c * PER, p.dffm);
    }
#pragma unroll
    for (int c = 0; c < K; ++c) {
      a[c] = fmaf(xa[m], sa[c], a[c]);
      b[c] = fmaf(xb[m], sb[c], b[c]);
    }
  }
  float pv = 0.f;
#pragma unroll
  for (int c = 0; c < K; ++c) pv = fmaf(a[c], b[c], pv);
  return pv;
}

// Two pairs per lane with all four segment loads in flight before any math
// (single-slot fields: cfg1/4/5): doubles the gather's memory-level
// parallelism where each pair is only 2 x 32 B.  Pair b is skipped (returns 0)
// when !act_b; pair a likewise.
template <int K, typename T>
__device__ __forceinline__ float2 pair_dot_x2(const FwdParams& p, const int* sidx,
                                              const float* sval, bool act_a, int fa1, int fa2,
                                              bool act_b, int fb1, int fb2) {
  constexpr int SEGB = K * (int)sizeof(T);
  constexpr int NU = SEGB / 16;
  constexpr int PER = 16 / (int)sizeof(T);
  const T* ffm = (const T*)p.ffm;
  const int ja1 = act_a ? sidx[fa1] : -1, ja2 = act_a ? sidx[fa2] : -1;
  const int jb1 = act_b ? sidx[fb1] : -1, jb2 = act_b ? sidx[fb2] : -1;
  uint4 r[4][NU];
  ldg_chunks_pred<NU>(ffm + ((int64_t)(ja1 > 0 ? ja1 : 0) * p.F + fa2) * K, ja1 >= 0, r[0]);
  ldg_chunks_pred<NU>(ffm + ((int64_t)(ja2 > 0 ? ja2 : 0) * p.F + fa1) * K, ja2 >= 0, r[1]);
  ldg_chunks_pred<NU>(ffm + ((int64_t)(jb1 > 0 ? jb1 : 0) * p.F + fb2) * K, jb1 >= 0, r[2]);
  ldg_chunks_pred<NU>(ffm + ((int64_t)(jb2 > 0 ? jb2 : 0) * p.F + fb1) * K, jb2 >= 0, r[3]);
  const float x[4] = {ja1 >= 0 ? sval[fa1] : 0.f, ja2 >= 0 ? sval[fa2] : 0.f,
                      jb1 >= 0 ? sval[fb1] : 0.f, jb2 >= 0 ? sval[fb2] : 0.f};
  float out[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    float sa[K], sb[K];
#pragma unroll
    for (int c = 0; c < NU; ++c) {
      unpack16<T>(r[2 * q][c], sa + c * PER, p.dffm);
      unpack16<T>(r[2 * q + 1][c], sb + c * PER, p.dffm);
    }
    float pv = 0.f;
#pragma unroll
    for (int c = 0; c < K; ++c)
      pv = fmaf(x[2 * q] * sa[c], x[2 * q + 1] * sb[c], pv);
    out[q] = pv;
  }
  return make_float2(out[0], out[1]);
}

// MergeNorm tail for one example held by one warp (M:355-360).  The raw pair
// values are already in column `el` of X (rows 1..P); lane-partial sums of
// the pairs in `s1`.  Writes the standardised vector back in place, row 0 =
// lr_out, and the per-example residual terms / non-finite flags.
__device__ __forceinline__ void merge_finish(float* X, double* exd, int* flag, int el, int TE,
                                             int XS, int P, int D, int lane, double lr_out,
                                             double s1, int pbad) {
  const double psum = warp_sum(s1);
  const double mu = (psum + lr_out) / D;
  double s2 = 0.0;
  for (int pp = lane; pp < P; pp += 32) {
    const double d = (double)X[(pp + 1) * XS + el] - mu;
    s2 += d * d;
  }
  s2 = warp_sum(s2) + (lr_out - mu) * (lr_out - mu);
  const double denom = sqrt(s2 / D) + 1e-6;  // population std + MERGE_EPS (M:37, M:359-360)
  const double rden = 1.0 / denom;            // one f64 division per example
  int mbad = 0;
  for (int pp = lane; pp < P; pp += 32) {
    const float m = (float)(((double)X[(pp + 1) * XS + el] - mu) * rden);
    X[(pp + 1) * XS + el] = m;
    mbad |= !isfinite(m);
  }
  pbad = __any_sync(0xffffffffu, pbad);
  mbad = __any_sync(0xffffffffu, mbad);
  if (lane == 0) {
    const float m0 = (float)((lr_out - mu) * rden);
    X[el] = m0;
    mbad |= !isfinite(m0);
    exd[el] = lr_out;
    exd[TE + el] = psum;
    flag[el] = (!isfinite(lr_out) ? 1 : 0) | (pbad ? 2 : 0) | (mbad ? 4 : 0);
  }
}

__device__ __forceinline__ void zero_column(float* X, double* exd, int* flag, int el, int TE,
                                            int XS, int D, int lane) {
  for (int i = lane; i < D; i += 32) X[i * XS + el] = 0.f;
  if (lane == 0) { exd[el] = 0.0; exd[TE + el] = 0.0; flag[el] = 0; }
}

// Phase B: MLP over a tile of TE merged columns, residual logit, sigmoid.
// Output slot of column el is out_base + el (valid for el < nvalid).
// Must be entered by the whole CTA; ends with __syncthreads().
__device__ __forceinline__ void mlp_tile(const FwdParams& p, float* X, float* Ha, float* Hb,
                                         double* exd, int* flag, int64_t out_base, int nvalid) {
  const int TE = p.TE, XS = p.XS;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (p.xout) {  // staging mode (mlp_tc.cu): rows, residuals, stage bits; row index = out_base + el
    for (int el = warp; el < nvalid; el += FWD_WARPS) {
      const int64_t e = out_base + el;
      for (int i = lane; i < p.Kp; i += 32)
        xstore1(p.xout, p.xplane, e * p.Kp + i, i < p.D ? X[i * XS + el] : 0.f);
      if (lane == 0) {
        p.rout[e] = exd[el] + exd[TE + el];
        p.fout[e] = flag[el];
      }
    }
    __syncthreads();
    return;
  }
  const float* xin = X;
  int I = p.D;
  float* outb = Ha;
  for (int l = 0; l + 1 < p.n_layers; ++l) {
    const int O = p.dims[l + 1];
    const float* __restrict__ W = p.W[l];
    const float* __restrict__ bl = p.b[l];
    const int O4 = (O + 3) >> 2;
    const int units = O4 * (TE >> 1);
    for (int u = threadIdx.x; u < units; u += FWD_THREADS) {
      const int og = u % O4, eg = u / O4;
      const int o0 = og * 4, e0 = eg * 2;
      float acc0[4], acc1[4];
      if ((O & 3) == 0) {
        const float4 bv = __ldg((const float4*)(bl + o0));
        acc0[0] = acc1[0] = bv.x; acc0[1] = acc1[1] = bv.y;
        acc0[2] = acc1[2] = bv.z; acc0[3] = acc1[3] = bv.w;
#pragma unroll 4
        for (int i = 0; i < I; ++i) {
          const float2 x = *(const float2*)(xin + i * XS + e0);
          const float4 w = __ldg((const float4*)(W + (int64_t)i * O + o0));
          acc0[0] = fmaf(x.x, w.x, acc0[0]); acc0[1] = fmaf(x.x, w.y, acc0[1]);
          acc0[2] = fmaf(x.x, w.z, acc0[2]); acc0[3] = fmaf(x.x, w.w, acc0[3]);
          acc1[0] = fmaf(x.y, w.x, acc1[0]); acc1[1] = fmaf(x.y, w.y, acc1[1]);
          acc1[2] = fmaf(x.y, w.z, acc1[2]); acc1[3] = fmaf(x.y, w.w, acc1[3]);
        }
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c) acc0[c] = acc1[c] = (o0 + c < O) ? __ldg(bl + o0 + c) : 0.f;
        for (int i = 0; i < I; ++i) {
          const float2 x = *(const float2*)(xin + i * XS + e0);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            if (o0 + c < O) {
              const float w = __ldg(W + (int64_t)i * O + o0 + c);
              acc0[c] = fmaf(x.x, w, acc0[c]);
              acc1[c] = fmaf(x.y, w, acc1[c]);
            }
          }
        }
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (o0 + c < O) {
          if (!isfinite(acc0[c])) atomicOr(&flag[e0], 8);
          if (!isfinite(acc1[c])) atomicOr(&flag[e0 + 1], 8);
          *(float2*)(outb + (o0 + c) * XS + e0) =
              make_float2(relu_nan(acc0[c]), relu_nan(acc1[c]));
        }
      }
    }
    __syncthreads();
    xin = outb;
    I = O;
    outb = (outb == Ha) ? Hb : Ha;
  }

  // output unit + residual logit + sigmoid
  for (int el = warp; el < nvalid; el += FWD_WARPS) {
    const int64_t e = out_base + el;
    double nn = 0.0;
    if (p.n_layers > 0) {
      const float* __restrict__ Wo = p.W[p.n_layers - 1];
      float s = 0.f;
      for (int i = lane; i < I; i += 32) s = fmaf(xin[i * XS + el], __ldg(Wo + i), s);
      s = warp_sumf(s);
      nn = (double)s + (double)__ldg(p.b[p.n_layers - 1]);  // M:372-373
    }
    if (lane == 0) {
      const double logit = nn + exd[el] + exd[TE + el];  // M:377
      p.prob[e] = (float)sigmoid_clamped(logit);
      if (p.logit) p.logit[e] = (float)logit;
      if (!isfinite(logit)) {
        const int fl = flag[el];
        const int blk = (fl & 1) ? DFFM_BLOCK_LR : (fl & 2) ? DFFM_BLOCK_FFM
                      : (fl & 4) ? DFFM_BLOCK_MERGE : (fl & 8) ? DFFM_BLOCK_NN
                      : DFFM_BLOCK_LOGIT;
        atomicMin((unsigned long long*)p.status,
                  (unsigned long long)status_key(p.status_base + e, blk, DFFM_NUMERIC));
      }
    }
  }
  __syncthreads();
}

__device__ __forceinline__ void build_pairtab(uint16_t* pairtab, int F) {
  // DiagMask pair order (M:113-117): strict upper triangle, row-major
  for (int f1 = threadIdx.x; f1 < F; f1 += FWD_THREADS) {
    const int base = f1 * F - f1 * (f1 + 1) / 2;
    for (int f2 = f1 + 1; f2 < F; ++f2) pairtab[base + f2 - f1 - 1] = (uint16_t)(f1 | (f2 << 8));
  }
}

// Stage one example's padded slots (F fields x M) into the warp's buffers,
// returning the f64 lr partial sum (M:338) and flagging out-of-range indices.
template <typename T>
__device__ __forceinline__ double stage_slots(const FwdParams& p, const int32_t* gi,
                                              const float* gv, int nslots, int* sidx,
                                              float* sval, int lane, int& bad) {
  const T* lrt = (const T*)p.lr;
  double lrs = 0.0;
  for (int s = lane; s < nslots; s += 32) {
    int j = __ldg(gi + s);
    const float x = __ldg(gv + s);
    if (j >= p.n_buckets || j < -1) { bad = 1; j = -1; }
    sidx[s] = j;
    sval[s] = x;
    if (j >= 0) lrs += (double)x * (double)load_elem<T>(lrt + j, p.dlr);
  }
  return lrs;
}

template <int K, int MU, typename T>
__global__ void __launch_bounds__(FWD_THREADS, FWD_MIN_BLOCKS)
fwd_kernel(FwdParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  const FwdSmem L = fwd_smem_layout(p.F, p.M, p.P, p.D, p.TE, p.XS, p.hmax);
  uint16_t* pairtab = (uint16_t*)(smem + L.off_pair);
  float* X = (float*)(smem + L.off_X);
  float* Ha = (float*)(smem + L.off_Ha);
  float* Hb = (float*)(smem + L.off_Hb);
  double* exd = (double*)(smem + L.off_exd);
  int* flag = (int*)(smem + L.off_flag);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int FM = p.F * p.M;
  unsigned char* spres = smem + L.off_pres + warp * p.F;
  int* sidx = (int*)(smem + L.off_sidx) + warp * FM;
  float* sval = (float*)(smem + L.off_sval) + warp * FM;
  const int TE = p.TE, XS = p.XS, P = p.P, D = p.D;
  constexpr int KA = K ? K : 32;
  const int k = K ? K : p.k;

  build_pairtab(pairtab, p.F);
  __syncthreads();
  const float bias = load_elem<T>((const T*)p.lr + p.n_buckets, p.dlr);
  const int64_t ntiles = (p.n + TE - 1) / TE;

  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    // ------------------------------------------------ phase A: one warp per example
    for (int el = warp; el < TE; el += FWD_WARPS) {
      const int64_t e = tile * TE + el;
      if (e >= p.n) { zero_column(X, exd, flag, el, TE, XS, D, lane); continue; }
      int bad = 0;
      const double lrs = stage_slots<T>(p, p.idx + e * FM, p.val + e * FM, FM, sidx, sval,
                                        lane, bad);
      __syncwarp();
      for (int f = lane; f < p.F; f += 32) {
        unsigned char pr = 0;
        for (int m = 0; m < p.M; ++m) pr |= (sidx[f * p.M + m] >= 0);
        spres[f] = pr;
      }
      if (__any_sync(0xffffffffu, bad) && lane == 0)
        atomicMin((unsigned long long*)p.status,
                  (unsigned long long)status_key(p.status_base + e, DFFM_BLOCK_NONE,
                                                 DFFM_CONTRACT));
      const double lr_out = (double)bias + warp_sum(lrs);  // M:327, M:338
      __syncwarp();

      double s1 = 0.0;
      int pbad = 0;
      for (int pp = lane; pp < P; pp += 32) {
        const uint32_t pr = pairtab[pp];
        const int f1 = pr & 0xFF, f2 = pr >> 8;
        float pv = 0.f;
        if (spres[f1] & spres[f2]) {  // inactive pairs stay exactly 0 (M:346-351)
          const int M = p.M;
          if constexpr (K > 0 && MU > 0 && (K * sizeof(T)) % 16 == 0) {
            pv = pair_dot_batched<K, MU, T>(p, sidx + f1 * M, sval + f1 * M, sidx + f2 * M,
                                            sval + f2 * M, M, f1, f2);
          } else {
            float a[KA], bb[KA];
#pragma unroll
            for (int c = 0; c < KA; ++c) { a[c] = 0.f; bb[c] = 0.f; }
            accum_slots<K, MU, T>(p, sidx + f1 * M, sval + f1 * M, M, f2, a);   // S[f1][f2]
            accum_slots<K, MU, T>(p, sidx + f2 * M, sval + f2 * M, M, f1, bb);  // S[f2][f1]
#pragma unroll
            for (int c = 0; c < KA; ++c)
              if (K || c < k) pv = fmaf(a[c], bb[c], pv);
          }
        }
        X[(pp + 1) * XS + el] = pv;
        s1 += (double)pv;
        pbad |= !isfinite(pv);
      }
      merge_finish(X, exd, flag, el, TE, XS, P, D, lane, lr_out, s1, pbad);
    }
    __syncthreads();
    // ------------------------------------------------ phase B: MLP over the tile
    const int64_t base = tile * TE;
    const int nvalid = (p.n - base) < TE ? (int)(p.n - base) : TE;
    mlp_tile(p, X, Ha, Hb, exd, flag, base, nvalid);
  }
}

// MLP over one X tile by NM warps (thread index mt in [0, 32*NM)); named
// barrier 1 synchronises the MLP warps between layers.
template <int NM>
__device__ __forceinline__ void mlp_warps_tile(const FwdParams& p, const float* xin,
                                               const double* exd, int* flag, float* Ha,
                                               float* Hb, int64_t base, int mt) {
  const int TE = p.TE, XS = p.XS;
  const int lane = mt & 31, mw = mt >> 5;
  if (p.xout) {  // staging mode: rows for the tensor-core MLP (mlp_tc.cu)
    for (int el = mw; el < TE; el += NM) {
      const int64_t e = base + el;
      if (e >= p.n) continue;
      for (int i = lane; i < p.Kp; i += 32)
        xstore1(p.xout, p.xplane, e * p.Kp + i, i < p.D ? xin[i * XS + el] : 0.f);
      if (lane == 0) {
        p.rout[e] = exd[el] + exd[TE + el];
        p.fout[e] = flag[el];
      }
    }
    __syncwarp();
    return;
  }
  int I = p.D;
  float* outb = Ha;
  for (int l = 0; l + 1 < p.n_layers; ++l) {
    const int O = p.dims[l + 1];
    const float* __restrict__ W = p.W[l];
    const float* __restrict__ bl = p.b[l];
    const int O4 = O >> 2;
    const int units = O4 * (TE >> 2);
    for (int u = mt; u < units; u += 32 * NM) {
      const int o0 = (u % O4) * 4, e0 = (u / O4) * 4;
      const float4 bv = __ldg((const float4*)(bl + o0));
      float acc[4][4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        acc[r][0] = bv.x; acc[r][1] = bv.y; acc[r][2] = bv.z; acc[r][3] = bv.w;
      }
#pragma unroll 8
      for (int i = 0; i < I; ++i) {
        const float4 x = *(const float4*)(xin + i * XS + e0);
        const float4 w = __ldg((const float4*)(W + (int64_t)i * O + o0));
        const float xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          acc[r][0] = fmaf(xs[r], w.x, acc[r][0]);
          acc[r][1] = fmaf(xs[r], w.y, acc[r][1]);
          acc[r][2] = fmaf(xs[r], w.z, acc[r][2]);
          acc[r][3] = fmaf(xs[r], w.w, acc[r][3]);
        }
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        float4 o;
        o.x = relu_nan(acc[0][c]);  // M:370
        o.y = relu_nan(acc[1][c]);
        o.z = relu_nan(acc[2][c]);
        o.w = relu_nan(acc[3][c]);
#pragma unroll
        for (int r = 0; r < 4; ++r)
          if (!isfinite(acc[r][c])) atomicOr(&flag[e0 + r], 8);
        *(float4*)(outb + (o0 + c) * XS + e0) = o;
      }
    }
    named_bar_sync(1, 32 * NM);
    xin = outb;
    I = O;
    outb = (outb == Ha) ? Hb : Ha;
  }
  for (int el = mw; el < TE; el += NM) {
    const int64_t e = base + el;
    if (e >= p.n) continue;
    double nn = 0.0;
    if (p.n_layers > 0) {
      const float* __restrict__ Wo = p.W[p.n_layers - 1];
      float sacc = 0.f;
      for (int i = lane; i < I; i += 32) sacc = fmaf(xin[i * XS + el], __ldg(Wo + i), sacc);
      sacc = warp_sumf(sacc);
      nn = (double)sacc + (double)__ldg(p.b[p.n_layers - 1]);  // M:372-373
    }
    if (lane == 0) {
      const double logit = nn + exd[el] + exd[TE + el];  // M:377
      p.prob[e] = (float)sigmoid_clamped(logit);
      if (p.logit) p.logit[e] = (float)logit;
      if (!isfinite(logit)) {
        const int fl = flag[el];
        const int blk = (fl & 1) ? DFFM_BLOCK_LR : (fl & 2) ? DFFM_BLOCK_FFM
                      : (fl & 4) ? DFFM_BLOCK_MERGE : (fl & 8) ? DFFM_BLOCK_NN
                      : DFFM_BLOCK_LOGIT;
        atomicMin((unsigned long long*)p.status,
                  (unsigned long long)status_key(p.status_base + e, blk, DFFM_NUMERIC));
      }
    }
  }
  named_bar_sync(1, 32 * NM);  // Ha/Hb and this X buffer are free again
}

}  // namespace dffm
