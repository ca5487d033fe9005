// K2: sequential Adagrad trainer (replaces training._train_lines T:172-185 =
// forward M:321 -> predict_proba M:300 -> backward_update M:440-533, batch 1,
// in the reference's exact example order).
//
// One persistent CTA (1024 threads) walks the whole stream; every example is
// a dependent step, so the design goal is per-example latency:
//   * the MLP weights and their accumulators are staged into shared memory
//     for the whole launch (159 KB at cfg3) and written back at the end, so
//     every GEMV and every MLP Adagrad step runs at shared-memory latency;
//   * GEMVs use conflict-free mappings with deterministic split-K
//     reductions (fixed order: results do not depend on scheduling);
//   * the hashed lr / ffm rows stay in HBM (L2-hot) and are read-modified-
//     written in place, coalesced along the row.
// All model arithmetic is f64 over f32 storage like the reference
// (M:15-18), with the roundings it performs:
//   forward   S[f][g] = sum_m x_m * f64(w)       (M:339), pairs in f64 (M:351),
//             MergeNorm (M:355-360), MLP in f64 with f32 weights (M:367-373)
//   Adagrad   acc64 = f64(acc32) + g*g ; acc32 <- f32(acc64) ;
//             w32 <- f32(f64(w32) - (lr*g) * (1/sqrt(acc64)))     (M:510-513, M:545-554)
//             -- separate IEEE mul / add / sqrt / div, never FMA-contracted
//   duplicate buckets across fields: gradients summed in occurrence order
//             before one update (sort-and-segment, M:424-437)
//   sparse    zero-gradient slots are skipped; byte-identical to dense (M:536-572)
#include <algorithm>
#include <cooperative_groups.h>
#include <math.h>
#include <stdlib.h>

#include "common.cuh"

namespace dffm {

#ifndef DFFM_TR_THREADS
#define DFFM_TR_THREADS 1024
#endif
constexpr int TR_THREADS = DFFM_TR_THREADS;
constexpr int TR_WARPS = TR_THREADS / 32;
#ifndef DFFM_TR_HW_THREADS
#define DFFM_TR_HW_THREADS 512
#endif
constexpr int TR_HW_THREADS = DFFM_TR_HW_THREADS;  // threads per Hogwild worker (K6)
constexpr int TR_CLUSTER = 8;  // CTAs per cluster for the split trainer

// Phase timestamps (debug builds only, -DDFFM_TR_TRACE): SM clock of thread 0
// of rank 0 at each phase boundary, for examples [TR_T0, TR_T0 + TR_TN).
#ifdef DFFM_TR_TRACE
constexpr int TR_T0 = 16, TR_TN = 64, TR_NPH = 40;
__device__ long long g_tr_trace[TR_TN * TR_NPH];
#define TR_MARK(ph)                                                            \
  do {                                                                         \
    if (threadIdx.x == 0 && rank == 0 && e >= TR_T0 && e < TR_T0 + TR_TN)      \
      g_tr_trace[(e - TR_T0) * TR_NPH + (ph)] = clock64();                     \
  } while (0)
#define TR_MARK_T(ph, thr)                                                     \
  do {                                                                         \
    if (threadIdx.x == (thr) && rank == 0 && e >= TR_T0 && e < TR_T0 + TR_TN)  \
      g_tr_trace[(e - TR_T0) * TR_NPH + (ph)] = clock64();                     \
  } while (0)
#else
#define TR_MARK(ph) do { } while (0)
#define TR_MARK_T(ph, thr) do { } while (0)
#endif

struct TrainParams {
  const int32_t* idx;
  const float* val;
  const uint8_t* labels;
  double* prob_out;
  uint64_t* status;
  int64_t n;
  int64_t n_buckets;
  int F, M, k, P, D;
  int n_layers;
  int dims[DFFM_MAX_LAYERS + 1];
  int hsum;      // sum of hidden sizes
  int dmax;      // max layer width incl. D
  int mlp_size;  // floats in W+b over all layers
  int mlp_dup;   // floats in W+b of layers >= 1 (second weight buffer of the cluster trainer)
  int mlp_smem;  // 1: MLP weights + accumulators resident in shared memory
  int hogwild;   // K6: each CTA is an independent worker over examples blockIdx.x + i*gridDim.x
  float* lr;
  float* ffm;
  float* W[DFFM_MAX_LAYERS];
  float* b[DFFM_MAX_LAYERS];
  float* lr_acc;
  float* ffm_acc;
  float* W_acc[DFFM_MAX_LAYERS];
  float* b_acc[DFFM_MAX_LAYERS];
  double lr_ffm, lr_lr, lr_nn, power_t;
  int sparse;
};

struct TrSmem {
  int off_sidx, off_sval, off_pres, off_lrp, off_S, off_v, off_merged, off_pre, off_act, off_d0,
      off_d1, off_dv, off_nxt, off_lead, off_fact, off_red, off_part, off_dpm, off_ptab, off_ulist,
      off_gkg, off_sfield, off_zbuf, off_dpart, off_dg, off_mlp, total;
};

__host__ __device__ inline int a16(int x) { return (x + 15) & ~15; }

// S[f][g][c] in shared memory (f64): segment stride k + 1 and an odd row stride, so
// the strided walks -- pairs read S[f1][f2] / S[f2][f1] with lanes along f2, the
// backward reads S[g][f] with lanes along g -- spread over the banks.  (With the dense
// [F][F][k] layout a row is F*k*8 = 1,536 B at cfg3, a multiple of 128: 32-way conflicts
// made the pair loop 5.2k cycles and the dp/fact loop 5.3k of the 70k per example.)
__host__ __device__ inline int tr_s_seg(int k) { return k + 1; }
__host__ __device__ inline int tr_s_row(int F, int k) { return (F * (k + 1)) | 1; }

__host__ __device__ inline TrSmem tr_smem_layout(int F, int M, int k, int D, int hsum, int dmax,
                                                 int mlp_floats) {
  TrSmem s;
  const int FM = F * M;
  int o = 0;
  s.off_sidx = o; o = a16(o + FM * 4);
  s.off_sval = o; o = a16(o + FM * 8);
  s.off_pres = o; o = a16(o + F * 4);
  s.off_lrp = o; o = a16(o + F * 8);
  s.off_S = o; o = a16(o + F * tr_s_row(F, k) * 8);
  s.off_v = o; o = a16(o + D * 8);
  s.off_merged = o; o = a16(o + D * 8);
  s.off_pre = o; o = a16(o + (hsum + 1) * 8);
  s.off_act = o; o = a16(o + (hsum + 1) * 8);
  s.off_d0 = o; o = a16(o + dmax * 8);
  s.off_d1 = o; o = a16(o + dmax * 8);
  s.off_dv = o; o = a16(o + D * 8);
  s.off_nxt = o; o = a16(o + FM * 4);
  s.off_lead = o; o = a16(o + FM * 4);
  s.off_fact = o; o = a16(o + F * 4);
  s.off_red = o; o = a16(o + 2 * TR_WARPS * 8);  // two ping-pong slots
  s.off_part = o; o = a16(o + TR_THREADS * 8);
  s.off_dpm = o; o = a16(o + F * F * 8);
  s.off_ptab = o; o = a16(o + (F * (F - 1) / 2) * 2);
  s.off_ulist = o; o = a16(o + FM * 4 + 16);
  s.off_gkg = o; o = a16(o + F * k);
  s.off_sfield = o; o = a16(o + FM);
  s.off_zbuf = o; o = a16(o + dmax * 8);
  s.off_dpart = o; o = a16(o + D * 8);
  s.off_dg = o; o = a16(o + (hsum + 1) * 8);
  s.off_mlp = o; o = a16(o + mlp_floats * 4);
  s.total = o;
  return s;
}

// acc**(-power_t) (M:400-404).  For power_t = 0.5 the reference evaluates
// 1.0/np.sqrt(acc): two correctly rounded f64 ops, reproduced exactly.  (A
// 1-ulp rsqrt() was measured: ~8% faster, but over thousands of sequential
// steps the last-bit differences compound through the training dynamics and
// 13% of slots drifted past the 1e-5 contract -- so it is opt-in only.)
#ifndef DFFM_FAST_INVSQRT
#define DFFM_FAST_INVSQRT 0
#endif
// The general power is kept out of line: inlined at every Adagrad call site it made the
// trainer 166 KB of SASS, more than the SM's instruction cache, and every phase of the
// per-example chain then started with instruction-fetch misses.
__device__ __noinline__ double inv_pow_general(double acc, double pt) { return pow(acc, -pt); }
__device__ __forceinline__ double inv_pow(double acc, double pt) {
  if (pt == 0.5) return DFFM_FAST_INVSQRT ? rsqrt(acc) : __ddiv_rn(1.0, __dsqrt_rn(acc));
  return inv_pow_general(acc, pt);
}

// One Adagrad element step with the reference's rounding (M:510-513) on values in
// registers: returns {new weight, new accumulator}.  (One out-of-line copy instead of
// eight inlined ones was measured: 32.6k vs 32.9k examples/s -- instruction fetch is
// not what bounds the chain.)
__device__ __forceinline__
float2 adagrad_core(float w, float acc, double g, double lr, double pt) {
  const double a64 = __dadd_rn((double)acc, __dmul_rn(g, g));
  const double step = __dmul_rn(__dmul_rn(lr, g), inv_pow(a64, pt));
  return make_float2(__double2float_rn(__dsub_rn((double)w, step)), __double2float_rn(a64));
}

__device__ __forceinline__ void adagrad(float* w, float* acc, double g, double lr, double pt) {
  const float2 r = adagrad_core(*w, *acc, g, lr, pt);
  *acc = r.y;
  *w = r.x;
}

// The same step on a weight held in a register: returns the new weight (the caller
// publishes it); the accumulator is updated in place.
__device__ __forceinline__ float adagrad_val(float w, float* acc, double g, double lr, double pt) {
  const float2 r = adagrad_core(w, *acc, g, lr, pt);
  *acc = r.y;
  return r.x;
}

// MLP element of the working copy: shared memory, or global (L2-only reads so
// no SM keeps a stale L1 line of a weight another SM -- Hogwild worker or
// cluster peer -- updated)
__device__ __forceinline__ double ldm(const float* q, bool glob) {
  return (double)(glob ? __ldcg(q) : *q);
}

// Same step on a global-memory slot shared across the cluster's SMs: L2-only
// accesses so no CTA can read a stale L1 line of another SM's update.
__device__ __forceinline__ void adagrad_g(float* w, float* acc, double g, double lr, double pt) {
  const float2 r = adagrad_core(__ldcg(w), __ldcg(acc), g, lr, pt);
  __stcg(acc, r.y);
  __stcg(w, r.x);
}

__device__ __forceinline__ void adagrad_m(float* w, float* acc, double g, double lr, double pt,
                                          bool glob) {
  if (glob) adagrad_g(w, acc, g, lr, pt);
  else adagrad(w, acc, g, lr, pt);
}

// Block-wide f64 sum (all threads call); result broadcast to all.  One
// barrier: warps publish partials into a ping-pong slot, then every thread
// folds the TR_WARPS partials itself in a fixed order (deterministic).
template <int NW = TR_WARPS>
__device__ double block_sum(double v, double* red, int& ctr) {
  constexpr int TR_WARPS = NW;
  // every thread calls block_sum the same number of times, so the per-thread
  // call counter selects the same ping-pong slot block-wide; reusing a slot
  // two calls later is ordered by the intervening call's barrier
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  double* slot = red + (++ctr & 1) * TR_WARPS;
  if (lane == 0) slot[warp] = v;
  __syncthreads();
  double t = lane < TR_WARPS ? slot[lane] : 0.0;  // fixed-order tree fold, every warp
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  return t;
}

// block_sum that also or-reduces a per-thread flag in its one barrier
template <int NW = TR_WARPS>
__device__ double block_sum_or(double v, int& flag, double* red, int& ctr) {
  constexpr int TR_WARPS = NW;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  double* slot = red + (++ctr & 1) * TR_WARPS;
  if (lane == 0) slot[warp] = v;
  flag = __syncthreads_or(flag);
  double t = lane < TR_WARPS ? slot[lane] : 0.0;  // the same fixed-order fold as block_sum
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  return t;
}

__device__ __forceinline__ int tr_pair_pos(int a, int b, int F) {
  return a * F - a * (a + 1) / 2 + (b - a - 1);
}

__device__ __forceinline__ double sigmoid_raw(double logit) {  // M:293-297
  if (logit >= 0.0) return 1.0 / (1.0 + exp(-fmin(logit, 60.0)));
  const double e = exp(fmax(logit, -60.0));
  return e / (1.0 + e);
}

// NT threads per CTA: 1024 for the sequential trainer (one chain, all of the
// SM); the Hogwild workers use NT = 512 so two workers share an SM
template <int C, int NT = TR_THREADS>
__global__ void __launch_bounds__(NT, 1024 / NT) train_kernel(TrainParams p) {
  constexpr int TR_THREADS = NT;  // shadow the file-wide defaults inside the kernel
  constexpr int TR_WARPS = NT / 32;
  extern __shared__ __align__(128) unsigned char smem[];
  const int F = p.F, M = p.M, k = p.k, P = p.P, D = p.D, FM = F * M, Fk = F * k;
  const TrSmem L =
      tr_smem_layout(F, M, k, D, p.hsum, p.dmax, p.mlp_smem ? 2 * p.mlp_size + p.mlp_dup : 0);
  int* sidx = (int*)(smem + L.off_sidx);
  double* sval = (double*)(smem + L.off_sval);
  int* pres = (int*)(smem + L.off_pres);
  double* lrp = (double*)(smem + L.off_lrp);
  double* S = (double*)(smem + L.off_S);
  const int SK = tr_s_seg(p.k), SR = tr_s_row(p.F, p.k);  // segment / row stride of S
  double* v = (double*)(smem + L.off_v);
  double* merged = (double*)(smem + L.off_merged);
  double* pre = (double*)(smem + L.off_pre);
  double* act = (double*)(smem + L.off_act);
  double* d0 = (double*)(smem + L.off_d0);
  double* d1 = (double*)(smem + L.off_d1);
  double* dv = (double*)(smem + L.off_dv);
  int* nxt = (int*)(smem + L.off_nxt);
  int* lead = (int*)(smem + L.off_lead);
  int* fact = (int*)(smem + L.off_fact);
  double* red = (double*)(smem + L.off_red);
  double* part = (double*)(smem + L.off_part);
  double* dpm = (double*)(smem + L.off_dpm);
  uint16_t* ptab = (uint16_t*)(smem + L.off_ptab);
  int* ulist = (int*)(smem + L.off_ulist);
  int* nuniq = ulist + FM;
  unsigned char* gkg = smem + L.off_gkg;
  unsigned char* sfield = smem + L.off_sfield;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NL = p.n_layers;
  const double pt = p.power_t;
  int bsc = 0;  // block_sum call counter (same in every thread)

  // constant tables: pair order (M:113-117), latent column -> target field,
  // slot -> field
  for (int f1 = tid; f1 < F; f1 += TR_THREADS) {
    const int base = f1 * F - f1 * (f1 + 1) / 2;
    for (int f2 = f1 + 1; f2 < F; ++f2) ptab[base + f2 - f1 - 1] = (uint16_t)(f1 | (f2 << 8));
  }
  for (int t = tid; t < Fk; t += TR_THREADS) gkg[t] = (unsigned char)(t / k);
  for (int t = tid; t < FM; t += TR_THREADS) sfield[t] = (unsigned char)(t / M);

  // ---- cluster split (C > 1): CTA `rank` owns layer-0 columns [c0, c0+W0)
  // (weights, accumulators, GEMV partials, updates), every other layer and the
  // forward chain are replicated (identical deterministic updates in every CTA)
  const int rank = C > 1 ? (int)cooperative_groups::this_cluster().block_rank() : 0;
  const int W0 = (C > 1 && NL > 1) ? p.dims[1] / C : (NL > 0 ? p.dims[1] : 0);
  const int c0 = (C > 1 && NL > 1) ? rank * W0 : 0;
  double* zbuf = (double*)(smem + L.off_zbuf);
  double* dpart = (double*)(smem + L.off_dpart);
  double* dg = (double*)(smem + L.off_dg);  // gradients w.r.t. the layers' pre-activations

  // ---- MLP working copies: shared memory for the whole launch when they fit.
  // Layer 0 is stored as its [I][W0] column slice (W0 = O when C == 1).
  float* Wl[DFFM_MAX_LAYERS];
  float* bl[DFFM_MAX_LAYERS];
  float* Wal[DFFM_MAX_LAYERS];
  float* bal[DFFM_MAX_LAYERS];
  int ldw[DFFM_MAX_LAYERS];  // row stride of the working copy
  // Cluster trainer: the replicated layers (l >= 1) are UPDATED by one owner CTA per
  // row (row r on rank r % C; bias element c on rank c % C) instead of by every CTA --
  // the Adagrad step is FP64 division / square-root / conversion throughput
  // (tools/fp64_bench.cu), so 8 copies of it cost 8x the pipe time of one.  The owner
  // publishes the new weights to every CTA's copy through DSMEM.  Other CTAs may
  // still be reading the old values (upstream gradients use the PRE-update weights,
  // M:473-475), so the layers' weights are double-buffered: example e reads buffer
  // wp, the owners write every element of their rows (updated or not) into buffer
  // wp ^ 1 of all CTAs, and the end-of-example cluster barrier flips wp.
  const bool dsplit = C > 1 && p.mlp_smem && NL > 1;
  int wp = 0;
  float* Wl2[DFFM_MAX_LAYERS];  // second buffers (dsplit, l >= 1)
  float* bl2[DFFM_MAX_LAYERS];
  {
    float* mw = (float*)(smem + L.off_mlp);
    float* ma = mw + p.mlp_size;
    float* md = ma + p.mlp_size;
    int off = 0, off2 = 0;
    for (int l = 0; l < NL; ++l) {
      const int I = p.dims[l], O = p.dims[l + 1];
      const bool split = (C > 1 && l == 0 && NL > 1);
      const int Ow = split ? W0 : O, cb = split ? c0 : 0;
      ldw[l] = p.mlp_smem ? Ow : O;
      if (p.mlp_smem) {
        Wl[l] = mw + off; bl[l] = mw + off + I * Ow;
        Wal[l] = ma + off; bal[l] = ma + off + I * Ow;
        for (int t = tid; t < I * Ow; t += TR_THREADS) {
          const int i = t / Ow, c = t - i * Ow;
          Wl[l][t] = p.W[l][(int64_t)i * O + cb + c];
          Wal[l][t] = p.W_acc[l][(int64_t)i * O + cb + c];
        }
        for (int t = tid; t < Ow; t += TR_THREADS) { bl[l][t] = p.b[l][cb + t]; bal[l][t] = p.b_acc[l][cb + t]; }
        off += I * Ow + Ow;
        Wl2[l] = Wl[l];
        bl2[l] = bl[l];
        if (dsplit && l > 0) {
          Wl2[l] = md + off2;
          bl2[l] = md + off2 + I * O;
          off2 += I * O + O;
        }
      } else {
        Wl[l] = p.W[l] + cb; bl[l] = p.b[l] + cb; Wal[l] = p.W_acc[l] + cb; bal[l] = p.b_acc[l] + cb;
        Wl2[l] = Wl[l];
        bl2[l] = bl[l];
      }
    }
  }
  if (C > 1) cooperative_groups::this_cluster().sync();  // every CTA resident before DSMEM use
  else __syncthreads();

  // The next example's slots are loaded one example ahead (thread s < FM
  // holds slot s), and its latent / lr rows are prefetched into L2 while the
  // current example's backward pass runs; the current example's accumulator
  // rows are prefetched at its start for its update phase.  (Prefetches only
  // warm L2 -- the values are always re-read after the preceding update.)
  const bool pf_on = FM <= TR_THREADS;
  int pf_j = -1;
  float pf_x = 0.f;
  const bool mg = !p.mlp_smem;  // MLP working copy in global memory
  const int64_t e0 = p.hogwild ? blockIdx.x : 0, estep = p.hogwild ? gridDim.x : 1;
  if (pf_on && tid < FM && e0 < p.n) { pf_j = p.idx[e0 * FM + tid]; pf_x = p.val[e0 * FM + tid]; }
  const int row_bytes = Fk * 4;

  for (int64_t e = e0; e < p.n; e += estep) {
    if (p.hogwild) {  // a worker that hit an error stops the pool (T:253-256)
      if (__syncthreads_or(tid == 0 && __ldcg((const unsigned long long*)p.status) != ~0ull))
        break;
    }
    // ---------------------------------------------------------- stage example
    TR_MARK(0);
    const int label = p.labels[e];
    if (label > 1) {  // M:453-454 ContractError, before touching anything
      if (tid == 0)
        atomicMin((unsigned long long*)p.status,
                  (unsigned long long)status_key(e, DFFM_BLOCK_NONE, DFFM_CONTRACT));
      break;
    }
    int bad = 0;
    if (pf_on) {
      if (tid < FM) {
        int j = pf_j;
        if (j >= p.n_buckets || j < -1) { bad = 1; j = -1; }
        sidx[tid] = j;
        sval[tid] = (double)pf_x;
        if (j >= 0) {  // this example's accumulator rows, for its update phase
          const unsigned char* ar = (const unsigned char*)(p.ffm_acc + (int64_t)j * Fk);
          for (int off = 0; off < row_bytes; off += 128) prefetch_l2(ar + off);
        }
        if (e + estep < p.n) {
          pf_j = p.idx[(e + estep) * FM + tid];
          pf_x = p.val[(e + estep) * FM + tid];
        }
      }
    } else {
      for (int s = tid; s < FM; s += TR_THREADS) {
        int j = p.idx[e * FM + s];
        if (j >= p.n_buckets || j < -1) { bad = 1; j = -1; }
        sidx[s] = j;
        sval[s] = (double)p.val[e * FM + s];
      }
    }
    if (tid < F) fact[tid] = 0;
    if (__syncthreads_or(bad)) {
      if (tid == 0)
        atomicMin((unsigned long long*)p.status,
                  (unsigned long long)status_key(e, DFFM_BLOCK_NONE, DFFM_CONTRACT));
      break;
    }
    TR_MARK(1);
    for (int f = tid; f < F; f += TR_THREADS) {
      int pr = 0;
      double lp = 0.0;
      for (int m = 0; m < M; ++m) {
        const int j = sidx[f * M + m];
        if (j >= 0) {
          pr = 1;
          lp += (double)__ldcg(p.lr + j) * sval[f * M + m];  // M:338 np.dot(lr[idx], x)
        }
      }
      pres[f] = pr;
      lrp[f] = lp;
    }
    // S[f][g][c] = sum_m x_m * ffm[j_m][g][c]  (M:339): warp per field,
    // lanes along the row (coalesced).  Rows of <= 256 floats and <= 4 slots:
    // every load of the field is issued before the first sum (one memory
    // latency per example instead of one per 32-wide column step), sums in
    // slot order as before.
    // Spare warps (warp >= F) build the duplicate lists meanwhile (below).
    const bool dup_split = Fk <= 256 && M <= 4 && (k & 3) == 0 && TR_WARPS - F >= 4;
    if (dup_split && warp >= F) {
      const int dt = tid - F * 32, dn = (TR_WARPS - F) * 32;
      // thread per slot: one pass over the slots (broadcast reads) gives the first slot
      // holding the same bucket (lead) and the next one after it (nxt)
      for (int s = dt; s < FM; s += dn) {
        const int js = sidx[s];
        int ld_ = js >= 0 ? s : -1, nx = 0x7fffffff;
        if (js >= 0)
          for (int s2 = 0; s2 < FM; ++s2) {
            const bool eq = s2 != s && sidx[s2] == js;
            if (eq && s2 < s) ld_ = min(ld_, s2);
            if (eq && s2 > s) nx = min(nx, s2);
          }
        lead[s] = ld_;
        nxt[s] = nx == 0x7fffffff ? -1 : nx;
      }
      named_bar_sync(2, dn);
      if (warp == F) {
        int cnt = 0;
        for (int s0 = 0; s0 < FM; s0 += 32) {
          const int s = s0 + lane;
          const bool isl = s < FM && lead[s] == s;
          const unsigned bm = __ballot_sync(0xffffffffu, isl);
          if (isl) ulist[cnt + __popc(bm & ((1u << lane) - 1u))] = s;
          cnt += __popc(bm);
        }
        if (lane == 0) *nuniq = cnt;
      }
      TR_MARK_T(36, F * 32);
    } else if (Fk <= 256 && M <= 4 && (k & 3) == 0) {
      // 16-byte row loads, lanes along the row: an `ld.cg` is a strong GPU-scope load
      // and the SM issues a thread's strong loads one at a time (~290 cycles each:
      // the 18 scalar loads of a field warp took 5.2k cycles to issue), so the
      // fewer, wider loads are what shortens the gather
      const int nv = Fk >> 2;  // float4 vectors per row (<= 64: two per lane)
      for (int f = warp; f < F; f += TR_WARPS) {
        int js[4];
        double xs[4];
        float4 v[4][2];
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          js[m] = m < M ? sidx[f * M + m] : -1;
          xs[m] = m < M ? sval[f * M + m] : 0.0;
        }
        TR_MARK_T(30, 32);
#pragma unroll
        for (int m = 0; m < 4; ++m)
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int q = lane + 32 * i;
            v[m][i] = (js[m] >= 0 && q < nv)
                          ? __ldcg((const float4*)(p.ffm + (int64_t)js[m] * Fk) + q)
                          : make_float4(0.f, 0.f, 0.f, 0.f);
          }
        TR_MARK_T(31, 32);
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int q = lane + 32 * i;
          if (q < nv) {
            const int gk = 4 * q, gg = gkg[gk];
            double* dst = S + f * SR + gg * SK + (gk - gg * k);
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              double s = 0.0;
#pragma unroll
              for (int m = 0; m < 4; ++m)
                if (js[m] >= 0) s += xs[m] * (double)(&v[m][i].x)[t];
              dst[t] = s;
            }
          }
        }
      }
      TR_MARK_T(37, 32);
      TR_MARK_T(38, 0);
    } else {
      for (int f = warp; f < F; f += TR_WARPS) {
        for (int gk = lane; gk < Fk; gk += 32) {
          double s = 0.0;
          for (int m = 0; m < M; ++m) {
            const int j = sidx[f * M + m];
            if (j >= 0) s += sval[f * M + m] * (double)__ldcg(p.ffm + (int64_t)j * Fk + gk);
          }
          S[f * SR + gkg[gk] * SK + (gk - gkg[gk] * k)] = s;
        }
      }
    }
    // sort-and-segment bookkeeping for the update (M:424-437): lead = first
    // slot holding the bucket, nxt = next slot of the same bucket; the
    // leaders (one per unique bucket, occurrence order) are compacted into
    // ulist by warp 0
    if (!dup_split) {
      for (int s = tid; s < FM; s += TR_THREADS) {
        lead[s] = sidx[s] >= 0 ? s : -1;
        nxt[s] = 0x7fffffff;
      }
      __syncthreads();
      TR_MARK(2);
      // all (s, s2) slot pairs in parallel: lead = smallest equal slot, nxt =
      // smallest equal slot after s
      for (int t = tid; t < FM * FM; t += TR_THREADS) {
        const int s = t / FM, s2 = t - s * FM;
        if (s2 != s && sidx[s] >= 0 && sidx[s2] == sidx[s]) {
          if (s2 < s) atomicMin(&lead[s], s2);
          else atomicMin(&nxt[s], s2);
        }
      }
      __syncthreads();
      for (int s = tid; s < FM; s += TR_THREADS)
        if (nxt[s] == 0x7fffffff) nxt[s] = -1;
      __syncthreads();
      if (warp == 0) {
        int cnt = 0;
        for (int s0 = 0; s0 < FM; s0 += 32) {
          const int s = s0 + lane;
          const bool isl = s < FM && lead[s] == s;
          const unsigned bm = __ballot_sync(0xffffffffu, isl);
          if (isl) ulist[cnt + __popc(bm & ((1u << lane) - 1u))] = s;
          cnt += __popc(bm);
        }
        if (lane == 0) *nuniq = cnt;
      }
    }
    __syncthreads();
    TR_MARK(3);
    // ---------------------------------------------------------- pairs, MergeNorm
    double psum_part = 0.0;
    int ffm_bad = 0;
    for (int pp = tid; pp < P; pp += TR_THREADS) {
      const int f1 = ptab[pp] & 0xFF, f2 = ptab[pp] >> 8;
      double pv = 0.0;
      if (pres[f1] && pres[f2]) {  // M:346-351
        const double* a = S + f1 * SR + f2 * SK;
        const double* b = S + f2 * SR + f1 * SK;
        for (int c = 0; c < k; ++c) pv += a[c] * b[c];
      }
      v[1 + pp] = pv;
      psum_part += pv;
      ffm_bad |= !isfinite(pv);
    }
    TR_MARK(16);
    if (tid == TR_THREADS - 1) {  // a thread without a pair: the serial chain runs beside the pair loop
      double lo = (double)__ldcg(p.lr + p.n_buckets);  // bias, M:327
      for (int f = 0; f < F; ++f)
        if (pres[f]) lo += lrp[f];
      v[0] = lo;
    }
    TR_MARK(17);
    const double psum = block_sum_or<TR_WARPS>(psum_part, ffm_bad, red, bsc);
    TR_MARK(18);
    TR_MARK(19);
    const double lr_out = v[0];
    // the f64 divisions / square root below are computed by the warps that use them
    // (tid < D rounded up to a warp), not by all 32
    const bool dw = warp < (D + 31) / 32;
    const double mu = dw ? (psum + lr_out) / D : 0.0;
    double sq_part = 0.0;
    for (int i = tid; i < D; i += TR_THREADS) {
      const double c = v[i] - mu;
      sq_part += c * c;
    }
    const double sq_sum = block_sum<TR_WARPS>(sq_part, red, bsc);
    const double sd = dw ? sqrt(sq_sum / D) : 0.0;  // np.std (population)
    const double denom = sd + 1e-6;
    TR_MARK(20);
    int merge_bad = 0;
    for (int i = tid; i < D; i += TR_THREADS) {
      merged[i] = (v[i] - mu) / denom;
      merge_bad |= !isfinite(merged[i]);
    }
    merge_bad = __syncthreads_or(merge_bad);
    TR_MARK(4);
    // ---------------------------------------------------------- MLP forward (f64)
    double nn_out = 0.0;
    int nn_bad = 0;
    if (NL > 0) {
      const double* a = merged;
      int hoff = 0;
      for (int l = 0; l + 1 < NL; ++l) {
        const int I = p.dims[l], O = p.dims[l + 1];
        const bool split = (C > 1 && l == 0);
        const int Ow = split ? W0 : O, ld = ldw[l];
        const float* W = wp ? Wl2[l] : Wl[l];
        const float* bcur = wp ? bl2[l] : bl[l];
        // split-K: thread (part, o), o fastest -> conflict-free W reads;
        // partials reduced in fixed part order (deterministic)
        const int G = Ow <= TR_THREADS ? TR_THREADS / Ow : 1;
        if (G > 1) {
          const int o = tid % Ow, pa = tid / Ow;
          if (pa < G) {
            double s = 0.0;
            for (int i = pa; i < I; i += G) s += a[i] * ldm(W + (int64_t)i * ld + o, mg);
            part[pa * Ow + o] = s;
          }
          __syncthreads();
        }
        for (int o = tid; o < Ow; o += TR_THREADS) {
          double z = 0.0;
          if (G > 1) {
            for (int q = 0; q < G; ++q) z += part[q * Ow + o];
          } else {
            for (int i = 0; i < I; ++i) z += a[i] * ldm(W + (int64_t)i * ld + o, mg);
          }
          z += ldm(&bcur[o], mg);  // M:368
          if (split) {
            // owner broadcasts its columns' pre-activations to every CTA (DSMEM)
            for (int rk = 0; rk < C; ++rk)
              cooperative_groups::this_cluster().map_shared_rank(zbuf, rk)[c0 + o] = z;
          } else {
            pre[hoff + o] = z;
            act[hoff + o] = (z != z) ? z : fmax(z, 0.0);  // np.maximum (M:370)
            nn_bad |= !isfinite(z);
          }
        }
        if (split) {
          cooperative_groups::this_cluster().sync();
          for (int o = tid; o < O; o += TR_THREADS) {
            const double z = zbuf[o];
            pre[hoff + o] = z;
            act[hoff + o] = (z != z) ? z : fmax(z, 0.0);
            nn_bad |= !isfinite(z);
          }
        }
        __syncthreads();
        TR_MARK(5 + (l > 0));
        a = act + hoff;
        hoff += O;
      }
      const int I = p.dims[NL - 1];
      double s = 0.0;
      const float* Wo = wp ? Wl2[NL - 1] : Wl[NL - 1];
      for (int i = tid; i < I; i += TR_THREADS) s += a[i] * ldm(&Wo[i], mg);
      nn_out = block_sum_or<TR_WARPS>(s, nn_bad, red, bsc) +
               ldm(wp ? &bl2[NL - 1][0] : &bl[NL - 1][0], mg);  // M:372-373
    }
    TR_MARK(7);
    const double logit = nn_out + lr_out + psum;  // M:377
    if (!isfinite(logit)) {  // M:392-396 (uniform across the block and the cluster)
      if (tid == 0 && rank == 0) {
        const int blk = !isfinite(lr_out) ? DFFM_BLOCK_LR : ffm_bad ? DFFM_BLOCK_FFM
                      : merge_bad ? DFFM_BLOCK_MERGE : nn_bad ? DFFM_BLOCK_NN : DFFM_BLOCK_LOGIT;
        atomicMin((unsigned long long*)p.status,
                  (unsigned long long)status_key(e, blk, DFFM_NUMERIC));
      }
      break;
    }
    if (pf_on && rank == 0 && tid < FM && e + estep < p.n && pf_j >= 0 && pf_j < p.n_buckets) {
      const unsigned char* wr = (const unsigned char*)(p.ffm + (int64_t)pf_j * Fk);
      for (int off = 0; off < row_bytes; off += 128) prefetch_l2(wr + off);
      prefetch_l2(p.lr + pf_j);
    }
    TR_MARK(21);
    // sigmoid and g = p - y (M:456-457) once per CTA, broadcast through shared memory
    // (32 warps each evaluating an f64 exp and a division is ~1.5k cycles of FP64 pipe)
    if (tid == 0) {
      const double p_raw = sigmoid_raw(logit);
      dg[p.hsum] = p_raw - (double)label;
      if (rank == 0) p.prob_out[e] = fmin(fmax(p_raw, 1e-7), 1.0 - 1e-7);
    }
    __syncthreads();
    const double g = dg[p.hsum];
    // ---------------------------------------------------------- MLP backward + update
    // Pass 1: the gradient chain top layer down, every upstream gradient from the
    // PRE-update weights (M:473-475); dg holds the gradient w.r.t. each layer's
    // pre-activations (hidden layer j at its pre/act offset, g at hsum).
    // Pass 2: every layer's Adagrad updates in ONE barrier-free phase -- the updates
    // have no consumer before the next example, and as separate phases each small
    // layer cost a barrier plus a full Adagrad latency (~1.2-2.4k cycles each in the
    // phase trace) that now hides under layer 0's rounds.
    double* dmerged = d1;
    if (NL > 0) {
      TR_MARK(22);
      TR_MARK(23);
      int oout = p.hsum;  // offset in dg of layer l's output gradient
      for (int l = NL - 1; l >= 0; --l) {
        const int I = p.dims[l];
        const bool split = (C > 1 && l == 0);
        const int Ow = split ? W0 : p.dims[l + 1], cb = split ? c0 : 0, ld = ldw[l];
        const float* W = wp ? Wl2[l] : Wl[l];
        const double* dcur = dg + oout;
        const int oin = oout - I;  // offset of layer l's input (pre / act / dg), l > 0
        // warp per row (split layer: partial over this CTA's columns, reduced across
        // the cluster); the ReLU mask of the layer below (M:479) applied on the way out
        if (Ow <= 8) {  // narrow (cluster-split) slice: thread per row
          for (int r = tid; r < I; r += TR_THREADS) {
            double s = 0.0;
            for (int c = 0; c < Ow; ++c) s += ldm(W + (int64_t)r * ld + c, mg) * dcur[cb + c];
            if (l > 0) dg[oin + r] = pre[oin + r] > 0.0 ? s : 0.0;
            else (split ? dpart : dmerged)[r] = s;
          }
        } else {
          for (int r = warp; r < I; r += TR_WARPS) {
            double s = 0.0;
            for (int c = lane; c < Ow; c += 32) s += ldm(W + (int64_t)r * ld + c, mg) * dcur[cb + c];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (lane == 0) {
              if (l > 0) dg[oin + r] = pre[oin + r] > 0.0 ? s : 0.0;
              else (split ? dpart : dmerged)[r] = s;
            }
          }
        }
        if (split) {
          cooperative_groups::this_cluster().sync();
          for (int r = tid; r < I; r += TR_THREADS) {
            double s = 0.0;
            for (int rk = 0; rk < C; ++rk)
              s += cooperative_groups::this_cluster().map_shared_rank(dpart, rk)[r];
            dmerged[r] = s;
          }
        }
        __syncthreads();
        TR_MARK(24 + l);
        oout = oin;
      }
      TR_MARK(8);
      // ---- pass 2: W[r][c] with grad = a_in[r]*d[c]; zero gradients skipped (M:536-554)
      const int rt = TR_THREADS - 1 - tid;  // the small jobs start from the top threads:
      int uo = 0;                           // the low ones have layer 0's extra round
      auto first_item = [&](int n) {  // item of this thread in a job of n items dealt from rt = uo
        const int t = rt - uo + (rt < uo ? TR_THREADS : 0);
        uo = (uo + n) % TR_THREADS;
        return t;
      };
      oout = p.hsum;
      for (int l = NL - 1; l >= 0; --l) {
        const int I = p.dims[l];
        const bool split = (C > 1 && l == 0);
        const int Ow = split ? W0 : p.dims[l + 1], cb = split ? c0 : 0, ld = ldw[l];
        float* W = wp ? Wl2[l] : Wl[l];
        float* Wa = Wal[l];
        const double* dcur = dg + oout;
        const int oin = oout - I;
        const double* a_in = l == 0 ? merged : act + oin;
        if (dsplit && l > 0) {
          // owner rows r = rank, rank + C, ...: one element per thread, the new (or
          // unchanged) weight stored into buffer wp ^ 1 of every CTA
          auto cl = cooperative_groups::this_cluster();
          float* Wn = wp ? Wl[l] : Wl2[l];
          const int nown = (I - rank + C - 1) / C;
          for (int t = first_item(nown * Ow); t < nown * Ow; t += TR_THREADS) {
            const int ro = t / Ow, c = t - ro * Ow, r = rank + C * ro;
            const double ar = a_in[r];
            const double gr = __dmul_rn(ar, dcur[c]);
            // the same skips as the replicated update: zero-gradient slots (M:536-554),
            // and whole dead-ReLU rows when the row is walked by a warp (Ow > 8)
            const bool skip = p.sparse && (gr == 0.0 || (Ow > 8 && ar == 0.0));
            float w = W[r * ld + c];
            if (!skip) w = adagrad_val(w, &Wa[r * ld + c], gr, p.lr_nn, pt);
            for (int rk = 0; rk < C; ++rk) cl.map_shared_rank(Wn, rk)[r * ld + c] = w;
          }
          // bias element c on rank c % C
          float* bc = wp ? bl2[l] : bl[l];
          float* bn = wp ? bl[l] : bl2[l];
          const int nbo = (Ow - rank + C - 1) / C;
          for (int t = first_item(nbo); t < nbo; t += TR_THREADS) {
            const int cbias = rank + C * t;
            const double gr = dcur[cbias];
            float w = bc[cbias];
            if (gr != 0.0 || !p.sparse) w = adagrad_val(w, &bal[l][cbias], gr, p.lr_nn, pt);
            for (int rk = 0; rk < C; ++rk) cl.map_shared_rank(bn, rk)[cbias] = w;
          }
        } else {
          if (Ow <= 8) {  // narrow slice: flat (row, column) per thread
            for (int t = tid; t < I * Ow; t += TR_THREADS) {
              const int r = t / Ow, c = t - r * Ow;
              const double gr = __dmul_rn(a_in[r], dcur[cb + c]);
              if (gr != 0.0 || !p.sparse) adagrad_m(&W[(int64_t)r * ld + c], &Wa[(int64_t)r * ld + c],
                                                    gr, p.lr_nn, pt, mg);
            }
          } else {  // warp per row (dead-ReLU rows skipped warp-uniformly), lanes along c
            for (int r = warp; r < I; r += TR_WARPS) {
              const double ar = a_in[r];
              if (ar == 0.0 && p.sparse) continue;
              float* wr = W + (int64_t)r * ld;
              float* war = Wa + (int64_t)r * ld;
              for (int c = lane; c < Ow; c += 32) {
                const double gr = __dmul_rn(ar, dcur[cb + c]);
                if (gr != 0.0 || !p.sparse) adagrad_m(&wr[c], &war[c], gr, p.lr_nn, pt, mg);
              }
            }
          }
          // bias (M:557-572); in the cluster trainer from the top threads
          for (int c = C > 1 ? first_item(Ow) : tid; c < Ow; c += TR_THREADS) {
            const double gr = dcur[cb + c];
            if (gr != 0.0 || !p.sparse) adagrad_m(&bl[l][c], &bal[l][c], gr, p.lr_nn, pt, mg);
          }
        }
        oout = oin;
      }
      TR_MARK(9);
    }
    // ---------------------------------------------------------- MergeNorm backward (M:413-421)
    double d_lr;
    if (NL > 0) {
      double s_d = 0.0, s_dc = 0.0;
      for (int i = tid; i < D; i += TR_THREADS) {
        s_d += dmerged[i];
        s_dc += dmerged[i] * (v[i] - mu);
      }
      const double sum_d = block_sum<TR_WARPS>(s_d, red, bsc);
      const double dot_dc = block_sum<TR_WARPS>(s_dc, red, bsc);
      if (dw) {
        const double mean_d = sum_d / D;
        const double coef = sd > 0.0 ? dot_dc / (D * sd * denom * denom) : 0.0;
        for (int i = tid; i < D; i += TR_THREADS) {
          double x = (dmerged[i] - mean_d) / denom;
          if (sd > 0.0) x = x - (v[i] - mu) * coef;
          dv[i] = x;
        }
      }
      __syncthreads();
      TR_MARK(10);
      d_lr = g + dv[0];  // M:483
    } else {
      d_lr = g;
      for (int i = tid; i < D; i += TR_THREADS) dv[i] = 0.0;
      __syncthreads();
    }
    // d_pairs[p] = g + dv[1+p] (M:484); dp symmetric (M:492-495).
    // t[g][:] = dp[f][g] * S[g][f][:]; fields whose t is all zero are skipped (M:502)
    // dp[f][g] precomputed per (field, target) into dpm (f64) so the update's
    // inner loop is division-free; fact[f] = field f's t row is not all zero
    for (int t = tid; t < F * F; t += TR_THREADS) {
      const int f = t / F, gg = t - f * F;
      double dpv = 0.0;
      if (gg != f) dpv = g + dv[1 + (gg < f ? tr_pair_pos(gg, f, F) : tr_pair_pos(f, gg, F))];
      dpm[t] = dpv;
      if (gg == f || !pres[f]) continue;
      const double* sgf = S + gg * SR + f * SK;
      int any = 0;
      for (int c = 0; c < k; ++c) any |= (dpv * sgf[c]) != 0.0;
      if (any) atomicOr(&fact[f], 1);
    }
    __syncthreads();
    TR_MARK(11);
    // ---------------------------------------------------------- FFM update (M:490-513)
    // merged gradient per (unique bucket, latent element) in occurrence order
    const int nu = *nuniq;
    // work item = (unique row u, 32-element chunk); items dealt round-robin
    // to the cluster's CTAs and then to warps, so every SM gets ~1/C of it
    const int nchunk = (Fk + 31) >> 5;
    for (int it = rank + C * warp; it < nu * nchunk; it += C * TR_WARPS) {
      const int u = it / nchunk, ch = it - u * nchunk;
      const int s = ulist[u];
      const int j = sidx[s];
      float* wrow = p.ffm + (int64_t)j * Fk;
      float* arow = p.ffm_acc + (int64_t)j * Fk;
      {
        const int gk = ch * 32 + lane;
        if (gk >= Fk) continue;
        const int gg = gkg[gk], c = gk - gg * k;
        double ug = 0.0;
        bool touched = false;
        for (int s2 = s; s2 >= 0; s2 = nxt[s2]) {
          const int f = sfield[s2];
          if (!fact[f]) continue;
          const double tv = dpm[f * F + gg] * S[gg * SR + f * SK + c];  // t[g][c] (M:501)
          ug += sval[s2] * tv;  // x * t (M:505), add.at order
          touched = true;
        }
        if (touched && (ug != 0.0 || !p.sparse))
          adagrad_g(&wrow[gk], &arow[gk], ug, p.lr_ffm, pt);  // M:509-513
      }
    }
    TR_MARK(12);
    // ---------------------------------------------------------- LR + bias (M:516-530)
    if (rank == C - 1) {  // the last CTA gets the fewest FFM work items
      for (int s = tid; s < FM; s += TR_THREADS) {
        if (lead[s] != s) continue;
        const int j = sidx[s];
        double ug = 0.0;
        for (int s2 = s; s2 >= 0; s2 = nxt[s2]) ug += d_lr * sval[s2];
        adagrad_g(&p.lr[j], &p.lr_acc[j], ug, p.lr_lr, pt);
      }
      if (tid == 0) adagrad_g(&p.lr[p.n_buckets], &p.lr_acc[p.n_buckets], d_lr, p.lr_lr, pt);
    }
    // every table write of this example is visible cluster-wide before the
    // next example reads (release/acquire at cluster scope; table reads are L2-only)
    TR_MARK(13);
    if (C > 1) cooperative_groups::this_cluster().sync();
    else __syncthreads();
    if (dsplit) wp ^= 1;
    TR_MARK(14);
  }

  // ---- write the MLP working copies back (also after an error: the reference
  // keeps every update applied before the failing example)
  __syncthreads();
  if (p.mlp_smem) {
    for (int l = 0; l < NL; ++l) {
      const int I = p.dims[l], O = p.dims[l + 1];
      const bool split = (C > 1 && l == 0 && NL > 1);
      if (dsplit && l > 0) {
        // weights: identical in every CTA (buffer wp), rank 0 writes; accumulators:
        // each owner writes its rows / bias elements
        const float* Wc = wp ? Wl2[l] : Wl[l];
        const float* bc = wp ? bl2[l] : bl[l];
        for (int t = tid; t < I * O; t += TR_THREADS) {
          if (rank == 0) p.W[l][t] = Wc[t];
          if ((t / O) % C == rank) p.W_acc[l][t] = Wal[l][t];
        }
        for (int t = tid; t < O; t += TR_THREADS) {
          if (rank == 0) p.b[l][t] = bc[t];
          if (t % C == rank) p.b_acc[l][t] = bal[l][t];
        }
        continue;
      }
      if (!split && rank != 0) continue;  // replicated layers: one writer
      const int Ow = split ? W0 : O, cb = split ? c0 : 0;
      for (int t = tid; t < I * Ow; t += TR_THREADS) {
        const int i = t / Ow, c = t - i * Ow;
        p.W[l][(int64_t)i * O + cb + c] = Wl[l][t];
        p.W_acc[l][(int64_t)i * O + cb + c] = Wal[l][t];
      }
      for (int t = tid; t < Ow; t += TR_THREADS) { p.b[l][cb + t] = bl[l][t]; p.b_acc[l][cb + t] = bal[l][t]; }
    }
  }
  if (C > 1) cooperative_groups::this_cluster().sync();  // no CTA exits while DSMEM is in use
}

}  // namespace dffm

using namespace dffm;

static int tr_validate(const dffm_model* m, int32_t M, int C, TrainParams& p, int* smem_out) {
  if (!m) { set_error("null model"); return DFFM_CONTRACT; }
  if (m->wdtype != DFFM_W_F32) { set_error("training needs f32 tables"); return DFFM_CONTRACT; }
  if (m->n_fields < 1 || m->k < 1 || M < 1) { set_error("bad shape"); return DFFM_CONTRACT; }
  if (m->n_layers < 0 || m->n_layers > DFFM_MAX_LAYERS || m->n_layers == 1) {
    set_error("n_layers=%d invalid", m->n_layers);
    return DFFM_CONTRACT;
  }
  p.F = m->n_fields;
  p.k = m->k;
  p.M = M;
  p.P = p.F * (p.F - 1) / 2;
  p.D = 1 + p.P;
  p.n_buckets = (int64_t)1 << m->hash_bits;
  p.n_layers = m->n_layers;
  p.hsum = 0;
  p.dmax = p.D;
  p.mlp_size = 0;
  for (int l = 0; l <= DFFM_MAX_LAYERS; ++l) p.dims[l] = m->dims[l];
  if (p.n_layers) {
    if (m->dims[0] != p.D || m->dims[p.n_layers] != 1) {
      set_error("MLP dims do not match 1+F(F-1)/2 -> ... -> 1");
      return DFFM_CONTRACT;
    }
    for (int l = 1; l < p.n_layers; ++l) {
      p.hsum += m->dims[l];
      if (m->dims[l] > p.dmax) p.dmax = m->dims[l];
    }
    for (int l = 0; l < p.n_layers; ++l) {
      const int Ow = (C > 1 && l == 0) ? m->dims[1] / C : m->dims[l + 1];  // layer-0 slice
      p.mlp_size += m->dims[l] * Ow + Ow;
    }
  }
  p.lr = (float*)m->lr;
  p.ffm = (float*)m->ffm;
  for (int l = 0; l < p.n_layers; ++l) {
    p.W[l] = (float*)m->W[l];
    p.b[l] = (float*)m->b[l];
  }
  const int smax = max_smem_optin_current();
  p.mlp_dup = 0;
  if (C > 1)
    for (int l = 1; l < p.n_layers; ++l) p.mlp_dup += m->dims[l] * m->dims[l + 1] + m->dims[l + 1];
  TrSmem L = tr_smem_layout(p.F, p.M, p.k, p.D, p.hsum, p.dmax, 2 * p.mlp_size + p.mlp_dup);
  p.mlp_smem = L.total <= smax;
  if (!p.mlp_smem) L = tr_smem_layout(p.F, p.M, p.k, p.D, p.hsum, p.dmax, 0);
  if (L.total > smax) {
    set_error("trainer needs %d B of shared memory per example state (> %d)", L.total, smax);
    return DFFM_SIZING;
  }
  *smem_out = L.total;
  return DFFM_OK;
}

#ifdef DFFM_TR_TRACE
extern "C" int dffm_tr_trace_read(long long* host) {
  return (int)cudaMemcpyFromSymbol(host, g_tr_trace, sizeof(g_tr_trace));
}
#endif

extern "C" int64_t dffm_train_scratch_bytes(const dffm_model*, int32_t) { return 0; }

extern "C" int dffm_train_sequential(const dffm_model* model, const dffm_train_state* state,
                                     const int32_t* idx, const float* val, const uint8_t* labels,
                                     int32_t max_per_field, int64_t n, double* prob_out,
                                     void* scratch, uint64_t* status, void* stream) {
  (void)scratch;
  TrainParams p{};
  int smem = 0;
  // cluster split when layer 0 divides evenly (DFFM_TRAIN_CLUSTER=1 forces one CTA)
  int C = 1;
  {
    static int env = -1;
    if (env < 0) {
      const char* v = getenv("DFFM_TRAIN_CLUSTER");
      env = v ? atoi(v) : TR_CLUSTER;
    }
    if (env == TR_CLUSTER && model && model->n_layers >= 2 && model->dims[1] % TR_CLUSTER == 0)
      C = TR_CLUSTER;
  }
  int rc = tr_validate(model, max_per_field, C, p, &smem);
  if (rc == DFFM_SIZING && C > 1) {
    C = 1;
    rc = tr_validate(model, max_per_field, C, p, &smem);
  }
  if (rc) return rc;
  if (!state || !state->lr_acc || !state->ffm_acc) {
    set_error("null optimizer state");
    return DFFM_CONTRACT;
  }
  if (n < 0) { set_error("negative n"); return DFFM_CONTRACT; }
  if (n == 0) return DFFM_OK;
  if (!idx || !val || !labels || !prob_out || !status) {
    set_error("null buffer");
    return DFFM_CONTRACT;
  }
  for (int l = 0; l < p.n_layers; ++l) {
    if (!state->W_acc[l] || !state->b_acc[l]) { set_error("null MLP acc"); return DFFM_CONTRACT; }
    p.W_acc[l] = state->W_acc[l];
    p.b_acc[l] = state->b_acc[l];
  }
  p.lr_acc = state->lr_acc;
  p.ffm_acc = state->ffm_acc;
  p.lr_ffm = state->lr_ffm;
  p.lr_lr = state->lr_lr;
  p.lr_nn = state->lr_nn;
  p.power_t = state->power_t;
  p.sparse = state->sparse;
  p.idx = idx;
  p.val = val;
  p.labels = labels;
  p.prob_out = prob_out;
  p.status = status;
  p.n = n;
  int occ = 0;
  if (C == 1) {
    rc = kernel_occupancy((const void*)train_kernel<1>, TR_THREADS, smem, &occ);
    if (rc) return rc;
    note_launches(1), train_kernel<1><<<1, TR_THREADS, smem, (cudaStream_t)stream>>>(p);
  } else {
    // one thread-block cluster of C CTAs on C SMs (DSMEM exchange per example)
    rc = kernel_occupancy((const void*)train_kernel<TR_CLUSTER>, TR_THREADS, smem, &occ);
    if (rc) return rc;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(TR_CLUSTER);
    cfg.blockDim = dim3(TR_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = TR_CLUSTER;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    note_launches(1);
    DFFM_CUDA_TRY(cudaLaunchKernelEx(&cfg, train_kernel<TR_CLUSTER>, p), "launch(train cluster)");
  }
  DFFM_CUDA_TRY(cudaGetLastError(), "launch(train)");
  return DFFM_OK;
}

// K6: Hogwild-style trainer (T:242-336).  n_workers CTAs, each an
// independent predict-then-learn loop over examples w, w + W, w + 2W, ...
// against the SHARED store: no locks, no ordering between workers (a lost or
// overwritten update is allowed, T:1-11; individual f32 stores never tear).
// MLP state stays in global memory (L2-only accesses).  n_workers == 1 is the
// sequential kernel itself, so its result is identical to train_sequential.
extern "C" int dffm_train_hogwild(const dffm_model* model, const dffm_train_state* state,
                                  const int32_t* idx, const float* val, const uint8_t* labels,
                                  int32_t max_per_field, int64_t n, int32_t n_workers,
                                  double* prob_out, void* scratch, uint64_t* status,
                                  void* stream) {
  if (n_workers < 1) { set_error("n_workers must be >= 1"); return DFFM_CONTRACT; }
  if (n_workers == 1)
    return dffm_train_sequential(model, state, idx, val, labels, max_per_field, n, prob_out,
                                 scratch, status, stream);
  (void)scratch;
  TrainParams p{};
  int smem = 0;
  int rc = tr_validate(model, max_per_field, 1, p, &smem);
  if (rc) return rc;
  if (p.mlp_smem) {  // workers share the MLP in global memory
    p.mlp_smem = 0;
    smem = tr_smem_layout(p.F, p.M, p.k, p.D, p.hsum, p.dmax, 0).total;
  }
  p.hogwild = 1;
  if (!state || !state->lr_acc || !state->ffm_acc) {
    set_error("null optimizer state");
    return DFFM_CONTRACT;
  }
  if (n < 0) { set_error("negative n"); return DFFM_CONTRACT; }
  if (n == 0) return DFFM_OK;
  if (!idx || !val || !labels || !prob_out || !status) {
    set_error("null buffer");
    return DFFM_CONTRACT;
  }
  for (int l = 0; l < p.n_layers; ++l) {
    if (!state->W_acc[l] || !state->b_acc[l]) { set_error("null MLP acc"); return DFFM_CONTRACT; }
    p.W_acc[l] = state->W_acc[l];
    p.b_acc[l] = state->b_acc[l];
  }
  p.lr_acc = state->lr_acc;
  p.ffm_acc = state->ffm_acc;
  p.lr_ffm = state->lr_ffm;
  p.lr_lr = state->lr_lr;
  p.lr_nn = state->lr_nn;
  p.power_t = state->power_t;
  p.sparse = state->sparse;
  p.idx = idx;
  p.val = val;
  p.labels = labels;
  p.prob_out = prob_out;
  p.status = status;
  p.n = n;
  int occ = 0;
  rc = kernel_occupancy((const void*)train_kernel<1, TR_HW_THREADS>, TR_HW_THREADS, smem, &occ);
  if (rc) return rc;
  // concurrent workers only: a CTA that could not be resident would run later,
  // in series with the others
  const int64_t W = std::min<int64_t>({(int64_t)n_workers, (int64_t)occ * sm_count_current(), n});
  note_launches(1), train_kernel<1, TR_HW_THREADS><<<(unsigned)W, TR_HW_THREADS, smem,
                                                      (cudaStream_t)stream>>>(p);
  DFFM_CUDA_TRY(cudaGetLastError(), "launch(train hogwild)");
  return DFFM_OK;
}

extern "C" int dffm_hogwild_max_workers(const dffm_model* model, int32_t max_per_field) {
  TrainParams p{};
  int smem = 0;
  if (tr_validate(model, max_per_field, 1, p, &smem)) return 0;
  smem = tr_smem_layout(p.F, p.M, p.k, p.D, p.hsum, p.dmax, 0).total;
  int occ = 0;
  if (kernel_occupancy((const void*)train_kernel<1, TR_HW_THREADS>, TR_HW_THREADS, smem, &occ))
    return 0;
  return occ * sm_count_current();
}
