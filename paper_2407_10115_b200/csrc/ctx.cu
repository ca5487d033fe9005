#include <atomic>
// K3: context-cached candidate scorer (no reference code --
// the truth is model.forward on the merged context+candidate example).
//
// One CTA owns a request at a time (persistent over requests):
//   cache build (once per request, cost independent of the candidate count,
//   S:257): lr partial over the context features, the context latent
//   sums Sctx[x][g][:] = sum_{j in x} x_j * ffm[j][g][:] for every context field
//   x and every target field g, and the ctx x ctx pair values -- all in shared
//   memory, never written to HBM.
//   candidates, in tiles of TE: one warp per candidate gathers only the
//   candidate's own rows; cand x ctx pairs use <S[c][x] (gathered), Sctx[x][c]
//   (cached)>, cand x cand pairs are formed as in K1, ctx x ctx pairs are
//   copied from the cache.  MergeNorm and the MLP are not cached and
//   run through the same phase-B tile code as K1.
#include <algorithm>
#include <stdlib.h>
#include <string.h>
#include <mutex>
#include <unordered_map>

#include "forward_kernel.cuh"
#include "mlp_tc.cuh"

namespace dffm {

int fill_model_params(const dffm_model* m, FwdParams& p);
int pick_k_template(int k, int wdtype);

struct CtxParams {
  FwdParams f;
  const int32_t* cidx;
  const float* cval;
  const int32_t* didx;
  const float* dval;
  int Fc, Mc, Fd, Md;
  int64_t R;
  int C;
  int cblk;  // candidates per work unit (a multiple of TE)
  const unsigned char* cache_in;  // K3 v2: prebuilt context caches (dffm_ctx_build), or null
};

struct CtxSmem {
  FwdSmem b;
  int off_S, off_cpair, off_cpres, off_csidx, off_csval, off_lrp, total;
};

__host__ __device__ inline CtxSmem ctx_smem_layout(const CtxParams& q) {
  const FwdParams& p = q.f;
  CtxSmem s;
  // per-warp slot buffers sized for the candidate part (Fd x Md)
  s.b = fwd_smem_layout(p.F, 1, p.P, p.D, p.TE, p.XS, p.hmax);
  int o = s.b.off_sidx;
  s.b.off_sidx = o; o = align16(o + FWD_WARPS * q.Fd * q.Md * 4);
  s.b.off_sval = o; o = align16(o + FWD_WARPS * q.Fd * q.Md * 4);
  s.off_S = o; o = align16(o + q.Fc * p.F * p.k * 4);
  s.off_cpair = o; o = align16(o + p.P * 4);
  s.off_cpres = o; o = align16(o + q.Fc);
  s.off_csidx = o; o = align16(o + q.Fc * q.Mc * 4);
  s.off_csval = o; o = align16(o + q.Fc * q.Mc * 4);
  s.off_lrp = o; o = align16(o + 8);
  s.total = o;
  return s;
}

template <int K, int MU, typename T>
__global__ void __launch_bounds__(FWD_THREADS)
ctx_kernel(CtxParams q) {
  extern __shared__ __align__(128) unsigned char smem[];
  const FwdParams& p = q.f;
  const CtxSmem L = ctx_smem_layout(q);
  uint16_t* pairtab = (uint16_t*)(smem + L.b.off_pair);
  float* X = (float*)(smem + L.b.off_X);
  float* Ha = (float*)(smem + L.b.off_Ha);
  float* Hb = (float*)(smem + L.b.off_Hb);
  double* exd = (double*)(smem + L.b.off_exd);
  int* flag = (int*)(smem + L.b.off_flag);
  float* Sctx = (float*)(smem + L.off_S);
  float* cpair = (float*)(smem + L.off_cpair);
  unsigned char* cpres = smem + L.off_cpres;
  int* csidx = (int*)(smem + L.off_csidx);
  float* csval = (float*)(smem + L.off_csval);
  double* lrp = (double*)(smem + L.off_lrp);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int F = p.F, Fc = q.Fc, Mc = q.Mc, Fd = q.Fd, Md = q.Md;
  const int DM = Fd * Md;
  unsigned char* spres = smem + L.b.off_pres + warp * F;
  int* sidx = (int*)(smem + L.b.off_sidx) + warp * DM;
  float* sval = (float*)(smem + L.b.off_sval) + warp * DM;
  const int TE = p.TE, XS = p.XS, P = p.P, D = p.D;
  constexpr int KA = K ? K : 32;
  const int k = K ? K : p.k;
  const T* ffm = (const T*)p.ffm;

  build_pairtab(pairtab, F);
  const float bias = load_elem<T>((const T*)p.lr + p.n_buckets, p.dlr);

  // work unit = (request, block of cblk candidates): balances the tail and
  // keeps every SM busy when requests are few; the context cache is rebuilt
  // only when a unit starts a different request
  const int nub = (q.C + q.cblk - 1) / q.cblk;
  const int64_t nunits = q.R * nub;
  int64_t cached_r = -1;
  for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
    const int64_t r = u / nub;
    const int cbeg = (int)(u % nub) * q.cblk, cend = min(q.C, cbeg + q.cblk);
    __syncthreads();
    if (r != cached_r) {
      cached_r = r;
      // ---------------------------------------------- build_context_cache
      if (warp == 0) {
        int bad = 0;
        const double lrs = stage_slots<T>(p, q.cidx + r * Fc * Mc, q.cval + r * Fc * Mc, Fc * Mc,
                                          csidx, csval, lane, bad);
        const double tot = warp_sum(lrs);
        if (lane == 0) *lrp = tot;
        if (__any_sync(0xffffffffu, bad) && lane == 0)
          atomicMin((unsigned long long*)p.status,
                    (unsigned long long)status_key(p.status_base + r * q.C, DFFM_BLOCK_NONE,
                                                   DFFM_CONTRACT));
      }
      __syncthreads();
      for (int x = threadIdx.x; x < Fc; x += FWD_THREADS) {
        unsigned char pr = 0;
        for (int m = 0; m < Mc; ++m) pr |= (csidx[x * Mc + m] >= 0);
        cpres[x] = pr;
      }
      for (int t = threadIdx.x; t < Fc * F * k; t += FWD_THREADS) {
        const int x = t / (F * k), gk = t % (F * k);
        float acc = 0.f;
        for (int m = 0; m < Mc; ++m) {
          const int j = csidx[x * Mc + m];
          if (j >= 0) acc = fmaf(csval[x * Mc + m], load_elem<T>(ffm + (int64_t)j * F * k + gk, p.dffm), acc);
        }
        Sctx[t] = acc;
      }
      __syncthreads();
      for (int pp = threadIdx.x; pp < P; pp += FWD_THREADS) {
        const uint32_t pr = pairtab[pp];
        const int f1 = pr & 0xFF, f2 = pr >> 8;
        float pv = 0.f;
        if (f2 < Fc && (cpres[f1] & cpres[f2])) {
          const float* a = Sctx + (f1 * F + f2) * k;
          const float* b = Sctx + (f2 * F + f1) * k;
          for (int c = 0; c < k; ++c) pv = fmaf(a[c], b[c], pv);
        }
        cpair[pp] = pv;
      }
      __syncthreads();
    }  // cache for request r built
    const double lr_ctx = (double)bias + *lrp;

    // ---------------------------------------------- predict_batch
    for (int c0 = cbeg; c0 < cend; c0 += TE) {
      for (int el = warp; el < TE; el += FWD_WARPS) {
        const int cand = c0 + el;
        if (cand >= cend) { zero_column(X, exd, flag, el, TE, XS, D, lane); continue; }
        const int64_t e = r * q.C + cand;
        int bad = 0;
        const double lrs = stage_slots<T>(p, q.didx + e * DM, q.dval + e * DM, DM, sidx, sval,
                                          lane, bad);
        __syncwarp();
        for (int f = lane; f < Fd; f += 32) {
          unsigned char pr = 0;
          for (int m = 0; m < Md; ++m) pr |= (sidx[f * Md + m] >= 0);
          spres[Fc + f] = pr;
        }
        if (__any_sync(0xffffffffu, bad) && lane == 0)
          atomicMin((unsigned long long*)p.status,
                    (unsigned long long)status_key(p.status_base + e, DFFM_BLOCK_NONE,
                                                   DFFM_CONTRACT));
        const double lr_out = lr_ctx + warp_sum(lrs);
        __syncwarp();
        double s1 = 0.0;
        int pbad = 0;
        for (int pp = lane; pp < P; pp += 32) {
          const uint32_t pr = pairtab[pp];
          const int f1 = pr & 0xFF, f2 = pr >> 8;
          float pv;
          if (f2 < Fc) {
            pv = cpair[pp];  // ctx x ctx: cached
          } else {
            pv = 0.f;
            const int d2 = f2 - Fc;
            float a[KA], bb[KA];
#pragma unroll
            for (int c = 0; c < KA; ++c) { a[c] = 0.f; bb[c] = 0.f; }
            if (f1 < Fc) {  // ctx x cand: S[f1][f2] from the cache
              if (cpres[f1] & spres[f2]) {
                const float* sc = Sctx + (f1 * F + f2) * k;
#pragma unroll
                for (int c = 0; c < KA; ++c)
                  if (K || c < k) a[c] = sc[c];
                accum_slots<K, MU, T>(p, sidx + d2 * Md, sval + d2 * Md, Md, f1, bb);
#pragma unroll
                for (int c = 0; c < KA; ++c)
                  if (K || c < k) pv = fmaf(a[c], bb[c], pv);
              }
            } else if (spres[f1] & spres[f2]) {  // cand x cand
              const int d1 = f1 - Fc;
              accum_slots<K, MU, T>(p, sidx + d1 * Md, sval + d1 * Md, Md, f2, a);
              accum_slots<K, MU, T>(p, sidx + d2 * Md, sval + d2 * Md, Md, f1, bb);
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
      const int nvalid = (cend - c0) < TE ? (cend - c0) : TE;
      mlp_tile(p, X, Ha, Hb, exd, flag, r * q.C + c0, nvalid);
    }
  }
}

}  // namespace dffm

#include "ctx_ring.cuh"

namespace dffm {

using CtxRingKernel = void (*)(CtxParams, CrSmem);

template <typename T>
static CtxRingKernel select_ctx_ring(int K, int MD) {
#define DFFM_SEL(KK)                                        \
  if (K == KK) {                                            \
    if (MD == 1) return ctx_ring_kernel<KK, T, 1>;          \
    if (MD == 2) return ctx_ring_kernel<KK, T, 2>;          \
    if (MD == 3) return ctx_ring_kernel<KK, T, 3>;          \
    if (MD == 4) return ctx_ring_kernel<KK, T, 4>;          \
  }
  if constexpr (sizeof(T) == 4) { DFFM_SEL(4) }
  DFFM_SEL(8)
  DFFM_SEL(16)
#undef DFFM_SEL
  return nullptr;
}

using CtxKernel = void (*)(CtxParams);

template <typename T>
static CtxKernel select_ctx(int K, int MU) {
#define DFFM_SEL(KK)                                   \
  if (K == KK) {                                       \
    if (MU == 1) return ctx_kernel<KK, 1, T>;          \
    if (MU == 2) return ctx_kernel<KK, 2, T>;          \
    if (MU == 3) return ctx_kernel<KK, 3, T>;          \
    if (MU == 4) return ctx_kernel<KK, 4, T>;          \
    return ctx_kernel<KK, 0, T>;                       \
  }
  DFFM_SEL(4)
  DFFM_SEL(8)
  DFFM_SEL(16)
  DFFM_SEL(0)
#undef DFFM_SEL
  return nullptr;
}

static int launch_ctx(CtxKernel kern, const CtxParams& q, int smem, cudaStream_t s) {
  {  // DFFM_CTX_SMEM_KB: pad the per-CTA shared memory (fewer CTAs per SM, more L1 for W)
    static int pad = -1;
    if (pad < 0) {
      const char* v = getenv("DFFM_CTX_SMEM_KB");
      pad = v ? atoi(v) * 1024 : 0;
    }
    if (pad > smem && pad <= max_smem_optin_current()) smem = pad;
  }
  int occ = 0;
  int rc = kernel_occupancy((const void*)kern, FWD_THREADS, smem, &occ);
  if (rc) return rc;
  const int64_t nunits = q.R * ((q.C + q.cblk - 1) / q.cblk);
  const int64_t grid = std::min<int64_t>(nunits, (int64_t)sm_count_current() * occ);
  note_launches(1), kern<<<(unsigned)grid, FWD_THREADS, smem, s>>>(q);
  DFFM_CUDA_TRY(cudaGetLastError(), "launch(ctx)");
  return DFFM_OK;
}

// request context caches the library has built (host count; dffm_ctx_build_count)
static std::atomic<long long> g_ctx_builds{0};

// build_context_cache for R requests into per-request blobs (cache_bytes each):
// one CTA per request builds it in shared memory and copies it out
template <typename T>
__global__ void __launch_bounds__(256) ctx_build_kernel(CtxParams q, CrSmem L,
                                                        unsigned char* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int64_t r = blockIdx.x;
  cr_build_cache<T>(smem, q, L, r, r, threadIdx.x, 256);
  uint4* dst = (uint4*)(out + (size_t)r * L.cache_bytes);
  for (int v = threadIdx.x; v < L.cache_bytes / 16; v += 256) dst[v] = ((const uint4*)smem)[v];
}

// the K3 v2 context-cache layout (cache_bytes per request) for this model shape
static CrSmem ctx_cache_layout(const FwdParams& p, int wdtype, int Fc, int Mc) {
  const int esz = wdtype == DFFM_W_F32 ? 4 : 2;
  return cr_smem_layout(p.F, Fc, Mc, p.F - Fc, 1, p.k, esz, 1, max_smem_optin_current());
}

}  // namespace dffm

using namespace dffm;

static int ctx_score_impl(const dffm_model* model, const int32_t* ctx_idx, const float* ctx_val,
                          int32_t n_ctx_fields, int32_t ctx_m, const int32_t* cand_idx,
                          const float* cand_val, int32_t cand_m, int64_t n_requests,
                          int32_t n_cand, float* prob, uint64_t* status, void* stream,
                          const unsigned char* cache_in);

extern "C" int dffm_ctx_score(const dffm_model* model, const int32_t* ctx_idx,
                              const float* ctx_val, int32_t n_ctx_fields, int32_t ctx_m,
                              const int32_t* cand_idx, const float* cand_val, int32_t cand_m,
                              int64_t n_requests, int32_t n_cand, float* prob, uint64_t* status,
                              void* stream) {
  return ctx_score_impl(model, ctx_idx, ctx_val, n_ctx_fields, ctx_m, cand_idx, cand_val, cand_m,
                        n_requests, n_cand, prob, status, stream, nullptr);
}

extern "C" int64_t dffm_ctx_build_count(void) { return g_ctx_builds.load(); }

extern "C" int64_t dffm_ctx_cache_bytes(const dffm_model* model, int32_t n_ctx_fields,
                                        int32_t ctx_m) {
  FwdParams p{};
  if (fill_model_params(model, p)) return -1;
  if (n_ctx_fields < 1 || n_ctx_fields >= p.F || ctx_m < 1 || ctx_m > 64) {
    set_error("bad context shape");
    return -1;
  }
  return ctx_cache_layout(p, model->wdtype, n_ctx_fields, ctx_m).cache_bytes;
}

extern "C" int dffm_ctx_build(const dffm_model* model, const int32_t* ctx_idx,
                              const float* ctx_val, int32_t n_ctx_fields, int32_t ctx_m,
                              int64_t n_requests, void* cache_out, uint64_t* status,
                              void* stream) {
  CtxParams q{};
  int rc = fill_model_params(model, q.f);
  if (rc) return rc;
  FwdParams& p = q.f;
  if (n_ctx_fields < 1 || n_ctx_fields >= p.F || ctx_m < 1 || ctx_m > 64 || n_requests < 0 ||
      n_requests > (1ll << 31) - 1) {
    set_error("bad context shape");
    return DFFM_CONTRACT;
  }
  if (n_requests == 0) return DFFM_OK;
  if (!ctx_idx || !ctx_val || !cache_out || !status) { set_error("null buffer"); return DFFM_CONTRACT; }
  const int k = p.k, esz = model->wdtype == DFFM_W_F32 ? 4 : 2;
  if (!(k == 4 || k == 8 || k == 16) || (k * esz) % 16 || ((uintptr_t)p.ffm & 15) ||
      ((uintptr_t)cache_out & 15)) {
    set_error("context cache needs k in {4, 8, 16} with 16-byte rows");
    return DFFM_SIZING;
  }
  q.cidx = ctx_idx;
  q.cval = ctx_val;
  q.Fc = n_ctx_fields;
  q.Mc = ctx_m;
  q.Fd = p.F - n_ctx_fields;
  p.status = status;
  const CrSmem L = ctx_cache_layout(p, model->wdtype, n_ctx_fields, ctx_m);
  const void* kern = model->wdtype == DFFM_W_F32 ? (const void*)ctx_build_kernel<float>
                     : model->wdtype == DFFM_W_BF16 ? (const void*)ctx_build_kernel<__nv_bfloat16>
                                                    : (const void*)ctx_build_kernel<uint16_t>;
  int occ = 0;
  if ((rc = kernel_occupancy(kern, 256, L.cache_bytes, &occ))) return rc;
  const cudaStream_t s = (cudaStream_t)stream;
  switch (model->wdtype) {
    case DFFM_W_F32:
      note_launches(1), ctx_build_kernel<float><<<(unsigned)n_requests, 256, L.cache_bytes, s>>>(
                            q, L, (unsigned char*)cache_out);
      break;
    case DFFM_W_BF16:
      note_launches(1), ctx_build_kernel<__nv_bfloat16>
                            <<<(unsigned)n_requests, 256, L.cache_bytes, s>>>(q, L,
                                                                 (unsigned char*)cache_out);
      break;
    default:
      note_launches(1), ctx_build_kernel<uint16_t><<<(unsigned)n_requests, 256, L.cache_bytes, s>>>(
                            q, L, (unsigned char*)cache_out);
  }
  DFFM_CUDA_TRY(cudaGetLastError(), "launch(ctx_build)");
  g_ctx_builds += n_requests;
  return DFFM_OK;
}

extern "C" int dffm_ctx_score_cached(const dffm_model* model, const void* cache,
                                     const int32_t* ctx_idx, const float* ctx_val,
                                     int32_t n_ctx_fields, int32_t ctx_m, const int32_t* cand_idx,
                                     const float* cand_val, int32_t cand_m, int64_t n_requests,
                                     int32_t n_cand, float* prob, uint64_t* status, void* stream) {
  if (!cache || ((uintptr_t)cache & 15)) { set_error("null / misaligned cache"); return DFFM_CONTRACT; }
  return ctx_score_impl(model, ctx_idx, ctx_val, n_ctx_fields, ctx_m, cand_idx, cand_val, cand_m,
                        n_requests, n_cand, prob, status, stream,
                        (const unsigned char*)cache);
}

static int ctx_score_impl(const dffm_model* model, const int32_t* ctx_idx, const float* ctx_val,
                          int32_t n_ctx_fields, int32_t ctx_m, const int32_t* cand_idx,
                          const float* cand_val, int32_t cand_m, int64_t n_requests,
                          int32_t n_cand, float* prob, uint64_t* status, void* stream,
                          const unsigned char* cache_in) {
  CtxParams q{};
  int rc = fill_model_params(model, q.f);
  if (rc) return rc;
  FwdParams& p = q.f;
  if (n_ctx_fields < 0 || n_ctx_fields > p.F || ctx_m < 1 || cand_m < 1 || ctx_m > 64 ||
      cand_m > 64 || n_requests < 0 || n_cand < 0) {
    set_error("bad request shape");
    return DFFM_CONTRACT;
  }
  if (n_requests == 0 || n_cand == 0) return DFFM_OK;
  if (!prob || !status || (n_ctx_fields && (!ctx_idx || !ctx_val)) ||
      (n_ctx_fields < p.F && (!cand_idx || !cand_val))) {
    set_error("null buffer");
    return DFFM_CONTRACT;
  }
  q.cidx = ctx_idx;
  q.cval = ctx_val;
  q.didx = cand_idx;
  q.dval = cand_val;
  q.Fc = n_ctx_fields;
  q.Mc = ctx_m;
  q.Fd = p.F - n_ctx_fields;
  q.Md = cand_m;
  q.R = n_requests;
  q.C = n_cand;
  p.n = n_requests * (int64_t)n_cand;
  p.M = cand_m;
  p.prob = prob;
  p.logit = nullptr;
  p.status = status;
  const int smax = max_smem_optin_current();
  // DFFM_CTX_MLP=tc: MLP on the tensor cores (staged rows + mlp_tc, as K1 v6).
  // Off by default: at cfg4 (277-64-32-1) K3's candidate gather, not its MLP,
  // bounds the kernel, and staging costs more than it saves (measured
  // 93M vs 153M candidates/s).  Read per call.
  const char* ctx_mlp = getenv("DFFM_CTX_MLP");
  const bool use_tc = ctx_mlp && strcmp(ctx_mlp, "tc") == 0 && tc_eligible(p, smax);
  if (use_tc) p.hmax = 0;
  CtxSmem L;
  static int te_env = -1, cblk_env = -1;
  if (te_env < 0) {
    const char* v = getenv("DFFM_CTX_TE");
    te_env = v ? atoi(v) : 32;
    if (te_env < 2 || te_env > 32 || (te_env & 1)) te_env = 32;
    const char* c = getenv("DFFM_CTX_CBLK");
    cblk_env = c ? atoi(c) : 128;
  }
  int TE = te_env;
  for (;; TE >>= 1) {
    p.TE = TE;
    p.XS = TE + 2;
    L = ctx_smem_layout(q);
    if (L.total <= smax || TE <= 2) break;
  }
  if (L.total > smax) {
    set_error("context scorer needs %d B shared memory (> %d)", L.total, smax);
    return DFFM_SIZING;
  }
  q.cblk = std::max(p.TE, cblk_env / p.TE * p.TE);
  const int K = pick_k_template(p.k, model->wdtype);
  const int MU = cand_m <= 4 ? cand_m : 0;
  CtxKernel kern = nullptr;
  switch (model->wdtype) {
    case DFFM_W_F32: kern = select_ctx<float>(K, MU); break;
    case DFFM_W_BF16: kern = select_ctx<__nv_bfloat16>(K, MU); break;
    default: kern = select_ctx<uint16_t>(K, MU); break;
  }
  if (!kern) { set_error("no context kernel for k=%d", p.k); return DFFM_SIZING; }
  // K3 v2 (default when it takes the shape): candidates through the K1 v8 row
  // ring with the context cache in shared memory, MLP on the tensor cores
  {
    static int ring_env = -1;
    if (ring_env < 0) {
      const char* v = getenv("DFFM_CTX_RING");
      ring_env = v ? atoi(v) : 1;
    }
    const int esz = model->wdtype == DFFM_W_F32 ? 4 : 2;
    const int k = p.k;
    const int NX = CR_MAXX;  // candidates in flight (CR_MAXX / B bundle slots)
    const int64_t per_cta = ((n_requests + 147) / 148 + 1) * (int64_t)n_cand;
    bool ok = ring_env && ctx_mlp == nullptr && tc_eligible(p, smax) && n_ctx_fields >= 1 &&
              per_cta < (1ll << 30) &&
              q.Fd >= 1 && cand_m <= 4 && q.Fd * cand_m <= CR_MAXFM && n_cand >= NX &&
              (k == 4 || k == 8 || k == 16) && (k * esz) % 16 == 0 && ctx_idx && ctx_val &&
              !((uintptr_t)p.ffm & 15) && !((uintptr_t)p.lr & 3);
    CrSmem CL{};
    if (ok) {
      static int bun_env = -1;  // DFFM_CTX_BUNDLE=1: one candidate per slot (A/B knob)
      if (bun_env < 0) {
        const char* v = getenv("DFFM_CTX_BUNDLE");
        bun_env = v ? atoi(v) : 4;
      }
      int B = cr_bundle(q.Fd * cand_m, n_cand);
      while (B > bun_env && B > 1) B >>= 1;
      CL = cr_smem_layout(p.F, q.Fc, q.Mc, q.Fd, cand_m, k, esz, B, smax);
      ok = CL.R >= 2 * B * q.Fd * cand_m;
    }
    CtxRingKernel rk = nullptr;
    if (ok) {
      switch (model->wdtype) {
        case DFFM_W_F32: rk = select_ctx_ring<float>(k, cand_m); break;
        case DFFM_W_BF16: rk = select_ctx_ring<__nv_bfloat16>(k, cand_m); break;
        default: rk = select_ctx_ring<uint16_t>(k, cand_m); break;
      }
    }
    if (rk) {
      const cudaStream_t s = (cudaStream_t)stream;
      p.hmax = 0;
      const int64_t rows_all = n_requests * (int64_t)n_cand;
      const int64_t cap = std::max<int64_t>(n_cand, std::min<int64_t>(rows_all, 1 << 22));
      const int64_t req_per = std::max<int64_t>(1, cap / n_cand);
      const int64_t rows_max = std::min<int64_t>(req_per, n_requests) * n_cand;
      TcPlan plan;
      if ((rc = tc_plan(p, smax, (rows_max + TC_M - 1) / TC_M * TC_M, s, &plan))) return rc;
      int occ = 0;
      if ((rc = kernel_occupancy((const void*)rk, CR_THREADS, CL.total, &occ))) return rc;
      const int DM = q.Fd * q.Md;
      for (int64_t r0 = 0; r0 < n_requests; r0 += req_per) {
        const int64_t nr = std::min<int64_t>(req_per, n_requests - r0);
        CtxParams a = q;
        a.cidx = ctx_idx + r0 * q.Fc * q.Mc;
        a.cval = ctx_val + r0 * q.Fc * q.Mc;
        a.didx = cand_idx + r0 * n_cand * DM;
        a.dval = cand_val + r0 * n_cand * DM;
        a.R = nr;
        a.f.n = nr * n_cand;
        a.f.status_base = r0 * n_cand;
        a.f.prob = prob + r0 * n_cand;
        a.f.xout = plan.X;
        a.f.xplane = plan.xplane;
        a.f.rout = plan.resid;
        a.f.fout = plan.flags;
        a.f.Kp = plan.Kp;
        a.cache_in = cache_in ? cache_in + (size_t)r0 * CL.cache_bytes : nullptr;
        const int64_t grid = std::min<int64_t>(nr, (int64_t)sm_count_current());
        note_launches(1), rk<<<(unsigned)grid, CR_THREADS, CL.total, s>>>(a, CL);
        DFFM_CUDA_TRY(cudaGetLastError(), "launch(ctx_ring)");
        if ((rc = tc_mlp_slice(plan, nr * n_cand, r0 * n_cand, prob + r0 * n_cand, nullptr, s)))
          return rc;
        if (!cache_in) g_ctx_builds += nr;
      }
      return DFFM_OK;
    }
  }
  // other shapes build every request's context inside the kernel (a prebuilt
  // cache is not consumed there; the context rows give the same result)
  g_ctx_builds += n_requests;
  if (!use_tc) return launch_ctx(kern, q, L.total, (cudaStream_t)stream);
  // requests in slices: K3 stages each candidate's MergeNorm row, mlp_tc scores them
  const cudaStream_t s = (cudaStream_t)stream;
  const int64_t req_per = std::max<int64_t>(1, tc_default_slice_rows() / n_cand);
  const int64_t rows_max = std::min<int64_t>(req_per, n_requests) * n_cand;
  TcPlan plan;
  if ((rc = tc_plan(p, smax, (rows_max + TC_M - 1) / TC_M * TC_M, s, &plan))) return rc;
  const int DM = q.Fd * q.Md;
  for (int64_t r0 = 0; r0 < n_requests; r0 += req_per) {
    const int64_t nr = std::min<int64_t>(req_per, n_requests - r0);
    CtxParams a = q;
    a.cidx = ctx_idx ? ctx_idx + r0 * q.Fc * q.Mc : nullptr;
    a.cval = ctx_val ? ctx_val + r0 * q.Fc * q.Mc : nullptr;
    a.didx = cand_idx ? cand_idx + r0 * n_cand * DM : nullptr;
    a.dval = cand_val ? cand_val + r0 * n_cand * DM : nullptr;
    a.R = nr;
    a.f.n = nr * n_cand;
    a.f.status_base = r0 * n_cand;
    a.f.prob = prob + r0 * n_cand;
    a.f.xout = plan.X;
    a.f.xplane = plan.xplane;
    a.f.rout = plan.resid;
    a.f.fout = plan.flags;
    a.f.Kp = plan.Kp;
    if ((rc = launch_ctx(kern, a, L.total, s))) return rc;
    if ((rc = tc_mlp_slice(plan, nr * n_cand, r0 * n_cand, prob + r0 * n_cand, nullptr, s)))
      return rc;
  }
  return DFFM_OK;
}
