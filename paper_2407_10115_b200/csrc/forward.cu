// C ABI entry for K1 (dffm_forward): validation, tile sizing, dispatch.
#include <algorithm>
#include <mutex>
#include <unordered_map>

#include <stdlib.h>
#include <string.h>

#include "forward_kernel.cuh"
#include "forward_ws.cuh"
#include "mlp_tc.cuh"
#include "forward_rsw.cuh"

#include <cudaTypedefs.h>

namespace dffm {

template <typename T>
int launch_forward_t(const FwdParams& p, int K, int MU, int smem, cudaStream_t s);
template <typename T>
int launch_forward_ws_t(const FwdParams& p, int K, int MU, int smem, cudaStream_t s);
template <typename T>
int launch_forward_rsw_t(const FwdParams& p, const RswSmem& L, int K, cudaStream_t s);

// Kernel family: default (-1) = the dispatcher's choice per shape (row-ring
// gather + tcgen05 MLP where it applies, else the fused ws kernel, else v1);
// FAM_WS / FAM_V1 / FAM_TC force one for A/B measurements and tests
// (DFFM_FORWARD_KERNEL=ws|v1|tc, or dffm_set_forward_family on this thread).
// The choice is thread-local: concurrent host threads (one per GPU, or two
// streams on one GPU) never see each other's setting.
enum FwdFamily { FAM_WS = 1, FAM_V1 = 2, FAM_TC = 5 };
static thread_local int t_family = -2;  // -2: not read yet; -1: default
static int forward_family() {
  if (t_family == -2) {
    const char* v = getenv("DFFM_FORWARD_KERNEL");
    int f = -1;
    if (v && strcmp(v, "ws") == 0) f = FAM_WS;
    if (v && strcmp(v, "v1") == 0) f = FAM_V1;
    if (v && strcmp(v, "tc") == 0) f = FAM_TC;
    t_family = f;
  }
  return t_family;
}

// Optional per-thread launch trace (dffm_set_event_trace): after every kernel
// dffm_forward launches, an event is recorded on the launch stream and the
// kernel's role tagged (0 weight blocking, 1 gather, 2 MLP, 3 fused), so a
// caller can split a step's device time per kernel with CUDA events.
struct EventTrace {
  void** events = nullptr;
  int32_t* tags = nullptr;
  int32_t cap = 0;
  int32_t* count = nullptr;
};
static thread_local EventTrace t_trace;
static void trace_launch(int tag, cudaStream_t s) {
  EventTrace& t = t_trace;
  if (!t.events || !t.count || *t.count >= t.cap) return;
  cudaEventRecord((cudaEvent_t)t.events[*t.count], s);
  t.tags[*t.count] = tag;
  ++*t.count;
}

int pick_k_template(int k, int wdtype);

// ---- driver entry point for tensor-map encoding (no -lcuda)
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  if (!fn) {
    cudaDriverEntryPointQueryResult qr;
    void* ptr = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &qr) ==
            cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)ptr;
  }
  return fn;
}

static bool try_ws_forward(const dffm_model* m, FwdParams& p, int smax, cudaStream_t s, int* rc,
                           bool force = false) {
  const int fam = forward_family();
  if (!force && fam != FAM_WS && fam != -1) return false;
  for (int l = 1; l < p.n_layers; ++l)
    if (p.dims[l] % 4) return false;
  for (int TE = p.xout ? 8 : 32; TE >= 8; TE >>= 1) {  // staging: small tile, big ring
    p.TE = TE;
    p.XS = TE + 4;
    const WsSmem L = ws_smem_layout(p.F, p.M, p.P, p.D, p.TE, p.XS, p.hmax);
    if (L.total > smax) continue;
    const int K = pick_k_template(p.k, m->wdtype);
    const int MU = p.M <= 4 ? p.M : 0;
    switch (m->wdtype) {
      case DFFM_W_F32: *rc = launch_forward_ws_t<float>(p, K, MU, L.total, s); break;
      case DFFM_W_BF16: *rc = launch_forward_ws_t<__nv_bfloat16>(p, K, MU, L.total, s); break;
      default: *rc = launch_forward_ws_t<uint16_t>(p, K, MU, L.total, s); break;
    }
    return true;
  }
  return false;
}

// ---- K1 v6: gather (ws family, staging mode) + tcgen05 MLP (mlp_tc.cu), per slice.
// Chosen explicitly (family 5 / DFFM_FORWARD_KERNEL=tc) or, by default, when
// the MLP is heavy enough that CUDA-core FMAs would bound the fused kernel.
static bool tc_auto(const FwdParams& p) {
  int64_t macs = 0;
  for (int l = 0; l < p.n_layers; ++l) macs += (int64_t)p.dims[l] * p.dims[l + 1];
  return macs >= 65536;  // cfg5 (781-256-128-1): 232,832; cfg2 (277-64-32-1): 19,808
}

// device workspace per (device, stream), grow-only: staged rows of one slice
// and the blocked hi/lo MLP weights
static int tc_workspace(cudaStream_t s, size_t bytes, unsigned char** out) {
  struct Ws { void* ptr = nullptr; size_t bytes = 0; };
  static std::mutex mu;
  static std::unordered_map<uint64_t, Ws> ws;
  int dev = 0;
  DFFM_CUDA_TRY(cudaGetDevice(&dev), "cudaGetDevice");
  const uint64_t key = (uint64_t)(uintptr_t)s ^ ((uint64_t)dev << 56);
  std::lock_guard<std::mutex> lk(mu);
  Ws& w = ws[key];
  if (w.bytes < bytes) {
    if (w.ptr) DFFM_CUDA_TRY(cudaFree(w.ptr), "cudaFree(tc workspace)");
    w.ptr = nullptr;
    w.bytes = 0;
    DFFM_CUDA_TRY(cudaMalloc(&w.ptr, bytes), "cudaMalloc(tc workspace)");
    w.bytes = bytes;
  }
  *out = (unsigned char*)w.ptr;
  return DFFM_OK;
}

// staged rows as two fp16 planes [2][rows][Kp]: 4-D map {8 halfs, rows, Kp/8
// K cores, 2 planes}; one box {8, 128, 2, 2} lands as the A0 | A1 tiles of a
// 16-wide chunk in the K-major core-matrix layout of mlp_tc.cu
static int rows_tensor_map_x(const __half* X, int Kp, int64_t rows, int64_t xplane,
                             CUtensorMap* tm) {
  auto fn = encode_fn();
  if (!fn) { set_error("cuTensorMapEncodeTiled unavailable"); return DFFM_CUDA; }
  cuuint64_t dims[4] = {8, (cuuint64_t)rows, (cuuint64_t)(Kp / 8), 2};
  cuuint64_t strides[3] = {(cuuint64_t)Kp * 2, 16, (cuuint64_t)xplane * 2};
  cuuint32_t box[4] = {8, (cuuint32_t)TC_M, 2, 2};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, const_cast<__half*>(X), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled(staged rows) failed (%d)", (int)r);
    return DFFM_CUDA;
  }
  return DFFM_OK;
}

// shapes the K1 v8 row-ring gather takes
static bool rsw_shape_ok(const dffm_model* m, const FwdParams& p) {
  if (p.M < 1 || p.M > 4 || p.P < 1 || p.F * p.M > RSW_MAXFM || p.F > 255) return false;
  const int esz = m->wdtype == DFFM_W_F32 ? 4 : 2;
  const int k = p.k;
  if (!(k == 4 || k == 8 || k == 16) || (k * esz) % 16 != 0) return false;
  return !(((uintptr_t)p.ffm & 15) || ((uintptr_t)p.lr & 3));
}

// K1 v8 staging gather: warp-specialised circular row ring (M <= 4)
static bool try_rsw_forward(const dffm_model* m, FwdParams& p, int smax, cudaStream_t s,
                            int* rc) {
  if (!p.xout || !rsw_shape_ok(m, p)) return false;
  const int esz = m->wdtype == DFFM_W_F32 ? 4 : 2;
  const int k = p.k;
  static int nx_env = -1;
  if (nx_env < 0) {
    const char* v = getenv("DFFM_RSW_NX");
    nx_env = v ? std::min(RSW_MAXX, std::max(2, atoi(v))) : 8;
  }

  const int row_bytes = p.F * k * esz;
  int npw = RSW_NPW, nmw = RSW_NMW;
  {
    static int roles_env = -1;  // DFFM_RSW_ROLES=0: the fixed 16 / 6 layout (A/B knob)
    if (roles_env < 0) {
      const char* v = getenv("DFFM_RSW_ROLES");
      roles_env = v ? atoi(v) : 1;
    }
    if (roles_env) rsw_role_layout((p.P + 31) / 32, &npw, &nmw);
  }
  for (int nx = std::max(nx_env, nmw); nx >= std::max(2, nmw); --nx) {
    RswSmem L = rsw_smem_layout(p.F, p.M, p.P, row_bytes, nx, smax);
    if (L.R < p.F * p.M || L.R < 2 * p.F) continue;
    L.npw = npw;
    L.nmw = nmw;
    switch (m->wdtype) {
      case DFFM_W_F32: *rc = launch_forward_rsw_t<float>(p, L, k, s); break;
      case DFFM_W_BF16: *rc = launch_forward_rsw_t<__nv_bfloat16>(p, L, k, s); break;
      default: *rc = launch_forward_rsw_t<uint16_t>(p, L, k, s); break;
    }
    return true;
  }
  return false;
}

bool tc_eligible(const FwdParams& p, int smax) {
  const int NH = p.n_layers - 1;
  if (NH < 1 || NH > TC_MAXH) return false;
  int nmax = 0;
  for (int l = 1; l <= NH; ++l) {
    const int w = p.dims[l];
    if (w < TC_WIDTH_MULT || w > 256 || w % TC_WIDTH_MULT) return false;  // 16-col blocks per part
    nmax = std::max(nmax, w);
  }
  // one TMEM accumulation group per layer: layer 0's K (D padded to 16) <= 16 TC_GROUP
  if (((p.D + 15) & ~15) > 16 * TC_GROUP) return false;
  return tc_smem_bytes(2, tc_stage_bytes(nmax)) <= smax;
}

int64_t tc_default_slice_rows() {
  static int64_t slice_env = -1;
  if (slice_env < 0) {
    const char* v = getenv("DFFM_TC_SLICE");
    slice_env = v ? atoll(v) : (int64_t)32 * 148 * TC_M;  // 606,208 rows: fewer pipeline fills (cfg2 +4%)
    slice_env = std::max<int64_t>(TC_M, slice_env / TC_M * TC_M);
  }
  return slice_env;
}

int tc_plan(const FwdParams& p, int smax, int64_t slice_rows, cudaStream_t s, TcPlan* plan) {
  MlpTcParams& q = plan->q;
  q = MlpTcParams{};
  const int NH = p.n_layers - 1;
  int nmax = 0;
  for (int l = 1; l <= NH; ++l) nmax = std::max(nmax, p.dims[l]);
  q.n_hidden = NH;
  const int Kp = (p.D + 15) & ~15;
  size_t whalfs = 0;
  for (int l = 0; l < NH; ++l) {
    q.kin[l] = l == 0 ? Kp : p.dims[l];
    q.nout[l] = p.dims[l + 1];
    whalfs += (size_t)q.kin[l] * q.nout[l] * 2;
  }
  q.stage_bytes = tc_stage_bytes(nmax);
  static int stages_env = -1;
  if (stages_env < 0) {
    const char* v = getenv("DFFM_TC_STAGES");
    stages_env = v ? std::max(2, std::min(TC_MAX_STAGES, atoi(v))) : TC_MAX_STAGES;
  }
  q.stages = stages_env;
  while (q.stages > 2 && tc_smem_bytes(q.stages, q.stage_bytes) > smax) --q.stages;
  int cols = 32;
  while (cols < 2 * nmax) cols <<= 1;
  q.tmem_cols = cols;
  plan->smem = tc_smem_bytes(q.stages, q.stage_bytes);
  plan->Kp = Kp;
  plan->slice_rows = slice_rows;
  auto a256 = [](size_t b) { return (b + 255) & ~(size_t)255; };
  const size_t b_e = 256, b_w = a256(whalfs * 2), b_x = a256((size_t)slice_rows * Kp * 4),  // 2 fp16 planes
               b_r = a256((size_t)slice_rows * 8), b_f = a256((size_t)slice_rows * 4);
  unsigned char* ws = nullptr;
  int rc = tc_workspace(s, b_e + b_w + b_x + b_r + b_f, &ws);
  if (rc) return rc;
  int* wexp = (int*)ws;            // [TC_MAXH] per-layer weight scale exponents
  int* wmax = wexp + TC_MAXH;      // [TC_MAXH] max |w| scratch
  __half* wblk = (__half*)(ws + b_e);
  plan->X = (__half*)(ws + b_e + b_w);
  plan->xplane = (int64_t)slice_rows * Kp;
  plan->resid = (double*)(ws + b_e + b_w + b_x);
  plan->flags = (int*)(ws + b_e + b_w + b_x + b_r);
  __half* wl = wblk;
  for (int l = 0; l < NH; ++l) {
    const int kreal = l == 0 ? p.D : p.dims[l];
    if ((rc = launch_tc_prep_weights(p.W[l], kreal, q.nout[l], q.kin[l], wl, wmax + l, wexp + l,
                                     s)))
      return rc;
    q.wblk[l] = wl;
    q.bias[l] = p.b[l];
    wl += (size_t)q.kin[l] * q.nout[l] * 2;
  }
  q.wexp = wexp;
  q.w_out = p.W[NH];
  q.b_out = p.b[NH];
  q.resid = plan->resid;
  q.flags = plan->flags;
  q.status = p.status;
  return DFFM_OK;
}

int tc_mlp_slice(TcPlan& plan, int64_t rows, int64_t status_base, float* prob, float* logit,
                 cudaStream_t s) {
  CUtensorMap tm;
  int rc = rows_tensor_map_x(plan.X, plan.Kp, rows, plan.xplane, &tm);
  if (rc) return rc;
  plan.q.rows = rows;
  plan.q.status_base = status_base;
  plan.q.prob = prob;
  plan.q.logit = logit;
  return launch_mlp_tc(tm, plan.q, plan.smem, s);
}

static bool try_tc_forward(const dffm_model* m, FwdParams& p, int smax, cudaStream_t s,
                           int* rc) {
  const int fam = forward_family();
  // default: the row-ring gather + tensor-core MLP wherever the ring takes the
  // shape (cfg2: 135 vs 111 M preds/s for the fused ws kernel), or whenever
  // the MLP is too heavy for CUDA cores (cfg5)
  if (fam != FAM_TC && !(fam == -1 && (tc_auto(p) || rsw_shape_ok(m, p)))) return false;
  if (!tc_eligible(p, smax)) return false;
  FwdParams pg = p;
  pg.hmax = 0;  // staging mode: the gather kernels keep no hidden-layer buffers
  {
    const WsSmem L = ws_smem_layout(p.F, p.M, p.P, p.D, 8, 12, 0);
    if (L.total > smax) return false;  // the ws gather (the fallback) must fit
  }
  static int gather_env = -2;
  if (gather_env == -2) {
    const char* v = getenv("DFFM_TC_GATHER");
    gather_env = (v && strcmp(v, "ws") == 0) ? FAM_WS : -1;  // default: row ring when it applies
  }
  const int64_t sl = std::min<int64_t>(tc_default_slice_rows(), (p.n + TC_M - 1) / TC_M * TC_M);
  TcPlan plan;
  if ((*rc = tc_plan(p, smax, sl, s, &plan))) return true;
  trace_launch(0, s);
  const int64_t FM = (int64_t)p.F * p.M;
  for (int64_t s0 = 0; s0 < p.n; s0 += sl) {
    const int64_t ns = std::min<int64_t>(sl, p.n - s0);
    FwdParams a = pg;
    a.idx = p.idx + s0 * FM;
    a.val = p.val + s0 * FM;
    a.n = ns;
    a.status_base = p.status_base + s0;
    a.prob = p.prob + s0;
    a.logit = nullptr;
    a.xout = plan.X;
    a.xplane = plan.xplane;
    a.rout = plan.resid;
    a.fout = plan.flags;
    a.Kp = plan.Kp;
    bool launched = false;
    if (gather_env < 0) launched = try_rsw_forward(m, a, smax, s, rc);
    if (!launched) launched = try_ws_forward(m, a, smax, s, rc, true);
    if (!launched) { set_error("no gather kernel fits the staging slice"); *rc = DFFM_SIZING; }
    if (*rc) return true;
    trace_launch(1, s);
    if ((*rc = tc_mlp_slice(plan, ns, p.status_base + s0, p.prob + s0,
                            p.logit ? p.logit + s0 : nullptr, s)))
      return true;
    trace_launch(2, s);
  }
  *rc = DFFM_OK;
  return true;
}

// shared with ctx.cu: fills FwdParams' model part, validates
int fill_model_params(const dffm_model* m, FwdParams& p) {
  if (!m) { set_error("null model"); return DFFM_CONTRACT; }
  if (m->n_fields < 1 || m->n_fields > 255) {
    set_error("n_fields=%d outside [1, 255]", m->n_fields);
    return DFFM_SIZING;
  }
  if (m->k < 1 || m->k > 32) {
    set_error("k=%d unsupported (1..32)", m->k);
    return DFFM_SIZING;
  }
  if (m->hash_bits < 1 || m->hash_bits > 29) {
    set_error("hash_bits=%d outside [1, 29]", m->hash_bits);
    return DFFM_CONTRACT;
  }
  if (m->n_layers < 0 || m->n_layers > DFFM_MAX_LAYERS || m->n_layers == 1) {
    set_error("n_layers=%d invalid", m->n_layers);
    return DFFM_CONTRACT;
  }
  if (m->wdtype < 0 || m->wdtype > 2) { set_error("bad wdtype"); return DFFM_CONTRACT; }
  if (!m->lr || !m->ffm) { set_error("null table"); return DFFM_CONTRACT; }
  p.F = m->n_fields;
  p.k = m->k;
  p.P = p.F * (p.F - 1) / 2;
  p.D = 1 + p.P;
  p.n_buckets = (int64_t)1 << m->hash_bits;
  p.n_layers = m->n_layers;
  p.hmax = 0;
  for (int l = 0; l <= DFFM_MAX_LAYERS; ++l) p.dims[l] = m->dims[l];
  if (p.n_layers) {
    if (m->dims[0] != p.D || m->dims[p.n_layers] != 1) {
      set_error("MLP dims do not match 1+F(F-1)/2 -> ... -> 1");
      return DFFM_CONTRACT;
    }
    for (int l = 0; l < p.n_layers; ++l) {
      if (!m->W[l] || !m->b[l]) { set_error("null MLP layer %d", l); return DFFM_CONTRACT; }
      if (((uintptr_t)m->W[l] & 15) || ((uintptr_t)m->b[l] & 15)) {
        set_error("MLP layer %d not 16-byte aligned", l);
        return DFFM_CONTRACT;
      }
      p.W[l] = m->W[l];
      p.b[l] = m->b[l];
      if (l + 1 < p.n_layers) p.hmax = std::max(p.hmax, m->dims[l + 1]);
    }
  }
  p.lr = m->lr;
  p.ffm = m->ffm;
  p.dlr = Deq{m->q_lr_min, m->q_lr_bucket};
  p.dffm = Deq{m->q_ffm_min, m->q_ffm_bucket};
  return DFFM_OK;
}

int fwd_dispatch(int wdtype, const FwdParams& p, int K, int MU, int smem, cudaStream_t s) {
  switch (wdtype) {
    case DFFM_W_F32: return launch_forward_t<float>(p, K, MU, smem, s);
    case DFFM_W_BF16: return launch_forward_t<__nv_bfloat16>(p, K, MU, smem, s);
    default: return launch_forward_t<uint16_t>(p, K, MU, smem, s);
  }
}

int pick_k_template(int k, int wdtype) {
  const int esz = wdtype == DFFM_W_F32 ? 4 : 2;
  if ((k == 4 || k == 8 || k == 16) && (k * esz) % 8 == 0) return k;
  return 0;
}

}  // namespace dffm

using namespace dffm;

extern "C" int dffm_set_forward_family(int32_t family) {
  if (family != -1 && family != FAM_WS && family != FAM_V1 && family != FAM_TC) {
    set_error("bad forward family %d (-1 default, 1 ws, 2 v1, 5 tc)", family);
    return DFFM_CONTRACT;
  }
  t_family = family;  // this host thread only
  return DFFM_OK;
}

extern "C" int dffm_set_event_trace(void** events, int32_t* tags, int32_t capacity,
                                    int32_t* count) {
  if (events && (!tags || !count || capacity < 0)) {
    set_error("event trace needs tags, count and capacity >= 0");
    return DFFM_CONTRACT;
  }
  t_trace = EventTrace{events, tags, events ? capacity : 0, count};
  return DFFM_OK;
}

extern "C" int dffm_forward(const dffm_model* model, const int32_t* idx, const float* val,
                            int32_t max_per_field, int64_t n, float* prob, float* logit_opt,
                            int64_t status_base, uint64_t* status, void* stream) {
  FwdParams p{};
  int rc = fill_model_params(model, p);
  if (rc) return rc;
  if (n < 0 || max_per_field < 1 || max_per_field > 64) {
    set_error("bad batch shape n=%lld M=%d", (long long)n, max_per_field);
    return DFFM_CONTRACT;
  }
  if (n == 0) return DFFM_OK;
  if (!idx || !val || !prob || !status) { set_error("null buffer"); return DFFM_CONTRACT; }
  p.idx = idx;
  p.val = val;
  p.prob = prob;
  p.logit = logit_opt;
  p.status = status;
  p.n = n;
  p.status_base = status_base;
  p.M = max_per_field;
  const int smax = max_smem_optin_current();
  if (try_tc_forward(model, p, smax, (cudaStream_t)stream, &rc)) return rc;
  if (try_ws_forward(model, p, smax, (cudaStream_t)stream, &rc)) {
    if (!rc) trace_launch(3, (cudaStream_t)stream);
    return rc;
  }
  // Tile width: 16 keeps the per-block footprint small enough that the MLP
  // weights stay L1-resident next to three blocks per SM (DFFM_FWD_TE overrides).
  static int te_env = -1;
  if (te_env < 0) {
    const char* v = getenv("DFFM_FWD_TE");
    te_env = v ? atoi(v) : 16;
    if (te_env < 2 || te_env > 64 || (te_env & 1)) te_env = 16;
  }
  int TE = te_env;
  FwdSmem L;
  for (;; TE >>= 1) {
    p.TE = TE;
    p.XS = TE + 2;
    L = fwd_smem_layout(p.F, p.M, p.P, p.D, p.TE, p.XS, p.hmax);
    if (L.total <= smax || TE <= 2) break;
  }
  if (L.total > smax) {
    set_error("forward tile needs %d B shared memory (> %d)", L.total, smax);
    return DFFM_SIZING;
  }
  const int K = pick_k_template(p.k, model->wdtype);
  const int MU = p.M <= 4 ? p.M : 0;
  rc = fwd_dispatch(model->wdtype, p, K, MU, L.total, (cudaStream_t)stream);
  if (!rc) trace_launch(3, (cudaStream_t)stream);
  return rc;
}
