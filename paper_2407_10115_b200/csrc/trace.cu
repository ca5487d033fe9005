// K11: single-example forward trace and dense loss gradient (f64), the
// per-example API of the reference that keeps every intermediate:
//   dffm_forward_trace   <- M:321-397 forward() -> ForwardState (M:275-290)
//   dffm_loss_gradients  <- M:575-634 loss_gradients()
// One CTA walks the reference's stages in order; every sum is f64 with the
// f32 (or dequantised bf16 / u16) table values promoted exactly as numpy
// promotes them.  Used by model.forward / model.loss_gradients for one
// example at a time -- the batched paths (K1, K2) never need the trace.
#include "common.cuh"

namespace dffm {

constexpr int TR_THREADS = 256;

template <typename T>
__device__ __forceinline__ double tab(const void* base, int64_t i, const Deq& d) {
  return (double)load_elem<T>((const T*)base + i, d);
}

struct TrLayout {  // offsets (in doubles) into the trace buffer
  int64_t S, pairs, v, merged, acts, total;
};

__host__ __device__ inline TrLayout tr_layout(int F, int k, int n_layers, const int32_t* dims) {
  TrLayout L;
  const int64_t P = (int64_t)F * (F - 1) / 2, D = 1 + P;
  L.S = DFFM_TRACE_HEAD;
  L.pairs = L.S + (int64_t)F * F * k;
  L.v = L.pairs + P;
  L.merged = L.v + D;
  L.acts = L.merged + D;
  int64_t h = 0;
  for (int l = 1; l < n_layers; ++l) h += 2 * dims[l];
  L.total = L.acts + h;
  return L;
}

__device__ void block_sum2(double a, double b, double* red, double& ra, double& rb) {
  a = warp_sum(a);
  b = warp_sum(b);
  const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
  __syncthreads();
  if (ln == 0) { red[w] = a; red[32 + w] = b; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double x = 0, y = 0;
    for (int i = 0; i < TR_THREADS / 32; ++i) { x += red[i]; y += red[32 + i]; }
    red[64] = x;
    red[65] = y;
  }
  __syncthreads();
  ra = red[64];
  rb = red[65];
}

template <typename T>
__global__ void __launch_bounds__(TR_THREADS) trace_kernel(dffm_model m, const int32_t* idx,
                                                           const float* val, int M, double* out) {
  __shared__ double red[66];
  __shared__ int present[256];
  const int F = m.n_fields, k = m.k, P = F * (F - 1) / 2, D = 1 + P;
  const int64_t nf = (int64_t)1 << m.hash_bits;
  const Deq dl{m.q_lr_min, m.q_lr_bucket}, df{m.q_ffm_min, m.q_ffm_bucket};
  const TrLayout L = tr_layout(F, k, m.n_layers, m.dims);
  double* S = out + L.S;
  for (int f = threadIdx.x; f < F; f += TR_THREADS) {
    int pr = 0;
    for (int s = 0; s < M; ++s) pr |= idx[f * M + s] >= 0;
    present[f] = pr;
  }
  __syncthreads();
  // lr_out = bias + sum_f dot(lr[idx_f], x_f)  (M:327, M:338), fields in order
  if (threadIdx.x == 0) {
    double lr_out = tab<T>(m.lr, nf, dl);
    for (int f = 0; f < F; ++f) {
      double dot = 0.0;
      for (int s = 0; s < M; ++s) {
        const int j = idx[f * M + s];
        if (j >= 0) dot += tab<T>(m.lr, j, dl) * (double)val[f * M + s];
      }
      lr_out += dot;
    }
    out[0] = lr_out;
  }
  // S[f][g][:] = sum_{j in f} x_j ffm[j][g][:]  (M:328, M:339)
  for (int e = threadIdx.x; e < F * F * k; e += TR_THREADS) {
    const int f = e / (F * k), r = e - f * F * k;  // r = g*k + kk
    double acc = 0.0;
    for (int s = 0; s < M; ++s) {
      const int j = idx[f * M + s];
      if (j >= 0) acc += (double)val[f * M + s] * tab<T>(m.ffm, (int64_t)j * F * k + r, df);
    }
    S[e] = acc;
  }
  __syncthreads();
  // pairs (M:344-353): active iff both fields present; strict upper triangle order
  double* pairs = out + L.pairs;
  double* v = out + L.v;
  double loc = 0.0;
  for (int p = threadIdx.x; p < P; p += TR_THREADS) {
    int f1 = 0, rem = p;
    while (rem >= F - 1 - f1) { rem -= F - 1 - f1; ++f1; }
    const int f2 = f1 + 1 + rem;
    double d = 0.0;
    if (present[f1] && present[f2]) {
      const double* a = S + ((int64_t)f1 * F + f2) * k;
      const double* b = S + ((int64_t)f2 * F + f1) * k;
      for (int t = 0; t < k; ++t) d += a[t] * b[t];
    }
    pairs[p] = d;
    v[1 + p] = d;
  }
  __syncthreads();
  if (threadIdx.x == 0) v[0] = out[0];
  __syncthreads();
  // MergeNorm (M:355-360): population mean / std over D values
  for (int c = threadIdx.x; c < D; c += TR_THREADS) loc += v[c];
  double sum, dummy;
  block_sum2(loc, 0.0, red, sum, dummy);
  const double mu = sum / D;
  loc = 0.0;
  for (int c = threadIdx.x; c < D; c += TR_THREADS) loc += (v[c] - mu) * (v[c] - mu);
  double ss;
  block_sum2(loc, 0.0, red, ss, dummy);
  const double sd = sqrt(ss / D);
  double* merged = out + L.merged;
  for (int c = threadIdx.x; c < D; c += TR_THREADS) merged[c] = (v[c] - mu) / (sd + 1e-6);
  double psum_loc = 0.0;
  for (int p = threadIdx.x; p < P; p += TR_THREADS) psum_loc += pairs[p];
  double psum;
  block_sum2(psum_loc, 0.0, red, psum, dummy);
  // MLP (M:362-373): z = a @ W + b, a = max(z, 0) (NaN kept)
  double nn = 0.0;
  if (m.n_layers) {
    const double* a = merged;
    double* acts = out + L.acts;
    for (int l = 0; l + 1 < m.n_layers; ++l) {
      const int in = m.dims[l], o = m.dims[l + 1];
      const float* W = m.W[l];
      double* pre = acts;
      double* act = acts + o;
      for (int c = threadIdx.x; c < o; c += TR_THREADS) {
        double z = 0.0;
        for (int i = 0; i < in; ++i) z += a[i] * (double)W[(int64_t)i * o + c];
        z += (double)m.b[l][c];
        pre[c] = z;
        act[c] = z != z ? z : fmax(z, 0.0);
      }
      __syncthreads();
      a = act;
      acts += 2 * o;
    }
    const int in = m.dims[m.n_layers - 1];
    const float* w = m.W[m.n_layers - 1];
    loc = 0.0;
    for (int i = threadIdx.x; i < in; i += TR_THREADS) loc += a[i] * (double)w[i];
    block_sum2(loc, 0.0, red, nn, dummy);
    nn += (double)m.b[m.n_layers - 1][0];
  }
  if (threadIdx.x == 0) {
    out[1] = nn + out[0] + psum;  // logit, M:377
    out[2] = mu;
    out[3] = sd;
    out[4] = nn;
    out[5] = psum;
  }
}

// sigma without the probability clamp (M:293-297)
__device__ inline double sigmoid_raw(double logit) {
  if (logit >= 0.0) return 1.0 / (1.0 + exp(-fmin(logit, 60.0)));
  const double e = exp(fmax(logit, -60.0));
  return e / (1.0 + e);
}

// Dense f64 gradient over the weights' flat layout (lr | ffm | per layer W, b):
// M:575-634, from a trace buffer of the same example.
__global__ void __launch_bounds__(TR_THREADS) grad_kernel(dffm_model m, const int32_t* idx,
                                                          const float* val, int M,
                                                          const double* tr, int label,
                                                          double* grad, double* scratch) {
  __shared__ double red[66];
  const int F = m.n_fields, k = m.k, P = F * (F - 1) / 2, D = 1 + P;
  const int64_t nf = (int64_t)1 << m.hash_bits;
  const TrLayout L = tr_layout(F, k, m.n_layers, m.dims);
  const int64_t lr_size = nf + 1, ffm_off = lr_size, nn_off = ffm_off + nf * F * k;
  const double g = sigmoid_raw(tr[1]) - (double)label;
  // scratch: d_pairs-with-lr dv [D], two ping-pong d vectors of the widest layer
  double* dv = scratch;
  int wmax = 1;
  for (int l = 0; l <= m.n_layers; ++l) wmax = max(wmax, (int)m.dims[l]);
  double* dA = scratch + D;
  double* dB = dA + wmax;
  if (m.n_layers) {
    int64_t loff[DFFM_MAX_LAYERS];
    int64_t off = nn_off;
    for (int l = 0; l < m.n_layers; ++l) {
      loff[l] = off;
      off += (int64_t)m.dims[l] * m.dims[l + 1] + m.dims[l + 1];
    }
    // layer inputs: merged, then each hidden layer's activations
    const double* acts = tr + L.acts;
    if (threadIdx.x == 0) dA[0] = g;
    __syncthreads();
    double* d = dA;
    double* dn = dB;
    for (int i = m.n_layers - 1; i >= 0; --i) {
      const int in = m.dims[i], o = m.dims[i + 1];
      const double* a_in = tr + L.merged;
      int64_t hoff = 0;
      for (int l = 0; l < i; ++l) hoff += 2 * m.dims[l + 1];
      if (i > 0) a_in = acts + hoff - m.dims[i];  // act of layer i-1
      const float* W = m.W[i];
      for (int64_t e = threadIdx.x; e < (int64_t)in * o; e += TR_THREADS) {
        const int r = (int)(e / o), c = (int)(e - (int64_t)r * o);
        grad[loff[i] + e] = a_in[r] * d[c];  // outer(a_in, d)
      }
      for (int c = threadIdx.x; c < o; c += TR_THREADS) grad[loff[i] + (int64_t)in * o + c] = d[c];
      // da_in = W @ d, then the ReLU mask of the layer below (M:479) or MergeNorm
      for (int r = threadIdx.x; r < in; r += TR_THREADS) {
        double s = 0.0;
        for (int c = 0; c < o; ++c) s += (double)W[(int64_t)r * o + c] * d[c];
        if (i > 0) {  // da_in * (pre > 0): a non-finite da_in times 0 stays NaN, as in numpy
          const double pre = acts[hoff - 2 * m.dims[i] + r];
          s = s * (pre > 0.0 ? 1.0 : 0.0);
        }
        dn[r] = s;
      }
      __syncthreads();
      double* t = d; d = dn; dn = t;
    }
    // _merge_backward (M:413-421) on d = d_merged [D]
    const double mu = tr[2], sd = tr[3], denom = sd + 1e-6;
    const double* vv = tr + L.v;
    double l1 = 0.0, l2 = 0.0;
    for (int c = threadIdx.x; c < D; c += TR_THREADS) {
      l1 += d[c];
      l2 += d[c] * (vv[c] - mu);
    }
    double sdm, dotc;
    block_sum2(l1, l2, red, sdm, dotc);
    const double mean = sdm / D;
    for (int c = threadIdx.x; c < D; c += TR_THREADS) {
      double x = (d[c] - mean) / denom;
      if (sd > 0.0) x = x - (vv[c] - mu) * (dotc / (D * sd * denom * denom));
      dv[c] = g + x;  // d_lr = g + dv[0], d_pairs = g + dv[1:]
    }
  } else {
    for (int c = threadIdx.x; c < D; c += TR_THREADS) dv[c] = g;
  }
  __syncthreads();
  // FFM rows: out[j][gg][:] += x_j * dp[f][gg] * S[gg][f][:], fields in order
  const double* S = tr + L.S;
  for (int r = threadIdx.x; r < F * k; r += TR_THREADS) {
    const int gg = r / k, kk = r - gg * k;
    for (int f = 0; f < F; ++f) {
      double dp = 0.0;
      if (gg != f) {
        const int a = min(f, gg), b = max(f, gg);
        const int p = a * (2 * F - a - 1) / 2 + (b - a - 1);
        dp = dv[1 + p];
      }
      const double t = dp * S[((int64_t)gg * F + f) * k + kk];
      for (int s = 0; s < M; ++s) {
        const int j = idx[f * M + s];
        if (j >= 0) grad[ffm_off + (int64_t)j * F * k + r] += (double)val[f * M + s] * t;
      }
    }
  }
  // LR weights and bias (np.add.at in field order, then the bias)
  if (threadIdx.x == 0) {
    const double d_lr = dv[0];
    for (int f = 0; f < F; ++f)
      for (int s = 0; s < M; ++s) {
        const int j = idx[f * M + s];
        if (j >= 0) grad[j] += d_lr * (double)val[f * M + s];
      }
    grad[nf] += d_lr;
  }
}

static int check_model(const dffm_model* m) {
  if (!m || !m->lr || !m->ffm) { set_error("null model"); return DFFM_CONTRACT; }
  if (m->n_fields < 1 || m->n_fields > 255 || m->k < 1 || m->k > 64 || m->hash_bits < 1 ||
      m->hash_bits > 29 || m->n_layers < 0 || m->n_layers == 1 ||
      m->n_layers > DFFM_MAX_LAYERS || m->wdtype < 0 || m->wdtype > 2) {
    set_error("bad model shape");
    return DFFM_CONTRACT;
  }
  const int D = 1 + m->n_fields * (m->n_fields - 1) / 2;
  if (m->n_layers && (m->dims[0] != D || m->dims[m->n_layers] != 1)) {
    set_error("MLP dims do not match 1+F(F-1)/2 -> ... -> 1");
    return DFFM_CONTRACT;
  }
  return DFFM_OK;
}

}  // namespace dffm

using namespace dffm;

extern "C" int64_t dffm_trace_len(const dffm_model* model) {
  if (check_model(model)) return -1;
  return tr_layout(model->n_fields, model->k, model->n_layers, model->dims).total;
}

extern "C" int dffm_forward_trace(const dffm_model* model, const int32_t* idx, const float* val,
                                  int32_t max_per_field, double* trace, void* stream) {
  if (int rc = check_model(model)) return rc;
  if (!idx || !val || !trace || max_per_field < 1 || max_per_field > 4096) {
    set_error("bad trace arguments");
    return DFFM_CONTRACT;
  }
  cudaStream_t s = (cudaStream_t)stream;
  switch (model->wdtype) {
    case DFFM_W_F32:
      note_launches(1), trace_kernel<float><<<1, TR_THREADS, 0, s>>>(*model, idx, val,
                                                                      max_per_field, trace);
      break;
    case DFFM_W_BF16:
      note_launches(1), trace_kernel<__nv_bfloat16><<<1, TR_THREADS, 0, s>>>(
                            *model, idx, val, max_per_field, trace);
      break;
    default:
      note_launches(1), trace_kernel<uint16_t><<<1, TR_THREADS, 0, s>>>(*model, idx, val,
                                                                         max_per_field, trace);
  }
  DFFM_CUDA_TRY(cudaGetLastError(), "launch(trace)");
  return DFFM_OK;
}

extern "C" int64_t dffm_grad_scratch_len(const dffm_model* model) {
  if (check_model(model)) return -1;
  int wmax = 1;
  for (int l = 0; l <= model->n_layers; ++l) wmax = wmax > model->dims[l] ? wmax : model->dims[l];
  return 1 + model->n_fields * (model->n_fields - 1) / 2 + 2 * (int64_t)wmax;
}

extern "C" int dffm_loss_gradients(const dffm_model* model, const int32_t* idx, const float* val,
                                   int32_t max_per_field, const double* trace, int32_t label,
                                   double* grad, int64_t grad_len, double* scratch,
                                   void* stream) {
  if (int rc = check_model(model)) return rc;
  if (label != 0 && label != 1) { set_error("label must be 0 or 1"); return DFFM_CONTRACT; }
  const int64_t nf = (int64_t)1 << model->hash_bits;
  int64_t total = nf + 1 + nf * model->n_fields * model->k;
  for (int l = 0; l < model->n_layers; ++l)
    total += (int64_t)model->dims[l] * model->dims[l + 1] + model->dims[l + 1];
  if (!idx || !val || !trace || !grad || !scratch || grad_len != total) {
    set_error("bad gradient arguments (grad_len %lld, layout wants %lld)", (long long)grad_len,
              (long long)total);
    return DFFM_CONTRACT;
  }
  cudaStream_t s = (cudaStream_t)stream;
  DFFM_CUDA_TRY(cudaMemsetAsync(grad, 0, (size_t)total * 8, s), "memset(grad)");
  note_launches(1), grad_kernel<<<1, TR_THREADS, 0, s>>>(*model, idx, val, max_per_field, trace,
                                                         label, grad, scratch);
  DFFM_CUDA_TRY(cudaGetLastError(), "launch(loss_gradients)");
  return DFFM_OK;
}
