// K8: streaming evaluator (replaces metrics.StreamingEvaluator, Me:109-129,
// and window_auc, Me:21-34) over a device stream of progressive predictions.
//
// Windows are non-overlapping, `window` examples each; a window with one
// label class has no AUC (NaN = the reference's None).  The rank-based AUC
// with midranks for ties equals the Mann-Whitney statistic
//     AUC = (#{(p, n): s_p > s_n} + 0.5 #{(p, n): s_p == s_n}) / (P N)
// so one CTA per window computes the numerator EXACTLY as an integer
// 2 #gt + #eq: the smaller class's scores are staged in shared memory (f64,
// <= window/2 entries) and every thread streams elements of the other class
// against them.  No sort, no floating-point rank sums.
// The same CTA sums its window's clamped log-losses (Me:117-120) in f64; the
// trailing partial window gets its own loss slot.  Per-element logs are the
// CUDA f64 log/log1p (<= 1 ulp from the host libm), so loss sums agree with
// the reference to ~1e-15 relative, not bitwise.
#include <mutex>
#include <unordered_set>

#include "common.cuh"

namespace dffm {

constexpr int EV_THREADS = 1024;
constexpr double EV_CLAMP = 1e-7;  // LOSS_CLAMP, Me:18

__device__ __forceinline__ double clamped_loss(double p, int y) {
  p = fmin(fmax(p, EV_CLAMP), 1.0 - EV_CLAMP);
  return y ? -log(p) : -log1p(-p);
}

__global__ void __launch_bounds__(EV_THREADS) eval_window_kernel(const double* probs,
                                                                 const uint8_t* labels, int64_t n,
                                                                 int window, int64_t n_full,
                                                                 double* auc_out,
                                                                 double* loss_out) {
  extern __shared__ double sbuf[];
  __shared__ unsigned long long red_u[EV_THREADS / 32];
  __shared__ double red_d[EV_THREADS / 32];
  __shared__ int npos_s;
  const int64_t w = blockIdx.x;
  const int64_t a = w * window;
  const int len = (int)((n - a) < window ? (n - a) : (int64_t)window);
  const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
  const double* s = probs + a;
  const uint8_t* y = labels + a;

  // losses + positive count
  double ls = 0.0;
  int np = 0;
  for (int i = tid; i < len; i += EV_THREADS) {
    ls += clamped_loss(s[i], y[i]);
    np += y[i] != 0;
  }
  ls = warp_sum(ls);
  np = __reduce_add_sync(0xffffffffu, np);
  if (lane == 0) { red_d[wp] = ls; red_u[wp] = (unsigned long long)np; }
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    unsigned long long c = 0;
    for (int k = 0; k < EV_THREADS / 32; ++k) { t += red_d[k]; c += red_u[k]; }
    loss_out[w] = t;
    npos_s = (int)c;
  }
  __syncthreads();
  if (w >= n_full) return;  // trailing partial window: loss only
  const int P = npos_s, N = len - P;
  if (P == 0 || N == 0) {
    if (tid == 0) auc_out[w] = __longlong_as_double(0x7ff8000000000000ll);  // None
    return;
  }
  // stage the smaller class (order of staging irrelevant: counting is symmetric)
  const int small_pos = P <= N;
  __shared__ int fill;
  if (tid == 0) fill = 0;
  __syncthreads();
  for (int i = tid; i < len; i += EV_THREADS) {
    if ((y[i] != 0) == small_pos) sbuf[atomicAdd(&fill, 1)] = s[i];
  }
  __syncthreads();
  const int ns = small_pos ? P : N;
  // 2*#(pos > neg) + #(pos == neg), from each large-class element's view
  unsigned long long cnt = 0;
  for (int i = tid; i < len; i += EV_THREADS) {
    if ((y[i] != 0) == small_pos) continue;
    const double v = s[i];
    unsigned int c = 0;
    for (int j = 0; j < ns; ++j) {
      const double u = sbuf[j];
      // small = positives: pair (u, v) = (pos, neg) -> count u > v
      // small = negatives: pair (v, u) = (pos, neg) -> count v > u
      const bool gt = small_pos ? (u > v) : (v > u);
      c += gt ? 2u : (u == v ? 1u : 0u);
    }
    cnt += c;
  }
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  __syncthreads();
  if (lane == 0) red_u[wp] = cnt;
  __syncthreads();
  if (tid == 0) {
    unsigned long long c = 0;
    for (int k = 0; k < EV_THREADS / 32; ++k) c += red_u[k];
    auc_out[w] = (double)c / (2.0 * (double)P * (double)N);
  }
}

}  // namespace dffm

using namespace dffm;

// auc_out[n / window] (NaN = undefined window), loss_out[ceil(n / window)]
// (per-window sums of clamped log-losses, the last one partial when
// window does not divide n).  window in [2, 57344] (the smaller class of a
// window is staged in 227 KB of shared memory).
extern "C" int fw_eval_stream(const double* probs, const uint8_t* labels, int64_t n,
                              int32_t window, double* auc_out, double* loss_out, void* stream) {
  if (n < 0 || window < 2 || window > 57344 || (n && (!probs || !labels || !loss_out))) {
    set_error("bad evaluator arguments (window %d)", window);
    return DFFM_CONTRACT;
  }
  if (n == 0) return DFFM_OK;
  const int64_t n_full = n / window, n_win = (n + window - 1) / window;
  if (n_full && !auc_out) { set_error("null auc_out"); return DFFM_CONTRACT; }
  const int smem = (window / 2) * 8;
  // the dynamic-smem limit is a per-device (context) attribute: set it once per device
  {
    static std::mutex mu;
    static std::unordered_set<int> done;
    int dev = 0;
    DFFM_CUDA_TRY(cudaGetDevice(&dev), "cudaGetDevice");
    std::lock_guard<std::mutex> lk(mu);
    if (!done.count(dev)) {
      DFFM_CUDA_TRY(cudaFuncSetAttribute(eval_window_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         max_smem_optin_current() - 1024),
                    "cudaFuncSetAttribute(eval)");
      done.insert(dev);
    }
  }
  note_launches(1), eval_window_kernel<<<(unsigned)n_win, EV_THREADS, smem, (cudaStream_t)stream>>>(
      probs, labels, n, window, n_full, auc_out, loss_out);
  DFFM_CUDA_TRY(cudaGetLastError(), "launch(eval)");
  return DFFM_OK;
}
