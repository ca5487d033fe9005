/*
 * dffm.h -- C ABI of libdffm.so, the B200 (sm_100a) DeepFFM hot path.
 *
 * The reference (`fieldwise`, /root/reference/pkg/src/fieldwise) has no FFI:
 * its boundary is the Python API of model.py.  Each entry point below
 * replaces one reference function (cited file:line) and is what a ctypes /
 * cffi binding of that Python API calls.
 *
 * Conventions
 *   - Every pointer argument is a caller-owned DEVICE pointer unless named
 *     *_host.  Nothing here allocates on the hot path or frees caller memory.
 *   - `stream` is a cudaStream_t passed as void*; every call is asynchronous
 *     on it.  Results that need a host decision (status words) are read back
 *     by the caller.
 *   - Return value: DFFM_OK or an error class mirroring fieldwise/errors.py;
 *     dffm_last_error() gives a thread-local message for the last failure.
 *   - Device status word (uint64, initialise to all-ones): kernels report
 *     the first offending example with atomicMin on
 *         (example_index << 8) | (block << 4) | code
 *     so the host raises the same exception class, for the same (first)
 *     example, with the same `block` name as the reference would.
 */
#ifndef DFFM_H
#define DFFM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* error classes (E: errors.py) */
enum dffm_status {
  DFFM_OK = 0,
  DFFM_CONTRACT = 1, /* ContractError  E:32  (bad field id, index, label, stale state) */
  DFFM_FORMAT = 2,   /* FormatError    E:16 */
  DFFM_NUMERIC = 3,  /* NumericError   E:40  (block code in the status word) */
  DFFM_SIZING = 4,   /* SizingError    E:36 */
  DFFM_CUDA = 5      /* CUDA runtime failure */
};

/* NumericError.block, in the reference's diagnosis order (M:308-318, M:458) */
enum dffm_block {
  DFFM_BLOCK_NONE = 0, DFFM_BLOCK_LR = 1, DFFM_BLOCK_FFM = 2, DFFM_BLOCK_MERGE = 3,
  DFFM_BLOCK_NN = 4, DFFM_BLOCK_LOGIT = 5, DFFM_BLOCK_LOSS = 6
};

/* storage type of the hashed lr / ffm tables */
enum dffm_wdtype { DFFM_W_F32 = 0, DFFM_W_BF16 = 1, DFFM_W_U16Q = 2 };

#define DFFM_MAX_LAYERS 5 /* <= 4 hidden layers (M:70-71) + the output layer */

/*
 * Device-resident model (replaces WeightStore, M:142-230).  Each block is a
 * separate 256-byte-aligned allocation instead of the reference's one flat
 * array (whose ffm block starts 4 bytes past a 16-byte boundary, M:182):
 *   lr   [2^b + 1]        lr weights, bias at index 2^b        (M:148-149)
 *   ffm  [2^b][F][k]      field-aware latent rows, row-major   (M:150-151)
 *   W[l] [in][out] f32, b[l] [out] f32 per MLP layer           (M:152, M:198-210)
 * For DFFM_W_U16Q the lr/ffm tables hold 16-bit bucket indices and are
 * dequantised inline as  w = q_min + idx * q_bucket  (f32 mul, then f32 add).
 */
typedef struct dffm_model {
  int32_t n_fields;
  int32_t k;
  int32_t hash_bits;
  int32_t n_layers;                    /* 0 (no MLP) or len(hidden)+1 */
  int32_t dims[DFFM_MAX_LAYERS + 1];   /* dims[0] = 1+F(F-1)/2 ... dims[n_layers] = 1 */
  int32_t wdtype;                      /* enum dffm_wdtype */
  int32_t _pad;
  const void* lr;
  const void* ffm;
  const float* W[DFFM_MAX_LAYERS];
  const float* b[DFFM_MAX_LAYERS];
  float q_lr_min, q_lr_bucket;         /* per-table FWQ1 headers (u16 only) */
  float q_ffm_min, q_ffm_bucket;
} dffm_model;

/* Library identity / diagnostics */
int dffm_abi_version(void);
const char* dffm_last_error(void);
/* sha256 prefix of the kernel sources + Makefile the library was built from */
const char* dffm_build_id(void);
int dffm_device_sm_count(int device);

/*
 * K1 fused forward, batched: replaces model.forward + predict_proba
 * (M:300-397) as called per example by training.evaluate_stream
 * (T:221-236).  Inputs are canonical padded examples (Fe:121-172):
 *   idx [n][F][max_per_field] int32, -1 = empty slot, indices strictly
 *   increasing within a field; val same shape, f32.
 * Outputs prob[n] (clamped sigmoid, M:304-305) and optionally logit[n].
 * status_base is added to example numbers reported in the status word, so
 * chunked or sharded launches report the caller's global example index.
 */
int dffm_forward(const dffm_model* model, const int32_t* idx, const float* val,
                 int32_t max_per_field, int64_t n, float* prob, float* logit_opt,
                 int64_t status_base, uint64_t* status, void* stream);

/*
 * K1 kernel family (all compute identical results within the 1e-5 contract;
 * shapes a family cannot take fall back to family 2):
 *   1 warp-specialised (fused MLP on CUDA cores), 2 CTA-synchronous,
 *   5 staged rows + tcgen05 3xTF32 MLP (hidden widths multiples of 16, <= 256),
 *   -1 = default: DFFM_FORWARD_KERNEL (ws|v1|tc) if set, else 5 (K1 v8
 *   row-ring gather + tcgen05 MLP) when the ring takes the shape (M <= 4,
 *   F*M <= 128, k in {4, 8, 16}) and the hidden widths are multiples of 16,
 *   or when the MLP has >= 64K multiply-adds per example; otherwise 1.
 * Family 5 keeps a per-(device, stream) device workspace (staged rows of one
 * slice + the blocked hi/lo MLP weights), allocated on first use.
 * Thread-local: applies to dffm_forward calls made by the calling host
 * thread only (reentrant across host threads). Other values: DFFM_CONTRACT.
 */
int dffm_set_forward_family(int32_t family);

/*
 * Per-thread launch trace for measurement (bench.py): while set, every
 * kernel dffm_forward launches is followed by cudaEventRecord(events[i])
 * on the launch stream and tags[i] = its role (0 weight blocking for the
 * tensor-core MLP, 1 row gather, 2 tcgen05 MLP, 3 fused forward); *count
 * advances, up to capacity. events = NULL clears the trace. The events are
 * caller-created cudaEvent_t handles.
 */
int dffm_set_event_trace(void** events, int32_t* tags, int32_t capacity, int32_t* count);

/*
 * K3 context-cached scorer (no reference code).  Request r
 * has ctx fields [0, n_ctx_fields) in ctx_idx[r][n_ctx_fields][ctx_m] and
 * n_cand candidates with fields [n_ctx_fields, F) in
 * cand_idx[r][n_cand][F - n_ctx_fields][cand_m].  prob[r][n_cand] equals
 * forward+predict_proba on the merged example.
 */
int dffm_ctx_score(const dffm_model* model, const int32_t* ctx_idx, const float* ctx_val,
                   int32_t n_ctx_fields, int32_t ctx_m, const int32_t* cand_idx,
                   const float* cand_val, int32_t cand_m, int64_t n_requests, int32_t n_cand,
                   float* prob, uint64_t* status, void* stream);

/*
 * Device-resident context caches (SPEC S:248-262 build_context_cache, S:263-271
 * predict_batch): dffm_ctx_build writes, per request, a blob of
 * dffm_ctx_cache_bytes() bytes (16-byte aligned) holding the context slots,
 * the context lr partial, the context latent sums S[x][g][:] and the
 * ctx x ctx pair outputs with their f64 moments; a bad context index is a
 * ContractError at that request.  dffm_ctx_score_cached scores candidates
 * against prebuilt blobs (no context pass; the context rows are still passed
 * for shapes the row-ring kernel does not take, which rebuild in-kernel).
 * dffm_ctx_build_count(): request caches built so far by this library.
 */
int64_t dffm_ctx_cache_bytes(const dffm_model* model, int32_t n_ctx_fields, int32_t ctx_m);
int dffm_ctx_build(const dffm_model* model, const int32_t* ctx_idx, const float* ctx_val,
                   int32_t n_ctx_fields, int32_t ctx_m, int64_t n_requests, void* cache_out,
                   uint64_t* status, void* stream);
int dffm_ctx_score_cached(const dffm_model* model, const void* cache, const int32_t* ctx_idx,
                          const float* ctx_val, int32_t n_ctx_fields, int32_t ctx_m,
                          const int32_t* cand_idx, const float* cand_val, int32_t cand_m,
                          int64_t n_requests, int32_t n_cand, float* prob, uint64_t* status,
                          void* stream);
int64_t dffm_ctx_build_count(void);

/*
 * K2 sequential Adagrad trainer: replaces the predict-then-learn loop of
 * training._train_lines (T:172-185) = forward (M:321) + predict_proba
 * (M:300) + backward_update (M:440-533), in the reference's exact example
 * order, f64 arithmetic over f32 storage.  Mutates the weights of `model`
 * (which must be DFFM_W_F32) and the accumulators in place.
 *   lr_acc [2^b+1], ffm_acc [2^b][F][k], W_acc[l], b_acc[l]   f32, same shapes
 *   labels[n] in {0,1} (else ContractError, M:453-454)
 *   prob_out[n]: the clamped progressive prediction of each example (f64)
 *   scratch: device workspace of dffm_train_scratch_bytes() bytes
 */
typedef struct dffm_train_state {
  float* lr_acc;
  float* ffm_acc;
  float* W_acc[DFFM_MAX_LAYERS];
  float* b_acc[DFFM_MAX_LAYERS];
  double lr_ffm, lr_lr, lr_nn, power_t;
  int32_t sparse;                      /* M:536-572 sparse skip (results identical) */
  int32_t _pad;
} dffm_train_state;

int64_t dffm_train_scratch_bytes(const dffm_model* model, int32_t max_per_field);
int dffm_train_sequential(const dffm_model* model, const dffm_train_state* state,
                          const int32_t* idx, const float* val, const uint8_t* labels,
                          int32_t max_per_field, int64_t n, double* prob_out,
                          void* scratch, uint64_t* status, void* stream);

/*
 * K6 Hogwild-style trainer: replaces hogwild_train (T:269-336).
 * n_workers independent predict-then-learn loops run concurrently on the
 * GPU (one CTA each; worker w takes examples w, w + W, ...) against the SHARED
 * store with no locks -- concurrent updates may overwrite each other (T:1-11),
 * f32 stores never tear.  prob_out[e] is example e's progressive prediction.
 * n_workers == 1 is dffm_train_sequential exactly.  Workers beyond what can be
 * resident at once are not launched (dffm_hogwild_max_workers).  An error in
 * any worker stops every worker at its next example; the status word holds
 * the smallest failing example index.
 */
int dffm_train_hogwild(const dffm_model* model, const dffm_train_state* state,
                       const int32_t* idx, const float* val, const uint8_t* labels,
                       int32_t max_per_field, int64_t n, int32_t n_workers, double* prob_out,
                       void* scratch, uint64_t* status, void* stream);
int dffm_hogwild_max_workers(const dffm_model* model, int32_t max_per_field);

/*
 * K4 16-bit quantisation (formula PAPER.md:291-305).
 *   fwq_minmax:     minmax_out[2] = {min, max} of w[n] (device); *first_nonfinite
 *                   (device, initialise to all-ones) = smallest offset of a
 *                   non-finite weight (SPEC S:317 NumericError "with offset")
 *   fwq_header:     host-side header from min/max, pinned rounding
 *   fwq_quantize:   q[i] = clamp(rint((f64(w)-f64(hmin))/f64(hbucket)), 0, 65535)
 *   fwq_dequantize: out[i] = hmin + q[i]*hbucket  (f32 mul then f32 add, no FMA)
 */
int fwq_minmax(const float* w, int64_t n, float* minmax_out, uint64_t* first_nonfinite,
               void* stream);
int fwq_header(float wmin, float wmax, int32_t alpha, int32_t beta, float* hmin_host,
               float* hbucket_host);
int fwq_quantize(const float* w, int64_t n, float hmin, float hbucket, uint16_t* q,
                 void* stream);
int fwq_dequantize(const uint16_t* q, int64_t n, float hmin, float hbucket, float* out,
                   void* stream);

/*
 * K9 ragged batch -> padded layout (the batched form of Fe:121-172 examples):
 * ex_off int64 [n+1] (absolute; this call reads idx/val at ex_off[e] - nnz_base),
 * cnt u8 [n][n_fields] features per field, idx i32 / val f32 [nnz] in example,
 * field, slot order  ->  out_idx i32 / out_val f32 [n][n_fields][max_per_field]
 * (-1 / 0 padding), ready for dffm_forward.  A count above max_per_field or a
 * count sum that disagrees with ex_off sets DFFM_CONTRACT for that example in
 * the status word (status_base + e).  Device pointers, async on `stream`.
 */
int dffm_unpack_ragged(const int64_t* ex_off, const uint8_t* cnt, const int32_t* idx,
                       const float* val, int64_t n, int32_t n_fields, int32_t max_per_field,
                       int64_t nnz_base, int32_t* out_idx, float* out_val, int64_t status_base,
                       uint64_t* status, void* stream);

/*
 * K10 text parse (Fe:175-235, H:28-50): lines text[line_off[i]:line_off[i+1]]
 * (no newline) of the reference's example grammar -> canonical hashed features.
 *   fw_parse_scratch_bytes -> device scratch size for (n_lines, text_bytes)
 *   fw_parse_lines: labels u8 [n], line_status i32 [n] (0 ok, else the kind of
 *     ParseError: 1 label, 2 no blocks, 3 empty block, 4 unknown field, 5 bad
 *     value, 6 non-finite value, 7 raw index out of range, 8 unsupported
 *     (non-ASCII whitespace / non-ASCII digits), 9 > 1024 features, 10 > 255
 *     features in one field), cnt u8 [n][n_fields], ex_off int64 [n+1]
 *     (ex_off[n] = total features), max_cnt (largest field count, device i32).
 *     Schema: field names as bytes[name_off[f]:name_off[f+1]], numeric u8 [F].
 *   fw_parse_emit (after reading ex_off[n]): idx i32 / val f32 [nnz] (val64
 *     f64 optional) in field-id order, ascending index within a field.
 * Failed lines hold no features; the caller raises at the first failed line.
 */
int64_t fw_parse_scratch_bytes(int64_t n_lines, int64_t text_bytes);
int fw_parse_lines(const uint8_t* text, const int64_t* line_off, int64_t n_lines,
                   int64_t text_bytes, const uint8_t* names, const int32_t* name_off,
                   const uint8_t* numeric, int32_t n_fields, int32_t hash_bits, void* scratch,
                   uint8_t* labels, int32_t* line_status, uint8_t* cnt, int64_t* ex_off,
                   int32_t* max_cnt, void* stream);
int fw_parse_emit(const int64_t* line_off, int64_t n_lines, int64_t text_bytes,
                  const void* scratch, const int64_t* ex_off, int32_t* idx, float* val,
                  double* val64_opt, void* stream);

/*
 * K9b packed wire format -> padded layout: as dffm_unpack_ragged, but each
 * index is idx_width (3 or 4) little-endian bytes and values equal to 1.0 are
 * elided: bit (bit_base + t) of vbits (LSB first) is set iff feature t of this
 * call carries an explicit f32, stored in vals[voff[e] - val_base + rank].
 * n_fields * max_per_field <= 128.
 */
int dffm_unpack_packed(const int64_t* ex_off, const uint8_t* cnt, const uint8_t* idx_bytes,
                       int32_t idx_width, const uint8_t* vbits, const float* vals,
                       const int64_t* voff, int64_t n, int32_t n_fields, int32_t max_per_field,
                       int64_t nnz_base, int64_t bit_base, int64_t val_base, int32_t* out_idx,
                       float* out_val, int64_t status_base, uint64_t* status, void* stream);

/* Kernels launched by this library so far (all devices and threads). */
int64_t dffm_launch_count(void);

/*
 * K5 feature hashing (H:28-50): out[i] = fnv1a32(bytes[off[i]:off[i+1]]) & (2^bits-1)
 * (bits = 32 returns the raw hash).
 */
int fw_hash_fnv1a32(const uint8_t* bytes, const int64_t* offsets, int64_t n, int32_t bits,
                    uint32_t* out, void* stream);

/*
 * K7 FWP1 byte patches (file format S:381; no reference code).
 * create (device buffers old[old_len], new[new_len]):
 *   fwp_diff_count  -> number of ops (scratch: fwp_scratch_bytes(new_len) B)
 *   fwp_diff_ops    -> ordered op ranges [starts[k], ends[k]) into new
 *   fwp_encode_size -> offsets[k] of each op in the op stream, total bytes
 *   fwp_encode      -> the op stream: varint(skip) varint(length) payload ...
 * apply: fwp_parse_ops (HOST: the op headers are serial by format) then
 *   fwp_scatter (device payload copy into the target buffer).
 * fw_fnv1a64_host: the FNV-1a 64 digest of the header, host bytes.
 * fwp_diff_count / fwp_encode_size synchronise `stream` to return a count.
 */
int64_t fwp_scratch_bytes(int64_t new_len);
int fwp_diff_count(const uint8_t* old_, int64_t old_len, const uint8_t* new_, int64_t new_len,
                   void* scratch, int64_t* n_ops_host, void* stream);
int fwp_diff_ops(const uint8_t* old_, int64_t old_len, const uint8_t* new_, int64_t new_len,
                 const void* scratch, int64_t* starts, int64_t* ends, void* stream);
int fwp_encode_size(const int64_t* starts, const int64_t* ends, int64_t n_ops,
                    int64_t* offsets, void* scratch, int64_t* total_host, void* stream);
int fwp_encode(const uint8_t* new_, const int64_t* starts, const int64_t* ends,
               const int64_t* offsets, int64_t n_ops, uint8_t* out, void* stream);
int fwp_parse_ops(const uint8_t* ops_host, int64_t ops_len, int64_t target_len,
                  int64_t* dst_off_host, int64_t* src_off_host, int64_t* len_host,
                  int64_t max_ops, int64_t* n_ops_out);
int fwp_scatter(uint8_t* dst, const uint8_t* src, const int64_t* dst_off, const int64_t* src_off,
                const int64_t* len, int64_t n_ops, void* stream);
uint64_t fw_fnv1a64_host(const uint8_t* data_host, int64_t n);

/*
 * K8 streaming evaluator: replaces StreamingEvaluator (Me:109-129) and
 * window_auc (Me:21-34) over a device stream.  probs f64 [n] (clamped
 * progressive predictions), labels u8 [n] in {0,1}.  Non-overlapping windows:
 *   auc_out[n / window]            midrank (Mann-Whitney) AUC, NaN if one class
 *   loss_out[ceil(n / window)]     per-window sums of clamped log-losses
 *                                  (the last partial when window does not divide n)
 * window in [2, 57344].
 */
int fw_eval_stream(const double* probs, const uint8_t* labels, int64_t n, int32_t window,
                   double* auc_out, double* loss_out, void* stream);

/*
 * K11 single-example trace (M:321-397 forward with every intermediate the
 * reference's ForwardState keeps, M:275-290) and dense loss gradient
 * (M:575-634 loss_gradients), f64, one CTA.  idx/val: ONE example in the
 * padded layout [n_fields][max_per_field] (device).  trace: device f64
 * buffer of dffm_trace_len(model) values:
 *   [0] lr_out  [1] logit  [2] merge mu  [3] merge sd  [4] nn output
 *   [5] sum of pair outputs  [6..7] reserved
 *   [DFFM_TRACE_HEAD ..] latent sums S [F][F][k], pair outputs [P],
 *   merge vector v [D], merged input [D], then per hidden layer
 *   pre-activations [h] followed by activations [h].
 * dffm_loss_gradients zero-fills grad (f64, the weights' flat layout
 * lr | ffm | per layer W, b: dffm's weights_total values) and writes the
 * log-loss gradient of that example and label; scratch holds
 * dffm_grad_scratch_len(model) doubles.
 */
#define DFFM_TRACE_HEAD 8
int64_t dffm_trace_len(const dffm_model* model);
int dffm_forward_trace(const dffm_model* model, const int32_t* idx, const float* val,
                       int32_t max_per_field, double* trace, void* stream);
int64_t dffm_grad_scratch_len(const dffm_model* model);
int dffm_loss_gradients(const dffm_model* model, const int32_t* idx, const float* val,
                        int32_t max_per_field, const double* trace, int32_t label,
                        double* grad, int64_t grad_len, double* scratch, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DFFM_H */
