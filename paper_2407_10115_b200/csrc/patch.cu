// K7: FWP1 byte patches between two weight files.
//
// create: a byte at offset i < new_len differs if i >= old_len or
// old[i] != new[i]; differing runs separated by fewer than GAP_MERGE = 4
// identical bytes form one op.  With d(i) the differ flag, an
// op STARTS at i iff d(i) and none of d(i-4..i-1), and ENDS at i iff d(i) and
// none of d(i+1..i+4) -- local rules, so the diff is a data-parallel pass over
// both buffers (HBM-bound: 2 bytes read per byte of new):
//   count   one CTA per 32 KB block; each thread owns 16-byte chunks, builds
//           the differ mask of its chunk plus a 4-byte halo on each side and
//           pops the start / end bits
//   scan    one CTA: exclusive prefix of the per-block counts (ordered ops)
//   ops     the same pass again, writing start / end offsets at the scanned
//           positions in byte order
//   size    per op: varint(skip) + varint(length) + length; scan -> offsets
//   encode  one warp per op: the two LEB128 varints and the payload bytes
// apply: op headers are parsed on the host (each op's position depends on the
// previous one by format), payloads are scattered on the device.
// Digests (FNV-1a 64 over the whole content) are serial by definition
// and computed on the host.
#include "common.cuh"

namespace dffm {

constexpr int PB_THREADS = 256;
constexpr int PB_ITERS = 8;
constexpr int64_t PB_BLOCK = (int64_t)PB_THREADS * 16 * PB_ITERS;  // bytes per CTA
constexpr int PATCH_GAP = 4;

struct PatchIn {
  const uint8_t* old_;
  int64_t old_len;
  const uint8_t* new_;
  int64_t new_len;
};

__device__ __forceinline__ int differs(const PatchIn& in, int64_t i) {
  if (i < 0 || i >= in.new_len) return 0;
  if (i >= in.old_len) return 1;
  return in.old_[i] != in.new_[i];
}

// bit b (0..15) of the result = byte base+b starts / ends an op
__device__ __forceinline__ void chunk_masks(const PatchIn& in, int64_t base, uint32_t* smask,
                                            uint32_t* emask) {
  // d bits: bit j <-> byte base - 4 + j, j in [0, 24)
  uint32_t d = 0;
  if (base + 16 <= in.old_len && base + 16 <= in.new_len && ((base & 15) == 0) &&
      (((uintptr_t)in.old_ & 15) == 0) && (((uintptr_t)in.new_ & 15) == 0)) {
    const uint4 a = *(const uint4*)(in.old_ + base);
    const uint4 b = *(const uint4*)(in.new_ + base);
    const uint32_t aw[4] = {a.x, a.y, a.z, a.w}, bw[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const uint32_t x = aw[w] ^ bw[w];
#pragma unroll
      for (int k = 0; k < 4; ++k) d |= (uint32_t)(((x >> (8 * k)) & 0xFF) != 0) << (4 + 4 * w + k);
    }
  } else {
    for (int j = 0; j < 16; ++j) d |= (uint32_t)differs(in, base + j) << (4 + j);
  }
  for (int j = 0; j < 4; ++j) {
    d |= (uint32_t)differs(in, base - 4 + j) << j;
    d |= (uint32_t)differs(in, base + 16 + j) << (20 + j);
  }
  const uint32_t before = (d << 1) | (d << 2) | (d << 3) | (d << 4);  // any of the 4 bytes before
  const uint32_t after = (d >> 1) | (d >> 2) | (d >> 3) | (d >> 4);   // any of the 4 bytes after
  *smask = ((d & ~before) >> 4) & 0xFFFFu;
  *emask = ((d & ~after) >> 4) & 0xFFFFu;
}

__global__ void __launch_bounds__(PB_THREADS) patch_count_kernel(PatchIn in, int64_t* cnt_s,
                                                                 int64_t* cnt_e) {
  const int64_t b0 = (int64_t)blockIdx.x * PB_BLOCK;
  int cs = 0, ce = 0;
#pragma unroll 1
  for (int it = 0; it < PB_ITERS; ++it) {
    const int64_t base = b0 + ((int64_t)it * PB_THREADS + threadIdx.x) * 16;
    if (base >= in.new_len) break;
    uint32_t sm, em;
    chunk_masks(in, base, &sm, &em);
    cs += __popc(sm);
    ce += __popc(em);
  }
  __shared__ int red[2][PB_THREADS / 32];
  cs = __reduce_add_sync(0xffffffffu, cs);
  ce = __reduce_add_sync(0xffffffffu, ce);
  if ((threadIdx.x & 31) == 0) { red[0][threadIdx.x >> 5] = cs; red[1][threadIdx.x >> 5] = ce; }
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t a = 0, b = 0;
    for (int w = 0; w < PB_THREADS / 32; ++w) { a += red[0][w]; b += red[1][w]; }
    cnt_s[blockIdx.x] = a;
    cnt_e[blockIdx.x] = b;
  }
}

// single-CTA exclusive scan in place; total -> *total
__global__ void __launch_bounds__(1024) scan_i64_kernel(int64_t* v, int64_t n, int64_t* total) {
  __shared__ int64_t part[1024];
  const int t = threadIdx.x;
  const int64_t per = (n + 1023) / 1024;
  const int64_t a = min(n, (int64_t)t * per), b = min(n, a + per);
  int64_t s = 0;
  for (int64_t i = a; i < b; ++i) s += v[i];
  part[t] = s;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {  // inclusive Hillis-Steele
    const int64_t x = t >= o ? part[t - o] : 0;
    __syncthreads();
    part[t] += x;
    __syncthreads();
  }
  int64_t run = t ? part[t - 1] : 0;
  for (int64_t i = a; i < b; ++i) {
    const int64_t x = v[i];
    v[i] = run;
    run += x;
  }
  if (t == 1023) *total = part[1023];
}

// ordered positions of the starts / ends in this CTA's block
__global__ void __launch_bounds__(PB_THREADS) patch_ops_kernel(PatchIn in, const int64_t* off_s,
                                                               const int64_t* off_e,
                                                               int64_t* starts, int64_t* ends) {
  const int64_t b0 = (int64_t)blockIdx.x * PB_BLOCK;
  __shared__ int ws[PB_THREADS / 32], we[PB_THREADS / 32];
  int64_t ps = off_s[blockIdx.x], pe = off_e[blockIdx.x];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll 1
  for (int it = 0; it < PB_ITERS; ++it) {
    const int64_t base = b0 + ((int64_t)it * PB_THREADS + threadIdx.x) * 16;
    uint32_t sm = 0, em = 0;
    if (base < in.new_len) chunk_masks(in, base, &sm, &em);
    const int cs = __popc(sm), ce = __popc(em);
    // CTA-wide exclusive prefix of (cs, ce) in thread order = byte order
    int is = cs, ie = ce;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int xs = __shfl_up_sync(0xffffffffu, is, o), xe = __shfl_up_sync(0xffffffffu, ie, o);
      if (lane >= o) { is += xs; ie += xe; }
    }
    if (lane == 31) { ws[warp] = is; we[warp] = ie; }
    __syncthreads();
    int wps = 0, wpe = 0, ts = 0, te = 0;
    for (int w = 0; w < PB_THREADS / 32; ++w) {
      if (w < warp) { wps += ws[w]; wpe += we[w]; }
      ts += ws[w];
      te += we[w];
    }
    int64_t qs = ps + wps + is - cs, qe = pe + wpe + ie - ce;
    while (sm) { const int j = __ffs(sm) - 1; sm &= sm - 1; starts[qs++] = base + j; }
    while (em) { const int j = __ffs(em) - 1; em &= em - 1; ends[qe++] = base + j + 1; }
    ps += ts;
    pe += te;
    __syncthreads();
  }
}

__device__ __forceinline__ int varint_len(uint64_t x) {
  int n = 1;
  while (x >= 0x80) { x >>= 7; ++n; }
  return n;
}

__global__ void patch_size_kernel(const int64_t* starts, const int64_t* ends, int64_t n_ops,
                                  int64_t* sizes) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n_ops;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t prev = k ? ends[k - 1] : 0;
    const uint64_t skip = (uint64_t)(starts[k] - prev), len = (uint64_t)(ends[k] - starts[k]);
    sizes[k] = varint_len(skip) + varint_len(len) + (int64_t)len;
  }
}

__device__ __forceinline__ int put_varint(uint8_t* o, uint64_t x) {
  int n = 0;
  while (x >= 0x80) { o[n++] = (uint8_t)(x | 0x80); x >>= 7; }
  o[n++] = (uint8_t)x;
  return n;
}

// one warp per op: varints by lane 0, payload bytes by all lanes
__global__ void patch_encode_kernel(const uint8_t* new_, const int64_t* starts,
                                    const int64_t* ends, const int64_t* offsets, int64_t n_ops,
                                    uint8_t* out) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t k = wid; k < n_ops; k += nw) {
    const int64_t prev = k ? ends[k - 1] : 0;
    const int64_t s = starts[k], len = ends[k] - s;
    uint8_t* o = out + offsets[k];
    const int h = varint_len((uint64_t)(s - prev)) + varint_len((uint64_t)len);
    if (lane == 0) {
      const int n1 = put_varint(o, (uint64_t)(s - prev));
      put_varint(o + n1, (uint64_t)len);
    }
    for (int64_t i = lane; i < len; i += 32) o[h + i] = new_[s + i];
  }
}

// apply: payload scatter, one warp per op
__global__ void patch_scatter_kernel(uint8_t* dst, const uint8_t* src, const int64_t* dst_off,
                                     const int64_t* src_off, const int64_t* len, int64_t n_ops) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t k = wid; k < n_ops; k += nw) {
    const int64_t d = dst_off[k], s = src_off[k], n = len[k];
    for (int64_t i = lane; i < n; i += 32) dst[d + i] = src[s + i];
  }
}

static int64_t n_blocks(int64_t new_len) { return (new_len + PB_BLOCK - 1) / PB_BLOCK; }

}  // namespace dffm

using namespace dffm;

extern "C" int64_t fwp_scratch_bytes(int64_t new_len) {
  return (2 * std::max<int64_t>(n_blocks(new_len), 1) + 4) * 8;
}

extern "C" int fwp_diff_count(const uint8_t* old_, int64_t old_len, const uint8_t* new_,
                              int64_t new_len, void* scratch, int64_t* n_ops_host,
                              void* stream) {
  if (old_len < 0 || new_len < 0 || !scratch || !n_ops_host || (old_len && !old_) ||
      (new_len && !new_)) {
    set_error("bad patch arguments");
    return DFFM_CONTRACT;
  }
  *n_ops_host = 0;
  if (new_len == 0) return DFFM_OK;
  const cudaStream_t s = (cudaStream_t)stream;
  const int64_t nb = n_blocks(new_len);
  int64_t* cnt_s = (int64_t*)scratch;
  int64_t* cnt_e = cnt_s + nb;
  int64_t* tot = cnt_e + nb;
  PatchIn in{old_, old_len, new_, new_len};
  note_launches(1), patch_count_kernel<<<(unsigned)nb, PB_THREADS, 0, s>>>(in, cnt_s, cnt_e);
  note_launches(1), scan_i64_kernel<<<1, 1024, 0, s>>>(cnt_s, nb, tot);
  note_launches(1), scan_i64_kernel<<<1, 1024, 0, s>>>(cnt_e, nb, tot + 1);
  DFFM_CUDA_TRY(cudaGetLastError(), "launch(patch count)");
  int64_t h[2];
  DFFM_CUDA_TRY(cudaMemcpyAsync(h, tot, 16, cudaMemcpyDeviceToHost, s), "copy(patch count)");
  DFFM_CUDA_TRY(cudaStreamSynchronize(s), "sync(patch count)");
  if (h[0] != h[1]) {
    set_error("patch diff: %lld starts vs %lld ends", (long long)h[0], (long long)h[1]);
    return DFFM_CUDA;
  }
  *n_ops_host = h[0];
  return DFFM_OK;
}

// after fwp_diff_count (same scratch): ordered op ranges [starts[k], ends[k])
extern "C" int fwp_diff_ops(const uint8_t* old_, int64_t old_len, const uint8_t* new_,
                            int64_t new_len, const void* scratch, int64_t* starts, int64_t* ends,
                            void* stream) {
  if (new_len == 0) return DFFM_OK;
  const int64_t nb = n_blocks(new_len);
  const int64_t* off_s = (const int64_t*)scratch;
  PatchIn in{old_, old_len, new_, new_len};
  note_launches(1), patch_ops_kernel<<<(unsigned)nb, PB_THREADS, 0, (cudaStream_t)stream>>>(in, off_s, off_s + nb,
                                                                          starts, ends);
  DFFM_CUDA_TRY(cudaGetLastError(), "launch(patch ops)");
  return DFFM_OK;
}

// encoded op-stream size: offsets[n_ops] (device) gets each op's output offset
extern "C" int fwp_encode_size(const int64_t* starts, const int64_t* ends, int64_t n_ops,
                               int64_t* offsets, void* scratch, int64_t* total_host,
                               void* stream) {
  *total_host = 0;
  if (n_ops == 0) return DFFM_OK;
  const cudaStream_t s = (cudaStream_t)stream;
  const int grid = (int)std::min<int64_t>((n_ops + 255) / 256, (int64_t)sm_count_current() * 8);
  note_launches(1), patch_size_kernel<<<grid, 256, 0, s>>>(starts, ends, n_ops, offsets);
  int64_t* tot = (int64_t*)scratch;
  note_launches(1), scan_i64_kernel<<<1, 1024, 0, s>>>(offsets, n_ops, tot);
  DFFM_CUDA_TRY(cudaGetLastError(), "launch(patch size)");
  DFFM_CUDA_TRY(cudaMemcpyAsync(total_host, tot, 8, cudaMemcpyDeviceToHost, s), "copy(size)");
  DFFM_CUDA_TRY(cudaStreamSynchronize(s), "sync(patch size)");
  return DFFM_OK;
}

extern "C" int fwp_encode(const uint8_t* new_, const int64_t* starts, const int64_t* ends,
                          const int64_t* offsets, int64_t n_ops, uint8_t* out, void* stream) {
  if (n_ops == 0) return DFFM_OK;
  const int grid = (int)std::min<int64_t>((n_ops * 32 + 255) / 256, (int64_t)sm_count_current() * 16);
  note_launches(1), patch_encode_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(new_, starts, ends, offsets, n_ops,
                                                              out);
  DFFM_CUDA_TRY(cudaGetLastError(), "launch(patch encode)");
  return DFFM_OK;
}

// host: parse the op stream (after the 32-byte header) into scatter lists;
// *n_ops_out = ops found (if > max_ops only the count is returned).  Errors
// mirror the reference's apply_patch: truncated or over-long
// varints, payloads past the end, ops overrunning the target -> FORMAT.
extern "C" int fwp_parse_ops(const uint8_t* ops, int64_t ops_len, int64_t target_len,
                             int64_t* dst_off, int64_t* src_off, int64_t* len, int64_t max_ops,
                             int64_t* n_ops_out) {
  int64_t pos = 0, cur = 0, k = 0;
  auto varint = [&](uint64_t* v) -> int {
    uint64_t x = 0;
    for (int i = 0; i < 10; ++i) {
      if (pos >= ops_len) return DFFM_FORMAT;
      const uint8_t b = ops[pos++];
      if (i == 9 && (b & 0x7E)) return DFFM_FORMAT;  // > 64 bits
      x |= (uint64_t)(b & 0x7F) << (7 * i);
      if (!(b & 0x80)) { *v = x; return DFFM_OK; }
    }
    return DFFM_FORMAT;
  };
  while (pos < ops_len) {
    uint64_t skip, n;
    if (varint(&skip) || varint(&n)) { set_error("truncated or over-long varint"); return DFFM_FORMAT; }
    const uint64_t start = (uint64_t)cur + skip;
    if (start < (uint64_t)cur || start + n < start || start + n > (uint64_t)target_len) {
      set_error("op overruns target length");
      return DFFM_FORMAT;
    }
    if ((uint64_t)pos + n > (uint64_t)ops_len) { set_error("truncated payload"); return DFFM_FORMAT; }
    if (k < max_ops) { dst_off[k] = (int64_t)start; src_off[k] = pos; len[k] = (int64_t)n; }
    ++k;
    pos += (int64_t)n;
    cur = (int64_t)(start + n);
  }
  *n_ops_out = k;
  return DFFM_OK;
}

extern "C" int fwp_scatter(uint8_t* dst, const uint8_t* src, const int64_t* dst_off,
                           const int64_t* src_off, const int64_t* len, int64_t n_ops,
                           void* stream) {
  if (n_ops == 0) return DFFM_OK;
  const int grid = (int)std::min<int64_t>((n_ops * 32 + 255) / 256, (int64_t)sm_count_current() * 16);
  note_launches(1), patch_scatter_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(dst, src, dst_off, src_off, len,
                                                               n_ops);
  DFFM_CUDA_TRY(cudaGetLastError(), "launch(patch scatter)");
  return DFFM_OK;
}

// FNV-1a 64 over host bytes: serial by definition
extern "C" uint64_t fw_fnv1a64_host(const uint8_t* data, int64_t n) {
  uint64_t h = 0xCBF29CE484222325ull;
  for (int64_t i = 0; i < n; ++i) h = (h ^ data[i]) * 0x100000001B3ull;
  return h;
}
