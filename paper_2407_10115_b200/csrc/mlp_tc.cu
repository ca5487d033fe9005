// K1 MLP stage on tcgen05 tensor cores (M:362-377 for a slice of examples whose
// MergeNorm rows the gather kernel staged in HBM/L2; see forward.cu).
//
// Precision: every f32 operand is split into two fp16 pieces and the products
// run as kind::f16 MMAs with f32 accumulation (twice the tensor rate of tf32
// and half its operand bytes):
//     x = x0 + x1     x0 = fp16(x),  x1 = fp16(x - x0)      (22 significant bits)
//     x.w ~= x0.w0 + x0.w1 + x1.w0                           (x1.w1 ~ 2^-22 x.w dropped)
// so one K=16 chunk is three MMAs into the same accumulator.  fp16's exponent
// range is narrow, so each layer's weights and each example row of hidden
// activations are scaled by a power of two (exact) that puts their maximum in
// [2^14, 2^15): nothing overflows and the residual pieces stay normal.  The
// epilogue undoes both scales exactly.  Non-finite values stay non-finite
// (NaN/inf propagate), as the diagnosis of M:308-318 needs.
//
// One persistent CTA per SM walks tiles of 128 examples.  For each hidden
// layer l the tile's pre-activations Z_l[128 x N_l] accumulate in TMEM (f32,
// one lane per example) as a K-loop of 16-wide chunks through a ring of
// shared-memory stages:
//   warp 0     TMA producer: layer 0's A tiles (one 4-D TMA of the staged hi /
//              lo planes the gather kernel wrote, xstore4) and every layer's
//              blocked fp16 W chunk (1-D bulk copy)
//   warp 1     MMA issuer (one thread): three tcgen05.mma.kind::f16 per chunk
//   epilogue   (four column parts per TMEM lane quadrant) drain each
//              accumulation group from TMEM into IEEE f32 register sums, then
//              unscale, +bias, ReLU (NaN kept, M:370) -> the next layer's fp16
//              A tiles straight from registers; last: output column dot
//              product (parts meet in shared memory), residual logit (M:377),
//              clamped sigmoid (M:304-305), status.
// Operand layouts are the canonical no-swizzle K-major core-matrix layouts
// (8 rows x 16 bytes per core matrix; LBO = K-direction core stride, SBO =
// 8-row group stride), as validated for tf32 by tools/tc_probe.cu.
#include "mlp_tc.cuh"

namespace dffm {

#ifdef DFFM_TC_TRACE  // measurement variant: MMA-issuer timeline of CTA 0
constexpr int TCT_N = 4096;
__device__ long long g_tct[TCT_N];
__device__ int g_tct_n;
#define TCT(tag) do { if (blockIdx.x == 0) { int i_ = atomicAdd(&g_tct_n, 1); if (i_ < TCT_N) \
    g_tct[i_] = (clock64() << 8) | (tag); } } while (0)
#define TCE(tag) do { if (threadIdx.x == 64) TCT(tag); } while (0)
#else
#define TCT(tag) do { } while (0)
#define TCE(tag) do { } while (0)
#endif

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* tm, int c0, int c1,
                                            int c2, int c3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// shared-memory matrix descriptor (sm_100 version bit 46; base offset 0, no swizzle)
__device__ __forceinline__ uint64_t umma_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}

// instruction descriptor: D f32, A/B f16, both K-major, M x N
__device__ __forceinline__ uint32_t idesc_f16(int m, int n) {
  return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void mma_f16(uint32_t d, uint64_t a, uint64_t b, uint32_t id,
                                        uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc));
}

// same, A (M x 16 fp16) read from TMEM: one lane per row, 8 columns of packed pairs
__device__ __forceinline__ void mma_f16_ta(uint32_t d, uint32_t a, uint64_t b, uint32_t id,
                                           uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
      "r"(a), "l"(b), "r"(id), "r"(acc));
}

// 32 lanes x 8 consecutive 32-bit columns of TMEM <- 8 registers per thread
__device__ __forceinline__ void tmem_st8(uint32_t addr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(addr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
      : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

// 32 lanes x 16 consecutive f32 columns of TMEM -> 16 registers per thread
__device__ __forceinline__ void tmem_ld16(uint32_t addr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(addr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
}

__device__ __forceinline__ float pow2f(int e) {  // 2^e, e in [-126, 127]
  return __int_as_float((127 + e) << 23);
}

// fp16 pieces (hi, lo) of 2 consecutive values, packed in pairs (paired cvts)
__device__ __forceinline__ void split2(float x, float y, uint32_t& hi, uint32_t& lo) {
  const __half2 h = __floats2half2_rn(x, y);
  const float2 b = __half22float2(h);
  const __half2 l = __floats2half2_rn(x - b.x, y - b.y);
  hi = *(const uint32_t*)&h;
  lo = *(const uint32_t*)&l;
}

// power-of-two exponent putting a maximum magnitude m in [2^14, 2^15)
__device__ __forceinline__ int range_exp(float m) {
  return m > 0.f ? max(-100, min(100, TC_HEXP - ilogbf(m))) : 0;
}

// Accumulation: each layer accumulates in one TMEM region (regions alternate
// per layer, so the MMAs of the next layer or tile run while the epilogue
// reads the previous accumulator).  The tensor core's f32 accumulation is
// coarser than IEEE round-to-nearest (tools/tc_accuracy.cu); with the fp16
// pieces a whole cfg5 layer 0 (49 chunks) stays at 3e-6 relative error on the
// probabilities against the 1e-5 contract, so layers are one group of at most
// TC_GROUP chunks (the host checks kin <= 16 * TC_GROUP).

// first 16-column block of part h of an N-wide layer (N % 16 == 0): the
// N/16 blocks are dealt to the TC_PARTS parts as evenly as possible
__device__ __forceinline__ int part_blk(int h, int N) { return (h * (N >> 4)) / TC_PARTS; }

__global__ void __launch_bounds__(TC_THREADS, 1)
mlp_tc_kernel(const __grid_constant__ CUtensorMap tmx, const MlpTcParams p) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int S = p.stages, SB = p.stage_bytes, NH = p.n_hidden;
  uint64_t* full = (uint64_t*)(smem + S * SB);
  uint64_t* empty = full + S;
  uint64_t* abar = empty + S;    // [1] the epilogue wrote the next layer's A buffer
  uint64_t* accf = abar + 2;     // [2] TMEM region holds a finished group
  uint64_t* tempty = accf + 2;   // [2] TMEM region drained by the epilogue
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);
  float* xpart = (float*)((unsigned char*)full + (2 * S + 6) * 8 + 16);  // [2][TC_PARTS][TC_M]
  int* xbad = (int*)(xpart + 2 * TC_PARTS * TC_M);                 // [2][TC_PARTS][TC_M]
  int* xexp = xbad + 2 * TC_PARTS * TC_M;                          // [2][TC_PARTS][TC_M]
  float* cst = (float*)(xexp + 2 * TC_PARTS * TC_M);  // biases | w_out | b_out | 2^-wexp
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(abar, TC_EPI_WARPS);
    for (int r = 0; r < 2; ++r) {
      mbar_init(&accf[r], 1);
      mbar_init(&tempty[r], TC_EPI_WARPS);
    }
    mbar_fence_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(p.tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // stage the constants the epilogue reads for every tile (layer l's bias at
  // offset 256 l, w_out at 1024, b_out at 1280, 2^-wexp[l] at 1281 + l)
  for (int l = 0; l < NH; ++l)
    for (int i = threadIdx.x; i < p.nout[l]; i += blockDim.x) cst[256 * l + i] = p.bias[l][i];
  for (int i = threadIdx.x; i < p.nout[NH - 1]; i += blockDim.x) cst[1024 + i] = p.w_out[i];
  if (threadIdx.x == 0) cst[1280] = *p.b_out;
  if (threadIdx.x < NH) cst[1281 + threadIdx.x] = pow2f(-p.wexp[threadIdx.x]);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t RS = (uint32_t)p.tmem_cols >> 1;  // accumulator region stride (columns)
  const int64_t ntiles = (p.rows + TC_M - 1) / TC_M;
  // newest rows first: the gather kernel wrote the slice in row order just
  // before, so its last rows are the ones still resident in L2
  auto tile_row = [&](int64_t t) { return ntiles - 1 - t; };

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      uint32_t s = 0, ph = 0, wrapped = 0;  // ring stage, its phase, past the first round
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int row0 = (int)(tile_row(t) * TC_M);
        for (int l = 0; l < NH; ++l) {
          const int nck = p.kin[l] >> 4;
          const uint32_t wbytes = (uint32_t)p.nout[l] * 64u;
          const unsigned char* wsrc = (const unsigned char*)p.wblk[l];
          for (int c = 0; c < nck; ++c) {
            if (wrapped) mbar_wait(&empty[s], ph ^ 1u);
            unsigned char* st = smem + s * SB;
            mbar_arrive_expect_tx(&full[s], wbytes + (l == 0 ? 8192u : 0u));
            if (l == 0)  // {8 halfs, 128 rows, 2 K cores, 2 planes} -> A0 | A1
              tma_load_4d(st + TC_OFF_A, &tmx, 0, row0, 2 * c, 0, &full[s]);
            tma_load_1d(st + TC_OFF_B, wsrc, wbytes, &full[s]);
            wsrc += wbytes;
            if (++s == (uint32_t)S) { s = 0; ph ^= 1u; wrapped = 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      uint32_t s = 0, ph = 0;  // ring stage and its phase
      uint32_t gg = 0;         // accumulation-group (= layer) counter
      uint32_t abph = 0;       // phase of abar (one completion per tile and layer >= 1)
      uint32_t d = tmem, dprev = tmem;  // this / the previous layer's accumulator region
      // descriptors of stage 0; stage s adds (s * SB) >> 4 to the 14-bit address field
      const uint32_t st0 = smem_u32(smem);
      const uint64_t a0_0 = umma_desc(st0 + TC_OFF_A, 2048, 128);
      const uint64_t a1_0 = umma_desc(st0 + TC_OFF_A + 4096, 2048, 128);
      const uint32_t sstep = (uint32_t)SB >> 4;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        for (int l = 0; l < NH; ++l) {
          const int nck = p.kin[l] >> 4, N = p.nout[l];
          const uint32_t id = idesc_f16(TC_M, N);
          const uint32_t lboW = (uint32_t)(N >> 3) * 128u;
          const uint64_t b0_0 = umma_desc(st0 + TC_OFF_B, lboW, 128);
          const uint64_t b1_0 = umma_desc(st0 + TC_OFF_B + (uint32_t)N * 32u, lboW, 128);
          if (l > 0) {  // the epilogue rewrote the previous layer's region as this layer's A
            mbar_wait(abar, abph);
            abph ^= 1u;
            dprev = d;
          }
          {  // one accumulation group per layer: its region must have been released
            const uint32_t reg = gg & 1;
            if (gg >= 2) mbar_wait(&tempty[reg], ((gg >> 1) - 1) & 1);
            d = tmem + reg * RS;
          }
          for (int c = 0; c < nck; ++c) {
            if (c == 0) TCT(l * 2);
            mbar_wait(&full[s], ph);
            if (c == 0) TCT(l * 2 + 1);
            tc_fence_after();
            const uint64_t so = (uint64_t)(s * sstep);
            const uint64_t b0 = b0_0 + so, b1 = b1_0 + so;
            if (l == 0) {
              mma_f16(d, a0_0 + so, b0, id, c != 0);
              mma_f16(d, a0_0 + so, b1, id, 1);
              mma_f16(d, a1_0 + so, b0, id, 1);
            } else {  // chunk c of A: hi pieces at column 16c, lo pieces at 16c + 8
              const uint32_t a0 = dprev + (uint32_t)c * 16u, a1 = a0 + 8u;
              mma_f16_ta(d, a0, b0, id, c != 0);
              mma_f16_ta(d, a0, b1, id, 1);
              mma_f16_ta(d, a1, b0, id, 1);
            }
            mma_commit(&empty[s]);  // stage reusable once these MMAs finish
            if (++s == (uint32_t)S) { s = 0; ph ^= 1u; }
          }
          TCT(16 + l);
          mma_commit(&accf[gg & 1]);  // the layer's accumulator is complete
          ++gg;
        }
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue warps
    // One accumulation group per layer (nck <= TC_GROUP, checked on the host):
    // each layer's accumulator is read from TMEM in 16-column blocks, twice
    // for hidden->hidden layers (pass 1: the row's maximum for its power-of-
    // two scale; pass 2: the scaled fp16 A pieces of the next layer), so only
    // one block is live in registers at a time.
    const int ew = warp - 2;               // 0 .. TC_EPI_WARPS-1
    const int h = ew >> 2;                 // column part owned by this warp
    const int q = warp & 3;                // TMEM lane quadrant this warp may access
    const int r = q * 32 + lane;           // tile row = example of this thread
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
    uint32_t dg = 0;                       // drained-group counter
    int tl = 0;                            // local tile counter (exchange buffer parity)
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++tl) {
      int nn_bad = 0;
      int row_e = 0;                       // power-of-two scale of this row's layer input
      float part = 0.f;                    // this part's share of the output dot (M:372)
      for (int l = 0; l < NH; ++l) {
        const int N = p.nout[l];
        // this part's 16-column blocks [b0, b0 + nb) of layer l (parts may be
        // empty when N < 64); they are also the K chunks of layer l + 1 that
        // this part writes (as fp16 pieces, in place) into the accumulator region
        const int b0 = part_blk(h, N), nb = part_blk(h + 1, N) - b0;
        const uint32_t reg = dg & 1;
        mbar_wait(&accf[reg], (dg >> 1) & 1);
        tc_fence_after();
        const uint32_t ta = lane_base + reg * RS + (uint32_t)(b0 * 16);
        // acc * 2^-(weight scale) * 2^-(row scale) = pre-activations (M:368)
        const float zs = cst[1281 + l] * pow2f(-row_e);
        const float* bl = cst + 256 * l + b0 * 16;
        if (l + 1 < NH) {
          float amax = 0.f;
          for (int cb = 0; cb < nb; ++cb) {  // pass 1: ReLU (M:370) maxima
            float v[16];
            tmem_ld16(ta + (uint32_t)cb * 16, v);
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const float z = v[j] * zs + bl[cb * 16 + j];
              nn_bad |= !isfinite(z);
              const float a = relu_nan(z);
              if (a < 3.0e38f) amax = fmaxf(amax, a);  // finite maximum (NaN compares false)
            }
          }
          int* xe = xexp + (l & 1) * TC_PARTS * TC_M;
          xe[h * TC_M + r] = __float_as_int(amax);  // non-negative: int order = float order
          named_bar_sync(2, 32 * TC_EPI_WARPS);
          int mb = 0;
#pragma unroll
          for (int k2 = 0; k2 < TC_PARTS; ++k2) mb = max(mb, xe[k2 * TC_M + r]);
          const int e_next = range_exp(__int_as_float(mb));
          const float a_scale = pow2f(e_next);
          for (int cb = 0; cb < nb; ++cb) {  // pass 2: layer l + 1's A, in place in TMEM
            float v[16];
            tmem_ld16(ta + (uint32_t)cb * 16, v);
            uint32_t hi[8], lo[8];
#pragma unroll
            for (int j = 0; j < 8; ++j)
              split2(relu_nan(v[2 * j] * zs + bl[cb * 16 + 2 * j]) * a_scale,
                     relu_nan(v[2 * j + 1] * zs + bl[cb * 16 + 2 * j + 1]) * a_scale, hi[j], lo[j]);
            tmem_st8(ta + (uint32_t)cb * 16, hi);
            tmem_st8(ta + (uint32_t)cb * 16 + 8, lo);
          }
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          row_e = e_next;
        } else {
          const float* wo = cst + 1024 + b0 * 16;
          for (int cb = 0; cb < nb; ++cb) {  // last hidden layer: straight into the dot
            float v[16];
            tmem_ld16(ta + (uint32_t)cb * 16, v);
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const float z = v[j] * zs + bl[cb * 16 + j];
              nn_bad |= !isfinite(z);
              part = fmaf(relu_nan(z), wo[cb * 16 + j], part);
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          // region release: layer l's MMAs have consumed layer l's A, which
          // lived in layer l-1's region; the last layer's own region is read
          if (l > 0) mbar_arrive(&tempty[reg ^ 1u]);
          if (l + 1 < NH) mbar_arrive(abar);
          else mbar_arrive(&tempty[reg]);
        }
        ++dg;
      }
      // ---- output (M:372-373): the parts' partial dots meet in shared memory
      float* xp = xpart + (tl & 1) * TC_PARTS * TC_M;
      int* xb = xbad + (tl & 1) * TC_PARTS * TC_M;
      if (h > 0) { xp[h * TC_M + r] = part; xb[h * TC_M + r] = nn_bad; }
      named_bar_sync(1, 32 * TC_EPI_WARPS);
      const int64_t e = tile_row(t) * TC_M + r;
      if (h == 0 && e < p.rows) {
        float acc_nn = part;
#pragma unroll
        for (int k2 = 1; k2 < TC_PARTS; ++k2) {  // fixed order: deterministic
          acc_nn += xp[k2 * TC_M + r];
          nn_bad |= xb[k2 * TC_M + r];
        }
        const double nn = (double)acc_nn + (double)cst[1280];
        const double logit = nn + p.resid[e];  // M:377
        p.prob[e] = (float)sigmoid_clamped(logit);
        if (p.logit) p.logit[e] = (float)logit;
        if (!isfinite(logit)) {  // first non-finite stage, M:308-318
          const int fl = p.flags[e] | (nn_bad || !isfinite(acc_nn) ? 8 : 0);
          const int blk = (fl & 1) ? DFFM_BLOCK_LR : (fl & 2) ? DFFM_BLOCK_FFM
                        : (fl & 4) ? DFFM_BLOCK_MERGE : (fl & 8) ? DFFM_BLOCK_NN
                        : DFFM_BLOCK_LOGIT;
          atomicMin((unsigned long long*)p.status,
                    (unsigned long long)status_key(p.status_base + e, blk, DFFM_NUMERIC));
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(p.tmem_cols));
  }
}

// max |w| over the finite weights of one layer (bit pattern of a non-negative
// float: integer order = float order) -> *wmax (zeroed by the host first)
__global__ void tc_wmax_kernel(const float* __restrict__ W, int64_t n, int* wmax) {
  int m = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float a = fabsf(W[i]);
    if (a < 3.0e38f) m = max(m, __float_as_int(a));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m) atomicMax(wmax, m);
}

// W [K][N] f32 row-major (M:198-210) -> kin/16 chunks, each [B0 N x 16][B1 N x 16]
// fp16 in the K-major core-matrix layout the B descriptor expects (rows =
// outputs, 8 K values = 16 bytes per core-matrix row).  The layer is scaled
// by 2^e, e = range_exp(max |w|), so the pieces fit fp16 and the residuals
// stay normal; *wexp = e.
__global__ void tc_prep_weights_kernel(const float* __restrict__ W, int K, int N, int Kp,
                                       const int* __restrict__ wmax, __half* __restrict__ dst,
                                       int* __restrict__ wexp) {
  const int e = range_exp(__int_as_float(*wmax));
  const float sc = pow2f(e);
  if (blockIdx.x == 0 && threadIdx.x == 0) *wexp = e;
  const int64_t total = (int64_t)Kp * N;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(i / N), n = (int)(i - (int64_t)k * N);
    const float w = k < K ? W[(int64_t)k * N + n] * sc : 0.f;
    const __half w0 = __float2half_rn(w);
    const __half w1 = __float2half_rn(w - __half2float(w0));
    const int c = k >> 4, kk = k & 15;
    __half* chunk = dst + (int64_t)c * N * 32;
    const int off = (((kk >> 3) * (N >> 3) + (n >> 3)) * 64) + (n & 7) * 8 + (kk & 7);
    chunk[off] = w0;
    chunk[N * 16 + off] = w1;
  }
}

int launch_tc_prep_weights(const float* W, int K, int N, int Kp, __half* dst, int* wmax,
                           int* wexp, cudaStream_t s) {
  const int64_t total = (int64_t)Kp * N;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 4096);
  DFFM_CUDA_TRY(cudaMemsetAsync(wmax, 0, sizeof(int), s), "memset(wmax)");
  const int64_t nw = (int64_t)K * N;
  note_launches(1), tc_wmax_kernel<<<(int)std::min<int64_t>((nw + 255) / 256, 1024), 256, 0, s>>>(
                        W, nw, wmax);
  DFFM_CUDA_TRY(cudaGetLastError(), "launch(tc_wmax)");
  note_launches(1), tc_prep_weights_kernel<<<blocks, 256, 0, s>>>(W, K, N, Kp, wmax, dst, wexp);
  DFFM_CUDA_TRY(cudaGetLastError(), "launch(tc_prep_weights)");
  return DFFM_OK;
}

int launch_mlp_tc(const CUtensorMap& tmx, const MlpTcParams& p, int smem, cudaStream_t s) {
  int occ = 0;
  int rc = kernel_occupancy((const void*)mlp_tc_kernel, TC_THREADS, smem, &occ);
  if (rc) return rc;
  const int64_t ntiles = (p.rows + TC_M - 1) / TC_M;
  const int64_t grid = std::min<int64_t>(ntiles, (int64_t)sm_count_current());
  note_launches(1), mlp_tc_kernel<<<(unsigned)grid, TC_THREADS, smem, s>>>(tmx, p);
  DFFM_CUDA_TRY(cudaGetLastError(), "launch(mlp_tc)");
  return DFFM_OK;
}

}  // namespace dffm

#ifdef DFFM_TC_TRACE
extern "C" int dffm_debug_tc_trace(long long* out, int n) {
  int cnt = 0;
  cudaMemcpyFromSymbol(&cnt, dffm::g_tct_n, sizeof(int));
  cnt = cnt < n ? cnt : n;
  if (cnt > dffm::TCT_N) cnt = dffm::TCT_N;
  cudaMemcpyFromSymbol(out, dffm::g_tct, sizeof(long long) * cnt);
  int z = 0;
  cudaMemcpyToSymbol(dffm::g_tct_n, &z, sizeof(int));
  return cnt;
}
#endif
