// K1 MLP stage on tcgen05 tensor cores (M:362-377 for a slice of examples whose
// MergeNorm rows the gather kernel staged in HBM/L2; see forward.cu).
//
// One persistent CTA per SM walks tiles of 128 examples.  For each hidden
// layer l the tile's pre-activations Z_l[128 x N_l] accumulate in TMEM (f32,
// one lane per example) as a K-loop of 16-wide chunks through a ring of
// shared-memory stages:
//   warp 0     TMA producer: layer 0's A chunk (X rows, 2-D tensor map, 64-B
//              swizzle) and every layer's W chunk (pre-blocked hi/lo, 1-D bulk)
//   warp 1     MMA issuer (one thread): per 8-wide K step three
//              tcgen05.mma.kind::tf32 -- A_hi*W_hi + A_hi*W_lo + A_lo*W_hi
//              (3xTF32: ~fp32 accuracy from the TF32 tensor cores; the
//              tensor core truncates f32 operands to tf32, so A_hi is the raw
//              f32 and A_lo = x - trunc_tf32(x))
//   warps 2-9  (two per TMEM lane quadrant, each owning half of a layer's
//              columns) layer 0: A_lo for each landed X chunk; every layer:
//              drain each accumulation group from TMEM into f32 register sums
//              (see below), then +bias, ReLU (NaN kept, M:370) -> the next
//              layer's hi/lo A chunks straight from registers; last: output
//              column dot product (halves meet in shared memory), residual
//              logit (M:377), clamped sigmoid (M:304-305), status.
// All operand layouts are the canonical K-major core-matrix layouts
// (validated by tools/tc_probe.cu).
#include "mlp_tc.cuh"

namespace dffm {

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(tm), "r"(c0), "r"(c1), "r"(smem_u32(bar))
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

// shared-memory matrix descriptor (sm_100 version bit 46; base offset 0)
__device__ __forceinline__ uint64_t umma_desc(uint32_t addr, uint32_t lbo, uint32_t sbo,
                                              uint32_t layout) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) |
         ((uint64_t)layout << 61);
}

// instruction descriptor: D f32, A/B tf32, both K-major, M x N
__device__ __forceinline__ uint32_t idesc_tf32(int m, int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t id,
                                         uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc));
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

__device__ __forceinline__ float tf32_lo(float x) {
  return x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}

// Accumulation precision: the tensor core's f32 accumulation is coarser than
// IEEE round-to-nearest (tools/tc_accuracy.cu: one accumulator over K=784 at
// cfg5 scale errs 2.5e-5 x rms vs 3.7e-6 for a sequential fp32 FMA chain), so
// each layer's K-loop is cut into groups of TC_GROUP chunks: a group
// accumulates in one TMEM region (regions alternate), and the epilogue drains
// it into IEEE f32 register sums while the MMAs run the next group.

// one thread's part of a row of accumulators, statically indexed (registers)
struct HalfRow {
  float v[TC_PART_MAX];
};

__device__ __forceinline__ void drain_group(HalfRow& acc, uint32_t taddr, int nblk, bool first) {
#pragma unroll
  for (int cb = 0; cb < TC_PART_MAX / 16; ++cb) {
    if (cb < nblk) {
      float v[16];
      tmem_ld16(taddr + (uint32_t)cb * 16, v);
#pragma unroll
      for (int j = 0; j < 16; ++j) acc.v[cb * 16 + j] = first ? v[j] : acc.v[cb * 16 + j] + v[j];
    }
  }
}

// drain accumulation group #dg (region dg & 1) into this thread's half-row
__device__ __forceinline__ void epi_drain(HalfRow& acc, uint64_t* accf, uint64_t* tempty,
                                          uint32_t& dg, uint32_t lane_base, uint32_t RS,
                                          int col0, int nblk, bool first, int lane) {
  const uint32_t reg = dg & 1;
  mbar_wait(&accf[reg], (dg >> 1) & 1);
  tc_fence_after();
  drain_group(acc, lane_base + reg * RS + (uint32_t)col0, nblk, first);
  tc_fence_before();
  __syncwarp();
  if (lane == 0) mbar_arrive(&tempty[reg]);
  ++dg;
}

// first 16-column block of part h of an N-wide layer (N % 16 == 0): the
// N/16 blocks are dealt to the TC_PARTS parts as evenly as possible
__device__ __forceinline__ int part_blk(int h, int N) { return (h * (N >> 4)) / TC_PARTS; }

__global__ void __launch_bounds__(TC_THREADS, 1)
mlp_tc_kernel(const __grid_constant__ CUtensorMap tmx, const MlpTcParams p) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int S = p.stages, SB = p.stage_bytes, NH = p.n_hidden;
  uint64_t* full = (uint64_t*)(smem + S * SB);
  uint64_t* aready = full + S;
  uint64_t* empty = aready + S;
  uint64_t* lready = empty + S;  // [S] split warps: the stage's A_lo is written (every chunk)
  uint64_t* accf = lready + S;   // [2] TMEM region holds a finished group
  uint64_t* tempty = accf + 2;   // [2] TMEM region drained by the epilogue
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);
  float* xpart = (float*)(smem + S * SB + (4 * S + 4) * 8 + 16);  // [2][TC_PARTS][TC_M]
  int* xbad = (int*)(xpart + 2 * TC_PARTS * TC_M);                 // [2][TC_PARTS][TC_M]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&aready[s], TC_EPI_WARPS);
      mbar_init(&empty[s], 1);
      mbar_init(&lready[s], TC_SPLIT_WARPS);
    }
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
      uint32_t g = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        for (int l = 0; l < NH; ++l) {
          const int nck = p.kin[l] >> 4;
          const uint32_t wbytes = (uint32_t)p.nout[l] * 128u;
          for (int c = 0; c < nck; ++c, ++g) {
            const int s = (int)(g % S);
            const uint32_t u = g / S;
            if (u > 0) mbar_wait(&empty[s], (u - 1) & 1);
            unsigned char* st = smem + s * SB;
            mbar_arrive_expect_tx(&full[s], wbytes + (l == 0 ? 8192u : 0u));
            if (l == 0) tma_load_2d(st, &tmx, c * TC_KC, (int)(tile_row(t) * TC_M), &full[s]);
            tma_load_1d(st + 16384, p.wblk[l] + (size_t)c * p.nout[l] * 32, wbytes, &full[s]);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      uint32_t g = 0, gg = 0;  // chunk counter, accumulation-group counter
      uint32_t apar = 0;       // per-stage phase bits of aready (used by layer >= 1 chunks only)
      uint32_t d = tmem;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        for (int l = 0; l < NH; ++l) {
          const int nck = p.kin[l] >> 4, N = p.nout[l];
          const uint32_t id = idesc_tf32(TC_M, N);
          const uint32_t lboW = (uint32_t)(N >> 3) * 128u;
          for (int c = 0; c < nck; ++c, ++g) {
            const int cg = c % TC_GROUP;
            if (cg == 0) {  // a new group: its region must have been drained
              const uint32_t reg = gg & 1;
              if (gg >= 2) mbar_wait(&tempty[reg], ((gg >> 1) - 1) & 1);
              d = tmem + reg * RS;
            }
            const int s = (int)(g % S);
            const uint32_t u = g / S;
            if (l > 0) {  // A chunk written by the epilogue from the previous layer
              mbar_wait(&aready[s], (apar >> s) & 1u);
              apar ^= 1u << s;
            }
            mbar_wait(&lready[s], u & 1);
            mbar_wait(&full[s], u & 1);
            tc_fence_after();
            const uint32_t st = smem_u32(smem + s * SB);
            const uint32_t whi = st + 16384, wlo = whi + (uint32_t)N * 64u;
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) {
              uint64_t ahi, alo;
              if (l == 0) {  // TMA tile: 128 rows x 64 B, 64-byte swizzle
                ahi = umma_desc(st + ks * 32, 16, 512, 4);
                alo = umma_desc(st + 8192 + ks * 32, 16, 512, 4);
              } else {       // epilogue-written: core-matrix blocked, no swizzle
                ahi = umma_desc(st + ks * 4096, 2048, 128, 0);
                alo = umma_desc(st + 8192 + ks * 4096, 2048, 128, 0);
              }
              const uint64_t bhi = umma_desc(whi + ks * 2 * lboW, lboW, 128, 0);
              const uint64_t blo = umma_desc(wlo + ks * 2 * lboW, lboW, 128, 0);
              mma_tf32(d, ahi, bhi, id, (cg | ks) != 0);
              mma_tf32(d, ahi, blo, id, 1);
              mma_tf32(d, alo, bhi, id, 1);
            }
            mma_commit(&empty[s]);  // stage reusable once these MMAs finish
            if (cg == TC_GROUP - 1 || c == nck - 1) {
              mma_commit(&accf[gg & 1]);  // group complete in its region
              ++gg;
            }
          }
        }
      }
    }
  } else if (warp >= 2 + TC_EPI_WARPS) {
    // ------------------------------------------------------------ split warps
    // A_lo = x - trunc_tf32(x) of each landed layer-0 X chunk (same swizzled
    // positions), off the epilogue warps so accumulator drains never hold
    // the MMAs back; they walk every chunk in order and arrive on lready[s]
    // for each (layer >= 1 chunks: nothing to split), which keeps the
    // mbarrier phases of full/lready in lock step with the MMA issuer.
    const int sw = warp - 2 - TC_EPI_WARPS;
    uint32_t g = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      for (int l = 0; l < NH; ++l) {
        const int nck = p.kin[l] >> 4;
        for (int c = 0; c < nck; ++c, ++g) {
          const int s = (int)(g % S);
          mbar_wait(&full[s], (g / S) & 1);
          if (l == 0) {
            unsigned char* st = smem + s * SB;
            const float4* a = (const float4*)st;
            float4* lo = (float4*)(st + 8192);
#pragma unroll
            for (int i = sw * 32 + lane; i < 512; i += 32 * TC_SPLIT_WARPS) {
              const float4 x = a[i];
              lo[i] = make_float4(tf32_lo(x.x), tf32_lo(x.y), tf32_lo(x.z), tf32_lo(x.w));
            }
            fence_async_smem();
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&lready[s]);
        }
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue warps
    const int ew = warp - 2;               // 0 .. TC_EPI_WARPS-1
    const int h = ew >> 2;                 // column part owned by this warp
    const int q = warp & 3;                // TMEM lane quadrant this warp may access
    const int r = q * 32 + lane;           // tile row = example of this thread
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
    uint32_t g = 0, dg = 0;                // chunk counter, drained-group counter
    HalfRow acc;
    int tl = 0;                            // local tile counter (exchange buffer parity)
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++tl) {
      int nn_bad = 0;
      for (int l = 0; l < NH; ++l) {
        const int nck = p.kin[l] >> 4, N = p.nout[l];
        // this part's 16-column blocks [b0, b1) of layer l (parts may be empty
        // when N < 64) and of the previous layer (ownership of its A chunks)
        const int b0 = part_blk(h, N), hc = (part_blk(h + 1, N) - b0) * 16;
        const int ngr = (nck + TC_GROUP - 1) / TC_GROUP;
        const int pb0 = l > 0 ? part_blk(h, p.nout[l - 1]) : 0;
        const int pb1 = l > 0 ? part_blk(h + 1, p.nout[l - 1]) : 0;
        for (int gi = 0; gi < ngr; ++gi) {
          const int cend = min(nck, (gi + 1) * TC_GROUP);
          for (int c = gi * TC_GROUP; c < cend; ++c, ++g) {
            if (l == 0) continue;  // layer 0's A (hi: TMA, lo: split warps)
            const int s = (int)(g % S);
            mbar_wait(&full[s], (g / S) & 1);  // stage free again (W landed)
            unsigned char* st = smem + s * SB;
            if (c >= pb0 && c < pb1) {  // this part holds the chunk's 16 columns
              const int cbl = c - pb0;
#pragma unroll
              for (int cb = 0; cb < TC_PART_MAX / 16; ++cb) {
                if (cb == cbl) {
#pragma unroll
                  for (int kq = 0; kq < 4; ++kq) {
                    const float* a4 = acc.v + cb * 16 + kq * 4;
                    const int off = ((kq * 16 + (r >> 3)) * 128) + (r & 7) * 16;
                    *(float4*)(st + off) = make_float4(a4[0], a4[1], a4[2], a4[3]);
                    *(float4*)(st + 8192 + off) =
                        make_float4(tf32_lo(a4[0]), tf32_lo(a4[1]), tf32_lo(a4[2]), tf32_lo(a4[3]));
                  }
                }
              }
            }
            fence_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&aready[s]);
          }
          if (gi > 0)  // one group behind the MMAs
            epi_drain(acc, accf, tempty, dg, lane_base, RS, b0 * 16, hc >> 4, gi == 1, lane);
        }
        epi_drain(acc, accf, tempty, dg, lane_base, RS, b0 * 16, hc >> 4, ngr == 1, lane);
        // acc = this part's pre-activations of layer l: + bias, ReLU (M:368-370)
        const float* __restrict__ bl = p.bias[l] + b0 * 16;
#pragma unroll
        for (int cb = 0; cb < TC_PART_MAX / 16; ++cb) {
          if (cb < (hc >> 4)) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const float z = acc.v[cb * 16 + j] + __ldg(bl + cb * 16 + j);
              nn_bad |= !isfinite(z);
              acc.v[cb * 16 + j] = relu_nan(z);
            }
          }
        }
      }
      // ---- output layer (M:372-373): the parts' partial dots meet in shared memory
      const int lb0 = part_blk(h, p.nout[NH - 1]);
      const int hcl = (part_blk(h + 1, p.nout[NH - 1]) - lb0) * 16;
      const float* __restrict__ wo = p.w_out + lb0 * 16;
      float part = 0.f;
#pragma unroll
      for (int cb = 0; cb < TC_PART_MAX / 16; ++cb) {
        if (cb < (hcl >> 4)) {
#pragma unroll
          for (int j = 0; j < 16; ++j) part = fmaf(acc.v[cb * 16 + j], __ldg(wo + cb * 16 + j), part);
        }
      }
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
        const double nn = (double)acc_nn + (double)__ldg(p.b_out);
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

// W [K][N] f32 row-major (M:198-210) -> kin/16 chunks, each [hi N x 16][lo N x 16]
// in the K-major core-matrix layout the B descriptor expects (rows = outputs).
// hi = tf32 round-to-nearest of w, lo = w - hi (exact in f32).
__global__ void tc_prep_weights_kernel(const float* __restrict__ W, int K, int N, int Kp,
                                       float* __restrict__ dst) {
  const int64_t total = (int64_t)Kp * N;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(i / N), n = (int)(i - (int64_t)k * N);
    const float w = k < K ? W[(int64_t)k * N + n] : 0.f;
    uint32_t hb;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hb) : "f"(w));
    const float hi = __uint_as_float(hb);
    const int c = k >> 4, kk = k & 15;
    float* chunk = dst + (int64_t)c * N * 32;
    const int off = (((kk >> 2) * (N >> 3) + (n >> 3)) * 32) + (n & 7) * 4 + (kk & 3);
    chunk[off] = hi;
    chunk[N * 16 + off] = w - hi;
  }
}

int launch_tc_prep_weights(const float* W, int K, int N, int Kp, float* dst, cudaStream_t s) {
  const int64_t total = (int64_t)Kp * N;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 4096);
  note_launches(1), tc_prep_weights_kernel<<<blocks, 256, 0, s>>>(W, K, N, Kp, dst);
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
