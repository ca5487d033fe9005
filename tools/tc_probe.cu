// tcgen05 kind::tf32 probe: one CTA computes D[128 x N] = A[128 x K] . B[N x K]^T
// (both K-major, no swizzle, core-matrix blocked) with the 3xTF32 split
// (hi*hi + hi*lo + lo*hi), reads D back from TMEM and compares with a host f64
// GEMM.  Validates the shared-memory / instruction descriptor encodings used by
// csrc/mlp_tc.cu.   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tc_probe tools/tc_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include <cuda.h>
#include <cudaTypedefs.h>

constexpr int M = 128, N = 256, K = 64;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
// blocked K-major layout of a [R x K] operand, K-chunks of 4 elements (16 B):
// byte offset of (r, k) = ((k/4) * (R/8) + r/8) * 128 + (r%8) * 16 + (k%4) * 4
__device__ __forceinline__ int blk_off(int r, int k, int R) {
  return ((k >> 2) * (R >> 3) + (r >> 3)) * 128 + (r & 7) * 16 + (k & 3) * 4;
}
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (sm_100)
  return d;                // base_offset 0, lbo_mode 0, layout SWIZZLE_NONE (0)
}
__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n) {
  return (1u << 4)            // D f32
       | (2u << 7)            // A tf32
       | (2u << 10)           // B tf32
       | ((uint32_t)(n >> 3) << 17)
       | ((uint32_t)(m >> 4) << 24);
}
__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__global__ void probe(const float* A, const float* B, float* D, int split) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* ah = sm;                 // M*K*4
  unsigned char* al = ah + M * K * 4;
  unsigned char* bh = al + M * K * 4;     // N*K*4
  unsigned char* bl = bh + N * K * 4;
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int t = tid; t < M * K; t += blockDim.x) {
    const int r = t / K, k = t % K;
    const float x = A[t], h = split == 2 ? __uint_as_float(__float_as_uint(x) & 0xFFFFE000u)
                                         : tf32_rna(x), l = x - h;
    *(float*)(ah + blk_off(r, k, M)) = split == 1 ? h : x;
    *(float*)(al + blk_off(r, k, M)) = l;
  }
  for (int t = tid; t < N * K; t += blockDim.x) {
    const int r = t / K, k = t % K;
    const float x = B[t], h = split == 2 ? __uint_as_float(__float_as_uint(x) & 0xFFFFE000u)
                                         : tf32_rna(x), l = x - h;
    *(float*)(bh + blk_off(r, k, N)) = split == 1 ? h : x;
    *(float*)(bl + blk_off(r, k, N)) = l;
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(smem_u32(&tmem_base)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&mbar)));
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    const uint32_t id = idesc_tf32(M, N);
    const uint32_t lboA = (M / 8) * 128, lboB = (N / 8) * 128, sbo = 128;
    int first = 1;
    for (int ks = 0; ks < K / 8; ++ks) {
      const uint32_t koffA = ks * 2 * lboA, koffB = ks * 2 * lboB;
      const int npass = split ? 3 : 1;
      for (int ps = 0; ps < npass; ++ps) {
        const unsigned char* a = (ps == 2) ? al : ah;
        const unsigned char* b = (ps == 1) ? bl : bh;
        const uint64_t da = sdesc(smem_u32(a) + koffA, lboA, sbo);
        const uint64_t db = sdesc(smem_u32(b) + koffB, lboB, sbo);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
            :: "r"(tmem), "l"(da), "l"(db), "r"(id), "r"(first ? 0 : 1));
        first = 0;
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                 :: "r"(smem_u32(&mbar)) : "memory");
  }
  // wait for the MMAs (phase 0)
  {
    uint32_t done = 0;
    while (!done) {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                   "selp.u32 %0, 1, 0, p;\n\t}\n"
                   : "=r"(done) : "r"(smem_u32(&mbar)), "r"(0));
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp < 4) {
    const int row = warp * 32 + (tid & 31);
    for (int c0 = 0; c0 < N; c0 += 8) {
      uint32_t v[8];
      const uint32_t addr = tmem + ((uint32_t)(warp * 32) << 16) + c0;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                     "=r"(v[6]), "=r"(v[7]) : "r"(addr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int j = 0; j < 8; ++j) D[row * N + c0 + j] = __uint_as_float(v[j]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(256));
}


// Variant: A arrives by 2-D TMA (box 16 f32 x 128 rows, 64-byte swizzle), one
// 16-wide K chunk at a time; lo = x - trunc_tf32(x) is computed elementwise in
// the same swizzled positions; A descriptors use SWIZZLE_64B (layout 4,
// SBO = 8 rows * 64 B, K-step = +32 B inside the atom).
__global__ void probe_tma(const __grid_constant__ CUtensorMap tmA, const float* B, float* D) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* ah = sm;                       // K/16 chunks x 8 KB
  unsigned char* al = ah + M * K * 4;
  unsigned char* bh = al + M * K * 4;
  unsigned char* bl = bh + N * K * 4;
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar, tbar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int t = tid; t < N * K; t += blockDim.x) {
    const int r = t / K, k = t % K;
    const float x = B[t], h = tf32_rna(x), l = x - h;
    *(float*)(bh + blk_off(r, k, N)) = h;
    *(float*)(bl + blk_off(r, k, N)) = l;
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(smem_u32(&tmem_base)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&mbar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&tbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                 :: "r"(smem_u32(&tbar)), "r"(M * K * 4) : "memory");
    for (int c = 0; c < K / 16; ++c)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3}], [%4];"
          :: "r"(smem_u32(ah + c * 8192)), "l"(&tmA), "r"(c * 16), "r"(0),
             "r"(smem_u32(&tbar)) : "memory");
  }
  {
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                   "selp.u32 %0, 1, 0, p;\n\t}\n" : "=r"(done) : "r"(smem_u32(&tbar)), "r"(0));
  }
  for (int t = tid; t < M * K; t += blockDim.x) {
    const float x = ((const float*)ah)[t];
    ((float*)al)[t] = x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    const uint32_t id = idesc_tf32(M, N);
    const uint32_t lboB = (N / 8) * 128, sbo = 128;
    int first = 1;
    for (int ks = 0; ks < K / 8; ++ks) {
      const int c = ks >> 1, h = ks & 1;
      for (int ps = 0; ps < 3; ++ps) {
        const unsigned char* a = ((ps == 2) ? al : ah) + c * 8192 + h * 32;
        const unsigned char* b = (ps == 1) ? bl : bh;
        uint64_t da = sdesc(smem_u32(a), 16, 512);
        da |= (uint64_t)4 << 61;  // SWIZZLE_64B
        const uint64_t db = sdesc(smem_u32(b) + ks * 2 * lboB, lboB, sbo);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
            :: "r"(tmem), "l"(da), "l"(db), "r"(id), "r"(first ? 0 : 1));
        first = 0;
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                 :: "r"(smem_u32(&mbar)) : "memory");
  }
  {
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                   "selp.u32 %0, 1, 0, p;\n\t}\n" : "=r"(done) : "r"(smem_u32(&mbar)), "r"(0));
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp < 4) {
    const int row = warp * 32 + (tid & 31);
    for (int c0 = 0; c0 < N; c0 += 8) {
      uint32_t v[8];
      const uint32_t addr = tmem + ((uint32_t)(warp * 32) << 16) + c0;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                     "=r"(v[6]), "=r"(v[7]) : "r"(addr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int j = 0; j < 8; ++j) D[row * N + c0 + j] = __uint_as_float(v[j]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(256));
}

static void check(const std::vector<float>& A, const std::vector<float>& B,
                  const std::vector<float>& D, const char* what) {
  double maxerr = 0, maxref = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += (double)A[i * K + k] * B[j * K + k];
      maxerr = fmax(maxerr, fabs(s - D[i * N + j]));
      maxref = fmax(maxref, fabs(s));
    }
  printf("%s max|err|=%.3e rel=%.3e\n", what, maxerr, maxerr / maxref);
}

int main() {
  std::vector<float> A(M * K), B(N * K), D(M * N);
  srand(1);
  for (auto& x : A) x = (float)rand() / RAND_MAX * 2.f - 1.f;
  for (auto& x : B) x = (float)rand() / RAND_MAX * 2.f - 1.f;
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  const int smem = 2 * (M + N) * K * 4;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int split = 0; split < 3; ++split) {
    cudaMemset(dD, 0, D.size() * 4);
    probe<<<1, 128, smem>>>(dA, dB, dD, split);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxref = 0;
    for (int i = 0; i < M; ++i)
      for (int j = 0; j < N; ++j) {
        double s = 0;
        for (int k = 0; k < K; ++k) s += (double)A[i * K + k] * B[j * K + k];
        maxerr = fmax(maxerr, fabs(s - D[i * N + j]));
        maxref = fmax(maxref, fabs(s));
      }
    printf("split=%d max|err|=%.3e max|ref|=%.3e rel=%.3e  D[0]=%f D[1,2]=%f\n", split, maxerr,
           maxref, maxerr / maxref, D[0], D[1 * N + 2]);
  }
  {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult qr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr);
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)M};
    cuuint64_t strides[1] = {(cuuint64_t)K * 4};
    cuuint32_t box[2] = {16, 128};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = ((PFN_cuTensorMapEncodeTiled_v12000)fn)(
        &tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dA, dims, strides, box, estr,
        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode rc=%d\n", (int)r);
    cudaFuncSetAttribute(probe_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaMemset(dD, 0, D.size() * 4);
    probe_tma<<<1, 128, smem>>>(tm, dB, dD);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    check(A, B, D, "tma-sw64");
  }
  return 0;
}
