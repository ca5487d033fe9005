// Accuracy of the tcgen05 kind::tf32 3xTF32 GEMM at MLP layer-0 scale:
// D[128 x 256] = X[128 x K] . W[K x 256], X ~ N(0,1) (standardised MergeNorm
// rows), W ~ N(0, 0.05), K = 784.  Accumulation split over NACC TMEM
// accumulators (chunk c -> accumulator c % NACC), summed on CUDA cores.
// Reports max |err| / rms(ref) against a host f64 GEMM.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cmath>
#include <random>
#include <vector>
#include <cuda_runtime.h>

constexpr int M = 128, N = 128, K = 784;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ int blk_off(int r, int k, int R) {
  return ((k >> 2) * (R >> 3) + (r >> 3)) * 128 + (r & 7) * 16 + (k & 3) * 4;
}
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r; asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x)); return __uint_as_float(r);
}

// one CTA, K in chunks of 16 staged through smem one at a time (simple, not fast)
__global__ void gemm(const float* A, const float* B, float* D, int nacc, int passes) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* ah = sm; unsigned char* al = ah + M * 16 * 4;
  unsigned char* bh = al + M * 16 * 4; unsigned char* bl = bh + N * 16 * 4;
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(&tmem_base)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&mbar)));
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  const uint32_t id = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
  uint32_t phase = 0;
  for (int c = 0; c < K / 16; ++c) {
    for (int t = tid; t < M * 16; t += blockDim.x) {
      const int r = t / 16, k = t % 16;
      const float x = A[r * K + c * 16 + k];
      *(float*)(ah + blk_off(r, k, M)) = x;
      *(float*)(al + blk_off(r, k, M)) = x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
    }
    for (int t = tid; t < N * 16; t += blockDim.x) {
      const int r = t / 16, k = t % 16;
      const float x = B[r * K + c * 16 + k], h = tf32_rna(x);
      *(float*)(bh + blk_off(r, k, N)) = h;
      *(float*)(bl + blk_off(r, k, N)) = x - h;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (tid == 0) {
      const int a = c % nacc;
      const uint32_t d = tmem + a * N;
      for (int ks = 0; ks < 2; ++ks) {
        const uint64_t dah = sdesc(smem_u32(ah) + ks * 4096, 2048, 128), dal = sdesc(smem_u32(al) + ks * 4096, 2048, 128);
        const uint64_t dbh = sdesc(smem_u32(bh) + ks * 2 * (N / 8) * 128, (N / 8) * 128, 128);
        const uint64_t dbl = sdesc(smem_u32(bl) + ks * 2 * (N / 8) * 128, (N / 8) * 128, 128);
        const uint32_t first = (c < nacc && ks == 0) ? 0 : 1;
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
                     :: "r"(d), "l"(dah), "l"(dbh), "r"(id), "r"(first));
        if (passes > 1) {
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
                       :: "r"(d), "l"(dah), "l"(dbl), "r"(id), "r"(1));
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
                       :: "r"(d), "l"(dal), "l"(dbh), "r"(id), "r"(1));
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&mbar)) : "memory");
    }
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n" : "=r"(done) : "r"(smem_u32(&mbar)), "r"(phase));
    phase ^= 1;
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    __syncthreads();
  }
  if (warp < 4) {
    const int row = warp * 32 + (tid & 31);
    for (int c0 = 0; c0 < N; c0 += 8) {
      float s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      for (int a = 0; a < nacc; ++a) {
        uint32_t v[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                     : "r"(tmem + ((uint32_t)(warp * 32) << 16) + a * N + c0));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int j = 0; j < 8; ++j) s[j] += __uint_as_float(v[j]);
      }
      for (int j = 0; j < 8; ++j) D[row * N + c0 + j] = s[j];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(512));
}

int main() {
  std::mt19937 g(7);
  std::normal_distribution<float> nx(0.f, 1.f), nw(0.f, 0.05f);
  std::vector<float> A(M * K), B(N * K), D(M * N);
  for (auto& x : A) x = nx(g);
  for (auto& x : B) x = nw(g);
  std::vector<double> ref(M * N);
  double rms = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += (double)A[i * K + k] * B[j * K + k];
      ref[i * N + j] = s; rms += s * s;
    }
  rms = sqrt(rms / (M * N));
  // f32 sequential reference error for scale
  double f32err = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      float s = 0;
      for (int k = 0; k < K; ++k) s = fmaf(A[i * K + k], B[j * K + k], s);
      f32err = fmax(f32err, fabs(s - ref[i * N + j]));
    }
  printf("rms(ref)=%.4f  fp32-FMA sequential max err/rms = %.3e\n", rms, f32err / rms);
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  const int smem = 2 * (M + N) * 16 * 4 + 1024;
  cudaFuncSetAttribute(gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int passes : {1, 3})
    for (int nacc : {1, 2, 4}) {
      gemm<<<1, 128, smem>>>(dA, dB, dD, nacc, passes);
      if (cudaDeviceSynchronize() != cudaSuccess) { printf("err\n"); return 1; }
      cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
      double mx = 0, mean = 0;
      for (int i = 0; i < M * N; ++i) { const double e = D[i] - ref[i]; mx = fmax(mx, fabs(e)); mean += e; }
      printf("passes=%d nacc=%d  max err/rms = %.3e  mean err/rms = %.3e\n", passes, nacc, mx / rms, mean / (M * N) / rms);
    }
  return 0;
}
