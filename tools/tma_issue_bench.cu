// Microbenchmark: issue rate of 1-D TMA bulk row copies (768 B) from W producer
// warps into a shared-memory ring, vs row gathers with plain 256-bit loads.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_issue_bench tma_issue_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void tma_kernel(const float* table, const int* rows, int n_rows_per_warp, int nwarps,
                           int row_bytes, unsigned long long* cycles) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bar = (uint64_t*)smem;
  unsigned char* ring = smem + 1024;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x < nwarps) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar + threadIdx.x)));
  asm volatile("fence.mbarrier_init.release.cluster;");
  __syncthreads();
  if (warp >= nwarps) return;
  long long t0 = clock64();
  const int per_batch = 64;  // rows per barrier phase
  uint32_t phase = 0;
  for (int b0 = 0; b0 < n_rows_per_warp; b0 += per_batch) {
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar + warp)), "r"(per_batch * row_bytes));
    __syncwarp();
    for (int i = lane; i < per_batch; i += 32) {
      const int r = rows[(blockIdx.x * nwarps + warp) * n_rows_per_warp + b0 + i];
      unsigned char* dst = ring + (size_t)(warp * per_batch + i) * (row_bytes + 16);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(su32(dst)), "l"(table + (size_t)r * (row_bytes / 4)), "r"(row_bytes), "r"(su32(bar + warp)) : "memory");
    }
    asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W;}" ::"r"(su32(bar + warp)), "r"(phase));
    phase ^= 1;
  }
  long long t1 = clock64();
  if (lane == 0) atomicAdd(cycles, (unsigned long long)(t1 - t0));
}

__global__ void ldg_kernel(const float* table, const int* rows, int n_rows_per_warp, int nwarps,
                           int row_bytes, float* sink) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp >= nwarps) return;
  float acc = 0.f;
  const int n32 = row_bytes / 32;  // 256-bit chunks per row
  for (int i = 0; i < n_rows_per_warp; i += 4) {
    float4 v[4][2];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int r = rows[(blockIdx.x * nwarps + warp) * n_rows_per_warp + i + u];
      const float* p = table + (size_t)r * (row_bytes / 4) + (lane % n32) * 8;
      v[u][0] = __ldg((const float4*)p); v[u][1] = __ldg((const float4*)p + 1);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) acc += v[u][0].x + v[u][1].w;
  }
  if (acc == 12345.f) sink[0] = acc;
}

int main() {
  const int row_bytes = 768;
  const size_t n_table_rows = 1 << 24;
  float* table;
  cudaMalloc(&table, n_table_rows * row_bytes);
  cudaMemset(table, 0, n_table_rows * row_bytes);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int n_per_warp = 4096;
  for (int nw : {1, 2, 4, 8}) {
    size_t nrows = (size_t)sms * nw * n_per_warp;
    int* rows_h = new int[nrows];
    uint64_t x = 88172645463325252ull;
    for (size_t i = 0; i < nrows; ++i) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; rows_h[i] = (int)(x % n_table_rows); }
    int* rows;
    cudaMalloc(&rows, nrows * 4);
    cudaMemcpy(rows, rows_h, nrows * 4, cudaMemcpyHostToDevice);
    unsigned long long* cyc;
    cudaMalloc(&cyc, 8);
    int smem = 1024 + nw * 64 * (row_bytes + 16);
    cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(cyc, 0, 8);
      cudaEventRecord(a);
      tma_kernel<<<sms, nw * 32, smem>>>(table, rows, n_per_warp, nw, row_bytes, cyc);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
    }
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("TMA  warps/SM=%d: %.3f ms, %.1f Mrows/s chip, %.1f GB/s, err=%s\n", nw, ms, nrows / ms / 1e3,
           nrows * row_bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      ldg_kernel<<<sms, nw * 32>>>(table, rows, n_per_warp, nw, row_bytes, (float*)cyc);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
    }
    cudaEventElapsedTime(&ms, a, b);
    printf("LDG  warps/SM=%d: %.3f ms, %.1f Mrows/s chip, %.1f GB/s\n", nw, ms, nrows / ms / 1e3, nrows * row_bytes / ms / 1e6);
    cudaFree(rows); cudaFree(cyc); delete[] rows_h;
  }
  return 0;
}
