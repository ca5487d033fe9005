// Microbenchmark: useful-byte bandwidth of random gathers from a 12.9 GB table
// of 768 B rows: (a) scattered 32 B segments (each lane its own random row) vs
// (b) row-coalesced (lanes 0..23 read one row's 24 segments), U loads in flight.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_bench gather_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void ld32(const void* p, uint4& a, uint4& b) {
  asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z),
                 "=r"(b.w)
               : "l"(p));
}
__device__ __forceinline__ uint32_t hsh(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16;
  return x;
}

template <int U, bool COAL>
__global__ void __launch_bounds__(512) gather(const unsigned char* table, uint32_t nrows,
                                              int iters, uint32_t* sink) {
  const int lane = threadIdx.x & 31;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
    uint4 a[U], b[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint32_t row, seg;
      if (COAL) {
        row = hsh(gw * 7919u + it * 131u + u) % nrows;
        seg = lane % 24;
      } else {
        row = hsh((gw * 32 + lane) * 7919u + it * 131u + u) % nrows;
        seg = hsh(lane + it) % 24;
      }
      ld32(table + (size_t)row * 768 + seg * 32, a[u], b[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc += a[u].x ^ b[u].w;
  }
  if (acc == 0x12345) sink[0] = acc;
}

template <typename Kern>
void run(Kern kern, const char* name, int threads, int bps, int U, bool coal,
         const unsigned char* table, uint32_t nrows, uint32_t* sink, int sms) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 64, blocks = sms * bps;
  float ms = 0;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a);
    kern<<<blocks, threads>>>(table, nrows, iters, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
  }
  cudaEventElapsedTime(&ms, a, b);
  double useful = (double)blocks * threads * iters * U * 32.0;
  if (coal) useful *= 24.0 / 32.0;
  printf("%-10s U=%d %dthr x %d/SM: %.3f ms %6.0f GB/s useful (%s)\n", name, U, threads, bps, ms,
         useful / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const size_t nrows = 1u << 24;
  unsigned char* table;
  cudaMalloc(&table, nrows * 768);
  cudaMemset(table, 1, nrows * 768);
  uint32_t* sink;
  cudaMalloc(&sink, 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run(gather<2, false>, "scattered", 512, 2, 2, false, table, nrows, sink, sms);
  run(gather<6, false>, "scattered", 512, 2, 6, false, table, nrows, sink, sms);
  run(gather<6, false>, "scattered", 256, 3, 6, false, table, nrows, sink, sms);
  run(gather<2, true>, "coalesced", 512, 2, 2, true, table, nrows, sink, sms);
  run(gather<6, true>, "coalesced", 512, 2, 6, true, table, nrows, sink, sms);
  run(gather<6, true>, "coalesced", 256, 3, 6, true, table, nrows, sink, sms);
  return 0;
}
