// FP64 latency / throughput on one SM (K2 is a chain of f64 phases): cycles per dependent
// DFMA for one warp, and per warp-instruction with 1..32 warps issuing independent chains;
// the same for the correctly rounded division and square root K2's Adagrad step uses.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_bench tools/fp64_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(double* out, long long* cyc, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-3 + 1.0, x1 = x0 + 0.5, x2 = x0 + 0.25, x3 = x0 + 0.125;
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (OP == 0) { x0 = fma(x0, a, b); }  // dependent chain
    if (OP == 1) { x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b); }
    if (OP == 2) { x0 = __ddiv_rn(a, x0) + b; }
    if (OP == 3) { x0 = __dsqrt_rn(x0) + b; }
    if (OP == 4) { x0 = __ddiv_rn(1.0, __dsqrt_rn(x0)) + b; x1 = __ddiv_rn(1.0, __dsqrt_rn(x1)) + b; }
    if (OP == 5) { x0 = (double)((float)x0) * a + b; }  // F2F round trip + DFMA
  }
  const long long t1 = clock64();
  __syncthreads();
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * 8);
  cudaMalloc(&cyc, 8);
  const char* names[] = {"DFMA dependent", "DFMA x4 independent", "ddiv_rn dependent", "dsqrt_rn dependent",
                         "1/sqrt (div+sqrt) x2 indep", "F2F.F32<->F64 + DFMA"};
  const int per[] = {1, 4, 1, 1, 2, 1};
  const int iters = 2000;
  for (int op = 0; op < 6; ++op)
    for (int warps : {1, 4, 8, 16, 32}) {
      for (int rep = 0; rep < 2; ++rep) {
        switch (op) {
          case 0: k<0><<<1, warps * 32>>>(out, cyc, iters, 1.0000001, 1e-9); break;
          case 1: k<1><<<1, warps * 32>>>(out, cyc, iters, 1.0000001, 1e-9); break;
          case 2: k<2><<<1, warps * 32>>>(out, cyc, iters, 1.0000001, 1e-9); break;
          case 3: k<3><<<1, warps * 32>>>(out, cyc, iters, 1.0000001, 1e-9); break;
          case 4: k<4><<<1, warps * 32>>>(out, cyc, iters, 1.0000001, 1e-9); break;
          case 5: k<5><<<1, warps * 32>>>(out, cyc, iters, 1.0000001, 1e-9); break;
        }
        cudaDeviceSynchronize();
      }
      long long c;
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      printf("%-30s warps %2d: %7.1f cycles per op per thread-chain, %6.2f cycles per warp-op on the SM\n",
             names[op], warps, (double)c / iters / per[op], (double)c / iters / per[op] / warps);
    }
  return 0;
}
