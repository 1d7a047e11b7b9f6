// Microbenchmark: do 64-bit warp shuffles share the L1/shared-memory data pipe
// with LDS.64 on sm_100a?  Times LDS-only, SHFL-only and interleaved loops.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/microbench9.cu -o tools/microbench9
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>   // 0 lds, 1 shfl, 2 both
__global__ void __launch_bounds__(256) k(int iters, double* out) {
  __shared__ double s[8][64];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  s[w][lane] = lane;
  s[w][lane + 32] = -lane;
  __syncwarp();
  double a = lane, b = 0;
  int idx = lane;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (MODE != 1) { b += s[w][(idx + u) & 63]; }
      if (MODE != 0) { a = __shfl_sync(0xffffffffu, a, (lane + u + 1) & 31) + 1.0; }
    }
    idx = (idx + 3) & 63;
  }
  if (a + b == 12345.0) out[0] = a + b;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int blocks = 148 * 8, iters = 4096;
  const char* names[3] = {"LDS.64", "SHFL f64", "LDS.64 + SHFL f64"};
  for (int m = 0; m < 3; ++m) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (m == 0) k<0><<<blocks, 256>>>(iters, out);
      if (m == 1) k<1><<<blocks, 256>>>(iters, out);
      if (m == 2) k<2><<<blocks, 256>>>(iters, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double warp_ops = (double)blocks * 8 * iters * 8;   // per op kind
      if (rep) printf("%-20s %8.3f ms  %.3f warp-ops/clk/SM (at %d MHz nominal)\n", names[m], ms,
                      warp_ops / 148 / (ms * 1e-3 * clk * 1e3), clk / 1000);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
