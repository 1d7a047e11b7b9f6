// Microbenchmark: FP64 FMA throughput of one B200 (the FP64 peak SURVEY 8(d)
// asks for; MEASURED_PEAKS.json has none).  8 independent DFMA chains per
// thread, 148 x 8 blocks of 256 threads.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/microbench10.cu -o tools/microbench10
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) dfma_loop(int iters, double a, double b, double* out) {
  double x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = threadIdx.x + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = fma(x[j], a, b);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += x[j];
  if (s == 1.2345) out[0] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int blocks = sms * 8, threads = 256, iters = 1 << 16;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    dfma_loop<<<blocks, threads>>>(iters, 0.999999, 1e-7, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 8 * iters * (double)blocks * threads;
    if (rep) printf("DFMA: %.2f TFLOP/s fp64 (%d SMs, %.3f ms; %.1f DFMA/clk/SM at the %d MHz nominal clock)\n",
                    flops / (ms * 1e-3) / 1e12, sms, ms, flops / 2 / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
