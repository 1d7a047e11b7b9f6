// address-offset sensitivity of a 5-read/3-write streaming kernel (design experiment)
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
__global__ void cheb2(long n2, const double2* __restrict__ g, const double2* __restrict__ Dinv, double2* __restrict__ t,
                      double2* __restrict__ dv, double2* __restrict__ x, double c1, double c2) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n2) return;
  double2 G = g[i], T = t[i], D = Dinv[i], V = dv[i], X = x[i];
  double2 d;
  d.x = fma(c1, V.x, c2 * D.x * (G.x - T.x));
  d.y = fma(c1, V.y, c2 * D.y * (G.y - T.y));
  t[i] = make_double2(0, 0); dv[i] = d; x[i] = make_double2(X.x + d.x, X.y + d.y);
}
__global__ void cheb1(long n, const double* __restrict__ g, const double* __restrict__ Dinv, double* __restrict__ t,
                      double* __restrict__ dv, double* __restrict__ x, double c1, double c2) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double r = g[i] - t[i];
  t[i] = 0.0;
  double d = fma(c1, dv[i], c2 * Dinv[i] * r);
  dv[i] = d;
  x[i] = x[i] + d;
}
int main() {
  const long n = 35587930, n2 = n / 2;
  const long cap = (1L << 30) / 8 * 2;  // 2 GB per buffer
  double* buf[5];
  for (int k = 0; k < 5; ++k) { CK(cudaMalloc(&buf[k], cap * sizeof(double))); CK(cudaMemset(buf[k], 0, cap * 8)); }
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  auto timeit = [&](auto f, int reps) { f(); cudaEventRecord(a); for (int r = 0; r < reps; ++r) f(); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b); return ms / reps; };
  long offs_mb[] = {0, 2, 32, 64, 128, 182, 256, 384, 512, 1024};
  for (long omb : offs_mb) {
    long o = omb * (1L << 20) / 8;
    double* p[5]; for (int k = 0; k < 5; ++k) p[k] = buf[k] + o;
    float t2 = timeit([&] { cheb2<<<(n2 + 255) / 256, 256>>>(n2, (double2*)p[0], (double2*)p[1], (double2*)p[2], (double2*)p[3], (double2*)p[4], .5, .3); }, 50);
    float t1 = timeit([&] { cheb1<<<(n + 255) / 256, 256>>>(n, p[0], p[1], p[2], p[3], p[4], .5, .3); }, 50);
    // staggered bases: each array at a different offset
    double* q[5]; for (int k = 0; k < 5; ++k) q[k] = buf[k] + o + k * (long)(3 << 20) / 8;
    float t3 = timeit([&] { cheb1<<<(n + 255) / 256, 256>>>(n, q[0], q[1], q[2], q[3], q[4], .5, .3); }, 50);
    printf("offset %5ld MB: double2 %.3f ms (%.0f GB/s)  double %.3f ms (%.0f GB/s)  staggered %.3f ms (%.0f GB/s)\n", omb, t2, 64.0 * n / t2 / 1e6, t1, 64.0 * n / t1 / 1e6, t3, 64.0 * n / t3 / 1e6);
  }
  // single buffer, arrays packed back to back (MG-layout like)
  {
    double* big; CK(cudaMalloc(&big, 5 * n * sizeof(double) + 4096)); CK(cudaMemset(big, 0, 5 * n * 8));
    float t1 = timeit([&] { cheb1<<<(n + 255) / 256, 256>>>(n, big, big + n, big + 2 * n, big + 3 * n, big + 4 * n, .5, .3); }, 50);
    printf("packed single buffer (unaligned n): double %.3f ms (%.0f GB/s)\n", t1, 64.0 * n / t1 / 1e6);
  }
  CK(cudaDeviceSynchronize());
  return 0;
}
