// streaming-structure microbenchmark (design experiment, not product code)
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
template <int U>
__global__ void cheb2u(long n2, const double2* __restrict__ g, const double2* __restrict__ Dinv, double2* __restrict__ t,
                       double2* __restrict__ dv, double2* __restrict__ x, double c1, double c2) {
  long i0 = ((long)blockIdx.x * blockDim.x) * U + threadIdx.x;
  double2 G[U], T[U], D[U], V[U], X[U];
#pragma unroll
  for (int u = 0; u < U; ++u) { long i = i0 + u * blockDim.x; if (i < n2) { G[u] = g[i]; T[u] = t[i]; D[u] = Dinv[i]; V[u] = dv[i]; X[u] = x[i]; } }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    long i = i0 + u * blockDim.x;
    if (i >= n2) continue;
    double2 d;
    d.x = fma(c1, V[u].x, c2 * D[u].x * (G[u].x - T[u].x));
    d.y = fma(c1, V[u].y, c2 * D[u].y * (G[u].y - T[u].y));
    t[i] = make_double2(0, 0); dv[i] = d; x[i] = make_double2(X[u].x + d.x, X[u].y + d.y);
  }
}
__global__ void reads5(long n2, const double2* __restrict__ a, const double2* __restrict__ b, const double2* __restrict__ c,
                       const double2* __restrict__ d, const double2* __restrict__ e, double2* __restrict__ o) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n2) return;
  double2 A = a[i], B = b[i], C = c[i], D = d[i], E = e[i];
  o[i] = make_double2(A.x + B.x + C.x + D.x + E.x, A.y + B.y + C.y + D.y + E.y);
}
__global__ void rmw3(long n2, double2* __restrict__ a, double2* __restrict__ b, double2* __restrict__ c) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n2) return;
  double2 A = a[i], B = b[i], C = c[i];
  a[i] = make_double2(A.x + 1, A.y); b[i] = make_double2(B.x + C.x, B.y); c[i] = make_double2(0, 0);
}
// AoS: gd = (g, Dinv), xv = (x, dv), t separate
__global__ void cheb_aos(long n, const double2* __restrict__ gd, double2* __restrict__ xv, double* __restrict__ t, double c1, double c2) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double2 GD = gd[i], XV = xv[i]; double T = t[i];
  double d = fma(c1, XV.y, c2 * GD.y * (GD.x - T));
  t[i] = 0; xv[i] = make_double2(XV.x + d, d);
}
__global__ void copy2(long n2, const double2* __restrict__ a, double2* __restrict__ b) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n2) b[i] = a[i];
}
int main() {
  const long n = 35587930, n2 = n / 2;
  double* buf[8];
  for (int k = 0; k < 8; ++k) { CK(cudaMalloc(&buf[k], 2 * n * sizeof(double))); CK(cudaMemset(buf[k], 0, 2 * n * 8)); }
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  auto timeit = [&](auto f, int reps) { f(); cudaEventRecord(a); for (int r = 0; r < reps; ++r) f(); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b); return ms / reps; };
  auto D2 = [&](int k) { return (double2*)buf[k]; };
  float t;
  for (int round = 0; round < 3; ++round) {
  printf("round %d\n", round);
  t = timeit([&] { copy2<<<(n2 + 255) / 256, 256>>>(n2, D2(0), D2(1)); }, 100); printf("copy2 %.3f ms %.0f GB/s\n", t, 16.0 * n / t / 1e6);
  t = timeit([&] { copy2<<<(n + 255) / 256, 256>>>(n, D2(0), D2(1)); }, 100); printf("copy2 2x %.3f ms %.0f GB/s\n", t, 32.0 * n / t / 1e6);
  t = timeit([&] { cheb2u<1><<<(n2 + 255) / 256, 256>>>(n2, D2(0), D2(1), D2(2), D2(3), D2(4), .5, .3); }, 100); printf("cheb2u1 %.3f ms %.0f GB/s\n", t, 64.0 * n / t / 1e6);
  t = timeit([&] { cheb2u<2><<<(n2 + 511) / 512, 256>>>(n2, D2(0), D2(1), D2(2), D2(3), D2(4), .5, .3); }, 100); printf("cheb2u2 %.3f ms %.0f GB/s\n", t, 64.0 * n / t / 1e6);
  t = timeit([&] { cheb2u<4><<<(n2 + 1023) / 1024, 256>>>(n2, D2(0), D2(1), D2(2), D2(3), D2(4), .5, .3); }, 100); printf("cheb2u4 %.3f ms %.0f GB/s\n", t, 64.0 * n / t / 1e6);
  t = timeit([&] { cheb2u<2><<<(n2 + 255) / 256, 128>>>(n2, D2(0), D2(1), D2(2), D2(3), D2(4), .5, .3); }, 100); printf("cheb2u2b128 %.3f ms %.0f GB/s\n", t, 64.0 * n / t / 1e6);
  t = timeit([&] { reads5<<<(n2 + 255) / 256, 256>>>(n2, D2(0), D2(1), D2(2), D2(3), D2(4), D2(5)); }, 100); printf("reads5+w1 %.3f ms %.0f GB/s\n", t, 48.0 * n / t / 1e6);
  t = timeit([&] { rmw3<<<(n2 + 255) / 256, 256>>>(n2, D2(0), D2(1), D2(2)); }, 100); printf("rmw3 %.3f ms %.0f GB/s\n", t, 48.0 * n / t / 1e6);
  t = timeit([&] { cheb_aos<<<(n + 255) / 256, 256>>>(n, D2(0), D2(1), buf[2], .5, .3); }, 100); printf("cheb_aos %.3f ms %.0f GB/s\n", t, 56.0 * n / t / 1e6);
  }
  CK(cudaDeviceSynchronize());
  return 0;
}
