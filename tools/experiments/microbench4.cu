// is it the code or the buffers? (design experiment)
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
__global__ void fill(long n, double* p, double v) { long i = (long)blockIdx.x * blockDim.x + threadIdx.x; if (i < n) p[i] = v * (1 + (i % 7)); }
int main(int argc, char** argv) {
  const long n = 35587930, n2 = n / 2;
  long per = 2 * n;
  double* buf[5];
  for (int k = 0; k < 5; ++k) { CK(cudaMalloc(&buf[k], per * sizeof(double))); CK(cudaMemset(buf[k], 0, per * 8)); }
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  auto timeit = [&](auto f, int reps) { f(); cudaEventRecord(a); for (int r = 0; r < reps; ++r) f(); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b); return ms / reps; };
  auto D2 = [&](int k) { return (double2*)buf[k]; };
  for (int pass = 0; pass < 2; ++pass) {
    if (pass == 1) { for (int k = 0; k < 5; ++k) fill<<<(per + 255) / 256, 256>>>(per, buf[k], 0.1 + k); CK(cudaDeviceSynchronize()); printf("nonzero data:\n"); }
    float t1 = timeit([&] { cheb2u<1><<<(n2 + 255) / 256, 256>>>(n2, D2(0), D2(1), D2(2), D2(3), D2(4), .5, .3); }, 50);
    float t2 = timeit([&] { cheb2<<<(n2 + 255) / 256, 256>>>(n2, D2(0), D2(1), D2(2), D2(3), D2(4), .5, .3); }, 50);
    printf("cheb2u<1> %.3f ms (%.0f GB/s)   cheb2 %.3f ms (%.0f GB/s)\n", t1, 64.0 * n / t1 / 1e6, t2, 64.0 * n / t2 / 1e6);
  }
  return 0;
}
