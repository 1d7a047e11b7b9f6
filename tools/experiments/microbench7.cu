// production cheb_step vs the fast microbench variant (design experiment)
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
template <bool READ_T, bool READ_DV, bool WRITE_DV, bool X_ZERO>
__global__ void __launch_bounds__(256) cheb_step(const double2* __restrict__ g, const double2* __restrict__ Dinv,
                                                    double2* __restrict__ t, double2* __restrict__ dv,
                                                    double2* __restrict__ x, double c1, double c2) {
  const long i = (long)blockIdx.x * 256 + threadIdx.x;
  const double2 G = g[i];
  double2 T = make_double2(0.0, 0.0), V = T, X = T;
  if (READ_T) T = t[i];
  const double2 Di = Dinv[i];
  if (READ_DV) V = dv[i];
  if (!X_ZERO) X = x[i];
  if (READ_T) t[i] = make_double2(0.0, 0.0);
  double dx = c2 * Di.x * (G.x - T.x), dy = c2 * Di.y * (G.y - T.y);
  if (READ_DV) { dx = fma(c1, V.x, dx); dy = fma(c1, V.y, dy); }
  if (WRITE_DV) dv[i] = make_double2(dx, dy);
  x[i] = make_double2(X.x + dx, X.y + dy);
}
__global__ void fill(long n, double* p, double v) { long i = (long)blockIdx.x * blockDim.x + threadIdx.x; if (i < n) p[i] = v * (1 + (i % 7)); }
int main() {
  const long n = 35588096, n2 = n / 2;   // multiple of 512
  double* buf[5];
  for (int k = 0; k < 5; ++k) { CK(cudaMalloc(&buf[k], n * sizeof(double))); fill<<<(n+255)/256,256>>>(n, buf[k], 0.1 + k); }
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  auto timeit = [&](auto f, int reps) { f(); cudaEventRecord(a); for (int r = 0; r < reps; ++r) f(); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b); return ms / reps; };
  auto D2 = [&](int k) { return (double2*)buf[k]; };
  for (int round = 0; round < 2; ++round) {
    float t1 = timeit([&] { cheb2u<1><<<(n2 + 255) / 256, 256>>>(n2, D2(0), D2(1), D2(2), D2(3), D2(4), .5, .3); }, 30);
    float t2 = timeit([&] { cheb_step<true, true, true, false><<<n / 512, 256>>>(D2(0), D2(1), D2(2), D2(3), D2(4), .5, .3); }, 30);
    float t3 = timeit([&] { cheb_step<false, false, true, true><<<n / 512, 256>>>(D2(0), D2(1), D2(2), D2(3), D2(4), .5, .3); }, 30);
    float t4 = timeit([&] { cheb2u<2><<<(n2 + 511) / 512, 256>>>(n2, D2(0), D2(1), D2(2), D2(3), D2(4), .5, .3); }, 30);
    printf("cheb2u<1> %.3f  prod<1,1,1,0> %.3f  prod<0,0,1,1> %.3f  cheb2u<2> %.3f ms\n", t1, t2, t3, t4);
  }
  return 0;
}
