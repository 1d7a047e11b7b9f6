// store-after-load to the same address: hoisted zero store vs data-dependent store (design experiment)
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
template <bool DEP>
__global__ void __launch_bounds__(256) cheb_step(const double2* __restrict__ g, const double2* __restrict__ Dinv,
                                                    double2* __restrict__ t, double2* __restrict__ dv,
                                                    double2* __restrict__ x, double c1, double c2) {
  const long i = (long)blockIdx.x * 256 + threadIdx.x;
  const double2 G = g[i];
  double2 T = t[i];
  const double2 Di = Dinv[i];
  double2 V = dv[i], X = x[i];
  if (DEP) t[i] = make_double2(T.x - T.x, T.y - T.y);
  else t[i] = make_double2(0.0, 0.0);
  double dx = c2 * Di.x * (G.x - T.x), dy = c2 * Di.y * (G.y - T.y);
  dx = fma(c1, V.x, dx); dy = fma(c1, V.y, dy);
  dv[i] = make_double2(dx, dy);
  x[i] = make_double2(X.x + dx, X.y + dy);
}
__global__ void fill(long n, double* p, double v) { long i = (long)blockIdx.x * blockDim.x + threadIdx.x; if (i < n) p[i] = v * (1 + (i % 7)); }
int main() {
  const long n = 35588096;
  double* buf[5];
  for (int k = 0; k < 5; ++k) { CK(cudaMalloc(&buf[k], n * sizeof(double))); fill<<<(n+255)/256,256>>>(n, buf[k], 0.1 + k); }
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  auto timeit = [&](auto f, int reps) { f(); cudaEventRecord(a); for (int r = 0; r < reps; ++r) f(); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b); return ms / reps; };
  auto D2 = [&](int k) { return (double2*)buf[k]; };
  float t0 = timeit([&] { cheb_step<false><<<n / 512, 256>>>(D2(0), D2(1), D2(2), D2(3), D2(4), .5, .3); }, 30);
  float t1 = timeit([&] { cheb_step<true><<<n / 512, 256>>>(D2(0), D2(1), D2(2), D2(3), D2(4), .5, .3); }, 30);
  printf("hoisted zero store %.3f ms   data-dependent store %.3f ms\n", t0, t1);
  return 0;
}
