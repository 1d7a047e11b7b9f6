// Microbenchmarks for the design of the level kernels on B200 (not part of
// the library): streaming vector updates with several arrays, and fp64
// atomic scatter throughput.   nvcc -O3 -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void copyk(long n, const double* __restrict__ a, double* __restrict__ b) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) b[i] = a[i];
}

template <bool GS>
__global__ void cheb(long n, const double* __restrict__ g, const double* __restrict__ Dinv, double* __restrict__ t,
                     double* __restrict__ dv, double* __restrict__ x, double c1, double c2) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const long stride = GS ? (long)gridDim.x * blockDim.x : n;
  for (; i < n; i += stride) {
    double r = g[i] - t[i];
    t[i] = 0.0;
    double d = fma(c1, dv[i], c2 * Dinv[i] * r);
    dv[i] = d;
    x[i] = x[i] + d;
  }
}

__global__ void cheb2(long n2, const double2* __restrict__ g, const double2* __restrict__ Dinv, double2* __restrict__ t,
                      double2* __restrict__ dv, double2* __restrict__ x, double c1, double c2) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n2) return;
  double2 G = g[i], T = t[i], D = Dinv[i], V = dv[i], X = x[i];
  t[i] = make_double2(0, 0);
  double2 d;
  d.x = fma(c1, V.x, c2 * D.x * (G.x - T.x));
  d.y = fma(c1, V.y, c2 * D.y * (G.y - T.y));
  dv[i] = d;
  x[i] = make_double2(X.x + d.x, X.y + d.y);
}

__global__ void scatter_atomic(long n, const int* __restrict__ idx, double* __restrict__ y) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) atomicAdd(y + idx[i], 1.0);
}
__global__ void scatter_store(long n, const int* __restrict__ idx, double* __restrict__ y) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[idx[i]] = 1.0;
}

int main() {
  const long n = 35587930;
  const long nbig = 58297952;
  double *buf[8];
  for (int k = 0; k < 8; ++k) { CK(cudaMalloc(&buf[k], nbig * sizeof(double))); CK(cudaMemset(buf[k], 0, nbig * 8)); }
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  float ms;
  auto timeit = [&](auto f, int reps) { f(); cudaEventRecord(a); for (int r = 0; r < reps; ++r) f(); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b); return ms / reps; };
  double off = 22709000;  // finest level offset in MG layout
  long o = (long)off / 32 * 32;
  float t;
  t = timeit([&] { copyk<<<(n + 255) / 256, 256>>>(n, buf[0] + o, buf[1] + o); }, 20);
  printf("copy         %.3f ms  %.0f GB/s\n", t, 16.0 * n / t / 1e6);
  t = timeit([&] { cheb<true><<<148 * 16, 256>>>(n, buf[0] + o, buf[1] + o, buf[2] + o, buf[3] + o, buf[4] + o, 0.5, 0.3); }, 20);
  printf("cheb gs2368  %.3f ms  %.0f GB/s\n", t, 64.0 * n / t / 1e6);
  t = timeit([&] { cheb<false><<<(n + 255) / 256, 256>>>(n, buf[0] + o, buf[1] + o, buf[2] + o, buf[3] + o, buf[4] + o, 0.5, 0.3); }, 20);
  printf("cheb full    %.3f ms  %.0f GB/s\n", t, 64.0 * n / t / 1e6);
  t = timeit([&] { cheb<true><<<148 * 64, 256>>>(n, buf[0] + o, buf[1] + o, buf[2] + o, buf[3] + o, buf[4] + o, 0.5, 0.3); }, 20);
  printf("cheb gs9472  %.3f ms  %.0f GB/s\n", t, 64.0 * n / t / 1e6);
  t = timeit([&] { cheb2<<<(n / 2 + 255) / 256, 256>>>(n / 2, (double2*)(buf[0] + o), (double2*)(buf[1] + o), (double2*)(buf[2] + o), (double2*)(buf[3] + o), (double2*)(buf[4] + o), 0.5, 0.3); }, 20);
  printf("cheb v2      %.3f ms  %.0f GB/s\n", t, 64.0 * n / t / 1e6);
  // offsets staggered
  t = timeit([&] { cheb<false><<<(n + 255) / 256, 256>>>(n, buf[0], buf[1] + 1024, buf[2] + 4096, buf[3] + 77777 * 4, buf[4] + 333 * 32, 0.5, 0.3); }, 20);
  printf("cheb stagger %.3f ms  %.0f GB/s\n", t, 64.0 * n / t / 1e6);
  // atomics: random-ish (cell-like) vs sequential
  std::vector<int> hidx(27 * (n / 8));
  long m = hidx.size();
  unsigned s = 1;
  for (long i = 0; i < m; ++i) { s = s * 1664525u + 1013904223u; hidx[i] = (int)((i / 27) * 8 + (s >> 8) % 27) % n; }
  int* didx;
  CK(cudaMalloc(&didx, m * 4));
  CK(cudaMemcpy(didx, hidx.data(), m * 4, cudaMemcpyHostToDevice));
  t = timeit([&] { scatter_atomic<<<(m + 255) / 256, 256>>>(m, didx, buf[5]); }, 10);
  printf("atomic scatter (27 per cell, local) %.3f ms  %.2f G atomics/s\n", t, m / t / 1e6);
  t = timeit([&] { scatter_store<<<(m + 255) / 256, 256>>>(m, didx, buf[5]); }, 10);
  printf("store scatter                        %.3f ms  %.2f G stores/s\n", t, m / t / 1e6);
  for (long i = 0; i < m; ++i) hidx[i] = (int)(i % n);
  CK(cudaMemcpy(didx, hidx.data(), m * 4, cudaMemcpyHostToDevice));
  t = timeit([&] { scatter_atomic<<<(m + 255) / 256, 256>>>(m, didx, buf[5]); }, 10);
  printf("atomic sequential                    %.3f ms  %.2f G atomics/s\n", t, m / t / 1e6);
  CK(cudaDeviceSynchronize());
  return 0;
}
