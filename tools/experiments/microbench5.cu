// load order / early-exit structure experiment (design experiment)
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
#define BODY \
  double2 d; d.x = fma(c1, V.x, c2 * D.x * (G.x - T.x)); d.y = fma(c1, V.y, c2 * D.y * (G.y - T.y)); \
  t[i] = make_double2(0, 0); dv[i] = d; x[i] = make_double2(X.x + d.x, X.y + d.y);
// A: early exit, t loaded first
__global__ void kA(long n2, const double2* __restrict__ g, const double2* __restrict__ Dinv, double2* __restrict__ t, double2* __restrict__ dv, double2* __restrict__ x, double c1, double c2) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x; if (i >= n2) return;
  double2 T = t[i]; double2 G = g[i]; double2 D = Dinv[i]; double2 V = dv[i]; double2 X = x[i]; BODY }
// B: predicated loads, g first
__global__ void kB(long n2, const double2* __restrict__ g, const double2* __restrict__ Dinv, double2* __restrict__ t, double2* __restrict__ dv, double2* __restrict__ x, double c1, double c2) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  double2 G, T, D, V, X;
  if (i < n2) { G = g[i]; D = Dinv[i]; T = t[i]; V = dv[i]; X = x[i]; }
  if (i >= n2) return; BODY }
// C: no const on g/Dinv (no .CONSTANT path)
__global__ void kC(long n2, double2* g, double2* Dinv, double2* t, double2* dv, double2* x, double c1, double c2) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x; if (i >= n2) return;
  double2 G = __ldcg(g + i), T = __ldcg(t + i), D = __ldcg(Dinv + i), V = __ldcg(dv + i), X = __ldcg(x + i); BODY }
// D: only non-constant loads through ld.global (no restrict)
__global__ void kD(long n2, const double2* g, const double2* Dinv, double2* t, double2* dv, double2* x, double c1, double c2) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x; if (i >= n2) return;
  double2 G = g[i]; double2 D = Dinv[i]; double2 T = t[i]; double2 V = dv[i]; double2 X = x[i]; BODY }
int main() {
  const long n = 35587930, n2 = n / 2;
  double* buf[5];
  for (int k = 0; k < 5; ++k) { CK(cudaMalloc(&buf[k], 2 * n * sizeof(double))); CK(cudaMemset(buf[k], 0, 2 * n * 8)); }
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  auto timeit = [&](auto f, int reps) { f(); cudaEventRecord(a); for (int r = 0; r < reps; ++r) f(); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b); return ms / reps; };
  auto D2 = [&](int k) { return (double2*)buf[k]; };
  int g = (n2 + 255) / 256;
  float tA = timeit([&] { kA<<<g, 256>>>(n2, D2(0), D2(1), D2(2), D2(3), D2(4), .5, .3); }, 50);
  float tB = timeit([&] { kB<<<g, 256>>>(n2, D2(0), D2(1), D2(2), D2(3), D2(4), .5, .3); }, 50);
  float tC = timeit([&] { kC<<<g, 256>>>(n2, D2(0), D2(1), D2(2), D2(3), D2(4), .5, .3); }, 50);
  float tD = timeit([&] { kD<<<g, 256>>>(n2, D2(0), D2(1), D2(2), D2(3), D2(4), .5, .3); }, 50);
  printf("A(t first) %.3f  B(pred, g first) %.3f  C(ldcg) %.3f  D(no restrict) %.3f ms\n", tA, tB, tC, tD);
  return 0;
}
