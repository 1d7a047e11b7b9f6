// sm_100a kernels of the local-smoothing GMG hot path (fp64, no tensor cores).
//
//  cell_apply      y += a_T h^(d-2) (sum_i (x)_j K|M) x_T   sum-factorised Q_k
//                  Laplace cell operator, thread per cell, register
//                  resident 1-D passes, gathers through the level DoF table,
//                  fp64 atomic scatter (RED.ADD.F64 at L2)
//  cell_diag       diagonal of the level operator
//  cell_load       b += f h^d (w (x) w (x) w) on leaf cells (f = const)
//  cheb_*          fused Chebyshev-Jacobi vector updates, reset of the
//                  apply accumulator
//  fam_restrict    d_{l-1} += P^T r, warp per refined parent (family of 2^d
//                  children), r = d - K x computed on the fly for the V-cycle
//                  residual (edge rows included); owned patch nodes
//                  only => exact P^T without weights
//  fam_prolongate  x_l += P x_{l-1} (owned fine nodes, exclusive writes) or
//                  x_l[E] = (P x_{l-1})[E] (hanging / edge values, leaf operator)
//  dot / axpy      CG vector kernels with deterministic two-stage reductions
#pragma once
#include <cstdint>

namespace gmg {
namespace dev {

// ------------------------------------------------------------- 1-D matrices
// Closed forms on the reference interval [0,1] with nodes {0, 1/k, .., 1}:
//   Q1: K = [[1,-1],[-1,1]],  M = [[1/3,1/6],[1/6,1/3]],  int phi = (1/2, 1/2)
//   Q2: K = 1/3 [[7,-8,1],[-8,16,-8],[1,-8,7]],  M = 1/30 [[4,2,-1],[2,16,2],[-1,2,4]],
//       int phi = (1/6, 2/3, 1/6)
template <int K> struct Q;
template <> struct Q<1> {
  static __device__ __forceinline__ double Km(int i, int j) { return i == j ? 1.0 : -1.0; }
  static __device__ __forceinline__ double Mm(int i, int j) { return i == j ? (1.0 / 3.0) : (1.0 / 6.0); }
  static __device__ __forceinline__ double w(int) { return 0.5; }
  // coarse basis j at fine patch coordinate a / 2 (a = 0..2)
  static __device__ __forceinline__ double P(int a, int j) {
    if (a == 1) return 0.5;
    return (a == 2 * j) ? 1.0 : 0.0;
  }
};
template <> struct Q<2> {
  static __device__ __forceinline__ double Km(int i, int j) {
    if (i == 1 && j == 1) return 16.0 / 3.0;
    if (i == 1 || j == 1) return -8.0 / 3.0;
    return i == j ? 7.0 / 3.0 : 1.0 / 3.0;
  }
  static __device__ __forceinline__ double Mm(int i, int j) {
    if (i == 1 && j == 1) return 16.0 / 30.0;
    if (i == 1 || j == 1) return 2.0 / 30.0;
    return i == j ? 4.0 / 30.0 : -1.0 / 30.0;
  }
  static __device__ __forceinline__ double w(int i) { return i == 1 ? (2.0 / 3.0) : (1.0 / 6.0); }
  // coarse basis phi_j at t = a/4: phi0 = 2t^2-3t+1, phi1 = 4t(1-t), phi2 = 2t^2-t
  static __device__ __forceinline__ double P(int a, int j) {
    switch (a) {
      case 0: return j == 0 ? 1.0 : 0.0;
      case 1: return j == 0 ? 0.375 : (j == 1 ? 0.75 : -0.125);
      case 2: return j == 1 ? 1.0 : 0.0;
      case 3: return j == 0 ? -0.125 : (j == 1 ? 0.75 : 0.375);
      default: return j == 2 ? 1.0 : 0.0;
    }
  }
};

template <int D, int K> struct Shape {
  static constexpr int N1 = K + 1;
  static constexpr int NN = D == 2 ? N1 * N1 : N1 * N1 * N1;
  static constexpr int NP1 = 2 * K + 1;
  static constexpr int NP = D == 2 ? NP1 * NP1 : NP1 * NP1 * NP1;
  static constexpr int NCH = 1 << D;
};

// out = A_ref u on one cell (x fastest local numbering)
template <int D, int K>
__device__ __forceinline__ void elem_apply(const double (&u)[Shape<D, K>::NN], double (&out)[Shape<D, K>::NN]) {
  constexpr int N = K + 1;
  if constexpr (D == 2) {
    double a[N * N], b[N * N];
#pragma unroll
    for (int y = 0; y < N; ++y)
#pragma unroll
      for (int x = 0; x < N; ++x) {
        double sa = 0, sb = 0;
#pragma unroll
        for (int q = 0; q < N; ++q) {
          sa = fma(Q<K>::Km(x, q), u[y * N + q], sa);
          sb = fma(Q<K>::Mm(x, q), u[y * N + q], sb);
        }
        a[y * N + x] = sa;
        b[y * N + x] = sb;
      }
#pragma unroll
    for (int y = 0; y < N; ++y)
#pragma unroll
      for (int x = 0; x < N; ++x) {
        double s = 0;
#pragma unroll
        for (int q = 0; q < N; ++q) {
          s = fma(Q<K>::Mm(y, q), a[q * N + x], s);
          s = fma(Q<K>::Km(y, q), b[q * N + x], s);
        }
        out[y * N + x] = s;
      }
  } else {
    constexpr int NN = N * N * N;
    double t1[NN], t2[NN];
    // z direction: t1 = M_z u, t2 = K_z u
#pragma unroll
    for (int z = 0; z < N; ++z)
#pragma unroll
      for (int yx = 0; yx < N * N; ++yx) {
        double s1 = 0, s2 = 0;
#pragma unroll
        for (int q = 0; q < N; ++q) {
          s1 = fma(Q<K>::Mm(z, q), u[q * N * N + yx], s1);
          s2 = fma(Q<K>::Km(z, q), u[q * N * N + yx], s2);
        }
        t1[z * N * N + yx] = s1;
        t2[z * N * N + yx] = s2;
      }
    // y direction: a = M_y t1, b = K_y t1 + M_y t2
    double a[NN], b[NN];
#pragma unroll
    for (int z = 0; z < N; ++z)
#pragma unroll
      for (int y = 0; y < N; ++y)
#pragma unroll
        for (int x = 0; x < N; ++x) {
          double sa = 0, sb = 0;
#pragma unroll
          for (int q = 0; q < N; ++q) {
            const int iq = z * N * N + q * N + x;
            sa = fma(Q<K>::Mm(y, q), t1[iq], sa);
            sb = fma(Q<K>::Km(y, q), t1[iq], sb);
            sb = fma(Q<K>::Mm(y, q), t2[iq], sb);
          }
          a[z * N * N + y * N + x] = sa;
          b[z * N * N + y * N + x] = sb;
        }
    // x direction: out = K_x a + M_x b
#pragma unroll
    for (int zy = 0; zy < N * N; ++zy)
#pragma unroll
      for (int x = 0; x < N; ++x) {
        double s = 0;
#pragma unroll
        for (int q = 0; q < N; ++q) {
          s = fma(Q<K>::Km(x, q), a[zy * N + q], s);
          s = fma(Q<K>::Mm(x, q), b[zy * N + q], s);
        }
        out[zy * N + x] = s;
      }
  }
}

template <int D, int K>
__device__ __forceinline__ double elem_diag(int i) {
  constexpr int N = K + 1;
  int ix = i % N, iy = (i / N) % N, iz = i / (N * N);
  if constexpr (D == 2) return Q<K>::Km(ix, ix) * Q<K>::Mm(iy, iy) + Q<K>::Mm(ix, ix) * Q<K>::Km(iy, iy);
  return Q<K>::Km(ix, ix) * Q<K>::Mm(iy, iy) * Q<K>::Mm(iz, iz) +
         Q<K>::Mm(ix, ix) * Q<K>::Km(iy, iy) * Q<K>::Mm(iz, iz) +
         Q<K>::Mm(ix, ix) * Q<K>::Mm(iy, iy) * Q<K>::Km(iz, iz);
}

// ------------------------------------------------------------- cell kernels
// cell_dofs is SoA: dof of local node b of cell c at cell_dofs[b * ldc + c]
template <int D, int K>
__global__ void __launch_bounds__(128) cell_apply(int n, const int* __restrict__ list,
                                                  const int* __restrict__ cell_dofs, long ldc,
                                                  const double* __restrict__ coef, double scale,
                                                  const double* __restrict__ x, double* __restrict__ y) {
  constexpr int NN = Shape<D, K>::NN;
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int c = list ? list[t] : t;
  int idx[NN];
  double u[NN], v[NN];
#pragma unroll
  for (int b = 0; b < NN; ++b) idx[b] = __ldg(cell_dofs + (long)b * ldc + c);
#pragma unroll
  for (int b = 0; b < NN; ++b) u[b] = idx[b] >= 0 ? __ldg(x + idx[b]) : 0.0;
  elem_apply<D, K>(u, v);
  const double s = coef ? scale * __ldg(coef + c) : scale;
#pragma unroll
  for (int b = 0; b < NN; ++b)
    if (idx[b] >= 0) atomicAdd(y + idx[b], s * v[b]);
}

template <int D, int K>
__global__ void cell_diag(int n, const int* __restrict__ cell_dofs, long ldc, const double* __restrict__ coef,
                          double scale, double* __restrict__ diag) {
  constexpr int NN = Shape<D, K>::NN;
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  const double s = coef ? scale * coef[c] : scale;
#pragma unroll
  for (int b = 0; b < NN; ++b) {
    int i = cell_dofs[(long)b * ldc + c];
    if (i >= 0) atomicAdd(diag + i, s * elem_diag<D, K>(b));
  }
}

template <int D, int K>
__global__ void cell_load(int n, const int* __restrict__ list, const int* __restrict__ cell_dofs, long ldc,
                          double fh, double* __restrict__ y) {
  constexpr int NN = Shape<D, K>::NN;
  constexpr int N = K + 1;
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int c = list[t];
#pragma unroll
  for (int b = 0; b < NN; ++b) {
    int i = cell_dofs[(long)b * ldc + c];
    double w = Q<K>::w(b % N) * Q<K>::w((b / N) % N);
    if (D == 3) w *= Q<K>::w(b / (N * N));
    if (i >= 0) atomicAdd(y + i, fh * w);
  }
}

// ------------------------------------------------------------- Chebyshev
// dv = c1 dv + c2 Dinv (g - t);  x += dv (x = dv if X_ZERO);  t = 0
template <bool READ_T, bool READ_DV, bool WRITE_DV, bool X_ZERO>
__global__ void cheb_step(long n, const double* __restrict__ g, const double* __restrict__ Dinv,
                          double* __restrict__ t, double* __restrict__ dv, double* __restrict__ x,
                          double c1, double c2) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const long stride = (long)gridDim.x * blockDim.x;
  for (; i < n; i += stride) {
    double r = g[i];
    if (READ_T) {
      r -= t[i];
      t[i] = 0.0;
    }
    double d = c2 * Dinv[i] * r;
    if (READ_DV) d = fma(c1, dv[i], d);
    if (WRITE_DV) dv[i] = d;
    x[i] = X_ZERO ? d : x[i] + d;
  }
}

// ------------------------------------------------------------- transfers
// Family f: parent fam_parent[f] in level l-1, children 2^d f .. 2^d f + 2^d - 1 in
// level l.  Patch node a (coordinates in [0,2k]^d) of child c = (a_j > k), local
// node b_j = a_j - k c_j.  own_mask: bit a set iff this family owns the fine node.
template <int D, int K>
__device__ __forceinline__ int patch_dof(int f, int a, const int* __restrict__ cell_dofs_f, long ldc) {
  constexpr int NP1 = 2 * K + 1, N = K + 1;
  int c = 0, b = 0, mul = 1;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    int aj = a % NP1;
    a /= NP1;
    int cj = aj > K ? 1 : 0;
    c |= cj << j;
    b += (aj - K * cj) * mul;
    mul *= N;
  }
  return cell_dofs_f[(long)b * ldc + (long)f * (1 << D) + c];
}

// tensor weight P(a, j) of fine patch node a and coarse local node j
template <int D, int K>
__device__ __forceinline__ double patch_weight(int a, int j) {
  constexpr int NP1 = 2 * K + 1, N = K + 1;
  double w = 1.0;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    w *= Q<K>::P(a % NP1, j % N);
    a /= NP1;
    j /= N;
  }
  return w;
}

enum : int { XFER_ADD = 0, XFER_SET_E = 1 };
enum : int { RES_PLAIN = 0, RES_VCYCLE = 1, RES_EONLY = 2 };

constexpr int XFER_WARPS = 4;

template <int D, int K, int MODE>
__global__ void __launch_bounds__(32 * XFER_WARPS)
fam_prolongate(int nfam, const int* __restrict__ fam_list, const int* __restrict__ fam_parent,
               const unsigned long long* __restrict__ own_mask, int mask_words,
               const int* __restrict__ cdofs_coarse, long ldc_coarse,
               const int* __restrict__ cdofs_fine, long ldc_fine, const unsigned char* __restrict__ cls_fine,
               const double* __restrict__ xc, double* __restrict__ xf) {
  constexpr int NC = Shape<D, K>::NN, NP = Shape<D, K>::NP;
  __shared__ double sc[XFER_WARPS][NC];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int t = blockIdx.x * XFER_WARPS + w;
  if (t >= nfam) return;
  const int f = fam_list ? fam_list[t] : t;
  const int p = fam_parent[f];
  for (int j = lane; j < NC; j += 32) {
    int i = cdofs_coarse[(long)j * ldc_coarse + p];
    sc[w][j] = i >= 0 ? xc[i] : 0.0;
  }
  __syncwarp();
  for (int a = lane; a < NP; a += 32) {
    if (!((own_mask[(long)f * mask_words + (a >> 6)] >> (a & 63)) & 1ull)) continue;
    int i = patch_dof<D, K>(f, a, cdofs_fine, ldc_fine);
    if (i < 0) continue;
    if (MODE == XFER_SET_E && !(cls_fine[i] & 1)) continue;
    double v = 0.0;
#pragma unroll
    for (int j = 0; j < NC; ++j) v = fma(patch_weight<D, K>(a, j), sc[w][j], v);
    if (MODE == XFER_SET_E) xf[i] = v;
    else xf[i] += v;
  }
}

// d_c += P^T r with r = (MODE == RES_VCYCLE ? d - t (and t := 0) : v) on owned fine nodes
template <int D, int K, int MODE>
__global__ void __launch_bounds__(32 * XFER_WARPS)
fam_restrict(int nfam, const int* __restrict__ fam_list, const int* __restrict__ fam_parent,
             const unsigned long long* __restrict__ own_mask, int mask_words,
             const int* __restrict__ cdofs_coarse, long ldc_coarse,
             const int* __restrict__ cdofs_fine, long ldc_fine, const unsigned char* __restrict__ cls_fine,
             const double* __restrict__ v, double* __restrict__ t, double* __restrict__ dc) {
  constexpr int NC = Shape<D, K>::NN, NP = Shape<D, K>::NP;
  constexpr int NP1 = 2 * K + 1, N = K + 1;
  __shared__ double sr[XFER_WARPS][NP];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int tt = blockIdx.x * XFER_WARPS + w;
  if (tt >= nfam) return;
  const int f = fam_list ? fam_list[tt] : tt;
  for (int a = lane; a < NP; a += 32) {
    double r = 0.0;
    if ((own_mask[(long)f * mask_words + (a >> 6)] >> (a & 63)) & 1ull) {
      int i = patch_dof<D, K>(f, a, cdofs_fine, ldc_fine);
      if (i >= 0) {
        if (MODE == RES_VCYCLE) {
          r = v[i] - t[i];
          t[i] = 0.0;
        } else if (MODE == RES_EONLY) {
          r = (cls_fine[i] & 1) ? v[i] : 0.0;
        } else {
          r = v[i];
        }
      }
    }
    sr[w][a] = r;
  }
  __syncwarp();
  const int p = fam_parent[f];
  for (int j = lane; j < NC; j += 32) {
    int ci = cdofs_coarse[(long)j * ldc_coarse + p];
    if (ci < 0) continue;
    // fine patch coordinates with a nonzero weight for coarse node j_d: the
    // coincident node 2 j_d and the odd (mid-edge) nodes 1 (and 3 for K = 2)
    constexpr int NA = K + 1;
    int jj[3] = {j % N, (j / N) % N, D == 3 ? j / (N * N) : 0};
    double s = 0.0;
#pragma unroll
    for (int qz = 0; qz < (D == 3 ? NA : 1); ++qz) {
      const int az = D == 3 ? (qz == 0 ? 2 * jj[2] : 2 * qz - 1) : 0;
#pragma unroll
      for (int qy = 0; qy < NA; ++qy) {
        const int ay = qy == 0 ? 2 * jj[1] : 2 * qy - 1;
#pragma unroll
        for (int qx = 0; qx < NA; ++qx) {
          const int ax = qx == 0 ? 2 * jj[0] : 2 * qx - 1;
          double wgt = Q<K>::P(ax, jj[0]) * Q<K>::P(ay, jj[1]);
          if (D == 3) wgt *= Q<K>::P(az, jj[2]);
          const int a = ax + NP1 * ay + (D == 3 ? NP1 * NP1 * az : 0);
          s = fma(wgt, sr[w][a], s);
        }
      }
    }
    atomicAdd(dc + ci, s);
  }
}

// ------------------------------------------------------------- misc vector kernels
__global__ void coarse_solve(int n, const int* __restrict__ sidx, const double* __restrict__ Ainv,
                             const double* __restrict__ d, double* __restrict__ x) {
  int i = threadIdx.x;
  for (; i < n; i += blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < n; ++j) s = fma(Ainv[(long)i * n + j], d[sidx[j]], s);
    x[sidx[i]] = s;
  }
}

// MG layout <- leaf order: out[m] = (inv[m] >= 0 ? in[inv[m]] : 0)
__global__ void gather_to_mg(long n, const long long* __restrict__ inv, const double* __restrict__ in,
                             double* __restrict__ out) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const long stride = (long)gridDim.x * blockDim.x;
  for (; i < n; i += stride) {
    long long s = inv[i];
    out[i] = s >= 0 ? in[s] : 0.0;
  }
}
// leaf order <- MG layout
__global__ void gather_from_mg(long n, const long long* __restrict__ perm, const double* __restrict__ in,
                               double* __restrict__ out) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const long stride = (long)gridDim.x * blockDim.x;
  for (; i < n; i += stride) out[i] = in[perm[i]];
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// block partial of sum_i a_i b_i (mask: lambda slots only when lam != null)
template <int NT>
__device__ __forceinline__ void block_store_partial(double s, double* partial) {
  __shared__ double sh[NT / 32];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < NT / 32 ? sh[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) partial[blockIdx.x] = v;
  }
}

constexpr int RED_NT = 256;

__global__ void __launch_bounds__(RED_NT) dot_partial(long n, const double* __restrict__ a,
                                                      const double* __restrict__ b, double* __restrict__ partial) {
  double s = 0.0;
  for (long i = (long)blockIdx.x * RED_NT + threadIdx.x; i < n; i += (long)gridDim.x * RED_NT) s = fma(a[i], b[i], s);
  block_store_partial<RED_NT>(s, partial);
}

// deterministic final sum of nb partials into out[slot]
__global__ void __launch_bounds__(RED_NT) reduce_final(int nb, const double* __restrict__ partial,
                                                       double* __restrict__ out) {
  double s = 0.0;
  for (int i = threadIdx.x; i < nb; i += RED_NT) s += partial[i];
  __shared__ double sh[RED_NT / 32];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < RED_NT / 32 ? sh[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) *out = v;
  }
}

// q = mask * y ; partial (p, q)
__global__ void __launch_bounds__(RED_NT) mask_dot(long n, const unsigned char* __restrict__ lam,
                                                   const double* __restrict__ y, const double* __restrict__ p,
                                                   double* __restrict__ q, double* __restrict__ partial) {
  double s = 0.0;
  for (long i = (long)blockIdx.x * RED_NT + threadIdx.x; i < n; i += (long)gridDim.x * RED_NT) {
    double v = lam[i] ? y[i] : 0.0;
    q[i] = v;
    s = fma(p[i], v, s);
  }
  block_store_partial<RED_NT>(s, partial);
}

// CG: alpha = sc[0]/sc[1];  x += alpha p;  r -= alpha q;  partial (r, r)
__global__ void __launch_bounds__(RED_NT) cg_update_xr(long n, const double* __restrict__ sc,
                                                       const double* __restrict__ p, const double* __restrict__ q,
                                                       double* __restrict__ x, double* __restrict__ r,
                                                       double* __restrict__ partial) {
  const double alpha = sc[0] / sc[1];
  double s = 0.0;
  for (long i = (long)blockIdx.x * RED_NT + threadIdx.x; i < n; i += (long)gridDim.x * RED_NT) {
    x[i] = fma(alpha, p[i], x[i]);
    double ri = fma(-alpha, q[i], r[i]);
    r[i] = ri;
    s = fma(ri, ri, s);
  }
  block_store_partial<RED_NT>(s, partial);
}

// z = lam * X ; partial (r, z)
__global__ void __launch_bounds__(RED_NT) mask_copy_dot(long n, const unsigned char* __restrict__ lam,
                                                        const double* __restrict__ X, const double* __restrict__ r,
                                                        double* __restrict__ z, double* __restrict__ partial) {
  double s = 0.0;
  for (long i = (long)blockIdx.x * RED_NT + threadIdx.x; i < n; i += (long)gridDim.x * RED_NT) {
    double v = lam[i] ? X[i] : 0.0;
    z[i] = v;
    s = fma(r[i], v, s);
  }
  block_store_partial<RED_NT>(s, partial);
}

// beta = sc[2]/sc[0]; p = z + beta p; then sc[0] = sc[2]
__global__ void cg_update_p(long n, const double* __restrict__ sc, const double* __restrict__ z,
                            double* __restrict__ p) {
  const double beta = sc[2] / sc[0];
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const long stride = (long)gridDim.x * blockDim.x;
  for (; i < n; i += stride) p[i] = fma(beta, p[i], z[i]);
}
__global__ void copy_scalar(const double* __restrict__ src, double* __restrict__ dst) { *dst = *src; }

// eigen CG: r -= alpha q on S rows, 0 on E rows (cls bit0 = E)
__global__ void eig_update_r(long n, double alpha, const unsigned char* __restrict__ cls,
                             const double* __restrict__ q, double* __restrict__ r) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) r[i] = (cls[i] & 1) ? 0.0 : fma(-alpha, q[i], r[i]);
}
__global__ void eig_z(long n, const double* __restrict__ Dinv, const double* __restrict__ r, double* __restrict__ z) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) z[i] = Dinv[i] * r[i];
}
__global__ void axpby(long n, double a, const double* __restrict__ x, double b, double* __restrict__ y) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = fma(a, x[i], b * y[i]);
}
__global__ void invert_diag(long n, const unsigned char* __restrict__ cls, double* __restrict__ d, int* bad) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (cls[i] & 1) {
    d[i] = 0.0;
  } else {
    double v = d[i];
    if (!(v > 0.0)) atomicAdd(bad, 1);
    d[i] = v > 0.0 ? 1.0 / v : 0.0;
  }
}
__global__ void recip_s(long n, const unsigned char* __restrict__ cls, const double* __restrict__ Dinv,
                        double* __restrict__ diag) {
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) diag[i] = (cls[i] & 1) ? 0.0 : 1.0 / Dinv[i];
}

}  // namespace dev
}  // namespace gmg
